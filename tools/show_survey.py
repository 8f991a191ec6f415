import json, sys
for ln in open(sys.argv[1]):
    try:
        d = json.loads(ln)
    except Exception:
        print(ln.rstrip()[:200]); continue
    if "case" in d:
        w = d["worst"][0]
        print(f"  {d['case'][:36]:36s} max {d['max']:.2e} p999 {d['p999']:.1e} >.01 {d['gt01']:3d} bad {d['bad']} fb {d['fallback']:6d} | k {w['kappa']:.0f} lam {w['lam']:.1f} t0 {w['t0']:.2f} c {w['code']}")
    else:
        print("  time", d["cfg"], [round(x * 1e3, 1) for x in d["stage_ms"]], round(d["mpix_s"]))
