"""Per-phase totals of k_filter from a source CSV (ncu --page source --csv
--print-source cuda,sass, optionally gzipped): stall samples and warp
instructions by phase.  python tools/ncu_phases.py source.csv[.gz]"""
import csv, gzip, io, sys, collections
p = sys.argv[1]
txt = (gzip.open(p, "rt") if p.endswith(".gz") else open(p)).read()
# phase ranges by file and line, found from the phase-marker comments of
# k_filter in the CURRENT sources (capture and sources must match) and the
# helper functions of fabf_device.cuh
import os, re
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cu = open(os.path.join(ROOT, "paper_1811_02308_b200", "csrc", "fabf.cu")).read().splitlines()
dv = open(os.path.join(ROOT, "paper_1811_02308_b200", "csrc", "fabf_device.cuh")).read().splitlines()
def find(lines, pat, start=0):
    for i in range(start, len(lines)):
        if re.search(pat, lines[i]):
            return i + 1
    raise SystemExit("marker not found: " + pat)
k0 = find(cu, r"k_filter\(FilterArgs a\) \{")
la = find(cu, r"---- phase A", k0); lb = find(cu, r"---- phase B", la)
lc1 = find(cu, r"---- phase C1", lb); lc2 = find(cu, r"---- phase C2", lc1)
lp = find(cu, r"const int qb = step & 1;", k0)
kend = find(cu, r"^}", lc2)
ds = find(dv, r"bool stretch_flagged"); dr = find(dv, r"int reflect_hi")
PH = [("fabf.cu", k0, lp - 1, "setup+prologue"), ("fabf.cu", lp, la - 1, "pixel params"),
      ("fabf.cu", la, lb - 1, "A"), ("fabf.cu", lb, lc1 - 1, "B"), ("fabf.cu", lc1, lc2 - 1, "C1"),
      ("fabf.cu", lc2, kend, "C2"), ("fabf_device.cuh", ds, dr - 1, "C1"),
      ("fabf_device.cuh", dr, dr + 8, "A"), ("fabf_device.cuh", 1, ds - 1, "C2"),
      ("fabf_erfcx.cuh", 1, 99, "C2")]
fname, hdr = "?", None
acc = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        ins = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    ln = int(r[0])
    g = "other:" + fname
    for f, lo, hi, name in PH:
        if f == fname and lo <= ln <= hi:
            g = name
            break
    a = acc[g]
    a[0] += s
    a[1] += ins
    for k, v in d.items():
        if k.startswith("stall_") and v not in ("", "0"):
            try:
                a[2][k[6:]] += int(v)
            except ValueError:
                pass
ts = sum(a[0] for a in acc.values()); ti = sum(a[1] for a in acc.values())
for g, (s, ins, st) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    top = ", ".join(f"{k}:{100*v/max(1,s):.0f}%" for k, v in st.most_common(4))
    print(f"{g:16s} samples {100*s/ts:5.1f}%  instr {100*ins/ti:5.1f}%  {top}")
