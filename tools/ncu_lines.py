"""Per-source-line summary of an ncu report (stall samples, instructions, top
stall reasons):  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
tot_s = tot_i = 0
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = ["Line No", "Source", "Address", "Sass"] + r[4:]
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        ins = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    if s == 0 and ins == 0:
        continue
    stalls = {k[6:]: int(v or 0) for k, v in d.items()
              if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0")}
    st = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    rows.append((s, ins, fname, d["Line No"], d["Source"].strip()[:70], st))
    tot_s += s
    tot_i += ins
import os
rows.sort(key=lambda x: -x[1] if os.environ.get("SORT") == "instr" else -x[0])
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, ins, f, ln, src, st in rows[:top]:
    sts = " ".join(f"{k}:{100*v/max(s,1):.0f}%" for k, v in st)
    print(f"{100*s/tot_s:5.1f}% {100*ins/tot_i:5.1f}%i {f}:{ln:>4} {src:70s} {sts}")

# phase groups (fabf.cu line ranges of k_filter, device helpers by function)
if len(sys.argv) > 3:
    import json
    groups = json.loads(sys.argv[3])  # {"name": [file, lo, hi], ...}
    acc = {}
    for s, ins, f, ln, src, st in rows:
        g = "other"
        for name, (gf, lo, hi) in groups.items():
            if f == gf and lo <= int(ln) <= hi:
                g = name
                break
        a = acc.setdefault(g, [0, 0])
        a[0] += s
        a[1] += ins
    for g, (s, ins) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{g:12s} samples {100*s/tot_s:5.1f}%  instr {100*ins/tot_i:5.1f}%")
