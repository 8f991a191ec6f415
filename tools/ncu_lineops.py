"""Per-CUDA-line dynamic SASS counts (thread-instr per pixel) and opcode mix:
python tools/ncu_lineops.py rep [top] [pixels]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
px = float(sys.argv[3]) if len(sys.argv) > 3 else 8294400
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, src = "?", "?", ""
lines = collections.defaultdict(collections.Counter)
srcs = {}
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = ["Line No", "Source", "Address", "Sass"] + r[4:]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0] != "":
        line = r[0]
        srcs[(fname, line)] = r[1].strip()[:60]
        continue
    d = dict(zip(hdr, r))
    try:
        n = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    op = d["Sass"].strip().split()
    if not op or n == 0:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = "IMAD.MOV" if o.startswith("IMAD.MOV") else o.split(".")[0]
    lines[(fname, line)][o] += n
tot = sum(sum(c.values()) for c in lines.values())
rows = sorted(lines.items(), key=lambda kv: -sum(kv[1].values()))
print(f"total {tot * 32 / px:.0f} thread-instr/px")
for (f, ln), c in rows[:top]:
    n = sum(c.values())
    mix = " ".join(f"{o}:{v * 32 / px:.0f}" for o, v in c.most_common(5))
    print(f"{n * 32 / px:6.1f} {f}:{ln:>4} {srcs.get((f, ln), '')[:58]:58s} {mix}")
