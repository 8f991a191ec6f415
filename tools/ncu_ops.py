"""Dynamic SASS opcode mix of an ncu report: python tools/ncu_ops.py rep [pixels]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
px = float(sys.argv[2]) if len(sys.argv) > 2 else 8294400
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
cnt = collections.Counter()
tot = 0
for row in csv.reader(io.StringIO(txt)):
    if row and row[0] == "Address":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    try:
        n = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    op = d["Source"].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    cnt[o] += n
    tot += n
print(f"total {tot} warp instr = {tot * 32 / px:.0f} thread-instr/px")
for o, n in cnt.most_common(32):
    print(f"{o:10s} {n:12d} {100 * n / tot:5.1f}%  {n * 32 / px:7.1f}/px")
