"""Per-launch DRAM traffic and headline metrics of ncu --set full captures ->
profiles/traffic.json (read by bench.py for roofline.traffic).
  python tools/ncu_traffic.py kernel=report.ncu-rep [kernel=report ...]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__time_duration.sum": "duration",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
}
out_path = os.path.join(ROOT, "profiles", "traffic.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
for arg in sys.argv[1:]:
    kern, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, v = rows[0], rows[1], rows[2]
    d = {"report": os.path.basename(rep)}
    for name, unit, val in zip(h, units, v):
        if name in KEYS:
            x = float(val.replace(",", ""))
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
                     "nsecond": 1e-3}.get(unit, 1.0)
            d[KEYS[name]] = x * scale
            if unit in ("usecond", "msecond", "nsecond"):
                d["duration_unit"] = "us"
    d["dram_bytes"] = d.get("dram_read_bytes", 0.0) + d.get("dram_write_bytes", 0.0)
    res[kern] = d
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
