#!/usr/bin/env python3
"""Per-launch DRAM traffic of each kernel in an .ncu-rep -> JSON (bench.py
reads the decode entry as roofline.traffic).

  python tools/ncu_traffic.py full.ncu-rep > profiles/ncu_traffic.json
"""
import csv
import json
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    short = name.split("::")[-1].split("(")[0]
    rd = float(r[h.index("dram__bytes_read.sum")])
    wr = float(r[h.index("dram__bytes_write.sum")])
    res.setdefault(short, {"dram_read_bytes": rd, "dram_write_bytes": wr,
                           "traffic_bytes": rd + wr,
                           "duration_us": float(r[h.index("gpu__time_duration.sum")]) / 1e3})
dec = [v for k, v in res.items() if k.startswith("decode_kernel<float")]
if dec:
    res["c3_g1_decode_bytes"] = dec[0]["traffic_bytes"]
res["note"] = ("ncu --set full --clock-control none, bench.py --steps 3 (C3: ring M=8, D=25.6M, "
               "1 GPU), one launch per kernel after warm-up; per-launch DRAM traffic")
print(json.dumps(res, indent=1))
