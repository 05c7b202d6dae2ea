"""DRAM traffic per launch of the roofline kernel from an ncu --set full
capture of one step's schur_trailing_kernel launches (tools/ncu_round2.sh):
writes profiles/trailing_traffic_<tag>.json, which bench.py reports as
roofline.traffic (bytes per launch, averaged over the mode-0 trailing
updates: the subdomain elimination's K = 128 launches and the dual-block
LU's K = 64 launches).

    python tools/traffic.py gpurun_out/full_trailing_r01c.ncu-rep r01c
"""
import csv
import io
import json
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "launch__grid_size"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(head)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "": 1}
def val(r, name):
    v = r[col[name]].replace(",", "")
    return float(v) * scale.get(units[col[name]], 1)
launches = []
for r in data:
    launches.append(dict(grid=int(val(r, "launch__grid_size")),
                         ms=val(r, "gpu__time_duration.sum") * 1e3,
                         dram_bytes=val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")))
# elimination order: [strip, big] x 3 (128-wide panels), then the dual LU's 64-wide panels
mode0 = [l for i, l in enumerate(launches) if (i >= 6 or i % 2 == 1)]
res = {
    "kernel": "schur_trailing_kernel",
    "capture": rep.split("/")[-1],
    "how": "ncu --set full --clock-control none -k regex:schur_trailing_kernel -c 16 "
           "python tools/profile_step.py --steps 1 (cfg5)",
    "launches": launches,
    "mode0_launches": len(mode0),
    "traffic_bytes_per_launch": sum(l["dram_bytes"] for l in mode0) / max(len(mode0), 1),
}
json.dump(res, open(f"profiles/trailing_traffic_{tag}.json", "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}))
