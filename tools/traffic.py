"""DRAM traffic per launch of the roofline kernel from an ncu --set full
capture of one step's schur_trailing_kernel launches (tools/ncu_round2.sh):
writes profiles/trailing_traffic_<tag>.json, which bench.py reports as
roofline.traffic (bytes per launch, averaged over the mode-0 trailing
updates: the subdomain elimination's K = 128 launches and the dual-block
LU's K = 64 launches).

    python tools/traffic.py gpurun_out/full_trailing_r01d.ncu-rep r01d [nI_max nB_max]

The launch order of one step is rebuilt from the 128-wide panel sequence of the
two eliminations (strip launch when a panel has a second 64-wide sub-panel,
then the mode-0 trailing update): cfg5 has nI_max = 343, nB_max = 386.
"""
import csv
import io
import json
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
nI_max = int(sys.argv[3]) if len(sys.argv) > 3 else 343
nB_max = int(sys.argv[4]) if len(sys.argv) > 4 else 386
seq = []
for npiv in (nI_max, nB_max):
    for k in range(0, npiv, 128):
        if k + 64 < npiv:
            seq.append("strip")
        seq.append("update")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "launch__grid_size"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(head)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "": 1}
def val(r, name):
    v = r[col[name]].replace(",", "")
    return float(v) * scale.get(units[col[name]], 1)
launches = []
for r in data:
    launches.append(dict(grid=int(val(r, "launch__grid_size")),
                         ms=val(r, "gpu__time_duration.sum") * 1e3,
                         dram_bytes=val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")))
mode0 = [l for l, kind in zip(launches, seq) if kind == "update"]
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
