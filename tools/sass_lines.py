"""Per-source-line warp-stall samples of one kernel from an ncu --set full
report (needs -lineinfo): python tools/sass_lines.py REP KERNEL_SUBSTR CUBIN [N]
Maps ncu's SASS addresses to file:line with nvdisasm -g."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, kname, cubin = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
samples = {}
for r in rows[1:]:
    try:
        samples[int(r[ia], 16)] = (float(r[iss] or 0), {hdr[i]: float(r[i] or 0) for i in stall_cols})
    except (ValueError, IndexError):
        pass
base = min(samples) if samples else 0
samples = {a - base: v for a, v in samples.items()}
# function name in the cubin
syms = subprocess.run(["cuobjdump", "-symbols", cubin], capture_output=True, text=True).stdout
fn = [s.split()[-1] for s in syms.splitlines() if kname in s and "STO_ENTRY" in s]
if not fn:
    sys.exit(f"{kname} not in {cubin}")
full_dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = full_dis.split(".text." + fn[0] + ":")
if len(sec) < 2:
    sys.exit("function section not found")
dis = sec[1].split(".section")[0]
cur = None
agg = defaultdict(float)
why = defaultdict(lambda: defaultdict(float))
for l in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a = int(m.group(1), 16)
        if a in samples:
            agg[cur] += samples[a][0]
            for k, v in samples[a][1].items():
                why[cur][k] += v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    w = sorted(why[k].items(), key=lambda kv: -kv[1])[:3]
    print(f"{v / tot:6.3f} {k:28s} " + " ".join(f"{a[6:]}={b / max(v, 1):.2f}" for a, b in w))
