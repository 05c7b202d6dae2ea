"""Summarise ncu outputs for profiles/:
   python tools/ncu_summary.py launches.csv [full.ncu-rep ...] > profiles/ncu_summary_rNN.md

* launch list (gpu__time_duration.sum per launch, cold and serialised): per
  kernel name, launches, total / mean ms and share of all kernel time;
* full captures: duration, DRAM bytes read + written, achieved DRAM GB/s,
  SM / DMMA pipe utilisation, registers, occupancy, smem per block."""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").strip()


def launches(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}[r["Metric Unit"]]
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        out.append(f"| {k} | {n} | {ms:.2f} | {1e3 * ms / n:.1f} | {ms / tot:.3f} |")
    out.append(f"\nall kernels: {sum(a[0] for a in agg.values())} launches, {tot:.1f} ms")
    return "\n".join(out)


METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_subpipe_pct (DMMA on the tensor pipe)",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct (DFMA, not DMMA)",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard": "stall_long_sb",
}


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        line = [f"### {short(d.get('Kernel Name', '?'))}  ({path.split('/')[-1]})"]
        for m, lab in METRICS.items():
            if m in d:
                line.append(f"- {lab} ({m}): {d[m]} {u.get(m, '')}")
        out.append("\n".join(line))
    return "\n\n".join(out)


if __name__ == "__main__":
    print("## launch list\n")
    print(launches(sys.argv[1]))
    for p in sys.argv[2:]:
        print("\n## full capture\n")
        print(full(p))
