"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

    python tools/ncu_summary.py rep gpurun_out/prof.ncu-rep > profiles/ncu_<name>_r01.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/launches_<name>_r01.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {r[i]:>18s} {units[i]}")
        stalls = [(float(r[i] or 0), h[i]) for i in range(len(h))
                  if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")]
        stalls.sort(reverse=True)
        print("  top stall reasons (warps per issue):")
        for v, k in stalls[:8]:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "ns": 1e-3, "s": 1e6}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0][:60]][0] += 1
        agg[r[ki].split("(")[0][:60]][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"total device time {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches "
          f"(ncu serialised, cold cache: compare shares)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:62s} n={c:6d} {t / 1e3:10.3f} ms {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
