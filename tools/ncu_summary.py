"""Summarise ncu output for profiles/: key metrics of an `ncu --set full`
report (per kernel) or the per-kernel totals of a `--metrics
gpu__time_duration.sum` launch list (CSV).

    python tools/ncu_summary.py rep  gpurun_out/prof.ncu-rep  > profiles/...txt
    python tools/ncu_summary.py list gpurun_out/launches.csv  > profiles/...txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sass__inst_executed_local_loads",
    "sass__inst_executed_local_stores",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        print(f"kernel: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {vals[i]:>18s} {units[i]}")
        print()


def launch_list(path):
    """Per (kernel, grid) totals -- the grid separates the bench legs that
    launch the same kernel (single fit: (148,1,1); population batch:
    (x, saccades, 1); NM: one block per problem group)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    d = defaultdict(list)
    for r in rows[1:]:
        d[(r[ki], r[gi])].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(f"{'launches':>8s} {'mean_ns':>12s} {'total_ns':>12s} {'share':>6s}  {'grid':>16s}  kernel")
    for (k, g), v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v)/len(v):12.1f} {sum(v):12.1f} {100*sum(v)/tot:5.1f}%  {g:>16s}  {k}")
    # every launch in order (us), so the legs that share a (kernel, grid) --
    # e.g. the 10^6-candidate step and the latency leg's 10^5..10^8 fits --
    # can be told apart
    print("\n# launches in order: id  grid  us  kernel")
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        print(f"{r[0]:>5s} {r[gi]:>16s} {float(r[vi].replace(',', '')) / 1e3:12.1f}  {name}")


if __name__ == "__main__":
    {"rep": rep, "list": launch_list}[sys.argv[1]](sys.argv[2])
