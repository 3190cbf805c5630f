"""Summarise an ncu --set full report: per kernel, the headline metrics and
the top warp-stall reasons (reads `ncu -i REP --page details/raw --csv`)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "No Eligible", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__average_warp_latency_issue_stalled_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio"]


def main(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    out = {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] in WANT:
            out.setdefault((r[ii], r[ki]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    for r in rr[2:]:
        key = (r[h.index("ID")], r[h.index("Kernel Name")])
        for m in RAW:
            if m in h:
                out.setdefault(key, {})[m] = r[h.index(m)]
    for (i, k), d in out.items():
        print(f"== [{i}] {k[:90]}")
        for m, v in d.items():
            print(f"   {m:80s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
