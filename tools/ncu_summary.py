"""Summarise an ncu --set full report: key counters and warp-stall breakdown.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:100])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:88s} {v[i]:>14s} {u[i]}")
        stalls = [(float(v[i] or 0), n) for i, n in enumerate(h)
                  if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio")]
        if not stalls:
            stalls = [(float(v[i] or 0), n) for i, n in enumerate(h)
                      if n.startswith("smsp__pcsamp_warps_issue_stalled_") and v[i]]
        for val, n in sorted(stalls, reverse=True)[:8]:
            print(f"  stall {n:86s} {val:>10.2f}")


if __name__ == "__main__":
    main()
