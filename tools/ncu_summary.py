"""Text summary of an ncu --set full capture (first kernel): the metrics DESIGN.md and the bench
cite (duration, DRAM bytes, throughput, issue / tensor-pipe activity, occupancy, warp stall mix).
    python tools/ncu_summary.py report.ncu-rep "title" > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum"]


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    print(f"# {title}")
    print(f"# kernel: {v[h.index('Kernel Name')][:120]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {v[i]:>20s} {units[i]}")
    stalls = {k: float(x) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
              not k.endswith("not_issued") and x.replace(".", "").isdigit()}
    tot = sum(stalls.values()) or 1.0
    print("# warp-state samples (share of all samples)")
    for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        print(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', 'stall_'):40s} {100 * x / tot:6.1f} %")


if __name__ == "__main__":
    main()
