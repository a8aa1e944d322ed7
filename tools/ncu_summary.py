"""Key metrics of one ncu --set full report (first kernel) as text: duration, DRAM traffic, pipe utilisation,
occupancy, stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name[:120])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print("  %-80s %14s %s" % (k, v[i], u[i]))
        stalls = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled_")
                  and h[i].endswith("_per_issue_active.ratio")]
        stalls = sorted(((float(x.replace(",", "")), n) for n, x in stalls if x), reverse=True)[:6]
        print("  top stalls (warps per issue):", ", ".join("%s %.2f" % (n.split("stalled_")[1].split("_per")[0], s)
                                                         for s, n in stalls))


if __name__ == "__main__":
    main(sys.argv[1])
