"""Prints the key counters of an ncu --set full report (one kernel launch per report)."""
import csv, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "sm__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size"]
def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:100])
        for i, h in enumerate(hdr):
            if h in KEYS or ("stalled" in h and h.endswith("per_issue_active.ratio") and float(vals[i] or 0) > 0.3):
                print(f"  {h} [{units[i]}] = {vals[i]}")
if __name__ == "__main__":
    main(sys.argv[1])
