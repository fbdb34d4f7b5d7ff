"""Print key metrics + warp stall breakdown from an ncu report (raw page)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:60])
        for k in KEYS:
            if k in hdr:
                print(f"  {k:62s} {r[hdr.index(k)]:>16s} {units[hdr.index(k)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warp_latency_issue_stalled_"):-6]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  stalls (avg cycles per issued instr):",
              ", ".join(f"{n}={v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
