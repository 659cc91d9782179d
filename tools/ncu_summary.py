"""Prints the key counters of an ncu --set full report (run here, no GPU needed)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): d[h] for h in hdr
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(float(v.replace(",", "") or 0) for v in stalls.values())
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
        print("  stall samples (top):", ", ".join(f"{k} {100 * float(v.replace(',', '')) / tot:.1f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
