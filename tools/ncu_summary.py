"""Per-kernel summary of an ncu --set full report (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/xxx.txt
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("sm__inst_executed.sum.per_cycle_active", "IPC (SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_static", "static smem/block"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    stall = [i for i, n in enumerate(h)
             if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        print(f"== {r[ki].split('(')[0]}")
        for m, label in WANT:
            if m in h:
                i = h.index(m)
                print(f"   {label:28s} {r[i]} {units[i]}")
        vals = sorted(((float(r[i] or 0), h[i][len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')])
                       for i in stall), reverse=True)[:6]
        print("   top stalls (cycles/issue)   " + ", ".join(f"{n} {v:.2f}" for v, n in vals))


if __name__ == "__main__":
    main(sys.argv[1])
