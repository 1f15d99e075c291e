"""Key metrics of every kernel in an `ncu --page raw --csv` export (one line per metric)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "barrier / issue"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "membar / issue"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    units = rows[1] if len(rows) > 1 else [""] * len(hdr)
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:90]}")
        for k, name in KEYS:
            if k in d:
                print(f"   {name:28s} {d[k]} {u.get(k, '')}")


if __name__ == "__main__":
    main(sys.argv[1])
