"""Summarise `ncu --set full` captures (.ncu-rep) into one text table per kernel: duration,
DRAM bytes, throughput and pipe utilisation, occupancy.  Usage:
  python tools/ncu_summary.py OUT.txt rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe % (active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem) blocks"),
    ("smsp__average_warp_latency_issue_stalled_short_scoreboard", "stall short scoreboard"),
]


def main(out, reps):
    lines = []
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(h, r))
            lines.append(f"== {rep.split('/')[-1]}: {d.get('Kernel Name', '?')}")
            for k, label in KEYS:
                if k in d:
                    lines.append(f"  {label:34s} {d[k]:>14s} {units[h.index(k)]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
