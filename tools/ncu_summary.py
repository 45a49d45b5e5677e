"""Summarise ncu reports (run here, no GPU): key roofline counters per kernel.

    python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/<round>_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("dram__bytes_read.sum.per_second", "dram read BW"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor mem active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict((h, (r[i], units[i])) for i, h in enumerate(hdr)) for r in rows[2:]]


def main(paths):
    print("| report | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|" + "---|" * (len(KEYS) + 2))
    for p in paths:
        for rec in raw(p):
            name = rec.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("void ", "")[-40:]
            cells = []
            for k, _ in KEYS:
                v = rec.get(k)
                cells.append(f"{v[0]} {v[1]}".strip() if v else "-")
            print(f"| {p.split('/')[-1]} | {name} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
