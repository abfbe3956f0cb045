"""Summarise ncu --set full reports (raw page) into a compact markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/r01_attn_*.ncu-rep > profiles/r01_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (realtime)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return [(dict(zip(head, r)), dict(zip(head, units))) for r in rows[2:]]


def main(paths):
    print("| report | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for p in paths:
        for d, u in raw(p):
            name = d.get("Kernel Name", "?").split("(")[0].split("::")[-1][:40]
            cells = []
            for k, _ in KEYS:
                v = d.get(k, "")
                unit = u.get(k, "")
                cells.append(f"{v} {unit}".strip() if v else "n/a")
            print(f"| {p.split('/')[-1]} | {name} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
