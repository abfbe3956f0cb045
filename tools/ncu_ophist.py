"""Executed-instruction histogram by opcode from an ncu report's source page (SASS).

    python tools/ncu_ophist.py gpurun_out/x.ncu-rep [per_unit_divisor]

Weights every SASS line by its 'Instructions Executed' (warp-level) count; with a divisor (e.g.
engine warps x tiles) prints per-unit counts.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(path, div=1.0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[1]
    recs = [dict(zip(head, r)) for r in rows[2:] if len(r) == len(head)]
    hist = collections.Counter()
    for r in recs:
        src = r["Source"].strip()
        src = re.sub(r"^@!?U?P\w+\s+", "", src)
        op = src.split()[0] if src else "?"
        hist[op] += float(r["Instructions Executed"] or 0)
    tot = sum(hist.values())
    print(f"total {tot:.0f} warp-instructions ({tot / div:.1f} per unit)")
    for op, c in hist.most_common(45):
        print(f"{op:28s} {c / div:10.1f} {c / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
