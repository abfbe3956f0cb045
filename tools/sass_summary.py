"""Per-kernel SASS instruction summary of libbbm.so (cuobjdump -sass), the evidence that the hot
kernels are tcgen05/TMA-native (UTCHMMA / UTMALDG / UTMASTG / LDTM / STTM, no HMMA) and where
local-memory spills (STL / LDL) sit.

    python tools/sass_summary.py [--lib paper_2409_15097_b200/libbbm.so] [--filter attn_] [--spills]
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "LDGSTS", "UTMAPF", "LDTM", "STTM", "HMMA", "MUFU.EX2",
        "FFMA2", "FADD2", "FMUL2", "F2FP", "FMNMX", "SYNCS", "BAR", "LDS", "STS", "LDG", "STG", "STL", "LDL",
        "NANOSLEEP", "ELECT"]


def demangle(name: str) -> str:
    try:
        return subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2409_15097_b200", "libbbm.so"))
    ap.add_argument("--filter", default="attn_")
    ap.add_argument("--spills", action="store_true", help="print the instructions around each STL/LDL")
    a = ap.parse_args()
    out = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)[1:]
    rows = []
    for f in funcs:
        name, _, body = f.partition("\n")
        if a.filter not in name and a.filter not in demangle(name.strip()):
            continue
        ops = collections.Counter()
        lines = [ln for ln in body.splitlines() if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln)]
        for ln in lines:
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
            if not m:
                continue
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    ops[k] += 1
        rows.append((demangle(name.strip()), len(lines), ops))
        if a.spills:
            for i, ln in enumerate(lines):
                if re.search(r"\b(STL|LDL)\b", ln):
                    ctx = " | ".join(re.sub(r"\s+", " ", x.split("*/", 1)[-1]).strip()[:40] for x in lines[max(0, i - 2):i + 3])
                    print(f"   {demangle(name.strip())[:60]}: {ctx}")
    print("| kernel | instructions | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for name, n, ops in rows:
        short = re.sub(r"bbm::\(anonymous namespace\)::", "", name)
        short = re.sub(r"\(CUtensorMap_st.*", "", short)
        print(f"| `{short}` | {n} | " + " | ".join(str(ops.get(k, 0)) for k in KEYS) + " |")
    return 0


if __name__ == "__main__":
    sys.exit(main())
