"""Top stalled SASS instructions of an ncu report (source page, --print-source sass).

    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[1]
    recs = [dict(zip(head, r)) for r in rows[2:] if len(r) == len(head)]
    stall_cols = [h for h in head if h.startswith("stall_") and "Not Issued" not in h]
    total = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in recs)
    agg = {c: sum(float(r[c] or 0) for r in recs) for c in stall_cols}
    print(f"total samples {total:.0f}")
    print("by reason:", ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
    recs.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in recs[:top]:
        s = float(r["Warp Stall Sampling (All Samples)"] or 0)
        reasons = sorted(((float(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{s / total:6.2%} {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} " +
              " ".join(f"{n}:{v / max(s, 1):.0%}" for v, n in reasons if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
