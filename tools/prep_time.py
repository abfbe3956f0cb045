"""Device time of bbm_prep_update_bool_device (the fused one-launch preprocessor) on the configs'
dense bool masks, back-to-back updates (bench.device_ms), for preprocessor A/B runs.

    python tools/prep_time.py [--configs c2,c5] [--reps 50]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2409_15097_b200 as bbm

    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c5")
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    for name in a.configs.split(","):
        mask, *_ = bench.make_config(name)
        n = mask.size()
        dense = torch.from_numpy(mask.to_dense()).to(dev)
        prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
        with torch.cuda.stream(stream):
            for _ in range(5):
                prep.update(dense, stream.cuda_stream)
            best = min(bench.device_ms(stream, lambda: prep.update(dense, stream.cuda_stream), a.reps)
                       for _ in range(3))
        print(json.dumps({"config": name, "n": n, "us": best * 1e3, "gbs_bool": n * n / (best * 1e-3) / 1e9,
                          "lib": os.environ.get("BBM_LIB", "in-tree")}))


if __name__ == "__main__":
    main()
