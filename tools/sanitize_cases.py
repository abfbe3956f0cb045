"""Small launches for compute-sanitizer (racecheck / synccheck / memcheck): every forward variant
on C1/C3-shaped problems incl. ragged n, multi-slot and split-KV rows, the backward, and the
fused preprocessor update path.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_15097_b200 as bbm  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    cases = [("causal", 640, 64, 2), ("packed-seq[100;260;37;243]", 0, 128, 3),
             ("global(w=64;g=100)", 2048, 64, 1), ("all-ones", 300, 128, 2)]
    for spec, n, d, slots in cases:
        mask = bbm.generate(spec, n)
        n = mask.size()
        prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(dev), bbm.BlockSpec(128, 128))
        q, k, v, go = ((torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
                       for _ in range(4))
        for var in bbm.Variant:
            r = bbm.blocked_forward(q, k, v, d ** -0.5, mask, prep, var)
            b = bbm.blocked_backward(q, k, v, d ** -0.5, mask, prep, var, r, go)
            torch.cuda.synchronize()
            assert bool(torch.isfinite(r.out.float()).all()) and bool(torch.isfinite(b.dq.float()).all())
        prep.update(torch.from_numpy(mask.to_dense()).to(dev))
        bbm.blocked_forward(q, k, v, d ** -0.5, mask, prep, bbm.Variant.binblk)
        torch.cuda.synchronize()
        print(f"ok {spec} n={n} d={d} slots={slots}", flush=True)


if __name__ == "__main__":
    main()
