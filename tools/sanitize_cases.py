"""Small launches for compute-sanitizer (racecheck / synccheck / memcheck): every forward variant
on C1/C3-shaped problems incl. ragged n, multi-slot and split-KV rows, the backward, and the
fused preprocessor update path; band masks whose repeated launches skip empty 64-row halves
(forward and backward), the device RCM application in all four modes, and the opt-in two-stream
forward.

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
             ("global(w=64;g=100)", 2048, 64, 1), ("all-ones", 300, 128, 2),
             ("windowed(w=40)", 1500, 128, 2), ("windowed(w=30)", 1000, 64, 2)]
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
        # repeated launches: the plan header has reached the host, half skipping (if the mask has
        # enough empty halves) is on in the forward and both backward kernels
        for _ in range(2):
            r = bbm.blocked_forward(q, k, v, d ** -0.5, mask, prep, bbm.Variant.binblk)
            b = bbm.blocked_backward(q, k, v, d ** -0.5, mask, prep, bbm.Variant.binblk, r, go)
        torch.cuda.synchronize()
        prep.update(torch.from_numpy(mask.to_dense()).to(dev))
        bbm.blocked_forward(q, k, v, d ** -0.5, mask, prep, bbm.Variant.binblk)
        torch.cuda.synchronize()
        print(f"ok {spec} n={n} d={d} slots={slots}", flush=True)
    # device RCM application (passes / TMA gather4 / hybrid / LSU gather) and the two-stream forward
    base = bbm.relabel(bbm.generate("windowed(w=40)", 1000), 5)
    perm = bbm.rcm_order(base)
    prep = bbm.preprocess_mask(bbm.permute_mask(base, perm), bbm.BlockSpec(128, 128))
    rows = torch.from_numpy(perm.forward.astype(np.int32)).to(dev)
    q, k, v = ((torch.rand((2, 1000, 128), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    m = torch.empty((2, 1000), dtype=torch.float32, device=dev)
    l = torch.empty_like(m)
    for mode in (1, 2, 3, 4):  # passes, TMA gather4, hybrid, LSU cp.async gather
        for var in bbm.Variant:
            bbm.attn_fwd_device(prep, var, q, k, v, out, m, l, 0.08, rows=rows, gather_mode=mode)
    bbm.set_fwd_kernel("pair")
    bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k, v, out, m, l, 0.08)
    bbm.set_fwd_kernel("auto")
    torch.cuda.synchronize()
    print("ok rcm passes / tma gather / pair kernel", flush=True)


if __name__ == "__main__":
    main()
