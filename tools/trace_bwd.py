"""Per-role event trace of one backward kernel (dq or dkdv) and a per-half time budget.

    python tools/trace_bwd.py [--config c2] [--variant binblk] [--side dq|dkdv] [--ctas 1]

Runs the forward for the row statistics, one warm backward, then one traced backward with
BBM_TRACE_BWD_SIDE selecting the kernel (attn_bwd.cu event codes 40-55).
"""
from __future__ import annotations

import argparse
import collections
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LABELS = {(50, 51): "wait S/dP", (51, 52): "elementwise (P, dS)", (52, 50): "tile gap",
          (52, 53): "wait last accumulate (item end)", (53, 54): "epilogue", (54, 55): "next item",
          (55, 50): "item start", (55, 54): "empty item"}


def main():
    import numpy as np
    import torch

    import bench
    import paper_2409_15097_b200 as bbm
    from paper_2409_15097_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", default="binblk")
    ap.add_argument("--side", default="dq", choices=["dq", "dkdv"])
    ap.add_argument("--ctas", type=int, default=1)
    a = ap.parse_args()
    os.environ["BBM_TRACE_BWD_SIDE"] = "0" if a.side == "dq" else "1"

    dev = torch.device("cuda", 0)
    mask, B, H, d, _ = bench.make_config(a.config)
    slots, n = B * H, mask.size()
    prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(dev), bbm.BlockSpec(128, 128))
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = ((torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4))
    var = bbm.parse_variant(a.variant)
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=dev)
    rsum = torch.empty_like(rmax)
    bbm.attn_fwd_device(prep, var, q, k, v, out, rmax, rsum, d ** -0.5)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    bbm.attn_bwd_device(prep, var, q, k, v, out, rmax, rsum, do, dq, dk, dv, d ** -0.5)
    buf = torch.zeros(a.ctas * 8192, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib.bbm_set_trace(C.c_void_p(buf.data_ptr()), a.ctas))
    bbm.attn_bwd_device(prep, var, q, k, v, out, rmax, rsum, do, dq, dk, dv, d ** -0.5)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.bbm_set_trace(None, 0))
    ev = buf.cpu().numpy().view(np.uint64).reshape(a.ctas, 8192)

    for c in range(a.ctas):
        evs = sorted((int(x >> 24), int((x >> 16) & 0xFF), int((x >> 15) & 1), int(x & 0x7FFF)) for x in ev[c] if x)
        if not evs:
            print(f"CTA {c}: no events")
            continue
        t0, t1 = evs[0][0], evs[-1][0]
        n_items = sum(1 for e in evs if e[1] == 43)
        n_tiles = sum(1 for e in evs if e[1] == 41) // 2
        print(f"CTA {c} ({a.side}): span {t1 - t0} cycles, {n_items} items, {n_tiles} tiles, "
              f"{(t1 - t0) / max(1, n_tiles):.0f} cycles/tile")
        for h in (0, 1):
            eng = [e for e in evs if e[2] == h and 50 <= e[1] <= 55]
            budget = collections.Counter()
            for (ta, ca, _, _), (tb, cb, _, _) in zip(eng, eng[1:]):
                budget[LABELS.get((ca, cb), f"{ca}->{cb}")] += tb - ta
            tot = sum(budget.values())
            print(f"  half {h} engine budget over {tot} cycles:")
            for name, val in budget.most_common():
                print(f"     {name:36s} {val / tot:6.1%}  ({val / max(1, n_tiles):6.0f} / tile)")
        # MMA-side latencies per half
        lat = collections.defaultdict(list)
        last = {}
        for t, code, s, aux in evs:
            last[(s, code)] = t
            if code == 51 and (s, 40) in last:
                lat[f"h{s} S/dP issued -> engine has S"].append(t - last[(s, 40)])
            if code == 42 and (s, 52) in last:
                lat[f"h{s} P arrive -> MMA sees P"].append(t - last[(s, 52)])
            if code == 41 and (s, 42) in last:
                lat[f"h{s} MMA sees P -> accumulate issued"].append(t - last[(s, 42)])
            if code == 40 and (s, 41) in last:
                lat[f"h{s} accumulate issued -> next S/dP issued"].append(t - last[(s, 41)])
        for k2 in sorted(lat):
            vals = np.array(lat[k2])
            print(f"   {k2:44s} n={len(vals):4d} mean={vals.mean():7.0f} p50={np.median(vals):7.0f}")


if __name__ == "__main__":
    main()
