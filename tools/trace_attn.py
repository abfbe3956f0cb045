"""Per-role event trace of the attention kernel (bbm_set_trace) and a latency breakdown.

    python tools/trace_attn.py [--config c2] [--variant binblk] [--ctas 2] [--dump out.txt]

Runs one traced launch after a warm launch, decodes the events of the first CTAs and prints, per
stream, the average cycles between consecutive stages of a tile (S issue -> softmax start ->
P ready -> PV issue) and across item boundaries.
"""
from __future__ import annotations

import argparse
import collections
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {1: "P:Q", 2: "P:K", 3: "P:V", 10: "M:S", 11: "M:PV", 12: "M:Vready", 13: "M:Kready", 14: "M:Pseen", 25: "X:sregs", 26: "X:maxed", 27: "X:pcomp", 20: "X:swait", 21: "X:sready",
         22: "X:pready", 23: "X:oready", 24: "X:epi_done", 28: "X:stats", 29: "X:item"}


def main():
    import numpy as np
    import torch

    import bench
    import paper_2409_15097_b200 as bbm
    from paper_2409_15097_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--variant", default="binblk")
    ap.add_argument("--ctas", type=int, default=2)
    ap.add_argument("--dump", default=None)
    a = ap.parse_args()

    dev = torch.device("cuda", 0)
    mask, B, H, d, desc = bench.make_config(a.config)
    slots, n = B * H, mask.size()
    prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(dev), bbm.BlockSpec(128, 128))
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = ((torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    var = bbm.parse_variant(a.variant)
    bbm.attn_fwd_device(prep, var, q, k, v, out, None, None, d ** -0.5)
    buf = torch.zeros(a.ctas * 8192, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib.bbm_set_trace(C.c_void_p(buf.data_ptr()), a.ctas))
    bbm.attn_fwd_device(prep, var, q, k, v, out, None, None, d ** -0.5)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.bbm_set_trace(None, 0))
    ev = buf.cpu().numpy().view(np.uint64).reshape(a.ctas, 8192)

    lines = []
    for c in range(a.ctas):
        evs = [(int(x >> 24), int((x >> 16) & 0xFF), int((x >> 15) & 1), int(x & 0x7FFF)) for x in ev[c] if x]
        evs.sort()
        t0 = evs[0][0]
        for t, code, s, aux in evs:
            lines.append(f"cta{c} {t - t0:9d} s{s} {str(NAMES.get(code, code)):10s} {aux}")
        # per stream stage latencies
        per = collections.defaultdict(list)
        last = {}
        for t, code, s, aux in evs:
            key = (s, code)
            last[key] = t
            if code == 21 and (s, 10) in last:
                per["S issue -> softmax has S"].append(t - last[(s, 10)])
            if code == 21 and (s, 20) in last:
                per["softmax waited for S"].append(t - last[(s, 20)])
            if code == 25 and (s, 21) in last:
                per["  S ready -> S in registers"].append(t - last[(s, 21)])
            if code == 26 and (s, 25) in last:
                per["  S in registers -> row max exchanged"].append(t - last[(s, 25)])
            if code == 27 and (s, 26) in last:
                per["  max exchanged -> P computed"].append(t - last[(s, 26)])
            if code == 22 and (s, 27) in last:
                per["  P computed -> P stored + arrive"].append(t - last[(s, 27)])
            if code == 22 and (s, 21) in last:
                per["softmax compute (S ready -> P ready)"].append(t - last[(s, 21)])
            if code == 11 and (s, 22) in last:
                per["P ready -> PV issued"].append(t - last[(s, 22)])
            if code == 14 and (s, 22) in last:
                per["  P ready -> MMA sees P"].append(t - last[(s, 22)])
            if code == 12 and (s, 14) in last:
                per["  MMA sees P -> V landed"].append(t - last[(s, 14)])
            if code == 11 and (s, 12) in last:
                per["  V landed -> PV issued"].append(t - last[(s, 12)])
            if code == 13 and (s, 11) in last:
                per["  PV issued -> K landed"].append(t - last[(s, 11)])
            if code == 10 and (s, 13) in last:
                per["  K landed -> S issued"].append(t - last[(s, 13)])
            if code == 10 and (s, 11) in last:
                per["PV issued -> next S issued"].append(t - last[(s, 11)])
            if code == 23 and (s, 22) in last:
                per["last P ready -> O ready (epilogue start)"].append(t - last[(s, 22)])
            if code == 24 and (s, 23) in last:
                per["epilogue (O ready -> done)"].append(t - last[(s, 23)])
            if code == 20 and (s, 24) in last:
                per["epilogue done -> next softmax wait"].append(t - last.pop((s, 24)))
        # engine time budget: every cycle between consecutive engine events gets one label
        eng = [e for e in evs if e[1] in (20, 21, 22, 25, 26, 27, 28, 29)]  # 23/24: epilogue warpgroup
        lab = {(20, 21): "wait S", (21, 25): "S tmem load", (25, 26): "mask + max + exchange",
               (26, 27): "exp + P pack", (27, 22): "P store + arrive", (22, 20): "tile gap",
               (22, 28): "item end: stats hand-over", (28, 29): "next item descriptor",
               (29, 20): "item start: first mask bits etc."}
        budget = collections.Counter()
        for (ta, ca, _, _), (tb, cb, _, ab) in zip(eng, eng[1:]):
            name = lab.get((ca, cb), f"{ca}->{cb}")
            if cb in (20, 21):
                name += " (item start)" if ab == 0 else " (in item)"
            budget[name] += tb - ta
        tot = sum(budget.values())
        print(f"  engine budget over {tot} cycles:")
        for name, v in budget.most_common():
            print(f"     {name:40s} {v / tot:6.1%}")
        span = evs[-1][0] - t0
        n_s = sum(1 for e in evs if e[1] == 10)
        print(f"CTA {c}: span {span} cycles, {n_s} S tiles, {span / max(1, n_s):.0f} cycles/tile (both streams)")
        for k2, vals in per.items():
            vals = np.array(vals)
            print(f"   {k2:42s} n={len(vals):4d} mean={vals.mean():8.0f} p50={np.median(vals):8.0f} max={vals.max():8.0f}")
    if a.dump:
        with open(a.dump, "w") as f:
            f.write("\n".join(lines))


if __name__ == "__main__":
    main()
