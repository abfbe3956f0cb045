"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref/libbbm_ref.so).

Run in the container that has /root/reference (after `make -C oracle`):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz. The fixtures pin both the C oracle restatement and the GPU path when
the reference itself is not available (e.g. on the GPU box), and are small enough to commit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def family_specs(n: int):
    """test_util.hpp:63-84 family_masks(n) as spec strings."""
    w8 = max(1, n // 8)
    return [
        ("causal", n), ("all-ones", n), (f"windowed(w={w8})", n), (f"windowed(w={w8};causal=1)", n),
        (f"dilated(w={max(1, n // 16)};d=2)", n), (f"global(w={w8};g={min(4, n)})", n),
        (f"packed-seq[{n // 2};{n - n // 2}]", 0),
        (f"packed-bidir[{n // 4}:{n // 4};{n // 4}:{n - 3 * (n // 4)}]", 0),
        ("random(p=0.05;seed=17)", n), ("random(p=0.4;seed=18)", n),
    ]


def main():
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libbbm_ref.so missing: run `make -C oracle` where /root/reference exists")

    # ---- mask model: masks x specs -> sums/occ/runs/stats (mask.hpp:184-247)
    cases = {}
    specs = [(2, 2), (3, 5), (16, 16), (32, 16), (64, 64), (128, 128), (128, 64), (128, 32), (8, 8)]
    idx = 0
    for n in (15, 64, 100, 130, 257):
        for spec_str, nn in family_specs(n):
            words = oracle.ref_generate(spec_str, nn)
            m = words.shape[0]
            for bi, bj in specs:
                sums, occ, off, tot, st = oracle.ref_preprocess(words, m, bi, bj)
                key = f"c{idx}"
                idx += 1
                cases[key + "_spec"] = np.array([m, bi, bj], np.uint64)
                cases[key + "_name"] = np.array(spec_str)
                cases[key + "_words"] = words
                cases[key + "_sums"] = sums
                cases[key + "_occ"] = occ
                cases[key + "_off"] = off
                cases[key + "_tot"] = tot
                cases[key + "_stats_u"] = np.array([st["blocks_total"], st["blocks_nonzero"],
                                                    st["blocks_full"]], np.uint64)
                cases[key + "_stats_f"] = np.array([st["block_density"], st["element_density"]])
    # MEDUSA trees (generators.hpp:22-63) incl. the paper's [4;4;4;4]
    for tree in ("medusa[4;4;4;4]", "medusa[8;7]", "medusa[16;15]"):
        words = oracle.ref_generate(tree)
        m = words.shape[0]
        for bi, bj in ((128, 32), (128, 128), (64, 64)):
            sums, occ, off, tot, st = oracle.ref_preprocess(words, m, bi, bj)
            key = f"c{idx}"
            idx += 1
            cases[key + "_spec"] = np.array([m, bi, bj], np.uint64)
            cases[key + "_name"] = np.array(tree)
            cases[key + "_words"] = words
            cases[key + "_sums"] = sums
            cases[key + "_occ"] = occ
            cases[key + "_off"] = off
            cases[key + "_tot"] = tot
            cases[key + "_stats_u"] = np.array([st["blocks_total"], st["blocks_nonzero"],
                                                st["blocks_full"]], np.uint64)
            cases[key + "_stats_f"] = np.array([st["block_density"], st["element_density"]])
    cases["count"] = np.array(idx)
    np.savez_compressed(os.path.join(HERE, "mask_model.npz"), **cases)
    print(f"mask_model.npz: {idx} cases")

    # ---- counters per variant (engine.hpp:118-153) on a few masks, d=4 (values irrelevant)
    cnt = {}
    j = 0
    for spec_str, nn in family_specs(96)[:8]:
        words = oracle.ref_generate(spec_str, nn)
        m = words.shape[0]
        q, k, v, _ = oracle.ref_make_problem_f32(5, 1, m, 4)
        for bi, bj in ((16, 16), (32, 16), (128, 128)):
            for var in range(4):
                _, _, _, c = oracle.ref_blocked_forward(q, k, v, 0.5, words, m, bi, bj, var, threads=2)
                cnt[f"k{j}"] = np.array([m, bi, bj, var, *c], np.uint64)
                cnt[f"k{j}_words"] = words
                j += 1
    cnt["count"] = np.array(j)
    np.savez_compressed(os.path.join(HERE, "counters.npz"), **cnt)
    print(f"counters.npz: {j} cases")

    # ---- forward: config C1 (causal N=1024, d=64) slot 0 and a ragged MEDUSA case, reference
    # blocked_forward<float> (binblk, 128x128) on bf16-rounded make_problem inputs.
    fwd = {}
    for name, spec_str, nn, d in (("c1", "causal", 1024, 64), ("medusa", "medusa[4;4;4;4]", 0, 128),
                                  ("packed", "packed-seq[100;300;57;311]", 0, 128)):
        words = oracle.ref_generate(spec_str, nn)
        m = words.shape[0]
        q, k, v, _ = oracle.make_problem(1, 1, m, d)
        qb, kb, vb = (oracle.bf16_round(a) for a in (q, k, v))
        scale = 1.0 / np.sqrt(d)
        out, rmax, rsum, c = oracle.ref_blocked_forward(qb.astype(np.float32), kb.astype(np.float32),
                                                        vb.astype(np.float32), scale, words, m, 128, 128,
                                                        2, threads=8)
        fwd[f"{name}_words"] = words
        fwd[f"{name}_meta"] = np.array([m, d, 1], np.uint64)
        fwd[f"{name}_out"] = out[0].astype(np.float32)
        fwd[f"{name}_row_max"] = rmax[0]
        fwd[f"{name}_row_sum"] = rsum[0]
        fwd[f"{name}_counters"] = np.array(c, np.uint64)
    np.savez_compressed(os.path.join(HERE, "forward.npz"), **fwd)
    print("forward.npz written")

    # ---- RCM permutations (reorder.hpp:85-133)
    rcm = {}
    j = 0
    masks = [oracle.ref_generate(s, n) for s, n in (
        ("random(p=0.02;seed=3)", 200), ("random(p=0.005;seed=4;diag=0)", 300), ("windowed(w=5)", 150),
        ("causal", 40), ("dilated(w=3;d=4)", 90), ("global(w=3;g=2)", 64))]
    for words in masks:
        m = words.shape[0]
        fwd_perm, bw0, bw1 = oracle.ref_rcm(words, m)
        rcm[f"r{j}_words"] = words
        rcm[f"r{j}_fwd"] = fwd_perm
        rcm[f"r{j}_bw"] = np.array([bw0, bw1], np.uint64)
        j += 1
    rcm["count"] = np.array(j)
    np.savez_compressed(os.path.join(HERE, "rcm.npz"), **rcm)
    print(f"rcm.npz: {j} cases")


if __name__ == "__main__":
    main()
