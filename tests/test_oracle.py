"""Pin the CPU oracle (oracle/bbm_oracle.c) before trusting it.

1. The reference's own known-answer tests (test_mask_model.cpp, test_engine.cpp,
   test_reorder.cpp), re-asserted against the C restatement.
2. Golden vectors produced by the real reference headers (tests/golden/*.npz, made by
   tests/golden/make_golden.py through oracle/_ref), compared bit-for-bit / to 1e-6.
3. When oracle/_ref is present, direct comparisons against the reference on fresh inputs.
"""
import os

import numpy as np
import pytest

import oracle
from tests.conftest import GOLDEN


def words_from_dense(dense):
    n = dense.shape[0]
    wpr = (n + 63) // 64
    pad = np.zeros((n, wpr * 64), np.uint8)
    pad[:, :n] = dense
    return np.packbits(pad, axis=1, bitorder="little").view(np.uint64).reshape(n, wpr)


def causal(n):
    return words_from_dense(np.tril(np.ones((n, n), bool)))


# ------------------------------------------------------------------ KATs (test_mask_model.cpp)

def test_kat_causal_four_by_four():  # test_mask_model.cpp:81-107
    sums, occ, off, tot, st = oracle.preprocess(causal(4), 4, 2, 2)
    assert sums.tolist() == [[3, 0], [4, 3]]
    assert occ.tolist() == [[1, 0], [1, 1]]
    assert off.tolist() == [0, 0] and tot.tolist() == [0, 1]
    assert (st["blocks_total"], st["blocks_nonzero"], st["blocks_full"]) == (4, 3, 1)
    assert st["block_density"] == 0.75 and st["element_density"] == 10.0 / 16.0


def test_kat_ragged_edges_use_true_area():  # test_mask_model.cpp:109-125
    sums, _, off, tot, _ = oracle.preprocess(words_from_dense(np.ones((5, 5), bool)), 5, 2, 2)
    assert sums.tolist() == [[4, 4, 2], [4, 4, 2], [2, 2, 1]]
    assert off.tolist() == [0, 0, 0] and tot.tolist() == [3, 3, 3]


def test_kat_first_maximal_run_wins():  # test_mask_model.cpp:145-159
    d = np.zeros((16, 16), bool)
    d[0:2, 2:6] = True
    d[0:2, 8:10] = True
    _, _, off, tot, _ = oracle.preprocess(words_from_dense(d), 16, 2, 2)
    assert off[0] == 1 and tot[0] == 2


def test_popcount_range_matches_per_bit():  # test_mask_model.cpp:64-79
    rng = np.random.default_rng(21)
    d = rng.random((130, 130)) < 0.25
    w = words_from_dense(d)
    L = oracle.orc()
    import ctypes as C
    L.orc_popcount_range.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.c_uint64]
    L.orc_popcount_range.restype = C.c_uint32
    for _ in range(200):
        i = int(rng.integers(130))
        a, b = sorted(int(x) for x in rng.integers(0, 131, size=2))
        row = np.ascontiguousarray(w[i])
        got = L.orc_popcount_range(row.ctypes.data_as(C.POINTER(C.c_uint64)), a, b)
        assert got == int(d[i, a:b].sum())


@pytest.mark.parametrize("spec", [(2, 2), (3, 5), (16, 16), (32, 16), (64, 64)])
def test_sums_match_brute_force(spec):  # test_mask_model.cpp:127-143
    bi, bj = spec
    for seed in range(1, 5):
        n = 30 + seed * 25
        d = np.random.default_rng(seed).random((n, n)) < 0.2
        sums = oracle.block_sums(words_from_dense(d), n, bi, bj)
        rows, cols = -(-n // bi), -(-n // bj)
        pad = np.zeros((rows * bi, cols * bj), np.uint32)
        pad[:n, :n] = d
        want = pad.reshape(rows, bi, cols, bj).sum(axis=(1, 3))
        assert np.array_equal(sums, want)


# ------------------------------------------------------------------ counters (test_engine.cpp)

def test_kat_counters_causal_four():  # test_engine.cpp:23-50
    w = causal(4)
    assert oracle.counters(w, 4, 2, 2, 0) == (4, 4, 0, 0, 0)
    assert oracle.counters(w, 4, 2, 2, 1) == (4, 4, 4, 0, 0)
    assert oracle.counters(w, 4, 2, 2, 2) == (4, 3, 3, 1, 0)
    assert oracle.counters(w, 4, 2, 2, 3) == (4, 3, 2, 1, 1)


def test_kat_counters_full_mask_runs():  # test_engine.cpp:52-61
    w = words_from_dense(np.ones((256, 256), bool))
    assert oracle.counters(w, 256, 64, 64, 3) == (16, 16, 0, 0, 16)


def test_kat_causal_256_processes_10_of_16():  # acceptance.cpp:160-168
    assert oracle.counters(causal(256), 256, 64, 64, 2)[1] == 10


# ------------------------------------------------------------------ golden vectors

def load(name):
    path = os.path.join(GOLDEN, name)
    return np.load(path, allow_pickle=False)


def test_mask_model_matches_reference_golden():
    g = load("mask_model.npz")
    for i in range(int(g["count"])):
        n, bi, bj = (int(x) for x in g[f"c{i}_spec"])
        sums, occ, off, tot, st = oracle.preprocess(g[f"c{i}_words"], n, bi, bj)
        ctx = f"{g[f'c{i}_name']} n={n} spec={bi}x{bj}"
        assert np.array_equal(sums, g[f"c{i}_sums"]), ctx
        assert np.array_equal(occ, g[f"c{i}_occ"]), ctx
        assert np.array_equal(off, g[f"c{i}_off"]), ctx
        assert np.array_equal(tot, g[f"c{i}_tot"]), ctx
        assert [st["blocks_total"], st["blocks_nonzero"], st["blocks_full"]] == g[f"c{i}_stats_u"].tolist()
        assert [st["block_density"], st["element_density"]] == g[f"c{i}_stats_f"].tolist()


def test_counters_match_reference_golden():
    g = load("counters.npz")
    for i in range(int(g["count"])):
        n, bi, bj, var, *want = (int(x) for x in g[f"k{i}"])
        assert oracle.counters(g[f"k{i}_words"], n, bi, bj, var) == tuple(want)


def test_naive_forward_matches_reference_golden():
    g = load("forward.npz")
    for name in ("c1", "medusa", "packed"):
        n, d, _ = (int(x) for x in g[f"{name}_meta"])
        q, k, v, _ = oracle.make_problem(1, 1, n, d)
        qb, kb, vb = (oracle.bf16_round(a[0]) for a in (q, k, v))
        out, rmax, rsum = oracle.naive_forward(qb, kb, vb, 1.0 / np.sqrt(d), g[f"{name}_words"], n)
        # reference float engine accumulates in double: ~1e-7 from the double oracle
        assert np.max(np.abs(out - g[f"{name}_out"])) < 1e-6
        assert np.allclose(rmax, g[f"{name}_row_max"], rtol=1e-12, atol=1e-12)
        assert np.allclose(rsum, g[f"{name}_row_sum"], rtol=1e-12)


def test_rcm_matches_reference_golden():
    g = load("rcm.npz")
    for i in range(int(g["count"])):
        words = g[f"r{i}_words"]
        n = words.shape[0]
        fwd = oracle.rcm_order(words, n)
        assert np.array_equal(fwd, g[f"r{i}_fwd"])
        bw0, bw1 = (int(x) for x in g[f"r{i}_bw"])
        assert oracle.bandwidth(words, n) == bw0
        assert oracle.bandwidth(oracle.permute_mask(words, n, fwd), n) == bw1


def test_rcm_kats():  # test_reorder.cpp:109-127, 174-186
    # edgeless 5 -> forward [4,3,2,1,0]
    assert oracle.rcm_order(words_from_dense(np.eye(5, dtype=bool)), 5).tolist() == [4, 3, 2, 1, 0]
    # ring of 8 -> bandwidth 2 after RCM
    d = np.eye(8, dtype=bool)
    for i in range(8):
        d[i, (i + 1) % 8] = True
    w = words_from_dense(d)
    assert oracle.bandwidth(oracle.permute_mask(w, 8, oracle.rcm_order(w, 8)), 8) == 2


# ------------------------------------------------------------------ against the live reference

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built here")


@needs_ref
def test_make_problem_stream_matches_reference():
    q, k, v, do = oracle.make_problem(7, 2, 33, 5)
    rq, rk, rv, rdo = oracle.ref_make_problem_f32(7, 2, 33, 5)
    for a, b in ((q, rq), (k, rk), (v, rv), (do, rdo)):
        assert np.array_equal(a.astype(np.float32), b)


@needs_ref
def test_preprocess_matches_reference_on_large_random():
    words = oracle.ref_generate("random(p=0.3;seed=9)", 1000)
    for bi, bj in ((128, 128), (64, 64), (100, 37)):
        a = oracle.preprocess(words, 1000, bi, bj)
        b = oracle.ref_preprocess(words, 1000, bi, bj)
        for x, y in zip(a[:4], b[:4]):
            assert np.array_equal(x, y)
        assert a[4] == b[4]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("spec,n,d", [("causal", 70, 16), ("packed-seq[20;33;14]", 0, 8), ("random(p=0.2;seed=5;diag=0)", 45, 12)])
def test_naive_backward_matches_reference(spec, n, d):
    # pins the C restatement of naive_backward (reference.hpp:84-139) on the reference itself
    words = oracle.ref_generate(spec, n)
    n = words.shape[0]
    q, k, v, g = (a[0] for a in oracle.make_problem(3, 1, n, d))
    for threads in (1, 3):
        got = oracle.naive_backward(q, k, v, g, 0.37, words, n, threads=threads)
        want = oracle.ref_naive_backward(q, k, v, g, 0.37, words, n)
        for a, b in zip(got, want):
            assert np.allclose(a, b, rtol=1e-12, atol=1e-13)
    # dense = every key visible: the all-ones mask
    got = oracle.naive_backward(q, k, v, g, 0.37, None, n)
    want = oracle.ref_naive_backward(q, k, v, g, 0.37, np.full_like(words, 0) | oracle.ref_generate("all-ones", n), n)
    for a, b in zip(got, want):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-13)


def test_naive_rows_equals_full_oracle():
    # the row-sampled oracle is the full one restricted to the listed rows
    words = oracle.ref_generate("global(w=9;g=2)", 70)
    n = words.shape[0]
    q, k, v, g = (a[0] for a in oracle.make_problem(4, 1, n, 16))
    rows = [0, 1, 5, 33, 69]
    out, rmax, rsum, dq = oracle.naive_rows(q, k, v, 0.3, words, n, rows, d_out=g)
    o2, m2, l2 = oracle.naive_forward(q, k, v, 0.3, words, n, threads=1)
    dq2, _, _ = oracle.naive_backward(q, k, v, g, 0.3, words, n, threads=1)
    assert np.allclose(out, o2[rows], rtol=1e-13, atol=1e-14)
    assert np.allclose(rmax, m2[rows]) and np.allclose(rsum, l2[rows], rtol=1e-13)
    assert np.allclose(dq, dq2[rows], rtol=1e-12, atol=1e-13)
