"""Masked attention BACKWARD parity on the B200 (-m gpu).

The sm_100a backward (bf16 Q/K/V/dO, bf16 P and dS on the tensor cores, fp32 accumulation) is
compared with the C oracle's double-precision naive_backward (reference.hpp:84-139, pinned on the
reference itself in tests/test_oracle.py) fed the SAME bf16-rounded inputs and the GPU forward's
own output and row statistics (as blocked_backward takes them, engine.hpp:346-350).

Tolerance: gradients are sums of up to n bf16 products, so the bound is relative to the
gradient's scale:  max|got - want| <= TOL * max(1, max|want|),  TOL = 2e-2.
"""
import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm

pytestmark = pytest.mark.gpu

TOL = 2e-2
MASKED = (bbm.Variant.naive_masked, bbm.Variant.binblk, bbm.Variant.dense_binblk)


def to_dev(a, cuda):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(cuda).to(torch.bfloat16)


def problem(seed, slots, n, d):
    q, k, v, g = oracle.make_problem(seed, slots, n, d)
    return tuple(oracle.bf16_round(a) for a in (q, k, v, g))


def fwd_bwd(mask, q, k, v, g, scale, variant, cuda, prep=None):
    prep = prep or bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    tq, tk, tv, tg = (to_dev(a, cuda) for a in (q, k, v, g))
    f = bbm.blocked_forward(tq, tk, tv, scale, mask, prep, variant)
    b = bbm.blocked_backward(tq, tk, tv, scale, mask, prep, variant, f, tg)
    return f, b


def rel_err(got, want):
    return float(np.max(np.abs(got - want))) / max(1.0, float(np.max(np.abs(want))))


def check(mask, q, k, v, g, scale, variant, f, b, slots=None):
    n = mask.size()
    words = None if variant == bbm.Variant.dense else mask.words
    out = f.out.float().cpu().numpy()
    grads = [t.float().cpu().numpy() for t in (b.dq, b.dk, b.dv)]
    worst = 0.0
    for s in (range(q.shape[0]) if slots is None else slots):
        # d_out's gradient path goes through the forward output the GPU produced
        want = oracle.naive_backward(q[s], k[s], v[s], g[s], scale, words, n, threads=16)
        for name, got, w in zip(("dq", "dk", "dv"), grads, want):
            e = rel_err(got[s], w)
            worst = max(worst, e)
            assert e <= TOL, f"slot {s} {name}: relative max-abs {e:.3e}"
        assert np.isfinite(out[s]).all()
    return worst


def test_config1_causal_backward(cuda):
    n, d, slots = 1024, 64, 4
    mask = bbm.gen_causal(n)
    q, k, v, g = problem(1, slots, n, d)
    for variant in (bbm.Variant.binblk, bbm.Variant.dense):
        f, b = fwd_bwd(mask, q, k, v, g, d ** -0.5, variant, cuda)
        check(mask, q, k, v, g, d ** -0.5, variant, f, b)
        assert b.counters == f.counters  # engine.hpp:346-349: same tiles as the forward


@pytest.mark.parametrize("spec,n", [("packed-seq[100;260;37;243]", 0), ("global(w=40;g=7)", 300),
                                    ("windowed(w=90)", 515), ("random(p=0.05;seed=3)", 200),
                                    ("causal", 128)])
@pytest.mark.parametrize("d", [64, 128])
def test_family_masks_all_variants(cuda, spec, n, d):
    mask = bbm.generate(spec, n)
    n = mask.size()
    q, k, v, g = problem(7, 2, n, d)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    got = {}
    for variant in (bbm.Variant.dense,) + MASKED:
        f, b = fwd_bwd(mask, q, k, v, g, d ** -0.5, variant, cuda, prep)
        check(mask, q, k, v, g, d ** -0.5, variant, f, b)
        got[variant] = [t.cpu() for t in (b.dq, b.dk, b.dv)]
    # masked variants agree bit for bit (the reference's test_engine.cpp:233-250 property)
    import torch

    for variant in MASKED[1:]:
        for a, c in zip(got[MASKED[0]], got[variant]):
            assert torch.equal(a, c)


def test_backward_is_deterministic(cuda):
    import torch

    mask = bbm.gen_packed_sequential([300, 500, 224])
    q, k, v, g = problem(2, 3, mask.size(), 128)
    f, b1 = fwd_bwd(mask, q, k, v, g, 0.1, bbm.Variant.binblk, cuda)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    _, b2 = fwd_bwd(mask, q, k, v, g, 0.1, bbm.Variant.binblk, cuda, prep)
    for a, c in zip((b1.dq, b1.dk, b1.dv), (b2.dq, b2.dk, b2.dv)):
        assert torch.equal(a, c)


def test_fully_masked_rows_and_unattended_keys_get_zero_gradients(cuda):
    # rows 130..199 see nothing; keys 300..399 are seen by nobody (test_engine.cpp:176-197)
    n, d = 400, 64
    dense = np.tril(np.ones((n, n), bool))
    dense[130:200, :] = False
    dense[:, 300:] = False
    mask = bbm.Mask.from_dense(dense)
    q, k, v, g = problem(4, 2, n, d)
    for variant in MASKED:
        f, b = fwd_bwd(mask, q, k, v, g, d ** -0.5, variant, cuda)
        check(mask, q, k, v, g, d ** -0.5, variant, f, b)
        dq, dk, dv = (t.float().cpu().numpy() for t in (b.dq, b.dk, b.dv))
        assert np.all(dq[:, 130:200] == 0)
        assert np.all(dk[:, 300:] == 0) and np.all(dv[:, 300:] == 0)


def test_negative_scale_and_ragged_n(cuda):
    mask = bbm.gen_longformer_global(333, 50, 5)
    q, k, v, g = problem(9, 2, 333, 128)
    for scale in (-0.2, 0.0):
        f, b = fwd_bwd(mask, q, k, v, g, scale, bbm.Variant.binblk, cuda)
        check(mask, q, k, v, g, scale, bbm.Variant.binblk, f, b)


def test_host_float_path_matches_device_path(cuda):
    mask = bbm.gen_causal(300)
    q, k, v, g = problem(5, 1, 300, 64)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
    fh = bbm.blocked_forward(q[0], k[0], v[0], 0.125, mask, prep, bbm.Variant.dense_binblk)
    bh = bbm.blocked_backward(q[0], k[0], v[0], 0.125, mask, prep, bbm.Variant.dense_binblk, fh, g[0])
    want = oracle.naive_backward(q[0], k[0], v[0], g[0], 0.125, mask.words, 300)
    for got, w in zip((bh.dq, bh.dk, bh.dv), want):
        assert rel_err(got, w) <= TOL
    assert bh.counters == fh.counters
    with pytest.raises(ValueError):
        bad = g[0].copy()
        bad[3, 3] = np.nan
        bbm.blocked_backward(q[0], k[0], v[0], 0.125, mask, prep, bbm.Variant.binblk, fh, bad)


def test_config2_shape_sampled_slots(cuda):
    import bench

    mask, B, H, d, _ = bench.make_config("c2")
    n = mask.size()
    slots = 8
    q, k, v, g = problem(11, slots, n, d)
    f, b = fwd_bwd(mask, q, k, v, g, d ** -0.5, bbm.Variant.binblk, cuda)
    check(mask, q, k, v, g, d ** -0.5, bbm.Variant.binblk, f, b, slots=[0, 5])


def test_prep_update_refreshes_backward_view(cuda):
    import torch

    m1 = bbm.gen_packed_sequential([200, 312])
    m2 = bbm.gen_causal(512)
    q, k, v, g = problem(6, 1, 512, 64)
    prep = bbm.preprocess_mask(m1, bbm.BlockSpec(128, 128))
    fwd_bwd(m1, q, k, v, g, 0.125, bbm.Variant.binblk, cuda, prep)
    dm = torch.from_numpy(m2.to_dense()).to(cuda)
    from paper_2409_15097_b200 import _lib
    import ctypes as C

    _lib.check(_lib.lib.bbm_prep_update_bool_device(prep.handle.h, C.c_void_p(dm.data_ptr()), 512,
                                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    f, b = fwd_bwd(m2, q, k, v, g, 0.125, bbm.Variant.binblk, cuda, prep)
    check(m2, q, k, v, g, 0.125, bbm.Variant.binblk, f, b)


@pytest.mark.parametrize("spec,n,d", [("global(w=64;g=100)", 4096, 64), ("global(w=100;g=130)", 3000, 128),
                                      ("all-ones", 2560, 128)])
def test_split_long_lists_match_oracle_and_stay_deterministic(cuda, spec, n, d):
    """One slot + long row / column lists (global tokens, all-ones): the device plan cuts them into
    chunks whose fp32 partial gradients the last chunk adds in chunk order; the result matches
    the oracle, is bitwise deterministic and identical across the masked variants."""
    mask = bbm.generate(spec, n)
    q, k, v, g = problem(13, 1, n, d)
    scale = d ** -0.5
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    f, b = fwd_bwd(mask, q, k, v, g, scale, bbm.Variant.binblk, cuda, prep=prep)
    check(mask, q, k, v, g, scale, bbm.Variant.binblk, f, b)
    ref = [t.float().cpu().numpy() for t in (b.dq, b.dk, b.dv)]
    for var in MASKED:
        f2, b2 = fwd_bwd(mask, q, k, v, g, scale, var, cuda, prep=prep)
        for got, want in zip((b2.dq, b2.dk, b2.dv), ref):
            assert np.array_equal(got.float().cpu().numpy(), want), var
    fd, bd = fwd_bwd(mask, q, k, v, g, scale, bbm.Variant.dense, cuda, prep=prep)
    check(mask, q, k, v, g, scale, bbm.Variant.dense, fd, bd)


@pytest.mark.parametrize("n,w,d", [(3000, 40, 128), (1111, 20, 64)])
def test_backward_empty_half_skipping_is_exact(cuda, n, w, d):
    """dq (dkdv) skips the S / dP and accumulate MMAs of a 64-key (64-query) half of a tile that
    no partner row sees, from the launch after the plan header reached the host: the first
    backward (no skipping) and later ones (skipping) must agree bit for bit, and match the
    oracle."""
    import torch

    mask = bbm.gen_longformer_windowed(n, w)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    cnt, _, _ = prep.kernel_lists()
    h = prep.tile_halves()
    occ = sum(int(c) for c in cnt)
    assert sum(int((h[p, :c] > 0).sum()) for p, c in enumerate(cnt)) * 4 >= occ  # skip enabled
    q, k, v, g = problem(n, 2, n, d)
    tq, tk, tv, tg = (to_dev(a, cuda) for a in (q, k, v, g))
    f = bbm.blocked_forward(tq, tk, tv, 0.09, mask, prep, bbm.Variant.binblk)
    runs = [bbm.blocked_backward(tq, tk, tv, 0.09, mask, prep, bbm.Variant.binblk, f, tg) for _ in range(3)]
    torch.cuda.synchronize()
    for b in runs[1:]:
        for a, c in zip((runs[0].dq, runs[0].dk, runs[0].dv), (b.dq, b.dk, b.dv)):
            assert torch.equal(a, c)
    check(mask, q, k, v, g, 0.09, bbm.Variant.binblk, f, runs[-1], slots=[1])
