"""Head dims other than the kernels' 64 / 128 on the B200 (-m gpu).

The reference accepts any positive d_k and an independent d_v (validate_forward_args,
engine.hpp:244-258; EngineForward.ValueHeadDimMayDifferFromKeyDim, test_engine.cpp:198-209). The
sm_100a kernels tile the head dim at 64 or 128, so every entry that takes the caller's layout
(the float host-buffer C ABI, the C++ drop-in, the Python mirror) zero-pads Q/K/V to
kernel_dim(d_k, d_v) on the device and crops the outputs: zero Q/K columns add exact zeros to every
score, zero V / dO columns give output columns that are dropped. Parity: the double oracle at the
same tolerance as the native dims (2e-2 relative); the padded run must also equal an explicitly
zero-padded native run bit for bit. d_v above 128 runs as column passes over V (the forward's
P is the same on every pass; the backward's dq / dk are sums over the passes, dv their
concatenation); d_k above 128 stays rejected (documented narrowing).
"""
import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm

pytestmark = pytest.mark.gpu

TOL = 2e-2
DIMS = [(21, 5, 3), (130, 3, 100), (300, 96, 96), (200, 128, 7), (257, 64, 40), (150, 40, 200), (77, 128, 300)]


def rel_err(got, want):
    return float(np.max(np.abs(np.asarray(got, np.float64) - want))) / max(1.0, float(np.max(np.abs(want))))


def inputs(n, dk, dv, seed, slots=2):
    rng = np.random.default_rng(seed)
    q = oracle.bf16_round(rng.uniform(-1, 1, (slots, n, dk)).astype(np.float32))
    k = oracle.bf16_round(rng.uniform(-1, 1, (slots, n, dk)).astype(np.float32))
    v = oracle.bf16_round(rng.uniform(-1, 1, (slots, n, dv)).astype(np.float32))
    g = oracle.bf16_round(rng.uniform(-1, 1, (slots, n, dv)).astype(np.float32))
    return q, k, v, g


def pad(a, D):
    return np.pad(a, [(0, 0)] * (a.ndim - 1) + [(0, D - a.shape[-1])])


def oracle_backward(q, k, v, g, scale, words, n):
    """naive_backward (reference.hpp:84-139) for d_v != d_k: the C restatement takes one head dim,
    so both sides are zero-padded to max(d_k, d_v) in double (exact) and the gradients cropped."""
    dk, dv = q.shape[1], v.shape[1]
    D = max(dk, dv)
    gq, gk, gv = oracle.naive_backward(pad(q, D), pad(k, D), pad(v, D), pad(g, D), scale, words, n, threads=16)
    return gq[:, :dk], gk[:, :dk], gv[:, :dv]


@pytest.mark.parametrize("n,dk,dv", DIMS)
def test_host_path_any_head_dims_match_oracle(n, dk, dv):
    mask = bbm.gen_random_sparse(n, 0.3, 7, True)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(8, 8))
    q, k, v, g = inputs(n, dk, dv, seed=n + dk)
    scale = 0.4
    for variant in (bbm.Variant.dense, bbm.Variant.binblk, bbm.Variant.dense_binblk, bbm.Variant.naive_masked):
        words = None if variant == bbm.Variant.dense else mask.words
        f = bbm.blocked_forward(q, k, v, scale, mask, prep, variant)
        assert f.out.shape == (2, n, dv)
        for s in range(2):
            want, wmax, _ = oracle.naive_forward(q[s], k[s], v[s], scale, words, n)
            assert rel_err(f.out[s], want) <= TOL, (variant, s)
            fin = np.isfinite(wmax)
            assert np.array_equal(np.isfinite(f.row_max[s]), fin)
            assert np.max(np.abs(f.row_max[s][fin] - wmax[fin])) <= 1e-2 * max(1.0, np.max(np.abs(wmax[fin])))
        b = bbm.blocked_backward(q, k, v, scale, mask, prep, variant, f, g)
        assert b.dq.shape == (2, n, dk) and b.dk.shape == (2, n, dk) and b.dv.shape == (2, n, dv)
        for s in range(2):
            want = oracle_backward(q[s], k[s], v[s], g[s], scale, words, n)
            for name, got, w in zip(("dq", "dk", "dv"), (b.dq[s], b.dk[s], b.dv[s]), want):
                assert rel_err(got, w) <= TOL, (variant, s, name)


@pytest.mark.parametrize("n,dk,dv", DIMS[:3])
def test_padded_run_equals_explicitly_padded_native_run(cuda, n, dk, dv):
    """The padding is exact: the same inputs zero-padded by the caller to the kernel dim give the
    same bits on every output (forward and backward, host and device paths)."""
    import torch

    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
    q, k, v, g = inputs(n, dk, dv, seed=3)
    D = 128 if max(dk, dv) > 64 else 64
    scale = 0.25
    f = bbm.blocked_forward(q, k, v, scale, mask, prep, bbm.Variant.binblk)
    fp = bbm.blocked_forward(pad(q, D), pad(k, D), pad(v, D), scale, mask, prep, bbm.Variant.binblk)
    assert np.array_equal(f.out, fp.out[..., :dv])
    assert np.array_equal(f.row_max, fp.row_max) and np.array_equal(f.row_sum, fp.row_sum)
    b = bbm.blocked_backward(q, k, v, scale, mask, prep, bbm.Variant.binblk, f, g)
    bp = bbm.blocked_backward(pad(q, D), pad(k, D), pad(v, D), scale, mask, prep, bbm.Variant.binblk, fp, pad(g, D))
    assert np.array_equal(b.dq, bp.dq[..., :dk]) and np.array_equal(b.dk, bp.dk[..., :dk])
    assert np.array_equal(b.dv, bp.dv[..., :dv])
    # device path (CUDA bf16 tensors) gives the host path's bits
    dev = lambda a: torch.from_numpy(a).to(cuda).to(torch.bfloat16)  # noqa: E731
    fd = bbm.blocked_forward(dev(q), dev(k), dev(v), scale, mask, prep, bbm.Variant.binblk)
    assert tuple(fd.out.shape) == (2, n, dv)
    assert np.array_equal(fd.out.float().cpu().numpy(), f.out)
    bd = bbm.blocked_backward(dev(q), dev(k), dev(v), scale, mask, prep, bbm.Variant.binblk, fd, dev(g))
    assert tuple(bd.dq.shape) == (2, n, dk) and tuple(bd.dv.shape) == (2, n, dv)
    for got, want in ((bd.dq, b.dq), (bd.dk, b.dk), (bd.dv, b.dv)):
        assert rel_err(got.float().cpu().numpy(), want) <= 1e-3


def test_key_dim_above_128_or_zero_rejected():
    n = 64
    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
    ok = np.zeros((n, 64), np.float32)
    with pytest.raises(ValueError):
        bbm.blocked_forward(np.zeros((n, 129), np.float32), np.zeros((n, 129), np.float32), ok, 0.1, mask, prep,
                            bbm.Variant.binblk)
    # d_v above 128 runs as column passes (test_host_path_any_head_dims_match_oracle); d_k cannot
    f = bbm.blocked_forward(ok, ok, np.ones((n, 200), np.float32), 0.1, mask, prep, bbm.Variant.binblk)
    assert f.out.shape == (n, 200) and np.allclose(f.out, 1.0)
    with pytest.raises(ValueError):
        bbm.blocked_forward(np.zeros((n, 0), np.float32), np.zeros((n, 0), np.float32), ok, 0.1, mask, prep,
                            bbm.Variant.binblk)


def test_device_path_value_dim_above_128(cuda):
    """CUDA bf16 tensors with d_v > 128 (column passes in the Python mirror) agree with the float
    host entries (column passes in the C ABI) and with the oracle."""
    import torch

    n, dk, dv = 300, 64, 200
    mask = bbm.gen_longformer_windowed(n, 50)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
    q, k, v, g = inputs(n, dk, dv, seed=5)
    scale = 0.3
    dev = lambda a: torch.from_numpy(a).to(cuda).to(torch.bfloat16)  # noqa: E731
    f = bbm.blocked_forward(q, k, v, scale, mask, prep, bbm.Variant.binblk)
    fd = bbm.blocked_forward(dev(q), dev(k), dev(v), scale, mask, prep, bbm.Variant.binblk)
    assert tuple(fd.out.shape) == (2, n, dv)
    assert np.array_equal(fd.out.float().cpu().numpy(), f.out)
    b = bbm.blocked_backward(q, k, v, scale, mask, prep, bbm.Variant.binblk, f, g)
    bd = bbm.blocked_backward(dev(q), dev(k), dev(v), scale, mask, prep, bbm.Variant.binblk, fd, dev(g))
    for got, want in ((bd.dq, b.dq), (bd.dk, b.dk), (bd.dv, b.dv)):
        assert tuple(got.shape) == want.shape
        assert rel_err(got.float().cpu().numpy(), want) <= 1e-2
    for s in range(2):
        want = oracle_backward(q[s], k[s], v[s], g[s], scale, mask.words, n)
        for got, w in zip((b.dq[s], b.dk[s], b.dv[s]), want):
            assert rel_err(got, w) <= TOL
