"""BASELINE configurations at FULL size on the B200 (-m gpu).

The double oracle cannot run whole full-size problems in seconds, so these tests use what stays
cheap at any size: (1) sampled query rows checked against the row-restricted oracle
(oracle.naive_rows, reference.hpp:42-139 restated per row — pinned on the full oracle in
test_oracle.py), including each config's first / last / ragged rows; (2) size-independent
properties: run-to-run determinism, masked variants bitwise identical (test_engine.cpp:112-134),
and for the backward the identities  sum_j dV_j = sum_i dO_i  over rows with a visible key (the
rows of P sum to one) and  sum_j dK_j = 0  (the rows of dS sum to zero).
Tolerances: outputs max-abs 2e-2; dq relative max-abs 2e-2; the identities 2e-2 relative to
max(|reference side|, sqrt(n)).
"""
import numpy as np
import pytest

import bench
import oracle
import paper_2409_15097_b200 as bbm

pytestmark = pytest.mark.gpu

TOL = 2e-2


def inputs(slots, n, d, dev, seed):
    import torch

    g = torch.Generator(device=dev).manual_seed(seed)
    return [(torch.rand((slots, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(4)]


def sample_rows(n, extra=()):
    rng = np.random.default_rng(n)
    rows = set(rng.choice(n, size=min(n, 24), replace=False).tolist())
    rows |= {0, 1, n - 1, n // 2} | {r for r in extra if 0 <= r < n}
    return sorted(rows)


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_forward_full_size_sampled_rows(cuda, cfg):
    import torch

    mask, B, H, d, _ = bench.make_config(cfg)
    variant = bbm.Variant.dense_binblk if cfg == "c4" else bbm.Variant.binblk
    n, slots = mask.size(), B * H
    prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(cuda), bbm.BlockSpec(128, 128))
    q, k, v, _ = inputs(slots, n, d, cuda, 5)
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=cuda)
    rsum = torch.empty_like(rmax)
    bbm.attn_fwd_device(prep, variant, q, k, v, out, rmax, rsum, d ** -0.5)
    out2 = torch.empty_like(q)
    bbm.attn_fwd_device(prep, variant, q, k, v, out2, None, None, d ** -0.5)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)  # deterministic at full size
    rows = sample_rows(n, extra=(127, 128, 2047, 2048, 16383))
    for s in (0, slots - 1):
        o, m, l, _ = oracle.naive_rows(host(q[s]), host(k[s]), host(v[s]), d ** -0.5, mask.words, n, rows)
        got = host(out[s])[rows]
        assert float(np.abs(got - o).max()) <= TOL, f"{cfg} slot {s}"
        fin = np.isfinite(m)
        gm, gl = host(rmax[s])[rows], host(rsum[s])[rows]
        assert np.array_equal(fin, np.isfinite(gm))
        assert np.allclose(gm[fin], m[fin], rtol=1e-2, atol=1e-2) and np.allclose(gl[fin], l[fin], rtol=1e-2)


def test_masked_variants_bitwise_identical_full_c2(cuda):
    import torch

    mask, B, H, d, _ = bench.make_config("c2")
    n, slots = mask.size(), 16
    prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(cuda), bbm.BlockSpec(128, 128))
    q, k, v, _ = inputs(slots, n, d, cuda, 6)
    outs = []
    for var in (bbm.Variant.naive_masked, bbm.Variant.binblk, bbm.Variant.dense_binblk):
        o = torch.empty_like(q)
        bbm.attn_fwd_device(prep, var, q, k, v, o, None, None, d ** -0.5)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_backward_full_size_rows_and_identities(cuda, cfg):
    import torch

    mask, B, H, d, _ = bench.make_config(cfg)
    variant = bbm.Variant.dense_binblk if cfg == "c4" else bbm.Variant.binblk
    n, slots = mask.size(), min(B * H, 8)
    prep = bbm.preprocess_mask(torch.from_numpy(mask.to_dense()).to(cuda), bbm.BlockSpec(128, 128))
    q, k, v, g = inputs(slots, n, d, cuda, 7)
    out = torch.empty_like(q)
    rmax = torch.empty((slots, n), dtype=torch.float32, device=cuda)
    rsum = torch.empty_like(rmax)
    bbm.attn_fwd_device(prep, variant, q, k, v, out, rmax, rsum, d ** -0.5)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    bbm.attn_bwd_device(prep, variant, q, k, v, out, rmax, rsum, g, dq, dk, dv, d ** -0.5)
    dq2, dk2, dv2 = (torch.empty_like(q) for _ in range(3))
    bbm.attn_bwd_device(prep, variant, q, k, v, out, rmax, rsum, g, dq2, dk2, dv2, d ** -0.5)
    torch.cuda.synchronize()
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)  # deterministic
    rows = sample_rows(n)
    has_key = mask.to_dense().any(axis=1)
    for s in (0, slots - 1):
        _, _, _, want = oracle.naive_rows(host(q[s]), host(k[s]), host(v[s]), d ** -0.5, mask.words, n, rows,
                                          d_out=host(g[s]))
        got = host(dq[s])[rows]
        assert float(np.abs(got - want).max()) <= TOL * max(1.0, float(np.abs(want).max())), f"{cfg} dq slot {s}"
        # identities over the whole slot
        sdv = host(dv[s]).sum(0)
        sdo = host(g[s])[has_key].sum(0)
        scale_ref = max(float(np.abs(sdo).max()), np.sqrt(n))
        assert float(np.abs(sdv - sdo).max()) <= TOL * scale_ref, f"{cfg} sum dV slot {s}"
        sdk = host(dk[s]).sum(0)
        assert float(np.abs(sdk).max()) <= TOL * max(float(np.abs(host(dk[s])).sum(0).max()) / np.sqrt(n), 1.0), \
            f"{cfg} sum dK slot {s}"


@pytest.mark.parametrize("mode", [2, 3, 4])
def test_full_c5_rcm_gather_modes_bitwise(cuda, mode):
    """f2 at the headline size: the C5 forward (bench.py's RCM-reordered mask and its permutation)
    on ORIGINAL-order inputs with the RCM permutation
    applied on the device (in-kernel TMA gather, hybrid, in-kernel LSU gather) equals the forward
    on pre-permuted inputs scattered back, bit for bit, on every slot — three launches each (the
    LSU mode's cp.async gathers hand shared memory to tcgen05 through mbarrier + proxy fence; a
    missing ordering would show here as sporadic differences)."""
    import torch

    words, fwd_perm = bench.mask_words("c5", *bench.bbm_backends(bbm, 0))  # the RCM-reordered mask
    _, _, d, _, _, n = bench.CONFIGS["c5"]
    prep = bbm.preprocess_mask(bbm.Mask(n, words), bbm.BlockSpec(128, 128))
    slots = 16  # 16 of C5's 128 slots: the full per-slot size, a bounded test time
    q, k, v, _ = inputs(slots, n, d, cuda, 7)
    fwd = torch.from_numpy(np.ascontiguousarray(fwd_perm, dtype=np.int64)).to(cuda)
    rows = fwd.to(torch.int32)
    qp, kp, vp = (t[:, fwd].contiguous() for t in (q, k, v))  # row a <- token forward[a]
    op = torch.empty_like(qp)
    mp = torch.empty((slots, n), dtype=torch.float32, device=cuda)
    bbm.attn_fwd_device(prep, bbm.Variant.binblk, qp, kp, vp, op, mp, None, d ** -0.5)
    want_o = torch.empty_like(op)
    want_o[:, fwd] = op
    want_m = torch.empty_like(mp)
    want_m[:, fwd] = mp
    for _ in range(3):
        out = torch.empty_like(q)
        m = torch.empty_like(mp)
        bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k, v, out, m, None, d ** -0.5, rows=rows, gather_mode=mode)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), want_o.view(torch.int16))
        assert torch.equal(m.view(torch.int32), want_m.view(torch.int32))
