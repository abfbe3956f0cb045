"""The two-stream forward kernel (attn_fwd_pair.cu) on the B200 (-m gpu).

It must reproduce the single-stream kernel (attn_fwd.cu) bit for bit wherever that kernel splits
no row (outputs and row statistics, every variant), and match the double oracle
(reference.hpp:42-81) within the north-star tolerance. Masks cover the list shapes the merged
K/V schedule has to handle: identical adjacent lists (dense, causal), shifted lists (bands),
disjoint lists (packed sequences), an odd number of row tiles (last pair with one row), fully
masked row tiles and ragged n.
"""
import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm

pytestmark = pytest.mark.gpu


def _inputs(cuda, slots, n, d, seed):
    import torch

    g = torch.Generator(device=cuda).manual_seed(seed)
    return tuple((torch.rand((slots, n, d), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16) for _ in range(3))


def _run(prep, var, q, k, v, scale, mode):
    import torch

    bbm.set_fwd_kernel(mode)
    try:
        slots, n, _ = q.shape
        out = torch.empty_like(q)
        m = torch.empty((slots, n), dtype=torch.float32, device=q.device)
        l = torch.empty_like(m)
        bbm.attn_fwd_device(prep, var, q, k, v, out, m, l, scale)
        torch.cuda.synchronize()
        return out, m, l
    finally:
        bbm.set_fwd_kernel("auto")


def _masks():
    fully_masked = bbm.gen_packed_sequential([300, 200, 500])
    w = fully_masked.words.copy()
    w[128:256] = 0  # row tile 1 sees nothing
    return [
        ("causal", bbm.gen_causal(1024)),
        ("band", bbm.gen_longformer_windowed(1500, 90)),
        ("packed", bbm.gen_packed_sequential([100, 260, 37, 243, 512, 90, 330])),
        ("global", bbm.generate("global(w=64;g=20)", 1408)),
        ("random", bbm.generate("random(p=0.02;seed=5)", 896)),
        ("odd_rows", bbm.gen_causal(640)),
        ("masked_tile", bbm.Mask(1000, w)),
    ]


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("name,mask", _masks(), ids=[m[0] for m in _masks()])
def test_pair_kernel_bitwise_equals_single_stream(cuda, name, mask, d):
    n = mask.size()
    slots = 3
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = _inputs(cuda, slots, n, d, n + d)
    for var in bbm.Variant:
        ref = _run(prep, var, q, k, v, d ** -0.5, "single")
        got = _run(prep, var, q, k, v, d ** -0.5, "pair")
        for a, b, what in zip(got, ref, ("out", "row_max", "row_sum")):
            import torch

            view = torch.int16 if a.dtype == torch.bfloat16 else torch.int32
            assert torch.equal(a.view(view), b.view(view)), f"{name} d={d} {var.name}: {what} differs"


@pytest.mark.parametrize("name,mask", _masks()[:4], ids=[m[0] for m in _masks()[:4]])
def test_pair_kernel_matches_oracle(cuda, name, mask):
    import torch

    n, d, slots = mask.size(), 128, 2
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v, _ = oracle.make_problem(11, slots, n, d)
    q, k, v = (oracle.bf16_round(a) for a in (q, k, v))
    t = [torch.from_numpy(a.astype(np.float32)).to(cuda).to(torch.bfloat16) for a in (q, k, v)]
    out, rmax, rsum = _run(prep, bbm.Variant.binblk, *t, d ** -0.5, "pair")
    out = out.float().cpu().numpy()
    rmax, rsum = rmax.cpu().numpy(), rsum.cpu().numpy()
    for s in range(slots):
        o, m, l = oracle.naive_forward(q[s], k[s], v[s], d ** -0.5, mask.words, n, threads=16)
        assert float(np.abs(out[s] - o).max()) <= 2e-2
        fin = np.isfinite(m)
        assert np.array_equal(fin, np.isfinite(rmax[s]))
        assert np.allclose(rmax[s][fin], m[fin], rtol=1e-2, atol=1e-2)
        assert np.allclose(rsum[s][fin], l[fin], rtol=1e-2)


def test_pair_kernel_negative_and_zero_scale(cuda):
    """Sentinel handling under a negative scale and the zero-scale substitute (same as the
    single-stream kernel)."""
    mask = bbm.gen_longformer_windowed(777, 50)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = _inputs(cuda, 2, 777, 128, 3)
    import torch

    for scale in (-0.3, 0.0):
        ref = _run(prep, bbm.Variant.binblk, q, k, v, scale, "single")
        got = _run(prep, bbm.Variant.binblk, q, k, v, scale, "pair")
        for a, b in zip(got, ref):
            view = torch.int16 if a.dtype == torch.bfloat16 else torch.int32
            assert torch.equal(a.view(view), b.view(view))


def test_default_selection_is_the_single_stream_kernel(cuda):
    """The default forward is attn_fwd.cu; selecting "pair" changes which kernel runs, not the bits."""
    import torch

    mask = bbm.gen_longformer_windowed(2048, 200)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = _inputs(cuda, 8, 2048, 128, 9)
    first = _run(prep, bbm.Variant.binblk, q, k, v, 0.09, "auto")
    for mode in ("single", "pair", "auto"):
        again = _run(prep, bbm.Variant.binblk, q, k, v, 0.09, mode)
        for a, b in zip(again, first):
            view = torch.int16 if a.dtype == torch.bfloat16 else torch.int32
            assert torch.equal(a.view(view), b.view(view)), mode
