"""Masked attention forward parity on the B200 (-m gpu).

The sm_100a kernel (bf16 inputs, bf16 P, fp32 accumulation) is compared with the C oracle's
double-precision naive_forward (reference.hpp:42-81) fed the SAME bf16-rounded inputs.
Tolerance (north star): max-abs <= 2e-2 on outputs; row_max / row_sum relative 1e-2.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL_OUT = 2e-2
TOL_STAT = 1e-2
MASKED = (bbm.Variant.naive_masked, bbm.Variant.binblk, bbm.Variant.dense_binblk)


def problem(seed, slots, n, d):
    q, k, v, _ = oracle.make_problem(seed, slots, n, d)
    return tuple(oracle.bf16_round(a) for a in (q, k, v))


def to_dev(a, cuda):
    import torch

    return torch.from_numpy(a.astype(np.float32)).to(cuda).to(torch.bfloat16)


def run_gpu(mask, q, k, v, scale, variant, cuda, spec=bbm.BlockSpec(128, 128), prep=None):
    prep = prep or bbm.preprocess_mask(mask, spec)
    r = bbm.blocked_forward(to_dev(q, cuda), to_dev(k, cuda), to_dev(v, cuda), scale, mask, prep, variant)
    return (r.out.float().cpu().numpy(), r.row_max.cpu().numpy(), r.row_sum.cpu().numpy(), r.counters)


def check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, variant, slots_to_check=None):
    n = mask.size()
    slots = q.shape[0]
    idx = range(slots) if slots_to_check is None else slots_to_check
    words = None if variant == bbm.Variant.dense else mask.words
    worst = 0.0
    for s in idx:
        o, m, l = oracle.naive_forward(q[s], k[s], v[s], scale, words, n, threads=16)
        err = float(np.max(np.abs(out[s] - o)))
        worst = max(worst, err)
        assert err <= TOL_OUT, f"slot {s}: max-abs {err}"
        fin = np.isfinite(m)
        assert np.array_equal(fin, np.isfinite(rmax[s])), "fully-masked rows differ"
        assert np.all(rmax[s][~fin] == -np.inf) and np.all(rsum[s][~fin] == 0)
        assert np.all(out[s][~fin] == 0)
        assert np.allclose(rmax[s][fin], m[fin], rtol=TOL_STAT, atol=TOL_STAT)
        assert np.allclose(rsum[s][fin], l[fin], rtol=TOL_STAT)
    return worst


def test_config1_causal_b1_h4_n1024_d64(cuda):
    """BASELINE config 1: causal, B=1 H=4 N=1024 d=64, all four variants."""
    mask = bbm.gen_causal(1024)
    q, k, v = problem(1, 4, 1024, 64)
    scale = 1 / 8.0
    for var in bbm.Variant:
        out, rmax, rsum, c = run_gpu(mask, q, k, v, scale, var, cuda)
        err = check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, var)
        assert err < 5e-3  # expected ~3e-3 for bf16 P
    assert c.blocks_processed == 4 * 36  # 36 of 64 tiles at 128x128


def test_forward_matches_reference_golden(cuda):
    g = np.load(os.path.join(GOLDEN, "forward.npz"))
    for name in ("c1", "medusa", "packed"):
        n, d, _ = (int(x) for x in g[f"{name}_meta"])
        mask = bbm.Mask(n, g[f"{name}_words"])
        q, k, v = problem(1, 1, n, d)
        out, rmax, rsum, c = run_gpu(mask, q, k, v, 1 / np.sqrt(d), bbm.Variant.binblk, cuda)
        assert np.max(np.abs(out[0] - g[f"{name}_out"])) <= TOL_OUT, name
        fin = np.isfinite(g[f"{name}_row_max"])
        assert np.allclose(rmax[0][fin], g[f"{name}_row_max"][fin], rtol=TOL_STAT, atol=TOL_STAT)
        assert np.allclose(rsum[0][fin], g[f"{name}_row_sum"][fin], rtol=TOL_STAT)
        assert [c.blocks_visited, c.blocks_processed, c.mask_block_reads, c.skipped_by_binblk,
                c.skipped_mask_reads_by_run] == g[f"{name}_counters"].tolist()


FAMILY = ["causal", "all-ones", "windowed(w={w8})", "windowed(w={w8};causal=1)", "dilated(w={w16};d=2)",
          "global(w={w8};g=4)", "random(p=0.05;seed=17)", "random(p=0.4;seed=18)"]


@pytest.mark.parametrize("n", [128, 200, 256, 700])
@pytest.mark.parametrize("d", [64, 128])
def test_family_masks_all_variants(cuda, n, d):
    q, k, v = problem(n, 2, n, d)
    scale = 1 / np.sqrt(d)
    for tmpl in FAMILY:
        spec = tmpl.format(w8=max(1, n // 8), w16=max(1, n // 16))
        mask = bbm.generate(spec, n)
        for var in bbm.Variant:
            out, rmax, rsum, _ = run_gpu(mask, q, k, v, scale, var, cuda)
            check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, var)


@pytest.mark.parametrize("spec,n", [("packed-seq[{a};{b}]", 300), ("packed-bidir[{a}:{a};{a}:{b}]", 515),
                                    ("medusa[4;4;4;4]", 0), ("medusa[8;7]", 0)])
def test_packed_and_tree_masks(cuda, spec, n):
    s = spec.format(a=n // 4, b=n - 3 * (n // 4)) if n else spec
    mask = bbm.generate(s, n)
    N = mask.size()
    q, k, v = problem(3, 2, N, 128)
    for var in MASKED:
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, 0.088, var, cuda)
        check_against_oracle(mask, q, k, v, 0.088, out, rmax, rsum, var)


def test_masked_variants_bitwise_identical_and_deterministic(cuda):
    """test_engine.cpp:112-134 on the GPU: the masked variants share one tile kernel, so their
    outputs are bitwise equal; repeated calls are bitwise equal (no atomics)."""
    for spec, n in (("random(p=0.3;seed=4)", 333), ("global(w=40;g=5)", 512), ("causal", 384)):
        mask = bbm.generate(spec, n)
        q, k, v = problem(11, 3, n, 64)
        prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
        base = run_gpu(mask, q, k, v, 0.125, bbm.Variant.naive_masked, cuda, prep=prep)
        for var in (bbm.Variant.binblk, bbm.Variant.dense_binblk, bbm.Variant.binblk):
            r = run_gpu(mask, q, k, v, 0.125, var, cuda, prep=prep)
            assert np.array_equal(r[0], base[0]), (spec, var)
            assert np.array_equal(r[1], base[1]) and np.array_equal(r[2], base[2])


def test_all_variants_agree_bitwise_on_full_mask(cuda):  # test_engine.cpp:136-148
    mask = bbm.gen_all_ones(384)
    q, k, v = problem(9, 2, 384, 128)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    base = run_gpu(mask, q, k, v, 0.1, bbm.Variant.dense, cuda, prep=prep)
    for var in MASKED:
        r = run_gpu(mask, q, k, v, 0.1, var, cuda, prep=prep)
        assert np.array_equal(r[0], base[0]) and np.array_equal(r[2], base[2])


def test_fully_masked_rows_produce_zero_rows(cuda):  # test_engine.cpp:176-197
    n = 300
    mask = bbm.gen_random_sparse(n, 0.2, 11)
    for i in (5, 20, 129, 299):
        for j in range(n):
            mask.set(i, j, False)
    # and a whole 128-row tile with no ones: empty tile list
    for i in range(128, 256):
        for j in range(n):
            mask.set(i, j, False)
    q, k, v = problem(12, 2, n, 64)
    for var in MASKED:
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, 0.2, var, cuda)
        check_against_oracle(mask, q, k, v, 0.2, out, rmax, rsum, var)
        for i in (5, 20, 150, 299):
            assert rsum[0, i] == 0 and rmax[0, i] == -np.inf and np.all(out[0, i] == 0)


def test_tiny_and_ragged_shapes(cuda):  # test_engine.cpp:387-405
    for n in (1, 15, 100, 129):
        mask = bbm.gen_causal(n)
        q, k, v = problem(22, 1, n, 64)
        for spec in (bbm.BlockSpec(64, 64), bbm.BlockSpec(128, 32)):
            out, rmax, rsum, c = run_gpu(mask, q, k, v, 0.3, bbm.Variant.dense_binblk, cuda, spec=spec)
            check_against_oracle(mask, q, k, v, 0.3, out, rmax, rsum, bbm.Variant.dense_binblk)
            assert c.blocks_visited == (-(-n // spec.block_i)) * (-(-n // spec.block_j))


def test_negative_and_zero_scale(cuda):
    mask = bbm.gen_longformer_windowed(256, 20)
    q, k, v = problem(5, 1, 256, 64)
    for scale in (-0.3, 0.0, 2.5):
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, scale, bbm.Variant.binblk, cuda)
        check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, bbm.Variant.binblk)


def test_validation_errors(cuda):  # test_engine.cpp:349-385
    import torch

    n = 256
    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = (to_dev(a, cuda) for a in problem(21, 1, n, 64))
    bad = q.clone()
    bad[0, 3, 2] = float("nan")
    with pytest.raises(ValueError):
        bbm.blocked_forward(bad, k, v, 0.1, mask, prep, bbm.Variant.binblk)
    with pytest.raises(ValueError):
        bbm.blocked_forward(q, k, v, float("inf"), mask, prep, bbm.Variant.binblk)
    with pytest.raises(ValueError):
        bbm.blocked_forward(q, k, v, 0.1, mask, prep, bbm.Variant.binblk, threads=0)
    wrong = bbm.preprocess_mask(bbm.gen_causal(n + 8), bbm.BlockSpec(128, 128))
    with pytest.raises(ValueError):
        bbm.blocked_forward(q, k, v, 0.1, mask, wrong, bbm.Variant.binblk)
    with pytest.raises(ValueError):
        bbm.blocked_forward(q[:, :-1], k, v, 0.1, mask, prep, bbm.Variant.binblk)
    with pytest.raises(ValueError):  # documented narrowing: d <= 128 (smaller dims run padded)
        z = torch.zeros((1, n, 160), dtype=torch.bfloat16, device=cuda)
        bbm.blocked_forward(z, z, z, 0.1, mask, prep, bbm.Variant.binblk)
    with pytest.raises(ValueError):
        bbm.run_attention([], 0.1, mask, prep, bbm.Variant.binblk)


def test_host_float_path_equals_device_path(cuda):
    mask = bbm.gen_longformer_global(500, 60, 3)
    q, k, v = problem(30, 1, 500, 128)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    dev = run_gpu(mask, q, k, v, 0.09, bbm.Variant.binblk, cuda, prep=prep)
    host = bbm.blocked_forward(q[0].astype(np.float32), k[0].astype(np.float32), v[0].astype(np.float32),
                               0.09, mask, prep, bbm.Variant.binblk)
    assert np.array_equal(host.out, dev[0][0])
    assert np.array_equal(host.row_sum.astype(np.float32), dev[2][0].astype(np.float32))


def test_run_attention_equals_per_slot(cuda):  # test_engine.cpp:323-347
    n = 256
    mask = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = problem(100, 4, n, 64)
    slots = [bbm.SlotInputs(to_dev(q[s], cuda), to_dev(k[s], cuda), to_dev(v[s], cuda)) for s in range(4)]
    multi = bbm.run_attention(slots, 0.125, mask, prep, bbm.Variant.binblk)
    total = bbm.EngineCounters()
    for s in range(4):
        single = bbm.blocked_forward(slots[s].q, slots[s].k, slots[s].v, 0.125, mask, prep, bbm.Variant.binblk)
        assert np.array_equal(multi.slots[s].out.float().cpu().numpy(), single.out.float().cpu().numpy())
        total += single.counters
    assert multi.counters == total


def test_multi_gpu_driver_single_device(cuda):
    import torch

    n = 512
    mask = bbm.gen_longformer_windowed(n, 100)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v = problem(8, 6, n, 128)
    bits = [to_dev(a, cuda).view(torch.int16).cpu().numpy().view(np.uint16) for a in (q, k, v)]
    out, rmax, rsum, ms = bbm.run_attention_multi(prep, bbm.Variant.binblk, *bits, 0.088,
                                                  list(range(torch.cuda.device_count())))
    got = torch.from_numpy(out.view(np.int16)).view(torch.bfloat16).float().numpy()
    check_against_oracle(mask, q, k, v, 0.088, got, rmax, rsum, bbm.Variant.binblk, slots_to_check=[0, 5])
    assert ms > 0


def test_permutation_kernels_match_oracle(cuda):
    import torch

    n = 777
    mask = bbm.gen_random_sparse(n, 0.01, 4)
    perm = bbm.rcm_order(mask)
    got = bbm.permute_mask(mask, perm)
    assert np.array_equal(got.words, oracle.permute_mask(mask.words, n, perm.forward))
    x = torch.randn(3, n, 128, device=cuda).to(torch.bfloat16)
    px = bbm.permute_rows(x, perm)
    assert torch.equal(px, x[:, torch.from_numpy(perm.forward.astype(np.int64)).to(cuda)])
    assert torch.equal(bbm.unpermute_rows(px, perm), x)


def test_rcm_end_to_end_reordered_attention(cuda):  # test_reorder.cpp:202-216
    n = 640
    base = bbm.gen_longformer_windowed(n, 12)
    mask = bbm.relabel(base, 3)
    perm = bbm.rcm_order(mask)
    pmask = bbm.permute_mask(mask, perm)
    assert bbm.bandwidth(pmask) <= 2 * 12 + 1
    q, k, v = problem(40, 2, n, 64)
    dq, dk, dv = (to_dev(a, cuda) for a in (q, k, v))
    pq, pk, pv = (bbm.permute_rows(t, perm) for t in (dq, dk, dv))
    prep = bbm.preprocess_mask(pmask, bbm.BlockSpec(128, 128))
    r = bbm.blocked_forward(pq, pk, pv, 0.125, pmask, prep, bbm.Variant.binblk)
    out = bbm.unpermute_rows(r.out, perm).float().cpu().numpy()
    direct = run_gpu(mask, q, k, v, 0.125, bbm.Variant.binblk, cuda)
    assert np.max(np.abs(out - direct[0])) <= TOL_OUT
    assert prep.stats.blocks_nonzero < bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128)).stats.blocks_nonzero


def test_config2_shape_sampled_slots(cuda):
    """BASELINE config 2 shape (packed-seq N=4096 d=128), 2 of the 256 slots vs the oracle; the
    rest through size-independent properties (finite, every row sees itself -> row_sum >= 1)."""
    import torch

    from bench import alpaca_lengths

    mask = bbm.gen_packed_sequential(alpaca_lengths(4096, 7))
    q, k, v = problem(1, 2, 4096, 128)
    out, rmax, rsum, _ = run_gpu(mask, q, k, v, 1 / np.sqrt(128), bbm.Variant.binblk, cuda)
    check_against_oracle(mask, q, k, v, 1 / np.sqrt(128), out, rmax, rsum, bbm.Variant.binblk)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    g = torch.Generator(device=cuda).manual_seed(0)
    big = [(torch.rand((64, 4096, 128), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    r = bbm.blocked_forward(*big, 1 / np.sqrt(128), mask, prep, bbm.Variant.binblk, check_finite=False)
    assert bool(torch.isfinite(r.out.float()).all())
    assert bool((r.row_sum >= 1.0 - 1e-3).all())


@pytest.mark.parametrize("spec,n,d", [("global(w=64;g=100)", 4096, 64), ("all-ones", 2560, 128),
                                      ("causal", 3000, 128), ("dilated(w=40;d=30)", 2600, 64)])
def test_split_kv_long_rows_match_oracle(cuda, spec, n, d):
    """One slot + long KV lists -> the launch splits rows into chunks (split-KV) and the last
    chunk combines the partials; every variant must still match the oracle."""
    mask = bbm.generate(spec, n)
    # a fully masked stretch inside long rows: some chunks see no key for some rows
    for i in range(0, 40):
        for j in range(1024, n):
            mask.set(i, j, False)
    q, k, v = problem(7, 1, n, d)
    scale = 1 / np.sqrt(d)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    for var in bbm.Variant:
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, scale, var, cuda, prep=prep)
        check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, var)
    # repeated launches reuse the per-prep counters (reset in-kernel): identical results
    first = run_gpu(mask, q, k, v, scale, bbm.Variant.binblk, cuda, prep=prep)
    again = run_gpu(mask, q, k, v, scale, bbm.Variant.binblk, cuda, prep=prep)
    assert np.array_equal(again[0], first[0])


@pytest.mark.parametrize("spec,n,d", [("global(w=64;g=100)", 4096, 64), ("causal", 1024, 64),
                                      ("packed-seq[700;1200;900;1296]", 0, 128)])
def test_masked_variants_bitwise_identical_with_split_rows(cuda, spec, n, d):
    # long rows are split into key-range chunks at boundaries set by the occupied tiles, so the
    # masked variants stay bit-identical even when rows are split (test_engine.cpp:112-134)
    mask = bbm.generate(spec, n)
    n = mask.size()
    q, k, v = problem(21, 3, n, d)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    outs = [run_gpu(mask, q, k, v, d ** -0.5, var, cuda, prep=prep) for var in MASKED]
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])
    check_against_oracle(mask, q, k, v, d ** -0.5, *outs[1][:3], bbm.Variant.binblk, slots_to_check=[0])


def test_rcm_host_pipeline_equals_explicit_permutation(cuda):
    # bbm_attn_fwd_rcm_host_bf16: original-order inputs through the device-side permutation
    # equal the explicit host permutation + forward on the reordered mask + host unpermutation
    # (bit for bit: the same kernel runs on the same reordered data), and the attention with the
    # original mask (equivariance, test_reorder.cpp:202-216) to the bf16 tolerance
    import ctypes as C

    from paper_2409_15097_b200 import _lib

    base = bbm.gen_longformer_windowed(1000, 7)
    shuffled = bbm.relabel(base, 3)
    perm = bbm.rcm_order(shuffled)
    pmask = bbm.permute_mask(shuffled, perm)
    slots, n, d = 5, 1000, 128
    q, k, v = problem(31, slots, n, d)
    to_u16 = lambda a: (np.ascontiguousarray(a, np.float32).view(np.uint32) >> 16).astype(np.uint16)  # noqa: E731
    hq, hk, hv = (to_u16(a) for a in (q, k, v))  # inputs are already bf16-exact
    prep = bbm.preprocess_mask(pmask, bbm.BlockSpec(128, 128))
    out = np.empty_like(hq)
    rmax = np.empty((slots, n), np.float32)
    rsum = np.empty((slots, n), np.float32)
    fwd = np.ascontiguousarray(perm.forward, dtype=np.uint32)
    u16, f32 = C.POINTER(C.c_uint16), C.POINTER(C.c_float)
    _lib.check(_lib.lib.bbm_attn_fwd_rcm_host_bf16(
        prep.handle.h, int(bbm.Variant.binblk), fwd.ctypes.data_as(C.POINTER(C.c_uint32)),
        hq.ctypes.data_as(u16), hk.ctypes.data_as(u16), hv.ctypes.data_as(u16), out.ctypes.data_as(u16),
        rmax.ctypes.data_as(f32), rsum.ctypes.data_as(f32), slots, d, d ** -0.5))
    # explicit: permute on the host, plain host-buffer forward, unpermute on the host
    pq, pk, pv = (np.ascontiguousarray(a[:, fwd]) for a in (hq, hk, hv))
    pout = np.empty_like(pq)
    pmax = np.empty((slots, n), np.float32)
    psum = np.empty((slots, n), np.float32)
    _lib.check(_lib.lib.bbm_attn_fwd_host_bf16(
        prep.handle.h, int(bbm.Variant.binblk), pq.ctypes.data_as(u16), pk.ctypes.data_as(u16),
        pv.ctypes.data_as(u16), pout.ctypes.data_as(u16), pmax.ctypes.data_as(f32), psum.ctypes.data_as(f32),
        slots, d, d ** -0.5))
    want = np.empty_like(pout)
    want[:, fwd] = pout
    assert np.array_equal(out, want)
    wmax = np.empty_like(pmax)
    wmax[:, fwd] = pmax
    assert np.array_equal(rmax, wmax)
    got = (out.astype(np.uint32) << 16).view(np.float32)
    check_against_oracle(shuffled, q, k, v, d ** -0.5, got, rmax.astype(np.float64),
                         rsum.astype(np.float64), bbm.Variant.binblk, slots_to_check=[0, 4])


@pytest.mark.parametrize("d", [64, 128])
def test_mixed_items_in_one_launch(cuda, d):
    """Every item shape in one multi-slot launch: fully masked row tiles (no tiles), one-tile rows,
    a long global row that the launch splits (split-KV), a ragged last tile, and both O
    accumulators / statistics slots in turn — the hand-off between the softmax engine and the
    epilogue warpgroup must keep each item's statistics with its own accumulator."""
    n = 2900
    mask = bbm.gen_longformer_windowed(n, 40)
    for j in range(n):  # global row and column: row 0 sees everything, everyone sees key 0
        mask.set(0, j, True)
        mask.set(j, 0, True)
    for i in range(1280, 1408):  # a whole row tile with no key
        for j in range(n):
            mask.set(i, j, False)
    q, k, v = problem(31, 3, n, d)
    scale = 1 / np.sqrt(d)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    for var in (bbm.Variant.binblk, bbm.Variant.dense_binblk):
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, scale, var, cuda, prep=prep)
        check_against_oracle(mask, q, k, v, scale, out, rmax, rsum, var)
        assert np.all(out[:, 1280:1408] == 0) and np.all(rmax[:, 1280:1408] == -np.inf)


@pytest.mark.parametrize("n,d,slots,spec", [(1000, 64, 3, "windowed(w=40)"), (2304, 128, 2, "global(w=90;g=70)"),
                                            (640, 128, 5, "causal")])
@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_in_kernel_rcm_gather_equals_explicit_permutation(cuda, n, d, slots, spec, mode):
    """bbm_attn_fwd_gather_ex (f2): original-order Q/K/V, the prep of the RCM-permuted mask, the
    permutation applied on the device — by permute passes around the plain kernel (mode 1, the
    default 0), by TMA tile::gather4 / scatter4 inside the kernel (mode 2), or K/V by passes with
    Q/O gathered / scattered in the kernel (mode 3) — == permute_rows +
    forward + unpermute_rows, bit for bit, for every variant (incl. ragged n and split-KV rows)."""
    import torch

    base = bbm.generate(spec, n)
    shuffled = bbm.relabel(base, 5)
    perm = bbm.rcm_order(shuffled)
    pm = bbm.permute_mask(shuffled, perm)
    prep = bbm.preprocess_mask(pm, bbm.BlockSpec(128, 128))
    g = torch.Generator(device=cuda).manual_seed(n + d)
    q, k, v = ((torch.rand((slots, n, d), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    rows = torch.from_numpy(perm.forward.astype(np.int32)).to(cuda)
    fwd = torch.from_numpy(perm.forward.astype(np.int64)).to(cuda)
    for var in bbm.Variant:
        out = torch.empty_like(q)
        m = torch.empty((slots, n), dtype=torch.float32, device=cuda)
        l = torch.empty_like(m)
        bbm.attn_fwd_device(prep, var, q, k, v, out, m, l, d ** -0.5, rows=rows, gather_mode=mode)
        qp, kp, vp = (bbm.permute_rows(t, perm) for t in (q, k, v))
        op = torch.empty_like(qp)
        mp = torch.empty_like(m)
        lp = torch.empty_like(m)
        bbm.attn_fwd_device(prep, var, qp, kp, vp, op, mp, lp, d ** -0.5)
        want_o = bbm.unpermute_rows(op, perm)
        want_m = torch.empty_like(mp)
        want_l = torch.empty_like(lp)
        want_m[:, fwd] = mp
        want_l[:, fwd] = lp
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), want_o.view(torch.int16)), var
        assert torch.equal(m.view(torch.int32), want_m.view(torch.int32)), var
        assert torch.equal(l.view(torch.int32), want_l.view(torch.int32)), var


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("scale_sign", [1.0, -1.0])
def test_empty_half_skip_build_is_bitwise_identical(cuda, d, scale_sign):
    """Masks whose occupied tiles are mostly partial run the engine build that skips a warp's
    empty 32 x 64 score halves (the plan header's occupied/full counts select it once they have
    reached the host, one launch after a new prep). The first launch runs the plain build, later
    ones the skipping build: outputs and statistics must be bitwise equal, and match the oracle."""
    import torch

    n = 2900
    mask = bbm.gen_longformer_windowed(n, 40)  # a band: ~all occupied tiles partial
    q, k, v = problem(5, 2, n, d)
    scale = scale_sign / np.sqrt(d)
    import ctypes as C

    from paper_2409_15097_b200 import _lib

    def builds():
        a, b = C.c_uint64(), C.c_uint64()
        _lib.check(_lib.lib.bbm_fwd_build_counts(C.byref(a), C.byref(b)))
        return a.value, b.value

    for var in (bbm.Variant.binblk, bbm.Variant.dense_binblk):
        prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
        c0 = builds()
        first = run_gpu(mask, q, k, v, scale, var, cuda, prep=prep)
        c1 = builds()
        assert c1[0] == c0[0] + 1 and c1[1] == c0[1], "a fresh plan runs the plain build"
        torch.cuda.synchronize()
        for _ in range(2):
            again = run_gpu(mask, q, k, v, scale, var, cuda, prep=prep)
            for a, b in zip(first[:3], again[:3]):
                assert np.array_equal(a, b), var
        assert builds()[1] == c1[1] + 2, "the band mask runs the skipping build once known"
        check_against_oracle(mask, q, k, v, scale, *again[:3], var, slots_to_check=[1])
    # a mask of mostly full tiles keeps the plain build
    causal = bbm.gen_causal(n)
    prep = bbm.preprocess_mask(causal, bbm.BlockSpec(128, 128))
    run_gpu(causal, q, k, v, scale, bbm.Variant.binblk, cuda, prep=prep)
    torch.cuda.synchronize()
    c2 = builds()
    run_gpu(causal, q, k, v, scale, bbm.Variant.binblk, cuda, prep=prep)
    assert builds() == (c2[0] + 1, c2[1])


@pytest.mark.parametrize("n,w", [(3000, 40), (2048, 30), (1111, 20)])
def test_empty_key_half_skipping_is_exact(cuda, n, w):
    """Bands leave whole 64-key halves of their edge tiles empty; binblk / dense_binblk load and
    multiply only the other half, naive always multiplies whole tiles. All three must agree bit
    for bit (a skipped half contributes exactly nothing) and match the oracle."""
    import torch

    mask = bbm.gen_longformer_windowed(n, w)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    assert (prep.tile_halves() > 0).any()
    q, k, v = problem(n + w, 2, n, 128)
    outs = {}
    for var in MASKED:
        for _ in range(2):  # the skip is enabled from the plan header, one launch after a new mask
            r = bbm.blocked_forward(to_dev(q, cuda), to_dev(k, cuda), to_dev(v, cuda), 0.1, mask, prep, var)
            torch.cuda.synchronize()
        outs[var] = (r.out.view(torch.int16).cpu().numpy(), r.row_max.cpu().numpy(), r.row_sum.cpu().numpy())
    base = outs[bbm.Variant.naive_masked]
    for var in MASKED:
        for a, b in zip(outs[var], base):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), var
    out = outs[bbm.Variant.binblk][0].view(np.uint16).astype(np.uint32) << 16
    check_against_oracle(mask, q, k, v, 0.1, out.view(np.float32), outs[bbm.Variant.binblk][1],
                         outs[bbm.Variant.binblk][2], bbm.Variant.binblk)
