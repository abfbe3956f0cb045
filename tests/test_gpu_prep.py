"""GPU mask preprocessor parity (-m gpu): bit-exact against the reference's golden vectors and
the C oracle, through the C ABI (packed host, packed device and dense-bool device inputs)."""
import os

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def check_prep(prep, sums, occ, off, tot, stats_u, stats_f, ctx=""):
    assert np.array_equal(prep.sums.values, sums), ctx
    assert np.array_equal(prep.occupancy.values, occ), ctx
    assert prep.runs.offset == list(off) and prep.runs.total_ones == list(tot), ctx
    st = prep.stats
    assert [st.blocks_total, st.blocks_nonzero, st.blocks_full] == list(stats_u), ctx
    assert [st.block_density, st.element_density] == list(stats_f), ctx


def test_prep_matches_reference_golden_every_case(cuda):
    g = np.load(os.path.join(GOLDEN, "mask_model.npz"))
    for i in range(int(g["count"])):
        n, bi, bj = (int(x) for x in g[f"c{i}_spec"])
        m = bbm.Mask(n, g[f"c{i}_words"])
        prep = bbm.preprocess_mask(m, bbm.BlockSpec(bi, bj))
        check_prep(prep, g[f"c{i}_sums"], g[f"c{i}_occ"], g[f"c{i}_off"], g[f"c{i}_tot"],
                   g[f"c{i}_stats_u"].tolist(), g[f"c{i}_stats_f"].tolist(),
                   f"{g[f'c{i}_name']} n={n} {bi}x{bj}")


def test_kats_on_gpu(cuda):  # test_mask_model.cpp:81-125
    p = bbm.preprocess_mask(bbm.gen_causal(4), bbm.BlockSpec(2, 2))
    assert p.sums.values.tolist() == [[3, 0], [4, 3]]
    assert p.runs.offset == [0, 0] and p.runs.total_ones == [0, 1]
    assert p.stats.block_density == 0.75 and p.stats.element_density == 10 / 16
    p = bbm.preprocess_mask(bbm.gen_all_ones(5), bbm.BlockSpec(2, 2))
    assert p.sums.values.tolist() == [[4, 4, 2], [4, 4, 2], [2, 2, 1]]
    assert p.runs.total_ones == [3, 3, 3]
    occ = bbm.preprocess_mask(bbm.gen_medusa([4, 4, 4, 4]), bbm.BlockSpec(128, 32)).occupancy
    assert (occ.rows(), occ.cols()) == (3, 11) and all(occ.at(p, 0) for p in range(3))
    with pytest.raises(ValueError):
        bbm.preprocess_mask(bbm.gen_causal(4), bbm.BlockSpec(0, 2))


@pytest.mark.parametrize("spec,n", [("packed-seq[700;1200;900;1296]", 0), ("global(w=512;g=128)", 4096),
                                    ("random(p=0.01;seed=3)", 2500), ("causal", 1024),
                                    ("medusa[16;15]", 0), ("windowed(w=200)", 3000)])
@pytest.mark.parametrize("bs", [(128, 128), (64, 64), (128, 64), (100, 37)])
def test_prep_matches_oracle_at_scale(cuda, spec, n, bs):
    m = bbm.generate(spec, n)
    N = m.size()
    prep = bbm.preprocess_mask(m, bbm.BlockSpec(*bs))
    sums, occ, off, tot, st = oracle.preprocess(m.words, N, *bs)
    check_prep(prep, sums, occ, off, tot,
               [st["blocks_total"], st["blocks_nonzero"], st["blocks_full"]],
               [st["block_density"], st["element_density"]], spec)


def expected_kernel_lists(words, n):
    sums, _, _, _, _ = oracle.preprocess(words, n, 128, 128)
    kr = sums.shape[0]
    ri = np.minimum(128, n - np.arange(kr) * 128)
    area = np.outer(ri, ri)
    cnt = (sums > 0).sum(axis=1).astype(np.uint32)
    lists = []
    for p in range(kr):
        qs = np.flatnonzero(sums[p] > 0)
        # full flag (bit 31) is never set on a ragged right-edge tile (the kernel masks it)
        lists.append([int(q) | (0x80000000 if sums[p, q] == area[p, q] and (q + 1) * 128 <= n else 0)
                      for q in qs])
    order = sorted(range(kr), key=lambda p: (-int(cnt[p]), p))
    return cnt, lists, order


@pytest.mark.parametrize("spec,n", [("packed-seq[64;300;128;555;1]", 0), ("global(w=100;g=3)", 1000),
                                    ("random(p=0.002;seed=5;diag=0)", 777), ("all-ones", 130)])
def test_kernel_lists_ascending_and_lpt_order(cuda, spec, n):
    m = bbm.generate(spec, n)
    N = m.size()
    prep = bbm.preprocess_mask(m, bbm.BlockSpec(128, 128))
    cnt, lst, order = prep.kernel_lists()
    want_cnt, want_lists, want_order = expected_kernel_lists(m.words, N)
    assert np.array_equal(cnt, want_cnt)
    for p in range(len(want_lists)):
        assert lst[p, : cnt[p]].tolist() == want_lists[p]
    assert order.tolist() == want_order


@pytest.mark.parametrize("n", [4096, 1000, 2388, 16384])
def test_bool_device_path_equals_packed_path(cuda, n):
    import torch

    m = bbm.gen_longformer_global(n, min(512, n - 1), 64) if n != 1000 else bbm.gen_random_sparse(n, 0.05, 2)
    dense = torch.from_numpy(m.to_dense()).to(cuda)
    for bs in ((128, 128), (64, 32)):
        a = bbm.preprocess_mask(dense, bbm.BlockSpec(*bs))
        b = bbm.preprocess_mask(m, bbm.BlockSpec(*bs))
        assert np.array_equal(a.sums.values, b.sums.values)
        assert a.runs == b.runs and a.stats == b.stats
        ca, la, oa = a.kernel_lists()
        cb, lb, ob = b.kernel_lists()
        assert np.array_equal(ca, cb) and np.array_equal(oa, ob)
        for p in range(len(ca)):
            assert np.array_equal(la[p, : ca[p]], lb[p, : cb[p]])


def test_packed_device_path(cuda):
    import torch

    m = bbm.gen_random_sparse(1500, 0.01, 8)
    dev = torch.from_numpy(m.words.view(np.int64)).to(cuda)
    a = bbm.preprocess_mask(dev, bbm.BlockSpec(128, 128))
    b = bbm.preprocess_mask(m, bbm.BlockSpec(128, 128))
    assert np.array_equal(a.sums.values, b.sums.values) and a.stats == b.stats


def test_counters_match_reference_golden(cuda):
    g = np.load(os.path.join(GOLDEN, "counters.npz"))
    for i in range(int(g["count"])):
        n, bi, bj, var, *want = (int(x) for x in g[f"k{i}"])
        prep = bbm.preprocess_mask(bbm.Mask(n, g[f"k{i}_words"]), bbm.BlockSpec(bi, bj))
        c = prep.counters(bbm.Variant(var), 1)
        got = [c.blocks_visited, c.blocks_processed, c.mask_block_reads, c.skipped_by_binblk,
               c.skipped_mask_reads_by_run]
        assert got == want, (n, bi, bj, var)
        c3 = prep.counters(bbm.Variant(var), 3)
        assert c3.blocks_visited == 3 * want[0]


@pytest.mark.parametrize("n", [4096, 1000])
def test_uint8_mask_any_nonzero_is_true(cuda, n):
    """A uint8 mask holding arbitrary nonzero values (not just 0 / 1) means the same as its 0 / 1
    version: identical metadata and bitwise identical attention output (the fast pack path
    normalizes 16-byte chunks that contain values > 1)."""
    import torch

    m = bbm.gen_random_sparse(n, 0.05, 4)
    ones = torch.from_numpy(m.to_dense()).to(cuda)
    g = torch.Generator(device=cuda).manual_seed(1)
    vals = torch.randint(1, 256, (n, n), generator=g, device=cuda, dtype=torch.uint8)
    # half the rows keep plain 0 / 1 bytes, so both pack paths meet in one launch
    vals[::2] = 1
    wild = torch.where(ones, vals, torch.zeros_like(vals))
    a = bbm.preprocess_mask(ones, bbm.BlockSpec(128, 128))
    b = bbm.preprocess_mask(wild, bbm.BlockSpec(128, 128))
    assert np.array_equal(a.sums.values, b.sums.values) and a.runs == b.runs and a.stats == b.stats
    ca, la, _ = a.kernel_lists()
    cb, lb, _ = b.kernel_lists()
    assert np.array_equal(ca, cb)
    q, k, v = ((torch.rand((2, n, 64), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16) for _ in range(3))
    outs = []
    for prep in (a, b):
        o = torch.empty_like(q)
        bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k, v, o, None, None, 0.125)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def _expected_halves(m, cnt, lst):
    """Empty key halves of every occupied 128x128 tile at its list position (numpy)."""
    n = m.size()
    kt = (n + 127) // 128
    pad = np.zeros((kt * 128, kt * 128), bool)
    pad[:n, :n] = m.to_dense()
    want = np.zeros((kt, kt), np.uint8)
    for p in range(kt):
        for k in range(cnt[p]):
            q = int(lst[p, k] & 0x7FFFFFFF)
            blk = pad[p * 128:(p + 1) * 128, q * 128:(q + 1) * 128]
            want[p, k] = (0 if blk[:, :64].any() else 1) | (0 if blk[:, 64:].any() else 2)
    return want


@pytest.mark.parametrize("n,kind", [(4096, "band"), (1000, "band"), (2304, "causal"), (1500, "random"),
                                    (3000, "packed")])
def test_tile_halves_match_the_mask(cuda, n, kind):
    """The forward skips a 64-key half of a tile that no row sees; the flags come from the fused
    preprocessor (n % 16 == 0), the kernel chain (bool rows with n % 16 != 0) and the packed path."""
    import torch

    m = {"band": lambda: bbm.gen_longformer_windowed(n, 40),
         "causal": lambda: bbm.gen_causal(n),
         "random": lambda: bbm.gen_random_sparse(n, 0.002, 4),
         "packed": lambda: bbm.gen_packed_sequential([50, 300, 30, 700, 100, 1820])}[kind]()
    for src in (m, torch.from_numpy(m.to_dense()).to(cuda)):
        prep = bbm.preprocess_mask(src, bbm.BlockSpec(128, 128))
        cnt, lst, _ = prep.kernel_lists()
        got = prep.tile_halves()
        want = _expected_halves(m, cnt, lst)
        for p in range(len(cnt)):
            assert np.array_equal(got[p, : cnt[p]], want[p, : cnt[p]]), p
    if kind == "band":
        assert (want > 0).any()  # the case the forward's half skipping is for
