"""CPU tests of libbbm's host side: the C-ABI surface, generators, RCM, mask model helpers.

No compute calls here (no GPU in the build container); the GPU parity tests are in
tests/test_gpu_*.py (-m gpu).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from paper_2409_15097_b200 import _lib
from tests.conftest import GOLDEN, ROOT


def test_library_loads_and_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "bbm_capi.h")).read()
    declared = set(re.findall(r"\b(bbm_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = C.CDLL(bbm.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, f"symbols declared in bbm_capi.h but not exported: {missing}"
    assert declared == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"
    assert lib.bbm_abi_version() == 2


def test_device_count_is_safe_without_gpu():
    c = C.c_int(-1)
    assert _lib.lib.bbm_device_count(C.byref(c)) == 0
    assert c.value >= 0


def test_generators_bit_identical_to_reference_golden():
    g = np.load(os.path.join(GOLDEN, "mask_model.npz"))
    seen = set()
    for i in range(int(g["count"])):
        name = str(g[f"c{i}_name"])
        words = g[f"c{i}_words"]
        n = words.shape[0]
        if (name, n) in seen:
            continue
        seen.add((name, n))
        m = bbm.generate(name, n)
        assert m.size() == n and np.array_equal(m.words, words), name


def test_generator_errors_match_reference():  # test_generators.cpp:212-230
    for bad in ("nope", "windowed(w=3", "windowed(x=1)", "medusa[0]", "random(p=abc)",
                "packed-bidir[3]"):
        with pytest.raises(ValueError):
            bbm.generate(bad, 8)
    with pytest.raises(ValueError):
        bbm.gen_longformer_windowed(4, 4)


def test_medusa_size_without_root():  # generators.hpp:22-32, test_generators.cpp:27-33
    assert bbm.blockmask.medusa_size([4, 4, 4, 4]) == 340
    assert bbm.gen_medusa([4, 4, 4, 4]).size() == 340


def test_rcm_matches_reference_golden():
    g = np.load(os.path.join(GOLDEN, "rcm.npz"))
    for i in range(int(g["count"])):
        words = g[f"r{i}_words"]
        m = bbm.Mask(words.shape[0], words)
        perm = bbm.rcm_order(m)
        assert np.array_equal(perm.forward, g[f"r{i}_fwd"])
        assert bbm.bandwidth(m) == int(g[f"r{i}_bw"][0])


def test_rcm_matches_oracle_on_random_graphs():
    for seed, n, p in ((1, 97, 0.03), (2, 300, 0.01), (3, 64, 0.2), (4, 513, 0.004)):
        m = bbm.gen_random_sparse(n, p, seed, force_diagonal=(seed % 2 == 0))
        assert np.array_equal(bbm.rcm_order(m).forward, oracle.rcm_order(m.words, n))


def test_rcm_kats():  # test_reorder.cpp:109-127, 174-186
    assert bbm.rcm_order(bbm.generate("random(p=0;seed=1)", 5)).forward.tolist() == [4, 3, 2, 1, 0]
    path = bbm.Mask(12)
    for i in range(12):
        path.set(i, i, True)
        if i + 1 < 12:
            path.set(i, i + 1, True)
    shuffled = bbm.relabel(path, 5)
    perm = bbm.rcm_order(shuffled)
    re_words = oracle.permute_mask(shuffled.words, 12, perm.forward)
    assert oracle.bandwidth(re_words, 12) == 1


def test_relabel_is_a_conjugation():
    m = bbm.gen_longformer_windowed(50, 3)
    r = bbm.relabel(m, 3)
    assert r.count_ones() == m.count_ones()
    assert bbm.bandwidth(r) > bbm.bandwidth(m)


def test_mask_helpers_and_permutation():
    m = bbm.Mask(70)
    m.set(3, 69, True)
    m.set(3, 0, True)
    m.set(69, 64, True)
    assert m.get(3, 69) and m.get(3, 0) and not m.get(3, 1) and m.count_ones() == 3
    m.set(3, 69, False)
    assert m.count_ones() == 2
    d = np.random.default_rng(0).random((70, 70)) < 0.3
    assert np.array_equal(bbm.Mask.from_dense(d).to_dense(), d)
    with pytest.raises(ValueError):
        bbm.Permutation.from_forward([0, 0, 1])
    p = bbm.Permutation.from_forward([2, 0, 1])
    assert p.inverse.tolist() == [1, 2, 0]


@pytest.mark.gpu  # the helpers run the preprocessor's row kernel on the device
def test_host_metadata_helpers_match_golden():
    g = np.load(os.path.join(GOLDEN, "mask_model.npz"))
    for i in range(0, int(g["count"]), 7):
        n, bi, bj = (int(x) for x in g[f"c{i}_spec"])
        sums = bbm.BlockSums(n, bbm.BlockSpec(bi, bj), g[f"c{i}_sums"])
        assert np.array_equal(bbm.build_block_occupancy(sums).values, g[f"c{i}_occ"])
        runs = bbm.build_dense_runs(sums)
        assert runs.offset == g[f"c{i}_off"].tolist() and runs.total_ones == g[f"c{i}_tot"].tolist()
        st = bbm.block_stats(sums)
        assert [st.blocks_total, st.blocks_nonzero, st.blocks_full] == g[f"c{i}_stats_u"].tolist()
        assert [st.block_density, st.element_density] == g[f"c{i}_stats_f"].tolist()


def test_variant_names():  # engine.hpp:28-45
    for v in bbm.Variant:
        assert bbm.parse_variant(bbm.to_string(v)) == v
    with pytest.raises(ValueError):
        bbm.parse_variant("fast")


def test_spec_validation():
    with pytest.raises(ValueError):
        bbm.BlockSpec(0, 4).validate()
    with pytest.raises(ValueError):
        bbm.BlockSpec(4, 0).validate()


def test_shard_slots_cover_all_slots():
    for slots in (1, 7, 128, 256):
        for g in (1, 2, 4, 8):
            ranges = [bbm.shard_slots(slots, g, r) for r in range(g)]
            assert ranges[0][0] == 0 and ranges[-1][1] == slots
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
