"""bench.py's two arms build the SAME workload (CPU, no GPU needed).

The reference arm composes each BASELINE config's mask from the reference's own code
(oracle/_ref: generators.hpp, reorder.hpp compiled from /root/reference), the GPU arm from this
framework's host generators / relabel / RCM and its device permute_mask; the masks must be
identical bit for bit, and both arms print the identical `config` object.
"""
import numpy as np
import pytest

import bench
import oracle
import paper_2409_15097_b200 as bbm

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def ours_host(name):
    """Our arm's composition with the (GPU) permute_mask replaced by the oracle's restatement."""
    gen, relabel, rcm, _ = bench.bbm_backends(bbm)
    return bench.mask_words(name, gen, relabel, rcm, lambda w, n, f: oracle.permute_mask(w, n, f))


@needs_ref
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_masks_identical_across_arms(name):
    ours, _ = ours_host(name)
    ref, _ = bench.ref_mask(name)
    assert ours.shape == ref.shape and np.array_equal(ours, ref)
    assert ours.shape[0] == bench.CONFIGS[name][5]


@needs_ref
def test_config5_rcm_pipeline_identical_across_arms():
    n = bench.CONFIGS["c5"][5]
    band = oracle.ref_generate("windowed(w=164)", n)
    assert np.array_equal(bbm.generate("windowed(w=164)", n).words, band)
    shuffled_ref = oracle.ref_relabel(band, n, 3)
    shuffled = bbm.relabel(bbm.Mask(n, band), 3).words
    assert np.array_equal(shuffled, shuffled_ref)
    fwd_ref, bw0, bw1 = oracle.ref_rcm(shuffled_ref, n)
    fwd = bbm.rcm_order(bbm.Mask(n, shuffled)).forward
    assert np.array_equal(fwd, fwd_ref)
    assert bw0 > 30000 and bw1 == 164  # bandwidth 32758 -> 164
    assert np.array_equal(oracle.permute_mask(shuffled, n, fwd), oracle.ref_permute_mask(shuffled_ref, n, fwd_ref))


def test_config_dict_is_arm_independent():
    for name in bench.CONFIGS:
        a = bench.config_dict(name, "binblk", 4, "strong")
        assert a == bench.config_dict(name, "binblk", 4, "strong")
        assert a["slots"] == bench.CONFIGS[name][0] * bench.CONFIGS[name][1]


def test_alpaca_lengths_fill_the_sequence():
    lengths = bench.alpaca_lengths(4096, 7)
    assert sum(lengths) == 4096 and all(1 <= x <= 512 for x in lengths)
    assert all(64 <= x for x in lengths[:-1])
