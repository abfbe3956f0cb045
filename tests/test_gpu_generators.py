"""Device mask generators (f4, gen.cu) against the reference's own generators.hpp (oracle/_ref)
and the host fixture: bit-identical packed words, including the random family's single
mt19937_64 stream over all n^2 entries at the config-5 size (-m gpu)."""
import time

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

SPECS = [("causal", 1000), ("all-ones", 130), ("windowed(w=37)", 777), ("windowed(w=5;causal=1)", 300),
         ("dilated(w=9;d=3)", 500), ("global(w=64;g=100)", 4096), ("global(w=3;g=7)", 65),
         ("random(p=0.01;seed=1)", 100), ("random(p=0.3;seed=7)", 1000), ("random(p=0.02;seed=3;diag=0)", 4099),
         ("random(p=0;seed=1)", 64), ("random(p=1;seed=2;diag=0)", 70), ("medusa[4;4]", 0), ("packed-seq[5;9;3]", 0)]


@needs_ref
@pytest.mark.parametrize("spec,n", SPECS)
def test_device_generator_matches_reference(cuda, spec, n):
    dev = bbm.generate_device(spec, n).cpu().numpy().view(np.uint64)
    ref = oracle.ref_generate(spec, n)
    assert dev.shape == ref.shape and np.array_equal(dev, ref)
    assert np.array_equal(dev, bbm.generate(spec, n).words)


@needs_ref
@pytest.mark.parametrize("spec", ["random(p=0.01;seed=1)", "windowed(w=164)", "global(w=512;g=128)"])
def test_device_generator_config_sizes(cuda, spec):
    import torch

    n = 32768 if "global" not in spec else 16384
    t0 = time.perf_counter()
    dev = bbm.generate_device(spec, n)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = oracle.ref_generate(spec, n)
    t_ref = time.perf_counter() - t0
    assert np.array_equal(dev.cpu().numpy().view(np.uint64), ref)
    print(f"{spec} n={n}: device {t_dev * 1e3:.1f} ms, reference host {t_ref * 1e3:.1f} ms")
