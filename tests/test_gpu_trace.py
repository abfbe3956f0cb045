"""The event-tracing builds of the attention kernels (bbm_set_trace; tools/trace_attn.py,
tools/trace_bwd.py) record events and compute exactly what the untraced kernels compute (-m gpu)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from paper_2409_15097_b200 import _lib

pytestmark = pytest.mark.gpu


def test_traced_kernels_record_events_and_match(cuda):
    import torch

    n, d, slots = 700, 128, 2
    mask = bbm.gen_longformer_windowed(n, 150)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    q, k, v, g = (torch.from_numpy(a.astype(np.float32)).to(cuda).to(torch.bfloat16)
                  for a in oracle.make_problem(3, slots, n, d))
    scale = d ** -0.5

    def run():
        out = torch.empty_like(q)
        rmax = torch.empty((slots, n), dtype=torch.float32, device=cuda)
        rsum = torch.empty_like(rmax)
        bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k, v, out, rmax, rsum, scale)
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        bbm.attn_bwd_device(prep, bbm.Variant.binblk, q, k, v, out, rmax, rsum, g, dq, dk, dv, scale)
        torch.cuda.synchronize()
        return out, dq, dk, dv

    plain = run()
    buf = torch.zeros(2 * 8192, dtype=torch.int64, device=cuda)
    os.environ["BBM_TRACE_BWD_SIDE"] = "1"
    try:
        _lib.check(_lib.lib.bbm_set_trace(C.c_void_p(buf.data_ptr()), 2))
        traced = run()
    finally:
        _lib.check(_lib.lib.bbm_set_trace(None, 0))
        del os.environ["BBM_TRACE_BWD_SIDE"]
    for a, b in zip(plain, traced):
        assert torch.equal(a, b)
    codes = set(((buf.cpu().numpy().view(np.uint64) >> 16) & 0xFF).tolist()) - {0}
    assert {10, 11, 20, 21, 22} <= codes or {40, 41, 50, 51, 52} <= codes, codes
