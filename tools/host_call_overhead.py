"""Per-call cost of the float host-buffer entries at small sizes (acceptance.cpp:267-289's shape:
one head, N=4096, d=64, windowed(w=256)): blocked_forward / blocked_backward on numpy float32,
timed on the host (synchronous API) against the device-resident kernels of the same problem."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_15097_b200 as bbm  # noqa: E402

n, d = 4096, 64
mask = bbm.generate("windowed(w=256)", n) if hasattr(bbm, "generate") else bbm.gen_longformer_windowed(n, 256)
prep = bbm.preprocess_mask(mask, bbm.BlockSpec(64, 64))
rng = np.random.default_rng(0)
q, k, v, g = (rng.uniform(-1, 1, (n, d)).astype(np.float32) for _ in range(4))
for var in (bbm.Variant.dense, bbm.Variant.binblk):
    for _ in range(3):
        f = bbm.blocked_forward(q, k, v, 0.125, mask, prep, var)
        b = bbm.blocked_backward(q, k, v, 0.125, mask, prep, var, f, g)
    tf, tb = [], []
    for _ in range(10):
        t0 = time.perf_counter()
        f = bbm.blocked_forward(q, k, v, 0.125, mask, prep, var)
        t1 = time.perf_counter()
        b = bbm.blocked_backward(q, k, v, 0.125, mask, prep, var, f, g)
        t2 = time.perf_counter()
        tf.append(t1 - t0)
        tb.append(t2 - t1)
    dev = torch.device("cuda", 0)
    tq, tk, tv, tg = (torch.from_numpy(a).to(dev).to(torch.bfloat16) for a in (q, k, v, g))
    fd = bbm.blocked_forward(tq, tk, tv, 0.125, mask, prep, var)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        fd = bbm.blocked_forward(tq, tk, tv, 0.125, mask, prep, var, check_finite=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"{var.name}: host fwd {np.median(tf) * 1e3:.3f} ms, host bwd {np.median(tb) * 1e3:.3f} ms, "
          f"device fwd {e0.elapsed_time(e1) / 20:.3f} ms")
