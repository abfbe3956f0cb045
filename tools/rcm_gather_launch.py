"""C5 forward on original-order inputs with the RCM permutation applied on the device (f2), for ncu:
    ncu --set full -k regex:attn_fwd_kernel -s 2 -c 1 python tools/rcm_gather_launch.py [mode]
mode: 1 passes, 2 TMA gather4, 3 hybrid, 4 LSU gather (default)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2409_15097_b200 as bbm  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 4
words, fwd_perm = bench.mask_words("c5", *bench.bbm_backends(bbm, 0))
B, H, d, _, _, n = bench.CONFIGS["c5"]
prep = bbm.preprocess_mask(bbm.Mask(n, words), bbm.BlockSpec(128, 128))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = ((torch.rand((B * H, n, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
rows = torch.from_numpy(np.ascontiguousarray(fwd_perm, dtype=np.int32)).to(dev)
for _ in range(4):
    bbm.attn_fwd_device(prep, bbm.Variant.binblk, q, k, v, out, None, None, d ** -0.5, rows=rows, gather_mode=mode)
torch.cuda.synchronize()
print("ok")
