"""compute-sanitizer on one device-RCM gather mode: python tools/sanitize_gather_mode.py <mode 1-4>"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_15097_b200 as bbm
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
base = bbm.relabel(bbm.generate("windowed(w=40)", 1000), 5)
perm = bbm.rcm_order(base)
prep = bbm.preprocess_mask(bbm.permute_mask(base, perm), bbm.BlockSpec(128, 128))
rows = torch.from_numpy(perm.forward.astype(np.int32)).to(dev)
q, k, v = ((torch.rand((2, 1000, 128), generator=g, device=dev) * 2 - 1).to(torch.bfloat16) for _ in range(3))
out = torch.empty_like(q); m = torch.empty((2, 1000), dtype=torch.float32, device=dev); l = torch.empty_like(m)
mode = int(sys.argv[1])
for var in bbm.Variant:
    bbm.attn_fwd_device(prep, var, q, k, v, out, m, l, 0.08, rows=rows, gather_mode=mode)
torch.cuda.synchronize(); print("ok", mode)
