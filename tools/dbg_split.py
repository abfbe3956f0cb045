import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import oracle, paper_2409_15097_b200 as bbm
from tests.test_gpu_attn import problem, run_gpu
cuda = torch.device('cuda', 0)
for spec, n, d, cut in [("global(w=64;g=100)", 4096, 64, True), ("global(w=64;g=100)", 4096, 64, False), ("global(w=64;g=100)", 4096, 128, True), ("causal", 1024, 64, False)]:
    mask = bbm.generate(spec, n)
    if cut:
        for i in range(0, 40):
            for j in range(1024, n):
                mask.set(i, j, False)
    q, k, v = problem(7, 1, n, d)
    scale = 1 / np.sqrt(d)
    prep = bbm.preprocess_mask(mask, bbm.BlockSpec(128, 128))
    for var in bbm.Variant:
        out, rmax, rsum, _ = run_gpu(mask, q, k, v, scale, var, cuda, prep=prep)
        words = None if var == bbm.Variant.dense else mask.words
        o, m, l = oracle.naive_forward(q[0], k[0], v[0], scale, words, n, threads=16)
        err = np.abs(out[0] - o).max(axis=1)
        bad = np.nonzero(err > 2e-2)[0]
        print(spec, n, d, cut, var.name, 'max', err.max(), 'bad rows', bad[:10], len(bad))
