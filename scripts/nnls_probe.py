"""Config-4-shaped NNLS (r = 8192, d = 512, Uniform[0,1) sketch-like columns) for profiling the
GPU solvers: python scripts/nnls_probe.py [lh|bpp] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0812_4547_b200 as srht  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "bpp"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(44)
r, d = 8192, 512
SA = rng.random((r, d), dtype=np.float32)
xs = rng.random(d)
xs[rng.choice(d, d // 2, replace=False)] = 0.0
Sb = (SA.astype(np.float64) @ xs + 0.01 * rng.standard_normal(r)).astype(np.float32)
M = torch.from_numpy(np.asfortranarray(np.column_stack([SA, Sb]))).t().contiguous().t().cuda()
G = srht.gram(M)
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x, it = srht.nnls_gram(G, method=method)
    b.record()
    torch.cuda.synchronize()
    print(method, "ms", a.elapsed_time(b), "iters", int(it))
