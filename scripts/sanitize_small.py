"""Small sketches through every kernel path, for compute-sanitizer runs (no timing)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

rng = np.random.default_rng(0)
for (n, c, r) in [(40000, 3, 1000), (1 << 15, 2, 16384), (70000, 5, 300)]:
    M = torch.from_numpy(rng.random((n, c), dtype=np.float32)).cuda().t().contiguous().t()
    plan = srht.Plan(n, c - 1, r, 1)
    SM = plan.sketch_columns(M)
    part = plan.sketch_rows_partial(M[: plan.row_shard_rows()], 0) if n > plan.row_shard_rows() else None
    torch.cuda.synchronize()
    print("dense", n, c, r, float(SM.abs().sum()))
G = srht.gram(SM)
x, it = srht.nnls_gram(G[:2, :2].contiguous() if G.shape[0] > 2 else G)
A = rng.standard_normal((600, 200)).astype(np.float32)
Gb = srht.gram(torch.from_numpy(A).cuda().t().contiguous().t())
xb, itb = srht.nnls_gram(Gb)
torch.cuda.synchronize()
print("nnls", int(itb))
