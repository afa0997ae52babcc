"""Time Algorithm 2 SubspaceSampling on the GPU at the config-4 shape (n = 2^20, d = 512,
r = 8192, p_i proportional to the squared row norms of Phi).  CUDA events, median of 5."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

n, d, r = 1 << 20, 512, 8192
Phi = torch.empty((d, n), device="cuda").t()
srht.gen_uniform(3, 0, Phi)
p = (Phi.double() ** 2).sum(1)
p /= p.sum()
ts = []
for i in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    K, rows = srht.subspace_sampling(Phi, r, p, seed=5)
    b.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(a.elapsed_time(b))
print(json.dumps({"n": n, "d": d, "r": r, "kept": int(K.numel()), "ms": statistics.median(ts),
                  "out_MB": rows.numel() * 4 / 1e6}))
