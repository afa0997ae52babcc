"""Per-GPU throughput of config 5 at the column-shard sizes of a 1/2/4/8-GPU run (128, 64, 32, 16
columns of n = 2^26), measured on one GPU: CUDA events around each sketch, 10 launches after 3."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = 1 << 26, 127, 16384
plan = srht.Plan(n, d, r, 0)
lib = _lib.load()
res = {}
for cols in (128, 64, 32, 16):
    M = torch.empty((cols, n), dtype=torch.float32, device="cuda").t()
    srht.gen_uniform(0, 0, M)
    ws = plan.workspace(cols)
    out = torch.empty((cols, r), device="cuda").t()
    for _ in range(3):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        plan.sketch_columns(M, out=out, workspace=ws)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    res[cols] = {"ms": ms, "GBps": 4.0 * n * cols / ms / 1e6}
    del M, out, ws
    torch.cuda.empty_cache()
print(json.dumps(res))
