"""Time the FP64-accumulation parity mode (plan accum="fp64") on config 4 (2^20 x 513, r = 8192)."""
import json
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

n, d, r = 1 << 20, 512, 8192
M = torch.empty((d + 1, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
res = {}
for accum in ("fp32", "fp64"):
    plan = srht.Plan(n, d, r, 0, accum=accum)
    ws = plan.workspace(d + 1)
    ts = []
    for i in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.sketch_columns(M, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    res[accum] = statistics.median(ts)
print(json.dumps({"config": 4, "ms": res}))
