"""Config 4: eager step time vs CUDA-graph replay of the same step (sketch + slab reduction)."""
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

n, d, r = 1 << 20, 512, 8192
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
step = lambda: plan.sketch_columns(M, out=out, workspace=ws)
for _ in range(3):
    step()
torch.cuda.synchronize()


def timeit(fn, k=50):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


eager = timeit(step)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    step()
graph = timeit(g.replay)
print(json.dumps({"eager_ms": eager, "graph_ms": graph}))
