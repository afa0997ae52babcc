"""Stress run of the config-5 sketch: many launches in one process, output compared bit for bit
with the first launch after every 25 (kernel v3 is deterministic).  python scripts/stress_v3.py [launches]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n, d, r = 1 << 26, 127, 16384
M = torch.empty((d + 1, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(d + 1)
out = torch.empty((d + 1, r), device="cuda").t()
plan.sketch_columns(M, out=out, workspace=ws)
ref = out.clone()
bad = 0
for i in range(k):
    plan.sketch_columns(M, out=out, workspace=ws)
    if i % 25 == 24:
        torch.cuda.synchronize()
        bad += int(not torch.equal(out, ref))
torch.cuda.synchronize()
print("launches", k + 1, "mismatching checks", bad, "kernel", srht.library().srht_debug_last_kernel(), flush=True)
