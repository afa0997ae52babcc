"""Kernel time per launch, back to back vs with idle gaps (power / thermal drift check).

python scripts/step_drift.py [5|4]  -- prints the k_sketch_tma duration of each launch."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = (1 << 26, 127, 16384) if len(sys.argv) < 2 or sys.argv[1] == "5" else (1 << 20, 512, 8192)
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()


def run(k, gap):
    lib.srht_profile_start(k)
    for _ in range(k):
        plan.sketch_columns(M, out=out, workspace=ws)
        if gap:
            torch.cuda.synchronize()
            time.sleep(gap)
    torch.cuda.synchronize()
    arr = (ctypes.c_float * k)()
    cnt = ctypes.c_int()
    lib.srht_profile_stop(arr, k, ctypes.byref(cnt))
    return [round(arr[i], 3) for i in range(cnt.value)]


run(3, 0)
print("gap 0.5 s:", run(6, 0.5))
print("back to back:", run(120, 0))
print("gap 0.5 s:", run(6, 0.5))
