"""Knock-out experiments on kernel v2 (timing only; results are wrong when mode != 0)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1 << 20, 512, 8192))]
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
res = {}
modes = [int(x) for x in sys.argv[4].split(',')] if len(sys.argv) > 4 else [0, 1, 2, 3, 4, 5, 6, 7]
for mode in modes:
    lib.srht_debug_set_mode(mode)
    for _ in range(3):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    lib.srht_profile_start(10)
    for _ in range(10):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    arr = (ctypes.c_float * 10)()
    cnt = ctypes.c_int()
    lib.srht_profile_stop(arr, 10, ctypes.byref(cnt))
    ms = sum(arr[i] for i in range(cnt.value)) / cnt.value
    res[mode] = (ms, 4.0 * n * c / ms / 1e6)
    names = {0: 'full', 1: 'no loads', 2: 'no gather', 3: 'no loads+gather', 4: 'no butterflies', 5: 'no loads+bfly',
             6: 'no gather+bfly', 7: 'barriers+smem only', 16: 'ALT tokens', 17: 'ALT no loads', 20: 'ALT no bfly', 32: 'SOLO group', 33: 'SOLO no loads', 35: 'SOLO no loads/gather'}
    print("mode %d (%s): %.3f ms  %.0f GB/s-equivalent" % (mode, names.get(mode, '?'), ms, res[mode][1]), flush=True)
lib.srht_debug_set_mode(0)
