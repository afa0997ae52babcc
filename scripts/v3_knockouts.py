"""Knock-out experiments on kernel v3 (debug build libsrht_dbg.so; timing only, results wrong).

SRHT_LIB=libsrht_dbg.so python scripts/v3_knockouts.py [n d r]
mode bits: 1 = consumers skip the gather loads, 2 = producers skip butterflies,
4 = producers skip round-1/round-2 shared-memory traffic."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1 << 26, 127, 16384))]
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
names = {0: "full", 1: "no gather loads", 2: "no butterflies", 3: "no gather, no butterflies",
         4: "no round smem", 5: "no gather, no round smem", 6: "no bfly, no round smem", 7: "TMA + barriers only"}
for mode in range(8):
    lib.srht_debug_set_mode(mode)
    for _ in range(2):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    lib.srht_profile_start(5)
    for _ in range(5):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    arr = (ctypes.c_float * 5)()
    cnt = ctypes.c_int()
    lib.srht_profile_stop(arr, 5, ctypes.byref(cnt))
    ms = sum(arr[i] for i in range(cnt.value)) / cnt.value
    print("mode %d (%-26s): %7.3f ms  %6.0f GB/s-equivalent  kernel %d" % (
        mode, names[mode], ms, 4.0 * n * c / ms / 1e6, lib.srht_debug_last_kernel()), flush=True)
lib.srht_debug_set_mode(0)
