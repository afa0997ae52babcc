"""Knock-out experiments on kernel v3 (debug build libsrht_dbg.so; timing only, results wrong).

SRHT_LIB=libsrht_dbg.so python scripts/v3_knockouts.py [n d r] [modes]
mode bits: 1 = consumers skip the gather loads, 4 = producers skip the round shared-memory
traffic.  (Modes with bit 2 (no butterflies) or bit 8 (no transform) fail to launch in the debug
build and are not used.)"""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1 << 26, 127, 16384))]
modes = [int(x) for x in sys.argv[4].split(',')] if len(sys.argv) > 4 else [0, 1, 4, 5]
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
names = {0: "full", 1: "no gather loads", 4: "no round smem", 5: "no gather, no round smem",
         8: "no transform", 9: "no transform, no gather"}
for mode in modes:
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
    print("mode %d (%-26s): %7.3f ms  %6.0f GB/s-equivalent" % (mode, names.get(mode, "?"), ms, 4.0 * n * c / ms / 1e6),
          flush=True)
lib.srht_debug_set_mode(0)
