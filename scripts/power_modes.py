"""Sustained-load kernel time and power per knock-out mode (debug build; timing only).

SRHT_LIB=libsrht_dbg.so python scripts/power_modes.py modes  (nvidia-smi samples alongside;
each mode: 150 back-to-back launches, then 2 s idle).  Prints wall-clock windows per mode."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = 1 << 26, 127, 16384
modes = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [0]
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
K = 150
for mode in modes:
    if hasattr(lib, "srht_debug_set_mode"):
        lib.srht_debug_set_mode(mode)
    plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    time.sleep(2.0)
    lib.srht_profile_start(K)
    t0 = time.time()
    for _ in range(K):
        plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    t1 = time.time()
    arr = (ctypes.c_float * K)()
    cnt = ctypes.c_int()
    lib.srht_profile_stop(arr, K, ctypes.byref(cnt))
    a = [arr[i] for i in range(cnt.value)]
    print("mode %d: wall %.3f-%.3f  first5 %.3f ms  last50 %.3f ms" % (mode, t0, t1, sum(a[:5]) / 5, sum(a[-50:]) / 50),
          flush=True)
