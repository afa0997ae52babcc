"""Per-phase producer timing of kernel v2 (debug build, mode 8): CTA 0, warp 0 of each producer warp."""
import ctypes
import sys

import numpy as np
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
tr = torch.zeros(8 * 64 * 10, dtype=torch.int64, device="cuda")
lib.srht_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 8
print("trace mode", mode)
lib.srht_debug_set_mode(mode)
for _ in range(3):
    plan.sketch_columns(M, out=out, workspace=ws)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(8, 64, 10).astype(np.float64)
names = ["loads", "signs", "round0", "EMPTY wait", "STS.128", "GRP wait", "LDS", "round1", "STS+arrive"]
for wgi in [0, 4]:
    rows = t[wgi, 8:60]
    ph = np.diff(rows, axis=1)                      # phase k: t[k+1]-t[k]
    cyc = np.diff(rows[:, 0])                      # tile to tile
    print("group %d warp0: tile-to-tile %.0f cycles (median)" % (wgi // 4, np.median(cyc)))
    for k in range(9):
        print("   %-12s %7.0f" % (names[k], np.median(ph[:, k])))
    print("   %-12s %7.0f" % ("next start", np.median(rows[1:, 0] - rows[:-1, 9])))
lib.srht_debug_set_mode(0)
