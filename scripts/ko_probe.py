import ctypes, sys, time
sys.path.insert(0, '.')
import torch
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib
n, d, r = 1 << 20, 512, 8192
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
for mode in [int(x) for x in sys.argv[1].split(',')]:
    lib.srht_debug_set_mode(mode)
    t = time.time()
    plan.sketch_columns(M, out=out, workspace=ws)
    torch.cuda.synchronize()
    print("mode", mode, "ok", round(time.time() - t, 3), "s", "kernel", lib.srht_debug_last_kernel(), flush=True)
