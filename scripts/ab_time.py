"""A/B timing of one library build (SRHT_LIB=lib<name>.so): tile-kernel ms per launch on
config 5 and config 4, launched alone (0.3 s gaps) and back to back, plus a parity spot check
of 2 config-4 columns against the float64 oracle.  python scripts/ab_time.py [5,4]"""
import ctypes
import json
import math
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

lib = _lib.load()
res = {"lib": os.environ.get("SRHT_LIB", "libsrht.so")}
cfgs = [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ["5", "4"])]
for cfg in cfgs:
    n, d, r = (1 << 26, 127, 16384) if cfg == 5 else (1 << 20, 512, 8192)
    c = d + 1
    M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
    srht.gen_uniform(0, 0, M)
    if os.environ.get("AB_SYNC"):  # stress runs: name the stage an asynchronous fault surfaces in
        torch.cuda.synchronize()
        print("progress: config %d inputs generated" % cfg, file=sys.stderr, flush=True)
    plan = srht.Plan(n, d, r, 0)
    if os.environ.get("AB_SYNC"):
        torch.cuda.synchronize()
        print("progress: config %d plan built" % cfg, file=sys.stderr, flush=True)
    ws = plan.workspace(c)
    out = torch.empty((c, r), device="cuda").t()

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
        return [arr[i] for i in range(cnt.value)]

    print("progress: config %d first sketches" % cfg, file=sys.stderr, flush=True)
    run(3, 0)
    print("progress: config %d first sketches done" % cfg, file=sys.stderr, flush=True)
    ref_out = out.clone()
    alone = run(6, 0.3)
    print("progress: config %d alone runs done" % cfg, file=sys.stderr, flush=True)
    b2b = run(20 if cfg == 5 else 200, 0)
    print("progress: config %d back-to-back runs done" % cfg, file=sys.stderr, flush=True)
    res["c%d" % cfg] = {"alone_med": statistics.median(alone), "b2b_first10": statistics.mean(b2b[:10]),
                        "b2b_last10": statistics.mean(b2b[-10:]), "kernel": lib.srht_debug_last_kernel(),
                        "deterministic": bool(torch.equal(out, ref_out))}
    if cfg == 4:  # parity spot check: columns 0 and d against the oracle
        from oracle import srht as osr
        for j in (0, d):
            x = M[:, j].double().cpu().numpy()
            ref = osr.sketch(x[:, None], 0, r)[:, 0]
            got = out[:, j].double().cpu().numpy()
            bound = 1e-5 * math.sqrt(n) * np.abs(x).max()
            res["c4_err_over_bound_col%d" % j] = float(np.abs(got - ref).max() / bound)
    del M, out, ws, plan
    torch.cuda.empty_cache()
    if os.environ.get("AB_SLEEP"):  # stress runs: let the clocks recover between configurations
        torch.cuda.synchronize()
        time.sleep(float(os.environ["AB_SLEEP"]))
print(json.dumps(res), flush=True)
