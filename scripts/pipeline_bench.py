"""Time the GPU RandomizedNNLS pipeline stages (Algorithm 1 on the GPU): sketch, Gram, NNLS.

python scripts/pipeline_bench.py [config]   (2: 3000 batched CSC problems; 4: 2^20 x 512 dense;
1: the tiny dense problem).  CUDA-event times per stage, median of 5 after 2 warm-ups.
"""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
import workloads

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = workloads.CONFIGS[cfg_id]
seed = workloads.SEED
dev = torch.device("cuda", 0)


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


if cfg_id == 2:
    w = workloads.config2_host(seed)
    n, d, batch, r = w["n"], w["d"], w["batch"], w["r"]
    c = d + 1
    plan = srht.Plan(n, d, r, seed, batch=batch)
    M = srht.CSC(torch.from_numpy(w["colptr"]).to(dev), torch.from_numpy(w["rowidx"]).to(dev),
                 torch.from_numpy(w["vals"]).to(dev), (n, batch * c))
    ws = plan.workspace(batch * c)
    t_s, SM = timed(lambda: plan.sketch_batched(M, workspace=ws))
else:
    n, d, r = cfg["n"], cfg["d"], cfg["r"]
    batch, c = 1, cfg["d"] + 1
    Md, _ = workloads.dense_device(n, d, seed=seed)
    plan = srht.Plan(n, d, r, seed)
    ws = plan.workspace(c)
    t_s, SM = timed(lambda: plan.sketch_columns(Md, workspace=ws))
t_g, G = timed(lambda: srht.gram(SM))
res = {"config": cfg_id, "batch": batch, "n": n, "d": d, "r": r, "ms": {"sketch": t_s, "gram": t_g},
       "gram_gflops": 2.0 * batch * r * c * c / 2 / (t_g * 1e-3) / 1e9}
xs = {}
for method in ("lh", "bpp"):
    if method == "bpp" and d > 580:
        continue
    t_n, (x, it) = timed(lambda: srht.nnls_gram(G, method=method), reps=3, warm=1)
    it = it.cpu().numpy().reshape(-1)
    xs[method] = x
    res["ms"]["nnls_" + method] = t_n
    res["iterations_" + method] = {"min": int(it.min()), "median": float(np.median(it)), "max": int(it.max())}
if len(xs) == 2:
    a, b = xs["lh"].double(), xs["bpp"].double()
    res["bpp_vs_lh_max_abs_diff"] = float((a - b).abs().max())
    res["bpp_vs_lh_same_support"] = bool(torch.equal(a > 0, b > 0))
res["ms"]["total_bpp" if "nnls_bpp" in res["ms"] else "total_lh"] = t_s + t_g + res["ms"].get("nnls_bpp", res["ms"]["nnls_lh"])
print(json.dumps(res))
