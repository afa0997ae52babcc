"""End-to-end NNLS gate (reading R14) for config 4 at full size (too slow for pytest).

x~_gpu = Lawson-Hanson on the GPU sketch (promoted to f64), x~_ora = Lawson-Hanson
on the oracle's f64 sketch; both evaluated as R(x~) = ||A x~ - b|| on the
original data.  Prints one JSON line with the relative difference.
"""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_0812_4547_b200 as srht  # noqa: E402
import workloads  # noqa: E402
from oracle import nnls, srht as osr  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = workloads.CONFIGS[cfg_id]
n, d, r, seed = c["n"], c["d"], c["r"], workloads.SEED
t0 = time.time()
M, xt = workloads.dense_device(n, d, seed=seed)
plan = srht.Plan(n, d, r, seed)
SM = plan.sketch_columns(M, workspace=plan.workspace(d + 1)).cpu().numpy().astype(np.float64)
Mh = M.cpu().numpy()
del M
torch.cuda.empty_cache()
A = Mh[:, :d].astype(np.float64)
b = Mh[:, d].astype(np.float64)
ref = np.empty((r, d + 1))
for j0 in range(0, d + 1, 32):
    ref[:, j0:j0 + 32] = osr.sketch(Mh[:, j0:j0 + 32].astype(np.float64), seed, r)
t1 = time.time()
tol = 1e-5 * np.sqrt(n) * np.max(np.abs(Mh), axis=0)
elem = float(np.max(np.abs(SM - ref) / tol))
x_g, it_g = nnls.lawson_hanson(SM[:, :d], SM[:, d])
x_o, it_o = nnls.lawson_hanson(ref[:, :d], ref[:, d])
Rg, Ro = nnls.residual_norm(A, x_g, b), nnls.residual_norm(A, x_o, b)
sk_g = float(np.linalg.norm(SM[:, :d] @ x_g - SM[:, d]))
sk_o = float(np.linalg.norm(ref[:, :d] @ x_o - ref[:, d]))
out = {"config": cfg_id, "n": n, "d": d, "r": r, "max_err_over_tol": elem,
       "R_gpu": Rg, "R_oracle": Ro, "rel_diff_R": abs(Rg - Ro) / Ro, "gate_1e-6": abs(Rg - Ro) / Ro <= 1e-6,
       "sketched_R_gpu": sk_g, "sketched_R_oracle": sk_o, "rel_diff_sketched_R": abs(sk_g - sk_o) / sk_o,
       "lh_iters": [it_g, it_o], "residual_over_norm_b": Ro / float(np.linalg.norm(b)),
       "seconds": {"sketch+oracle": t1 - t0, "nnls": time.time() - t1}}
print(json.dumps(out), flush=True)
