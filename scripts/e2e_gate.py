"""North-star end-to-end NNLS gate (reading R14) at full size, configs 4 and 5.

    python scripts/e2e_gate.py [config] > profiles/r02_e2e_nnls_c<config>.json

For each sketch mode (FP32 throughput path, FP64-accumulation mode) and for the oracle's
float64 sketch: x~ = the oracle's Lawson-Hanson on (SA, Sb) (Algorithm 1 step 5),
then R(x~) = ||A x~ - b|| on the ORIGINAL data, computed on the device in FP64 (2^26 x 128 is
too big for the host).  Gate: |R(x~_gpu) - R(x~_oracle)| / R(x~_oracle) <= 1e-6.  Also:
element-wise parity of every column against the north_star tolerance, the FP64 mode against
one FP32 spacing, and the Fig. 1 relative error R(x~) / R(x_opt), with x_opt from
Lawson-Hanson on the Cholesky form of the full problem (reading C13: Q = A^T A, q = A^T b on
the device in FP64; min ||L^T x - L^-1 q|| has the same minimiser).
The oracle sketches all columns column-parallel on the host cores (tests/par_oracle.py).
"""

import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0812_4547_b200 as srht  # noqa: E402
import workloads  # noqa: E402
from oracle import nnls  # noqa: E402
from tests import par_oracle  # noqa: E402


def residual(M, x, d, chunk=8):
    """||A x - b|| in FP64 on the device, A = M[:, :d] (FP32), b = M[:, d]."""
    res = -M[:, d].double()
    xt = torch.from_numpy(np.asarray(x, dtype=np.float64)).to(M.device)
    for j0 in range(0, d, chunk):
        j1 = min(d, j0 + chunk)
        res += M[:, j0:j1].double() @ xt[j0:j1]
    return float(torch.linalg.vector_norm(res))


def gram_full(M, d, chunk=8):
    """G = [A | b]^T [A | b] in FP64 on the device (exact products, FP64 sums)."""
    c = d + 1
    G = torch.zeros((c, c), dtype=torch.float64, device=M.device)
    rows = M.shape[0]
    step = 1 << 22
    for i0 in range(0, rows, step):
        blk = M[i0:i0 + step].double()
        G += blk.t() @ blk
    return G.cpu().numpy()


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = workloads.CONFIGS[cfg_id]
    n, d, r, seed = c["n"], c["d"], c["r"], workloads.SEED
    t0 = time.time()
    M, x_true = workloads.dense_device(n, d, seed=seed)
    sk = {}
    for accum in ("fp32", "fp64"):
        plan = srht.Plan(n, d, r, seed, accum=accum)
        ws = plan.workspace(d + 1)
        SM = plan.sketch_columns(M, workspace=ws)
        torch.cuda.synchronize()
        kern = srht.library().srht_debug_last_kernel()
        sk[accum] = (SM.cpu().numpy().astype(np.float64), kern)
        del plan, ws, SM
        torch.cuda.empty_cache()
    bcol = M[:, d].cpu().numpy()
    colmax = M.abs().amax(dim=0).cpu().numpy().astype(np.float64)
    t1 = time.time()
    specs = [("gen", (j, n)) for j in range(d)] + [("array", bcol)]
    ref, workers = par_oracle.sketch_columns(specs, seed, r)
    t2 = time.time()
    bound = 1e-5 * math.sqrt(n) * colmax
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    out = {"config": cfg_id, "n": n, "d": d, "r": r, "columns_checked": d + 1,
           "oracle": {"workers": workers, "seconds": t2 - t1}}
    x_o = nnls.solve_sketched(ref[:, :d], ref[:, d])
    R_o = residual(M, x_o, d)
    # x_opt of the full problem through its Cholesky form (same minimiser, reading C13)
    G = gram_full(M, d)
    L = np.linalg.cholesky(G[:d, :d])
    y = np.linalg.solve(L, G[:d, d])
    x_opt = nnls.solve_sketched(L.T, y)
    R_opt = residual(M, x_opt, d)
    out["oracle_sketch"] = {"R": R_o, "relative_error_fig1": R_o / R_opt}
    out["R_opt"] = R_opt
    out["residual_over_norm_b"] = R_opt / float(np.linalg.norm(bcol.astype(np.float64)))
    for accum, (SM, kern) in sk.items():
        err = np.abs(SM - ref)
        x_g = nnls.solve_sketched(SM[:, :d], SM[:, d])
        R_g = residual(M, x_g, d)
        rel = abs(R_g - R_o) / R_o
        e = {"kernel": {3: "k_sketch_tma", 6: "k_sketch_tma64"}.get(kern, str(kern)),
             "max_err_over_tol": float(np.max(err / bound[None, :])),
             "max_err_over_fp32_ulp": float(np.max(err / np.maximum(ulp, 1e-300))),
             "R": R_g, "rel_diff_R": rel, "gate_1e-6": bool(rel <= 1e-6),
             "relative_error_fig1": R_g / R_opt,
             "sketched_R": float(np.linalg.norm(SM[:, :d] @ x_g - SM[:, d])),
             "support_equal_to_oracle": bool(np.array_equal(x_g > 0, x_o > 0))}
        out[accum] = e
    out["seconds"] = {"generate+sketch": t1 - t0, "oracle": t2 - t1, "nnls+residuals": time.time() - t2}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
