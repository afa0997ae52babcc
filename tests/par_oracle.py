"""Column-parallel runs of the CPU oracle (test infrastructure only).

The oracle sketches one column of a 2^26-row problem in ~20 s single-threaded; the
full-size config-5 checks run it over many columns at once, one process per host
core.  Columns of A are regenerated in each worker from the counter-based generator
(bit-identical to srht_gen_uniform, pinned by test_config4_full_sampled_columns); any
other column (b) is passed in as an array.
"""

import multiprocessing as mp
import os

import numpy as np


def _work(args):
    seed, r, spec = args
    import workloads
    from oracle import srht as osr
    kind, payload = spec
    if kind == "gen":
        j, n = payload
        col = workloads.host_uniform_column(seed, j, n)
    else:
        col = payload
    return osr.sketch(np.asarray(col, dtype=np.float64), seed, r)[:, 0]


def sketch_columns(specs, seed, r, workers=None):
    """Oracle sketches (float64, (r, len(specs))) of the given columns.

    specs: list of ("gen", (j, n)) for column j of the uniform generator, or ("array", col).
    workers: processes (default: host cores, at most one per ~5 GB of available memory).
    """
    if workers is None:
        try:
            import psutil
            by_mem = int(0.7 * psutil.virtual_memory().available // 5e9)
        except Exception:
            by_mem = 4
        workers = max(1, min(len(os.sched_getaffinity(0)), by_mem, len(specs)))
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        cols = pool.map(_work, [(seed, r, s) for s in specs], chunksize=1)
    return np.stack(cols, axis=1), workers
