#!/usr/bin/env python
"""Benchmark: SRHT sketch throughput of [A | b] (input GB/s and fraction of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl srht|reference]

Default workload: BASELINE.json config 5 (A = 2^26 x 127 FP32 Uniform[0,1) plus b,
128 columns, 34.4 GB, r = 16384), the configuration the metric is quoted on at
1/2/4/8 GPUs.  One "step" = one SRHT sketch of all 128 columns: the tile kernel
(load + sign + FWHT + pruned accumulate) and the slab reduction, plus, for N > 1,
one NCCL all_gather of the r x c_g shards (columns are sharded across ranks;
total work is fixed, so scaling is "strong").  Plan creation (Algorithm 1 steps
2 and 4) is excluded, as in SURVEY.md 8(d).  Inputs (34 GB) are far larger than
L2 (126 MB), so no L2 flush is needed between steps.

Under torchrun every rank runs its shard; timing is CUDA events on the launch
stream between barriers + synchronize, max over ranks; rank 0 prints one JSON line.
"""

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "SRHT sketch throughput: input GB/s of [A|b] and % of B200 HBM peak, 1/2/4/8 GPUs"
UNIT = "GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="srht", choices=["srht", "reference"])
    ap.add_argument("--accum", default="fp32", choices=["fp32", "fp64"],
                    help="fp32: the throughput path; fp64: the FP64-accumulation parity mode "
                         "(DESIGN.md reading R14), which meets the 1e-6 end-to-end gate on configs 4/5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sustain-seconds", type=float, default=1.0,
                    help="after the timed steps, run back to back for about this long and report the "
                         "steady-state step (the 1000 W board cap engages after ~50 ms); 0 = skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1, column shards: p2p = the sketch's reduction stores every rank's columns "
                         "straight into all ranks' outputs over NVLink (CUDA IPC, fused gather); nccl = one "
                         "all_gather_into_tensor after the sketch")
    ap.add_argument("--shard", default="columns", choices=["columns", "rows"],
                    help="multi-GPU partition of [A|b]: column ranges + all-gather (default) or "
                         "row ranges + one FP64 all-reduce of the partial sums")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def column_range(c, world, rank):
    base, rem = divmod(c, world)
    c0 = rank * base + min(rank, rem)
    return c0, c0 + base + (1 if rank < rem else 0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return 6650.0, "fallback", {}


def load_traffic(config, kernel):
    """dram read+write bytes per launch of the tile kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("config%d" % config)
    except Exception:
        return None


KERNEL_NAMES = {1: "k_sketch_tiles", 2: "k_sketch_ws", 3: "k_sketch_tma", 4: "k_sketch_f64", 5: "k_sketch_col",
                6: "k_sketch_tma64"}


def last_kernel(lib):
    """Name of the tile kernel the library ran for the last sketch call."""
    return KERNEL_NAMES.get(lib.srht_debug_last_kernel(), "unknown")


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": getattr(pynvml, "nvmlClocksEventReasonGpuIdle", 0x1),
                "applications_clocks_setting": getattr(pynvml, "nvmlClocksEventReasonApplicationsClocksSetting", 0x2),
                "sw_power_cap": getattr(pynvml, "nvmlClocksEventReasonSwPowerCap", 0x4),
                "hw_slowdown": getattr(pynvml, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "sync_boost": 0x10,
                "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40,
                "hw_power_brake_slowdown": 0x80,
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, v in names.items():
                            if mask & v and k != "gpu_idle":
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(0.02)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": "NVML sampling unavailable"}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# Oracle timing (cpu_baseline leg and --impl reference): the only places bench
# executes oracle/.
# ---------------------------------------------------------------------------

def oracle_sample(cfg_id, seed=workloads.SEED, part=0):
    """One bounded sample of the workload for the CPU oracle: (callable, bytes, description).

    `part` selects a different column of a dense workload (the column-parallel leg gives each
    worker its own column); sparse samples are the same for every part."""
    from oracle import srht as osr
    cfg = workloads.CONFIGS[cfg_id]
    n, r = cfg["n"], cfg["r"]
    if cfg["kind"] == "dense":
        j = int(part) % cfg["d"]
        col = workloads.host_uniform_column(seed, j, n).astype(np.float64)
        return (lambda: osr.sketch(col, seed, r)), 4 * n, "1 column (A[:,%d]) of config %d, n=%d, r=%d" % (
            j, cfg_id, n, r)
    if cfg_id == 3:
        w = workloads.config3_host(seed)
        dense = workloads.csc_to_dense(w["colptr"], w["rowidx"], w["vals"], n, 4)
        nbytes = 8 * int(w["colptr"][4]) + 8 * 5
        return (lambda: osr.sketch(dense, seed, r)), nbytes, "4 CSC columns of config 3 (densified), n=%d, r=%d" % (n, r)
    w = workloads.config2_host(seed, batch=2)
    c = w["d"] + 1
    dense = workloads.csc_to_dense(w["colptr"], w["rowidx"], w["vals"], n, 2 * c)
    nbytes = 8 * int(w["colptr"][2 * c]) + 8 * (2 * c + 1)

    def run():
        for p in range(2):
            osr.sketch(dense[:, p * c:(p + 1) * c], seed, r, p=p)
    return run, nbytes, "2 of 3000 batched CSC problems of config 2 (densified), n=%d, r=%d" % (n, r)


def _oracle_worker(cfg_id, part, barrier, q):
    """Column-parallel leg: build this worker's sample, wait for every worker, time the oracle."""
    try:
        fn, nbytes, desc = oracle_sample(cfg_id, part=part)
        barrier.wait(timeout=600)
        t0 = time.time()
        fn()
        q.put((part, t0, time.time(), nbytes, desc))
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((part, None, None, 0, repr(e)))


def oracle_workers(cfg_id):
    """Workers for the all-cores leg: the host cores this process may use, at most one per
    column of a dense workload, and at most one per ~5 GB of available RAM (the float64
    oracle holds several N-long temporaries per column)."""
    import psutil
    cores = len(os.sched_getaffinity(0))
    cfg = workloads.CONFIGS[cfg_id]
    per_worker = 40.0 * max(cfg["n"], 1 << 16) + 256e6 if cfg["kind"] == "dense" else 1.5e9
    by_mem = int(0.7 * psutil.virtual_memory().available // per_worker)
    w = min(cores, max(1, by_mem))
    if cfg["kind"] == "dense":
        w = min(w, cfg["d"])
    return max(1, w), cores


def time_oracle_parallel(cfg_id, workers):
    """The oracle as it stands, one process per host core, each on its own sample; throughput =
    all samples' bytes / (last finish - first start)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(workers)
    q = ctx.Queue()
    procs = [ctx.Process(target=_oracle_worker, args=(cfg_id, k, barrier, q)) for k in range(workers)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=1800) for _ in range(workers)]
    for pr in procs:
        pr.join(timeout=60)
    ok = [x for x in res if x[1] is not None]
    if len(ok) < workers:
        raise RuntimeError("oracle worker failed: %s" % [x[4] for x in res if x[1] is None][:1])
    t = max(x[2] for x in ok) - min(x[1] for x in ok)
    nbytes = sum(x[3] for x in ok)
    desc = "%d worker processes, each on its own sample (worker 0: %s)" % (workers, ok[0][4])
    return nbytes / t / 1e9, t, desc


def cpu_baseline_line(cfg_id):
    """cpu_baseline: the oracle on 1 core and column-parallel on all host cores (rank 0, N = 1)."""
    v1, t1, desc1 = time_oracle(cfg_id)
    w, cores = oracle_workers(cfg_id)
    try:
        vp, tp, descp = time_oracle_parallel(cfg_id, w)
        allc = {"value": vp, "unit": UNIT, "cores": w, "host_cores": cores, "sample": descp, "seconds": tp}
    except Exception as e:  # keep the single-core number if the parallel leg cannot run
        allc = {"value": None, "unit": UNIT, "cores": w, "host_cores": cores, "error": repr(e)[:200]}
    best = allc if allc.get("value") and allc["value"] > v1 else None
    return {"value": best["value"] if best else v1, "unit": UNIT, "cores": best["cores"] if best else 1,
            "kind": "oracle", "sample": best["sample"] if best else desc1,
            "single_core": {"value": v1, "unit": UNIT, "cores": 1, "sample": desc1, "seconds": t1},
            "all_cores": allc}


def time_oracle(cfg_id, reps=1):
    fn, nbytes, desc = oracle_sample(cfg_id)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    return nbytes / t / 1e9, t, desc


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    fn, nbytes, desc = oracle_sample(args.config)
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    t = (time.perf_counter() - t0) / args.steps
    value = nbytes / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config%d_%s" % (args.config, cfg["name"]), "n": cfg["n"], "d": cfg["d"],
                   "r": cfg["r"], "sample": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# The GPU arm
# ---------------------------------------------------------------------------

def build_dense_shard(cfg, c0, c1, seed, device, srht):
    """Column shard [c0, c1) of M = [A | b] on the device (A generated, b = A x + noise)."""
    import torch
    n, d = cfg["n"], cfg["d"]
    c = d + 1
    Ml = torch.empty((c1 - c0, n), dtype=torch.float32, device=device).t()
    a1 = min(c1, d)
    if a1 > c0:
        srht.gen_uniform(seed, c0, Ml[:, : a1 - c0])
    if c1 == c:  # this rank holds b
        x = workloads.x_true_half_zeros(seed, d)
        e = workloads._rng(seed, 2).standard_normal(n) * 0.01
        b64 = torch.from_numpy(e).to(device)
        xt = torch.from_numpy(x).to(device)
        chunk = 8
        tmp = torch.empty((chunk, n), dtype=torch.float32, device=device).t()
        for j0 in range(0, d, chunk):
            j1 = min(d, j0 + chunk)
            if c0 <= j0 and j1 <= a1:
                blk = Ml[:, j0 - c0:j1 - c0]
            else:
                blk = tmp[:, : j1 - j0]
                srht.gen_uniform(seed, j0, blk)
            b64 += blk.double() @ xt[j0:j1]
        Ml[:, c - 1 - c0] = b64.float()
        del tmp, b64
    torch.cuda.synchronize()
    return Ml


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_0812_4547_b200 as srht
    from paper_0812_4547_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    cfg = workloads.CONFIGS[args.config]
    if cfg["kind"] != "dense":
        return bench_sparse(args, cfg, srht, _lib, world, rank, device)
    n, d, r, seed = cfg["n"], cfg["d"], cfg["r"], workloads.SEED
    c = d + 1
    rows_mode = args.shard == "rows"
    plan = srht.Plan(n, d, r, seed, accum=args.accum)
    if rows_mode:
        # every rank holds rows [row0, row1) of all c columns (Uniform[0,1) from rank-specific
        # streams: the timing does not depend on the values)
        from paper_0812_4547_b200 import dist as sdist
        row0, row1 = sdist.row_range(n, world, rank, plan.row_shard_rows())
        c0, c1, cl = 0, c, c
        Ml = torch.empty((c, row1 - row0), dtype=torch.float32, device=device).t()
        if row1 > row0:
            srht.gen_uniform(seed, 1000003 * (rank + 1), Ml)
        torch.cuda.synchronize()
    else:
        c0, c1 = column_range(c, world, rank)
        cl = c1 - c0
        Ml = build_dense_shard(cfg, c0, c1, seed, device, srht)
    ws = plan.workspace(cl)
    stream = torch.cuda.current_stream(device)
    lib = _lib.load()
    if world > 1:
        from paper_0812_4547_b200 import dist as sdist
        sdist.check_same_plan(plan, device=device)  # untimed: every rank derived the same D and S
    peers = None
    gather_mode = "nccl" if (world == 1 or rows_mode) else args.gather
    if gather_mode == "p2p":
        try:
            peers = sdist.PeerOutputs(plan, c)
        except Exception as exc:  # IPC mapping not possible here: the NCCL all-gather
            if rank == 0:
                print("fused gather unavailable (%s); using NCCL all_gather" % exc, file=sys.stderr)
            gather_mode = "nccl"
        full_out = torch.empty((c, r), dtype=torch.float32, device=device).t()
    else:
        full_out = torch.empty((c, r), dtype=torch.float32, device=device).t()

    part_buf = torch.empty((c, r), dtype=torch.float64, device=device).t() if rows_mode else None

    def step():
        if rows_mode:
            if Ml.shape[0]:
                plan.sketch_rows_partial(Ml, row0, out=part_buf, workspace=ws)
            else:
                part_buf.zero_()
            if world > 1:
                dist.all_reduce(part_buf.t(), op=dist.ReduceOp.SUM)
            plan.rows_finish(part_buf, out=full_out)  # r^{-1/2} + FP32 rounding in the library
        elif world > 1 and peers is not None:
            sdist.sketch_sharded_p2p(plan, Ml, c, peers, workspace=ws)
        elif world > 1:
            sdist.sketch_sharded(plan, Ml, c, out=full_out, workspace=ws)
        else:
            plan.sketch_columns(Ml, out=full_out, workspace=ws)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # inputs that fit in L2 (config 1): flush L2 (256 MB write) before every step, outside
    # the per-step events; larger inputs stream through L2 and run back to back
    small = 4.0 * n * c <= 2 * 126e6
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=device) if small else None
    with ClockSampler(local) as clk:
        _lib.check(lib.srht_profile_start(args.steps), "srht_profile_start")
        pairs = []
        if small:
            for i in range(args.steps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                pairs.append((e0, e1))
        else:
            ev0.record(stream)
            for i in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
        kms_arr = (ctypes.c_float * args.steps)()
        kcount = ctypes.c_int()
        _lib.check(lib.srht_profile_stop(kms_arr, args.steps, ctypes.byref(kcount)), "srht_profile_stop")
    if world > 1:
        dist.barrier()
    ms = (statistics.mean(a.elapsed_time(b) for a, b in pairs) if small else ev0.elapsed_time(ev1) / args.steps)
    kms = statistics.mean(kms_arr[i] for i in range(kcount.value))
    t = torch.tensor([ms, kms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kms_max = float(t[0]), float(t[1])  # max over ranks

    total_in = 4.0 * n * c
    value = total_in / (ms * 1e-3) / 1e9
    kname = last_kernel(lib)
    peak, peak_kind, peaks = load_peaks()
    # read the shard once, write r x c_l (rows mode: the shard's rows, FP64 r x c partials)
    alg_bytes_launch = (4.0 * Ml.shape[0] * c + 8.0 * r * c) if rows_mode else (4.0 * n * cl + 4.0 * r * cl)
    achieved = alg_bytes_launch / (kms_max * 1e-3) / 1e9  # slowest rank's kernel
    clk_now = clk.summary()
    if args.accum == "fp64":
        # FP64 mode: bound by the FP64 add pipe.  Algorithmic adds per padded element: log2 r + 1
        # (SURVEY 8(d)); peak = 148 SMs x 64 FP64 lanes x the median SM clock under load
        # (scripts/mb_dadd.cu measures the lanes).
        lg = max(1, (r - 1).bit_length())
        alg_adds = (lg + 1) * float(plan.N) * cl
        clk_mhz = clk_now.get("sm_mhz") or 1965.0
        dpeak = 148 * 64 * clk_mhz * 1e6 / 1e12
        dach = alg_adds / (kms_max * 1e-3) / 1e12
        roofline = {"bound": "alu", "achieved": dach, "peak": dpeak, "unit": "TFLOP/s", "frac": dach / dpeak,
                    "traffic": None, "kernel": kname,
                    "peak_source": "148 SMs x 64 FP64 add lanes x %.0f MHz (derived; DESIGN.md 6.1b)" % clk_mhz,
                    "kernel_ms": kms_max, "share_of_step": kms_max / ms, "adds_per_padded_element": lg + 1,
                    "hbm_achieved_GBps": achieved, "hbm_frac": achieved / peak}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": load_traffic(args.config, kname), "kernel": kname,
                    "peak_source": "%s (MEASURED_PEAKS.json hbm_gbs)" % peak_kind if peak_kind == "measured"
                    else "fallback 6650 GB/s (B200_PROFILING.md)",
                    "kernel_ms": kms_max, "share_of_step": kms_max / ms}

    # ---- sustained: back-to-back steps for ~sustain_seconds, per-step events, second half ----
    sustained = None
    if args.sustain_seconds > 0 and not small:
        k = max(8, int(args.sustain_seconds / (ms * 1e-3)))
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k + 1)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk2:
            _lib.check(lib.srht_profile_start(k), "srht_profile_start")
            evs[0].record(stream)
            for i in range(k):
                step()
                evs[i + 1].record(stream)
            torch.cuda.synchronize()
            sk_arr = (ctypes.c_float * k)()
            skc = ctypes.c_int()
            _lib.check(lib.srht_profile_stop(sk_arr, k, ctypes.byref(skc)), "srht_profile_stop")
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(k)]
        half = per[k // 2:]
        kh = [sk_arr[i] for i in range(k // 2, skc.value)]
        st = torch.tensor([statistics.median(half), statistics.median(kh) if kh else 0.0], dtype=torch.float64,
                          device=device)
        if world > 1:
            dist.all_reduce(st, op=dist.ReduceOp.MAX)
        s_ms, s_kms = float(st[0]), float(st[1])
        sustained = {"steps": k, "ms_per_step": s_ms, "value": 4.0 * n * c / (s_ms * 1e-3) / 1e9, "unit": UNIT,
                     "kernel_ms": s_kms, "note": "median of the second half of %d back-to-back steps" % k,
                     "clocks": clk2.summary()}
        if args.accum != "fp64" and s_kms > 0:
            sustained["roofline_frac"] = alg_bytes_launch / (s_kms * 1e-3) / 1e9 / peak

    # ---- config 1: steady-state CUDA-graph replay of the step (launch bound) ----
    graph = None
    if small and world == 1 and not rows_mode:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device)
        side.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream(device).wait_stream(side)
        with torch.cuda.graph(g):
            step()
        reps = 200
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = {"us_per_step": 1e3 * e0.elapsed_time(e1) / reps, "replays": reps,
                 "l2": "not flushed (steady-state replay)"}

    # ---- e2e: the same sketch through the host-buffer C-ABI call ----
    e2e = None
    if not args.no_e2e and not rows_mode:
        e2e = measure_e2e(args, plan, Ml, n, r, c, cl, world, rank, device, peers)

    # ---- cpu_baseline: the oracle on the host cores (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if args.accum == "fp64" else "f32", "data": "synthetic",
            "config": {"workload": "config%d_%s" % (args.config, cfg["name"]), "n": n, "d": d, "r": r,
                       "accum": args.accum,
                       "columns": c, "input_bytes": total_in,
                       "parallelism": ("rows/%d" if rows_mode else "columns/%d") % world,
                       "gather": None if world == 1 else ("allreduce (rows)" if rows_mode else
                                                          ("fused p2p" if peers is not None else "nccl all_gather")),
                       "l2": "flushed (256 MB write) before each step" if small else "inputs larger than L2 (no flush)"},
            "hbm_frac_of_measured": value / peak,
            "hbm_frac_of_8TBs": value / 8000.0,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": args.steps * (2 if (plan_has_reduce(plan) or rows_mode) else 1) + (
                args.steps if rows_mode else 0),
        }
        if graph is not None:
            line["graph_replay"] = graph
        if sustained is not None:
            line["sustained"] = sustained
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_sparse(args, cfg, srht, _lib, world, rank, device):
    """Configs 2 (3000 batched CSC problems) and 3 (CSC A + dense b), single GPU.

    Metric: input GB/s of the CSC bytes (8 nnz + 8 (c+1), plus the dense b) per
    sketch.  These paths are FP32-ALU / latency bound (the inputs are small and
    the transform is dense work), so the roofline reported is the FP32 add rate
    (148 SMs x 128 lanes x SM clock) against the pruned adds per element.
    """
    import torch
    if world > 1:
        raise SystemExit("sparse configs are single-GPU in bench.py")
    seed = workloads.SEED
    if args.config == 2:
        w = workloads.config2_host(seed)
        n, d, batch, r = w["n"], w["d"], w["batch"], w["r"]
        c = d + 1
        ncols = batch * c
        M = srht.CSC(torch.from_numpy(w["colptr"]).cuda(), torch.from_numpy(w["rowidx"]).cuda(),
                     torch.from_numpy(w["vals"]).cuda(), (n, ncols))
        plan = srht.Plan(n, d, r, seed, batch=batch)
        out = torch.empty((batch, c, r), dtype=torch.float32, device=device)
        ws = plan.workspace(ncols)

        def step():
            plan.sketch_batched(M, out=out, workspace=ws)
        in_bytes = workloads.input_bytes_csc(int(w["colptr"][-1]), ncols)
        out_bytes = 4.0 * r * ncols
    else:
        w = workloads.config3_host(seed)
        n, d, r = w["n"], w["d"], w["r"]
        ncols = d + 1
        A = srht.CSC(torch.from_numpy(w["colptr"]).cuda(), torch.from_numpy(w["rowidx"]).cuda(),
                     torch.from_numpy(w["vals"]).cuda(), (n, d))
        bvec = torch.from_numpy(w["b"]).cuda()
        plan = srht.Plan(n, d, r, seed)
        SA = torch.empty((d, r), dtype=torch.float32, device=device).t()
        Sb = torch.empty(r, dtype=torch.float32, device=device)
        ws = plan.workspace(ncols)

        def step():
            plan.sketch(A, bvec, SA=SA, Sb=Sb, workspace=ws)
        in_bytes = workloads.input_bytes_csc(int(w["colptr"][-1]), d, dense_b_rows=n)
        out_bytes = 4.0 * r * ncols
    # L2 flush buffer (inputs of config 3 fit in L2): 2x L2
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=device)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    lib = _lib.load()
    times = []
    with ClockSampler(0) as clk:
        _lib.check(lib.srht_profile_start(args.steps), "srht_profile_start")
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
        kms_arr = (ctypes.c_float * args.steps)()
        kcount = ctypes.c_int()
        _lib.check(lib.srht_profile_stop(kms_arr, args.steps, ctypes.byref(kcount)), "srht_profile_stop")
    ms = statistics.mean(a.elapsed_time(b) for a, b in times)
    kms = statistics.mean(kms_arr[i] for i in range(kcount.value)) if kcount.value else ms
    N = plan.N
    kname = last_kernel(lib)
    # algorithmic adds per padded element with Ailon-Liberty pruning = log2 r + 1
    # (the kernels' own counts are reported beside it: the whole-column kernel does log2 N, the
    # tiled kernel log2 B + r / B with B = 2r capped at N)
    adds_per_el = float((r - 1).bit_length() + 1)
    if kname == "k_sketch_col":
        kernel_adds = float(N.bit_length() - 1)
    else:
        lb = min((r - 1).bit_length() + 1, N.bit_length() - 1, 14)
        kernel_adds = lb + r / float(1 << lb)
    adds = adds_per_el * N * ncols
    clk_mhz = clk.summary()["sm_mhz"] or 1965.0
    alu_peak = 148 * 128 * clk_mhz * 1e6 / 1e12  # T adds/s
    value = in_bytes / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "config%d_%s" % (args.config, cfg["name"]), "n": n, "d": d, "r": r,
                   "columns": ncols, "input_bytes": in_bytes, "output_bytes": out_bytes,
                   "l2": "flushed (256 MB write) before each step"},
        "roofline": {"bound": "alu", "achieved": adds / (kms * 1e-3) / 1e12, "peak": alu_peak, "unit": "Tadd/s",
                     "frac": adds / (kms * 1e-3) / 1e12 / alu_peak, "traffic": None, "kernel": kname,
                     "kernel_ms": kms, "adds_per_padded_element": adds_per_el,
                     "kernel_adds_per_padded_element": kernel_adds,
                     "hbm_equiv_GBps": (in_bytes + out_bytes) / (kms * 1e-3) / 1e9},
        "clocks": clk.summary(),
        "gpu_launches": args.steps * (2 if plan.workspace_bytes(1) > 0 else 1),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def plan_has_reduce(plan):
    return plan.workspace_bytes(1) > 0


def bind_near_gpu(device):
    """Restrict this process to the CPUs NVML reports as local to `device` (so the pinned host
    buffers are first-touched, and DMA'd, on the GPU's NUMA node).  Returns (previous affinity, note)."""
    prev = os.sched_getaffinity(0)
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            bus = torch.cuda.get_device_properties(device).pci_bus_id  # torch >= 2.x
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus if isinstance(bus, bytes) else bus.encode())
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        words = (os.cpu_count() + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        cpus = {64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1} & prev
        if cpus:
            os.sched_setaffinity(0, cpus)
            return prev, "%d host cpus local to the GPU (NVML affinity)" % len(cpus)
    except Exception as e:  # no NVML affinity: keep the current binding
        return prev, "unbound (%s)" % type(e).__name__
    return prev, "unbound"


def measure_e2e(args, plan, Ml, n, r, c, cl, world, rank, device, peers=None):
    """Host-buffer end-to-end: pinned host [A|b] shard -> device -> sketch -> host, every step."""
    import psutil
    import torch
    import torch.distributed as dist
    prev_aff, binding = bind_near_gpu(device)
    need = 4 * n * cl
    avail = psutil.virtual_memory().available
    cols = cl
    if need > 0.6 * avail:
        cols = max(1, int(0.6 * avail // (4 * n)))
    host = torch.empty((cols, n), dtype=torch.float32).pin_memory().t()
    host.copy_(Ml[:, :cols])
    if world == 1:
        # one GPU: the host-buffer C-ABI call (chunked H2D / sketch / D2H pipeline inside)
        out = torch.empty((cols, r), dtype=torch.float32).pin_memory().t()

        def e2e_step():
            plan.sketch_columns_host(host, out=out)
        api = "srht_sketch_columns_host (pinned host buffers, chunked H2D/sketch/D2H pipeline)"
        d2h = 4 * r * cols
    else:
        # N GPUs: the public multi-GPU call -- each rank copies its host shard to its device, then
        # dist.sketch_sharded (sketch + NCCL all-gather), and the full r x c sketch is read back
        from paper_0812_4547_b200 import dist as sdist
        full_h = torch.empty((c, r), dtype=torch.float32).pin_memory().t()
        full_d = torch.empty((c, r), dtype=torch.float32, device=device).t()
        ws = plan.workspace(cl)

        def e2e_step():
            Ml[:, :cols].copy_(host, non_blocking=True)
            if peers is not None:
                res = sdist.sketch_sharded_p2p(plan, Ml, c, peers, workspace=ws)
            else:
                res = sdist.sketch_sharded(plan, Ml, c, out=full_d, workspace=ws)
            full_h.copy_(res, non_blocking=True)
            torch.cuda.synchronize()
        api = ("host shard -> device (H2D), dist.sketch_sharded%s (sketch + %s), D2H of the r x c result"
               % (("_p2p", "fused gather over peer memory") if peers is not None else ("", "NCCL all-gather")))
        d2h = 4 * r * c
    e2e_step()  # warm-up
    if world > 1:
        dist.barrier()
    ts = []
    for _ in range(max(1, args.e2e_steps)):
        t0 = time.perf_counter()
        e2e_step()
        ts.append(time.perf_counter() - t0)
    t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t[0])
    total_cols = cols * world
    e2e = {"value": 4.0 * n * total_cols / sec / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * n * cols,
           "d2h_bytes_per_step": d2h, "seconds_per_step": sec, "api": api}
    if cols < cl:
        e2e["sample"] = "%d of %d columns per rank (host RAM %.0f GB available)" % (cols, cl, avail / 1e9)
    e2e["host_binding"] = binding
    del host
    os.sched_setaffinity(0, prev_aff)
    return e2e


if __name__ == "__main__":
    main()
