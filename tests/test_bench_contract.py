"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle) prints one JSON
line with the metric, the e2e and cpu_baseline objects, and only rank 0 prints under torchrun."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                        "--warmup", "1", *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return [l for l in p.stdout.splitlines() if l.strip().startswith("{")]


def test_reference_arm_json_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("config1")


def test_reference_arm_only_rank0_prints():
    env = {"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2", "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": "29533"}
    assert _run(env, "--gpus", "2") == []


def test_cpu_baseline_workers_bounded():
    # the all-cores oracle leg: at most one process per host core and per column, at least one
    sys.path.insert(0, ROOT)
    import bench
    for cfg in (1, 4, 5):
        w, cores = bench.oracle_workers(cfg)
        assert 1 <= w <= cores == len(os.sched_getaffinity(0))
        import workloads
        assert w <= workloads.CONFIGS[cfg]["d"]


def test_cpu_baseline_parallel_leg_runs():
    # two workers on config 1 (tiny): the JSON object carries both legs and the core counts
    sys.path.insert(0, ROOT)
    import bench
    v, t, desc = bench.time_oracle_parallel(1, 2)
    assert v > 0 and t > 0 and desc.startswith("2 worker processes")
