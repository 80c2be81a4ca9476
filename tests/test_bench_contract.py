"""bench.py contract checks that run without a GPU: the reference arm (the oracle on
the host cores) prints one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "2",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["value"] > 0 and j["steps"] == 2
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in j["config"]
    # the same workload object the product arm prints (driver: same_config)
    sys.path.insert(0, ROOT)
    import bench
    from synth import argus_inputs as gen
    cfg = gen.CONFIGS["C1"]
    assert j["config"] == bench.workload_config(cfg, bench.batch_sizes(cfg, bench.n_trace(cfg)), 0, 1)


def test_product_bench_refuses_without_gpu():
    """No CPU fallback: the product arm needs the CUDA path."""
    import torch
    if torch.cuda.is_available():
        return
    out = subprocess.run([sys.executable, "bench.py", "--config", "C1", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode != 0


def test_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks (torchrun,
    127.0.0.1) which rendezvous; rank 0 alone prints the line (launcher check on CPU)."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and sorted(j["ranks"]) == [0, 1] and j["max_over_ranks"] == 1.0


def test_gpus_mismatch_refused():
    """A WORLD_SIZE that disagrees with --gpus is an error, not a silent 1-GPU run."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode != 0


def test_timed_schedule_represents_trace():
    """Any K samples the bursty trace's low / high states in proportion (the best
    matching contiguous window of the trace, in order); K >= NT runs whole passes first."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from synth import argus_inputs as gen
    sizes = gen.bursty_sizes(256, seed=2018, lo=16, hi=512)
    full = np.mean(sizes)
    hi_frac = np.mean(np.asarray(sizes) > 256)
    for K in (20, 30, 64, 100, 600):
        sch = bench.timed_schedule(sizes, K)
        assert len(sch) == K
        ts = np.asarray([sizes[b] for b in sch])
        assert abs(ts.mean() / full - 1) < 0.05, (K, ts.mean(), full)
        assert abs(np.mean(ts > 256) - hi_frac) <= 1.0 / K + 0.02, K
        rem = sch[(K // 256) * 256:]
        assert all((b - a) % 256 == 1 for a, b in zip(rem, rem[1:]))   # contiguous, in trace order
    assert bench.timed_schedule(sizes, 512) == list(range(256)) * 2
