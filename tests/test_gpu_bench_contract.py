"""bench.py end to end on a small configuration (GPU): the JSON line the driver parses keeps its
contract — metric, value, unit, n_gpus, steps, warmup, ms_per_step, higher_is_better, scaling,
dtype, data, config.workload, gpu_launches, roofline, kernel_shares, e2e, clocks — and the reference
arm prints its line with impl = reference.  (The headline numbers come from the full default run.)"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run(["--config", "3", "--steps", "3", "--warmup", "3", "--no-driver-baselines", "--no-hybrid",
              "--cpu-sample-batches", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "kernel_shares", "e2e",
              "clocks", "cpu_baseline", "payload_roofline", "batch_latency_ms", "engine_chain"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["workload"] == "cfg3-tlsf-4GiB"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["engine_chain"]["chunks"] > 0


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "3", "--steps", "2", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_per_config_side_line():
    """bench.py's per-config side measurement (configs 1-4 beside the headline): the timed batches
    captured as one CUDA graph with the library launching directly under capture, replayed once,
    every returned offset compared with Oracle-L afterwards.  Config 1 (the single-launch small-heap
    path) and config 4 (binary buddies, ~40 launches per batch) on a few batches."""
    sys.path.insert(0, ROOT)
    import torch
    import bench
    import tracegen as tg
    dev = torch.device("cuda", 0)
    flush = torch.empty(1 << 20, dtype=torch.int32, device=dev)
    for cid, nb in ((1, 0), (4, 6)):
        r = bench.run_config(tg.CONFIGS[cid], nb, dev, flush)
        assert r["parity_ok"], (cid, r["mismatch"])
        assert r["device_ops_s"] > 0 and r["oracle_ops_s"] > 0 and r["timing"].startswith("the timed batches")
