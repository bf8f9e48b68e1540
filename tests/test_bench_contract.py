"""bench.py's reference arm (the fp64 oracle on the host cores, the one leg that runs
without a GPU) prints one JSON line with the driver's contract keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("flightline 598x20000x72")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_json_contract():
    """The GPU arm's line: roofline (bound, achieved, peak, unit, frac, traffic), clocks,
    gpu_launches, and an end-to-end number with the H2D/D2H bytes it moved."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3",
                          "--e2e-steps", "1", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] == 2 * 65   # K0, K1, K2-init, 31 sweeps, 30 updates, status copy
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 598 * 20000 * 72 * 4 and e["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_gpu_arm_multi_rank_plumbing():
    """The N > 1 launch path (torchrun, --split columns): each rank retrieves its contiguous
    column range of one flightline, the time is the max over ranks, rank 0 prints one line.
    On a one-GPU box the two ranks share the device (gloo): checks the plumbing and the
    contract keys only -- the number is not a measurement."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--config", "segment", "--steps", "2", "--warmup", "3", "--e2e-steps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["parallelism"] == "columns/2"
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 598 * 2000 * 72 * 4
