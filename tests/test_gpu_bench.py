"""bench.py's product arm on the GPU prints exactly one JSON line with every
field of the benchmark contract (a small configs[0] run), and the same metric
and unit as the reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_json_contract(cuda):
    d = _run("--config", "c1", "--steps", "5", "--warmup", "3")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e",
                "cpu_baseline"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["dtype"] == "u64"
    assert "workload" in d["config"] and d["config"]["workload"].startswith("configs[0]")
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    # L2-resident filter: the binding bound is the live L2 random-sector probe
    assert r["bound"] == "l2" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 2e-3
    assert 0 < r["frac"] <= 1.1 and set(d["roofline_kernels"]) == {"add", "contains"}
    assert d["gpu_launches"] >= 2 * d["steps"]
    n = 1 << 20
    assert d["config"]["keys_per_step"] == 3 * n and d["fpr"]["negatives"] == n
    assert 0 < d["fpr"]["measured"] < 0.05
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["h2d_bytes_per_step"] == 8 * 3 * n and e["unit"] == d["unit"]
    assert e["d2h_bytes_per_step"] == 4 * (2 * n // 32)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    ref = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    rl = json.loads(ref.stdout.strip().splitlines()[-1])
    assert rl["metric"] == d["metric"] and rl["unit"] == d["unit"] and rl["config"]["workload"] == d["config"]["workload"]


def test_bench_default_legs(cuda):
    """The default line (configs[1] at iso FPR) carries the HBM leg
    (configs[2] at full size) and the fixed-load leg, each with its own
    roofline; the measured FPR of the iso leg is within 4 sigma of the
    exact model."""
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e")
    assert d["config"]["workload"].startswith("configs[1] at iso FPR")
    assert abs(d["fpr"]["z"]) <= 4
    assert d["roofline"]["bound"] == "l2"
    h = d["hbm"]
    if "skipped" not in h:
        assert h["workload"].startswith("configs[2]") and h["value"] > 0
        assert h["roofline_kernels"]["contains"]["bound"] == "hbm"
        assert h["add_path"] == "binned"
    assert d["fixed_load"]["workload"].startswith("configs[1] fixed load")


@pytest.mark.parametrize("merge", ["alltoall", "allgather", "route"])
def test_bench_under_torchrun(cuda, merge):
    """The driver's multi-GPU launch form (torch.distributed.run, one rank
    per GPU, NCCL, rendezvous on 127.0.0.1) at one rank: RANK / LOCAL_RANK /
    WORLD_SIZE come from the environment, rank 0 prints one contract line
    with n_gpus = WORLD_SIZE, for each merge strategy."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--config", "c1", "--steps", "3", "--warmup", "3", "--merge", merge,
                        "--no-cpu", "--no-e2e", "--no-probe"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("configs[0]")
