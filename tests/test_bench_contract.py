"""bench.py's one-line JSON contract: the reference arm on the CPU, the
device arm (small workload) on a GPU, and the weak-scaling size rule."""

import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--workload", "pack100", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["higher_is_better"] is True
    # the reference itself (baseline/_ref) when installed, else the oracle port
    import bench
    kind = "reference" if bench.reference_package() is not None else "port"
    assert d["cpu_baseline"]["kind"] == kind and d["cpu_baseline"]["value"] == d["value"]
    assert d["config"]["same_config"] is True
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"] == "pack100"


def test_points_per_rank_rule(monkeypatch):
    import bench
    args = types.SimpleNamespace(points_per_rank=3_000_000)
    assert bench.points_per_rank(args, 8) == 3_000_000
    args = types.SimpleNamespace(points_per_rank=None)
    import psutil

    class VM:
        def __init__(self, avail):
            self.available = avail

    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    monkeypatch.setattr(psutil, "virtual_memory", lambda: VM(2 * 2**40))
    assert bench.points_per_rank(args, 8) == 8_000_000          # 2 TB host: configs[4]
    monkeypatch.setattr(psutil, "virtual_memory", lambda: VM(2**40))
    assert bench.points_per_rank(args, 8) == 8_000_000          # 1 TB host: configs[4]
    monkeypatch.setattr(psutil, "virtual_memory", lambda: VM(200 * 2**30))
    assert bench.points_per_rank(args, 8) == 2_000_000
    monkeypatch.setattr(psutil, "virtual_memory", lambda: VM(50 * 2**30))
    assert bench.points_per_rank(args, 8) == 1_000_000          # floor
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    n = bench.points_per_rank(args, 1)
    assert 1_000_000 <= n <= 8_000_000 and n % 1_000_000 == 0


@pytest.mark.gpu
def test_device_arm_line(gpu):
    d = _run(["--workload", "pack100", "--steps", "20", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == r["achieved"] / r["peak"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


@pytest.mark.gpu
def test_multi_gpu_mpc_rank_graph_arm_at_one_rank(gpu):
    """The strong-scaled MPC arm builds its rank graph from the spec alone
    (partition.mpc_rank_graph) and runs it through NcclRank at one rank."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--partition", "--workload", "mpc100k",
                        "--steps", "12", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert BASE_KEYS <= set(d)
    assert d["scaling"] == "strong" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["rank_graph"] == "mpc_rank_graph" and d["config"]["edges"] == 300002


@pytest.mark.gpu
def test_multi_gpu_packing_rank_graph_arm_at_one_rank(gpu):
    """The strong-scaled packing arm builds its rank graph from the spec
    alone (partition.packing_rank_graph) and runs it through NcclRank."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--partition", "--workload", "pack100",
                        "--steps", "10", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["scaling"] == "strong" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["rank_graph"] == "packing_rank_graph" and d["config"]["edges"] == 20500


@pytest.mark.gpu
def test_multi_gpu_arm_line_at_one_rank(gpu):
    """The torchrun / NCCL arm (factor-partitioned SVM rank graph, NCCL
    all-gather inside the captured iteration) end to end at one rank."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--partition", "--points-per-rank", "200000",
                        "--steps", "6", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["points_per_rank"] == 200000 and d["chain_form"] in ("unit", "fast")
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
