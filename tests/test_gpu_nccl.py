"""The torchrun / NCCL strong-scaling path for packing and MPC (and SVM
through the generic partition) end to end at one rank: NcclRank builds the
rank's partition plan, attaches NCCL and runs the captured iteration; the
gathered state must equal the single-plan run.  (At world 1 every
variable is local; the cut exchange itself is validated on one device by
tests/test_gpu_partition.py's LocalGroup and over gloo by
tests/test_partition.py.)"""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["pack", "mpc", "svm", "mpc_rank", "pack_rank"])
def test_nccl_rank_world1_matches_single_plan(gpu, name):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port),
                        os.path.join(ROOT, "tests", "nccl_rank_check.py"), name, "12"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["world"] == 1 and d["iterations"] == 12 and d["launches"] > 0
    assert d["history_rows"] == 12
    assert d["bitwise"], d["rel_err"]


def _torchrun(name, nproc, env_extra, iters=12):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", str(nproc), "--master-addr", "127.0.0.1",
                        "--master-port", str(port),
                        os.path.join(ROOT, "tests", "nccl_rank_check.py"), name, str(iters)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("name", ["pack", "mpc_rank"])
def test_p2p_rank_world1_matches_single_plan(gpu, name):
    """Peer-memory transport at one rank: the exchange kernel stores into
    the rank's own receive buffer and raises its own flag."""
    d = _torchrun(name, 1, {"FG_TRANSPORT": "p2p"})
    assert d["transport"] == "p2p" and d["iterations"] == 12 and d["history_rows"] == 12
    # counted from the captured graph's kernel nodes: the partition passes
    # and the residual step (local sums, exchange and commit in one
    # k_reduce_p2p launch) every iteration
    assert d["launches"] >= 2 * d["iterations"]
    assert d["bitwise"], d["rel_err"]


@pytest.mark.parametrize("name", ["pack", "mpc", "svm"])
def test_p2p_two_ranks_one_device(gpu, name):
    """Two processes, both on device 0, exchanging the cut and residual
    partials through CUDA IPC peer memory inside the captured iteration --
    the real multi-rank exchange the one-GPU pool can run (NCCL refuses two
    ranks on one device).  The gathered state equals the same partition
    run as a local group bit for bit, and the single-plan run to 1e-9."""
    d = _torchrun(name, 2, {"FG_TRANSPORT": "p2p", "FG_ONE_DEVICE": "1"})
    assert d["world"] == 2 and d["iterations"] == 12 and d["history_rows"] == 12
    assert d["ncut"] > 0 and d["launches"] >= 4 * d["iterations"]
    assert d["group_bitwise"] is True
    assert max(d["rel_err"].values()) <= 1e-9, d["rel_err"]


def test_p2p_lost_peer_fails_instead_of_hanging(gpu):
    """A rank that attached but never runs: the other rank's exchange kernel
    waits for its flags for the bounded 10 s, stops the run, and fg_run
    reports the lost peer (no hung GPU)."""
    d = _torchrun("lost_peer", 2, {"FG_TRANSPORT": "p2p", "FG_ONE_DEVICE": "1"}, iters=8)
    assert d["error"] is not None and "stopped answering" in d["error"], d
    assert 9.0 < d["seconds"] < 60.0, d
