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
