"""Multi-GPU parity: p ranks, one process per GPU, each owning a contiguous
cost-balanced slice of both leaf lists, partial products summed over the ranks
(P:578-587): NCCL, then libhm's peer-memory collectives (hm_p2p_import; the GMRES
normalisation publishes the next product's x).  Runs tools/multi_rank_check.py under torchrun
when the box has >= 2 GPUs; skipped on a 1-GPU box.  Bars: owned ranges tile both lists;
p-rank matvec vs the 1-rank matvec <= 1e-13 relative; p-rank GMRES / CG solutions vs 1-rank
<= 1e-8; P2P vs NCCL solutions <= 1e-12 with equal iteration counts (see the script)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg", ["C1", "C2", "C1odd"])   # C1odd: N = 1279, N mod p != 0
def test_two_rank_matvec_and_solve(cfg):
    if _ngpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "multi_rank_check.py"), cfg]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["world"] == 2
