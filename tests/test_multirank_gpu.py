"""Row sharding across processes through the product library: two torchrun ranks
share cuda:0 (gloo collectives on host-staged tensors -- NCCL needs one GPU per rank) and run the
exact library calls of the one-process-per-GPU path; rank 0's response must equal the reference's
(C1 full size, by hash) and a single-context answer (C4 parameters).  See tests/multirank_worker.py."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_row_sharded_answer(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "multirank_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "multirank ok" in out.stdout
