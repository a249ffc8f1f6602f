"""Head-sharded TP = 2 on two GPUs through the library (§8 a9): both ranks' all-reduced
outputs equal the unsharded oracle (bf16 tolerance), temporal and spatial.  One GPU per process
(tests/tp2_worker.py under torch.distributed.run, NCCL).  Skipped on a box with fewer than two GPUs —
the sharding recipe itself is pinned on CPU by tests/test_dist_cpu.py (gloo, world size 2)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="TP = 2 needs two GPUs on this box")
def test_tp2_head_sharded_matches_unsharded_oracle():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "tp2_worker.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("rel_err") == 8, r.stdout
