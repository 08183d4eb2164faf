"""Data-parallel gradient exchange: the copy-engine push all-reduce vs NCCL on >= 2 GPUs."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_push_allreduce_multi_gpu():
    # every visible GPU up to 4; on a 1-GPU box the same check at world 1 (the code path
    # over a 1-rank communicator; the cross-rank sums need gpurun --gpus 2 / 4)
    n = max(1, min(torch.cuda.device_count(), 4))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), str(ROOT / "tests" / "dp_check.py")],
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "DP_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
