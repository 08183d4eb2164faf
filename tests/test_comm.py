"""C-ABI communicator (tlora_comm_*, tlora_layer_allreduce_grads): argument checks and
the no-device failure on CPU; the multi-rank NCCL check (tests/comm_check.py) when >= 2
GPUs are visible."""
import ctypes as C
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

from paper_2602_07263_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_comm_argument_errors():
    lib = capi.lib()
    h = C.c_void_p()
    idb = (C.c_uint8 * capi.UNIQUE_ID_BYTES)()
    assert lib.tlora_comm_create(0, idb, 4, 0, 3, C.byref(h)) == capi.ERR_ARG  # 3 ∤ 4
    assert "tp_size" in lib.tlora_last_error().decode()
    assert lib.tlora_comm_create(0, idb, 2, 2, 1, C.byref(h)) == capi.ERR_ARG
    assert lib.tlora_comm_create(0, None, 2, 0, 1, C.byref(h)) == capi.ERR_ARG
    assert lib.tlora_comm_info(None, None, None, None, None) == capi.ERR_ARG
    assert lib.tlora_comm_all_reduce(None, 0, None, None, 0, capi.F32, 0, None) == capi.ERR_ARG
    assert lib.tlora_comm_destroy(None) == capi.OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_comm_create_without_device_fails_cleanly():
    lib = capi.lib()
    h = C.c_void_p()
    idb = (C.c_uint8 * capi.UNIQUE_ID_BYTES)()
    assert lib.tlora_comm_create(0, idb, 1, 0, 1, C.byref(h)) == capi.ERR_NO_DEVICE
    assert h.value is None


@pytest.mark.gpu
def test_comm_multi_gpu():
    # every visible GPU up to 4; on a 1-GPU box the same check at world 1 (the code path
    # over a 1-rank communicator; the cross-rank sums need gpurun --gpus 2 / 4)
    n = max(1, min(torch.cuda.device_count(), 4))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), str(ROOT / "tests" / "comm_check.py")],
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "COMM_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
