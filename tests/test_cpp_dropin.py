"""The reference's hot-path tests restated in C++ against the drop-in headers
(include/lora_fleet/*.hpp -> C-ABI). Built by `make` (tests/cpp/_build/test_dropin)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "_build" / "test_dropin"


def _run(mode):
    if not BIN.exists():
        subprocess.run(["make", "-C", str(ROOT), "tests/cpp/_build/test_dropin"], check=True)
    p = subprocess.run([str(BIN), mode], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout


def test_dropin_cpu_cases():
    _run("cpu")


@pytest.mark.gpu
def test_dropin_gpu_cases():
    _run("gpu")
