"""The C++ host mirror (include/skl.hpp over the C-ABI, no PyTorch) checked
against the oracle by tests/cpp/test_sklinear.cpp (acceptance-style: one
PASS/FAIL line per criterion, exit code = failures, 77 = no GPU)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_sklinear")


def _run():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built (run __graft_entry__.build())")
    return subprocess.run([BIN], capture_output=True, text=True, timeout=600)


def test_cpp_host_binary_builds_and_skips_without_gpu():
    """CPU: the binary links libskl.so + the oracle and exits 77 (skip) when no GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    r = _run()
    assert r.returncode == 77, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_host_parity_on_gpu():
    r = _run()
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
