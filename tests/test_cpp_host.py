"""The C++ hosts over the C-ABI (no PyTorch), acceptance-style binaries (one
PASS/FAIL line per criterion, exit code = failures, 77 = no GPU):
  tests/cpp/test_sklinear  -- include/skl.hpp (SkLinear) against the oracle;
  tests/cpp/test_chain_dp  -- include/skl_chain.hpp / skl_model.hpp / skl_dp.hpp:
      a reference-saved Linear/SKLinear/ReLU model file through model_forward,
      the chain backward, and the overlapped gradient all-reduce over NCCL."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINS = {"sklinear": os.path.join(ROOT, "tests", "cpp", "test_sklinear"),
        "chain_dp": os.path.join(ROOT, "tests", "cpp", "test_chain_dp")}


def _run(which):
    b = BINS[which]
    if not os.path.exists(b):
        pytest.fail(f"{b} not built (run __graft_entry__.build())")
    return subprocess.run([b, ROOT], capture_output=True, text=True, timeout=900)


@pytest.mark.parametrize("which", sorted(BINS))
def test_cpp_host_binary_builds_and_skips_without_gpu(which):
    """CPU: the binaries link libskl.so (+ the oracle / NCCL) and exit 77 (skip) when no GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    r = _run(which)
    assert r.returncode == 77, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("which", sorted(BINS))
def test_cpp_host_on_gpu(which):
    r = _run(which)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
