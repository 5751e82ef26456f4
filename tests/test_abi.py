"""CPU tests of the C-ABI boundary (include/skl.h <-> libskl.so): the library
loads, exports exactly what the header declares, its host-side logic matches
the reference contracts, and without a GPU every compute entry point fails
loudly (no CPU fallback)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

import paper_2601_15473_b200 as skl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "skl.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_path():
    fns = declared_functions()
    for f in ("sketched_linear_forward", "sketched_linear_backward", "skl_generate_sketches", "skl_init_params",
              "skl_workspace_size", "skl_allreduce_grads", "skl_last_error", "skl_derive_seed"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = skl.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", skl.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for f in declared_functions():
        assert f in exported, f
        assert getattr(lib, f) is not None
    assert set(skl.ABI_SYMBOLS) <= set(declared_functions())


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", skl.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_contracts(port):
    assert skl.lib().skl_rng_algorithm().decode() == "splitmix64-boxmuller-v1"  # rng.hpp:10
    for m, i in ((42, 0), (42, 1000), (0, 7), (2**64 - 1, 3)):
        assert skl.derive_seed(m, i) == port.derive_seed(m, i)
    s = skl.shape(8192, 8192, 1, 16)
    learn, stored, dense = skl.params(s)
    assert stored - 8192 == 524288 and dense - 8192 == 67108864 and learn == 16 * 16384 + 8192
    assert skl.exceeds_dense(2, 64, 256, 256) and not skl.exceeds_dense(1, 64, 256, 256)


def test_parameter_and_shape_errors():
    with pytest.raises(skl.ParameterError):
        skl.params(skl.shape(8, 8, 0, 4))          # nn_layers.cpp:116
    with pytest.raises(skl.ParameterError):
        skl.workspace_size(skl.shape(8, 8, 2, 0), 16)
    with pytest.raises(skl.ShapeError):
        skl.workspace_size(skl.shape(8, 8, 1, 4), -1)
    with pytest.raises(skl.ShapeError):
        skl.params(skl.shape(0, 8, 1, 4))


def test_workspace_plan_is_monotone_in_tokens():
    s = skl.shape(768, 3072, 2, 128)
    f1, b1 = skl.workspace_size(s, 1024)
    f2, b2 = skl.workspace_size(s, 32768)
    assert 0 < f1 <= f2 and 0 < b1 <= b2
    assert b2 >= 32768 * 512 * 2  # backward keeps P [T, R] (bf16)


def test_compute_fails_loudly_without_gpu():
    """No CPU fallback: compute entry points report SKL_ERR_CUDA on a GPU-less host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    s = skl.shape(64, 64, 1, 16)
    lib = skl.lib()
    rc = lib.skl_generate_sketches(ctypes.byref(s), 0, 1, None, None, None)
    assert rc == 3 and b"no CUDA device" in lib.skl_last_error()
    rc = lib.sketched_linear_forward(ctypes.byref(s), 16, *([ctypes.c_void_p(16)] * 9), 1 << 30, None)
    assert rc == 3


def test_unaligned_shapes_are_accepted():
    """Any shape the reference accepts is a valid call (nn_layers.cpp:61-101):
    rows that are not 16-byte multiples are staged as zero-padded copies, so the
    workspace query covers the padded layer plus the copies, and a compute call
    gets as far as the device check (no SKL_ERR_UNSUPPORTED)."""
    import torch
    s = skl.shape(6, 8, 2, 3)  # test_nn_layers.cpp:158 GradCheck shape: d_in*2 bytes not 16-B aligned
    f, b = skl.workspace_size(s, 4)
    fa, ba = skl.workspace_size(skl.shape(8, 8, 2, 3), 4)  # the padded layer itself
    assert f > fa and b > ba
    for dt in (skl.BF16, skl.F32_TF32):
        assert min(skl.workspace_size(skl.shape(7, 13, 1, 5, dt), 33)) > 0
    n = ctypes.c_size_t()
    assert skl.lib().skl_from_dense_workspace_size(ctypes.byref(skl.shape(6, 8, 4, 3)), ctypes.byref(n)) == 0
    assert n.value > 0
    if torch.cuda.is_available():
        return
    rc = skl.lib().sketched_linear_forward(ctypes.byref(s), 4, *([ctypes.c_void_p(16)] * 9), 1 << 30, None)
    assert rc == 3 and b"no CUDA device" in skl.lib().skl_last_error()


def test_dense_linear_contract():
    """DenseLinear entry points (skl.h): workspace query for aligned and ragged
    shapes, shape / parameter errors before any device work."""
    import torch
    s = skl.dense_shape(768, 3072)
    f, b = skl.dense_workspace_size(s, 1024)
    assert f > 0 and b >= 768 * 1024 * 2          # backward stages xᵀ
    assert min(skl.dense_workspace_size(skl.dense_shape(6, 8, skl.F32_TF32), 2)) > 0
    with pytest.raises(skl.ShapeError):
        skl.dense_workspace_size(skl.dense_shape(0, 8), 2)
    with pytest.raises(skl.ShapeError):
        skl.dense_workspace_size(s, -1)
    lib = skl.lib()
    vp = ctypes.c_void_p
    # bad fuse flag / missing grad_W: parameter errors
    assert lib.dense_linear_forward(ctypes.byref(s), 4, skl.FUSE_RELU_IN, *([vp(16)] * 4), vp(16), 1 << 30,
                                    None) == 2
    assert lib.dense_linear_backward(ctypes.byref(s), 4, 0, *([vp(16)] * 4), None, None, vp(16), 1 << 30,
                                     None) == 2
    if not torch.cuda.is_available():
        assert lib.dense_linear_forward(ctypes.byref(s), 4, 0, *([vp(16)] * 4), vp(16), 1 << 30, None) == 3


def test_relu_bits_contract():
    """1-bit ReLU mask entry points (skl.h SKL_FUSE_RELU_BITS): row stride in
    64-column groups, support query, and parameter errors raised before any
    device work."""
    import ctypes
    assert skl.relu_bits_row_words(1) == 2
    assert skl.relu_bits_row_words(64) == 2
    assert skl.relu_bits_row_words(160) == 6
    assert skl.relu_bits_row_words(3072) == 96
    assert skl.relu_bits_supported(skl.shape(768, 3072, 2, 128, skl.BF16))       # CTA-pair b2b kernel
    assert not skl.relu_bits_supported(skl.shape(4096, 4096, 3, 256, skl.BF16))  # R = 1536: unfused chain
    lib = skl.lib()
    s = skl.shape(768, 3072, 2, 128, skl.BF16)
    vp = ctypes.c_void_p
    dummy = vp(16)
    # BITS without RELU_OUT, and RELU_OUT|BITS without a buffer: parameter errors
    # forward_bits(shape, T, fuse, x, S1s, S2s, U1s, U2s, bias, y, saved, relu_bits, ws, ws_bytes, stream)
    st = lib.sketched_linear_forward_bits(ctypes.byref(s), 8, skl.FUSE_RELU_BITS, *([dummy] * 8), dummy, None, 0, None)
    assert st == 2
    st = lib.sketched_linear_forward_bits(ctypes.byref(s), 8, skl.FUSE_RELU_OUT | skl.FUSE_RELU_BITS,
                                          *([dummy] * 8), None, None, 0, None)
    assert st == 2
    # backward_bits(shape, T, phases, fuse, g, x, saved, S1s, S2s, U1s, U2s, gx, dU1s, dU2s, db, relu_bits, ws, ...)
    st = lib.sketched_linear_backward_bits(ctypes.byref(s), 8, skl.BWD_ALL, skl.FUSE_RELU_BITS, *([dummy] * 11),
                                           dummy, None, 0, None)
    assert st == 2
