"""Model files (nn_model.cpp:396-531): the reference's JSON manifest + PNTR
blob.  Fixtures tests/golden/ref_model_{f32,f64}.json(+.bin) were written by
the reference's own model_save (tests/golden/make_golden_model.py), with the
reference's model_forward output of a seeded input stored beside them."""
from __future__ import annotations

import json
import os
import shutil

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _fromhex(lst):
    return np.array([float.fromhex(v) for v in lst])


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_reference_blob_layout(dt):
    """Blob = 'PNTR' + version 1 + per SKLinear (u1_i, u2_i)*L + bias, f32/f64 LE."""
    path = os.path.join(GOLD, f"ref_model_{dt}.json")
    m = json.load(open(path))
    blob = open(path + ".bin", "rb").read()
    assert blob[:4] == b"PNTR" and blob[4] == 1
    n = sum(l["num_terms"] * l["low_rank"] * (l["d_in"] + l["d_out"]) + l["d_out"]
            for l in m["layers"] if l["type"] == "SKLinear")
    assert len(blob) == 5 + n * (4 if dt == "f32" else 8)
    assert m["rng_algorithm"] == "splitmix64-boxmuller-v1"


def _tamper(tmp_path, key=None, value=None, blob_edit=None):
    src = os.path.join(GOLD, "ref_model_f32.json")
    dst = str(tmp_path / "m.json")
    m = json.load(open(src))
    if key:
        m[key] = value
    json.dump(m, open(dst, "w"))
    b = bytearray(open(src + ".bin", "rb").read())
    if blob_edit:
        b = blob_edit(b)
    open(dst + ".bin", "wb").write(bytes(b))
    return dst


@pytest.mark.parametrize("case", ["rng", "version", "dtype", "magic", "blobver"])
def test_load_errors_before_any_device_work(tmp_path, case):
    """model_load's guards (nn_model.cpp:448-466) raise LoadError."""
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.model_io import model_load
    p = {"rng": lambda: _tamper(tmp_path, "rng_algorithm", "mt19937"),
         "version": lambda: _tamper(tmp_path, "format_version", 2),
         "dtype": lambda: _tamper(tmp_path, "dtype", "f16"),
         "magic": lambda: _tamper(tmp_path, blob_edit=lambda b: b"XXXX" + b[4:]),
         "blobver": lambda: _tamper(tmp_path, blob_edit=lambda b: b[:4] + bytes([2]) + b[5:])}[case]()
    with pytest.raises(skl.LoadError):
        model_load(p)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("variant", ["bf16", "tf32"])
def test_reference_saved_model_runs_on_device(dt, variant):
    """A model the REFERENCE saved loads here (sketches re-realised on the GPU
    from their seeds) and reproduces the reference's model_forward."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.model_io import model_load
    from tests._util import check_close
    g = json.load(open(os.path.join(GOLD, "ref_model_forward.json")))
    T = g["T"]
    x = _fromhex(g["x"]).reshape(64, T)             # column convention
    y_ref = _fromhex(g[f"y_{dt}"]).reshape(40, T)
    dtype = skl.BF16 if variant == "bf16" else skl.F32_TF32
    chain, names = model_load(os.path.join(GOLD, f"ref_model_{dt}.json"), dtype=dtype)
    assert names == [f"layer{i}" for i in range(5)]
    X = torch.from_numpy(x.T.copy()).to("cuda", skl.torch_dtype(dtype))
    y = chain.forward(X, train=False)
    torch.cuda.synchronize()
    # compare against the reference on the same (rounded) input
    check_close(f"model_forward {dt} -> {variant}", y.double().cpu().numpy(), y_ref.T, variant)


@pytest.mark.gpu
def test_model_saved_here_loads_in_reference(tmp_path):
    """Round trip: model_save of the device layers -> the reference's own
    model_load + model_forward (oracle/_ref) == the device forward."""
    import ctypes
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.model_io import model_load, model_save
    from tests._util import check_close
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    ref = oracle.Oracle("reference")
    if not hasattr(ref.lib, "ref_model_forward_file"):
        pytest.skip("reference built without nn_model.cpp")
    chain, names = model_load(os.path.join(GOLD, "ref_model_f32.json"), dtype=skl.F32_TF32)
    out = str(tmp_path / "saved.json")
    model_save(chain.layers(), out, dtype="f64", names=names)
    g = json.load(open(os.path.join(GOLD, "ref_model_forward.json")))
    T = g["T"]
    x = _fromhex(g["x"]).reshape(64, T)
    y = np.empty((40, T))
    f = ref.lib.ref_model_forward_file
    f.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double),
                  ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
    assert f(out.encode(), 64, T, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 40,
             y.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
    X = torch.from_numpy(x.T.copy()).to("cuda", torch.float32)
    y_dev = chain.forward(X, train=False).double().cpu().numpy()
    check_close("reference model_forward of a file saved here", y_dev, y.T, "tf32")


def test_mixed_reference_blob_layout():
    """A reference-saved model with a Linear layer: w [d_out][d_in] then b in the
    blob (nn_model.cpp:405-407), between the SKLinear records."""
    path = os.path.join(GOLD, "ref_model_mixed_f64.json")
    m = json.load(open(path))
    assert [l["type"] for l in m["layers"]] == ["SKLinear", "ReLU", "Linear", "ReLU", "SKLinear"]
    n = 0
    for l in m["layers"]:
        if l["type"] == "SKLinear":
            n += l["num_terms"] * l["low_rank"] * (l["d_in"] + l["d_out"]) + l["d_out"]
        elif l["type"] == "Linear":
            n += l["d_in"] * l["d_out"] + l["d_out"]
    assert len(open(path + ".bin", "rb").read()) == 5 + 8 * n


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("variant", ["bf16", "tf32"])
def test_reference_saved_mixed_model_runs_on_device(dt, variant, tmp_path):
    """A reference-saved Linear/SKLinear/ReLU model with ragged widths (50, k = 5)
    loads here and reproduces the reference's model_forward; saving it again
    here gives a file the reference's model_load + model_forward accept with the
    same output."""
    import ctypes
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.model_io import model_load, model_save
    from tests._util import check_close
    g = json.load(open(os.path.join(GOLD, "ref_model_mixed_forward.json")))
    T = g["T"]
    x = _fromhex(g["x"]).reshape(64, T)
    y_ref = _fromhex(g[f"y_{dt}"]).reshape(40, T)
    dtype = skl.BF16 if variant == "bf16" else skl.F32_TF32
    model = model_load(os.path.join(GOLD, f"ref_model_mixed_{dt}.json"), dtype=dtype)
    assert isinstance(model.layers[2], skl.DenseLinear)
    X = torch.from_numpy(x.T.copy()).to("cuda", skl.torch_dtype(dtype))
    y = model.forward(X)
    torch.cuda.synchronize()
    check_close(f"mixed model_forward {dt} -> {variant}", y.double().cpu().numpy(), y_ref.T, variant)
    if variant != "tf32" or not oracle.available("reference"):
        return
    ref = oracle.Oracle("reference")
    out = str(tmp_path / "mixed.json")
    model_save(model.layers, out, dtype="f64", names=model.names)
    y2 = np.empty((40, T))
    f = ref.lib.ref_model_forward_file
    f.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_double),
                  ctypes.c_uint64, ctypes.POINTER(ctypes.c_double)]
    assert f(out.encode(), 64, T, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 40,
             y2.ctypes.data_as(ctypes.POINTER(ctypes.c_double))) == 0
    check_close("reference model_forward of the re-saved mixed model", y.double().cpu().numpy(), y2.T, "tf32")


@pytest.mark.gpu
def test_conv_layers_load_but_model_forward_refuses(tmp_path):
    """SKConv2d / Conv2d layers load (nn_model.cpp:483-500) but, as in the
    reference's model_forward (nn_model.cpp:117-119), a chain refuses them."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("layers are device-resident")
    import paper_2601_15473_b200 as skl
    from paper_2601_15473_b200.conv import ConvShape, SkConv2d
    from paper_2601_15473_b200.model_io import DenseConv2d, model_load, model_save
    conv = SkConv2d(ConvShape(2, 3, 3, 3, 1, 1), 1, 4, seed=3, dtype=skl.F32_TF32)
    dconv = DenseConv2d(ConvShape(3, 2, 1, 1, 1, 0), skl.DenseLinear(3, 2, seed=4, dtype=skl.F32_TF32))
    p = str(tmp_path / "conv.json")
    model_save([conv, dconv], p, dtype="f32")
    m = model_load(p, dtype=skl.F32_TF32)
    assert isinstance(m.layers[0], SkConv2d) and isinstance(m.layers[1], DenseConv2d)
    assert torch.equal(m.layers[0].inner.U1s, conv.inner.U1s)
    with pytest.raises(skl.ShapeError):
        m.forward(torch.zeros(4, 18, device="cuda"))
