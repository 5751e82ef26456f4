"""Model files: the reference's JSON manifest + 'PNTR' blob, on the device.

Mirror of rnla::nn::model_save / model_load (nn_model.cpp:396-531) for the
layers of Linear/SKLinear/ReLU chains plus SKConv2d / Conv2d.  A manifest stores each SKLinear's
sketches as DESCRIPTORS (dist, rows, cols, seed; nn_model.cpp:250-265) and the
blob stores only the learnable U1/U2 and the bias, f32 or f64 little-endian,
after the 5-byte header 'PNTR' + version 1 (nn_model.cpp:196-246,303-311).
Loading re-realises the sketches on the GPU from their seeds -- bit-identical
to SketchOp::realized -- under the same rng_algorithm guard
(nn_model.cpp:453-454), so a model the reference saved runs here unchanged,
and a model saved here loads in the reference.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import BF16, DenseLinear, LoadError, ParameterError, ShapeError, SkLinear, lib
from .model import Relu, SkChain

MAGIC = b"PNTR"
BLOB_VERSION = 1


def _blob_path(path):
    return path + ".bin"   # blob_path_for, nn_model.cpp:392


class _Reader:
    def __init__(self, data: bytes, f32: bool, offset: int):
        self.data, self.f32, self.pos = data, f32, offset

    def read(self, count: int) -> np.ndarray:
        width = 4 if self.f32 else 8
        end = self.pos + count * width
        if end > len(self.data):
            raise LoadError(9, "model blob too short for declared layers")
        a = np.frombuffer(self.data, dtype="<f4" if self.f32 else "<f8", count=count, offset=self.pos)
        self.pos = end
        return a.astype(np.float64)


class DenseConv2d:
    """A dense Conv2d layer of a model file (layers.hpp:122-142): its conv shape
    and lowered DenseLinear.  Loaded and saved so that files holding one round
    trip; like the reference's model_forward (nn_model.cpp:117-119), a chain
    refuses it."""

    def __init__(self, shape, inner: DenseLinear):
        self.shape, self.inner = shape, inner


class Model:
    """rnla::nn::Model (model.hpp): named layers of one model file.  forward()
    is model_forward (nn_model.cpp:111-122): Linear / SKLinear / ReLU only,
    ShapeError on any other layer, as in the reference."""

    def __init__(self, layers, names, dtype="f32"):
        self.layers, self.names, self.dtype = list(layers), list(names), dtype
        self._chain = None

    def chain(self) -> SkChain:
        if self._chain is None:
            self._chain = SkChain(self.layers)
        return self._chain

    def forward(self, x, train=False):
        return self.chain().forward(x, train=train)

    def find(self, name):
        return self.layers[self.names.index(name)] if name in self.names else None

    def __iter__(self):  # `chain, names = model_load(...)` (Linear/SKLinear/ReLU files)
        return iter((self.chain(), self.names))


def _conv_shape(j):
    from .conv import ConvShape
    return ConvShape(j["c_in"], j["c_out"], j["kernel_h"], j["kernel_w"], j["stride"], j["padding"])


def _sk_from_json(j, rd, dtype, device):
    """sk_linear_from_json (nn_model.cpp:290-311)."""
    d_in, d_out, L, k = j["d_in"], j["d_out"], j["num_terms"], j["low_rank"]
    sk = j["sketches"]
    if len(sk) != 2 * L:
        raise LoadError(9, "SKLinear manifest: expected 2*num_terms sketches")
    u1 = np.empty((L, k, d_in))
    u2 = np.empty((L, d_out, k))
    for i in range(L):        # blob order: u1_0, u2_0, u1_1, u2_1, ..., bias
        u1[i] = rd.read(k * d_in).reshape(k, d_in)
        u2[i] = rd.read(d_out * k).reshape(d_out, k)
    bias = rd.read(d_out)
    desc = [(s["dist"], s["rows"], s["cols"], s["seed"]) for s in sk]
    return SkLinear.from_parts(d_in, d_out, L, k, desc, u1, u2, bias, dtype=dtype, device=device)


def model_load(path, dtype=BF16, device="cuda"):
    """-> Model (unpacks as (SkChain, [layer names]) for chain files).  Raises
    LoadError like model_load (nn_model.cpp:448-531).  Layer types: Linear,
    SKLinear, ReLU, SKConv2d and Conv2d; attention layers are not on this path."""
    try:
        with open(path, "rb") as f:
            root = json.loads(f.read().decode())
    except OSError as e:
        raise LoadError(9, f"model_load: cannot open {path}") from e
    except (ValueError, UnicodeDecodeError) as e:
        raise LoadError(9, f"model_load: malformed manifest: {e}") from e
    try:
        if root["format_version"] != 1:
            raise LoadError(9, "model_load: unsupported format_version")
        if root["rng_algorithm"] != lib().skl_rng_algorithm().decode():
            raise LoadError(9, "model_load: manifest uses an unknown rng_algorithm")
        mdt = root["dtype"]
        if mdt not in ("f32", "f64"):
            raise LoadError(9, f"model_load: unsupported dtype {mdt}")
        try:
            with open(_blob_path(path), "rb") as f:
                blob = f.read()
        except OSError as e:
            raise LoadError(9, f"model_load: cannot open {_blob_path(path)}") from e
        if len(blob) < 5 or blob[:4] != MAGIC:
            raise LoadError(9, "model_load: bad blob magic")
        if blob[4] != BLOB_VERSION:
            raise LoadError(9, "model_load: unsupported blob version")
        rd = _Reader(blob, mdt == "f32", 5)
        layers, names = [], []
        for j in root["layers"]:
            name, typ = j["name"], j["type"]
            if name in names:
                raise LoadError(9, f"model_load: duplicate layer name {name}")
            if typ == "SKLinear":
                layers.append(_sk_from_json(j, rd, dtype, device))
            elif typ == "Linear":      # nn_model.cpp:473-481: w [d_out][d_in] then b
                d_in, d_out = j["d_in"], j["d_out"]
                w = rd.read(d_out * d_in).reshape(d_out, d_in)
                layers.append(DenseLinear.from_parts(w, rd.read(d_out), dtype=dtype, device=device))
            elif typ == "ReLU":
                layers.append(Relu())
            elif typ == "SKConv2d":    # nn_model.cpp:492-500
                from .conv import SkConv2d
                shape = _conv_shape(j)
                inner = _sk_from_json(j, rd, dtype, device)
                if inner.d_in != shape.lowered_d_in() or inner.d_out != shape.c_out:
                    raise LoadError(9, "SKConv2d manifest: inner dims disagree with conv shape")
                layers.append(SkConv2d(shape, inner.num_terms, inner.low_rank, dtype=dtype, inner=inner))
            elif typ == "Conv2d":      # nn_model.cpp:483-490
                shape = _conv_shape(j)
                d_in = shape.lowered_d_in()
                w = rd.read(shape.c_out * d_in).reshape(shape.c_out, d_in)
                layers.append(DenseConv2d(shape, DenseLinear.from_parts(w, rd.read(shape.c_out), dtype=dtype,
                                                                        device=device)))
            elif typ in ("MultiheadAttention", "RandMultiheadAttention"):
                raise ShapeError(1, f"model_load: layer '{name}' ({typ}) is not on the SKLinear path")
            else:
                raise LoadError(9, f"unknown layer type: {typ}")   # layer_type_from_name, nn_model.cpp:43-52
            names.append(name)
        if rd.pos != len(blob):
            raise LoadError(9, "model_load: blob length does not match manifest")
    except KeyError as e:
        raise LoadError(9, f"model_load: malformed manifest: missing {e}") from e
    return Model(layers, names, mdt)


def model_save(layers, path, dtype="f32", names=None):
    """model_save (nn_model.cpp:396-440) of a list of SkLinear / DenseLinear / Relu /
    SkConv2d / DenseConv2d layers.  Parameters are read back from the device
    (their stored precision)."""
    if dtype not in ("f32", "f64"):
        raise ParameterError(2, "model_save: dtype must be f64 or f32")
    layers = list(layers)
    names = list(names) if names is not None else [f"layer{i}" for i in range(len(layers))]
    if len(names) != len(layers):
        raise ParameterError(2, f"model_save: {len(names)} names for {len(layers)} layers")
    out = bytearray(MAGIC + bytes([BLOB_VERSION]))
    npdt = "<f4" if dtype == "f32" else "<f8"
    js = []

    def put(t):
        nonlocal out
        out += t.detach().double().cpu().numpy().astype(npdt).tobytes()

    def conv_json(shape):
        return {"c_in": shape.c_in, "c_out": shape.c_out, "kernel_h": shape.kernel_h, "kernel_w": shape.kernel_w,
                "stride": shape.stride, "padding": shape.padding}

    from .conv import SkConv2d
    for name, lyr in zip(names, layers):
        if isinstance(lyr, Relu):
            js.append({"name": name, "type": "ReLU"})
            continue
        if isinstance(lyr, DenseLinear):   # nn_model.cpp:369-371, 405-407
            put(lyr.W)
            put(lyr.bias)
            js.append({"name": name, "type": "Linear", "d_in": lyr.d_in, "d_out": lyr.d_out})
            continue
        if isinstance(lyr, DenseConv2d):
            put(lyr.inner.W)
            put(lyr.inner.bias)
            js.append({"name": name, "type": "Conv2d", **conv_json(lyr.shape)})
            continue
        conv = None
        if isinstance(lyr, SkConv2d):
            conv, lyr = lyr, lyr.inner
        if not isinstance(lyr, SkLinear):
            raise ShapeError(1, f"model_save: layer '{name}' is not on the SKLinear path")
        L, k = lyr.num_terms, lyr.low_rank
        U2 = lyr.U2s.detach().double().cpu().numpy()   # [L, d_in, k] = u1ᵀ
        U1 = lyr.U1s.detach().double().cpu().numpy()   # [L, k, d_out] = u2ᵀ
        for i in range(L):
            out += np.ascontiguousarray(U2[i].T).astype(npdt).tobytes()
            out += np.ascontiguousarray(U1[i].T).astype(npdt).tobytes()
        out += lyr.bias.detach().double().cpu().numpy().astype(npdt).tobytes()
        ent = {"name": name, "type": "SKConv2d" if conv else "SKLinear"}
        if conv:
            ent.update(conv_json(conv.shape))
        ent.update({"d_in": lyr.d_in, "d_out": lyr.d_out, "num_terms": L, "low_rank": k,
                    "sketches": [{"dist": d, "rows": r, "cols": c, "seed": int(sd)} for (d, r, c, sd) in lyr.sketches]})
        js.append(ent)
    manifest = {"format_version": 1, "rng_algorithm": lib().skl_rng_algorithm().decode(), "dtype": dtype,
                "layers": js}
    with open(path, "w") as f:
        f.write(json.dumps(manifest, indent=2) + "\n")
    with open(_blob_path(path), "wb") as f:
        f.write(bytes(out))
