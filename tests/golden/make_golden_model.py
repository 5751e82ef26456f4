#!/usr/bin/env python3
"""Generate tests/golden/ref_model_{f32,f64}.json(+.bin) with the REFERENCE's own
model_save (nn_model.cpp:396-440, via oracle/_ref/librnla_ref.so built from the
unmodified sources + oracle/ref_model_shim.cpp), and the reference's
model_forward (nn_model.cpp:111-122) of a seeded input through each file.

    make -C oracle && python tests/golden/make_golden_model.py

The chain: SKLinear(64->96, L2, k16, Gaussian) + ReLU + SKLinear(96->48, L1,
k32, Rademacher) + ReLU + SKLinear(48->40, L1, k8, Gaussian); nonzero biases.
The mixed chain (ref_model_mixed_*): SKLinear(64->96, L2, k16) + ReLU +
Linear(96->50, dense_linear_init) + ReLU + SKLinear(50->40, L1, k5) -- a dense
layer and ragged widths (50, k = 5), as a tuner-produced model has them.
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

# type (0 SKLinear, 1 ReLU), d_in, d_out, l, k, seed, dist
SPEC = [(0, 64, 96, 2, 16, 101, 0), (1, 0, 0, 0, 0, 0, 0), (0, 96, 48, 1, 32, 202, 1), (1, 0, 0, 0, 0, 0, 0),
        (0, 48, 40, 1, 8, 303, 0)]
T = 20
MIXED = [(0, 64, 96, 2, 16, 101, 0), (1, 0, 0, 0, 0, 0, 0), (2, 96, 50, 0, 0, 202, 0), (1, 0, 0, 0, 0, 0, 0),
         (0, 50, 40, 1, 5, 303, 0)]


def main():
    ref = oracle.Oracle("reference")
    lib = ref.lib
    lib.ref_model_save_chain.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_uint64)]
    lib.ref_model_forward_file.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_double), ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_double)]
    lib.ref_model_last_error.restype = ctypes.c_char_p
    spec = np.array(SPEC, dtype=np.uint64).ravel()
    x = ref.gaussian_matrix(64, T, 7)  # column convention [d_in x T]
    out = {"generator": "tests/golden/make_golden_model.py", "spec": SPEC, "T": T, "x_seed": 7,
           "x": [float(v).hex() for v in x.ravel()]}
    for dt in ("f32", "f64"):
        path = os.path.join(HERE, f"ref_model_{dt}.json")
        rc = lib.ref_model_save_chain(path.encode(), 1 if dt == "f32" else 0, len(SPEC),
                                      spec.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        assert rc == 0, lib.ref_model_last_error()
        y = np.empty((40, T))
        rc = lib.ref_model_forward_file(path.encode(), 64, T, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        40, y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        assert rc == 0, lib.ref_model_last_error()
        out[f"y_{dt}"] = [float(v).hex() for v in y.ravel()]
        print("wrote", path)
    with open(os.path.join(HERE, "ref_model_forward.json"), "w") as f:
        json.dump(out, f, indent=1)
    mspec = np.array(MIXED, dtype=np.uint64).ravel()
    mout = {"generator": "tests/golden/make_golden_model.py", "spec": MIXED, "T": T, "x_seed": 7,
            "x": out["x"]}
    for dt in ("f32", "f64"):
        path = os.path.join(HERE, f"ref_model_mixed_{dt}.json")
        rc = lib.ref_model_save_chain(path.encode(), 1 if dt == "f32" else 0, len(MIXED),
                                      mspec.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        assert rc == 0, lib.ref_model_last_error()
        y = np.empty((40, T))
        rc = lib.ref_model_forward_file(path.encode(), 64, T, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        40, y.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        assert rc == 0, lib.ref_model_last_error()
        mout[f"y_{dt}"] = [float(v).hex() for v in y.ravel()]
        print("wrote", path)
    with open(os.path.join(HERE, "ref_model_mixed_forward.json"), "w") as f:
        json.dump(mout, f, indent=1)


if __name__ == "__main__":
    main()
