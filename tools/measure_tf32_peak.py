"""Dense TF32 tensor-core peak of this B200, measured like MEASURED_PEAKS.json's
bf16 figure: cuBLAS fp32 8192^3 matmul with TF32 allowed (2*N^3 FLOPs), best of
10 (burst) and back to back for 4 s (sustained), CUDA events.  The bf16 figure
is re-measured beside it for the ratio.  Prints one JSON line."""
import json
import time

import torch


def measure(dtype, n=8192):
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2 * n ** 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    cnt = 0
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            a @ b
        cnt += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / cnt
    return flops / (best / 1e3) / 1e12, flops / (sus / 1e3) / 1e12


torch.backends.cuda.matmul.allow_tf32 = True
torch.backends.cudnn.allow_tf32 = True
tf_b, tf_s = measure(torch.float32)
bf_b, bf_s = measure(torch.bfloat16)
print(json.dumps({"tf32_tflops": round(tf_b, 1), "tf32_tflops_sustained": round(tf_s, 1),
                  "bf16_tflops": round(bf_b, 1), "bf16_tflops_sustained": round(bf_s, 1),
                  "ratio_tf32_bf16": round(tf_b / bf_b, 3), "gpu": torch.cuda.get_device_name(0),
                  "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS), best of 10 (burst) and back to back "
                         "for 4 s (sustained), CUDA events; bf16 re-measured the same way"}))
