"""FC1-shaped GEMM (T x 4h x h) under each epilogue variant the executor can
use: plain store, bias, BIAS_GELU without / with the gelu' side output, and
the backward's DGELU (dgrad of FC2 times gelu'). CUDA events, L2 flushed."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

T, H = (int(x) for x in sys.argv[1:3]) if len(sys.argv) >= 3 else (32768, 1024)
N = 4 * H
x = torch.randn(T, H, device="cuda").bfloat16()
w1 = torch.randn(N, H, device="cuda").bfloat16()
b1 = torch.randn(N, device="cuda").bfloat16()
h = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
aux = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
dy = torch.randn(T, H, device="cuda").bfloat16()
w2 = torch.randn(H, N, device="cuda").bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def t(fn, iters=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


fl = 2 * T * N * H
res = {}
for name, fn in {
    "store": lambda: K.gemm(x, w1, h),
    "bias": lambda: K.gemm(x, w1, h, epilogue=K.EPI_BIAS, bias=b1),
    "bias_gelu": lambda: K.gemm(x, w1, h, epilogue=K.EPI_BIAS_GELU, bias=b1),
    "bias_gelu_save": lambda: K.gemm(x, w1, h, epilogue=K.EPI_BIAS_GELU, bias=b1, aux=aux),
    "dgelu": lambda: K.gemm(dy, w2, h, b_kmajor=False, epilogue=K.EPI_DGELU, aux=aux),
    "dgrad_store": lambda: K.gemm(dy, w2, h, b_kmajor=False),
}.items():
    us = t(fn)
    res[name] = {"us": round(us, 1), "tflops": round(fl / us / 1e6, 1)}
print(json.dumps({"T": T, "h": H, **res}))
