"""The last FC2 of a non-last stage writes the next stage's ring slot. Time
the options at the bench shape (m=32: 32768 x 1024 x 4096, BIAS_RESID):
(a) the 1-SM direct-store GEMM into the destination (what the executor does
for a peer pointer), (b) the 2-CTA TMA-store GEMM into a local buffer, (c)
(b) + the put kernel copying the result to another buffer (the alternative).
Same device (the copy over NVLink is ~105 us at 64 MiB, profiles/r02)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

M, N, KD = 32768, 1024, 4096
a = (torch.randn(M, KD, device="cuda") * 0.05).bfloat16()
w = (torch.randn(N, KD, device="cuda") * 0.02).bfloat16()
bias = torch.zeros(N, device="cuda").bfloat16()
res = torch.randn(M, N, device="cuda").bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
dst = torch.empty_like(out)


def t(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


direct = t(lambda: K.gemm(a, w, None, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=res,
                          out_ptr=dst.data_ptr(), ldd=N, direct=True))
tma = t(lambda: K.gemm(a, w, out, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=res))


def tma_put():
    K.gemm(a, w, out, epilogue=K.EPI_BIAS_RESID, bias=bias, aux=res)
    K.p2p_put(dst.data_ptr(), out)


both = t(tma_put)
f = 2 * M * N * KD
print(json.dumps({"direct_us": round(direct, 1), "direct_tflops": round(f / direct / 1e6, 1),
                  "tma_us": round(tma, 1), "tma_tflops": round(f / tma / 1e6, 1),
                  "tma_plus_local_put_us": round(both, 1)}))
