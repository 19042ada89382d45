"""Time vp_gemm_bf16 on the BASELINE shapes with CUDA events (L2-flushed)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402


def bench(M, N, Kd, layout="nt", epi=K.EPI_STORE, iters=20):
    a_k, b_k = layout[0] == "n", layout[1] == "t"
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = torch.randn(N, Kd, device="cuda").bfloat16()
    a = A if a_k else A.t().contiguous()
    b = B if b_k else B.t().contiguous()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi >= K.EPI_ACC_F32 else torch.bfloat16)
    bias = torch.randn(N, device="cuda").bfloat16()
    aux = torch.randn(M, N, device="cuda").bfloat16()
    kw = {}
    if epi in (K.EPI_BIAS, K.EPI_BIAS_GELU, K.EPI_BIAS_RESID):
        kw["bias"] = bias
    if epi in (K.EPI_BIAS_GELU, K.EPI_BIAS_RESID, K.EPI_DGELU):
        kw["aux"] = aux
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        K.gemm(a, b, out, a_kmajor=a_k, b_kmajor=b_k, epilogue=epi, **kw)
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        K.gemm(a, b, out, a_kmajor=a_k, b_kmajor=b_k, epilogue=epi, **kw)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    t = ts[len(ts) // 2]
    tf = 2 * M * N * Kd / t / 1e9
    # cuBLAS for comparison (library baseline, not the product)
    for _ in range(3):
        torch.matmul(A, B.t())
    cts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(A, B.t())
        e.record()
        torch.cuda.synchronize()
        cts.append(s.elapsed_time(e))
    cts.sort()
    ct = cts[len(cts) // 2]
    return {"M": M, "N": N, "K": Kd, "layout": layout, "epi": epi, "ms": round(t, 4),
            "tflops": round(tf, 1), "cublas_tflops": round(2 * M * N * Kd / ct / 1e9, 1)}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "one":
    # python microbench.py one M N K layout epi
    M, N, Kd = map(int, sys.argv[2:5])
    print(json.dumps(bench(M, N, Kd, sys.argv[5], int(sys.argv[6]), iters=5)), flush=True)
    sys.exit(0)

if __name__ == "__main__":
    shapes = [
        (8192, 3072, 1024, "nt"), (8192, 1024, 1024, "nt"), (8192, 4096, 1024, "nt"),
        (8192, 1024, 4096, "nt"), (8192, 1024, 4096, "nn"), (4096, 1024, 8192, "tn"),
        (4096, 9216, 3072, "nt"), (4096, 3072, 12288, "nt"), (4096, 12288, 3072, "nt"),
        (3072, 12288, 4096, "tn"), (4096, 5760, 1920, "nt"), (8192, 8192, 8192, "nt"),
        (8192, 51200, 1024, "nt"),
    ]
    for M, N, Kd, lay in shapes:
        print(json.dumps(bench(M, N, Kd, lay)), flush=True)
    # the 355M stage GEMMs with their fused epilogues (fwd, dgrad, wgrad)
    for M, N, Kd, lay, epi in [(8192, 3072, 1024, "nt", K.EPI_BIAS), (8192, 1024, 1024, "nt", K.EPI_BIAS_RESID),
                               (8192, 4096, 1024, "nt", K.EPI_BIAS_GELU), (8192, 1024, 4096, "nt", K.EPI_BIAS_RESID),
                               (8192, 4096, 1024, "nn", K.EPI_DGELU), (8192, 1024, 4096, "nn", K.EPI_STORE),
                               (1024, 4096, 8192, "tn", K.EPI_ACC_F32), (3072, 1024, 8192, "tn", K.EPI_ACC_F32),
                               (1024, 1024, 8192, "tn", K.EPI_ACC_F32)]:
        print(json.dumps(bench(M, N, Kd, lay, epi)), flush=True)
