"""clock64 breakdown of one persistent GEMM launch (traced library): the
MMA warp's waits for operands (full) and for a drained accumulator (tempty),
and epilogue warp 4's time in the accumulator wait, TMEM loads, epilogue
math, staging-buffer waits and smem stores + TMA issue. Averages over CTAs.

    VP_BUILD_TAG=gtrace VP_EXTRA_NVCC=-DVP_GEMM_TRACE python paper_2111_04007_b200/build.py
    VP_LIB_PATH=paper_2111_04007_b200/libvpipe_gtrace.so python tools/gemm_trace.py M N K layout epi
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

M, N, Kd = (int(x) for x in sys.argv[1:4])
layout, epi = sys.argv[4], int(sys.argv[5])
a_k, b_k = layout[0] == "n", layout[1] == "t"
A = torch.randn(M, Kd, device="cuda").bfloat16()
B = torch.randn(N, Kd, device="cuda").bfloat16()
a = A if a_k else A.t().contiguous()
b = B if b_k else B.t().contiguous()
out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi >= K.EPI_ACC_F32 else torch.bfloat16)
kw = {}
if epi in (K.EPI_BIAS, K.EPI_BIAS_GELU, K.EPI_BIAS_RESID):
    kw["bias"] = torch.randn(N, device="cuda").bfloat16()
if epi in (K.EPI_BIAS_GELU, K.EPI_BIAS_RESID, K.EPI_DGELU):
    kw["aux"] = torch.randn(M, N, device="cuda").bfloat16()
for _ in range(3):
    K.gemm(a, b, out, a_kmajor=a_k, b_kmajor=b_k, epilogue=epi, **kw)
torch.cuda.synchronize()
mma = np.zeros((296, 4), dtype=np.uint64)
ep = np.zeros((296, 6), dtype=np.uint64)
K.L.vp_debug_gemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
assert K.L.vp_debug_gemm_trace(mma.ctypes.data, ep.ctypes.data) == 0
lead = mma[0::2][mma[0::2, 2] > 0].astype(np.float64)
e = ep[ep[:, 5] > 0].astype(np.float64)
res = {"shape": [M, N, Kd, layout, epi],
       "mma_total_clk": lead[:, 2].mean(), "mma_wait_full_pct": 100 * (lead[:, 0] / lead[:, 2]).mean(),
       "mma_wait_tempty_pct": 100 * (lead[:, 1] / lead[:, 2]).mean(), "tiles_per_cluster": lead[:, 3].mean(),
       "epi_total_clk": e[:, 5].mean()}
for i, name in enumerate(("tfull_wait", "tmem_ld", "math", "buf_wait", "store_issue")):
    res[f"epi_{name}_pct"] = round(100 * (e[:, i] / e[:, 5]).mean(), 1)
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}))
