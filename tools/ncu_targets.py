"""One launch of each hot kernel at the GPT-2 355M m=32 shapes, bracketed by
cudaProfilerStart/Stop for

    ncu --profile-from-start off --set full --clock-control none --import-source on \\
        -o profiles/r01e_kernels_355m_m32 python paper_2111_04007_b200/ncu_targets.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K
torch.manual_seed(0)
M, H, F = 32768, 1024, 4096
B, S, NH, D = 32, 1024, 16, 64
x = torch.randn(M, H, device="cuda").bfloat16()
w1 = torch.randn(F, H, device="cuda").bfloat16() * 0.02
b1 = torch.zeros(F, device="cuda").bfloat16()
pre = torch.empty(M, F, device="cuda").bfloat16(); f = torch.empty_like(pre)
w2 = torch.randn(H, F, device="cuda").bfloat16() * 0.02
dy = torch.randn(M, H, device="cuda").bfloat16()
dpre = torch.empty_like(pre)
db = torch.zeros(F, device="cuda"); dws = torch.zeros(K.gemm_dbias_ws_elems(M, F), device="cuda")
g = torch.ones(H, device="cuda").bfloat16(); bt = torch.zeros(H, device="cuda").bfloat16()
y = torch.empty_like(x); mean = torch.empty(M, device="cuda"); rstd = torch.empty(M, device="cuda")
dx = torch.randn_like(x); dg = torch.zeros(H, device="cuda"); dbb = torch.zeros(H, device="cuda")
ds = torch.zeros(H, device="cuda"); lws = torch.zeros(K.layernorm_ws_elems(H), device="cuda")
qkv = torch.randn(M, 3 * H, device="cuda").bfloat16(); o = torch.empty(M, H, device="cuda").bfloat16()
lse = torch.empty(B * NH * S, device="cuda"); do = torch.randn_like(o); dqkv = torch.empty_like(qkv)
aws = torch.empty(K.attention_bwd_ws_elems(B, S, NH, D), device="cuda")
bq = torch.zeros(3 * H, device="cuda")
def run():
    K.gemm(x, w1, f, epilogue=K.EPI_BIAS_GELU, bias=b1, aux=pre)                       # FC1 fwd
    K.gemm(dy, w2, dpre, b_kmajor=False, epilogue=K.EPI_DGELU, aux=pre, dbias=db, dbias_ws=dws)  # FC2 dgrad+DGELU
    K.layernorm_fwd(x, g, bt, y, mean, rstd)
    K.layernorm_bwd(dy, x, g, mean, rstd, dx, dg, dbb, lws, accumulate=True, dsum=ds)
    K.attention_fwd(qkv, o, lse, B, S, NH, D, True)
    K.attention_bwd(qkv, o, do, lse, dqkv, aws, B, S, NH, D, True, dbias=bq)
run(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
run(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
