"""Time vp_attention_fwd/bwd (CUDA events) at the BASELINE shapes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402


def t(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


cases = [(8, 1024, 16, 64, True), (4, 1024, 20, 96, True), (4, 1024, 32, 96, True),
         (32, 512, 16, 64, False)]
if len(sys.argv) > 1 and sys.argv[1] == "long":
    cases = [(2, 4096, 16, 64, False), (2, 4096, 16, 64, True), (8, 1024, 16, 64, False)]
for B, S, H, D, causal in cases:
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty_like(lse)
    f = 4 * B * S * S * H * D * (0.5 if causal else 1.0)
    ms_f = t(lambda: K.attention_fwd(qkv, o, lse, B, S, H, D, causal))
    ms_b = t(lambda: K.attention_bwd(qkv, o, do, lse, dqkv, delta, B, S, H, D, causal))
    print(json.dumps({"B": B, "S": S, "H": H, "D": D, "causal": causal,
                      "fwd_ms": round(ms_f, 4), "fwd_tflops": round(f / ms_f / 1e9, 1),
                      "bwd_ms": round(ms_b, 4), "bwd_tflops": round(2.5 * f / ms_b / 1e9, 1)}))
