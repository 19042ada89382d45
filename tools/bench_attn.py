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
if len(sys.argv) > 1 and sys.argv[1] == "big":   # planner-chosen m=32 (dQ accumulator > L2)
    cases = [(8, 1024, 16, 64, True), (16, 1024, 16, 64, True), (32, 1024, 16, 64, True),
             (64, 512, 16, 64, False)]
for B, S, H, D, causal in cases:
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
    f = 4 * B * S * S * H * D * (0.5 if causal else 1.0)
    ms_f = t(lambda: K.attention_fwd(qkv, o, lse, B, S, H, D, causal))
    ms_b = t(lambda: K.attention_bwd(qkv, o, do, lse, dqkv, delta, B, S, H, D, causal))
    ms_bd = t(lambda: K.attention_bwd(qkv, o, do, lse, dqkv, delta, B, S, H, D, causal,
                                      deterministic=True))
    print(json.dumps({"B": B, "S": S, "H": H, "D": D, "causal": causal,
                      "fwd_ms": round(ms_f, 4), "fwd_tflops": round(f / ms_f / 1e9, 1),
                      "bwd_ms": round(ms_b, 4), "bwd_tflops": round(2.5 * f / ms_b / 1e9, 1),
                      "bwd_det_ms": round(ms_bd, 4)}))

if len(sys.argv) > 1 and sys.argv[1] == "sdpa":
    # library reference points (not on the product path): torch SDPA backends
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel
    for B, S, H, D, causal in [(8, 1024, 16, 64, True), (4, 1024, 32, 96, True)]:
        q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16,
                               requires_grad=True) for _ in range(3))
        f = 4 * B * S * S * H * D * (0.5 if causal else 1.0)
        for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
            try:
                with sdpa_kernel(be):
                    out = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                    go = torch.randn_like(out)
                    ms_f = t(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=causal))
                    ms_fb = t(lambda: torch.autograd.grad(
                        F.scaled_dot_product_attention(q, k, v, is_causal=causal), (q, k, v), go))
                ms_b = ms_fb - ms_f
                print(json.dumps({"backend": str(be), "B": B, "S": S, "H": H, "D": D,
                                  "fwd_ms": round(ms_f, 4), "fwd_tflops": round(f / ms_f / 1e9, 1),
                                  "bwd_ms": round(ms_b, 4),
                                  "bwd_tflops": round(2.5 * f / ms_b / 1e9, 1)}))
            except Exception as ex:  # noqa: BLE001
                print(json.dumps({"backend": str(be), "error": str(ex)[:200]}))
