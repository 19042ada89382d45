"""Attention microbenchmark at the bench shapes: forward / backward time and
TFLOP/s (causal FLOPs: 4*B*S^2*H*D/2 forward, 2.5x that backward), with and
without K7 dropout, plus torch SDPA (cuDNN / flash) as library reference
points. CUDA events, 3 warm-up + 10 timed calls.

    python tools/attn_micro.py [B S H D causal] ...
"""
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


def run(B, S, H, D, causal):
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
    seed = torch.full((1,), 12345, dtype=torch.int64, device="cuda")
    nw = max(1, K.attention_mask_words(B, S, H))
    mq = torch.zeros(nw, dtype=torch.int32, device="cuda")
    mk = torch.zeros(nw, dtype=torch.int32, device="cuda")
    f = 4 * B * S * S * H * D * (0.5 if causal else 1.0)
    out = {"B": B, "S": S, "H": H, "D": D, "causal": causal}
    for p in (0.0, 0.1):
        ms_m = t(lambda: K.attention_dropout_mask(B, S, H, causal, 0.1, seed, 3, mq, mk)) \
            if p > 0 else 0.0
        ms_f = t(lambda: K.attention_fwd(qkv, o, lse, B, S, H, D, causal, p=p, seed=seed,
                                         mask=mq))
        db = torch.zeros(3 * H * D, device="cuda")
        ms_b = t(lambda: K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, causal, dbias=db,
                                         p=p, seed=seed, mask_q=mq, mask_k=mk))
        tag = "" if p == 0 else "_p0.1"
        out.update({f"fwd_us{tag}": round(ms_f * 1e3, 1),
                    f"fwd_tflops{tag}": round(f / ms_f / 1e9, 1),
                    f"bwd_us{tag}": round(ms_b * 1e3, 1),
                    f"bwd_tflops{tag}": round(2.5 * f / ms_b / 1e9, 1)})
        if p > 0:
            out["mask_us_p0.1"] = round(ms_m * 1e3, 1)
        elif "det" in sys.argv:
            ms_d = t(lambda: K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, causal,
                                             deterministic=True))
            out["bwd_two_kernel_us"] = round(ms_d * 1e3, 1)
            out["bwd_two_kernel_tflops"] = round(2.5 * f / ms_d / 1e9, 1)
    if "sdpa" in sys.argv:
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel
        q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16,
                               requires_grad=True) for _ in range(3))
        for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
            try:
                with sdpa_kernel(be):
                    y = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
                    go = torch.randn_like(y)
                    ms_f = t(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=causal))
                    ms_fb = t(lambda: torch.autograd.grad(
                        F.scaled_dot_product_attention(q, k, v, is_causal=causal), (q, k, v), go))
                out[str(be).split(".")[-1]] = {"fwd_tflops": round(f / ms_f / 1e9, 1),
                                               "bwd_tflops": round(2.5 * f / (ms_fb - ms_f) / 1e9, 1)}
            except Exception as ex:  # noqa: BLE001
                out[str(be).split(".")[-1]] = str(ex)[:100]
    print(json.dumps(out), flush=True)


args = [a for a in sys.argv[1:] if a not in ("sdpa", "det")]
cases = [(32, 1024, 16, 64, True), (8, 1024, 16, 64, True), (4, 1024, 20, 96, True),
         (4, 1024, 32, 96, True), (16, 1024, 20, 96, True),
         (64, 512, 16, 64, False)]
if len(args) >= 5:
    cases = [tuple(int(x) for x in args[:4]) + (args[4] in ("1", "True", "true"),)]
for c in cases:
    run(*c)
