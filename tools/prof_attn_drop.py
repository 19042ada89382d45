"""Attention forward + backward at 32x1024x16x64 causal without and with K7
dropout (keep-bit mask written by the forward, read by the backward), one
launch each after a warm-up — the ncu target for the dropout overhead."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

B, S, H, D = 32, 1024, 16, 64
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
seed = torch.full((1,), 12345, dtype=torch.int64, device="cuda")
mq = torch.zeros(K.attention_mask_words(B, S, H), dtype=torch.int32, device="cuda")
mk = torch.zeros_like(mq)
for it in range(2):
    for p in (0.0, 0.1):
        if p > 0:
            K.attention_dropout_mask(B, S, H, True, p, seed, 0, mq, mk)
        K.attention_fwd(qkv, o, lse, B, S, H, D, True, p=p, seed=seed, mask=mq)
        K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, True, p=p, seed=seed, mask_q=mq,
                        mask_k=mk)
torch.cuda.synchronize()
print("ok")
