"""One fwd+bwd attention call at a BASELINE shape (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

B, S, H, D = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 1024, 16, 64))]
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
delta = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
for _ in range(2):
    K.attention_fwd(qkv, o, lse, B, S, H, D, True)
    K.attention_bwd(qkv, o, do, lse, dqkv, delta, B, S, H, D, True)
torch.cuda.synchronize()
print("ok")
