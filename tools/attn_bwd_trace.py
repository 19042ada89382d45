"""clock64 timeline of the fused attention backward's first CTAs (key block
0 of four (b, h) pairs: 8 query blocks each at S=1024): per query block,
the softmax-gradient warp's waits and compute, and the MMA warp's S/dP
issue. Needs the traced library (see tools/attn_trace.py)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

B, S, H, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) >= 5 else (32, 1024, 16, 64)
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
K.attention_fwd(qkv, o, lse, B, S, H, D, True)
for _ in range(3):
    K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, True)
torch.cuda.synchronize()
buf = np.zeros((4, 16, 16), dtype=np.uint64)
K.L.vp_debug_bwd_trace.argtypes = [ctypes.c_void_p]
assert K.L.vp_debug_bwd_trace(buf.ctypes.data) == 0
for cta in range(2):
    t = buf[cta].astype(np.int64)
    base = t[0, 0]
    print("  softmax start(0) abs:", [int(t[i, 0] - base) for i in range(8)])
    print(f"CTA {cta}: it | q_wait+S0_wait(0-1) | half0(1-2) | S1_wait(2-3) | half1(3-4) | "
          f"grad_waits(2-5) | store+arrive(4-6) | MMA S/dP issue(9) | p_full->(10) | "
          f"dq_empty(11) | grads issued(12) | dq_full(13) | iter time")
    for it in range(8):
        r = t[it] - base
        nxt = (t[it + 1, 0] - t[it, 0]) if it < 7 else 0
        print(f"  {it} {r[1]-r[0]:6d} {r[2]-r[1]:6d} {r[3]-r[2]:6d} {r[4]-r[3]:6d} {r[5]-r[2]:6d} "
              f"{r[6]-r[4]:6d} {r[9]:8d} {r[10]:8d} {r[11]:8d} {r[12]:8d} {r[13]:8d} {nxt:6d}")
