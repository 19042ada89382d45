"""clock64 timeline of the attention forward's first (heaviest) CTAs: per key
block j, the softmax warp's wait for S_j (slot 0->1), its softmax (1->2), the
P store incl. waits (2->3), and the MMA warp's S_j issue (4) and PV_j issue
(5), in cycles from the first stamp. Needs the traced library:

    VP_BUILD_TAG=trace VP_EXTRA_NVCC=-DVP_BWD_TRACE python paper_2111_04007_b200/build.py
    VP_LIB_PATH=paper_2111_04007_b200/libvpipe_trace.so python tools/attn_trace.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402

B, S, H, D = 32, 1024, 16, 64
qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
for _ in range(3):
    K.attention_fwd(qkv, o, lse, B, S, H, D, True)
torch.cuda.synchronize()
buf = np.zeros((4, 32, 8), dtype=np.uint64)
K.L.vp_debug_fwd_trace.argtypes = [ctypes.c_void_p]
rc = K.L.vp_debug_fwd_trace(buf.ctypes.data)
assert rc == 0, rc
for cta in range(2):
    t = buf[cta].astype(np.int64)
    base = t[0, 0]
    print(f"CTA {cta}: j | s_wait(0-1) | softmax(1-2) | Pstore(2-3) | S_issue(4) | PV_issue(5) | "
          f"block time")
    for j in range(16):
        r = t[j] - base
        nxt = (t[j + 1, 0] - t[j, 0]) if j < 15 else 0
        print(f"  {j:2d} {r[1] - r[0]:6d} {r[2] - r[1]:6d} {r[3] - r[2]:6d} {r[4]:8d} {r[5]:8d} {nxt:6d}")
