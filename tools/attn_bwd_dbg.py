"""Fused attention backward with parts of its work switched off (traced
library, diagnostic only — results are garbage): which side's traffic slows
the tensor pipe. VP_LIB_PATH=paper_2111_04007_b200/libvpipe_trace.so."""
import ctypes
import json
import os
import sys

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
K.L.vp_debug_bwd_set.argtypes = [ctypes.c_int]
res = {}
for dbg in (0, 1, 2, 4, 3, 7):
    K.L.vp_debug_bwd_set(dbg)
    for _ in range(3):
        K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, True)
    e.record()
    torch.cuda.synchronize()
    res[dbg] = round(s.elapsed_time(e) / 10 * 1e3, 1)
K.L.vp_debug_bwd_set(0)
print(json.dumps({"shape": [B, S, H, D], "bwd_us_by_dbg": res}))
