"""Time the HBM-bound row/column kernels (LayerNorm fwd/bwd, bias-gradient
column sums) at the GPT-2 355M shapes, CUDA events, inputs rotated over
sets larger than L2 (cold) or a single set (warm)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import kernels as K  # noqa: E402


def timed(fn, n_sets, iters=20):
    for i in range(3):
        fn(i % n_sets)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(iters):
        fn(i % n_sets)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    out = {}
    for cols in (1024, 1920, 3072):
        n = 4
        xs = [torch.randn(rows, cols, device="cuda").bfloat16() for _ in range(n)]
        dys = [torch.randn(rows, cols, device="cuda").bfloat16() for _ in range(n)]
        ys = [torch.empty_like(xs[0]) for _ in range(n)]
        g = torch.randn(cols, device="cuda").bfloat16()
        bt = torch.randn(cols, device="cuda").bfloat16()
        mean = torch.empty(rows, device="cuda")
        rstd = torch.empty(rows, device="cuda")
        dg = torch.zeros(cols, device="cuda")
        db = torch.zeros(cols, device="cuda")
        ws = torch.zeros(K.layernorm_ws_elems(cols), device="cuda")
        bws = torch.zeros(K.bias_grad_ws_elems(4 * cols), device="cuda")
        mb = 2 * rows * cols * 2 / 1e6
        for tag, sets in (("cold", n), ("warm", 1)):
            t = timed(lambda i: ys[i].copy_(xs[i]), sets)
            out[f"copy_{cols}_{tag}_us"] = round(t, 2)
            t = timed(lambda i: K.layernorm_fwd(xs[i], g, bt, ys[i], mean, rstd), sets)
            out[f"ln_fwd_{cols}_{tag}_us"] = round(t, 2)
            out[f"ln_fwd_{cols}_{tag}_GBs"] = round(mb / t * 1e3, 0)
            K.layernorm_fwd(xs[0], g, bt, ys[0], mean, rstd)
            t = timed(lambda i: K.layernorm_bwd(dys[i], xs[i], g, mean, rstd, ys[i], dg, db, ws,
                                                accumulate=True), sets)
            out[f"ln_bwd_{cols}_{tag}_us"] = round(t, 2)
            out[f"ln_bwd_{cols}_{tag}_GBs"] = round(2 * mb / t * 1e3, 0)
            t = timed(lambda i: K.bias_grad(dys[i], db, bws), sets)
            out[f"colsum_{cols}_{tag}_us"] = round(t, 2)
            out[f"colsum_{cols}_{tag}_GBs"] = round(mb / 2 / t * 1e3, 0)
    big = torch.randn(rows, 4096, device="cuda").bfloat16()
    db4 = torch.zeros(4096, device="cuda")
    bws = torch.zeros(K.bias_grad_ws_elems(4096), device="cuda")
    t = timed(lambda i: K.bias_grad(big, db4, bws), 1)
    out["colsum_4096_warm_us"] = round(t, 2)
    lg = torch.randn(8192, 51200, device="cuda").bfloat16()
    lab = torch.randint(0, 51200, (8192,), device="cuda")
    lr = torch.empty(8192, device="cuda")
    t = timed(lambda i: K.xent_fwd_bwd(lg, lab, lr, 1e-6), 1, iters=5)
    out["xent_8192x51200_us"] = round(t, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
