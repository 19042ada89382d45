"""In-step per-op timing: wraps every kernel entry point of ``kernels`` with
CUDA events on the current (= executor) stream and runs Varuna steps on one
GPU. Unlike an ncu launch list (serialised, caches flushed per kernel), this
is the time each op takes inside the real step, L2 state included.

    python -m paper_2111_04007_b200.op_profile --config gpt2_355m --m 8 --N 4
"""
import argparse
import collections
import functools
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import ParallelConfig  # noqa: E402
from paper_2111_04007_b200 import kernels as K  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS  # noqa: E402
from paper_2111_04007_b200.runtime import Varuna, synthetic_batch  # noqa: E402

OPS = ("gemm", "layernorm_fwd", "layernorm_bwd", "attention_fwd", "attention_bwd", "embed_fwd",
       "embed_bwd", "embed_typed_fwd", "embed_typed_bwd", "gelu_bwd", "xent_fwd_bwd",
       "bias_grad", "dropout_", "add", "grad_norm_sq", "adam_step", "p2p_put")
RECORDS = []
ON = [False]


def _key(name, args, kw):
    if name == "gemm":
        a, b = args[0], args[1]
        ak, bk = kw.get("a_kmajor", True), kw.get("b_kmajor", True)
        M = a.shape[0] if ak else a.shape[1]
        Kd = a.shape[1] if ak else a.shape[0]
        N = b.shape[0] if bk else b.shape[1]
        return f"gemm {M}x{N}x{Kd} {'T' if ak else 'N'}{'T' if bk else 'N'} " \
               f"epi{kw.get('epilogue', 0)}", 2 * M * N * Kd
    if name == "bias_grad":
        return f"bias_grad cols={args[0].shape[1]}", 0
    return name, 0


def _wrap(name, fn):
    @functools.wraps(fn)
    def inner(*args, **kw):
        if not ON[0]:
            return fn(*args, **kw)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        out = fn(*args, **kw)
        e1.record(st)
        RECORDS.append((_key(name, args, kw), e0, e1))
        return out
    return inner


def install():
    for n in OPS:
        if hasattr(K, n):
            setattr(K, n, _wrap(n, getattr(K, n)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt2_355m")
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--N", type=int, default=4)
    a = ap.parse_args()
    install()
    cfg = CONFIGS[a.config]
    # eager launches (no CUDA graphs): the timing wrappers must run per call
    v = Varuna(cfg, ParallelConfig(1, 1, a.m, a.N, (0,) * cfg.n_layer), seed=0,
               init_device="cuda", graphs=False)
    b = {k: t.cuda() for k, t in synthetic_batch(cfg, a.m * a.N, 0).items()}
    for _ in range(2):
        v.step(b)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(v.stream)
    v.step(b)
    s1.record(v.stream)
    torch.cuda.synchronize()
    plain = s0.elapsed_time(s1) * 1e3
    ON[0] = True
    v.step(b)
    torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0.0, 0, 0])
    for (key, flops), e0, e1 in RECORDS:
        t = e0.elapsed_time(e1) * 1e3
        agg[key][0] += t
        agg[key][1] += 1
        agg[key][2] += flops
    total = sum(x[0] for x in agg.values())
    print(f"step {plain:.0f} us un-instrumented ({plain / a.N:.0f} us per micro-batch); "
          f"instrumented op total {total:.0f} us")
    print(f"{'us/mb':>9} {'share':>6} {'n/mb':>5} {'us/call':>8} {'TF/s':>7}  op")
    for key, (t, n, fl) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        tf = f"{fl / (t * 1e-6) / 1e12:7.0f}" if fl else "       "
        print(f"{t / a.N:9.1f} {t / total:6.1%} {n / a.N:5.1f} {t / n:8.1f} {tf}  {key}")


if __name__ == "__main__":
    main()
