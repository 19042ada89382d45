"""Oracle: fp32 PyTorch-CPU GPT-2 + a sequential Varuna pipeline executor.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The reference has no
tensor math, so this loss/gradient oracle is PARITY-
UNPINNED against the reference itself; it follows the semantics SURVEY
§8(c)2 derives from it:

* stages own contiguous CutPoints (layers) per ``stage_map``;
* each stage walks its Varuna task list (restated in oracle/schedule.py,
  pinned to the reference's plans): F(j) discards intermediates on k < P-1,
  R(j) recomputes from the stashed input, B(j) consumes the downstream
  gradient; the last stage runs F(j) then B(j) (sp/engine/py_kernel.py:
  156-175, 216-234);
* micro-batch gradients accumulate in schedule order (sp/scheduler.py:237);
* loss = mean over all M_total·S label tokens; tied wte between stage 0
  and the LM head; global grad-norm clipping; AdamW with fp32 master state
  (the 16 B/param model, sp/core.py:17-18).

Weights start from the same seeded init as the GPU executor (re-derived
here, not imported from the product) rounded to bf16, so both sides see
identical parameters.
"""

from __future__ import annotations

import math
from typing import Dict, List

import numpy as np
import torch

from . import schedule as osch


def _round(t):
    return t.to(torch.bfloat16).to(torch.float32)


def init_params(n_layer, hidden, vocab, seq, seed=0, init_std=0.02, arch="gpt2", type_vocab=2):
    """Same generator streams as the product's per-layer init (seeded by
    (seed, layer)); returns fp32 tensors rounded to bf16."""
    h = hidden
    out = {}
    g = torch.Generator()
    g.manual_seed(seed * 1000003)
    out["wte"] = _round(torch.randn((vocab, h), generator=g) * init_std)
    out["wpe"] = _round(torch.randn((seq, h), generator=g) * 0.01)
    if arch == "bert":
        out["tte"] = _round(torch.randn((type_vocab, h), generator=g) * init_std)
        out["lne_g"] = torch.ones(h)
        out["lne_b"] = torch.zeros(h)
    proj = init_std / math.sqrt(2 * n_layer)
    shapes = [("ln1_g", (h,)), ("ln1_b", (h,)), ("w_qkv", (3 * h, h)), ("b_qkv", (3 * h,)),
              ("w_o", (h, h)), ("b_o", (h,)), ("ln2_g", (h,)), ("ln2_b", (h,)),
              ("w_fc1", (4 * h, h)), ("b_fc1", (4 * h,)), ("w_fc2", (h, 4 * h)), ("b_fc2", (h,))]
    for li in range(n_layer):
        g = torch.Generator()
        g.manual_seed(seed * 1000003 + li + 1)
        for name, shape in shapes:
            if name.endswith("_g"):
                v = torch.ones(shape)
            elif name.startswith("b_") or name.endswith("_b"):
                v = torch.zeros(shape)
            else:
                std = proj if name in ("w_o", "w_fc2") else init_std
                v = torch.randn(shape, generator=g) * std
            out[f"l{li}.{name}"] = _round(v)
    if arch == "bert":
        g = torch.Generator()
        g.manual_seed(seed * 1000003 + n_layer + 1)
        out["w_mlm"] = _round(torch.randn((h, h), generator=g) * init_std)
        out["b_mlm"] = torch.zeros(h)
        out["lnm_g"] = torch.ones(h)
        out["lnm_b"] = torch.zeros(h)
        out["b_dec"] = torch.zeros(vocab)
    else:
        out["lnf_g"] = torch.ones(h)
        out["lnf_b"] = torch.zeros(h)
    return out


# ------------------------------------------------------------------ dropout
# Restatement of the K7 mask (include/vpipe.h vp_set_seed / vp_dropout_dev,
# csrc/common.cuh drop_key / drop_bits) and of the executor's per-(step,
# micro-batch) seed (paper_2111_04007_b200/runtime.py task_seed), so the
# oracle draws exactly the GPU's masks. Dropout is not in the reference
# (SPEC.md:18); its recompute-correctness requirement is PAPER.md:577.
_M32 = np.uint64(0xFFFFFFFF)
_M64 = (1 << 64) - 1


def task_seed(seed: int, step: int, mb: int) -> int:
    x = (seed * 0x9E3779B97F4A7C15 + step * 0xD1B54A32D192ED03 + mb * 0xBF58476D1CE4E5B9 + 1) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _fmix32(h):
    """murmur3 finalizer on uint64 arrays holding 32-bit values."""
    h = h ^ (h >> np.uint64(16))
    h = (h * np.uint64(0x85EBCA6B)) & _M32
    h = h ^ (h >> np.uint64(13))
    h = (h * np.uint64(0xC2B2AE35)) & _M32
    return h ^ (h >> np.uint64(16))


def drop_threshold(p: float) -> int:
    return min(65535, int(p * 65536.0 + 0.5))


def drop_keep(seed64: int, salt: int, e: np.ndarray, p: float) -> np.ndarray:
    """Keep flags of flat element indices ``e`` (uint64) at one call site."""
    lo = np.uint64(seed64 & 0xFFFFFFFF)
    hi = np.uint64(seed64 >> 32)
    key = _fmix32(lo ^ _fmix32(hi ^ _fmix32(np.uint64(salt & 0xFFFFFFFF))))
    pair = e >> np.uint64(1)
    b = _fmix32(key ^ (((pair & _M32) * np.uint64(0x9E3779B1)) & _M32)
                ^ (((pair >> np.uint64(32)) * np.uint64(0x85EBCA77)) & _M32))
    u = np.where((e & np.uint64(1)) == 1, b >> np.uint64(16), b & np.uint64(0xFFFF))
    return u >= np.uint64(drop_threshold(p))


def dropout(x: torch.Tensor, p: float, seed64, salt: int) -> torch.Tensor:
    """x * mask / (1 - p) over the flat (row-major) element index."""
    if p <= 0 or seed64 is None:
        return x
    thr = drop_threshold(p)
    e = np.arange(x.numel(), dtype=np.uint64)
    keep = torch.from_numpy(drop_keep(seed64, salt, e, p)).view(x.shape)
    return x * keep.to(x.dtype) * (65536.0 / (65536 - thr))


def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


# dropout call-site salts (paper_2111_04007_b200/model.py drop_salt)
def _salt(li, site):
    return li * 4 + site


SALT_EMBED = 0x7FFFFFF0


def layer_forward_post(p, li, x, B, S, H, eps=1e-12, drop=0.0, seed64=None):
    """BERT post-LN layer (bidirectional attention); hidden dropout on the
    proj / FC2 branches, attention-probability dropout."""
    h = x.shape[-1]
    D = h // H
    pre = f"l{li}."
    qkv = x @ p[pre + "w_qkv"].t() + p[pre + "b_qkv"]
    q, k, v = qkv.view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    o = (dropout(s.softmax(-1), drop, seed64, _salt(li, 0)) @ v).permute(0, 2, 1, 3).reshape(B * S, h)
    y1 = x + dropout(o @ p[pre + "w_o"].t() + p[pre + "b_o"], drop, seed64, _salt(li, 1))
    x1 = torch.nn.functional.layer_norm(y1, (h,), p[pre + "ln1_g"], p[pre + "ln1_b"], eps)
    f = gelu(x1 @ p[pre + "w_fc1"].t() + p[pre + "b_fc1"])
    y2 = x1 + dropout(f @ p[pre + "w_fc2"].t() + p[pre + "b_fc2"], drop, seed64, _salt(li, 2))
    return torch.nn.functional.layer_norm(y2, (h,), p[pre + "ln2_g"], p[pre + "ln2_b"], eps)


def layer_forward(p, li, x, B, S, H, eps=1e-5, drop=0.0, seed64=None):
    h = x.shape[-1]
    D = h // H
    pre = f"l{li}."
    a = torch.nn.functional.layer_norm(x, (h,), p[pre + "ln1_g"], p[pre + "ln1_b"], eps)
    qkv = a @ p[pre + "w_qkv"].t() + p[pre + "b_qkv"]
    q, k, v = qkv.view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    mask = torch.ones(S, S, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    o = (dropout(s.softmax(-1), drop, seed64, _salt(li, 0)) @ v).permute(0, 2, 1, 3).reshape(B * S, h)
    x1 = x + dropout(o @ p[pre + "w_o"].t() + p[pre + "b_o"], drop, seed64, _salt(li, 1))
    c = torch.nn.functional.layer_norm(x1, (h,), p[pre + "ln2_g"], p[pre + "ln2_b"], eps)
    f = gelu(c @ p[pre + "w_fc1"].t() + p[pre + "b_fc1"])
    return x1 + dropout(f @ p[pre + "w_fc2"].t() + p[pre + "b_fc2"], drop, seed64, _salt(li, 2))


class PipelineOracle:
    """Sequential execution of a P-stage Varuna pipeline on CPU fp32."""

    def __init__(self, n_layer, hidden, heads, vocab, seq, stage_map, micro_batch, n_micro,
                 seed=0, arch="gpt2", dropout=0.0):
        self.L, self.h, self.H, self.V, self.S = n_layer, hidden, heads, vocab, seq
        self.arch = arch
        self.eps = 1e-12 if arch == "bert" else 1e-5
        self.stage_map = list(stage_map)
        self.P = max(stage_map) + 1
        self.m, self.N = micro_batch, n_micro
        self.params = {k: v.clone().requires_grad_(True)
                       for k, v in init_params(n_layer, hidden, vocab, seq, seed,
                                               arch=arch).items()}
        self.layers = [[i for i, s in enumerate(stage_map) if s == k] for k in range(self.P)]
        self.seed, self.drop = seed, dropout
        self._seed64 = None   # of the micro-batch being run

    def _stage_forward(self, k, x_or_ids, types=None):
        p = self.params
        if k == 0:
            ids = x_or_ids
            x = p["wte"][ids] + p["wpe"][torch.arange(self.S).repeat(self.m)]
            if self.arch == "bert":
                x = x + p["tte"][types]
                x = torch.nn.functional.layer_norm(x, (self.h,), p["lne_g"], p["lne_b"], self.eps)
            x = dropout(x, self.drop, self._seed64, SALT_EMBED)
        else:
            x = x_or_ids
        for li in self.layers[k]:
            if self.arch == "bert":
                x = layer_forward_post(p, li, x, self.m, self.S, self.H, self.eps, self.drop,
                                       self._seed64)
            else:
                x = layer_forward(p, li, x, self.m, self.S, self.H, drop=self.drop,
                                  seed64=self._seed64)
        return x

    def _head_loss(self, x, labels, scale):
        p = self.params
        if self.arch == "bert":
            hm = gelu(x @ p["w_mlm"].t() + p["b_mlm"])
            z = torch.nn.functional.layer_norm(hm, (self.h,), p["lnm_g"], p["lnm_b"], self.eps)
            logits = z @ p["wte"].t() + p["b_dec"]
            l = torch.nn.functional.cross_entropy(logits, labels, ignore_index=-100,
                                                  reduction="sum")
            return l * scale
        y = torch.nn.functional.layer_norm(x, (self.h,), p["lnf_g"], p["lnf_b"], 1e-5)
        logits = y @ p["wte"].t()
        l = torch.nn.functional.cross_entropy(logits, labels, ignore_index=-100, reduction="sum")
        return l * scale

    def run_minibatch(self, ids, labels, total_tokens, types=None, step=1, replica=0):
        """ids/labels: [N*m, S] int64. Returns the (scaled) loss; grads are
        accumulated in ``self.params[*].grad`` in schedule order. With
        dropout, micro-batch j of ``replica`` in training step ``step`` draws
        the executor's masks (seed task_seed(seed, step, replica*N + j))."""
        P, N = self.P, self.N
        plan = osch.varuna_plan(P, N, 1_000_000, 2_000_000, 1_000_000)
        order = _global_order(plan, P)
        rows = N * self.m
        if ids.shape[0] < rows:
            # M_total semantics (sp/planner.py:99-103): N_m = ceil(M/(m*D)),
            # the last micro-batch partially filled; padded rows carry no label
            pad = rows - ids.shape[0]
            ids = torch.cat([ids, torch.zeros(pad, ids.shape[1], dtype=ids.dtype)], 0)
            labels = torch.cat([labels, torch.full((pad, labels.shape[1]), -100,
                                                   dtype=labels.dtype)], 0)
            if types is not None:
                types = torch.cat([types, torch.zeros(pad, types.shape[1], dtype=types.dtype)], 0)
        ids = ids.view(N, self.m * self.S)
        labels = labels.view(N, self.m * self.S)
        if types is not None:
            types = types.reshape(N, self.m * self.S)
        scale = 1.0 / total_tokens
        act = {}     # (k, j) -> activation entering stage k (detached)
        saved = {}   # (k, j) -> (input leaf, output) with graph
        grad_in = {}  # (k, j) -> gradient of stage k output
        loss = 0.0
        for k, kind, j in order:
            last = k == P - 1
            self._seed64 = task_seed(self.seed, step, replica * N + j) if self.drop > 0 else None
            inp = ids[j] if k == 0 else act[(k, j)]
            tj = types[j] if (types is not None and k == 0) else None
            if kind == osch.F and not last:
                with torch.no_grad():
                    out = self._stage_forward(k, inp, tj)
                act[(k + 1, j)] = out.detach()
            elif kind == osch.R or (kind == osch.F and last):
                leaf = inp if k == 0 else inp.detach().requires_grad_(True)
                out = self._stage_forward(k, leaf, tj)
                saved[(k, j)] = (leaf, out)
            else:  # backward
                leaf, out = saved.pop((k, j))
                if last:
                    l = self._head_loss(out, labels[j], scale)
                    loss += float(l.detach())
                    l.backward()
                else:
                    out.backward(grad_in.pop((k, j)))
                if k > 0:
                    grad_in[(k - 1, j)] = leaf.grad.detach()
        return loss

    def grads(self) -> Dict[str, torch.Tensor]:
        return {k: (v.grad.clone() if v.grad is not None else torch.zeros_like(v))
                for k, v in self.params.items()}

    def adamw_step(self, step, lr=1e-4, betas=(0.9, 0.999), eps=1e-8, wd=0.01, max_norm=1.0):
        """Global-norm clip then AdamW (decoupled decay), fp32 state."""
        with torch.no_grad():
            gs = [v.grad for v in self.params.values() if v.grad is not None]
            norm = math.sqrt(sum(float((g * g).sum()) for g in gs))
            coef = 1.0
            if max_norm > 0 and norm > max_norm:
                coef = max_norm / (norm + 1e-6)
            if not hasattr(self, "_m"):
                self._m = {k: torch.zeros_like(v) for k, v in self.params.items()}
                self._v = {k: torch.zeros_like(v) for k, v in self.params.items()}
            b1, b2 = betas
            for k, p in self.params.items():
                g = (p.grad if p.grad is not None else torch.zeros_like(p)) * coef
                self._m[k].mul_(b1).add_(g, alpha=1 - b1)
                self._v[k].mul_(b2).addcmul_(g, g, value=1 - b2)
                mh = self._m[k] / (1 - b1 ** step)
                vh = self._v[k] / (1 - b2 ** step)
                p.sub_(lr * (mh / (vh.sqrt() + eps) + wd * p))
                p.grad = None
        return norm


def _global_order(plan, P) -> List[tuple]:
    """A dependency-respecting interleaving of the per-stage lists: the
    zero-delay replay's start-time order (ties by stage)."""
    tf, tb, tr = 1, 2, 1
    times = {}
    ptr = [0] * P
    free = [0] * P
    moved = True
    while moved:
        moved = False
        for k in range(P):
            while ptr[k] < len(plan[k]):
                kind, j = plan[k][ptr[k]]
                if kind == osch.F:
                    dep = 0 if k == 0 else times.get((k - 1, osch.F, j))
                elif kind == osch.R or k == P - 1:
                    dep = times.get((k, osch.F, j))
                else:
                    a, b = times.get((k + 1, osch.B, j)), times.get((k, osch.R, j))
                    dep = None if a is None or b is None else max(a, b)
                if dep is None:
                    break
                s = max(free[k], dep)
                d = {osch.F: tf, osch.B: tb, osch.R: tr}[kind]
                times[(k, kind, j)] = s + d
                free[k] = s + d
                ptr[k] += 1
                moved = True
    ends = sorted(times.items(), key=lambda kv: (kv[1], kv[0][0]))
    # start order = end - duration
    dur = {osch.F: tf, osch.B: tb, osch.R: tr}
    return [key for key, _ in sorted(times.items(),
                                     key=lambda kv: (kv[1] - dur[kv[0][1]], kv[0][0]))]
