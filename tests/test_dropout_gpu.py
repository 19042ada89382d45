"""K7 dropout-recompute on the GPU against the oracle's restatement of the
mask (oracle/gpt2_fp32.py drop_keep / dropout; the mask is a pure function
of (seed, salt, element), so the oracle reproduces it exactly).

Bitwise: the kept/dropped pattern of every site (embedding in place, GEMM
epilogue, backward colsum pass, attention probabilities) and R == F at
p = 0.1 in-model. Numerics: against fp32 torch references of the same ops
at the tolerances of tests/test_kernels_gpu.py (bf16 storage); end-to-end
loss / gradient parity at p = 0.1 with tests/test_pipeline_gpu.py's
tolerances (loss 5e-3, gradients 3e-2)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P = 0.1
SEED = 0x1234_5678_9ABC_DEF1


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


def _seed_buf(v=SEED):
    from paper_2111_04007_b200 import kernels as K
    buf = torch.zeros(1, dtype=torch.int64, device="cuda")
    K.set_seed(buf, v)
    return buf


def test_mask_matches_oracle_and_rate():
    from paper_2111_04007_b200 import kernels as K
    from oracle.gpt2_fp32 import dropout
    x = torch.ones(4096, 1024, device="cuda", dtype=torch.bfloat16)
    K.dropout_dev_(x, P, _seed_buf(), 77)
    ref = dropout(torch.ones(4096, 1024), P, SEED, 77)
    assert torch.equal((x.float().cpu() == 0), (ref == 0))
    rate = (x == 0).float().mean().item()
    assert abs(rate - P) < 2e-3, rate
    # a different salt or seed gives a different mask
    y = torch.ones_like(x)
    K.dropout_dev_(y, P, _seed_buf(), 78)
    assert not torch.equal(x, y)
    z = torch.ones_like(x)
    K.dropout_dev_(z, P, _seed_buf(SEED + 1), 77)
    assert not torch.equal(x, z)


@pytest.mark.parametrize("M,N,K_", [(4096, 1024, 1024), (1000, 768, 256), (512, 192, 64)])
@pytest.mark.parametrize("direct", [False, True])
def test_gemm_dropout_epilogue(M, N, K_, direct):
    from paper_2111_04007_b200 import kernels as K
    from oracle.gpt2_fp32 import dropout
    torch.manual_seed(0)
    a = (torch.randn(M, K_, device="cuda") / math.sqrt(K_)).bfloat16()
    w = torch.randn(N, K_, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    res = torch.randn(M, N, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    if direct:
        K.gemm_dropout(a, w, None, bias, res, P, _seed_buf(), 5, out_ptr=out.data_ptr(), ldd=N,
                       direct=True)
    else:
        K.gemm_dropout(a, w, out, bias, res, P, _seed_buf(), 5)
    y = (a.float() @ w.float().t() + bias.float()).cpu()
    ref = res.float().cpu() + dropout(y, P, SEED, 5)
    assert rel(out.cpu(), ref) < 1e-2
    keep = dropout(torch.ones(M, N), P, SEED, 5) != 0
    branch = out.float().cpu() - res.float().cpu()
    # dropped elements carry exactly the residual
    assert branch[~keep].abs().max().item() == 0.0


def test_dropout_bwd_mask_and_bias():
    from paper_2111_04007_b200 import kernels as K
    from oracle.gpt2_fp32 import dropout
    torch.manual_seed(1)
    rows, cols = 3000, 1024
    g = torch.randn(rows, cols, device="cuda").bfloat16()
    gy = torch.empty_like(g)
    db = torch.ones(cols, device="cuda")
    ws = torch.zeros(K.bias_grad_ws_elems(cols), device="cuda")
    K.dropout_bwd(g, gy, P, _seed_buf(), 9, db, ws)
    ref = dropout(g.float().cpu(), P, SEED, 9)
    assert torch.equal(gy.float().cpu() == 0, ref == 0)
    assert rel(gy.cpu(), ref) < 1e-2
    assert rel(db.cpu(), 1 + gy.float().cpu().sum(0)) < 1e-4


@pytest.mark.parametrize("rows,cols,acc", [(3000, 1024, True), (2048, 1920, False),
                                           (1000, 3072, True)])
def test_layernorm_bwd_dropout_fused(rows, cols, acc):
    """vp_layernorm_bwd_dropout == layernorm_bwd followed by dropout_bwd:
    dx and gy bitwise, dgamma / dbeta / the branch bias gradient to fp32
    summation-order noise (widths of GPT-2 355M, 2.5B, 8.3B)."""
    from paper_2111_04007_b200 import kernels as K
    torch.manual_seed(5)
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    dy = torch.randn(rows, cols, device="cuda").bfloat16()
    gamma = (1 + 0.1 * torch.randn(cols, device="cuda")).bfloat16()
    mu = x.float().mean(1)
    rs = torch.rsqrt(x.float().var(1, unbiased=False) + 1e-5)
    base = torch.randn(rows, cols, device="cuda").bfloat16()
    ws = torch.zeros(K.layernorm_ws_elems(cols), device="cuda")
    bws = torch.zeros(K.bias_grad_ws_elems(cols), device="cuda")
    sb = _seed_buf()
    out = {}
    for fused in (False, True):
        dx = base.clone()
        dg, db, ds = (torch.zeros(cols, device="cuda") for _ in range(3))
        gy = torch.empty_like(dx)
        if fused:
            assert K.layernorm_bwd_dropout(dy, x, gamma, mu, rs, dx, dg, db, ws, ds, gy, P, sb, 21,
                                           accumulate=acc)
        else:
            K.layernorm_bwd(dy, x, gamma, mu, rs, dx, dg, db, ws, accumulate=acc)
            K.dropout_bwd(dx, gy, P, sb, 21, ds, bws)
        torch.cuda.synchronize()
        out[fused] = (dx, gy, dg, db, ds)
    a, b = out[False], out[True]
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    for u, v in zip(a[2:], b[2:]):
        assert rel(v, u) < 1e-5


def ref_attention_drop(qkv, B, S, H, D, causal, seed, salt):
    from oracle.gpt2_fp32 import dropout
    q, k, v = qkv.float().view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    if causal:
        mask = torch.ones(S, S, device=qkv.device, dtype=torch.bool).triu(1)
        s = s.masked_fill(mask, float("-inf"))
    p = dropout(s.softmax(-1).cpu(), P, seed, salt).to(qkv.device)
    return (p @ v).permute(0, 2, 1, 3).reshape(B * S, H * D)


@pytest.mark.parametrize("B,S,H,D,causal", [(2, 256, 4, 64, True), (1, 512, 2, 64, False),
                                            (1, 256, 2, 96, True), (1, 128, 2, 128, True)])
def test_attention_dropout_fwd_bwd(B, S, H, D, causal):
    from paper_2111_04007_b200 import kernels as K
    torch.manual_seed(2)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda").bfloat16()
    o = torch.empty(B * S, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    sb = _seed_buf()
    K.attention_fwd(qkv, o, lse, B, S, H, D, causal, p=P, seed=sb, salt=3)
    q = qkv.float().requires_grad_()
    ref = ref_attention_drop(q, B, S, H, D, causal, SEED, 3)
    assert rel(o, ref) < 1e-2
    do = torch.randn_like(o)
    ref.backward(do.float())
    g = q.grad.view(B * S, 3, H * D)
    ws = torch.empty(K.attention_bwd_ws_elems(B, S, H, D), device="cuda")
    # the pre-drawn keep bits (both layouts): forward and backward reading
    # them draw exactly the hashed masks (dK / dV bitwise: one CTA each)
    nw = K.attention_mask_words(B, S, H)
    mq = torch.zeros(nw, dtype=torch.int32, device="cuda")
    mk = torch.zeros(nw, dtype=torch.int32, device="cuda")
    K.attention_dropout_mask(B, S, H, causal, P, sb, 3, mq, mk)
    o2 = torch.empty_like(o)
    K.attention_fwd(qkv, o2, lse, B, S, H, D, causal, p=P, seed=sb, salt=3, mask=mq)
    assert torch.equal(o, o2)
    for det in (False, True):
        outs = []
        for m in ((None, None), (mq, mk)):
            dqkv = torch.full_like(qkv, float("nan"))
            K.attention_bwd(qkv, o, do, lse, dqkv, ws, B, S, H, D, causal, deterministic=det,
                            p=P, seed=sb, salt=3, mask_q=m[0], mask_k=m[1])
            d = dqkv.view(B * S, 3, H * D)
            for i, name in enumerate("qkv"):
                assert rel(d[:, i], g[:, i]) < 2e-2, (name, det, m[0] is None)
            outs.append(d)
        assert torch.equal(outs[0][:, 1:], outs[1][:, 1:]), det


def test_recompute_is_bitwise_forward_with_dropout():
    """Varuna's R(j) regenerates F(j)'s masks: the saving
    forward equals the checkpointed one bit for bit at p = 0.1."""
    import dataclasses
    from paper_2111_04007_b200.model import CONFIGS, GPT2Stage, StageSpec
    cfg = dataclasses.replace(CONFIGS["tiny"], dropout=P)
    for spec, x in ((StageSpec(1, 3, (1, 2)), "act"), (StageSpec(0, 2, (0, 1)), "ids")):
        st = GPT2Stage(cfg, spec, 4, "cuda", seed=0)
        if x == "act":
            inp, ids = torch.randn(st.T, cfg.hidden, device="cuda").bfloat16(), None
        else:
            inp, ids = None, torch.randint(0, cfg.vocab_size, (st.T,), device="cuda")
        y1 = st.forward(inp, ids, save=False, dseed=SEED).clone()
        y2 = st.forward(inp, ids, save=True, dseed=SEED).clone()
        assert torch.equal(y1, y2)
        y3 = st.forward(inp, ids, save=True, dseed=SEED + 1).clone()
        assert not torch.equal(y1, y3)   # the seed matters
        y0 = GPT2Stage(dataclasses.replace(cfg, dropout=0.0), spec, 4, "cuda", seed=0).forward(
            inp, ids, save=True)
        assert not torch.equal(y1, y0)   # dropout is active


@pytest.mark.parametrize("name", ["tiny", "tiny_bert"])
def test_single_gpu_parity_with_dropout(name):
    """A whole Varuna mini-batch at p = 0.1 (embedding, attention and hidden
    dropout in F and R, differentiated in B) against the fp32 oracle drawing
    the same masks; two steps so the per-step seeds change."""
    import dataclasses
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from oracle.gpt2_fp32 import PipelineOracle
    cfg = dataclasses.replace(CONFIGS[name], dropout=P)
    m, N = 4, 3
    pc = ParallelConfig(1, 1, m, N, (0,) * cfg.n_layer)
    v = Varuna(cfg, pc, seed=0)
    tok = cfg.mlm_per_seq if cfg.arch == "bert" else cfg.seq_len
    for step in (1, 2):
        batch = synthetic_batch(cfg, m * N, 0, step=step)
        res = v.step(batch, apply=False)
        torch.cuda.synchronize()
        o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                           pc.stage_map, m, N, seed=0, arch=cfg.arch, dropout=P)
        loss = o.run_minibatch(batch["input_ids"], batch["labels"], m * N * tok,
                               types=batch.get("token_type_ids"), step=step)
        assert abs(res.loss - loss) / abs(loss) < 5e-3, (step, res.loss, loss)
        og = o.grads()
        for pname, g in v.param_tensors("grad").items():
            assert rel(g, og[pname]) < 3e-2, (step, pname, rel(g, og[pname]))
        v.stage.params.grad.zero_()
    v.close()


def test_graph_replay_with_dropout_matches_eager():
    """Captured task graphs read the seed from device memory: replayed steps
    give the eager steps' losses (fresh masks every step)."""
    import dataclasses
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg = dataclasses.replace(CONFIGS["tiny"], dropout=P)
    losses = {}
    for graphs in (False, True):
        v = Varuna(cfg, ParallelConfig(1, 1, 4, 3, (0,) * cfg.n_layer), seed=0, graphs=graphs)
        losses[graphs] = [v.step(synthetic_batch(cfg, 12, 0, step=s)).loss for s in range(4)]
        if graphs:
            assert len(v._graphs) == 2
        v.close()
    for a, b in zip(losses[False], losses[True]):
        assert abs(a - b) <= 1e-4 * abs(a)
    assert len(set(losses[True])) == 4
