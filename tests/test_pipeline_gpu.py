"""End-to-end parity of the Varuna executor (GPU, bf16 kernels) against the
fp32 CPU oracle (oracle/gpt2_fp32.py) on the tiny GPT-2/BERT configs and on
layer-count cuts of the BASELINE widths (355M, 2.5B, 8.3B, BERT-large).

Tolerances (stated here): loss |Δ|/|loss| <= 5e-3;
per-tensor gradient relative L2 <= 3e-2; weights after one AdamW step
relative L2 <= 1e-2 (of the update-carrying tensors). Dropout p = 0.
"""

import math
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tiny_setup(P=1, D=1, N=4, m=4, name="tiny"):
    from paper_2111_04007_b200 import ParallelConfig, assign_stages, make_block_model, uniform_profile
    from paper_2111_04007_b200.model import CONFIGS
    cfg = CONFIGS[name]
    model = make_block_model(name, cfg.n_layer, cfg.hidden, cfg.seq_len)
    a = assign_stages(model, P, m, uniform_profile(cfg.n_layer, 1.0, 2.0, m_grid=(m,)))
    pc = ParallelConfig(P, D, m, N, a.stage_map)
    return cfg, pc


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


def oracle_run(cfg, pc, batch, steps=0):
    from oracle.gpt2_fp32 import PipelineOracle
    o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                       pc.stage_map, pc.micro_batch_size, pc.num_micro_batches, seed=0)
    total = pc.micro_batch_size * pc.num_micro_batches * pc.data_parallel * cfg.seq_len
    loss = o.run_minibatch(batch["input_ids"], batch["labels"], total)
    return o, loss


@pytest.mark.parametrize("name", ["tiny", "tiny_ragged"])
def test_single_gpu_loss_grads_and_update(name):
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg, pc = tiny_setup(name=name)
    batch = synthetic_batch(cfg, pc.micro_batch_size * pc.num_micro_batches, 0)
    v = Varuna(cfg, pc, seed=0)
    res = v.step(batch, apply=False)
    torch.cuda.synchronize()
    o, loss = oracle_run(cfg, pc, batch)
    assert abs(res.loss - loss) / abs(loss) < 5e-3, (res.loss, loss)
    og = o.grads()
    got = v.param_tensors("grad")
    for name, g in got.items():
        key = name
        assert key in og, name
        assert rel(g, og[key]) < 3e-2, (name, rel(g, og[key]))
    # optimizer: apply on both sides. Adam's first update is ~lr*sign(g), so
    # compare the UPDATE direction (cosine >= 0.9 over entries whose oracle
    # gradient is >= 5% of the tensor's RMS gradient — entries with ~zero
    # true gradient, e.g. the key bias, get a noise-sign update) and the weights (rel L2 <= 1e-2 where non-zero).
    before = {k: t.clone() for k, t in v.param_tensors("master").items()}
    ref_before = {k: p.detach().clone() for k, p in o.params.items()}
    v._optimizer_step()
    o.adamw_step(1)
    torch.cuda.synchronize()
    for name, t in v.param_tensors("master").items():
        ref = o.params[name].detach()
        d_gpu = (t - before[name]).float().cpu().flatten()
        d_ref = (ref - ref_before[name]).flatten()
        gref = og[name].flatten().abs()
        keep = gref >= 0.05 * gref.pow(2).mean().sqrt()  # drop ~zero-gradient entries
        cos = torch.nn.functional.cosine_similarity(d_gpu[keep], d_ref[keep], dim=0).item()
        assert cos > 0.9, (name, cos)
        if ref_before[name].norm() > 0:
            assert rel(t, ref) < 1e-2, name


def test_bert_single_gpu_loss_and_grads():
    """Post-LN BERT (tiny_bert: 4x256, s=128, bidirectional, MLM head with
    tied decoder) vs the fp32 oracle."""
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from oracle.gpt2_fp32 import PipelineOracle
    cfg = CONFIGS["tiny_bert"]
    m, N = 4, 4
    pc = ParallelConfig(1, 1, m, N, (0,) * cfg.n_layer)
    batch = synthetic_batch(cfg, m * N, 0)
    v = Varuna(cfg, pc, seed=0)
    res = v.step(batch, apply=False)
    torch.cuda.synchronize()
    o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                       pc.stage_map, m, N, seed=0, arch="bert")
    loss = o.run_minibatch(batch["input_ids"], batch["labels"], m * N * cfg.mlm_per_seq,
                           types=batch["token_type_ids"])
    assert abs(res.loss - loss) / abs(loss) < 5e-3, (res.loss, loss)
    og = o.grads()
    for name, g in v.param_tensors("grad").items():
        if name == "tte":  # only rows 0/1 exist; compare whole table
            pass
        assert rel(g, og[name]) < 3e-2, (name, rel(g, og[name]))


def test_partial_minibatch_and_loss_scale():
    """M_total not divisible by m*D (sp/planner.py:99-103: N_m = ceil(M/(m*D)),
    the last micro-batch partial): the loss is the mean over M_total samples
    and the gradients match the oracle's; with a loss scale of 1024 the
    reported loss is unscaled and the stored gradients carry the scale."""
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from oracle.gpt2_fp32 import PipelineOracle
    cfg = CONFIGS["tiny"]
    m, N, M, scale = 4, 4, 14, 1024.0
    pc = ParallelConfig(1, 1, m, N, (0,) * cfg.n_layer)
    batch = synthetic_batch(cfg, M, 0)
    v = Varuna(cfg, pc, seed=0, global_batch=M, loss_scale=scale)
    res = v.step(batch, apply=False)
    torch.cuda.synchronize()
    o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                       pc.stage_map, m, N, seed=0)
    loss = o.run_minibatch(batch["input_ids"], batch["labels"], M * cfg.seq_len)
    assert abs(res.loss - loss) / abs(loss) < 5e-3, (res.loss, loss)
    og = o.grads()
    for name, g in v.param_tensors("grad").items():
        assert rel(g / scale, og[name]) < 3e-2, (name, rel(g / scale, og[name]))
    assert abs(res.grad_norm - math.sqrt(sum(float((t * t).sum()) for t in og.values()))) \
        < 3e-2 * res.grad_norm
    with pytest.raises(Exception):
        Varuna(cfg, pc, seed=0, global_batch=12)   # would need only 3 micro-batches
    v.close()


def test_recompute_is_bitwise_forward():
    from paper_2111_04007_b200.model import CONFIGS, GPT2Stage, StageSpec
    cfg = CONFIGS["tiny"]
    st = GPT2Stage(cfg, StageSpec(1, 3, (1, 2)), 4, "cuda", seed=0)
    x = torch.randn(st.T, cfg.hidden, device="cuda").bfloat16()
    y1 = st.forward(x, None, save=False).clone()
    y2 = st.forward(x, None, save=True).clone()
    assert torch.equal(y1, y2)


def test_loss_decreases_over_steps():
    from paper_2111_04007_b200.runtime import AdamWConfig, Varuna, synthetic_batch
    cfg, pc = tiny_setup()
    batch = synthetic_batch(cfg, pc.micro_batch_size * pc.num_micro_batches, 0)
    v = Varuna(cfg, pc, seed=0, optimizer=AdamWConfig(lr=1e-3))
    losses = [v.step(batch).loss for _ in range(8)]
    assert losses[-1] < losses[0] - 0.1, losses


def test_gantt_export_format():
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg = CONFIGS["tiny"]
    v = Varuna(cfg, ParallelConfig(1, 1, 4, 2, (0,) * 4), seed=0, trace=True)
    res = v.step(synthetic_batch(cfg, 8, 0))
    rows = v.gantt_rows(res.timeline)
    text = v.gantt_csv(rows)
    lines = text.strip().splitlines()
    assert lines[0] == "stage,kind,microbatch,start_us,end_us"
    assert len(lines) - 1 == 2 * 2 + 1  # F,B per micro-batch + allreduce row
    kinds = [ln.split(",")[1] for ln in lines[1:]]
    assert kinds.count("F") == 2 and kinds.count("B") == 2 and kinds.count("A") == 1


def test_graph_replay_matches_eager():
    """Steps replayed from captured CUDA graphs give the losses of eager
    execution (attention dQ is summed in CTA order: fp32-level tolerance)."""
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg = CONFIGS["tiny"]
    losses = {}
    for graphs in (False, True):
        v = Varuna(cfg, ParallelConfig(1, 1, 4, 3, (0,) * cfg.n_layer), seed=0, graphs=graphs)
        out = []
        for s in range(4):
            b = synthetic_batch(cfg, 12, 0, step=s)
            out.append(v.step(b).loss)
        losses[graphs] = out
        if graphs:
            assert len(v._graphs) == 2  # one F and one B graph serve every micro-batch
        v.close()
    for a, b in zip(losses[False], losses[True]):
        assert abs(a - b) <= 1e-4 * abs(a)


@pytest.mark.parametrize("name,n_layer,m,N", [("gpt2_355m", 2, 1, 2), ("gpt2_2_5b", 1, 1, 1),
                                                 ("gpt2_8_3b", 1, 1, 1)])
def test_full_width_layers_match_oracle(name, n_layer, m, N):
    """The BASELINE model widths (355M: h=1024, 16 heads; 2.5B: h=1920, 20
    heads of 96; 8.3B: h=3072, 32 heads; s=1024, V=51200) with the layer count cut to what the fp32 CPU
    oracle runs in ~10 s: loss and every gradient under the tolerances of
    the module docstring, so the full-size GEMM/attention/LN tilings run
    in-model, not just the tiny ones."""
    import dataclasses
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg = dataclasses.replace(CONFIGS[name], n_layer=n_layer)
    pc = ParallelConfig(1, 1, m, N, (0,) * n_layer)
    batch = synthetic_batch(cfg, m * N, 0)
    v = Varuna(cfg, pc, seed=0)
    res = v.step(batch, apply=False)
    torch.cuda.synchronize()
    o, loss = oracle_run(cfg, pc, batch)
    assert abs(res.loss - loss) / abs(loss) < 5e-3, (res.loss, loss)
    og = o.grads()
    for pname, g in v.param_tensors("grad").items():
        assert rel(g, og[pname]) < 3e-2, (pname, rel(g, og[pname]))


def test_bert_large_width_layer_matches_oracle():
    """BERT-large width (h=1024, 16 heads, s=512, V=30528, post-LN, MLM head)
    with one layer, two micro-batches of 2, against the fp32 oracle."""
    import dataclasses
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from oracle.gpt2_fp32 import PipelineOracle
    cfg = dataclasses.replace(CONFIGS["bert_large"], n_layer=1)
    m, N = 2, 2
    pc = ParallelConfig(1, 1, m, N, (0,))
    batch = synthetic_batch(cfg, m * N, 0)
    v = Varuna(cfg, pc, seed=0)
    res = v.step(batch, apply=False)
    torch.cuda.synchronize()
    o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                       pc.stage_map, m, N, seed=0, arch="bert")
    loss = o.run_minibatch(batch["input_ids"], batch["labels"], m * N * cfg.mlm_per_seq,
                           types=batch["token_type_ids"])
    assert abs(res.loss - loss) / abs(loss) < 5e-3, (res.loss, loss)
    og = o.grads()
    for pname, g in v.param_tensors("grad").items():
        assert rel(g, og[pname]) < 3e-2, (pname, rel(g, og[pname]))


def test_dynamic_loss_scaler_skip_and_recover():
    """Dynamic loss scaling (LossScaler, device-resident state): a step whose
    gradients hold a non-finite value is skipped on the device (master and
    Adam moments untouched, Adam's applied-step count unchanged, gradients
    zeroed) and the scale backs off; the next clean step is applied as Adam
    step 1 and equals a fresh run's first step at that scale; after
    ``window`` clean steps the scale grows."""
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import AdamWConfig, LossScaler, Varuna, synthetic_batch
    cfg = CONFIGS["tiny"]
    pc = ParallelConfig(1, 1, 4, 2, (0,) * cfg.n_layer)
    opt = AdamWConfig(lr=1e-3)
    b = [synthetic_batch(cfg, 8, 0, step=s) for s in range(4)]
    v = Varuna(cfg, pc, seed=0, optimizer=opt,
               loss_scale=LossScaler(init=2.0 ** 16, dynamic=True, window=2))
    P = v.stage.params
    w0 = P.master.clone()
    m0 = P.exp_avg.clone()
    v.step(b[0], apply=False)
    P.grad[123] = float("inf")            # an overflowed gradient
    with torch.cuda.stream(v.stream):
        v._sync_grads()
        v._optimizer_step()
    torch.cuda.synchronize()
    assert v.flags[1].item() > 0
    assert torch.equal(P.master, w0) and torch.equal(P.exp_avg, m0)
    assert P.grad.abs().max().item() == 0.0
    assert v._ss.tolist()[:3] == [2.0 ** 15, 0.0, 0.0]
    r = v.step(b[1])
    assert not r.overflow and r.loss_scale == 2.0 ** 15
    ref = Varuna(cfg, pc, seed=0, optimizer=opt, loss_scale=2.0 ** 15)
    rr = ref.step(b[1])
    torch.cuda.synchronize()
    assert abs(r.loss - rr.loss) <= 1e-6 * abs(rr.loss)
    assert (P.master - ref.stage.params.master).abs().max().item() <= 1e-6
    assert v._ss.tolist()[:3] == [2.0 ** 15, 1.0, 1.0]
    r = v.step(b[2])                       # second clean step: window reached
    torch.cuda.synchronize()
    assert v._ss.tolist()[:3] == [2.0 ** 16, 2.0, 0.0]
    v.close()
    ref.close()


def test_module_with_cutpoints_equals_config():
    """Varuna over a model structure with user CutPoints (every 2 layers) runs
    the same math as over the config (one CutPoint per layer)."""
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.modules import GPT2
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    cfg = CONFIGS["tiny"]
    batch = synthetic_batch(cfg, 8, 0)
    a = Varuna(GPT2(cfg, cut_every=2), ParallelConfig(1, 1, 4, 2, (0, 0)), seed=0)
    b = Varuna(cfg, ParallelConfig(1, 1, 4, 2, (0,) * cfg.n_layer), seed=0)
    assert a.pc.stage_map == (0,) * cfg.n_layer
    la, lb = a.step(batch).loss, b.step(batch).loss
    assert abs(la - lb) <= 2e-6 * abs(lb), (la, lb)   # fp32 atomic loss sum order
    a.close()
    b.close()
