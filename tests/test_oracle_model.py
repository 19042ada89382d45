"""Self-consistency of the fp32 GPT-2 pipeline oracle (CPU): the Varuna
schedule with recompute on P stages must reproduce the single-stage
(non-pipelined) gradients — recompute and micro-batch accumulation are
exact in fp32 up to summation order."""

import torch

from oracle.gpt2_fp32 import PipelineOracle


def _run(stage_map, N=4, m=2, seed=0):
    L, h, H, V, S = 4, 64, 4, 512, 32
    o = PipelineOracle(L, h, H, V, S, stage_map, m, N, seed=seed)
    g = torch.Generator()
    g.manual_seed(5)
    toks = torch.randint(0, V, (N * m, S + 1), generator=g)
    loss = o.run_minibatch(toks[:, :-1].contiguous(), toks[:, 1:].contiguous(), N * m * S)
    return o, loss


def test_pipeline_equals_single_stage():
    o1, l1 = _run([0, 0, 0, 0])
    o2, l2 = _run([0, 0, 1, 1])
    o4, l4 = _run([0, 1, 2, 3])
    assert abs(l1 - l2) < 1e-5 and abs(l1 - l4) < 1e-5
    g1, g2, g4 = o1.grads(), o2.grads(), o4.grads()
    for k in g1:
        for g in (g2, g4):
            err = ((g[k] - g1[k]).norm() / g1[k].norm().clamp_min(1e-12)).item()
            assert err < 1e-4, k


def test_loss_is_mean_token_xent_at_init():
    o, l = _run([0, 0, 0, 0])
    import math
    assert abs(l - math.log(512)) < 0.2  # near-uniform predictions at init


def test_bert_pipeline_equals_single_stage():
    L, h, H, V, S, N, m = 4, 64, 4, 512, 32, 4, 2
    g = torch.Generator()
    g.manual_seed(9)
    ids = torch.randint(0, V, (N * m, S), generator=g)
    types = torch.zeros(N * m, S, dtype=torch.int64)
    types[:, S // 2:] = 1
    labels = torch.full((N * m, S), -100, dtype=torch.int64)
    labels[:, ::5] = torch.randint(0, V, (N * m, (S + 4) // 5), generator=g)
    outs = []
    for sm in ([0, 0, 0, 0], [0, 0, 1, 1]):
        o = PipelineOracle(L, h, H, V, S, sm, m, N, seed=0, arch="bert")
        outs.append((o.run_minibatch(ids, labels, int((labels >= 0).sum()), types=types), o.grads()))
    (l1, g1), (l2, g2) = outs
    assert abs(l1 - l2) < 1e-5
    for k in g1:
        err = ((g2[k] - g1[k]).norm() / g1[k].norm().clamp_min(1e-12)).item()
        assert err < 1e-4, k
