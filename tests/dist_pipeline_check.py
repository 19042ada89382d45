"""torchrun helper: run one Varuna mini-batch on P*D GPUs and compare each
rank's gradients / the loss with the fp32 CPU oracle (tiny GPT-2)."""

import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def skewed_profile(m=4):
    """Unbalanced 4-cut-point profile with slow, jittery links under which the
    opportunistic replica kernel departs from the static order at P=2, N=4."""
    from paper_2111_04007_b200.calibration import CalibrationProfile, CutpointTimes
    cps = tuple(CutpointTimes({m: f}, {m: 2 * f}, {m: 195}, {m: 16}, {m: 195}, {m: 16},
                              {m: 195}, {m: 16}, {1: 0}) for f in (84, 195, 266, 255))
    return CalibrationProfile((m,), (1,), cps)



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--D", type=int, default=1)
    ap.add_argument("--N", type=int, default=4)
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--dispatch", default="static")
    ap.add_argument("--layers", type=int, default=0, help="cut the config to this many layers")
    ap.add_argument("--micro-batch", type=int, default=4)
    ap.add_argument("--dropout", type=float, default=0.0)
    ap.add_argument("--cut-every", type=int, default=0,
                    help="build the model as modules.GPT2 with a CutPoint every this many "
                         "layers (stage map over the CutPoint blocks)")
    ap.add_argument("--steps", type=int, default=1,
                    help="train steps-1 steps (AdamW on both sides), check the last")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="M_total (default m*N*D); smaller values leave partial micro-batches")
    args = ap.parse_args()
    from tests._dist import init
    dev, _ = init()
    from paper_2111_04007_b200 import ParallelConfig, assign_stages, make_block_model, uniform_profile
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from oracle.gpt2_fp32 import PipelineOracle
    cfg = CONFIGS[args.config]
    import dataclasses
    if args.layers:
        cfg = dataclasses.replace(cfg, n_layer=args.layers)
    if args.dropout:
        cfg = dataclasses.replace(cfg, dropout=args.dropout)
    P, D, N, m = args.P, args.D, args.N, args.micro_batch
    module = None
    if args.cut_every:
        from paper_2111_04007_b200.modules import GPT2
        module = GPT2(cfg, cut_every=args.cut_every)
        spec = module.model_spec()
        a = assign_stages(spec, P, m, uniform_profile(spec.num_cutpoints, 1.0, 2.0, m_grid=(m,)))
    else:
        model = make_block_model("tiny", cfg.n_layer, cfg.hidden, cfg.seq_len)
        a = assign_stages(model, P, m, uniform_profile(cfg.n_layer, 1.0, 2.0, m_grid=(m,)))
    pc = ParallelConfig(P, D, m, N, a.stage_map)
    prof = None
    if args.dispatch == "opportunistic":
        # unbalanced per-cut-point times + slow, jittery links: the replica
        # kernel reorders tasks relative to the static schedule
        prof = skewed_profile(m)
    M = args.global_batch or m * N * D
    v = Varuna(module if module is not None else cfg, pc, seed=0, dispatch=args.dispatch,
               profile=prof, global_batch=M)
    if module is not None:
        pc = v.pc        # the per-layer stage map the oracle walks
    if args.dispatch == "opportunistic":
        kinds, mbs = v.schedule.stage_slice(v.stage_id)
        moved = sum(a != b for a, b in zip(zip(kinds.tolist(), mbs.tolist()), v.tasks))
        print(f"rank {v.rank} dispatch order differs from static at {moved} positions", flush=True)
    print(f"rank {v.rank} ring slots {v.n_ring} (act) {v.n_grad} (grad) for N_m = {N}", flush=True)
    shares = [min(max(M - r * m * N, 0), m * N) for r in range(D)]
    o = PipelineOracle(cfg.n_layer, cfg.hidden, cfg.heads, cfg.vocab_size, cfg.seq_len,
                       pc.stage_map, m, N, seed=0, arch=cfg.arch, dropout=cfg.dropout)
    total = M * (cfg.mlm_per_seq if cfg.arch == "bert" else cfg.seq_len)
    for step in range(1, args.steps + 1):
        batches = [{k: t[:shares[r]] for k, t in synthetic_batch(cfg, m * N, r,
                                                                   step=step - 1).items()}
                   for r in range(D)]
        final = step == args.steps
        res = v.step(batches[v.replica], apply=not final)
        torch.cuda.synchronize()
        if v.dispatch == "live":
            # the executed order is a valid Varuna execution: rule 2 and the
            # last stage's F/B alternation (checked against the policy's own
            # bookkeeping: every task exactly once)
            assert sorted(v.executed) == sorted(v.tasks), v.executed
            for i, (kind, j) in enumerate(v.executed):
                if kind == 0:
                    assert v.executed[i - 1] == ((2 if v.spec.last else 1), j), v.executed
        # oracle: D replicas' mini-batches, summed gradients
        loss = sum(o.run_minibatch(b["input_ids"], b["labels"], total,
                                   types=b.get("token_type_ids"), step=step, replica=r)
                   for r, b in enumerate(batches))
        if not final:
            o.adamw_step(step)
    og = o.grads()
    ok = True
    for name, g in v.param_tensors("grad").items():
        key = "wte" if name == "wte_head" else name
        ref = og[key]
        err = ((g.float().cpu() - ref).norm() / ref.norm().clamp_min(1e-12)).item()
        if err > 3e-2:
            print(f"rank {v.rank} {name}: rel err {err:.3e}", flush=True)
            ok = False
    if v.spec.last:
        lerr = abs(res.loss - loss) / abs(loss)
        print(f"rank {v.rank} loss {res.loss:.6f} oracle {loss:.6f} rel {lerr:.2e}", flush=True)
        ok = ok and lerr < 5e-3
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    v.close()
    if dist.get_rank() == 0:
        print("PARITY OK" if flag.item() == 0 else "PARITY FAIL", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
