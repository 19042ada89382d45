"""torchrun helper (2 ranks): train at 2x1 (pipeline), morph twice through
the reference's morph decision (``replan`` = plan(gpus, ...,
micro_batch_size=cached m), sp/morphing.py:327-346) — first with 2 GPUs
available (the planner picks 1x2, data parallel), then with 1 GPU (1x1,
rank 1 becomes a spare) — via per-layer sharded checkpoints written into
the SAME directory each time. The loss trajectory and the final Adam state
must match an unmorphed single-GPU 1x1 run of the same global mini-batches
(same math, different parallelisation)."""

import os
import sys
import tempfile

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STEPS = 5


def main():
    from tests._dist import init, same_device
    dev, backend = init()
    from paper_2111_04007_b200 import ParallelConfig, uniform_profile
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import AdamWConfig, Varuna, morph, synthetic_batch
    cfg = CONFIGS["tiny"]
    m = 4
    opt = AdamWConfig(lr=1e-3)
    rows = 16  # M_total
    full = [synthetic_batch(cfg, rows, 0, step=s) for s in range(STEPS)]
    prof = uniform_profile(cfg.n_layer, 1000.0, 2000.0, m_grid=(m,), d_grid=(1, 2))

    def share(b, v):
        if not v.active:
            return {}
        n = rows // v.D
        return {k: t[v.replica * n:(v.replica + 1) * n] for k, t in b.items()}

    v = Varuna(cfg, ParallelConfig(2, 1, m, 4, (0, 0, 1, 1)), optimizer=opt, seed=0,
               global_batch=rows)
    losses = []
    ck = os.path.join(tempfile.gettempdir(), f"vp_morph_{os.environ.get('MASTER_PORT', '0')}")
    if dist.get_rank() == 0:
        import shutil
        shutil.rmtree(ck, ignore_errors=True)
    dist.barrier()
    configs = []
    for s in range(STEPS):
        if s == 2:
            v = morph(v, ck, gpus=2, profile=prof, seed=0)
        if s == 4:
            v = morph(v, ck, gpus=1, profile=prof, seed=0)
        configs.append((v.P, v.D))
        res = v.step(share(full[s], v))
        losses.append(res.loss)
    # the last-stage rank(s) hold the losses; DP replicas each hold the global mean
    tr = torch.tensor([x if x is not None else 0.0 for x in losses], device=dev)
    cnt = torch.tensor([1.0 if x is not None else 0.0 for x in losses], device=dev)
    dist.all_reduce(tr)
    dist.all_reduce(cnt)
    got = (tr / cnt).tolist()
    # final fp32 master + Adam moments of rank 0 (1x1 owns everything)
    state = None
    if dist.get_rank() == 0:
        state = {k: v.param_tensors(k) for k in ("master",)}
        P = v.stage.params
        state["exp_avg"] = {n: P.view(P.exp_avg, n).float().cpu() for n in P.names}
        state["exp_avg_sq"] = {n: P.view(P.exp_avg_sq, n).float().cpu() for n in P.names}
        step_count = v.step_count
    ok = True
    dist.barrier()
    if dist.get_rank() == 0:
        import subprocess
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "morph_ref_run.py"),
                              str(STEPS), os.path.join(ck, "ref_state.pt")],
                             capture_output=True, text=True,
                             env=dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0"))
        ref_losses = [float(x) for x in out.stdout.strip().split()[-STEPS:]]
        ref = torch.load(os.path.join(ck, "ref_state.pt"))
        print("configs", configs, flush=True)
        print("morph losses", got, "reference", ref_losses, flush=True)
        ok = configs == [(2, 1), (2, 1), (1, 2), (1, 2), (1, 1)]
        ok = ok and all(abs(a - b) / abs(b) < 1e-4 for a, b in zip(got, ref_losses))
        assert step_count == ref["step_count"] == STEPS, (step_count, ref["step_count"])
        # global relative L2 over all tensors (per-tensor errors of the
        # near-zero-gradient entries, e.g. the key bias, are Adam sign noise)
        worst, glob = {}, {}
        for key in ("master", "exp_avg", "exp_avg_sq"):
            num = den = 0.0
            for n, t in state[key].items():
                r = ref[key][n]
                d = (t.float().cpu() - r).norm().item()
                num += d * d
                den += r.norm().item() ** 2
                e = d / max(r.norm().item(), 1e-20)
                if e > worst.get(key, ("", 0.0))[1]:
                    worst[key] = (n, e)
            glob[key] = (num / max(den, 1e-30)) ** 0.5
        print("state rel err (global)", glob, "worst tensor", worst, flush=True)
        ok = ok and glob["master"] < 1e-3 and glob["exp_avg"] < 5e-2 and glob["exp_avg_sq"] < 5e-2
        print("MORPH OK" if ok else "MORPH FAIL", flush=True)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    v.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
