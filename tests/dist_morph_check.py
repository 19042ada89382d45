"""torchrun helper (2 ranks): train 2 mini-batches at 2x1 (pipeline), morph to
1x2 (data parallel) via per-layer sharded checkpoints, train a third; the
loss trajectory must match an unmorphed single-GPU 1x1 run of the same
global mini-batches (same math, different parallelisation)."""

import os
import sys
import tempfile

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import AdamWConfig, Varuna, morph, synthetic_batch
    cfg = CONFIGS["tiny"]
    m = 4
    opt = AdamWConfig(lr=1e-3)
    rows = 16  # M_total
    full = [synthetic_batch(cfg, rows, 0, step=s) for s in range(3)]

    def half(b, r):
        return {k: t[r * rows // 2:(r + 1) * rows // 2] for k, t in b.items()}

    v = Varuna(cfg, ParallelConfig(2, 1, m, 4, (0, 0, 1, 1)), optimizer=opt, seed=0)
    losses = []
    for s in range(2):
        res = v.step(full[s])
        losses.append(res.loss)
    ck = os.path.join(tempfile.gettempdir(), f"vp_morph_{os.environ.get('MASTER_PORT', '0')}")
    if dist.get_rank() == 0:
        import shutil
        shutil.rmtree(ck, ignore_errors=True)
    dist.barrier()
    v = morph(v, ParallelConfig(1, 2, m, 2, (0, 0, 0, 0)), ck, seed=0)
    res = v.step(half(full[2], v.replica))
    losses.append(res.loss)
    loss_tr = torch.tensor([x if x is not None else 0.0 for x in losses], device="cuda")
    # rank 1 was the last stage before the morph; after it both ranks have losses
    dist.all_reduce(loss_tr[:2])
    ok = True
    dist.barrier()
    if dist.get_rank() == 0:
        # unmorphed reference on this GPU alone (separate process group not needed)
        import subprocess
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "morph_ref_run.py")],
                             capture_output=True, text=True, env=dict(os.environ, RANK="0",
                                                                     WORLD_SIZE="1",
                                                                     LOCAL_RANK="0"))
        ref_losses = [float(x) for x in out.stdout.strip().split()[-3:]]
        got = loss_tr.tolist()
        print("morph losses", got, "reference", ref_losses, flush=True)
        ok = all(abs(a - b) / abs(b) < 2e-2 for a, b in zip(got, ref_losses))
        print("MORPH OK" if ok else "MORPH FAIL", flush=True)
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    v.close()
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
