"""Unmorphed reference trajectory for dist_morph_check.py: 1x1, same data.
argv: steps, path for the final state (fp32 master + Adam moments)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for k in ("MASTER_ADDR", "MASTER_PORT", "TORCHELASTIC_RUN_ID", "GROUP_RANK", "LOCAL_WORLD_SIZE"):
    os.environ.pop(k, None)
from paper_2111_04007_b200 import ParallelConfig  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS  # noqa: E402
from paper_2111_04007_b200.runtime import AdamWConfig, Varuna, synthetic_batch  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
torch.cuda.set_device(0)
cfg = CONFIGS["tiny"]
v = Varuna(cfg, ParallelConfig(1, 1, 4, 4, (0, 0, 0, 0)), optimizer=AdamWConfig(lr=1e-3), seed=0)
losses = [v.step(synthetic_batch(cfg, 16, 0, step=s)).loss for s in range(steps)]
if len(sys.argv) > 2:
    P = v.stage.params
    torch.save({"master": {n: P.view(P.master, n).float().cpu() for n in P.names},
                "exp_avg": {n: P.view(P.exp_avg, n).float().cpu() for n in P.names},
                "exp_avg_sq": {n: P.view(P.exp_avg_sq, n).float().cpu() for n in P.names},
                "step_count": v.step_count}, sys.argv[2])
print(" ".join(str(x) for x in losses))
