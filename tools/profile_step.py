"""One short Varuna step for profiling (ncu launch lists / --set full):
GPT-2 config, P=1, N_m micro-batches of m rows, after one warm-up step."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_04007_b200 import ParallelConfig  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS  # noqa: E402
from paper_2111_04007_b200.runtime import Varuna, synthetic_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt2_355m")
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--N", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
cfg = CONFIGS[a.config]
pc = ParallelConfig(1, 1, a.m, a.N, (0,) * cfg.n_layer)
v = Varuna(cfg, pc, seed=0, init_device="cuda")
b = synthetic_batch(cfg, a.m * a.N, 0)
b = {k: t.cuda() for k, t in b.items()}
for _ in range(a.steps):
    v.step(b)
torch.cuda.synchronize()
print("profile_step done")
