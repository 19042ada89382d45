"""torchrun helper (2 ranks): re-derive the opportunistic dispatch order from
a traced step's measured task times (Varuna.retune_dispatch) and check the
following steps reproduce the static-order run's losses."""

import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from tests._dist import init
    dev, _ = init()
    from paper_2111_04007_b200 import ParallelConfig
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import AdamWConfig, Varuna, synthetic_batch
    cfg = CONFIGS["tiny"]
    pc = ParallelConfig(2, 1, 2, 12, (0, 0, 0, 1))   # unbalanced: stage 0 slower
    losses = {}
    for retune in (False, True):
        v = Varuna(cfg, pc, optimizer=AdamWConfig(lr=1e-3), seed=0)
        out = []
        for s in range(4):
            b = synthetic_batch(cfg, 24, 0, step=s)
            if retune and s == 1:
                v.trace = True
                res = v.step(b)
                v.trace = False
                v.retune_dispatch(res.timeline)
                # grow the bounded activation rings between steps (what a
                # retuned order needing more in-flight slots triggers)
                assert v.n_ring < 12, v.n_ring
                v._resize_rings(12)
                assert v.links.rx_n.get(0, 12) == 12 and v.links.tx_n.get(0, 12) == 12
            else:
                res = v.step(b)
            out.append(res.loss if res.loss is not None else 0.0)
        t = torch.tensor(out, device=dev, dtype=torch.float64)
        dist.all_reduce(t)   # the last stage (rank 1) holds the losses
        losses[retune] = t.tolist()
        v.close()
    ok = all(abs(a - b) <= 1e-3 * abs(a) for a, b in zip(losses[False], losses[True]))
    if dist.get_rank() == 0:
        print("static", losses[False], "retuned", losses[True], flush=True)
        print("RETUNE OK" if ok else "RETUNE FAIL", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
