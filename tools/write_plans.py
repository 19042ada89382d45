"""Write profiles/plans.json: the (P, D) -> (m, N_m, stage_map) plan of every
bench configuration, as the reference planner chooses it over the committed
B200 calibration profiles (bench.choose_micro_batch / stage_map_for). Both
bench arms read the committed file, so the reference arm never runs the
product's planner and both arms time the same workload.

    python tools/write_plans.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2111_04007_b200 import JobSpec, micro_batches_for  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS  # noqa: E402

PDS = [(1, 1), (2, 1), (4, 1), (2, 2), (4, 2), (8, 1), (2, 4), (1, 2), (1, 4), (1, 8)]


def main():
    out = {}
    for name, (M, m_default) in bench.MODEL_CONFIGS.items():
        cfg = CONFIGS[name]
        ent = {}
        for P, D in PDS:
            if P > cfg.n_layer:
                continue
            m = bench.choose_micro_batch(cfg, P, D, M, name)
            how = "planner: fastest simulated mini-batch over the B200 calibration m grid"
            if m is None:
                m, how = m_default, "config default (no multi-m calibration profile)"
            N = micro_batches_for(JobSpec(M), m, D)
            ent[f"{P}x{D}"] = {"m": m, "N": N, "M_total": M, "m_choice": how,
                               "stage_map": list(bench.stage_map_for(cfg, P, m, name))}
        out[name] = ent
    path = os.path.join(ROOT, "profiles", "plans.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(path)


if __name__ == "__main__":
    main()
