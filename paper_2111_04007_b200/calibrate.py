"""B200 calibration writer.

Measures, on one B200, the per-CutPoint forward / backward time of a
transformer layer at micro-batch sizes ``m``, the LM/MLM head and the
embedding, and writes a ``CalibrationProfile`` in the reference's YAML format
(``format_version: 1``, sp/calibration.py:321-393) so the reference planner
and simulator (and ours) run on measured B200 numbers:

    python -m paper_2111_04007_b200.calibrate --config gpt2_355m --m 8 \\
        --out profiles/b200_gpt2_355m.yaml

* forward_us[i][m]  = one layer's forward (checkpointed, no saving); the
  embedding is added to cut-point 0, the head's forward to the last one;
* backward_us[i][m] = the layer's backward from its saved working set (the
  recompute is priced by the simulator as R = F, sp/simulator.py:241-253);
* act/grad transfer  = m·s·h·2 bytes over NVLink at the measured 770 GB/s
  peer bandwidth + 5 µs (intra-node; every peer is one NVSwitch hop);
* allreduce_us[i][D] = ring allreduce of the cut-point's fp32 gradient at
  the measured 725 GB/s NVLink bus bandwidth (B200_PROFILING.md).
"""

from __future__ import annotations

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_04007_b200.calibration import (CalibrationProfile, CutpointTimes,  # noqa: E402
                                               ring_allreduce_seconds, save_profile)
from paper_2111_04007_b200.core import us_from_seconds  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS, GPT2Stage, StageSpec  # noqa: E402
from paper_2111_04007_b200.runtime import synthetic_batch  # noqa: E402

PEER_BW = 770e9
AR_BW = 725e9


def _time(fn, iters=5):
    """GPU time of ``fn`` (µs): captured once into a CUDA graph and replayed,
    as the executor runs it, so host launch cost does not inflate it."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        for _ in range(2):
            g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(iters):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # µs


def measure(cfg_name: str, m: int):
    """(layer_f, layer_b, head_f, head_b, embed_f) in µs at micro-batch m."""
    cfg = CONFIGS[cfg_name]
    dev = torch.device("cuda", torch.cuda.current_device())
    mid = GPT2Stage(cfg, StageSpec(1, 3, (1,)), m, dev, seed=0, init_device="cuda")
    x = torch.randn(mid.T, cfg.hidden, device=dev).bfloat16()
    g = torch.randn_like(x) * 1e-3
    # the simulator prices F and R alike (recompute_scale 1): use the saving
    # forward, which is what R (and a last stage's F) executes
    layer_f = _time(lambda: mid.forward(x, None, save=True))
    mid.forward(x, None, save=True)
    layer_b = _time(lambda: mid.backward(g, None))
    del mid
    last = GPT2Stage(cfg, StageSpec(1, 2, (1,)), m, dev, seed=0, init_device="cuda")
    b = synthetic_batch(cfg, m, 0)
    labels = b["labels"].to(dev).view(-1)
    last.forward(x, None, save=True)
    head_fb = _time(lambda: last.loss_and_head_backward(labels, 1e-6))
    del last
    first = GPT2Stage(cfg, StageSpec(0, 2, (0,)), m, dev, seed=0, init_device="cuda")
    ids = b["input_ids"].to(dev).view(-1)
    types = b.get("token_type_ids")
    types = types.to(dev).view(-1) if types is not None else None
    full_f = _time(lambda: first.forward(None, ids, save=True, types=types))
    embed_f = max(full_f - layer_f, 0.0)
    del first
    torch.cuda.empty_cache()
    # head forward ~ 1/3 of its forward+backward (two GEMMs of equal size in bwd)
    return layer_f, layer_b, head_fb / 3.0, 2.0 * head_fb / 3.0, embed_f


def build_profile(cfg_name: str, m_grid, d_grid=(1, 2, 4, 8)) -> CalibrationProfile:
    cfg = CONFIGS[cfg_name]
    meas = {m: measure(cfg_name, m) for m in m_grid}
    grad_bytes = 4 * cfg.layer_param_count()
    cps = []
    for i in range(cfg.n_layer):
        fwd, bwd, tx = {}, {}, {}
        for m in m_grid:
            lf, lb, hf, hb, ef = meas[m]
            f, bb = lf, lb
            if i == 0:
                f += ef
                bb += ef
            if i == cfg.n_layer - 1:
                f += hf
                bb += hb
            fwd[m] = max(1, round(f))
            bwd[m] = max(1, round(bb))
            tx[m] = us_from_seconds(m * cfg.seq_len * cfg.hidden * 2 / PEER_BW) + 5
        ar = {d: us_from_seconds(ring_allreduce_seconds(grad_bytes, d, AR_BW, 5e-6))
              for d in d_grid}
        cps.append(CutpointTimes(fwd, bwd, dict(tx), dict(tx), dict(tx), {m: 0 for m in m_grid},
                                 dict(tx), {m: 0 for m in m_grid}, ar))
    return CalibrationProfile(tuple(sorted(m_grid)), tuple(d_grid), tuple(cps))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt2_355m")
    ap.add_argument("--m", type=int, nargs="+", default=[8])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    prof = build_profile(a.config, a.m)
    out = a.out or f"profiles/b200_{a.config}.yaml"
    save_profile(prof, out)
    cp0, cpl = prof.cutpoints[0], prof.cutpoints[-1]
    m = a.m[0]
    print(f"wrote {out}: layer F/B = {prof.cutpoints[1].forward_us[m]}/"
          f"{prof.cutpoints[1].backward_us[m]} us, first F {cp0.forward_us[m]}, "
          f"last F/B {cpl.forward_us[m]}/{cpl.backward_us[m]} us at m={m}")


if __name__ == "__main__":
    main()
