"""B200 calibration writer.

Measures on B200s what the reference's ``CalibrationProfile`` prices
(sp/calibration.py:95-110, 162-176, 219-221) and writes it in the
reference's YAML format (``format_version: 1``, sp/calibration.py:321-393),
so the reference planner and simulator (and ours) run on B200 numbers:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        -m paper_2111_04007_b200.calibrate --config gpt2_355m --m 4 8 16 32
    # or, keeping the committed F/B columns and re-measuring the network only:
    ... -m paper_2111_04007_b200.calibrate --config gpt2_355m --comm-only

* forward_us[i][m]  = one layer's saving forward (what R and a last stage's
  F execute); the embedding is added to cut-point 0, the head's forward
  (final LN + logits GEMM, timed by itself) to the last one;
* backward_us[i][m] = the layer's backward from its saved working set; the
  last cut-point adds the head backward (loss + head GEMMs + LN backward =
  head F+B minus the head forward, both measured);
* act/grad transfer  = the K9 put kernel (vp_p2p_put) writing one
  m*s*h*2-byte slot from GPU 0 into GPU 1's IPC-mapped ring, CUDA events on
  the sender's stream (needs >= 2 GPUs; one GPU writes the model at the
  measured-peak NVLink rate instead and says so);
* allreduce_us[i][D] = NCCL allreduce of the cut-point's bf16 gradient
  bucket (2 B/param, the executor's C1 payload) over D of the box's GPUs,
  median of 10; D above the GPUs present is extrapolated from the largest
  measured D's bus bandwidth with the reference's ring formula
  (ring_allreduce_seconds, sp/calibration.py:162-176).

Provenance (measured vs extrapolated, GPU count, clocks) goes to
``<out>.provenance.json`` beside the YAML.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_04007_b200 import kernels as K  # noqa: E402
from paper_2111_04007_b200.calibration import (CalibrationProfile, CutpointTimes,  # noqa: E402
                                               load_profile, ring_allreduce_seconds, save_profile)
from paper_2111_04007_b200.core import us_from_seconds  # noqa: E402
from paper_2111_04007_b200.model import CONFIGS, GPT2Stage, StageSpec  # noqa: E402
from paper_2111_04007_b200.runtime import synthetic_batch  # noqa: E402

PEER_BW_MODEL = 770e9   # used only when a single GPU is present (said in provenance)


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


def measure_compute(cfg_name: str, m: int):
    """(layer_f, layer_b, head_f, head_b, embed_f) in µs at micro-batch m."""
    cfg = CONFIGS[cfg_name]
    dev = torch.device("cuda", torch.cuda.current_device())
    mid = GPT2Stage(cfg, StageSpec(1, 3, (1,)), m, dev, seed=0, init_device="cuda")
    x = torch.randn(mid.T, cfg.hidden, device=dev).bfloat16()
    g = torch.randn_like(x) * 1e-3
    layer_f = _time(lambda: mid.forward(x, None, save=True))
    mid.forward(x, None, save=True)
    layer_b = _time(lambda: mid.backward(g, None))
    del mid
    last = GPT2Stage(cfg, StageSpec(1, 2, (1,)), m, dev, seed=0, init_device="cuda")
    b = synthetic_batch(cfg, m, 0)
    labels = b["labels"].to(dev).view(-1)
    last.forward(x, None, save=True)
    head_fb = _time(lambda: last.loss_and_head_backward(labels, 1e-6))
    if cfg.arch == "bert":
        P = last.params
        xs = last.xs[-1]

        def head_fwd():
            K.gemm(xs, P.w("w_mlm"), last.mlm_act, epilogue=K.EPI_BIAS_GELU, bias=P.w("b_mlm"),
                   aux=last.mlm_pre)
            K.layernorm_fwd(last.mlm_act, P.w("lnm_g"), P.w("lnm_b"), last.lnf_out,
                            last.lnf_mean, last.lnf_rstd, cfg.ln_eps)
            K.gemm(last.lnf_out, P.w(last.head_weight_name), last.logits, epilogue=K.EPI_BIAS,
                   bias=P.w("b_dec"))
    else:
        P = last.params
        xs = last.xs[-1]

        def head_fwd():
            K.layernorm_fwd(xs, P.w("lnf_g"), P.w("lnf_b"), last.lnf_out, last.lnf_mean,
                            last.lnf_rstd, cfg.ln_eps)
            K.gemm(last.lnf_out, P.w(last.head_weight_name), last.logits)
    head_f = _time(head_fwd)
    del last
    first = GPT2Stage(cfg, StageSpec(0, 2, (0,)), m, dev, seed=0, init_device="cuda")
    ids = b["input_ids"].to(dev).view(-1)
    types = b.get("token_type_ids")
    types = types.to(dev).view(-1) if types is not None else None
    full_f = _time(lambda: first.forward(None, ids, save=True, types=types))
    embed_f = max(full_f - layer_f, 0.0)
    del first
    torch.cuda.empty_cache()
    return layer_f, layer_b, head_f, max(head_fb - head_f, 1.0), embed_f


def measure_k9(cfg, m_grid, world, rank, dev):
    """{m: µs} of one K9 slot write GPU 0 -> GPU 1 (IPC-mapped ring), or the
    bandwidth model on one GPU. Collective over the world."""
    from paper_2111_04007_b200.runtime import _Links
    out = {}
    nbytes = {m: m * cfg.seq_len * cfg.hidden * 2 for m in m_grid}
    if world < 2:
        return {m: us_from_seconds(n / PEER_BW_MODEL) + 5 for m, n in nbytes.items()}, "model"
    big = max(nbytes.values())
    buf = None
    info = None
    if rank == 1:
        buf = K.DeviceBuffer(big)
        info = _Links._mem_handle(buf.ptr)
    allinfo = [None] * world
    dist.all_gather_object(allinfo, info)
    if rank == 0:
        dst = _Links._open_mem(allinfo[1])
        src = torch.randn(big // 2, device=dev).bfloat16()
        st = torch.cuda.Stream()
        for m, n in nbytes.items():
            ts = []
            for i in range(11):
                a = torch.cuda.Event(enable_timing=True)
                b_ = torch.cuda.Event(enable_timing=True)
                a.record(st)
                K.p2p_put(dst, src, nbytes=n, stream=st)
                b_.record(st)
                b_.synchronize()
                if i:
                    ts.append(a.elapsed_time(b_) * 1e3)
            out[m] = max(1, round(statistics.median(ts)))
        K.L.vp_ipc_close_mem_handle(dst)
    dist.barrier()
    if buf is not None:
        buf.free()
    res = [out]
    dist.broadcast_object_list(res, src=0)
    return res[0], "measured"


def measure_allreduce(cfg, d_grid, world, rank, dev):
    """{D: µs} of one cut-point's bf16 gradient bucket allreduce (NCCL)."""
    n = cfg.layer_param_count()
    res, how = {1: 0}, {1: "none"}
    meas = [d for d in d_grid if 1 < d <= world]
    busbw = None
    for d in meas:
        grp = dist.new_group(list(range(d)))
        t = None
        if rank < d:
            x = torch.ones(n, dtype=torch.bfloat16, device=dev)
            for _ in range(3):
                dist.all_reduce(x, group=grp)
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                dist.all_reduce(x, group=grp)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            t = statistics.median(ts)
        dist.barrier()
        obj = [t]
        dist.broadcast_object_list(obj, src=0)
        res[d], how[d] = max(1, round(obj[0])), f"measured NCCL on {d} GPUs"
        busbw = 2.0 * (d - 1) / d * 2 * n / (obj[0] * 1e-6)
    for d in d_grid:
        if d not in res:
            bw = busbw or 725e9
            res[d] = us_from_seconds(ring_allreduce_seconds(2 * n, d, bw, 5e-6))
            how[d] = (f"extrapolated (ring formula at the measured {bw / 1e9:.0f} GB/s bus "
                      f"bandwidth of D={max(meas)})" if meas else "model (725 GB/s)")
    return res, how


def build_profile(cfg_name, m_grid, d_grid, world, rank, dev, base=None):
    cfg = CONFIGS[cfg_name]
    if base is None:
        meas = {}
        if rank == 0:
            meas = {m: measure_compute(cfg_name, m) for m in m_grid}
        obj = [meas]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        meas = obj[0]
    else:
        m_grid = base.m_grid
    tx, tx_how = measure_k9(cfg, m_grid, world, rank, dev)
    ar, ar_how = measure_allreduce(cfg, d_grid, world, rank, dev)
    cps = []
    for i in range(cfg.n_layer):
        if base is not None:
            fwd = dict(base.cutpoints[i].forward_us)
            bwd = dict(base.cutpoints[i].backward_us)
        else:
            fwd, bwd = {}, {}
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
        zero = {m: 0 for m in m_grid}
        cps.append(CutpointTimes(fwd, bwd, dict(tx), dict(tx), dict(tx), dict(zero), dict(tx),
                                 dict(zero), dict(ar)))
    prov = {"gpus": world, "transfer": tx_how, "transfer_us": tx,
            "allreduce": {str(d): h for d, h in ar_how.items()},
            "allreduce_us": {str(d): v for d, v in ar.items()},
            "compute": "kept from the base profile" if base is not None else
            "measured (graph-replayed, one B200)",
            "device": torch.cuda.get_device_name(dev)}
    return CalibrationProfile(tuple(sorted(m_grid)), tuple(d_grid), tuple(cps)), prov


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt2_355m")
    ap.add_argument("--m", type=int, nargs="+", default=[8])
    ap.add_argument("--d", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--out", default=None)
    ap.add_argument("--comm-only", action="store_true",
                    help="keep the F/B columns of the existing profile; re-measure K9 and AR")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    out = a.out or f"profiles/b200_{a.config}.yaml"
    base = load_profile(out) if a.comm_only else None
    prof, prov = build_profile(a.config, a.m, a.d, world, rank, dev, base)
    if rank == 0:
        save_profile(prof, out)
        with open(out.replace(".yaml", "") + ".provenance.json", "w") as f:
            json.dump(prov, f, indent=1)
        m = prof.m_grid[0]
        c1 = prof.cutpoints[1]
        print(f"wrote {out}: layer F/B {c1.forward_us[m]}/{c1.backward_us[m]} us at m={m}; "
              f"K9 {prov['transfer_us']} ({prov['transfer']}); AR {prov['allreduce_us']}")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
