"""Benchmark: Varuna pipeline training throughput (samples/s) on 1/2/4/8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt2_355m]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...     # the reference-side CPU arm

One step = one mini-batch of M_total samples (BASELINE config 2: GPT-2 355M,
M_total = 512, m = 8) through the Varuna schedule on P×D GPUs, with the
gradient allreduce and the AdamW update — the whole training step. The P×D
ladder at fixed M_total (strong scaling): 1 → 1×1, 2 → 2×1, 4 → 4×1,
8 → 4×2 (the BASELINE.json configuration). Stage maps come from the
reference's ``assign_stages`` over a FLOP-proportional calibration profile
with the LM head folded into the last cut-point and the last stage weighted
0.75 (it runs no recompute), which is how the planner would balance it.

Rank 0 prints ONE JSON line (see the driver contract in the task). Timing:
CUDA events on the executor's compute stream, barrier + synchronize on both
sides, max over ranks. The step's working set (weights, optimizer state,
activations: several GB) is far larger than the 126 MB L2, so no explicit
flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LADDER = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
METRIC_NAMES = {"gpt2_355m": "GPT-2 355M", "gpt2_2_5b": "GPT-2 2.5B", "gpt2_8_3b": "GPT-2 8.3B",
                "tiny": "tiny GPT-2", "bert_large": "BERT-large"}
MODEL_CONFIGS = {  # name: (M_total, m)
    "gpt2_355m": (512, 8),
    "gpt2_2_5b": (256, 4),
    "gpt2_8_3b": (512, 4),
    "bert_large": (8192, 32),
    "tiny": (16, 4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vpipe", choices=["vpipe", "reference"])
    ap.add_argument("--config", default="gpt2_355m", choices=sorted(MODEL_CONFIGS))
    ap.add_argument("--pd", default=None, help="override P x D, e.g. 4x2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--m", default="auto",
                    help="micro-batch size: 'auto' (the planner's choice over the calibration "
                         "profile's m grid) or an integer")
    ap.add_argument("--dispatch", default="opportunistic",
                    choices=["opportunistic", "live", "static"],
                    help="P>1 task order: the reference's opportunistic policy replayed over "
                         "the calibration profile (default), run live on real arrivals, or the "
                         "static Varuna schedule")
    ap.add_argument("--no-retune", action="store_true",
                    help="opportunistic replay: keep the order derived from the calibration "
                         "profile instead of re-deriving it (reference policy, replica kernel) "
                         "from one traced step's MEASURED stage times")
    ap.add_argument("--retune-perturb", action="store_true",
                    help="also try the replica kernel's orders under x0.85..1.15-scaled "
                         "times (off by default)")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    ap.add_argument("--dropout", type=float, default=None,
                    help="hidden + attention dropout of the run (default: the config's)")
    ap.add_argument("--side-dropout", type=float, default=0.1,
                    help="also time the same workload at this dropout (SURVEY §8(d): 0.1 for "
                         "perf runs) and report it beside the headline; 0 disables")
    ap.add_argument("--trace-dir", default=None,
                    help="write every rank's measured Gantt CSV of the traced step here")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    except Exception:  # noqa: BLE001
        return 1590.0, 1400.0, 6650.0, "fallback"


def stage_map_for(cfg, P, m, config_name=None):
    """Stage map by the reference DP (assign_stages). With a B200 calibration
    profile (profiles/b200_<config>.yaml, written by
    paper_2111_04007_b200.calibrate) each cut-point is priced at its executed
    cost on a recomputing stage, 2F_i + B_i, and the last stage (no
    recompute) is weighted by (F+B)/(2F+B); otherwise a FLOP-proportional
    profile with the head folded into the last cut-point, weight 0.75."""
    from paper_2111_04007_b200 import assign_stages, load_profile, make_block_model
    from paper_2111_04007_b200.calibration import CalibrationProfile, CutpointTimes
    path = os.path.join(ROOT, "profiles", f"b200_{config_name}.yaml") if config_name else ""
    if P > 1 and path and os.path.exists(path):
        prof = load_profile(path)
        if m in prof.m_grid and prof.num_cutpoints == cfg.n_layer:
            cost = [2 * prof.forward_us(i, m) + prof.backward_us(i, m) for i in range(cfg.n_layer)]
            f1, b1 = prof.forward_us(1, m), prof.backward_us(1, m)
            z = {m: 0}
            cps = tuple(CutpointTimes({m: c}, {m: c}, z, z, z, z, z, z, {1: 0}) for c in cost)
            model = make_block_model(cfg_name(cfg), cfg.n_layer, cfg.hidden, cfg.seq_len)
            return assign_stages(model, P, m, CalibrationProfile((m,), (1,), cps),
                                 last_stage_weight=(f1 + b1) / (2 * f1 + b1)).stage_map
    per_layer = cfg.flops_per_token_layer() * cfg.seq_len * m
    head = cfg.head_flops_per_token() * cfg.seq_len * m
    us = [max(1, round(per_layer / 1e9))] * cfg.n_layer
    us[-1] += max(1, round(head / 1e9))
    z = {m: 0}
    cps = tuple(CutpointTimes({m: t}, {m: 2 * t}, z, z, z, z, z, z, {1: 0}) for t in us)
    prof = CalibrationProfile((m,), (1,), cps)
    model = make_block_model(cfg_name(cfg), cfg.n_layer, cfg.hidden, cfg.seq_len)
    return assign_stages(model, P, m, prof, last_stage_weight=0.75 if P > 1 else 1.0).stage_map


def choose_micro_batch(cfg, P, D, M, config_name):
    """Micro-batch size as the reference planner chooses it (sp/planner.py:
    106-145): simulate the mini-batch for every m of the B200 calibration
    profile's grid (Varuna schedule, opportunistic dispatch, the stage map
    assign_stages picks at that m) and keep the fastest. None without a
    multi-m profile."""
    from paper_2111_04007_b200 import (ParallelConfig, build_placement, generate_varuna_schedule,
                                       load_profile, make_block_model, simulate_minibatch,
                                       uniform_cluster, JobSpec, micro_batches_for)
    path = os.path.join(ROOT, "profiles", f"b200_{config_name}.yaml")
    if not os.path.exists(path):
        return None
    prof = load_profile(path)
    if len(prof.m_grid) < 2 or prof.num_cutpoints != cfg.n_layer:
        return None
    model = make_block_model(cfg_name(cfg), cfg.n_layer, cfg.hidden, cfg.seq_len)
    place = build_placement(uniform_cluster(P * D, 8), P, D)
    best, best_t = None, None
    for m in prof.m_grid:
        N = micro_batches_for(JobSpec(M), m, D)
        if N < P:  # fewer micro-batches than stages: the pipeline cannot fill
            continue
        sm = stage_map_for(cfg, P, m, config_name)
        pc = ParallelConfig(P, D, m, N, tuple(sm))
        t = simulate_minibatch(generate_varuna_schedule(P, N, 1.0, 2.0, 1.0), pc, prof, place,
                               model, opportunistic=P > 1).minibatch_us
        if best_t is None or t < best_t:
            best, best_t = m, t
    return best


def gemm_traffic():
    """DRAM bytes per launch of the representative GEMM (FC1 shape) from the
    committed ncu --set full capture (profiles/r01e_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "r02t_traffic.json")) as f:
            t = json.load(f)
        return {"bytes_per_launch": t["dram_bytes"], "algorithmic_bytes": t["algorithmic_bytes"],
                "kernel": t["kernel"], "source": t["source"]}
    except (OSError, KeyError, ValueError):
        return None


def cfg_name(cfg):
    return f"{getattr(cfg, 'arch', 'gpt2')}-L{cfg.n_layer}-h{cfg.hidden}"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-i", str(index), "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        loaded = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU arm
# Everything in this section runs WITHOUT importing the product package
# (paper_2111_04007_b200 / libvpipe.so): the reference arm times the
# reference's own control plane (spotpipe from baseline/_ref) and the fp32
# CPU port of the executor's tensor path (oracle/gpt2_fp32.py — the reference
# has no tensor math), on a plan read from the committed
# profiles/plans.json.

# (n_layer, hidden, heads, vocab, seq, arch, mlm_per_seq) — the BASELINE
# model shapes, restated here so the CPU arm does not import the product
MODEL_DIMS = {
    "tiny": (4, 256, 4, 50304, 128, "gpt2", 0),
    "gpt2_355m": (24, 1024, 16, 51200, 1024, "gpt2", 0),
    "gpt2_2_5b": (54, 1920, 20, 51200, 1024, "gpt2", 0),
    "gpt2_8_3b": (72, 3072, 32, 51200, 1024, "gpt2", 0),
    "bert_large": (24, 1024, 16, 30528, 512, "bert", 77),
}
# north-star P x D of each BASELINE config (BASELINE.json "configs")
NORTH_STAR_PD = {"tiny": (2, 1), "gpt2_355m": (4, 2), "bert_large": (2, 4),
                 "gpt2_2_5b": (8, 1), "gpt2_8_3b": (4, 2)}
# the fp32 CPU port keeps params + grads + Adam state on the host: models
# above this many layers x hidden^2 run a layer cut, extrapolated
CPU_FULL_MODEL_MAX = 24 * 1024 ** 2


def load_plan(config, P, D):
    """The committed plan (tools/write_plans.py) for this config at P x D."""
    with open(os.path.join(ROOT, "profiles", "plans.json")) as f:
        plans = json.load(f)
    ent = plans.get(config, {}).get(f"{P}x{D}")
    if ent is None:
        raise SystemExit(f"no committed plan for {config} {P}x{D} in profiles/plans.json "
                         "(run tools/write_plans.py)")
    return ent


def _ladder_pd(args, world):
    if args.pd:
        return tuple(map(int, args.pd.lower().split("x")))
    return LADDER.get(world, (world, 1))


def _timeit(fn, min_s=0.2, max_reps=2000):
    """Median wall time (s) of fn() over repetitions filling ~min_s."""
    ts = []
    t_end = time.perf_counter() + min_s
    while len(ts) < 3 or (time.perf_counter() < t_end and len(ts) < max_reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def control_plane_times(api, plans, configs=None):
    """Single-threaded wall time (us) of the control-plane entry points the
    executor depends on: the Varuna plan (uncached),
    assign_stages over the B200 calibration profile, and simulate_minibatch
    (opportunistic), at each BASELINE config's north-star P x D. ``api`` is
    the reference's spotpipe module or the product package (C++ twins)."""
    out = {}
    for name in configs or NORTH_STAR_PD:
        P, D = NORTH_STAR_PD[name]
        ent = plans.get(name, {}).get(f"{P}x{D}")
        prof_path = os.path.join(ROOT, "profiles", f"b200_{name}.yaml")
        if ent is None or not os.path.exists(prof_path):
            continue
        L, h, _, _, S, _, _ = MODEL_DIMS[name]
        m, N = ent["m"], ent["N"]
        prof = api.load_profile(prof_path)
        if m not in prof.m_grid:
            continue
        model = api.make_block_model(name, L, h, S)
        gen = getattr(api.generate_varuna_schedule, "__wrapped__", api.generate_varuna_schedule)
        sched = gen(P, N, 1.0, 2.0, 1.0)
        pc = api.ParallelConfig(P, D, m, N, tuple(ent["stage_map"]))
        place = api.build_placement(api.uniform_cluster(P * D, 8), P, D)
        out[f"{name} {P}x{D} N_m={N}"] = {
            "generate_varuna_schedule_us": round(1e6 * _timeit(
                lambda: gen(P, N, 1.0, 2.0, 1.0)), 1),
            "assign_stages_us": round(1e6 * _timeit(
                lambda: api.assign_stages(model, P, m, prof)), 1),
            "simulate_minibatch_us": round(1e6 * _timeit(
                lambda: api.simulate_minibatch(sched, pc, prof, place, model,
                                               opportunistic=True)), 1),
        }
    return out


def reference_control_plane(plans):
    """The reference's own CPU control plane (spotpipe 0.1.0 installed
    unmodified into baseline/_ref; its compiled Cython replica kernel when
    it built), or a one-line reason it is unavailable."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "spotpipe")):
        return {"unavailable": "baseline/_ref/spotpipe not installed"}
    sys.path.insert(0, ref)
    try:
        import spotpipe
        import spotpipe.engine as eng
        res = control_plane_times(spotpipe, plans)
        res["engine"] = eng.ENGINE_NAME
        return res
    except Exception as ex:  # noqa: BLE001
        return {"unavailable": f"spotpipe import/run failed: {ex}"}
    finally:
        sys.path.remove(ref)


class CpuPipelineSample:
    """The executor's tensor path on the host cores: the fp32 torch-CPU port
    (oracle/gpt2_fp32.py) walking the Varuna plan of this config's stage map
    for ONE sample per step (m = 1, one micro-batch: F, R on every
    recomputing stage, B), plus 1/M_total of one AdamW update over all
    parameters (timed once). Models too large to hold fp32 params + grads +
    Adam state on the host run a cut of the layers and the time is scaled by
    the layer count (said in ``sample``)."""

    def __init__(self, config, stage_map):
        import torch
        from oracle.gpt2_fp32 import PipelineOracle
        self.threads = os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        L, h, H, V, S, arch, mlm = MODEL_DIMS[config]
        self.config, self.S, self.V, self.arch, self.mlm = config, S, V, arch, mlm
        self.L = L
        P = max(stage_map) + 1
        cut = L
        if L * h * h > CPU_FULL_MODEL_MAX:
            cut = max(P, (CPU_FULL_MODEL_MAX // (h * h)) // P * P)
        # the same P-stage structure on the cut: layers spread evenly
        smap = [min(P - 1, i * P // cut) for i in range(cut)] if cut != L else list(stage_map)
        self.cut = cut
        self.o = PipelineOracle(cut, h, H, V, S, smap, 1, 1, seed=0, arch=arch)
        self.P = P
        g = torch.Generator()
        g.manual_seed(1234)
        toks = torch.randint(0, V, (1, S + 1), generator=g)
        if arch == "bert":
            self.ids = toks[:, :S].contiguous()
            self.types = torch.zeros(1, S, dtype=torch.int64)
            self.types[:, S // 2:] = 1
            self.labels = torch.full((1, S), -100, dtype=torch.int64)
            self.labels[0, :mlm] = toks[0, 1:mlm + 1]
        else:
            self.ids, self.labels, self.types = toks[:, :-1].contiguous(), toks[:, 1:].contiguous(), None
        self.adam_s = None

    def step(self, M_total):
        """Seconds for one sample's F(+R)+B (+ its AdamW share)."""
        t0 = time.perf_counter()
        self.o.run_minibatch(self.ids, self.labels, self.S if self.arch != "bert" else self.mlm,
                             types=self.types)
        t = time.perf_counter() - t0
        if self.adam_s is None:
            t1 = time.perf_counter()
            self.o.adamw_step(1)
            self.adam_s = time.perf_counter() - t1
        for p in self.o.params.values():
            p.grad = None
        return (t + self.adam_s / M_total) * (self.L / self.cut)

    def describe(self):
        L, h = self.L, MODEL_DIMS[self.config][1]
        cut = "" if self.cut == L else (f"; {self.cut} of {L} layers run, time scaled x{L / self.cut:.2f} "
                                         "(extrapolated)")
        return (f"1 sample per step: fp32 torch-CPU port of the executor (oracle/gpt2_fp32.py) walking "
                f"the Varuna plan over {self.P} stage(s) — F, R on recomputing stages, B — at s={self.S}, "
                f"h={h}, plus 1/M_total of one AdamW update{cut}")


def run_reference(args):
    """--impl reference: the reference-side CPU arm. Rank 0 alone runs (other
    ranks exit at once). No product import: the plan comes from the committed
    profiles/plans.json, the control plane is spotpipe's own, the tensor path
    the fp32 CPU port."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    with open(os.path.join(ROOT, "profiles", "plans.json")) as f:
        plans = json.load(f)
    P, D = _ladder_pd(args, args.gpus)
    ent = load_plan(args.config, P, D)
    M, m, N = ent["M_total"], ent["m"], ent["N"]
    L, h, H, V, S, arch, _ = MODEL_DIMS[args.config]
    cp = reference_control_plane(plans)
    sample = CpuPipelineSample(args.config, ent["stage_map"])
    times = []
    for i in range(args.warmup + args.steps):
        t = sample.step(M)
        if i >= args.warmup:
            times.append(t)
    total = sum(times)
    value = len(times) / total
    line = {"metric": f"samples/sec ({METRIC_NAMES[args.config]} Varuna pipeline step)",
            "value": round(value, 5), "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / len(times), 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config} P{P}xD{D} m={m} N_m={N} M_total={M}",
                       "global_batch": M, "seq_len": S, "parallelism": f"pp{P}xdp{D}",
                       "plan": "profiles/plans.json (committed)"},
            "cpu_baseline": {"value": round(value, 5), "unit": "samples/s",
                             "cores": sample.threads, "kind": "port",
                             "sample": sample.describe()},
            "e2e": {"value": round(value, 5), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "control_plane_reference_cpu_us": cp}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm

def workload_shape(args, cfg, world):
    """(M_total, P, D, m, how m was chosen, stage_map) — from the committed
    plan (profiles/plans.json) so both arms time the same workload; an
    explicit --m recomputes N_m and the stage map."""
    M, m = MODEL_CONFIGS[args.config]
    P, D = _ladder_pd(args, world)
    if args.m == "auto":
        try:
            ent = load_plan(args.config, P, D)
            return ent["M_total"], P, D, ent["m"], ent["m_choice"] + " (profiles/plans.json)", \
                tuple(ent["stage_map"])
        except (SystemExit, OSError):
            m_sel = choose_micro_batch(cfg, P, D, M, args.config)
            if m_sel is not None:
                m = m_sel
            how = "planner (computed: no committed plan)"
    else:
        m, how = int(args.m), "command line"
    return M, P, D, m, how, tuple(stage_map_for(cfg, P, m, args.config))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2111_04007_b200 import ParallelConfig, micro_batches_for, JobSpec
    from paper_2111_04007_b200 import kernels as K
    from paper_2111_04007_b200.model import CONFIGS
    from paper_2111_04007_b200.runtime import Varuna, synthetic_batch
    from paper_2111_04007_b200.simulator import bubble_fraction

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    if args.dropout is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, dropout=args.dropout)
    M, P, D, m, m_how, stage_map = workload_shape(args, cfg, world)
    N = micro_batches_for(JobSpec(M), m, D)
    pc = ParallelConfig(P, D, m, N, stage_map)
    init_dev = "cuda"
    # P > 1: the reference's opportunistic policy (sp/engine decide) run over
    # the B200 calibration profile gives each stage its dispatch order; the
    # static Varuna order would idle the faster stage (it is generated for
    # uniform stage times).
    prof_path = os.path.join(ROOT, "profiles", f"b200_{args.config}.yaml")
    dispatch, prof = "static", None
    if P > 1 and args.dispatch == "live":
        dispatch = "live"
    elif P > 1 and os.path.exists(prof_path) and args.dispatch == "opportunistic":
        from paper_2111_04007_b200 import load_profile
        prof = load_profile(prof_path)
        if m in prof.m_grid and prof.num_cutpoints == cfg.n_layer:
            dispatch = "opportunistic"
        else:
            prof = None
    v = Varuna(cfg, pc, seed=0, init_device=init_dev, dispatch=dispatch, profile=prof)
    st = v.stream
    rows = m * N
    host = synthetic_batch(cfg, rows, v.replica)
    host = {k: t.pin_memory() for k, t in host.items()}
    dbatch = {k: t.to(dev) for k, t in host.items()}

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        v.step(dbatch)
    barrier()
    if P > 1 and dispatch == "opportunistic" and not args.no_retune:
        # one traced step: the dispatch order is re-derived by the reference's
        # opportunistic replica kernel from the MEASURED per-stage task times
        v.trace = True
        tl0 = v.step(dbatch).timeline
        v.trace = False
        v.retune_dispatch(tl0, perturb=args.retune_perturb)
        v.step(dbatch)
        barrier()

    # ---- timed region 1: inputs resident in HBM
    clocks = ClockSampler(local)
    l0 = K.LAUNCHES[0]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(st)
    for _ in range(args.steps):
        v.step(dbatch)
    e1.record(st)
    barrier()
    launches = K.LAUNCHES[0] - l0
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    clk = clocks.stop()
    value = M / (ms / 1e3)

    # ---- timed region 2: end to end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        h2d = sum(t.numel() * t.element_size() for k, t in host.items()
                  if (k == "input_ids" and v.spec.first) or (k == "labels" and v.spec.last))
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.steps):
            res = v.step(host)
            if v.spec.last:
                _ = res.loss  # D2H read of the step's loss (forces completion)
        t1.record(st)
        barrier()
        ms_e2e = max_over_ranks(t0.elapsed_time(t1)) / args.steps
        tot = torch.tensor([h2d, 4 if v.spec.last else 0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tot)
        e2e = {"value": round(M / (ms_e2e / 1e3), 3), "unit": "samples/s",
               "h2d_bytes_per_step": int(tot[0].item()), "d2h_bytes_per_step": int(tot[1].item())}

    # ---- instrumented steps (not timed): the task timeline of a normal
    # (graph-replayed) step, then GEMM launch durations of an eager step
    barrier()
    v.trace = True
    res = v.step(dbatch)
    torch.cuda.synchronize()
    v.trace = False
    barrier()
    K.GEMM_TIMING["on"] = True
    K.GEMM_TIMING["records"].clear()
    v.step(dbatch)
    torch.cuda.synchronize()
    K.GEMM_TIMING["on"] = False
    recs = K.GEMM_TIMING["records"]
    g_flops = sum(r[0] for r in recs)
    g_ms = sum(r[1].elapsed_time(r[2]) for r in recs)
    tl = res.timeline
    step_us = tl["step_us"]
    # measured bubble by the reference definition (sp/simulator.py:107-114):
    # 1 - (sum of task busy + sum of AR WORK) / (P*D*T_mb). AR work is the
    # C1 bucket spans on the comm stream (not the sync bracket, which also
    # holds C2/C3 waits on other stages); T_mb the latest task / AR end.
    # Every rank's clock starts at its step's first event, right after a
    # barrier with idle streams (one common origin to ~0.1 ms).
    ends = [b for _, _, _, b in tl["tasks"]] + [b for _, b in tl["ar_spans"]]
    busy_all = torch.tensor([tl["busy_us"], tl["ar_work_us"]], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(busy_all)
    mb_us = max_over_ranks(max(ends) if ends else 0.0)
    bubble = 1.0 - (busy_all[0].item() + busy_all[1].item()) / (world * mb_us) if mb_us else 0.0
    k9_us = measure_k9(v, P, dev)
    if args.trace_dir:
        os.makedirs(args.trace_dir, exist_ok=True)
        with open(os.path.join(args.trace_dir, f"gantt_{P}x{D}_{dispatch}_rank{rank}.csv"),
                  "w") as f:
            f.write(v.gantt_csv(v.gantt_rows(tl)))
    gemm_tf = g_flops / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    # per GEMM class of the step (per-GEMM TFLOP/s vs burst and
    # sustained): launches grouped by shape, operand layouts and epilogue
    epi_names = {K.EPI_STORE: "store", K.EPI_BIAS: "bias", K.EPI_BIAS_GELU: "bias_gelu",
                 K.EPI_BIAS_RESID: "bias_resid", K.EPI_DGELU: "dgelu",
                 K.EPI_ACC_F32: "acc_f32", K.EPI_STORE_F32: "store_f32", K.EPI_RESID: "resid"}
    groups = {}
    for fl, e0, e1, key in recs:
        gsum = groups.setdefault(key, [0, 0.0, 0])
        gsum[0] += fl
        gsum[1] += e0.elapsed_time(e1)
        gsum[2] += 1
    gemm_classes = []
    for (gm, gn, gk, ak, bk, ep), (fl, ms_, n) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        gemm_classes.append({"MxNxK": f"{gm}x{gn}x{gk}", "layout": ("n" if ak else "t") + ("t" if bk else "n"),
                             "epilogue": epi_names.get(ep, str(ep)), "launches": n,
                             "us_per_launch": round(1e3 * ms_ / n, 1),
                             "tflops": round(fl / (ms_ / 1e3) / 1e12, 1),
                             "share_of_gemm_time": round(ms_ / g_ms, 3) if g_ms else None})
    gemm_share = g_ms / (step_us / 1e3) if step_us else 0.0
    burst, sustained, hbm, src = peaks()

    # per-stage roofline: T_k = max(X_k / peak, act_bytes / NVLink)
    flops_layer_tok = cfg.flops_per_token_layer()
    worst = 0.0
    for s in range(P):
        nl = sum(1 for x in stage_map if x == s)
        F = nl * flops_layer_tok * m * cfg.seq_len
        if s == P - 1:
            F += cfg.head_flops_per_token() * m * cfg.seq_len
        X = (3 if (s == P - 1 or P == 1) else 4) * F
        t = max(X / (burst * 1e12), m * cfg.seq_len * cfg.hidden * 2 / 900e9)
        worst = max(worst, t)
    roof_samples = D * m / worst

    # measured stage profile -> reference bubble predictor (simulate_minibatch)
    # the dispatch used: the replayed opportunistic order is a FIXED order
    # (computed by the replica kernel from the calibration profile), so it is
    # predicted as that order run statically; live and static dispatch are
    # the reference policy itself on the Varuna schedule
    predicted = predicted_bubble(v, tl, P, D, N, m, world, dev, dist,
                                 opportunistic=dispatch == "live", k9_us=k9_us,
                                 replay=dispatch == "opportunistic")

    cpu = None
    control_plane = None
    if rank == 0:
        try:   # bounded: ~cpu_sample_s of host work after one warm-up sample
            cs = CpuPipelineSample(args.config, stage_map)
            cs.step(M)
            ts = []
            while sum(ts) < args.cpu_sample_s and len(ts) < 50:
                ts.append(cs.step(M))
            cpu = {"value": round(len(ts) / sum(ts), 5), "unit": "samples/s",
                   "cores": cs.threads, "kind": "port",
                   "sample": cs.describe() + f"; {len(ts)} samples timed"}
            del cs
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {ex}"}
        import paper_2111_04007_b200 as vpapi
        with open(os.path.join(ROOT, "profiles", "plans.json")) as f:
            control_plane = control_plane_times(vpapi, json.load(f))
    # ---- the same workload at the perf-run dropout (fused K7: masks in the
    # GEMM epilogues and attention, recompute-exact), device-resident inputs
    side = None
    if args.side_dropout and args.side_dropout != cfg.dropout:
        import dataclasses
        v.close()
        torch.cuda.empty_cache()
        cfg_d = dataclasses.replace(cfg, dropout=args.side_dropout)
        vd = Varuna(cfg_d, pc, seed=0, init_device=init_dev, dispatch=dispatch, profile=prof)
        for _ in range(args.warmup):
            vd.step(dbatch)
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(vd.stream)
        for _ in range(args.steps):
            vd.step(dbatch)
        a1.record(vd.stream)
        barrier()
        ms_d = max_over_ranks(a0.elapsed_time(a1)) / args.steps
        side = {"dropout": args.side_dropout, "value": round(M / (ms_d / 1e3), 3),
                "unit": "samples/s", "ms_per_step": round(ms_d, 2),
                "note": "hidden (GEMM-epilogue) + attention-probability + embedding dropout, "
                        "masks regenerated bit-exactly by recompute; CUDA graphs on"}
        v = vd
    if rank == 0:
        line = {
            "metric": f"samples/sec ({METRIC_NAMES[args.config]} Varuna pipeline step)",
            "value": round(value, 3), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic tokens, random-init weights",
            "config": {"workload": f"{args.config} P{P}xD{D} m={m} N_m={N} M_total={M}",
                       "model": cfg_name(cfg), "global_batch": M, "seq_len": cfg.seq_len,
                       "parallelism": f"pp{P}xdp{D}", "stage_map_sizes":
                           [sum(1 for x in stage_map if x == s) for s in range(P)],
                       "l2": "working set >> 126 MB L2 (no flush needed)", "dropout": cfg.dropout,
                       "dispatch": dispatch, "micro_batch": m, "micro_batch_choice": m_how},
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "achieved": round(gemm_tf, 1),
                         "peak": sustained, "unit": "TFLOP/s",
                         "frac": round(gemm_tf / sustained, 4),
                         "traffic": gemm_traffic(),
                         "kernel": "vp_gemm_bf16 (tcgen05), all GEMM launches of one step",
                         "peak_kind": f"{src} bf16 sustained", "share_of_step": round(gemm_share, 3),
                         "burst_peak": burst, "by_class": gemm_classes[:12]},
            "stage_roofline": {"roofline_samples_per_s": round(roof_samples, 1),
                               "frac": round(value / roof_samples, 4)},
            "bubble": {"measured": round(bubble, 4), "predicted": predicted["bubble"],
                       "rel_err": (round(abs(bubble - predicted["bubble"]) / predicted["bubble"], 4)
                                   if predicted["bubble"] else None),
                       "measured_minibatch_us": round(mb_us, 1),
                       "predicted_minibatch_us": predicted["minibatch_us"],
                       "basis": "reference formula (sp/simulator.py:107-114); predicted = "
                                "simulate_minibatch twin on the Varuna schedule with the "
                                f"dispatch used ({dispatch}), over an in-step profile: measured "
                                "per-stage F/B/R, K9 put time, C1 bucket work",
                       "k9_put_us": k9_us},
            "cpu_baseline": cpu,
            "control_plane_cpp_us": control_plane,
            "with_dropout": side,
        }
        print(json.dumps(line), flush=True)
    v.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_k9(v, P, dev):
    """K9 transfer time: the gradient put of one m*s*h*2-byte slot into the
    upstream stage's ring (median of 5 after one warm-up, CUDA events on
    the executor stream; all stages idle). Max over ranks; 0 at P = 1."""
    import torch
    import torch.distributed as dist
    from paper_2111_04007_b200 import kernels as K
    t = 0.0
    if P > 1 and v.active and not v.spec.first:
        src = v.stage.g
        dst = v.links.peer_slot_ptr(1, 1)
        st = v.stream
        times = []
        for i in range(6):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            K.p2p_put(dst, src, stream=st)
            b.record(st)
            b.synchronize()
            if i:
                times.append(a.elapsed_time(b) * 1e3)
        t = statistics.median(times)
    if dist.is_initialized() and dist.get_world_size() > 1:
        x = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        t = float(x.item())
    return round(t, 2)


def predicted_bubble(v, tl, P, D, N, m, world, dev, dist, opportunistic=False, k9_us=0.0,
                     replay=False):
    """The reference's prediction for this run (simulate_minibatch,
    sp/simulator.py:259-389, on the C++ replica kernel): the Varuna schedule
    generate_varuna_schedule(P, N, 1, 2, 1) under the dispatch policy used
    (opportunistic for the replayed and the live dispatch), over an IN-STEP
    calibration profile — one cut-point per stage carrying that stage's
    measured mean F and B (replica 0), R as a measured R/F ratio, the
    measured K9 put time as the intra-node act/grad transfer, and the stage's
    measured C1 bucket work as its AR time. ``replay``: the schedule is the
    per-stage order actually executed (replica 0), simulated statically."""
    import torch
    from paper_2111_04007_b200 import (ModelSpec, ParallelConfig, build_placement,
                                       generate_varuna_schedule, simulate_minibatch,
                                       uniform_cluster)
    from paper_2111_04007_b200.calibration import CalibrationProfile, CutpointTimes
    from paper_2111_04007_b200.core import KIND_BACKWARD, KIND_FORWARD, KIND_RECOMPUTE
    sums = torch.zeros(world, 4, device=dev, dtype=torch.float64)
    cnt = {0: [], 1: [], 2: []}
    for kind, j, a, b in tl["tasks"]:
        cnt[kind].append(b - a)
    for kind, col in ((KIND_FORWARD, 0), (KIND_BACKWARD, 1), (KIND_RECOMPUTE, 2)):
        if cnt[kind]:
            sums[v.rank, col] = statistics.mean(cnt[kind])
    sums[v.rank, 3] = tl["ar_work_us"]
    if world > 1:
        dist.all_reduce(sums)
    stage_f = [float(sums[s, 0].item()) for s in range(P)]
    stage_b = [float(sums[s, 1].item()) for s in range(P)]
    stage_ar = [float(sums[[r * P + s for r in range(D)], 3].mean().item()) for s in range(P)]
    rec = [float(sums[s, 2].item()) / stage_f[s] for s in range(P) if sums[s, 2] > 0 and stage_f[s]]
    rscale = statistics.mean(rec) if rec else 1.0
    tx = {m: int(round(k9_us))}
    d_grid = tuple(sorted({1, D}))
    cps = tuple(CutpointTimes({m: max(1, round(stage_f[s]))}, {m: max(1, round(stage_b[s]))},
                              tx, tx, tx, {m: 0}, tx, {m: 0},
                              {d: (int(round(stage_ar[s])) if d == D and D > 1 else 0)
                               for d in d_grid}) for s in range(P))
    prof = CalibrationProfile((m,), d_grid, cps)
    model = ModelSpec("stages", (1,) * P, (1,) * P)
    pc = ParallelConfig(P, D, m, N, tuple(range(P)))
    sched = generate_varuna_schedule(P, N, 1.0, 2.0, 1.0)
    if replay:
        import numpy as np
        from paper_2111_04007_b200.scheduler import Schedule
        orders = [None] * world
        if world > 1:
            dist.all_gather_object(orders, v.executed)
        else:
            orders = [v.executed]
        kinds, mbs, offs = [], [], [0]
        for s in range(P):          # replica 0's ranks are 0..P-1
            kinds += [k for k, _ in orders[s]]
            mbs += [j for _, j in orders[s]]
            offs.append(len(kinds))
        sched = Schedule("executed", P, N, np.array(kinds, np.int64), np.array(mbs, np.int64),
                         np.array(offs, np.int64), 1, 2, 1)
    r = simulate_minibatch(sched, pc, prof,
                           build_placement(uniform_cluster(P * D, 8), P, D), model,
                           opportunistic=opportunistic, recompute_scale=rscale)
    return {"bubble": round(r.bubble_fraction, 4), "minibatch_us": int(r.minibatch_us)}


if __name__ == "__main__":
    sys.exit(main())
