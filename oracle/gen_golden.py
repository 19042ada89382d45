"""Generate the committed golden fixtures under tests/golden/ by running the
REFERENCE implementation (spotpipe 0.1.0, /root/reference/pkg/src) in this
container.

TEST INFRASTRUCTURE ONLY. This script is the provenance of every fixture the
parity tests check against; nothing in the product imports it, and it is
never run on the GPU box (the reference tree does not exist there).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

Reference entry points exercised (all paths relative to /root/reference):
  generate_varuna_schedule / generate_gpipe_schedule  pkg/src/spotpipe/scheduler.py:128-176
  Schedule.in_flight_bound                            pkg/src/spotpipe/scheduler.py:88-97
  makespan_us / schedule_to_csv                       pkg/src/spotpipe/scheduler.py:370-373, 467-473
  engine.py_kernel.run_replica                        pkg/src/spotpipe/engine/py_kernel.py:41-360
  assign_stages / identify_cutpoints / memory_check   pkg/src/spotpipe/partitioner.py:124-436
  build_placement / simulate_minibatch                pkg/src/spotpipe/simulator.py:58-389
  micro_batches_for / select_microbatch / plan        pkg/src/spotpipe/planner.py:72-208
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from spotpipe import engine  # noqa: E402
from spotpipe.calibration import synthesize_profile, uniform_profile  # noqa: E402
from spotpipe.core import (  # noqa: E402
    HardwareSpec,
    JobSpec,
    ModelSpec,
    ParallelConfig,
    make_block_model,
    uniform_cluster,
    uniform_stage_map,
)
from spotpipe.engine import py_kernel  # noqa: E402
from spotpipe.partitioner import (  # noqa: E402
    Operation,
    OpProfile,
    assign_stages,
    identify_cutpoints,
    load_op_profile,
    memory_check,
)
from spotpipe.planner import micro_batches_for, plan, select_microbatch  # noqa: E402
from spotpipe.scheduler import (  # noqa: E402
    generate_gpipe_schedule,
    generate_varuna_schedule,
    makespan_us,
    schedule_to_csv,
)
from spotpipe.simulator import build_placement, simulate_minibatch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
UNIT = (1.0, 2.0, 1.0)

# BASELINE.json configs: name, blocks, hidden, seq, P, D, m, M_total
CONFIGS = [
    ("tiny", 4, 256, 128, 2, 1, 4, 16),
    ("gpt2_355m", 24, 1024, 1024, 4, 2, 8, 512),
    ("bert_large", 24, 1024, 512, 2, 4, 32, 8192),
    ("gpt2_2_5b", 54, 1920, 1024, 8, 1, 4, 256),
    ("gpt2_8_3b", 72, 3072, 1024, 4, 2, 4, 512),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def sched_record(s):
    p = s.pipeline_depth
    return {
        "kinds": s.kinds.tolist(),
        "mbs": s.mbs.tolist(),
        "offsets": s.offsets.tolist(),
        "in_flight_bound": [s.in_flight_bound(k + 1) for k in range(p)],
        "makespan_us": makespan_us(s),
    }


def gen_schedules():
    small = {}
    for p in range(1, 9):
        for n in range(1, 17):
            small[f"varuna,{p},{n}"] = sched_record(generate_varuna_schedule(p, n, *UNIT))
            small[f"gpipe,{p},{n}"] = sched_record(generate_gpipe_schedule(p, n, *UNIT))
    # Non-canonical time ratios change the plan; pin a few.
    ratios = {}
    for (tf, tb, tr) in ((1.0, 3.0, 1.0), (1.3, 2.0, 1.0), (1.0, 2.2, 1.0), (0.5, 1.0, 0.5)):
        for (p, n) in ((4, 32), (8, 64), (4, 64), (3, 7)):
            s = generate_varuna_schedule(p, n, tf, tb, tr)
            ratios[f"{tf},{tb},{tr},{p},{n}"] = {
                "csv_sha256": hashlib.sha256(schedule_to_csv(s).encode()).hexdigest(),
                "n_tasks": int(s.offsets[-1]),
            }
    big = {}
    for (p, n) in ((2, 4), (4, 32), (2, 64), (8, 64), (4, 64), (2, 128), (8, 16),
                   (4, 1024), (8, 512), (1, 64), (2, 32), (4, 16), (8, 32), (4, 8)):
        s = generate_varuna_schedule(p, n, *UNIT)
        g = generate_gpipe_schedule(p, n, *UNIT)
        big[f"{p},{n}"] = {
            "csv_sha256": hashlib.sha256(schedule_to_csv(s).encode()).hexdigest(),
            "kinds_sha256": sha(s.kinds),
            "mbs_sha256": sha(s.mbs),
            "n_tasks": int(s.offsets[-1]),
            "in_flight_bound": [s.in_flight_bound(k + 1) for k in range(p)],
            "makespan_us": makespan_us(s),
            "gpipe_makespan_us": makespan_us(g),
        }
    golden_csv_2_2 = schedule_to_csv(generate_varuna_schedule(2, 2, *UNIT))
    return {"small": small, "ratios": ratios, "configs": big, "csv_2_2": golden_csv_2_2}


def gen_engine_cases():
    cases = []
    for opp in (False, True):
        for ser in (False, True):
            rng = np.random.default_rng(20_240 + int(opp) * 2 + int(ser))
            for trial in range(60):
                P = int(rng.integers(1, 9))
                N = int(rng.integers(1, 13))
                policy = "varuna" if trial % 2 else "gpipe"
                gen = generate_varuna_schedule if trial % 2 else generate_gpipe_schedule
                s = gen(P, N, *UNIT)
                fwd = np.full(P, 1_000_000, dtype=np.int64)
                bwd = np.full(P, 2_000_000, dtype=np.int64)
                rec = np.full(P, 1_000_000, dtype=np.int64)
                act = rng.integers(0, 500_000, size=max(P - 1, 0) * N).astype(np.int64)
                grad = rng.integers(0, 500_000, size=max(P - 1, 0) * N).astype(np.int64)
                expg = rng.integers(0, 500_000, size=max(P - 1, 1)).astype(np.int64)
                in_act = np.full(P, 128, dtype=np.int64)
                work = np.full(P, 1024, dtype=np.int64)
                cap = np.array([s.in_flight_bound(k + 1) + 4 for k in range(P)], dtype=np.int64)
                out = py_kernel.run_replica(P, N, s.kinds, s.mbs, s.offsets, fwd, bwd, rec,
                                            act, grad, expg, in_act, work, cap, opp, ser)
                cases.append(_engine_case(P, N, policy, s, fwd, bwd, rec, act, grad, expg,
                                          in_act, work, cap, opp, ser, out))
    # Heterogeneous stage times (the illustrative B200-like profile shape,
    # SURVEY A.5): per-stage F/B/R differ, zero and 200 us latency.
    rng = np.random.default_rng(77)
    for trial in range(40):
        P = int(rng.integers(2, 9))
        N = int(rng.integers(P, 3 * P + 8))
        s = generate_varuna_schedule(P, N, *UNIT)
        fwd = rng.integers(500, 3000, size=P).astype(np.int64)
        bwd = (2 * fwd + rng.integers(0, 300, size=P)).astype(np.int64)
        rec = fwd.copy()
        lat = int(rng.choice([0, 10, 200]))
        act = (lat + rng.integers(0, 50, size=(P - 1) * N)).astype(np.int64)
        grad = (lat + rng.integers(0, 50, size=(P - 1) * N)).astype(np.int64)
        expg = np.full(P - 1, lat + 25, dtype=np.int64)
        in_act = rng.integers(1, 1 << 20, size=P).astype(np.int64)
        work = rng.integers(1, 1 << 22, size=P).astype(np.int64)
        cap = np.array([s.in_flight_bound(k + 1) + 4 for k in range(P)], dtype=np.int64)
        for opp in (False, True):
            out = py_kernel.run_replica(P, N, s.kinds, s.mbs, s.offsets, fwd, bwd, rec,
                                        act, grad, expg, in_act, work, cap, opp, True)
            cases.append(_engine_case(P, N, "varuna", s, fwd, bwd, rec, act, grad, expg,
                                      in_act, work, cap, opp, True, out))
    return cases


def _engine_case(P, N, policy, s, fwd, bwd, rec, act, grad, expg, in_act, work, cap,
                 opp, ser, out):
    return {
        "P": P, "N": N, "policy": policy,
        "opportunistic": bool(opp), "serialize_links": bool(ser),
        "fwd_us": fwd.tolist(), "bwd_us": bwd.tolist(), "rec_us": rec.tolist(),
        "act_tx_us": act.tolist(), "grad_tx_us": grad.tolist(),
        "exp_grad_tx_us": expg.tolist(), "in_act_bytes": in_act.tolist(),
        "work_bytes": work.tolist(), "stash_cap": cap.tolist(),
        "makespan": int(out["makespan"]),
        "sha256": {k: sha(v) for k, v in out.items() if k != "makespan"},
        "task_start_head": out["task_start"][:16].tolist(),
        "peak_stash": out["peak_stash"].tolist(),
    }


def profile_from_forward_us(times):
    # Same construction as the reference tests' helper (pkg/tests/test_partitioner.py).
    from spotpipe.calibration import CalibrationProfile, CutpointTimes
    cps = []
    for t in times:
        cps.append(CutpointTimes(
            forward_us={1: t}, backward_us={1: 2 * t},
            act_intra_us={1: 0}, grad_intra_us={1: 0},
            act_inter_mean_us={1: 0}, act_inter_jitter_us={1: 0},
            grad_inter_mean_us={1: 0}, grad_inter_jitter_us={1: 0},
            allreduce_us={1: 0},
        ))
    return CalibrationProfile(m_grid=(1,), d_grid=(1,), cutpoints=tuple(cps))


def assignment_record(a):
    return {
        "stage_map": list(a.stage_map),
        "boundaries": list(a.boundaries),
        "stage_parameters": list(a.stage_parameters),
        "stage_forward_us": list(a.stage_forward_us),
        "stage_input_activation_bytes": list(a.stage_input_activation_bytes),
        "stage_working_activation_bytes": list(a.stage_working_activation_bytes),
        "stage_boundary_activation_bytes": list(a.stage_boundary_activation_bytes),
    }


B200_HW = HardwareSpec(
    gpu_memory_bytes=180_000_000_000, gpus_per_node=8,
    intra_node_bandwidth=900e9, inter_node_bandwidth=50e9,
    inter_node_latency_us=5, inter_node_jitter_us=0, intra_node_latency_us=2,
)

COMMODITY_HW = HardwareSpec(
    gpu_memory_bytes=16_000_000_000, gpus_per_node=1,
    intra_node_bandwidth=12_500_000_000, inter_node_bandwidth=325_000_000,
    inter_node_latency_us=2_000, inter_node_jitter_us=2_000, intra_node_latency_us=5,
)


def gen_partition():
    out = {"configs": {}, "random": [], "weighted": [], "cutpoints": [], "memory": []}
    for name, L, h, s, P, D, m, M in CONFIGS:
        model = make_block_model(name, L, h, s)
        uni = uniform_profile(L, 1.0, 2.0, m_grid=(m,), d_grid=(1, D) if D > 1 else (1,))
        a = assign_stages(model, P, m, uni)
        syn = synthesize_profile(model, B200_HW, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
        a2 = assign_stages(model, P, m, syn)
        rec = {"uniform": assignment_record(a), "synth_b200": assignment_record(a2),
               "uniform_stage_map": list(uniform_stage_map(L, P))}
        out["configs"][name] = rec
    rng = random.Random(7)
    for trial in range(300):
        k = rng.randint(2, 16)
        p = rng.randint(1, min(6, k))
        times = [rng.randint(1, 100) for _ in range(k)]
        acts = [rng.randint(1, 50) for _ in range(k)]
        params = [rng.randint(1, 1000) for _ in range(k)]
        model = ModelSpec("m", tuple(params), tuple(acts))
        a = assign_stages(model, p, 1, profile_from_forward_us(times))
        out["random"].append({"times": times, "acts": acts, "params": params, "P": p,
                              "result": assignment_record(a)})
    for trial in range(60):
        k = rng.randint(3, 12)
        p = rng.randint(2, min(4, k))
        times = [rng.randint(1, 60) for _ in range(k)]
        acts = [rng.randint(1, 50) for _ in range(k)]
        w = rng.choice([0.5, 0.75, 1.25, 0.9])
        model = ModelSpec("m", tuple([1] * k), tuple(acts))
        a = assign_stages(model, p, 1, profile_from_forward_us(times), last_stage_weight=w)
        out["weighted"].append({"times": times, "acts": acts, "P": p, "weight": w,
                                "result": assignment_record(a)})
    # identify_cutpoints on the shipped op profile and random profiles.
    prof = load_op_profile("/root/reference/pkg/configs/sample_ops.yaml")
    ops = [{"name": o.name, "compute_us": o.compute_us, "activation_bytes": o.output_activation_bytes,
            "parameters": o.owned_parameters, "param_groups": sorted(o.param_groups)} for o in prof.ops]
    for k in range(1, 11):
        for tol in (0.0, 0.2, 0.5):
            try:
                r = identify_cutpoints(prof, k, tolerance=tol)
                res = {"boundaries": list(r.boundaries),
                       "shared_crossings": [list(x) for x in r.shared_crossings],
                       "section_compute_us": list(r.section_compute_us),
                       "max_section_us": r.max_section_us,
                       "total_boundary_activation": r.total_boundary_activation,
                       "cutpoint_parameters": list(r.model.cutpoint_parameters),
                       "cutpoint_activation_bytes": list(r.model.cutpoint_activation_bytes)}
            except Exception as e:  # noqa: BLE001
                res = {"error": type(e).__name__}
            out["cutpoints"].append({"ops": ops, "shared_groups": sorted(prof.shared_groups),
                                     "K": k, "tolerance": tol, "result": res})
    for trial in range(120):
        n = rng.randint(2, 12)
        groups = ["g0", "g1", "g2"]
        opl = []
        for i in range(n):
            pg = sorted({g for g in groups if rng.random() < 0.15})
            opl.append({"name": f"op{i}", "compute_us": rng.randint(0, 50),
                        "activation_bytes": rng.randint(0, 40),
                        "parameters": rng.randint(0, 30), "param_groups": pg})
        shared = sorted({g for g in groups if rng.random() < 0.5})
        k = rng.randint(1, n)
        tol = rng.choice([0.0, 0.1, 0.2, 0.35])
        prof_r = OpProfile(ops=tuple(Operation(o["name"], o["compute_us"], o["activation_bytes"],
                                               o["parameters"], frozenset(o["param_groups"]))
                                     for o in opl), shared_groups=frozenset(shared))
        try:
            r = identify_cutpoints(prof_r, k, tolerance=tol)
            res = {"boundaries": list(r.boundaries),
                   "shared_crossings": [list(x) for x in r.shared_crossings],
                   "section_compute_us": list(r.section_compute_us),
                   "max_section_us": r.max_section_us,
                   "total_boundary_activation": r.total_boundary_activation,
                   "cutpoint_parameters": list(r.model.cutpoint_parameters),
                   "cutpoint_activation_bytes": list(r.model.cutpoint_activation_bytes)}
        except Exception as e:  # noqa: BLE001
            res = {"error": type(e).__name__}
        out["cutpoints"].append({"ops": opl, "shared_groups": shared, "K": k,
                                 "tolerance": tol, "result": res})
    # memory_check on the configs with schedule bounds.
    for name, L, h, s, P, D, m, M in CONFIGS:
        model = make_block_model(name, L, h, s)
        uni = uniform_profile(L, 1.0, 2.0, m_grid=(m,))
        a = assign_stages(model, P, m, uni)
        n_m = micro_batches_for(JobSpec(M), m, D)
        sch = generate_varuna_schedule(P, n_m, *UNIT)
        rep = memory_check(a, m, n_m, B200_HW,
                           in_flight_bound=[sch.in_flight_bound(k + 1) + 4 for k in range(P)])
        out["memory"].append({"config": name, "N_m": n_m, "stages": [
            {"parameter_state_bytes": st.parameter_state_bytes,
             "stashed_activation_bytes": st.stashed_activation_bytes,
             "working_activation_bytes": st.working_activation_bytes,
             "feasible": st.feasible} for st in rep.stages]})
    return out


def gen_simulator():
    out = {"configs": {}, "uniform_small": [], "jitter": [], "placement": {}, "planner": {}}
    for name, L, h, s, P, D, m, M in CONFIGS:
        model = make_block_model(name, L, h, s)
        d_grid = tuple(sorted({1, D}))
        uni = uniform_profile(L, 1.0, 2.0, m_grid=(m,), d_grid=d_grid)
        a = assign_stages(model, P, m, uni)
        n_m = micro_batches_for(JobSpec(M), m, D)
        cfg = ParallelConfig(P, D, m, n_m, a.stage_map)
        sch = generate_varuna_schedule(P, n_m, *UNIT)
        gp = generate_gpipe_schedule(P, n_m, *UNIT)
        pl = build_placement(uniform_cluster(P * D, gpus_per_vm=8), P, D)
        rec = {"N_m": n_m, "stage_map": list(a.stage_map)}
        for tag, sc in (("varuna", sch), ("gpipe", gp)):
            for opp in (False, True):
                r = simulate_minibatch(sc, cfg, uni, pl, model, opportunistic=opp)
                rec[f"{tag},{int(opp)}"] = {"minibatch_us": r.minibatch_us,
                                            "makespan_us": r.makespan_us,
                                            "bubble_fraction": r.bubble_fraction,
                                            "stage_idle_us": [list(x) for x in r.stage_idle_us],
                                            "peak_memory_bytes": list(r.peak_memory_bytes)}
        out["configs"][name] = rec
    for p in range(1, 7):
        for n in (1, 2, 5, 8, 13):
            for d in (1, 2):
                model = ModelSpec("u", tuple([1] * p), tuple([8] * p))
                prof = uniform_profile(p, 1.0, 2.0, d_grid=tuple(range(1, d + 1)))
                cfg = ParallelConfig(p, d, 1, n, uniform_stage_map(p, p))
                pl = build_placement(uniform_cluster(p * d), p, d)
                s = generate_varuna_schedule(p, n, *UNIT)
                r = simulate_minibatch(s, cfg, prof, pl, model)
                out["uniform_small"].append({"P": p, "N": n, "D": d,
                                             "minibatch_us": r.minibatch_us,
                                             "bubble_fraction": r.bubble_fraction})
    # Jittered commodity profile: exercises the splitmix64/Box-Muller transfer
    # sampler and inter-node link classes (pkg/src/spotpipe/simulator.py:173-208).
    model = make_block_model("gpt-2.5b-like", 54, 1920, 1024)
    prof = synthesize_profile(model, COMMODITY_HW, [1, 2, 4], [1, 2, 3],
                              allreduce_bandwidth=1_250_000_000)
    for (P, D, m, n, seed, gpv) in ((6, 2, 2, 12, 4, 1), (9, 3, 2, 8, 1, 1), (3, 2, 4, 6, 7, 2),
                                    (6, 1, 1, 9, 11, 4), (2, 3, 2, 5, 0, 1)):
        cfg = ParallelConfig(P, D, m, n, uniform_stage_map(54, P))
        pl = build_placement(uniform_cluster(P * D, gpus_per_vm=gpv), P, D)
        s = generate_varuna_schedule(P, n, *UNIT)
        for opp in (False, True):
            r = simulate_minibatch(s, cfg, prof, pl, model, seed=seed, opportunistic=opp)
            out["jitter"].append({"P": P, "D": D, "m": m, "N": n, "seed": seed,
                                  "gpus_per_vm": gpv, "opportunistic": opp,
                                  "minibatch_us": r.minibatch_us, "makespan_us": r.makespan_us,
                                  "bubble_fraction": r.bubble_fraction,
                                  "allreduce_us": list(r.allreduce_us),
                                  "allreduce_start_us": list(r.allreduce_start_us),
                                  "task_start_sha256": [sha(x["task_start"]) for x in r.replicas],
                                  "msg_arrive_sha256": [sha(x["msg_arrive"]) for x in r.replicas]})
    for (P, D) in ((1, 1), (2, 1), (4, 1), (2, 2), (4, 2), (8, 1), (2, 4), (1, 8)):
        pl = build_placement(uniform_cluster(8, gpus_per_vm=8), P, D)
        out["placement"][f"{P},{D}"] = {f"{s},{r}": list(v) for (s, r), v in pl.assignments.items()}
    # Planner: micro_batches_for and select_microbatch, plus one plan() per config.
    mb = {}
    for M in (16, 256, 512, 8192, 100, 7):
        for m in (1, 2, 4, 8, 32):
            for d in (1, 2, 3, 4, 8):
                mb[f"{M},{m},{d}"] = micro_batches_for(JobSpec(M), m, d)
    out["planner"]["micro_batches_for"] = mb
    sel = {}
    for name, L, h, s, P, D, m, M in CONFIGS:
        model = make_block_model(name, L, h, s)
        for thr in (0.02, 0.05, 0.0):
            syn = synthesize_profile(model, B200_HW, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
            sel[f"{name},{thr}"] = select_microbatch(syn, thr)
    out["planner"]["select_microbatch"] = sel
    plans = {}
    for name, L, h, s, P, D, m, M in CONFIGS:
        model = make_block_model(name, L, h, s)
        syn = synthesize_profile(model, B200_HW, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
        for G in (1, 2, 4, 8):
            r = plan(G, model, JobSpec(M), syn, B200_HW, uniform_cluster(G, gpus_per_vm=8),
                     micro_batch_size=m)
            plans[f"{name},{G}"] = {"P": r.chosen.pipeline_depth, "D": r.chosen.data_parallel,
                                    "m": r.chosen.micro_batch_size,
                                    "N_m": r.chosen.num_micro_batches,
                                    "stage_map": list(r.chosen.stage_map),
                                    "minibatch_us": r.minibatch_us,
                                    "candidates": [[c.config.pipeline_depth, c.config.data_parallel,
                                                    c.minibatch_us] for c in r.candidates]}
    out["planner"]["plan"] = plans
    return out


def main():
    assert engine.ENGINE_NAME in ("python", "compiled")
    os.makedirs(OUT, exist_ok=True)
    for name, fn in (("schedules", gen_schedules), ("engine_cases", gen_engine_cases),
                     ("partition", gen_partition), ("simulator", gen_simulator)):
        data = fn()
        path = os.path.join(OUT, f"{name}.json")
        with open(path, "w") as f:
            json.dump({"generator": "oracle/gen_golden.py", "reference": "spotpipe 0.1.0",
                       "data": data}, f, separators=(",", ":"))
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
