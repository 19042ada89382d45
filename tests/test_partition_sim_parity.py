"""Partitioner, placement, simulator (bubble predictor) and planner parity
against the reference's outputs (tests/golden/partition.json,
simulator.json, produced by spotpipe 0.1.0)."""

import hashlib

import numpy as np
import pytest

import paper_2111_04007_b200 as vp
from paper_2111_04007_b200.calibration import CalibrationProfile, CutpointTimes
from oracle import partition as opart

CONFIGS = {  # name: (L, h, s, P, D, m, M)
    "tiny": (4, 256, 128, 2, 1, 4, 16),
    "gpt2_355m": (24, 1024, 1024, 4, 2, 8, 512),
    "bert_large": (24, 1024, 512, 2, 4, 32, 8192),
    "gpt2_2_5b": (54, 1920, 1024, 8, 1, 4, 256),
    "gpt2_8_3b": (72, 3072, 1024, 4, 2, 4, 512),
}
FIELDS = ["stage_map", "boundaries", "stage_parameters", "stage_forward_us",
          "stage_input_activation_bytes", "stage_working_activation_bytes",
          "stage_boundary_activation_bytes"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def prof_from_f(times):
    cps = tuple(CutpointTimes({1: t}, {1: 2 * t}, {1: 0}, {1: 0}, {1: 0}, {1: 0}, {1: 0}, {1: 0},
                              {1: 0}) for t in times)
    return CalibrationProfile((1,), (1,), cps)


def test_assign_stages_configs(golden):
    for name, rec in golden("partition")["configs"].items():
        L, h, s, P, D, m, M = CONFIGS[name]
        model = vp.make_block_model(name, L, h, s)
        a = vp.assign_stages(model, P, m, vp.uniform_profile(L, 1.0, 2.0, m_grid=(m,)))
        for f in FIELDS:
            assert list(getattr(a, f)) == rec["uniform"][f], (name, f)
        syn = vp.synthesize_profile(model, vp.B200_NVL8, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
        a2 = vp.assign_stages(model, P, m, syn)
        for f in FIELDS:
            assert list(getattr(a2, f)) == rec["synth_b200"][f], (name, f)
        assert list(vp.uniform_stage_map(L, P)) == rec["uniform_stage_map"]
    # The 2.5B case is the one where the DP differs from uniform_stage_map.
    sm = golden("partition")["configs"]["gpt2_2_5b"]["uniform"]["stage_map"]
    assert [sm.count(k) for k in range(8)] == [5, 7, 7, 7, 7, 7, 7, 7]


def test_assign_stages_random(golden):
    for rec in golden("partition")["random"]:
        model = vp.ModelSpec("m", tuple(rec["params"]), tuple(rec["acts"]))
        a = vp.assign_stages(model, rec["P"], 1, prof_from_f(rec["times"]))
        for f in FIELDS:
            assert list(getattr(a, f)) == rec["result"][f], (rec, f)
    for rec in golden("partition")["weighted"]:
        model = vp.ModelSpec("m", (1,) * len(rec["times"]), tuple(rec["acts"]))
        a = vp.assign_stages(model, rec["P"], 1, prof_from_f(rec["times"]),
                             last_stage_weight=rec["weight"])
        assert list(a.boundaries) == rec["result"]["boundaries"]


def test_assign_stages_vs_oracle_fresh():
    rng = np.random.default_rng(5)
    for _ in range(200):
        k = int(rng.integers(1, 30))
        p = int(rng.integers(1, k + 1))
        t = rng.integers(1, 1000, size=k).tolist()
        acts = rng.integers(1, 100, size=k).tolist()
        a = vp.assign_stages(vp.ModelSpec("m", (1,) * k, tuple(acts)), p, 1, prof_from_f(t))
        o = opart.assign_stages(t, acts, [1] * k, None, p)
        assert list(a.boundaries) == o["boundaries"]


def test_assign_stages_errors():
    model = vp.make_block_model("m", 3, 32, 8)
    with pytest.raises(vp.InfeasibleError):
        vp.assign_stages(model, 4, 1, vp.uniform_profile(3, 0.01, 0.02))
    with pytest.raises(vp.ConfigError):
        vp.assign_stages(model, 2, 1, vp.uniform_profile(4, 0.01, 0.02))


def test_identify_cutpoints(golden):
    for rec in golden("partition")["cutpoints"]:
        prof = vp.OpProfile(tuple(vp.Operation(o["name"], o["compute_us"], o["activation_bytes"],
                                               o["parameters"], frozenset(o["param_groups"]))
                                  for o in rec["ops"]), frozenset(rec["shared_groups"]))
        res = rec["result"]
        if "error" in res:
            with pytest.raises((vp.InfeasibleError, vp.ConfigError)):
                vp.identify_cutpoints(prof, rec["K"], rec["tolerance"])
            continue
        r = vp.identify_cutpoints(prof, rec["K"], rec["tolerance"])
        assert list(r.boundaries) == res["boundaries"]
        assert [list(x) for x in r.shared_crossings] == res["shared_crossings"]
        assert list(r.section_compute_us) == res["section_compute_us"]
        assert r.max_section_us == res["max_section_us"]
        assert r.total_boundary_activation == res["total_boundary_activation"]
        assert list(r.model.cutpoint_parameters) == res["cutpoint_parameters"]


def test_memory_check(golden):
    for rec in golden("partition")["memory"]:
        L, h, s, P, D, m, M = CONFIGS[rec["config"]]
        model = vp.make_block_model(rec["config"], L, h, s)
        a = vp.assign_stages(model, P, m, vp.uniform_profile(L, 1.0, 2.0, m_grid=(m,)))
        n_m = vp.micro_batches_for(vp.JobSpec(M), m, D)
        assert n_m == rec["N_m"]
        sch = vp.generate_varuna_schedule(P, n_m, 1.0, 2.0, 1.0)
        hw = vp.HardwareSpec(180_000_000_000, 8, 900e9, 50e9, 5, 0, 2)
        r = vp.memory_check(a, m, n_m, hw, [sch.in_flight_bound(k + 1) + 4 for k in range(P)])
        for st, want in zip(r.stages, rec["stages"]):
            assert st.parameter_state_bytes == want["parameter_state_bytes"]
            assert st.stashed_activation_bytes == want["stashed_activation_bytes"]
            assert st.working_activation_bytes == want["working_activation_bytes"]
            assert st.feasible == want["feasible"]


def test_placement(golden):
    for key, rec in golden("simulator")["placement"].items():
        P, D = map(int, key.split(","))
        pl = vp.build_placement(vp.uniform_cluster(8, gpus_per_vm=8), P, D)
        assert {f"{s},{r}": list(v) for (s, r), v in pl.assignments.items()} == rec
        for (s, r), v in pl.assignments.items():
            assert v[1] == pl.rank_of(s, r)  # GPU index == executor rank


def test_simulator_configs(golden):
    for name, rec in golden("simulator")["configs"].items():
        L, h, s, P, D, m, M = CONFIGS[name]
        model = vp.make_block_model(name, L, h, s)
        uni = vp.uniform_profile(L, 1.0, 2.0, m_grid=(m,), d_grid=tuple(sorted({1, D})))
        a = vp.assign_stages(model, P, m, uni)
        n_m = vp.micro_batches_for(vp.JobSpec(M), m, D)
        cfg = vp.ParallelConfig(P, D, m, n_m, a.stage_map)
        pl = vp.build_placement(vp.uniform_cluster(P * D, gpus_per_vm=8), P, D)
        for tag in ("varuna", "gpipe"):
            gen = vp.generate_varuna_schedule if tag == "varuna" else vp.generate_gpipe_schedule
            for opp in (0, 1):
                r = vp.simulate_minibatch(gen(P, n_m, 1.0, 2.0, 1.0), cfg, uni, pl, model,
                                          opportunistic=bool(opp))
                want = rec[f"{tag},{opp}"]
                assert r.minibatch_us == want["minibatch_us"], (name, tag, opp)
                assert r.makespan_us == want["makespan_us"]
                assert r.bubble_fraction == want["bubble_fraction"]
                assert [list(x) for x in r.stage_idle_us] == want["stage_idle_us"]
                assert list(r.peak_memory_bytes) == want["peak_memory_bytes"]


def test_simulator_small_uniform(golden):
    for rec in golden("simulator")["uniform_small"]:
        p, n, d = rec["P"], rec["N"], rec["D"]
        model = vp.ModelSpec("u", (1,) * p, (8,) * p)
        prof = vp.uniform_profile(p, 1.0, 2.0, d_grid=tuple(range(1, d + 1)))
        cfg = vp.ParallelConfig(p, d, 1, n, vp.uniform_stage_map(p, p))
        pl = vp.build_placement(vp.uniform_cluster(p * d), p, d)
        r = vp.simulate_minibatch(vp.generate_varuna_schedule(p, n, 1.0, 2.0, 1.0), cfg, prof,
                                  pl, model)
        assert r.minibatch_us == rec["minibatch_us"] and r.bubble_fraction == rec["bubble_fraction"]


def test_simulator_jitter_commodity(golden):
    model = vp.make_block_model("gpt-2.5b-like", 54, 1920, 1024)
    hw = vp.HardwareSpec(16_000_000_000, 1, 12_500_000_000, 325_000_000, 2_000, 2_000, 5)
    prof = vp.synthesize_profile(model, hw, [1, 2, 4], [1, 2, 3], allreduce_bandwidth=1_250_000_000)
    for rec in golden("simulator")["jitter"]:
        P, D, m, n = rec["P"], rec["D"], rec["m"], rec["N"]
        cfg = vp.ParallelConfig(P, D, m, n, vp.uniform_stage_map(54, P))
        pl = vp.build_placement(vp.uniform_cluster(P * D, gpus_per_vm=rec["gpus_per_vm"]), P, D)
        r = vp.simulate_minibatch(vp.generate_varuna_schedule(P, n, 1.0, 2.0, 1.0), cfg, prof,
                                  pl, model, seed=rec["seed"], opportunistic=rec["opportunistic"])
        assert r.minibatch_us == rec["minibatch_us"], rec
        assert r.bubble_fraction == rec["bubble_fraction"]
        assert list(r.allreduce_us) == rec["allreduce_us"]
        assert list(r.allreduce_start_us) == rec["allreduce_start_us"]
        assert [_sha(x["task_start"]) for x in r.replicas] == rec["task_start_sha256"]
        assert [_sha(x["msg_arrive"]) for x in r.replicas] == rec["msg_arrive_sha256"]


def test_planner(golden):
    pl = golden("simulator")["planner"]
    for key, want in pl["micro_batches_for"].items():
        M, m, d = map(int, key.split(","))
        assert vp.micro_batches_for(vp.JobSpec(M), m, d) == want
    for key, want in pl["select_microbatch"].items():
        name, thr = key.split(",")
        L, h, s, *_ = CONFIGS[name]
        model = vp.make_block_model(name, L, h, s)
        syn = vp.synthesize_profile(model, vp.B200_NVL8, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
        assert vp.select_microbatch(syn, float(thr)) == want
    for key, want in pl["plan"].items():
        name, G = key.split(",")
        L, h, s, P, D, m, M = CONFIGS[name]
        model = vp.make_block_model(name, L, h, s)
        syn = vp.synthesize_profile(model, vp.B200_NVL8, [1, 2, 4, 8, 16, 32], [1, 2, 4, 8])
        r = vp.plan(int(G), model, vp.JobSpec(M), syn, vp.B200_NVL8,
                    vp.uniform_cluster(int(G), gpus_per_vm=8), micro_batch_size=m)
        assert (r.chosen.pipeline_depth, r.chosen.data_parallel) == (want["P"], want["D"])
        assert r.chosen.num_micro_batches == want["N_m"]
        assert list(r.chosen.stage_map) == want["stage_map"]
        assert r.minibatch_us == want["minibatch_us"]
        assert [[c.config.pipeline_depth, c.config.data_parallel, c.minibatch_us]
                for c in r.candidates] == want["candidates"]


def test_profile_yaml_roundtrip(tmp_path):
    model = vp.make_block_model("m", 6, 256, 128)
    prof = vp.synthesize_profile(model, vp.B200_NVL8, [1, 2, 4], [1, 2])
    path = str(tmp_path / "p.yaml")
    vp.save_profile(prof, path)
    back = vp.load_profile(path)
    assert back == prof
