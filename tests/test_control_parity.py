"""Product control plane (libvpipe.so, C++) vs the reference's own outputs
(tests/golden/*, produced by spotpipe 0.1.0) and vs the pinned oracle on
fresh random cases. Bit-exact: integer arrays must be identical."""

import sys
import os
import hashlib

import numpy as np
import pytest

import paper_2111_04007_b200 as vp
from paper_2111_04007_b200 import engine as veng
from oracle import engine as oeng
from oracle import schedule as osch

UNIT = (1.0, 2.0, 1.0)
KEYS = ["task_stage", "task_kind", "task_mb", "task_start", "task_end", "msg_send",
        "msg_grant", "msg_arrive", "msg_boundary", "msg_dir", "msg_mb",
        "last_bwd_end", "peak_stash", "peak_sets", "peak_mem"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def test_library_version():
    assert b"vpipe" in vp._lib.lib.vp_version()


def test_small_plans_bit_exact(golden):
    for key, rec in golden("schedules")["small"].items():
        policy, p, n = key.split(",")
        gen = vp.generate_varuna_schedule if policy == "varuna" else vp.generate_gpipe_schedule
        s = gen(int(p), int(n), *UNIT)
        assert s.kinds.tolist() == rec["kinds"], key
        assert s.mbs.tolist() == rec["mbs"], key
        assert s.offsets.tolist() == rec["offsets"], key
        assert [s.in_flight_bound(k + 1) for k in range(int(p))] == rec["in_flight_bound"]
        assert vp.makespan_us(s) == rec["makespan_us"], key


def test_config_plans_bit_exact(golden):
    for key, rec in golden("schedules")["configs"].items():
        p, n = map(int, key.split(","))
        s = vp.generate_varuna_schedule(p, n, *UNIT)
        assert hashlib.sha256(vp.schedule_to_csv(s).encode()).hexdigest() == rec["csv_sha256"]
        assert _sha(s.kinds) == rec["kinds_sha256"] and _sha(s.mbs) == rec["mbs_sha256"]
        assert int(s.offsets[-1]) == rec["n_tasks"]
        assert [s.in_flight_bound(k + 1) for k in range(p)] == rec["in_flight_bound"]
        if n <= 128:
            assert vp.makespan_us(s) == rec["makespan_us"]
            g = vp.generate_gpipe_schedule(p, n, *UNIT)
            assert vp.makespan_us(g) == rec["gpipe_makespan_us"]


def test_noncanonical_ratios(golden):
    for key, rec in golden("schedules")["ratios"].items():
        tf, tb, tr, p, n = key.split(",")
        s = vp.generate_varuna_schedule(int(p), int(n), float(tf), float(tb), float(tr))
        assert hashlib.sha256(vp.schedule_to_csv(s).encode()).hexdigest() == rec["csv_sha256"], key


def test_reference_known_answers():
    # pkg/tests/test_scheduler.py:30-49, 116-120, 228-242 and
    # pkg/tests/test_acceptance.py:50-63 known answers.
    s = vp.generate_varuna_schedule(1, 4, *UNIT)
    assert [t.kind + str(t.micro_batch) for t in s.stage_tasks[0]] == \
        ["F1", "B1", "F2", "B2", "F3", "B3", "F4", "B4"]
    v, g = vp.generate_varuna_schedule(4, 5, *UNIT), vp.generate_gpipe_schedule(4, 5, *UNIT)
    assert vp.makespan_us(g) - vp.makespan_us(v) == 1_000_000
    assert vp.makespan_us(v) == 27_000_000
    assert v.in_flight_bound(1) == 5 and v.in_flight_bound(4) == 1
    assert vp.generate_varuna_schedule(2, 2, *UNIT).stage_tasks[1] == (
        vp.Task("F", 1, 2), vp.Task("B", 1, 2), vp.Task("F", 2, 2), vp.Task("B", 2, 2))
    with pytest.raises(vp.ConfigError):
        vp.generate_varuna_schedule(0, 5, *UNIT)
    with pytest.raises(vp.ConfigError):
        vp.generate_varuna_schedule(2, 2, 0.0, 1.0, 1.0)


def test_golden_csv(golden):
    assert vp.schedule_to_csv(vp.generate_varuna_schedule(2, 2, *UNIT)) == \
        golden("schedules")["csv_2_2"]
    s = vp.generate_varuna_schedule(3, 4, *UNIT)
    back = vp.schedule_from_csv(vp.schedule_to_csv(s), vp.POLICY_VARUNA, *UNIT)
    assert back.stage_tasks == s.stage_tasks


def test_validator_clean_and_dominance():
    for p in range(1, 9):
        for n in range(1, 17):
            v = vp.generate_varuna_schedule(p, n, *UNIT)
            assert vp.validate_schedule(v) == []
            assert vp.makespan_us(v) <= vp.makespan_us(vp.generate_gpipe_schedule(p, n, *UNIT))


def test_engine_bit_exact_vs_reference(golden):
    for i, c in enumerate(golden("engine_cases")):
        gen = vp.generate_varuna_schedule if c["policy"] == "varuna" else vp.generate_gpipe_schedule
        s = gen(c["P"], c["N"], *UNIT)
        out = veng.run_replica(c["P"], c["N"], s.kinds, s.mbs, s.offsets, c["fwd_us"],
                               c["bwd_us"], c["rec_us"], c["act_tx_us"], c["grad_tx_us"],
                               c["exp_grad_tx_us"], c["in_act_bytes"], c["work_bytes"],
                               c["stash_cap"], c["opportunistic"], c["serialize_links"])
        assert out["makespan"] == c["makespan"], i
        for k in KEYS:
            assert _sha(out[k]) == c["sha256"][k], (i, k)


def test_engine_matches_oracle_random():
    rng = np.random.default_rng(99)
    for trial in range(150):
        P = int(rng.integers(1, 11))
        N = int(rng.integers(1, 20))
        s = vp.generate_varuna_schedule(P, N, *UNIT) if trial % 3 else \
            vp.generate_gpipe_schedule(P, N, *UNIT)
        fwd = rng.integers(100, 5000, size=P)
        bwd = fwd * 2 + rng.integers(0, 100, size=P)
        rec = fwd + rng.integers(0, 10, size=P)
        act = rng.integers(0, 800, size=max(P - 1, 0) * N)
        grad = rng.integers(0, 800, size=max(P - 1, 0) * N)
        expg = rng.integers(0, 800, size=max(P - 1, 1))
        in_act = rng.integers(1, 1000, size=P)
        work = rng.integers(1, 1000, size=P)
        cap = np.array([s.in_flight_bound(k + 1) + int(rng.integers(0, 5)) for k in range(P)])
        for opp in (False, True):
            for ser in (False, True):
                args = (P, N, s.kinds, s.mbs, s.offsets, fwd, bwd, rec, act, grad, expg,
                        in_act, work, cap, opp, ser)
                a, b = veng.run_replica(*args), oeng.run_replica(*args)
                assert a["makespan"] == b["makespan"]
                for k in KEYS:
                    assert np.array_equal(a[k], b[k]), (trial, k)


def test_zero_delay_collapse_to_static_plan():
    for P, N in ((4, 5), (1, 4), (7, 9)):
        s = vp.generate_varuna_schedule(P, N, *UNIT)
        f = np.full(P, 1_000_000)
        zero = np.zeros(max(P - 1, 0) * N)
        spans = {veng.run_replica(P, N, s.kinds, s.mbs, s.offsets, f, 2 * f, f, zero, zero,
                                  np.zeros(max(P - 1, 1)), np.ones(P), np.ones(P),
                                  np.full(P, N), opp, True)["makespan"] for opp in (0, 1)}
        assert spans == {vp.makespan_us(s)}


def test_schedule_matches_oracle_large():
    for p, n in ((8, 200), (3, 333), (6, 97), (5, 128)):
        s = vp.generate_varuna_schedule(p, n, *UNIT)
        k, m, o = osch.flatten(osch.varuna_plan(p, n, 1_000_000, 2_000_000, 1_000_000))
        assert s.kinds.tolist() == k and s.mbs.tolist() == m and s.offsets.tolist() == o


def test_opportunistic_execution_order():
    from paper_2111_04007_b200 import ParallelConfig, generate_varuna_schedule, make_block_model
    from paper_2111_04007_b200.simulator import execution_order
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from dist_pipeline_check import skewed_profile
    sch = generate_varuna_schedule(2, 4, 1.0, 2.0, 1.0)
    pc = ParallelConfig(2, 1, 4, 4, (0, 0, 1, 1))
    order = execution_order(sch, pc, skewed_profile(), make_block_model("t", 4, 256, 128))
    moved = 0
    for k in range(2):
        kinds, mbs = sch.stage_slice(k)
        static = list(zip(kinds.tolist(), mbs.tolist()))
        assert sorted(static) == sorted(order[k])          # a permutation of the stage's tasks
        moved += sum(a != b for a, b in zip(static, order[k]))
        for i, (kind, j) in enumerate(order[k]):           # rule 2 holds in the replayed order
            if kind == 0 and k < 1:
                assert order[k][i - 1] == (1, j)
            if kind == 0:
                assert (2, j) in order[k][:i]
    assert moved > 0
