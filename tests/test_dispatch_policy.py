"""The live per-stage dispatcher (paper_2111_04007_b200/dispatch.py
StagePolicy) against the reference's replica kernel: P independent
StagePolicy objects — each seeing only its own stage, the arrivals that
reached it and the rule-1 deadlines announced to it — driven by the
reference engine's event loop (sp/engine/py_kernel.py:322-333, restated
below) must start every task at the same time, in the same order, as the
compiled kernel (vp_run_replica, bit-exact to spotpipe's) on random
heterogeneous cases, static and opportunistic, serialized links or not."""

import heapq

import numpy as np
import pytest

import paper_2111_04007_b200 as vp
from paper_2111_04007_b200 import engine as veng
from paper_2111_04007_b200.core import KIND_BACKWARD as B, KIND_FORWARD as F
from paper_2111_04007_b200.dispatch import StagePolicy

UNIT = (1.0, 2.0, 1.0)


def drive(P, N, s, fwd, bwd, rec, act_tx, grad_tx, expg, cap, opp, ser):
    """Event loop of run_replica with the decisions made by StagePolicy."""
    offs = s.offsets.tolist()
    pols = []
    for k in range(P):
        tasks = list(zip(s.kinds[offs[k]:offs[k + 1]].tolist(),
                         s.mbs[offs[k]:offs[k + 1]].tolist()))
        pols.append(StagePolicy(tasks, N, k == P - 1, int(cap[k]), opp))
    act_arr = [[-1] * N for _ in range(P)]
    act_arr[0] = [0] * N
    grad_arr = [[-1] * N for _ in range(P)]
    deadline = [[-1] * N for _ in range(P)]
    act_free = [0] * max(P - 1, 1)
    grad_free = [0] * max(P - 1, 1)
    running = [None] * P      # (pos, kind, mb, end)
    out = []
    heap = [(0, k) for k in range(P)]
    heapq.heapify(heap)

    def send(boundary, direction, mb, now):
        dur = int((act_tx if direction == 0 else grad_tx)[boundary * N + mb])
        free = act_free if direction == 0 else grad_free
        if ser:
            grant = max(now, free[boundary])
            arrive = grant + dur
            free[boundary] = arrive
        else:
            arrive = now + dur
        if direction == 0:
            act_arr[boundary + 1][mb] = arrive
            heapq.heappush(heap, (arrive, boundary + 1))
        else:
            grad_arr[boundary][mb] = arrive
            heapq.heappush(heap, (arrive, boundary))
            jit = arrive - int(rec[boundary])
            heapq.heappush(heap, (max(jit, now), boundary))

    def decide(k, now):
        if running[k] is not None:
            return
        pol = pols[k]
        pos = pol.decide(now, lambda mb: act_arr[k][mb], lambda mb: grad_arr[k][mb],
                         lambda mb: deadline[k][mb], int(fwd[k]), int(rec[k]))
        if pos is None:
            return
        kind, mb = pol.kinds[pos], pol.mbs[pos]
        dur = int({F: fwd, B: bwd}.get(kind, rec)[k])
        pol.start(pos)
        running[k] = (pos, kind, mb, now + dur)
        out.append((k, kind, mb, now, now + dur))
        if kind == B and k > 0:
            dl = now + dur + int(expg[k - 1]) - int(rec[k - 1])
            deadline[k - 1][mb] = dl
            heapq.heappush(heap, (max(dl, now), k - 1))
        heapq.heappush(heap, (now + dur, k))

    while heap:
        now = heap[0][0]
        touched = set()
        while heap and heap[0][0] == now:
            _, k = heapq.heappop(heap)
            r = running[k]
            if r is not None and r[3] == now:
                pos, kind, mb, _ = r
                running[k] = None
                pols[k].complete(pos)
                if kind == F and k < P - 1:
                    send(k, 0, mb, now)
                elif kind == B and k > 0:
                    send(k - 1, 1, mb, now)
            touched.add(k)
        for k in sorted(touched):
            decide(k, now)
    assert all(p.done for p in pols)
    return out


@pytest.mark.parametrize("seed", range(6))
def test_stage_policies_reproduce_replica_kernel(seed):
    rng = np.random.default_rng(1000 + seed)
    for trial in range(25):
        P = int(rng.integers(1, 9))
        N = int(rng.integers(1, 17))
        s = vp.generate_varuna_schedule(P, N, *UNIT)
        fwd = rng.integers(100, 5000, size=P)
        bwd = fwd * 2 + rng.integers(0, 300, size=P)
        rec = fwd + rng.integers(0, 50, size=P)
        act = rng.integers(0, 2000, size=max(P - 1, 0) * N)
        grad = rng.integers(0, 2000, size=max(P - 1, 0) * N)
        expg = rng.integers(0, 2000, size=max(P - 1, 1))
        cap = np.array([s.in_flight_bound(k + 1) + int(rng.integers(0, 5)) for k in range(P)])
        ones = np.ones(P, dtype=np.int64)
        for opp in (False, True):
            for ser in (False, True):
                ref = veng.run_replica(P, N, s.kinds, s.mbs, s.offsets, fwd, bwd, rec, act, grad,
                                       expg, ones, ones, cap, opp, ser)
                got = drive(P, N, s, fwd, bwd, rec, act, grad, expg, cap, opp, ser)
                want = list(zip(*[ref[k].tolist() for k in ("task_stage", "task_kind", "task_mb",
                                                            "task_start", "task_end")]))
                assert got == want, (seed, trial, opp, ser)


def test_zero_delay_is_the_static_plan():
    P, N = 4, 8
    s = vp.generate_varuna_schedule(P, N, *UNIT)
    f = np.full(P, 1000)
    z = np.zeros((P - 1) * N, dtype=np.int64)
    got = drive(P, N, s, f, 2 * f, f, z, z, np.zeros(P - 1), np.full(P, N), True, True)
    for k in range(P):
        order = [(kind, mb) for st, kind, mb, _, _ in got if st == k]
        a, b = s.stage_slice(k)
        assert order == list(zip(a.tolist(), b.tolist()))
