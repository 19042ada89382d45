"""Oracle: Varuna / GPipe static plans restated in plain Python.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Pinned against
tests/golden/schedules.json, which the reference itself produced.

Kind codes follow sp/core.py:22-26: B=0, R=1, F=2; micro-batches are 0-based
in the flat arrays.
"""

from __future__ import annotations

import heapq

B, R, F = 0, 1, 2


def us(seconds: float) -> int:
    """sp/core.py:37-38 — round-half-even of seconds*1e6."""
    return int(round(seconds * 1_000_000))


def varuna_plan(p: int, n: int, tf: int, tb: int, tr: int):
    """Zero-delay joint simulation of Varuna's three rules.

    Restates sp/scheduler.py:179-284. Returns one list of (kind, mb) per
    stage in start order.

    Rule 3 (backward first, :239-245), rule 2 (after R(j) only B(j) may run,
    :228-235), rule 1 (just-in-time recompute: R(j) is due at downstream
    B(j)'s start + tb - tr, :273-279; a forward fills the gap only if it ends
    by that deadline, :254-258); the last stage alternates F/B and never
    recomputes (:239-241).
    """
    last = p - 1
    plan = [[] for _ in range(p)]
    end_at = [0] * p
    cur = [None] * p                      # (kind, mb) while running
    nf = [0] * p                          # forwards started-and-finished count
    nb = [0] * p
    act = [[0 if k == 0 else None for _ in range(n)] for k in range(p)]
    grad = [[None] * n for _ in range(p)]
    due = [[None] * n for _ in range(p)]
    recomputed = [[False] * n for _ in range(p)]
    hold = [None] * p                     # rule-2 lock
    times = [0]

    def arrived(t, now):
        return t is not None and t <= now

    while times:
        now = heapq.heappop(times)
        while times and times[0] == now:
            heapq.heappop(times)
        # Completions first (all stages), then decisions in stage order.
        for k in range(p):
            if cur[k] is not None and end_at[k] == now:
                kind, mb = cur[k]
                cur[k] = None
                if kind == F:
                    nf[k] += 1
                    if k < last:
                        act[k + 1][mb] = now
                elif kind == R:
                    recomputed[k][mb] = True
                    hold[k] = mb
                else:
                    nb[k] += 1
                    if k > 0:
                        grad[k - 1][mb] = now
        for k in range(p):
            if cur[k] is not None or nb[k] >= n:
                continue
            pick = None
            if hold[k] is not None:
                j = hold[k]
                if arrived(grad[k][j], now):
                    pick = (B, j)
                else:
                    continue
            else:
                j = nb[k]
                if k == last:
                    if nf[k] > j:
                        pick = (B, j)
                elif arrived(grad[k][j], now) and recomputed[k][j]:
                    pick = (B, j)
                elif nf[k] > j and not recomputed[k][j]:
                    if arrived(grad[k][j], now):
                        pick = (R, j)
                    elif due[k][j] is not None:
                        d = due[k][j]
                        if now >= d:
                            pick = (R, j)
                        else:
                            f = nf[k]
                            if f < n and arrived(act[k][f], now) and now + tf <= d:
                                pick = (F, f)
                            else:
                                heapq.heappush(times, d)
                                continue
                if pick is None:
                    f = nf[k]
                    if f < n and arrived(act[k][f], now):
                        pick = (F, f)
                    else:
                        continue
            kind, mb = pick
            dur = tf if kind == F else (tb if kind == B else tr)
            plan[k].append(pick)
            cur[k] = pick
            end_at[k] = now + dur
            heapq.heappush(times, now + dur)
            if kind == B:
                hold[k] = None
                if k > 0:
                    d = now + tb - tr
                    due[k - 1][mb] = d
                    heapq.heappush(times, max(d, now))
    for k in range(p):
        if nb[k] != n:
            raise AssertionError(f"rule simulation deadlocked at stage {k + 1}")
    return plan


def gpipe_plan(p: int, n: int):
    """sp/scheduler.py:148-176: all forwards, then (R,B) pairs in reverse
    micro-batch order; the last stage skips R for its final micro-batch."""
    out = []
    for k in range(p):
        tasks = [(F, j) for j in range(n)]
        first = n - 1
        if k == p - 1:
            tasks.append((B, n - 1))
            first = n - 2
        for j in range(first, -1, -1):
            tasks += [(R, j), (B, j)]
        out.append(tasks)
    return out


def flatten(plan):
    """sp/scheduler.py:100-117 — flat kinds/mbs/offsets arrays."""
    kinds, mbs, offsets = [], [], [0]
    for tasks in plan:
        for kind, mb in tasks:
            kinds.append(kind)
            mbs.append(mb)
        offsets.append(len(kinds))
    return kinds, mbs, offsets


def in_flight_bound(plan_stage) -> int:
    """sp/scheduler.py:88-97: max prefix (#F - #B), floored at 0."""
    best = run = 0
    for kind, _ in plan_stage:
        run += (kind == F) - (kind == B)
        best = max(best, run)
    return best


def replay_makespan(plan, tf: int, tb: int, tr: int) -> int:
    """Zero-delay in-order replay; restates sp/scheduler.py:307-373."""
    p = len(plan)
    dur = {F: tf, B: tb, R: tr}
    done = {}  # (kind, mb, stage) -> end time
    ptr = [0] * p
    free = [0] * p
    moved = True
    while moved:
        moved = False
        for k in range(p):
            while ptr[k] < len(plan[k]):
                kind, j = plan[k][ptr[k]]
                if kind == F:
                    dep = 0 if k == 0 else done.get((F, j, k - 1))
                elif kind == R:
                    dep = done.get((F, j, k))
                elif k == p - 1:
                    dep = done.get((F, j, k))
                else:
                    a, b = done.get((B, j, k + 1)), done.get((R, j, k))
                    dep = None if a is None or b is None else max(a, b)
                if dep is None:
                    break
                start = max(free[k], dep)
                done[(kind, j, k)] = free[k] = start + dur[kind]
                ptr[k] += 1
                moved = True
    if any(ptr[k] != len(plan[k]) for k in range(p)):
        raise ValueError("unsatisfiable dependency order")
    return max(done.values()) if done else 0


def to_csv(plan) -> str:
    """sp/scheduler.py:467-473: ``stage,seq,kind,microbatch`` 1-based."""
    name = {F: "F", B: "B", R: "R"}
    rows = ["stage,seq,kind,microbatch"]
    for k, tasks in enumerate(plan):
        for i, (kind, mb) in enumerate(tasks):
            rows.append(f"{k + 1},{i + 1},{name[kind]},{mb + 1}")
    return "\n".join(rows) + "\n"
