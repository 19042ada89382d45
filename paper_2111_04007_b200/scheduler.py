"""Micro-batch schedules: the Varuna plan (generated natively), the GPipe
baseline, rule validation and the CSV wire format.

Public names and semantics follow spotpipe's scheduler (sp/scheduler.py):
``generate_varuna_schedule`` (:128-145) computes the plan by zero-delay
simulation of Varuna's three rules — here in C++ (``vp_varuna_schedule``,
paper_2111_04007_b200/csrc/control.cpp) — and returns the same flat
``kinds``/``mbs``/``offsets`` arrays bit for bit. The executor ships each
stage its slice of these arrays.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property, lru_cache
from typing import Dict, List, NamedTuple, Optional, Tuple

import numpy as np

from . import _lib
from .core import (KIND_BACKWARD, KIND_CODES, KIND_FORWARD, KIND_NAMES, KIND_RECOMPUTE,
                   ConfigError, us_from_seconds)

FORWARD, BACKWARD, RECOMPUTE = "F", "B", "R"
POLICY_VARUNA = "varuna"
POLICY_GPIPE = "gpipe"


class Task(NamedTuple):
    kind: str        # "F" | "B" | "R"
    micro_batch: int  # 1-based
    stage: int        # 1-based


@dataclass(frozen=True, eq=False)
class Schedule:
    """Per-stage ordered task lists as flat int64 arrays: stage k (0-based)
    owns ``kinds[offsets[k]:offsets[k+1]]`` (codes B=0 R=1 F=2) and the
    matching 0-based ``mbs``."""

    policy: str
    pipeline_depth: int
    num_micro_batches: int
    kinds: np.ndarray
    mbs: np.ndarray
    offsets: np.ndarray
    forward_us: int
    backward_us: int
    recompute_us: int

    def stage_slice(self, stage0: int) -> Tuple[np.ndarray, np.ndarray]:
        lo, hi = int(self.offsets[stage0]), int(self.offsets[stage0 + 1])
        return self.kinds[lo:hi], self.mbs[lo:hi]

    @cached_property
    def stage_tasks(self) -> Tuple[Tuple[Task, ...], ...]:
        out = []
        for k in range(self.pipeline_depth):
            kinds, mbs = self.stage_slice(k)
            out.append(tuple(Task(KIND_NAMES[int(a)], int(b) + 1, k + 1)
                             for a, b in zip(kinds.tolist(), mbs.tolist())))
        return tuple(out)

    def in_flight_bound(self, stage: int) -> int:
        """Largest prefix (#F − #B) of stage ``stage`` (1-based): the number of
        stashed micro-batches the stage must hold; sizes its receive ring."""
        return self.in_flight_bounds[stage - 1]

    @cached_property
    def in_flight_bounds(self) -> Tuple[int, ...]:
        out = []
        for k in range(self.pipeline_depth):
            kinds, _ = self.stage_slice(k)
            if kinds.size == 0:
                out.append(0)
                continue
            step = ((kinds == KIND_FORWARD).astype(np.int64)
                    - (kinds == KIND_BACKWARD).astype(np.int64))
            out.append(max(int(np.cumsum(step).max()), 0))
        return tuple(out)

    @cached_property
    def recompute_counts(self) -> Tuple[int, ...]:
        """Number of R tasks per stage (0-based order)."""
        return tuple(int((self.stage_slice(k)[0] == KIND_RECOMPUTE).sum())
                     for k in range(self.pipeline_depth))


def _make(policy, p, n, kinds, mbs, offsets, tf, tb, tr) -> Schedule:
    for a in (kinds, mbs, offsets):
        a.setflags(write=False)
    return Schedule(policy, p, n, kinds, mbs, offsets, tf, tb, tr)


def _times(forward_s, backward_s, recompute_s):
    tf, tb, tr = (us_from_seconds(x) for x in (forward_s, backward_s, recompute_s))
    if min(tf, tb, tr) <= 0:
        raise ConfigError("schedule: task times must be > 0")
    return tf, tb, tr


@lru_cache(maxsize=512)
def generate_varuna_schedule(pipeline_depth: int, num_micro_batches: int, forward_s: float,
                             backward_s: float, recompute_s: float) -> Schedule:
    p, n = pipeline_depth, num_micro_batches
    if p < 1 or n < 1:
        raise ConfigError("schedule: P and N_m must be >= 1")
    tf, tb, tr = _times(forward_s, backward_s, recompute_s)
    cap = 3 * p * n
    kinds = np.empty(cap, dtype=np.int64)
    mbs = np.empty(cap, dtype=np.int64)
    offsets = np.empty(p + 1, dtype=np.int64)
    rc = _lib.lib.vp_varuna_schedule(p, n, tf, tb, tr, cap, _lib.ptr(kinds), _lib.ptr(mbs),
                                     _lib.ptr(offsets))
    if rc == _lib.VP_ERR_DEADLOCK:
        raise AssertionError("rule simulation deadlocked")
    _lib.check(rc, "generate_varuna_schedule")
    total = int(offsets[p])
    return _make(POLICY_VARUNA, p, n, kinds[:total].copy(), mbs[:total].copy(), offsets,
                 tf, tb, tr)


@lru_cache(maxsize=512)
def generate_gpipe_schedule(pipeline_depth: int, num_micro_batches: int, forward_s: float,
                            backward_s: float, recompute_s: float) -> Schedule:
    p, n = pipeline_depth, num_micro_batches
    if p < 1 or n < 1:
        raise ConfigError("schedule: P and N_m must be >= 1")
    tf, tb, tr = _times(forward_s, backward_s, recompute_s)
    cap = 3 * p * n
    kinds = np.empty(cap, dtype=np.int64)
    mbs = np.empty(cap, dtype=np.int64)
    offsets = np.empty(p + 1, dtype=np.int64)
    _lib.check(_lib.lib.vp_gpipe_schedule(p, n, cap, _lib.ptr(kinds), _lib.ptr(mbs),
                                          _lib.ptr(offsets)), "generate_gpipe_schedule")
    total = int(offsets[p])
    return _make(POLICY_GPIPE, p, n, kinds[:total].copy(), mbs[:total].copy(), offsets,
                 tf, tb, tr)


def schedule_from_tasks(policy: str, stage_task_lists, forward_s: float, backward_s: float,
                        recompute_s: float) -> Schedule:
    """Schedule from explicit per-stage ``(letter, 1-based mb)`` lists."""
    p = len(stage_task_lists)
    n = max((mb for tasks in stage_task_lists for _, mb in tasks), default=0)
    kinds, mbs, offsets = [], [], [0]
    for tasks in stage_task_lists:
        for letter, mb in tasks:
            kinds.append(KIND_CODES[letter])
            mbs.append(mb - 1)
        offsets.append(len(kinds))
    return _make(policy, p, n, np.array(kinds, dtype=np.int64), np.array(mbs, dtype=np.int64),
                 np.array(offsets, dtype=np.int64), us_from_seconds(forward_s),
                 us_from_seconds(backward_s), us_from_seconds(recompute_s))


# ---------------------------------------------------------------------------
# Zero-delay replay and rule validation.
# ---------------------------------------------------------------------------

def _dependency(task: Task, p: int, end: Dict[Task, Tuple[int, int]]) -> Optional[int]:
    """End time of ``task``'s dependency; None while it has not run (0 = none).
    F waits for the activation from above, R for its own F, B for the
    gradient from below and its own R (the last stage: its own F)."""
    k, j = task.stage, task.micro_batch
    if task.kind == FORWARD:
        if k == 1:
            return 0
        up = end.get(Task(FORWARD, j, k - 1))
        return None if up is None else up[1]
    if task.kind == RECOMPUTE or k == p:
        own = end.get(Task(FORWARD, j, k))
        return None if own is None else own[1]
    down, rec = end.get(Task(BACKWARD, j, k + 1)), end.get(Task(RECOMPUTE, j, k))
    if down is None or rec is None:
        return None
    return max(down[1], rec[1])


def replay_uniform(schedule: Schedule) -> Dict[Task, Tuple[int, int]]:
    """Run the static lists in order under the schedule's uniform time model
    with zero network delay; (start_us, end_us) per task."""
    p = schedule.pipeline_depth
    dur = {FORWARD: schedule.forward_us, BACKWARD: schedule.backward_us,
           RECOMPUTE: schedule.recompute_us}
    lists = schedule.stage_tasks
    times: Dict[Task, Tuple[int, int]] = {}
    head = [0] * p
    free = [0] * p
    changed = True
    while changed:
        changed = False
        for k in range(p):
            while head[k] < len(lists[k]):
                t = lists[k][head[k]]
                dep = _dependency(t, p, times)
                if dep is None:
                    break
                s = max(free[k], dep)
                times[t] = (s, s + dur[t.kind])
                free[k] = s + dur[t.kind]
                head[k] += 1
                changed = True
    for k in range(p):
        if head[k] != len(lists[k]):
            t = lists[k][head[k]]
            raise ConfigError(f"schedule: stage {k + 1} deadlocks at {t.kind}{t.micro_batch} "
                              "(unsatisfiable dependency order)")
    return times


def makespan_us(schedule: Schedule) -> int:
    return max(e for _, e in replay_uniform(schedule).values())


@dataclass(frozen=True)
class RuleViolation:
    stage: int
    micro_batch: int
    rule: str
    message: str


def validate_schedule(schedule: Schedule) -> List[RuleViolation]:
    """Structure + Varuna rules 1–3 on the zero-delay replay."""
    p, n = schedule.pipeline_depth, schedule.num_micro_batches
    out: List[RuleViolation] = []
    for k, tasks in enumerate(schedule.stage_tasks, start=1):
        for letter in (FORWARD, BACKWARD):
            c = sum(t.kind == letter for t in tasks)
            if c != n:
                out.append(RuleViolation(k, 0, "structure",
                                         f"stage {k} has {c} {letter} tasks, expected {n}"))
        if schedule.policy == POLICY_VARUNA:
            want = 0 if (k == p or p == 1) else n
            c = sum(t.kind == RECOMPUTE for t in tasks)
            if c != want:
                out.append(RuleViolation(k, 0, "structure",
                                         f"stage {k} has {c} recomputes, expected {want}"))
        for i, t in enumerate(tasks):
            if t.kind != RECOMPUTE:
                continue
            nxt = tasks[i + 1] if i + 1 < len(tasks) else None
            if nxt is None or nxt.kind != BACKWARD or nxt.micro_batch != t.micro_batch:
                out.append(RuleViolation(k, t.micro_batch, "rule2",
                                         f"stage {k}: task between R{t.micro_batch} and "
                                         f"B{t.micro_batch}"))
    if out:
        return out
    try:
        times = replay_uniform(schedule)
    except ConfigError as e:
        return [RuleViolation(0, 0, "structure", str(e))]
    tr = schedule.recompute_us
    for k in range(1, p):
        for j in range(1, n + 1):
            r, d = times.get(Task(RECOMPUTE, j, k)), times.get(Task(BACKWARD, j, k + 1))
            if r is not None and d is not None and r[0] > d[1] - tr:
                out.append(RuleViolation(k, j, "rule1",
                                         f"stage {k}: R{j} starts at {r[0]}us, after gradient "
                                         f"arrival {d[1]}us - T_r"))
    for k, tasks in enumerate(schedule.stage_tasks, start=1):
        b_start = {t.micro_batch: times[t][0] for t in tasks if t.kind == BACKWARD}
        for t in tasks:
            if t.kind == BACKWARD:
                continue
            s = times[t][0]
            for j in range(1, n + 1):
                if j in b_start and b_start[j] <= s:
                    continue
                if k == p:
                    own = times.get(Task(FORWARD, j, k))
                    ready = None if own is None else own[1]
                else:
                    d, r = times.get(Task(BACKWARD, j, k + 1)), times.get(Task(RECOMPUTE, j, k))
                    ready = None if d is None or r is None else max(d[1], r[1])
                if ready is not None and ready <= s:
                    out.append(RuleViolation(k, t.micro_batch, "rule3",
                                             f"stage {k}: ran {t.kind}{t.micro_batch} at {s}us "
                                             f"while B{j} was ready"))
                    break
    return out


def schedule_to_csv(schedule: Schedule) -> str:
    """``stage,seq,kind,microbatch`` with 1-based stage/seq/micro-batch."""
    rows = ["stage,seq,kind,microbatch"]
    for k, tasks in enumerate(schedule.stage_tasks, start=1):
        rows += [f"{k},{i},{t.kind},{t.micro_batch}" for i, t in enumerate(tasks, start=1)]
    return "\n".join(rows) + "\n"


def schedule_from_csv(text: str, policy: str, forward_s: float, backward_s: float,
                      recompute_s: float) -> Schedule:
    lines = [ln for ln in text.strip().splitlines() if ln.strip()]
    if lines and lines[0].startswith("stage"):
        lines = lines[1:]
    per_stage: Dict[int, list] = {}
    for ln in lines:
        parts = ln.split(",")
        if len(parts) != 4:
            raise ConfigError(f"schedule csv: malformed line {ln!r}")
        k, seq, letter, mb = int(parts[0]), int(parts[1]), parts[2], int(parts[3])
        if letter not in (FORWARD, BACKWARD, RECOMPUTE):
            raise ConfigError(f"schedule csv: unknown kind {letter!r}")
        per_stage.setdefault(k, []).append((seq, letter, mb))
    if not per_stage or sorted(per_stage) != list(range(1, max(per_stage) + 1)):
        raise ConfigError("schedule csv: stages must be contiguous from 1")
    lists = [[(letter, mb) for _, letter, mb in sorted(per_stage[k])]
             for k in range(1, max(per_stage) + 1)]
    return schedule_from_tasks(policy, lists, forward_s, backward_s, recompute_s)
