"""Configuration search — the morph decision (sp/planner.py:72-208).

``plan(gpus, ...)`` sweeps P = 1..min(K, G) with D = ⌊G/P⌋, balances stages
with ``assign_stages``, sizes N_m = ⌈M/(m·D)⌉ so M_total is preserved across
reconfigurations, prices each candidate with ``simulate_minibatch`` and
returns the fastest (ties: shallower pipeline, then more replicas). The
schedule shape is always built with (T_f, T_b, T_r) = (1, 2, 1).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

from .calibration import CalibrationProfile
from .core import (ClusterState, ConfigError, HardwareSpec, InfeasibleError, JobSpec, ModelSpec,
                   ParallelConfig, seconds_from_us)
from .partitioner import assign_stages, memory_check
from .scheduler import POLICY_VARUNA, Schedule, generate_gpipe_schedule, generate_varuna_schedule
from .simulator import DEFAULT_STASH_PAD, build_placement, simulate_minibatch

CANONICAL_TIMES = (1.0, 2.0, 1.0)


@dataclass(frozen=True)
class Candidate:
    config: ParallelConfig
    minibatch_us: int

    @property
    def minibatch_seconds(self) -> float:
        return seconds_from_us(self.minibatch_us)


@dataclass(frozen=True)
class PlanResult:
    chosen: ParallelConfig
    minibatch_us: int
    total_gpus: int
    candidates: Tuple[Candidate, ...]

    @property
    def minibatch_seconds(self) -> float:
        return seconds_from_us(self.minibatch_us)

    def throughput(self, job: JobSpec) -> float:
        return job.minibatch_examples / self.minibatch_seconds

    def throughput_per_gpu(self, job: JobSpec) -> float:
        return self.throughput(job) / self.chosen.gpus_used

    @property
    def unused_gpus(self) -> int:
        return self.total_gpus - self.chosen.gpus_used


def select_microbatch(profile: CalibrationProfile, improvement_threshold: float = 0.02) -> int:
    """First grid m after which mean per-example forward time (over cut-points)
    improves by no more than the threshold; the last grid point otherwise."""
    grid = profile.m_grid
    if not grid:
        raise ConfigError("select_microbatch: profile has an empty m grid")
    K = profile.num_cutpoints

    def per_example(m):
        return sum(profile.forward_us(i, m) for i in range(K)) / (m * K)

    for cur, nxt in zip(grid, grid[1:]):
        if per_example(nxt) >= per_example(cur) * (1.0 - improvement_threshold):
            return cur
    return grid[-1]


def micro_batches_for(job: JobSpec, m: int, d: int) -> int:
    """N_m = max(1, ⌈M / (m·D)⌉): the last micro-batch may be partial so that
    M_total is preserved exactly."""
    return max(1, math.ceil(job.minibatch_examples / (m * d)))


def schedule_for(policy: str, p: int, n_m: int) -> Schedule:
    gen = generate_varuna_schedule if policy == POLICY_VARUNA else generate_gpipe_schedule
    return gen(p, n_m, *CANONICAL_TIMES)


def _faster(a: Candidate, b: Candidate) -> bool:
    return (a.minibatch_us, a.config.pipeline_depth, -a.config.data_parallel) < \
        (b.minibatch_us, b.config.pipeline_depth, -b.config.data_parallel)


def _sweep(gpus, model, job, profile, hw, cluster, m, seed, opportunistic,
           policy) -> Optional[PlanResult]:
    cands: List[Candidate] = []
    best = None
    for p in range(1, min(model.num_cutpoints, gpus) + 1):
        d = gpus // p
        if d == 0:
            break
        a = assign_stages(model, p, m, profile)
        n_m = micro_batches_for(job, m, d)
        sched = schedule_for(policy, p, n_m)
        bounds = [sched.in_flight_bound(s + 1) + DEFAULT_STASH_PAD for s in range(p)]
        if not memory_check(a, m, n_m, hw, in_flight_bound=bounds,
                            bytes_per_param=profile.optimizer_bytes_per_param).feasible:
            continue
        cfg = ParallelConfig(p, d, m, n_m, a.stage_map)
        res = simulate_minibatch(sched, cfg, profile, build_placement(cluster, p, d), model,
                                 seed=seed, opportunistic=opportunistic)
        c = Candidate(cfg, res.minibatch_us)
        cands.append(c)
        if best is None or _faster(c, best):
            best = c
    if best is None:
        return None
    return PlanResult(best.config, best.minibatch_us, gpus, tuple(cands))


def plan(gpus: int, model: ModelSpec, job: JobSpec, profile: CalibrationProfile,
         hw: HardwareSpec, cluster: ClusterState, seed: int = 0,
         micro_batch_size: Optional[int] = None, opportunistic: bool = True,
         improvement_threshold: float = 0.02, schedule_policy: str = POLICY_VARUNA) -> PlanResult:
    if gpus < 1:
        raise InfeasibleError("no feasible configuration: zero GPUs available")
    if profile.num_cutpoints != model.num_cutpoints:
        raise ConfigError(f"plan: profile has {profile.num_cutpoints} cut-points, "
                          f"model has {model.num_cutpoints}")
    m = micro_batch_size or select_microbatch(profile, improvement_threshold)
    res = _sweep(gpus, model, job, profile, hw, cluster, m, seed, opportunistic, schedule_policy)
    if res is None and micro_batch_size is None:
        for smaller in sorted((g for g in profile.m_grid if g < m), reverse=True):
            res = _sweep(gpus, model, job, profile, hw, cluster, smaller, seed, opportunistic,
                         schedule_policy)
            if res is not None:
                break
    if res is None:
        raise InfeasibleError("no feasible configuration: the model does not fit at any "
                              f"pipeline depth up to {min(model.num_cutpoints, gpus)}")
    return res
