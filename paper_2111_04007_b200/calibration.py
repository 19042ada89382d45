"""Calibration profile: per-cut-point F/B times, transfer and allreduce times.

Same data model and YAML wire format (``format_version: 1``) as spotpipe's
profile (sp/calibration.py:57-159, 321-393), so a profile MEASURED on B200 by
``paper_2111_04007_b200.measure`` can be fed to the reference planner and
simulator unchanged, and vice versa. Grid lookups never interpolate.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Sequence, Tuple

import numpy as np
import yaml

from .core import OPTIMIZER_BYTES_PER_PARAM, ConfigError, HardwareSpec, ModelSpec, us_from_seconds

PROFILE_FORMAT_VERSION = 1

#: per-m tables, in file order (sp/calibration.py:45-54)
PER_M_FIELDS = ("forward_us", "backward_us", "act_intra_us", "grad_intra_us",
                "act_inter_mean_us", "act_inter_jitter_us", "grad_inter_mean_us",
                "grad_inter_jitter_us")


@dataclass(frozen=True)
class CutpointTimes:
    forward_us: Dict[int, int]
    backward_us: Dict[int, int]
    act_intra_us: Dict[int, int]
    grad_intra_us: Dict[int, int]
    act_inter_mean_us: Dict[int, int]
    act_inter_jitter_us: Dict[int, int]
    grad_inter_mean_us: Dict[int, int]
    grad_inter_jitter_us: Dict[int, int]
    allreduce_us: Dict[int, int]


def _lookup(table, key, i, axis):
    if key not in table:
        raise ConfigError(f"calibration: cut-point {i} has no grid point {axis}={key} "
                          "(no interpolation; regenerate the profile with this grid value)")
    return table[key]


@dataclass(frozen=True)
class CalibrationProfile:
    m_grid: Tuple[int, ...]
    d_grid: Tuple[int, ...]
    cutpoints: Tuple[CutpointTimes, ...]
    optimizer_bytes_per_param: int = OPTIMIZER_BYTES_PER_PARAM

    def __post_init__(self):
        self._validate()

    def _validate(self):
        for name, grid in (("m_grid", self.m_grid), ("d_grid", self.d_grid)):
            if not grid:
                raise ConfigError(f"calibration: {name} must be non-empty")
            if list(grid) != sorted(set(grid)):
                raise ConfigError(f"calibration: {name} must be strictly increasing")
        for i, cp in enumerate(self.cutpoints):
            for name in PER_M_FIELDS:
                table = getattr(cp, name)
                for m in self.m_grid:
                    if m not in table:
                        raise ConfigError(f"calibration: cutpoint[{i}].{name} missing m={m}")
                    if table[m] < 0:
                        raise ConfigError(f"calibration: cutpoint[{i}].{name}[{m}] is negative")
            for name in ("forward_us", "backward_us"):
                seq = [getattr(cp, name)[m] for m in self.m_grid]
                if any(b < a for a, b in zip(seq, seq[1:])):
                    raise ConfigError(f"calibration: cutpoint[{i}].{name} must be "
                                      "non-decreasing in m")
            for d in self.d_grid:
                if d not in cp.allreduce_us:
                    raise ConfigError(f"calibration: cutpoint[{i}].allreduce_us missing D={d}")
                if cp.allreduce_us[d] < 0:
                    raise ConfigError(f"calibration: cutpoint[{i}].allreduce_us[{d}] is negative")
            if cp.allreduce_us.get(1, 0) != 0:
                raise ConfigError(f"calibration: cutpoint[{i}].allreduce_us[1] must be 0 "
                                  "(allreduce over a ring of one is a no-op)")

    @property
    def num_cutpoints(self) -> int:
        return len(self.cutpoints)

    def column(self, name: str, key: int):
        """int64 vector over cut-points of table ``name`` at grid point ``key``
        (m, or D for ``allreduce_us``); memoised — the profile is frozen."""
        cache = self.__dict__.setdefault("_columns", {})
        col = cache.get((name, key))
        if col is None:
            axis = "D" if name == "allreduce_us" else "m"
            col = np.array([_lookup(getattr(cp, name), key, i, axis)
                            for i, cp in enumerate(self.cutpoints)], dtype=np.int64)
            col.setflags(write=False)
            cache[(name, key)] = col
        return col

    def forward_us(self, i: int, m: int) -> int:
        return _lookup(self.cutpoints[i].forward_us, m, i, "m")

    def backward_us(self, i: int, m: int) -> int:
        return _lookup(self.cutpoints[i].backward_us, m, i, "m")

    def allreduce_us(self, i: int, d: int) -> int:
        return _lookup(self.cutpoints[i].allreduce_us, d, i, "D")

    def transfer_us(self, i: int, m: int, inter_node: bool, gradient: bool) -> Tuple[int, int]:
        """(mean, jitter stddev) µs of one boundary message."""
        cp = self.cutpoints[i]
        if not inter_node:
            table = cp.grad_intra_us if gradient else cp.act_intra_us
            return _lookup(table, m, i, "m"), 0
        mean = cp.grad_inter_mean_us if gradient else cp.act_inter_mean_us
        jit = cp.grad_inter_jitter_us if gradient else cp.act_inter_jitter_us
        return _lookup(mean, m, i, "m"), _lookup(jit, m, i, "m")


def ring_allreduce_seconds(payload_bytes: float, ring_size: int, bandwidth: float,
                           latency_s: float, contention_multiplier: float = 1.0) -> float:
    """α-β ring allreduce: 2(D-1)/D payload passes + 2(D-1) hops."""
    if ring_size <= 1:
        return 0.0
    d = ring_size
    return contention_multiplier * (2.0 * (d - 1) / d * payload_bytes / bandwidth
                                    + 2.0 * (d - 1) * latency_s)


def uniform_profile(stages: int, forward_s: float, backward_s: float,
                    m_grid: Sequence[int] = (1,), d_grid: Sequence[int] = (1,)) -> CalibrationProfile:
    """One cut-point per stage, identical times, zero network cost."""
    f, b = us_from_seconds(forward_s), us_from_seconds(backward_s)
    m_grid = tuple(m_grid)
    zero = {m: 0 for m in m_grid}
    cp = CutpointTimes({m: f for m in m_grid}, {m: b for m in m_grid}, dict(zero), dict(zero),
                       dict(zero), dict(zero), dict(zero), dict(zero), {d: 0 for d in d_grid})
    return CalibrationProfile(m_grid, tuple(d_grid), (cp,) * stages)


def synthesize_profile(model: ModelSpec, hw: HardwareSpec, m_grid: Sequence[int],
                       d_grid: Sequence[int],
                       seconds_per_unit_work: float = 0.010 / (12 * 1920 * 1920 * 4),
                       fixed_work_fraction: float = 0.15, backward_ratio: float = 2.0,
                       grad_bytes_per_param: int = 4, contention_multiplier: float = 1.0,
                       allreduce_bandwidth=None) -> CalibrationProfile:
    """Analytic profile, F = c·params·(m + 0.15), B = ratio·F, transfers =
    bytes/bw + latency (sp/calibration.py:179-255). Kept for planner parity;
    the executor itself uses MEASURED profiles."""
    if not m_grid or not d_grid:
        raise ConfigError("synthesize_profile: grids must be non-empty")
    ar_bw = hw.inter_node_bandwidth if allreduce_bandwidth is None else allreduce_bandwidth
    m_grid = tuple(sorted({int(m) for m in m_grid}))
    d_grid = tuple(sorted({int(d) for d in d_grid}))
    cps = []
    for params, act in zip(model.cutpoint_parameters, model.cutpoint_activation_bytes):
        f, b, intra, inter, jit = {}, {}, {}, {}, {}
        for m in m_grid:
            sec = seconds_per_unit_work * params * (m + fixed_work_fraction)
            f[m] = us_from_seconds(sec)
            b[m] = us_from_seconds(backward_ratio * sec)
            intra[m] = us_from_seconds(act * m / hw.intra_node_bandwidth) + hw.intra_node_latency_us
            inter[m] = us_from_seconds(act * m / hw.inter_node_bandwidth) + hw.inter_node_latency_us
            jit[m] = hw.inter_node_jitter_us
        ar = {d: us_from_seconds(ring_allreduce_seconds(float(params * grad_bytes_per_param), d,
                                                        ar_bw, hw.inter_node_latency_us / 1e6,
                                                        contention_multiplier))
              for d in d_grid}
        cps.append(CutpointTimes(f, b, dict(intra), dict(intra), dict(inter), dict(jit),
                                 dict(inter), dict(jit), ar))
    return CalibrationProfile(m_grid, d_grid, tuple(cps))


def save_profile(profile: CalibrationProfile, path: str) -> None:
    doc = {"format_version": PROFILE_FORMAT_VERSION,
           "optimizer_bytes_per_param": profile.optimizer_bytes_per_param,
           "m_grid": list(profile.m_grid), "d_grid": list(profile.d_grid),
           "cutpoints": [{name: dict(getattr(cp, name)) for name in PER_M_FIELDS + ("allreduce_us",)}
                         for cp in profile.cutpoints]}
    with open(path, "w") as f:
        yaml.safe_dump(doc, f, sort_keys=False)


def load_profile(path: str) -> CalibrationProfile:
    try:
        with open(path) as f:
            doc = yaml.safe_load(f)
    except FileNotFoundError:
        raise ConfigError(f"{path}: file not found")
    except yaml.YAMLError as e:
        raise ConfigError(f"{path}: parse error: {e}")
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: expected a mapping at top level")
    if doc.get("format_version") != PROFILE_FORMAT_VERSION:
        raise ConfigError(f"{path}.format_version: unsupported version "
                          f"{doc.get('format_version')!r}")
    allowed = {"format_version", "optimizer_bytes_per_param", "m_grid", "d_grid", "cutpoints"}
    for key in doc:
        if key not in allowed:
            raise ConfigError(f"{path}.{key}: unknown key")
    for key in ("m_grid", "d_grid", "cutpoints"):
        if key not in doc:
            raise ConfigError(f"{path}: missing required key {key}")
    raw = doc["cutpoints"]
    if not isinstance(raw, list) or not raw:
        raise ConfigError(f"{path}.cutpoints: expected a non-empty list")
    cps = []
    names = PER_M_FIELDS + ("allreduce_us",)
    for i, entry in enumerate(raw):
        if not isinstance(entry, dict):
            raise ConfigError(f"{path}.cutpoints[{i}]: expected a mapping")
        for key in entry:
            if key not in names:
                raise ConfigError(f"{path}.cutpoints[{i}].{key}: unknown key")
        tables = {}
        for name in names:
            if name not in entry:
                raise ConfigError(f"{path}.cutpoints[{i}].{name}: missing required table")
            if not isinstance(entry[name], dict):
                raise ConfigError(f"{path}.cutpoints[{i}].{name}: expected a mapping")
            tables[name] = {int(k): int(v) for k, v in entry[name].items()}
        cps.append(CutpointTimes(**tables))
    return CalibrationProfile(tuple(int(m) for m in doc["m_grid"]),
                              tuple(int(d) for d in doc["d_grid"]), tuple(cps),
                              int(doc.get("optimizer_bytes_per_param", OPTIMIZER_BYTES_PER_PARAM)))
