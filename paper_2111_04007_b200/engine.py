"""Replica event kernel: ``run_replica`` with the reference's 16-argument
contract (sp/engine/_kernel.pyx:334-351), implemented natively by
``vp_run_replica`` (csrc/control.cpp). The same C++ policy object is what the
live per-stage dispatcher would drive; ENGINE_NAME reports the native path."""

from __future__ import annotations

import numpy as np

from . import _lib

ENGINE_NAME = "native"

_OUT_KEYS = ("task_stage", "task_kind", "task_mb", "task_start", "task_end",
             "msg_send", "msg_grant", "msg_arrive", "msg_boundary", "msg_dir", "msg_mb")
_STAGE_KEYS = ("last_bwd_end", "peak_stash", "peak_sets", "peak_mem")


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def run_replica(n_stages, n_micro, kinds, mbs, offsets, fwd_us, bwd_us, rec_us, act_tx_us,
                grad_tx_us, exp_grad_tx_us, in_act_bytes, work_bytes, stash_cap,
                opportunistic, serialize_links) -> dict:
    P, N = int(n_stages), int(n_micro)
    ins = [_i64(x) for x in (kinds, mbs, offsets, fwd_us, bwd_us, rec_us, act_tx_us, grad_tx_us,
                             exp_grad_tx_us, in_act_bytes, work_bytes, stash_cap)]
    if ins[2].size < P + 1:
        raise ValueError("offsets must have P+1 entries")
    if ins[8].size == 0:
        ins[8] = np.zeros(1, dtype=np.int64)
    for i in (6, 7):
        if ins[i].size == 0:
            ins[i] = np.zeros(1, dtype=np.int64)
    n_tasks = int(ins[2][P])
    n_msgs = max(2 * (P - 1) * N, 1)
    bufs = {k: np.empty(max(n_tasks, 1), dtype=np.int64) for k in _OUT_KEYS[:5]}
    bufs.update({k: np.empty(n_msgs, dtype=np.int64) for k in _OUT_KEYS[5:]})
    bufs.update({k: np.empty(P, dtype=np.int64) for k in _STAGE_KEYS})
    out = _lib.ReplicaOut(**{k: _lib.ptr(v) for k, v in bufs.items()})
    rc = _lib.lib.vp_run_replica(P, N, *[_lib.ptr(a) for a in ins], int(bool(opportunistic)),
                                 int(bool(serialize_links)), out)
    if rc == _lib.VP_ERR_DEADLOCK:
        raise RuntimeError("replica simulation deadlocked")
    _lib.check(rc, "run_replica")
    res = {k: bufs[k][:out.n_tasks] for k in _OUT_KEYS[:5]}
    res.update({k: bufs[k][:out.n_msgs] for k in _OUT_KEYS[5:]})
    res.update({k: bufs[k] for k in _STAGE_KEYS})
    res["makespan"] = int(out.makespan)
    return res
