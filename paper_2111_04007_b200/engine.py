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
    a = np.asarray(a, dtype=np.int64).ravel()
    return a if a.size else np.zeros(1, dtype=np.int64)


def run_replica(n_stages, n_micro, kinds, mbs, offsets, fwd_us, bwd_us, rec_us, act_tx_us,
                grad_tx_us, exp_grad_tx_us, in_act_bytes, work_bytes, stash_cap,
                opportunistic, serialize_links) -> dict:
    P, N = int(n_stages), int(n_micro)
    ins = [_i64(x) for x in (kinds, mbs, offsets, fwd_us, bwd_us, rec_us, act_tx_us, grad_tx_us,
                             exp_grad_tx_us, in_act_bytes, work_bytes, stash_cap)]
    if ins[2].size < P + 1:
        raise ValueError("offsets must have P+1 entries")
    # one packed input block and one output block: two address lookups per
    # call instead of 27 (the ctypes marshalling dominated small replicas)
    packed = np.concatenate(ins)
    base_in = _lib.ptr(packed)
    in_ptrs, off = [], 0
    for a in ins:
        in_ptrs.append(base_in + 8 * off)
        off += a.size
    n_tasks = int(ins[2][P])
    n_msgs = max(2 * (P - 1) * N, 1)
    T = max(n_tasks, 1)
    sizes = [T] * 5 + [n_msgs] * 6 + [P] * 4
    block = np.empty(sum(sizes), dtype=np.int64)
    base_out = _lib.ptr(block)
    views, addrs, off = [], [], 0
    for n in sizes:
        views.append(block[off:off + n])
        addrs.append(base_out + 8 * off)
        off += n
    out = _lib.ReplicaOut(*addrs)
    rc = _lib.lib.vp_run_replica(P, N, *in_ptrs, int(bool(opportunistic)),
                                 int(bool(serialize_links)), out)
    if rc == _lib.VP_ERR_DEADLOCK:
        raise RuntimeError("replica simulation deadlocked")
    _lib.check(rc, "run_replica")
    nt, nm = out.n_tasks, out.n_msgs
    res = {k: v[:nt] for k, v in zip(_OUT_KEYS[:5], views[:5])}
    res.update({k: v[:nm] for k, v in zip(_OUT_KEYS[5:], views[5:11])})
    res.update(zip(_STAGE_KEYS, views[11:]))
    res["makespan"] = int(out.makespan)
    return res
