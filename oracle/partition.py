"""Oracle: cut-point identification and stage grouping DPs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Plain-Python restatements
of sp/partitioner.py:109-246 (identify_cutpoints), :269-374 (assign_stages)
and :404-436 (memory_check); pinned against tests/golden/partition.json.
"""

from __future__ import annotations

import math

INF = float("inf")


def _best_split(n_items, parts, seg, last_cost=None):
    """Min over contiguous ``parts``-way splits of the max segment cost.
    ``table[j][i]`` = best for items i.. split into j parts. Early exit when
    the leading segment alone already exceeds the best (segments grow)."""
    last_cost = last_cost or (lambda i: seg(i, n_items - 1))
    table = [[INF] * (n_items + 1) for _ in range(parts + 1)]
    for i in range(n_items):
        table[1][i] = last_cost(i)
    for j in range(2, parts + 1):
        for i in range(n_items):
            best = INF
            for e in range(i, n_items - 1):
                head = seg(i, e)
                if head >= best:
                    break
                best = min(best, max(head, table[j - 1][e + 1]))
            table[j][i] = best
    return table


def assign_stages(forward_us, acts, params, in_bytes0, P, last_stage_weight=1.0):
    """sp/partitioner.py:269-374. ``forward_us[i]`` = F_i(m); returns a dict
    with the same fields as the reference ``StageAssignment``.
    ``in_bytes0`` is the model's stage-0 input bytes per example (None =
    first boundary activation, sp/core.py:84-90)."""
    K = len(forward_us)
    if P > K:
        raise OverflowError("P exceeds K")
    pre = [0]
    for t in forward_us:
        pre.append(pre[-1] + t)

    def seg(i, j):
        return pre[j + 1] - pre[i]

    def last_cost(i):
        return last_stage_weight * seg(i, K - 1)

    best = _best_split(K, P, seg, last_cost)[P][0]
    # Phase 2: minimum total boundary activation among splits whose
    # non-final segments stay <= best and final segment cost <= best.
    act_tab = [[INF] * (K + 1) for _ in range(P + 1)]
    for i in range(K):
        if last_cost(i) <= best:
            act_tab[1][i] = 0
    for j in range(2, P + 1):
        for i in range(K):
            cand = INF
            for e in range(i, K - 1):
                if seg(i, e) > best:
                    break
                rest = act_tab[j - 1][e + 1]
                if rest < INF:
                    cand = min(cand, acts[e] + rest)
            act_tab[j][i] = cand
    ends = []
    i = 0
    for j in range(P, 1, -1):
        want = act_tab[j][i]
        for e in range(i, K - 1):
            if seg(i, e) > best:
                break
            rest = act_tab[j - 1][e + 1]
            if rest < INF and acts[e] + rest == want:
                ends.append(e)
                i = e + 1
                break
    ends.append(K - 1)
    stage_map, sp, sf, sin, swork, sbound = [], [], [], [], [], []
    lo = 0
    for s, e in enumerate(ends):
        stage_map += [s] * (e - lo + 1)
        sp.append(sum(params[lo:e + 1]))
        sf.append(seg(lo, e))
        if lo == 0:
            sin.append(acts[0] if in_bytes0 is None else in_bytes0)
        else:
            sin.append(acts[lo - 1])
        swork.append(sum(acts[lo:e + 1]))
        sbound.append(acts[e])
        lo = e + 1
    return {"stage_map": stage_map, "boundaries": ends, "stage_parameters": sp,
            "stage_forward_us": sf, "stage_input_activation_bytes": sin,
            "stage_working_activation_bytes": swork, "stage_boundary_activation_bytes": sbound}


def identify_cutpoints(ops, shared_groups, K, tolerance=0.2):
    """sp/partitioner.py:109-246. ``ops`` = list of dicts with compute_us,
    activation_bytes, parameters, param_groups."""
    n = len(ops)
    if K < 1:
        raise ValueError("K < 1")
    if K > n:
        raise OverflowError("K > n")
    after = [set() for _ in range(n + 1)]
    for i in range(n - 1, -1, -1):
        after[i] = after[i + 1] | set(ops[i]["param_groups"])
    spans, before = [], set()
    for b in range(n - 1):
        before |= set(ops[b]["param_groups"])
        spans.append(before & after[b + 1])
    ok = [all(g in shared_groups for g in spans[b]) for b in range(n - 1)]
    pre = [0]
    for o in ops:
        pre.append(pre[-1] + o["compute_us"])

    def seg(i, j):
        return pre[j + 1] - pre[i]

    mm = [[INF] * (n + 1) for _ in range(K + 1)]
    for i in range(n):
        mm[1][i] = seg(i, n - 1)
    for j in range(2, K + 1):
        for i in range(n):
            best = INF
            for e in range(i, n - 1):
                if not ok[e]:
                    continue
                head = seg(i, e)
                if head >= best:
                    break
                best = min(best, max(head, mm[j - 1][e + 1]))
            mm[j][i] = best
    if mm[K][0] == INF:
        raise OverflowError("no breakable partition")
    cap = max(int(mm[K][0]), math.ceil((1.0 + tolerance) * pre[n] / K))
    acts = [o["activation_bytes"] for o in ops]
    at = [[INF] * (n + 1) for _ in range(K + 1)]
    for i in range(n):
        if seg(i, n - 1) <= cap:
            at[1][i] = 0
    for j in range(2, K + 1):
        for i in range(n):
            best = INF
            for e in range(i, n - 1):
                if seg(i, e) > cap:
                    break
                if ok[e] and at[j - 1][e + 1] < INF:
                    best = min(best, acts[e] + at[j - 1][e + 1])
            at[j][i] = best
    if at[K][0] == INF:
        raise OverflowError("no partition fits the window")
    ends, i = [], 0
    for j in range(K, 1, -1):
        for e in range(i, n - 1):
            if seg(i, e) > cap:
                break
            if ok[e] and at[j - 1][e + 1] < INF and acts[e] + at[j - 1][e + 1] == at[j][i]:
                ends.append(e)
                i = e + 1
                break
    ends.append(n - 1)
    params, bacts, secs = [], [], []
    lo = 0
    for e in ends:
        params.append(max(sum(o["parameters"] for o in ops[lo:e + 1]), 1))
        bacts.append(max(ops[e]["activation_bytes"], 1))
        secs.append(seg(lo, e))
        lo = e + 1
    crossings = [[g, e] for e in ends[:-1] for g in sorted(spans[e])]
    return {"boundaries": ends, "shared_crossings": crossings, "section_compute_us": secs,
            "max_section_us": max(secs), "total_boundary_activation": sum(acts[e] for e in ends[:-1]),
            "cutpoint_parameters": params, "cutpoint_activation_bytes": bacts}


def memory_check(stage_params, stage_in_act, stage_work, m, n_m, gpu_bytes,
                 bounds=None, bytes_per_param=16):
    """sp/partitioner.py:404-436."""
    out = []
    for s in range(len(stage_params)):
        bound = n_m if bounds is None else min(n_m, bounds[s])
        p = bytes_per_param * stage_params[s]
        st = bound * m * stage_in_act[s]
        w = m * stage_work[s]
        out.append({"parameter_state_bytes": p, "stashed_activation_bytes": st,
                    "working_activation_bytes": w, "feasible": p + st + w <= gpu_bytes})
    return out
