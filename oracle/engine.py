"""Oracle: the replica event kernel (opportunistic Varuna runtime policy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). A plain-Python
restatement of sp/engine/py_kernel.py:41-360 (≡ sp/engine/_kernel.pyx:
334-567), pinned bit-exactly against tests/golden/engine_cases.json, which
the reference kernel produced. The product's C++ twin is
``vp_run_replica`` in paper_2111_04007_b200/csrc/engine.cpp.
"""

from __future__ import annotations

import heapq

import numpy as np

B, R, F = 0, 1, 2
FAR = 1 << 60


class _Replica:
    def __init__(self, P, N, kinds, mbs, offsets, fwd, bwd, rec, act_tx, grad_tx,
                 exp_grad, in_act, work, cap, opportunistic, serialize):
        self.P, self.N = P, N
        self.kinds = [int(x) for x in kinds]
        self.mbs = [int(x) for x in mbs]
        self.off = [int(x) for x in offsets]
        self.dur = {F: [int(x) for x in fwd], B: [int(x) for x in bwd], R: [int(x) for x in rec]}
        self.act_tx = [int(x) for x in act_tx]
        self.grad_tx = [int(x) for x in grad_tx]
        self.exp_grad = [int(x) for x in exp_grad]
        self.in_act = [int(x) for x in in_act]
        self.work = [int(x) for x in work]
        self.cap = [int(x) for x in cap]
        self.opp = bool(opportunistic)
        self.serialize = bool(serialize)
        n_tasks = self.off[P]
        self.done_pos = [False] * n_tasks
        self.head = self.off[:P]
        self.head = list(self.head)
        self.run = [None] * P          # (kind, mb) or None
        self.until = [0] * P
        self.lock = [-1] * P
        self.prev_kind = [-1] * P
        self.n_f = [0] * P
        self.n_b = [0] * P
        # Per-stage indices into the task list (sp/engine/py_kernel.py:94-113).
        self.f_at = [[-1] * N for _ in range(P)]
        self.b_at = [[-1] * N for _ in range(P)]
        self.b_mb = [[-1] * N for _ in range(P)]
        self.r_at = [[-1] * N for _ in range(P)]
        for k in range(P):
            cf = cb = 0
            for pos in range(self.off[k], self.off[k + 1]):
                kd, mb = self.kinds[pos], self.mbs[pos]
                if kd == F:
                    self.f_at[k][cf] = pos
                    cf += 1
                elif kd == B:
                    self.b_at[k][cb] = pos
                    self.b_mb[k][cb] = mb
                    cb += 1
                else:
                    self.r_at[k][mb] = pos
        self.act_at = [[0] * N if k == 0 else [-1] * N for k in range(P)]
        self.grad_at = [[-1] * N for _ in range(P)]
        self.jit = [[-1] * N for _ in range(P)]
        self.link_free = ([0] * max(P - 1, 1), [0] * max(P - 1, 1))
        self.stash = [0] * P
        self.sets = [0] * P
        self.peak_stash = [0] * P
        self.peak_sets = [0] * P
        self.peak_mem = [0] * P
        self.last_bwd_end = [0] * P
        self.tasks = []   # (stage, kind, mb, start, end)
        self.msgs = []    # (send, grant, arrive, boundary, dir, mb)
        self.q = [(0, k) for k in range(P)]
        heapq.heapify(self.q)

    # -- memory accounting (sp/engine/py_kernel.py:156-173) ---------------
    def _account(self, k):
        self.peak_stash[k] = max(self.peak_stash[k], self.stash[k])
        self.peak_sets[k] = max(self.peak_sets[k], self.sets[k])
        mem = self.stash[k] * self.in_act[k] + self.sets[k] * self.work[k]
        self.peak_mem[k] = max(self.peak_mem[k], mem)

    def start(self, k, pos, now):
        """sp/engine/py_kernel.py:136-182."""
        kind, mb = self.kinds[pos], self.mbs[pos]
        d = self.dur[kind][k]
        self.done_pos[pos] = True
        self.run[k] = (kind, mb)
        self.until[k] = now + d
        self.tasks.append((k, kind, mb, now, now + d))
        if kind == F:
            self.n_f[k] += 1
            self.stash[k] += 1
            self.sets[k] += 1
            self._account(k)
        elif kind == R:
            self.sets[k] += 1
            self._account(k)
        else:
            self.lock[k] = -1
            if k > 0:
                due = now + d + self.exp_grad[k - 1] - self.dur[R][k - 1]
                self.jit[k - 1][mb] = due
                heapq.heappush(self.q, (max(due, now), k - 1))
        heapq.heappush(self.q, (now + d, k))

    def send(self, boundary, direction, mb, now):
        """sp/engine/py_kernel.py:184-214: one message per directed link at a
        time when links are serialized."""
        tx = (self.act_tx if direction == 0 else self.grad_tx)[boundary * self.N + mb]
        free = self.link_free[direction]
        if self.serialize:
            grant = max(now, free[boundary])
            free[boundary] = grant + tx
        else:
            grant = now
        arrive = grant + tx
        self.msgs.append((now, grant, arrive, boundary, direction, mb))
        if direction == 0:
            self.act_at[boundary + 1][mb] = arrive
            heapq.heappush(self.q, (arrive, boundary + 1))
        else:
            self.grad_at[boundary][mb] = arrive
            heapq.heappush(self.q, (arrive, boundary))
            heapq.heappush(self.q, (max(arrive - self.dur[R][boundary], now), boundary))

    def complete(self, k, now):
        """sp/engine/py_kernel.py:216-234."""
        kind, mb = self.run[k]
        self.run[k] = None
        self.prev_kind[k] = kind
        if kind == F:
            if k < self.P - 1:
                self.sets[k] -= 1
                self.send(k, 0, mb, now)
        elif kind == R:
            self.lock[k] = mb
        else:
            self.sets[k] -= 1
            self.stash[k] -= 1
            self.n_b[k] += 1
            self.last_bwd_end[k] = now
            if k > 0:
                self.send(k - 1, 1, mb, now)

    def rec_due(self, k, mb, now):
        """sp/engine/py_kernel.py:238-248."""
        g = self.grad_at[k][mb]
        if g >= 0:
            return now if g <= now else g - self.dur[R][k]
        d = self.jit[k][mb]
        return d if d >= 0 else FAR

    def decide(self, k, now):
        """The runtime policy, sp/engine/py_kernel.py:250-322."""
        if self.run[k] is not None:
            return
        last = k == self.P - 1
        if self.lock[k] >= 0:
            if last or 0 <= self.grad_at[k][self.lock[k]] <= now:
                self.start(k, self.b_at[k][self.n_b[k]], now)
            return
        pos = self.head[k]
        while pos < self.off[k + 1] and self.done_pos[pos]:
            pos += 1
        self.head[k] = pos
        if pos >= self.off[k + 1]:
            return
        kind, mb = self.kinds[pos], self.mbs[pos]
        if kind == B:
            if last or 0 <= self.grad_at[k][mb] <= now:
                self.start(k, pos, now)
            return
        if kind == F:
            full = self.opp and self.stash[k] >= self.cap[k]
            if not full and 0 <= self.act_at[k][mb] <= now:
                self.start(k, pos, now)
                return
            if not self.opp:
                return
            c = self.n_b[k]
            if c < self.N and not last:
                jb = self.b_mb[k][c]
                rp = self.r_at[k][jb]
                if rp >= 0 and not self.done_pos[rp] and self.n_f[k] > jb \
                        and now >= self.rec_due(k, jb, now):
                    self.start(k, rp, now)
            return
        # Recompute at the head of the list.
        if not self.opp or last:
            self.start(k, pos, now)
            return
        f = self.n_f[k]
        f_ready = f < self.N and 0 <= self.act_at[k][f] <= now and self.stash[k] < self.cap[k]
        if 0 <= self.grad_at[k][mb] <= now:
            if f_ready and self.prev_kind[k] == B:
                self.start(k, self.f_at[k][f], now)
            else:
                self.start(k, pos, now)
            return
        due = self.rec_due(k, mb, now)
        if now >= due:
            self.start(k, pos, now)
            return
        if f_ready:
            if now + self.dur[F][k] <= due:
                self.start(k, self.f_at[k][f], now)
            return
        self.start(k, pos, now)

    def loop(self):
        """sp/engine/py_kernel.py:324-340: drain every event at the current
        instant (including zero-delay messages pushed while draining), then
        let each touched stage decide in index order."""
        q = self.q
        while q:
            now = q[0][0]
            touched = set()
            while q and q[0][0] == now:
                _, k = heapq.heappop(q)
                if self.run[k] is not None and self.until[k] == now:
                    self.complete(k, now)
                touched.add(k)
            for k in sorted(touched):
                self.decide(k, now)
        for k in range(self.P):
            if self.n_b[k] != self.N:
                raise RuntimeError(
                    f"replica simulation deadlocked: stage {k} completed "
                    f"{self.n_b[k]}/{self.N} backwards")

    def result(self):
        i64 = lambda xs: np.array(xs, dtype=np.int64).reshape(-1)  # noqa: E731
        t = list(zip(*self.tasks)) if self.tasks else [[]] * 5
        m = list(zip(*self.msgs)) if self.msgs else [[]] * 6
        return {
            "task_stage": i64(t[0]), "task_kind": i64(t[1]), "task_mb": i64(t[2]),
            "task_start": i64(t[3]), "task_end": i64(t[4]),
            "msg_send": i64(m[0]), "msg_grant": i64(m[1]), "msg_arrive": i64(m[2]),
            "msg_boundary": i64(m[3]), "msg_dir": i64(m[4]), "msg_mb": i64(m[5]),
            "last_bwd_end": i64(self.last_bwd_end), "peak_stash": i64(self.peak_stash),
            "peak_sets": i64(self.peak_sets), "peak_mem": i64(self.peak_mem),
            "makespan": max((x[4] for x in self.tasks), default=0),
        }


def run_replica(n_stages, n_micro, kinds, mbs, offsets, fwd_us, bwd_us, rec_us,
                act_tx_us, grad_tx_us, exp_grad_tx_us, in_act_bytes, work_bytes,
                stash_cap, opportunistic, serialize_links):
    """Same 16-argument contract as sp/engine/_kernel.pyx:334-351."""
    rep = _Replica(int(n_stages), int(n_micro), kinds, mbs, offsets, fwd_us, bwd_us, rec_us,
                   act_tx_us, grad_tx_us, exp_grad_tx_us, in_act_bytes, work_bytes,
                   stash_cap, opportunistic, serialize_links)
    rep.loop()
    return rep.result()
