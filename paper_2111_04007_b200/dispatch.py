"""On-line per-stage dispatch: the reference's opportunistic replica policy
(``decide``, sp/engine/py_kernel.py:250-322; compiled twin
sp/engine/_kernel.pyx:244-331) restated for ONE stage that only sees its own
state and the messages that reached it, so the executor can run it live,
against real arrivals, instead of replaying a simulated order.

The stage's state machine is the reference's: the static Varuna list is the
plan; rule 2 locks the stage after R(j) until B(j) runs (:253-259); a B at
the list head waits for its gradient (:269-272); a forward runs when its
activation has arrived and the stash is under its cap (:273-279), otherwise
a due R/B pair may jump ahead (:282-291); an R at the head waits for its
just-in-time start — gradient arrival minus T_r when the gradient is known,
else the deadline announced when the downstream B started (:176-181,
240-248) — filling with forwards that fit in front of it (:294-322), and a
backlog of arrived gradients is paced with one ready forward per R/B pair
(:301-310). ``start``/``complete`` mirror start_task/complete (:136-173,
216-234) for this stage's bookkeeping.

Times are in the caller's unit (the executor uses microseconds of
CLOCK_MONOTONIC, shared by the processes of one box). Arrival callbacks
return -1 when the message is not known yet, else its (possibly future)
arrival time; ``deadline(mb)`` returns -1 or the R(mb) start deadline.
``tests/test_dispatch_policy.py`` drives P of these with the reference
engine's event loop and checks the executed order and times equal the
compiled replica kernel's bit for bit.
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

from .core import KIND_BACKWARD as B
from .core import KIND_FORWARD as F
from .core import KIND_RECOMPUTE as R

_FAR = 1 << 60


class StagePolicy:
    """Opportunistic (or static, ``opportunistic=False``) dispatch of one
    stage's task list."""

    def __init__(self, tasks: Sequence[Tuple[int, int]], n_micro: int, last: bool,
                 stash_cap: int, opportunistic: bool = True):
        self.kinds = [k for k, _ in tasks]
        self.mbs = [j for _, j in tasks]
        self.N, self.last = n_micro, last
        self.cap, self.opp = stash_cap, opportunistic
        self.executed = [False] * len(tasks)
        self.ptr = 0
        self.locked = -1
        self.last_done = -1
        self.fwd_exec = self.bwd_exec = 0
        self.stash = 0
        self.fwd_pos = [-1] * n_micro
        self.rec_pos = [-1] * n_micro
        self.bwd_pos: List[int] = []
        self.bwd_mb: List[int] = []
        nf = 0
        for pos, (kind, mb) in enumerate(tasks):
            if kind == F:
                self.fwd_pos[nf] = pos
                nf += 1
            elif kind == B:
                self.bwd_pos.append(pos)
                self.bwd_mb.append(mb)
            else:
                self.rec_pos[mb] = pos

    @property
    def done(self) -> bool:
        return self.bwd_exec == self.N

    # -------------------------------------------------------- bookkeeping
    def start(self, pos: int) -> None:
        kind = self.kinds[pos]
        self.executed[pos] = True
        if kind == F:
            self.fwd_exec += 1
            self.stash += 1
        elif kind == B:
            self.locked = -1

    def complete(self, pos: int) -> None:
        kind, mb = self.kinds[pos], self.mbs[pos]
        self.last_done = kind
        if kind == R:
            self.locked = mb
        elif kind == B:
            self.stash -= 1
            self.bwd_exec += 1

    # ----------------------------------------------------------- decision
    def _rec_due_at(self, mb, now, grad_arr, deadline, t_rec) -> int:
        g = grad_arr(mb)
        if g >= 0:
            return now if g <= now else g - t_rec
        dl = deadline(mb)
        return dl if dl >= 0 else _FAR

    def decide(self, now, act_arr: Callable[[int], int], grad_arr: Callable[[int], int],
               deadline: Callable[[int], int], t_fwd, t_rec) -> Optional[int]:
        """Position of the task to start now (the stage is idle), or None."""
        j = self.locked
        if j >= 0:   # rule 2: only the matching backward may run next
            if self.last or 0 <= grad_arr(j) <= now:
                return self.bwd_pos[self.bwd_exec]
            return None
        p = self.ptr
        end = len(self.kinds)
        while p < end and self.executed[p]:
            p += 1
        self.ptr = p
        if p >= end:
            return None
        kind, mb = self.kinds[p], self.mbs[p]
        if kind == B:
            return p if (self.last or 0 <= grad_arr(mb) <= now) else None
        if kind == F:
            capped = self.opp and self.stash >= self.cap
            if not capped and 0 <= act_arr(mb) <= now:
                return p
            if not self.opp:
                return None
            c = self.bwd_exec
            if c < self.N and not self.last:
                jb = self.bwd_mb[c]
                rp = self.rec_pos[jb]
                if rp >= 0 and not self.executed[rp] and self.fwd_exec > jb:
                    if now >= self._rec_due_at(jb, now, grad_arr, deadline, t_rec):
                        return rp
            return None
        # recompute at the head
        if not self.opp or self.last:
            return p
        f = self.fwd_exec
        f_ready = f < self.N and 0 <= act_arr(f) <= now and self.stash < self.cap
        g = grad_arr(mb)
        if 0 <= g <= now:
            if f_ready and self.last_done == B:
                return self.fwd_pos[f]
            return p
        due_at = self._rec_due_at(mb, now, grad_arr, deadline, t_rec)
        if now >= due_at:
            return p
        if f_ready:
            if now + t_fwd <= due_at:
                return self.fwd_pos[f]
            return None
        return p
