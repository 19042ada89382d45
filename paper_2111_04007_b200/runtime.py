"""The Varuna executor: ``Varuna`` wrapper, ``CutPoint`` markers, ``step()``.

One process per GPU. Rank = r·P + s — the reference placement (stage s of
replica r on slot r·P + s, sp/simulator.py:58-81). Each rank instantiates
only the layers ``ParallelConfig.stage_map`` gives its stage (the CutPoint
→ stage assignment computed by ``assign_stages``, sp/partitioner.py:269-374)
and walks its slice of the Varuna plan (``generate_varuna_schedule(P, N_m,
1, 2, 1)``, sp/scheduler.py:128-145; always (1,2,1): sp/planner.py:204-208):

* F(j): stage forward WITHOUT saving intermediates (k < P-1); the last
  layer's FC2 epilogue writes the stage output straight into stage k+1's
  activation ring slot j over NVLink (IPC-mapped peer memory), then an
  interprocess event is recorded that stage k+1's stream waits on.
* R(j): the same forward from the stashed input (the received ring slot),
  this time saving the working set (Varuna's recompute; bitwise ≡ F).
* B(j): backward from the gradient ring slot j; the input gradient is put
  into stage k-1's gradient ring slot j by an SM copy kernel over NVLink.
* the last stage runs F(j) with saving and B(j) right after (no R).

End of mini-batch (per stage, as soon as its last B is done —
allreduce_barrier=False, sp/simulator.py:334-342): NCCL allreduce of the
flat fp32 gradient over the stage's DP group (C1), tied-embedding gradient
allreduce between stage 0 and P-1 (C3), a pipeline-wide (grad-norm²,
non-finite count) allreduce (C2), then one fused unscale + overflow-skip +
clip + AdamW kernel over the stage's flat parameters.

Host↔host ordering uses per-slot sequence counters in POSIX shared memory
(all ranks of one box); device ordering uses the IPC events only — no host
synchronisation on the data path.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from multiprocessing import shared_memory
from typing import Dict, List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from ._lib import check
from .core import KIND_BACKWARD, KIND_FORWARD, KIND_RECOMPUTE, ConfigError, ParallelConfig
from .model import GPT2Config, GPT2Stage, StageSpec
from .scheduler import Schedule, generate_varuna_schedule
from .simulator import bubble_fraction

F, R, B = KIND_FORWARD, KIND_RECOMPUTE, KIND_BACKWARD


from .modules import GPT2 as GPT2Module  # noqa: E402  (drop-in model structure)
from .modules import CutPoint  # noqa: E402,F401


@dataclass(frozen=True)
class AdamWConfig:
    lr: float = 1e-4
    betas: tuple = (0.9, 0.999)
    eps: float = 1e-8
    weight_decay: float = 0.01
    max_grad_norm: float = 1.0


@dataclass
class LossScaler:
    """Loss scaling for mixed precision. ``dynamic``: the apex / Megatron
    schedule (start at ``init``, x``backoff`` on overflow — the step is
    skipped on every rank, the overflow decision being global, PAPER.md:547 —
    x``growth`` after ``window`` clean steps); otherwise a static ``init``.
    The state lives on the device (vp_loss_scaler_update), so no step ever
    waits on the host for it."""

    init: float = 1.0
    dynamic: bool = False
    growth: float = 2.0
    backoff: float = 0.5
    window: int = 2000
    min_scale: float = 1.0

    @classmethod
    def of(cls, x) -> "LossScaler":
        if isinstance(x, LossScaler):
            return x
        if x == "dynamic":
            return cls(init=2.0 ** 16, dynamic=True)
        return cls(init=float(x))


@dataclass
class StepResult:
    """Loss is only known on last-stage ranks (None elsewhere). ``_scale``:
    device copy of the loss scale this step ran with."""

    _loss: Optional[torch.Tensor]
    _flags: torch.Tensor
    _scale: Optional[torch.Tensor]
    timeline: Optional[dict] = None

    @property
    def loss_scale(self) -> float:
        return 1.0 if self._scale is None else float(self._scale.item())

    @property
    def loss(self) -> Optional[float]:
        """Mean loss over the mini-batch's M_total samples (the device sum
        carries the loss scale; it is removed here)."""
        return None if self._loss is None else float(self._loss.item()) / self.loss_scale

    @property
    def overflow(self) -> bool:
        return bool(self._flags[1].item() != 0)

    @property
    def grad_norm(self) -> float:
        return math.sqrt(max(float(self._flags[0].item()), 0.0)) / self.loss_scale


_M64 = (1 << 64) - 1


def task_seed(seed: int, step: int, mb: int) -> int:
    """64-bit dropout seed of micro-batch ``mb`` (global index r*N_m + j, so
    DP replicas draw different masks) in training step ``step``: F(j), R(j)
    and B(j) of one step share it, so recompute regenerates the forward's
    masks. splitmix64 of a linear combination; restated in
    oracle/gpt2_fp32.py."""
    x = (seed * 0x9E3779B97F4A7C15 + step * 0xD1B54A32D192ED03 + mb * 0xBF58476D1CE4E5B9 + 1) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def synthetic_batch(cfg: GPT2Config, rows: int, replica: int, step: int = 0, seed: int = 1234):
    """Deterministic token rows for one replica: global row g = replica·rows + i
    (DP replicas partition M_total). GPT-2: labels are inputs shifted by one.
    BERT: two segments (token types 0 | 1), exactly ``mlm_per_seq`` masked
    positions per row with random targets, -100 elsewhere."""
    g = torch.Generator()
    g.manual_seed(seed + 7919 * replica + 104729 * step)
    if cfg.arch == "bert":
        S = cfg.seq_len
        ids = torch.randint(0, cfg.vocab_size, (rows, S), generator=g)
        types = torch.zeros(rows, S, dtype=torch.int64)
        types[:, S // 2:] = 1
        labels = torch.full((rows, S), -100, dtype=torch.int64)
        pos = torch.argsort(torch.rand(rows, S, generator=g), dim=1)[:, :cfg.mlm_per_seq]
        tgt = torch.randint(0, cfg.vocab_size, (rows, cfg.mlm_per_seq), generator=g)
        labels.scatter_(1, pos, tgt)
        return {"input_ids": ids, "token_type_ids": types, "labels": labels}
    toks = torch.randint(0, cfg.vocab_size, (rows, cfg.seq_len + 1), generator=g)
    return {"input_ids": toks[:, :-1].contiguous(), "labels": toks[:, 1:].contiguous()}


class _Shm:
    """Per-(rank, channel, slot) int64 sequence counters in POSIX shared
    memory, shared by the processes of one box. Channels: data posted by a
    ring's producer (ACT, GRAD) and credits posted by its consumer
    (FREE_ACT, FREE_GRAD)."""

    CHANNELS = 6   # ACT, GRAD data; FREE_ACT, FREE_GRAD credits; DL_SEQ, DL_TIME (live dispatch)

    def __init__(self, name: str, world: int, slots: int, create: bool):
        self.shape = (world, self.CHANNELS, slots)
        nbytes = 8 * world * self.CHANNELS * slots
        if create:
            try:
                old = shared_memory.SharedMemory(name=name)
                old.close()
                old.unlink()
            except FileNotFoundError:
                pass
            self.shm = shared_memory.SharedMemory(name=name, create=True, size=nbytes)
            np.ndarray(self.shape, dtype=np.int64, buffer=self.shm.buf)[:] = 0
        else:
            self.shm = shared_memory.SharedMemory(name=name)
            try:  # the creator owns unlinking; keep the tracker out of it
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:  # noqa: BLE001
                pass
        self.arr = np.ndarray(self.shape, dtype=np.int64, buffer=self.shm.buf)
        self.owner = create

    def post(self, rank, channel, slot, seq):
        self.arr[rank, channel, slot] = seq

    def ready(self, rank, channel, slot, seq) -> bool:
        return self.arr[rank, channel, slot] >= seq

    def wait(self, rank, channel, slot, seq, timeout=600.0):
        a = self.arr
        if a[rank, channel, slot] >= seq:
            return
        t0 = time.monotonic()
        while a[rank, channel, slot] < seq:
            if time.monotonic() - t0 > timeout:
                raise TimeoutError(f"p2p handshake timed out (peer {rank}, channel {channel}, "
                                   f"slot {slot}, seq {seq})")
            time.sleep(20e-6)

    def close(self):
        self.shm.close()
        if self.owner:
            try:
                self.shm.unlink()
            except FileNotFoundError:
                pass


def in_flight(order) -> int:
    """Largest number of forwards a stage has issued whose backward it has
    not yet started, over its task order (max prefix #F - #B; the
    reference's Schedule.in_flight_bound, sp/scheduler.py:88-97, taken on
    the order actually dispatched)."""
    cur = best = 0
    for kind, _ in order:
        if kind == F:
            cur += 1
            best = max(best, cur)
        elif kind == B:
            cur -= 1
    return best


# Ring slots beyond the producer's in-flight bound (the reference pads the
# opportunistic stash the same way, DEFAULT_STASH_PAD, sp/simulator.py:
# 256, 309-312), and gradient-ring credits: a stage consumes gradients in
# ascending micro-batch order right after they land (rule 1 JIT recompute).
RING_PAD = 2
GRAD_SLOTS = 4


def ring_slots(orders, P: int, N: int):
    """(activation slots, gradient slots) of every stage's receive rings.
    Stage k >= 1 receives activations F(j) of stage k-1 and holds slot j
    until its own B(j); k-1 starts B(j) only after k's B(j) (the gradient
    dependency), so at most in_flight(order[k-1]) slots are live."""
    act = [0] + [min(N, in_flight(orders[k - 1]) + RING_PAD) for k in range(1, P)]
    grad = [min(N, GRAD_SLOTS) for _ in range(P - 1)] + [0]
    return act, grad


class _Links:
    """IPC-registered activation / gradient rings between adjacent stages of
    one replica, BOUNDED: the receiver's activation ring has in_flight(
    upstream order) + RING_PAD slots, its gradient ring GRAD_SLOTS, not one
    per micro-batch (8.3B at N_m = 1024 would need 24 GiB per ring).

    Micro-batch g (a global counter, (step-1)*N + j + 1) uses slot g mod n.
    Data: the producer writes the slot on its stream, records the slot's
    data event (IPC) and posts g (shm); the consumer waits for g on the host,
    then makes its stream wait on the event. Credits: when the consumer's
    last reader of the slot (B(j)) is enqueued it records the slot's free
    event and posts g; before writing g the producer waits for credit
    g - n on the host and on the device. No host synchronisation with the
    GPU on the data path."""

    ACT, GRAD = 0, 1
    FREE = 2   # channel offset of the credits

    def __init__(self, rank, stage, P, slots_act, slots_grad, slot_elems, gloo_group, shm,
                 epoch_g: int = 1):
        self.rank, self.stage, self.P = rank, stage, P
        self.epoch_g = epoch_g   # first micro-batch written through these rings
        self.slot_bytes = slot_elems * 2
        self.shm = shm
        up, down = rank - 1, rank + 1
        # direction -> (local ring, slots) I receive into
        self.rx, self.rx_n = {}, {}
        self.data_tx, self.free_tx = {}, {}   # events I record: data (I produce), free (I consume)
        mine = {"rank": rank}
        if stage > 0:        # receive activations from up, send gradients to up
            self.rx_n[self.ACT] = slots_act[stage]
            self.rx[self.ACT] = K.DeviceBuffer(slots_act[stage] * self.slot_bytes)
            mine["act_ring"] = self._mem_handle(self.rx[self.ACT].ptr)
            self.free_tx[self.ACT], mine["act_free"] = self._events(slots_act[stage])
            self.data_tx[self.GRAD], mine["grad_data"] = self._events(slots_grad[stage - 1])
        if stage < P - 1:    # receive gradients from down, send activations to down
            self.rx_n[self.GRAD] = slots_grad[stage]
            self.rx[self.GRAD] = K.DeviceBuffer(slots_grad[stage] * self.slot_bytes)
            mine["grad_ring"] = self._mem_handle(self.rx[self.GRAD].ptr)
            self.free_tx[self.GRAD], mine["grad_free"] = self._events(slots_grad[stage])
            self.data_tx[self.ACT], mine["act_data"] = self._events(slots_act[stage + 1])
        world = dist.get_world_size()
        allinfo = [None] * world
        dist.all_gather_object(allinfo, mine, group=gloo_group)
        self.peer_ring, self.tx_n = {}, {}   # direction -> mapped peer ring I write, its slots
        self.data_rx, self.free_rx = {}, {}  # opened peer events I wait on
        if stage > 0:
            info = allinfo[up]
            self.peer_ring[self.GRAD] = self._open_mem(info["grad_ring"])
            self.tx_n[self.GRAD] = slots_grad[stage - 1]
            self.data_rx[self.ACT] = [self._open_event(h) for h in info["act_data"]]
            self.free_rx[self.GRAD] = [self._open_event(h) for h in info["grad_free"]]
        if stage < P - 1:
            info = allinfo[down]
            self.peer_ring[self.ACT] = self._open_mem(info["act_ring"])
            self.tx_n[self.ACT] = slots_act[stage + 1]
            self.data_rx[self.GRAD] = [self._open_event(h) for h in info["grad_data"]]
            self.free_rx[self.ACT] = [self._open_event(h) for h in info["act_free"]]
        self.peer = {self.ACT: up, self.GRAD: down}   # producer of what I receive
        self.consumer = {self.ACT: down, self.GRAD: up}

    @property
    def ring_bytes(self) -> int:
        return sum(n * self.slot_bytes for n in self.rx_n.values())

    @staticmethod
    def _mem_handle(ptr):
        h = ctypes.create_string_buffer(64)
        check(K.L.vp_ipc_get_mem_handle(ptr, h), "vp_ipc_get_mem_handle")
        return h.raw

    @staticmethod
    def _open_mem(handle):
        p = ctypes.c_void_p()
        check(K.L.vp_ipc_open_mem_handle(handle, ctypes.byref(p)), "vp_ipc_open_mem_handle")
        return p.value

    @staticmethod
    def _events(n):
        evs, hs = [], []
        for _ in range(n):
            e = ctypes.c_void_p()
            h = ctypes.create_string_buffer(64)
            check(K.L.vp_ipc_event_create(ctypes.byref(e), h), "vp_ipc_event_create")
            evs.append(e.value)
            hs.append(h.raw)
        return evs, hs

    @staticmethod
    def _open_event(handle):
        e = ctypes.c_void_p()
        check(K.L.vp_ipc_event_open(handle, ctypes.byref(e)), "vp_ipc_event_open")
        return e.value

    def close(self):
        """Unmap the peer rings and destroy the IPC events (every rank of the
        job calls this before any rank frees its rings, Varuna.close)."""
        for ptr in self.peer_ring.values():
            check(K.L.vp_ipc_close_mem_handle(ptr), "vp_ipc_close_mem_handle")
        self.peer_ring = {}
        for d in (self.data_rx, self.free_rx, self.data_tx, self.free_tx):
            for evs in d.values():
                for e in evs:
                    check(K.L.vp_event_destroy(e), "vp_event_destroy")
            d.clear()

    def free_local(self):
        for buf in self.rx.values():
            buf.free()
        self.rx = {}

    # ---- receiver side
    def rx_slot(self, direction, g, shape):
        s = g % self.rx_n[direction]
        return self.rx[direction].tensor(shape, torch.bfloat16, s * self.slot_bytes)

    def arrived(self, direction, g) -> bool:
        """Host view: the producer has enqueued micro-batch g's write."""
        return self.shm.ready(self.peer[direction], direction, g % self.rx_n[direction], g)

    def landed(self, direction, g) -> bool:
        """Device view (after ``arrived``): the write has completed."""
        s = g % self.rx_n[direction]
        return K.L.vp_event_query(self.data_rx[direction][s]) == 0

    def wait(self, direction, g, stream):
        """Order ``stream`` after the producer's write of micro-batch g."""
        s = g % self.rx_n[direction]
        self.shm.wait(self.peer[direction], direction, s, g)
        check(K.L.vp_stream_wait_event(stream.cuda_stream, self.data_rx[direction][s]),
              "vp_stream_wait_event")

    def release(self, direction, g, stream):
        """After the last reader of micro-batch g's slot is enqueued on
        ``stream``: record the slot's free event and post the credit."""
        s = g % self.rx_n[direction]
        check(K.L.vp_event_record(self.free_tx[direction][s], stream.cuda_stream),
              "vp_event_record")
        self.shm.post(self.rank, self.FREE + direction, s, g)

    # ---- producer side
    def peer_slot_ptr(self, direction, g):
        return self.peer_ring[direction] + (g % self.tx_n[direction]) * self.slot_bytes

    def acquire(self, direction, g, stream):
        """Before writing micro-batch g into the peer ring: wait (host, then
        device) until the slot's previous occupant g - n was released."""
        n = self.tx_n[direction]
        if g - n < self.epoch_g:   # the slot has not been used by these rings yet
            return
        s = g % n
        self.shm.wait(self.consumer[direction], self.FREE + direction, s, g - n)
        check(K.L.vp_stream_wait_event(stream.cuda_stream, self.free_rx[direction][s]),
              "vp_stream_wait_event")

    def signal(self, direction, g, stream):
        """After the producing work on ``stream``: record the slot's data
        event, then publish g to the receiver's host."""
        s = g % self.tx_n[direction]
        check(K.L.vp_event_record(self.data_tx[direction][s], stream.cuda_stream),
              "vp_event_record")
        self.shm.post(self.rank, direction, s, g)


def group_ranks(P: int, D: int) -> Dict[str, List[List[int]]]:
    """Process groups of a P x D job under the reference placement
    rank = r*P + s (sp/simulator.py:71-76): ``dp[s]`` the D replicas of stage
    s (C1), ``pipe[r]`` the P stages of replica r (C2), ``tie[r]`` the first
    and last stage of replica r (C3, tied embedding; P > 1 only)."""
    return {"dp": [[r * P + s for r in range(D)] for s in range(P)],
            "pipe": [[r * P + s for s in range(P)] for r in range(D)],
            "tie": [[r * P, r * P + P - 1] for r in range(D)] if P > 1 else []}


def stage_means(timeline: dict):
    """Mean F, B, R duration (us) of one stage's traced step (0 if absent)."""
    by = {KIND_FORWARD: [], KIND_BACKWARD: [], KIND_RECOMPUTE: []}
    for kind, _, a, b in timeline["tasks"]:
        by[kind].append(b - a)
    return tuple(sum(v) / len(v) if v else 0.0
                 for v in (by[KIND_FORWARD], by[KIND_BACKWARD], by[KIND_RECOMPUTE]))


def exchange_stage_means(means, rank: int, world: int, device="cpu", group=None) -> torch.Tensor:
    """[world, 3] table of every rank's (F, B, R) means (one all-reduce)."""
    sums = torch.zeros(world, 3, dtype=torch.float64, device=device)
    sums[rank] = torch.tensor(means, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(sums, group=group)
    return sums


def retune_order(schedule: Schedule, P: int, D: int, m: int, N: int, hidden: int, seq_len: int,
                 table: torch.Tensor, current, max_in_flight: Optional[int] = None,
                 perturb: bool = False) -> list:
    """Pick the per-stage dispatch order with the shortest simulated
    mini-batch under the measured stage times (replica 0's rows of
    ``table``): candidates are the static Varuna order, the order in use
    (``current``, one task list per stage) and the reference's opportunistic
    replica kernel's order under the MEASURED times (the reference policy
    fed a B200-measured profile); ``perturb`` adds the
    kernel's orders with backward / recompute scaled x0.85..1.15 (the policy
    is a heuristic). Deterministic: every rank given the same table and
    current orders returns the same order."""
    from .calibration import CalibrationProfile, CutpointTimes
    from .core import make_block_model, uniform_cluster
    from .simulator import build_placement, execution_order, simulate_minibatch
    f = [max(1.0, float(table[s, 0])) for s in range(P)]     # replica 0: ranks 0..P-1
    bw = [max(1.0, float(table[s, 1])) for s in range(P)]
    rr = [float(table[s, 2]) / f[s] for s in range(P) if table[s, 2] > 0]
    rscale = sum(rr) / len(rr) if rr else 1.0
    z = {m: 0}
    d_grid = tuple(sorted({1, D}))

    def profile(fb):
        c = tuple(CutpointTimes({m: round(f[s])}, {m: max(1, round(bw[s] * fb))}, z, z, z, z, z,
                                z, {d: 0 for d in d_grid}) for s in range(P))
        return CalibrationProfile((m,), d_grid, c)
    prof = profile(1.0)
    pc = ParallelConfig(P, D, m, N, tuple(range(P)))
    model = make_block_model("stages", P, hidden, seq_len)
    cands = [[list(zip(*[a.tolist() for a in schedule.stage_slice(k)])) for k in range(P)],
             [list(t) for t in current]]
    scales = (1.0, 0.85, 1.15) if perturb else (1.0,)
    for fb in scales:
        for rs in scales:
            o = execution_order(schedule, pc, profile(fb), model, opportunistic=True,
                                recompute_scale=rscale * rs)
            if o not in cands:
                cands.append(o)
    place = build_placement(uniform_cluster(P * D, max(P * D, 1)), P, D)
    best, best_t = None, None
    for order in cands:
        if max_in_flight is not None and any(in_flight(o) > max_in_flight for o in order):
            continue   # would overrun the bounded activation rings
        kinds, mbs, offs = [], [], [0]
        for k in range(P):
            kinds += [a for a, _ in order[k]]
            mbs += [j for _, j in order[k]]
            offs.append(len(kinds))
        sch = Schedule("candidate", P, N, np.array(kinds, np.int64), np.array(mbs, np.int64),
                       np.array(offs, np.int64), 1, 2, 1)
        t = simulate_minibatch(sch, pc, prof, place, model, opportunistic=False,
                               recompute_scale=rscale).minibatch_us
        if best_t is None or t < best_t:
            best, best_t = order, t
    return best


@dataclass
class _StepCtx:
    g0: int                 # global micro-batch number of this step's j = 0
    data: dict
    scale: float
    ev: Optional[list]
    graphs: bool
    x_in: dict = field(default_factory=dict)
    executed: list = field(default_factory=list)


class Varuna:
    """Pipeline-parallel training of a GPT-2 described by ``model`` under the
    ``config`` (P, D, m, N_m, stage_map) chosen by the reference planner."""

    def __init__(self, model, config: ParallelConfig, *,
                 optimizer: AdamWConfig = AdamWConfig(), seed: int = 0, loss_scale: float = 1.0,
                 device=None, init_device: str = "cpu", trace: bool = False,
                 dispatch: str = "static", profile=None, graphs: Optional[bool] = None,
                 backend: Optional[str] = None, global_batch: Optional[int] = None):
        # ``model``: a GPT2Config (one CutPoint after every layer) or a model
        # structure with user-placed CutPoints (modules.GPT2): the stage map
        # then covers its CutPoint blocks and is expanded to layers here
        self.module = None
        if isinstance(model, GPT2Module):
            self.module = model
            config = ParallelConfig(config.pipeline_depth, config.data_parallel,
                                    config.micro_batch_size, config.num_micro_batches,
                                    model.layer_stage_map(config.stage_map))
            model = model.cfg
        if len(config.stage_map) != model.n_layer:
            raise ConfigError(f"stage_map covers {len(config.stage_map)} cut-points, model has "
                              f"{model.n_layer} (one CutPoint per transformer layer)")
        P, D = config.pipeline_depth, config.data_parallel
        self.cfg, self.pc, self.opt = model, config, optimizer
        self.P, self.D = P, D
        self.m, self.N = config.micro_batch_size, config.num_micro_batches
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(), dist.get_world_size()
        else:
            self.rank, self.world = 0, 1
        if self.world < P * D:
            raise ConfigError(f"world size {self.world} < P*D = {P * D}")
        # ranks >= P*D are spares (the planner may leave GPUs unused,
        # PlanResult.unused_gpus, sp/planner.py): they join the collective
        # setup and teardown but own no stage and run no tasks
        self.active = self.rank < P * D
        self.stage_id, self.replica = (self.rank % P, self.rank // P) if self.active else (-1, -1)
        # M_total (sp/planner.py:99-103): N_m = ceil(M/(m*D)); the last
        # micro-batches may be partial (padded rows carry ignored labels) and
        # the loss is the mean over M_total samples, not over the padded count
        cap = self.m * self.N * D
        self.global_batch = cap if global_batch is None else int(global_batch)
        if not (cap - self.m * D < self.global_batch <= cap):
            raise ConfigError(f"global_batch {self.global_batch} does not need N_m = {self.N} "
                              f"micro-batches of {self.m} on {D} replicas "
                              f"(ceil(M/(m*D)) = {-(-self.global_batch // (self.m * D))})")
        # collective backend of the DP / pipeline / tie groups: NCCL when each
        # rank has its own GPU (the product); gloo when several ranks share
        # one device (NCCL refuses duplicate GPUs). The data plane is the same.
        self.backend = backend
        self.scaler = LossScaler.of(loss_scale)
        self.loss_scale = loss_scale
        self.links = None
        self.shm = None
        self._graphs = {}
        self.step_count = 0
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        if not self.active:
            self.spec = self.stage = None
            self._setup_groups()
            if P > 1:   # the peer-handle exchange of _Links is collective
                dist.all_gather_object([None] * self.world, {"rank": self.rank}, group=self.gloo)
            return
        layers = tuple(i for i, s in enumerate(config.stage_map) if s == self.stage_id)
        if not layers:
            raise ConfigError(f"stage {self.stage_id} owns no cut-points")
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.Stream(self.device)
        self.spec = StageSpec(self.stage_id, P, layers)
        self.stage = GPT2Stage(model, self.spec, self.m, self.device, seed, init_device)
        self.schedule: Schedule = generate_varuna_schedule(P, self.N, 1.0, 2.0, 1.0)
        plan = [list(zip(*[a.tolist() for a in self.schedule.stage_slice(k)])) for k in range(P)]
        if dispatch in ("static", "live"):
            orders = plan
        elif dispatch == "opportunistic":
            orders = self._opportunistic_orders(profile)
        else:
            raise ConfigError(f"dispatch must be 'static', 'opportunistic' or 'live', "
                              f"not {dispatch!r}")
        self.tasks = list(orders[self.stage_id])
        self.dispatch = dispatch
        self._check_plan()
        if dispatch == "static":
            assert self.tasks == plan[self.stage_id]   # executed order == the plan arrays
        # bounded rings: one slot count for every activation ring (so a
        # task's slot pointers repeat every n_ring micro-batches and its
        # captured graph can be reused), a multiple of the gradient ring's
        self.n_grad = min(self.N, GRAD_SLOTS)
        need = max(in_flight(o) for o in orders) + RING_PAD
        self.n_ring = min(self.N, -(-need // self.n_grad) * self.n_grad)
        # live dispatch: per-stage policy state + measured task durations
        self._profile = profile
        self._est = {F: 0.0, R: 0.0, B: 0.0}
        self.trace = trace
        self.loss_sum = torch.zeros(1, device=self.device)
        self.flags = torch.zeros(2, device=self.device)
        # device loss-scaler state {scale, applied Adam steps, good steps, scale used}
        s0 = self.scaler.init
        self._ss = torch.tensor([s0, 0.0, 0.0, s0], dtype=torch.float32, device=self.device)
        self._scale_used = None
        self._setup_groups()
        if P > 1:
            slot_elems = self.m * model.seq_len * model.hidden
            self.links = _Links(self.rank, self.stage_id, P, [0] + [self.n_ring] * (P - 1),
                                [self.n_grad] * (P - 1) + [0], slot_elems, self.gloo, self.shm)
        self.gpu_launches_per_step = None
        self._setup_dp()
        # Each task's launch sequence (tens to hundreds of kernels) is captured
        # once into a CUDA graph and replayed: the per-launch host cost would
        # otherwise approach the GPU time of the short kernels. Inputs reach
        # the graph through fixed buffers; IPC waits / signals stay outside.
        # Dropout masks stay fresh under replay: every site reads the
        # (step, micro-batch) seed from a device buffer written by a kernel
        # launched before each task, outside the graph. Disabled while kernel
        # timing hooks are active.
        self.use_graphs = True if graphs is None else bool(graphs)
        self.seed = seed
        T = self.m * model.seq_len
        self._in_ids = torch.zeros(T, dtype=torch.int64, device=self.device)
        self._in_types = torch.zeros(T, dtype=torch.int64, device=self.device)
        self._in_labels = torch.zeros(T, dtype=torch.int64, device=self.device)

    # ---------------------------------------------------------------- setup
    def _opportunistic_orders(self, profile):
        """Every stage's dispatch order as the reference's opportunistic
        replica kernel runs the schedule under ``profile`` (default: the
        generator's own 1:2:1 F:B:R times per cut-point, no transfer cost)."""
        from .calibration import uniform_profile
        from .core import make_block_model
        from .simulator import execution_order
        cfg, pc = self.cfg, self.pc
        if profile is None:
            profile = uniform_profile(cfg.n_layer, 1.0, 2.0, m_grid=(self.m,),
                                      d_grid=tuple(sorted({1, self.D})))
        model = make_block_model("stages", cfg.n_layer, cfg.hidden, cfg.seq_len)
        return execution_order(self.schedule, pc, profile, model, opportunistic=True)

    def retune_dispatch(self, timeline: dict, perturb: bool = False) -> None:
        """Re-derive the opportunistic dispatch order from MEASURED task
        times: every rank contributes its stage's mean F/R/B of a traced step
        (``step(trace=True)`` timeline), and the replica kernel re-runs the
        schedule over one cut-point per stage with those times. Collective
        over the pipeline ranks; all ranks compute the same orders."""
        table = exchange_stage_means(stage_means(timeline), self.rank, self.world, self.device)
        current = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(current, self.tasks)
        else:
            current = [self.tasks]
        best = retune_order(self.schedule, self.P, self.D, self.m, self.N, self.cfg.hidden,
                            self.cfg.seq_len, table, current[:self.P], perturb=perturb)
        self.tasks = best[self.stage_id]
        self.dispatch = "opportunistic"
        self._check_plan()
        need = max(in_flight(o) for o in best) + RING_PAD
        if self.P > 1 and need > self.n_ring and self.n_ring < self.N:
            self._resize_rings(min(self.N, -(-need // self.n_grad) * self.n_grad))

    def _resize_rings(self, n_ring: int) -> None:
        """Rebuild the activation rings with ``n_ring`` slots (every rank of
        the job, between steps): unmap and free the old rings, exchange new
        IPC handles, drop the captured graphs (their slot keys changed)."""
        torch.cuda.synchronize(self.device)
        self.links.close()
        dist.barrier(group=self.gloo)
        self.links.free_local()
        self.n_ring = n_ring
        slot_elems = self.m * self.cfg.seq_len * self.cfg.hidden
        self.links = _Links(self.rank, self.stage_id, self.P, [0] + [n_ring] * (self.P - 1),
                            [self.n_grad] * (self.P - 1) + [0], slot_elems, self.gloo, self.shm,
                            epoch_g=self.step_count * self.N + 1)
        self._graphs = {}

    def _check_plan(self):
        """The executor relies on rule 2 (R(j) directly before B(j)), on the
        last stage's F(j)/B(j) alternation (sp/scheduler.py:228-241) and on
        backwards in ascending micro-batch order (the gradient rings are
        consumed in order)."""
        last = self.spec.last
        bs = [j for kind, j in self.tasks if kind == B]
        if bs != sorted(bs):
            raise ConfigError(f"stage {self.stage_id}: backwards out of micro-batch order")
        for i, (kind, j) in enumerate(self.tasks):
            if kind == B:
                prev = self.tasks[i - 1] if i else None
                want = F if last else R
                if prev != (want, j):
                    raise ConfigError(f"stage {self.stage_id}: B{j + 1} not preceded by "
                                      f"{'F' if last else 'R'}{j + 1}")

    def _setup_dp(self):
        """C1 buckets: one per transformer layer of the stage (its gradients
        are final once the LAST backward of the step has passed it — they are
        exchanged on a side stream while that backward continues down the
        stage) plus the embedding / head remainder after it. The payload is
        bf16 (2 B/param, the reference's pricing, sp/calibration.py:162-176)
        packed from the fp32 accumulators and unpacked after the sum."""
        self._comm = None
        self._ar_spans = []
        if self.D == 1:
            return
        from .model import layer_param_shapes
        P = self.stage.params
        self._comm = torch.cuda.Stream(self.device)
        self._gbf = torch.empty(P.numel, dtype=torch.bfloat16, device=self.device)
        names = [n for n, _ in layer_param_shapes(self.cfg)]
        self._layer_seg = {li: P.segment([f"l{li}.{n}" for n in names])
                           for li in self.spec.layers}
        cuts = sorted(self._layer_seg.values())
        rest, pos = [], 0
        for lo, hi in cuts:
            if lo > pos:
                rest.append((pos, lo))
            pos = max(pos, hi)
        if pos < P.numel:
            rest.append((pos, P.numel))
        self._rest_seg = rest
        self._layer_ev = {li: torch.cuda.Event(external=True) for li in self.spec.layers}
        self._last_b = max(j for kind, j in self.tasks if kind == B)

    def _dp_bucket(self, lo, hi):
        """Pack, allreduce (bf16) and unpack gradient[lo:hi] on the comm
        stream; the span is timed (the measured AR work of the bubble)."""
        P, comm = self.stage.params, self._comm
        with torch.cuda.stream(comm):
            e0 = torch.cuda.Event(enable_timing=True) if self.trace else None
            if e0 is not None:
                e0.record(comm)
            K.grad_pack_bf16(P.grad[lo:hi], self._gbf[lo:hi], stream=comm)
            w = dist.all_reduce(self._gbf[lo:hi], group=self.dp_group, async_op=True)
            w.wait()
            K.grad_unpack_bf16(self._gbf[lo:hi], P.grad[lo:hi], stream=comm)
            if e0 is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(comm)
                self._ar_spans.append((e0, e1))

    def _layer_mark(self, li):
        self._layer_ev[li].record(self.stream)

    def _start_dp_layers(self):
        """After the last backward is enqueued: one bucket per layer, each
        behind the event its layer's backward recorded (top layer first)."""
        for li in reversed(self.spec.layers):
            self._comm.wait_event(self._layer_ev[li])
            lo, hi = self._layer_seg[li]
            self._dp_bucket(lo, hi)

    def _setup_groups(self):
        P, D = self.P, self.D
        self.dp_group = self.pipe_group = self.tie_group = None
        self.gloo = None
        self.shm = None
        if self.world == 1:
            return
        gr = group_ranks(P, D)
        self._groups = []

        def new(ranks):   # collective over the whole world, members or not
            g = dist.new_group(ranks, backend=self.backend)
            self._groups.append(g)
            return g
        for s, ranks in enumerate(gr["dp"]):
            g = new(ranks)
            if s == self.stage_id:
                self.dp_group = g
        for r, ranks in enumerate(gr["pipe"]):
            g = new(ranks)
            if r == self.replica:
                self.pipe_group = g
        for r, ranks in enumerate(gr["tie"]):
            g = new(ranks)
            if r == self.replica and self.active and (self.spec.first or self.spec.last):
                self.tie_group = g
        self.gloo = dist.new_group(list(range(self.world)), backend="gloo")
        self._groups.append(self.gloo)
        tag = os.environ.get("MASTER_PORT", "0")
        name = f"vpipe_{tag}_{os.getuid()}"
        if self.rank == 0:
            self.shm = _Shm(name, self.world, self.N, create=True)
        dist.barrier(group=self.gloo)
        if self.rank != 0:
            self.shm = _Shm(name, self.world, self.N, create=False)
        dist.barrier(group=self.gloo)

    # ----------------------------------------------------------------- data
    def _device_batch(self, batch):
        """Micro-batch views of this replica's rows; a partial last
        micro-batch is padded with ignored labels (M_total semantics,
        sp/planner.py:99-103). Host tensors are copied H2D here."""
        ids = batch.get("input_ids") if self.spec.first else None
        labels = batch.get("labels") if self.spec.last else None
        types = None
        if self.spec.first and self.cfg.arch == "bert":
            types = batch.get("token_type_ids")
            if types is None:
                types = torch.zeros_like(ids)
        rows = self.N * self.m
        share = min(max(self.global_batch - self.replica * rows, 0), rows)
        out = {}
        for key, t, fill in (("ids", ids, 0), ("labels", labels, -100), ("types", types, 0)):
            if t is None:
                continue
            if t.shape[0] not in (share, rows):
                raise ConfigError(f"replica {self.replica} got {t.shape[0]} rows; its share of "
                                  f"M_total = {self.global_batch} is {share}")
            if t.shape[0] < rows:
                pad = torch.full((rows - t.shape[0], t.shape[1]), fill, dtype=torch.int64,
                                 device=t.device)
                t = torch.cat([t, pad], 0)
            if t.device != self.device:
                t = t.to(self.device, non_blocking=True)
            out[key] = t.view(self.N, self.m * self.cfg.seq_len)
        return out

    # ----------------------------------------------------------------- step
    def step(self, batch: Dict[str, torch.Tensor], apply: bool = True) -> StepResult:
        """One mini-batch: N_m micro-batches through this stage's task list,
        then gradient synchronisation and the optimizer update."""
        self.step_count += 1
        if not self.active:
            return StepResult(None, torch.zeros(2), None)
        st = self.stream
        cfg, stage = self.cfg, self.stage
        # loss = mean over the M_total samples' label tokens (BERT: the
        # generator fixes mlm_per_seq masked positions per sequence)
        total_tokens = self.global_batch * (cfg.mlm_per_seq if cfg.arch == "bert" else cfg.seq_len)
        scale = 1.0 / total_tokens      # x the device loss scale, in the xent kernel
        ev = [] if self.trace else None
        self._ar_spans = []
        st.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(st):
            data = self._device_batch(batch)
            if self.spec.last:
                K.fill_f32_(self.loss_sum, 0.0, st)
            t_start = self._mark(ev)
            ctx = _StepCtx(g0=(self.step_count - 1) * self.N + 1, data=data, scale=scale, ev=ev,
                           graphs=self.use_graphs and not K.GEMM_TIMING["on"]
                           and self.step_count > 1)
            if self.dispatch == "live":
                self._run_live(ctx)
            else:
                for kind, j in self.tasks:
                    self._launch(kind, j, ctx)
            self.executed = ctx.executed
            t_ar0 = self._mark(ev)
            self._sync_grads()
            t_ar1 = self._mark(ev)
            self._scale_used = self._ss[0:1].clone()   # before the scaler moves it
            if apply:
                self._optimizer_step()
            t_end = self._mark(ev)
        # the caller's stream is ordered after the step (loss, flags, updated
        # weights): the executor stream is non-blocking w.r.t. the default one
        torch.cuda.current_stream(self.device).wait_stream(st)
        timeline = None
        if ev is not None:
            st.synchronize()
            timeline = self._timeline(t_start, ev, t_ar0, t_ar1, t_end)
        loss = self.loss_sum if self.spec.last else None
        return StepResult(loss, self.flags, self._scale_used, timeline)

    def _launch(self, kind, j, ctx):
        """Enqueue task (kind, j) on the compute stream: ring waits / credits,
        the task's launches (graph replay), then the data signals and slot
        releases. Micro-batch j of this step is global micro-batch g."""
        st, stage, cfg, links = self.stream, self.stage, self.cfg, self.links
        g = ctx.g0 + j
        data = ctx.data
        # inputs first (the stream waits on the peer's IPC event), so the
        # task's timing events bracket compute only
        if kind != B and not self.spec.first and j not in ctx.x_in:
            links.wait(_Links.ACT, g, st)
            ctx.x_in[j] = links.rx_slot(_Links.ACT, g, (stage.T, cfg.hidden))
        g_in = None
        if kind == B and not self.spec.last:
            links.wait(_Links.GRAD, g, st)
            g_in = links.rx_slot(_Links.GRAD, g, (stage.T, cfg.hidden))
        # credits: the peer slot this task writes must have been released
        if kind == F and not self.spec.last:
            links.acquire(_Links.ACT, g, st)
        if kind == B and not self.spec.first:
            links.acquire(_Links.GRAD, g, st)
        if self.spec.first:
            self._in_ids.copy_(data["ids"][j], non_blocking=True)
            if "types" in data:
                self._in_types.copy_(data["types"][j], non_blocking=True)
        if self.spec.last and kind == B:
            self._in_labels.copy_(data["labels"][j], non_blocking=True)
        if cfg.dropout > 0:
            K.set_seed(stage.seed_buf, task_seed(self.seed, self.step_count,
                                                 self.replica * self.N + j), st)
        e0 = self._mark(ctx.ev)
        x = ctx.x_in.get(j)

        dp_hook = kind == B and self.D > 1 and j == self._last_b

        def body():
            self._task(kind, g, x, g_in, ctx.scale, st, "types" in data,
                       layer_done=self._layer_mark if dp_hook else None)
        if ctx.graphs:
            key = (kind, g % self.n_ring) if links is not None else (kind, 0)
            self._replay(key + (dp_hook,), body, st)
        else:
            body()
        if dp_hook:
            self._start_dp_layers()
        if kind == F and not self.spec.last:
            links.signal(_Links.ACT, g, st)
        if kind == B:
            if not self.spec.first:
                links.signal(_Links.GRAD, g, st)
                links.release(_Links.ACT, g, st)    # B(j) was the stash slot's last reader
            if not self.spec.last:
                links.release(_Links.GRAD, g, st)
            ctx.x_in.pop(j, None)
        if ctx.ev is not None:
            ctx.ev.append((kind, j, e0, self._mark(ctx.ev)))
        ctx.executed.append((kind, j))

    # ------------------------------------------------------- live dispatch
    def _run_live(self, ctx):
        """Run this stage's tasks as the reference's opportunistic policy
        decides them ON LINE (dispatch.StagePolicy = decide(),
        sp/engine/py_kernel.py:250-322) from real arrivals: an activation has
        arrived when the producer posted it and its IPC event completed; a
        gradient is known once posted (arriving) and arrived on completion;
        the rule-1 deadline of R(j) is announced by the downstream stage when
        it starts B(j) (its start + measured T_b, minus our T_r). The stage
        decides only when idle (its previous task complete), as the
        reference does, so the host stays at most one task ahead."""
        from .dispatch import StagePolicy
        links = self.links
        last, first = self.spec.last, self.spec.first
        pol = StagePolicy(self.tasks, self.N, last, self.n_ring if not last else self.N,
                          opportunistic=True)
        down = self.rank + 1

        def now_us():
            return time.monotonic_ns() / 1000.0

        def act_arr(mb):
            if first:
                return 0
            g = ctx.g0 + mb
            if links.arrived(_Links.ACT, g) and links.landed(_Links.ACT, g):
                return 0
            return -1

        def grad_arr(mb):
            g = ctx.g0 + mb
            if not links.arrived(_Links.GRAD, g):
                return -1
            return 0 if links.landed(_Links.GRAD, g) else now_us() + 1.0

        def deadline(mb):
            a = self.shm.arr
            if a[down, 4, mb] != ctx.g0 + mb:
                return -1
            return a[down, 5, mb] / 1000.0 - self._est[R]

        pending = None   # (pos, kind, done event, start event)
        while not pol.done:
            if pending is not None:
                pos, kind, done, t0 = pending
                if not done.query():
                    time.sleep(10e-6)
                    continue
                pol.complete(pos)
                dur = t0.elapsed_time(done) * 1e3
                self._est[kind] = dur if self._est[kind] == 0 else 0.7 * self._est[kind] + 0.3 * dur
                pending = None
            now = now_us()
            pos = pol.decide(now, act_arr, grad_arr, deadline, self._est[F], self._est[R])
            if pos is None:
                time.sleep(10e-6)
                continue
            kind, j = pol.kinds[pos], pol.mbs[pos]
            pol.start(pos)
            if kind == B and not first:
                # rule-1 announcement to the stage below: our B(j) ends at
                # now + T_b; its R(j) should then be done
                self.shm.arr[self.rank, 5, j] = int((now + self._est[B]) * 1000.0)
                self.shm.arr[self.rank, 4, j] = ctx.g0 + j
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(self.stream)
            self._launch(kind, j, ctx)
            done = torch.cuda.Event(enable_timing=True)
            done.record(self.stream)
            pending = (pos, kind, done, t0)
        if pending is not None:
            pass   # the last task is left running; the step's tail orders after it

    def _task(self, kind, g, x, g_in, scale, st, typed, layer_done=None):
        """The launches of one schedule task on this stage (graph-capturable:
        every pointer is fixed for a given (kind, ring slot))."""
        stage = self.stage
        ids = self._in_ids if self.spec.first else None
        types = self._in_types if (self.spec.first and typed) else None
        if kind == F or kind == R:
            save = kind == R or self.spec.last
            out_ptr = None
            if kind == F and not self.spec.last:
                out_ptr = self.links.peer_slot_ptr(_Links.ACT, g)
            stage.forward(x, ids, save=save, stream=st, out_ptr=out_ptr, types=types)
        else:
            if self.spec.last:
                stage.loss_and_head_backward(self._in_labels, scale, self.loss_sum, stream=st,
                                             scale_dev=self._ss)
            out = stage.backward(g_in, ids, stream=st, types=types, layer_done=layer_done)
            if not self.spec.first:
                K.p2p_put(self.links.peer_slot_ptr(_Links.GRAD, g), out, stream=st)

    def _replay(self, key, body, st):
        """Run ``body`` through a CUDA graph captured on first use, keyed by
        (task kind, ring slot): the slot pointers repeat every n_ring
        micro-batches. Stages without rings use one graph per task kind."""
        g = self._graphs.get(key)
        if g is None:
            n0 = K.LAUNCHES[0]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                body()
            self._graphs[key] = (g, K.LAUNCHES[0] - n0)
            g, n = self._graphs[key]
        else:
            g, n = g
            K.LAUNCHES[0] += n
        g.replay()

    def _mark(self, ev):
        if ev is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def _timeline(self, t0, ev, ar0, ar1, t_end):
        """Per-task (kind, mb, start, end) in us from the step start on the
        compute stream; ``allreduce_us`` the sync bracket (C1 tail, C3, C2 —
        including waits on other stages), ``ar_work_us`` the C1 bucket work
        itself (pack + NCCL + unpack spans on the comm stream, overlapping
        the last backward) — the AR busy time of the bubble formula."""
        tasks = [(k, j, t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3) for k, j, a, b in ev]
        busy = sum(b - a for _, _, a, b in tasks)
        spans = [(t0.elapsed_time(a) * 1e3, t0.elapsed_time(b) * 1e3) for a, b in self._ar_spans]
        return {"tasks": tasks, "allreduce_us": (t0.elapsed_time(ar0) * 1e3,
                                                 t0.elapsed_time(ar1) * 1e3),
                "ar_spans": spans, "ar_work_us": sum(b - a for a, b in spans),
                "step_us": t0.elapsed_time(t_end) * 1e3, "busy_us": busy}

    # --------------------------------------------------- gradients + update
    def _tied_segment(self):
        P = self.stage.params
        if self.P == 1:
            return None
        name = "wte" if self.spec.first else ("wte_head" if self.spec.last else None)
        if name is None:
            return None
        return P.segment([name])

    def _sync_grads(self):
        P = self.stage.params
        if self.D > 1:
            # C1: the per-layer buckets are in flight since the last backward;
            # the embedding / head remainder follows, then the compute stream
            # joins the comm stream
            self._comm.wait_stream(self.stream)
            for lo, hi in self._rest_seg:
                self._dp_bucket(lo, hi)
            self.stream.wait_stream(self._comm)
            if self.spec.last:
                dist.all_reduce(self.loss_sum, group=self.dp_group)
        seg = self._tied_segment()
        if seg is not None:
            dist.all_reduce(P.grad[seg[0]:seg[1]], group=self.tie_group)       # C3
        K.fill_f32_(self.flags, 0.0, self.stream)
        n_unique = P.numel
        if self.spec.last and not self.spec.first:
            n_unique = P.offsets["wte_head"]   # the tied copy is counted on stage 0
        K.grad_norm_sq(P.grad[:n_unique], self.flags, stream=self.stream)
        if self.P > 1:
            dist.all_reduce(self.flags, group=self.pipe_group)                 # C2

    def _optimizer_step(self):
        """Unscale + skip-on-overflow + clip + AdamW (bias corrections of the
        applied-step count on the device), then the loss-scaler update."""
        P, o, ls = self.stage.params, self.opt, self.scaler
        K.adam_step_dev(P.master, P.weight, P.grad, P.exp_avg, P.exp_avg_sq, self.flags, o.lr,
                        o.betas[0], o.betas[1], o.eps, o.weight_decay, o.max_grad_norm,
                        self._ss, stream=self.stream)
        if ls.dynamic:
            K.loss_scaler_update(self._ss, self.flags, ls.growth, ls.backoff, ls.window,
                                 ls.min_scale, stream=self.stream)
        else:
            K.loss_scaler_update(self._ss, self.flags, 1.0, 1.0, 1 << 40, stream=self.stream)

    # ---------------------------------------------------------------- traces
    def gantt_rows(self, timeline: dict):
        """Measured per-task rows of this stage in the reference Gantt format
        (stage, kind, micro_batch, start_us, end_us), 1-based stage and
        micro-batch, plus the allreduce row 'A' (sp/simulator.py:116-131,
        sp/gantt.py:26-32)."""
        from .core import KIND_NAMES
        rows = [(self.stage_id + 1, KIND_NAMES[k], j + 1, int(round(a)), int(round(b)))
                for k, j, a, b in timeline["tasks"]]
        spans = timeline.get("ar_spans") or [timeline["allreduce_us"]]
        for a0, a1 in spans:   # the C1 bucket work (or the sync bracket at D = 1)
            rows.append((self.stage_id + 1, "A", 0, int(round(a0)), int(round(a1))))
        return sorted(rows, key=lambda r: (r[0], r[3], r[1]))

    @staticmethod
    def gantt_csv(rows) -> str:
        """``stage,kind,microbatch,start_us,end_us`` — loadable by the
        reference's ``spotpipe gantt --from-csv`` (sp/cli.py:429-445)."""
        out = ["stage,kind,microbatch,start_us,end_us"]
        out += [f"{s},{k},{mb},{a},{b}" for s, k, mb, a, b in rows]
        return "\n".join(out) + "\n"

    # ------------------------------------------------------------- inspection
    def param_tensors(self, which: str = "master") -> Dict[str, torch.Tensor]:
        """Named fp32 views (``master``/``grad``) or bf16 ``weight`` views of
        this stage's parameters, keyed like the CPU oracle."""
        P = self.stage.params
        buf = {"master": P.master, "grad": P.grad, "weight": P.weight}[which]
        return {n: P.view(buf, n) for n in P.names}

    # ------------------------------------------------------ checkpoint / morph
    def _owner_replica(self, name: str) -> int:
        """Per-layer checkpoint sharding across the D replicas:
        layer li is written by replica li mod D; embedding/head by replica 0."""
        if name.startswith("l") and "." in name:
            return int(name[1:name.index(".")]) % self.D
        return 0

    def save_layer_state(self, ckpt_dir: str) -> str:
        """Write this rank's share of the stage's per-layer state (fp32 master,
        Adam moments) keyed by GLOBAL parameter names, so a resume may use a
        different stage map / P x D. Each save goes to its own ``step<N>/``
        subdirectory, and rank 0 writes ``manifest.json`` (step, P, D, shard
        list), so shards of an earlier save — possibly under another P x D —
        are never mixed in. Collective: call on every rank. Returns the shard
        written (None on a spare rank)."""
        sub = os.path.join(ckpt_dir, f"step{self.step_count:08d}")
        path = None
        if self.active:
            os.makedirs(sub, exist_ok=True)
            P = self.stage.params
            state = {}
            for name in P.names:
                if name == "wte_head":      # tied copy: stage 0 owns "wte"
                    continue
                if self._owner_replica(name) != self.replica:
                    continue
                state[name] = {k: P.view(getattr(P, buf), name).detach().cpu().clone()
                               for k, buf in (("master", "master"), ("exp_avg", "exp_avg"),
                                              ("exp_avg_sq", "exp_avg_sq"))}
            path = os.path.join(sub, f"stage{self.stage_id}_replica{self.replica}.pt")
            torch.save({"step": self.step_count, "P": self.P, "D": self.D, "state": state}, path)
        if self.world > 1:
            dist.barrier(group=self.gloo)
        if self.rank == 0:
            import json
            man = {"step": self.step_count, "P": self.P, "D": self.D,
                   "scaler": self._ss.tolist() if self.active else None,
                   "stage_map": list(self.pc.stage_map), "micro_batch_size": self.m,
                   "global_batch": self.global_batch,
                   "shards": [f"stage{s_}_replica{r_}.pt" for r_ in range(self.D)
                              for s_ in range(self.P)]}
            tmp = os.path.join(ckpt_dir, "manifest.json.tmp")
            with open(tmp, "w") as f:
                json.dump(man, f)
            os.replace(tmp, os.path.join(ckpt_dir, "manifest.json"))   # the latest save
        if self.world > 1:
            dist.barrier(group=self.gloo)
        return path

    @staticmethod
    def read_manifest(ckpt_dir: str) -> dict:
        import json
        with open(os.path.join(ckpt_dir, "manifest.json")) as f:
            return json.load(f)

    def load_layer_state(self, ckpt_dir: str) -> None:
        """Load every parameter this rank owns from the shards the manifest
        lists; every shard must carry the manifest's step and P x D."""
        man = self.read_manifest(ckpt_dir)
        self.step_count = int(man["step"])
        if not self.active:
            return
        if man.get("scaler") is not None:   # loss scale + Adam's applied-step count
            self._ss.copy_(torch.tensor(man["scaler"], dtype=torch.float32))
        sub = os.path.join(ckpt_dir, f"step{man['step']:08d}")
        P = self.stage.params
        want = set(P.names)
        found = set()
        for fn in man["shards"]:
            blob = torch.load(os.path.join(sub, fn), map_location="cpu")
            if (blob["step"], blob["P"], blob["D"]) != (man["step"], man["P"], man["D"]):
                raise ConfigError(f"checkpoint shard {fn}: step {blob['step']} at "
                                  f"{blob['P']}x{blob['D']}, manifest: step {man['step']} at "
                                  f"{man['P']}x{man['D']}")
            for name, st in blob["state"].items():
                targets = [name] + (["wte_head"] if name == "wte" else [])
                for t in targets:
                    if t not in want:
                        continue
                    for k in ("master", "exp_avg", "exp_avg_sq"):
                        P.view(getattr(P, k), t).copy_(st[k].to(self.device))
                    P.view(P.weight, t).copy_(st["master"].to(self.device).to(torch.bfloat16))
                    found.add(t)
        missing = want - found
        if missing:
            raise ConfigError(f"checkpoint {ckpt_dir} lacks {sorted(missing)[:4]}...")
        torch.cuda.synchronize()

    def close(self):
        """Release what the executor holds: CUDA graphs, peer mappings, IPC
        events, rings, the stage's parameters / optimizer state / working
        sets, the shm handshake and the process groups. Collective over the
        job's ranks (every peer unmaps a ring before its owner frees it)."""
        if getattr(self, "_closed", False):
            return
        self._closed = True
        if self.active:
            torch.cuda.synchronize(self.device)
        self._graphs = {}
        if self.links is not None:
            self.links.close()
        if self.world > 1 and getattr(self, "gloo", None) is not None:
            dist.barrier(group=self.gloo)
        if self.links is not None:
            self.links.free_local()
            self.links = None
        if self.shm is not None:
            self.shm.close()
            self.shm = None
        for g in getattr(self, "_groups", []):
            try:
                dist.destroy_process_group(g)
            except Exception:  # noqa: BLE001 - torn down with the world group already
                pass
        self._groups = []
        self.dp_group = self.pipe_group = self.tie_group = self.gloo = None
        self.stage = None
        self._in_ids = self._in_types = self._in_labels = None
        torch.cuda.empty_cache()


def memory_plan(cfg: GPT2Config, config: ParallelConfig) -> List[Dict[str, int]]:
    """Per-stage HBM plan of a P x D job (bytes per rank): the stage's own
    allocation (``GPT2Stage.memory_plan``) plus the receiver-owned
    activation / gradient rings (one m*s*h*2-byte slot per micro-batch per
    direction). Compare the reference's feasibility model, ``memory_check``
    (16 B/param + stash + one working set, sp/partitioner.py:404-436)."""
    P = config.pipeline_depth
    out = []
    slot = config.micro_batch_size * cfg.seq_len * cfg.hidden * 2
    for s in range(P):
        layers = tuple(i for i, x in enumerate(config.stage_map) if x == s)
        plan = GPT2Stage.memory_plan(cfg, StageSpec(s, P, layers), config.micro_batch_size)
        rings = (int(s > 0) + int(s < P - 1)) * config.num_micro_batches * slot
        plan["rings"] = rings
        plan["total"] += rings
        out.append(plan)
    return out


def replan(cfg: GPT2Config, gpus: int, profile, global_batch: int, micro_batch_size: int,
           hw=None, seed: int = 0) -> ParallelConfig:
    """The morph decision (sp/morphing.py:327-346 → planner.plan,
    sp/planner.py:106-145): the fastest P x D for ``gpus`` GPUs of one
    NVSwitch box, keeping the job's cached micro-batch size and M_total
    (N_m = ceil(M/(m*D)))."""
    from .core import B200_NVL8, JobSpec, make_block_model, uniform_cluster
    from .planner import plan
    model = make_block_model(f"{cfg.arch}-L{cfg.n_layer}-h{cfg.hidden}", cfg.n_layer, cfg.hidden,
                             cfg.seq_len)
    res = plan(gpus, model, JobSpec(global_batch), profile, hw or B200_NVL8,
               uniform_cluster(gpus, 8), seed=seed, micro_batch_size=micro_batch_size)
    return res.chosen


def morph(v: Varuna, ckpt_dir: str, new_config: Optional[ParallelConfig] = None, *,
          gpus: Optional[int] = None, profile=None, **kwargs) -> Varuna:
    """Re-partition a running job: every rank writes its
    per-layer shard, the old executor is torn down and its device memory
    released (``v`` is closed — callers must rebind to the returned
    executor), a new executor is built for the new (P, D, stage_map) on the
    same ranks, and each rank loads exactly the layers its new stage owns.

    Without ``new_config`` the configuration comes from the reference's morph
    decision, ``replan`` (``plan(gpus, ..., micro_batch_size=cached m)``) over
    ``profile`` for ``gpus`` available GPUs (default: the world size); ranks
    beyond the chosen P x D become spares. M_total is preserved."""
    if new_config is None:
        if profile is None:
            raise ConfigError("morph: pass new_config, or a calibration profile to plan with")
        gpus = v.world if gpus is None else gpus
        if not 1 <= gpus <= v.world:
            raise ConfigError(f"morph: {gpus} GPUs available, job has {v.world} ranks")
        new_config = replan(v.cfg, gpus, profile, v.global_batch, v.m)
    v.save_layer_state(ckpt_dir)
    cfg, opt = v.cfg, v.opt
    kwargs.setdefault("global_batch", v.global_batch)
    kwargs.setdefault("backend", v.backend)
    kwargs.setdefault("loss_scale", v.loss_scale)
    v.close()
    nv = Varuna(cfg, new_config, optimizer=opt, **kwargs)
    nv.load_layer_state(ckpt_dir)
    if dist.is_initialized():
        dist.barrier()
    return nv
