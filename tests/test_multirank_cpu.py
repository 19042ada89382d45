"""Multi-rank host logic on CPU (gloo, world size 2 and 4): the process
groups of the reference placement (rank = r*P + s, sp/simulator.py:71-76),
the measured-time exchange and dispatch re-tuning consensus of
``Varuna.retune_dispatch``, the shared-memory sequence handshake of the
NVLink P2P links, and the bench's max-over-ranks timing reduction. The GPU
data path itself is covered by the ``-m gpu`` tests."""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, P, D, errq):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2111_04007_b200.core import KIND_BACKWARD, KIND_FORWARD, KIND_RECOMPUTE
        from paper_2111_04007_b200.core import uniform_cluster
        from paper_2111_04007_b200.runtime import (_Shm, exchange_stage_means, group_ranks,
                                                   retune_order)
        from paper_2111_04007_b200.scheduler import generate_varuna_schedule
        from paper_2111_04007_b200.simulator import build_placement, rank_layout

        # 1. groups: membership matches the reference placement, and an
        #    all-reduce over each group sums exactly its members
        gr = group_ranks(P, D)
        pipelines, dp_groups = rank_layout(P, D)
        assert gr["dp"] == dp_groups and gr["pipe"] == pipelines
        place = build_placement(uniform_cluster(P * D, 8), P, D)
        slots = sorted(place.assignments.values())
        for (s_, r_), slot in place.assignments.items():   # slot order == rank order
            assert slots.index(slot) == r_ * P + s_
        s_id, r_id = rank % P, rank // P
        for kind in ("dp", "pipe", "tie"):
            for ranks in gr[kind]:
                g = dist.new_group(ranks, backend="gloo")
                if rank in ranks:
                    t = torch.tensor([float(1 << rank)])
                    dist.all_reduce(t, group=g)
                    assert t.item() == float(sum(1 << x for x in ranks)), (kind, ranks, t)
        assert rank in gr["dp"][s_id] and rank in gr["pipe"][r_id]

        # 2. re-tuning: every rank contributes its stage's measured means,
        #    all ranks derive the same valid order
        N, m = 8, 4
        sch = generate_varuna_schedule(P, N, 1.0, 2.0, 1.0)
        f_us = 1000.0 * (1 + 0.5 * s_id)            # skewed stages
        means = (f_us, 2.1 * f_us, 0.0 if s_id == P - 1 else 0.9 * f_us)
        table = exchange_stage_means(means, rank, world)
        assert table.shape == (world, 3) and torch.allclose(
            table[rank], torch.tensor(means, dtype=torch.float64))
        static = [list(zip(*[a.tolist() for a in sch.stage_slice(k)])) for k in range(P)]
        order = retune_order(sch, P, D, m, N, 256, 128, table, static)
        allo = [None] * world
        dist.all_gather_object(allo, order)
        assert all(o == allo[0] for o in allo)
        for k in range(P):
            assert sorted(order[k]) == sorted(static[k])       # same tasks, maybe reordered
            for i, (kind, j) in enumerate(order[k]):            # rule 2 / last-stage F-B
                if kind == KIND_BACKWARD:
                    want = KIND_FORWARD if k == P - 1 else KIND_RECOMPUTE
                    assert order[k][i - 1] == (want, j), (k, i, order[k])

        # 3. P2P sequence handshake through shared memory
        name = f"vpipe_test_{port}_{os.getuid()}"
        if rank == 0:
            shm = _Shm(name, world, 4, create=True)
        dist.barrier()
        if rank != 0:
            shm = _Shm(name, world, 4, create=False)
        dist.barrier()
        shm.post(rank, 0, 1, 7 + rank)
        peer = (rank + 1) % world
        shm.wait(peer, 0, 1, 7 + peer, timeout=30.0)
        dist.barrier()
        shm.close()

        # 4. the bench's device-time reduction: max over ranks
        t = torch.tensor([float(10 + rank)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == 10 + world - 1
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("P,D", [(2, 1), (1, 2), (2, 2), (4, 1), (4, 2), (2, 4), (8, 1)])
def test_multirank_host_logic(P, D):
    world = P * D
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, D, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not alive, "ranks hung"
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
