"""world_size-2 gloo run of the N > 1 host logic (CPU only): every rank plans
its shard independently from the full problem (as each torchrun process of
bench.py does), the plans agree across processes, and the halo reduction of
point-space partials equals the reference's full-size
all-reduce (dba/solver.hpp:161, 375) value for value."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2112_01349_b200 as dba
        p = dba.generate_synthetic(dba.SyntheticOptions(cameras=30, points=301, num_observations=1507, seed=5))
        cams, pts, cid, pid, *_ = p.arrays()
        part = dba.partition_edges(p, world)[rank]
        shared = dba.shared_points(p, world)
        # plans agree across processes
        got = [None] * world
        dist.all_gather_object(got, (part.edge_ids.tolist(), shared.tolist()))
        edges = sorted(e for g in got for e in g[0])
        assert edges == list(range(p.num_observations)), "partition not exhaustive/disjoint"
        assert all(g[1] == got[0][1] for g in got), "halo plans differ between ranks"
        # point-space partials of a per-edge quantity, reference style: full 3n
        rng = np.random.default_rng(0)
        val = rng.standard_normal((p.num_observations, 3))
        local = np.zeros((p.num_points, 3))
        for e in part.edge_ids:
            local[pid[e]] += val[e]
        full = torch.from_numpy(local.copy())
        dist.all_reduce(full)
        # halo style: only shared points cross ranks
        halo = torch.from_numpy(local[shared].copy())
        dist.all_reduce(halo)
        mine = np.unique(pid[part.edge_ids])
        result = local.copy()
        result[shared] = halo.numpy()
        assert np.array_equal(result[mine], full.numpy()[mine]), "halo reduction differs from full all-reduce"
        # the NCCL unique id travels as bench.py sends it
        uid = [b"x" * 128 if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        assert uid[0] == b"x" * 128
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_two_rank_gloo_plans_and_halo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _shard_worker(rank, world, port, q):
    """One process per shard on the same GPU (the partitions of a torchrun
    job): the library's linearize + assembly of partition `rank` of `world`
    (local collectives), all-reduced over gloo, equals one context's
    assembly of the whole problem; the partition costs add up to the total."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2112_01349_b200 as dba
        p = dba.generate_synthetic(dba.SyntheticOptions(cameras=30, points=301, num_observations=1507, seed=5,
                                                        pixel_noise=0.5))
        with dba.RankContext(0, 8, shard=(rank, world)) as c:
            c.upload(p)
            cost, _ = c.cost()
            c.linearize()
            B, Cm, E, v, w = (np.array(a, copy=True) for a in c.system())
        part = dba.partition_edges(p, world)[rank]
        sums = [torch.from_numpy(x.copy()) for x in (B, Cm, v, w)] + [torch.tensor([cost], dtype=torch.float64)]
        for t in sums:
            dist.all_reduce(t)
        Es = [None] * world
        dist.all_gather_object(Es, (part.edge_ids.tolist(), E))
        if rank == 0:
            with dba.RankContext(0, 8) as c1:
                c1.upload(p)
                cost1, _ = c1.cost()
                c1.linearize()
                B1, C1, E1, v1, w1 = c1.system()
            rel = lambda a, b: float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
            assert rel(sums[0].numpy(), B1) < 1e-13 and rel(sums[2].numpy(), v1) < 1e-13
            assert rel(sums[1].numpy(), C1) < 1e-13 and rel(sums[3].numpy(), w1) < 1e-13
            assert abs(float(sums[4][0]) - cost1) <= 1e-13 * cost1
            for ids, Ek in Es:  # the coupling blocks are per edge: identical wherever the edge lives
                assert np.array_equal(np.asarray(Ek)[:len(ids)], np.asarray(E1)[ids])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))


@pytest.mark.gpu
def test_shard_processes_assemble_the_whole_system():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
