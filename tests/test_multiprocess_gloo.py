"""world_size-2 gloo run of the N > 1 host logic (CPU only): every rank plans
its shard independently from the full problem (as each torchrun process of
bench.py does), the plans agree across processes, and the halo reduction of
point-space partials equals the reference's full-size
all-reduce (dba/solver.hpp:161, 375) value for value."""
import os
import socket

import numpy as np
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
