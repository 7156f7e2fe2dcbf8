"""Integer-exact partitioning (north_star: bit-exact edge-to-partition
assignment and index ordering): the product's host code vs the oracle and the
reference's partition KATs (tests/test_partition.cpp)."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from oracle import oracle as O
from tests.factory import ProblemFactory


def test_even_split_and_remainder():
    """tests/test_partition.cpp:12-24."""
    f = ProblemFactory(3)
    parts = dba.partition_edges(f.random_problem(2, 2, 4), 2)
    assert list(parts[0].edge_ids) == [0, 1] and list(parts[1].edge_ids) == [2, 3]
    parts = dba.partition_edges(f.random_problem(2, 2, 5), 2)
    assert len(parts[0].edge_ids) == 3 and len(parts[1].edge_ids) == 2


def test_invalid_worker_counts():
    """tests/test_partition.cpp:39-44."""
    p = ProblemFactory(9).random_problem(2, 2, 3)
    for k in (0, 4):
        with pytest.raises(dba.dba.InvalidArgumentError):
            dba.partition_edges(p, k)


def test_first_appearance_order():
    """tests/test_partition.cpp:46-71: cameras {3 -> 0, 1 -> 1}."""
    cams = np.zeros((5, 9))
    cams[:, 6] = 1
    p = dba.BAProblem.from_arrays(cams, [[0, 0, -1]], [3, 1, 3], [0, 0, 0], np.zeros((3, 2)))
    part = dba.partition_edges(p, 1)[0]
    assert list(part.camera_map.to_global) == [3, 1]
    assert part.camera_map.local(3) == 0 and part.camera_map.local(1) == 1 and part.camera_map.local(0) == -1


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7])
def test_matches_oracle_integer_exact(k):
    """Partition ranges, LocalIndexMap orders and build_groups ptr/ids arrays
    (dba/partition.hpp:76-103, dba/block_matrix.hpp:309-320)."""
    p = ProblemFactory(17).random_problem(6, 9, 60)
    parts = dba.partition_edges(p, k)
    for r in range(k):
        o = O.partition(p, k, r)
        g = parts[r]
        assert g.edge_ids[0] == o["start"] and len(g.edge_ids) == o["count"]
        for a, b in ((g.camera_map.to_global, o["cam_g"]), (g.point_map.to_global, o["pt_g"]),
                     (g.cam_ptr, o["cam_ptr"]), (g.cam_blocks, o["cam_blk"]), (g.pt_ptr, o["pt_ptr"]),
                     (g.pt_blocks, o["pt_blk"])):
            assert np.array_equal(a, b)


def test_disjoint_exhaustive_order_preserving():
    """tests/test_partition.cpp:91-111."""
    f = ProblemFactory(29)
    for n in (5, 12, 31):
        p = f.random_problem(3, 4, n)
        for k in range(1, min(n, 6) + 1):
            parts = dba.partition_edges(p, k)
            cat = np.concatenate([q.edge_ids for q in parts])
            assert np.array_equal(cat, np.arange(n))
            sizes = [len(q.edge_ids) for q in parts]
            assert max(sizes) - min(sizes) <= 1


def test_halo_plan_point_major():
    """Point-major input: at most K-1 points are shared between ranks
    (SURVEY.md §8e), and exactly the points whose edges straddle a boundary."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=30, points=200, obs_per_point=5))
    cams, pts, cid, pid, *_ = p.arrays()
    for k in (2, 3, 8):
        sh = dba.shared_points(p, k)
        assert len(sh) <= k - 1
        owners = {}
        for r, part in enumerate(dba.partition_edges(p, k)):
            for q in set(pid[part.edge_ids].tolist()):
                owners.setdefault(q, set()).add(r)
        expect = sorted(q for q, s in owners.items() if len(s) > 1)
        assert list(sh) == expect


@pytest.mark.parametrize("shape,split", [
    ((1778, 993923, 5001946), [625244] * 2 + [625243] * 6),
    ((13682, 4456117, 28987644), [3623456] * 4 + [3623455] * 4),
], ids=["venice-1778", "final-13682"])
def test_k8_integer_exact_at_baseline_shapes(shape, split):
    """K = 8 on the BASELINE.json instances: the split
    (dba/partition.hpp:76-103: first N mod K ranks +1), every LocalIndexMap
    and build_groups array equal to the oracle's, integer for integer, and
    the halo plan (points touched by more than one rank) equal to an
    independent numpy count and at most K - 1 points (point-major edges)."""
    m, n, N = shape
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=m, points=n, num_observations=N, seed=1, pixel_noise=0.5))
    k = 8
    parts = dba.partition_edges(p, k)
    assert [len(g.edge_ids) for g in parts] == split
    for r in range(k):
        o = O.partition(p, k, r)
        g = parts[r]
        assert g.edge_ids[0] == o["start"] and len(g.edge_ids) == o["count"]
        for a, b in ((g.camera_map.to_global, o["cam_g"]), (g.point_map.to_global, o["pt_g"]),
                     (g.cam_ptr, o["cam_ptr"]), (g.cam_blocks, o["cam_blk"]), (g.pt_ptr, o["pt_ptr"]),
                     (g.pt_blocks, o["pt_blk"])):
            assert a.dtype.kind == b.dtype.kind and np.array_equal(a, b)
    pid = p.arrays()[3]
    bounds = np.cumsum([0] + split)
    first = pid[bounds[:-1]]
    last = pid[bounds[1:] - 1]
    expect = sorted({int(a) for a, b in zip(last[:-1], first[1:]) if a == b})
    shared = dba.shared_points(p, k)
    assert list(shared) == expect and len(shared) <= k - 1


def test_single_partition_identity_maps():  # tests/test_partition.cpp:26-37
    p = ProblemFactory(5).random_problem(3, 4, 8)
    parts = dba.partition_edges(p, 1)
    assert len(parts) == 1 and len(parts[0].edge_ids) == 8
    assert parts[0].camera_map.size() == 3 and parts[0].point_map.size() == 4
    assert all(parts[0].camera_map.local(c) == c for c in range(3))
    assert all(parts[0].point_map.local(q) == q for q in range(4))


def test_map_composed_with_inverse_is_identity():  # tests/test_partition.cpp:73-89
    p = ProblemFactory(17).random_problem(6, 9, 30)
    cid = p.arrays()[2]
    for k in (1, 2, 3, 4, 7):
        for part in dba.partition_edges(p, k):
            touched = set(int(c) for c in cid[part.edge_ids])
            cm = part.camera_map
            assert cm.size() == len(touched)
            assert all(cm.global_(cm.local(g)) == g for g in touched)
            assert all(cm.local(cm.global_(l)) == l for l in range(cm.size()))


def test_touched_camera_counts_bound_the_global_count():  # tests/test_partition.cpp:113-123
    p = ProblemFactory(31).random_problem(6, 8, 24)
    for k in (1, 2, 3):
        assert sum(part.camera_map.size() for part in dba.partition_edges(p, k)) >= p.num_cameras
