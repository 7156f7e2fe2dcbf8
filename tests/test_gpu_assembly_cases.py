"""The reference's assembly unit cases (tests/test_linear.cpp:42-138) on the
fused GPU linearize + assemble_local (lin.cuh) — one-chunk problems, the
blocks compared with products of the GPU's own Jacobians."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from paper_2112_01349_b200.dba import CameraState, Observation, PointState
from tests.factory import ProblemFactory

pytestmark = pytest.mark.gpu


def _system(p):
    with dba.RankContext(0, 8) as c:
        c.upload(p)
        c.linearize()
        _, jac = c.jacobians()
        return jac, c.system()


def test_single_edge_gram_blocks():  # tests/test_linear.cpp:42-58
    p = ProblemFactory(41).random_problem(1, 1, 1)
    jac, (B, Cb, E, _, _) = _system(p)
    jc, jp = jac[:, :9, 0], jac[:, 9:, 0]
    assert np.linalg.norm(B[0] - jc.T @ jc) < 1e-12 * max(1.0, np.linalg.norm(B[0]))
    assert np.linalg.norm(Cb[0] - jp.T @ jp) < 1e-12 * max(1.0, np.linalg.norm(Cb[0]))
    assert np.linalg.norm(E[0] - jc.T @ jp) < 1e-12 * max(1.0, np.linalg.norm(E[0]))


def test_two_edges_on_one_camera_add_their_gram_blocks():  # tests/test_linear.cpp:60-85
    f = ProblemFactory(43)
    p = dba.BAProblem()
    cam = f.random_camera()
    p.add_node(CameraState(rotation=tuple(cam[:3]), translation=tuple(cam[3:6]), focal=cam[6], k1=cam[7], k2=cam[8]))
    p.add_node(PointState(position=tuple(f.random_point())))
    p.add_node(PointState(position=tuple(f.random_point())))
    for q in (0, 1):
        p.add_edge(Observation(camera_id=0, point_id=q, pixel=tuple(f.u(-50, 50, 2))))
    jac, (B, _, _, _, _) = _system(p)
    expected = sum(jac[:, :9, e].T @ jac[:, :9, e] for e in range(2))
    assert np.linalg.norm(B[0] - expected) / np.linalg.norm(expected) < 1e-14


def test_assembled_diagonal_blocks_symmetric_psd():  # tests/test_linear.cpp:123-138
    p = ProblemFactory(53).random_problem(4, 6, 20)
    _, (B, Cb, _, _, _) = _system(p)
    for blocks in (B, Cb):
        for b in blocks:
            assert np.linalg.norm(b - b.T) <= 1e-10 * max(1.0, np.linalg.norm(b))
    rng = np.random.default_rng(5)
    Bd = np.zeros((9 * len(B), 9 * len(B)))
    for i, b in enumerate(B):
        Bd[9 * i:9 * i + 9, 9 * i:9 * i + 9] = b
    for _ in range(10):
        x = rng.uniform(-1, 1, Bd.shape[0])
        assert x @ (Bd @ x) >= -1e-10 * (x @ x)
