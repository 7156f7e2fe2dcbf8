"""Pins the CPU oracle against the reference's own known-answer tests and
properties: every assertion below restates a doctest case of
/root/reference/proj/tests (file:line in each docstring). CPU only."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from oracle import oracle as O
from tests.dense import (damp_dense, dense_blockdiag, dense_coupling, dense_jacobian, fd_jacobian, rel,
                         residual_reference, schur)
from tests.factory import ProblemFactory


def single(cam, pt, pix):
    return dba.BAProblem.from_arrays(np.array([cam], float), np.array([pt], float), [0], [0], [pix])


CAM_ID = [0, 0, 0, 0, 0, 0, 1, 0, 0]


# ------------------------------------------------------------ problem.hpp ---
def test_residual_kats():
    """tests/test_problem.cpp:118-130: (0,0) on the optical axis, (2,0) by hand."""
    assert np.array_equal(O.residual(CAM_ID, [0, 0, -1], [0, 0]), [0, 0])
    cam = list(CAM_ID)
    cam[6] = 2
    r = O.residual(cam, [1, 0, -1], [0, 0])
    assert abs(r[0] - 2.0) <= 1e-14 * 2 and abs(r[1]) <= 1e-14


def test_residual_zero_depth_throws():
    """tests/test_problem.cpp:132-138."""
    with pytest.raises(O.OracleError) as e:
        O.residual(CAM_ID, [1, 0, 0], [0, 0])
    assert e.value.code == 1


def test_residual_vs_independent_reference():
    """tests/test_problem.cpp:140-151: 200 trials, 1e-12."""
    f = ProblemFactory(11)
    for _ in range(200):
        cam, pt, pix = f.random_camera(), f.random_point(), f.u(-50, 50, 2)
        ours = O.residual(cam, pt, pix)
        ref = residual_reference(cam, pt, pix)
        assert np.linalg.norm(ours - ref) / max(1.0, np.linalg.norm(ref)) < 1e-12


def test_cost_kat_and_mse():
    """tests/test_problem.cpp:153-180: cost 5.0, MSE 2.5 / 1.25, zero cost."""
    p = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1]], [0, 0], [0, 0], [[-1, 0], [0, -2]])
    c = O.total_cost(p)
    assert c == pytest.approx(5.0, rel=1e-15)
    assert dba.dba.mse_from_cost(c, 2, dba.dba.MSE_PER_OBSERVATION) == pytest.approx(2.5, rel=1e-15)
    assert dba.dba.mse_from_cost(c, 2, dba.dba.MSE_HALF_PER_OBSERVATION) == pytest.approx(1.25, rel=1e-15)
    clean = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1]], [0], [0], [[0, 0]])
    assert O.total_cost(clean) == 0.0


def test_cost_permutation_invariant():
    """tests/test_problem.cpp:182-196."""
    p = ProblemFactory(23).random_problem(4, 6, 20)
    cams, pts, cid, pid, px, py, w = p.arrays()
    perm = np.random.default_rng(99).permutation(len(cid))
    q = dba.BAProblem.from_arrays(cams, pts, cid[perm], pid[perm], np.stack([px, py], 1)[perm])
    assert O.total_cost(q) == pytest.approx(O.total_cost(p), rel=1e-12)
    assert O.total_cost(p) >= 0


def test_cost_degenerate_edge_id():
    """tests/test_problem.cpp:198-218: edge 1."""
    p = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1], [1, 0, 0]], [0, 0], [0, 1], [[0, 0], [0, 0]])
    with pytest.raises(O.OracleError) as e:
        O.total_cost(p)
    assert e.value.code == 1 and e.value.index == 1


# --------------------------------------------------------- jet_vector.hpp ---
def test_jet_product_quotient_sqrt():
    """tests/test_jet.cpp:24-61."""
    v, g = O.jet_op("mul", [2.0], [[1.0], [0.0]], [3.0], [[0.0], [1.0]])
    assert v[0] == 6.0 and g[0, 0] == 3.0 and g[1, 0] == 2.0
    v, g = O.jet_op("div", [6.0], [[1.0], [0.0]], [2.0], [[0.0], [1.0]])
    assert v[0] == 3.0 and g[0, 0] == pytest.approx(0.5, rel=1e-15) and g[1, 0] == pytest.approx(-1.5, rel=1e-15)
    v, g = O.jet_op("sqrt", [4.0], [[4.0]])
    assert v[0] == 2.0 and g[0, 0] == 1.0
    v1, g1 = O.jet_op("neg", [4.0], [[4.0]])
    v2, g2 = O.jet_op("neg", v1, g1)
    assert v2[0] == 4.0 and g2[0, 0] == 4.0
    with pytest.raises(O.OracleError):
        O.jet_op("sqrt", [0.0], [[1.0]])
    v, g = O.jet_op("add_scalar", [1.5], [[2.0], [-3.0]], s=0.0)
    assert v[0] == 1.5 and list(g[:, 0]) == [2.0, -3.0]


def test_jet_errors():
    """tests/test_jet.cpp:63-78: shape mismatch, division by zero names element 1."""
    with pytest.raises(O.OracleError) as e:
        O.jet_op("div", [1.0, 1.0], [[0.0, 0.0]], [2.0, 0.0], [[0.0, 0.0]])
    assert "element 1" in str(e.value)


def test_jet_seed_linearity():
    """tests/test_jet.cpp:89-109: f = (x y + x) / (y + 5)."""
    def f(sx, sy):
        xy_v, xy_g = O.jet_op("mul", [1.3], sx, [0.4], sy)
        num_v, num_g = O.jet_op("add", xy_v, xy_g, [1.3], sx)
        den_v, den_g = O.jet_op("add_scalar", [0.4], sy, s=5.0)
        return O.jet_op("div", num_v, num_g, den_v, den_g)[1][:, 0]
    a, b = 0.7, -2.3
    base = f([[1.0], [0.0]], [[0.0], [1.0]])
    comb = f([[a], [0.0]], [[0.0], [b]])
    assert comb[0] == pytest.approx(a * base[0], rel=1e-14)
    assert comb[1] == pytest.approx(b * base[1], rel=1e-14)


def test_rotation_identity_and_quarter_turn():
    """tests/test_jet.cpp:126-141."""
    v, _ = O.rotate_jets([0, 0, 0], [0.3, -0.7, 1.1])
    assert list(v) == [0.3, -0.7, 1.1]
    v, _ = O.rotate_jets([0, 0, np.pi / 2], [1, 0, 0])
    assert np.allclose(v, [0, 1, 0], atol=1e-12)


def test_rotation_gradients_vs_fd():
    """tests/test_jet.cpp:143-171 (small-angle branch every 7th trial)."""
    rng = np.random.default_rng(1234)
    for trial in range(50):
        aa, x = rng.uniform(-1.5, 1.5, 3), rng.uniform(-1.5, 1.5, 3)
        if trial % 7 == 0:
            aa *= 1e-8
        _, g = O.rotate_jets(aa, x)
        params = np.concatenate([aa, x])
        for j in range(6):
            h = 1e-7 * max(1.0, abs(params[j]))
            hi, lo = params.copy(), params.copy()
            hi[j] += h
            lo[j] -= h
            fd = (O.rotate(hi[:3], hi[3:]) - O.rotate(lo[:3], lo[3:])) / (2 * h)
            assert np.all(np.abs(g[:, j] - fd) / np.maximum(1.0, np.abs(fd)) < 1e-6)


def test_fp32_rotation_small_angle():
    """tests/test_jet.cpp:354-367."""
    rng = np.random.default_rng(555)
    for trial in range(20):
        aa = rng.uniform(-0.5, 0.5, 3).astype(np.float32)
        if trial % 3 == 0:
            aa *= np.float32(1e-4)
        x = rng.uniform(-0.5, 0.5, 3).astype(np.float32)
        ours = O.rotate(aa, x, np.float32).astype(float)
        ref = O.rotate(aa.astype(float), x.astype(float))
        assert np.linalg.norm(ours - ref) <= 1e-5 * max(1.0, np.linalg.norm(ref))


# ---------------------------------------------------------- edge_eval.hpp ---
def test_batched_zero_residual():
    """tests/test_jet.cpp:173-193."""
    cam = list(CAM_ID)
    cam[6] = 2.0
    pix = O.residual(cam, [0.5, -0.25, -1.0], [0, 0])
    res, jac = O.linearize(single(cam, [0.5, -0.25, -1.0], pix))
    assert np.linalg.norm(res[:, 0]) < 1e-15 and np.isfinite(jac).all()


def test_batched_jacobian_vs_fd_and_scalar():
    """tests/test_jet.cpp:195-232."""
    p = ProblemFactory(77).random_problem(4, 7, 25)
    cams, pts, cid, pid, px, py, w = p.arrays()
    res, jac = O.linearize(p)
    for e in range(len(cid)):
        scalar = O.residual(cams[cid[e]], pts[pid[e]], [px[e], py[e]])
        assert np.linalg.norm(res[:, e] - scalar) / max(1.0, np.linalg.norm(scalar)) < 1e-13
        fd = fd_jacobian(lambda c, x, q: O.residual(c, x, q), cams[cid[e]], pts[pid[e]], [px[e], py[e]])
        assert np.all(np.abs(jac[:, :, e] - fd) / np.maximum(1.0, np.abs(fd)) < 1e-6)


def test_batched_bit_identical_across_partitions():
    """tests/test_jet.cpp:250-274."""
    p = ProblemFactory(303).random_problem(4, 6, 21)
    ref_r, ref_j = O.linearize(p)
    for k in (2, 3, 4):
        start = 0
        for r in range(k):
            res, jac = O.linearize(p, k, r)
            n = res.shape[1]
            assert np.array_equal(res, ref_r[:, start:start + n])
            assert np.array_equal(jac, ref_j[:, :, start:start + n])
            start += n


def test_linearize_degenerate_edge_id():
    """tests/test_jet.cpp:276-301: edge 2."""
    p = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1], [0, 1, 0]], [0, 0, 0], [0, 0, 1], np.zeros((3, 2)))
    with pytest.raises(O.OracleError) as e:
        O.linearize(p)
    assert e.value.code == 1 and e.value.index == 2


def test_analytic_matches_autodiff():
    """tests/test_jet.cpp:303-352, incl. the small-angle branch."""
    f = ProblemFactory(909)
    p = f.random_problem(5, 8, 30)
    ra, ja = O.linearize(p, mode=0)
    rn, jn = O.linearize(p, mode=1)
    for e in range(ra.shape[1]):
        assert np.linalg.norm(ra[:, e] - rn[:, e]) <= 1e-12 * max(1.0, np.linalg.norm(ra[:, e]))
        assert np.linalg.norm(ja[:, :9, e] - jn[:, :9, e]) <= 1e-12 * max(1.0, np.linalg.norm(ja[:, :9, e]))
        assert np.linalg.norm(ja[:, 9:, e] - jn[:, 9:, e]) <= 1e-12 * max(1.0, np.linalg.norm(ja[:, 9:, e]))
    cam = f.random_camera()
    cam[:3] *= 1e-8
    tiny = single(cam, f.random_point(), f.u(-50, 50, 2))
    _, ta = O.linearize(tiny, mode=0)
    _, tn = O.linearize(tiny, mode=1)
    assert np.linalg.norm(ta[:, :9] - tn[:, :9]) <= 1e-12 * max(1.0, np.linalg.norm(ta[:, :9]))


# ------------------------------------------------------- block_matrix.hpp ---
def _dense_system(p, k=1, rank=0):
    cams, pts, cid, pid, px, py, w = p.arrays()
    B, Cb, E, v, wv = O.assemble(p, k, rank)
    cnt = E.shape[0]
    start = sum(len(cid) // k + (1 if r < len(cid) % k else 0) for r in range(rank))
    return B, Cb, E, v, wv, cid[start:start + cnt], pid[start:start + cnt]


def test_assembly_matches_dense_gram():
    """tests/test_linear.cpp:87-121 at 1e-12."""
    p = ProblemFactory(47).random_problem(3, 4, 14)
    cams, pts, cid, pid, px, py, w = p.arrays()
    m, n = len(cams), len(pts)
    res, jac = O.linearize(p)
    J, r = dense_jacobian(jac, res, cid, pid, w, m, n)
    gram, rhs = J.T @ J, -J.T @ r
    B, Cb, E, v, wv, ci, pi = _dense_system(p)
    b, c, e = dense_blockdiag(B), dense_blockdiag(Cb), dense_coupling(E, ci, pi, m, n)
    assert rel(b, gram[:9 * m, :9 * m]) < 1e-12
    assert rel(c, gram[9 * m:, 9 * m:]) < 1e-12
    assert rel(e, gram[:9 * m, 9 * m:]) < 1e-12
    assert rel(v, rhs[:9 * m]) < 1e-12 and rel(wv, rhs[9 * m:]) < 1e-12


def test_partitioned_assembly_sums_to_whole():
    """tests/test_linear.cpp:140-182."""
    p = ProblemFactory(59).random_problem(4, 7, 23)
    m, n = p.num_cameras, p.num_points
    B1, C1, E1, v1, w1, ci, pi = _dense_system(p)
    e1 = dense_coupling(E1, ci, pi, m, n)
    for k in (2, 3, 5):
        acc = [0, 0, 0, 0, 0]
        for r in range(k):
            B, Cb, E, v, wv, ci, pi = _dense_system(p, k, r)
            for i, x in enumerate((dense_blockdiag(B), dense_blockdiag(Cb), dense_coupling(E, ci, pi, m, n), v, wv)):
                acc[i] = acc[i] + x
        assert rel(acc[0], dense_blockdiag(B1)) < 1e-12 and rel(acc[1], dense_blockdiag(C1)) < 1e-12
        assert rel(acc[2], e1) < 1e-12 and rel(acc[3], v1) < 1e-12 and rel(acc[4], w1) < 1e-12


def test_damping_kats():
    """tests/test_linear.cpp:284-298."""
    d = np.diag([2.0, 4.0, 8.0])[None]
    assert np.array_equal(O.damp(d, 0.0, 0), d)
    assert np.array_equal(O.damp(np.zeros((1, 3, 3)), 1.0, 0)[0], np.eye(3))
    assert np.array_equal(O.damp(d, 0.5, 1)[0], np.diag([3.0, 6.0, 12.0]))


def test_factor_solve_kats():
    """tests/test_linear.cpp:231-282: solve 2I x = (2,4,6); singular block 1."""
    assert np.linalg.norm(O.factor_solve((2.0 * np.eye(3))[None], [2, 4, 6]) - [1, 2, 3]) < 1e-14
    with pytest.raises(O.OracleError) as e:
        O.factor_solve(np.stack([np.eye(3), -np.eye(3)]), np.zeros(6))
    assert e.value.code == 2 and e.value.index == 1 and e.value.block_size == 3
    rng = np.random.default_rng(11)
    M = rng.uniform(-1, 1, (4, 9, 9))
    D = M @ M.transpose(0, 2, 1) + 0.5 * np.eye(9)
    x = rng.uniform(-1, 1, 36)
    y = O.factor_solve(D, x)
    back = np.concatenate([D[i] @ y[9 * i:9 * i + 9] for i in range(4)])
    assert np.linalg.norm(back - x) / np.linalg.norm(x) < 1e-10


# -------------------------------------------------------------- comms.hpp ---
def test_allreduce_kats():
    """tests/test_comms.cpp:12-59."""
    out = O.allreduce([[1, 2], [3, 4]])
    assert np.array_equal(out, [[4, 6], [4, 6]])
    rng = np.random.default_rng(2024)
    loc = rng.uniform(-1e6, 1e6, (4, 257))
    exp = loc[0].copy()
    for r in range(1, 4):
        exp += loc[r]
    once = O.allreduce(loc)
    assert all(np.array_equal(once[r], exp) for r in range(4))
    assert np.array_equal(O.allreduce(loc), once)


# ------------------------------------------------------------- solver.hpp ---
def _one_edge_problem(cams=1):
    return dba.BAProblem.from_arrays([CAM_ID] * cams, [[0, 0, -1]], [0], [0], [[0, 0]])


def test_dse_zero_coupling_is_bx():
    """tests/test_solver.cpp:75-105."""
    p = _one_edge_problem(2)
    B = np.stack([2 * np.eye(9), 3 * np.eye(9)])
    Cb = np.eye(3)[None]
    x = np.arange(1, 19, dtype=float)
    out, _, _ = O.blocks_solve(p, 1, B, Cb, np.zeros((1, 27)), 0, x)
    assert np.array_equal(out, np.concatenate([2 * x[:9], 3 * x[9:]]))
    out, _, _ = O.blocks_solve(p, 1, B, Cb, np.zeros((1, 27)), 0, np.zeros(18))
    assert np.linalg.norm(out) == 0.0


def test_dse_vs_dense_schur_and_across_k():
    """tests/test_solver.cpp:107-140."""
    rng = np.random.default_rng(31)
    for trial in range(10):
        p = ProblemFactory(1000 + trial).random_problem(3, 4, 9 + trial)
        m, n = p.num_cameras, p.num_points
        B, Cb, E, v, wv, ci, pi = _dense_system(p)
        S = schur(damp_dense(dense_blockdiag(B), 1e-3, 0), damp_dense(dense_blockdiag(Cb), 1e-3, 0),
                  dense_coupling(E, ci, pi, m, n))
        x = rng.uniform(-1, 1, 9 * m)
        ref = S @ x
        k1 = None
        for k in (1, 2, 3):
            out, ident = O.dse(p, k, 1e-3, 0, x)
            assert ident
            assert rel(out, ref) < 1e-10
            k1 = out if k1 is None else k1
            assert rel(out, k1) < 1e-10


def test_dpcg_zero_rhs_and_identity():
    """tests/test_solver.cpp:179-229."""
    p = ProblemFactory(88).random_problem(2, 3, 6)
    x, it, conv, _ = O.dpcg(p, 1, 1e-2, 0, np.zeros(18), 1e-6, 100)
    assert it == 0 and conv and np.linalg.norm(x) == 0.0
    q = _one_edge_problem(1)
    g = np.array([1, -2, 3, -4, 5, -6, 7, -8, 9.0])
    out, it, _ = O.blocks_solve(q, 1, np.eye(9)[None], np.eye(3)[None], np.zeros((1, 27)), 1, g, 1e-10, 100)
    assert it == 1 and np.linalg.norm(out - g) < 1e-14


def test_dpcg_vs_direct_across_k():
    """tests/test_solver.cpp:231-270."""
    rng = np.random.default_rng(41)
    for trial in range(6):
        p = ProblemFactory(2000 + trial).random_problem(3, 5, 11 + trial, normalized=True)
        m, n = p.num_cameras, p.num_points
        B, Cb, E, v, wv, ci, pi = _dense_system(p)
        S = schur(damp_dense(dense_blockdiag(B), 1e-2, 0), damp_dense(dense_blockdiag(Cb), 1e-2, 0),
                  dense_coupling(E, ci, pi, m, n))
        g = rng.uniform(-1, 1, 9 * m)
        direct = np.linalg.solve(S, g)
        for k in (1, 2, 4):
            x, _, _, ident = O.dpcg(p, k, 1e-2, 0, g, 1e-12, 500)
            assert ident and rel(x, direct) < 1e-8


def test_lm_zero_residual_converges_in_one():
    """tests/test_solver.cpp:335-359."""
    f = ProblemFactory(9)
    cams = np.stack([f.random_camera() for _ in range(2)])
    pts = np.stack([f.random_point() for _ in range(3)])
    cid, pid, pix = [], [], []
    for c in range(2):
        for q in range(3):
            cid.append(c)
            pid.append(q)
            pix.append(O.residual(cams[c], pts[q], [0, 0]))
    p = dba.BAProblem.from_arrays(cams, pts, cid, pid, pix)
    assert O.total_cost(p) == 0.0
    st = O.lm_solve(p, dba.SolverConfig())
    assert st.termination == "converged" and st.iteration == 1 and st.cost == 0.0 and st.history[0].accepted


def test_lm_ring_down_and_monotone():
    """tests/test_solver.cpp:361-384."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=20, points=80, obs_per_point=10, seed=1))
    init = O.total_cost(p)
    st = O.lm_solve(p, dba.SolverConfig(max_iterations=50))
    assert st.cost <= 0.1 * init
    last = init
    for r in st.history:
        if r.accepted:
            assert r.cost <= last * (1 + 1e-12)
            last = r.cost
    assert st.cost == st.history[-1].cost


def test_lm_k_equivalence():
    """tests/test_solver.cpp:386-426."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=12, points=40, obs_per_point=6, seed=3))
    cfg = dba.SolverConfig(max_iterations=12, check_rank_identity=True, pcg_tol=1e-12, pcg_max_iters=2000)
    ref = O.lm_solve(p, cfg)
    for k in (2, 4):
        cfg.workers = k
        st = O.lm_solve(p, cfg)
        assert len(st.history) == len(ref.history)
        for a, b in zip(st.history, ref.history):
            assert a.accepted == b.accepted
            if a.accepted:
                assert abs(a.cost - b.cost) / max(1.0, b.cost) < 1e-10
        scale = max(1.0, np.abs(ref.x_c).max(), np.abs(ref.x_p).max())
        assert max(np.abs(st.x_c - ref.x_c).max(), np.abs(st.x_p - ref.x_p).max()) / scale < 1e-8


def test_lm_reject_reuses_system():
    """tests/test_solver.cpp:428-455: edge tallies n (reject) vs 2n (accept)."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=8, points=20, obs_per_point=4, seed=5))
    n = p.num_observations
    st = O.lm_solve(p, dba.SolverConfig(lambda0=1e8, max_iterations=6))
    for r in st.history:
        assert r.worker_edges[0] == (2 * n if r.accepted else n)
    assert st.history[0].worker_edges[0] == 2 * n


def test_lm_stalled():
    """tests/test_solver.cpp:488-504."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=4, points=8, obs_per_point=2))
    st = O.lm_solve(p, dba.SolverConfig(lambda0=1e31, lambda_max=1e32, step_tol=0.0, max_iterations=50))
    assert st.termination == "stalled"


def test_lm_analytic_vs_autodiff():
    """tests/test_solver.cpp:506-528."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=12, points=36, obs_per_point=5, seed=21))
    a = O.lm_solve(p, dba.SolverConfig(max_iterations=12))
    b = O.lm_solve(p, dba.SolverConfig(max_iterations=12, jacobian=1))
    assert len(a.history) == len(b.history)
    for x, y in zip(a.history, b.history):
        assert abs(x.cost - y.cost) <= 1e-6 * max(1.0, x.cost)


def test_lm_fp32_tracks_fp64():
    """tests/test_solver.cpp:530-562."""
    p64 = dba.generate_synthetic(dba.SyntheticOptions(cameras=14, points=50, obs_per_point=6, seed=11))
    p32 = p64.astype(np.float32)
    s64 = O.lm_solve(p64, dba.SolverConfig(max_iterations=15))
    s32 = O.lm_solve(p32, dba.SolverConfig(max_iterations=15, workers=2))
    n = p64.num_observations
    init = O.total_cost(p64) / (2 * n)
    m64, m32 = s64.cost / (2 * n), s32.cost / (2 * n)
    assert m64 < 1e-3 * init and m32 < 1e-3 * init
    assert abs(m32 - m64) <= 0.02 * max(m64, 1e-12) + 1e-9


def test_lm_work_scales_as_one_over_k():
    """tests/test_solver.cpp:564-599."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=16, points=64, obs_per_point=8, seed=7))
    k1 = O.lm_solve(p, dba.SolverConfig(max_iterations=5, pcg_tol=1e-4))
    k4 = O.lm_solve(p, dba.SolverConfig(max_iterations=5, pcg_tol=1e-4, workers=4))
    assert len(k1.history) == len(k4.history)
    for a, b in zip(k1.history, k4.history):
        q = a.worker_edges[0] / 4
        for r in range(4):
            assert abs(b.worker_edges[r] - q) <= 0.05 * q
            o = a.worker_block_ops[0] / 4
            if o > 0:
                assert abs(b.worker_block_ops[r] - o) <= 0.05 * o
