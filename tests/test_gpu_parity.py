"""GPU parity: the sm_100a path (libdbag.so, through the C ABI) against the CPU
oracle on identical inputs. Tolerances are those of SURVEY.md §7-§8d and the
reference's own tests (file:line per test)."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from oracle import oracle as O
from tests.dense import damp_dense, dense_blockdiag, dense_coupling, fd_jacobian, rel, schur
from tests.factory import ProblemFactory

pytestmark = pytest.mark.gpu

CAM_ID = [0, 0, 0, 0, 0, 0, 1, 0, 0]


def ctx_for(p, mode=0):
    c = dba.RankContext(0, p.precision)
    c.upload(p, mode)
    return c


def ring(cams, pts, q, seed=1, radius=8.0, noise=0.0, nobs=0, dtype=np.float64):
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=cams, points=pts, obs_per_point=q, seed=seed,
                                                    circle_radius=radius, pixel_noise=noise, num_observations=nobs))
    return p if dtype == np.float64 else p.astype(dtype)


# ------------------------------------------------------------- linearize ----
@pytest.mark.parametrize("mode", [0, 1])
def test_linearize_matches_oracle(mode):
    """Residual 1e-13 and J 1e-12 relative vs the oracle's EdgeJacobianBatch
    (tests/test_jet.cpp:195-232, 303-329)."""
    p = ring(40, 300, 6, noise=0.5)
    with ctx_for(p, mode) as c:
        c.linearize()
        res, jac = c.jacobians()
    r0, j0 = O.linearize(p, mode=mode)
    for e in range(res.shape[1]):
        assert np.linalg.norm(res[:, e] - r0[:, e]) <= 1e-13 * max(1.0, np.linalg.norm(r0[:, e]))
        assert np.linalg.norm(jac[:, :, e] - j0[:, :, e]) <= 1e-12 * max(1.0, np.linalg.norm(j0[:, :, e]))


def test_linearize_vs_fd_random_problem():
    """tests/test_jet.cpp:195-232 on the GPU: J vs central differences 1e-6."""
    p = ProblemFactory(77).random_problem(4, 7, 25)
    cams, pts, cid, pid, px, py, w = p.arrays()
    with ctx_for(p) as c:
        c.linearize()
        res, jac = c.jacobians()
    for e in range(len(cid)):
        fd = fd_jacobian(lambda a, b, q: O.residual(a, b, q), cams[cid[e]], pts[pid[e]], [px[e], py[e]])
        assert np.all(np.abs(jac[:, :, e] - fd) / np.maximum(1.0, np.abs(fd)) < 1e-6)


def test_linearize_degenerate_edge_id():
    """tests/test_jet.cpp:276-301: DegenerateDepthError names global edge 2."""
    p = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1], [0, 1, 0]], [0, 0, 0], [0, 0, 1], np.zeros((3, 2)))
    with ctx_for(p) as c:
        with pytest.raises(dba.dba.DegenerateDepthError) as e:
            c.linearize()
        assert e.value.edge_id == 2


def test_cost_matches_oracle_and_degenerate():
    """EdgeEvaluator::cost vs total_cost 1e-12; degenerate trial -> +inf with edge id
    (tests/test_problem.cpp:198-218)."""
    p = ring(30, 200, 5, noise=0.5)
    assert dba.total_cost(p) == pytest.approx(O.total_cost(p), rel=1e-12)
    q = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1], [1, 0, 0]], [0, 0], [0, 1], [[0, 0], [0, 0]])
    with pytest.raises(dba.dba.DegenerateDepthError) as e:
        dba.total_cost(q)
    assert e.value.edge_id == 1


# -------------------------------------------------------------- assembly ----
@pytest.mark.parametrize("seed", [47, 59])
def test_assembly_matches_oracle(seed):
    """B, C, E, v, w vs the oracle's assemble_local at 1e-12 (tests/test_linear.cpp:87-121)."""
    p = ProblemFactory(seed).random_problem(4, 7, 40)
    with ctx_for(p) as c:
        c.linearize()
        B, Cb, E, v, w = c.system()
    B0, C0, E0, v0, w0 = O.assemble(p)
    for a, b in ((B, B0), (Cb, C0), (E, E0), (v, v0), (w, w0)):
        assert rel(a, b) < 1e-12


# ------------------------------------------------------- damping / factor ----
def test_singular_block_reports_index():
    """tests/test_linear.cpp:270-282 via the trial: a C block with a negative
    pivot raises SingularBlockError naming global point 1, size 3."""
    p = ProblemFactory(5).random_problem(2, 3, 6)
    with ctx_for(p) as c:
        c.linearize()
        B, Cb, E, v, w = c.system()
        Cb[1] = -np.eye(3)
        c.set_system(B=B, Cb=Cb)
        with pytest.raises(dba.dba.SingularBlockError) as e:
            c.damp_factor(0.0, 0)
        assert e.value.block_index == 1 and e.value.block_size == 3


# ------------------------------------------------------------------- DSE ----
def test_dse_zero_coupling_is_bx():
    """tests/test_solver.cpp:75-105 (exact)."""
    p = dba.BAProblem.from_arrays([CAM_ID, CAM_ID], [[0, 0, -1]], [0], [0], [[0, 0]])
    B = np.stack([2 * np.eye(9), 3 * np.eye(9)])
    x = np.arange(1, 19, dtype=float)
    out, _, _ = dba.group_operator(p, 1, x, mode=0, blocks=(B, np.eye(3)[None], np.zeros((1, 27))))
    assert np.array_equal(out, np.concatenate([2 * x[:9], 3 * x[9:]]))


def test_dse_vs_dense_schur_and_oracle_across_k():
    """tests/test_solver.cpp:107-140: 1e-10 vs dense Schur, rank-identical,
    cross-K 1e-10; plus 1e-12 vs the oracle at the same K."""
    rng = np.random.default_rng(31)
    for trial in range(6):
        p = ProblemFactory(1000 + trial).random_problem(3, 4, 9 + trial)
        m = p.num_cameras
        B0, C0, E0, _, _ = O.assemble(p)
        cams, pts, cid, pid, *_ = p.arrays()
        S = schur(damp_dense(dense_blockdiag(B0), 1e-3, 0), damp_dense(dense_blockdiag(C0), 1e-3, 0),
                  dense_coupling(E0, cid, pid, m, p.num_points))
        x = rng.uniform(-1, 1, 9 * m)
        ref = S @ x
        for k in (1, 2, 3):
            out, _, ident = dba.group_operator(p, k, x, mode=0, lam=1e-3, policy=0)
            orc, _ = O.dse(p, k, 1e-3, 0, x)
            assert ident
            assert rel(out, ref) < 1e-10
            assert rel(out, orc) < 1e-12


def test_dpcg_identity_one_iteration_and_zero_rhs():
    """tests/test_solver.cpp:179-229."""
    p = dba.BAProblem.from_arrays([CAM_ID], [[0, 0, -1]], [0], [0], [[0, 0]])
    g = np.array([1, -2, 3, -4, 5, -6, 7, -8, 9.0])
    x, it, _ = dba.group_operator(p, 1, g, mode=1, blocks=(np.eye(9)[None], np.eye(3)[None], np.zeros((1, 27))),
                                  tol=1e-10, max_iters=100)
    assert it == 1 and np.linalg.norm(x - g) < 1e-14
    q = ProblemFactory(88).random_problem(2, 3, 6)
    x, it, _ = dba.group_operator(q, 1, np.zeros(18), mode=1, lam=1e-2, policy=0, tol=1e-6, max_iters=100)
    assert it == 0 and np.linalg.norm(x) == 0.0


def test_dpcg_vs_direct_and_oracle_across_k():
    """tests/test_solver.cpp:231-270: dense direct 1e-8, rank-identical."""
    rng = np.random.default_rng(41)
    for trial in range(4):
        p = ProblemFactory(2000 + trial).random_problem(3, 5, 11 + trial, normalized=True)
        m = p.num_cameras
        B0, C0, E0, _, _ = O.assemble(p)
        cams, pts, cid, pid, *_ = p.arrays()
        S = schur(damp_dense(dense_blockdiag(B0), 1e-2, 0), damp_dense(dense_blockdiag(C0), 1e-2, 0),
                  dense_coupling(E0, cid, pid, m, p.num_points))
        g = rng.uniform(-1, 1, 9 * m)
        direct = np.linalg.solve(S, g)
        for k in (1, 2, 4):
            x, it, ident = dba.group_operator(p, k, g, mode=1, lam=1e-2, policy=0, tol=1e-12, max_iters=500)
            assert ident and rel(x, direct) < 1e-8


def test_dpcg_iterates_across_k_fabricated():
    """tests/test_solver.cpp:272-333: fixed 12 iterations on a benign operator,
    bitwise rank-identical, cross-K 1e-10, and 1e-12 vs the oracle."""
    cams, pts, edges = 4, 6, 16
    p = ProblemFactory(4242).random_problem(cams, pts, edges)
    rng = np.random.default_rng(17)
    Mb = 0.05 * rng.uniform(-1, 1, (cams, 9, 9))
    B = np.eye(9) + Mb @ Mb.transpose(0, 2, 1)
    Mc = 0.05 * rng.uniform(-1, 1, (pts, 3, 3))
    Cb = np.eye(3) + Mc @ Mc.transpose(0, 2, 1)
    E = 0.02 * rng.uniform(-1, 1, (edges, 27))
    g = rng.uniform(-1, 1, 9 * cams)
    ref = None
    for k in (1, 2, 4):
        x, _, ident = dba.group_operator(p, k, g, mode=1, blocks=(B, Cb, E), tol=0.0, max_iters=12)
        xo, _, _ = O.blocks_solve(p, k, B, Cb, E, 1, g, 0.0, 12)
        assert ident and rel(x, xo) < 1e-12
        ref = x if ref is None else ref
        assert rel(x, ref) < 1e-10


def test_group_allreduce_bitwise_sequential():
    """tests/test_comms.cpp:12-59: ascending-rank sum, bit-identical, rank-identical."""
    assert np.array_equal(dba.group_allreduce(np.array([[1.0, 2], [3, 4]])), [[4, 6], [4, 6]])
    rng = np.random.default_rng(2024)
    loc = rng.uniform(-1e6, 1e6, (4, 257))
    exp = loc[0].copy()
    for r in range(1, 4):
        exp += loc[r]
    out = dba.group_allreduce(loc)
    assert all(np.array_equal(out[r], exp) for r in range(4))
    assert np.array_equal(dba.group_allreduce(loc), out)


# ------------------------------------------------------------ LM solver ----
def _compare_histories(g, o, cost_tol, check_lambda=True):
    assert len(g.history) == len(o.history), (len(g.history), len(o.history))
    assert [r.accepted for r in g.history] == [r.accepted for r in o.history]
    for a, b in zip(g.history, o.history):
        assert abs(a.cost - b.cost) <= cost_tol * max(abs(b.cost), 1e-300) or abs(a.cost - b.cost) < 1e-20
        if check_lambda:
            assert a.lambda_ == pytest.approx(b.lambda_, rel=1e-9)
    assert g.termination == o.termination


@pytest.mark.parametrize("k", [1, 2, 4])
def test_lm_trajectory_tight_pcg(k):
    """K-equivalence protocol of tests/acceptance.cpp:108-176 (pcg_tol 1e-12,
    pcg_max_iters 2000) applied GPU vs oracle at the same K: identical
    accept/reject sequence and lambda schedule, per-iteration costs within
    1e-9 relative (north_star asks 1e-6), final parameters within 1e-8,
    identical per-worker edge tallies."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024)
    cfg = dba.SolverConfig(max_iterations=10, workers=k, check_rank_identity=True, pcg_tol=1e-12, pcg_max_iters=2000)
    g = dba.lm_solve(p, cfg)
    o = O.lm_solve(p, cfg)
    _compare_histories(g, o, 1e-9)
    for a, b in zip(g.history, o.history):
        assert a.worker_edges == b.worker_edges
    scale = max(1.0, np.abs(o.x_c).max(), np.abs(o.x_p).max())
    assert max(np.abs(g.x_c - o.x_c).max(), np.abs(g.x_p - o.x_p).max()) / scale < 1e-8


@pytest.mark.parametrize("k", [2, 3, 4])
def test_lm_trajectory_with_shared_points(k):
    """Count-exact edge totals that split points across shard boundaries
    (SURVEY.md §8e halo: <= K - 1 shared points, exchanged instead of the
    reference's full point-space all-reduce). Same protocol as above."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024, nobs=3197)
    assert len(dba.shared_points(p, k)) > 0
    cfg = dba.SolverConfig(max_iterations=6, workers=k, check_rank_identity=True, pcg_tol=1e-12, pcg_max_iters=2000)
    g = dba.lm_solve(p, cfg)
    o = O.lm_solve(p, cfg)
    _compare_histories(g, o, 1e-9)
    for a, b in zip(g.history, o.history):
        assert a.worker_edges == b.worker_edges


@pytest.mark.parametrize("nobs", [3197, 3203])
def test_trial_pieces_across_k_with_shared_points(nobs):
    """One LM trial's pieces on K in-process ranks (group_operator modes 2-5):
    rhs g, DPCG dx_c, trial cost and model terms equal K = 1 to reassociation
    level when shard boundaries split points."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024, nobs=nobs)
    z = np.zeros(9 * p.num_cameras)
    base = {m: dba.group_operator(p, 1, z, mode=m, lam=1e-4, policy=1, tol=1e-12, max_iters=2000)[0] for m in (2, 3, 4, 5)}
    for k in (2, 3, 4):
        assert len(dba.shared_points(p, k)) > 0
        for m, tol in ((5, 1e-14), (2, 1e-12), (3, 1e-10), (4, 1e-10)):
            out, _, ident = dba.group_operator(p, k, z, mode=m, lam=1e-4, policy=1, tol=1e-12, max_iters=2000)
            assert ident
            a, b = (out[:4], base[m][:4]) if m == 4 else (out, base[m])
            assert rel(a, b) < tol, (k, m, rel(a, b))


@pytest.mark.parametrize("k", [1, 2])
def test_lm_trajectory_defaults(k):
    """SolverConfig defaults (pcg_tol 1e-6): same accept/reject sequence; costs
    within 1e-5 relative. With the inner solve stopped at 1e-6 the
    reference's own K = 1 vs K = 2 runs differ by up to ~1e-6 on this
    instance (reassociation only), so 1e-6 is the noise floor here."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024)
    cfg = dba.SolverConfig(max_iterations=8, workers=k)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-5, check_lambda=False)


def test_lm_pcg_counts_and_tallies():
    """With a coarse, decisive inner stop (pcg_tol 1e-4, as the reference's
    work-scaling test, tests/test_solver.cpp:571-576) the PCG iteration counts
    match the oracle within +-2, and the block-op tallies follow
    N_k (2 + 2 (1 + I + floor(I/50)))."""
    p = ring(12, 40, 6, seed=3)
    cfg = dba.SolverConfig(max_iterations=10, pcg_tol=1e-4, pcg_max_iters=2000)
    g = dba.lm_solve(p, cfg)
    o = O.lm_solve(p, cfg)
    _compare_histories(g, o, 1e-4)
    n = p.num_observations
    for a, b in zip(g.history, o.history):
        assert abs(a.pcg_iterations - b.pcg_iterations) <= 2
        i = a.pcg_iterations
        assert a.worker_block_ops[0] == n * (2 + 2 * (1 + i + i // 50))


def test_lm_fp32():
    """FP32 path, the reference's own protocol (tests/test_solver.cpp:530-562):
    both precisions cut the MSE by 1e3 and land within 2 %; the model
    evaluation itself (initial cost) matches the FP32 oracle to 1e-6. (Per
    iteration the reference's own FP32 K=1 vs K=2 runs already differ by
    1e-3..4e-2 through reassociation, so that is not a usable FP32 bar.)"""
    p64 = ring(14, 50, 6, seed=11)
    p32 = p64.astype(np.float32)
    s64 = O.lm_solve(p64, dba.SolverConfig(max_iterations=15))
    s32 = dba.lm_solve(p32, dba.SolverConfig(max_iterations=15, workers=2))
    n = p64.num_observations
    init = O.total_cost(p64) / (2 * n)
    m64, m32 = s64.cost / (2 * n), s32.cost / (2 * n)
    assert m64 < 1e-3 * init and m32 < 1e-3 * init
    assert abs(m32 - m64) <= 0.02 * max(m64, 1e-12) + 1e-9
    assert dba.total_cost(p32) == pytest.approx(O.total_cost(p32), rel=1e-6)


def test_lm_analytic_matches_oracle():
    p = ring(30, 300, 6, radius=1.0, noise=0.5, seed=9)
    cfg = dba.SolverConfig(max_iterations=8, jacobian=1, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


def test_lm_zero_residual_converges_in_one():
    """tests/test_solver.cpp:335-359. Pixels are the GPU model's own
    projections, so the start is an exact zero of its residual."""
    f = ProblemFactory(9)
    cams = np.stack([f.random_camera() for _ in range(2)])
    pts = np.stack([f.random_point() for _ in range(3)])
    cid = [c for c in range(2) for _ in range(3)]
    pid = [q for _ in range(2) for q in range(3)]
    p0 = dba.BAProblem.from_arrays(cams, pts, cid, pid, np.zeros((6, 2)))
    with ctx_for(p0) as c:
        proj = c.residuals()
    p = dba.BAProblem.from_arrays(cams, pts, cid, pid, proj.T)
    assert dba.total_cost(p) == 0.0
    st = dba.lm_solve(p)
    assert st.termination == "converged" and st.iteration == 1 and st.cost == 0.0 and st.history[0].accepted


def test_jet_value_lanes_equal_scalar_residual():
    """The batched jet values and the scalar model agree bit-for-bit
    (dba/problem.hpp:146-150 contract), on the GPU."""
    p = ring(40, 300, 6, noise=0.5)
    with ctx_for(p) as c:
        c.linearize()
        res, _ = c.jacobians()
        assert np.array_equal(res, c.residuals())


def test_full_size_first_iteration_properties():
    """Trafalgar-257-shaped instance (the bench workload, PCG capped at 500):
    linearize parity at full size, and the first LM step's cost/accept agree
    with the oracle to the truncated-PCG level (1e-3)."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=257, points=65132, num_observations=225911, seed=1,
                                                    pixel_noise=0.5))
    with ctx_for(p) as c:
        c.linearize()
        res, jac = c.jacobians()
        cfg = dba.SolverConfig()
        cost1, it, acc = c.probe_step(cfg.lambda0, cfg)
    r0, j0 = O.linearize(p)
    assert rel(res, r0) < 1e-13 and rel(jac, j0) < 1e-12
    secs, its = O.lm_probe_steps(p, dba.SolverConfig(workers=4), 1)
    st = O.lm_solve(p, dba.SolverConfig(max_iterations=1, workers=4))
    assert acc == st.history[0].accepted
    assert abs(cost1 - st.history[0].cost) <= 1e-3 * st.history[0].cost
    assert it == its[0]


def test_lm_reject_reuses_system_tallies():
    """tests/test_solver.cpp:428-455."""
    p = ring(8, 20, 4, seed=5)
    n = p.num_observations
    st = dba.lm_solve(p, dba.SolverConfig(lambda0=1e8, max_iterations=6))
    for r in st.history:
        assert r.worker_edges[0] == (2 * n if r.accepted else n)
    assert st.history[0].worker_edges[0] == 2 * n


def test_lm_stalled():
    """tests/test_solver.cpp:488-504."""
    p = ring(4, 8, 2)
    st = dba.lm_solve(p, dba.SolverConfig(lambda0=1e31, lambda_max=1e32, step_tol=0.0, max_iterations=50))
    assert st.termination == "stalled"


def test_lm_ring_down_monotone():
    """tests/test_solver.cpp:361-384."""
    p = ring(20, 80, 10)
    init = O.total_cost(p)
    st = dba.lm_solve(p, dba.SolverConfig(max_iterations=50))
    assert st.cost <= 0.1 * init
    last = init
    for r in st.history:
        if r.accepted:
            assert r.cost <= last * (1 + 1e-12)
            last = r.cost


def test_probe_step_matches_first_iteration():
    """The bench step (one LM iteration from x0, not committed) reproduces the
    first IterationRecord of a full solve."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024)
    cfg = dba.SolverConfig(max_iterations=1)
    st = dba.lm_solve(p, cfg)
    with ctx_for(p) as c:
        for _ in range(2):
            cost, it, acc = c.probe_step(cfg.lambda0, cfg)
            assert acc == st.history[0].accepted and it == st.history[0].pcg_iterations
            assert cost == pytest.approx(st.history[0].cost, rel=1e-12)


def test_full_size_venice_operator_properties():
    """venice-1778-shaped instance (5.0 M observations, E 1.2 GB, the bench's
    HBM-bound secondary): properties that hold at any size, where the oracle
    would take minutes. The reduced camera operator S of the graph path is
    symmetric, linear and positive definite; DPCG's answer satisfies the true
    residual bound; the first LM iteration agrees between K = 1 (graph DPCG)
    and K = 2 (host-driven DPCG over the in-process group) to the reference's
    own cross-K noise at pcg_tol 1e-6."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=1778, points=993923, num_observations=5001946, seed=1,
                                                    pixel_noise=0.5))
    m = p.num_cameras
    rng = np.random.default_rng(5)
    with dba.RankContext(0, 8) as c:
        c.upload(p)
        c.linearize()
        c.damp_factor(10.0, dba.DAMPING_DIAG_SCALED)  # well conditioned: DPCG converges tightly
        x, y = rng.standard_normal(9 * m), rng.standard_normal(9 * m)
        Sx, Sy = c.dse(x), c.dse(y)
        assert abs(y @ Sx - x @ Sy) <= 1e-12 * np.linalg.norm(y) * np.linalg.norm(Sx)
        assert rel(c.dse(2.0 * x - 3.0 * y), 2.0 * Sx - 3.0 * Sy) < 1e-12
        assert x @ Sx > 0 and y @ Sy > 0
        g = rng.standard_normal(9 * m)
        sol, it, conv = c.dpcg(g, 1e-10, 2000)
        assert conv and 0 < it < 2000
        assert np.linalg.norm(g - c.dse(sol)) <= 1e-8 * np.linalg.norm(g)
    s1 = dba.lm_solve(p, dba.SolverConfig(max_iterations=1))
    s2 = dba.lm_solve(p, dba.SolverConfig(max_iterations=1, workers=2), devices=[0])
    h1, h2 = s1.history[0], s2.history[0]
    assert len(dba.shared_points(p, 2)) == 1  # the boundary splits a point: the halo path runs
    assert h1.accepted == h2.accepted and h1.pcg_iterations == h2.pcg_iterations == 500
    assert abs(h1.cost - h2.cost) <= 1e-5 * h1.cost
    assert h2.worker_edges == [2 * 2500973, 2 * 2500973]


@pytest.mark.parametrize("k", [1, 2, 3])
def test_long_tiles_dse_and_lm(k):
    """Points observed by more than 128 cameras take the long-tile path
    (dse_long: one CTA per point, chunks of one tile), here mixed with shard
    boundaries inside such points: DSE vs the oracle at 1e-12, LM trajectory
    vs the oracle at the same K."""
    p = ring(220, 30, 150, seed=7, radius=1.0, noise=0.5, nobs=30 * 150 + 17)
    x = np.random.default_rng(2).standard_normal(9 * p.num_cameras)
    out, _, ident = dba.group_operator(p, k, x, mode=0, lam=1e-3, policy=0)
    orc, _ = O.dse(p, k, 1e-3, 0, x)
    assert ident and rel(out, orc) < 1e-12
    cfg = dba.SolverConfig(max_iterations=4, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


@pytest.mark.parametrize("variant", ["cluster-2-per-warp", "grid-barrier", "fold+step kernels"])
def test_graph_fold_step_variants(variant, monkeypatch):
    """The three fold + step forms of the graph DPCG (k_g_fsc for m <= 544,
    k_g_fs up to 4736 cameras, k_g_fold + k_g_step beyond) give the oracle's
    trajectory. m = 300 makes k_g_fsc fold two cameras per warp; the
    environment switches force the larger-m forms on the same instance."""
    if variant == "grid-barrier":
        monkeypatch.setenv("DBAG_FSC", "0")
    elif variant == "fold+step kernels":
        monkeypatch.setenv("DBAG_FSC", "0")
        monkeypatch.setenv("DBAG_FS", "0")
    p = ring(300, 900, 4, radius=1.0, noise=0.5, seed=11)
    cfg = dba.SolverConfig(max_iterations=4, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


def test_coupling_fp32_memory_lean_variant():
    """Row f4: FP64 solve with the coupling blocks stored in
    FP32. Not the reference's numerics — E carries ~6e-8 relative rounding,
    which this ill-conditioned ring amplifies to a few 1e-6 in the cost — so
    the bar is closeness to the FP64 path: S x within 1e-6, the same
    accept/reject sequence and costs within 1e-4 relative (the north star's
    FP32 bar) at tight PCG; K = 2 reproduces K = 1 of the same variant."""
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024, nobs=3197)
    x = np.random.default_rng(3).standard_normal(9 * p.num_cameras)
    outs = []
    for lean in (False, True):
        with dba.RankContext(0, 8, coupling_fp32=lean) as c:
            c.upload(p)
            c.linearize()
            c.damp_factor(1e-3, dba.DAMPING_DIAG_SCALED)
            outs.append(c.dse(x))
    assert 0 < rel(outs[1], outs[0]) < 1e-6
    cfg = dba.SolverConfig(max_iterations=6, pcg_tol=1e-12, pcg_max_iters=2000)
    a = dba.lm_solve(p, cfg)
    b = dba.lm_solve(p, dba.SolverConfig(max_iterations=6, pcg_tol=1e-12, pcg_max_iters=2000, coupling_fp32=True))
    _compare_histories(b, a, 1e-4, check_lambda=False)
    b2 = dba.lm_solve(p, dba.SolverConfig(max_iterations=6, pcg_tol=1e-12, pcg_max_iters=2000, coupling_fp32=True,
                                          workers=2))
    # K = 2 reassociates the camera sums and the PCG dots; this ring amplifies
    # that rounding like the FP32 E rounding above (measured 1.2e-6 at
    # iteration 4)
    _compare_histories(b2, b, 1e-5, check_lambda=False)


@pytest.mark.parametrize("k", [1, 2])
def test_unobserved_camera_and_point(k):
    """A camera and a point no observation references (BAProblem::validate
    warns, dba/problem.hpp:231-255): their parameters stay untouched and the
    trajectory matches the oracle; an edge-less problem fails like
    partition_edges (K > N, dba/partition.hpp:76-103)."""
    base = ring(12, 80, 4, seed=9, radius=1.0, noise=0.5)
    cams, pts, cid, pid, px, py, _ = base.arrays()
    cams2, pts2 = np.vstack([cams, cams[0] + 0.01]), np.vstack([pts, pts[0] + 0.02])
    p = dba.BAProblem.from_arrays(cams2, pts2, cid, pid, np.stack([px, py], 1))
    assert len(p.validate()) == 2
    cfg = dba.SolverConfig(max_iterations=4, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    g, o = dba.lm_solve(p, cfg), O.lm_solve(p, cfg)
    _compare_histories(g, o, 1e-9)
    assert np.array_equal(g.x_c.reshape(-1, 9)[12], cams2[12]) and np.array_equal(g.x_p.reshape(-1, 3)[80], pts2[80])
    assert np.abs(g.x_c - o.x_c).max() < 1e-6 and np.abs(g.x_p - o.x_p).max() < 1e-8
    # lambda0 = 0: the reference factors the unobserved point's zero block
    # too and names it (dba/block_matrix.hpp:123-134; C before B)
    with dba.RankContext(0, 8) as c:
        c.upload(p)
        c.linearize()
        for policy in (dba.DAMPING_IDENTITY, dba.DAMPING_DIAG_SCALED):
            with pytest.raises(dba.SingularBlockError) as ei:
                c.damp_factor(0.0, policy)
            assert ei.value.block_index == 80 and ei.value.block_size == 3
        c.damp_factor(1e-4, dba.DAMPING_DIAG_SCALED)  # damped: factorable
    # inside LM the failure is a reject (dba/solver.hpp:426-430), as in the oracle
    cfg0 = dba.SolverConfig(max_iterations=2, workers=k, lambda0=0.0)
    g0, o0 = dba.lm_solve(p, cfg0), O.lm_solve(p, cfg0)
    assert [r.accepted for r in g0.history] == [r.accepted for r in o0.history] == [False, False]
    empty = dba.BAProblem.from_arrays(cams[:2], pts[:3], np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 2)))
    with pytest.raises(dba.InvalidArgumentError):
        dba.lm_solve(empty, dba.SolverConfig(max_iterations=3))


@pytest.mark.parametrize("k", [1, 2])
def test_host_driven_dpcg_loop(k, monkeypatch):
    """DBAG_PCG=host: the one-launch-per-step DPCG loop (a host round trip per
    PCG iteration) kept as the reference implementation of the device-driven
    forms; same oracle trajectory, split points included."""
    monkeypatch.setenv("DBAG_PCG", "host")
    p = ring(40, 400, 8, radius=1.0, noise=0.5, seed=2024, nobs=3197)
    cfg = dba.SolverConfig(max_iterations=4, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("lean", [False, True])
def test_memory_pool_matches_prediction(lean):
    """Predicted-size pool: upload reserves exactly the
    host-side prediction in one allocation and fills it; the device's free
    memory drops by that much (up to the driver's 2 MiB granularity); the
    solve afterwards allocates nothing more than the per-context scratch."""
    import torch
    p = ring(60, 3000, 6, noise=0.5, seed=7)
    pred = dba.predict_memory(p, coupling_fp32=lean)
    with dba.RankContext(0, 8, coupling_fp32=lean) as c:
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info(0)[0]
        c.upload(p)
        assert c.memory_pool() == (pred, pred)
        free1 = torch.cuda.mem_get_info(0)[0]
        assert pred <= free0 - free1 <= pred + 4 * 2**20
        c.linearize()
        c.damp_factor(1e-4, dba.DAMPING_DIAG_SCALED)
        c.rhs()
        c.pcg(1e-6, 100)
        assert free1 - torch.cuda.mem_get_info(0)[0] <= 4 * 2**20
        c.upload(p)  # re-upload replaces the pool
        assert c.memory_pool() == (pred, pred)
    for k in (2, 3):
        preds = [dba.predict_memory(p, k, r, coupling_fp32=lean) for r in range(k)]
        assert max(preds) < pred


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2])
def test_batched_assembly_scratch(monkeypatch, k):
    """The row-based assembly (DBAG_LIN=rows: Jb, the per-edge rows linearize
    hands to two assembly kernels) in batches of whole points
    (DBAG_JB_BATCH slots): C, w and E are computed exactly as in one batch; B
    and v add the batches' double-precision sums, so they agree to rounding;
    the LM trajectory matches; the pool shrinks accordingly."""
    monkeypatch.setenv("DBAG_LIN", "rows")
    p = ring(50, 2000, 6, noise=0.5, seed=11)
    out = {}
    for cap in (0, 700):
        if cap:
            monkeypatch.setenv("DBAG_JB_BATCH", str(cap))
        else:
            monkeypatch.delenv("DBAG_JB_BATCH", raising=False)
        with dba.RankContext(0, 8) as c:
            c.upload(p)
            c.linearize()
            out[cap] = [np.array(a, copy=True) for a in c.system()]
            out[cap].append(c.memory_pool()[0])
        out[cap].append(dba.lm_solve(p, dba.SolverConfig(max_iterations=4, pcg_tol=1e-10, pcg_max_iters=1000,
                                                         workers=k)))
    B0, C0, E0, v0, w0, pool0, st0 = out[0]
    B1, C1, E1, v1, w1, pool1, st1 = out[700]
    assert np.array_equal(C1, C0) and np.array_equal(w1, w0) and np.array_equal(E1, E0)
    assert rel(B1, B0) < 1e-14 and rel(v1, v0) < 1e-14
    assert pool0 - pool1 >= (p.num_observations - 700 - 200) * 28 * 8
    _compare_histories(st1, st0, 1e-9, check_lambda=False)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["cluster", "grid-barrier", "fold+step kernels"])
@pytest.mark.parametrize("k", [1, 2])
def test_dpcg_pq_breakdown(variant, k, monkeypatch):
    """p'q <= 0 stops DPCG with PcgBreakdownError (dba/solver.hpp:238-241),
    uniformly over the graph's fold + step forms and the K > 1 loop: an
    indefinite reduced system S = I - E C^-1 E^T (B = C = I, large E) and a
    right-hand side along a negative direction of S."""
    if variant != "cluster":
        monkeypatch.setenv("DBAG_FSC", "0")
    if variant == "fold+step kernels":
        monkeypatch.setenv("DBAG_FS", "0")
    p = ProblemFactory(123).random_problem(2, 3, 6)
    m, n, N = p.num_cameras, p.num_points, p.num_observations
    E = np.random.default_rng(5).uniform(-3, 3, (N, 27))
    blocks = (np.tile(np.eye(9), (m, 1, 1)), np.tile(np.eye(3), (n, 1, 1)), E)
    cams, pts, cid, pid, *_ = p.arrays()
    Ed = dense_coupling(E.reshape(N, 9, 3), cid, pid, m, n)
    S = np.eye(9 * m) - Ed @ Ed.T
    w, V = np.linalg.eigh(S)
    assert w[0] < 0
    with pytest.raises(dba.PcgBreakdownError):
        dba.group_operator(p, k, V[:, 0], mode=1, blocks=blocks, tol=1e-12, max_iters=100)


@pytest.mark.parametrize("shape", ["chunks", "long-tiles"])
@pytest.mark.parametrize("k", [1, 2])
def test_streaming_pass_variant(shape, k, monkeypatch):
    """The opt-in persistent TMA-fed DSE pass (stream.cuh, DBAG_STREAM=1:
    cp.async.bulk record + C-factor stages, mbarrier ring, gather warps) gives
    the oracle's trajectory in the graph DPCG (K = 1) and in the run-ahead
    loop of K = 2 ranks (halo points), with ordinary chunks and with long
    tiles (points observed by more than 128 cameras)."""
    monkeypatch.setenv("DBAG_STREAM", "1")
    monkeypatch.setenv("DBAG_NST", "2")
    if shape == "chunks":
        p = ring(60, 800, 6, radius=1.0, noise=0.5, seed=4, nobs=800 * 6 + 13)
    else:
        p = ring(220, 30, 150, seed=7, radius=1.0, noise=0.5, nobs=30 * 150 + 17)
    cfg = dba.SolverConfig(max_iterations=4, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


@pytest.mark.parametrize("k", [2, 3, 5])
def test_peer_graph_dpcg_matches_host_loop(k, monkeypatch):
    """K > 1 DPCG as one CUDA graph per rank with the device-side peer
    all-reduces (peer.cuh: epoch handshake over peer memory, ascending-rank
    fold) against the host-driven run-ahead loop over the group collectives
    (DBAG_PEER=0), with shard boundaries inside points (halo): same accept
    sequence, costs to 1e-9 (the graph's fused fold + step reassociates the
    rho / |r|^2 reductions, so the tight-tolerance PCG may stop an iteration
    apart); and the oracle's trajectory at the same K."""
    p = ring(40, 600, 6, radius=1.0, noise=0.5, seed=9, nobs=600 * 6 - 7)
    assert len(dba.shared_points(p, k)) > 0
    cfg = dba.SolverConfig(max_iterations=4, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    g = dba.lm_solve(p, cfg, devices=[0])
    monkeypatch.setenv("DBAG_PEER", "0")
    h = dba.lm_solve(p, cfg, devices=[0])
    _compare_histories(g, h, 1e-9)
    _compare_histories(g, O.lm_solve(p, cfg), 1e-9)


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("mode", [0, 1])
def test_fused_linearize_assembly_matches_rows(k, mode, monkeypatch):
    """The fused linearize + assemble pass (lin.cuh: point sums in the chunk,
    camera terms folded per (chunk, camera) partial) against the row-based
    two-kernel assembly (DBAG_LIN=rows) and the oracle: C, w, E bit-identical
    (same per-point association), B and v to double-sum rounding, with long
    tiles (points seen by more than 128 cameras) and K = 2 halos; LM
    trajectories equal."""
    p = ring(200, 40, 130, seed=5, radius=1.0, noise=0.5, nobs=40 * 130 - 9)
    sysm = {}
    for lin in ("fused", "rows"):
        if lin == "rows":
            monkeypatch.setenv("DBAG_LIN", "rows")
        with dba.RankContext(0, 8) as c:
            c.upload(p, mode)
            c.linearize()
            sysm[lin] = [np.array(a, copy=True) for a in c.system()]
    (B0, C0, E0, v0, w0), (B1, C1, E1, v1, w1) = sysm["fused"], sysm["rows"]
    if mode == 0:  # jets: IEEE-rn operations only, identical in both kernels
        assert np.array_equal(C0, C1) and np.array_equal(w0, w1) and np.array_equal(E0, E1)
    else:  # the closed form's products may contract differently per kernel
        assert rel(C0, C1) < 1e-14 and rel(w0, w1) < 1e-14 and rel(E0, E1) < 1e-14
    assert rel(B0, B1) < 1e-14 and rel(v0, v1) < 1e-14
    Bo, Co, Eo, vo, wo = O.assemble(p, mode=mode)
    for a, b in ((B0, Bo), (C0, Co), (E0, Eo), (v0, vo), (w0, wo)):
        assert rel(a, np.asarray(b).reshape(a.shape)) < 1e-12
    monkeypatch.delenv("DBAG_LIN")
    cfg = dba.SolverConfig(max_iterations=3, workers=k, pcg_tol=1e-12, pcg_max_iters=2000,
                           jacobian=dba.JACOBIAN_ANALYTIC if mode else dba.JACOBIAN_AUTODIFF)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)


def test_peer_graph_timeout_names_absent_rank():
    """The device-side peer waits of the K > 1 DPCG graph are bounded by the
    collective timeout (SolverConfig::collective_timeout, dba/solver.hpp:54):
    a rank whose peer never enters the solve gets CollectiveError naming the
    absent rank (dba/comms.hpp:136-193 semantics) instead of spinning
    forever; the graph drains once the first wait gives up."""
    import time
    p = ring(30, 300, 6, radius=1.0, noise=0.5, seed=21, nobs=300 * 6 - 5)
    g = dba.WorkerGroup(2, timeout_ms=300)
    ctx = [dba.RankContext(0, 8, group=(g, r)) for r in range(2)]
    out = {}

    def body(r):
        c = ctx[r]
        c.upload(p)
        c.linearize()
        c.damp_factor(1e-4)
        c.rhs()
        out[r] = c.pcg(1e-12, 200)

    dba.run_on_workers(g, body)  # both ranks: peer sites and graphs built
    assert out[0] == out[1] and out[0][0] > 0
    t0 = time.monotonic()
    with pytest.raises(dba.CollectiveError, match=r"rank\(s\) 1 did not arrive"):
        ctx[0].pcg(1e-12, 200)  # rank 1 never joins
    assert time.monotonic() - t0 < 30.0
    for c in ctx:
        c.close()
    g.close()


def test_peer_site_selftest_fallback(monkeypatch):
    """Every peer site is verified before use (k_peer_selftest: two
    all-reduces of closed-form values per slice, agreed over the ranks); a
    failed check (forced here) makes every rank fall back to the
    host-driven loop, with the same oracle trajectory."""
    p = ring(30, 300, 6, radius=1.0, noise=0.5, seed=21, nobs=300 * 6 - 5)
    cfg = dba.SolverConfig(max_iterations=3, workers=2, pcg_tol=1e-12, pcg_max_iters=2000)
    ok = dba.lm_solve(p, cfg, devices=[0])
    monkeypatch.setenv("DBAG_PEER_SELFTEST_FAIL", "1")
    fb = dba.lm_solve(p, cfg, devices=[0])
    o = O.lm_solve(p, cfg)
    _compare_histories(ok, o, 1e-9)
    _compare_histories(fb, o, 1e-9)


@pytest.mark.parametrize("k", [1, 2])
def test_chunks_with_many_cameras(k):
    """Chunks whose points are seen by more than 32 distinct cameras (the
    unstaged gather path of the pass, camera vectors read per slot) and by
    more than 14 (the fold runs more than one round of (camera, component)
    items per thread): 100 cameras, points of 40-70 observations each, DSE
    vs the oracle at 1e-12 and the LM trajectory at the same K."""
    rng = np.random.default_rng(17)
    base = ring(100, 2, 2, seed=3, radius=1.0, noise=0.5)
    cams = base.arrays()[0]
    pts = rng.uniform(-0.3, 0.3, (60, 3))
    cid, pid = [], []
    for q in range(60):
        obs = rng.choice(100, size=int(rng.integers(40, 71)), replace=False)
        cid += sorted(obs.tolist())
        pid += [q] * len(obs)
    cid, pid = np.array(cid, np.int32), np.array(pid, np.int32)
    P = np.zeros((len(cid), 2))
    p0 = dba.BAProblem.from_arrays(cams, pts, cid, pid, P)
    # pixels = the projection plus noise (a well-posed problem)
    r, _ = O.linearize(p0)  # r = projection - pixel, pixel = 0
    P = np.asarray(r).T + rng.uniform(-0.5, 0.5, P.shape)
    p = dba.BAProblem.from_arrays(cams, pts, cid, pid, P)
    x = rng.uniform(-1, 1, 9 * p.num_cameras)
    out, _, ident = dba.group_operator(p, k, x, mode=0, lam=1e-3, policy=0)
    orc, _ = O.dse(p, k, 1e-3, 0, x)
    assert ident and rel(out, orc) < 1e-12
    cfg = dba.SolverConfig(max_iterations=3, workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
    _compare_histories(dba.lm_solve(p, cfg), O.lm_solve(p, cfg), 1e-9)
