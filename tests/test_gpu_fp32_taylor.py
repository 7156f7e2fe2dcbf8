"""FP32 operator parity against the FP32 oracle (the reference's Scalar =
float instantiation: tests/test_jet.cpp:354-367, tests/test_solver.cpp:530-562)
and the small-angle Taylor branch of the rotation coefficients
(dba/problem.hpp:75-118; tests/test_jet.cpp:143-171, 303-352), on the GPU."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba
from oracle import oracle as O
from tests.dense import rel
from tests.factory import ProblemFactory

pytestmark = pytest.mark.gpu


def ctx_for(p, mode=0):
    c = dba.RankContext(0, p.precision)
    c.upload(p, mode)
    return c


def ring32(cams, pts, q, seed=1, noise=0.5):
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=cams, points=pts, obs_per_point=q, seed=seed,
                                                    pixel_noise=noise, circle_radius=1.0))
    return p.astype(np.float32)


# FP32 bars: the operators differ from the oracle only in association /
# FMA contraction of the same float operations, i.e. a few float ulps
# relative to the operand magnitudes.
F32_LIN, F32_SYS, F32_DSE = 2e-6, 2e-5, 5e-5


@pytest.mark.parametrize("mode", [0, 1])
def test_fp32_linearize_matches_fp32_oracle(mode):
    p = ring32(30, 200, 6, seed=3)
    with ctx_for(p, mode) as c:
        c.linearize()
        res, jac = c.jacobians()
    r0, j0 = O.linearize(p, mode=mode)
    assert res.dtype == np.float32 and r0.dtype == np.float32
    px, py = p.arrays()[4:6]
    for e in range(res.shape[1]):
        # r = projection - pixel cancels: float ulps scale with |projection|
        scale = max(1.0, float(np.hypot(px[e], py[e])), float(np.linalg.norm(r0[:, e])))
        assert np.linalg.norm(res[:, e] - r0[:, e]) <= F32_LIN * scale
        assert np.linalg.norm(jac[:, :, e] - j0[:, :, e]) <= F32_LIN * max(1.0, np.linalg.norm(j0[:, :, e]))


def test_fp32_assembly_and_cost_match_fp32_oracle():
    p = ring32(24, 150, 5, seed=8)
    with ctx_for(p) as c:
        c.linearize()
        B, Cb, E, v, w = c.system()
        cost, _ = c.cost()
    B0, C0, E0, v0, w0 = O.assemble(p)
    for a, b in ((B, B0), (Cb, C0), (E, E0), (v, v0), (w, w0)):
        assert a.dtype == np.float32 and rel(a, b) < F32_SYS
    assert cost == pytest.approx(O.total_cost(p), rel=1e-6)


@pytest.mark.parametrize("k", [1, 2])
def test_fp32_dse_matches_fp32_oracle(k):
    p = ring32(20, 120, 5, seed=12)
    x = np.random.default_rng(4).uniform(-1, 1, 9 * p.num_cameras).astype(np.float32)
    out, _, ident = dba.group_operator(p, k, x, mode=0, lam=1e-3, policy=1)
    ref, oident = O.dse(p, k, 1e-3, 1, x)
    assert ident and oident and out.dtype == np.float32 and ref.dtype == np.float32
    assert rel(out, ref) < F32_DSE


def small_angle_problem(scale, dtype, seed=21):
    """Cameras near the identity rotation (|aa| ~ scale), points in front of
    them (P_z < 0 after the translation), BAL-normalized focal."""
    rng = np.random.default_rng(seed)
    m, n, q = 6, 40, 4
    cams = np.zeros((m, 9))
    cams[:, :3] = rng.uniform(-1, 1, (m, 3)) * scale
    cams[:, 3:6] = rng.uniform(-0.1, 0.1, (m, 3)) + [0, 0, -4.0]
    cams[:, 6] = rng.uniform(1.0, 2.0, m)
    cams[:, 7] = rng.uniform(-0.1, 0.1, m)
    cams[:, 8] = rng.uniform(-0.05, 0.05, m)
    truth = rng.uniform(-0.5, 0.5, (n, 3))
    cid = np.array([(p + j) % m for p in range(n) for j in range(q)], np.int32)
    pid = np.repeat(np.arange(n, dtype=np.int32), q)
    # observations: projections of the true points (+ 1e-3 noise); stored
    # points perturbed, so the solve has work to do
    pix = np.stack([O.residual(cams[c], truth[t], [0.0, 0.0]) for c, t in zip(cid, pid)])
    pix += rng.uniform(-1e-3, 1e-3, pix.shape)
    pts = truth + rng.uniform(-0.02, 0.02, truth.shape)
    return dba.BAProblem.from_arrays(cams, pts, cid, pid, pix, dtype=dtype)


@pytest.mark.parametrize("dtype,scale,tol", [(np.float64, 1e-8, 1e-12), (np.float32, 1e-3, 2e-6)],
                         ids=["fp64-t1e-16", "fp32-t1e-6"])
def test_taylor_branch_linearize_and_cost(dtype, scale, tol):
    """theta^2 below rotation_taylor_threshold (1e-12 FP64, 1e-4 FP32,
    dba/problem.hpp:75-82): the GPU takes the 2nd-order Taylor branch of
    c, s1, c2 and their t-derivatives exactly where the oracle does; its
    residuals and Jacobians (autodiff and analytic) match the oracle's."""
    p = small_angle_problem(scale, dtype)
    cams = p.arrays()[0]
    t = (cams[:, :3].astype(np.float64) ** 2).sum(1)
    thr = 1e-12 if dtype == np.float64 else 1e-4
    assert np.all(t < thr) and np.all(t > 0)
    for mode in (0, 1):
        with ctx_for(p, mode) as c:
            c.linearize()
            res, jac = c.jacobians()
            cost, bad = c.cost()
        r0, j0 = O.linearize(p, mode=mode)
        assert bad < 0
        assert rel(res, r0) < tol and rel(jac, j0) < tol
        assert cost == pytest.approx(O.total_cost(p), rel=tol * 10)


def test_taylor_branch_lm_trajectory_fp64():
    """A short LM solve that starts inside the Taylor branch: same accept
    sequence and costs as the oracle (tight PCG, K-equivalence protocol)."""
    p = small_angle_problem(1e-8, np.float64)
    cfg = dba.SolverConfig(max_iterations=5, pcg_tol=1e-12, pcg_max_iters=2000)
    g, o = dba.lm_solve(p, cfg), O.lm_solve(p, cfg)
    assert [r.accepted for r in g.history] == [r.accepted for r in o.history]
    for a, b in zip(g.history, o.history):
        assert abs(a.cost - b.cost) <= 1e-9 * max(b.cost, 1e-300)
