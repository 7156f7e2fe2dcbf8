"""The reference's acceptance runner (tests/acceptance.cpp:1-635,
`dba_acceptance`) on the B200 path: the same eight criteria, instances,
tolerances and PASS/FAIL report, with every solve / operator evaluated by
libdbag.so on the GPU and the dense checks done in numpy (tests/dense.py,
the restatement of tests/oracles.hpp). Test infrastructure: run it as

    python tests/acceptance.py [--criterion N]... [--data-dir PATH]

(exit 0 when every selected criterion passes, 1 otherwise, 2 on a bad
argument), or through tests/test_acceptance.py (`-m gpu`).

Deviations, each forced by this environment and named in the report:
* ProblemFactory (tests/oracles.hpp:147-236) is restated with numpy's RNG
  (tests/factory.py): same distributions, not the same draws.
* Criteria 5 and 7 replay published BAL files (problem-49/21/16-...-pre.txt)
  from --data-dir / DBA_DATA_DIR; there is no network here, so without the
  files they FAIL exactly as the reference does ("dataset file ... not
  found").
* Criterion 8's SpMV-adjointness item: the product has no standalone E / E^T
  SpMV (both live inside the fused DSE pass, dse.cuh), so the adjointness is
  checked on the operator that pass applies, S = B_d - E C_d^-1 E^T:
  y.(S x) against x.(S y) at the reference's 1e-12.

Criteria 1 and 6 are borderline for the reference on its own instances:
the CPU restatement of the reference (oracle/) spreads by 9.3e-9 / 9.5e-9
in final parameters between K = 1 and K = 2 / 4 (tolerance 1e-8), and its
K = 4 work-scaling solve takes 330 PCG iterations in LM iteration 5 where
K = 1 takes 279 (18 % block-op deviation, tolerance 5 %) — the runner
reports what it measures; tests/test_acceptance.py holds the GPU to the
reference's own numbers there.
"""
import argparse
import os
import sys

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2112_01349_b200 as dba  # noqa: E402
from paper_2112_01349_b200 import bal_io  # noqa: E402
from tests.dense import damp_dense, dense_blockdiag, dense_coupling, fd_jacobian, residual_reference  # noqa: E402
from tests.factory import ProblemFactory  # noqa: E402

DATA_DIR = "data"

# (label, file, published MSE under the calibrated cost / 2N convention),
# tests/acceptance.cpp:51-56
LADYBUG49 = ("Ladybug-49", "problem-49-7776-pre.txt", 0.42)
TRAFALGAR21 = ("Trafalgar-21", "problem-21-11315-pre.txt", 0.83)
DUBROVNIK16 = ("Dubrovnik-16", "problem-16-22106-pre.txt", 0.22)

NAMES = {
    1: "K-equivalence of the distributed solve",
    2: "auto-diff Jacobians vs finite differences",
    3: "DSE vs dense Schur oracle",
    4: "DPCG vs dense direct solve",
    5: "MSE reproduction on BAL datasets",
    6: "per-worker work scales as 1/K",
    7: "fp32/fp64 reach the same MSE",
    8: "property suites",
}


class Outcome:
    """tests/acceptance.cpp:27-36."""

    def __init__(self):
        self.ok = True
        self.details = []

    def fail(self, msg):
        self.ok = False
        self.details.append(msg)

    def note(self, msg):
        self.details.append(msg)


def fmt(v):
    return f"{v:.3e}"


def load_dataset(spec, out, dtype=np.float64):
    """tests/acceptance.cpp:58-71: a missing file is a failure."""
    label, fname, _ = spec
    path = os.path.join(DATA_DIR, fname)
    if not os.path.isfile(path):
        out.fail(f"{label}: dataset file {path} not found; place the BAL file there (see README, Datasets)")
        return None
    return bal_io.parse_bal(path, dtype=dtype)


def acceptance_synthetic():
    """tests/acceptance.cpp:79-100: 200 / 800 / 8000, radius-1 ring, seed
    2024, U(-0.5, 0.5) pixel noise from a second mt19937_64(2024) stream in
    edge order (the generator's pixel_noise extension, bit-identical)."""
    return dba.generate_synthetic(dba.SyntheticOptions(cameras=200, points=800, obs_per_point=10, seed=2024,
                                                       circle_radius=1.0, pixel_noise=0.5))


def check_k_equivalence(label, problem, out):
    """tests/acceptance.cpp:107-167: K = 1, 2, 4 at pcg_tol 1e-12 / 2000:
    final parameters 1e-8 (rel. inf-norm), accepted-cost trajectories 1e-10."""
    runs = []
    for k in (1, 2, 4):
        cfg = dba.SolverConfig(workers=k, pcg_tol=1e-12, pcg_max_iters=2000)
        runs.append((k, dba.lm_solve(problem, cfg, devices=[0])))
    ref = runs[0][1]
    scale = max(1.0, np.abs(ref.x_c).max(initial=0.0), np.abs(ref.x_p).max(initial=0.0))
    ref_costs = [r.cost for r in ref.history if r.accepted]
    for k, st in runs[1:]:
        dparam = max(np.abs(st.x_c - ref.x_c).max(initial=0.0), np.abs(st.x_p - ref.x_p).max(initial=0.0)) / scale
        if dparam > 1e-8:
            out.fail(f"{label}: K={k} final parameters differ from K=1 by {fmt(dparam)} rel inf-norm (tol 1e-8)")
        else:
            out.note(f"{label}: K={k} param agreement {fmt(dparam)} (tol 1e-8)")
        costs = [r.cost for r in st.history if r.accepted]
        if len(costs) != len(ref_costs):
            out.fail(f"{label}: K={k} took {len(costs)} accepted steps vs {len(ref_costs)} at K=1")
            continue
        worst = max((abs(a - b) / max(1.0, b) for a, b in zip(costs, ref_costs)), default=0.0)
        if worst > 1e-10:
            out.fail(f"{label}: K={k} accepted-cost trajectories differ by {fmt(worst)} rel (tol 1e-10)")
        else:
            out.note(f"{label}: K={k} cost-trajectory agreement {fmt(worst)} (tol 1e-10)")


def criterion_1():
    out = Outcome()
    check_k_equivalence("synthetic-200/800/8000", acceptance_synthetic(), out)
    ladybug = load_dataset(LADYBUG49, out)
    if ladybug is not None:
        check_k_equivalence(LADYBUG49[0], ladybug, out)
    return out


def criterion_2():
    """tests/acceptance.cpp:178-220: 1000 random (camera, point, pixel)
    edges, GPU auto-diff Jacobians (the JetVector path, k_lin_chunk) vs
    central differences of the straight-line residual, rel. error with a
    max(1, |fd|) floor < 1e-6. The edges are evaluated as one 1000-edge
    problem (edge i: camera i, point i) — each edge's jets depend only on
    its own camera and point."""
    out = Outcome()
    f = ProblemFactory(12345)
    cams = np.stack([f.random_camera() for _ in range(1000)])
    pts = np.stack([f.random_point() for _ in range(1000)])
    pix = f.u(-50, 50, (1000, 2))
    ids = np.arange(1000, dtype=np.int32)
    p = dba.BAProblem.from_arrays(cams, pts, ids, ids, pix)
    with dba.RankContext(0, 8) as ctx:
        ctx.upload(p, dba.JACOBIAN_AUTODIFF)
        ctx.linearize()
        _, jac = ctx.jacobians()
    worst = 0.0
    for e in range(1000):
        fd = fd_jacobian(residual_reference, cams[e], pts[e], pix[e])
        worst = max(worst, float(np.max(np.abs(jac[:, :, e] - fd) / np.maximum(1.0, np.abs(fd)))))
    out.note(f"max relative auto-diff vs finite-difference error over 1000 edges: {fmt(worst)} (tol 1e-6)")
    if not worst < 1e-6:
        out.fail("Jacobian mismatch above tolerance")
    return out


def small_system(f, index, normalized=False, lam=1e-3):
    """tests/acceptance.cpp:222-249: m <= 5 cameras, n <= 8 points, the
    damped (identity, lambda 1e-3) dense B, C and E of the assembled system —
    here the GPU's own assembly (RankContext.system, K = 1)."""
    cams = 2 + index % 4
    pts = 3 + index % 6
    edges = max(cams, pts) + 3 + index % 5
    p = f.random_problem(cams, pts, edges, normalized=normalized)
    with dba.RankContext(0, 8) as ctx:
        ctx.upload(p)
        ctx.linearize()
        B, Cb, E, _, _ = ctx.system()
    _, _, cid, pid, *_ = p.arrays()
    b = damp_dense(dense_blockdiag(B), lam, 0)
    c = damp_dense(dense_blockdiag(Cb), lam, 0)
    e = dense_coupling(E, cid, pid, cams, pts)
    return p, b, c, e


def criterion_3():
    """tests/acceptance.cpp:279-312: 50 problems, K in {1, 2, 3}: every
    rank's DSE output vs the dense Schur operator applied to x, < 1e-10."""
    out = Outcome()
    f = ProblemFactory(777)
    rng = np.random.default_rng(31337)
    worst = 0.0
    identical = True
    for trial in range(50):
        p, b, c, e = small_system(f, trial)
        x = rng.uniform(-1, 1, b.shape[0])
        expected = b @ x - e @ np.linalg.solve(c, e.T @ x)
        for k in (1, 2, 3):
            r, _, ident = dba.group_operator(p, k, x, mode=0, lam=1e-3, policy=dba.DAMPING_IDENTITY)
            identical &= ident
            worst = max(worst, float(np.linalg.norm(r - expected) / max(1.0, np.linalg.norm(expected))))
    out.note(f"max DSE vs dense Schur relative error over 50 problems, K in {{1,2,3}}: {fmt(worst)} (tol 1e-10)")
    if not identical:
        out.fail("DSE results differ across ranks")
    if not worst < 1e-10:
        out.fail("DSE deviates from the dense oracle")
    return out


def criterion_4():
    """tests/acceptance.cpp:314-354: 50 unit-focal problems, DPCG (tol 1e-12,
    1000 iterations) at K in {1, 2, 3} vs the dense direct solve of the
    Schur system, < 1e-8."""
    out = Outcome()
    f = ProblemFactory(888)
    rng = np.random.default_rng(4242)
    worst = 0.0
    identical = True
    for trial in range(50):
        p, b, c, e = small_system(f, trial, normalized=True)
        schur = b - e @ np.linalg.solve(c, e.T)
        g = rng.uniform(-1, 1, schur.shape[0])
        direct = np.linalg.solve(schur, g)
        for k in (1, 2, 3):
            x, _, ident = dba.group_operator(p, k, g, mode=1, lam=1e-3, policy=dba.DAMPING_IDENTITY, tol=1e-12,
                                             max_iters=1000)
            identical &= ident
            worst = max(worst, float(np.linalg.norm(x - direct) / max(1.0, np.linalg.norm(direct))))
    out.note(f"max DPCG vs dense direct-solve relative error: {fmt(worst)} (tol 1e-8)")
    if not identical:
        out.fail("DPCG results differ across ranks")
    if not worst < 1e-8:
        out.fail("DPCG deviates from the dense direct solve")
    return out


def check_mse(spec, out):
    """tests/acceptance.cpp:356-372."""
    p = load_dataset(spec, out)
    if p is None:
        return
    st = dba.lm_solve(p, dba.SolverConfig(), devices=[0])
    n = p.num_observations
    mse = dba.mse_from_cost(st.cost, n, dba.MSE_HALF_PER_OBSERVATION)
    mse_n = dba.mse_from_cost(st.cost, n, dba.MSE_PER_OBSERVATION)
    rel = abs(mse - spec[2]) / spec[2]
    out.note(f"{spec[0]}: final MSE {fmt(mse)} (cost/2N, calibrated) / {fmt(mse_n)} (cost/N); published "
             f"{fmt(spec[2])}, deviation {fmt(100 * rel)}% (tol 10%)")
    if rel > 0.10:
        out.fail(f"{spec[0]}: MSE outside the 10% band")


def criterion_5():
    out = Outcome()
    for spec in (LADYBUG49, TRAFALGAR21, DUBROVNIK16):
        check_mse(spec, out)
    return out


def criterion_6():
    """tests/acceptance.cpp:382-431: 100 / 400 / 10 synthetic (seed 99),
    5 LM iterations at pcg_tol 1e-4, K = 1 vs K = 4: every worker's edge and
    block-op tallies within 5 % of a quarter of K = 1's."""
    out = Outcome()
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=100, points=400, obs_per_point=10, seed=99))
    k1 = dba.lm_solve(p, dba.SolverConfig(max_iterations=5, pcg_tol=1e-4), devices=[0])
    k4 = dba.lm_solve(p, dba.SolverConfig(max_iterations=5, pcg_tol=1e-4, workers=4), devices=[0])
    if len(k1.history) != len(k4.history):
        out.fail(f"K=1 and K=4 ran different iteration counts ({len(k1.history)} vs {len(k4.history)})")
        return out
    worst = 0.0
    for a, b in zip(k1.history, k4.history):
        eq, oq = a.worker_edges[0] / 4.0, a.worker_block_ops[0] / 4.0
        for r in range(4):
            worst = max(worst, abs(b.worker_edges[r] - eq) / eq)
            if oq > 0:
                worst = max(worst, abs(b.worker_block_ops[r] - oq) / oq)
    out.note(f"worst per-worker deviation from one quarter of the K=1 edge-proportional work: "
             f"{fmt(100 * worst)}% (tol 5%)")
    if worst > 0.05:
        out.fail("per-worker work does not scale as 1/K")
    return out


def criterion_7():
    """tests/acceptance.cpp:433-458: Trafalgar-21 in FP64 and FP32, final
    MSE within 2 %."""
    out = Outcome()
    p64 = load_dataset(TRAFALGAR21, out)
    if p64 is None:
        return out
    p32 = load_dataset(TRAFALGAR21, out, dtype=np.float32)
    s64 = dba.lm_solve(p64, dba.SolverConfig(), devices=[0])
    s32 = dba.lm_solve(p32, dba.SolverConfig(), devices=[0])
    n = p64.num_observations
    m64 = dba.mse_from_cost(s64.cost, n)
    m32 = dba.mse_from_cost(s32.cost, n)
    rel = abs(m32 - m64) / m64
    out.note(f"Trafalgar-21 final MSE: fp64 {fmt(m64)}, fp32 {fmt(m32)}, deviation {fmt(100 * rel)}% (tol 2%)")
    if rel > 0.02:
        out.fail("fp32 and fp64 runs disagree beyond 2%")
    return out


def criterion_8():
    """tests/acceptance.cpp:460-562."""
    out = Outcome()
    # accepted-cost monotonicity on a solve
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=24, points=96, obs_per_point=8))
    st = dba.lm_solve(p, dba.SolverConfig(max_iterations=20), devices=[0])
    last, mono = float("inf"), True
    for r in st.history:
        if r.accepted:
            mono &= not (r.cost > last * (1 + 1e-12))
            last = r.cost
    (out.note if mono else out.fail)("accepted-cost sequence is non-increasing" if mono
                                     else "accepted-cost sequence increased")

    # all-reduce rank identity and determinism (WorkerGroup on the device)
    k = 4
    locals_ = np.random.default_rng(55).uniform(-1e3, 1e3, (k, 101))

    def run(data):
        data = [row.copy() for row in data]
        g = dba.WorkerGroup(k)
        dba.run_on_workers(g, lambda r: g.allreduce_sum(r, data[r]))
        g.close()
        return data

    a, b = run(locals_), run(locals_)
    ident = all(np.array_equal(a[r], a[0]) and np.array_equal(a[r], b[r]) for r in range(k))
    (out.note if ident else out.fail)("all-reduce results are rank-identical and repeatable" if ident
                                      else "all-reduce results differ across ranks or runs")

    # partition disjointness / union
    q = ProblemFactory(66).random_problem(5, 9, 47)
    ok = True
    for kk in range(1, 7):
        concat = np.concatenate([part.edge_ids for part in dba.partition_edges(q, kk)])
        ok &= concat.size == 47 and np.array_equal(concat, np.arange(47))
    (out.note if ok else out.fail)("partitions are disjoint and cover the edge list in order" if ok
                                   else "partition union/disjointness violated")

    # adjointness of the fused E^T x / E b pass: S = B_d - E C_d^-1 E^T is
    # symmetric, so y.(S x) = x.(S y) (see the module docstring)
    q = ProblemFactory(67).random_problem(4, 7, 22)
    rng = np.random.default_rng(68)
    worst = 0.0
    for _ in range(20):
        x, y = rng.uniform(-1, 1, 36), rng.uniform(-1, 1, 36)
        sx, _, _ = dba.group_operator(q, 1, x, mode=0, lam=1e-3, policy=dba.DAMPING_IDENTITY)
        sy, _, _ = dba.group_operator(q, 1, y, mode=0, lam=1e-3, policy=dba.DAMPING_IDENTITY)
        lhs, rhs = float(y @ sx), float(x @ sy)
        worst = max(worst, abs(lhs - rhs) / max(1.0, abs(lhs), abs(rhs)))
    out.note(f"DSE-operator adjointness worst relative defect: {fmt(worst)} (tol 1e-12)")
    if worst > 1e-12:
        out.fail("the DSE pass's E^T and E are not numerical adjoints")
    return out


CRITERIA = {1: criterion_1, 2: criterion_2, 3: criterion_3, 4: criterion_4, 5: criterion_5, 6: criterion_6,
            7: criterion_7, 8: criterion_8}


def run_criterion(index):
    """tests/acceptance.cpp:564-580 (an exception is a failure)."""
    if index not in CRITERIA:
        o = Outcome()
        o.fail(f"unknown criterion {index}")
        return o
    try:
        return CRITERIA[index]()
    except Exception as e:  # noqa: BLE001 - reported, as the reference does
        o = Outcome()
        o.fail(f"unexpected exception: {e}")
        return o


def main(argv=None):
    """tests/acceptance.cpp:598-635."""
    global DATA_DIR
    ap = argparse.ArgumentParser(prog="dba_acceptance", usage="dba_acceptance [--criterion N]... [--data-dir PATH]")
    ap.add_argument("--criterion", type=int, action="append", default=[])
    ap.add_argument("--data-dir", default="data")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    DATA_DIR = args.data_dir
    if DATA_DIR == "data" and os.environ.get("DBA_DATA_DIR"):
        DATA_DIR = os.environ["DBA_DATA_DIR"]
    failures = 0
    for index in args.criterion or list(range(1, 9)):
        o = run_criterion(index)
        print(f"{'[PASS] ' if o.ok else '[FAIL] '}criterion {index}: {NAMES.get(index, '?')}")
        for line in o.details:
            print(f"       {line}")
        failures += not o.ok
    return 0 if failures == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
