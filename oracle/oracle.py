"""ctypes binding of the CPU oracle (oracle/liboracle_dba.so).

TEST INFRASTRUCTURE ONLY — the checker, never the product. Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module.
The oracle restates the reference (see dba_oracle.hpp for the file:line map).
This module is self-contained: it never imports the product package, so a
process that only runs the oracle (bench.py --impl reference) loads no
product library. Problems and configs are duck-typed: anything with
``arrays()`` -> (cameras (m,9), points (n,3), camera_id, point_id, pixel_x,
pixel_y, weight) and a float32/float64 ``dtype`` (the product's BAProblem, or
OracleProblem below), and any object carrying SolverConfig's field names.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from dataclasses import dataclass, field
from typing import List

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_dba.so")

_lib = None

i32, i64, u64, f64, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p


class Problem(C.Structure):  # orc_problem (oracle_capi.cpp)
    _fields_ = [("num_cameras", i32), ("num_points", i32), ("num_observations", i64),
                ("cameras", vp), ("points", vp), ("camera_id", C.POINTER(i32)),
                ("point_id", C.POINTER(i32)), ("pixel_x", vp), ("pixel_y", vp), ("weight", vp)]


class Config(C.Structure):  # orc_config
    _fields_ = [("workers", i32), ("max_iterations", i32), ("pcg_tol", f64), ("pcg_max_iters", i32),
                ("_pad0", i32), ("lambda0", f64), ("lambda_max", f64), ("rel_tol", f64), ("step_tol", f64),
                ("damping", i32), ("mse_half", i32), ("jacobian", i32), ("check_rank_identity", i32)]


class Result(C.Structure):  # orc_result
    _fields_ = [("iterations", i32), ("termination", i32), ("cost", f64), ("lam", f64), ("nu", f64),
                ("capacity", i32), ("workers", i32), ("rec_iteration", C.POINTER(i32)),
                ("rec_cost", C.POINTER(f64)), ("rec_mse", C.POINTER(f64)), ("rec_lambda", C.POINTER(f64)),
                ("rec_pcg", C.POINTER(i32)), ("rec_accepted", C.POINTER(i32)), ("rec_wall", C.POINTER(f64)),
                ("rec_worker_edges", C.POINTER(u64)), ("rec_worker_block_ops", C.POINTER(u64)),
                ("x_c", vp), ("x_p", vp)]


class Synth(C.Structure):  # orc_synth (= dbag_synthetic_options layout)
    _fields_ = [("cameras", i32), ("points", i32), ("obs_per_point", i32), ("exhaustive_search", i32), ("seed", u64),
                ("circle_radius", f64), ("base_focal", f64), ("pose_noise", f64), ("intrinsic_noise", f64),
                ("point_noise", f64), ("num_observations", i64), ("pixel_noise", f64)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        h = C.CDLL(LIB_PATH)
        P = C.POINTER
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_last_error_index": (C.c_int64, []),
            "orc_last_error_block_size": (C.c_int, []),
            "orc_residual": (C.c_int, [C.c_int, vp, vp, vp, vp]),
            "orc_rotate": (C.c_int, [C.c_int, vp, vp, vp]),
            "orc_total_cost": (C.c_int, [C.c_int, P(Problem), P(C.c_double)]),
            "orc_jet_op": (C.c_int, [C.c_int, C.c_int64, C.c_int, vp, vp, C.c_int, vp, vp, C.c_double, P(C.c_int),
                                     vp, vp]),
            "orc_rotate_jets": (C.c_int, [vp, vp, vp, vp]),
            "orc_partition": (C.c_int, [P(Problem), C.c_int, C.c_int, P(C.c_int64), P(C.c_int64), P(C.c_int), vp,
                                        P(C.c_int), vp, vp, vp, vp, vp]),
            "orc_linearize": (C.c_int, [C.c_int, P(Problem), C.c_int, C.c_int, C.c_int, vp, vp, P(C.c_int64)]),
            "orc_assemble": (C.c_int, [C.c_int, P(Problem), C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
            "orc_damp": (C.c_int, [C.c_int, C.c_int64, vp, C.c_double, C.c_int, vp]),
            "orc_factor_solve": (C.c_int, [C.c_int, C.c_int64, vp, vp]),
            "orc_dse": (C.c_int, [C.c_int, P(Problem), C.c_int, C.c_double, C.c_int, vp, vp, P(C.c_int)]),
            "orc_dpcg": (C.c_int, [C.c_int, P(Problem), C.c_int, C.c_double, C.c_int, vp, C.c_double, C.c_int, vp,
                                   P(C.c_int), P(C.c_int), P(C.c_int)]),
            "orc_blocks_solve": (C.c_int, [P(Problem), C.c_int, vp, vp, vp, C.c_int, vp, C.c_double, C.c_int, vp,
                                           P(C.c_int), P(C.c_int)]),
            "orc_allreduce": (C.c_int, [C.c_int, C.c_int64, vp]),
            "orc_lm_solve": (C.c_int, [C.c_int, P(Problem), P(Config), P(Result)]),
            "orc_lm_probe_phases": (C.c_int, [C.c_int, P(Problem), P(Config), C.c_int, C.c_int, vp, vp, vp]),
            "orc_synthetic_count": (C.c_int, [P(Synth), P(C.c_int64)]),
            "orc_generate_synthetic": (C.c_int, [P(Synth), C.c_int, vp, vp, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _lib = h
    return _lib


# ------------------------------------------------------------ containers --

@dataclass
class OracleConfig:
    """SolverConfig (dba/solver.hpp:39-55): same field names and defaults."""
    workers: int = 1
    max_iterations: int = 50
    pcg_tol: float = 1e-6
    pcg_max_iters: int = 500
    lambda0: float = 1e-4
    lambda_max: float = 1e32
    rel_tol: float = 1e-6
    step_tol: float = 1e-8
    damping: int = 1  # diag_scaled
    mse: int = 1      # half_per_observation
    jacobian: int = 0  # autodiff
    check_rank_identity: bool = False


class OracleProblem:
    """Flat BAProblem (dba/problem.hpp:171-261) held by the oracle alone."""

    def __init__(self, cams, pts, cid, pid, px, py, w=None, dtype=np.float64):
        d = np.dtype(dtype)
        self.dtype = d
        self._a = (np.ascontiguousarray(np.asarray(cams, d).reshape(-1, 9)),
                   np.ascontiguousarray(np.asarray(pts, d).reshape(-1, 3)),
                   np.ascontiguousarray(cid, np.int32), np.ascontiguousarray(pid, np.int32),
                   np.ascontiguousarray(px, d), np.ascontiguousarray(py, d),
                   np.ascontiguousarray(np.ones(len(cid), d) if w is None else w, d))

    def arrays(self):
        return self._a

    @property
    def num_cameras(self):
        return len(self._a[0])

    @property
    def num_points(self):
        return len(self._a[1])

    @property
    def num_observations(self):
        return len(self._a[2])

    @property
    def precision(self):
        return self.dtype.itemsize

    def astype(self, dtype):
        a = self._a
        return OracleProblem(*a, dtype=dtype)


def _ps(problem) -> Problem:
    cams, pts, cid, pid, px, py, w = problem.arrays()
    s = Problem()
    s.num_cameras, s.num_points, s.num_observations = len(cams), len(pts), len(cid)
    s.cameras, s.points = cams.ctypes.data, pts.ctypes.data
    s.camera_id = cid.ctypes.data_as(C.POINTER(C.c_int32))
    s.point_id = pid.ctypes.data_as(C.POINTER(C.c_int32))
    s.pixel_x, s.pixel_y, s.weight = px.ctypes.data, py.ctypes.data, w.ctypes.data
    s._keep = (cams, pts, cid, pid, px, py, w)
    return s


def _prec(problem) -> int:
    return np.dtype(problem.dtype).itemsize


def _cfg(config) -> Config:
    c = Config()
    c.workers, c.max_iterations, c.pcg_tol = config.workers, config.max_iterations, config.pcg_tol
    c.pcg_max_iters, c.lambda0, c.lambda_max = config.pcg_max_iters, config.lambda0, config.lambda_max
    c.rel_tol, c.step_tol, c.damping = config.rel_tol, config.step_tol, config.damping
    c.mse_half, c.jacobian = config.mse, config.jacobian
    c.check_rank_identity = int(config.check_rank_identity)
    return c


class OracleError(RuntimeError):
    def __init__(self, code, msg, index=-1, block_size=0):
        super().__init__(f"[{code}] {msg}")
        self.code, self.index, self.block_size = code, index, block_size


def check(rc):
    if rc:
        L = lib()
        raise OracleError(rc, L.orc_last_error().decode(), int(L.orc_last_error_index()),
                          int(L.orc_last_error_block_size()))


def _d(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype)


def residual(cam, pt, pix, dtype=np.float64):
    out = np.zeros(2, dtype)
    a, b, c = _d(cam, dtype), _d(pt, dtype), _d(pix, dtype)
    check(lib().orc_residual(np.dtype(dtype).itemsize, a.ctypes.data, b.ctypes.data, c.ctypes.data,
                             out.ctypes.data))
    return out


def rotate(aa, x, dtype=np.float64):
    out = np.zeros(3, dtype)
    a, b = _d(aa, dtype), _d(x, dtype)
    check(lib().orc_rotate(np.dtype(dtype).itemsize, a.ctypes.data, b.ctypes.data, out.ctypes.data))
    return out


def total_cost(problem) -> float:
    s = _ps(problem)
    c = C.c_double()
    check(lib().orc_total_cost(_prec(problem), C.byref(s), C.byref(c)))
    return c.value


JET_OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "sqrt": 4, "neg": 5, "add_scalar": 6}


def jet_op(op, a_v, a_g, b_v=None, b_g=None, s=0.0):
    """Elementwise JetVector kernel on fp64 batches; grads are (d, n) lane-major."""
    a_v = _d(np.atleast_1d(a_v))
    n = len(a_v)
    a_g = _d(np.zeros((0, n)) if a_g is None else np.asarray(a_g).reshape(-1, n))
    b_v = _d(np.zeros(n) if b_v is None else np.atleast_1d(b_v))
    b_g = _d(np.zeros((0, n)) if b_g is None else np.asarray(b_g).reshape(-1, n))
    d = max(a_g.shape[0], b_g.shape[0])
    ov = np.zeros(n)
    og = np.zeros((max(d, 1), n))
    dout = C.c_int()
    check(lib().orc_jet_op(JET_OPS[op], n, a_g.shape[0], a_v.ctypes.data, a_g.ctypes.data, b_g.shape[0],
                           b_v.ctypes.data, b_g.ctypes.data, s, C.byref(dout), ov.ctypes.data, og.ctypes.data))
    return ov, og[:dout.value]


def rotate_jets(aa, x):
    out = np.zeros(3)
    g = np.zeros((3, 6))
    a, b = _d(aa), _d(x)
    check(lib().orc_rotate_jets(a.ctypes.data, b.ctypes.data, out.ctypes.data, g.ctypes.data))
    return out, g


def partition(problem, k, rank):
    s = _ps(problem)
    m, n, nobs = s.num_cameras, s.num_points, s.num_observations
    start, count, nc, npt = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
    cam_g, pt_g = np.zeros(max(m, 1), np.int32), np.zeros(max(n, 1), np.int32)
    cam_ptr, pt_ptr = np.zeros(m + 1, np.int64), np.zeros(n + 1, np.int64)
    cam_blk, pt_blk = np.zeros(max(nobs, 1), np.int64), np.zeros(max(nobs, 1), np.int64)
    check(lib().orc_partition(C.byref(s), k, rank, C.byref(start), C.byref(count), C.byref(nc), cam_g.ctypes.data,
                              C.byref(npt), pt_g.ctypes.data, cam_ptr.ctypes.data, cam_blk.ctypes.data,
                              pt_ptr.ctypes.data, pt_blk.ctypes.data))
    c = count.value
    return dict(start=start.value, count=c, cam_g=cam_g[:nc.value], pt_g=pt_g[:npt.value],
                cam_ptr=cam_ptr[:nc.value + 1], cam_blk=cam_blk[:c], pt_ptr=pt_ptr[:npt.value + 1],
                pt_blk=pt_blk[:c])


def _count(problem, k, rank):
    n = problem.num_observations
    return n // k + (1 if rank < n % k else 0)


def linearize(problem, k=1, rank=0, mode=0):
    """(res (2, N_k), jac (2, 12, N_k)) or raises OracleError(1, ..., edge)."""
    cnt = _count(problem, k, rank)
    d = problem.dtype
    res = np.zeros(2 * cnt, d)
    jac = np.zeros(24 * cnt, d)
    bad = C.c_int64(-1)
    s = _ps(problem)
    check(lib().orc_linearize(_prec(problem), C.byref(s), k, rank, mode, res.ctypes.data, jac.ctypes.data,
                              C.byref(bad)))
    return res.reshape(2, cnt), jac.reshape(2, 12, cnt)


def assemble(problem, k=1, rank=0, mode=0):
    """Local (not all-reduced) B (m,9,9), C (n,3,3), E (N_k,9,3), v, w."""
    cnt = _count(problem, k, rank)
    d = problem.dtype
    m, n = problem.num_cameras, problem.num_points
    B, Cc, E = np.zeros(81 * m, d), np.zeros(9 * n, d), np.zeros(27 * cnt, d)
    v, w = np.zeros(9 * m, d), np.zeros(3 * n, d)
    s = _ps(problem)
    check(lib().orc_assemble(_prec(problem), C.byref(s), k, rank, mode, B.ctypes.data, Cc.ctypes.data,
                             E.ctypes.data, v.ctypes.data, w.ctypes.data))
    return B.reshape(m, 9, 9), Cc.reshape(n, 3, 3), E.reshape(cnt, 9, 3), v, w


def damp(blocks, lam, policy):
    b = _d(blocks)
    bs = b.shape[-1]
    out = np.zeros_like(b)
    check(lib().orc_damp(bs, b.shape[0], b.ctypes.data, lam, policy, out.ctypes.data))
    return out


def factor_solve(blocks, x):
    b = _d(blocks)
    xx = _d(x).copy()
    check(lib().orc_factor_solve(b.shape[-1], b.shape[0], b.ctypes.data, xx.ctypes.data))
    return xx


def dse(problem, k, lam, policy, x):
    """dse on the problem's own damped system at the problem's precision."""
    s = _ps(problem)
    d = np.dtype(problem.dtype)
    out = np.zeros(9 * problem.num_cameras, d)
    ident = C.c_int()
    xx = _d(x, d)
    check(lib().orc_dse(_prec(problem), C.byref(s), k, lam, policy, xx.ctypes.data, out.ctypes.data, C.byref(ident)))
    return out, bool(ident.value)


def dpcg(problem, k, lam, policy, rhs, tol, max_iters):
    s = _ps(problem)
    d = np.dtype(problem.dtype)
    x = np.zeros(9 * problem.num_cameras, d)
    it, conv, ident = C.c_int(), C.c_int(), C.c_int()
    rr = _d(rhs, d)
    check(lib().orc_dpcg(_prec(problem), C.byref(s), k, lam, policy, rr.ctypes.data, tol, max_iters, x.ctypes.data,
                         C.byref(it), C.byref(conv), C.byref(ident)))
    return x, it.value, bool(conv.value), bool(ident.value)


def blocks_solve(problem, k, B, Cb, E_table, mode, x, tol=1e-12, max_iters=500):
    s = _ps(problem)
    out = np.zeros(9 * problem.num_cameras)
    it, ident = C.c_int(), C.c_int()
    bb, cc, ee, xx = _d(B), _d(Cb), _d(E_table), _d(x)
    check(lib().orc_blocks_solve(C.byref(s), k, bb.ctypes.data, cc.ctypes.data, ee.ctypes.data,
                                 mode, xx.ctypes.data, tol, max_iters, out.ctypes.data, C.byref(it),
                                 C.byref(ident)))
    return out, it.value, bool(ident.value)


def allreduce(data):
    a = _d(data).copy()
    check(lib().orc_allreduce(a.shape[0], a.shape[1], a.ctypes.data))
    return a


@dataclass
class Record:
    """IterationRecord (dba/solver.hpp:57-68)."""
    iteration: int
    cost: float
    mse: float
    lambda_: float
    pcg_iterations: int
    accepted: bool
    wall_seconds: float
    worker_edges: List[int] = field(default_factory=list)
    worker_block_ops: List[int] = field(default_factory=list)


@dataclass
class State:
    """SolverState (dba/solver.hpp:70-85), rank 0's."""
    x_c: np.ndarray
    x_p: np.ndarray
    lambda_: float
    nu: float
    iteration: int
    cost: float
    termination: str
    history: List[Record]


def lm_solve(problem, config):
    """dba::lm_solve restated on the CPU with config.workers threads."""
    s = _ps(problem)
    cap, k = config.max_iterations, config.workers
    d = np.dtype(problem.dtype)
    it, cost, mse, lam = np.zeros(cap, np.int32), np.zeros(cap), np.zeros(cap), np.zeros(cap)
    pcg, acc, wall = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(cap)
    we, wb = np.zeros(cap * k, np.uint64), np.zeros(cap * k, np.uint64)
    xc, xp = np.zeros(9 * s.num_cameras, d), np.zeros(max(3 * s.num_points, 1), d)
    r = Result()
    r.capacity, r.workers = cap, k
    P = C.POINTER
    r.rec_iteration, r.rec_cost = it.ctypes.data_as(P(i32)), cost.ctypes.data_as(P(f64))
    r.rec_mse, r.rec_lambda = mse.ctypes.data_as(P(f64)), lam.ctypes.data_as(P(f64))
    r.rec_pcg, r.rec_accepted = pcg.ctypes.data_as(P(i32)), acc.ctypes.data_as(P(i32))
    r.rec_wall = wall.ctypes.data_as(P(f64))
    r.rec_worker_edges, r.rec_worker_block_ops = we.ctypes.data_as(P(u64)), wb.ctypes.data_as(P(u64))
    r.x_c, r.x_p = xc.ctypes.data, xp.ctypes.data
    cfg = _cfg(config)
    check(lib().orc_lm_solve(_prec(problem), C.byref(s), C.byref(cfg), C.byref(r)))
    hist = [Record(int(it[i]), float(cost[i]), float(mse[i]), float(lam[i]), int(pcg[i]), bool(acc[i]), float(wall[i]),
                   [int(v) for v in we[i * k:(i + 1) * k]], [int(v) for v in wb[i * k:(i + 1) * k]])
            for i in range(min(r.iterations, cap))]
    term = {0: "converged", 1: "max_iterations", 2: "stalled"}[r.termination]
    return State(xc.copy(), xp[:3 * s.num_points].copy(), r.lam, r.nu, r.iterations, r.cost, term, hist)


PHASES = ("linearize_assemble", "damp_factor", "rhs", "dpcg_setup", "dpcg_loop", "backsub_trial", "cost_model")


def lm_probe_phases(problem, config, steps, pcg_sample=0):
    """The bench step (one LM iteration from x0 at lambda0, K = config.workers
    rank threads) `steps` times. Returns (phases (steps, 7) seconds, max over
    ranks, in PHASES order; pcg iterations; DSE calls). pcg_sample > 0 caps
    the DPCG at that many iterations: a bounded sample of the step."""
    s = _ps(problem)
    cfg = _cfg(config)
    ph = np.zeros(steps * 7)
    its = np.zeros(steps, np.int32)
    dse = np.zeros(steps, np.int32)
    check(lib().orc_lm_probe_phases(_prec(problem), C.byref(s), C.byref(cfg), steps, int(pcg_sample),
                                    ph.ctypes.data, its.ctypes.data, dse.ctypes.data))
    return ph.reshape(steps, 7), its, dse


def lm_probe_steps(problem, config, steps):
    """Seconds per full bench step and the PCG count of each step."""
    ph, its, _ = lm_probe_phases(problem, config, steps)
    return ph.sum(1), its


@dataclass
class SynthOptions:
    """SyntheticOptions (dba/synthetic.hpp:19-30) + count-exact / pixel noise."""
    cameras: int = 20000
    points: int = 80000
    obs_per_point: int = 1000
    seed: int = 1
    circle_radius: float = 8.0
    base_focal: float = 1000.0
    pose_noise: float = 0.01
    intrinsic_noise: float = 0.5
    point_noise: float = 0.1
    num_observations: int = 0
    pixel_noise: float = 0.0


def generate_synthetic(opt: SynthOptions, threads: int = 0) -> OracleProblem:
    """The reference's generator (exhaustive nearest-camera scan), fp64."""
    o = Synth()
    for f in dataclasses.fields(opt):
        setattr(o, f.name, getattr(opt, f.name))
    o.exhaustive_search = 1
    n = C.c_int64()
    check(lib().orc_synthetic_count(C.byref(o), C.byref(n)))
    N = n.value
    cams, pts = np.zeros((opt.cameras, 9)), np.zeros((opt.points, 3))
    cid, pid, px, py = np.zeros(N, np.int32), np.zeros(N, np.int32), np.zeros(N), np.zeros(N)
    check(lib().orc_generate_synthetic(C.byref(o), int(threads or os.cpu_count() or 1), cams.ctypes.data,
                                       pts.ctypes.data, cid.ctypes.data, pid.ctypes.data, px.ctypes.data,
                                       py.ctypes.data))
    return OracleProblem(cams, pts, cid, pid, px, py)
