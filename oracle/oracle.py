"""ctypes binding of the CPU oracle (oracle/liboracle_dba.so).

TEST INFRASTRUCTURE ONLY — the checker, never the product. Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module.
The oracle restates the reference (see dba_oracle.hpp for the file:line map);
its struct layouts are the same as include/dbag.h, so the product's ctypes
structures are reused.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_dba.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        from paper_2112_01349_b200._native import Config, Problem, Result
        h = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
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
            "orc_dse": (C.c_int, [P(Problem), C.c_int, C.c_double, C.c_int, vp, vp, P(C.c_int)]),
            "orc_dpcg": (C.c_int, [P(Problem), C.c_int, C.c_double, C.c_int, vp, C.c_double, C.c_int, vp,
                                   P(C.c_int), P(C.c_int), P(C.c_int)]),
            "orc_blocks_solve": (C.c_int, [P(Problem), C.c_int, vp, vp, vp, C.c_int, vp, C.c_double, C.c_int, vp,
                                           P(C.c_int), P(C.c_int)]),
            "orc_allreduce": (C.c_int, [C.c_int, C.c_int64, vp]),
            "orc_lm_solve": (C.c_int, [C.c_int, P(Problem), P(Config), P(Result)]),
            "orc_lm_probe_steps": (C.c_int, [C.c_int, P(Problem), P(Config), C.c_int, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _lib = h
    return _lib


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
    s = problem.c_struct()
    c = C.c_double()
    check(lib().orc_total_cost(problem.precision, C.byref(s), C.byref(c)))
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
    s = problem.c_struct()
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
    s = problem.c_struct()
    check(lib().orc_linearize(problem.precision, C.byref(s), k, rank, mode, res.ctypes.data, jac.ctypes.data,
                              C.byref(bad)))
    return res.reshape(2, cnt), jac.reshape(2, 12, cnt)


def assemble(problem, k=1, rank=0, mode=0):
    """Local (not all-reduced) B (m,9,9), C (n,3,3), E (N_k,9,3), v, w."""
    cnt = _count(problem, k, rank)
    d = problem.dtype
    m, n = problem.num_cameras, problem.num_points
    B, Cc, E = np.zeros(81 * m, d), np.zeros(9 * n, d), np.zeros(27 * cnt, d)
    v, w = np.zeros(9 * m, d), np.zeros(3 * n, d)
    s = problem.c_struct()
    check(lib().orc_assemble(problem.precision, C.byref(s), k, rank, mode, B.ctypes.data, Cc.ctypes.data,
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
    s = problem.c_struct()
    out = np.zeros(9 * problem.num_cameras)
    ident = C.c_int()
    xx = _d(x)
    check(lib().orc_dse(C.byref(s), k, lam, policy, xx.ctypes.data, out.ctypes.data, C.byref(ident)))
    return out, bool(ident.value)


def dpcg(problem, k, lam, policy, rhs, tol, max_iters):
    s = problem.c_struct()
    x = np.zeros(9 * problem.num_cameras)
    it, conv, ident = C.c_int(), C.c_int(), C.c_int()
    rr = _d(rhs)
    check(lib().orc_dpcg(C.byref(s), k, lam, policy, rr.ctypes.data, tol, max_iters, x.ctypes.data,
                         C.byref(it), C.byref(conv), C.byref(ident)))
    return x, it.value, bool(conv.value), bool(ident.value)


def blocks_solve(problem, k, B, Cb, E_table, mode, x, tol=1e-12, max_iters=500):
    s = problem.c_struct()
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


def lm_solve(problem, config):
    """dba::lm_solve restated on the CPU with config.workers threads."""
    from paper_2112_01349_b200.dba import _ResultBuf
    s = problem.c_struct()
    buf = _ResultBuf(config.max_iterations, config.workers, s.num_cameras, s.num_points, problem.dtype)
    cfg = config.c_struct()
    check(lib().orc_lm_solve(problem.precision, C.byref(s), C.byref(cfg), C.byref(buf.r)))
    return buf.state(s.num_points)


def lm_probe_steps(problem, config, steps):
    """Seconds per bench step (one LM iteration from x0, K = config.workers
    threads) and the PCG count of each step."""
    s = problem.c_struct()
    cfg = config.c_struct()
    secs = np.zeros(steps)
    its = np.zeros(steps, np.int32)
    check(lib().orc_lm_probe_steps(problem.precision, C.byref(s), C.byref(cfg), steps, secs.ctypes.data,
                                   its.ctypes.data))
    return secs, its
