"""Host-side mirror of the reference's ``dba`` API for the LM inner loop.

Same names, argument meaning and error behaviour as the header-only C++ API
of the reference:

  BAProblem / CameraState / PointState / Observation   dba/problem.hpp:34-261
  partition_edges / EdgePartition / LocalIndexMap       dba/partition.hpp:14-103
  SolverConfig / IterationRecord / SolverState          dba/solver.hpp:39-85
  lm_solve                                              dba/solver.hpp:523-534
  generate_synthetic / SyntheticOptions                 dba/synthetic.hpp:19-146
  errors                                                dba/errors.hpp:17-84

Every numeric operator runs in libdbag.so (hand-written sm_100a kernels); this
module only marshals arrays and maps status codes back to exceptions.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

# ------------------------------------------------------------------ errors --


class Error(RuntimeError):
    """dba::Error (dba/errors.hpp:10-13)."""


class ParseError(Error):
    """Malformed input text (dba/errors.hpp:17-26); ``line`` is 1-based, 0 if unknown."""

    def __init__(self, msg: str, line: int = 0):
        super().__init__(msg)
        self.line = line


class InvalidArgumentError(Error):
    pass


class DegenerateDepthError(Error):
    def __init__(self, msg: str = "degenerate depth (P_z = 0)", edge_id: int = -1):
        super().__init__(msg)
        self.edge_id = edge_id


class ShapeError(Error):
    pass


class SingularBlockError(Error):
    def __init__(self, msg: str, block_index: int, block_size: int):
        super().__init__(msg)
        self.block_index = block_index
        self.block_size = block_size


class CollectiveError(Error):
    pass


class PcgBreakdownError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    lib = N.lib()
    msg = (lib.dbag_last_error() or b"").decode(errors="replace")
    idx = int(lib.dbag_last_error_index())
    if rc == 1:
        raise DegenerateDepthError(msg, idx)
    if rc == 2:
        raise SingularBlockError(msg, idx, int(lib.dbag_last_error_block_size()))
    if rc == 10:
        raise ParseError(msg, max(idx, 0))
    raise {3: PcgBreakdownError, 4: ShapeError, 5: InvalidArgumentError, 6: CollectiveError, 7: CudaError,
           8: NcclError}.get(rc, Error)(msg)


# ----------------------------------------------------------------- problem --

MSE_PER_OBSERVATION, MSE_HALF_PER_OBSERVATION = 0, 1


def pack_cameras(problem: "BAProblem"):
    """dba/problem.hpp:294-306: x_c (9m)."""
    return problem.pack_cameras()


def pack_points(problem: "BAProblem"):
    """dba/problem.hpp:308-318: x_p (3n)."""
    return problem.pack_points()


def unpack_states(x_c, x_p, problem: "BAProblem") -> None:
    """dba/problem.hpp:341-353: writes packed parameter vectors back into the
    problem's camera and point states (in place)."""
    cams, pts, cid, pid, px, py, w = problem.arrays()
    x_c = np.asarray(x_c, dtype=problem.dtype).reshape(-1)
    x_p = np.asarray(x_p, dtype=problem.dtype).reshape(-1)
    if x_c.size != cams.size or x_p.size != pts.size:
        raise ShapeError(f"unpack_states: expected {cams.size} + {pts.size} parameters, got {x_c.size} + {x_p.size}")
    problem._frozen = (np.ascontiguousarray(x_c.reshape(-1, 9)), np.ascontiguousarray(x_p.reshape(-1, 3)),
                       cid, pid, px, py, w)


def mse_from_cost(cost: float, num_observations: int, convention: int = MSE_HALF_PER_OBSERVATION) -> float:
    """dba/problem.hpp:22-29."""
    if num_observations <= 0:
        return 0.0
    return cost / (2.0 * num_observations if convention == MSE_HALF_PER_OBSERVATION else float(num_observations))


@dataclass
class CameraState:
    """BAL 9-parameter camera (dba/problem.hpp:34-49)."""
    rotation: Sequence[float] = (0.0, 0.0, 0.0)
    translation: Sequence[float] = (0.0, 0.0, 0.0)
    focal: float = 1.0
    k1: float = 0.0
    k2: float = 0.0

    def params(self):
        return [*self.rotation, *self.translation, self.focal, self.k1, self.k2]


@dataclass
class PointState:
    position: Sequence[float] = (0.0, 0.0, 0.0)


@dataclass
class Observation:
    camera_id: int = 0
    point_id: int = 0
    pixel: Sequence[float] = (0.0, 0.0)
    weight: float = 1.0


class BAProblem:
    """Camera nodes, point nodes and observation edges (dba/problem.hpp:171-261).

    ``dtype`` is the reference's Scalar template parameter (float32 or float64).
    Storage is packed: cameras (m, 9) as pack_cameras, points (n, 3) as
    pack_points, observations as SoA arrays in canonical edge order.
    """

    def __init__(self, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.float32, np.float64):
            raise InvalidArgumentError("BAProblem dtype must be float32 or float64")
        self._cams: list = []
        self._pts: list = []
        self._obs: list = []
        self._frozen = None

    @classmethod
    def from_arrays(cls, cameras, points, camera_id, point_id, pixels, weight=None, dtype=None):
        if dtype is None:
            src = np.asarray(cameras).dtype
            dtype = src if src in (np.float32, np.float64) else np.float64
        dtype = np.dtype(dtype)
        p = cls(dtype)
        cams = np.ascontiguousarray(np.asarray(cameras, dtype=dtype).reshape(-1, 9))
        pts = np.ascontiguousarray(np.asarray(points, dtype=dtype).reshape(-1, 3))
        cid = np.ascontiguousarray(np.asarray(camera_id, dtype=np.int32))
        pid = np.ascontiguousarray(np.asarray(point_id, dtype=np.int32))
        pix = np.asarray(pixels, dtype=dtype).reshape(-1, 2)
        w = np.ones(len(cid), dtype=dtype) if weight is None else np.ascontiguousarray(np.asarray(weight, dtype=dtype))
        if not (np.isfinite(cams).all() and np.isfinite(pts).all()):
            raise InvalidArgumentError("node has non-finite components")
        if len(cid) and (cid.min() < 0 or cid.max() >= len(cams)):
            raise InvalidArgumentError("edge references unknown camera")
        if len(pid) and (pid.min() < 0 or pid.max() >= len(pts)):
            raise InvalidArgumentError("edge references unknown point")
        if not (w >= 0).all():
            raise InvalidArgumentError("edge weight must be >= 0")
        p._frozen = (cams, pts, cid, pid, np.ascontiguousarray(pix[:, 0]), np.ascontiguousarray(pix[:, 1]), w)
        return p

    # -- append API (dba/problem.hpp:180-207)
    def _thaw(self):
        if self._frozen is not None:
            cams, pts, cid, pid, px, py, w = self._frozen
            self._cams = [list(r) for r in cams]
            self._pts = [list(r) for r in pts]
            self._obs = [(int(a), int(b), float(x), float(y), float(ww)) for a, b, x, y, ww in zip(cid, pid, px, py, w)]
            self._frozen = None

    def add_node(self, node) -> int:
        self._thaw()
        if isinstance(node, CameraState):
            v = [float(x) for x in node.params()]
            if not np.isfinite(v).all():
                raise InvalidArgumentError("camera node has non-finite components")
            self._cams.append(v)
            return len(self._cams) - 1
        if isinstance(node, PointState):
            v = [float(x) for x in node.position]
            if not np.isfinite(v).all():
                raise InvalidArgumentError("point node has non-finite components")
            self._pts.append(v)
            return len(self._pts) - 1
        raise InvalidArgumentError("add_node expects a CameraState or PointState")

    def add_edge(self, obs: Observation) -> int:
        self._thaw()
        if not 0 <= obs.camera_id < len(self._cams):
            raise InvalidArgumentError(f"edge references unknown camera {obs.camera_id}")
        if not 0 <= obs.point_id < len(self._pts):
            raise InvalidArgumentError(f"edge references unknown point {obs.point_id}")
        if not obs.weight >= 0:
            raise InvalidArgumentError("edge weight must be >= 0")
        self._obs.append((obs.camera_id, obs.point_id, float(obs.pixel[0]), float(obs.pixel[1]), float(obs.weight)))
        return len(self._obs) - 1

    def arrays(self):
        """(cameras (m,9), points (n,3), camera_id, point_id, pixel_x, pixel_y, weight)."""
        if self._frozen is None:
            d = self.dtype
            cams = np.ascontiguousarray(np.array(self._cams, dtype=d).reshape(-1, 9))
            pts = np.ascontiguousarray(np.array(self._pts, dtype=d).reshape(-1, 3))
            o = np.array(self._obs, dtype=np.float64).reshape(-1, 5)
            self._frozen = (cams, pts, np.ascontiguousarray(o[:, 0].astype(np.int32)),
                            np.ascontiguousarray(o[:, 1].astype(np.int32)), np.ascontiguousarray(o[:, 2].astype(d)),
                            np.ascontiguousarray(o[:, 3].astype(d)), np.ascontiguousarray(o[:, 4].astype(d)))
            self._cams, self._pts, self._obs = [], [], []
        return self._frozen

    @property
    def num_cameras(self) -> int:
        return len(self.arrays()[0])

    @property
    def num_points(self) -> int:
        return len(self.arrays()[1])

    @property
    def num_observations(self) -> int:
        return len(self.arrays()[2])

    # node / edge accessors (dba/problem.hpp:219-227), as value objects
    def camera(self, i: int) -> CameraState:
        c = self.arrays()[0][i]
        return CameraState(tuple(float(v) for v in c[:3]), tuple(float(v) for v in c[3:6]), float(c[6]),
                           float(c[7]), float(c[8]))

    def point(self, i: int) -> PointState:
        return PointState(tuple(float(v) for v in self.arrays()[1][i]))

    def observation(self, e: int) -> Observation:
        _, _, cid, pid, px, py, w = self.arrays()
        return Observation(int(cid[e]), int(pid[e]), (float(px[e]), float(py[e])), float(w[e]))

    def cameras(self) -> List[CameraState]:
        return [self.camera(i) for i in range(self.num_cameras)]

    def points(self) -> List[PointState]:
        return [self.point(i) for i in range(self.num_points)]

    def observations(self) -> List[Observation]:
        return [self.observation(e) for e in range(self.num_observations)]

    def pack_cameras(self):
        return self.arrays()[0].reshape(-1).copy()

    def pack_points(self):
        return self.arrays()[1].reshape(-1).copy()

    def astype(self, dtype) -> "BAProblem":
        cams, pts, cid, pid, px, py, w = self.arrays()
        return BAProblem.from_arrays(cams, pts, cid, pid, np.stack([px, py], 1), w, dtype=dtype)

    def validate(self) -> List[str]:
        """Non-fatal warnings (dba/problem.hpp:214-241)."""
        cams, pts, cid, pid, *_ = self.arrays()
        out = []
        used_c = np.zeros(len(cams), bool)
        used_c[cid] = True
        used_p = np.zeros(len(pts), bool)
        used_p[pid] = True
        out += [f"camera {i} is not referenced by any observation" for i in np.flatnonzero(~used_c)]
        out += [f"point {i} is not referenced by any observation" for i in np.flatnonzero(~used_p)]
        out += [f"camera {i} has non-positive focal length" for i in np.flatnonzero(~(cams[:, 6] > 0))]
        return out

    def c_struct(self) -> N.Problem:
        cams, pts, cid, pid, px, py, w = self.arrays()
        s = N.Problem()
        s.num_cameras, s.num_points, s.num_observations = len(cams), len(pts), len(cid)
        s.cameras, s.points = cams.ctypes.data, pts.ctypes.data
        s.camera_id = cid.ctypes.data_as(C.POINTER(C.c_int32))
        s.point_id = pid.ctypes.data_as(C.POINTER(C.c_int32))
        s.pixel_x, s.pixel_y, s.weight = px.ctypes.data, py.ctypes.data, w.ctypes.data
        s._keep = (cams, pts, cid, pid, px, py, w)
        return s

    @property
    def precision(self) -> int:
        return self.dtype.itemsize


# --------------------------------------------------------------- partition --


@dataclass
class LocalIndexMap:
    """First-appearance local <-> global map (dba/partition.hpp:14-45)."""
    to_global: np.ndarray
    global_count: int

    def local(self, global_id: int) -> int:
        hit = np.flatnonzero(self.to_global == global_id)
        return int(hit[0]) if len(hit) else -1

    def global_(self, local_id: int) -> int:
        return int(self.to_global[local_id])

    def size(self) -> int:
        return len(self.to_global)


@dataclass
class EdgePartition:
    """dba/partition.hpp:49-54, plus the E grouping of block_matrix.hpp:309-320."""
    worker_rank: int
    edge_ids: np.ndarray
    camera_map: LocalIndexMap
    point_map: LocalIndexMap
    cam_ptr: np.ndarray
    cam_blocks: np.ndarray
    pt_ptr: np.ndarray
    pt_blocks: np.ndarray


def partition_edges(problem: BAProblem, worker_count: int) -> List[EdgePartition]:
    """dba/partition.hpp:76-103 (bit-exact), computed by the library's host code."""
    s = problem.c_struct()
    m, n, nobs = s.num_cameras, s.num_points, s.num_observations
    if worker_count < 1:
        raise InvalidArgumentError("worker count must be >= 1")
    if worker_count > nobs:
        raise InvalidArgumentError(f"worker count {worker_count} exceeds number of edges {nobs}")
    out = []
    lib = N.lib()
    for r in range(worker_count):
        start, count = C.c_int64(), C.c_int64()
        nc, npt = C.c_int32(), C.c_int32()
        cam_g = np.zeros(max(m, 1), np.int32)
        pt_g = np.zeros(max(n, 1), np.int32)
        cam_ptr = np.zeros(m + 1, np.int64)
        pt_ptr = np.zeros(n + 1, np.int64)
        cam_blk = np.zeros(max(nobs, 1), np.int64)
        pt_blk = np.zeros(max(nobs, 1), np.int64)
        _check(lib.dbag_partition(C.byref(s), worker_count, r, C.byref(start), C.byref(count), C.byref(nc),
                                  cam_g.ctypes.data, C.byref(npt), pt_g.ctypes.data, cam_ptr.ctypes.data,
                                  cam_blk.ctypes.data, pt_ptr.ctypes.data, pt_blk.ctypes.data))
        k = count.value
        out.append(EdgePartition(r, np.arange(start.value, start.value + k, dtype=np.int32),
                                 LocalIndexMap(cam_g[:nc.value].copy(), m), LocalIndexMap(pt_g[:npt.value].copy(), n),
                                 cam_ptr[:nc.value + 1].copy(), cam_blk[:k].copy(), pt_ptr[:npt.value + 1].copy(),
                                 pt_blk[:k].copy()))
    return out


def shared_points(problem: BAProblem, worker_count: int) -> np.ndarray:
    """Global ids of points touched by more than one rank (the halo)."""
    s = problem.c_struct()
    cnt = C.c_int64()
    _check(N.lib().dbag_shared_points(C.byref(s), worker_count, C.byref(cnt), None))
    ids = np.zeros(max(cnt.value, 1), np.int32)
    _check(N.lib().dbag_shared_points(C.byref(s), worker_count, C.byref(cnt), ids.ctypes.data))
    return ids[:cnt.value]


def predict_memory(problem: BAProblem, worker_count: int = 1, rank: int = 0, coupling_fp32: bool = False) -> int:
    """Device bytes rank `rank` of `worker_count` reserves in its one pool
    allocation at upload (the paper's predicted-size memory pool, SURVEY.md
    §8f f4). Host-only: runs the partition and the device layout, no GPU."""
    s = problem.c_struct()
    b = C.c_uint64()
    _check(N.lib().dbag_predict_memory(C.byref(s), problem.precision, int(coupling_fp32), worker_count, rank,
                                       C.byref(b)))
    return b.value


# ------------------------------------------------------------------ solver --

DAMPING_IDENTITY, DAMPING_DIAG_SCALED = 0, 1
JACOBIAN_AUTODIFF, JACOBIAN_ANALYTIC = 0, 1
TERMINATION = {0: "converged", 1: "max_iterations", 2: "stalled"}


@dataclass
class SolverConfig:
    """dba/solver.hpp:39-55 (same fields and defaults)."""
    workers: int = 1
    max_iterations: int = 50
    pcg_tol: float = 1e-6
    pcg_max_iters: int = 500
    lambda0: float = 1e-4
    lambda_max: float = 1e32
    rel_tol: float = 1e-6
    step_tol: float = 1e-8
    damping: int = DAMPING_DIAG_SCALED
    mse: int = MSE_HALF_PER_OBSERVATION
    jacobian: int = JACOBIAN_AUTODIFF
    check_rank_identity: bool = False
    collective_timeout: float = 60000.0  # milliseconds (std::chrono::milliseconds, dba/solver.hpp:54)
    # B200 extension: FP64 solve with the coupling blocks E
    # stored in FP32 (half the DSE stream; not the reference's numerics)
    coupling_fp32: bool = False

    def c_struct(self) -> N.Config:
        c = N.Config()
        c.workers, c.max_iterations, c.pcg_tol = self.workers, self.max_iterations, self.pcg_tol
        c.pcg_max_iters, c.lambda0, c.lambda_max = self.pcg_max_iters, self.lambda0, self.lambda_max
        c.rel_tol, c.step_tol, c.damping = self.rel_tol, self.step_tol, self.damping
        c.mse_half, c.jacobian, c.check_rank_identity = self.mse, self.jacobian, int(self.check_rank_identity)
        c.coupling_fp32 = int(self.coupling_fp32)
        c.collective_timeout_ms = int(self.collective_timeout)
        return c


@dataclass
class IterationRecord:
    """dba/solver.hpp:57-68."""
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
class SolverState:
    """dba/solver.hpp:70-85 (rank 0's state)."""
    x_c: np.ndarray
    x_p: np.ndarray
    lambda_: float
    nu: float
    iteration: int
    cost: float
    termination: str
    history: List[IterationRecord]
    # the most recent trial, feeding the convergence decision (dba/solver.hpp:80-84)
    last_accepted: bool = False
    last_cost_change: float = float("inf")
    last_step_inf: float = float("inf")
    previous_cost: float = float("inf")


CONVERGENCE = {0: "keep_going", 1: "converged", 2: "max_iterations", 3: "stalled"}


def check_convergence(state: SolverState, config: SolverConfig) -> str:
    """dba::check_convergence (dba/solver.hpp:91-104): "converged" when an
    accepted step changed the cost by less than rel_tol (relatively) or moved
    the state by less than step_tol; "stalled" when lambda exceeds
    lambda_max; "max_iterations" at the cap; else "keep_going"."""
    if state.last_accepted:
        denom = max(state.previous_cost, 1e-300)
        if abs(state.last_cost_change) / denom < config.rel_tol or state.last_step_inf < config.step_tol:
            return "converged"
    if state.lambda_ > config.lambda_max:
        return "stalled"
    if state.iteration >= config.max_iterations:
        return "max_iterations"
    return "keep_going"


class _ResultBuf:
    def __init__(self, cap: int, workers: int, m: int, n: int, dtype):
        self.cap, self.k = cap, workers
        self.it = np.zeros(cap, np.int32)
        self.cost = np.zeros(cap)
        self.mse = np.zeros(cap)
        self.lam = np.zeros(cap)
        self.pcg = np.zeros(cap, np.int32)
        self.acc = np.zeros(cap, np.int32)
        self.wall = np.zeros(cap)
        self.we = np.zeros(cap * workers, np.uint64)
        self.wb = np.zeros(cap * workers, np.uint64)
        self.xc = np.zeros(9 * m, dtype)
        self.xp = np.zeros(max(3 * n, 1), dtype)
        r = N.Result()
        r.capacity, r.workers = cap, workers
        P = C.POINTER
        r.rec_iteration = self.it.ctypes.data_as(P(C.c_int32))
        r.rec_cost = self.cost.ctypes.data_as(P(C.c_double))
        r.rec_mse = self.mse.ctypes.data_as(P(C.c_double))
        r.rec_lambda = self.lam.ctypes.data_as(P(C.c_double))
        r.rec_pcg = self.pcg.ctypes.data_as(P(C.c_int32))
        r.rec_accepted = self.acc.ctypes.data_as(P(C.c_int32))
        r.rec_wall = self.wall.ctypes.data_as(P(C.c_double))
        r.rec_worker_edges = self.we.ctypes.data_as(P(C.c_uint64))
        r.rec_worker_block_ops = self.wb.ctypes.data_as(P(C.c_uint64))
        r.x_c, r.x_p = self.xc.ctypes.data, self.xp.ctypes.data
        self.r = r

    def state(self, n: int) -> SolverState:
        r = self.r
        k = self.k
        hist = [IterationRecord(int(self.it[i]), float(self.cost[i]), float(self.mse[i]), float(self.lam[i]),
                                int(self.pcg[i]), bool(self.acc[i]), float(self.wall[i]),
                                [int(v) for v in self.we[i * k:(i + 1) * k]],
                                [int(v) for v in self.wb[i * k:(i + 1) * k]])
                for i in range(min(r.iterations, self.cap))]
        return SolverState(self.xc.copy(), self.xp[:3 * n].copy(), r.lam, r.nu, r.iterations, r.cost,
                           TERMINATION[r.termination], hist, bool(r.last_accepted), float(r.last_cost_change),
                           float(r.last_step_inf), float(r.previous_cost))


def lm_solve(problem: BAProblem, config: Optional[SolverConfig] = None, devices: Sequence[int] = (0,)) -> SolverState:
    """dba::lm_solve (dba/solver.hpp:523-534) on B200: partitions into
    config.workers ranks (one host thread + one rank context each, placed on
    devices[rank % len(devices)]), runs the distributed LM loop and returns
    rank 0's state."""
    config = config or SolverConfig()
    s = problem.c_struct()
    buf = _ResultBuf(config.max_iterations, config.workers, s.num_cameras, s.num_points, problem.dtype)
    devs = (C.c_int * len(devices))(*devices)
    cfg = config.c_struct()
    _check(N.lib().dbag_lm_solve(problem.precision, C.byref(s), C.byref(cfg), devs, len(devices), C.byref(buf.r)))
    return buf.state(s.num_points)


def nccl_unique_id() -> bytes:
    b = C.create_string_buffer(128)
    _check(N.lib().dbag_nccl_unique_id(b))
    return b.raw


def lm_solve_rank(problem: BAProblem, config: SolverConfig, rank: int, nranks: int, uid: bytes,
                  device: int) -> SolverState:
    """dba::lm_solve_rank (dba/solver.hpp:295-518) for one process per GPU over NCCL."""
    s = problem.c_struct()
    buf = _ResultBuf(config.max_iterations, nranks, s.num_cameras, s.num_points, problem.dtype)
    cfg = config.c_struct()
    idb = C.create_string_buffer(bytes(uid), 128)
    _check(N.lib().dbag_lm_solve_rank(problem.precision, C.byref(s), C.byref(cfg), rank, nranks, idb, device,
                                      C.byref(buf.r)))
    return buf.state(s.num_points)


def total_cost(problem: BAProblem, device: int = 0) -> float:
    """dba::total_cost (dba/problem.hpp:266-283) on the GPU."""
    with RankContext(device, problem.precision) as ctx:
        ctx.upload(problem)
        c, bad = ctx.cost()
        if bad >= 0:
            raise DegenerateDepthError(f"degenerate depth (P_z = 0) at edge {bad}", bad)
        return c


# ------------------------------------------------------------- synthetic --


@dataclass
class SyntheticOptions:
    """dba/synthetic.hpp:19-30 plus the count-exact / pixel-noise extension."""
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
    exhaustive_search: bool = False

    def c_struct(self) -> N.SynthOptions:
        o = N.SynthOptions()
        for f in dataclasses.fields(self):
            setattr(o, f.name, getattr(self, f.name))
        return o


def synthetic_observation_count(opt: SyntheticOptions) -> int:
    o = opt.c_struct()
    n = C.c_int64()
    _check(N.lib().dbag_synthetic_count(C.byref(o), C.byref(n)))
    return n.value


def generate_synthetic(opt: SyntheticOptions) -> BAProblem:
    """generate_synthetic (dba/synthetic.hpp:70-146), fp64, host-side."""
    nobs = synthetic_observation_count(opt)
    o = opt.c_struct()
    cams = np.zeros((opt.cameras, 9))
    pts = np.zeros((opt.points, 3))
    cid = np.zeros(nobs, np.int32)
    pid = np.zeros(nobs, np.int32)
    px = np.zeros(nobs)
    py = np.zeros(nobs)
    _check(N.lib().dbag_generate_synthetic(C.byref(o), cams.ctypes.data, pts.ctypes.data, cid.ctypes.data,
                                           pid.ctypes.data, px.ctypes.data, py.ctypes.data))
    return BAProblem.from_arrays(cams, pts, cid, pid, np.stack([px, py], 1))


# ------------------------------------------------------------ rank context --


class RankContext:
    """One rank's device context (include/dbag.h "rank context"): the operator
    level of lm_solve_rank. K = 1 unless created with ``nccl=(rank, nranks, uid)``."""

    def __init__(self, device: int = 0, precision: int = 8, nccl=None, coupling_fp32: bool = False, shard=None,
                 group=None):
        """shard=(rank, nranks): partition `rank` of `nranks` with local
        collectives (EdgeEvaluator / assemble_local semantics: costs and the
        assembled system are this partition's own contribution).
        group=(WorkerGroup, rank): rank `rank` of an in-process group (the
        reference's run_on_workers model; the device is the group's)."""
        self.precision = precision
        self.dtype = np.float64 if precision == 8 else np.float32
        h = C.c_void_p()
        if group is not None:
            g, rank = group
            _check(N.lib().dbag_create_group_rank(g.h, int(rank), precision, int(coupling_fp32), C.byref(h)))
        elif shard is not None:
            _check(N.lib().dbag_create_shard(device, precision, int(coupling_fp32), int(shard[0]), int(shard[1]),
                                             C.byref(h)))
        elif nccl is None:
            _check(N.lib().dbag_create_ex(device, precision, int(coupling_fp32), C.byref(h)))
        else:
            rank, nranks, uid = nccl
            _check(N.lib().dbag_create_nccl_ex(device, rank, nranks, C.create_string_buffer(bytes(uid), 128),
                                               precision, int(coupling_fp32), C.byref(h)))
        self.h = h
        self._group = group[0] if group is not None else None  # the group outlives its rank contexts
        self.m = self.n = self.nobs = 0

    def close(self):
        if self.h:
            N.lib().dbag_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, problem: BAProblem, jacobian: int = JACOBIAN_AUTODIFF):
        if problem.precision != self.precision:
            raise InvalidArgumentError("problem dtype does not match the context precision")
        s = problem.c_struct()
        self.m, self.n, self.nobs = s.num_cameras, s.num_points, s.num_observations
        _check(N.lib().dbag_upload_problem(self.h, C.byref(s), jacobian))

    def set_state(self, x_c, x_p):
        xc = np.ascontiguousarray(x_c, self.dtype)
        xp = np.ascontiguousarray(x_p, self.dtype)
        _check(N.lib().dbag_set_state(self.h, xc.ctypes.data, xp.ctypes.data))

    def get_state(self, out=None):
        """(x_c, x_p); ``out`` = preallocated (9m, >= 3n) arrays of the context
        dtype (e.g. pinned) to copy into."""
        if out is None:
            xc = np.zeros(9 * self.m, self.dtype)
            xp = np.zeros(max(3 * self.n, 1), self.dtype)
        else:
            xc, xp = out
            if xc.dtype != self.dtype or xp.dtype != self.dtype or xc.size < 9 * self.m or xp.size < 3 * self.n \
                    or not (xc.flags.c_contiguous and xp.flags.c_contiguous):
                raise InvalidArgumentError("get_state out arrays must be contiguous, sized and of the context dtype")
        _check(N.lib().dbag_get_state(self.h, xc.ctypes.data, xp.ctypes.data))
        return xc, xp[:3 * self.n]

    def cost(self, trial: bool = False):
        c, bad = C.c_double(), C.c_int64()
        _check(N.lib().dbag_cost(self.h, int(trial), C.byref(c), C.byref(bad)))
        return c.value, bad.value

    def linearize(self):
        bad = C.c_int64()
        _check(N.lib().dbag_linearize(self.h, C.byref(bad)))

    def damp_factor(self, lam: float, policy: int = DAMPING_DIAG_SCALED):
        self._damping = (float(lam), int(policy))
        _check(N.lib().dbag_damp_factor(self.h, lam, policy, None, None))

    def rhs(self):
        _check(N.lib().dbag_rhs(self.h))

    def pcg(self, tol: float, max_iters: int):
        it, conv = C.c_int(), C.c_int()
        _check(N.lib().dbag_pcg(self.h, tol, max_iters, C.byref(it), C.byref(conv)))
        return it.value, bool(conv.value)

    def backsub_trial(self):
        _check(N.lib().dbag_backsub_trial(self.h))

    def model_terms(self, lam: Optional[float] = None, policy: Optional[int] = None):
        """(step_inf, damping term, dx.v + dx.w) of the last trial; lam/policy
        default to the preceding damp_factor's (others raise)."""
        d_lam, d_pol = getattr(self, "_damping", (0.0, DAMPING_DIAG_SCALED))
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _check(N.lib().dbag_model_terms(self.h, d_lam if lam is None else lam, d_pol if policy is None else policy,
                                        C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def accept(self):
        _check(N.lib().dbag_accept(self.h))

    def probe_step(self, lam: float, config: SolverConfig):
        cost, it, acc = C.c_double(), C.c_int(), C.c_int()
        cfg = config.c_struct()
        _check(N.lib().dbag_lm_probe_step(self.h, lam, C.byref(cfg), C.byref(cost), C.byref(it), C.byref(acc)))
        return cost.value, it.value, bool(acc.value)

    def profile(self, enable: Optional[bool] = None):
        t, n, a, b = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(N.lib().dbag_profile(self.h, -1 if enable is None else int(enable), C.byref(t), C.byref(n),
                                    C.byref(a), C.byref(b)))
        return {"dse_ms": t.value, "dse_launches": n.value, "point_ms": a.value, "cam_ms": b.value}

    def mark(self, which: int):
        _check(N.lib().dbag_event_mark(self.h, which))

    def elapsed_ms(self) -> float:
        ms = C.c_double()
        _check(N.lib().dbag_event_elapsed(self.h, C.byref(ms)))
        return ms.value

    def synchronize(self):
        _check(N.lib().dbag_synchronize(self.h))

    def time_dse_pass(self, reps: int = 20) -> float:
        """Device ms per launch of the graph DPCG's DSE pass launched alone."""
        t = C.c_double()
        _check(N.lib().dbag_time_dse_pass(self.h, int(reps), C.byref(t)))
        return t.value

    def memory_pool(self):
        """(reserved, used) bytes of this context's device pool."""
        r, u = C.c_uint64(), C.c_uint64()
        _check(N.lib().dbag_memory_pool(self.h, C.byref(r), C.byref(u)))
        return r.value, u.value

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(N.lib().dbag_launch_count(self.h, C.byref(n)))
        return n.value

    def residuals(self, trial: bool = False):
        """Scalar-model residuals (2, N) in shard edge order (NaN on zero depth)."""
        out = np.zeros(max(2 * self.nobs, 1), self.dtype)
        _check(N.lib().dbag_residuals(self.h, int(trial), out.ctypes.data))
        return out[:2 * self.nobs].reshape(2, self.nobs)

    def jacobians(self):
        """EdgeJacobianBatch in shard edge order: residuals (2, N), J (2, 12, N)."""
        res = np.zeros(2 * self.nobs, self.dtype)
        jac = np.zeros(24 * self.nobs, self.dtype)
        _check(N.lib().dbag_get_jacobians(self.h, res.ctypes.data, jac.ctypes.data))
        return res.reshape(2, self.nobs), jac.reshape(2, 12, self.nobs)

    def system(self):
        """B (m,9,9), C (n,3,3), E (N,9,3), v (9m), w (3n) as assembled (all-reduced)."""
        B = np.zeros(81 * self.m, self.dtype)
        Cm = np.zeros(max(9 * self.n, 1), self.dtype)
        E = np.zeros(max(27 * self.nobs, 1), self.dtype)
        v = np.zeros(9 * self.m, self.dtype)
        w = np.zeros(max(3 * self.n, 1), self.dtype)
        _check(N.lib().dbag_get_system(self.h, B.ctypes.data, Cm.ctypes.data, E.ctypes.data, v.ctypes.data,
                                       w.ctypes.data))
        return (B.reshape(-1, 9, 9), Cm[:9 * self.n].reshape(-1, 3, 3), E[:27 * self.nobs].reshape(-1, 9, 3), v,
                w[:3 * self.n])

    def set_system(self, B=None, Cb=None, E_table=None, v=None, w=None):
        arr = [None if a is None else np.ascontiguousarray(a, self.dtype) for a in (B, Cb, E_table, v, w)]
        ptr = [None if a is None else a.ctypes.data for a in arr]
        _check(N.lib().dbag_set_system(self.h, *ptr))

    def dse(self, x):
        x = np.ascontiguousarray(x, self.dtype)
        out = np.zeros_like(x)
        _check(N.lib().dbag_dse(self.h, x.ctypes.data, out.ctypes.data))
        return out

    def dpcg(self, rhs, tol: float, max_iters: int):
        rhs = np.ascontiguousarray(rhs, self.dtype)
        x = np.zeros_like(rhs)
        it, conv = C.c_int(), C.c_int()
        _check(N.lib().dbag_dpcg(self.h, rhs.ctypes.data, tol, max_iters, x.ctypes.data, C.byref(it),
                                 C.byref(conv)))
        return x, it.value, bool(conv.value)


def group_operator(problem: BAProblem, k: int, x, mode: int = 0, lam: float = 0.0, policy: int = DAMPING_IDENTITY,
                   blocks=None, tol: float = 1e-12, max_iters: int = 500, device: int = 0):
    """K in-process ranks on one device: mode 0 -> dse(x), mode 1 -> dpcg(rhs=x)
    on the problem's own damped system, or on fabricated (B, C, E_table);
    modes 2-5 expose one LM trial's pieces on the problem's system (rank 0's
    values): 2 the right-hand side g, 3 dx_c after DPCG(tol, max_iters),
    4 [trial cost, step_inf, damping term, dx.v + dx.w], 5 the gradient v."""
    s = problem.c_struct()
    d = problem.dtype
    x = np.ascontiguousarray(x, d)
    out = np.zeros_like(x)
    it, ident = C.c_int(), C.c_int()
    if blocks is not None:
        B, Cb, E = (np.ascontiguousarray(a, d) for a in blocks)
        bp, cp, ep = B.ctypes.data, Cb.ctypes.data, E.ctypes.data
    else:
        bp = cp = ep = None
    _check(N.lib().dbag_group_operator(problem.precision, C.byref(s), k, device, lam, policy, bp, cp, ep, mode,
                                       x.ctypes.data, tol, max_iters, out.ctypes.data, C.byref(it), C.byref(ident)))
    return out, it.value, bool(ident.value)


def group_allreduce(data: np.ndarray, device: int = 0) -> np.ndarray:
    """WorkerGroup::allreduce_sum over K = data.shape[0] in-process ranks."""
    a = np.ascontiguousarray(data, np.float64).copy()
    _check(N.lib().dbag_group_allreduce(a.shape[0], device, a.shape[1], a.ctypes.data))
    return a


class WorkerGroup:
    """dba::WorkerGroup (dba/comms.hpp:35-234) over K in-process ranks on
    GPUs: every rank calls from its own thread (run_on_workers). Collectives
    validate sequence / kind / type / length; a missing rank trips the
    timeout (CollectiveError naming the absent ranks); abort() fails every
    pending and later collective. allreduce_sum reduces in ascending rank
    order on the device: bit-identical on every rank."""

    def __init__(self, workers: int, timeout_ms: float = 60000.0, devices: Sequence[int] = (0,)):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(N.lib().dbag_group_create(int(workers), devs, len(devices), int(timeout_ms), C.byref(h)))
        self.h, self.k = h, int(workers)

    def workers(self) -> int:
        return self.k

    def close(self):
        if self.h:
            N.lib().dbag_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def barrier(self, rank: int):
        _check(N.lib().dbag_group_barrier(self.h, int(rank)))

    def allreduce_sum(self, rank: int, data: np.ndarray):
        """In place on a contiguous float32/float64 array."""
        if data.dtype not in (np.float32, np.float64) or not data.flags.c_contiguous:
            raise InvalidArgumentError("allreduce_sum needs a contiguous float32/float64 array")
        _check(N.lib().dbag_group_allreduce_sum(self.h, int(rank), data.ctypes.data, data.size, data.itemsize))
        return data

    def abort(self, reason: str = "aborted"):
        _check(N.lib().dbag_group_abort(self.h, reason.encode()))

    def sequence(self, rank: int) -> int:
        v = C.c_uint64()
        _check(N.lib().dbag_group_sequence(self.h, int(rank), C.byref(v)))
        return v.value


def run_on_workers(group: WorkerGroup, body):
    """dba::run_on_workers (dba/comms.hpp:214-234): body(rank) on one thread
    per rank; the first failure aborts the group and is re-raised after all
    threads joined."""
    import threading
    first = []
    lock = threading.Lock()

    def run(r):
        try:
            body(r)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            with lock:
                if not first:
                    first.append(e)
            try:
                group.abort(f"rank {r} failed: {e}")
            except Error:
                pass

    th = [threading.Thread(target=run, args=(r,)) for r in range(group.workers())]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if first:
        raise first[0]


def device_count() -> int:
    n = C.c_int()
    _check(N.lib().dbag_device_count(C.byref(n)))
    return n.value
