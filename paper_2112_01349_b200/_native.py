"""ctypes binding of libdbag.so (include/dbag.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2112_01349_b200/csrc``). There is no fallback: importing the package
without the library raises, and every GPU operator runs in the library.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBAG_LIB") or os.path.join(_HERE, "libdbag.so")

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp, cvp = C.c_void_p, C.c_void_p


class Problem(C.Structure):
    _fields_ = [("num_cameras", i32), ("num_points", i32), ("num_observations", i64),
                ("cameras", vp), ("points", vp), ("camera_id", C.POINTER(i32)),
                ("point_id", C.POINTER(i32)), ("pixel_x", vp), ("pixel_y", vp), ("weight", vp)]


class Config(C.Structure):
    _fields_ = [("workers", i32), ("max_iterations", i32), ("pcg_tol", f64), ("pcg_max_iters", i32),
                ("coupling_fp32", i32), ("lambda0", f64), ("lambda_max", f64), ("rel_tol", f64), ("step_tol", f64),
                ("damping", i32), ("mse_half", i32), ("jacobian", i32), ("check_rank_identity", i32),
                ("collective_timeout_ms", i64)]


class Result(C.Structure):
    _fields_ = [("iterations", i32), ("termination", i32), ("cost", f64), ("lam", f64), ("nu", f64),
                ("capacity", i32), ("workers", i32), ("rec_iteration", C.POINTER(i32)),
                ("rec_cost", C.POINTER(f64)), ("rec_mse", C.POINTER(f64)), ("rec_lambda", C.POINTER(f64)),
                ("rec_pcg", C.POINTER(i32)), ("rec_accepted", C.POINTER(i32)), ("rec_wall", C.POINTER(f64)),
                ("rec_worker_edges", C.POINTER(u64)), ("rec_worker_block_ops", C.POINTER(u64)),
                ("x_c", vp), ("x_p", vp), ("last_accepted", i32), ("last_cost_change", f64),
                ("last_step_inf", f64), ("previous_cost", f64)]


class SynthOptions(C.Structure):
    _fields_ = [("cameras", i32), ("points", i32), ("obs_per_point", i32), ("exhaustive_search", i32), ("seed", u64),
                ("circle_radius", f64), ("base_focal", f64), ("pose_noise", f64), ("intrinsic_noise", f64),
                ("point_noise", f64), ("num_observations", i64), ("pixel_noise", f64)]


_P = C.POINTER
_SIGS = {
    "dbag_version": (C.c_int, []),
    "dbag_last_error": (C.c_char_p, []),
    "dbag_last_error_index": (i64, []),
    "dbag_last_error_block_size": (C.c_int, []),
    "dbag_default_config": (None, [_P(Config)]),
    "dbag_device_count": (C.c_int, [_P(C.c_int)]),
    "dbag_partition": (C.c_int, [_P(Problem), C.c_int, C.c_int, _P(i64), _P(i64), _P(i32), vp, _P(i32), vp, vp,
                                 vp, vp, vp]),
    "dbag_shared_points": (C.c_int, [_P(Problem), C.c_int, _P(i64), vp]),
    "dbag_predict_memory": (C.c_int, [_P(Problem), C.c_int, C.c_int, C.c_int, C.c_int, _P(u64)]),
    "dbag_memory_pool": (C.c_int, [vp, _P(u64), _P(u64)]),
    "dbag_synthetic_count": (C.c_int, [_P(SynthOptions), _P(i64)]),
    "dbag_generate_synthetic": (C.c_int, [_P(SynthOptions), vp, vp, vp, vp, vp, vp]),
    "dbag_lm_solve": (C.c_int, [C.c_int, _P(Problem), _P(Config), _P(C.c_int), C.c_int, _P(Result)]),
    "dbag_nccl_unique_id": (C.c_int, [vp]),
    "dbag_lm_solve_rank": (C.c_int, [C.c_int, _P(Problem), _P(Config), C.c_int, C.c_int, vp, C.c_int,
                                     _P(Result)]),
    "dbag_create": (C.c_int, [C.c_int, C.c_int, _P(vp)]),
    "dbag_create_ex": (C.c_int, [C.c_int, C.c_int, C.c_int, _P(vp)]),
    "dbag_create_nccl": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.c_int, _P(vp)]),
    "dbag_create_nccl_ex": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, _P(vp)]),
    "dbag_group_create": (C.c_int, [C.c_int, _P(C.c_int), C.c_int, i64, _P(vp)]),
    "dbag_group_destroy": (C.c_int, [vp]),
    "dbag_group_barrier": (C.c_int, [vp, C.c_int]),
    "dbag_group_allreduce_sum": (C.c_int, [vp, C.c_int, vp, i64, C.c_int]),
    "dbag_group_abort": (C.c_int, [vp, C.c_char_p]),
    "dbag_group_sequence": (C.c_int, [vp, C.c_int, _P(u64)]),
    "dbag_destroy": (C.c_int, [vp]),
    "dbag_create_shard": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P(vp)]),
    "dbag_create_group_rank": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, _P(vp)]),
    "dbag_lm_solve_ctx": (C.c_int, [vp, _P(Config), _P(Result)]),
    "dbag_block_factor": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, vp, vp, _P(i64)]),
    "dbag_block_solve": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, vp, vp]),
    "dbag_upload_problem": (C.c_int, [vp, _P(Problem), C.c_int]),
    "dbag_set_state": (C.c_int, [vp, vp, vp]),
    "dbag_get_state": (C.c_int, [vp, vp, vp]),
    "dbag_cost": (C.c_int, [vp, C.c_int, _P(f64), _P(i64)]),
    "dbag_linearize": (C.c_int, [vp, _P(i64)]),
    "dbag_damp_factor": (C.c_int, [vp, f64, C.c_int, _P(i64), _P(C.c_int)]),
    "dbag_rhs": (C.c_int, [vp]),
    "dbag_pcg": (C.c_int, [vp, f64, C.c_int, _P(C.c_int), _P(C.c_int)]),
    "dbag_backsub_trial": (C.c_int, [vp]),
    "dbag_model_terms": (C.c_int, [vp, f64, C.c_int, _P(f64), _P(f64), _P(f64)]),
    "dbag_accept": (C.c_int, [vp]),
    "dbag_lm_probe_step": (C.c_int, [vp, f64, _P(Config), _P(f64), _P(C.c_int), _P(C.c_int)]),
    "dbag_profile": (C.c_int, [vp, C.c_int, _P(f64), _P(i64), _P(f64), _P(f64)]),
    "dbag_event_mark": (C.c_int, [vp, C.c_int]),
    "dbag_event_elapsed": (C.c_int, [vp, _P(f64)]),
    "dbag_synchronize": (C.c_int, [vp]),
    "dbag_time_dse_pass": (C.c_int, [vp, C.c_int, _P(f64)]),
    "dbag_launch_count": (C.c_int, [vp, _P(i64)]),
    "dbag_residuals": (C.c_int, [vp, C.c_int, vp]),
    "dbag_get_jacobians": (C.c_int, [vp, vp, vp]),
    "dbag_get_system": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "dbag_set_system": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "dbag_dse": (C.c_int, [vp, vp, vp]),
    "dbag_dpcg": (C.c_int, [vp, vp, f64, C.c_int, vp, _P(C.c_int), _P(C.c_int)]),
    "dbag_group_operator": (C.c_int, [C.c_int, _P(Problem), C.c_int, C.c_int, f64, C.c_int, vp, vp, vp, C.c_int,
                                      vp, f64, C.c_int, vp, _P(C.c_int), _P(C.c_int)]),
    "dbag_group_allreduce": (C.c_int, [C.c_int, C.c_int, i64, vp]),
    "dbag_bal_parse": (C.c_int, [C.c_char_p, i64, _P(vp)]),
    "dbag_bal_counts": (C.c_int, [vp, _P(i32), _P(i32), _P(i64)]),
    "dbag_bal_copy": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "dbag_bal_free": (C.c_int, [vp]),
    "dbag_bal_format": (C.c_int, [C.c_int, _P(Problem), _P(C.c_void_p), _P(i64)]),
    "dbag_free_text": (C.c_int, [vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """The loaded libdbag.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2112_01349_b200/csrc); there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib
