"""B200-native bundle-adjustment inner loop (MegBA, arXiv 2112.01349).

Drop-in for the reference's ``dba`` LM / DSE / DPCG path: the public names of
``dba.py`` mirror the reference's C++ API; every operator runs in the in-tree
``libdbag.so`` (hand-written sm_100a kernels + C++ host runtime, C ABI in
``include/dbag.h``). There is no CPU fallback.
"""
from . import _native
from .dba import *  # noqa: F401,F403
from .dba import (BAProblem, CameraState, PointState, Observation, SolverConfig, SolverState, IterationRecord,
                  SyntheticOptions, RankContext, lm_solve, lm_solve_rank, partition_edges, generate_synthetic,
                  group_operator, group_allreduce, shared_points, predict_memory, nccl_unique_id, total_cost,
                  device_count, check_convergence, pack_cameras, pack_points, unpack_states, mse_from_cost)
from .bal_io import parse_bal, serialize_bal, format_bal
from .report import RunReport, make_report, serialize_report, report_from_json, to_json

__all__ = ["BAProblem", "CameraState", "PointState", "Observation", "SolverConfig", "SolverState",
           "IterationRecord", "SyntheticOptions", "RankContext", "lm_solve", "lm_solve_rank", "partition_edges",
           "generate_synthetic", "group_operator", "group_allreduce", "shared_points", "predict_memory", "nccl_unique_id",
           "total_cost", "device_count", "check_convergence", "pack_cameras", "pack_points", "unpack_states", "mse_from_cost", "parse_bal", "serialize_bal", "format_bal", "RunReport", "make_report",
           "serialize_report", "report_from_json", "to_json"]
