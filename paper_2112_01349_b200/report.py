"""Run report, schema 1 (dba/report.hpp:13-166).

Same document as the reference's ``serialize_report``: fixed key order,
two-space indentation, doubles in nlohmann::json's shortest round-trip
format, so ``serialize_report(report_from_json(text)) == text`` byte for
byte (tests/test_generator_report.cpp:105-115).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List

from .dba import (DAMPING_DIAG_SCALED, DAMPING_IDENTITY, JACOBIAN_ANALYTIC, JACOBIAN_AUTODIFF,
                  MSE_HALF_PER_OBSERVATION, MSE_PER_OBSERVATION, InvalidArgumentError, IterationRecord, ParseError,
                  SolverConfig, SolverState, mse_from_cost)


@dataclass
class RunReport:
    """dba/report.hpp:13-25."""
    schema: int = 1
    dataset: str = ""
    workers: int = 1
    precision: str = "fp64"
    config: SolverConfig = field(default_factory=SolverConfig)
    iterations: List[IterationRecord] = field(default_factory=list)
    final_cost: float = 0.0
    final_mse: float = 0.0
    final_mse_alternate: float = 0.0
    termination: str = "converged"


# -- enum <-> string (dba/report.hpp:27-57)
def mse_to_string(c: int) -> str:
    return "2n" if c == MSE_HALF_PER_OBSERVATION else "n"


def mse_from_string(s: str) -> int:
    if s == "2n":
        return MSE_HALF_PER_OBSERVATION
    if s == "n":
        return MSE_PER_OBSERVATION
    raise InvalidArgumentError(f"unknown MSE convention '{s}' (use n or 2n)")


def jacobian_to_string(m: int) -> str:
    return "analytic" if m == JACOBIAN_ANALYTIC else "auto"


def jacobian_from_string(s: str) -> int:
    if s == "auto":
        return JACOBIAN_AUTODIFF
    if s == "analytic":
        return JACOBIAN_ANALYTIC
    raise InvalidArgumentError(f"unknown Jacobian mode '{s}' (use auto or analytic)")


def damping_to_string(p: int) -> str:
    return "identity" if p == DAMPING_IDENTITY else "diagonal"


def damping_from_string(s: str) -> int:
    if s == "identity":
        return DAMPING_IDENTITY
    if s == "diagonal":
        return DAMPING_DIAG_SCALED
    raise InvalidArgumentError(f"unknown damping policy '{s}' (use identity or diagonal)")


def make_report(dataset: str, config: SolverConfig, state: SolverState, num_observations: int,
                precision: str = "fp64") -> RunReport:
    """dba/report.hpp:59-79."""
    other = MSE_PER_OBSERVATION if config.mse == MSE_HALF_PER_OBSERVATION else MSE_HALF_PER_OBSERVATION
    return RunReport(dataset=dataset, workers=config.workers, precision=precision, config=config,
                     iterations=list(state.history), final_cost=state.cost,
                     final_mse=mse_from_cost(state.cost, num_observations, config.mse),
                     final_mse_alternate=mse_from_cost(state.cost, num_observations, other),
                     termination=state.termination)


def _fmt_double(v: float) -> str:
    """nlohmann::json's float output: shortest round-trip digits, fixed
    notation for decimal exponents in (-4, 15], else d.ddde+XX; non-finite
    values become null."""
    if not math.isfinite(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    mant, _, exp = repr(abs(v)).partition("e")
    e10 = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    lead = len(ip.lstrip("0")) if ip.strip("0") else -(len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    n = lead + e10  # value = 0.d1..dk x 10^n
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        out = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + out


def _dump(v, ind: int) -> str:
    pad, pad_in = " " * ind, " " * (ind + 2)
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _fmt_double(v)
    if isinstance(v, str):
        return json.dumps(v, ensure_ascii=False)
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(pad_in + _dump(x, ind + 2) for x in v) + "\n" + pad + "]"
    if isinstance(v, dict):
        if not v:
            return "{}"
        return "{\n" + ",\n".join(f"{pad_in}{json.dumps(k, ensure_ascii=False)}: {_dump(x, ind + 2)}"
                                  for k, x in v.items()) + "\n" + pad + "}"
    raise TypeError(type(v))


def to_json(r: RunReport) -> dict:
    """dba/report.hpp:81-119 (insertion order = key order)."""
    c = r.config
    return {
        "schema": r.schema, "dataset": r.dataset, "workers": r.workers, "precision": r.precision,
        "config": {"max_iterations": c.max_iterations, "pcg_tol": float(c.pcg_tol), "pcg_max_iters": c.pcg_max_iters,
                   "lambda0": float(c.lambda0), "lambda_max": float(c.lambda_max), "rel_tol": float(c.rel_tol),
                   "step_tol": float(c.step_tol), "damping": damping_to_string(c.damping),
                   "mse_convention": mse_to_string(c.mse), "jacobian": jacobian_to_string(c.jacobian)},
        "iterations": [{"iteration": it.iteration, "cost": float(it.cost), "mse": float(it.mse),
                        "lambda": float(it.lambda_), "pcg_iterations": it.pcg_iterations, "accepted": bool(it.accepted),
                        "wall_seconds": float(it.wall_seconds), "worker_edges": [int(x) for x in it.worker_edges],
                        "worker_block_ops": [int(x) for x in it.worker_block_ops]} for it in r.iterations],
        "final_cost": float(r.final_cost), "final_mse": float(r.final_mse),
        "final_mse_alternate": float(r.final_mse_alternate), "termination": r.termination,
    }


def serialize_report(r: RunReport) -> str:
    """dba/report.hpp:165-167: to_json(r).dump(2) + "\\n"."""
    return _dump(to_json(r), 0) + "\n"


def _num(x) -> float:
    return float("inf") if x is None else float(x)


def report_from_json(j) -> RunReport:
    """dba/report.hpp:121-163. ``j`` is the parsed document or its text."""
    if isinstance(j, (str, bytes)):
        j = json.loads(j)
    try:
        schema = int(j["schema"])
        if schema != 1:
            raise ParseError(f"unsupported report schema {schema}", 0)
        c = j["config"]
        cfg = SolverConfig(workers=int(j["workers"]), max_iterations=int(c["max_iterations"]), pcg_tol=_num(c["pcg_tol"]),
                           pcg_max_iters=int(c["pcg_max_iters"]), lambda0=_num(c["lambda0"]),
                           lambda_max=_num(c["lambda_max"]), rel_tol=_num(c["rel_tol"]), step_tol=_num(c["step_tol"]),
                           damping=damping_from_string(c["damping"]), mse=mse_from_string(c["mse_convention"]),
                           jacobian=jacobian_from_string(c["jacobian"]))
        its = [IterationRecord(int(i["iteration"]), _num(i["cost"]), _num(i["mse"]), _num(i["lambda"]),
                               int(i["pcg_iterations"]), bool(i["accepted"]), _num(i["wall_seconds"]),
                               [int(x) for x in i["worker_edges"]], [int(x) for x in i["worker_block_ops"]])
               for i in j["iterations"]]
        return RunReport(schema=schema, dataset=str(j["dataset"]), workers=int(j["workers"]),
                         precision="fp32" if j["precision"] == "fp32" else "fp64", config=cfg, iterations=its,
                         final_cost=_num(j["final_cost"]), final_mse=_num(j["final_mse"]),
                         final_mse_alternate=_num(j["final_mse_alternate"]), termination=str(j["termination"]))
    except KeyError as e:
        raise ParseError(f"report is missing key {e}", 0) from None
