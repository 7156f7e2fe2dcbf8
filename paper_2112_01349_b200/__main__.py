"""``python -m paper_2112_01349_b200 {solve,generate}`` — the reference's `dba`
front end (tools/dba_main.cpp:45-233) on the B200 solver.

solve     parse a BAL file, lm_solve on the GPU(s), schema-1 JSON run report
          (stdout or --output), per-iteration log on stderr. Exit 0; 2 on
          usage / parse / report-write errors; 3 on a fatal solver error
          (a partial report is still written) or a stalled run.
generate  emit a synthetic ring dataset (dba/synthetic.hpp) as BAL text.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

EXIT_USAGE, EXIT_SOLVER_FATAL = 2, 3


def _err(msg: str) -> None:
    sys.stderr.write(msg + "\n")


def _write_report(text: str, path: str) -> None:
    if not path:
        sys.stdout.write(text)
        sys.stdout.flush()
        return
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise RuntimeError(f"cannot write report to {path}") from None


def run_solve(a) -> int:
    """tools/dba_main.cpp:45-127."""
    from . import dba as D
    from .bal_io import parse_bal
    from .report import (RunReport, damping_from_string, jacobian_from_string, make_report, mse_from_string,
                         serialize_report)
    dtype = np.float32 if a.precision == "fp32" else np.float64
    try:
        with open(a.input, "rb") as f:
            text = f.read()
    except OSError:
        _err(f"error: cannot open {a.input}")
        return EXIT_USAGE
    try:
        warnings = []
        problem = parse_bal(text, dtype=dtype, warnings=warnings)
        for w in warnings:
            _err(f"warning: {w}")
    except D.ParseError as e:
        _err(f"error: {a.input}: {e}")
        return EXIT_USAGE
    config = D.SolverConfig(workers=a.workers, max_iterations=a.max_iters, pcg_tol=a.pcg_tol,
                            pcg_max_iters=a.pcg_max_iters, lambda0=a.lambda0, rel_tol=a.rel_tol, step_tol=a.step_tol,
                            mse=mse_from_string(a.mse_convention), damping=damping_from_string(a.damping),
                            jacobian=jacobian_from_string(a.jacobian))
    dataset = os.path.splitext(os.path.basename(a.input))[0]
    n_obs = problem.num_observations
    _err(f"{dataset}: {problem.num_cameras} cameras, {problem.num_points} points, {n_obs} observations, "
         f"K={config.workers}, {a.precision}")
    devices = [int(d) for d in a.devices.split(",")] if a.devices else [0]
    try:
        state = D.lm_solve(problem, config, devices=devices)
    except Exception as e:  # noqa: BLE001 — the reference catches std::exception here
        _err(f"solver error: {e}")
        partial = RunReport(dataset=dataset, workers=config.workers, precision=a.precision, config=config,
                            termination=f"fatal: {e}")
        try:
            _write_report(serialize_report(partial), a.output)
        except RuntimeError as io:
            _err(f"error: {io}")
        return EXIT_SOLVER_FATAL
    for rec in state.history:
        if a.log_every > 0 and (rec.iteration % a.log_every == 0 or rec.iteration == state.iteration):
            _err(f"iter {rec.iteration}{'  ' if rec.accepted else ' r'}  cost {rec.cost:g}  mse {rec.mse:g}  "
                 f"lambda {rec.lambda_:g}  pcg {rec.pcg_iterations}  t {rec.wall_seconds:g}s")
    _err(f"{state.termination} after {state.iteration} iterations, final mse "
         f"{D.mse_from_cost(state.cost, n_obs, config.mse):g}")
    try:
        _write_report(serialize_report(make_report(dataset, config, state, n_obs, a.precision)), a.output)
    except RuntimeError as e:
        _err(f"error: {e}")
        return EXIT_USAGE
    return EXIT_SOLVER_FATAL if state.termination == "stalled" else 0


def run_generate(a) -> int:
    """tools/dba_main.cpp:173-225."""
    from . import dba as D
    from .bal_io import serialize_bal

    def scaled(full: int) -> int:
        return max(1, int(full * a.scale))

    opt = D.SyntheticOptions(cameras=a.cameras if a.cameras is not None else scaled(20000),
                             points=a.points if a.points is not None else scaled(80000),
                             obs_per_point=a.obs_per_point if a.obs_per_point is not None else scaled(1000),
                             seed=a.seed, num_observations=a.num_observations or 0, pixel_noise=a.pixel_noise)
    problem = D.generate_synthetic(opt)
    if a.output:
        try:
            serialize_bal(problem, a.output)
        except OSError:
            _err(f"error: cannot write {a.output}")
            return EXIT_USAGE
    else:
        serialize_bal(problem, sys.stdout)
        sys.stdout.flush()
    _err(f"generated {opt.cameras} cameras, {opt.points} points, {problem.num_observations} observations "
         f"(seed {opt.seed})")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="dba", description="B200 bundle adjustment on BAL problems: distributed Schur "
                                 "elimination + PCG inside a Levenberg-Marquardt loop")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve a BAL problem file")
    s.add_argument("--input", required=True, help="BAL problem file")
    s.add_argument("--workers", type=int, default=1, help="number of ranks (K)")
    s.add_argument("--precision", default="fp64", choices=["fp32", "fp64"])
    s.add_argument("--max-iters", type=int, default=50, help="outer iteration cap")
    s.add_argument("--pcg-tol", type=float, default=1e-6, help="relative PCG residual tolerance")
    s.add_argument("--pcg-max-iters", type=int, default=500, help="PCG iteration cap")
    s.add_argument("--lambda0", type=float, default=1e-4, help="initial LM damping")
    s.add_argument("--rel-tol", type=float, default=1e-6, help="relative cost-change convergence tolerance")
    s.add_argument("--step-tol", type=float, default=1e-8, help="step infinity-norm convergence tolerance")
    s.add_argument("--mse-convention", default="2n", choices=["n", "2n"])
    s.add_argument("--damping", default="diagonal", choices=["identity", "diagonal"])
    s.add_argument("--jacobian", default="auto", choices=["auto", "analytic"])
    s.add_argument("--output", default="", help="write the JSON run report here (default: stdout)")
    s.add_argument("--log-every", type=int, default=1, help="print every Nth iteration (0 silences the log)")
    s.add_argument("--devices", default="0", help="CUDA devices for the ranks, comma separated (rank r on r mod D)")
    g = sub.add_parser("generate", help="emit a synthetic ring dataset as a BAL file")
    g.add_argument("--cameras", type=int)
    g.add_argument("--points", type=int)
    g.add_argument("--obs-per-point", type=int)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--scale", type=float, default=1.0,
                   help="scale the default full-size counts (20000/80000/1000); explicit count flags win")
    g.add_argument("--num-observations", type=int, default=0, help="count-exact edge total (BAL-shaped instances)")
    g.add_argument("--pixel-noise", type=float, default=0.0, help="U(-a, a) pixel noise (tests/acceptance.cpp:88-99)")
    g.add_argument("--output", default="", help="output BAL file (default: stdout)")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code else 0
    from . import dba as D
    try:
        return run_solve(a) if a.cmd == "solve" else run_generate(a)
    except D.Error as e:
        _err(f"error: {e}")
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001
        _err(f"error: {e}")
        return EXIT_SOLVER_FATAL


if __name__ == "__main__":
    sys.exit(main())
