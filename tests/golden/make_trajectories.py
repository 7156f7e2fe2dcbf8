"""Generates tests/golden/trajectories.json: the CPU oracle's LM trajectories
on the BASELINE.md §3 instances (dba/synthetic.hpp ring, seed 1, count-exact,
+-0.5 px noise) at SolverConfig defaults, max_iterations 10, for several
worker counts K. The reference's own results differ across K by float
reassociation only (dba/comms.hpp:32-33); the spread over K is the yardstick
the GPU parity tests use where the north_star's 1e-6 / 1e-4 per-iteration
bar is below the reference's own reproducibility.

The oracle is deterministic for a fixed K (fixed association everywhere), so
these files equal a live oracle run. Run from the repo root:
    python tests/golden/make_trajectories.py [config ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

SHAPES = {"ladybug-49": (49, 7776, 31843), "trafalgar-257": (257, 65132, 225911),
          "venice-1778": (1778, 993923, 5001946)}
ITERS = {"venice-1778/f64": 2}  # 4-6 CPU minutes per run on 8-16 threads: the first two iterations
RUNS = {  # name -> (shape, dtype, K values)
    "ladybug-49/f64": ("ladybug-49", np.float64, (1, 2, 3, 4, 5, 6, 7, 8)),
    "ladybug-49/f32": ("ladybug-49", np.float32, (1, 2, 3, 4, 5, 6, 7, 8)),
    "trafalgar-257/f64": ("trafalgar-257", np.float64, (1, 2, 3, 4, 5, 6, 7, 8)),
    "trafalgar-257/f32": ("trafalgar-257", np.float32, (1, 2, 3, 4, 5, 6, 7, 8)),
    "venice-1778/f64": ("venice-1778", np.float64, (4, 8, 16)),
}
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "trajectories.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        shape, dtype, ks = RUNS[name]
        m, n, N = SHAPES[shape]
        p = O.generate_synthetic(O.SynthOptions(cameras=m, points=n, num_observations=N, seed=1, pixel_noise=0.5))
        p = p.astype(dtype)
        iters = ITERS.get(name, 10)
        entry = {"shape": [m, n, N], "dtype": np.dtype(dtype).name, "max_iterations": iters, "runs": {}}
        for k in ks:
            t = time.time()
            st = O.lm_solve(p, O.OracleConfig(workers=k, max_iterations=iters))
            entry["runs"][str(k)] = {
                "cost": [r.cost for r in st.history], "lambda": [r.lambda_ for r in st.history],
                "accepted": [r.accepted for r in st.history], "pcg": [r.pcg_iterations for r in st.history],
                "final_cost": st.cost, "termination": st.termination, "seconds": time.time() - t}
            print(name, k, f"{time.time() - t:.1f}s", st.termination, [f"{c:.9e}" for c in entry["runs"][str(k)]["cost"]],
                  flush=True)
        data[name] = entry
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(RUNS))
