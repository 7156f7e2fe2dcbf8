"""Event-timed standalone DSE pass (k_g_pass) after one LM step: the kernel the
ncu full captures in profiles/ are taken from (-k regex:k_g_pass; ncu cannot
profile kernel nodes of a graph with conditional nodes, so the in-graph
launches are captured as these standalone launches on the same state).

  pass_only.py [workload] [precision 8|4] [lean]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import bench
import paper_2112_01349_b200 as dba
name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lean = len(sys.argv) > 3 and sys.argv[3] == "lean"
p = bench.make_problem(name, np.float64 if s == 8 else np.float32)
with dba.RankContext(0, s, coupling_fp32=lean) as ctx:
    ctx.upload(p)
    cfg = dba.SolverConfig()
    ctx.probe_step(cfg.lambda0, cfg)
    print(name, s, "lean" if lean else "", "k_g_pass ms", ctx.time_dse_pass(20), flush=True)
