"""Event-timed standalone DSE pass (k_g_pass) after one LM step: the kernel the
ncu full captures in profiles/ are taken from (-k regex:k_g_pass)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2112_01349_b200 as dba
name = sys.argv[1] if len(sys.argv) > 1 else "trafalgar-257"
p = bench.make_problem(name)
with dba.RankContext(0, 8) as ctx:
    ctx.upload(p)
    cfg = dba.SolverConfig()
    ctx.probe_step(cfg.lambda0, cfg)
    print(name, "k_g_pass ms", ctx.time_dse_pass(20), flush=True)
