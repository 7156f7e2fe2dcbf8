"""Per-PCG-iteration timeline of the graph DPCG: run with DBAG_LIB pointing at
the DBAG_GTIMING build (make -C paper_2112_01349_b200/csrc gt); one LM step
per workload, the library prints the averaged marks to stderr."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2112_01349_b200 as dba
for name in sys.argv[1:] or ["trafalgar-257", "venice-1778"]:
    p = bench.make_problem(name)
    with dba.RankContext(0, 8) as ctx:
        ctx.upload(p)
        cfg = dba.SolverConfig()
        for _ in range(3):
            ctx.synchronize(); ctx.mark(0)
            ctx.probe_step(cfg.lambda0, cfg)
            ctx.mark(1)
            print(name, "step ms", ctx.elapsed_ms(), flush=True)
        sys.stderr.flush()
