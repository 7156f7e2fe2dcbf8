"""One bounded CPU-reference sample at final-13682 (oracle port, all host
cores): DPCG capped at bench.PCG_SAMPLE iterations, scaled to the GPU step's
511 DSEs (500 PCG iterations + 10 refreshes + the DSE on x0)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
t0 = time.perf_counter()
p = bench.make_oracle_problem("final-13682")
tgen = time.perf_counter() - t0
k = bench.cpu_threads()
secs, info = bench.cpu_reference_steps(p, k, 1, dse_full=511, calibrate=False)
N = bench.WORKLOADS["final-13682"][2]
print(json.dumps({"workload": "final-13682", "cores": k, "host": bench.host_info(), "instance_generation_s": tgen,
                  "t_lm_s_scaled": secs[0], "edges_per_s": N / secs[0], "detail": info,
                  "sample": "one LM iteration from x0, DPCG capped at %d iterations, scaled to 511 DSEs" % bench.PCG_SAMPLE,
                  "wall_s": time.perf_counter() - t0}), flush=True)
