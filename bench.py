#!/usr/bin/env python
"""Bench: seconds per LM iteration and edges/sec (BASELINE.json `metric`).

A step is one LM iteration of the reference's inner loop
(dba/solver.hpp:330-425) on a synthetic BAL-shaped problem: linearize +
assemble (+ all-reduce), damp + factor, rhs, DPCG to pcg_tol / pcg_max_iters,
back-substitution, trial cost and model terms. Every step starts from the
same state x0 at lambda0 and the accept is not committed, so each step does
identical work (SURVEY.md §8d timing note). The headline workload is
Venice-1778 (BASELINE.json configs[2], the configuration the metric is quoted
"at 1/2/4/8 B200" on); a real 10-iteration solve's IterationRecord
wall-second deltas are reported beside it (BASELINE.md §3 t_LM).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload NAME]

N > 1: one process per GPU, NCCL between ranks. Under torchrun (the driver)
the ranks come from the environment; a bare `python bench.py --gpus N`
re-launches itself under torch.distributed.run with N processes.
`--impl reference` times the CPU restatement of the reference (oracle/; the
reference itself cannot be compiled here: Eigen/doctest/CLI11 are absent) on
the host's physical cores, K rank threads as dba/comms.hpp:214-234, on the
same workload. That process imports only oracle/ (its own generator, config
and ctypes structs), never the product package.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {  # (cameras, points, observations) — BASELINE.json configs
    "ladybug-49": (49, 7776, 31843),
    "trafalgar-257": (257, 65132, 225911),
    "venice-1778": (1778, 993923, 5001946),
    "final-13682": (13682, 4456117, 28987644),
    "city-50k": (50000, 20000000, 150000000),
}
DEFAULT_WORKLOAD = "venice-1778"  # configs[2]: the metric's "1/2/4/8 B200" configuration; fits one GPU
SECONDARY_WORKLOAD = "trafalgar-257"  # configs[1]: the FP32/FP64 1-B200 configuration
PCG_SAMPLE = 20  # PCG iterations per bounded CPU-reference sample step


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def synth_kwargs(name):
    """The BASELINE.md §3 instance: ring recipe, seed 1, count-exact, +-0.5 px noise."""
    m, n, N = WORKLOADS[name]
    return dict(cameras=m, points=n, num_observations=N, seed=1, pixel_noise=0.5)


def make_problem(name, dtype=np.float64):
    """The product's generator (windowed search; bit-identical to the oracle's
    exhaustive restatement of dba/synthetic.hpp, tests/test_generator.py)."""
    import paper_2112_01349_b200 as dba
    p = dba.generate_synthetic(dba.SyntheticOptions(**synth_kwargs(name)))
    return p if dtype == np.float64 else p.astype(dtype)


def make_oracle_problem(name, dtype=np.float64):
    """The same instance from the oracle's own generator (no product import)."""
    from oracle import oracle as O
    p = O.generate_synthetic(O.SynthOptions(**synth_kwargs(name)))
    return p if dtype == np.float64 else p.astype(dtype)


def host_info():
    """nproc / lscpu of this host: logical CPUs, physical cores, model."""
    info = {"nproc": os.cpu_count() or 1}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1"))
        info["physical_cores"] = int(kv.get("Core(s) per socket", "0")) * int(kv.get("Socket(s)", "1"))
    except Exception:
        pass
    if not info.get("physical_cores"):
        info["physical_cores"] = info["nproc"]
    return info


def dse_bytes(N, n, m, s):
    """Algorithmic bytes of one DSE (SURVEY.md §8d B_DSE): one pass over E plus
    one camera index per edge, C^-1 per point, B, x, out per camera."""
    return N * (27 * s + 4) + 9 * n * s + 108 * m * s


def dse_layout_bytes(N, n, m, s, t=None):
    """Compulsory bytes of one DSE pass over THIS layout: the factored
    coupling records (18 lanes of G = sqrt(w) Jc per edge, kernels.cuh
    kLanesFact, t bytes each) plus one camera index per edge, C^-1 per point,
    B, x, out and R per camera. The reference layout (dse_bytes) stores 27."""
    t = s if t is None else t
    return N * (18 * t + 4) + 9 * n * s + 117 * m * s


def lm_bytes(N, n, m, s, I, linearized=True):
    """Algorithmic bytes of one LM iteration (SURVEY.md §8d B_LM) with I PCG
    iterations and R = I // 50 residual refreshes; the leading 1 of B_PCG is
    the reference's DSE on x0 = 0, kept in the count."""
    b_lin = N * (3 * s + 8) + 3 * n * s + 9 * m * s + 27 * N * s + 90 * m * s + 12 * n * s
    b_fact = 162 * m * s + 18 * n * s
    b_rhs = N * (27 * s + 4) + 12 * n * s + 9 * m * s
    b_pcg = (1 + I + I // 50) * dse_bytes(N, n, m, s) + I * 153 * m * s
    b_back = N * (27 * s + 4) + 15 * n * s
    b_cost = N * (3 * s + 8) + 6 * n * s + 18 * m * s
    return (b_lin if linearized else 0) + b_fact + b_rhs + b_pcg + b_back + b_cost


def lm_roofline(N, n, m, s, I, world, peak, ms_step, prof, steps):
    """Whole-iteration roofline: B_LM / (K peak) against the
    measured t_LM, and the DSE edge throughput N (1 + I + R) / t_PCG."""
    b = lm_bytes(N, n, m, s, I)
    t_roof_ms = b / (world * peak * 1e9) * 1e3
    t_pcg_ms = prof["dse_ms"] / max(steps, 1)
    return {"bytes_per_step": b, "roofline_ms": t_roof_ms, "measured_ms": ms_step, "frac": t_roof_ms / ms_step,
            "pcg_ms_per_step": t_pcg_ms,
            "dse_edges_per_s": N * (1 + I + I // 50) / (t_pcg_ms / 1e3) if t_pcg_ms > 0 else None}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_threads():
    """K for the CPU reference: the host's physical core count (BASELINE.md
    §3), one rank thread each, as the reference's run_on_workers."""
    return max(1, host_info()["physical_cores"])


PCG_HEAD = 5  # DPCG iterations the oracle counts into its "dpcg head" phase


def scaled_lm_seconds(phases, dse_sample, dse_full):
    """One LM iteration's seconds from a bounded sample: every phase as
    measured (oracle.PHASES), the steady DPCG loop (phase 4: after the DSE on
    x0 and the first PCG_HEAD iterations) scaled from the sample's DSE count
    to the full iteration's — every loop DSE is the same work: one
    E^T x / C^-1 / E b round with its two all-reduces, dba/solver.hpp:149-181."""
    ph = np.asarray(phases, dtype=float)
    head = 1 + PCG_HEAD
    return float(ph.sum() - ph[4] + ph[4] * (dse_full - head) / max(int(dse_sample) - head, 1))


def cpu_reference_steps(p, k, n_steps, dse_full=None, calibrate=True):
    """Times the oracle's LM step on k rank threads. With calibrate, first one
    FULL LM iteration (unscaled, gives the full DSE count); then n_steps
    bounded samples (DPCG capped at PCG_SAMPLE iterations) scaled to the full
    iteration. Returns (per-step seconds, info)."""
    from oracle import oracle as O
    cfg = O.OracleConfig(workers=k)
    info = {"threads": k, "pcg_sample": PCG_SAMPLE}
    if calibrate:
        ph, its, dse = O.lm_probe_phases(p, cfg, 1)
        dse_full = int(dse[0])
        info.update(full_iteration_s=float(ph[0].sum()), full_pcg_iterations=int(its[0]),
                    full_phases_s=dict(zip(O.PHASES, map(float, ph[0]))))
    info["dse_per_full_iteration"] = int(dse_full)
    ph, its, dse = O.lm_probe_phases(p, cfg, n_steps, pcg_sample=PCG_SAMPLE)
    secs = [scaled_lm_seconds(ph[i], dse[i], dse_full) for i in range(n_steps)]
    info["sample_phases_s"] = dict(zip(O.PHASES, map(float, ph.mean(0))))
    info["sample_dse_calls"] = int(dse[-1])
    return secs, info


def run_reference(args):
    """The reference arm: the CPU restatement (oracle/) of the reference's
    solver on this host's physical cores. Imports oracle/ only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    m, n, N = WORKLOADS[args.workload]
    t_gen = time.perf_counter()
    p = make_oracle_problem(args.workload)
    t_gen = time.perf_counter() - t_gen
    host = host_info()
    k = cpu_threads()
    # warm-up: the first step is one FULL LM iteration (calibration: the full
    # DSE count and an unscaled t_LM); the rest are bounded samples.
    secs, info = cpu_reference_steps(p, k, args.warmup - 1 + args.steps if args.warmup >= 1 else args.steps)
    timed = secs[-args.steps:]
    t = float(np.mean(timed))
    value = N / t
    # K = 1: one bounded sample, scaled the same way
    secs1, info1 = cpu_reference_steps(p, 1, 1, dse_full=info["dse_per_full_iteration"], calibrate=False)
    sample = (f"{args.workload}: each step one LM iteration from x0 (oracle restatement, {k} rank threads), "
              f"DPCG capped at {PCG_SAMPLE} iterations and its time scaled to the full iteration's "
              f"{info['dse_per_full_iteration']} DSEs; warm-up step 1 ran the full iteration unscaled "
              f"({info['full_iteration_s']:.2f} s, {info['full_pcg_iterations']} PCG iterations)")
    print(json.dumps({
        "impl": "reference", "metric": "edges_per_sec_per_lm_iteration", "value": value, "unit": "edges/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, info["full_pcg_iterations"], max(args.gpus, 1)),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": k, "kind": "port", "sample": sample,
                         "host": host, "jacobian": "autodiff", "detail": info,
                         "k1": {"value": N / secs1[0], "unit": "edges/s", "cores": 1, "seconds": secs1[0],
                                "sample": f"one bounded sample at K = 1 (DPCG capped at {PCG_SAMPLE}, scaled)",
                                "detail": info1}},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "instance_generation_s": t_gen,
        "repo_libs_loaded": repo_libs_loaded(),
    }), flush=True)


def repo_libs_loaded():
    """In-tree shared objects mapped into this process (the reference arm
    must show oracle/ only)."""
    try:
        with open("/proc/self/maps") as f:
            return sorted({os.path.relpath(l.split()[-1], ROOT) for l in f
                           if l.rstrip().endswith(".so") and l.split()[-1].startswith(ROOT)})
    except Exception:
        return None


def workload_config(name, pcg):
    m, n, N = WORKLOADS[name]
    return {"workload": name, "cameras": m, "points": n, "observations": N, "pcg_iterations_per_step": int(pcg),
            "solver": "SolverConfig defaults (diag_scaled, lambda0 1e-4, pcg_tol 1e-6, pcg_max_iters 500)",
            "step": "one LM iteration from x0 (linearize+assemble, damp+factor, rhs, DPCG, backsub, trial cost)",
            "instance": "dba/synthetic.hpp ring, seed 1, count-exact, +-0.5 px noise (BASELINE.md §3)"}


def bench_config(name, pcg, world):
    """The `config` both arms print (identical for the same workload and N)."""
    return dict(workload_config(name, pcg), parallelism=f"edge-partitioned x{world}",
                l2="flushed (512 MiB write) between timed steps; the E stream exceeds L2 anyway at venice and above")


def flush_l2(buf):
    import torch
    buf.zero_()
    torch.cuda.synchronize()


def time_steps(ctx, cfg, steps, flush):
    """Per-step device time (CUDA events on the context's stream), L2 flushed
    between steps outside the timed window."""
    ms = []
    pcg = 0
    for _ in range(steps):
        if flush is not None:
            flush_l2(flush)
        ctx.synchronize()
        ctx.mark(0)
        _, pcg, _ = ctx.probe_step(cfg.lambda0, cfg)
        ctx.mark(1)
        ms.append(ctx.elapsed_ms())
    return ms, pcg


def dse_roofline(ctx, prof, b_dse, peak, steps, total_ms, world, b_layout=None):
    """Roofline of the dominant kernel, the DSE pass (B_DSE bytes
    per pass), timed inside the timed steps: CUDA events on the context's
    stream bracket every DPCG (one graph launch at K = 1), and the device time
    per DSE is that time over the DSE count — the pass plus its camera fold +
    PCG step and the launch gaps between them, so `achieved` is a lower bound
    on the pass kernel's own rate. standalone_pass_ms is the pass alone,
    launched back to back on the same state after the timed steps (ncu
    cannot profile kernel nodes of a graph with conditional nodes; the
    committed ncu captures are of these standalone launches)."""
    dse_per_step = prof["dse_launches"] / max(steps, 1)
    per = prof["dse_ms"] / max(prof["dse_launches"], 1)
    kernel = "k_g_pass DSE iteration of the graph DPCG (pass + camera fold / PCG step), per pass, in the timed steps"
    standalone = None
    if world == 1:
        try:
            standalone = ctx.time_dse_pass(20)
        except Exception:  # DBAG_PCG selected a non-graph DPCG
            kernel = "DPCG (DBAG_PCG=%s), device time per DSE" % os.environ.get("DBAG_PCG")
    else:
        kernel = "k_g_pass DSE iteration of the per-rank DPCG graph (pass, peer collectives, fold / step), per pass"
    achieved = b_dse / (per / 1e3) / 1e9
    lay = {} if b_layout is None else {
        "layout_bytes_per_launch": b_layout, "layout_achieved": b_layout / (per / 1e3) / 1e9,
        "layout_frac": b_layout / (per / 1e3) / 1e9 / peak}
    out = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": None, "bytes_per_launch": b_dse, "avg_launch_ms": per, **lay,
           "launches_per_step": dse_per_step,
           "share_of_step": per * dse_per_step / max(total_ms / max(steps, 1), 1e-9),
           "note": "achieved = algorithmic DSE bytes per pass (SURVEY 8d: 27 scalars of E per edge, the "
                   "reference's layout) / in-step device ms per DSE; layout_* = the same against the compulsory "
                   "bytes of the factored records this build streams (18 scalars per edge); traffic = ncu DRAM "
                   "bytes of one standalone pass launch (profiles/ncu_traffic.json)"}
    if standalone is not None:
        out["standalone_pass_ms"] = standalone
        out["standalone_achieved"] = b_dse / (standalone / 1e3) / 1e9
        out["standalone_frac"] = out["standalone_achieved"] / peak
        if b_layout is not None:
            out["standalone_layout_frac"] = b_layout / (standalone / 1e3) / 1e9 / peak
    return out


def solve_t_lm(p, world, rank, uid, device, iters=10):
    """BASELINE.md §3 t_LM: a real lm_solve (SolverConfig defaults,
    max_iterations 10), per-iteration seconds = consecutive
    IterationRecord.wall_seconds deltas (rejects, which do not relinearize,
    included). Iteration 1's figure also holds the initial cost."""
    import paper_2112_01349_b200 as dba
    cfg = dba.SolverConfig(workers=world, max_iterations=iters)
    if world == 1:
        st = dba.lm_solve(p, cfg, devices=[device])
    else:
        st = dba.lm_solve_rank(p, cfg, rank, world, uid, device)
    wall = [r.wall_seconds for r in st.history]
    dt = [wall[0]] + [b - a for a, b in zip(wall, wall[1:])]
    N = p.num_observations
    return {"iterations": len(dt), "t_lm_s": dt, "mean_t_lm_s": float(np.mean(dt)),
            "edges_per_s": N / float(np.mean(dt)), "pcg_iterations": [r.pcg_iterations for r in st.history],
            "accepted": [r.accepted for r in st.history], "cost": [r.cost for r in st.history],
            "termination": st.termination, "note": "host wall clock of the one-shot dbag_lm_solve (upload excluded)"}


def run_ours(args):
    import torch
    import paper_2112_01349_b200 as dba
    world, rank, local = dist_env()
    dist = None
    ndev = max(dba.device_count(), 1)
    device = local % ndev
    uid = uid_solve = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        # one ncclUniqueId per communicator: the bench context's and the
        # t_LM solve's (an id is spent by its communicator's bootstrap)
        uids = [(dba.nccl_unique_id(), dba.nccl_unique_id()) if rank == 0 else None]
        dist.broadcast_object_list(uids, src=0)
        uid, uid_solve = uids[0]
        ctx = dba.RankContext(device, 8, nccl=(rank, world, uid))
        print(f"[bench] rank {rank}/{world}: NCCL communicator up on cuda:{device}", file=sys.stderr, flush=True)
    else:
        ctx = dba.RankContext(device, 8)
    torch.cuda.set_device(device)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")
    m, n, N = WORKLOADS[args.workload]
    p = make_problem(args.workload)
    ctx.upload(p)
    cfg = dba.SolverConfig(workers=world)
    for _ in range(args.warmup):
        ctx.probe_step(cfg.lambda0, cfg)
    if dist:
        dist.barrier()
    ctx.synchronize()
    l0 = ctx.launch_count()
    ctx.profile(True)
    with ClockSampler(device) as clk:
        ms, pcg = time_steps(ctx, cfg, args.steps, flush)
    prof = ctx.profile()
    ctx.profile(False)
    launches = ctx.launch_count() - l0
    total_ms = float(sum(ms))
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    ms_step = total_ms / args.steps
    value = N / (ms_step / 1e3)

    # e2e through the public API with host buffers: per step the state goes
    # host -> device, one LM iteration runs, the trial state comes back.
    x_c, x_p = p.pack_cameras(), p.pack_points()
    hc = torch.from_numpy(x_c).pin_memory().numpy()
    hp = torch.from_numpy(x_p).pin_memory().numpy()
    oc = torch.empty(hc.size, dtype=torch.float64).pin_memory().numpy()
    op = torch.empty(hp.size, dtype=torch.float64).pin_memory().numpy()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.set_state(hc, hp)
        ctx.probe_step(cfg.lambda0, cfg)
        ctx.get_state(out=(oc, op))
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    state_bytes = 8 * (9 * m + 3 * n)

    peak, peak_kind = load_peaks()
    b_dse = dse_bytes(N // world, n, m, 8)
    roof = dse_roofline(ctx, prof, b_dse, peak, args.steps, total_ms, world, dse_layout_bytes(N // world, n, m, 8))
    roof["peak_kind"] = peak_kind
    roof["traffic"], roof["traffic_source"] = ncu_traffic(args.workload)
    ctx.close()
    line = {
        "metric": "edges_per_sec_per_lm_iteration", "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, pcg, world),
        "roofline": roof,
        "e2e": {"value": N / e2e_s, "unit": "edges/s", "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "lm_roofline": lm_roofline(N, n, m, 8, pcg, world, peak, ms_step, prof, args.steps),
    }
    if not args.no_solve:
        line["solve"] = solve_t_lm(p, world, rank, uid_solve if world > 1 else None, device)
    if world == 1 and rank == 0 and not args.no_secondary:
        line["secondary"] = secondary(flush, SECONDARY_WORKLOAD)
        line["secondary_fp32"] = secondary(flush, SECONDARY_WORKLOAD, np.float32)
        line["fp32"] = secondary(flush, args.workload, np.float32)
        # memory-lean variant
        line["coupling_fp32"] = secondary(flush, args.workload, coupling_fp32=True)
    if world == 1 and rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, p, pcg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def ncu_traffic(name, dtype="f64"):
    """dram__bytes_read + write per launch of the dominant kernel from the
    committed `ncu --set full` capture (the recipe's source for `traffic`)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(name if dtype == "f64" else f"{name}/{dtype}", {})
        return e.get("dram_bytes_per_launch"), e.get("source")
    except Exception:
        return None, None


def secondary(flush, name, dtype=np.float64, coupling_fp32=False):
    """The same step on another configuration / precision: Trafalgar-257
    (BASELINE.json configs[1], FP32/FP64), FP32, or the memory-lean variant."""
    import paper_2112_01349_b200 as dba
    m, n, N = WORKLOADS[name]
    s = np.dtype(dtype).itemsize
    p = make_problem(name, dtype)
    with dba.RankContext(0, s, coupling_fp32=coupling_fp32) as ctx:
        ctx.upload(p)
        cfg = dba.SolverConfig()
        for _ in range(3):
            ctx.probe_step(cfg.lambda0, cfg)
        ctx.profile(True)
        ms, pcg = time_steps(ctx, cfg, 5, flush)
        prof = ctx.profile()
        t = sum(ms) / len(ms)
        peak, _ = load_peaks()
        b_dse = dse_bytes(N, n, m, s)
        b_lay = dse_layout_bytes(N, n, m, s)
        if coupling_fp32:  # E lanes at 4 bytes, everything else FP64
            b_dse = N * (27 * 4 + 4) + 9 * n * 8 + 108 * m * 8
            b_lay = dse_layout_bytes(N, n, m, 8, 4)
        roof = dse_roofline(ctx, prof, b_dse, peak, len(ms), sum(ms), 1, b_lay)
    tag = "f64" if s == 8 and not coupling_fp32 else ("f64e32" if coupling_fp32 else "f32")
    roof["traffic"], roof["traffic_source"] = ncu_traffic(name, tag)
    return {"workload": name, "dtype": ("f64 (E blocks stored f32)" if coupling_fp32 else "f64") if s == 8 else "f32",
            "ms_per_step": t, "value": N / (t / 1e3),
            "unit": "edges/s", "pcg_iterations_per_step": pcg, "roofline": roof}


def cpu_baseline(args, p, pcg):
    """The CPU restatement on this host's physical cores: one bounded sample
    of the step (DPCG capped at PCG_SAMPLE iterations, scaled to the GPU
    step's 1 + I + I//50 DSEs; the same iteration count both sides)."""
    k = cpu_threads()
    dse_full = 1 + pcg + pcg // 50
    secs, info = cpu_reference_steps(p, k, 1, dse_full=dse_full, calibrate=False)
    N = WORKLOADS[args.workload][2]
    return {"value": N / secs[0], "unit": "edges/s", "cores": k, "kind": "port", "host": host_info(),
            "sample": f"1 LM-iteration step of {args.workload}, {k} rank threads, DPCG capped at {PCG_SAMPLE} "
                      f"iterations and scaled to {dse_full} DSEs", "seconds": secs[0], "detail": info}


def dry_run(args):
    """Launcher check without a GPU: every rank joins a gloo group and rank 0
    reports how many ranks reached it."""
    world, rank, _ = dist_env()
    n = 1
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        n = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": args.gpus, "world_size": world, "ranks_reached": n}), flush=True)


def relaunch(args):
    """`python bench.py --gpus N` without torchrun: re-run this script under
    torch.distributed.run with N processes (one per GPU), as the driver does."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher check only (no GPU work)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
