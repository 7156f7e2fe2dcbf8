// solver.cuh — the host LM loop over one rank context.
//
// Decision-for-decision restatement of lm_solve_rank (dba/solver.hpp:295-518)
// and check_convergence (:91-104): reject-reuse of the assembled system,
// diag-scaled or identity damping, gain ratio with the model decrease
// damping_term + dx_c.v + dx_p.w, Nielsen's lambda schedule, singular blocks
// and PCG breakdowns as rejects, the IterationRecord history with per-worker
// tallies all-reduced across ranks, and the optional rank-identity probe.
// Every scalar the decisions read is rank-identical (replicated camera space,
// all-reduced point-space terms), so all ranks take the same branch.
#pragma once

#include <chrono>
#include <cmath>
#include <limits>
#include <vector>

#include "rank.cuh"

namespace dbag {

struct Record {  // IterationRecord, dba/solver.hpp:57-68
  int iteration = 0;
  double cost = 0, mse = 0, lambda = 0;
  int pcg_iterations = 0;
  bool accepted = false;
  double wall_seconds = 0;
  std::vector<std::uint64_t> worker_edges, worker_block_ops;
};

struct Outcome {  // SolverState minus the parameter vectors
  double lambda = 0, nu = 2, cost = 0;
  int iteration = 0;
  int termination = 1;  // 0 converged, 1 max_iterations, 2 stalled
  std::vector<Record> history;
  bool last_accepted = false;
  double last_cost_change = std::numeric_limits<double>::infinity();
  double last_step_inf = std::numeric_limits<double>::infinity();
  double previous_cost = std::numeric_limits<double>::infinity();
};

inline double mse_from_cost(double cost, std::int64_t nobs, int half) {
  if (nobs <= 0) return 0.0;
  return cost / (half ? 2.0 * double(nobs) : double(nobs));
}

// dba/solver.hpp:91-104: 0 keep going, 1 converged, 2 max_iterations, 3 stalled
inline int check_convergence(const Outcome& s, const dbag_config& c) {
  if (s.last_accepted) {
    const double denom = std::max(s.previous_cost, 1e-300);
    if (std::abs(s.last_cost_change) / denom < c.rel_tol || s.last_step_inf < c.step_tol) return 1;
  }
  if (s.lambda > c.lambda_max) return 3;
  if (s.iteration >= c.max_iterations) return 2;
  return 0;
}

// Result of one trial (dba/solver.hpp:342-430).
struct Trial {
  bool accepted = false, factorization_ok = true;
  double cost_new = std::numeric_limits<double>::infinity();
  double step_inf = 0;
  int pcg_iterations = 0;
  double shrink = 1.0;  // lambda factor on accept
};

template <class R>
Trial run_trial(R& rk, const dbag_config& c, double lambda, double cost) {
  Trial t;
  try {
    rk.damp_factor(lambda, c.damping);
    rk.rhs();
    const PcgOut pcg = rk.pcg(c.pcg_tol, c.pcg_max_iters);
    t.pcg_iterations = pcg.iterations;
    rk.backsub_trial();
    std::int64_t bad = -1;
    t.cost_new = rk.cost(true, &bad);
    double step_inf, damp, gv;
    rk.model_terms(&step_inf, &damp, &gv);
    t.step_inf = step_inf;
    const double model = damp + gv;
    if (model <= 0) {
      t.accepted = step_inf < c.step_tol && t.cost_new <= cost;
      if (t.accepted) t.cost_new = std::min(t.cost_new, cost);
    } else {
      const double rho = (cost - t.cost_new) / model;
      t.accepted = std::isfinite(t.cost_new) && rho > 0;
      if (t.accepted) t.shrink = std::max(1.0 / 3.0, 1.0 - std::pow(2.0 * rho - 1.0, 3.0));
    }
  } catch (const Error& e) {
    if (e.code != DBAG_SINGULAR_BLOCK && e.code != DBAG_PCG_BREAKDOWN) throw;
    t.factorization_ok = false;
    t.accepted = false;
  }
  return t;
}

template <class R>
Outcome lm_solve_rank(R& rk, const dbag_config& c, std::int64_t num_obs) {
  const auto t0 = std::chrono::steady_clock::now();
  const int K = rk.plan().ranks, me = rk.plan().rank;
  Outcome st;
  st.lambda = c.lambda0;
  st.nu = 2.0;
  std::int64_t bad = -1;
  st.cost = rk.cost(false, &bad);
  if (!std::isfinite(st.cost)) throw degenerate_depth(bad);
  bool have_system = false;
  for (;;) {
    const Tally start = rk.tally();
    if (!have_system) {
      rk.linearize();
      have_system = true;
    }
    const double lambda = st.lambda;
    const Trial t = run_trial(rk, c, lambda, st.cost);
    double cost_new = t.cost_new;
    if (t.accepted) {
      st.lambda *= t.shrink;
      st.nu = 2.0;
    }
    st.previous_cost = st.cost;
    if (t.accepted) {
      rk.accept();
      st.last_cost_change = st.cost - cost_new;
      st.cost = cost_new;
      st.last_step_inf = t.step_inf;
      have_system = false;
    } else {
      st.lambda *= st.nu;
      st.nu *= 2.0;
      st.last_cost_change = std::numeric_limits<double>::infinity();
      st.last_step_inf = std::numeric_limits<double>::infinity();
    }
    st.last_accepted = t.accepted;
    ++st.iteration;
    Record rec;
    rec.iteration = st.iteration;
    rec.cost = st.cost;
    rec.mse = mse_from_cost(st.cost, num_obs, c.mse_half);
    rec.lambda = lambda;
    rec.pcg_iterations = t.factorization_ok ? t.pcg_iterations : 0;
    rec.accepted = t.accepted;
    rec.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<double> tal(static_cast<std::size_t>(2 * K), 0.0);
    tal[static_cast<std::size_t>(2 * me)] = double(rk.tally().edges - start.edges);
    tal[static_cast<std::size_t>(2 * me + 1)] = double(rk.tally().block_ops - start.block_ops);
    rk.allreduce_host(tal.data(), 2 * K);
    rec.worker_edges.resize(static_cast<std::size_t>(K));
    rec.worker_block_ops.resize(static_cast<std::size_t>(K));
    for (int r = 0; r < K; ++r) {
      rec.worker_edges[static_cast<std::size_t>(r)] = static_cast<std::uint64_t>(tal[static_cast<std::size_t>(2 * r)]);
      rec.worker_block_ops[static_cast<std::size_t>(r)] =
          static_cast<std::uint64_t>(tal[static_cast<std::size_t>(2 * r + 1)]);
    }
    st.history.push_back(rec);
    if (c.check_rank_identity) {  // dba/solver.hpp:479-501
      double ic, ip;
      rk.state_inf(&ic, &ip);
      std::vector<double> probe(static_cast<std::size_t>(4 * K), 0.0);
      const std::size_t self = static_cast<std::size_t>(4 * me);
      probe[self] = st.cost;
      probe[self + 1] = st.lambda;
      probe[self + 2] = ic;
      probe[self + 3] = ip;
      rk.allreduce_host(probe.data(), 4 * K);
      for (int r = 0; r < K; ++r) {
        const std::size_t o = static_cast<std::size_t>(4 * r);
        if (probe[o] != st.cost || probe[o + 1] != st.lambda || probe[o + 2] != ic || probe[o + 3] != ip)
          throw Error(DBAG_INTERNAL, "rank divergence detected at iteration " + std::to_string(st.iteration) +
                                         " between ranks " + std::to_string(me) + " and " + std::to_string(r));
      }
    }
    const int dec = check_convergence(st, c);
    if (dec == 1) { st.termination = 0; break; }
    if (dec == 3) { st.termination = 2; break; }
    if (dec == 2) { st.termination = 1; break; }
  }
  return st;
}

// One LM iteration from the current state (relinearized) without committing
// it: the bench "step" (identical work every call).
template <class R>
Trial probe_step(R& rk, const dbag_config& c, double lambda) {
  std::int64_t bad = -1;
  const double cost = rk.cost(false, &bad);
  if (!std::isfinite(cost)) throw degenerate_depth(bad);
  rk.linearize();
  return run_trial(rk, c, lambda, cost);
}

}  // namespace dbag
