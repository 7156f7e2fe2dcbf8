// oracle_capi.cpp — C ABI over the CPU restatement (dba_oracle.hpp).
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
// CPU legs of bench.py as the parity checker and the timed CPU baseline. The
// struct layouts mirror include/dbag.h so one ctypes definition serves both.
#include <cstdio>
#include <cstring>
#include <string>

#include "dba_oracle.hpp"

extern "C" {

typedef struct orc_problem {
  std::int32_t m, n;
  std::int64_t num_obs;
  const void* cameras;  // 9m Scalar
  const void* points;   // 3n Scalar
  const std::int32_t* cam_id;
  const std::int32_t* pt_id;
  const void* pixel_x;
  const void* pixel_y;
  const void* weight;
} orc_problem;

typedef struct orc_config {
  std::int32_t workers, max_iterations;
  double pcg_tol;
  std::int32_t pcg_max_iters, _pad0;
  double lambda0, lambda_max, rel_tol, step_tol;
  std::int32_t damping, mse_half, jacobian, check_rank_identity;
} orc_config;

typedef struct orc_result {
  std::int32_t iterations, termination;
  double cost, lambda, nu;
  std::int32_t capacity, workers;
  std::int32_t* rec_iteration;
  double* rec_cost;
  double* rec_mse;
  double* rec_lambda;
  std::int32_t* rec_pcg;
  std::int32_t* rec_accepted;
  double* rec_wall;
  std::uint64_t* rec_worker_edges;      // capacity x workers
  std::uint64_t* rec_worker_block_ops;  // capacity x workers
  void* x_c;                            // 9m Scalar (out)
  void* x_p;                            // 3n Scalar (out)
} orc_result;
}

namespace {

thread_local std::string g_err;
thread_local std::int64_t g_err_a = -1;
thread_local int g_err_b = 0;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return orc::kOk;
  } catch (const orc::OracleError& e) {
    g_err = e.what();
    g_err_a = e.a;
    g_err_b = e.b;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return orc::kInternal;
  }
}

template <class S>
orc::Problem<S> load(const orc_problem* p) {
  orc::Problem<S> pb;
  pb.m = p->m;
  pb.n = p->n;
  const S* c = static_cast<const S*>(p->cameras);
  const S* x = static_cast<const S*>(p->points);
  pb.cams.assign(c, c + std::size_t(p->m) * 9);
  pb.pts.assign(x, x + std::size_t(p->n) * 3);
  pb.cam_id.assign(p->cam_id, p->cam_id + p->num_obs);
  pb.pt_id.assign(p->pt_id, p->pt_id + p->num_obs);
  const S* px = static_cast<const S*>(p->pixel_x);
  const S* py = static_cast<const S*>(p->pixel_y);
  pb.px.assign(px, px + p->num_obs);
  pb.py.assign(py, py + p->num_obs);
  if (p->weight) {
    const S* w = static_cast<const S*>(p->weight);
    pb.weight.assign(w, w + p->num_obs);
  } else {
    pb.weight.assign(std::size_t(p->num_obs), S(1));
  }
  return pb;
}

orc::Config to_cfg(const orc_config* c) {
  orc::Config k;
  k.workers = c->workers;
  k.max_iterations = c->max_iterations;
  k.pcg_tol = c->pcg_tol;
  k.pcg_max_iters = c->pcg_max_iters;
  k.lambda0 = c->lambda0;
  k.lambda_max = c->lambda_max;
  k.rel_tol = c->rel_tol;
  k.step_tol = c->step_tol;
  k.damping = c->damping ? orc::Damping::diag_scaled : orc::Damping::identity;
  k.mse_half = c->mse_half;
  k.jacobian = c->jacobian ? orc::JacMode::analytic : orc::JacMode::autodiff;
  k.check_rank_identity = c->check_rank_identity != 0;
  return k;
}

// Builds every rank's (allreduced, damped, factored) system exactly as
// tests/test_solver.cpp:46-68 does, then runs fn(rank, group, hessian, Bd, Binv, Cinv).
template <class S, class Fn>
void with_system(const orc::Problem<S>& pb, int k, double lambda, int policy, Fn&& fn) {
  const auto parts = orc::partition_edges(pb, k);
  orc::Group g(k);
  orc::run_on_workers(g, [&](int r) {
    orc::Evaluator<S> ev(pb, parts[std::size_t(r)], orc::JacMode::autodiff);
    orc::Hessian<S> h(pb, parts[std::size_t(r)]);
    orc::assemble(ev.linearize(pb.cams.data(), pb.pts.data(), nullptr), ev, h);
    g.allreduce_sum(r, h.B.a.data(), h.B.a.size());
    g.allreduce_sum(r, h.C.a.data(), h.C.a.size());
    g.allreduce_sum(r, h.v.data(), h.v.size());
    g.allreduce_sum(r, h.w.data(), h.w.size());
    const auto pol = policy ? orc::Damping::diag_scaled : orc::Damping::identity;
    orc::BlockDiag<S, 9> Bd;
    orc::BlockDiag<S, 3> Cd;
    h.B.damp_into(static_cast<S>(lambda), pol, Bd);
    h.C.damp_into(static_cast<S>(lambda), pol, Cd);
    orc::Factored<S, 9> Bf;
    orc::Factored<S, 3> Cf;
    Bf.factor(Bd);
    Cf.factor(Cd);
    fn(r, g, h, Bd, Bf, Cf);
  });
}

template <class S>
int lm(const orc_problem* p, const orc_config* c, orc_result* out) {
  return guarded([&] {
    const auto pb = load<S>(p);
    const auto cfg = to_cfg(c);
    const auto st = orc::lm_solve(pb, cfg);
    out->iterations = st.iteration;
    out->termination = st.termination;
    out->cost = st.cost;
    out->lambda = st.lambda;
    out->nu = st.nu;
    out->workers = cfg.workers;
    const int n = std::min<int>(out->capacity, int(st.history.size()));
    for (int i = 0; i < n; ++i) {
      const auto& r = st.history[std::size_t(i)];
      if (out->rec_iteration) out->rec_iteration[i] = r.iteration;
      if (out->rec_cost) out->rec_cost[i] = r.cost;
      if (out->rec_mse) out->rec_mse[i] = r.mse;
      if (out->rec_lambda) out->rec_lambda[i] = r.lambda;
      if (out->rec_pcg) out->rec_pcg[i] = r.pcg_iterations;
      if (out->rec_accepted) out->rec_accepted[i] = r.accepted ? 1 : 0;
      if (out->rec_wall) out->rec_wall[i] = r.wall_seconds;
      for (int k = 0; k < cfg.workers; ++k) {
        if (out->rec_worker_edges) out->rec_worker_edges[std::size_t(i) * cfg.workers + k] = r.worker_edges[std::size_t(k)];
        if (out->rec_worker_block_ops)
          out->rec_worker_block_ops[std::size_t(i) * cfg.workers + k] = r.worker_block_ops[std::size_t(k)];
      }
    }
    if (out->x_c) std::memcpy(out->x_c, st.x_c.data(), st.x_c.size() * sizeof(S));
    if (out->x_p) std::memcpy(out->x_p, st.x_p.data(), st.x_p.size() * sizeof(S));
  });
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
std::int64_t orc_last_error_index(void) { return g_err_a; }
int orc_last_error_block_size(void) { return g_err_b; }

// residual of one edge; dba/problem.hpp:151-165
int orc_residual(int prec, const void* cam, const void* pt, const void* pix, void* out) {
  return guarded([&] {
    bool ok;
    if (prec == 8) {
      const double* q = static_cast<const double*>(pix);
      ok = orc::residual(static_cast<const double*>(cam), static_cast<const double*>(pt), q[0], q[1],
                         static_cast<double*>(out));
    } else {
      const float* q = static_cast<const float*>(pix);
      ok = orc::residual(static_cast<const float*>(cam), static_cast<const float*>(pt), q[0], q[1],
                         static_cast<float*>(out));
    }
    if (!ok) throw orc::DegenerateDepth(-1);
  });
}

int orc_rotate(int prec, const void* aa, const void* x, void* out) {
  return guarded([&] {
    if (prec == 8) orc::rotate(static_cast<const double*>(aa), static_cast<const double*>(x), static_cast<double*>(out));
    else orc::rotate(static_cast<const float*>(aa), static_cast<const float*>(x), static_cast<float*>(out));
  });
}

// dba/problem.hpp:266-283
int orc_total_cost(int prec, const orc_problem* p, double* cost) {
  return guarded([&] {
    if (prec == 8) *cost = orc::total_cost(load<double>(p));
    else *cost = orc::total_cost(load<float>(p));
  });
}

// Elementwise jet kernel on fp64 batches (KATs of tests/test_jet.cpp:24-109).
// op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt(a), 5 neg(a), 6 add_scalar(a, s).
int orc_jet_op(int op, std::int64_t n, int da, const double* av, const double* ag, int db, const double* bv,
               const double* bg, double s, int* dout, double* ov, double* og) {
  return guarded([&] {
    orc::Jets<double> a, b, o;
    a.shape(n, da);
    std::memcpy(a.v.data(), av, sizeof(double) * std::size_t(n));
    if (da) std::memcpy(a.g.data(), ag, sizeof(double) * std::size_t(n) * da);
    b.shape(n, db);
    if (bv) std::memcpy(b.v.data(), bv, sizeof(double) * std::size_t(n));
    if (db) std::memcpy(b.g.data(), bg, sizeof(double) * std::size_t(n) * db);
    switch (op) {
      case 0: orc::jet::add(a, b, o); break;
      case 1: orc::jet::sub(a, b, o); break;
      case 2: orc::jet::mul(a, b, o); break;
      case 3: orc::jet::div(a, b, o); break;
      case 4: orc::jet::sqrt(a, o); break;
      case 5: orc::jet::neg(a, o); break;
      case 6: orc::jet::add_scalar(a, s, o); break;
      default: throw orc::OracleError(orc::kInvalidArgument, "unknown jet op");
    }
    *dout = o.d;
    std::memcpy(ov, o.v.data(), sizeof(double) * std::size_t(n));
    std::memcpy(og, o.g.data(), sizeof(double) * std::size_t(n) * o.d);
  });
}

// Rodrigues on seeded jets (tests/test_jet.cpp:112-171): aa seeded on lanes
// 0..2, x on 3..5; out values (3) and gradients (3 x 6, row-major).
int orc_rotate_jets(const double* aa, const double* x, double* out, double* grad) {
  return guarded([&] {
    std::array<orc::Jets<double>, 3> A, X, O;
    for (int i = 0; i < 3; ++i) {
      A[i].shape(1, 6); X[i].shape(1, 6);
      std::fill(A[i].g.begin(), A[i].g.end(), 0.0);
      std::fill(X[i].g.begin(), X[i].g.end(), 0.0);
      A[i].v[0] = aa[i]; A[i].lane(i)[0] = 1.0;
      X[i].v[0] = x[i]; X[i].lane(3 + i)[0] = 1.0;
    }
    orc::JetPool<double> pool;
    orc::rotate_jets<double>({&A[0], &A[1], &A[2]}, {&X[0], &X[1], &X[2]}, {&O[0], &O[1], &O[2]}, pool);
    for (int i = 0; i < 3; ++i) {
      out[i] = O[i].v[0];
      for (int j = 0; j < 6; ++j) grad[i * 6 + j] = O[i].lane(j)[0];
    }
  });
}

// dba/partition.hpp:76-103 + dba/block_matrix.hpp:185-204,309-320 for one rank.
// Output buffers sized by the caller: cam_g[m], pt_g[n], cam_ptr[m+1],
// cam_blk[count], pt_ptr[n+1], pt_blk[count].
int orc_partition(const orc_problem* p, int k, int rank, std::int64_t* start, std::int64_t* count, int* n_cams,
                  std::int32_t* cam_g, int* n_pts, std::int32_t* pt_g, std::int64_t* cam_ptr, std::int64_t* cam_blk,
                  std::int64_t* pt_ptr, std::int64_t* pt_blk) {
  return guarded([&] {
    orc::Problem<double> pb;  // ids only
    pb.m = p->m;
    pb.n = p->n;
    pb.cam_id.assign(p->cam_id, p->cam_id + p->num_obs);
    pb.pt_id.assign(p->pt_id, p->pt_id + p->num_obs);
    const auto parts = orc::partition_edges(pb, k);
    if (rank < 0 || rank >= k) throw orc::OracleError(orc::kInvalidArgument, "rank out of range");
    const auto& part = parts[std::size_t(rank)];
    *start = part.start;
    *count = part.count;
    *n_cams = part.cams.size();
    *n_pts = part.pts.size();
    std::copy(part.cams.to_global.begin(), part.cams.to_global.end(), cam_g);
    std::copy(part.pts.to_global.begin(), part.pts.to_global.end(), pt_g);
    orc::EdgeBlocks<double> E(pb, part);
    std::copy(E.cam_ptr.begin(), E.cam_ptr.end(), cam_ptr);
    std::copy(E.cam_blk.begin(), E.cam_blk.end(), cam_blk);
    std::copy(E.pt_ptr.begin(), E.pt_ptr.end(), pt_ptr);
    std::copy(E.pt_blk.begin(), E.pt_blk.end(), pt_blk);
  });
}

// EdgeEvaluator::linearize for rank `rank` of K (dba/edge_eval.hpp:115-285).
// res: 2 x count (rx then ry); jac: 2 x 12 x count (row, lane, edge).
int orc_linearize(int prec, const orc_problem* p, int k, int rank, int mode, void* res, void* jac,
                  std::int64_t* bad_edge) {
  auto run = [&](auto tag) {
    using S = decltype(tag);
    return guarded([&] {
      const auto pb = load<S>(p);
      const auto parts = orc::partition_edges(pb, k);
      orc::Evaluator<S> ev(pb, parts[std::size_t(rank)], mode ? orc::JacMode::analytic : orc::JacMode::autodiff);
      try {
        const auto& b = ev.linearize(pb.cams.data(), pb.pts.data(), nullptr);
        const std::int64_t n = b.size();
        S* r = static_cast<S*>(res);
        S* j = static_cast<S*>(jac);
        std::memcpy(r, b.rx.v.data(), sizeof(S) * n);
        std::memcpy(r + n, b.ry.v.data(), sizeof(S) * n);
        std::memcpy(j, b.rx.g.data(), sizeof(S) * n * 12);
        std::memcpy(j + n * 12, b.ry.g.data(), sizeof(S) * n * 12);
      } catch (const orc::DegenerateDepth& e) {
        if (bad_edge) *bad_edge = e.a;
        throw;
      }
    });
  };
  return prec == 8 ? run(double{}) : run(float{});
}

// Per-rank local Gauss-Newton assembly (dba/block_matrix.hpp:358-400), not
// all-reduced: B[81m], C[9n], E[27 count] (shard edge order), v[9m], w[3n].
int orc_assemble(int prec, const orc_problem* p, int k, int rank, int mode, void* B, void* C, void* E, void* v,
                 void* w) {
  auto run = [&](auto tag) {
    using S = decltype(tag);
    return guarded([&] {
      const auto pb = load<S>(p);
      const auto parts = orc::partition_edges(pb, k);
      orc::Evaluator<S> ev(pb, parts[std::size_t(rank)], mode ? orc::JacMode::analytic : orc::JacMode::autodiff);
      orc::Hessian<S> h(pb, parts[std::size_t(rank)]);
      orc::assemble(ev.linearize(pb.cams.data(), pb.pts.data(), nullptr), ev, h);
      std::memcpy(B, h.B.a.data(), sizeof(S) * h.B.a.size());
      std::memcpy(C, h.C.a.data(), sizeof(S) * h.C.a.size());
      std::memcpy(E, h.E.blocks.data(), sizeof(S) * h.E.blocks.size());
      std::memcpy(v, h.v.data(), sizeof(S) * h.v.size());
      std::memcpy(w, h.w.data(), sizeof(S) * h.w.size());
    });
  };
  return prec == 8 ? run(double{}) : run(float{});
}

// BlockDiagonal::damp_into (dba/block_matrix.hpp:86-99), fp64.
int orc_damp(int bs, std::int64_t nb, const double* in, double lambda, int policy, double* out) {
  return guarded([&] {
    const auto pol = policy ? orc::Damping::diag_scaled : orc::Damping::identity;
    if (bs == 3) {
      orc::BlockDiag<double, 3> d, o;
      d.resize(nb);
      std::copy(in, in + nb * 9, d.a.begin());
      d.damp_into(lambda, pol, o);
      std::copy(o.a.begin(), o.a.end(), out);
    } else {
      orc::BlockDiag<double, 9> d, o;
      d.resize(nb);
      std::copy(in, in + nb * 81, d.a.begin());
      d.damp_into(lambda, pol, o);
      std::copy(o.a.begin(), o.a.end(), out);
    }
  });
}

// FactoredBlockDiagonal::factor + solve_in_place (dba/block_matrix.hpp:118-167), fp64.
int orc_factor_solve(int bs, std::int64_t nb, const double* blocks, double* x) {
  return guarded([&] {
    if (bs == 3) {
      orc::BlockDiag<double, 3> d;
      d.resize(nb);
      std::copy(blocks, blocks + nb * 9, d.a.begin());
      orc::Factored<double, 3> f;
      f.factor(d);
      f.solve_in_place(x);
    } else {
      orc::BlockDiag<double, 9> d;
      d.resize(nb);
      std::copy(blocks, blocks + nb * 81, d.a.begin());
      orc::Factored<double, 9> f;
      f.factor(d);
      f.solve_in_place(x);
    }
  });
}

// DSE (dba/solver.hpp:149-181) on the partitioned, damped system of the
// problem's own linearization (tests/test_solver.cpp:46-68). out = rank 0's
// result; *rank_identical = all ranks bitwise equal.
int orc_dse(int prec, const orc_problem* p, int k, double lambda, int policy, const void* xv, void* outv,
            int* rank_identical) {
  auto run = [&](auto tag) {
    using S = decltype(tag);
    return guarded([&] {
      const auto pb = load<S>(p);
      const S* x = static_cast<const S*>(xv);
      std::vector<std::vector<S>> outs(static_cast<std::size_t>(k));
      with_system<S>(pb, k, lambda, policy, [&](int r, orc::Group& g, orc::Hessian<S>& h, orc::BlockDiag<S, 9>& Bd,
                                                orc::Factored<S, 9>&, orc::Factored<S, 3>& Cf) {
        outs[std::size_t(r)].resize(std::size_t(pb.m) * 9);
        orc::DseWs<S> ws;
        orc::dse(x, Bd, h.E, Cf, g, r, outs[std::size_t(r)].data(), ws, nullptr);
      });
      *rank_identical = 1;
      for (int r = 1; r < k; ++r)
        if (std::memcmp(outs[std::size_t(r)].data(), outs[0].data(), outs[0].size() * sizeof(S)) != 0)
          *rank_identical = 0;
      std::copy(outs[0].begin(), outs[0].end(), static_cast<S*>(outv));
    });
  };
  return prec == 8 ? run(double{}) : run(float{});
}

// DPCG (dba/solver.hpp:202-257) on the same system.
int orc_dpcg(int prec, const orc_problem* p, int k, double lambda, int policy, const void* rhsv, double tol,
             int max_iters, void* x_out, int* iterations, int* converged, int* rank_identical) {
  auto run = [&](auto tag) {
    using S = decltype(tag);
    return guarded([&] {
      const auto pb = load<S>(p);
      std::vector<std::vector<S>> xs(static_cast<std::size_t>(k));
      std::vector<orc::PcgResult> res(static_cast<std::size_t>(k));
      const S* rhs = static_cast<const S*>(rhsv);
      const std::vector<S> g(rhs, rhs + std::size_t(pb.m) * 9);
      with_system<S>(pb, k, lambda, policy, [&](int r, orc::Group& grp, orc::Hessian<S>& h,
                                                orc::BlockDiag<S, 9>& Bd, orc::Factored<S, 9>& Bf,
                                                orc::Factored<S, 3>& Cf) {
        auto& x = xs[std::size_t(r)];
        x.assign(std::size_t(pb.m) * 9, S(0));
        res[std::size_t(r)] = orc::dpcg(x, Bd, Bf, h.E, Cf, g, grp, r, tol, max_iters, nullptr);
      });
      *rank_identical = 1;
      for (int r = 1; r < k; ++r)
        if (std::memcmp(xs[std::size_t(r)].data(), xs[0].data(), xs[0].size() * sizeof(S)) != 0) *rank_identical = 0;
      std::copy(xs[0].begin(), xs[0].end(), static_cast<S*>(x_out));
      *iterations = res[0].iterations;
      *converged = res[0].converged ? 1 : 0;
    });
  };
  return prec == 8 ? run(double{}) : run(float{});
}

// DSE / DPCG on caller-fabricated blocks (tests/test_solver.cpp:75-105,
// 198-229, 272-333): B[81m], C[9n] (already damped), E_table[27 N] in global
// edge order; the problem supplies only the graph. mode 0: out = dse(x);
// mode 1: out = dpcg(rhs=x, tol, max_iters).
int orc_blocks_solve(const orc_problem* p, int k, const double* B, const double* C, const double* E_table, int mode,
                     const double* x, double tol, int max_iters, double* out, int* iterations, int* rank_identical) {
  return guarded([&] {
    orc::Problem<double> pb;
    pb.m = p->m;
    pb.n = p->n;
    pb.cam_id.assign(p->cam_id, p->cam_id + p->num_obs);
    pb.pt_id.assign(p->pt_id, p->pt_id + p->num_obs);
    const auto parts = orc::partition_edges(pb, k);
    orc::BlockDiag<double, 9> b;
    b.resize(pb.m);
    std::copy(B, B + std::size_t(pb.m) * 81, b.a.begin());
    orc::BlockDiag<double, 3> c;
    c.resize(pb.n);
    std::copy(C, C + std::size_t(pb.n) * 9, c.a.begin());
    orc::Factored<double, 9> bf;
    orc::Factored<double, 3> cf;
    cf.factor(c);
    if (mode == 1) bf.factor(b);
    std::vector<std::vector<double>> outs(static_cast<std::size_t>(k));
    std::vector<int> its(std::size_t(k), 0);
    orc::Group g(k);
    orc::run_on_workers(g, [&](int r) {
      const auto& part = parts[std::size_t(r)];
      orc::EdgeBlocks<double> e(pb, part);
      for (std::int64_t i = 0; i < part.count; ++i)
        std::copy(E_table + (part.start + i) * 27, E_table + (part.start + i + 1) * 27, e.blk(i));
      auto& o = outs[std::size_t(r)];
      o.assign(std::size_t(pb.m) * 9, 0.0);
      if (mode == 0) {
        orc::DseWs<double> ws;
        orc::dse(x, b, e, cf, g, r, o.data(), ws, nullptr);
      } else {
        const std::vector<double> rhs(x, x + std::size_t(pb.m) * 9);
        its[std::size_t(r)] = orc::dpcg(o, b, bf, e, cf, rhs, g, r, tol, max_iters, nullptr).iterations;
      }
    });
    *rank_identical = 1;
    for (int r = 1; r < k; ++r)
      if (std::memcmp(outs[std::size_t(r)].data(), outs[0].data(), outs[0].size() * 8) != 0) *rank_identical = 0;
    std::copy(outs[0].begin(), outs[0].end(), out);
    if (iterations) *iterations = its[0];
  });
}

// WorkerGroup::allreduce_sum with K threads (dba/comms.hpp:67-84): data is
// K x len (rank-major), reduced in place on every rank's row.
int orc_allreduce(int k, std::int64_t len, double* data) {
  return guarded([&] {
    orc::Group g(k);
    orc::run_on_workers(g, [&](int r) { g.allreduce_sum(r, data + std::size_t(r) * len, std::size_t(len)); });
  });
}

// dba::lm_solve (dba/solver.hpp:523-534) with K = config->workers threads.
int orc_lm_solve(int prec, const orc_problem* p, const orc_config* c, orc_result* out) {
  return prec == 8 ? lm<double>(p, c, out) : lm<float>(p, c, out);
}

// The bench step on the CPU (the reference arm / cpu_baseline): `steps`
// times, one LM iteration of lm_solve_rank (dba/solver.hpp:330-425) from x0
// at lambda0 — linearize + assemble + all-reduce B, C, v, w, damp, factor,
// rhs, dpcg, back-substitution, trial cost, model terms — with
// K = config->workers threads. phases[step * 7 + i] (max over ranks) holds
// the seconds of: 0 linearize + assemble + all-reduces, 1 damp + factor,
// 2 rhs, 3 dpcg head (norms, r = g - S x0 and the first kHead = 5 loop
// iterations), 4 the rest of the dpcg loop, 5 back-substitution + trial
// state, 6 trial cost + model terms. pcg_sample > 0 caps the DPCG at that
// many iterations (a bounded sample of the step: the bench scales phase 4 by
// the full step's remaining DSE count over dse_calls[step] - 1 - kHead);
// pcg_iters / dse_calls report what ran.
int orc_lm_probe_phases(int prec, const orc_problem* p, const orc_config* c, int steps, int pcg_sample,
                        double* phases, int* pcg_iters, int* dse_calls) {
  auto run = [&](auto tag) {
    using S = decltype(tag);
    return guarded([&] {
      const auto pb = load<S>(p);
      const auto cfg = to_cfg(c);
      const auto parts = orc::partition_edges(pb, cfg.workers);
      orc::Group g(cfg.workers);
      const int K = cfg.workers;
      std::vector<double> ph(std::size_t(steps) * K * 7, 0.0);
      std::vector<int> its(std::size_t(steps), 0), dses(std::size_t(steps), 0);
      orc::run_on_workers(g, [&](int r) {
        const auto& part = parts[std::size_t(r)];
        orc::Evaluator<S> ev(pb, part, cfg.jacobian);
        orc::Hessian<S> h(pb, part);
        orc::BlockDiag<S, 9> Bd;
        orc::BlockDiag<S, 3> Cd;
        orc::Factored<S, 9> Bf;
        orc::Factored<S, 3> Cf;
        const std::size_t cdim = std::size_t(pb.m) * 9, pdim = std::size_t(pb.n) * 3;
        std::vector<S> gvec(cdim), dxc, dxp(pdim), txc(cdim), txp(pdim), ptmp, ctmp(cdim);
        const double lambda = cfg.lambda0;
        const int cap = pcg_sample > 0 ? std::min(pcg_sample, cfg.pcg_max_iters) : cfg.pcg_max_iters;
        using clk = std::chrono::steady_clock;
        for (int s = 0; s < steps; ++s) {
          double* P = &ph[(std::size_t(s) * K + r) * 7];
          auto t = clk::now();
          auto lap = [&](int i) {
            const auto now = clk::now();
            P[i] += std::chrono::duration<double>(now - t).count();
            t = now;
          };
          const auto& bt = ev.linearize(pb.cams.data(), pb.pts.data(), nullptr);
          orc::assemble(bt, ev, h);
          g.allreduce_sum(r, h.B.a.data(), h.B.a.size());
          g.allreduce_sum(r, h.C.a.data(), h.C.a.size());
          g.allreduce_sum(r, h.v.data(), h.v.size());
          g.allreduce_sum(r, h.w.data(), h.w.size());
          lap(0);
          int pcg = 0, dse = 0;
          try {
            h.B.damp_into(static_cast<S>(lambda), cfg.damping, Bd);
            h.C.damp_into(static_cast<S>(lambda), cfg.damping, Cd);
            Cf.factor(Cd);
            Bf.factor(Bd);
            lap(1);
            ptmp = h.w;
            Cf.solve_in_place(ptmp.data());
            ctmp.assign(cdim, S(0));
            h.E.apply(ptmp.data(), ctmp.data(), nullptr);
            g.allreduce_sum(r, ctmp.data(), ctmp.size());
            for (std::size_t i = 0; i < cdim; ++i) gvec[i] = h.v[i] - ctmp[i];
            lap(2);
            dxc.assign(cdim, S(0));
            double setup = 0;
            constexpr int kHead = 5;
            pcg = orc::dpcg(dxc, Bd, Bf, h.E, Cf, gvec, g, r, cfg.pcg_tol, cap, nullptr, &dse, &setup, kHead)
                      .iterations;
            lap(4);
            P[3] += setup;
            P[4] -= setup;
            ptmp.assign(pdim, S(0));
            h.E.apply_t(dxc.data(), ptmp.data(), nullptr);
            g.allreduce_sum(r, ptmp.data(), ptmp.size());
            for (std::size_t i = 0; i < pdim; ++i) dxp[i] = h.w[i] - ptmp[i];
            Cf.solve_in_place(dxp.data());
            for (std::size_t i = 0; i < cdim; ++i) txc[i] = pb.cams[i] + dxc[i];
            for (std::size_t i = 0; i < pdim; ++i) txp[i] = pb.pts[i] + dxp[i];
            lap(5);
            orc::distributed_cost(ev, txc.data(), txp.data(), g, r, nullptr);
            double step_inf = 0, damp = 0;
            for (std::size_t i = 0; i < cdim; ++i) step_inf = std::max(step_inf, std::abs(double(dxc[i])));
            for (std::size_t i = 0; i < pdim; ++i) step_inf = std::max(step_inf, std::abs(double(dxp[i])));
            for (std::size_t i = 0; i < cdim; ++i)
              damp += lambda * double(orc::clamp_curv(h.B.diag(std::int64_t(i)))) * double(dxc[i]) * double(dxc[i]);
            for (std::size_t i = 0; i < pdim; ++i)
              damp += lambda * double(orc::clamp_curv(h.C.diag(std::int64_t(i)))) * double(dxp[i]) * double(dxp[i]);
            volatile double model = damp + orc::dot_d(dxc.data(), h.v.data(), cdim) +
                                    orc::dot_d(dxp.data(), h.w.data(), pdim) + step_inf;
            (void)model;
            lap(6);
          } catch (const orc::SingularBlock&) {
          } catch (const orc::PcgBreakdown&) {
          }
          if (r == 0) {
            its[std::size_t(s)] = pcg;
            dses[std::size_t(s)] = dse;
          }
        }
      });
      for (int s = 0; s < steps; ++s) {
        for (int i = 0; i < 7; ++i) {
          double mx = 0;
          for (int r = 0; r < K; ++r) mx = std::max(mx, ph[(std::size_t(s) * K + r) * 7 + i]);
          phases[std::size_t(s) * 7 + i] = mx;
        }
        if (pcg_iters) pcg_iters[s] = its[std::size_t(s)];
        if (dse_calls) dse_calls[s] = dses[std::size_t(s)];
      }
    });
  };
  return prec == 8 ? run(double{}) : run(float{});
}

// generate_synthetic (dba/synthetic.hpp:70-146) + the count-exact / pixel
// noise extension, with the reference's exhaustive nearest-camera scan run
// on `threads` host threads. Options struct layout = dbag_synthetic_options.
typedef struct orc_synth {
  std::int32_t cameras, points, obs_per_point, exhaustive_search;
  std::uint64_t seed;
  double circle_radius, base_focal, pose_noise, intrinsic_noise, point_noise;
  std::int64_t num_observations;
  double pixel_noise;
} orc_synth;

static orc::SynthOptions to_synth(const orc_synth* s) {
  orc::SynthOptions o;
  o.cameras = s->cameras;
  o.points = s->points;
  o.obs_per_point = s->obs_per_point;
  o.seed = s->seed;
  o.circle_radius = s->circle_radius;
  o.base_focal = s->base_focal;
  o.pose_noise = s->pose_noise;
  o.intrinsic_noise = s->intrinsic_noise;
  o.point_noise = s->point_noise;
  o.num_observations = s->num_observations;
  o.pixel_noise = s->pixel_noise;
  return o;
}

int orc_synthetic_count(const orc_synth* s, std::int64_t* n_obs) {
  return guarded([&] { *n_obs = orc::synth_count(to_synth(s)); });
}

int orc_generate_synthetic(const orc_synth* s, int threads, double* cams, double* pts, std::int32_t* cam_id,
                           std::int32_t* pt_id, double* px, double* py) {
  return guarded([&] {
    const orc::Synthetic g = orc::generate_synthetic(to_synth(s), threads);
    std::copy(g.cams.begin(), g.cams.end(), cams);
    std::copy(g.pts.begin(), g.pts.end(), pts);
    std::copy(g.cam_id.begin(), g.cam_id.end(), cam_id);
    std::copy(g.pt_id.begin(), g.pt_id.end(), pt_id);
    std::copy(g.px.begin(), g.px.end(), px);
    std::copy(g.py.begin(), g.py.end(), py);
  });
}

}  // extern "C"
