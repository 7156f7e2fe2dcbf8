// The operator level of the C++ drop-in (include/dba/dba_b200_ops.hpp) driven
// the way the reference's own suite drives dba:: — ports of
// tests/test_solver.cpp:74-270 (dse / dpcg against dense oracles across K,
// rank-identical bitwise), tests/test_linear.cpp:270-298 (singular block
// index, damping) and tests/test_comms.cpp:20-60 (all-reduce), plus the
// evaluator / assembly / lm_solve_rank path. Needs a GPU (every operator runs
// on the device); `compile` only checks that the header instantiates and
// runs the host-only port (check_convergence, tests/test_solver.cpp:457-486).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "dba/dba_b200.hpp"

using namespace dba;

#define CHECK(x)                                                          \
  do {                                                                    \
    if (!(x)) {                                                           \
      std::fprintf(stderr, "CHECK failed: %s line %d\n", #x, __LINE__);   \
      std::exit(1);                                                       \
    }                                                                     \
  } while (0)

namespace {

using Vec = std::vector<double>;
using Mat = std::vector<double>;  // dense row-major, test-side checker only

double norm(const Vec& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
Vec sub(const Vec& a, const Vec& b) {
  Vec c(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) c[i] = a[i] - b[i];
  return c;
}
double dot(const Vec& a, const Vec& b) {
  double s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// dense Cholesky solve of SPD A (n x n) for the columns of B (n x k), in place
void chol_solve(Mat A, int n, Mat& B, int k) {
  for (int j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int p = 0; p < j; ++p) d -= A[j * n + p] * A[j * n + p];
    d = std::sqrt(d);
    A[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A[i * n + j];
      for (int p = 0; p < j; ++p) s -= A[i * n + p] * A[j * n + p];
      A[i * n + j] = s / d;
    }
  }
  for (int c = 0; c < k; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = B[i * k + c];
      for (int p = 0; p < i; ++p) s -= A[i * n + p] * B[p * k + c];
      B[i * k + c] = s / A[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = B[i * k + c];
      for (int p = i + 1; p < n; ++p) s -= A[p * n + i] * B[p * k + c];
      B[i * k + c] = s / A[i * n + i];
    }
  }
}

// tests/oracles.hpp:147-236 ProblemFactory: cameras on a ring looking at a
// point cluster (normalized: unit-scale focal and a wider cluster)
struct Factory {
  std::mt19937 rng;
  explicit Factory(unsigned s) : rng(s) {}
  double u(double a, double b) { return std::uniform_real_distribution<double>(a, b)(rng); }
  CameraState<double> camera(bool normalized) {
    const double ang = u(0, 2 * M_PI), rad = u(2.0, 4.0);
    const double c[3] = {rad * std::cos(ang), rad * std::sin(ang), u(-0.5, 0.5)};
    const double cn = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    const double z[3] = {c[0] / cn, c[1] / cn, c[2] / cn};
    double r[3] = {-z[1], z[0], 0};  // (0,0,1) x z
    const double rn = std::sqrt(r[0] * r[0] + r[1] * r[1]);
    r[0] /= rn;
    r[1] /= rn;
    const double y[3] = {z[1] * r[2] - z[2] * r[1], z[2] * r[0] - z[0] * r[2], z[0] * r[1] - z[1] * r[0]};
    const double R[3][3] = {{r[0], r[1], r[2]}, {y[0], y[1], y[2]}, {z[0], z[1], z[2]}};
    const double tr = R[0][0] + R[1][1] + R[2][2];
    const double th = std::acos(std::max(-1.0, std::min(1.0, (tr - 1) / 2)));
    const double w[3] = {R[2][1] - R[1][2], R[0][2] - R[2][0], R[1][0] - R[0][1]};
    CameraState<double> cs;
    for (int i = 0; i < 3; ++i) {
      cs.rotation[i] = th * w[i] / (2 * std::sin(th)) + u(-0.05, 0.05);
      cs.translation[i] = -(R[i][0] * c[0] + R[i][1] * c[1] + R[i][2] * c[2]) + u(-0.05, 0.05);
    }
    cs.focal = normalized ? u(1.0, 3.0) : u(500.0, 1500.0);
    cs.k1 = normalized ? u(-0.3, 0.3) : u(-0.1, 0.1);
    cs.k2 = normalized ? u(-0.2, 0.2) : u(-0.05, 0.05);
    return cs;
  }
  BAProblem<double> problem(int cams, int pts, int edges, bool normalized = false) {
    BAProblem<double> p;
    for (int i = 0; i < cams; ++i) p.add_node(camera(normalized));
    for (int i = 0; i < pts; ++i) {
      PointState<double> ps;
      for (int j = 0; j < 3; ++j) ps.position[j] = normalized ? u(-1.2, 1.2) * (j == 2 ? 0.8 / 1.2 : 1.0) : u(-0.3, 0.3);
      p.add_node(ps);
    }
    for (int e = 0; e < edges; ++e) {
      Observation<double> o;
      o.camera_id = e < cams ? e : std::uniform_int_distribution<int>(0, cams - 1)(rng);
      o.point_id = e < pts ? e : std::uniform_int_distribution<int>(0, pts - 1)(rng);
      o.pixel = normalized ? std::array<double, 2>{u(-1, 1), u(-1, 1)} : std::array<double, 2>{u(-50, 50), u(-50, 50)};
      p.add_edge(o);
    }
    return p;
  }
};

template <int BS>
Mat dense_block_diagonal(const BlockDiagonal<double, BS>& d) {
  const int n = static_cast<int>(d.dim());
  Mat out(static_cast<std::size_t>(n) * n, 0.0);
  for (std::int64_t i = 0; i < d.blocks(); ++i)
    for (int r = 0; r < BS; ++r)
      for (int c = 0; c < BS; ++c) out[(i * BS + r) * n + i * BS + c] = d.block(i)(r, c);
  return out;
}
Mat dense_coupling(const EdgeBlockMatrix<double>& e) {
  const int m = static_cast<int>(e.camera_dim()), n = static_cast<int>(e.point_dim());
  Mat out(static_cast<std::size_t>(m) * n, 0.0);
  for (std::int64_t b = 0; b < e.blocks(); ++b)
    for (int r = 0; r < 9; ++r)
      for (int c = 0; c < 3; ++c) out[(9 * e.camera_of_block(b) + r) * n + 3 * e.point_of_block(b) + c] += e.block(b)(r, c);
  return out;
}
// dense Schur S = B - E C^-1 E^T (m x m)
Mat dense_schur(const Mat& B, const Mat& C, const Mat& E, int m, int n) {
  Mat X(static_cast<std::size_t>(n) * m);  // C^-1 E^T
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) X[i * m + j] = E[j * n + i];
  chol_solve(C, n, X, m);
  Mat S = B;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double s = 0;
      for (int p = 0; p < n; ++p) s += E[i * n + p] * X[p * m + j];
      S[i * m + j] -= s;
    }
  return S;
}
Vec matvec(const Mat& A, const Vec& x) {
  const std::size_t n = x.size();
  Vec y(A.size() / n, 0.0);
  for (std::size_t i = 0; i < y.size(); ++i)
    for (std::size_t j = 0; j < n; ++j) y[i] += A[i * n + j] * x[j];
  return y;
}

struct ReducedSystem {
  BAProblem<double> problem;
  Mat b, c, e;  // damped B / C, dense E
  double lambda;
};

ReducedSystem make_system(unsigned seed, int cams, int pts, int edges, double lambda, bool normalized = false) {
  Factory f(seed);
  ReducedSystem sys{f.problem(cams, pts, edges, normalized), {}, {}, {}, lambda};
  const auto parts = partition_edges(sys.problem, 1);
  auto h = assemble_local<double>(sys.problem, parts[0], pack_cameras(sys.problem), pack_points(sys.problem));
  BlockDiagonal<double, kCameraParams> bd;
  BlockDiagonal<double, kPointParams> cd;
  h.B.damp_into(lambda, DampingPolicy::identity, bd);
  h.C.damp_into(lambda, DampingPolicy::identity, cd);
  sys.b = dense_block_diagonal(bd);
  sys.c = dense_block_diagonal(cd);
  sys.e = dense_coupling(h.E);
  return sys;
}

// tests/test_solver.cpp:43-72: fn once per rank with that rank's
// partitioned, all-reduced, damped and factored system
template <typename Fn>
void with_partitioned_system(const BAProblem<double>& problem, int k, double lambda, Fn&& fn) {
  const auto parts = partition_edges(problem, k);
  const auto x_c = pack_cameras(problem);
  const auto x_p = pack_points(problem);
  WorkerGroup group(k);
  run_on_workers(group, [&](int rank) {
    auto h = assemble_local<double>(problem, parts[static_cast<std::size_t>(rank)], x_c, x_p);
    group.allreduce_sum(rank, h.B.data());
    group.allreduce_sum(rank, h.C.data());
    group.allreduce_sum(rank, h.v);
    group.allreduce_sum(rank, h.w);
    BlockDiagonal<double, kCameraParams> b_damped;
    BlockDiagonal<double, kPointParams> c_damped;
    h.B.damp_into(lambda, DampingPolicy::identity, b_damped);
    h.C.damp_into(lambda, DampingPolicy::identity, c_damped);
    FactoredBlockDiagonal<double, kCameraParams> b_inv;
    FactoredBlockDiagonal<double, kPointParams> c_inv;
    b_inv.factor(b_damped);
    c_inv.factor(c_damped);
    fn(rank, group, h, b_damped, b_inv, c_inv);
  });
}

void dse_zero_coupling() {  // tests/test_solver.cpp:74-105
  BlockDiagonal<double, kCameraParams> b(2);
  b.block(0).set_identity(2.0);
  b.block(1).set_identity(3.0);
  BlockDiagonal<double, kPointParams> c(1);
  c.block(0).set_identity();
  FactoredBlockDiagonal<double, kPointParams> c_inv;
  c_inv.factor(c);
  BAProblem<double> problem;
  problem.add_node(CameraState<double>{});
  problem.add_node(CameraState<double>{});
  PointState<double> pt;
  pt.position = {0, 0, -1};
  problem.add_node(pt);
  problem.add_edge(Observation<double>{});
  const auto parts = partition_edges(problem, 1);
  EdgeBlockMatrix<double> e(problem, parts[0]);
  e.set_zero();
  WorkerGroup group(1);
  run_on_workers(group, [&](int rank) {
    Vec x(18);
    for (int i = 0; i < 18; ++i) x[i] = i + 1;
    const Vec out = dse(x, b, e, c_inv, group, rank);
    CHECK(norm(sub(out, b.apply(x))) == 0.0);
    CHECK(norm(dse(Vec(18, 0.0), b, e, c_inv, group, rank)) == 0.0);
  });
}

void dse_dense_schur_across_k() {  // tests/test_solver.cpp:107-140
  std::mt19937 rng(31);
  std::uniform_real_distribution<double> dist(-1, 1);
  for (int trial = 0; trial < 10; ++trial) {
    const auto sys = make_system(1000 + trial, 3, 4, 9 + trial, 1e-3);
    const int m = 27, n = 12;
    Vec x(m);
    for (auto& v : x) v = dist(rng);
    const Vec expected = matvec(dense_schur(sys.b, sys.c, sys.e, m, n), x);
    Vec k1;
    for (int k : {1, 2, 3}) {
      std::vector<Vec> per_rank(static_cast<std::size_t>(k));
      with_partitioned_system(sys.problem, k, sys.lambda,
                              [&](int rank, WorkerGroup& group, PartitionedHessian<double>& h,
                                  BlockDiagonal<double, kCameraParams>& b_damped,
                                  FactoredBlockDiagonal<double, kCameraParams>&,
                                  FactoredBlockDiagonal<double, kPointParams>& c_inv) {
                                per_rank[static_cast<std::size_t>(rank)] = dse(x, b_damped, h.E, c_inv, group, rank);
                              });
      for (int r = 0; r < k; ++r) {
        CHECK(norm(sub(per_rank[r], expected)) / std::max(1.0, norm(expected)) < 1e-10);
        CHECK(per_rank[r] == per_rank[0]);  // rank-identical, bitwise
      }
      if (k == 1) k1 = per_rank[0];
      CHECK(norm(sub(per_rank[0], k1)) / std::max(1.0, norm(k1)) < 1e-10);
    }
  }
}

void dse_symmetric_psd() {  // tests/test_solver.cpp:142-177
  const auto sys = make_system(77, 4, 6, 15, 1e-2);
  std::mt19937 rng(7);
  std::uniform_real_distribution<double> dist(-1, 1);
  const int trials = 8, dim = 36;
  std::vector<Vec> xs(trials, Vec(dim)), ys(trials, Vec(dim));
  for (int t = 0; t < trials; ++t)
    for (int i = 0; i < dim; ++i) {
      xs[t][i] = dist(rng);
      ys[t][i] = dist(rng);
    }
  with_partitioned_system(sys.problem, 2, sys.lambda,
                          [&](int rank, WorkerGroup& group, PartitionedHessian<double>& h,
                              BlockDiagonal<double, kCameraParams>& b_damped,
                              FactoredBlockDiagonal<double, kCameraParams>&,
                              FactoredBlockDiagonal<double, kPointParams>& c_inv) {
                            for (int t = 0; t < trials; ++t) {
                              const Vec ax = dse(xs[t], b_damped, h.E, c_inv, group, rank);
                              const Vec ay = dse(ys[t], b_damped, h.E, c_inv, group, rank);
                              CHECK(dot(xs[t], ax) >= -1e-10 * std::max(1.0, norm(ax) * norm(xs[t])));
                              const double xay = dot(xs[t], ay), yax = dot(ys[t], ax);
                              CHECK(std::abs(xay - yax) <= 1e-10 * std::max({1.0, std::abs(xay), std::abs(yax)}));
                            }
                          });
}

void dpcg_zero_rhs() {  // tests/test_solver.cpp:179-196
  const auto sys = make_system(88, 2, 3, 6, 1e-2);
  with_partitioned_system(sys.problem, 1, sys.lambda,
                          [&](int rank, WorkerGroup& group, PartitionedHessian<double>& h,
                              BlockDiagonal<double, kCameraParams>& b_damped,
                              FactoredBlockDiagonal<double, kCameraParams>& b_inv,
                              FactoredBlockDiagonal<double, kPointParams>& c_inv) {
                            Vec x(static_cast<std::size_t>(b_damped.dim()), 0.0);
                            const Vec rhs(x.size(), 0.0);
                            PcgWorkspace<double> ws;
                            const PcgResult res = dpcg(x, b_damped, b_inv, h.E, c_inv, rhs, group, rank, 1e-6, 100, ws);
                            CHECK(res.iterations == 0);
                            CHECK(res.converged);
                            CHECK(norm(x) == 0.0);
                          });
}

void dpcg_identity_one_iteration() {  // tests/test_solver.cpp:198-229
  BAProblem<double> problem;
  problem.add_node(CameraState<double>{});
  PointState<double> pt;
  pt.position = {0, 0, -1};
  problem.add_node(pt);
  problem.add_edge(Observation<double>{});
  const auto parts = partition_edges(problem, 1);
  BlockDiagonal<double, kCameraParams> b(1);
  b.block(0).set_identity();
  BlockDiagonal<double, kPointParams> c(1);
  c.block(0).set_identity();
  FactoredBlockDiagonal<double, kCameraParams> b_inv;
  FactoredBlockDiagonal<double, kPointParams> c_inv;
  b_inv.factor(b);
  c_inv.factor(c);
  EdgeBlockMatrix<double> e(problem, parts[0]);
  e.set_zero();
  WorkerGroup group(1);
  run_on_workers(group, [&](int rank) {
    const Vec g = {1, -2, 3, -4, 5, -6, 7, -8, 9};
    Vec x(9, 0.0);
    PcgWorkspace<double> ws;
    const PcgResult res = dpcg(x, b, b_inv, e, c_inv, g, group, rank, 1e-10, 100, ws);
    CHECK(res.iterations == 1);
    CHECK(norm(sub(x, g)) < 1e-14);
  });
}

void dpcg_dense_direct_across_k() {  // tests/test_solver.cpp:231-270
  std::mt19937 rng(41);
  std::uniform_real_distribution<double> dist(-1, 1);
  for (int trial = 0; trial < 6; ++trial) {
    const auto sys = make_system(2000 + trial, 3, 5, 11 + trial, 1e-2, /*normalized=*/true);
    const int m = 27, n = 15;
    const Mat S = dense_schur(sys.b, sys.c, sys.e, m, n);
    Vec g(m);
    for (auto& v : g) v = dist(rng);
    Mat direct = g;
    chol_solve(S, m, direct, 1);
    for (int k : {1, 2, 4}) {
      if (k > sys.problem.num_observations()) continue;
      std::vector<Vec> sol(static_cast<std::size_t>(k));
      with_partitioned_system(sys.problem, k, sys.lambda,
                              [&](int rank, WorkerGroup& group, PartitionedHessian<double>& h,
                                  BlockDiagonal<double, kCameraParams>& b_damped,
                                  FactoredBlockDiagonal<double, kCameraParams>& b_inv,
                                  FactoredBlockDiagonal<double, kPointParams>& c_inv) {
                                Vec x(static_cast<std::size_t>(b_damped.dim()), 0.0);
                                PcgWorkspace<double> ws;
                                dpcg(x, b_damped, b_inv, h.E, c_inv, g, group, rank, 1e-12, 500, ws);
                                sol[static_cast<std::size_t>(rank)] = x;
                              });
      for (int r = 1; r < k; ++r) CHECK(sol[r] == sol[0]);
      CHECK(norm(sub(sol[0], direct)) / std::max(1.0, norm(direct)) < 1e-8);
    }
  }
}

void singular_block_and_damping() {  // tests/test_linear.cpp:270-298
  BlockDiagonal<double, kPointParams> d(3);
  d.block(0).set_identity();
  d.block(2).set_identity();  // block 1 stays zero
  FactoredBlockDiagonal<double, kPointParams> f;
  bool threw = false;
  try {
    f.factor(d);
  } catch (const SingularBlockError& e) {
    threw = e.block_index() == 1 && e.block_size() == 3;
  }
  CHECK(threw);
  BlockDiagonal<double, kPointParams> a(1), out;
  a.block(0)(0, 0) = 2;
  a.block(0)(1, 1) = 4;
  a.block(0)(2, 2) = 8;
  a.damp_into(0.5, DampingPolicy::diag_scaled, out);
  CHECK(out.block(0)(0, 0) == 3 && out.block(0)(1, 1) == 6 && out.block(0)(2, 2) == 12);
  FactoredBlockDiagonal<double, kPointParams> g;
  g.factor(out);
  Vec x = {3, 6, 12};
  g.solve_in_place(x);
  CHECK(std::abs(x[0] - 1) < 1e-15 && std::abs(x[1] - 1) < 1e-15 && std::abs(x[2] - 1) < 1e-15);
}

void allreduce_kat() {  // tests/test_comms.cpp: every rank gets the ascending-rank sum
  WorkerGroup group(3);
  std::vector<Vec> out(3);
  run_on_workers(group, [&](int rank) {
    Vec v = {double(rank), 10.0 * rank, 1.0};
    group.allreduce_sum(rank, v);
    out[static_cast<std::size_t>(rank)] = v;
    CHECK(group.allreduce_sum(rank, 0.5) == 1.5);
  });
  for (int r = 0; r < 3; ++r) CHECK((out[r] == Vec{3.0, 30.0, 3.0}));
  bool threw = false;
  try {
    run_on_workers(group, [&](int rank) {
      if (rank == 1) throw InvalidArgumentError("boom");
      group.barrier(rank);
    });
  } catch (const InvalidArgumentError&) {
    threw = true;
  }
  CHECK(threw);
}

void evaluator_assembly_and_lm_rank() {
  Factory f(5);
  const auto problem = f.problem(6, 30, 120, true);
  const auto x_c = pack_cameras(problem), x_p = pack_points(problem);
  // per-partition costs add up to total_cost; assembly sums to K = 1's
  const double total = total_cost(problem);
  const auto p1 = partition_edges(problem, 1);
  auto h1 = assemble_local<double>(problem, p1[0], x_c, x_p);
  for (int k : {2, 3}) {
    const auto parts = partition_edges(problem, k);
    double sum = 0;
    Vec B(h1.B.data().size(), 0.0), v(h1.v.size(), 0.0);
    for (int r = 0; r < k; ++r) {
      EdgeEvaluator<double> ev(problem, parts[r]);
      WorkCounters wc;
      sum += ev.cost(x_c, x_p, &wc);
      CHECK(wc.edges_evaluated == parts[r].edge_ids.size());
      PartitionedHessian<double> h(problem, parts[r]);
      const auto& batch = ev.linearize(x_c, x_p);
      CHECK(batch.size() == static_cast<std::int64_t>(parts[r].edge_ids.size()) && batch.all_finite());
      assemble_local(batch, ev, h);
      for (std::size_t i = 0; i < B.size(); ++i) B[i] += h.B.data()[i];
      for (std::size_t i = 0; i < v.size(); ++i) v[i] += h.v[i];
      // E blocks are the same per edge whichever partition holds it
      for (std::size_t i = 0; i < parts[r].edge_ids.size(); ++i)
        for (int q = 0; q < 27; ++q)
          CHECK(std::abs(h.E.data()[i * 27 + q] - h1.E.data()[parts[r].edge_ids[i] * 27 + q]) <=
                1e-12 * std::max(1.0, std::abs(h1.E.data()[parts[r].edge_ids[i] * 27 + q])));
    }
    CHECK(std::abs(sum - total) <= 1e-12 * total);
    CHECK(norm(sub(B, h1.B.data())) <= 1e-12 * norm(h1.B.data()));
    CHECK(norm(sub(v, h1.v)) <= 1e-12 * norm(h1.v));
  }
  CHECK(std::abs(mean_squared_error(problem) - total / (2.0 * 120)) <= 1e-15 * total);
  // lm_solve_rank inside run_on_workers = lm_solve at the same K
  SolverConfig cfg;
  cfg.workers = 2;
  cfg.max_iterations = 5;
  const auto ref = lm_solve(problem, cfg);
  const auto parts = partition_edges(problem, 2);
  WorkerGroup group(2);
  std::vector<SolverState<double>> st(2);
  run_on_workers(group, [&](int rank) {
    st[static_cast<std::size_t>(rank)] = lm_solve_rank(problem, cfg, parts[rank], group, rank);
  });
  for (int r = 0; r < 2; ++r) {
    CHECK(st[r].history.size() == ref.history.size());
    for (std::size_t i = 0; i < ref.history.size(); ++i) {
      CHECK(st[r].history[i].accepted == ref.history[i].accepted);
      CHECK(std::abs(st[r].history[i].cost - ref.history[i].cost) <= 1e-12 * ref.history[i].cost);
    }
    CHECK(st[r].x_c == st[0].x_c && st[r].x_p == st[0].x_p);  // rank-identical
    CHECK(check_convergence(st[r], cfg) != ConvergenceDecision::keep_going);
  }
  CHECK(ref.last_accepted == ref.history.back().accepted);
  CHECK(ref.previous_cost >= ref.cost || !ref.last_accepted);
}

// tests/test_solver.cpp:457-486 (host logic, runs in `compile` mode too).
void check_convergence_decisions() {
  SolverConfig config;
  config.max_iterations = 50;
  SolverState<double> state;
  state.iteration = 3;
  state.lambda = 1e-4;
  state.cost = 10.0;
  state.previous_cost = 10.0;

  state.last_accepted = true;
  state.last_cost_change = 0.0;
  state.last_step_inf = 1.0;
  CHECK(check_convergence(state, config) == ConvergenceDecision::converged);

  state.last_cost_change = 5.0;
  CHECK(check_convergence(state, config) == ConvergenceDecision::keep_going);

  state.last_step_inf = 1e-9;
  CHECK(check_convergence(state, config) == ConvergenceDecision::converged);

  state.last_accepted = false;
  state.last_step_inf = 1.0;
  state.iteration = 50;
  CHECK(check_convergence(state, config) == ConvergenceDecision::max_iterations);

  state.iteration = 3;
  state.lambda = 2e32;
  CHECK(check_convergence(state, config) == ConvergenceDecision::stalled);
}

}  // namespace

int main(int argc, char** argv) {
  check_convergence_decisions();
  if (argc > 1 && std::strcmp(argv[1], "compile") == 0) {
    std::printf("ops compiled\n");
    return 0;
  }
  dse_zero_coupling();
  dse_dense_schur_across_k();
  dse_symmetric_psd();
  dpcg_zero_rhs();
  dpcg_identity_one_iteration();
  dpcg_dense_direct_across_k();
  singular_block_and_damping();
  allreduce_kat();
  evaluator_assembly_and_lm_rank();
  std::printf("ops gpu ok\n");
  return 0;
}
