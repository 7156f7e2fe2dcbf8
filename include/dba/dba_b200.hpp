// dba_b200.hpp — C++ drop-in facade of the reference's `dba` solver API over
// the B200 C ABI (include/dbag.h).
//
// Same names, argument meaning and error behaviour as the reference's
// header-only API, without its Eigen dependency:
//   BAProblem<Scalar>::add_node / add_edge   dba/problem.hpp:171-261
//   SolverConfig, IterationRecord, SolverState, TerminationReason
//                                            dba/solver.hpp:39-85
//   lm_solve(problem, config)                dba/solver.hpp:523-534
//   partition_edges(problem, K)              dba/partition.hpp:76-103
//   generate_synthetic(options)              dba/synthetic.hpp:70-146
//   parse_bal / serialize_bal                dba/bal_io.hpp:78-209
//   the exception hierarchy                  dba/errors.hpp:17-84
// A reference user switches by including this header instead of
// dba/solver.hpp and linking libdbag.so.
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <istream>
#include <limits>
#include <iterator>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../dbag.h"

namespace dba {

// ---- errors (dba/errors.hpp) ------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ParseError : public Error {  // message "line L: ..." (dba/errors.hpp:17-26)
 public:
  ParseError(const std::string& m, std::int64_t line) : Error(m), line_(line) {}
  std::int64_t line() const { return line_; }

 private:
  std::int64_t line_;
};
class InvalidArgumentError : public Error {
 public:
  using Error::Error;
};
class ShapeError : public Error {
 public:
  using Error::Error;
};
class CollectiveError : public Error {
 public:
  using Error::Error;
};
class PcgBreakdownError : public Error {
 public:
  using Error::Error;
};
class DegenerateDepthError : public Error {
 public:
  explicit DegenerateDepthError(std::int64_t edge_id = -1, const std::string& m = "degenerate depth (P_z = 0)")
      : Error(m), edge_id_(edge_id) {}
  std::int64_t edge_id() const { return edge_id_; }

 private:
  std::int64_t edge_id_;
};
class SingularBlockError : public Error {
 public:
  SingularBlockError(std::int64_t idx, int bs, const std::string& m) : Error(m), idx_(idx), bs_(bs) {}
  std::int64_t block_index() const { return idx_; }
  int block_size() const { return bs_; }

 private:
  std::int64_t idx_;
  int bs_;
};

namespace detail {
inline void check(int rc) {
  if (rc == DBAG_OK) return;
  const std::string msg = dbag_last_error();
  switch (rc) {
    case DBAG_DEGENERATE_DEPTH: throw DegenerateDepthError(dbag_last_error_index(), msg);
    case DBAG_SINGULAR_BLOCK: throw SingularBlockError(dbag_last_error_index(), dbag_last_error_block_size(), msg);
    case DBAG_PCG_BREAKDOWN: throw PcgBreakdownError(msg);
    case DBAG_SHAPE: throw ShapeError(msg);
    case DBAG_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
    case DBAG_COLLECTIVE: throw CollectiveError(msg);
    case DBAG_PARSE: throw ParseError(msg, dbag_last_error_index());
    default: throw Error(msg);
  }
}
}  // namespace detail

// ---- problem model (dba/problem.hpp) ----------------------------------------
enum class MseConvention { per_observation, half_per_observation };
enum class DampingPolicy { identity, diag_scaled };
enum class JacobianMode { autodiff, analytic };
enum class TerminationReason { converged, max_iterations, stalled };

inline constexpr int kCameraParams = 9;
inline constexpr int kPointParams = 3;

template <typename Scalar>
struct CameraState {
  std::array<Scalar, 3> rotation{};
  std::array<Scalar, 3> translation{};
  Scalar focal = Scalar(1);
  Scalar k1 = Scalar(0);
  Scalar k2 = Scalar(0);
  bool all_finite() const {
    for (Scalar v : rotation)
      if (!std::isfinite(double(v))) return false;
    for (Scalar v : translation)
      if (!std::isfinite(double(v))) return false;
    return std::isfinite(double(focal)) && std::isfinite(double(k1)) && std::isfinite(double(k2));
  }
};

template <typename Scalar>
struct PointState {
  std::array<Scalar, 3> position{};
  bool all_finite() const {
    for (Scalar v : position)
      if (!std::isfinite(double(v))) return false;
    return true;
  }
};

template <typename Scalar>
struct Observation {
  std::int32_t camera_id = 0;
  std::int32_t point_id = 0;
  std::array<Scalar, 2> pixel{};
  Scalar weight = Scalar(1);
};

template <typename Scalar>
class BAProblem {
 public:
  std::int32_t add_node(const CameraState<Scalar>& c) {
    if (!c.all_finite()) throw InvalidArgumentError("camera node has non-finite components");
    cams_.insert(cams_.end(), c.rotation.begin(), c.rotation.end());
    cams_.insert(cams_.end(), c.translation.begin(), c.translation.end());
    cams_.push_back(c.focal);
    cams_.push_back(c.k1);
    cams_.push_back(c.k2);
    return num_cameras() - 1;
  }
  std::int32_t add_node(const PointState<Scalar>& p) {
    if (!p.all_finite()) throw InvalidArgumentError("point node has non-finite components");
    pts_.insert(pts_.end(), p.position.begin(), p.position.end());
    return num_points() - 1;
  }
  std::int32_t add_edge(const Observation<Scalar>& o) {
    if (o.camera_id < 0 || o.camera_id >= num_cameras())
      throw InvalidArgumentError("edge references unknown camera " + std::to_string(o.camera_id));
    if (o.point_id < 0 || o.point_id >= num_points())
      throw InvalidArgumentError("edge references unknown point " + std::to_string(o.point_id));
    if (!(o.weight >= Scalar(0))) throw InvalidArgumentError("edge weight must be >= 0");
    cam_id_.push_back(o.camera_id);
    pt_id_.push_back(o.point_id);
    px_.push_back(o.pixel[0]);
    py_.push_back(o.pixel[1]);
    w_.push_back(o.weight);
    return static_cast<std::int32_t>(cam_id_.size()) - 1;
  }
  // Node / edge views (dba/problem.hpp:219-227): states are stored flat
  // (pack_cameras / pack_points layout), so these return copies.
  CameraState<Scalar> camera(std::int32_t i) const {
    const Scalar* q = cams_.data() + static_cast<std::size_t>(i) * kCameraParams;
    CameraState<Scalar> c;
    c.rotation = {q[0], q[1], q[2]};
    c.translation = {q[3], q[4], q[5]};
    c.focal = q[6];
    c.k1 = q[7];
    c.k2 = q[8];
    return c;
  }
  PointState<Scalar> point(std::int32_t i) const {
    const Scalar* q = pts_.data() + static_cast<std::size_t>(i) * kPointParams;
    PointState<Scalar> p;
    p.position = {q[0], q[1], q[2]};
    return p;
  }
  Observation<Scalar> observation(std::int64_t e) const {
    const std::size_t k = static_cast<std::size_t>(e);
    Observation<Scalar> o;
    o.camera_id = cam_id_[k];
    o.point_id = pt_id_[k];
    o.pixel = {px_[k], py_[k]};
    o.weight = w_[k];
    return o;
  }
  std::vector<CameraState<Scalar>> cameras() const {
    std::vector<CameraState<Scalar>> v;
    for (std::int32_t i = 0; i < num_cameras(); ++i) v.push_back(camera(i));
    return v;
  }
  std::vector<PointState<Scalar>> points() const {
    std::vector<PointState<Scalar>> v;
    for (std::int32_t i = 0; i < num_points(); ++i) v.push_back(point(i));
    return v;
  }
  std::vector<Observation<Scalar>> observations() const {
    std::vector<Observation<Scalar>> v;
    for (std::int64_t e = 0; e < num_observations(); ++e) v.push_back(observation(e));
    return v;
  }
  // BAProblem::validate (dba/problem.hpp:231-255): warnings, not errors.
  std::vector<std::string> validate() const {
    std::vector<std::string> w;
    std::vector<bool> cu(static_cast<std::size_t>(num_cameras())), pu(static_cast<std::size_t>(num_points()));
    for (std::size_t e = 0; e < cam_id_.size(); ++e) {
      cu[static_cast<std::size_t>(cam_id_[e])] = true;
      pu[static_cast<std::size_t>(pt_id_[e])] = true;
    }
    for (std::int32_t i = 0; i < num_cameras(); ++i)
      if (!cu[static_cast<std::size_t>(i)]) w.push_back("camera " + std::to_string(i) + " is not referenced by any observation");
    for (std::int32_t i = 0; i < num_points(); ++i)
      if (!pu[static_cast<std::size_t>(i)]) w.push_back("point " + std::to_string(i) + " is not referenced by any observation");
    for (std::int32_t i = 0; i < num_cameras(); ++i)
      if (!(cams_[static_cast<std::size_t>(i) * kCameraParams + 6] > Scalar(0)))
        w.push_back("camera " + std::to_string(i) + " has non-positive focal length");
    return w;
  }
  std::int32_t num_cameras() const { return static_cast<std::int32_t>(cams_.size() / kCameraParams); }
  std::int32_t num_points() const { return static_cast<std::int32_t>(pts_.size() / kPointParams); }
  std::int64_t num_observations() const { return static_cast<std::int64_t>(cam_id_.size()); }
  const std::vector<Scalar>& packed_cameras() const { return cams_; }  // pack_cameras
  const std::vector<Scalar>& packed_points() const { return pts_; }    // pack_points

  dbag_problem c_view() const {
    dbag_problem p;
    p.num_cameras = num_cameras();
    p.num_points = num_points();
    p.num_observations = num_observations();
    p.cameras = cams_.data();
    p.points = pts_.data();
    p.camera_id = cam_id_.data();
    p.point_id = pt_id_.data();
    p.pixel_x = px_.data();
    p.pixel_y = py_.data();
    p.weight = w_.data();
    return p;
  }

 private:
  std::vector<Scalar> cams_, pts_, px_, py_, w_;
  std::vector<std::int32_t> cam_id_, pt_id_;
};

// ---- solver (dba/solver.hpp) ------------------------------------------------
struct SolverConfig {
  int workers = 1;
  int max_iterations = 50;
  double pcg_tol = 1e-6;
  int pcg_max_iters = 500;
  double lambda0 = 1e-4;
  double lambda_max = 1e32;
  double rel_tol = 1e-6;
  double step_tol = 1e-8;
  DampingPolicy damping = DampingPolicy::diag_scaled;
  MseConvention mse = MseConvention::half_per_observation;
  JacobianMode jacobian = JacobianMode::autodiff;
  bool check_rank_identity = false;
  std::chrono::milliseconds collective_timeout{60000};  // dba/solver.hpp:54
  std::vector<int> devices{0};  // B200 placement: rank r -> devices[r % size]
  bool coupling_fp32 = false;     // B200 extension (row f4): E blocks stored in FP32 under an FP64 solve

  dbag_config c_view() const {
    dbag_config c;
    dbag_default_config(&c);
    c.workers = workers;
    c.max_iterations = max_iterations;
    c.pcg_tol = pcg_tol;
    c.pcg_max_iters = pcg_max_iters;
    c.lambda0 = lambda0;
    c.lambda_max = lambda_max;
    c.rel_tol = rel_tol;
    c.step_tol = step_tol;
    c.damping = damping == DampingPolicy::diag_scaled ? 1 : 0;
    c.mse_half = mse == MseConvention::half_per_observation ? 1 : 0;
    c.jacobian = jacobian == JacobianMode::analytic ? 1 : 0;
    c.check_rank_identity = check_rank_identity ? 1 : 0;
    c.collective_timeout_ms = static_cast<int64_t>(collective_timeout.count());
    c.coupling_fp32 = coupling_fp32 ? 1 : 0;
    return c;
  }
};

struct IterationRecord {
  int iteration = 0;
  double cost = 0, mse = 0, lambda = 0;
  int pcg_iterations = 0;
  bool accepted = false;
  double wall_seconds = 0;
  std::vector<std::uint64_t> worker_edges, worker_block_ops;
};

template <typename Scalar>
struct SolverState {
  std::vector<Scalar> x_c, x_p;
  double lambda = 0, nu = 2;
  int iteration = 0;
  double cost = 0;
  TerminationReason termination = TerminationReason::max_iterations;
  std::vector<IterationRecord> history;
  // Most recent trial, feeding the convergence decision (dba/solver.hpp:80-84).
  bool last_accepted = false;
  double last_cost_change = std::numeric_limits<double>::infinity();
  double last_step_inf = std::numeric_limits<double>::infinity();
  double previous_cost = std::numeric_limits<double>::infinity();
};

namespace detail {
// dbag_result -> SolverState (parameters already written through r.x_c / x_p).
template <typename Scalar>
void fill_state(const dbag_result& r, int cap, int k, const std::vector<std::int32_t>& it,
                const std::vector<double>& cost, const std::vector<double>& mse, const std::vector<double>& lam,
                const std::vector<std::int32_t>& pcg, const std::vector<std::int32_t>& acc,
                const std::vector<double>& wall, const std::vector<std::uint64_t>& we,
                const std::vector<std::uint64_t>& wb, SolverState<Scalar>& st) {
  st.lambda = r.lambda;
  st.nu = r.nu;
  st.iteration = r.iterations;
  st.cost = r.cost;
  st.termination = static_cast<TerminationReason>(r.termination);
  st.last_accepted = r.last_accepted != 0;
  st.last_cost_change = r.last_cost_change;
  st.last_step_inf = r.last_step_inf;
  st.previous_cost = r.previous_cost;
  for (int i = 0; i < std::min(cap, r.iterations); ++i) {
    IterationRecord rec;
    rec.iteration = it[static_cast<std::size_t>(i)];
    rec.cost = cost[static_cast<std::size_t>(i)];
    rec.mse = mse[static_cast<std::size_t>(i)];
    rec.lambda = lam[static_cast<std::size_t>(i)];
    rec.pcg_iterations = pcg[static_cast<std::size_t>(i)];
    rec.accepted = acc[static_cast<std::size_t>(i)] != 0;
    rec.wall_seconds = wall[static_cast<std::size_t>(i)];
    rec.worker_edges.assign(we.begin() + i * k, we.begin() + (i + 1) * k);
    rec.worker_block_ops.assign(wb.begin() + i * k, wb.begin() + (i + 1) * k);
    st.history.push_back(rec);
  }
}

// Runs fn(dbag_result&) with record buffers sized for cap iterations x k ranks.
template <typename Scalar, class Fn>
SolverState<Scalar> solve_into(std::size_t ncam, std::size_t npt, int cap, int k, Fn&& fn) {
  SolverState<Scalar> st;
  st.x_c.resize(ncam);
  st.x_p.resize(npt);
  std::vector<std::int32_t> it(cap), pcg(cap), acc(cap);
  std::vector<double> cost(cap), mse(cap), lam(cap), wall(cap);
  std::vector<std::uint64_t> we(static_cast<std::size_t>(cap) * k), wb(static_cast<std::size_t>(cap) * k);
  dbag_result r{};
  r.capacity = cap;
  r.rec_iteration = it.data();
  r.rec_cost = cost.data();
  r.rec_mse = mse.data();
  r.rec_lambda = lam.data();
  r.rec_pcg = pcg.data();
  r.rec_accepted = acc.data();
  r.rec_wall = wall.data();
  r.rec_worker_edges = we.data();
  r.rec_worker_block_ops = wb.data();
  r.x_c = st.x_c.data();
  r.x_p = st.x_p.data();
  fn(r);
  fill_state(r, cap, k, it, cost, mse, lam, pcg, acc, wall, we, wb, st);
  return st;
}
}  // namespace detail

// dba::lm_solve on B200: config.workers ranks, rank 0's state.
template <typename Scalar>
SolverState<Scalar> lm_solve(const BAProblem<Scalar>& problem, const SolverConfig& config) {
  static_assert(sizeof(Scalar) == 4 || sizeof(Scalar) == 8, "Scalar must be float or double");
  const dbag_problem p = problem.c_view();
  const dbag_config c = config.c_view();
  return detail::solve_into<Scalar>(problem.packed_cameras().size(), problem.packed_points().size(),
                                    config.max_iterations, config.workers, [&](dbag_result& r) {
                                      detail::check(dbag_lm_solve(static_cast<int>(sizeof(Scalar)), &p, &c,
                                                                  config.devices.data(),
                                                                  static_cast<int>(config.devices.size()), &r));
                                    });
}

// ---- partitioning (dba/partition.hpp) ----------------------------------------
struct EdgePartition {
  int worker_rank = 0;
  int worker_count = 1;  // B200 facade: K of the split this partition belongs to
  std::vector<std::int32_t> edge_ids;
  std::vector<std::int32_t> camera_to_global, point_to_global;  // LocalIndexMap::to_global
};

template <typename Scalar>
std::vector<EdgePartition> partition_edges(const BAProblem<Scalar>& problem, int worker_count) {
  const dbag_problem p = problem.c_view();
  std::vector<EdgePartition> out;
  if (worker_count < 1) throw InvalidArgumentError("worker count must be >= 1");
  const std::size_t m = static_cast<std::size_t>(p.num_cameras), n = static_cast<std::size_t>(p.num_points),
                    N = static_cast<std::size_t>(p.num_observations);
  for (int r = 0; r < worker_count; ++r) {
    std::int64_t start = 0, count = 0;
    std::int32_t nc = 0, np = 0;
    std::vector<std::int32_t> cg(std::max<std::size_t>(m, 1)), pg(std::max<std::size_t>(n, 1));
    std::vector<std::int64_t> cptr(m + 1), pptr(n + 1), cblk(std::max<std::size_t>(N, 1)),
        pblk(std::max<std::size_t>(N, 1));
    detail::check(dbag_partition(&p, worker_count, r, &start, &count, &nc, cg.data(), &np, pg.data(), cptr.data(),
                                 cblk.data(), pptr.data(), pblk.data()));
    EdgePartition e;
    e.worker_rank = r;
    e.worker_count = worker_count;
    for (std::int64_t i = 0; i < count; ++i) e.edge_ids.push_back(static_cast<std::int32_t>(start + i));
    e.camera_to_global.assign(cg.begin(), cg.begin() + nc);
    e.point_to_global.assign(pg.begin(), pg.begin() + np);
    out.push_back(std::move(e));
  }
  return out;
}

// ---- predicted-size memory pool (B200 extension) ------------
// Device bytes rank `rank` of `worker_count` reserves in its one pool
// allocation when lm_solve uploads its shard; host-only, no GPU needed.
template <typename Scalar>
std::uint64_t predict_memory(const BAProblem<Scalar>& problem, int worker_count = 1, int rank = 0,
                             bool coupling_fp32 = false) {
  const dbag_problem p = problem.c_view();
  std::uint64_t bytes = 0;
  detail::check(dbag_predict_memory(&p, static_cast<int>(sizeof(Scalar)), coupling_fp32 ? 1 : 0, worker_count, rank,
                                    &bytes));
  return bytes;
}

// ---- synthetic generator (dba/synthetic.hpp) ---------------------------------
struct SyntheticOptions {
  std::int32_t cameras = 20000, points = 80000, obs_per_point = 1000;
  std::uint64_t seed = 1;
  double circle_radius = 8.0, base_focal = 1000.0, pose_noise = 0.01, intrinsic_noise = 0.5, point_noise = 0.1;
  std::int64_t num_observations = 0;  // > 0: count-exact extension
  double pixel_noise = 0.0;
};

inline BAProblem<double> generate_synthetic(const SyntheticOptions& o) {
  dbag_synthetic_options c{};
  c.cameras = o.cameras;
  c.points = o.points;
  c.obs_per_point = o.obs_per_point;
  c.seed = o.seed;
  c.circle_radius = o.circle_radius;
  c.base_focal = o.base_focal;
  c.pose_noise = o.pose_noise;
  c.intrinsic_noise = o.intrinsic_noise;
  c.point_noise = o.point_noise;
  c.num_observations = o.num_observations;
  c.pixel_noise = o.pixel_noise;
  std::int64_t N = 0;
  detail::check(dbag_synthetic_count(&c, &N));
  std::vector<double> cams(static_cast<std::size_t>(o.cameras) * 9), pts(static_cast<std::size_t>(o.points) * 3),
      px(static_cast<std::size_t>(N)), py(static_cast<std::size_t>(N));
  std::vector<std::int32_t> cid(static_cast<std::size_t>(N)), pid(static_cast<std::size_t>(N));
  detail::check(dbag_generate_synthetic(&c, cams.data(), pts.data(), cid.data(), pid.data(), px.data(), py.data()));
  BAProblem<double> p;
  for (std::int32_t i = 0; i < o.cameras; ++i) {
    CameraState<double> cs;
    const double* q = cams.data() + static_cast<std::size_t>(i) * 9;
    cs.rotation = {q[0], q[1], q[2]};
    cs.translation = {q[3], q[4], q[5]};
    cs.focal = q[6];
    cs.k1 = q[7];
    cs.k2 = q[8];
    p.add_node(cs);
  }
  for (std::int32_t i = 0; i < o.points; ++i) {
    PointState<double> ps;
    ps.position = {pts[static_cast<std::size_t>(i) * 3], pts[static_cast<std::size_t>(i) * 3 + 1],
                   pts[static_cast<std::size_t>(i) * 3 + 2]};
    p.add_node(ps);
  }
  for (std::int64_t e = 0; e < N; ++e) {
    Observation<double> ob;
    ob.camera_id = cid[static_cast<std::size_t>(e)];
    ob.point_id = pid[static_cast<std::size_t>(e)];
    ob.pixel = {px[static_cast<std::size_t>(e)], py[static_cast<std::size_t>(e)]};
    p.add_edge(ob);
  }
  return p;
}

// ---- BAL text (dba/bal_io.hpp) ---------------------------------------------
// parse_bal<Scalar>: reals parsed in double and cast to Scalar, observations
// with weight 1; ParseError("line L: ...") on malformed text; validate()-style
// warnings (unreferenced nodes, non-positive focal) appended to `warnings`.
template <typename Scalar>
BAProblem<Scalar> parse_bal(std::istream& in, std::vector<std::string>* warnings = nullptr) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  dbag_bal* h = nullptr;
  detail::check(dbag_bal_parse(text.data(), static_cast<std::int64_t>(text.size()), &h));
  std::int32_t m = 0, n = 0;
  std::int64_t N = 0;
  std::vector<double> cams, pts, px, py;
  std::vector<std::int32_t> cid, pid;
  try {
    detail::check(dbag_bal_counts(h, &m, &n, &N));
    cams.resize(static_cast<std::size_t>(m) * 9);
    pts.resize(static_cast<std::size_t>(n) * 3);
    px.resize(static_cast<std::size_t>(N));
    py.resize(static_cast<std::size_t>(N));
    cid.resize(static_cast<std::size_t>(N));
    pid.resize(static_cast<std::size_t>(N));
    detail::check(dbag_bal_copy(h, cams.data(), pts.data(), cid.data(), pid.data(), px.data(), py.data()));
  } catch (...) {
    dbag_bal_free(h);
    throw;
  }
  dbag_bal_free(h);
  BAProblem<Scalar> p;
  std::vector<bool> cam_used(static_cast<std::size_t>(m)), pt_used(static_cast<std::size_t>(n));
  for (std::int32_t i = 0; i < m; ++i) {
    const double* q = cams.data() + static_cast<std::size_t>(i) * 9;
    CameraState<Scalar> c;
    for (int j = 0; j < 3; ++j) c.rotation[j] = static_cast<Scalar>(q[j]);
    for (int j = 0; j < 3; ++j) c.translation[j] = static_cast<Scalar>(q[3 + j]);
    c.focal = static_cast<Scalar>(q[6]);
    c.k1 = static_cast<Scalar>(q[7]);
    c.k2 = static_cast<Scalar>(q[8]);
    p.add_node(c);
  }
  for (std::int32_t i = 0; i < n; ++i) {
    PointState<Scalar> ps;
    for (int j = 0; j < 3; ++j) ps.position[j] = static_cast<Scalar>(pts[static_cast<std::size_t>(i) * 3 + j]);
    p.add_node(ps);
  }
  for (std::int64_t e = 0; e < N; ++e) {
    Observation<Scalar> o;
    o.camera_id = cid[static_cast<std::size_t>(e)];
    o.point_id = pid[static_cast<std::size_t>(e)];
    o.pixel = {static_cast<Scalar>(px[static_cast<std::size_t>(e)]), static_cast<Scalar>(py[static_cast<std::size_t>(e)])};
    p.add_edge(o);
    cam_used[static_cast<std::size_t>(o.camera_id)] = true;
    pt_used[static_cast<std::size_t>(o.point_id)] = true;
  }
  if (warnings) {  // BAProblem::validate (dba/problem.hpp:231-255)
    for (std::int32_t i = 0; i < m; ++i)
      if (!cam_used[static_cast<std::size_t>(i)])
        warnings->push_back("camera " + std::to_string(i) + " is not referenced by any observation");
    for (std::int32_t i = 0; i < n; ++i)
      if (!pt_used[static_cast<std::size_t>(i)])
        warnings->push_back("point " + std::to_string(i) + " is not referenced by any observation");
    for (std::int32_t i = 0; i < m; ++i)
      if (!(p.packed_cameras()[static_cast<std::size_t>(i) * 9 + 6] > Scalar(0)))
        warnings->push_back("camera " + std::to_string(i) + " has non-positive focal length");
  }
  return p;
}

template <typename Scalar>
void serialize_bal(const BAProblem<Scalar>& problem, std::ostream& out) {
  const dbag_problem v = problem.c_view();
  char* text = nullptr;
  std::int64_t len = 0;
  detail::check(dbag_bal_format(static_cast<int>(sizeof(Scalar)), &v, &text, &len));
  out.write(text, static_cast<std::streamsize>(len));
  dbag_free_text(text);
}

}  // namespace dba

// the operator level (WorkerGroup, BlockDiagonal, EdgeBlockMatrix, dse, dpcg,
// EdgeEvaluator, assemble_local, lm_solve_rank, ...)
#include "dba_b200_ops.hpp"
