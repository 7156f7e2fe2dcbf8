// dba_b200_ops.hpp — the operator level of the reference's dba:: API over the
// B200 C ABI (include/dbag.h), for code that drives the solver step by step
// the way the reference's tests and acceptance runner do:
//
//   WorkerGroup, run_on_workers                 dba/comms.hpp:35-234
//   BlockDiagonal, FactoredBlockDiagonal,
//   EdgeBlockMatrix, PartitionedHessian,
//   assemble_local                              dba/block_matrix.hpp:36-400
//   EdgeEvaluator, EdgeJacobianBatch            dba/edge_eval.hpp:21-309
//   dse, dpcg, PcgResult, workspaces            dba/solver.hpp:134-257
//   lm_solve_rank, check_convergence            dba/solver.hpp:91-104, 295-518
//   total_cost, mean_squared_error              dba/problem.hpp:266-290
//   WorkCounters                                dba/counters.hpp:11-24
//
// Included by dba_b200.hpp. Vectors are std::vector<Scalar> (the reference's
// Eigen vectors, same layout). The matrices are host containers — mirrors
// with the reference's accessors, for building and inspecting systems; every
// operator that computes (factor, solve, dse, dpcg, linearize, cost,
// assemble_local, lm_solve_rank) runs on the GPU through a rank context:
//   * EdgeEvaluator holds a shard context with local collectives (its cost
//     and assembly are the partition's own contribution, as in the
//     reference);
//   * dse / dpcg / lm_solve_rank run on the rank's context inside the
//     WorkerGroup, whose collectives are the group's (call them from
//     run_on_workers bodies, one thread per rank, like the reference).
// Each call uploads the blocks it is given (set_system), so a caller may edit
// the host blocks between calls exactly as with the reference's containers.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace dba {

// ---- counters (dba/counters.hpp:11-24) -----------------------------------------
struct WorkCounters {
  std::uint64_t edges_evaluated = 0;
  std::uint64_t edge_block_ops = 0;
};

// ---- WorkerGroup (dba/comms.hpp:35-234) ------------------------------------------
// K in-process ranks on devices[rank % size]: collectives validate call
// sequence, kind, element type and length; a missing rank trips the timeout
// naming the absent ranks (CollectiveError); abort() fails every pending and
// later collective.
class WorkerGroup {
 public:
  explicit WorkerGroup(int workers, std::chrono::milliseconds timeout = std::chrono::milliseconds(60000),
                       std::vector<int> devices = {0})
      : workers_(workers) {
    if (workers < 1) throw InvalidArgumentError("worker group needs at least one rank");
    detail::check(dbag_group_create(workers, devices.data(), static_cast<int>(devices.size()),
                                    static_cast<std::int64_t>(timeout.count()), &g_));
  }
  ~WorkerGroup() { dbag_group_destroy(g_); }
  WorkerGroup(const WorkerGroup&) = delete;
  WorkerGroup& operator=(const WorkerGroup&) = delete;

  int workers() const { return workers_; }
  std::uint64_t sequence(int rank) const {
    std::uint64_t s = 0;
    detail::check(dbag_group_sequence(g_, rank, &s));
    return s;
  }
  void barrier(int rank) { detail::check(dbag_group_barrier(g_, rank)); }
  // data := ascending-rank sum over the ranks' buffers (bit-identical on
  // every rank); float and double
  template <typename T>
  void allreduce_sum(int rank, T* data, std::size_t n) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "float or double");
    detail::check(dbag_group_allreduce_sum(g_, rank, data, static_cast<std::int64_t>(n), static_cast<int>(sizeof(T))));
  }
  template <typename T>
  void allreduce_sum(int rank, std::vector<T>& data) {
    allreduce_sum(rank, data.data(), data.size());
  }
  double allreduce_sum(int rank, double value) {
    allreduce_sum(rank, &value, 1);
    return value;
  }
  void abort(const std::string& reason, const std::exception_ptr& cause = nullptr) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (!first_failure_ && cause) first_failure_ = cause;
    }
    dbag_group_abort(g_, reason.c_str());
  }
  std::exception_ptr first_failure() const {
    std::lock_guard<std::mutex> lk(mu_);
    return first_failure_;
  }
  dbag_group* handle() { return g_; }

 private:
  int workers_;
  dbag_group* g_ = nullptr;
  mutable std::mutex mu_;
  std::exception_ptr first_failure_;
};

// run_on_workers (dba/comms.hpp:214-234): body(rank) on one thread per rank;
// a throwing rank aborts the group and its exception is rethrown after join.
template <typename Fn>
void run_on_workers(WorkerGroup& group, Fn&& body) {
  std::vector<std::thread> threads;
  for (int rank = 0; rank < group.workers(); ++rank) {
    threads.emplace_back([&group, &body, rank] {
      try {
        body(rank);
      } catch (const std::exception& e) {
        group.abort("rank " + std::to_string(rank) + " failed: " + e.what(), std::current_exception());
      } catch (...) {
        group.abort("rank " + std::to_string(rank) + " failed", std::current_exception());
      }
    });
  }
  for (auto& t : threads) t.join();
  if (auto f = group.first_failure()) std::rethrow_exception(f);
}

namespace detail {
// Owning handle of a rank context.
struct Ctx {
  dbag_ctx* c = nullptr;
  explicit Ctx(dbag_ctx* p) : c(p) {}
  ~Ctx() { dbag_destroy(c); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
};
template <typename Scalar>
constexpr int prec() {
  static_assert(sizeof(Scalar) == 4 || sizeof(Scalar) == 8, "Scalar must be float or double");
  return static_cast<int>(sizeof(Scalar));
}
}  // namespace detail

// ---- block containers (dba/block_matrix.hpp:17-167) -------------------------------
inline constexpr double kDampingDiagFloor = 1e-6;
inline constexpr double kDampingDiagCeiling = 1e32;

template <typename Scalar>
Scalar clamped_curvature(Scalar diag) {
  return std::min(static_cast<Scalar>(kDampingDiagCeiling), std::max(static_cast<Scalar>(kDampingDiagFloor), diag));
}

// A BS x BS row-major block viewed in place: b(r, c).
template <typename Scalar, int BS>
struct BlockRef {
  Scalar* p;
  Scalar& operator()(int r, int c) const { return p[r * BS + c]; }
  void set_identity(Scalar s = Scalar(1)) const {
    for (int r = 0; r < BS; ++r)
      for (int c = 0; c < BS; ++c) p[r * BS + c] = r == c ? s : Scalar(0);
  }
};

// BlockDiagonal<Scalar, BS> (dba/block_matrix.hpp:36-108): blocks stored
// contiguously, row-major within each block. Host container; the solver's
// own damping and factorization run on the device (k_damp_factor).
template <typename Scalar, int BS>
class BlockDiagonal {
 public:
  BlockDiagonal() = default;
  explicit BlockDiagonal(std::int64_t num_blocks) { resize(num_blocks); }
  void resize(std::int64_t num_blocks) {
    num_blocks_ = num_blocks;
    data_.assign(static_cast<std::size_t>(num_blocks) * BS * BS, Scalar(0));
  }
  void set_zero() { std::fill(data_.begin(), data_.end(), Scalar(0)); }
  std::int64_t blocks() const { return num_blocks_; }
  std::int64_t dim() const { return num_blocks_ * BS; }
  BlockRef<Scalar, BS> block(std::int64_t i) { return {data_.data() + static_cast<std::size_t>(i) * BS * BS}; }
  BlockRef<const Scalar, BS> block(std::int64_t i) const {
    return {data_.data() + static_cast<std::size_t>(i) * BS * BS};
  }
  std::vector<Scalar>& data() { return data_; }
  const std::vector<Scalar>& data() const { return data_; }
  // y = D x (the reference's container helper)
  std::vector<Scalar> apply(const std::vector<Scalar>& x) const {
    if (static_cast<std::int64_t>(x.size()) != dim()) throw ShapeError("block-diagonal apply: dimension mismatch");
    std::vector<Scalar> y(x.size(), Scalar(0));
    for (std::int64_t i = 0; i < num_blocks_; ++i)
      for (int r = 0; r < BS; ++r) {
        Scalar acc = Scalar(0);
        for (int c = 0; c < BS; ++c) acc += block(i)(r, c) * x[static_cast<std::size_t>(i * BS + c)];
        y[static_cast<std::size_t>(i * BS + r)] = acc;
      }
    return y;
  }
  // damped copy (dba/block_matrix.hpp:86-99); the undamped blocks stay
  void damp_into(Scalar lambda, DampingPolicy policy, BlockDiagonal& out) const {
    out.num_blocks_ = num_blocks_;
    out.data_ = data_;
    for (std::int64_t i = 0; i < num_blocks_; ++i)
      for (int j = 0; j < BS; ++j) {
        Scalar& d = out.block(i)(j, j);
        d += policy == DampingPolicy::identity ? lambda : lambda * clamped_curvature(d);
      }
  }
  std::vector<Scalar> diagonal() const {
    std::vector<Scalar> d(static_cast<std::size_t>(dim()));
    for (std::int64_t i = 0; i < num_blocks_; ++i)
      for (int j = 0; j < BS; ++j) d[static_cast<std::size_t>(i * BS + j)] = block(i)(j, j);
    return d;
  }

 private:
  std::int64_t num_blocks_ = 0;
  std::vector<Scalar> data_;
};

// FactoredBlockDiagonal<Scalar, BS> (dba/block_matrix.hpp:118-167): the LLT
// of every block, computed on the device (pivot <= 0 fails, lowest block
// first: SingularBlockError(i, BS)); solve_in_place runs the substitutions on
// the device. Keeps the factored blocks for the operators that factor on
// their own context (dse, dpcg).
template <typename Scalar, int BS>
class FactoredBlockDiagonal {
 public:
  FactoredBlockDiagonal() = default;
  explicit FactoredBlockDiagonal(int device) : device_(device) {}
  void factor(const BlockDiagonal<Scalar, BS>& d) {
    source_ = d;
    factor_.assign(d.data().size(), Scalar(0));
    std::int64_t bad = -1;
    detail::check(dbag_block_factor(device_, detail::prec<Scalar>(), BS, d.blocks(), d.data().data(), factor_.data(),
                                    &bad));
  }
  std::int64_t blocks() const { return source_.blocks(); }
  std::int64_t dim() const { return source_.dim(); }
  void solve_in_place(std::vector<Scalar>& x) const {
    if (static_cast<std::int64_t>(x.size()) != dim()) throw ShapeError("block-diagonal solve: dimension mismatch");
    detail::check(dbag_block_solve(device_, detail::prec<Scalar>(), BS, blocks(), factor_.data(), x.data()));
  }
  std::vector<Scalar> solve(const std::vector<Scalar>& x) const {
    std::vector<Scalar> y = x;
    solve_in_place(y);
    return y;
  }
  const BlockDiagonal<Scalar, BS>& source() const { return source_; }

 private:
  int device_ = 0;
  BlockDiagonal<Scalar, BS> source_;
  std::vector<Scalar> factor_;
};

// ---- EdgeBlockMatrix (dba/block_matrix.hpp:169-333) --------------------------------
// One 9x3 row-major block per partition edge, in partition edge order, with
// the global camera / point of each block. The operators run on the rank's
// context of the WorkerGroup they are called with (created on first use:
// the rank's shard of the problem on its device).
template <typename Scalar>
class EdgeBlockMatrix {
 public:
  EdgeBlockMatrix() = default;
  EdgeBlockMatrix(const BAProblem<Scalar>& problem, const EdgePartition& partition)
      : problem_(&problem),
        partition_(partition),
        num_cameras_(problem.num_cameras()),
        num_points_(problem.num_points()) {
    const std::size_t n = partition.edge_ids.size();
    cam_of_block_.resize(n);
    pt_of_block_.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      const auto o = problem.observation(partition.edge_ids[i]);
      cam_of_block_[i] = o.camera_id;
      pt_of_block_[i] = o.point_id;
    }
    blocks_.assign(n * kCameraParams * kPointParams, Scalar(0));
  }
  EdgeBlockMatrix(EdgeBlockMatrix&& o) noexcept { *this = std::move(o); }
  EdgeBlockMatrix& operator=(EdgeBlockMatrix&& o) noexcept {
    problem_ = o.problem_;
    partition_ = std::move(o.partition_);
    num_cameras_ = o.num_cameras_;
    num_points_ = o.num_points_;
    cam_of_block_ = std::move(o.cam_of_block_);
    pt_of_block_ = std::move(o.pt_of_block_);
    blocks_ = std::move(o.blocks_);
    ctx_ = std::move(o.ctx_);
    return *this;
  }

  std::int64_t blocks() const { return static_cast<std::int64_t>(cam_of_block_.size()); }
  std::int64_t camera_dim() const { return std::int64_t{num_cameras_} * kCameraParams; }
  std::int64_t point_dim() const { return std::int64_t{num_points_} * kPointParams; }
  BlockRef<Scalar, 3> block(std::int64_t i) {  // b(r, c), r < 9, c < 3
    return {blocks_.data() + static_cast<std::size_t>(i) * 27};
  }
  BlockRef<const Scalar, 3> block(std::int64_t i) const { return {blocks_.data() + static_cast<std::size_t>(i) * 27}; }
  std::int32_t camera_of_block(std::int64_t i) const { return cam_of_block_[static_cast<std::size_t>(i)]; }
  std::int32_t point_of_block(std::int64_t i) const { return pt_of_block_[static_cast<std::size_t>(i)]; }
  void set_zero() { std::fill(blocks_.begin(), blocks_.end(), Scalar(0)); }
  std::vector<Scalar>& data() { return blocks_; }
  const std::vector<Scalar>& data() const { return blocks_; }
  const EdgePartition& partition() const { return partition_; }

  // The rank's context in `group` with this system uploaded: B (damped),
  // the source blocks of C^-1 and these E blocks; damped with lambda 0, so the
  // context's operators use exactly B and C.
  dbag_ctx* system(WorkerGroup& group, int rank, const BlockDiagonal<Scalar, kCameraParams>& B,
                   const BlockDiagonal<Scalar, kPointParams>& C) const {
    if (!problem_) throw InvalidArgumentError("EdgeBlockMatrix without a problem");
    if (partition_.worker_count != group.workers() || partition_.worker_rank != rank)
      throw InvalidArgumentError("EdgeBlockMatrix partition " + std::to_string(partition_.worker_rank) + "/" +
                                 std::to_string(partition_.worker_count) + " used as rank " + std::to_string(rank) +
                                 " of " + std::to_string(group.workers()));
    if (B.blocks() != num_cameras_ || C.blocks() != num_points_) throw ShapeError("dse: block count mismatch");
    std::shared_ptr<Slot> slot;
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto& s = ctx_[&group];
      if (!s) {
        dbag_ctx* raw = nullptr;
        detail::check(dbag_create_group_rank(group.handle(), rank, detail::prec<Scalar>(), 0, &raw));
        s = std::make_shared<Slot>();
        s->ctx = std::make_unique<detail::Ctx>(raw);
      }
      slot = s;
    }
    dbag_ctx* c = slot->ctx->c;
    if (!slot->uploaded) {  // collective: every rank uploads its shard
      const dbag_problem p = problem_->c_view();
      detail::check(dbag_upload_problem(c, &p, 0));
      slot->uploaded = true;
    }
    // E in global edge order (the context reads its shard's edges)
    std::vector<Scalar> table(static_cast<std::size_t>(problem_->num_observations()) * 27, Scalar(0));
    for (std::size_t i = 0; i < partition_.edge_ids.size(); ++i)
      std::copy(blocks_.begin() + static_cast<std::ptrdiff_t>(i * 27),
                blocks_.begin() + static_cast<std::ptrdiff_t>(i * 27 + 27),
                table.begin() + static_cast<std::ptrdiff_t>(partition_.edge_ids[i]) * 27);
    detail::check(dbag_set_system(c, B.data().data(), C.data().data(), table.data(), nullptr, nullptr));
    std::int64_t bad = -1;
    int bs = 0;
    detail::check(dbag_damp_factor(c, 0.0, 0, &bad, &bs));
    return c;
  }

 private:
  const BAProblem<Scalar>* problem_ = nullptr;
  EdgePartition partition_;
  std::int32_t num_cameras_ = 0, num_points_ = 0;
  std::vector<std::int32_t> cam_of_block_, pt_of_block_;
  std::vector<Scalar> blocks_;
  struct Slot {
    std::unique_ptr<detail::Ctx> ctx;
    bool uploaded = false;
  };
  mutable std::mutex mu_;
  mutable std::map<const WorkerGroup*, std::shared_ptr<Slot>> ctx_;
};

// ---- the reduced camera operator (dba/solver.hpp:134-257) --------------------------
template <typename Scalar>
struct DseWorkspace {};  // device buffers live in the rank's context
template <typename Scalar>
struct PcgWorkspace {
  DseWorkspace<Scalar> dse_ws;
};
struct PcgResult {
  int iterations = 0;
  bool converged = false;
};

// dse (dba/solver.hpp:149-181): out = (B - E C^-1 E^T) x over the group's
// ranks (a = E_k^T x all-reduced, b = C^-1 a, c = E_k b all-reduced,
// out = B x - c). Collective; rank-identical.
template <typename Scalar>
void dse(const std::vector<Scalar>& x, const BlockDiagonal<Scalar, kCameraParams>& B, const EdgeBlockMatrix<Scalar>& E,
         const FactoredBlockDiagonal<Scalar, kPointParams>& C_inv, WorkerGroup& group, int rank,
         std::vector<Scalar>& out, DseWorkspace<Scalar>&, WorkCounters* counters = nullptr) {
  if (static_cast<std::int64_t>(x.size()) != E.camera_dim()) throw ShapeError("dse: dimension mismatch");
  dbag_ctx* c = E.system(group, rank, B, C_inv.source());
  out.resize(x.size());
  detail::check(dbag_dse(c, x.data(), out.data()));
  if (counters) counters->edge_block_ops += 2 * static_cast<std::uint64_t>(E.blocks());
}

template <typename Scalar>
std::vector<Scalar> dse(const std::vector<Scalar>& x, const BlockDiagonal<Scalar, kCameraParams>& B,
                        const EdgeBlockMatrix<Scalar>& E, const FactoredBlockDiagonal<Scalar, kPointParams>& C_inv,
                        WorkerGroup& group, int rank) {
  std::vector<Scalar> out;
  DseWorkspace<Scalar> ws;
  dse(x, B, E, C_inv, group, rank, out, ws);
  return out;
}

// dpcg (dba/solver.hpp:202-257): block-Jacobi PCG on the reduced camera
// system from x (the device solve starts at 0: a nonzero x solves for the
// correction of rhs - S x). B_inv is the factor of B_damped, as in the
// reference; the device refactors B_damped on the rank's context.
// Throws PcgBreakdownError on a rho / p'q breakdown.
template <typename Scalar>
PcgResult dpcg(std::vector<Scalar>& x, const BlockDiagonal<Scalar, kCameraParams>& B_damped,
               const FactoredBlockDiagonal<Scalar, kCameraParams>& B_inv, const EdgeBlockMatrix<Scalar>& E,
               const FactoredBlockDiagonal<Scalar, kPointParams>& C_inv, const std::vector<Scalar>& rhs,
               WorkerGroup& group, int rank, double tol, int max_iters, PcgWorkspace<Scalar>& ws,
               WorkCounters* counters = nullptr) {
  (void)B_inv;
  if (static_cast<std::int64_t>(rhs.size()) != E.camera_dim()) throw ShapeError("dpcg: dimension mismatch");
  x.resize(rhs.size(), Scalar(0));
  std::vector<Scalar> b = rhs;
  const bool warm = std::any_of(x.begin(), x.end(), [](Scalar v) { return v != Scalar(0); });
  dbag_ctx* c = E.system(group, rank, B_damped, C_inv.source());
  if (warm) {
    std::vector<Scalar> sx(x.size());
    detail::check(dbag_dse(c, x.data(), sx.data()));
    for (std::size_t i = 0; i < b.size(); ++i) b[i] -= sx[i];
  }
  std::vector<Scalar> d(x.size());
  int it = 0, conv = 0;
  detail::check(dbag_dpcg(c, b.data(), tol, max_iters, d.data(), &it, &conv));
  for (std::size_t i = 0; i < x.size(); ++i) x[i] = warm ? x[i] + d[i] : d[i];
  (void)ws;
  if (counters) counters->edge_block_ops += 2 * static_cast<std::uint64_t>(E.blocks()) * (1 + it + it / 50);
  return {it, conv != 0};
}

// ---- edge evaluation (dba/edge_eval.hpp:21-309) -------------------------------------
// EdgeJacobianBatch: per partition edge the residual r (2) and J = [Jc | Jp]
// (2 x 12), in partition edge order.
template <typename Scalar>
class EdgeJacobianBatch {
 public:
  std::int64_t size() const { return n_; }
  std::array<Scalar, 2> residual(std::int64_t i) const {
    return {res_[static_cast<std::size_t>(i)], res_[static_cast<std::size_t>(n_ + i)]};
  }
  // row r, column c of the 2 x 12 Jacobian (c < 9 camera, 9..11 point)
  Scalar jacobian(int r, int c, std::int64_t i) const {
    return jac_[(static_cast<std::size_t>(r) * 12 + static_cast<std::size_t>(c)) * static_cast<std::size_t>(n_) +
                static_cast<std::size_t>(i)];
  }
  std::array<std::array<Scalar, kCameraParams>, 2> camera_jacobian(std::int64_t i) const {
    std::array<std::array<Scalar, kCameraParams>, 2> j{};
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < kCameraParams; ++c) j[r][c] = jacobian(r, c, i);
    return j;
  }
  std::array<std::array<Scalar, kPointParams>, 2> point_jacobian(std::int64_t i) const {
    std::array<std::array<Scalar, kPointParams>, 2> j{};
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < kPointParams; ++c) j[r][c] = jacobian(r, kCameraParams + c, i);
    return j;
  }
  bool all_finite() const {
    for (Scalar v : res_)
      if (!std::isfinite(double(v))) return false;
    for (Scalar v : jac_)
      if (!std::isfinite(double(v))) return false;
    return true;
  }

 private:
  template <typename>
  friend class EdgeEvaluator;
  std::int64_t n_ = 0;
  std::vector<Scalar> res_, jac_;
};

// EdgeEvaluator (dba/edge_eval.hpp:75-309): the partition's edges on a shard
// context with local collectives (device `device`). linearize returns a
// reference valid until the next call; cost is the partition's own sum of
// w |r|^2 in double and throws DegenerateDepthError(global edge id).
template <typename Scalar>
class EdgeEvaluator {
 public:
  EdgeEvaluator(const BAProblem<Scalar>& problem, const EdgePartition& partition,
                JacobianMode mode = JacobianMode::autodiff, int device = 0)
      : problem_(&problem), partition_(partition), mode_(mode) {
    const std::size_t n = partition.edge_ids.size();
    for (std::size_t i = 0; i < n; ++i) {
      const auto o = problem.observation(partition.edge_ids[i]);
      cam_ids_.push_back(o.camera_id);
      pt_ids_.push_back(o.point_id);
      weights_.push_back(o.weight);
    }
    dbag_ctx* raw = nullptr;
    detail::check(dbag_create_shard(device, detail::prec<Scalar>(), 0, partition.worker_rank, partition.worker_count,
                                    &raw));
    ctx_ = std::make_shared<detail::Ctx>(raw);
    const dbag_problem p = problem.c_view();
    detail::check(dbag_upload_problem(raw, &p, mode == JacobianMode::analytic ? 1 : 0));
  }
  std::int64_t num_edges() const { return static_cast<std::int64_t>(cam_ids_.size()); }
  const std::vector<Scalar>& weights() const { return weights_; }
  const std::vector<std::int32_t>& camera_ids() const { return cam_ids_; }
  const std::vector<std::int32_t>& point_ids() const { return pt_ids_; }
  JacobianMode mode() const { return mode_; }

  const EdgeJacobianBatch<Scalar>& linearize(const std::vector<Scalar>& x_c, const std::vector<Scalar>& x_p,
                                             WorkCounters* counters = nullptr) {
    set_state(x_c, x_p);
    std::int64_t bad = -1;
    detail::check(dbag_linearize(ctx_->c, &bad));
    batch_.n_ = num_edges();
    batch_.res_.assign(static_cast<std::size_t>(2 * batch_.n_), Scalar(0));
    batch_.jac_.assign(static_cast<std::size_t>(24 * batch_.n_), Scalar(0));
    detail::check(dbag_get_jacobians(ctx_->c, batch_.res_.data(), batch_.jac_.data()));
    linearized_ = true;
    if (counters) counters->edges_evaluated += static_cast<std::uint64_t>(num_edges());
    return batch_;
  }

  double cost(const std::vector<Scalar>& x_c, const std::vector<Scalar>& x_p, WorkCounters* counters = nullptr) const {
    set_state(x_c, x_p);
    double c = 0;
    std::int64_t bad = -1;
    detail::check(dbag_cost(ctx_->c, 0, &c, &bad));
    if (bad >= 0) throw DegenerateDepthError(bad);
    if (counters) counters->edges_evaluated += static_cast<std::uint64_t>(num_edges());
    return c;
  }

  // the partition's assembled system of the last linearize (assemble_local)
  bool linearized() const { return linearized_; }
  dbag_ctx* context() const { return ctx_->c; }
  const EdgePartition& partition() const { return partition_; }

 private:
  void set_state(const std::vector<Scalar>& x_c, const std::vector<Scalar>& x_p) const {
    if (x_c.size() != problem_->packed_cameras().size() || x_p.size() != problem_->packed_points().size())
      throw ShapeError("evaluator: state dimension mismatch");
    detail::check(dbag_set_state(ctx_->c, x_c.data(), x_p.data()));
  }
  const BAProblem<Scalar>* problem_;
  EdgePartition partition_;
  JacobianMode mode_;
  std::vector<std::int32_t> cam_ids_, pt_ids_;
  std::vector<Scalar> weights_;
  std::shared_ptr<detail::Ctx> ctx_;
  EdgeJacobianBatch<Scalar> batch_;
  bool linearized_ = false;
};

// ---- assembly (dba/block_matrix.hpp:335-400) -----------------------------------------
template <typename Scalar>
struct PartitionedHessian {
  BlockDiagonal<Scalar, kCameraParams> B;
  BlockDiagonal<Scalar, kPointParams> C;
  EdgeBlockMatrix<Scalar> E;
  std::vector<Scalar> v, w;
  PartitionedHessian() = default;
  PartitionedHessian(const BAProblem<Scalar>& problem, const EdgePartition& partition)
      : B(problem.num_cameras()),
        C(problem.num_points()),
        E(problem, partition),
        v(static_cast<std::size_t>(problem.num_cameras()) * kCameraParams, Scalar(0)),
        w(static_cast<std::size_t>(problem.num_points()) * kPointParams, Scalar(0)) {}
};

// assemble_local (dba/block_matrix.hpp:358-388): the partition's B_k, C_k,
// E_k, v_k, w_k from the evaluator's last linearization (assembled on the
// device with the linearization; downloaded here).
template <typename Scalar>
void assemble_local(const EdgeJacobianBatch<Scalar>& batch, const EdgeEvaluator<Scalar>& evaluator,
                    PartitionedHessian<Scalar>& out) {
  if (!evaluator.linearized() || batch.size() != evaluator.num_edges())
    throw ShapeError("assemble: batch does not match partition");
  if (out.E.blocks() != evaluator.num_edges()) throw ShapeError("assemble: hessian does not match partition");
  detail::check(dbag_get_system(evaluator.context(), out.B.data().data(), out.C.data().data(), out.E.data().data(),
                                out.v.data(), out.w.data()));
}

template <typename Scalar>
PartitionedHessian<Scalar> assemble_local(const BAProblem<Scalar>& problem, const EdgePartition& partition,
                                          const std::vector<Scalar>& x_c, const std::vector<Scalar>& x_p) {
  EdgeEvaluator<Scalar> evaluator(problem, partition);
  PartitionedHessian<Scalar> h(problem, partition);
  assemble_local(evaluator.linearize(x_c, x_p), evaluator, h);
  return h;
}

// ---- costs (dba/problem.hpp:266-290) -------------------------------------------------
template <typename Scalar>
std::vector<Scalar> pack_cameras(const BAProblem<Scalar>& p) {
  return p.packed_cameras();
}
template <typename Scalar>
std::vector<Scalar> pack_points(const BAProblem<Scalar>& p) {
  return p.packed_points();
}

// total_cost: sum of w |r|^2 over every edge in edge order (double), on the
// device; DegenerateDepthError(edge) when an edge's depth is zero.
template <typename Scalar>
double total_cost(const BAProblem<Scalar>& problem) {
  const auto parts = partition_edges(problem, 1);
  EdgeEvaluator<Scalar> ev(problem, parts[0]);
  return ev.cost(problem.packed_cameras(), problem.packed_points());
}

template <typename Scalar>
double mean_squared_error(const BAProblem<Scalar>& problem,
                          MseConvention convention = MseConvention::half_per_observation) {
  const std::int64_t n = problem.num_observations();
  if (n <= 0) return 0.0;
  const double c = total_cost(problem);
  return convention == MseConvention::half_per_observation ? c / (2.0 * double(n)) : c / double(n);
}

// ---- LM control (dba/solver.hpp:86-104, 295-518) -------------------------------------
enum class ConvergenceDecision { keep_going, converged, max_iterations, stalled };

template <typename Scalar>
ConvergenceDecision check_convergence(const SolverState<Scalar>& state, const SolverConfig& config) {
  if (state.last_accepted) {
    const double denom = std::max(state.previous_cost, 1e-300);
    if (std::abs(state.last_cost_change) / denom < config.rel_tol || state.last_step_inf < config.step_tol)
      return ConvergenceDecision::converged;
  }
  if (state.lambda > config.lambda_max) return ConvergenceDecision::stalled;
  if (state.iteration >= config.max_iterations) return ConvergenceDecision::max_iterations;
  return ConvergenceDecision::keep_going;
}

// lm_solve_rank: this rank's body of the distributed LM loop over the group
// (call inside run_on_workers; every rank returns the full, rank-identical
// state).
template <typename Scalar>
SolverState<Scalar> lm_solve_rank(const BAProblem<Scalar>& problem, const SolverConfig& config,
                                  const EdgePartition& partition, WorkerGroup& group, int rank) {
  if (config.workers != group.workers() || partition.worker_count != group.workers() || partition.worker_rank != rank)
    throw InvalidArgumentError("lm_solve_rank: partition / config do not match the group rank");
  dbag_ctx* raw = nullptr;
  detail::check(dbag_create_group_rank(group.handle(), rank, detail::prec<Scalar>(), config.coupling_fp32 ? 1 : 0, &raw));
  detail::Ctx ctx(raw);
  const dbag_problem p = problem.c_view();
  detail::check(dbag_upload_problem(raw, &p, config.jacobian == JacobianMode::analytic ? 1 : 0));
  const dbag_config c = config.c_view();
  return detail::solve_into<Scalar>(problem.packed_cameras().size(), problem.packed_points().size(),
                                    config.max_iterations, group.workers(),
                                    [&](dbag_result& r) { detail::check(dbag_lm_solve_ctx(raw, &c, &r)); });
}

}  // namespace dba
