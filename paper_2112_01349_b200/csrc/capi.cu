// capi.cu — the extern "C" boundary (include/dbag.h).
//
// Status codes carry the reference's exception types across the ABI
// (dba/errors.hpp); every entry point catches, records the message and the
// payload (edge id / block index + size) in thread-local storage, and
// returns the code.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "common.hpp"
#include "bal.hpp"
#include "partition.hpp"
#include "rank.cuh"
#include "solver.cuh"

namespace dbag {
std::int64_t synthetic_count(const dbag_synthetic_options& o);
void generate_synthetic(const dbag_synthetic_options& o, double* cams, double* pts, std::int32_t* cam_id,
                        std::int32_t* pt_id, double* pix_x, double* pix_y);
}  // namespace dbag

using namespace dbag;

struct dbag_ctx {
  int precision = 8;
  std::unique_ptr<Comm> comm;
  std::unique_ptr<Rank<float>> r32;
  std::unique_ptr<Rank<double>> r64;
  std::unique_ptr<Rank<double, float>> r64l;  // FP64 arithmetic, FP32 coupling blocks (coupling_fp32)
  std::int64_t num_obs = 0;
  bool cost_valid = false;
  double cost = 0;
};

namespace {

thread_local std::string g_err;
thread_local std::int64_t g_err_index = -1;
thread_local int g_err_bs = 0;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return DBAG_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_index = e.index;
    g_err_bs = e.block_size;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_index = -1;
    g_err_bs = 0;
    return DBAG_INTERNAL;
  }
}

void check_precision(int p) {
  if (p != 4 && p != 8) throw Error(DBAG_INVALID_ARGUMENT, "precision must be 4 or 8");
}

void check_ctx(dbag_ctx* c) {
  if (!c || (!c->r32 && !c->r64 && !c->r64l)) throw Error(DBAG_INVALID_ARGUMENT, "null or empty context");
}

// Calls fn(Rank<S, T>&) on the context's typed rank.
template <class Fn>
void with_rank(dbag_ctx* c, Fn&& fn) {
  check_ctx(c);
  if (c->r64) fn(*c->r64);
  else if (c->r64l) fn(*c->r64l);
  else fn(*c->r32);
}

std::chrono::milliseconds timeout_of(const dbag_config& c) {
  return std::chrono::milliseconds(c.collective_timeout_ms > 0 ? c.collective_timeout_ms : 60000);
}

void fill_result(const Outcome& o, int K, dbag_result* out) {
  out->iterations = o.iteration;
  out->termination = o.termination;
  out->cost = o.cost;
  out->lambda = o.lambda;
  out->nu = o.nu;
  out->workers = K;
  out->last_accepted = o.last_accepted ? 1 : 0;
  out->last_cost_change = o.last_cost_change;
  out->last_step_inf = o.last_step_inf;
  out->previous_cost = o.previous_cost;
  const int n = std::min<int>(out->capacity, static_cast<int>(o.history.size()));
  for (int i = 0; i < n; ++i) {
    const Record& r = o.history[static_cast<std::size_t>(i)];
    if (out->rec_iteration) out->rec_iteration[i] = r.iteration;
    if (out->rec_cost) out->rec_cost[i] = r.cost;
    if (out->rec_mse) out->rec_mse[i] = r.mse;
    if (out->rec_lambda) out->rec_lambda[i] = r.lambda;
    if (out->rec_pcg) out->rec_pcg[i] = r.pcg_iterations;
    if (out->rec_accepted) out->rec_accepted[i] = r.accepted ? 1 : 0;
    if (out->rec_wall) out->rec_wall[i] = r.wall_seconds;
    for (int k = 0; k < K; ++k) {
      const std::size_t at = static_cast<std::size_t>(i) * K + k;
      if (out->rec_worker_edges) out->rec_worker_edges[at] = r.worker_edges[static_cast<std::size_t>(k)];
      if (out->rec_worker_block_ops) out->rec_worker_block_ops[at] = r.worker_block_ops[static_cast<std::size_t>(k)];
    }
  }
}

// Runs body(rank) on one host thread per rank (run_on_workers,
// dba/comms.hpp:214-234): the first failure aborts the group and is
// rethrown after every thread joined.
template <class Fn>
void run_ranks(Group& g, Fn&& body) {
  std::vector<std::thread> th;
  std::exception_ptr first;
  std::mutex mu;
  for (int r = 0; r < g.size(); ++r) {
    th.emplace_back([&, r] {
      try {
        DBAG_CUDA(cudaSetDevice(g.device_of(r)));
        body(r);
      } catch (const std::exception& e) {
        {
          std::lock_guard<std::mutex> lk(mu);
          if (!first) first = std::current_exception();
        }
        g.abort(std::string("rank ") + std::to_string(r) + " failed: " + e.what());
      }
    });
  }
  for (auto& t : th) t.join();
  if (first) std::rethrow_exception(first);
}

template <class S, class T = S>
void lm_group(const dbag_problem* p, const dbag_config* c, const int* devices, int n_devices, dbag_result* out) {
  const int K = c->workers;
  std::vector<int> devs(devices, devices + std::max(n_devices, 0));
  if (devs.empty()) devs.push_back(0);
  split_edges(p->num_observations, K);  // validates K like partition_edges
  Group g(K, devs, timeout_of(*c));
  run_ranks(g, [&](int r) {
    GroupComm comm(&g, r);
    Rank<S, T> rk(g.device_of(r), &comm);
    rk.upload(*p, c->jacobian);
    const Outcome o = lm_solve_rank(rk, *c, p->num_observations);
    // rank 0's state (dba/solver.hpp:533), x_p assembled over the group
    rk.gather_state(r == 0 ? static_cast<S*>(out->x_c) : nullptr, r == 0 ? static_cast<S*>(out->x_p) : nullptr);
    if (r == 0) fill_result(o, K, out);
  });
}

template <class S, class T = S>
void lm_nccl(const dbag_problem* p, const dbag_config* c, int rank, int nranks, const unsigned char* id, int device,
             dbag_result* out) {
  DBAG_CUDA(cudaSetDevice(device));
  if (c->workers != nranks) throw Error(DBAG_INVALID_ARGUMENT, "config.workers must equal nranks");
  NcclComm comm(rank, nranks, id);
  comm.set_timeout(timeout_of(*c));
  Rank<S, T> rk(device, &comm);
  rk.upload(*p, c->jacobian);
  const Outcome o = lm_solve_rank(rk, *c, p->num_observations);
  // Every rank returns the full, rank-identical state (dba/solver.hpp:533):
  // cameras are replicated; x_p is assembled over the communicator from
  // each point's owner (Rank::gather_state).
  rk.gather_state(static_cast<S*>(out->x_c), static_cast<S*>(out->x_p));
  fill_result(o, nranks, out);
}

template <class S>
void group_operator(const dbag_problem* p, int k, int device, double lambda, int policy, const void* B,
                    const void* C, const void* E, int mode, const void* x, double tol, int max_iters, void* out,
                    int* iterations, int* rank_identical) {
  split_edges(p->num_observations, k);
  Group g(k, {device});
  const std::size_t len = static_cast<std::size_t>(p->num_cameras) * 9;
  std::vector<std::vector<S>> outs(static_cast<std::size_t>(k), std::vector<S>(len));
  std::vector<int> its(static_cast<std::size_t>(k), 0);
  run_ranks(g, [&](int r) {
    GroupComm comm(&g, r);
    Rank<S> rk(device, &comm);
    rk.upload(*p, 0);
    if (B) {
      rk.set_system(static_cast<const S*>(B), static_cast<const S*>(C), static_cast<const S*>(E), nullptr, nullptr);
      rk.factor_as_is();
    } else {
      rk.linearize();
      rk.damp_factor(lambda, policy);
    }
    if (mode == 0) {
      rk.dse_host(static_cast<const S*>(x), outs[static_cast<std::size_t>(r)].data());
    } else if (mode >= 2) {  // diagnostics of one LM trial's pieces
      S* o = outs[static_cast<std::size_t>(r)].data();
      rk.trial_probe(mode, tol, max_iters, o);
    } else {
      its[static_cast<std::size_t>(r)] =
          rk.dpcg_host(static_cast<const S*>(x), tol, max_iters, outs[static_cast<std::size_t>(r)].data()).iterations;
    }
  });
  *rank_identical = 1;
  for (int r = 1; r < k; ++r)
    if (std::memcmp(outs[static_cast<std::size_t>(r)].data(), outs[0].data(), len * sizeof(S)) != 0) *rank_identical = 0;
  std::memcpy(out, outs[0].data(), len * sizeof(S));
  if (iterations) *iterations = its[0];
}

}  // namespace

extern "C" {

int dbag_version(void) { return 1; }
const char* dbag_last_error(void) { return g_err.c_str(); }
int64_t dbag_last_error_index(void) { return g_err_index; }
int dbag_last_error_block_size(void) { return g_err_bs; }

void dbag_default_config(dbag_config* c) {  // dba/solver.hpp:39-55
  std::memset(c, 0, sizeof(*c));
  c->workers = 1;
  c->max_iterations = 50;
  c->pcg_tol = 1e-6;
  c->pcg_max_iters = 500;
  c->lambda0 = 1e-4;
  c->lambda_max = 1e32;
  c->rel_tol = 1e-6;
  c->step_tol = 1e-8;
  c->damping = 1;
  c->mse_half = 1;
  c->jacobian = 0;
  c->check_rank_identity = 0;
  c->collective_timeout_ms = 60000;
}

int dbag_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    *out = e == cudaSuccess ? n : 0;
    (void)cudaGetLastError();
  });
}

int dbag_partition(const dbag_problem* p, int k, int rank, int64_t* start, int64_t* count, int32_t* n_cams,
                   int32_t* cam_g, int32_t* n_pts, int32_t* pt_g, int64_t* cam_ptr, int64_t* cam_blk, int64_t* pt_ptr,
                   int64_t* pt_blk) {
  return guarded([&] {
    const ShardPlan s = plan_shard(p->camera_id, p->point_id, p->num_observations, p->num_cameras, p->num_points, k,
                                   rank);
    *start = s.range.start;
    *count = s.range.count;
    *n_cams = s.cams.size();
    *n_pts = s.pts.size();
    std::copy(s.cams.to_global.begin(), s.cams.to_global.end(), cam_g);
    std::copy(s.pts.to_global.begin(), s.pts.to_global.end(), pt_g);
    std::copy(s.cam_ptr.begin(), s.cam_ptr.end(), cam_ptr);
    std::copy(s.cam_blk.begin(), s.cam_blk.end(), cam_blk);
    std::copy(s.pt_ptr.begin(), s.pt_ptr.end(), pt_ptr);
    std::copy(s.pt_blk.begin(), s.pt_blk.end(), pt_blk);
  });
}

int dbag_shared_points(const dbag_problem* p, int k, int64_t* n_shared, int32_t* ids) {
  return guarded([&] {
    const auto ranges = split_edges(p->num_observations, k);
    const Coverage cov = point_coverage(p->point_id, p->num_points, ranges);
    *n_shared = cov.n_shared;
    if (ids)
      for (std::int32_t q = 0; q < p->num_points; ++q)
        if (cov.shared_index[static_cast<std::size_t>(q)] >= 0) ids[cov.shared_index[static_cast<std::size_t>(q)]] = q;
  });
}

int dbag_predict_memory(const dbag_problem* p, int precision, int coupling_fp32, int k, int rank, uint64_t* bytes) {
  return guarded([&] {
    check_precision(precision);
    check_problem(*p);
    const ShardPlan s = plan_shard(p->camera_id, p->point_id, p->num_observations, p->num_cameras, p->num_points, k,
                                   rank, dev::kTile);
    const DeviceLayout d = build_device_layout(s, p->camera_id + s.range.start, dev::kTile);
    if (precision == 8 && coupling_fp32) *bytes = Rank<double, float>::predict_bytes(Rank<double, float>::shard_sizes(s, d));
    else if (precision == 8) *bytes = Rank<double>::predict_bytes(Rank<double>::shard_sizes(s, d));
    else *bytes = Rank<float>::predict_bytes(Rank<float>::shard_sizes(s, d));
  });
}

int dbag_memory_pool(dbag_ctx* ctx, uint64_t* reserved, uint64_t* used) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      *reserved = rk.pool_bytes();
      *used = rk.pool_used();
    });
  });
}

int dbag_synthetic_count(const dbag_synthetic_options* o, int64_t* n_obs) {
  return guarded([&] { *n_obs = synthetic_count(*o); });
}

int dbag_generate_synthetic(const dbag_synthetic_options* o, double* cameras, double* points, int32_t* camera_id,
                            int32_t* point_id, double* pixel_x, double* pixel_y) {
  return guarded([&] { generate_synthetic(*o, cameras, points, camera_id, point_id, pixel_x, pixel_y); });
}

struct dbag_bal {
  dbag::BalData d;
};

int dbag_bal_parse(const char* text, int64_t len, dbag_bal** out) {
  return guarded([&] {
    if (!out || (!text && len > 0) || len < 0) throw Error(DBAG_INVALID_ARGUMENT, "dbag_bal_parse: bad arguments");
    auto b = std::make_unique<dbag_bal>();
    b->d = dbag::parse_bal_text(text, static_cast<std::size_t>(len));
    *out = b.release();
  });
}

int dbag_bal_counts(const dbag_bal* b, int32_t* m, int32_t* n, int64_t* N) {
  return guarded([&] {
    if (!b) throw Error(DBAG_INVALID_ARGUMENT, "dbag_bal_counts: null handle");
    *m = b->d.m;
    *n = b->d.n;
    *N = b->d.N;
  });
}

int dbag_bal_copy(const dbag_bal* b, double* cameras, double* points, int32_t* camera_id, int32_t* point_id,
                  double* pixel_x, double* pixel_y) {
  return guarded([&] {
    if (!b) throw Error(DBAG_INVALID_ARGUMENT, "dbag_bal_copy: null handle");
    const auto& d = b->d;
    std::copy(d.cameras.begin(), d.cameras.end(), cameras);
    std::copy(d.points.begin(), d.points.end(), points);
    std::copy(d.cam.begin(), d.cam.end(), camera_id);
    std::copy(d.pt.begin(), d.pt.end(), point_id);
    std::copy(d.px.begin(), d.px.end(), pixel_x);
    std::copy(d.py.begin(), d.py.end(), pixel_y);
  });
}

int dbag_bal_free(dbag_bal* b) {
  return guarded([&] { delete b; });
}

int dbag_bal_format(int precision, const dbag_problem* p, char** text, int64_t* len) {
  return guarded([&] {
    if (!p || !text || !len) throw Error(DBAG_INVALID_ARGUMENT, "dbag_bal_format: bad arguments");
    std::string s;
    if (precision == 8)
      s = dbag::format_bal(p->num_cameras, p->num_points, p->num_observations, static_cast<const double*>(p->cameras),
                           static_cast<const double*>(p->points), p->camera_id, p->point_id,
                           static_cast<const double*>(p->pixel_x), static_cast<const double*>(p->pixel_y));
    else if (precision == 4)
      s = dbag::format_bal(p->num_cameras, p->num_points, p->num_observations, static_cast<const float*>(p->cameras),
                           static_cast<const float*>(p->points), p->camera_id, p->point_id,
                           static_cast<const float*>(p->pixel_x), static_cast<const float*>(p->pixel_y));
    else
      throw Error(DBAG_INVALID_ARGUMENT, "precision must be 4 or 8");
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    if (!buf) throw Error(DBAG_INTERNAL, "out of host memory");
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
    *text = buf;
    *len = static_cast<int64_t>(s.size());
  });
}

int dbag_free_text(char* text) {
  std::free(text);
  return DBAG_OK;
}

int dbag_lm_solve(int precision, const dbag_problem* p, const dbag_config* c, const int* devices, int n_devices,
                  dbag_result* out) {
  return guarded([&] {
    check_precision(precision);
    if (precision == 8 && c->coupling_fp32) lm_group<double, float>(p, c, devices, n_devices, out);
    else if (precision == 8) lm_group<double>(p, c, devices, n_devices, out);
    else lm_group<float>(p, c, devices, n_devices, out);
  });
}

int dbag_nccl_unique_id(unsigned char* out128) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw Error(DBAG_NCCL_ERROR, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, id.internal, 128);
  });
}

int dbag_lm_solve_rank(int precision, const dbag_problem* p, const dbag_config* c, int rank, int nranks,
                       const unsigned char* id, int device, dbag_result* out) {
  return guarded([&] {
    check_precision(precision);
    if (precision == 8 && c->coupling_fp32) lm_nccl<double, float>(p, c, rank, nranks, id, device, out);
    else if (precision == 8) lm_nccl<double>(p, c, rank, nranks, id, device, out);
    else lm_nccl<float>(p, c, rank, nranks, id, device, out);
  });
}

int dbag_create_ex(int device, int precision, int coupling_fp32, dbag_ctx** out) {
  return guarded([&] {
    check_precision(precision);
    auto ctx = std::make_unique<dbag_ctx>();
    ctx->precision = precision;
    ctx->comm = std::make_unique<SelfComm>();
    if (precision == 8 && coupling_fp32) ctx->r64l = std::make_unique<Rank<double, float>>(device, ctx->comm.get());
    else if (precision == 8) ctx->r64 = std::make_unique<Rank<double>>(device, ctx->comm.get());
    else ctx->r32 = std::make_unique<Rank<float>>(device, ctx->comm.get());
    *out = ctx.release();
  });
}

int dbag_create(int device, int precision, dbag_ctx** out) { return dbag_create_ex(device, precision, 0, out); }

namespace {
// A context over `comm` (owned by the context) on `device`.
void make_ctx(int device, int precision, int coupling_fp32, std::unique_ptr<Comm> comm, dbag_ctx** out) {
  check_precision(precision);
  if (coupling_fp32 && precision != 8)
    throw Error(DBAG_INVALID_ARGUMENT, "coupling_fp32 needs precision 8 (FP64 arithmetic, FP32 E blocks)");
  DBAG_CUDA(cudaSetDevice(device));
  auto ctx = std::make_unique<dbag_ctx>();
  ctx->precision = precision;
  ctx->comm = std::move(comm);
  if (precision == 8 && coupling_fp32) ctx->r64l = std::make_unique<Rank<double, float>>(device, ctx->comm.get());
  else if (precision == 8) ctx->r64 = std::make_unique<Rank<double>>(device, ctx->comm.get());
  else ctx->r32 = std::make_unique<Rank<float>>(device, ctx->comm.get());
  *out = ctx.release();
}
}  // namespace

int dbag_create_shard(int device, int precision, int coupling_fp32, int rank, int nranks, dbag_ctx** out) {
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(DBAG_INVALID_ARGUMENT, "bad shard rank / count");
    make_ctx(device, precision, coupling_fp32, std::make_unique<LocalComm>(rank, nranks), out);
  });
}

int dbag_create_nccl_ex(int device, int rank, int nranks, const unsigned char* id, int precision, int coupling_fp32,
                        dbag_ctx** out) {
  return guarded([&] {
    check_precision(precision);
    if (coupling_fp32 && precision != 8)
      throw Error(DBAG_INVALID_ARGUMENT, "coupling_fp32 needs precision 8 (FP64 arithmetic, FP32 E blocks)");
    DBAG_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<dbag_ctx>();
    ctx->precision = precision;
    ctx->comm = std::make_unique<NcclComm>(rank, nranks, id);
    if (precision == 8 && coupling_fp32) ctx->r64l = std::make_unique<Rank<double, float>>(device, ctx->comm.get());
    else if (precision == 8) ctx->r64 = std::make_unique<Rank<double>>(device, ctx->comm.get());
    else ctx->r32 = std::make_unique<Rank<float>>(device, ctx->comm.get());
    *out = ctx.release();
  });
}

int dbag_create_nccl(int device, int rank, int nranks, const unsigned char* id, int precision, dbag_ctx** out) {
  return dbag_create_nccl_ex(device, rank, nranks, id, precision, 0, out);
}

int dbag_destroy(dbag_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int dbag_upload_problem(dbag_ctx* ctx, const dbag_problem* p, int jacobian_mode) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) { rk.upload(*p, jacobian_mode); });
    ctx->num_obs = p->num_observations;
    ctx->cost_valid = false;
  });
}

int dbag_set_state(dbag_ctx* ctx, const void* x_c, const void* x_p) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.set_state(static_cast<const T*>(x_c), static_cast<const T*>(x_p));
    });
    ctx->cost_valid = false;
  });
}

int dbag_get_state(dbag_ctx* ctx, void* x_c, void* x_p) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.get_state(static_cast<T*>(x_c), static_cast<T*>(x_p));
    });
  });
}

int dbag_cost(dbag_ctx* ctx, int use_trial, double* cost, int64_t* bad_edge) {
  return guarded([&] {
    std::int64_t bad = -1;
    with_rank(ctx, [&](auto& rk) { *cost = rk.cost(use_trial != 0, &bad); });
    if (bad_edge) *bad_edge = bad;
  });
}

int dbag_linearize(dbag_ctx* ctx, int64_t* bad_edge) {
  if (bad_edge) *bad_edge = -1;
  const int rc = guarded([&] { with_rank(ctx, [&](auto& rk) { rk.linearize(); }); });
  if (rc == DBAG_DEGENERATE_DEPTH && bad_edge) *bad_edge = g_err_index;
  return rc;
}

int dbag_damp_factor(dbag_ctx* ctx, double lambda, int policy, int64_t* bad_block, int* bad_bs) {
  if (bad_block) *bad_block = -1;
  if (bad_bs) *bad_bs = 0;
  const int rc = guarded([&] { with_rank(ctx, [&](auto& rk) { rk.damp_factor(lambda, policy); }); });
  if (rc == DBAG_SINGULAR_BLOCK) {
    if (bad_block) *bad_block = g_err_index;
    if (bad_bs) *bad_bs = g_err_bs;
  }
  return rc;
}

int dbag_rhs(dbag_ctx* ctx) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { rk.rhs(); }); });
}

int dbag_pcg(dbag_ctx* ctx, double tol, int max_iters, int* iterations, int* converged) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      const PcgOut o = rk.pcg(tol, max_iters);
      if (iterations) *iterations = o.iterations;
      if (converged) *converged = o.converged ? 1 : 0;
    });
  });
}

int dbag_backsub_trial(dbag_ctx* ctx) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { rk.backsub_trial(); }); });
}

int dbag_model_terms(dbag_ctx* ctx, double lambda, int policy, double* step_inf, double* damping_term, double* gv) {
  // The reference's trial evaluates the damping term with the lambda and
  // policy it damped with (dba/solver.hpp:350-353, 389-408): the device sums
  // were formed with the preceding damp_factor's pair, so another pair is an
  // error rather than a silently different model.
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      if (lambda != rk.damping_lambda() || policy != rk.damping_policy())
        throw Error(DBAG_INVALID_ARGUMENT, "model_terms: lambda/policy differ from the preceding damp_factor's");
      rk.model_terms(step_inf, damping_term, gv);
    });
  });
}

int dbag_accept(dbag_ctx* ctx) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) { rk.accept(); });
    ctx->cost_valid = false;
  });
}

int dbag_lm_probe_step(dbag_ctx* ctx, double lambda, const dbag_config* c, double* cost_new, int* pcg_iterations,
                       int* accepted) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      if (!ctx->cost_valid) {
        std::int64_t bad = -1;
        ctx->cost = rk.cost(false, &bad);
        if (!std::isfinite(ctx->cost)) throw degenerate_depth(bad);
        ctx->cost_valid = true;
      }
      rk.linearize();
      const Trial t = run_trial(rk, *c, lambda, ctx->cost);
      if (cost_new) *cost_new = t.cost_new;
      if (pcg_iterations) *pcg_iterations = t.factorization_ok ? t.pcg_iterations : 0;
      if (accepted) *accepted = t.accepted ? 1 : 0;
    });
  });
}

int dbag_profile(dbag_ctx* ctx, int enable, double* dse_ms, int64_t* dse_launches, double* dse_point_ms,
                 double* dse_cam_ms) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      if (enable >= 0) {
        rk.set_profiling(enable != 0);
      } else {
        double t = 0, a = 0, b = 0;
        std::int64_t n = 0;
        rk.profile(&t, &n, &a, &b);
        if (dse_ms) *dse_ms = t;
        if (dse_launches) *dse_launches = n;
        if (dse_point_ms) *dse_point_ms = a;
        if (dse_cam_ms) *dse_cam_ms = b;
      }
    });
  });
}

int dbag_event_mark(dbag_ctx* ctx, int which) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { rk.mark(which); }); });
}

int dbag_event_elapsed(dbag_ctx* ctx, double* ms) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { *ms = rk.elapsed_ms(); }); });
}

int dbag_synchronize(dbag_ctx* ctx) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { rk.sync(); }); });
}

int dbag_time_dse_pass(dbag_ctx* ctx, int reps, double* ms_per_pass) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { *ms_per_pass = rk.time_dse_pass(reps); }); });
}

int dbag_launch_count(dbag_ctx* ctx, int64_t* out) {
  return guarded([&] { with_rank(ctx, [&](auto& rk) { *out = rk.launches(); }); });
}

int dbag_residuals(dbag_ctx* ctx, int use_trial, void* out) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.residuals(use_trial != 0, static_cast<T*>(out));
    });
  });
}

int dbag_get_jacobians(dbag_ctx* ctx, void* res, void* jac) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.get_jacobians(static_cast<T*>(res), static_cast<T*>(jac));
    });
  });
}

int dbag_get_system(dbag_ctx* ctx, void* B, void* C, void* E, void* v, void* w) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.get_system(static_cast<T*>(B), static_cast<T*>(C), static_cast<T*>(E), static_cast<T*>(v),
                    static_cast<T*>(w));
    });
  });
}

int dbag_set_system(dbag_ctx* ctx, const void* B, const void* C, const void* E_table, const void* v, const void* w) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.set_system(static_cast<const T*>(B), static_cast<const T*>(C), static_cast<const T*>(E_table),
                    static_cast<const T*>(v), static_cast<const T*>(w));
    });
  });
}

int dbag_dse(dbag_ctx* ctx, const void* x, void* out) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      rk.dse_host(static_cast<const T*>(x), static_cast<T*>(out));
    });
  });
}

int dbag_dpcg(dbag_ctx* ctx, const void* rhs, double tol, int max_iters, void* x_out, int* iterations,
              int* converged) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using S = std::remove_reference_t<decltype(rk)>;
      using T = typename S::Scalar;
      const PcgOut o = rk.dpcg_host(static_cast<const T*>(rhs), tol, max_iters, static_cast<T*>(x_out));
      if (iterations) *iterations = o.iterations;
      if (converged) *converged = o.converged ? 1 : 0;
    });
  });
}

int dbag_group_operator(int precision, const dbag_problem* p, int k, int device, double lambda, int policy,
                        const void* B, const void* C, const void* E_table, int mode, const void* x, double tol,
                        int max_iters, void* out, int* iterations, int* rank_identical) {
  return guarded([&] {
    check_precision(precision);
    if (precision == 8)
      group_operator<double>(p, k, device, lambda, policy, B, C, E_table, mode, x, tol, max_iters, out, iterations,
                             rank_identical);
    else
      group_operator<float>(p, k, device, lambda, policy, B, C, E_table, mode, x, tol, max_iters, out, iterations,
                            rank_identical);
  });
}

int dbag_group_allreduce(int k, int device, int64_t len, double* data) {
  return guarded([&] {
    Group g(k, {device});
    run_ranks(g, [&](int r) {
      GroupComm comm(&g, r);
      double* d = nullptr;
      DBAG_CUDA(cudaMalloc(&d, sizeof(double) * std::max<int64_t>(len, 1)));
      cudaStream_t s;
      DBAG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      DBAG_CUDA(cudaMemcpyAsync(d, data + static_cast<std::size_t>(r) * len, sizeof(double) * len,
                                cudaMemcpyHostToDevice, s));
      comm.allreduce_sum(d, len, DType::f64, s);
      DBAG_CUDA(cudaMemcpyAsync(data + static_cast<std::size_t>(r) * len, d, sizeof(double) * len,
                                cudaMemcpyDeviceToHost, s));
      DBAG_CUDA(cudaStreamSynchronize(s));
      cudaStreamDestroy(s);
      cudaFree(d);
    });
  });
}

// ---- WorkerGroup handle (dba/comms.hpp:35-234) -----------------------------
struct dbag_group {
  std::unique_ptr<Group> g;
  std::vector<cudaStream_t> streams;
};

int dbag_group_create(int k, const int* devices, int n_devices, int64_t timeout_ms, dbag_group** out) {
  return guarded([&] {
    std::vector<int> devs(devices, devices + std::max(n_devices, 0));
    if (devs.empty()) devs.push_back(0);
    auto h = std::make_unique<dbag_group>();
    h->g = std::make_unique<Group>(k, devs, std::chrono::milliseconds(timeout_ms > 0 ? timeout_ms : 60000));
    h->streams.resize(static_cast<std::size_t>(k));
    for (int r = 0; r < k; ++r) {
      DBAG_CUDA(cudaSetDevice(h->g->device_of(r)));
      DBAG_CUDA(cudaStreamCreateWithFlags(&h->streams[static_cast<std::size_t>(r)], cudaStreamNonBlocking));
    }
    *out = h.release();
  });
}

int dbag_group_destroy(dbag_group* h) {
  return guarded([&] {
    if (!h) return;
    for (std::size_t r = 0; r < h->streams.size(); ++r) {
      cudaSetDevice(h->g->device_of(static_cast<int>(r)));
      cudaStreamDestroy(h->streams[r]);
    }
    delete h;
  });
}

static void check_group_rank(dbag_group* h, int rank) {
  if (!h || rank < 0 || rank >= h->g->size()) throw Error(DBAG_INVALID_ARGUMENT, "bad group handle or rank");
}

int dbag_group_barrier(dbag_group* h, int rank) {
  return guarded([&] {
    check_group_rank(h, rank);
    h->g->barrier(rank);
  });
}

int dbag_group_allreduce_sum(dbag_group* h, int rank, void* data, int64_t len, int precision) {
  return guarded([&] {
    check_group_rank(h, rank);
    check_precision(precision);
    if (len < 0 || (len > 0 && !data)) throw Error(DBAG_INVALID_ARGUMENT, "bad all-reduce buffer");
    DBAG_CUDA(cudaSetDevice(h->g->device_of(rank)));
    cudaStream_t s = h->streams[static_cast<std::size_t>(rank)];
    const std::size_t bytes = static_cast<std::size_t>(len) * static_cast<std::size_t>(precision);
    void* d = nullptr;
    DBAG_CUDA(cudaMalloc(&d, std::max<std::size_t>(bytes, 8)));
    std::unique_ptr<void, void (*)(void*)> keep(d, [](void* q) { cudaFree(q); });
    DBAG_CUDA(cudaMemcpyAsync(d, data, bytes, cudaMemcpyHostToDevice, s));
    h->g->allreduce(rank, d, len, precision == 8 ? DType::f64 : DType::f32, false, s);
    DBAG_CUDA(cudaMemcpyAsync(data, d, bytes, cudaMemcpyDeviceToHost, s));
    DBAG_CUDA(cudaStreamSynchronize(s));
  });
}

int dbag_group_abort(dbag_group* h, const char* why) {
  return guarded([&] {
    if (!h) throw Error(DBAG_INVALID_ARGUMENT, "null group handle");
    h->g->abort(why ? why : "aborted by caller");
  });
}

int dbag_group_sequence(dbag_group* h, int rank, uint64_t* out) {
  return guarded([&] {
    check_group_rank(h, rank);
    *out = h->g->sequence(rank);
  });
}

int dbag_create_group_rank(dbag_group* h, int rank, int precision, int coupling_fp32, dbag_ctx** out) {
  return guarded([&] {
    check_group_rank(h, rank);
    make_ctx(h->g->device_of(rank), precision, coupling_fp32, std::make_unique<GroupComm>(h->g.get(), rank), out);
  });
}

int dbag_lm_solve_ctx(dbag_ctx* ctx, const dbag_config* c, dbag_result* out) {
  return guarded([&] {
    with_rank(ctx, [&](auto& rk) {
      using R = std::remove_reference_t<decltype(rk)>;
      using S = typename R::Scalar;
      if (c->workers != ctx->comm->size())
        throw Error(DBAG_INVALID_ARGUMENT, "config.workers must equal the context's rank count");
      if (ctx->num_obs <= 0) throw Error(DBAG_INVALID_ARGUMENT, "lm_solve_ctx needs an uploaded problem");
      if (c->max_iterations < 0 || !out) throw Error(DBAG_INVALID_ARGUMENT, "bad config or result");
      const Outcome o = lm_solve_rank(rk, *c, ctx->num_obs);
      rk.gather_state(static_cast<S*>(out->x_c), static_cast<S*>(out->x_p));
      fill_result(o, ctx->comm->size(), out);
    });
    ctx->cost_valid = false;
  });
}

}  // extern "C"

namespace {
template <class S, int BS>
void block_factor(std::int64_t nb, const void* blocks, void* factor, std::int64_t* bad) {
  S *a = nullptr, *ad = nullptr, *f = nullptr;
  unsigned long long* dbad = nullptr;
  const std::size_t bytes = static_cast<std::size_t>(std::max<std::int64_t>(nb, 1)) * BS * BS * sizeof(S);
  DBAG_CUDA(cudaMalloc(&a, bytes));
  std::unique_ptr<void, void (*)(void*)> k1(a, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMalloc(&ad, bytes));
  std::unique_ptr<void, void (*)(void*)> k2(ad, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMalloc(&f, bytes));
  std::unique_ptr<void, void (*)(void*)> k3(f, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMalloc(&dbad, sizeof(unsigned long long)));
  std::unique_ptr<void, void (*)(void*)> k4(dbad, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMemset(dbad, 0xff, sizeof(unsigned long long)));
  if (nb > 0) {
    DBAG_CUDA(cudaMemcpy(a, blocks, static_cast<std::size_t>(nb) * BS * BS * sizeof(S), cudaMemcpyHostToDevice));
    dev::k_damp_factor<S, BS><<<grid_for(nb, 64, 1 << 30), 64>>>(nb, a, S(0), 0, ad, f,
                                                                 static_cast<const std::int32_t*>(nullptr), dbad);
    DBAG_LAUNCH_CHECK();
    DBAG_CUDA(cudaMemcpy(factor, f, static_cast<std::size_t>(nb) * BS * BS * sizeof(S), cudaMemcpyDeviceToHost));
  }
  unsigned long long raw = ~0ull;
  DBAG_CUDA(cudaMemcpy(&raw, dbad, sizeof(raw), cudaMemcpyDeviceToHost));
  *bad = raw == ~0ull ? -1 : static_cast<std::int64_t>(raw);
}
template <class S, int BS>
void block_solve(std::int64_t nb, const void* factor, void* x) {
  if (nb <= 0) return;
  S *f = nullptr, *v = nullptr;
  DBAG_CUDA(cudaMalloc(&f, static_cast<std::size_t>(nb) * BS * BS * sizeof(S)));
  std::unique_ptr<void, void (*)(void*)> k1(f, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMalloc(&v, static_cast<std::size_t>(nb) * BS * sizeof(S)));
  std::unique_ptr<void, void (*)(void*)> k2(v, [](void* q) { cudaFree(q); });
  DBAG_CUDA(cudaMemcpy(f, factor, static_cast<std::size_t>(nb) * BS * BS * sizeof(S), cudaMemcpyHostToDevice));
  DBAG_CUDA(cudaMemcpy(v, x, static_cast<std::size_t>(nb) * BS * sizeof(S), cudaMemcpyHostToDevice));
  dev::k_block_solve<S, BS><<<grid_for(nb, 64, 1 << 30), 64>>>(nb, f, v);
  DBAG_LAUNCH_CHECK();
  DBAG_CUDA(cudaMemcpy(x, v, static_cast<std::size_t>(nb) * BS * sizeof(S), cudaMemcpyDeviceToHost));
}
void check_bs(int bs) {
  if (bs != 3 && bs != 9) throw Error(DBAG_INVALID_ARGUMENT, "block size must be 3 or 9");
}
}  // namespace

extern "C" {

int dbag_block_factor(int device, int precision, int bs, int64_t nblocks, const void* blocks, void* factor,
                      int64_t* bad_block) {
  return guarded([&] {
    check_precision(precision);
    check_bs(bs);
    if (nblocks < 0 || (nblocks > 0 && (!blocks || !factor))) throw Error(DBAG_INVALID_ARGUMENT, "bad block arrays");
    DBAG_CUDA(cudaSetDevice(device));
    std::int64_t bad = -1;
    if (precision == 8) {
      if (bs == 3) block_factor<double, 3>(nblocks, blocks, factor, &bad);
      else block_factor<double, 9>(nblocks, blocks, factor, &bad);
    } else {
      if (bs == 3) block_factor<float, 3>(nblocks, blocks, factor, &bad);
      else block_factor<float, 9>(nblocks, blocks, factor, &bad);
    }
    if (bad_block) *bad_block = bad;
    if (bad >= 0)  // SingularBlockError(i, BS) (dba/block_matrix.hpp:128-129)
      throw Error(DBAG_SINGULAR_BLOCK, "block " + std::to_string(bad) + " of size " + std::to_string(bs) +
                                           " is not positive definite", bad, bs);
  });
}

int dbag_block_solve(int device, int precision, int bs, int64_t nblocks, const void* factor, void* x) {
  return guarded([&] {
    check_precision(precision);
    check_bs(bs);
    if (nblocks < 0 || (nblocks > 0 && (!factor || !x))) throw Error(DBAG_INVALID_ARGUMENT, "bad block arrays");
    DBAG_CUDA(cudaSetDevice(device));
    if (precision == 8) {
      if (bs == 3) block_solve<double, 3>(nblocks, factor, x);
      else block_solve<double, 9>(nblocks, factor, x);
    } else {
      if (bs == 3) block_solve<float, 3>(nblocks, factor, x);
      else block_solve<float, 9>(nblocks, factor, x);
    }
  });
}

}  // extern "C"
