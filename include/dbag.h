/*
 * dbag.h — C ABI of the B200-native bundle-adjustment inner loop.
 *
 * The reference (MegBA re-creation, /root/reference/proj) exposes this path
 * only as the header-only C++ API in namespace dba (proj/README.md:154-176);
 * it has no C ABI and no plugin registry. Every entry point
 * below names the reference symbol it replaces. Conventions:
 *   - plain pointers and sizes; no torch or CUDA types;
 *   - `precision` is sizeof(Scalar): 4 (fp32) or 8 (fp64), the reference's
 *     Scalar template parameter (dba/problem.hpp:35, dba/solver.hpp:71);
 *   - host buffers are copied in, the caller keeps ownership; device buffers
 *     belong to the context;
 *   - every call is synchronous with respect to the scalars it returns;
 *   - status codes map 1:1 onto the reference's exception types
 *     (dba/errors.hpp:17-84); the host facade (include/dba/dba.hpp and the
 *     Python package) rethrows them.
 */
#ifndef DBAG_H_
#define DBAG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (dba/errors.hpp) ------------------------------------ */
#define DBAG_OK 0
#define DBAG_DEGENERATE_DEPTH 1   /* DegenerateDepthError(edge_id)        errors.hpp:35-46 */
#define DBAG_SINGULAR_BLOCK 2     /* SingularBlockError(index, size)      errors.hpp:56-70 */
#define DBAG_PCG_BREAKDOWN 3      /* PcgBreakdownError                    errors.hpp:81-84 */
#define DBAG_SHAPE 4              /* ShapeError                           errors.hpp:49-52 */
#define DBAG_INVALID_ARGUMENT 5   /* InvalidArgumentError                 errors.hpp:28-31 */
#define DBAG_COLLECTIVE 6         /* CollectiveError                      errors.hpp:75-78 */
#define DBAG_CUDA_ERROR 7
#define DBAG_NCCL_ERROR 8
#define DBAG_INTERNAL 9
#define DBAG_PARSE 10             /* ParseError(msg, line): line via dbag_last_error_index  errors.hpp:17-26 */

/* ---- problem / config / result ----------------------------------------- */

/* BAProblem<Scalar> (dba/problem.hpp:171-261) as flat arrays: cameras are the
 * packed x_c of pack_cameras (9 per camera: aa0 aa1 aa2 t0 t1 t2 f k1 k2),
 * points the packed x_p (3 per point), observations in canonical edge order.
 * weight may be NULL (all ones). Scalar arrays use `precision`. */
typedef struct dbag_problem {
  int32_t num_cameras, num_points;
  int64_t num_observations;
  const void* cameras;
  const void* points;
  const int32_t* camera_id;
  const int32_t* point_id;
  const void* pixel_x;
  const void* pixel_y;
  const void* weight;
} dbag_problem;

/* SolverConfig (dba/solver.hpp:39-55); defaults via dbag_default_config. */
typedef struct dbag_config {
  int32_t workers, max_iterations;
  double pcg_tol;
  int32_t pcg_max_iters;
  int32_t coupling_fp32;       /* B200 extension: FP64 solve with the E blocks stored in FP32; 0 = off */
  double lambda0, lambda_max, rel_tol, step_tol;
  int32_t damping;             /* 0 identity, 1 diag_scaled (default) */
  int32_t mse_half;            /* 1 half_per_observation (default), 0 per_observation */
  int32_t jacobian;            /* 0 autodiff (default), 1 analytic */
  int32_t check_rank_identity; /* rank-divergence probe, dba/solver.hpp:479-501 */
  int64_t collective_timeout_ms; /* SolverConfig::collective_timeout (dba/solver.hpp:54), default 60000; <= 0 = default */
} dbag_config;

/* SolverState + IterationRecord history (dba/solver.hpp:57-85). The caller
 * owns every array; `capacity` bounds the history rows written. */
typedef struct dbag_result {
  int32_t iterations, termination; /* 0 converged, 1 max_iterations, 2 stalled */
  double cost, lambda, nu;
  int32_t capacity, workers;
  int32_t* rec_iteration;
  double* rec_cost;
  double* rec_mse;
  double* rec_lambda;
  int32_t* rec_pcg;
  int32_t* rec_accepted;
  double* rec_wall;
  uint64_t* rec_worker_edges;     /* capacity x workers */
  uint64_t* rec_worker_block_ops; /* capacity x workers */
  void* x_c;                      /* 9m Scalar (out, may be NULL) */
  void* x_p;                      /* 3n Scalar (out, may be NULL) */
  /* SolverState's most recent trial (dba/solver.hpp:80-84) */
  int32_t last_accepted;
  double last_cost_change, last_step_inf, previous_cost;
} dbag_result;

/* SyntheticOptions (dba/synthetic.hpp:19-30) plus the count-exact extension of
 * num_observations > 0 selects Q_p = floor(N/n) + [p < N mod n]
 * nearest cameras per point (0 = reference behaviour, obs_per_point each), and
 * pixel_noise > 0 adds U(-noise, noise) per pixel coordinate from a second
 * mt19937_64(seed) stream in edge order (tests/acceptance.cpp:88-99). */
typedef struct dbag_synthetic_options {
  int32_t cameras, points, obs_per_point;
  int32_t exhaustive_search; /* 1: the reference's O(n m) nearest-camera scan */
  uint64_t seed;
  double circle_radius, base_focal, pose_noise, intrinsic_noise, point_noise;
  int64_t num_observations;
  double pixel_noise;
} dbag_synthetic_options;

int dbag_version(void);
const char* dbag_last_error(void);
/* Extra payload of the last error: edge id (DEGENERATE_DEPTH) or block index
 * (SINGULAR_BLOCK), and the block size for SINGULAR_BLOCK. */
int64_t dbag_last_error_index(void);
int dbag_last_error_block_size(void);
void dbag_default_config(dbag_config* out);
int dbag_device_count(int* out);

/* ---- host-only utilities ------------------------------------------------ */

/* partition_edges + LocalIndexMap + EdgeBlockMatrix::build_groups for one
 * rank (dba/partition.hpp:76-103, dba/block_matrix.hpp:185-204, 309-320).
 * Integer-exact. Buffers: cam_g[m], pt_g[n], cam_ptr[m+1], cam_blk[count],
 * pt_ptr[n+1], pt_blk[count]. */
int dbag_partition(const dbag_problem* p, int k, int rank, int64_t* start, int64_t* count, int32_t* n_cams,
                   int32_t* cam_g, int32_t* n_pts, int32_t* pt_g, int64_t* cam_ptr, int64_t* cam_blk,
                   int64_t* pt_ptr, int64_t* pt_blk);

/* Halo plan for K ranks: the global ids of points touched by more than one
 * rank, ascending. Returns the count in *n_shared; ids may be
 * NULL to query the count. */
int dbag_shared_points(const dbag_problem* p, int k, int64_t* n_shared, int32_t* ids);

/* Predicted-size memory pool: the exact
 * device bytes rank `rank` of `k` reserves in ONE allocation when the problem
 * is uploaded (E chunk records, shard arrays, state and system blocks, PCG
 * vectors), computed on the host from the partition and layout alone — no
 * GPU needed — so a caller can pick K or the FP32-E variant before
 * uploading. precision 4|8; coupling_fp32 as in dbag_create_ex. Not
 * included: the per-context fixed scratch (< 64 KB) and NCCL's buffers. */
int dbag_predict_memory(const dbag_problem* p, int precision, int coupling_fp32, int k, int rank, uint64_t* bytes);

/* generate_synthetic (dba/synthetic.hpp:70-146), fp64 output. Query the edge
 * count first with dbag_synthetic_count. Outputs: cameras[9m], points[3n],
 * camera_id/point_id/pixel_x/pixel_y[N]. */
int dbag_synthetic_count(const dbag_synthetic_options* o, int64_t* n_obs);
int dbag_generate_synthetic(const dbag_synthetic_options* o, double* cameras, double* points, int32_t* camera_id,
                            int32_t* point_id, double* pixel_x, double* pixel_y);

/* ---- BAL text: dba::parse_bal / serialize_bal (dba/bal_io.hpp:78-209) ----
 * dbag_bal_parse scans `len` bytes of BAL text (header, observations,
 * cameras, points) with the reference's validation and messages; on
 * malformed input it returns DBAG_PARSE, dbag_last_error() reads
 * "line L: <msg>" and dbag_last_error_index() the line L. Values are fp64;
 * callers cast to their Scalar exactly as parse_bal<Scalar> does.
 * dbag_bal_format emits the same text serialize_bal writes ("%.16e" reals);
 * free it with dbag_free_text. */
typedef struct dbag_bal dbag_bal;
int dbag_bal_parse(const char* text, int64_t len, dbag_bal** out);
int dbag_bal_counts(const dbag_bal* b, int32_t* num_cameras, int32_t* num_points, int64_t* num_observations);
int dbag_bal_copy(const dbag_bal* b, double* cameras, double* points, int32_t* camera_id, int32_t* point_id,
                  double* pixel_x, double* pixel_y);
int dbag_bal_free(dbag_bal* b);
int dbag_bal_format(int precision, const dbag_problem* p, char** text, int64_t* len);
int dbag_free_text(char* text);

/* ---- one-shot solve: dba::lm_solve (dba/solver.hpp:523-534) -------------- */

/* Partitions into config->workers ranks, runs one rank context per worker
 * thread on devices[rank % n_devices] (all ranks on one GPU when
 * n_devices == 1), all-reduces in ascending rank order like WorkerGroup, and
 * returns rank 0's state. */
int dbag_lm_solve(int precision, const dbag_problem* p, const dbag_config* c, const int* devices, int n_devices,
                  dbag_result* out);

/* One process per GPU (torchrun): rank `rank` of `nranks` over NCCL. Every
 * rank passes the full problem and the same 128-byte ncclUniqueId. */
int dbag_nccl_unique_id(unsigned char* out128);
int dbag_lm_solve_rank(int precision, const dbag_problem* p, const dbag_config* c, int rank, int nranks,
                       const unsigned char* nccl_id128, int device, dbag_result* out);

/* ---- rank context: the operator level of dba/solver.hpp:295-518 ---------- */
typedef struct dbag_ctx dbag_ctx;

/* K = 1 context on `device` (single rank, no collectives). */
int dbag_create(int device, int precision, dbag_ctx** out);
/* Same, with the memory-lean variant: precision 8 and
 * coupling_fp32 != 0 keep every vector, block and reduction in FP64 and store
 * only the coupling blocks E in FP32 (half the DSE stream). */
int dbag_create_ex(int device, int precision, int coupling_fp32, dbag_ctx** out);
/* Context for rank `rank` of an NCCL communicator (multi-process). */
int dbag_create_nccl(int device, int rank, int nranks, const unsigned char* nccl_id128, int precision,
                     dbag_ctx** out);
/* Same, with the memory-lean variant (coupling_fp32 needs precision 8). */
int dbag_create_nccl_ex(int device, int rank, int nranks, const unsigned char* nccl_id128, int precision,
                        int coupling_fp32, dbag_ctx** out);
int dbag_destroy(dbag_ctx* ctx);
/* Context holding shard `rank` of `nranks` (partition_edges) with LOCAL
 * collectives: the per-partition operators of EdgeEvaluator::linearize / cost
 * and assemble_local (dba/edge_eval.hpp:79-122, 289-309; dba/block_matrix.hpp:
 * 335-388): cost and the assembled B, C, v, w are this partition's own
 * contribution, not all-reduced. */
int dbag_create_shard(int device, int precision, int coupling_fp32, int rank, int nranks, dbag_ctx** out);

/* EdgeEvaluator ctor + PartitionedHessian ctor (dba/edge_eval.hpp:79-97,
 * dba/block_matrix.hpp:185-204, 344-352): partitions the full problem, keeps
 * this rank's shard on the device, sets the state to the problem's x0. */
int dbag_upload_problem(dbag_ctx* ctx, const dbag_problem* p, int jacobian_mode);
/* pack/unpack of x_c (9m) and x_p (3n); get writes only this rank's points. */
int dbag_set_state(dbag_ctx* ctx, const void* x_c, const void* x_p);
int dbag_get_state(dbag_ctx* ctx, void* x_c, void* x_p);

/* detail::distributed_cost (dba/solver.hpp:264-278): current state
 * (use_trial = 0) or the trial state (1). Degenerate depth gives +inf and
 * the lowest offending global edge id in *bad_edge (else -1). */
int dbag_cost(dbag_ctx* ctx, int use_trial, double* cost, int64_t* bad_edge);
/* EdgeEvaluator::linearize + assemble_local + all-reduce of B, C, v, w
 * (dba/solver.hpp:330-340). Returns DBAG_DEGENERATE_DEPTH with the edge id. */
int dbag_linearize(dbag_ctx* ctx, int64_t* bad_edge);
/* damp_into + factor of C then B (dba/solver.hpp:350-355). */
int dbag_damp_factor(dbag_ctx* ctx, double lambda, int policy, int64_t* bad_block, int* bad_bs);
/* g = v - allreduce(E_k C^-1 w) (dba/solver.hpp:357-363). */
int dbag_rhs(dbag_ctx* ctx);
/* dpcg from dx_c = 0 on the reduced camera system (dba/solver.hpp:202-257). */
int dbag_pcg(dbag_ctx* ctx, double tol, int max_iters, int* iterations, int* converged);
/* dx_p = C^-1 (w - allreduce(E_k^T dx_c)); trial = x + dx (dba/solver.hpp:371-379). */
int dbag_backsub_trial(dbag_ctx* ctx);
/* step_inf, damping term, dx_c.v + dx_p.w (dba/solver.hpp:383-410) of the
 * last backsub_trial. lambda / policy must be the preceding damp_factor's
 * (the reference's trial damps and scores with one pair); otherwise
 * DBAG_INVALID_ARGUMENT. */
int dbag_model_terms(dbag_ctx* ctx, double lambda, int policy, double* step_inf, double* damping_term, double* gv);
/* x <- trial (dba/solver.hpp:433-437). */
int dbag_accept(dbag_ctx* ctx);
/* One full LM iteration from the current state and lambda, decision
 * computed but the state NOT committed (the bench "step"): linearize,
 * damp+factor, rhs, dpcg, back-substitution, trial cost, model terms. */
int dbag_lm_probe_step(dbag_ctx* ctx, double lambda, const dbag_config* c, double* cost_new, int* pcg_iterations,
                       int* accepted);
/* Device time (ms) of the DSE kernels and their launch count since the last
 * reset (CUDA events on the context's stream; enable first). */
int dbag_profile(dbag_ctx* ctx, int enable, double* dse_ms, int64_t* dse_launches, double* dse_point_ms,
                 double* dse_cam_ms);
/* Device ms between two points of the context's stream (bench timing). */
int dbag_event_mark(dbag_ctx* ctx, int which);
int dbag_event_elapsed(dbag_ctx* ctx, double* ms);
int dbag_synchronize(dbag_ctx* ctx);
/* Device ms per launch of the single-rank graph DPCG's DSE pass (k_g_pass),
 * launched alone `reps` times back to back on the state the last dbag_pcg /
 * probe step left (bench roofline; needs a preceding graph DPCG). */
int dbag_time_dse_pass(dbag_ctx* ctx, int reps, double* ms_per_pass);
/* Number of kernels this context has launched (bench: gpu_launches). */
int dbag_launch_count(dbag_ctx* ctx, int64_t* out);
/* The context's pool after dbag_upload_problem: reserved == the prediction,
 * used == reserved (upload fails with DBAG_INTERNAL otherwise). */
int dbag_memory_pool(dbag_ctx* ctx, uint64_t* reserved, uint64_t* used);

/* ---- test hooks (operator-level parity) ------------------- */
/* Scalar-model residuals (dba/problem.hpp:151-165) of the current (0) or
 * trial (1) state, res[2][count] in shard edge order; NaN on P_z == 0. */
int dbag_residuals(dbag_ctx* ctx, int use_trial, void* out);
/* EdgeJacobianBatch in shard edge order: res[2][count], jac[2][12][count]. */
int dbag_get_jacobians(dbag_ctx* ctx, void* res, void* jac);
/* Assembled (all-reduced) system: B[81m], C[9n] and w[3n] full size (zeros
 * for points this rank does not touch), E[27 count] row-major 9x3 blocks in
 * shard edge order, v[9m]. */
int dbag_get_system(dbag_ctx* ctx, void* B, void* C, void* E, void* v, void* w);
/* Replace the assembled system with caller blocks (B[81m], C[9n] full-size,
 * E_table[27 N] in global edge order, v[9m], w[3n]); NULL keeps a part. */
int dbag_set_system(dbag_ctx* ctx, const void* B, const void* C, const void* E_table, const void* v, const void* w);
/* out = dse(x) with the damped B and C^-1 of the last damp_factor
 * (dba/solver.hpp:149-181). */
int dbag_dse(dbag_ctx* ctx, const void* x, void* out);
/* dpcg on an arbitrary rhs (dba/solver.hpp:202-257). */
int dbag_dpcg(dbag_ctx* ctx, const void* rhs, double tol, int max_iters, void* x_out, int* iterations,
              int* converged);
/* Multi-rank operator drivers with K in-process ranks on `device`, used by
 * the K-equivalence tests (tests/test_solver.cpp:107-333): the problem's own
 * linearization, all-reduced, damped with (lambda, policy) -> mode 0:
 * out = dse(x); mode 1: out = dpcg(rhs = x). With fabricated blocks when
 * B != NULL (B[81m], C[9n] already damped, E_table[27N]). rank_identical
 * reports whether all ranks produced bitwise-identical outputs. */
int dbag_group_operator(int precision, const dbag_problem* p, int k, int device, double lambda, int policy,
                        const void* B, const void* C, const void* E_table, int mode, const void* x, double tol,
                        int max_iters, void* out, int* iterations, int* rank_identical);
/* WorkerGroup::allreduce_sum over K in-process ranks on `device`:
 * data is K x len fp64 (rank-major), reduced in place. */
int dbag_group_allreduce(int k, int device, int64_t len, double* data);

/* ---- WorkerGroup handle: dba::WorkerGroup (dba/comms.hpp:35-234) ---------
 * K in-process ranks on devices[rank % n_devices]; each rank's calls come
 * from that rank's own host thread (run_on_workers). Collectives validate
 * call sequence, kind, element type and length, and a missing rank trips
 * the timeout with a message naming the absent ranks (DBAG_COLLECTIVE);
 * abort() makes every pending and later collective fail. Up to 256 ranks.
 * allreduce_sum reduces a HOST buffer in place (staged through the rank's
 * device, summed in ascending rank order: bit-identical on every rank). */
typedef struct dbag_group dbag_group;
int dbag_group_create(int k, const int* devices, int n_devices, int64_t timeout_ms, dbag_group** out);
int dbag_group_destroy(dbag_group* g);
int dbag_group_barrier(dbag_group* g, int rank);                                   /* comms.hpp:56-63 */
int dbag_group_allreduce_sum(dbag_group* g, int rank, void* data, int64_t len, int precision); /* :67-91 */
int dbag_group_abort(dbag_group* g, const char* why);                              /* :96-105 */
int dbag_group_sequence(dbag_group* g, int rank, uint64_t* out);                   /* :52-53 */
/* Rank `rank` of the group as an operator context (dba/solver.hpp:149-257,
 * 295-299 called inside run_on_workers): every collective of the context's
 * operators (cost, linearize, damp_factor, dse, dpcg, ...) goes through the
 * group. Call from that rank's own thread; the group outlives the context. */
int dbag_create_group_rank(dbag_group* g, int rank, int precision, int coupling_fp32, dbag_ctx** out);
/* lm_solve_rank (dba/solver.hpp:295-518) on an uploaded context: collective
 * over the context's ranks; out->x_c / x_p receive the full, rank-identical
 * state. */
int dbag_lm_solve_ctx(dbag_ctx* ctx, const dbag_config* c, dbag_result* out);

/* ---- FactoredBlockDiagonal (dba/block_matrix.hpp:118-167) on the device --- */
/* LLT of nblocks BS x BS row-major blocks (bs = 3 or 9): `factor` receives the
 * device format (lower factor, reciprocal pivots above the diagonal, bs*bs
 * per block); *bad_block = the lowest non-positive-definite block or -1
 * (DBAG_SINGULAR_BLOCK is returned then). */
int dbag_block_factor(int device, int precision, int bs, int64_t nblocks, const void* blocks, void* factor,
                      int64_t* bad_block);
/* x := D^-1 x blockwise from dbag_block_factor's factor. */
int dbag_block_solve(int device, int precision, int bs, int64_t nblocks, const void* factor, void* x);

#ifdef __cplusplus
}
#endif
#endif /* DBAG_H_ */
