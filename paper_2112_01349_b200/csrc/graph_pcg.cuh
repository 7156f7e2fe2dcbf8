// graph_pcg.cuh — DPCG as a CUDA graph with device-side control flow.
//
// dpcg (dba/solver.hpp:202-257) for a single rank, every recurrence on the
// device and the loop itself in the graph: k_g_init, then one conditional
// WHILE node whose body is DBAG_GRAPH_UNROLL copies of
//   k_g_pass   the DSE pass over E (one CTA per chunk, long tiles first),
//              gathering p = z + beta p_prev (or x) once per (chunk,
//              camera) and writing camera-major partials;
// followed by the camera fold + PCG step, in one of three forms chosen by m:
//   k_g_fsc    m <= 544: one thread-block cluster (<= 16 CTAs), warp per
//              camera; p'q and rho, |r|^2 over distributed shared memory;
//   k_g_fs     m <= 4736: warp per camera, software grid barrier for p'q,
//              last-block grid reduction for rho, |r|^2;
//   k_g_fold + k_g_step  beyond: the fold and the step as two kernels.
// Each computes c = fold(partials) in chunk order, q = B_d p - c, p'q (camera
// order), alpha, x += alpha p, r -= alpha q, z = B^-1 r, rho, |r|^2 and the
// loop decision (cudaGraphSetConditional). Consecutive kernels are linked by
// programmatic-dependent-launch edges: a kernel's constant loads run before
// it waits on its predecessor. Every 50th iteration the body runs once more
// as a residual-refresh pass (DSE on x, r = g - S x), selected by a device
// phase flag; once the loop is decided the copies left in the body return at
// entry (done flag). One graph launch runs the whole inner solve with no host
// round trip.
//
// Loop control matches the reference: stop when |r| <= tol |g| or
// n == max_iters; rho (after z = B^-1 r) and p'q breakdowns stop with status
// 1 / 2 in the reference's order (rho checked before the DSE, p'q after).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dse.cuh"

#ifndef DBAG_GRAPH_UNROLL
#define DBAG_GRAPH_UNROLL 16  // PCG iterations per WHILE-body launch (DBAG_UNROLL overrides)
#endif

namespace dbag {
namespace dev {
// k_g_fs: lane-strided partial rows per load batch (2: no spill at 128
// registers; 3 and 4 measured no faster)
constexpr int kFsBatch = 2;

#if DBAG_GTIMING  // per-iteration timeline of the graph body (development builds)
constexpr int kTlStride = 16;  // marks of one iteration: a 128-byte line of their own
__device__ unsigned long long g_tl[kTlStride * 1024];
__device__ __forceinline__ void tl_mark(int n, int k) {
  if (n < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl[n * kTlStride + k] = t;
  }
}
#define DBAG_TL(n, k, cond) \
  if (cond) tl_mark(n, k)
#else
#define DBAG_TL(n, k, cond)
#endif

template <class S>
struct GScal {
  double rho, rho_prev, pq, rnorm2, rhs_norm2, tol;
  S alpha, beta;
  int n, max_iters, status, dse_count;
  int phase;  // 0: PCG pass, 1: residual-refresh pass (DSE on x)
  int done;   // loop finished: the remaining kernels of an unrolled body return at once
  int peer_fail;  // K > 1: bit p = rank p missed a peer all-reduce (PeerSite::failed)
};

template <class S>
struct GBufs {
  std::int32_t m;
  const S* Bd;
  const S* Binv;
  const S* g;
  S* x;
  S* r;
  S* z;
  S* p0;  // p buffers: iteration n writes p[n & 1]
  S* p1;
  S* q;
  const std::int32_t* cam_part_ptr;
  const S* part;
  double* pq_cam;  // per-camera p.q of the running pass
  const S* c_total;  // K > 1: E C^-1 E^T p summed over ranks (k_g_fold reads it instead of the partials)
};

// The WHILE node's condition; kNoCond outside a graph (the run-ahead
// stream loop of K > 1 ranks, Rank::pcg_stream).
constexpr cudaGraphConditionalHandle kNoCond = ~0ull;
__device__ __forceinline__ void set_conditional(cudaGraphConditionalHandle h, unsigned v) {
  if (h != kNoCond) cudaGraphSetConditional(h, v);
}

template <class S>
__device__ __forceinline__ S* p_cur(const GBufs<S>& B, int n) {
  return (n & 1) ? B.p1 : B.p0;
}

// Programmatic dependent launch (graph edges of type programmatic): a kernel
// lets its dependent start launching early, and the dependent waits for the
// full completion (and memory) of its prerequisite only where it first needs
// it. Both are no-ops for kernels launched without such an edge.
__device__ __forceinline__ void pdl_allow_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Gather of the graph's DSE pass: the tile's E, metadata and C factors (all
// constant during the solve) are loaded before waiting on the previous
// kernel; then p = z + beta p_prev (PCG pass) or x (refresh pass).
template <class S>
struct GatherGraph {
  const GScal<S>* sc;
  const S* z;
  const S* x;
  const S* p0;
  const S* p1;
  const S* v;  // x (refresh) or z (PCG), set by ready()
  const S* pprev;
  S beta;
  bool first, pcg;
  __device__ __forceinline__ bool ready() {
    pdl_wait();
    if (sc->done) return false;
    const int n = sc->n;
    pcg = sc->phase == 0;
    beta = sc->beta;
    first = n == 0;
    v = pcg ? z : x;
    pprev = ((n + 1) & 1) ? p1 : p0;
    return true;
  }
  __device__ __forceinline__ S operator()(std::int32_t cam, int i) const {
    const std::size_t k = std::size_t(cam) * 9 + i;
    const S a = __ldg(v + k);
    return (!pcg || first) ? a : a + beta * __ldg(pprev + k);
  }
  struct Raw {
    S v, pp;
  };
  __device__ __forceinline__ Raw raw(std::int32_t cam, int i) const { return raw_at(int(cam) * 9 + i); }
  __device__ __forceinline__ Raw raw_at(int k) const {
    return {__ldg(v + k), (!pcg || first) ? S(0) : __ldg(pprev + k)};
  }
  __device__ __forceinline__ S combine(const Raw& r) const { return (!pcg || first) ? r.v : r.v + beta * r.pp; }
};

// Loop decision after rho / |r|^2 of iteration state n (dba/solver.hpp:223-230).
template <class S>
__device__ __forceinline__ bool continue_loop(GScal<S>* sc) {
  bool loop = sqrt(sc->rnorm2) > sc->tol * sqrt(sc->rhs_norm2) && sc->n < sc->max_iters;
  if (loop && (!(sc->rho > 0.0) || isinf(sc->rho))) {
    sc->status = 1;
    loop = false;
  }
  return loop;
}

// Lanes 0..26 of each warp: 3 cameras x 9 rows (thread = row of a camera).
__device__ __forceinline__ bool camera_lane(std::int32_t m, std::int32_t& cam, int& row, int& base) {
  const int lane = threadIdx.x & 31;
  const std::int64_t warp = (blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x) >> 5;
  row = lane % 9;
  base = lane - row;
  cam = std::int32_t(warp * 3 + lane / 9);
  return lane < 27 && cam < m;
}

// z = B^-1 r for a camera whose 9 rows sit in lanes base..base+8.
template <class S>
__device__ __forceinline__ S precond_lane(const S* Binv, std::int32_t cam, int row, int base, S rrow) {
  const S* bi = Binv + std::size_t(cam) * 81 + row * 9;
  S z = S(0);
#pragma unroll
  for (int k = 0; k < 9; ++k) z += bi[k] * __shfl_sync(0xffffffffu, rrow, base + k);
  return z;
}

// x = 0, r = g, z = B^-1 g, rho, |g|^2; sets the WHILE condition.
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_g_init(GBufs<S> B, RedWs ws, GScal<S>* sc,
                                                        cudaGraphConditionalHandle h_while) {
  std::int32_t cam;
  int row, base;
  const bool on = camera_lane(B.m, cam, row, base);
  double rho = 0.0, rn = 0.0;
  const std::size_t i = on ? std::size_t(cam) * 9 + row : 0;
  const S gi = on ? B.g[i] : S(0);
  const S zi = precond_lane(B.Binv, on ? cam : 0, row, base, gi);
  if (on) {
    B.x[i] = S(0);
    B.r[i] = gi;
    B.z[i] = zi;
    rho = double(gi) * double(zi);
    rn = double(gi) * double(gi);
  }
  const double v[2] = {rho, rn};
  __shared__ double fin[2];
  if (grid_reduce<SumOp, 2>(v, ws.partials, ws.counter, fin) && threadIdx.x == 0) {
    sc->rho = fin[0];
    sc->rnorm2 = fin[1];
    sc->rhs_norm2 = fin[1];
    sc->rho_prev = 0.0;
    sc->n = 0;
    sc->status = 0;
    sc->beta = S(0);
    sc->phase = 0;
    sc->dse_count = fin[1] != 0.0 ? 1 : 0;  // the reference's DSE on x0 (dba/solver.hpp:217)
    const bool loop = fin[1] != 0.0 && continue_loop(sc);
    sc->done = loop ? 0 : 1;
    set_conditional(h_while, loop ? 1u : 0u);
  }
}

// One camera, one warp: c = fold of the camera's partials in chunk order
// (lanes strided, fixed shuffle tree); v = p = z + beta p_prev (PCG pass,
// stored as p) or x (refresh pass); q = B_d v - c; the p.q term in double.
template <class S>
__device__ __forceinline__ void camera_fold(const GBufs<S>& B, std::int32_t cam, int lane, int n, S beta, bool pcg) {
  S acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = S(0);
  const std::size_t at = std::size_t(cam) * 9;
  const int row = lane < 9 ? lane : 0;
  if (B.c_total) {  // already folded and summed over ranks
    acc[0] = B.c_total[at + row];
  } else {
    for (std::int32_t k = B.cam_part_ptr[cam] + lane; k < B.cam_part_ptr[cam + 1]; k += 32) {
      const S* pp = B.part + std::size_t(k) * 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += pp[i];
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
      acc[i] = __shfl_sync(0xffffffffu, acc[i], 0);
    }
  }
  S v;
  if (pcg) {
    const S zr = B.z[at + row];
    v = n == 0 ? zr : zr + beta * p_cur(B, n + 1)[at + row];
    if (lane < 9) p_cur(B, n)[at + row] = v;
  } else {
    v = B.x[at + row];
  }
  S d = S(0);
#pragma unroll
  for (int k = 0; k < 9; ++k) d += B.Bd[std::size_t(cam) * 81 + row * 9 + k] * __shfl_sync(0xffffffffu, v, k);
  S c = acc[0];
  if (!B.c_total)
#pragma unroll
    for (int i = 1; i < 9; ++i)
      if (row == i) c = acc[i];
  const S qv = d - c;
  double pq = 0.0;
  if (lane < 9) {
    B.q[at + row] = qv;
    pq = double(v) * double(qv);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pq += __shfl_down_sync(0xffffffffu, pq, o);
  if (lane == 0) B.pq_cam[cam] = pq;
}

// The body's DSE pass: CTAs [0, n_long) take the long tiles, the rest one
// chunk each (GatherGraph).
template <class S, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(kTile, pass_min_blocks<T, S>()) k_g_pass(DseArgs<S, T> A, GBufs<S> B, const GScal<S>* sc) {
  __shared__ DseWork<S> sm;
  pdl_allow_dependents();
  const std::int32_t blk = blockIdx.x;
  const GatherGraph<S> gx{sc, B.z, B.x, B.p0, B.p1, nullptr, nullptr, S(0), false, true};
#if DBAG_GTIMING
  if (blk == 0 && threadIdx.x == 0) {
    unsigned long long t_s;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_s));
    pdl_wait();
    tl_mark(sc->n, 0);
    if (sc->n < 1024) g_tl[sc->n * kTlStride + 7] = t_s;
  }
#endif
  if (blk < A.n_long)
    dse_long<S, 0, L>(A, sm, blk, gx);
  else
    dse_chunk<S, 0, L>(A, sm, blk - A.n_long, gx);
}

// Finish of an iteration: rho_prev, rho, |r|^2, n + 1, beta, loop decision.
template <class S>
__device__ __forceinline__ void finish_iteration(GScal<S>* sc, double rho, double rn2,
                                                 cudaGraphConditionalHandle h_while) {
  sc->rho_prev = sc->rho;
  sc->rho = rho;
  sc->rnorm2 = rn2;
  sc->n += 1;
  sc->beta = S(rho / sc->rho_prev);
  const bool loop = continue_loop(sc);
  sc->done = loop ? 0 : 1;
  set_conditional(h_while, loop ? 1u : 0u);
}

// Camera fold of the pass: warp per camera (camera_fold).
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_g_fold(GBufs<S> B, const GScal<S>* sc) {
  pdl_allow_dependents();
  pdl_wait();
  if (sc->done) return;
  const int n = sc->n;
  DBAG_TL(n, 1, blockIdx.x == 0 && threadIdx.x == 0);
  const std::int32_t cam = std::int32_t((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (cam < B.m) camera_fold(B, cam, threadIdx.x & 31, n, sc->beta, sc->phase == 0);
}

// End of a body pass (dba/solver.hpp:238-254). PCG pass: p'q = sum of the
// per-camera terms (every CTA folds them in camera order: same value
// everywhere), breakdown check, alpha; x += alpha p; then either
// r -= alpha q, z = B^-1 r, rho, |r|^2 and the loop decision, or (every 50th
// iteration) hand over to a refresh pass. Refresh pass (q = S x): r = g - q,
// z, rho, |r|^2 and the loop decision. sc is written only by the CTA that
// finishes the grid reduction, after every CTA has read it.
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_g_step(GBufs<S> B, RedWs ws, GScal<S>* sc,
                                                        cudaGraphConditionalHandle h_while) {
  __shared__ double red[32];
  __shared__ double pq_all;
  pdl_allow_dependents();
  pdl_wait();
  if (sc->done) return;
  const int n = sc->n;
  DBAG_TL(n, 2, blockIdx.x == 0 && threadIdx.x == 0);
  const bool refresh_pass = sc->phase != 0;
  S alpha = S(0);
  double pq = 0.0;
  if (!refresh_pass) {
    for (std::int32_t c = threadIdx.x; c < B.m; c += blockDim.x) pq += __ldcg(B.pq_cam + c);
    pq = block_reduce<SumOp>(pq, red);
    if (threadIdx.x == 0) pq_all = pq;
    __syncthreads();
    pq = pq_all;
    if (!(pq > 0.0) || isinf(pq)) {  // p'q breakdown (uniform across the grid)
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->pq = pq;
        sc->status = 2;
        sc->dse_count += 1;
        sc->done = 1;
        set_conditional(h_while, 0u);
      }
      return;
    }
    alpha = S(sc->rho / pq);
  }
  const bool hand_over = !refresh_pass && (n + 1) % 50 == 0;
  std::int32_t cam;
  int row, base;
  const bool on = camera_lane(B.m, cam, row, base);
  const std::size_t i = on ? std::size_t(cam) * 9 + row : 0;
  S ri = S(0);
  if (refresh_pass) {
    if (on) ri = B.g[i] - B.q[i];
  } else if (on) {
    B.x[i] = B.x[i] + alpha * p_cur(B, n)[i];
    if (!hand_over) ri = B.r[i] - alpha * B.q[i];
  }
  double rho = 0.0, rn = 0.0;
  if (!hand_over) {
    const S zi = precond_lane(B.Binv, on ? cam : 0, row, base, ri);
    if (on) {
      B.r[i] = ri;
      B.z[i] = zi;
      rho = double(ri) * double(zi);
      rn = double(ri) * double(ri);
    }
  }
  const double v[2] = {rho, rn};
  __shared__ double fin[2];
  if (grid_reduce<SumOp, 2>(v, ws.partials, ws.counter, fin) && threadIdx.x == 0) {
    DBAG_TL(n, 3, true);
    sc->dse_count += 1;
    if (!refresh_pass) {
      sc->pq = pq;
      sc->alpha = alpha;
    }
    if (hand_over) {
      sc->phase = 1;
      set_conditional(h_while, 1u);
    } else {
      sc->phase = 0;
      finish_iteration(sc, fin[0], fin[1], h_while);
    }
  }
}

// Software grid barrier over co-resident CTAs: one monotonically increasing
// 64-bit arrival counter (never reset), so a barrier costs one atomic and
// the polls; the target is the next multiple of gridDim.x. Only for kernels
// whose CTAs are all co-resident: k_g_fs runs at most as many CTAs as the
// SMs hold (checked at graph build) and its PDL dependents cannot launch
// before every one of its CTAs has started.
__device__ __forceinline__ void grid_barrier(unsigned long long* count) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(count, 1ull);
    const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
    while (*reinterpret_cast<volatile unsigned long long*>(count) < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// Camera fold + PCG step in one kernel (m <= 8 x grid): one warp per camera,
// lane = row. The camera's B_d and B^-1 rows and its partial range are
// constant during the solve and are loaded before waiting on the pass; after
// it, every vector row the camera needs and the first partial rows are
// loaded in one round trip, before the scalars are checked:
//   c = fold(partials), v = p = z + beta p_prev (stored) or x (refresh),
//   q = B_d v - c, p.q per warp -> per-CTA sum (warp order) -> slot
//   blockIdx.x of pq_cam; grid barrier; p'q = sum of the CTA slots (one warp,
//   fixed tree: the same bits in every CTA), alpha; x += alpha p; r -= alpha
//   q (or r = g - q after a refresh pass); z = B^-1 r; rho, |r|^2 -> grid
//   reduce; the last CTA advances the scalars and sets the WHILE condition.
// Same per-camera arithmetic as k_g_fold + k_g_step; the cross-camera sums
// (p'q, rho, |r|^2) are associated differently (both fixed, deterministic).
// Measured against the plain form (scalars first, one partial row per load,
// every CTA summing all m camera terms): venice 14.3 -> 13.5 us per
// iteration outside the pass.
template <class S>
__global__ void __maxnreg__(128) k_g_fs(GBufs<S> B, RedWs ws, GScal<S>* sc,  // 125 registers, no spill
                                                      cudaGraphConditionalHandle h_while, unsigned long long* bar) {
  __shared__ double red[32];
  __shared__ double pq_all;
  pdl_allow_dependents();
  const int lane = threadIdx.x & 31;
  const int row = lane < 9 ? lane : 0;
  const std::int32_t cam = std::int32_t((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const bool on = cam < B.m;
  const std::int32_t c = on ? cam : 0;
  const std::int32_t k0 = B.cam_part_ptr[c], k1 = on ? B.cam_part_ptr[c + 1] : k0;
  S bd[9], bi[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    bd[k] = B.Bd[std::size_t(c) * 81 + row * 9 + k];
    bi[k] = B.Binv[std::size_t(c) * 81 + row * 9 + k];
  }
  pdl_wait();
#if DBAG_GTIMING
  unsigned long long t_w;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_w));
#endif
  // plain loads (L1 path): LDG.STRONG.GPU (__ldcg) measured slower here;
  // the producers are previous kernels, complete at the PDL wait
  const int done = sc->done, n = sc->n, phase = sc->phase;
  const S beta = sc->beta;
  const double rho_cur = sc->rho;
  // nothing below waits on the scalars before the fold's loads are out: both
  // p buffers are read (n picks one later), the partials in batches of
  // kFsBatch lane-strided rows (the same add order as one row at a time),
  // and the done check follows the fold
  const std::size_t at = std::size_t(c) * 9 + row;
  const S zr = *(B.z + at), pa = *(B.p0 + at), pb = *(B.p1 + at), xr = *(B.x + at);
  const S rr = *(B.r + at), gr = *(B.g + at);
  S acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = S(0);
  for (std::int32_t k = k0 + lane; k < k1; k += 32 * kFsBatch) {
    S v[kFsBatch][9];
#pragma unroll
    for (int q = 0; q < kFsBatch; ++q) {
      const bool in = k + 32 * q < k1;
      const S* p = B.part + std::size_t(in ? k + 32 * q : k) * 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) v[q][i] = in ? *(p + i) : S(0);
    }
#pragma unroll
    for (int q = 0; q < kFsBatch; ++q)
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += v[q][i];
  }
  if (done) return;
  const S pp = ((n + 1) & 1) ? pb : pa;  // p_cur(B, n + 1)
#if DBAG_GTIMING
  if (blockIdx.x == 0 && threadIdx.x == 0 && n < 1024) g_tl[n * kTlStride + 1] = t_w;
#endif
  DBAG_TL(n, 2, blockIdx.x == 0 && threadIdx.x == 0);
  const bool pcg = phase == 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
    acc[i] = __shfl_sync(0xffffffffu, acc[i], 0);
  }
  S cr = acc[0];
#pragma unroll
  for (int i = 1; i < 9; ++i)
    if (row == i) cr = acc[i];
  const S v = pcg ? (n == 0 ? zr : zr + beta * pp) : xr;
  if (pcg && on && lane < 9) p_cur(B, n)[at] = v;
  S d = S(0);
#pragma unroll
  for (int k = 0; k < 9; ++k) d += bd[k] * __shfl_sync(0xffffffffu, v, k);
  const S qv = d - cr;
  S alpha = S(0);
  double pq = 0.0;
  bool hand_over = false;
  S ri = S(0);
  if (pcg) {
    double t = lane < 9 ? double(v) * double(qv) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    // p'q: each CTA sums its warps' cameras in warp order into slot
    // blockIdx.x of pq_cam; after the barrier one warp per CTA sums the
    // gridDim.x slots (lane-strided, fixed xor tree): the same bits in every CTA
    if (lane == 0) red[threadIdx.x >> 5] = on ? t : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) b += red[w];
      B.pq_cam[blockIdx.x] = b;
    }
    DBAG_TL(n, 3, blockIdx.x == 0 && threadIdx.x == 0);
    grid_barrier(bar);
    DBAG_TL(n, 4, blockIdx.x == 0 && threadIdx.x == 0);
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (unsigned k = lane; k < gridDim.x; k += 32) s += __ldcg(B.pq_cam + k);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) pq_all = s;
    }
    __syncthreads();
    pq = pq_all;
    DBAG_TL(n, 5, blockIdx.x == 0 && threadIdx.x == 0);
    if (!(pq > 0.0) || isinf(pq)) {  // p'q breakdown (uniform across the grid)
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->pq = pq;
        sc->status = 2;
        sc->dse_count += 1;
        sc->done = 1;
        set_conditional(h_while, 0u);
      }
      return;
    }
    alpha = S(rho_cur / pq);
    hand_over = (n + 1) % 50 == 0;
    if (on && lane < 9) B.x[at] = xr + alpha * v;
    if (!hand_over) ri = rr - alpha * qv;
  } else {
    ri = gr - qv;
  }
  double rho = 0.0, rn = 0.0;
  if (!hand_over) {
    S zi = S(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) zi += bi[k] * __shfl_sync(0xffffffffu, ri, k);
    if (on && lane < 9) {
      B.r[at] = ri;
      B.z[at] = zi;
      rho = double(ri) * double(zi);
      rn = double(ri) * double(ri);
    }
  }
  const double vv[2] = {rho, rn};
  __shared__ double fin[2];
  if (grid_reduce<SumOp, 2>(vv, ws.partials, ws.counter, fin) && threadIdx.x == 0) {
    DBAG_TL(n, 6, true);
    sc->dse_count += 1;
    if (pcg) {
      sc->pq = pq;
      sc->alpha = alpha;
    }
    if (hand_over) {
      sc->phase = 1;
      set_conditional(h_while, 1u);
    } else {
      sc->phase = 0;
      finish_iteration(sc, fin[0], fin[1], h_while);
    }
  }
}


// Camera fold + PCG step for small m as ONE thread-block cluster (<= 16 CTAs
// of 544 threads, warp per camera, CPW cameras per warp): the p'q and
// rho / |r|^2 reductions go through distributed shared memory and hardware
// cluster barriers instead of global atomics, a software grid barrier and a
// last-block pass. Same per-camera arithmetic as k_g_fs; the cross-camera
// sums are taken in fixed (CTA, warp, camera) order, so deterministic.
constexpr int kFscThreads = 544;  // 17 warps: a 16-CTA cluster covers 272 cameras with one camera per warp
constexpr int kFscWarps = kFscThreads / 32;

// Cluster sums over distributed shared memory without remote reads: before
// the cluster barrier each CTA pushes its value into slot [its rank] of the
// inbox of every CTA that needs the sum (remote stores, issued in parallel
// by the lanes of one warp); after it, a warp reduces its local inbox in a
// fixed tree order, so every CTA gets the same bits and no CTA has to wait
// for another to finish reading before it exits.
__device__ __forceinline__ void cluster_push(const cooperative_groups::cluster_group& cluster, double* inbox,
                                             int rank, double v, int lane, int to_lo, int to_hi) {
  const int r = to_lo + lane;
  if (r < to_hi) *cluster.map_shared_rank(inbox + rank, r) = v;
}
__device__ __forceinline__ double inbox_sum(const double* inbox, int lane, int ncta) {
  double t = lane < ncta ? inbox[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  return t;  // lane 0
}

template <class S, int CPW>
__global__ void __launch_bounds__(kFscThreads, 1) k_g_fsc(GBufs<S> B, GScal<S>* sc, cudaGraphConditionalHandle h_while) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double w_pq[kFscWarps], w_rho[kFscWarps], w_rn[kFscWarps];
  __shared__ double in_pq[32], in_rho[32], in_rn[32];  // cluster_push inboxes, one slot per CTA
  __shared__ double pq_all;
  pdl_allow_dependents();
  // phase 0 of the cluster barrier: arrive now, wait before the first
  // remote store (every CTA of the cluster has started by then)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = lane < 9 ? lane : 0;
  const int rank = int(cluster.block_rank()), ncta = int(cluster.num_blocks());
  std::int32_t cam[CPW], k0[CPW], k1[CPW];
  bool on[CPW];
  S bd[CPW][9], bi[CPW][9];
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    const std::int32_t c = (rank * kFscWarps + warp) + j * ncta * kFscWarps;
    on[j] = c < B.m;
    cam[j] = on[j] ? c : 0;
    k0[j] = B.cam_part_ptr[cam[j]];
    k1[j] = on[j] ? B.cam_part_ptr[cam[j] + 1] : k0[j];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      bd[j][k] = B.Bd[std::size_t(cam[j]) * 81 + row * 9 + k];
      bi[j][k] = B.Binv[std::size_t(cam[j]) * 81 + row * 9 + k];
    }
  }
  pdl_wait();
  // the scalars, every vector row (both p buffers: n picks one) and the
  // partials go out in one round trip; the done check follows the fold
  const int done = sc->done, n = sc->n, phase = sc->phase;
  const S beta = sc->beta;
  const double rho_cur = sc->rho;
  S v[CPW], qv[CPW], xr[CPW], rr[CPW], gr[CPW], zr[CPW], pa[CPW], pb[CPW], cr[CPW];
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    const std::size_t at = std::size_t(cam[j]) * 9 + row;
    zr[j] = B.z[at];
    pa[j] = B.p0[at];
    pb[j] = B.p1[at];
    xr[j] = B.x[at];
    rr[j] = B.r[at];
    gr[j] = B.g[at];
    S acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = S(0);
    for (std::int32_t k = k0[j] + lane; k < k1[j]; k += 32) {
      const S* pa = B.part + std::size_t(k) * 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += pa[i];
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
      acc[i] = __shfl_sync(0xffffffffu, acc[i], 0);
    }
    cr[j] = acc[0];
#pragma unroll
    for (int i = 1; i < 9; ++i)
      if (row == i) cr[j] = acc[i];
  }
  if (done != 0 || n < 0 || beta != beta) return;  // uniform over the cluster (n < 0, NaN beta: never)
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  DBAG_TL(n, 1, rank == 0 && threadIdx.x == 0);
  DBAG_TL(n, 2, rank == 0 && threadIdx.x == 0);
  const bool pcg = phase == 0;
  double pq_w = 0.0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    const std::size_t at = std::size_t(cam[j]) * 9 + row;
    const S pp = ((n + 1) & 1) ? pb[j] : pa[j];  // p_cur(B, n + 1)
    v[j] = pcg ? (n == 0 ? zr[j] : zr[j] + beta * pp) : xr[j];
    if (pcg && on[j] && lane < 9) p_cur(B, n)[at] = v[j];
    S d = S(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) d += bd[j][k] * __shfl_sync(0xffffffffu, v[j], k);
    qv[j] = d - cr[j];
    double t = (lane < 9 && on[j]) ? double(v[j]) * double(qv[j]) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    pq_w += t;  // lane 0: this warp's cameras in order
  }
  S alpha = S(0);
  double pq = 0.0;
  bool hand_over = false;
  if (pcg) {
    if (lane == 0) w_pq[warp] = pq_w;
    __syncthreads();
    if (warp == 0) {
      double b = 0.0;
      for (int w = 0; w < kFscWarps; ++w) b += w_pq[w];
      cluster_push(cluster, in_pq, rank, b, lane, 0, ncta);  // to every CTA
    }
    DBAG_TL(n, 3, rank == 0 && threadIdx.x == 0);
    cluster.sync();
    DBAG_TL(n, 4, rank == 0 && threadIdx.x == 0);
    if (warp == 0) {
      const double t = inbox_sum(in_pq, lane, ncta);
      if (lane == 0) pq_all = t;
    }
    __syncthreads();
    pq = pq_all;
    DBAG_TL(n, 5, rank == 0 && threadIdx.x == 0);
    if (!(pq > 0.0) || isinf(pq)) {  // p'q breakdown (uniform over the cluster)
      if (rank == 0 && threadIdx.x == 0) {
        sc->pq = pq;
        sc->status = 2;
        sc->dse_count += 1;
        sc->done = 1;
        set_conditional(h_while, 0u);
      }
      return;
    }
    alpha = S(rho_cur / pq);
    hand_over = (n + 1) % 50 == 0;
  }
  double rho_w = 0.0, rn_w = 0.0;
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    const std::size_t at = std::size_t(cam[j]) * 9 + row;
    S ri = S(0);
    if (pcg) {
      if (on[j] && lane < 9) B.x[at] = xr[j] + alpha * v[j];
      if (!hand_over) ri = rr[j] - alpha * qv[j];
    } else {
      ri = gr[j] - qv[j];
    }
    if (!hand_over) {
      S zi = S(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) zi += bi[j][k] * __shfl_sync(0xffffffffu, ri, k);
      double rho = 0.0, rn = 0.0;
      if (on[j] && lane < 9) {
        B.r[at] = ri;
        B.z[at] = zi;
        rho = double(ri) * double(zi);
        rn = double(ri) * double(ri);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rho += __shfl_down_sync(0xffffffffu, rho, o);
        rn += __shfl_down_sync(0xffffffffu, rn, o);
      }
      rho_w += rho;
      rn_w += rn;
    }
  }
  if (lane == 0) {
    w_rho[warp] = rho_w;
    w_rn[warp] = rn_w;
  }
  __syncthreads();
  if (warp == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kFscWarps; ++w) {
      a += w_rho[w];
      b += w_rn[w];
    }
    cluster_push(cluster, in_rho, rank, a, lane, 0, 1);  // to CTA 0
    cluster_push(cluster, in_rn, rank, b, lane, 0, 1);
  }
  cluster.sync();
  if (rank != 0) return;
  double rho = 0.0, rn = 0.0;
  if (warp == 0) {
    rho = inbox_sum(in_rho, lane, ncta);
    rn = inbox_sum(in_rn, lane, ncta);
  }
  if (rank == 0 && threadIdx.x == 0) {
    DBAG_TL(n, 6, true);
    sc->dse_count += 1;
    if (pcg) {
      sc->pq = pq;
      sc->alpha = alpha;
    }
    if (hand_over) {
      sc->phase = 1;
      set_conditional(h_while, 1u);
    } else {
      sc->phase = 0;
      finish_iteration(sc, rho, rn, h_while);
    }
  }
}

}  // namespace dev
}  // namespace dbag
