// pcg.cuh — DPCG as one persistent cooperative kernel (single rank).
//
// dpcg (dba/solver.hpp:202-257) with the reduced camera operator applied by
// the fused DSE pass (dse.cuh) and every recurrence on the device: one
// launch runs the whole inner solve, so the LM loop pays one launch and one
// host read per trial instead of ~6 launches + a host round trip per PCG
// iteration. Phases are separated by a software grid barrier (all CTAs are
// co-resident: cooperative launch); the scalar reductions are computed
// redundantly by every CTA from per-CTA partials in a fixed order, so every
// CTA takes identical branches and the result is deterministic.
//
// Per iteration n (refresh iterations, (n+1) % 50 == 0, add one DSE on x):
//   B  DSE of p, p = z (n = 0) or z + beta p_prev formed on the fly   | barrier
//   C  per camera: c = fold(partials), q = B_d p - c, p.q partials    | barrier
//   D  x += alpha p, r -= alpha q, z = B^-1 r (explicit block inverse),
//      rho = r.z and |r|^2 partials                                   | barrier
// Breakdown checks (rho, p'q non-finite or <= 0) and the stopping rule
// |r| <= tol |g| or n == max_iters are the reference's, in its order.
#pragma once

#include <cstdint>

#include "dse.cuh"

namespace dbag {
namespace dev {

struct PcgDevOut {
  int iterations, converged, status, dse_count;
  double rho, pq, rnorm2, rhs_norm2;
};

template <class S>
struct PcgPArgs {
  DseArgs<S> dse;
  std::int32_t m;
  const std::int32_t* cam_part_ptr;
  const S* Bd;    // damped B, 81 per camera
  const S* Binv;  // explicit inverse of damped B, 81 per camera
  const S* g;
  S* x;
  S* r;
  S* z;
  S* pa;
  S* pb;
  S* q;
  double tol;
  int max_iters;
  double* bpart;  // 4 x gridDim.x
  unsigned* bar;  // [count, generation]
  PcgDevOut* out;
};

constexpr int kCamsPerGroup = kTile / 9;  // 14 cameras x 9 rows per CTA sweep

// Software grid barrier over co-resident CTAs; traps instead of hanging.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned long long spins = 0;
      while (*gen == g0) {
        __nanosleep(64);
        if (++spins > (1ull << 27)) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Block sum (fixed tree) of v into slot[blockIdx.x].
__device__ __forceinline__ void block_partial(double v, double* slot, double* red) {
  v = warp_reduce<SumOp>(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kTile / 32; ++w) s += red[w];
    slot[blockIdx.x] = s;
  }
  __syncthreads();
}

// Sum of the G per-block partials, same order in every CTA; all threads get it.
__device__ __forceinline__ double grid_fold(const double* v, double* red) {
  double s = 0.0;
  if (threadIdx.x < 32) {
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) s += __ldcg(v + i);
    s = warp_reduce<SumOp>(s);
    if (threadIdx.x == 0) red[4] = s;
  }
  __syncthreads();
  s = red[4];
  __syncthreads();
  return s;
}

template <class S>
__device__ __forceinline__ void dse_phase(const PcgPArgs<S>& P, DseWork<S>& sm, DseStages<S>* st, unsigned& parity,
                                          const GatherP<S>& gp) {
  if (st) {
    dse_stream_pass<S, 0>(P.dse, sm, *st, parity, gp);
  } else {
    for (std::int32_t c = blockIdx.x; c < P.dse.n_chunks; c += gridDim.x) dse_chunk<S, 0>(P.dse, sm, c, gp);
    for (std::int32_t l = blockIdx.x; l < P.dse.n_long; l += gridDim.x) dse_long<S, 0>(P.dse, sm, l, gp);
  }
}

// Phase C: q = B_d v - fold(partials) per camera (warp per camera); returns
// this thread's share of v.q.
template <class S>
__device__ __forceinline__ double camera_phase(const PcgPArgs<S>& P, const S* v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double vq = 0.0;
  for (std::int32_t cam = blockIdx.x * (kTile / 32) + warp; cam < P.m; cam += gridDim.x * (kTile / 32)) {
    S acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = S(0);
    for (std::int32_t k = P.cam_part_ptr[cam] + lane; k < P.cam_part_ptr[cam + 1]; k += 32) {
      const S* pp = P.dse.part + std::size_t(k) * 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += __ldcg(pp + i);
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
      acc[i] = __shfl_sync(0xffffffffu, acc[i], 0);
    }
    if (lane < 9) {
      S c = acc[0];
#pragma unroll
      for (int i = 1; i < 9; ++i)
        if (lane == i) c = acc[i];
      const S* b = P.Bd + std::size_t(cam) * 81 + lane * 9;
      const S* vv = v + std::size_t(cam) * 9;
      S d = S(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) d += __ldg(b + k) * __ldcg(vv + k);
      const S qv = d - c;
      P.q[std::size_t(cam) * 9 + lane] = qv;
      vq += double(__ldcg(vv + lane)) * double(qv);
    }
  }
  return vq;
}

// Camera-group sweep: this thread's element of camera cb*14 + tid/9.
template <class S, class F>
__device__ __forceinline__ void camera_groups(const PcgPArgs<S>& P, S* rs, F&& f) {
  const int tid = threadIdx.x;
  const int lc = tid / 9, row = tid % 9;
  for (std::int32_t cb = blockIdx.x; cb * kCamsPerGroup < P.m; cb += gridDim.x) {
    const std::int32_t cam = cb * kCamsPerGroup + lc;
    const bool on = tid < kCamsPerGroup * 9 && cam < P.m;
    f(on, cam, row, rs + lc * 9);
    __syncthreads();
  }
}

// z = B^-1 r for this thread's row, r of the camera staged in rs.
template <class S>
__device__ __forceinline__ S precond_row(const PcgPArgs<S>& P, std::int32_t cam, int row, const S* rs) {
  const S* bi = P.Binv + std::size_t(cam) * 81 + row * 9;
  S z = S(0);
#pragma unroll
  for (int k = 0; k < 9; ++k) z += __ldg(bi + k) * rs[k];
  return z;
}

template <class S, bool TMA>
__global__ void __launch_bounds__(kTile, TMA ? 3 : 5) k_pcg_persistent(PcgPArgs<S> P) {
  __shared__ DseWork<S> sm;
  __shared__ S rs[kTile];
  __shared__ double red[8];
  extern __shared__ __align__(128) unsigned char pcg_dyn[];
  DseStages<S>* st = TMA ? reinterpret_cast<DseStages<S>*>(pcg_dyn) : nullptr;
  if (TMA) stages_init(*st);
  unsigned parity = 0;
  const int G = gridDim.x;
  double* part_rho = P.bpart;
  double* part_rn = P.bpart + G;
  double* part_pq = P.bpart + 2 * G;
  // x = 0, r = g, z = B^-1 g, rho = r.z, |r|^2
  double lrho = 0.0, lrn = 0.0;
  camera_groups(P, rs, [&](bool on, std::int32_t cam, int row, S* rc) {
    const std::size_t i = std::size_t(cam) * 9 + row;
    S gi = S(0);
    if (on) {
      gi = P.g[i];
      P.x[i] = S(0);
      P.r[i] = gi;
      rc[row] = gi;
    }
    __syncthreads();
    if (on) {
      const S zi = precond_row(P, cam, row, rc);
      P.z[i] = zi;
      lrho += double(gi) * double(zi);
      lrn += double(gi) * double(gi);
    }
  });
  block_partial(lrho, part_rho, red);
  block_partial(lrn, part_rn, red);
  grid_barrier(P.bar);
  double rho = grid_fold(part_rho, red);
  double rn2 = grid_fold(part_rn, red);
  const double rhs2 = rn2;
  const double rhs_norm = sqrt(rhs2);
  int n = 0, status = 0, dse_count = 0;
  double rho_prev = 0.0, pq = 0.0;
  S* pcur = P.pa;
  S* pnext = P.pb;
  if (rhs2 != 0.0) {
    dse_count = 1;  // the reference's DSE on x0 = 0 (dba/solver.hpp:217), S 0 = 0
    while (sqrt(rn2) > P.tol * rhs_norm && n < P.max_iters) {
      if (!(rho > 0.0) || isinf(rho)) {
        status = 1;
        break;
      }
      const S beta = n == 0 ? S(0) : S(rho / rho_prev);
      const GatherP<S> gp{P.z, pcur, beta, n == 0};
      dse_phase(P, sm, st, parity, gp);
      for (std::size_t i = std::size_t(blockIdx.x) * kTile + threadIdx.x; i < std::size_t(P.m) * 9;
           i += std::size_t(G) * kTile)
        pnext[i] = n == 0 ? __ldcg(P.z + i) : __ldcg(P.z + i) + beta * __ldcg(pcur + i);
      grid_barrier(P.bar);
      block_partial(camera_phase(P, pnext), part_pq, red);
      grid_barrier(P.bar);
      pq = grid_fold(part_pq, red);
      ++dse_count;
      if (!(pq > 0.0) || isinf(pq)) {
        status = 2;
        break;
      }
      const S alpha = S(rho / pq);
      const bool refresh = (n + 1) % 50 == 0;
      lrho = 0.0;
      lrn = 0.0;
      if (!refresh) {
        camera_groups(P, rs, [&](bool on, std::int32_t cam, int row, S* rc) {
          const std::size_t i = std::size_t(cam) * 9 + row;
          S ri = S(0);
          if (on) {
            P.x[i] = P.x[i] + alpha * __ldcg(pnext + i);
            ri = P.r[i] - alpha * __ldcg(P.q + i);
            P.r[i] = ri;
            rc[row] = ri;
          }
          __syncthreads();
          if (on) {
            const S zi = precond_row(P, cam, row, rc);
            P.z[i] = zi;
            lrho += double(ri) * double(zi);
            lrn += double(ri) * double(ri);
          }
        });
      } else {
        // x += alpha p, then r = g - S x (dba/solver.hpp:246-249)
        for (std::size_t i = std::size_t(blockIdx.x) * kTile + threadIdx.x; i < std::size_t(P.m) * 9;
             i += std::size_t(G) * kTile)
          P.x[i] = __ldcg(P.x + i) + alpha * __ldcg(pnext + i);
        grid_barrier(P.bar);
        dse_phase(P, sm, st, parity, GatherP<S>{P.x, P.x, S(0), true});
        grid_barrier(P.bar);
        camera_phase(P, P.x);
        grid_barrier(P.bar);
        ++dse_count;
        camera_groups(P, rs, [&](bool on, std::int32_t cam, int row, S* rc) {
          const std::size_t i = std::size_t(cam) * 9 + row;
          S ri = S(0);
          if (on) {
            ri = P.g[i] - __ldcg(P.q + i);
            P.r[i] = ri;
            rc[row] = ri;
          }
          __syncthreads();
          if (on) {
            const S zi = precond_row(P, cam, row, rc);
            P.z[i] = zi;
            lrho += double(ri) * double(zi);
            lrn += double(ri) * double(ri);
          }
        });
      }
      block_partial(lrho, part_rho, red);
      block_partial(lrn, part_rn, red);
      grid_barrier(P.bar);
      rho_prev = rho;
      rho = grid_fold(part_rho, red);
      rn2 = grid_fold(part_rn, red);
      ++n;
      S* t = pcur;
      pcur = pnext;
      pnext = t;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.out->iterations = n;
    P.out->converged = sqrt(rn2) <= P.tol * rhs_norm ? 1 : 0;
    P.out->status = status;
    P.out->dse_count = dse_count;
    P.out->rho = rho;
    P.out->pq = pq;
    P.out->rnorm2 = rn2;
    P.out->rhs_norm2 = rhs2;
  }
}

}  // namespace dev
}  // namespace dbag
