// pipe.cuh — the DSE pass as a persistent, TMA-fed software pipeline.
//
// Same arithmetic as dse_chunk_at (dse.cuh; dba/solver.hpp:149-181, one pass
// over E per DSE), restructured so that no dependent global load sits on the
// per-chunk critical path:
//   * persistent CTAs walk chunks c = blockIdx.x + j * gridDim.x; one thread
//     keeps kPipeStages chunk records in flight through the TMA engine
//     (cp.async.bulk + mbarrier complete_tx), so the E stream never waits on
//     the compute phases of a tile;
//   * a chunk touches few distinct cameras (nu ~ 4-11 on the BAL-shaped
//     rings), so the camera vector is gathered once per (chunk, camera) —
//     9 values per camera, not 9 per slot — one chunk AHEAD, into registers,
//     and staged in shared memory (xs) for the next chunk; the points' C
//     factors (and w) are likewise loaded one chunk ahead;
//   * the four phases of a chunk (a_s = E_s^T x, b_p = C_p^-1 sum a_s,
//     y_s = E_s b_p, per-camera fold) then run on shared memory and
//     registers only. y_s overwrites the slot's own E lanes in the stage copy
//     (each thread owns its slot), so the fold reads it from there.
// Partials are written to their camera-major slots exactly as dse_chunk_at
// does (deterministic, no atomics): the two kernels are interchangeable.
// Chunks of long tiles (points with > kTile observations) are skipped in the
// pipeline and finished afterwards by dse_long.
#pragma once

#include <cstdint>

#include "dse.cuh"
#include "tma.cuh"

namespace dbag {
namespace dev {

constexpr int kPipeStages = 3;
constexpr int kPipeCams = 28;  // distinct cameras per chunk staged in xs (2 gathers per thread); more: direct path
static_assert(kPipeCams <= kXsCams, "staged cameras need RecMeta::ucam");

template <class S>
struct PipeSmem {
  S rec[kPipeStages][Rec<S>::kLen];
  S xs[2][kPipeCams * 9];
  S a[kTile][3];
  S b[kTile][3];
  alignas(8) std::uint64_t full[kPipeStages];
};

// Two-step camera-vector gathers for the one-chunk-ahead prefetch: load()
// issues the loads, combine() forms the value where it is consumed.
template <class S>
struct PipeGatherX {
  const S* x;
  struct Raw {
    S v;
  };
  __device__ __forceinline__ bool ready() { return true; }
  __device__ __forceinline__ Raw load(std::int32_t cam, int i) const { return {__ldg(x + std::size_t(cam) * 9 + i)}; }
  __device__ __forceinline__ S combine(const Raw& r) const { return r.v; }
  __device__ __forceinline__ S operator()(std::int32_t cam, int i) const { return combine(load(cam, i)); }
};

template <class S>
__device__ __forceinline__ void pipe_issue(const DseArgs<S>& A, PipeSmem<S>& sm, std::int32_t c, int k) {
  mbar_arrive_expect_tx(&sm.full[k], std::uint32_t(Rec<S>::kBytes));
  bulk_g2s(sm.rec[k], A.rec + std::size_t(c) * Rec<S>::kLen, std::uint32_t(Rec<S>::kBytes), &sm.full[k]);
}

// Per-chunk values prefetched one chunk ahead (registers of the thread that
// consumes them): up to two (camera, row) gathers, the point's C factor,
// w (MODE 1/2) and its halo index.
template <class S, class G>
struct PipeAhead {
  typename G::Raw g0, g1;
  S L[9], wv[3];
  std::int32_t halo;
};

template <class S, int MODE, class G>
__device__ __forceinline__ void pipe_prefetch(const DseArgs<S>& A, const RecMeta& M, const G& gx,
                                              PipeAhead<S, G>& ah) {
  const int tid = threadIdx.x;
  const int nu = M.nu;
  if (MODE != 2 && nu <= kPipeCams && M.nchunk == 1) {
    const int nv = nu * 9;
    if (tid < nv) {
      const int u = tid / 9, i = tid - u * 9;
      ah.g0 = gx.load(M.ucam[u], i);
    }
    if (tid + kTile < nv) {
      const int t = tid + kTile, u = t / 9, i = t - u * 9;
      ah.g1 = gx.load(M.ucam[u], i);
    }
  }
  if (M.nchunk == 1 && tid < M.np) {
    const std::int32_t p = M.p0 + tid;
    load_point<S, MODE>(A, p, ah.L, ah.wv);
    ah.halo = (MODE != 2 && A.halo_of) ? A.halo_of[p] : -1;
  }
}

template <class S, int MODE, class G>
__device__ __forceinline__ void pipe_commit(const RecMeta& M, const G& gx, const PipeAhead<S, G>& ah, S* xs) {
  const int tid = threadIdx.x;
  const int nu = M.nu;
  if (MODE != 2 && nu <= kPipeCams && M.nchunk == 1) {
    const int nv = nu * 9;
    if (tid < nv) xs[tid] = gx.combine(ah.g0);
    if (tid + kTile < nv) xs[tid + kTile] = gx.combine(ah.g1);
  }
}

// Point finish with the prefetched factor / halo index (finish_point's
// arithmetic).
template <class S, int MODE>
__device__ __forceinline__ void pipe_finish_point(const DseArgs<S>& A, std::int32_t p, std::int32_t h, const S* L,
                                                  const S* wv, S* tt, S* b) {
  if (h >= 0) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      A.halo_buf[std::size_t(h) * 3 + j] = tt[j];
      b[j] = S(0);
    }
    return;
  }
  if (MODE == 1)
#pragma unroll
    for (int j = 0; j < 3; ++j) tt[j] = wv[j] - tt[j];
  if (MODE == 2)
#pragma unroll
    for (int j = 0; j < 3; ++j) tt[j] = wv[j];
  llt_solve<S, 3>(L, tt);
#pragma unroll
  for (int j = 0; j < 3; ++j) b[j] = tt[j];
  if (MODE == 1)
#pragma unroll
    for (int j = 0; j < 3; ++j) A.out_pt[std::size_t(p) * 3 + j] = b[j];
}

template <class S>
struct YLanes {  // y written over the stage's E lanes 0..8 (lane-major)
  const S* R;
  __device__ __forceinline__ S operator()(int o, int i) const { return R[i * kTile + o]; }
};

// One chunk from its landed stage R; xs holds its cameras' values (fast
// path) and ah its prefetched point data.
template <class S, int MODE, class G>
__device__ __forceinline__ void pipe_chunk(const DseArgs<S>& A, PipeSmem<S>& sm, S* R, const S* xs, const G& gx,
                                           const PipeAhead<S, G>& ah) {
  const int tid = threadIdx.x;
  const RecMeta& M = *reinterpret_cast<const RecMeta*>(R + Rec<S>::kE);
  const int nslots = M.nslots, np = M.np;
  S e[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) e[k] = R[k * kTile + tid];  // padding slots hold zeros
  if (MODE != 2) {
    S a[3] = {S(0), S(0), S(0)};
    if (tid < nslots) {
      if (M.nu <= kPipeCams) {
        const S* xv = xs + int(M.su[tid]) * 9;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          a[0] += e[i * 3 + 0] * xv[i];
          a[1] += e[i * 3 + 1] * xv[i];
          a[2] += e[i * 3 + 2] * xv[i];
        }
      } else {
        const std::int32_t cam = M.cam[tid];
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          const S xv = gx(cam, i);
          a[0] += e[i * 3 + 0] * xv;
          a[1] += e[i * 3 + 1] * xv;
          a[2] += e[i * 3 + 2] * xv;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) sm.a[tid][j] = a[j];
  }
  __syncthreads();
  if (tid < np) {
    S tt[3] = {S(0), S(0), S(0)}, b[3];
    if (MODE != 2)
      for (int q = M.pbeg[tid]; q < M.pbeg[tid + 1]; ++q)
#pragma unroll
        for (int j = 0; j < 3; ++j) tt[j] += sm.a[q][j];
    pipe_finish_point<S, MODE>(A, M.p0 + tid, ah.halo, ah.L, ah.wv, tt, b);
#pragma unroll
    for (int j = 0; j < 3; ++j) sm.b[tid][j] = b[j];
  }
  __syncthreads();
  if constexpr (MODE != 1) {
    const int pti = M.pt[tid];
    const S b0 = sm.b[pti][0], b1 = sm.b[pti][1], b2 = sm.b[pti][2];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i * kTile + tid] = (e[i * 3] * b0 + e[i * 3 + 1] * b1) + e[i * 3 + 2] * b2;
    __syncthreads();
    fold_cameras(A, M.nu, M.ubeg, M.uslot, M.upart, YLanes<S>{R});
  }
}

// The whole pass of one CTA. gx.ready() is called once, after the first
// records are in flight (graph pass: waits for the previous kernel and reads
// the PCG scalars); false drains the issued copies and returns.
template <class S, int MODE, class G>
__device__ __forceinline__ void pipe_pass(const DseArgs<S>& A, PipeSmem<S>& sm, G& gx) {
  const int tid = threadIdx.x;
  const std::int32_t first = blockIdx.x, stride = gridDim.x;
  const std::int32_t nmine = first < A.n_chunks ? (A.n_chunks - 1 - first) / stride + 1 : 0;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < kPipeStages; ++k) mbar_init(&sm.full[k], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (std::int32_t j = 0; j < nmine && j < kPipeStages; ++j) pipe_issue(A, sm, first + j * stride, int(j));
  if (!gx.ready()) {
    for (std::int32_t j = 0; j < nmine && j < kPipeStages; ++j) mbar_wait(&sm.full[j], 0u);
    return;
  }
  PipeAhead<S, G> ah;
  ah.halo = -1;
  if (nmine > 0) {
    mbar_wait(&sm.full[0], 0u);
    const RecMeta& M0 = *reinterpret_cast<const RecMeta*>(sm.rec[0] + Rec<S>::kE);
    pipe_prefetch<S, MODE>(A, M0, gx, ah);
    pipe_commit<S, MODE>(M0, gx, ah, sm.xs[0]);
  }
  __syncthreads();
  for (std::int32_t j = 0; j < nmine; ++j) {
    const int k = int(j % kPipeStages);
    S* R = sm.rec[k];
    const RecMeta& M = *reinterpret_cast<const RecMeta*>(R + Rec<S>::kE);
    PipeAhead<S, G> cur = ah;  // this chunk's point data
    const RecMeta* Mn = nullptr;
    if (j + 1 < nmine) {
      const int kn = int((j + 1) % kPipeStages);
      mbar_wait(&sm.full[kn], std::uint32_t(((j + 1) / kPipeStages) & 1));
      Mn = reinterpret_cast<const RecMeta*>(sm.rec[kn] + Rec<S>::kE);
      pipe_prefetch<S, MODE>(A, *Mn, gx, ah);
    }
    if (M.nchunk == 1) pipe_chunk<S, MODE>(A, sm, R, sm.xs[j & 1], gx, cur);
    if (Mn) pipe_commit<S, MODE>(*Mn, gx, ah, sm.xs[(j + 1) & 1]);
    // y was written into stage k through the generic proxy; order it before
    // the TMA (async proxy) refill of the same bytes.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // stage k and xs[j & 1] are free
    if (tid == 0 && j + kPipeStages < nmine) pipe_issue(A, sm, first + (j + kPipeStages) * stride, k);
  }
  if (A.n_long > 0) {
    // every stage is drained: reuse stage 0 as dse_long's work area
    static_assert(sizeof(DseWork<S>) <= sizeof(S) * Rec<S>::kLen, "DseWork must fit in one stage");
    DseWork<S>& w = *reinterpret_cast<DseWork<S>*>(sm.rec[0]);
    for (std::int32_t l = first; l < A.n_long; l += stride) dse_long<S, MODE>(A, w, l, gx);
  }
}

template <class S, int MODE>
__global__ void __launch_bounds__(kTile) k_dse_pipe(DseArgs<S> A) {
  extern __shared__ __align__(128) unsigned char pipe_dyn[];
  PipeSmem<S>& sm = *reinterpret_cast<PipeSmem<S>*>(pipe_dyn);
  PipeGatherX<S> gx{A.x};
  pipe_pass<S, MODE>(A, sm, gx);
}

}  // namespace dev
}  // namespace dbag
