// dse.cuh — the streaming pass over the coupling blocks E.
//
// One pass over E per DSE (dba/solver.hpp:149-181):
//   a_p = sum_s E_s^T x[cam_s]   b_p = C_p^-1 a_p   y_s = E_s b_p
// E is stored as 128-slot chunk records: 27 lanes x 128 slots (lane-major:
// thread i reads lane k at k*128 + i, fully coalesced) followed by the
// chunk's static metadata (RecMeta: cameras, slot -> point, slots grouped by
// camera, camera-major partial positions). One CTA per chunk, one thread per
// slot; every index the tile needs arrives with the record, so the only
// dependent loads are the camera-vector gathers (once per distinct camera
// and row, L1/L2-resident) and the points' C factors. The E block stays in
// registers between the two products, so each coupling block is read exactly
// once per DSE. y is folded per (chunk, camera, component): one thread per
// item sums the camera's slots in slot-list order (fold_items) and writes its
// camera-major partial; the camera fold (graph_pcg.cuh, or k_cam_reduce on
// the host-driven path) sums each camera's contiguous partials. No atomics
// anywhere: deterministic.
//
// MODE 0  DSE          a from x, b = C^-1 a, y -> partials
// MODE 1  back-subst.  a from x (= dx_c), out_pt = C^-1 (w - a)   (dba/solver.hpp:371-376)
// MODE 2  rhs          b = C^-1 w, y -> partials                  (dba/solver.hpp:358-360)
// Halo points (shared with other ranks; MODE 0/1) deposit a_p in halo_buf and
// are finished after the halo all-reduce (k_halo_fix / k_halo_finish).
// Points with more than 128 slots span several chunks ("long" tiles); their
// chunks are skipped by k_dse_chunk and handled by k_dse_long.
#pragma once
#ifndef DBAG_FOLD_ITEMS
#define DBAG_FOLD_ITEMS 1
#endif

#include <cstdint>

#include "kernels.cuh"

namespace dbag {
namespace dev {

// S: arithmetic type; T: storage type of the E lanes in the records (T = S,
// or float under FP64 arithmetic: SolverConfig coupling_fp32, row f4).
template <class S, class T = S>
struct DseArgs {
  std::int32_t n_chunks;
  const T* rec;
  const S* x;
  const S* Cinv;
  const S* w;
  const std::int32_t* halo_of;
  S* halo_buf;
  S* part;
  S* out_pt;
  const std::int32_t* long_chunk;  // first chunk of each long tile
  std::int32_t n_long;
  std::int32_t pf_dist;  // > 0: chunk c prefetches record c + pf_dist into L2
  const S* Rm;           // per-camera R (9m, row-major): factored records only
};

// Shared work area of a chunk pass: a (3 x kTile), b (3 x kTile) and the
// staged camera vectors xs, then y (9 x kTile) in its own buffer (20 KB per
// CTA in FP64): writing y needs no barrier after the b reads. Overlaying y
// on a/b/xs (DBAG_Y_OVERLAY=1, 11 KB) costs that barrier and measured 3 %
// slower per LM iteration (trafalgar and venice).
#ifndef DBAG_Y_OVERLAY
#define DBAG_Y_OVERLAY 0
#endif
// y rows padded to 10 scalars (DBAG_FOLD_PAIRS): the y-phase writes each row
// with 16-byte (FP64) stores and the fold reads two components per load
// (fold_pairs).
#ifndef DBAG_FOLD_PAIRS
#define DBAG_FOLD_PAIRS 1
#endif
static_assert(!(DBAG_FOLD_PAIRS && DBAG_Y_OVERLAY), "padded y rows do not fit the overlay");
constexpr int kYW = DBAG_FOLD_PAIRS ? 10 : 9;
template <class S>
struct alignas(16) DseWork {
  S buf[kTile * 9];
#if !DBAG_Y_OVERLAY
  S ybuf[kTile * kYW];
#endif
  S rs[kXsCams * 9];  // R of the chunk's distinct cameras (factored records)
  std::int32_t upart[kTile];
  std::uint8_t uslot[kTile];
  std::uint8_t ubeg[kTile + 8];
  __device__ __forceinline__ S (*a())[3] { return reinterpret_cast<S(*)[3]>(buf); }
  __device__ __forceinline__ S (*b())[3] { return reinterpret_cast<S(*)[3]>(buf + 3 * kTile); }
  __device__ __forceinline__ S* xs() { return buf + 6 * kTile; }
#if DBAG_Y_OVERLAY
  __device__ __forceinline__ S (*y())[9] { return reinterpret_cast<S(*)[9]>(buf); }
#else
  __device__ __forceinline__ S (*y())[kYW] { return reinterpret_cast<S(*)[kYW]>(ybuf); }
#endif
};
static_assert(6 * kTile + kXsCams * 9 <= 9 * kTile, "a, b and xs must fit under y");

template <class T, int L>
__device__ __forceinline__ const RecMeta& rec_meta(const T* R) {
  return *reinterpret_cast<const RecMeta*>(R + Rec<T, L>::kE);
}

// Point finish: halo deposit or b = C^-1 a (MODE 0), dx_p = C^-1 (w - a)
// (MODE 1), b = C^-1 w (MODE 2). Returns b (zero for halo points).
template <class S, int MODE, class T>
__device__ __forceinline__ void finish_point(const DseArgs<S, T>& A, std::int32_t p, const S* L, const S* wv, S* tt,
                                             S* b) {
  const std::int32_t h = (MODE != 2 && A.halo_of) ? A.halo_of[p] : -1;
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

// The point's C factor (and w for MODE 1/2), loaded early.
template <class S, int MODE, class T>
__device__ __forceinline__ void load_point(const DseArgs<S, T>& A, std::int32_t p, S* L, S* wv) {
#pragma unroll
  for (int k = 0; k < 9; ++k) L[k] = A.Cinv[std::size_t(p) * 9 + k];
  if (MODE != 0)
#pragma unroll
    for (int j = 0; j < 3; ++j) wv[j] = A.w[std::size_t(p) * 3 + j];
}

// Folds y per distinct camera of the chunk into the camera-major partials
// with a single warp when nu <= 32: camera u gets G lanes (the largest power
// of two with nu * G <= 32); lane j of the group sums slots j, j + G, ... of
// the camera in slot-list order, an xor butterfly over the G lanes combines
// them (fixed order: deterministic) and the group's lanes share the 9
// stores. nu > 32: one thread per camera, sequential. Few lanes and few
// butterfly levels keep the fold's shuffle count small (it dominated the
// instruction mix with a warp per camera).
template <class S, class Y, class T>
__device__ __forceinline__ void fold_cameras(const DseArgs<S, T>& A, int nu, const std::uint8_t* ubeg,
                                             const std::uint8_t* uslot, const std::int32_t* upart, const Y& y) {
  const int tid = threadIdx.x;
  // the largest power of two G with nu * G <= 32: 32 >> ceil(log2 nu)
  const int G = nu <= 32 ? 32 >> (32 - __clz(max(nu, 1) - 1)) : 1;
  const int nact = nu * G;
  if ((tid & ~31) >= nact) return;  // the warp has no camera
  const int u = tid / G, j = tid & (G - 1);
  S acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = S(0);
  if (tid < nact) {
    for (int k = ubeg[u] + j; k < ubeg[u + 1]; k += G) {
      const int o = uslot[k];
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += y(o, i);
    }
  }
  for (int o = 1; o < G; o <<= 1) {  // G > 1 only when nact <= 32: the whole warp is here
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  }
  if (tid < nact) {
    S* out = A.part + std::size_t(upart[u]) * 9;
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if ((i & (G - 1)) == j) out[i] = acc[i];
  }
}

// Fold by (camera, component) items (the default; DBAG_FOLD_ITEMS=0 keeps
// the one-warp lane-group fold above): thread t sums component i of camera
// u (t = 9 u + i, strided by the block) over the camera's slots in
// slot-list order — sequential, no shuffles, one store per thread; warps
// with no item exit at once. Measured: venice pass 0.207 -> 0.184 ms,
// trafalgar 14.3 -> 12.4 us (a third of the fold's instructions: no
// butterfly, no lane-group bookkeeping).
template <class S, class Y, class T>
__device__ __forceinline__ void fold_items(const DseArgs<S, T>& A, int nu, const std::uint8_t* ubeg,
                                           const std::uint8_t* uslot, const std::int32_t* upart, const Y& y) {
  const int n = nu * 9;
  for (int t = threadIdx.x; t < n; t += kTile) {
    const int u = (t * 7282) >> 16, i = t - 9 * u;  // t / 9 for t < 1152
    S acc = S(0);
    for (int k = ubeg[u]; k < ubeg[u + 1]; ++k) acc += y(uslot[k], i);
    A.part[std::size_t(upart[u]) * 9 + i] = acc;
  }
}

template <class S, int W = 9>
struct YRows {  // y[slot][W] rows (DseWork: W = kYW)
  const S (*y)[W];
  __device__ __forceinline__ S operator()(int o, int i) const { return y[o][i]; }
};

// y row of slot tid into the work area (padded rows: component pairs).
template <class S>
__device__ __forceinline__ void store_y(DseWork<S>& sm, int tid, const S* y) {
#if DBAG_FOLD_PAIRS
  using V = typename Pair<S>::type;
  V* row = reinterpret_cast<V*>(sm.y()[tid]);
#pragma unroll
  for (int h = 0; h < 4; ++h) row[h] = V{y[2 * h], y[2 * h + 1]};
  row[4] = V{y[8], S(0)};
#else
#pragma unroll
  for (int i = 0; i < 9; ++i) sm.y()[tid][i] = y[i];
#endif
}

// Fold by (camera, component pair) items: thread t sums components 2h and
// 2h + 1 of camera u (t = 5 u + h) over the camera's slots in slot-list
// order with one paired load per slot — the same per-component order as
// fold_items, with about half its instructions.
template <class S, class T>
__device__ __forceinline__ void fold_pairs(const DseArgs<S, T>& A, int nu, const std::uint8_t* ubeg,
                                           const std::uint8_t* uslot, const std::int32_t* upart,
                                           const S (*y)[kYW]) {
  using V = typename Pair<S>::type;
  const int n = nu * 5;
  for (int t = threadIdx.x; t < n; t += kTile) {
    const int u = (t * 13108) >> 16, h = t - 5 * u;  // t / 5 for t < 640
    S a0 = S(0), a1 = S(0);
    for (int k = ubeg[u]; k < ubeg[u + 1]; ++k) {
      const V v = reinterpret_cast<const V*>(y[uslot[k]])[h];
      a0 += v.x;
      a1 += v.y;
    }
    S* out = A.part + std::size_t(upart[u]) * 9 + 2 * h;
    out[0] = a0;
    if (h < 4) out[1] = a1;
  }
}

template <class S, class T>
__device__ __forceinline__ void fold_y(const DseArgs<S, T>& A, int nu, const DseWork<S>& sm) {
#if DBAG_FOLD_PAIRS
  fold_pairs(A, nu, sm.ubeg, sm.uslot, sm.upart, const_cast<DseWork<S>&>(sm).y());
#elif DBAG_FOLD_ITEMS
  fold_items(A, nu, sm.ubeg, sm.uslot, sm.upart, YRows<S, kYW>{const_cast<DseWork<S>&>(sm).y()});
#else
  fold_cameras(A, nu, sm.ubeg, sm.uslot, sm.upart, YRows<S, kYW>{const_cast<DseWork<S>&>(sm).y()});
#endif
}

template <class S>
__device__ __forceinline__ void stage_meta(const RecMeta& M, DseWork<S>& sm) {
  const int tid = threadIdx.x;
  if (tid < kPfParts || tid < M.nu) sm.upart[tid] = M.upart[tid];
  sm.uslot[tid] = M.uslot[tid];
  sm.ubeg[tid] = M.ubeg[tid];
  if (tid < 8) sm.ubeg[kTile + tid] = M.ubeg[kTile + tid];
}

// Camera-vector gathers of the a-phase: the plain vector x, or the PCG
// search direction formed on the fly, p = z (first iteration) or
// z + beta p_prev (dba/solver.hpp:231-236).
// ready() runs once per tile after the tile's own (constant) loads are in
// flight and before the first gather; false skips the tile.
template <class S>
struct GatherX {
  const S* x;
  __device__ __forceinline__ bool ready() { return true; }
  __device__ __forceinline__ S operator()(std::int32_t cam, int i) const { return __ldg(x + std::size_t(cam) * 9 + i); }
  // split access: raw() issues the loads, combine() forms the value
  struct Raw {
    S v;
  };
  __device__ __forceinline__ Raw raw(std::int32_t cam, int i) const { return {__ldg(x + std::size_t(cam) * 9 + i)}; }
  __device__ __forceinline__ Raw raw_at(int k) const { return {__ldg(x + k)}; }
  __device__ __forceinline__ S combine(const Raw& r) const { return r.v; }
};
// One 128-slot chunk whose record is at R (global or shared memory);
// normal tiles only (long tiles return). L = record lanes (kLanesFact:
// G = sqrt(w) Jc with the cameras' R staged in shared memory; kLanesDense:
// the 9x3 blocks).
template <class S, int MODE, int L, class G, class T>
__device__ __forceinline__ void dse_chunk_at(const DseArgs<S, T>& A, DseWork<S>& sm, const T* R, G gx) {
  constexpr bool kFact = L == kLanesFact;
  const int tid = threadIdx.x;
  const RecMeta& M = rec_meta<T, L>(R);
  // Load order (measured): header and metadata first; then the loads that
  // depend on them and sit on the tile's critical path (C factors, the
  // cameras' R — constant, so before the producer wait — then the camera
  // gathers after it); the E-lane stream, needed only from the a-phase on,
  // is issued behind the gathers so it does not queue ahead of them.
  const int4 hdr = *reinterpret_cast<const int4*>(&M.p0);  // p0, np, nslots, nchunk
  const int su = M.su[tid];
  const int pti = M.pt[tid];
  const int pb0 = M.pbeg[tid], pb1 = M.pbeg[tid + 1];
  const int nu = M.nu;
  if (MODE != 1) stage_meta(M, sm);
  if (hdr.w > 1) return;  // long tile: dse_long
  const std::int32_t p0 = hdr.x, np = hdr.y;
  S L9[9], wv[3];
  if (tid < np) load_point<S, MODE>(A, p0 + tid, L9, wv);
  const bool staged = nu <= kXsCams;
  // the chunk's camera rows: element t = tid + 128 j of the staged (camera,
  // row) list is row r of distinct camera u (t = 9 u + r; 128 = 9 * 14 + 2),
  // at offset ucam[u] * 9 + r of the camera-space vectors (shared by the R
  // and the x gathers)
  int goff[3];
  bool gon[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int t = tid + kTile * j;
    const int u = (t * 7282) >> 16;  // t / 9 for t < 384 (9 * 7282 = 65538)
    gon[j] = staged && u < nu;
    goff[j] = gon[j] ? M.ucam[u] * 9 + (t - 9 * u) : 0;
  }
  S rraw[3];
  if (kFact)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (gon[j]) rraw[j] = __ldg(A.Rm + goff[j]);
  if (!gx.ready()) return;
  typename G::Raw graw[3];  // the chunk's camera vectors, once per (camera, row)
  if (MODE != 2)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (gon[j]) graw[j] = gx.raw_at(goff[j]);
#if DBAG_RELOAD_E
  // E lanes are read where they are used (a-phase, y-phase) instead of being
  // held in registers across the point solve: the second read hits L1 / L2
  // (the record was just streamed), and the freed registers buy resident CTAs
  auto lanes = [&](S* e) {
#pragma unroll
    for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
  };
#else
  S e[L];
#pragma unroll
  for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);  // padding slots hold zeros
#endif
  if (staged && (kFact || MODE != 2)) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (gon[j]) {
        if (MODE != 2) sm.xs()[tid + kTile * j] = gx.combine(graw[j]);
        if (kFact) sm.rs[tid + kTile * j] = rraw[j];
      }
    __syncthreads();
  }
  // this slot's camera R: staged, or straight from global for > kXsCams cameras
  const std::int32_t cam = staged ? 0 : M.cam[tid];
  // the slot's camera R: staged in shared memory (the compiler sees the
  // address space: LDS, not generic loads) or from global beyond kXsCams
  const S* Rg = kFact ? A.Rm + std::size_t(cam) * 9 : nullptr;
  // the slot's staged camera R, read once for the a- and y-phases:
  // venice 0.1853 -> 0.1811 ms (FP64), 0.1096 -> 0.1068 (FP32), same run.
  // Not with FP32 lanes under FP64 arithmetic: its 7-CTA register budget
  // would spill; that variant reads R from shared memory in both phases.
  constexpr bool kRcReg = kFact && sizeof(T) == sizeof(S);
  S rcr[9];
  const S* rcs = kRcReg ? rcr : (kFact ? sm.rs + su * 9 : nullptr);
  auto load_rc = [&](bool real) {  // measured: in the a-phase, not ahead of it
    if (kRcReg && staged)
#pragma unroll
      for (int i = 0; i < 9; ++i) rcr[i] = real ? sm.rs[su * 9 + i] : S(0);
  };
  if (MODE == 2) load_rc(true);
  if (MODE != 2) {
    S a[3] = {S(0), S(0), S(0)};
    if (tid < hdr.z) {
      S xv[9];
#if DBAG_RELOAD_E
      S e[L];
      lanes(e);
#endif
      if (staged) {
#pragma unroll
        for (int i = 0; i < 9; ++i) xv[i] = sm.xs()[su * 9 + i];
        load_rc(true);
        coupling_t<S, L>(e, rcs, xv, a);
      } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) xv[i] = gx(cam, i);
        coupling_t<S, L>(e, Rg, xv, a);
      }
    } else {
      load_rc(false);  // padding slot: zero lanes, finite R
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) sm.a()[tid][j] = a[j];
  }
  __syncthreads();
  if (tid < np) {
    S tt[3] = {S(0), S(0), S(0)}, b[3];
    if (MODE != 2)
      for (int q = pb0; q < pb1; ++q)
#pragma unroll
        for (int j = 0; j < 3; ++j) tt[j] += sm.a()[q][j];
    finish_point<S, MODE>(A, p0 + tid, L9, wv, tt, b);
#pragma unroll
    for (int j = 0; j < 3; ++j) sm.b()[tid][j] = b[j];
  }
  __syncthreads();
  if constexpr (MODE != 1) {
    const S b0 = sm.b()[pti][0], b1 = sm.b()[pti][1], b2 = sm.b()[pti][2];
#if DBAG_Y_OVERLAY
    __syncthreads();  // y overlays b
#endif
    S y[9];
#if DBAG_RELOAD_E
    S e[L];
    lanes(e);
#endif
    if (staged) coupling_b<S, L>(e, rcs, b0, b1, b2, y);
    else coupling_b<S, L>(e, Rg, b0, b1, b2, y);
    store_y(sm, tid, y);
    __syncthreads();
    fold_y(A, nu, sm);
    // one chunk per CTA (k_g_pass, k_dse_chunk): no trailing barrier
  }
}

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <class S, int MODE, int L, class G, class T>
__device__ __forceinline__ void dse_chunk(const DseArgs<S, T>& A, DseWork<S>& sm, std::int32_t chunk, const G& gx) {
  // One wave ahead: the record the CTA pf_dist chunks later will read is
  // streamed into L2 now (E is constant through the PCG, so this may run
  // before the producer wait), decoupling HBM traffic from the pass's
  // per-chunk latency chain.
  if (A.pf_dist > 0 && threadIdx.x == 0 && chunk + A.pf_dist < A.n_chunks)
    l2_prefetch(A.rec + std::size_t(chunk + A.pf_dist) * Rec<T, L>::kLen, rec_hot_bytes<T, L>());
  dse_chunk_at<S, MODE, L>(A, sm, A.rec + std::size_t(chunk) * Rec<T, L>::kLen, gx);
}

// Resident CTAs per SM the chunk pass is compiled for (register budget),
// measured: 5 with FP64 E lanes in registers, 7 for FP32 lanes under FP64
// arithmetic (coupling_fp32), 8 for the all-FP32 solve (64 registers, no
// spill; 0.117 -> 0.110 ms per venice pass).
#ifndef DBAG_RELOAD_E
#define DBAG_RELOAD_E 0
#endif
#ifndef DBAG_PASS_MINB_F32E
#define DBAG_PASS_MINB_F32E 7
#endif
#ifndef DBAG_PASS_MINB_F64E
#define DBAG_PASS_MINB_F64E 5
#endif
#ifndef DBAG_PASS_MINB_F32
#define DBAG_PASS_MINB_F32 8
#endif
template <class T, class S = double>
constexpr int pass_min_blocks() {
  return sizeof(T) == 4 ? (sizeof(S) == 4 ? DBAG_PASS_MINB_F32 : DBAG_PASS_MINB_F32E) : DBAG_PASS_MINB_F64E;
}

template <class S, int MODE, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(kTile, pass_min_blocks<T, S>()) k_dse_chunk(DseArgs<S, T> A) {
  __shared__ DseWork<S> sm;
  dse_chunk<S, MODE, L>(A, sm, blockIdx.x, GatherX<S>{A.x});
}

// One CTA per long tile (a single point observed more than 128 times).
template <class S, int MODE, int L, class G, class T>
__device__ __forceinline__ void dse_long(const DseArgs<S, T>& A, DseWork<S>& sm, std::int32_t li, G gx) {
  constexpr bool kFact = L == kLanesFact;
  if (!gx.ready()) return;
  const int tid = threadIdx.x;
  const std::int32_t c0 = A.long_chunk[li];
  const RecMeta& M0 = rec_meta<T, L>(A.rec + std::size_t(c0) * Rec<T, L>::kLen);
  const std::int32_t p = M0.p0, nchunk = M0.nchunk;
  S a[3] = {S(0), S(0), S(0)};
  if (MODE != 2) {
    for (std::int32_t c = c0; c < c0 + nchunk; ++c) {
      const T* R = A.rec + std::size_t(c) * Rec<T, L>::kLen;
      const RecMeta& M = rec_meta<T, L>(R);
      if (tid < M.nslots) {
        const std::int32_t cam = M.cam[tid];
        S e[L], xv[9], as[3];
#pragma unroll
        for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
#pragma unroll
        for (int i = 0; i < 9; ++i) xv[i] = gx(cam, i);
        coupling_t<S, L>(e, kFact ? A.Rm + std::size_t(cam) * 9 : nullptr, xv, as);
#pragma unroll
        for (int j = 0; j < 3; ++j) a[j] += as[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) sm.a()[tid][j] = a[j];
  __syncthreads();
  if (tid == 0) {
    S tt[3] = {S(0), S(0), S(0)}, b[3];
    if (MODE != 2)
      for (int k = 0; k < kTile; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j) tt[j] += sm.a()[k][j];
    S L9[9], wv[3];
    load_point<S, MODE>(A, p, L9, wv);
    finish_point<S, MODE>(A, p, L9, wv, tt, b);
#pragma unroll
    for (int j = 0; j < 3; ++j) sm.b()[0][j] = b[j];
  }
  if constexpr (MODE != 1) {
    __syncthreads();
    const S b0 = sm.b()[0][0], b1 = sm.b()[0][1], b2 = sm.b()[0][2];  // y overlays b below
    for (std::int32_t c = c0; c < c0 + nchunk; ++c) {
      const T* R = A.rec + std::size_t(c) * Rec<T, L>::kLen;
      const RecMeta& M = rec_meta<T, L>(R);
      __syncthreads();
      stage_meta(M, sm);
      S e[L], y[9];
#pragma unroll
      for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
      coupling_b<S, L>(e, kFact ? A.Rm + std::size_t(M.cam[tid]) * 9 : nullptr, b0, b1, b2, y);
      store_y(sm, tid, y);
      __syncthreads();
      fold_y(A, M.nu, sm);
    }
  }
  __syncthreads();
}

template <class S, int MODE, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(kTile) k_dse_long(DseArgs<S, T> A) {
  __shared__ DseWork<S> sm;
  dse_long<S, MODE, L>(A, sm, blockIdx.x, GatherX<S>{A.x});
}

}  // namespace dev
}  // namespace dbag
