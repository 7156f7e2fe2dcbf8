// stream.cuh — the graph DPCG's DSE pass as a persistent, TMA-fed kernel.
//
// Same arithmetic as k_g_pass (dse.cuh: a_p = sum_s E_s^T p[cam_s],
// b_p = C_p^-1 a_p, y_s = E_s b_p folded per (chunk, camera) into the
// camera-major partials; dba/solver.hpp:149-181), different machinery:
//
//   * one CTA per SM slot (grid = SMs x resident CTAs), each walking the
//     chunks b, b + G, b + 2G, ... of the staged-chunk table;
//   * a producer warp streams each chunk's whole record (E lanes + RecMeta)
//     and the C factors of its points (one contiguous range: points are in
//     device order) into an NST-deep ring of shared-memory stages with
//     cp.async.bulk, completion on an mbarrier per stage (expect_tx);
//   * a gather warp waits for each landed record and gathers the chunk's
//     camera vectors (p = z + beta p_prev, or x) and rotations R once per
//     (distinct camera, row) into the same stage, off the consumers' path;
//   * four consumer warps (thread per slot) compute the chunk from shared
//     memory only and release the stage through a third mbarrier.
//
// The record bytes of the next NST chunks are in flight while a chunk is
// computed, so the HBM stream no longer waits on the per-chunk dependency
// chain (header -> gathers -> a -> point solve -> y -> fold) that bounds the
// one-CTA-per-chunk pass. E and C are constant during the PCG, so the first
// NST stages are issued before the programmatic-dependent-launch wait.
//
// Long tiles (points with more than kTile observations) run after the staged
// chunks, straight from global memory.
#pragma once

#include <cstdint>

#include "graph_pcg.cuh"

namespace dbag {
namespace dev {

#ifndef DBAG_STREAM_SLEEP_NS
#define DBAG_STREAM_SLEEP_NS 100
#endif
#ifndef DBAG_CSTAGE
#define DBAG_CSTAGE 48
#endif
constexpr int kCStage = DBAG_CSTAGE;  // points of a chunk whose C factors travel with its record
constexpr int kGatherWarps = 2;  // chunk k is gathered by gather warp k % kGatherWarps
constexpr int kStreamThreads = kTile + 32 + 32 * kGatherWarps;  // 4 consumer warps, the copy warp, the gather warps

// One staged chunk: record index, Cinv source (16-byte units) and the bytes
// of its C copy (16-byte rounded; the chunk's first factor starts at byte
// (p0 * 9 * sizeof(S)) % 16 of the copy).
struct ChunkTab {
  std::int32_t chunk, c16, cbytes, pad;
};

template <class S, class T, int L>
struct StreamLayout {
  static constexpr int kRecBytes = Rec<T, L>::kBytes;
  static constexpr int kCBytes = (kCStage * 9 * int(sizeof(S)) + 16 + 15) / 16 * 16;
  static constexpr int kXsBytes = 2 * kXsCams * 9 * int(sizeof(S));  // the gathered camera vectors and R
  static constexpr int kStageBytes = kRecBytes + kCBytes + kXsBytes;
  static constexpr int kWorkBytes = 15 * kTile * int(sizeof(S));  // a, b (3 x kTile each), y (9 x kTile)
  static constexpr int kHead = 128;  // mbarriers
  static constexpr int bytes(int nst) { return kHead + kWorkBytes + nst * kStageBytes; }
  static_assert(kRecBytes % 16 == 0, "bulk copy size");
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(std::uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_addr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait of the copy and gather warps: back off between probes, so the
// waiting warps do not take issue slots from the consumer warps (a bare
// try_wait loop re-issues every ~10 cycles).
__device__ __forceinline__ void mbar_wait_sleep(std::uint64_t* b, unsigned parity) {
  while (!mbar_test(b, parity)) __nanosleep(DBAG_STREAM_SLEEP_NS);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// barrier of the four consumer warps (the producer warp never joins)
__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Fold of y per distinct camera of the chunk over all four consumer warps:
// camera u gets G lanes of one warp (G the largest power of two <= 32 with
// nu * G <= 128; warp w holds cameras [w * 32/G, (w + 1) * 32/G)); lane j of
// the group sums slots j, j + G, ... of the camera in slot-list order, an xor
// butterfly over the G lanes combines them (fixed order: deterministic) and
// the group's lanes share the 9 stores into the camera-major partial.
template <class S, class T>
__device__ __forceinline__ void fold_cameras4(const DseArgs<S, T>& A, int nu, const std::uint8_t* ubeg,
                                              const std::uint8_t* uslot, const std::int32_t* upart, const S (*y)[9]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int G = 32;
  while (G > 1 && nu * G > kTile) G >>= 1;
  const int cpw = 32 / G;
  if (warp * cpw >= nu) return;  // warp-uniform
  const int u = warp * cpw + lane / G, j = lane & (G - 1);
  S acc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = S(0);
  if (u < nu)
    for (int k = ubeg[u] + j; k < ubeg[u + 1]; k += G) {
      const int o = uslot[k];
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += y[o][i];
    }
  for (int o = 1; o < G; o <<= 1) {
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  }
  if (u < nu) {
    S* out = A.part + std::size_t(upart[u]) * 9;
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if ((i & (G - 1)) == j) out[i] = acc[i];
  }
}

// One staged chunk (record R and C factors Cst in shared memory).
template <class S, int L, class G, class T>
__device__ __forceinline__ void stream_chunk(const DseArgs<S, T>& A, S* work, T* R, const S* Cst, const S* xs,
                                             const G& gx) {
  constexpr bool kFact = L == kLanesFact;
  const int tid = threadIdx.x;
  const RecMeta& M = *reinterpret_cast<const RecMeta*>(R + Rec<T, L>::kE);
  const int4 hdr = *reinterpret_cast<const int4*>(&M.p0);  // p0, np, nslots, nchunk
  const std::int32_t p0 = hdr.x, np = hdr.y;
  const int nu = M.nu;
  const bool staged = nu <= kXsCams;
  S(*a)[3] = reinterpret_cast<S(*)[3]>(work);
  S(*b)[3] = reinterpret_cast<S(*)[3]>(work + 3 * kTile);
  const S* rs = xs + kXsCams * 9;
  S L9[9];
  if (tid < np) {
    const S* src = tid < kCStage
                       ? Cst + ((std::size_t(p0) * 9 * sizeof(S)) & 15) / sizeof(S) + tid * 9
                       : A.Cinv + std::size_t(p0 + tid) * 9;
#pragma unroll
    for (int k = 0; k < 9; ++k) L9[k] = src[k];
  }
  const std::int32_t cam = staged ? 0 : M.cam[tid];
  const S* Rc = kFact ? (staged ? rs + M.su[tid] * 9 : A.Rm + std::size_t(cam) * 9) : nullptr;
  {
    S av[3] = {S(0), S(0), S(0)};
    if (tid < hdr.z) {
      S xv[9];
      const int su = M.su[tid];
#pragma unroll
      for (int i = 0; i < 9; ++i) xv[i] = staged ? xs[su * 9 + i] : gx(cam, i);
      S e[L];
#pragma unroll
      for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
      coupling_t<S, L>(e, Rc, xv, av);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) a[tid][j] = av[j];
  }
  cbar();
  if (tid < np) {
    S tt[3] = {S(0), S(0), S(0)}, bv[3];
    for (int q = M.pbeg[tid]; q < M.pbeg[tid + 1]; ++q)
#pragma unroll
      for (int j = 0; j < 3; ++j) tt[j] += a[q][j];
    S wv[3];
    finish_point<S, 0>(A, p0 + tid, L9, wv, tt, bv);
#pragma unroll
    for (int j = 0; j < 3; ++j) b[tid][j] = bv[j];
  }
  cbar();  // b complete
  const int pti = M.pt[tid];
  S y[9];
  {
    S e[L];  // E lanes again from the stage (padding slots hold zeros)
#pragma unroll
    for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
    coupling_b<S, L>(e, Rc, b[pti][0], b[pti][1], b[pti][2], y);
  }
  S(*yb)[9] = reinterpret_cast<S(*)[9]>(work + 6 * kTile);
#pragma unroll
  for (int i = 0; i < 9; ++i) yb[tid][i] = y[i];
  cbar();
  fold_items(A, nu, M.ubeg, M.uslot, M.upart, YRows<S>{yb});
}

// A long tile (one point, several chunk records), from global memory.
template <class S, int L, class G, class T>
__device__ __forceinline__ void stream_long(const DseArgs<S, T>& A, S* work, S* ybuf, std::int32_t li, const G& gx) {
  constexpr bool kFact = L == kLanesFact;
  const int tid = threadIdx.x;
  S(*a)[3] = reinterpret_cast<S(*)[3]>(work);
  S(*b)[3] = reinterpret_cast<S(*)[3]>(work + 3 * kTile);
  S(*yb)[9] = reinterpret_cast<S(*)[9]>(ybuf);
  const std::int32_t c0 = A.long_chunk[li];
  const RecMeta& M0 = rec_meta<T, L>(A.rec + std::size_t(c0) * Rec<T, L>::kLen);
  const std::int32_t p = M0.p0, nchunk = M0.nchunk;
  S av[3] = {S(0), S(0), S(0)};
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
      for (int j = 0; j < 3; ++j) av[j] += as[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) a[tid][j] = av[j];
  cbar();
  if (tid == 0) {
    S tt[3] = {S(0), S(0), S(0)}, bv[3];
    for (int k = 0; k < kTile; ++k)
#pragma unroll
      for (int j = 0; j < 3; ++j) tt[j] += a[k][j];
    S L9[9], wv[3];
    load_point<S, 0>(A, p, L9, wv);
    finish_point<S, 0>(A, p, L9, wv, tt, bv);
#pragma unroll
    for (int j = 0; j < 3; ++j) b[0][j] = bv[j];
  }
  cbar();
  const S b0 = b[0][0], b1 = b[0][1], b2 = b[0][2];
  for (std::int32_t c = c0; c < c0 + nchunk; ++c) {
    const T* R = A.rec + std::size_t(c) * Rec<T, L>::kLen;
    const RecMeta& M = rec_meta<T, L>(R);
    S e[L], y[9];
#pragma unroll
    for (int k = 0; k < L; ++k) e[k] = S(R[k * kTile + tid]);
    coupling_b<S, L>(e, kFact ? A.Rm + std::size_t(M.cam[tid]) * 9 : nullptr, b0, b1, b2, y);
    cbar();  // the previous chunk's fold has read yb
#pragma unroll
    for (int i = 0; i < 9; ++i) yb[tid][i] = y[i];
    cbar();
    fold_cameras(A, M.nu, M.ubeg, M.uslot, M.upart, YRows<S>{yb});
  }
  cbar();  // a, b, yb are reused by the next tile
}

// The pass. Block = 4 consumer warps + 1 producer warp; dynamic shared
// memory = StreamLayout::bytes(NST).
template <class S, class T, int L, int NST>
__global__ void __launch_bounds__(kStreamThreads, 3) k_g_stream(DseArgs<S, T> A, GBufs<S> B, const GScal<S>* sc,
                                                          const ChunkTab* __restrict__ tab, std::int32_t n_norm) {
  using Lay = StreamLayout<S, T, L>;
  extern __shared__ __align__(128) unsigned char smem[];
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem);
  std::uint64_t* empty = full + NST;
  std::uint64_t* ready = empty + NST;
  int* flag = reinterpret_cast<int*>(ready + NST);
  S* work = reinterpret_cast<S*>(smem + Lay::kHead);
  unsigned char* stages = smem + Lay::kHead + Lay::kWorkBytes;
  const int tid = threadIdx.x;
  pdl_allow_dependents();
#if DBAG_GTIMING
  if (blockIdx.x == 0 && tid == 0) {
    unsigned long long t_s;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_s));
    pdl_wait();
    tl_mark(sc->n, 0);
    if (sc->n < 1024) g_tl[sc->n * kTlStride + 7] = t_s;
  }
#endif
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTile / 32);
      mbar_init(&ready[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // done only flips 0 -> 1 inside one graph launch, so an early read of 1
    // is final (this copy of the unrolled body has nothing to do)
    *flag = *reinterpret_cast<const volatile int*>(&sc->done);
  }
  __syncthreads();
  if (*flag) return;
  const std::int32_t G = gridDim.x, b0 = blockIdx.x;
  const int mine = n_norm > b0 ? (n_norm - b0 + G - 1) / G : 0;
  const int npre = mine < NST ? mine : NST;
  if (tid >= kTile + 32) {  // gather warps
    const int lane = tid & 31, gw = (tid - kTile - 32) >> 5;
    GatherGraph<S> gx{sc, B.z, B.x, B.p0, B.p1, nullptr, nullptr, S(0), false, true};
    if (!gx.ready()) return;
    constexpr int kG = (kXsCams * 9 + 31) / 32;
    int k = gw;
    for (std::int32_t j = b0 + gw * G; j < n_norm; j += kGatherWarps * G, k += kGatherWarps) {
      const int s = k % NST;
      mbar_wait_sleep(&full[s], (k / NST) & 1);
      unsigned char* st = stages + std::size_t(s) * Lay::kStageBytes;
      const RecMeta& M = *reinterpret_cast<const RecMeta*>(st + Rec<T, L>::kE * sizeof(T));
      const int nu = M.nu;
      if (nu <= kXsCams) {
        S* xs = reinterpret_cast<S*>(st + Lay::kRecBytes + Lay::kCBytes);
        typename GatherGraph<S>::Raw g[kG];
        S rr[kG];
#pragma unroll
        for (int i = 0; i < kG; ++i) {
          const int t = lane + 32 * i;
          if (t < nu * 9) {
            const int u = t / 9, r = t - u * 9;
            const std::int32_t cam = M.ucam[u];
            g[i] = gx.raw(cam, r);
            if (L == kLanesFact) rr[i] = __ldg(A.Rm + std::size_t(cam) * 9 + r);
          }
        }
#pragma unroll
        for (int i = 0; i < kG; ++i) {
          const int t = lane + 32 * i;
          if (t < nu * 9) {
            xs[t] = gx.combine(g[i]);
            if (L == kLanesFact) xs[kXsCams * 9 + t] = rr[i];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    }
    return;
  }
  if (tid >= kTile) {  // copy (producer) warp
    const int lane = tid - kTile;
    int k = 0;
    for (std::int32_t base = b0; base < n_norm; base += 32 * G) {
      const std::int32_t jl = base + lane * G;
      int4 t = make_int4(0, 0, 0, 0);
      if (jl < n_norm) t = __ldg(reinterpret_cast<const int4*>(tab) + jl);
      for (int i = 0; i < 32; ++i, ++k) {
        if (base + i * G >= n_norm) break;
        const int c = __shfl_sync(0xffffffffu, t.x, i);
        const int c16 = __shfl_sync(0xffffffffu, t.y, i);
        const int cb = __shfl_sync(0xffffffffu, t.z, i);
        if (k == npre) {  // past the constant prefetch: only for a live pass
          pdl_wait();
          if (*reinterpret_cast<const volatile int*>(&sc->done)) return;
        }
        const int s = k % NST;
        if (k >= NST) mbar_wait_sleep(&empty[s], ((k / NST) - 1) & 1);
        if (lane == 0) {
          unsigned char* st = stages + std::size_t(s) * Lay::kStageBytes;
          mbar_expect_tx(&full[s], unsigned(Lay::kRecBytes + cb));
          bulk_g2s(st, A.rec + std::size_t(c) * Rec<T, L>::kLen, Lay::kRecBytes, &full[s]);
          if (cb > 0)
            bulk_g2s(st + Lay::kRecBytes, reinterpret_cast<const unsigned char*>(A.Cinv) + std::size_t(c16) * 16,
                     unsigned(cb), &full[s]);
        }
        __syncwarp();
      }
    }
    return;
  }
  GatherGraph<S> gx{sc, B.z, B.x, B.p0, B.p1, nullptr, nullptr, S(0), false, true};
  if (!gx.ready()) {  // loop already decided: let the prefetched copies land, then leave
    for (int k = 0; k < npre; ++k) mbar_wait(&full[k], 0);
    return;
  }
  int k = 0;
  for (std::int32_t j = b0; j < n_norm; j += G, ++k) {
    const int s = k % NST;
    mbar_wait(&ready[s], (k / NST) & 1);  // record landed and its cameras gathered
    unsigned char* st = stages + std::size_t(s) * Lay::kStageBytes;
    stream_chunk<S, L>(A, work, reinterpret_cast<T*>(st), reinterpret_cast<const S*>(st + Lay::kRecBytes),
                       reinterpret_cast<const S*>(st + Lay::kRecBytes + Lay::kCBytes), gx);
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (A.n_long > 0) {
    cbar();
    for (std::int32_t li = G - 1 - b0; li < A.n_long; li += G) stream_long<S, L>(A, work, work + 6 * kTile, li, gx);
  }
}

}  // namespace dev
}  // namespace dbag
