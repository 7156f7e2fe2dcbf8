// peer.cuh — device-side all-reduce between the ranks of a group over peer
// memory: the collective of the K > 1 graph DPCG.
//
// WorkerGroup::allreduce_sum (dba/comms.hpp:67-91) as one kernel: every rank
// deposits its vector in its own slot buffer, raises a per-slice arrival
// epoch, waits for every peer's epoch of that slice, and folds the K slots in
// ascending rank order (acc = s0; acc += s1; ... — the reference's association,
// identical bits on every rank). Slots are double-buffered by epoch parity: a
// rank that reached collective e has seen every peer arrive at e - 1, i.e.
// finish reading collective e - 2's slots, so no second barrier is needed.
// Slices are independent (one CTA each, its own epoch), so no grid-wide sync.
// Peers are other devices reached over NVLink / NVSwitch (P2P in one process,
// CUDA IPC across processes) or other ranks on the same device; slot reads
// bypass L1 (ld.cg) and epochs use release/acquire at system scope.
//
// No host rendezvous and no host-visible state: the kernel is captured in the
// rank's DPCG graph, and the ranks' graphs synchronise on the device.
#pragma once

#include <cstdint>

#include "comm.hpp"
#include "kernels.cuh"

namespace dbag {
namespace dev {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kPeerThreads = 256;

// The exchange of one slice [b0, b1): fill(mine) deposits this rank's values
// into its slot, then the epoch handshake, then out[i] = ascending-rank sum.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Waiting for the peers: timeout_ns / failed given (the setup self-check,
// 2 s) or the site's own (SolverConfig::collective_timeout in the DPCG
// graph); past the timeout bit p of the absent rank p is ORed into *failed
// and the wait ends. A set *failed ends every later wait at once (the graph
// drains; the host raises CollectiveError naming the ranks). No timeout and
// no flag: wait for as long as the peers take.
template <class T, class Fill>
__device__ __forceinline__ void peer_slice(const PeerSite& s, int c, std::int64_t b0, std::int64_t b1, T* out,
                                           Fill fill, unsigned long long timeout_ns = 0, int* failed = nullptr) {
  const unsigned e = s.epoch[c] + 1u;
  fill(static_cast<T*>(s.slot[e & 1u][s.rank]));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // the CTA's deposits (ordered by bar.sync) before the epoch
    st_release_sys(s.flag[s.rank] + c, e);
    const unsigned long long tmo = timeout_ns ? timeout_ns : s.timeout_ns;
    int* fl = timeout_ns ? failed : s.failed;
    const volatile int* vfl = fl;
    const unsigned long long t0 = tmo ? global_ns() : 0;
    for (int p = 0; p < s.k; ++p) {
      unsigned spins = 0;
      while (static_cast<int>(ld_acquire_sys(s.flag[p] + c) - e) < 0) {
        if ((++spins & 255u) != 0u) continue;
        if (vfl && *vfl) break;  // a peer is already known absent
        if (tmo && global_ns() - t0 > tmo) {
          atomicOr(fl, 1 << p);
          break;
        }
      }
    }
    s.epoch[c] = e;
  }
  __syncthreads();
  for (std::int64_t i = b0 + threadIdx.x; i < b1; i += kPeerThreads) {
    T acc = __ldcg(static_cast<const T*>(s.slot[e & 1u][0]) + i);
    for (int p = 1; p < s.k; ++p) acc += __ldcg(static_cast<const T*>(s.slot[e & 1u][p]) + i);
    out[i] = acc;
  }
}

__device__ __forceinline__ bool peer_skip(const int* skip) {
  return skip && *reinterpret_cast<const volatile int*>(skip);
}

// out[0..len) := sum over ranks of in[0..len) (in may alias out). Grid =
// s.nslice CTAs of kPeerThreads. skip (may be null): when *skip != 0 every
// rank returns at once (the copies of an unrolled graph body after the loop
// decision; every rank sees the same flag).
template <class T>
__global__ void __launch_bounds__(kPeerThreads) k_peer_allreduce(PeerSite s, const T* in, T* out, std::int64_t len,
                                                                 const int* skip) {
  if (peer_skip(skip)) return;
  const int c = blockIdx.x;
  const std::int64_t b0 = std::int64_t(c) * s.slice;
  const std::int64_t b1 = b0 + s.slice < len ? b0 + s.slice : len;
  peer_slice<T>(s, c, b0, b1, out, [&](T* mine) {
    for (std::int64_t i = b0 + threadIdx.x; i < b1; i += kPeerThreads) mine[i] = in[i];
  });
}

// Setup self-check of a site (NcclComm, CUDA-IPC peers): `rounds`
// all-reduces of rank-dependent values (both slot parities), every slice,
// each compared with the closed-form sum; *bad = 1 on a mismatch or a peer
// that never arrives (2 s). Leaves every rank's epochs advanced alike.
template <class T = double>
__global__ void __launch_bounds__(kPeerThreads) k_peer_selftest(PeerSite s, T* buf, int rounds, int* bad) {
  const int c = blockIdx.x;
  const std::int64_t b0 = std::int64_t(c) * s.slice, b1 = b0 + s.slice < s.len ? b0 + s.slice : s.len;
  for (int q = 0; q < rounds; ++q) {
    peer_slice<T>(
        s, c, b0, b1, buf,
        [&](T* mine) {
          for (std::int64_t i = b0 + threadIdx.x; i < b1; i += kPeerThreads)
            mine[i] = T(s.rank + 1) * T(i % 1009 + q + 1);
        },
        2000000000ull, bad);
    const T k = T(s.k);
    for (std::int64_t i = b0 + threadIdx.x; i < b1; i += kPeerThreads)
      if (buf[i] != k * (k + 1) / 2 * T(i % 1009 + q + 1)) *bad = 1;
    __syncthreads();
  }
}

// The camera side of a K > 1 DSE in one kernel: fold of this rank's
// partials per camera (warp per camera, lanes strided over the camera's
// partials, fixed shuffle tree: k_cam_reduce's association) straight into
// the deposit slot, then the all-reduce of the 9m vector into out.
template <class S>
__global__ void __launch_bounds__(kPeerThreads) k_peer_cam(PeerSite s, std::int32_t m,
                                                           const std::int32_t* __restrict__ cam_part_ptr,
                                                           const S* __restrict__ part, S* out, const int* skip) {
  if (peer_skip(skip)) return;
  const int c = blockIdx.x;
  const std::int64_t len = std::int64_t(m) * 9;
  const std::int64_t b0 = std::int64_t(c) * s.slice;
  const std::int64_t b1 = b0 + s.slice < len ? b0 + s.slice : len;
  peer_slice<S>(s, c, b0, b1, out, [&](S* mine) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (std::int64_t cam = b0 / 9 + warp; cam < b1 / 9; cam += kPeerThreads / 32) {
      S acc[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] = S(0);
      for (std::int32_t k = cam_part_ptr[cam] + lane; k < cam_part_ptr[cam + 1]; k += 32) {
        const S* pp = part + std::size_t(k) * 9;
#pragma unroll
        for (int i = 0; i < 9; ++i) acc[i] += pp[i];
      }
#pragma unroll
      for (int i = 0; i < 9; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
      }
      if (lane == 0)
#pragma unroll
        for (int i = 0; i < 9; ++i) mine[cam * 9 + i] = acc[i];
    }
  });
}

// The halo of a K > 1 DSE in one kernel (one CTA: 3H <= 3(K - 1) values):
// all-reduce of the halo points' a_p deposits into hsum, then for this
// rank's halo slots b_p = C_p^-1 a_p, y_s = E_s b_p into the slot's partial
// (k_halo_fix).
template <class S, class T, int L>
__global__ void __launch_bounds__(kPeerThreads) k_peer_halo(PeerSite s, const S* hbuf, S* hsum, std::int64_t len,
                                                            const int* skip, std::int32_t n,
                                                            const std::int32_t* __restrict__ halo_slot,
                                                            const std::int32_t* __restrict__ slot_dpt,
                                                            const std::int32_t* __restrict__ halo_of,
                                                            const S* __restrict__ Cinv, const T* __restrict__ E,
                                                            const std::int32_t* __restrict__ slot_chunk,
                                                            const std::int32_t* __restrict__ chunk_slot,
                                                            const std::int32_t* __restrict__ halo_pos,
                                                            S* __restrict__ part,
                                                            const std::int32_t* __restrict__ slot_cam,
                                                            const S* __restrict__ Rm) {
  if (peer_skip(skip)) return;
  peer_slice<S>(s, 0, 0, len, hsum, [&](S* mine) {
    for (std::int64_t i = threadIdx.x; i < len; i += kPeerThreads) mine[i] = hbuf[i];
  });
  __syncthreads();
  for (std::int32_t i = threadIdx.x; i < n; i += kPeerThreads) {
    const std::int32_t sl = halo_slot[i];
    const std::int32_t p = slot_dpt[sl];
    S b[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) b[j] = hsum[std::size_t(halo_of[p]) * 3 + j];
    llt_solve<S, 3>(Cinv + std::size_t(p) * 9, b);
    const T* ep = E + rec_at<T, L>(slot_chunk, chunk_slot, sl);
    S e[L], y[9];
#pragma unroll
    for (int k = 0; k < L; ++k) e[k] = S(ep[std::size_t(k) * kTile]);
    coupling_b<S, L>(e, L == kLanesFact ? Rm + std::size_t(slot_cam[sl]) * 9 : nullptr, b[0], b[1], b[2], y);
#pragma unroll
    for (int r = 0; r < 9; ++r) part[std::size_t(halo_pos[i]) * 9 + r] = y[r];
  }
}

}  // namespace dev
}  // namespace dbag
