// lin.cuh — linearize + assemble_local in one pass over the chunk records.
//
// EdgeEvaluator::linearize + assemble_local (dba/edge_eval.hpp:115-191,
// dba/block_matrix.hpp:358-388) without the per-edge Jacobian rows in HBM:
// one CTA per 128-slot chunk (the DSE pass's tiles: whole points, slots in
// point-major edge order), thread per slot:
//   * gather x_c / x_p, jets (or the closed form), residual, 2 x 12 J;
//     G = sqrt(w) Jc into the chunk's record (the DSE stream);
//   * the slot's [Jc | Jp | r | w] row in shared memory;
//   * thread per point: C_p += w Jp^T Jp, w_p -= w Jp^T r over its slots in
//     edge order — the reference's per-point association (k_assemble_points'
//     arithmetic, bit for bit);
//   * per distinct camera of the chunk (the DSE fold's lane groups): the 45
//     upper-triangular terms of w Jc^T Jc and the 9 of -w Jc^T r summed in
//     double over the camera's slots into its camera-major partial (54
//     doubles at the DSE partial position); k_cam_assemble then folds each
//     camera's partials in chunk order into B and v.
// The previous form wrote 224 bytes of Jacobian row per edge and read them
// back twice (point- and camera-major assembly kernels): 2.1x the record
// writes in DRAM traffic plus two gathers (profiles/r2_ncu_all_venice.txt).
// Points observed more than 128 times (long tiles) take k_lin_long, one CTA
// per tile, its point sums sequential over the tile's slots.
#pragma once

#include <cstdint>

#include "dse.cuh"

namespace dbag {
namespace dev {

constexpr int kAsmTerms = 54;  // 45 upper-triangular B terms + 9 v terms per camera
constexpr int kRowW = 27;      // smem row per slot: Jc0[9] Jc1[9] Jp0[3] Jp1[3] r0 r1 w

template <class S, class T>
struct LinArgs {
  std::int32_t n_chunks;
  T* rec;
  const std::int32_t* chunk_slot;
  const std::int32_t* slot_cam;
  const std::int32_t* slot_pt;
  const std::int32_t* slot_edge;
  std::int64_t edge_base;
  const S* px;
  const S* py;
  const S* w;
  const S* xc;
  const S* xp;
  S* C;
  S* wv;
  double* bpart;  // kAsmTerms per camera-major partial position
  const std::int32_t* long_chunk;
  std::int32_t n_long;
  unsigned long long* bad_edge;
};

// term q of the camera assembly: (i, j) of the upper triangle for q < 45
__host__ __device__ constexpr int asm_i(int q) {
  return q < 9 ? 0 : q < 17 ? 1 : q < 24 ? 2 : q < 30 ? 3 : q < 35 ? 4 : q < 39 ? 5 : q < 42 ? 6 : q < 44 ? 7 : 8;
}
__host__ __device__ constexpr int asm_row0(int i) { return i * 9 - i * (i - 1) / 2; }  // first q of row i
__host__ __device__ constexpr int asm_j(int q) { return asm_i(q) + (q - asm_row0(asm_i(q))); }

// One slot: jets, G lanes into the record, the smem row. False: degenerate.
template <class S, int MODE, class T, int L>
__device__ __forceinline__ void lin_slot(const LinArgs<S, T>& a, T* R, std::int64_t s, S* row) {
  const S* cam = a.xc + std::size_t(a.slot_cam[s]) * 9;
  const S* x = a.xp + std::size_t(a.slot_pt[s]) * 3;
  S c[9], X[3], r[2], J[2][12];
#pragma unroll
  for (int k = 0; k < 9; ++k) c[k] = cam[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) X[k] = x[k];
  const bool ok = MODE == 0 ? edge_autodiff(c, X, a.px[s], a.py[s], r, J) : edge_analytic(c, X, a.px[s], a.py[s], r, J);
  const int tid = threadIdx.x;
  if (!ok) {
    atomicMin(a.bad_edge, (unsigned long long)(a.edge_base + a.slot_edge[s]));
#pragma unroll
    for (int k = 0; k < kRowW; ++k) row[k] = S(0);
#pragma unroll
    for (int k = 0; k < L; ++k) R[k * kTile + tid] = T(0);
    return;
  }
  const S wt = a.w[s];
  if constexpr (L == kLanesFact) {  // G = sqrt(w) Jc (exact copy for unit weights)
    const S sw = wt == S(1) ? S(1) : sqrt(wt);
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < 9; ++k) R[(q * 9 + k) * kTile + tid] = T(fm(sw, J[q][k]));
  } else {
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        R[(i * 3 + j) * kTile + tid] = T(fm(wt, fa(fm(J[0][i], J[0][9 + j]), fm(J[1][i], J[1][9 + j]))));
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    row[k] = J[0][k];
    row[9 + k] = J[1][k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    row[18 + k] = J[0][9 + k];
    row[21 + k] = J[1][9 + k];
  }
  row[24] = r[0];
  row[25] = r[1];
  row[26] = wt;
}

// C_p += w Jp^T Jp, w_p -= w Jp^T r over rows [k0, k1) in order
// (k_assemble_points' arithmetic).
template <class S>
__device__ __forceinline__ void point_accumulate(const S (*rows)[kRowW], int k0, int k1, S (*c)[3], S* g) {
  for (int k = k0; k < k1; ++k) {
    const S* row = rows[k];
    S jp0[3], jp1[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      jp0[q] = row[18 + q];
      jp1[q] = row[21 + q];
    }
    const S r0 = row[24], r1 = row[25], wt = row[26];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) c[i][j] = fa(c[i][j], fm(wt, fa(fm(jp0[i], jp0[j]), fm(jp1[i], jp1[j]))));
      g[i] = fs(g[i], fm(wt, fa(fm(jp0[i], r0), fm(jp1[i], r1))));
    }
  }
}

// Camera terms of one chunk: lane groups per distinct camera (as the DSE
// fold), three passes of 18 terms, butterfly over the group, stores shared
// by the group's lanes.
template <class S, class T>
__device__ __forceinline__ void camera_partials(const LinArgs<S, T>& a, const RecMeta& M, const S (*rows)[kRowW]) {
  const int nu = M.nu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int G = 32;
  while (G > 1 && nu * G > kTile) G >>= 1;
  const int cpw = 32 / G;
  if (warp * cpw >= nu) return;  // warp-uniform
  const int u = warp * cpw + lane / G, j = lane & (G - 1);
  const int k0 = u < nu ? M.ubeg[u] + j : 0, k1 = u < nu ? M.ubeg[u + 1] : 0;
  double* out = a.bpart + std::size_t(u < nu ? M.upart[u] : 0) * kAsmTerms;
#pragma unroll
  for (int pass = 0; pass < 3; ++pass) {
    double acc[18];
#pragma unroll
    for (int t = 0; t < 18; ++t) acc[t] = 0.0;
    for (int k = k0; k < k1; k += G) {
      const S* row = rows[M.uslot[k]];
      const S wt = row[26];
#pragma unroll
      for (int t = 0; t < 18; ++t) {
        const int q = pass * 18 + t;
        if (q < 45) {
          const int i = asm_i(q), jj = asm_j(q);
          acc[t] += double(fm(wt, fa(fm(row[i], row[jj]), fm(row[9 + i], row[9 + jj]))));
        } else {
          const int i = q - 45;
          acc[t] -= double(fm(wt, fa(fm(row[i], row[24]), fm(row[9 + i], row[25]))));
        }
      }
    }
    for (int o = 1; o < G; o <<= 1) {
#pragma unroll
      for (int t = 0; t < 18; ++t) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    }
    if (u < nu)
#pragma unroll
      for (int t = 0; t < 18; ++t)
        if ((t & (G - 1)) == j) out[pass * 18 + t] = acc[t];
  }
}

template <class S, int MODE, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(kTile) k_lin_chunk(LinArgs<S, T> a) {
  __shared__ S rows[kTile][kRowW];
  const int tid = threadIdx.x;
  T* R = a.rec + std::size_t(blockIdx.x) * Rec<T, L>::kLen;
  const RecMeta& M = rec_meta<T, L>(R);
  const int4 hdr = *reinterpret_cast<const int4*>(&M.p0);  // p0, np, nslots, nchunk
  if (hdr.w > 1) return;  // long tile: k_lin_long
  const std::int64_t s = std::int64_t(a.chunk_slot[blockIdx.x]) + tid;
  if (tid < hdr.z) lin_slot<S, MODE, T, L>(a, R, s, rows[tid]);
  __syncthreads();
  if (tid < hdr.y) {
    S c[3][3] = {}, g[3] = {};
    point_accumulate<S>(rows, M.pbeg[tid], M.pbeg[tid + 1], c, g);
    const std::size_t p = std::size_t(hdr.x + tid);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) a.C[p * 9 + i * 3 + jj] = c[i][jj];
      a.wv[p * 3 + i] = g[i];
    }
  }
  camera_partials<S, T>(a, M, rows);
}

template <class S, int MODE, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(kTile) k_lin_long(LinArgs<S, T> a) {
  __shared__ S rows[kTile][kRowW];
  const int tid = threadIdx.x;
  const std::int32_t c0 = a.long_chunk[blockIdx.x];
  const RecMeta& M0 = rec_meta<T, L>(a.rec + std::size_t(c0) * Rec<T, L>::kLen);
  const std::int32_t p = M0.p0, nchunk = M0.nchunk;
  S c[3][3] = {}, g[3] = {};
  for (std::int32_t ch = c0; ch < c0 + nchunk; ++ch) {
    T* R = a.rec + std::size_t(ch) * Rec<T, L>::kLen;
    const RecMeta& M = rec_meta<T, L>(R);
    const std::int64_t s = std::int64_t(a.chunk_slot[ch]) + tid;
    if (tid < M.nslots) lin_slot<S, MODE, T, L>(a, R, s, rows[tid]);
    __syncthreads();
    if (tid == 0) point_accumulate<S>(rows, 0, M.nslots, c, g);  // edge order across the tile's chunks
    camera_partials<S, T>(a, M, rows);
    __syncthreads();  // rows are rewritten by the next chunk
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) a.C[std::size_t(p) * 9 + i * 3 + jj] = c[i][jj];
      a.wv[std::size_t(p) * 3 + i] = g[i];
    }
  }
}

// B and v per camera from its partials in chunk order: warp per camera, lane
// owns terms lane and lane + 32 (coalesced 54-double partials), sequential
// over the partials (deterministic). Writes all m cameras (zero where the
// rank holds no edge of the camera).
template <class S>
__global__ void __launch_bounds__(256) k_cam_assemble(std::int32_t m, const std::int32_t* __restrict__ cam_part_ptr,
                                                      const double* __restrict__ bpart, S* __restrict__ B,
                                                      S* __restrict__ v) {
  const std::int32_t cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cam >= m) return;
  double a0 = 0.0, a1 = 0.0;
  for (std::int32_t k = cam_part_ptr[cam]; k < cam_part_ptr[cam + 1]; ++k) {
    const double* pp = bpart + std::size_t(k) * kAsmTerms;
    a0 += pp[lane];
    if (lane + 32 < kAsmTerms) a1 += pp[lane + 32];
  }
  S* b = B + std::size_t(cam) * 81;
  auto put = [&](int q, double val) {
    if (q < 45) {
      const int i = asm_i(q), j = asm_j(q);
      b[i * 9 + j] = S(val);
      b[j * 9 + i] = S(val);
    } else {
      v[std::size_t(cam) * 9 + (q - 45)] = S(val);
    }
  };
  put(lane, a0);
  if (lane + 32 < kAsmTerms) put(lane + 32, a1);
}

}  // namespace dev
}  // namespace dbag
