// kernels.cuh — the sm_100a kernels of the LM inner loop.
//
// Layout (per rank):
//   slot s        : point-major position of shard edge pt_blk[s]
//                   (dba/block_matrix.hpp:309-320 grouping); slot_* arrays are
//                   SoA and streamed coalesced.
//   cslot c       : camera-major position (cam_blk order); cslot_pslot maps it
//                   to the point-major slot.
//   E_pm / E_cm   : the 9x3 coupling blocks (dba/block_matrix.hpp:174-329),
//                   SoA by element (27 lanes x N), in slot / cslot order.
//   Jb            : per-slot residual + 2x12 Jacobian + weight, AoS of 28.
//   cameras       : global ids, 9m vectors, 81m blocks (replicated).
//   points        : local ids (first appearance), 3 n_loc vectors.
// Reductions that feed LM / PCG decisions are deterministic: fixed grid,
// fixed per-thread order, fixed shuffle tree, and a last-block finalize that
// sums per-block partials in block order.
#pragma once

#include <cstddef>

#include <cuda_runtime.h>

#include <cstdint>

#include "jets.cuh"

namespace dbag {
namespace dev {

constexpr int kTile = 128;        // point-pass tile (slots) == block size
constexpr int kRedThreads = 256;  // reduction kernels' block size
constexpr int kRedBlocksMax = 592;  // 4 x 148 SMs
constexpr int kXsCams = 32;  // distinct cameras of a chunk whose vectors are gathered once into shared memory

// Static per-chunk metadata stored after the E lanes of its record, so one
// coalesced read of a record brings every index a tile needs (no pointer
// chasing through global index arrays on the streaming path).
struct RecMeta {
  std::int32_t p0, np, nslots, nchunk;  // first device point, points, slots; nchunk > 1: long tile
  std::int32_t nu, ci, pad0, pad1;      // distinct cameras; chunk index inside its tile
  std::int32_t ucam[kXsCams];           // camera id of distinct camera u < kXsCams
  std::uint8_t pt[kTile];               // slot -> point index in the tile
  std::uint8_t uslot[kTile];            // slots grouped by camera
  std::uint8_t ubeg[kTile + 8];         // camera u's slots: uslot[ubeg[u] .. ubeg[u+1])
  std::uint8_t pbeg[kTile + 8];         // point i's slots: [pbeg[i], pbeg[i+1])
  std::uint8_t su[kTile];               // slot -> its distinct camera u (inverse of uslot / ubeg)
  std::int32_t upart[kTile];            // camera-major partial position of each distinct camera
  std::int32_t cam[kTile];              // camera of each slot (padding: 0); read only when nu > kXsCams
};
static_assert(sizeof(RecMeta) % 16 == 0, "record metadata must keep 16-byte alignment");
// Coupling-block storage per slot, the L lanes of a chunk record:
//   kLanesFact = 18  factored (the product path): G = sqrt(w) Jc, the
//       edge's 2x9 camera Jacobian scaled by sqrt(w), lanes r * 9 + k. The
//       reference's block E = w Jc^T Jp (dba/block_matrix.hpp:380-381) is
//       E = G^T Gt R with Gt = G[:, 3:6] (dr/dt = dr/dP) and R = dP/dX the
//       camera's rotation matrix (one per camera, Rank::Rm_), since
//       Jp = dr/dP R. E^T x = R^T Gt^T (G x), E b = G^T Gt (R b): 18 scalars
//       per edge instead of 27 (1/3 fewer bytes on the DSE stream), fewer
//       registers, every product the reference forms (rounding-level
//       reassociation only). This is the implicit-Schur storage of the
//       Jacobian blocks (cf. Ceres' ImplicitSchurComplement), here with Jp
//       folded into the camera's R.
//   kLanesDense = 27  the 9x3 block itself, row-major (i * 3 + j): used for
//       caller-fabricated blocks (Rank::set_system, any 9x3 E).
constexpr int kLanesFact = 18;
constexpr int kLanesDense = 27;

// Bytes of a record the pass reads for a chunk with at most kPfParts
// distinct cameras: the E lanes and the metadata up to upart[kPfParts)
// (cam[] and the rest of upart[] are read only by rarer chunks).
constexpr int kPfParts = 16;
template <class S, int L = kLanesFact>
constexpr unsigned rec_hot_bytes() {
  return unsigned(L * kTile * sizeof(S) + offsetof(RecMeta, upart) + kPfParts * sizeof(std::int32_t));
}
static_assert(rec_hot_bytes<double>() % 16 == 0 && rec_hot_bytes<float>() % 16 == 0, "bulk prefetch size");
static_assert(rec_hot_bytes<double, kLanesDense>() % 16 == 0 && rec_hot_bytes<float, kLanesDense>() % 16 == 0,
              "bulk prefetch size");

// double2 / float2: paired shared-memory rows (dse.cuh fold_pairs)
template <class T>
struct Pair;
template <>
struct Pair<double> {
  using type = double2;
};
template <>
struct Pair<float> {
  using type = float2;
};

// E chunk record: L lanes x kTile slots (lane-major) then RecMeta; one
// record per 128-slot chunk of the device slot order.
template <class S, int L = kLanesFact>
struct Rec {
  static constexpr int kE = L * kTile;
  static constexpr int kMeta = int(sizeof(RecMeta) / sizeof(S));
  static constexpr int kLen = kE + kMeta;
  static constexpr int kBytes = kLen * int(sizeof(S));
};

// Offset of lane 0 of slot s inside the record array.
template <class S, int L = kLanesFact>
__host__ __device__ __forceinline__ std::size_t rec_at(const std::int32_t* slot_chunk, const std::int32_t* chunk_slot,
                                                       std::int64_t s) {
  const std::int32_t c = slot_chunk[s];
  return std::size_t(c) * Rec<S, L>::kLen + std::size_t(s - chunk_slot[c]);
}

template <int BS>
__host__ __device__ constexpr int rcp_at(int k);

struct SumOp {
  __device__ static double id() { return 0.0; }
  __device__ static double op(double a, double b) { return a + b; }
};
struct MaxOp {
  __device__ static double id() { return 0.0; }  // used on |x| >= 0
  __device__ static double op(double a, double b) { return fmax(a, b); }
};

template <class Op>
__device__ __forceinline__ double warp_reduce(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = Op::op(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Block reduction, result valid in thread 0. smem: >= blockDim/32 doubles.
template <class Op>
__device__ __forceinline__ double block_reduce(double v, double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_reduce<Op>(v);
  __syncthreads();
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? smem[lane] : Op::id();
    v = warp_reduce<Op>(v);
  }
  return v;
}

// NV block reductions in one pass (one shared round trip for all values);
// results valid in thread 0. smem: >= NV * 32 doubles.
template <class Op, int NV>
__device__ __forceinline__ void block_reduce_n(double (&v)[NV], double* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_reduce<Op>(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[k * 32 + warp] = v[k];
  __syncthreads();
  if (warp == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_reduce<Op>(lane < nw ? smem[k * 32 + lane] : Op::id());
}

// Grid-wide deterministic reduction of NV values: every block calls this
// once; the last block to arrive reduces the per-block partials in block
// order and writes out[0..NV). Returns true in the finalizing block (all
// threads), after out[] is written and visible to that block. Only the
// partials' writer (thread 0) fences before arriving: the callers' other
// stores are for later kernels, which the kernel boundary orders.
template <class Op, int NV>
__device__ __forceinline__ bool grid_reduce(const double (&v)[NV], double* partials, unsigned* counter,
                                            double* out) {
  __shared__ double red[NV * 32];
  __shared__ bool last;
  double b[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) b[k] = v[k];
  block_reduce_n<Op, NV>(b, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * gridDim.x + blockIdx.x] = b[k];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    acc[k] = Op::id();
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) acc[k] = Op::op(acc[k], __ldcg(partials + k * gridDim.x + i));
  }
  block_reduce_n<Op, NV>(acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = acc[k];
    *counter = 0u;
  }
  __threadfence();
  __syncthreads();
  return true;
}

struct RedWs {  // per-launch scratch of the grid reductions
  double* partials;   // >= 8 * kRedBlocksMax
  unsigned* counter;  // zero-initialized
};

// ---------------------------------------------------------------- cost ----
// EdgeEvaluator::cost (dba/edge_eval.hpp:289-309): sum w |r|^2 with the
// squared norm in Scalar and the accumulation in double. Degenerate depth ->
// +inf and atomicMin of the global edge id.
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_cost(std::int64_t N, const std::int32_t* __restrict__ slot_cam,
                                                      const std::int32_t* __restrict__ slot_pt,
                                                      const std::int32_t* __restrict__ slot_edge,
                                                      std::int64_t edge_base, const S* __restrict__ px,
                                                      const S* __restrict__ py, const S* __restrict__ w,
                                                      const S* __restrict__ xc, const S* __restrict__ xp,
                                                      RedWs ws, double* out_cost, unsigned long long* bad_edge) {
  double acc = 0.0;
  bool bad = false;
  for (std::int64_t s = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; s < N;
       s += std::int64_t(gridDim.x) * blockDim.x) {
    const S* cam = xc + std::size_t(slot_cam[s]) * 9;
    const S* x = xp + std::size_t(slot_pt[s]) * 3;
    S c[9], X[3], r[2];
#pragma unroll
    for (int k = 0; k < 9; ++k) c[k] = cam[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) X[k] = x[k];
    if (edge_residual(c, X, px[s], py[s], r)) {
      acc += double(w[s]) * double(fa(fm(r[0], r[0]), fm(r[1], r[1])));
    } else {
      bad = true;
      atomicMin(bad_edge, (unsigned long long)(edge_base + slot_edge[s]));
    }
  }
  const double v[2] = {acc, bad ? 1.0 : 0.0};
  __shared__ double fin[2];
  if (grid_reduce<SumOp, 2>(v, ws.partials, ws.counter, fin)) {
    if (threadIdx.x == 0) *out_cost = fin[1] > 0 ? __longlong_as_double(0x7ff0000000000000LL) : fin[0];
  }
}

// Per-edge cost-path residuals in shard edge order (test hook).
template <class S>
__global__ void k_residuals(std::int64_t N, const std::int32_t* __restrict__ slot_cam,
                            const std::int32_t* __restrict__ slot_pt, const std::int32_t* __restrict__ slot_edge,
                            const S* __restrict__ px, const S* __restrict__ py, const S* __restrict__ xc,
                            const S* __restrict__ xp, S* __restrict__ out) {
  const std::int64_t s = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (s >= N) return;
  S c[9], X[3], r[2] = {S(0), S(0)};
#pragma unroll
  for (int k = 0; k < 9; ++k) c[k] = xc[std::size_t(slot_cam[s]) * 9 + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) X[k] = xp[std::size_t(slot_pt[s]) * 3 + k];
  if (!edge_residual(c, X, px[s], py[s], r)) r[0] = r[1] = S(NAN);
  const std::int64_t e = slot_edge[s];
  out[e] = r[0];
  out[N + e] = r[1];
}

// ---------------------------------------------------------- linearize ----
// Fused K1+K2(+K3)+K5-E: gather, jets (or closed form), residual, Jacobian,
// E = w Jc^T Jp. Jb row: [r0 r1 | J0[12] | J1[12] | w pad].
template <class S, int MODE, class T = S, int L = kLanesFact>
__global__ void __launch_bounds__(128) k_linearize(std::int64_t s0, std::int64_t s1,
                                                   const std::int32_t* __restrict__ slot_cam,
                                                   const std::int32_t* __restrict__ slot_pt,
                                                   const std::int32_t* __restrict__ slot_edge,
                                                   std::int64_t edge_base, const S* __restrict__ px,
                                                   const S* __restrict__ py, const S* __restrict__ w,
                                                   const S* __restrict__ xc, const S* __restrict__ xp,
                                                   S* __restrict__ Jb, T* __restrict__ E,
                                                   const std::int32_t* __restrict__ slot_chunk,
                                                   const std::int32_t* __restrict__ chunk_slot,
                                                   unsigned long long* bad_edge) {
  const std::int64_t s = s0 + blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (s >= s1) return;
  const S* cam = xc + std::size_t(slot_cam[s]) * 9;
  const S* x = xp + std::size_t(slot_pt[s]) * 3;
  S c[9], X[3], r[2], J[2][12];
#pragma unroll
  for (int k = 0; k < 9; ++k) c[k] = cam[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) X[k] = x[k];
  const bool ok = MODE == 0 ? edge_autodiff(c, X, px[s], py[s], r, J) : edge_analytic(c, X, px[s], py[s], r, J);
  if (!ok) {
    atomicMin(bad_edge, (unsigned long long)(edge_base + slot_edge[s]));
    return;
  }
  const S wt = w[s];
  S* row = Jb + std::size_t(s - s0) * 28;  // Jb holds the batch [s0, s1)
  row[0] = r[0];
  row[1] = r[1];
#pragma unroll
  for (int j = 0; j < 12; ++j) {
    row[2 + j] = J[0][j];
    row[14 + j] = J[1][j];
  }
  row[26] = wt;
  row[27] = S(0);
  const std::size_t base = rec_at<T, L>(slot_chunk, chunk_slot, s);
  if constexpr (L == kLanesFact) {  // G = sqrt(w) Jc (exact copy for unit weights)
    const S sw = wt == S(1) ? S(1) : sqrt(wt);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int k = 0; k < 9; ++k) E[base + std::size_t(r * 9 + k) * kTile] = T(fm(sw, J[r][k]));
  } else {
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        E[base + std::size_t(i * 3 + j) * kTile] = T(fm(wt, fa(fm(J[0][i], J[0][9 + j]), fm(J[1][i], J[1][9 + j]))));
  }
}

// R(aa) = c I + s1 [aa]x + c2 aa aa^T per camera (row-major, 9m), with the
// model's coefficients (dba/problem.hpp:89-118, Taylor branch included):
// dP/dX of the Snavely model, the factor that turns the stored dr/dt into
// Jp = dr/dP R (factored coupling records).
template <class S>
__global__ void k_cam_rotations(std::int32_t m, const S* __restrict__ xc, S* __restrict__ Rm) {
  const std::int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const S a0 = xc[std::size_t(c) * 9], a1 = xc[std::size_t(c) * 9 + 1], a2 = xc[std::size_t(c) * 9 + 2];
  const S t = fa(fa(fm(a0, a0), fm(a1, a1)), fm(a2, a2));
  S cs, s1, c2;
  rot_coeffs(t, cs, s1, c2);
  const S a[3] = {a0, a1, a2};
  const S k[3][3] = {{S(0), -a2, a1}, {a2, S(0), -a0}, {-a1, a0, S(0)}};
  S* o = Rm + std::size_t(c) * 9;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) o[i * 3 + j] = fa(fa(i == j ? cs : S(0), fm(s1, k[i][j])), fm(c2, fm(a[i], a[j])));
}

// E^T x (a 3-vector) and E b (a 9-vector) of one slot for either record
// layout: e = the slot's L lanes, Rc = its camera's R (factored only).
template <class S, int L>
__device__ __forceinline__ void coupling_t(const S* e, const S* Rc, const S* xv, S* a) {
  if constexpr (L == kLanesFact) {
    S u0 = S(0), u1 = S(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      u0 += e[k] * xv[k];
      u1 += e[9 + k] * xv[k];
    }
    S h[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) h[i] = e[3 + i] * u0 + e[12 + i] * u1;
#pragma unroll
    for (int j = 0; j < 3; ++j) a[j] = (Rc[j] * h[0] + Rc[3 + j] * h[1]) + Rc[6 + j] * h[2];
  } else {
#pragma unroll
    for (int j = 0; j < 3; ++j) a[j] = S(0);
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      a[0] += e[i * 3 + 0] * xv[i];
      a[1] += e[i * 3 + 1] * xv[i];
      a[2] += e[i * 3 + 2] * xv[i];
    }
  }
}
template <class S, int L>
__device__ __forceinline__ void coupling_b(const S* e, const S* Rc, S b0, S b1, S b2, S* y) {
  if constexpr (L == kLanesFact) {
    S g[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) g[i] = (Rc[i * 3] * b0 + Rc[i * 3 + 1] * b1) + Rc[i * 3 + 2] * b2;
    const S v0 = (e[3] * g[0] + e[4] * g[1]) + e[5] * g[2];
    const S v1 = (e[12] * g[0] + e[13] * g[1]) + e[14] * g[2];
#pragma unroll
    for (int k = 0; k < 9; ++k) y[k] = e[k] * v0 + e[9 + k] * v1;
  } else {
#pragma unroll
    for (int i = 0; i < 9; ++i) y[i] = (e[i * 3] * b0 + e[i * 3 + 1] * b1) + e[i * 3 + 2] * b2;
  }
}

// C[p] += w Jp^T Jp, w[p] -= w Jp^T r over the point's slots in edge order
// (dba/block_matrix.hpp:382-386). Thread per local point.
template <class S>
__global__ void k_assemble_points(std::int32_t d0, std::int32_t d1, const std::int32_t* __restrict__ pt_ptr,
                                  std::int64_t s0, const S* __restrict__ Jb, S* __restrict__ C,
                                  S* __restrict__ wv) {
  const std::int32_t p = d0 + static_cast<std::int32_t>(blockIdx.x * blockDim.x + threadIdx.x);
  if (p >= d1) return;
  S c[3][3] = {}, g[3] = {};
  for (std::int32_t s = pt_ptr[p]; s < pt_ptr[p + 1]; ++s) {
    const S* row = Jb + std::size_t(s - s0) * 28;
    const S r0 = row[0], r1 = row[1], wt = row[26];
    S jp0[3], jp1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      jp0[k] = row[2 + 9 + k];
      jp1[k] = row[14 + 9 + k];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) c[i][j] = fa(c[i][j], fm(wt, fa(fm(jp0[i], jp0[j]), fm(jp1[i], jp1[j]))));
      g[i] = fs(g[i], fm(wt, fa(fm(jp0[i], r0), fm(jp1[i], r1))));
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) C[std::size_t(p) * 9 + i * 3 + j] = c[i][j];
    wv[std::size_t(p) * 3 + i] = g[i];
  }
}

// B[c] += w Jc^T Jc, v[c] -= w Jc^T r (dba/block_matrix.hpp:378-385), one CTA
// per local camera over its camera-major slots of the Jb batch starting at
// slot s0. With several batches (carry != nullptr) a CTA per camera the
// batch touches (cam_list) adds its double sums to `carry` (54 per camera)
// and k_carry_out writes B and v after the last batch.
template <class S, int NT>
__global__ void __launch_bounds__(NT) k_assemble_cameras(const std::int32_t* __restrict__ cam_ptr,
                                                         const std::int32_t* __restrict__ cam_glob,
                                                         const std::int32_t* __restrict__ cslot_pslot,
                                                         std::int64_t s0, const S* __restrict__ Jb,
                                                         S* __restrict__ B, S* __restrict__ v,
                                                         double* __restrict__ carry,
                                                         const std::int32_t* __restrict__ cam_list) {
  const std::int32_t lc = cam_list ? cam_list[blockIdx.x] : static_cast<std::int32_t>(blockIdx.x);
  double acc[54];  // 45 upper-triangular B entries + 9 v entries
#pragma unroll
  for (int k = 0; k < 54; ++k) acc[k] = 0.0;
  for (std::int32_t cs = cam_ptr[lc] + threadIdx.x; cs < cam_ptr[lc + 1]; cs += NT) {
    const std::int32_t ps = cslot_pslot[cs];
    const S* row = Jb + std::size_t(ps - s0) * 28;
    S jc0[9], jc1[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      jc0[k] = row[2 + k];
      jc1[k] = row[14 + k];
    }
    const S r0 = row[0], r1 = row[1], wt = row[26];
    int q = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) acc[q++] += double(fm(wt, fa(fm(jc0[i], jc0[j]), fm(jc1[i], jc1[j]))));
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[45 + i] -= double(fm(wt, fa(fm(jc0[i], r0), fm(jc1[i], r1))));
  }
  __shared__ double red[32];
  const std::int32_t cg = cam_glob[lc];
  int q = 0;
  double out[54];
#pragma unroll
  for (int k = 0; k < 54; ++k) out[k] = block_reduce<SumOp>(acc[k], red);
  if (threadIdx.x == 0 && carry) {
    double* cy = carry + std::size_t(lc) * 54;
#pragma unroll
    for (int k = 0; k < 54; ++k) cy[k] += out[k];
  }
  if (threadIdx.x == 0 && !carry) {
    S* b = B + std::size_t(cg) * 81;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) {
        b[i * 9 + j] = S(out[q]);
        b[j * 9 + i] = S(out[q]);
        ++q;
      }
#pragma unroll
    for (int i = 0; i < 9; ++i) v[std::size_t(cg) * 9 + i] = S(out[45 + i]);
  }
}

// B and v of every local camera from the batch sums (multi-batch assembly).
template <class S>
__global__ void k_carry_out(std::int32_t m_loc, const std::int32_t* __restrict__ cam_glob,
                            const double* __restrict__ carry, S* __restrict__ B, S* __restrict__ v) {
  const std::int32_t lc = blockIdx.x * blockDim.x + threadIdx.x;
  if (lc >= m_loc) return;
  const double* cy = carry + std::size_t(lc) * 54;
  S* b = B + std::size_t(cam_glob[lc]) * 81;
  int q = 0;
  for (int i = 0; i < 9; ++i)
    for (int j = i; j < 9; ++j) {
      b[i * 9 + j] = S(cy[q]);
      b[j * 9 + i] = S(cy[q]);
      ++q;
    }
  for (int i = 0; i < 9; ++i) v[std::size_t(cam_glob[lc]) * 9 + i] = S(cy[45 + i]);
}

// ------------------------------------------------------ damp + factor ----
// damp_into (dba/block_matrix.hpp:86-99) + per-block LLT that fails on a
// pivot <= 0 (Eigen llt_inplace::unblocked semantics, :123-134); stores the
// lower factor for the solves. Thread per block.
template <class S, int BS>
__global__ void k_damp_factor(std::int64_t nb, const S* __restrict__ A, S lambda, int policy, S* __restrict__ Ad,
                              S* __restrict__ Ainv, const std::int32_t* __restrict__ index_map,
                              unsigned long long* bad) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i >= nb) return;
  S m[BS][BS];
  const S* a = A + std::size_t(i) * BS * BS;
#pragma unroll
  for (int r = 0; r < BS; ++r)
#pragma unroll
    for (int c = 0; c < BS; ++c) m[r][c] = a[r * BS + c];
#pragma unroll
  for (int j = 0; j < BS; ++j) {
    if (policy == 0) {
      m[j][j] += lambda;
    } else {
      const S d = m[j][j];
      const S cl = fmin(S(1e32), fmax(S(1e-6), d));
      m[j][j] += lambda * cl;
    }
  }
  S* ad = Ad + std::size_t(i) * BS * BS;
#pragma unroll
  for (int r = 0; r < BS; ++r)
#pragma unroll
    for (int c = 0; c < BS; ++c) ad[r * BS + c] = m[r][c];
  // Cholesky, lower factor in m's lower triangle
  bool ok = true;
#pragma unroll
  for (int k = 0; k < BS; ++k) {
    S x = m[k][k];
    if (k > 0) {
      S sq = S(0);
#pragma unroll
      for (int j = 0; j < k; ++j) sq += m[k][j] * m[k][j];
      x -= sq;
    }
    if (!(x > S(0)) && !(x != x)) {  // x <= 0 fails; NaN passes (Eigen)
      ok = false;
      break;
    }
    x = sqrt(x);
    m[k][k] = x;
#pragma unroll
    for (int r = k + 1; r < BS; ++r) {
      S acc = m[r][k];
#pragma unroll
      for (int j = 0; j < k; ++j) acc -= m[r][j] * m[k][j];
      m[r][k] = acc / x;
    }
  }
  if (!ok) {
    atomicMin(bad, (unsigned long long)(index_map ? index_map[i] : i));
    return;
  }
  // The factor L (row-major lower triangle, zeros above) — solves are the
  // reference's forward + back substitution (dba/block_matrix.hpp:140-150).
  S* ai = Ainv + std::size_t(i) * BS * BS;
#pragma unroll
  for (int r = 0; r < BS; ++r)
#pragma unroll
    for (int c = 0; c < BS; ++c) ai[r * BS + c] = c <= r ? m[r][c] : S(0);
#pragma unroll
  for (int k = 0; k < BS; ++k) ai[rcp_at<BS>(k)] = S(1) / m[k][k];
}

// Position of 1/L_kk in the (otherwise unused) upper triangle of a stored
// factor: row 0 for k < BS-1, (1, 2) for the last one.
template <int BS>
__host__ __device__ constexpr int rcp_at(int k) {
  return k < BS - 1 ? k + 1 : BS + 2;
}

// x := (L L^T)^-1 x — the reference's forward + back substitution
// (dba/block_matrix.hpp:140-150) with the divisions by L_kk replaced by
// multiplications with the stored reciprocals.
template <class S, int BS>
__device__ __forceinline__ void llt_solve(const S* __restrict__ L, S* x) {
#pragma unroll
  for (int r = 0; r < BS; ++r) {
    S acc = x[r];
#pragma unroll
    for (int c = 0; c < r; ++c) acc -= L[r * BS + c] * x[c];
    x[r] = acc * L[rcp_at<BS>(r)];
  }
#pragma unroll
  for (int r = BS - 1; r >= 0; --r) {
    S acc = x[r];
#pragma unroll
    for (int c = r + 1; c < BS; ++c) acc -= L[c * BS + r] * x[c];
    x[r] = acc * L[rcp_at<BS>(r)];
  }
}

// x := D^-1 x per block from the stored factor (FactoredBlockDiagonal::
// solve_in_place, dba/block_matrix.hpp:140-152). Thread per block.
template <class S, int BS>
__global__ void k_block_solve(std::int64_t nb, const S* __restrict__ L, S* __restrict__ x) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i >= nb) return;
  S v[BS];
#pragma unroll
  for (int r = 0; r < BS; ++r) v[r] = x[std::size_t(i) * BS + r];
  llt_solve<S, BS>(L + std::size_t(i) * BS * BS, v);
#pragma unroll
  for (int r = 0; r < BS; ++r) x[std::size_t(i) * BS + r] = v[r];
}

// Explicit inverse of SPD blocks from their stored factor (L with 1/L_kk in
// the upper triangle): A^-1 = L^-T L^-1. Used for the block-Jacobi
// preconditioner z = B^-1 r (dba/solver.hpp:224-225) as a 9x9 GEMV.
template <class S, int BS>
__global__ void k_block_inverse(std::int64_t nb, const S* __restrict__ L, S* __restrict__ out) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i >= nb) return;
  const S* l = L + std::size_t(i) * BS * BS;
  S li[BS][BS];
#pragma unroll
  for (int c = 0; c < BS; ++c)
#pragma unroll
    for (int r = 0; r < BS; ++r) {
      if (r < c) {
        li[r][c] = S(0);
      } else {
        S acc = (r == c) ? S(1) : S(0);
#pragma unroll
        for (int k = c; k < r; ++k) acc -= l[r * BS + k] * li[k][c];
        li[r][c] = acc * l[rcp_at<BS>(r)];
      }
    }
  S* o = out + std::size_t(i) * BS * BS;
#pragma unroll
  for (int r = 0; r < BS; ++r)
#pragma unroll
    for (int c = r; c < BS; ++c) {
      S acc = S(0);
#pragma unroll
      for (int k = c; k < BS; ++k) acc += li[k][r] * li[k][c];
      o[r * BS + c] = acc;
      o[c * BS + r] = acc;
    }
}

// -------------------------------------------------------------- halo ----
// Finish of the MODE 1 pass (dse.cuh) for halo points after the all-reduce.
template <class S, int MODE>
__global__ void k_halo_finish(std::int32_t n, const std::int32_t* __restrict__ lpts,
                              const std::int32_t* __restrict__ hidx, const S* __restrict__ halo_buf,
                              const S* __restrict__ Cinv, const S* __restrict__ wv, S* __restrict__ out) {
  const std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const std::int32_t p = lpts[i];
  S t[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) t[j] = halo_buf[std::size_t(hidx[i]) * 3 + j];
  if (MODE == 1)
#pragma unroll
    for (int j = 0; j < 3; ++j) t[j] = wv[std::size_t(p) * 3 + j] - t[j];
  llt_solve<S, 3>(Cinv + std::size_t(p) * 9, t);
#pragma unroll
  for (int r = 0; r < 3; ++r) out[std::size_t(p) * 3 + r] = t[r];
}

// Halo scatter / gather of W-wide point records.
template <class S, int W>
__global__ void k_halo_scatter(std::int32_t n, const std::int32_t* __restrict__ lpts,
                               const std::int32_t* __restrict__ hidx, const S* __restrict__ src,
                               S* __restrict__ halo) {
  const std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < W; ++k) halo[std::size_t(hidx[i]) * W + k] = src[std::size_t(lpts[i]) * W + k];
}
template <class S, int W>
__global__ void k_halo_gather(std::int32_t n, const std::int32_t* __restrict__ lpts,
                              const std::int32_t* __restrict__ hidx, const S* __restrict__ halo,
                              S* __restrict__ dst) {
  const std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < W; ++k) dst[std::size_t(lpts[i]) * W + k] = halo[std::size_t(hidx[i]) * W + k];
}

// -------------------------------------------------------- camera space ----
// PCG scalars kept on the device so the recurrences never round-trip.
template <class S>
struct PcgScal {
  double rho, rho_prev, pq, rnorm2, rhs_norm2;
  double dot_a, dot_b, dot_c;  // generic reduction outputs
  S alpha, beta;
  int status;  // bit 1: rho breakdown, bit 2: pq breakdown
  int n;
};

// ----------------------------------------------------- DSE camera side ----
// Halo slots after the all-reduce of their points' a_p: b_p = C_p^-1 a_p,
// y_s = E_s b_p into the slot's own partial.
template <class S, class T = S, int L = kLanesFact>
__global__ void k_halo_fix(std::int32_t n, const std::int32_t* __restrict__ halo_slot,
                           const std::int32_t* __restrict__ slot_dpt, const std::int32_t* __restrict__ halo_of,
                           const S* __restrict__ halo_buf, const S* __restrict__ Cinv, const T* __restrict__ E,
                           const std::int32_t* __restrict__ slot_chunk, const std::int32_t* __restrict__ chunk_slot,
                           const std::int32_t* __restrict__ halo_pos, S* __restrict__ part,
                           const std::int32_t* __restrict__ slot_cam, const S* __restrict__ Rm) {
  const std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const std::int32_t s = halo_slot[i];
  const std::int32_t p = slot_dpt[s];
  S b[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) b[j] = halo_buf[std::size_t(halo_of[p]) * 3 + j];
  llt_solve<S, 3>(Cinv + std::size_t(p) * 9, b);
  const T* ep = E + rec_at<T, L>(slot_chunk, chunk_slot, s);
  S e[L], y[9];
#pragma unroll
  for (int k = 0; k < L; ++k) e[k] = S(ep[std::size_t(k) * kTile]);
  coupling_b<S, L>(e, L == kLanesFact ? Rm + std::size_t(slot_cam[s]) * 9 : nullptr, b[0], b[1], b[2], y);
#pragma unroll
  for (int r = 0; r < 9; ++r) part[std::size_t(halo_pos[i]) * 9 + r] = y[r];
}

// Point rows between global order and device-point order:
// SCATTER = false: dev[d] = glob[idx[d]]; true: glob[idx[d]] = dev[d].
template <class S, bool SCATTER>
__global__ void k_point_rows(std::int32_t n, const std::int32_t* __restrict__ idx, const S* __restrict__ src,
                             S* __restrict__ dst) {
  const std::int32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const std::size_t g = std::size_t(idx[d]) * 3, l = std::size_t(d) * 3;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (SCATTER)
      dst[g + k] = src[l + k];
    else
      dst[l + k] = src[g + k];
  }
}

// glob[idx[d]] = dev[d] for the points this rank owns (gather_state).
template <class S>
__global__ void k_owned_rows(std::int32_t n, const std::int32_t* __restrict__ idx,
                             const std::uint8_t* __restrict__ owned, const S* __restrict__ src, S* __restrict__ dst) {
  const std::int32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n || !owned[d]) return;
  const std::size_t g = std::size_t(idx[d]) * 3, l = std::size_t(d) * 3;
#pragma unroll
  for (int k = 0; k < 3; ++k) dst[g + k] = src[l + k];
}

// rows[idx[i]] = 0 for W-wide rows.
template <class S, int W>
__global__ void k_zero_rows(std::int32_t n, const std::int32_t* __restrict__ idx, S* __restrict__ rows) {
  const std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < W; ++k) rows[std::size_t(idx[i]) * W + k] = S(0);
}

// c_cam = fold of the camera's partials in chunk order (warp per camera, lanes
// strided, fixed shuffle tree), then per EPI:
//   0: out = c (all m cameras written; the all-reduce follows for K > 1)
//   1: out = q = B_d x - c and p.q -> alpha (DSE, K = 1, dba/solver.hpp:166)
//   2: out = g = v - c (right-hand side, K = 1, dba/solver.hpp:363)
template <class S, int EPI>
__global__ void __launch_bounds__(kRedThreads) k_cam_reduce(std::int32_t m, const std::int32_t* __restrict__ cam_part_ptr,
                                                            const std::int32_t* __restrict__ cam_part,
                                                            const S* __restrict__ part, const S* __restrict__ Bd,
                                                            const S* __restrict__ x, const S* __restrict__ v,
                                                            S* __restrict__ out, RedWs ws, PcgScal<S>* sc) {
  const int lane = threadIdx.x & 31;
  const std::int32_t cam = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double pq = 0.0;
  if (cam < m) {
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
      acc[i] = __shfl_sync(0xffffffffu, acc[i], 0);
    }
    if (lane < 9) {
      S c = acc[0];
#pragma unroll
      for (int i = 1; i < 9; ++i)
        if (lane == i) c = acc[i];
      S o;
      if (EPI == 0) {
        o = c;
      } else if (EPI == 2) {
        o = v[std::size_t(cam) * 9 + lane] - c;
      } else {
        const S* b = Bd + std::size_t(cam) * 81 + lane * 9;
        const S* xv = x + std::size_t(cam) * 9;
        S d = S(0);
#pragma unroll
        for (int k = 0; k < 9; ++k) d += b[k] * xv[k];
        o = d - c;
        pq = double(xv[lane]) * double(o);
      }
      out[std::size_t(cam) * 9 + lane] = o;
    }
  }
  if (EPI == 1) {
    const double vv[1] = {pq};
    __shared__ double fin[1];
    if (grid_reduce<SumOp, 1>(vv, ws.partials, ws.counter, fin)) {
      if (threadIdx.x == 0) {
        const double r = fin[0];
        sc->pq = r;
        if (!(r > 0.0) || isinf(r)) sc->status |= 2;
        sc->alpha = S(sc->rho / r);
      }
    }
  }
}

// q = Bd x - c, and p.q in double when PQ (dba/solver.hpp:166-167, 238).
template <class S, bool PQ>
__global__ void __launch_bounds__(kRedThreads) k_cam_epilogue(std::int32_t m, const S* __restrict__ Bd,
                                                              const S* __restrict__ x, const S* __restrict__ c,
                                                              S* __restrict__ q, RedWs ws, PcgScal<S>* sc) {
  double acc = 0.0;
  for (std::int32_t cam = blockIdx.x * blockDim.x + threadIdx.x; cam < m; cam += gridDim.x * blockDim.x) {
    const S* b = Bd + std::size_t(cam) * 81;
    S xv[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) xv[k] = x[std::size_t(cam) * 9 + k];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      S s = S(0);
#pragma unroll
      for (int k = 0; k < 9; ++k) s += b[r * 9 + k] * xv[k];
      const S qv = s - c[std::size_t(cam) * 9 + r];
      q[std::size_t(cam) * 9 + r] = qv;
      if (PQ) acc += double(xv[r]) * double(qv);
    }
  }
  if (PQ) {
    const double v[1] = {acc};
    __shared__ double fin[1];
    if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin)) {
      if (threadIdx.x == 0) {
        const double pq = fin[0];
        sc->pq = pq;
        if (!(pq > 0.0) || isinf(pq)) sc->status |= 2;
        sc->alpha = S(sc->rho / pq);
      }
    }
  }
}

// z = B^-1 r, rho = r.z; beta = (S)(rho / rho_prev) (dba/solver.hpp:224-236).
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_pcg_precond(std::int32_t m, const S* __restrict__ Binv,
                                                             const S* __restrict__ r, S* __restrict__ z, RedWs ws,
                                                             PcgScal<S>* sc) {
  double acc = 0.0;
  for (std::int32_t cam = blockIdx.x * blockDim.x + threadIdx.x; cam < m; cam += gridDim.x * blockDim.x) {
    S rv[9], zv[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) zv[k] = rv[k] = r[std::size_t(cam) * 9 + k];
    llt_solve<S, 9>(Binv + std::size_t(cam) * 81, zv);
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      z[std::size_t(cam) * 9 + i] = zv[i];
      acc += double(rv[i]) * double(zv[i]);
    }
  }
  const double v[1] = {acc};
  __shared__ double fin[1];
  if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin)) {
    if (threadIdx.x == 0) {
      const double rho = fin[0];
      sc->rho = rho;
      if (!(rho > 0.0) || isinf(rho)) sc->status |= 1;
      sc->beta = sc->n == 0 ? S(0) : S(rho / sc->rho_prev);
    }
  }
}

// z = B^-1 r with the explicit inverse (thread per element) and rho = r.z
// in double; beta = (S)(rho / rho_prev) (dba/solver.hpp:224-236).
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_pcg_precond_inv(std::int32_t m, const S* __restrict__ Binv,
                                                                 const S* __restrict__ r, S* __restrict__ z, RedWs ws,
                                                                 PcgScal<S>* sc) {
  double acc = 0.0;
  const std::int64_t len = std::int64_t(m) * 9;
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t cam = i / 9, row = i % 9;
    const S* bi = Binv + cam * 81 + row * 9;
    const S* rc = r + cam * 9;
    S zv = S(0);
#pragma unroll
    for (int k = 0; k < 9; ++k) zv += bi[k] * rc[k];
    z[i] = zv;
    acc += double(r[i]) * double(zv);
  }
  const double v[1] = {acc};
  __shared__ double fin[1];
  if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin)) {
    if (threadIdx.x == 0) {
      const double rho = fin[0];
      sc->rho = rho;
      if (!(rho > 0.0) || isinf(rho)) sc->status |= 1;
      sc->beta = sc->n == 0 ? S(0) : S(rho / sc->rho_prev);
    }
  }
}

// p = z (n == 0) or z + beta p.
template <class S>
__global__ void k_pcg_p(std::int64_t len, const S* __restrict__ z, S* __restrict__ p, const PcgScal<S>* sc) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i >= len) return;
  if (sc->n == 0) p[i] = z[i];
  else p[i] = z[i] + sc->beta * p[i];
}

// x += alpha p; if UPD_R: r -= alpha q and |r|^2 (dba/solver.hpp:243-254).
template <class S, bool UPD_R>
__global__ void __launch_bounds__(kRedThreads) k_pcg_xr(std::int64_t len, const S* __restrict__ p,
                                                        const S* __restrict__ q, S* __restrict__ x,
                                                        S* __restrict__ r, RedWs ws, PcgScal<S>* sc) {
  const S alpha = sc->alpha;
  double acc = 0.0;
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    x[i] += alpha * p[i];
    if (UPD_R) {
      const S rv = r[i] - alpha * q[i];
      r[i] = rv;
      acc += double(rv) * double(rv);
    }
  }
  if (UPD_R) {
    const double v[1] = {acc};
    __shared__ double fin[1];
    if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin)) {
      if (threadIdx.x == 0) {
        sc->rnorm2 = fin[0];
        sc->rho_prev = sc->rho;
        sc->n += 1;
      }
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    // counter bookkeeping done by the refresh kernel
  }
}

// r = g - q and |r|^2 (the every-50 refresh, and the start r = g - S x0).
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_pcg_refresh(std::int64_t len, const S* __restrict__ g,
                                                             const S* __restrict__ q, S* __restrict__ r, RedWs ws,
                                                             PcgScal<S>* sc, int bump) {
  double acc = 0.0;
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const S rv = g[i] - q[i];
    r[i] = rv;
    acc += double(rv) * double(rv);
  }
  const double v[1] = {acc};
  __shared__ double fin[1];
  if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin)) {
    if (threadIdx.x == 0) {
      sc->rnorm2 = fin[0];
      if (bump) {
        sc->rho_prev = sc->rho;
        sc->n += 1;
      }
    }
  }
}

// Generic double dot of two S vectors into sc->dot_a.
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_dot(std::int64_t len, const S* __restrict__ a,
                                                     const S* __restrict__ b, RedWs ws, double* out) {
  double acc = 0.0;
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x)
    acc += double(a[i]) * double(b[i]);
  const double v[1] = {acc};
  __shared__ double fin[1];
  if (grid_reduce<SumOp, 1>(v, ws.partials, ws.counter, fin))
    if (threadIdx.x == 0) *out = fin[0];
}

// out = a - b.
template <class S>
__global__ void k_sub(std::int64_t len, const S* __restrict__ a, const S* __restrict__ b, S* __restrict__ out) {
  const std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  if (i < len) out[i] = a[i] - b[i];
}

// ---------------------------------------------------------- trial / model ----
// trial = x + dx, and the model terms of dba/solver.hpp:383-410 over one
// parameter block family: out[0] = max |dx|, out[1] = damping sum
// (identity: sum dx^2, scaled by lambda on the host; diag_scaled:
// sum lambda clamp(D_jj) dx^2), out[2] = dx . grad. BS = 9 (cameras, all
// entries) or 3 (local points, owned ones only for the sums).
template <class S, int BS>
__global__ void __launch_bounds__(kRedThreads) k_trial(std::int32_t nb, const S* __restrict__ x,
                                                       const S* __restrict__ dx, S* __restrict__ xt,
                                                       const S* __restrict__ D, const S* __restrict__ grad,
                                                       const std::uint8_t* __restrict__ owned, double lambda,
                                                       int policy, RedWs ws, double* out) {
  double smax = 0.0, damp = 0.0, gv = 0.0;
  for (std::int32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const bool own = owned ? owned[b] != 0 : true;
#pragma unroll
    for (int k = 0; k < BS; ++k) {
      const std::size_t i = std::size_t(b) * BS + k;
      const S d = dx[i];
      xt[i] = x[i] + d;
      if (own) {
        const double dd = double(d);
        smax = fmax(smax, fabs(dd));
        if (policy == 0) {
          damp += dd * dd;
        } else {
          const S djj = D[std::size_t(b) * BS * BS + k * BS + k];
          const S cl = fmin(S(1e32), fmax(S(1e-6), djj));
          damp += lambda * double(cl) * dd * dd;
        }
        gv += dd * double(grad[i]);
      }
    }
  }
  __shared__ double red[32];
  __shared__ bool last;
  const double bm = block_reduce<MaxOp>(smax, red);
  const double bd = block_reduce<SumOp>(damp, red);
  const double bg = block_reduce<SumOp>(gv, red);
  if (threadIdx.x == 0) {
    ws.partials[blockIdx.x] = bm;
    ws.partials[gridDim.x + blockIdx.x] = bd;
    ws.partials[2 * gridDim.x + blockIdx.x] = bg;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ws.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double m0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    m0 = fmax(m0, __ldcg(ws.partials + i));
    s1 += __ldcg(ws.partials + gridDim.x + i);
    s2 += __ldcg(ws.partials + 2 * gridDim.x + i);
  }
  m0 = block_reduce<MaxOp>(m0, red);
  s1 = block_reduce<SumOp>(s1, red);
  s2 = block_reduce<SumOp>(s2, red);
  if (threadIdx.x == 0) {
    out[0] = m0;
    out[1] = s1;
    out[2] = s2;
    *ws.counter = 0u;
  }
}

// Ascending-rank sum of K deposited buffers (WorkerGroup::allreduce_sum,
// dba/comms.hpp:76-81): out = ((s0 + s1) + s2) + ...
template <class T>
__global__ void k_sum_slots(std::int64_t len, int k, const T* const* __restrict__ slots, T* __restrict__ out) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < len;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    T acc = slots[0][i];
    for (int r = 1; r < k; ++r) acc += slots[r][i];
    out[i] = acc;
  }
}

}  // namespace dev
}  // namespace dbag
