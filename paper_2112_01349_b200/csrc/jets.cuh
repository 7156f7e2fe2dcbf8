// jets.cuh — register-resident forward-mode dual numbers for sm_100a.
//
// The reference's JetVector (dba/jet_vector.hpp:21-332) is a lane-major SoA
// batch where every elementwise op materializes a full (1 + 12) x N output:
// 56 sweeps over memory per linearization. Here one thread
// owns one edge and its jets live in registers. Each Jet carries a
// compile-time lane mask of the gradient lanes that can be nonzero (lanes
// 0..8 camera, 9..11 point, dba/edge_eval.hpp:132-144), so structurally-zero
// lanes are never stored or computed. For the lanes that are computed the
// arithmetic is the reference's: product rule ga*vb + va*gb
// (jet_vector.hpp:188-189), quotient (ga - q gb)/vb (:227-228), chain rule
// through the rotation coefficients (:321-331); the op sequence of
// edge_autodiff() is the one of EdgeEvaluator::linearize_autodiff
// (dba/edge_eval.hpp:126-191) and rotate_angle_axis (jet_vector.hpp:429-473).
#pragma once

#include <cuda_runtime.h>

namespace dbag {
namespace dev {

template <class S>
__host__ __device__ constexpr S taylor_threshold() {
  return sizeof(S) == 8 ? S(1e-12) : S(1e-4);
}

// Round-to-nearest arithmetic that the compiler may not contract into FMAs:
// the jet and residual code below then performs exactly the IEEE operation
// sequence of the reference (compiled for x86-64 without FMA), so values
// agree with the CPU restatement bit-for-bit wherever sin/cos agree.
__device__ __forceinline__ double fm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fs(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fd(float a, float b) { return __fdiv_rn(a, b); }

// dba/problem.hpp:89-118
template <class S>
__device__ __forceinline__ void rot_coeffs(S t, S& c, S& s1, S& c2) {
  if (t < taylor_threshold<S>()) {
    c = fa(fs(S(1), fd(t, S(2))), fd(fm(t, t), S(24)));
    s1 = fa(fs(S(1), fd(t, S(6))), fd(fm(t, t), S(120)));
    c2 = fa(fs(S(0.5), fd(t, S(24))), fd(fm(t, t), S(720)));
  } else {
    const S th = sqrt(t);
    S sn, cs;
    if constexpr (sizeof(S) == 8) sincos(th, &sn, &cs);
    else sincosf(th, &sn, &cs);
    c = cs;
    s1 = fd(sn, th);
    c2 = fd(fs(S(1), c), t);
  }
}
template <class S>
__device__ __forceinline__ void rot_dcoeffs(S t, S c, S s1, S c2, S& dc, S& ds1, S& dc2) {
  if (t < taylor_threshold<S>()) {
    dc = fa(S(-0.5), fd(t, S(12)));
    ds1 = fa(fd(S(-1), S(6)), fd(t, S(60)));
    dc2 = fa(fd(S(-1), S(24)), fd(t, S(360)));
  } else {
    dc = fd(-s1, S(2));
    ds1 = fd(fs(c, s1), fm(S(2), t));
    dc2 = fd(fs(fd(s1, S(2)), c2), t);
  }
}

template <class S, unsigned M>
struct Jet {
  S v;
  S g[12];
};

#define DBAG_LANES _Pragma("unroll") for (int j = 0; j < 12; ++j)

template <class S, int L>
__device__ __forceinline__ Jet<S, (1u << L)> seed(S v) {
  Jet<S, (1u << L)> o;
  o.v = v;
  DBAG_LANES o.g[j] = (j == L) ? S(1) : S(0);
  return o;
}

template <class S, unsigned A, unsigned B>
__device__ __forceinline__ Jet<S, A | B> operator+(const Jet<S, A>& a, const Jet<S, B>& b) {
  Jet<S, A | B> o;
  DBAG_LANES {
    const bool ia = (A >> j) & 1u, ib = (B >> j) & 1u;
    o.g[j] = (ia && ib) ? fa(a.g[j], b.g[j]) : ia ? a.g[j] : ib ? b.g[j] : S(0);
  }
  o.v = fa(a.v, b.v);
  return o;
}

template <class S, unsigned A, unsigned B>
__device__ __forceinline__ Jet<S, A | B> operator-(const Jet<S, A>& a, const Jet<S, B>& b) {
  Jet<S, A | B> o;
  DBAG_LANES {
    const bool ia = (A >> j) & 1u, ib = (B >> j) & 1u;
    o.g[j] = (ia && ib) ? fs(a.g[j], b.g[j]) : ia ? a.g[j] : ib ? -b.g[j] : S(0);
  }
  o.v = fs(a.v, b.v);
  return o;
}

template <class S, unsigned A, unsigned B>
__device__ __forceinline__ Jet<S, A | B> operator*(const Jet<S, A>& a, const Jet<S, B>& b) {
  Jet<S, A | B> o;
  DBAG_LANES {
    const bool ia = (A >> j) & 1u, ib = (B >> j) & 1u;
    o.g[j] = (ia && ib) ? fa(fm(a.g[j], b.v), fm(a.v, b.g[j])) : ia ? fm(a.g[j], b.v) : ib ? fm(a.v, b.g[j]) : S(0);
  }
  o.v = fm(a.v, b.v);
  return o;
}

template <class S, unsigned A, unsigned B>
__device__ __forceinline__ Jet<S, A | B> operator/(const Jet<S, A>& a, const Jet<S, B>& b) {
  Jet<S, A | B> o;
  o.v = fd(a.v, b.v);
  DBAG_LANES {
    const bool ia = (A >> j) & 1u, ib = (B >> j) & 1u;
    o.g[j] = (ia && ib) ? fd(fs(a.g[j], fm(o.v, b.g[j])), b.v)
             : ia       ? fd(a.g[j], b.v)
             : ib       ? fd(fs(S(0), fm(o.v, b.g[j])), b.v)
                        : S(0);
  }
  return o;
}

template <class S, unsigned A>
__device__ __forceinline__ Jet<S, A> scale(const Jet<S, A>& a, S s) {  // mul_scalar
  Jet<S, A> o;
  DBAG_LANES o.g[j] = ((A >> j) & 1u) ? fm(a.g[j], s) : S(0);
  o.v = fm(a.v, s);
  return o;
}

template <class S, unsigned A>
__device__ __forceinline__ Jet<S, A> shift(const Jet<S, A>& a, S s) {  // add_scalar
  Jet<S, A> o;
  DBAG_LANES o.g[j] = ((A >> j) & 1u) ? a.g[j] : S(0);
  o.v = fa(a.v, s);
  return o;
}

// rotation_coefficients (jet_vector.hpp:293-332)
template <class S, unsigned A>
__device__ __forceinline__ void rotation_coefficients(const Jet<S, A>& t, Jet<S, A>& c, Jet<S, A>& s1,
                                                      Jet<S, A>& c2) {
  S dc, ds1, dc2;
  rot_coeffs(t.v, c.v, s1.v, c2.v);
  rot_dcoeffs(t.v, c.v, s1.v, c2.v, dc, ds1, dc2);
  DBAG_LANES {
    const bool on = (A >> j) & 1u;
    c.g[j] = on ? fm(dc, t.g[j]) : S(0);
    s1.g[j] = on ? fm(ds1, t.g[j]) : S(0);
    c2.g[j] = on ? fm(dc2, t.g[j]) : S(0);
  }
}

// Residual and the 2 x 12 local Jacobian of one edge by forward-mode jets,
// in the op order of EdgeEvaluator::linearize_autodiff. False on P_z == 0.
template <class S>
__device__ __forceinline__ bool edge_autodiff(const S* cam, const S* X, S pixx, S pixy, S* r, S (*J)[12]) {
  const auto a0 = seed<S, 0>(cam[0]);
  const auto a1 = seed<S, 1>(cam[1]);
  const auto a2 = seed<S, 2>(cam[2]);
  const auto t0 = seed<S, 3>(cam[3]);
  const auto t1 = seed<S, 4>(cam[4]);
  const auto t2 = seed<S, 5>(cam[5]);
  const auto f = seed<S, 6>(cam[6]);
  const auto k1 = seed<S, 7>(cam[7]);
  const auto k2 = seed<S, 8>(cam[8]);
  const auto x0 = seed<S, 9>(X[0]);
  const auto x1 = seed<S, 10>(X[1]);
  const auto x2 = seed<S, 11>(X[2]);

  // rotate_angle_axis: t = (a0^2 + a1^2) + a2^2
  const auto t = (a0 * a0 + a1 * a1) + a2 * a2;
  Jet<S, 7u> c, s1, c2;
  rotation_coefficients(t, c, s1, c2);
  const auto dot = ((a0 * x0 + a1 * x1) + a2 * x2) * c2;
  const auto cr0 = (a1 * x2 - a2 * x1) * s1;
  const auto cr1 = (a2 * x0 - a0 * x2) * s1;
  const auto cr2 = (a0 * x1 - a1 * x0) * s1;
  const auto P0 = ((x0 * c + cr0) + a0 * dot) + t0;
  const auto P1 = ((x1 * c + cr1) + a1 * dot) + t1;
  const auto P2 = ((x2 * c + cr2) + a2 * dot) + t2;
  if (P2.v == S(0)) return false;

  // p = -(P_x, P_y) / P_z  (div then neg = mul_scalar(-1))
  const auto ux = scale(P0 / P2, S(-1));
  const auto uy = scale(P1 / P2, S(-1));
  // distortion = (n2 k1 + (n2 n2) k2) + 1, scale = distortion * f
  const auto n2 = ux * ux + uy * uy;
  const auto dist = shift(n2 * k1 + (n2 * n2) * k2, S(1)) * f;
  const auto rx = ux * dist;
  const auto ry = uy * dist;
  r[0] = fs(rx.v, pixx);
  r[1] = fs(ry.v, pixy);
  DBAG_LANES {
    J[0][j] = rx.g[j];
    J[1][j] = ry.g[j];
  }
  return true;
}

// Closed-form Jacobian (EdgeEvaluator::linearize_analytic,
// dba/edge_eval.hpp:199-285).
template <class S>
__device__ __forceinline__ bool edge_analytic(const S* cm, const S* x, S pixx, S pixy, S* r, S (*J)[12]) {
  const S aa[3] = {cm[0], cm[1], cm[2]};
  const S t = (aa[0] * aa[0] + aa[1] * aa[1]) + aa[2] * aa[2];
  S c, s1, c2, dc, ds1, dc2;
  rot_coeffs(t, c, s1, c2);
  rot_dcoeffs(t, c, s1, c2, dc, ds1, dc2);
  const S cr[3] = {aa[1] * x[2] - aa[2] * x[1], aa[2] * x[0] - aa[0] * x[2], aa[0] * x[1] - aa[1] * x[0]};
  const S dot = (aa[0] * x[0] + aa[1] * x[1]) + aa[2] * x[2];
  S P[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) P[k] = ((x[k] * c + cr[k] * s1) + aa[k] * (dot * c2)) + cm[3 + k];
  if (P[2] == S(0)) return false;
  S dtt[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dtt[k] = (x[k] * dc + cr[k] * ds1) + aa[k] * (dot * dc2);
  // e_j x x
  const S ejx[3][3] = {{S(0), -x[2], x[1]}, {x[2], S(0), -x[0]}, {-x[1], x[0], S(0)}};
  S dPda[3][3];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      dPda[k][j] = ((S(2) * aa[j] * dtt[k] + ejx[j][k] * s1) + (k == j ? S(1) : S(0)) * (dot * c2)) +
                   aa[k] * (x[j] * c2);
  const S skew[3][3] = {{S(0), -aa[2], aa[1]}, {aa[2], S(0), -aa[0]}, {-aa[1], aa[0], S(0)}};
  S R[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) R[a][b] = ((a == b ? c : S(0)) + s1 * skew[a][b]) + c2 * (aa[a] * aa[b]);
  const S u[2] = {-P[0] / P[2], -P[1] / P[2]};
  const S n2 = u[0] * u[0] + u[1] * u[1];
  const S dist = (S(1) + cm[7] * n2) + cm[8] * n2 * n2;
  const S iz = S(1) / P[2];
  const S dudp[2][3] = {{-iz, S(0), P[0] * iz * iz}, {S(0), -iz, P[1] * iz * iz}};
  const S kk = S(2) * (cm[7] + S(2) * cm[8] * n2);
  S drdu[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) drdu[a][b] = cm[6] * ((a == b ? dist : S(0)) + kk * (u[a] * u[b]));
  S drdp[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) drdp[a][b] = drdu[a][0] * dudp[0][b] + drdu[a][1] * dudp[1][b];
  r[0] = cm[6] * dist * u[0] - pixx;
  r[1] = cm[6] * dist * u[1] - pixy;
#pragma unroll
  for (int col = 0; col < 3; ++col) {
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      J[a][col] = (drdp[a][0] * dPda[0][col] + drdp[a][1] * dPda[1][col]) + drdp[a][2] * dPda[2][col];
      J[a][3 + col] = drdp[a][col];
      J[a][9 + col] = (drdp[a][0] * R[0][col] + drdp[a][1] * R[1][col]) + drdp[a][2] * R[2][col];
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    J[a][6] = dist * u[a];
    J[a][7] = cm[6] * n2 * u[a];
    J[a][8] = cm[6] * n2 * n2 * u[a];
  }
  return true;
}

// Scalar Snavely residual (dba/problem.hpp:125-165), same op order as the
// jet composition, so its value equals the jets' value lanes bit-for-bit.
template <class S>
__device__ __forceinline__ bool edge_residual(const S* cam, const S* x, S pixx, S pixy, S* r) {
  const S t = fa(fa(fm(cam[0], cam[0]), fm(cam[1], cam[1])), fm(cam[2], cam[2]));
  S c, s1, c2;
  rot_coeffs(t, c, s1, c2);
  const S dc2 = fm(fa(fa(fm(cam[0], x[0]), fm(cam[1], x[1])), fm(cam[2], x[2])), c2);
  const S cr0 = fs(fm(cam[1], x[2]), fm(cam[2], x[1]));
  const S cr1 = fs(fm(cam[2], x[0]), fm(cam[0], x[2]));
  const S cr2 = fs(fm(cam[0], x[1]), fm(cam[1], x[0]));
  const S P0 = fa(fa(fa(fm(x[0], c), fm(cr0, s1)), fm(cam[0], dc2)), cam[3]);
  const S P1 = fa(fa(fa(fm(x[1], c), fm(cr1, s1)), fm(cam[1], dc2)), cam[4]);
  const S P2 = fa(fa(fa(fm(x[2], c), fm(cr2, s1)), fm(cam[2], dc2)), cam[5]);
  if (P2 == S(0)) return false;
  const S ux = -fd(P0, P2);
  const S uy = -fd(P1, P2);
  const S n2 = fa(fm(ux, ux), fm(uy, uy));
  const S dist = fa(fa(fm(n2, cam[7]), fm(fm(n2, n2), cam[8])), S(1));
  const S sc = fm(dist, cam[6]);
  r[0] = fs(fm(ux, sc), pixx);
  r[1] = fs(fm(uy, sc), pixy);
  return true;
}

}  // namespace dev
}  // namespace dbag
