// synthetic.cpp — the reference's ring dataset generator, made count-exact and
// scalable.
//
// Follows generate_synthetic (dba/synthetic.hpp:70-146): radius-R ring of m
// cameras looking at the origin (look_at_origin :52-64, Eigen
// AngleAxisd(Matrix3d) via the quaternion, restated below), pose noise
// U(0, pose_noise), focal = base + U(0, intr), k1, k2 ~ U(0, intr); points
// (x, y, z) ~ (U(-.1,.1), U(-.1,.1), U(-.03,.03)) drawn in x -> y -> z order
// (the reference leaves this order to the compiler, dba/synthetic.hpp:108-109;
// here it is fixed), stored x, y get an extra U(-point_noise, point_noise);
// every point is observed by its Q nearest cameras (tie-break (dist2, id)),
// edges point-major with ascending camera ids, pixels = projections of the
// true points through the noisy cameras.
//
// Extensions: Q_p = floor(N/n) + [p < N mod n] when num_observations > 0, and
// U(-noise, noise) pixel noise from a second mt19937_64(seed) stream in edge
// order (tests/acceptance.cpp:88-99). The nearest-camera search is windowed
// around the point's azimuth (cameras sit at angles 2 pi i / m, so the Q
// nearest form an arc): O(n Q) instead of the reference's O(n m). It falls
// back to the exhaustive search when m is small.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "common.hpp"

namespace dbag {
namespace {

class Uniform {  // dba/synthetic.hpp:40-50
 public:
  explicit Uniform(std::uint64_t seed) : eng_(seed) {}
  double unit() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double range(double lo, double hi) { return lo + (hi - lo) * unit(); }

 private:
  std::mt19937_64 eng_;
};

struct V3 {
  double x, y, z;
};
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 normalized(const V3& a) {
  const double n2 = (a.x * a.x + a.y * a.y) + a.z * a.z;
  if (n2 > 0) {
    const double n = std::sqrt(n2);
    return {a.x / n, a.y / n, a.z / n};
  }
  return a;
}

// Eigen::AngleAxisd(Matrix3d): rotation matrix -> quaternion -> angle-axis.
void angle_axis_from_matrix(const double r[3][3], double out[3]) {
  double q[4];  // x y z w
  double t = (r[0][0] + r[1][1]) + r[2][2];
  if (t > 0) {
    t = std::sqrt(t + 1.0);
    q[3] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (r[2][1] - r[1][2]) * t;
    q[1] = (r[0][2] - r[2][0]) * t;
    q[2] = (r[1][0] - r[0][1]) * t;
  } else {
    int i = 0;
    if (r[1][1] > r[0][0]) i = 1;
    if (r[2][2] > r[i][i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = std::sqrt(r[i][i] - r[j][j] - r[k][k] + 1.0);
    q[i] = 0.5 * t;
    t = 0.5 / t;
    q[3] = (r[k][j] - r[j][k]) * t;
    q[j] = (r[j][i] + r[i][j]) * t;
    q[k] = (r[k][i] + r[i][k]) * t;
  }
  double n = std::sqrt((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]);
  if (n != 0.0) {
    const double angle = 2.0 * std::atan2(n, std::abs(q[3]));
    if (q[3] < 0) n = -n;
    for (int a = 0; a < 3; ++a) out[a] = angle * (q[a] / n);
  } else {
    out[0] = out[1] = out[2] = 0.0;
  }
}

// Snavely projection (dba/problem.hpp:125-165) of X through a camera.
bool project(const double* cam, const V3& X, double* pix) {
  const double aa[3] = {cam[0], cam[1], cam[2]};
  const double x[3] = {X.x, X.y, X.z};
  const double t = (aa[0] * aa[0] + aa[1] * aa[1]) + aa[2] * aa[2];
  double c, s1, c2;
  if (t < 1e-12) {
    c = 1.0 - t / 2.0 + t * t / 24.0;
    s1 = 1.0 - t / 6.0 + t * t / 120.0;
    c2 = 0.5 - t / 24.0 + t * t / 720.0;
  } else {
    const double th = std::sqrt(t);
    c = std::cos(th);
    s1 = std::sin(th) / th;
    c2 = (1.0 - c) / t;
  }
  const double dc2 = ((aa[0] * x[0] + aa[1] * x[1]) + aa[2] * x[2]) * c2;
  double p[3];
  for (int i = 0; i < 3; ++i) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
    const double cr = aa[i1] * x[i2] - aa[i2] * x[i1];
    p[i] = ((x[i] * c + cr * s1) + aa[i] * dc2) + cam[3 + i];
  }
  if (p[2] == 0.0) return false;
  const double ux = -(p[0] / p[2]), uy = -(p[1] / p[2]);
  const double n2 = ux * ux + uy * uy;
  const double dist = (n2 * cam[7] + (n2 * n2) * cam[8]) + 1.0;
  const double scale = dist * cam[6];
  pix[0] = ux * scale - 0.0;
  pix[1] = uy * scale - 0.0;
  return true;
}

void validate(const dbag_synthetic_options& o) {
  if (o.cameras < 1 || o.points < 1 || (o.num_observations <= 0 && o.obs_per_point < 1))
    throw Error(DBAG_INVALID_ARGUMENT, "synthetic counts must be positive");
  const std::int64_t qmax =
      o.num_observations > 0 ? (o.num_observations + o.points - 1) / o.points : std::int64_t(o.obs_per_point);
  if (o.num_observations > 0 && o.num_observations < o.points)
    throw Error(DBAG_INVALID_ARGUMENT, "count-exact mode needs at least one observation per point");
  if (qmax > o.cameras)
    throw Error(DBAG_INVALID_ARGUMENT,
                "obs-per-point " + std::to_string(qmax) + " exceeds camera count " + std::to_string(o.cameras));
}

inline std::int32_t q_of(const dbag_synthetic_options& o, std::int32_t p) {
  if (o.num_observations <= 0) return o.obs_per_point;
  const std::int64_t base = o.num_observations / o.points, extra = o.num_observations % o.points;
  return static_cast<std::int32_t>(base + (p < extra ? 1 : 0));
}

}  // namespace

std::int64_t synthetic_count(const dbag_synthetic_options& o) {
  validate(o);
  return o.num_observations > 0 ? o.num_observations : std::int64_t(o.points) * o.obs_per_point;
}

void generate_synthetic(const dbag_synthetic_options& o, double* cams, double* pts, std::int32_t* cam_id,
                        std::int32_t* pt_id, double* pix_x, double* pix_y) {
  validate(o);
  const std::int32_t m = o.cameras;
  Uniform rng(o.seed);
  std::vector<V3> centers(static_cast<std::size_t>(m));
  constexpr double kPi = 3.14159265358979323846;
  for (std::int32_t i = 0; i < m; ++i) {
    const double angle = 2.0 * kPi * static_cast<double>(i) / static_cast<double>(m);
    const V3 center{o.circle_radius * std::cos(angle), o.circle_radius * std::sin(angle), 0.0};
    centers[static_cast<std::size_t>(i)] = center;
    // look_at_origin (dba/synthetic.hpp:52-64)
    const V3 cz = normalized(center);
    const V3 right = normalized(cross(V3{0, 0, 1}, cz));
    const V3 up = cross(cz, right);
    const double rot[3][3] = {{right.x, right.y, right.z}, {up.x, up.y, up.z}, {cz.x, cz.y, cz.z}};
    double* cam = cams + static_cast<std::size_t>(i) * 9;
    angle_axis_from_matrix(rot, cam);
    const double cc[3] = {center.x, center.y, center.z};
    for (int r = 0; r < 3; ++r) cam[3 + r] = -((rot[r][0] * cc[0] + rot[r][1] * cc[1]) + rot[r][2] * cc[2]);
    for (int j = 0; j < 3; ++j) cam[j] += rng.range(0.0, o.pose_noise);
    for (int j = 0; j < 3; ++j) cam[3 + j] += rng.range(0.0, o.pose_noise);
    cam[6] = o.base_focal + rng.range(0.0, o.intrinsic_noise);
    cam[7] = rng.range(0.0, o.intrinsic_noise);
    cam[8] = rng.range(0.0, o.intrinsic_noise);
  }
  std::vector<V3> truth(static_cast<std::size_t>(o.points));
  for (std::int32_t i = 0; i < o.points; ++i) {
    V3 p;
    p.x = rng.range(-0.1, 0.1);
    p.y = rng.range(-0.1, 0.1);
    p.z = rng.range(-0.03, 0.03);
    truth[static_cast<std::size_t>(i)] = p;
    double* s = pts + static_cast<std::size_t>(i) * 3;
    s[0] = p.x + rng.range(-o.point_noise, o.point_noise);
    s[1] = p.y + rng.range(-o.point_noise, o.point_noise);
    s[2] = p.z;
  }
  auto dist2 = [&](std::int32_t c, const V3& p) {
    const V3& ce = centers[static_cast<std::size_t>(c)];
    const double dx = ce.x - p.x, dy = ce.y - p.y, dz = ce.z - p.z;
    return (dx * dx + dy * dy) + dz * dz;
  };
  std::vector<std::int32_t> order;
  std::vector<double> d2;
  std::int64_t e = 0;
  for (std::int32_t p = 0; p < o.points; ++p) {
    const V3& X = truth[static_cast<std::size_t>(p)];
    const std::int32_t q = q_of(o, p);
    const std::int32_t half = q + 4;
    order.clear();
    if (o.exhaustive_search || 2 * half + 1 >= m) {
      order.resize(static_cast<std::size_t>(m));
      std::iota(order.begin(), order.end(), 0);
    } else {
      double phi = std::atan2(X.y, X.x);
      if (phi < 0) phi += 2.0 * kPi;
      const std::int64_t i0 = std::llround(phi * m / (2.0 * kPi));
      for (std::int32_t k = -half; k <= half; ++k) order.push_back(static_cast<std::int32_t>(((i0 + k) % m + m) % m));
    }
    d2.resize(order.size());
    auto less = [&](std::int32_t a, std::int32_t b) {
      const double da = dist2(a, X), db = dist2(b, X);
      return da != db ? da < db : a < b;
    };
    std::nth_element(order.begin(), order.begin() + (q - 1), order.end(), less);
    std::sort(order.begin(), order.begin() + q);
    for (std::int32_t k = 0; k < q; ++k, ++e) {
      const std::int32_t c = order[static_cast<std::size_t>(k)];
      double px[2];
      if (!project(cams + static_cast<std::size_t>(c) * 9, X, px)) throw degenerate_depth(e);
      cam_id[e] = c;
      pt_id[e] = p;
      pix_x[e] = px[0];
      pix_y[e] = px[1];
    }
  }
  if (o.pixel_noise > 0) {
    std::mt19937_64 noise(o.seed);
    const double amp = 2.0 * o.pixel_noise;
    for (std::int64_t i = 0; i < e; ++i) {
      const double u = static_cast<double>(noise() >> 11) * 0x1.0p-53;
      const double v = static_cast<double>(noise() >> 11) * 0x1.0p-53;
      pix_x[i] += (u - 0.5) * amp;
      pix_y[i] += (v - 0.5) * amp;
    }
  }
}

}  // namespace dbag
