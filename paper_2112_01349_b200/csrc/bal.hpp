// bal.hpp — BAL text ingestion and emission.
//
// Same format, validation, error messages and line numbers as the
// reference's parse_bal / serialize_bal (dba/bal_io.hpp:19-209); the input
// is scanned in memory instead of one istream::get per character:
//   header           num_cameras num_points num_observations
//   observations     cam_idx pt_idx px py                  (x num_observations)
//   cameras          rotation[3] translation[3] f k1 k2    (x num_cameras)
//   points           X Y Z                                  (x num_points)
// Integers follow strtoll (whole token, no overflow), reals strtod (whole
// token, finite); std::from_chars takes the common decimal forms (same
// correctly rounded value as strtod) and strtod the rest ('+', hex, ...).
// Emission prints every real with "%.16e" so that parse -> serialize ->
// parse round-trips to identical values (dba/bal_io.hpp:146-156).
#pragma once

#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <string_view>
#include <vector>

#include "common.hpp"

namespace dbag {

struct BalData {
  std::int32_t m = 0, n = 0;
  std::int64_t N = 0;
  std::vector<double> cameras, points, px, py;  // 9m, 3n, N, N
  std::vector<std::int32_t> cam, pt;            // N
};

// ParseError(msg, line) of dba/errors.hpp:17-26: "line L: msg", L >= 1.
inline Error parse_error(const std::string& msg, std::int64_t line) {
  return Error(DBAG_PARSE, line > 0 ? "line " + std::to_string(line) + ": " + msg : msg, line);
}

class BalScanner {
 public:
  BalScanner(const char* text, std::size_t len) : p_(text), end_(text + len) {}

  // dba/bal_io.hpp:25-39: skip whitespace (counting '\n'), then the token;
  // the newline that ends a token is counted before the next token.
  std::string_view token() {
    while (p_ < end_ && is_space(*p_)) {
      if (*p_ == '\n') ++line_;
      ++p_;
    }
    if (p_ == end_) throw parse_error("unexpected end of input", line_);
    const char* b = p_;
    while (p_ < end_ && !is_space(*p_)) ++p_;
    return std::string_view(b, static_cast<std::size_t>(p_ - b));
  }

  std::int64_t next_int() {  // dba/bal_io.hpp:41-49
    const std::string_view t = token();
    std::int64_t v = 0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec == std::errc() && r.ptr == t.data() + t.size()) return v;
    const std::string s(t);  // '+', leading zeros past int64 range, ...: strtoll decides
    char* e = nullptr;
    errno = 0;
    const long long w = std::strtoll(s.c_str(), &e, 10);
    if (e != s.c_str() + s.size() || errno == ERANGE || s.empty())
      throw parse_error("expected integer, got '" + s + "'", line_);
    return w;
  }

  double next_real() {  // dba/bal_io.hpp:51-61
    const std::string_view t = token();
    double v = 0.0;
    const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (!(r.ec == std::errc() && r.ptr == t.data() + t.size())) {
      const std::string s(t);
      char* e = nullptr;
      errno = 0;
      v = std::strtod(s.c_str(), &e);
      if (e != s.c_str() + s.size() || s.empty()) throw parse_error("expected number, got '" + s + "'", line_);
    }
    if (!std::isfinite(v)) throw parse_error("non-finite value '" + std::string(t) + "'", line_);
    return v;
  }

  std::int64_t line() const { return line_; }

 private:
  static bool is_space(char c) { return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
  const char* p_;
  const char* end_;
  std::int64_t line_ = 1;
};

// parse_bal (dba/bal_io.hpp:78-144): observations are read (and their
// indices validated against the header) before the camera and point blocks.
inline BalData parse_bal_text(const char* text, std::size_t len) {
  BalScanner in(text, len);
  const std::int64_t m = in.next_int(), n = in.next_int(), N = in.next_int();
  if (m < 0 || n < 0 || N < 0) throw parse_error("negative count in header", in.line());
  if (m > INT32_MAX || n > INT32_MAX) throw parse_error("count exceeds int32 ids", in.line());
  BalData d;
  d.m = static_cast<std::int32_t>(m);
  d.n = static_cast<std::int32_t>(n);
  d.N = N;
  d.cam.reserve(static_cast<std::size_t>(N));
  d.pt.reserve(static_cast<std::size_t>(N));
  d.px.reserve(static_cast<std::size_t>(N));
  d.py.reserve(static_cast<std::size_t>(N));
  for (std::int64_t i = 0; i < N; ++i) {
    const std::int64_t c = in.next_int();
    const std::int64_t p = in.next_int();
    if (c < 0 || c >= m)
      throw parse_error("camera index " + std::to_string(c) + " out of range [0, " + std::to_string(m) + ")", in.line());
    if (p < 0 || p >= n)
      throw parse_error("point index " + std::to_string(p) + " out of range [0, " + std::to_string(n) + ")", in.line());
    d.cam.push_back(static_cast<std::int32_t>(c));
    d.pt.push_back(static_cast<std::int32_t>(p));
    d.px.push_back(in.next_real());
    d.py.push_back(in.next_real());
  }
  d.cameras.resize(static_cast<std::size_t>(m) * 9);
  for (double& v : d.cameras) v = in.next_real();
  d.points.resize(static_cast<std::size_t>(n) * 3);
  for (double& v : d.points) v = in.next_real();
  return d;
}

// serialize_bal (dba/bal_io.hpp:158-209): header, observation lines
// "cam pt px py", then one real per line for cameras and points.
template <class S>
std::string format_bal(std::int32_t m, std::int32_t n, std::int64_t N, const S* cameras, const S* points,
                       const std::int32_t* cam, const std::int32_t* pt, const S* px, const S* py) {
  std::string out;
  out.reserve(static_cast<std::size_t>(N) * 56 + (static_cast<std::size_t>(m) * 9 + static_cast<std::size_t>(n) * 3) * 24 + 64);
  char buf[64];
  out += std::to_string(m) + ' ' + std::to_string(n) + ' ' + std::to_string(N) + '\n';
  auto real = [&](S v) {
    const int k = std::snprintf(buf, sizeof(buf), "%.16e", static_cast<double>(v));
    out.append(buf, static_cast<std::size_t>(k));
  };
  for (std::int64_t e = 0; e < N; ++e) {
    out += std::to_string(cam[e]);
    out += ' ';
    out += std::to_string(pt[e]);
    out += ' ';
    real(px[e]);
    out += ' ';
    real(py[e]);
    out += '\n';
  }
  for (std::size_t i = 0; i < static_cast<std::size_t>(m) * 9; ++i) {
    real(cameras[i]);
    out += '\n';
  }
  for (std::size_t i = 0; i < static_cast<std::size_t>(n) * 3; ++i) {
    real(points[i]);
    out += '\n';
  }
  return out;
}

}  // namespace dbag
