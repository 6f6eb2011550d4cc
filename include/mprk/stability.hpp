// mprk drop-in (B200): stability-function analysis helpers
// (/root/reference/proj/include/mprk/stability.hpp:10-41).  Off the B200 hot
// path: provided host-only so that reference callers that also
// use them (e.g. the reference's acceptance gate) still compile against the
// drop-in.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <vector>

#include "mprk/errors.hpp"
#include "mprk/precision.hpp"
#include "mprk/tableau.hpp"

namespace mprk {

enum class FloatFormat { Binary16, Binary32 };

// R(z) = 1 + z b^T w with (I - zA) w = e solved by Gaussian elimination with
// partial pivoting in extended precision (the reference's dense solve, so the
// |R| = 1 boundary falls on the same lattice cells).
inline std::complex<double> stability_function(const ButcherTableau& t, std::complex<double> z) {
  using cl = std::complex<long double>;
  const int q = t.q;
  const cl zl(z.real(), z.imag());
  std::vector<cl> M((std::size_t)q * q), w(q, cl(1.0L));
  for (int r = 0; r < q; ++r)
    for (int c = 0; c < q; ++c)
      M[(std::size_t)r * q + c] =
          (r == c ? cl(1.0L) : cl()) - zl * ((long double)t.a_high[r][c] + (long double)t.a_eps[r][c]);
  long double big = 0.0L;
  for (const cl& v : M) big = std::max(big, std::abs(v));
  const long double tiny = big * q * std::numeric_limits<double>::epsilon();
  auto at = [&](int r, int c) -> cl& { return M[(std::size_t)r * q + c]; };
  for (int k = 0; k < q; ++k) {
    int p = k;
    for (int r = k + 1; r < q; ++r)
      if (std::abs(at(r, k)) > std::abs(at(p, k))) p = r;
    if (std::abs(at(p, k)) <= tiny) throw SingularSystem("stability_function: I - zA is singular");
    if (p != k) {
      for (int c = 0; c < q; ++c) std::swap(at(k, c), at(p, c));
      std::swap(w[k], w[p]);
    }
    for (int r = k + 1; r < q; ++r) {
      const cl f = at(r, k) / at(k, k);
      if (f == cl()) continue;
      for (int c = k; c < q; ++c) at(r, c) -= f * at(k, c);
      w[r] -= f * w[k];
    }
  }
  for (int r = q - 1; r >= 0; --r) {
    cl s = w[r];
    for (int c = r + 1; c < q; ++c) s -= at(r, c) * w[c];
    w[r] = s / at(r, r);
  }
  cl acc;
  for (int i = 0; i < q; ++i) acc += (long double)t.b[i] * w[i];
  const cl R = cl(1.0L) + zl * acc;
  return {(double)R.real(), (double)R.imag()};
}

inline std::complex<double> corrected_midpoint_reference(std::complex<double> z) {
  if (z == std::complex<double>(2.0, 0.0)) throw PoleAtTwo("corrected_midpoint_reference: pole at z = 2");
  return (z + 2.0) / (2.0 - z);
}

inline ButcherTableau truncate_eps(const ButcherTableau& t, FloatFormat fmt) {
  ButcherTableau o = t;
  for (auto& row : o.a_eps)
    for (double& v : row) v = fmt == FloatFormat::Binary16 ? round_binary16(v) : round_binary32(v);
  o.c = b200::row_sums(o.a_high, o.a_eps);
  o.name += fmt == FloatFormat::Binary16 ? "+b16" : "+b32";
  return o;
}

struct StabilityGrid {
  double re_min = 0, re_max = 0, im_min = 0, im_max = 0;
  int nx = 0, ny = 0;
  std::vector<double> values;        // |R|, index ix*ny + iy; +inf at poles
  std::vector<std::uint8_t> stable;  // values <= 1
  double re_at(int ix) const { return re_min + (re_max - re_min) * ix / (nx - 1); }
  double im_at(int iy) const { return im_min + (im_max - im_min) * iy / (ny - 1); }
  long stable_count() const {
    long c = 0;
    for (std::uint8_t s : stable) c += s;
    return c;
  }
};

inline StabilityGrid region_scan(const ButcherTableau& t, double re_min, double re_max, double im_min, double im_max,
                                 int nx, int ny) {
  if (nx < 2 || ny < 2 || (double)nx * ny > 1e7) throw Error("region_scan: lattice must be 2..1e7 points per side");
  StabilityGrid g{re_min, re_max, im_min, im_max, nx, ny, {}, {}};
  g.values.resize((std::size_t)nx * ny);
  g.stable.resize(g.values.size());
  for (int ix = 0; ix < nx; ++ix)
    for (int iy = 0; iy < ny; ++iy) {
      double v;
      try {
        v = std::abs(stability_function(t, {g.re_at(ix), g.im_at(iy)}));
        if (std::isnan(v)) v = std::numeric_limits<double>::infinity();
      } catch (const SingularSystem&) {
        v = std::numeric_limits<double>::infinity();
      }
      g.values[(std::size_t)ix * ny + iy] = v;
      g.stable[(std::size_t)ix * ny + iy] = v <= 1.0;
    }
  return g;
}

}  // namespace mprk
