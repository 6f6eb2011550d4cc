// mprk drop-in (B200): stability-function analysis helpers
// (/root/reference/proj/include/mprk/stability.hpp:10-41).  Off the B200 hot
// path: provided host-only so that reference callers that also
// use them (e.g. the reference's acceptance gate) still compile against the
// drop-in.  R(z) = 1 + z b^T (I - zA)^{-1} e; A = A_high + A_eps is lower
// triangular for every tableau validate() accepts, so (I - zA) y = e is a
// forward substitution, carried out in extended precision.
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

inline std::complex<double> stability_function(const ButcherTableau& t, std::complex<double> z) {
  using cl = std::complex<long double>;
  const int q = t.q;
  const cl zl(z.real(), z.imag());
  long double scale = 1.0L;
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) scale = std::max(scale, std::abs(zl * (long double)(t.a_high[i][j] + t.a_eps[i][j])));
  std::vector<cl> y(q);
  for (int i = 0; i < q; ++i) {
    cl rhs(1.0L, 0.0L);
    for (int j = 0; j < i; ++j) rhs += zl * (long double)(t.a_high[i][j] + t.a_eps[i][j]) * y[j];
    const cl d = cl(1.0L, 0.0L) - zl * (long double)(t.a_high[i][i] + t.a_eps[i][i]);
    if (std::abs(d) <= scale * q * std::numeric_limits<double>::epsilon())
      throw SingularSystem("stability_function: I - zA is singular");
    y[i] = rhs / d;
  }
  cl acc(0.0L, 0.0L);
  for (int i = 0; i < q; ++i) acc += (long double)t.b[i] * y[i];
  const cl r = cl(1.0L, 0.0L) + zl * acc;
  return {(double)r.real(), (double)r.imag()};
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
      } catch (const SingularSystem&) {
        v = std::numeric_limits<double>::infinity();
      }
      g.values[(std::size_t)ix * ny + iy] = v;
      g.stable[(std::size_t)ix * ny + iy] = v <= 1.0;
    }
  return g;
}

}  // namespace mprk
