// mprk drop-in (B200): closed-form 1D spectral factors
// (/root/reference/proj/include/mprk/spectral.hpp:8-37), computed by
// libmprk_b200's host setup code (glibc sin/cos in the reference's order).
#pragma once

#include <complex>
#include <vector>

#include "mprk/b200.hpp"

namespace mprk {

enum class Stencil1D {
  DirichletLaplace1D,    // tridiag(-1, 2, -1), zero ghosts
  PeriodicCentralDiff1D  // x_{i+1} - x_{i-1}, periodic
};

template <typename T>
struct SpectralFactor {
  int n = 0;
  std::vector<T> q;
  std::vector<T> q_inv;
  std::vector<T> lambda;
};

namespace b200 {
template <typename T>
SpectralFactor<T> spectral(int periodic, int n, double sigma, double gamma) {
  SpectralFactor<T> f;
  f.n = n;
  const std::size_t nn = n > 0 ? static_cast<std::size_t>(n) * n : 0;
  f.q.resize(nn);
  f.q_inv.resize(nn);
  f.lambda.resize(n > 0 ? n : 0);
  check(mprkb_spectral(periodic, n, sigma, gamma, f.q.data(), f.q_inv.data(), f.lambda.data()));
  return f;
}
template <typename D>
auto narrow_factor(const SpectralFactor<D>& f) {
  using N = std::conditional_t<std::is_same_v<D, double>, float, std::complex<float>>;
  SpectralFactor<N> o;
  o.n = f.n;
  auto cast = [](const std::vector<D>& v) {
    std::vector<N> r;
    r.reserve(v.size());
    for (const D& x : v) r.push_back(static_cast<N>(x));
    return r;
  };
  o.q = cast(f.q);
  o.q_inv = cast(f.q_inv);
  o.lambda = cast(f.lambda);
  return o;
}
}  // namespace b200

inline SpectralFactor<double> spectral_dirichlet(int n, double sigma, double gamma) {
  return b200::spectral<double>(0, n, sigma, gamma);
}
inline SpectralFactor<std::complex<double>> spectral_periodic(int n, double sigma, double gamma) {
  return b200::spectral<std::complex<double>>(1, n, sigma, gamma);
}
inline SpectralFactor<float> downcast_factor(const SpectralFactor<double>& f) { return b200::narrow_factor(f); }
inline SpectralFactor<std::complex<float>> downcast_factor(const SpectralFactor<std::complex<double>>& f) {
  return b200::narrow_factor(f);
}

}  // namespace mprk
