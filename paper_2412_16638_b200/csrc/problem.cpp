#include "problem.hpp"

#include <cmath>
#include <cstdlib>
#include <numbers>

#include "types.hpp"

namespace mprkb {

Problem make_problem(Equation eq, int n, double nu, int k0, int nz) {
  const bool heat = eq == Equation::Heat;
  if (n < (heat ? 2 : 3)) MPRKB_THROW(3, "make_problem: grid too small for the requested equation");
  if (nz <= 0) nz = n;
  if (k0 < 0 || k0 + nz > n) MPRKB_THROW(10, "make_problem: k-slab outside the grid");
  Problem p;
  p.eq = eq;
  p.n = n;
  p.k0 = k0;
  p.nz = nz;
  const size_t m = (size_t)n * n * nz;
  const double pi = std::numbers::pi;
  if (heat) {
    // nodes at i*h, h = 1/(n-1); boundary nodes are unknowns with zero ghosts
    p.h = 1.0 / (n - 1);
    p.gamma_k = -1.0 / (p.h * p.h);
    p.u0.assign(m, 0.0);
    p.forcing.resize(m);
    for (int k = k0; k < k0 + nz; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i)
          p.forcing[i + (size_t)j * n + (size_t)(k - k0) * n * n] =
              std::sin(pi * i * p.h) * std::sin(pi * j * p.h) * std::sin(pi * k * p.h);
  } else {
    // periodic unit cube, h = 1/n, Gaussian pulse
    p.h = 1.0 / n;
    p.gamma_k = -1.0 / (2.0 * p.h);
    if (eq == Equation::AdvectionDiffusion) p.gamma_d = -nu / (p.h * p.h);
    p.u0.resize(m);
    for (int k = k0; k < k0 + nz; ++k)
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
          const double dx = i * p.h - 0.5, dy = j * p.h - 0.5, dz = k * p.h - 0.5;
          p.u0[i + (size_t)j * n + (size_t)(k - k0) * n * n] = std::exp(-100.0 * (dx * dx + dy * dy + dz * dz));
        }
  }
  return p;
}

std::vector<double> heat_exact(const Problem& p, double t) {
  if (p.eq != Equation::Heat) MPRKB_THROW(8, "heat_exact: analytic solution exists for the heat problem only");
  const double pi2 = std::numbers::pi * std::numbers::pi;
  const double amp = (1.0 - std::exp(-3.0 * pi2 * t)) / (3.0 * pi2);
  std::vector<double> u(p.forcing.size());
  for (size_t i = 0; i < u.size(); ++i) u[i] = amp * p.forcing[i];
  return u;
}

void spectral_dirichlet(int n, double sigma, double gamma, std::vector<double>& q, std::vector<double>& q_inv,
                        std::vector<double>& lambda) {
  if (n < 2) MPRKB_THROW(3, "spectral_dirichlet: n must be at least 2");
  q.resize((size_t)n * n);
  lambda.resize(n);
  const double norm = std::sqrt(2.0 / (n + 1));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      q[(size_t)j * n + k] = norm * std::sin((j + 1) * (k + 1) * std::numbers::pi / (n + 1));
  q_inv = q;  // orthonormal and symmetric
  for (int k = 0; k < n; ++k)
    lambda[k] = sigma + gamma * (2.0 - 2.0 * std::cos((k + 1) * std::numbers::pi / (n + 1)));
}

void spectral_periodic(int n, double sigma, double gamma, std::vector<std::complex<double>>& q,
                       std::vector<std::complex<double>>& q_inv, std::vector<std::complex<double>>& lambda,
                       double gamma2) {
  if (n < 3) MPRKB_THROW(3, "spectral_periodic: n must be at least 3");
  q.resize((size_t)n * n);
  q_inv.resize(q.size());
  lambda.resize(n);
  const double norm = 1.0 / std::sqrt(static_cast<double>(n));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double angle = 2.0 * std::numbers::pi * ((static_cast<long long>(j) * k) % n) / n;
      q[(size_t)j * n + k] = std::polar(norm, angle);
      q_inv[(size_t)k * n + j] = std::polar(norm, -angle);
    }
  for (int k = 0; k < n; ++k) {
    lambda[k] = std::complex<double>(sigma, 0.0) +
                gamma * std::complex<double>(0.0, 2.0 * std::sin(2.0 * std::numbers::pi * k / n));
    if (gamma2 != 0.0)
      lambda[k] += std::complex<double>(gamma2 * (2.0 - 2.0 * std::cos(2.0 * std::numbers::pi * k / n)), 0.0);
  }
}

namespace {

double coeff(const char* text) {
  char* end = nullptr;
  const double v = std::strtod(text, &end);
  if (end == nullptr || *end != '\0') MPRKB_THROW(1, std::string("bad coefficient literal: ") + text);
  return v;
}

Tableau make(const std::string& name, int q) {
  Tableau t;
  t.name = name;
  t.q = q;
  t.a_high.assign((size_t)q * q, 0.0);
  t.a_eps.assign((size_t)q * q, 0.0);
  t.b.assign(q, 0.0);
  return t;
}

void finish(Tableau& t) {
  t.c.assign(t.q, 0.0);
  for (int i = 0; i < t.q; ++i) {
    double acc = 0.0;
    for (int j = 0; j < t.q; ++j) acc += t.ah(i, j) + t.ae(i, j);
    t.c[i] = acc;
  }
}

}  // namespace

// Published 15-digit coefficients (Grant, arXiv 2412.16638), parsed once by
// strtod (correctly rounded), with the reference's correction of the 4s3pB
// a_42 high part (tableau.cpp:78-85).
Tableau builtin_tableau(const std::string& name) {
  if (name.rfind("midpoint", 0) == 0) {
    const int p = std::atoi(name.c_str() + 8);
    if (p < 0 || name.size() == 8) MPRKB_THROW(1, "midpoint_corrected: corrector count must be nonnegative");
    Tableau t = make(name, p + 1);
    t.a_eps[0] = 0.5;
    for (int i = 1; i <= p; ++i) t.a_high[(size_t)i * t.q + i - 1] = 0.5;
    t.b[p] = 1.0;
    finish(t);
    return t;
  }
  Tableau t = make(name, 4);
  auto AH = [&](int i, int j, const char* s) { t.a_high[(size_t)i * 4 + j] = coeff(s); };
  auto AE = [&](int i, int j, const char* s) { t.a_eps[(size_t)i * 4 + j] = coeff(s); };
  if (name == "4s3pA") {
    AE(0, 0, "0.788675134594813");
    AH(1, 0, "0.211324865405187");
    AE(2, 0, "0.051944240459852");
    AH(2, 0, "0.709495523817170");
    AH(2, 1, "-0.86531425061942");
    AE(2, 2, "0.788675134594813");
    AH(3, 0, "0.705123240545107");
    AH(3, 1, "0.943370088535775");
    AH(3, 2, "-0.859818194486069");
    t.b = {0.0, 0.5, 0.0, 0.5};
  } else if (name == "4s3pB") {
    for (int i = 0; i < 4; ++i) t.a_eps[(size_t)i * 4 + i] = 0.5;
    AE(1, 0, "-2.376349376129689");
    AH(1, 0, "2.543016042796356");
    AE(2, 0, "-2.951484396921318");
    AH(2, 0, "2.451484396921318");
    AE(2, 1, "0.475891038758779");
    AH(2, 1, "0.024108961241221");
    AE(3, 0, "-0.573861819468268");
    AH(3, 0, "2.073861819468268");
    AE(3, 1, "0.051944240459852");
    AH(3, 1, "-1.551944240459852");  // corrected: a42 sums to -3/2
    AE(3, 2, "-1.211868223075524");
    AH(3, 2, "1.711868223075524");
    t.b = {1.5, -1.5, 0.5, 0.5};
  } else if (name == "4s3pC") {
    AE(0, 0, "0.511243008730995");
    AE(1, 0, "-1.999347282862640");
    AH(1, 0, "-0.050470366527530");
    AE(1, 1, "1.957161067302390");
    AE(2, 0, "0.443312893511937");
    AH(2, 0, "0.368613367355336");
    AE(2, 1, "-0.573131033672219");
    AH(2, 1, "0.273504374252976");
    AE(2, 2, "0.128283796414019");
    AE(3, 0, "-2");
    AH(3, 0, "1.803794668975043");
    AE(3, 1, "-0.160330320741428");
    AH(3, 1, "0.097485042980759");
    AE(3, 2, "0.579597314161362");
    AH(3, 2, "-1.895660952342050");
    AE(3, 3, "1.484688928981990");
    t.b = {coeff("0.002837446974069"), coeff("0.336264433650450"), coeff("0.806376720267787"),
           coeff("-0.145478600892306")};
  } else {
    MPRKB_THROW(1, "unknown method name: " + name);
  }
  finish(t);
  return t;
}

}  // namespace mprkb
