// Host-side problem setup: grids, forcing, closed-form spectral factors,
// Butcher tableaus.  Computed on the CPU once per Stepper with the same
// libm calls and expression order as the reference, then uploaded.
#pragma once

#include <complex>
#include <string>
#include <vector>

namespace mprkb {

enum class Equation { Heat = 0, Advection = 1, AdvectionDiffusion = 2 };

struct Problem {
  Equation eq = Equation::Heat;
  int n = 0;
  double h = 0.0;
  double gamma_k = 0.0;   // stencil scale of K (operators.cpp:37, 52)
  double gamma_d = 0.0;   // diffusion scale (advection-diffusion extension)
  int k0 = 0, nz = 0;     // this rank's k-slab [k0, k0 + nz) (the whole grid: 0, n)
  std::vector<double> u0;       // local slab
  std::vector<double> forcing;  // local slab; empty unless heat
  size_t size() const { return (size_t)n * n * nz; }
};

// make_problem (operators.cpp:29-65).  nu: diffusion coefficient of the
// advection-diffusion extension (K_d = nu/h^2 * periodic Laplacian).  k0/nz
// restrict u0 and forcing to one k-slab of a split grid (nz = 0: all of it);
// every value is the one the undivided grid holds at that point.
Problem make_problem(Equation eq, int n, double nu = 0.0, int k0 = 0, int nz = 0);
// heat_exact (operators.cpp:67-75)
std::vector<double> heat_exact(const Problem& p, double t);

// spectral_dirichlet (spectral.cpp:11-29): q, q_inv (n*n row-major), lambda
void spectral_dirichlet(int n, double sigma, double gamma, std::vector<double>& q,
                        std::vector<double>& q_inv, std::vector<double>& lambda);
// spectral_periodic (spectral.cpp:31-51), plus an optional periodic-Laplacian
// term gamma2*(2 - 2cos(2 pi k/n)) in lambda for advection-diffusion.
void spectral_periodic(int n, double sigma, double gamma, std::vector<std::complex<double>>& q,
                       std::vector<std::complex<double>>& q_inv,
                       std::vector<std::complex<double>>& lambda, double gamma2 = 0.0);

struct Tableau {
  std::string name;
  int q = 0;
  std::vector<double> a_high, a_eps, b, c;  // q*q row-major, q, q
  double ah(int i, int j) const { return a_high[(size_t)i * q + j]; }
  double ae(int i, int j) const { return a_eps[(size_t)i * q + j]; }
};
// builtin_tableau / midpoint_corrected (tableau.cpp:52-144)
Tableau builtin_tableau(const std::string& name);

}  // namespace mprkb
