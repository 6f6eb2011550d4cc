// Drop-in example: the reference's own usage pattern (tests/acceptance.cpp
// run_case, stepper.cpp integrate) written against mprk_b200.hpp.  Prints
// "<mean_iterations> <error_max> <error_l2>" for heat n^3, 4s3pB, fp32
// implicit, tau = 1/40, t_end = 0.1 (numerics from argv[2]: fast | parity).
#include <cstdio>
#include <cstdlib>
#include <string>

#include "mprk_b200.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 16;
  const bool parity = argc > 2 && std::string(argv[2]) == "parity";
  try {
    mprk_b200::IntegrationConfig cfg;
    cfg.equation = mprk_b200::Equation::Heat;
    cfg.n = n;
    cfg.tableau = mprk_b200::builtin_tableau("4s3pB");
    cfg.tau = 1.0 / 40.0;
    cfg.t_end = 0.1;
    cfg.tol = 1e-4;
    cfg.implicit = mprk_b200::Precision::F32;
    cfg.parity = parity;
    const auto r = mprk_b200::integrate(cfg);
    std::printf("%.17g %.17g %.17g\n", r.mean_iterations, *r.error_max, *r.error_l2);

    // Stepper form (stepper.hpp:53-65)
    mprk_b200::Stepper st(cfg);
    std::vector<double> u = st.initial_state();
    mprk_b200::StepTrace trace;
    st.step(u, trace);
    std::printf("solves %zu iterations %d\n", trace.solves.size(), trace.solves.at(0).iterations);
  } catch (const mprk_b200::DeviceError& e) {
    std::printf("device error: %s\n", e.what());
    return 3;
  } catch (const mprk_b200::Error& e) {
    std::printf("mprk error: %s\n", e.what());
    return 2;
  }
  return 0;
}
