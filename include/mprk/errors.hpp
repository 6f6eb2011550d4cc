// mprk drop-in (B200): the reference's exception hierarchy
// (/root/reference/proj/include/mprk/errors.hpp:9-58).  Every C-ABI status
// code of libmprk_b200 maps onto exactly one of these (include/mprk_b200.h).
#pragma once

#include <stdexcept>
#include <string>

namespace mprk {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LengthMismatch : Error {  // MPRKB_LENGTH_MISMATCH
  using Error::Error;
};
struct DimensionTooSmall : Error {  // MPRKB_DIMENSION_TOO_SMALL
  using Error::Error;
};
struct SingularSystem : Error {  // MPRKB_SINGULAR_SYSTEM
  using Error::Error;
};
struct PoleAtTwo : Error {  // MPRKB_POLE_AT_TWO
  using Error::Error;
};
struct OverflowToInfinity : Error {  // MPRKB_OVERFLOW_TO_INFINITY
  using Error::Error;
};
struct ZeroEigenvalueSum : Error {  // MPRKB_ZERO_EIGENVALUE_SUM
  using Error::Error;
};
struct WrongEquation : Error {  // MPRKB_WRONG_EQUATION
  using Error::Error;
};
struct NonFiniteState : Error {  // MPRKB_NONFINITE_STATE
  using Error::Error;
};
struct ConvergenceFailure : Error {
  using Error::Error;
};

}  // namespace mprk
