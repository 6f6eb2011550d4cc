// mprk drop-in (B200): precision tags and host-side narrowing helpers with the
// reference's semantics (/root/reference/proj/include/mprk/precision.hpp:12-202).
// These run on the host at the API boundary (setup / conversion of caller
// vectors); the device path narrows inside its fused kernels.
#pragma once

#include <cfenv>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "mprk/errors.hpp"

namespace mprk {

enum class Precision { F32, F64 };
enum class ScalarKind { Real, Complex };

inline const char* to_string(Precision p) { return p == Precision::F32 ? "f32" : "f64"; }

// Smallest double that rounds (RNE) to binary32 infinity: 2^128 - 2^103.
inline constexpr double kBinary32OverflowThreshold = 0x1.ffffffp+127;

inline double round_binary32(double x) {
  if (std::isnan(x)) return x;
  if (std::fabs(x) >= kBinary32OverflowThreshold) return x > 0 ? INFINITY : -INFINITY;
  return static_cast<double>(static_cast<float>(x));
}

// binary16 rounding straight from binary64 (no double rounding through
// binary32): the value is snapped to the binary16 grid of its binade with a
// ties-to-even rint (exact, since the scaling is by a power of two), then
// encoded.
inline std::uint16_t to_binary16_bits(double x) {
  const std::uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  if (std::isnan(x)) return static_cast<std::uint16_t>(sign | 0x7E00);
  const double a = std::fabs(x);
  if (std::isinf(a)) return static_cast<std::uint16_t>(sign | 0x7C00);
  if (a < 0x1p-1022) return sign;  // zero and binary64 subnormals
  int e2 = 0;
  std::frexp(a, &e2);                   // a = f 2^e2, f in [0.5, 1)
  const int e = std::max(e2 - 1, -14);  // binade exponent (subnormals share -14)
  const double ulp = std::ldexp(1.0, e - 10);
  const int saved = std::fegetround();
  std::fesetround(FE_TONEAREST);
  const double r = std::nearbyint(a / ulp) * ulp;
  std::fesetround(saved);
  if (r > 65504.0) return static_cast<std::uint16_t>(sign | 0x7C00);
  if (r == 0.0) return sign;
  int re = 0;
  std::frexp(r, &re);
  const int ue = re - 1;  // unbiased exponent of the rounded value
  if (ue < -14) {         // subnormal: units of 2^-24
    return static_cast<std::uint16_t>(sign | static_cast<std::uint16_t>(std::ldexp(r, 24)));
  }
  const unsigned mant = static_cast<unsigned>(std::ldexp(r, 10 - ue)) - 1024u;
  return static_cast<std::uint16_t>(sign | ((ue + 15) << 10) | mant);
}

inline double from_binary16_bits(std::uint16_t h) {
  const bool neg = (h & 0x8000) != 0;
  const int ef = (h >> 10) & 0x1F;
  const unsigned mant = h & 0x3FFu;
  double v;
  if (ef == 0x1F)
    v = mant ? std::numeric_limits<double>::quiet_NaN() : std::numeric_limits<double>::infinity();
  else if (ef == 0)
    v = std::ldexp(static_cast<double>(mant), -24);
  else
    v = std::ldexp(static_cast<double>(mant | 0x400u), ef - 25);
  return neg ? -v : v;
}

inline double round_binary16(double x) { return from_binary16_bits(to_binary16_bits(x)); }

inline float downcast_scalar(double x) {
  if (std::fabs(x) >= kBinary32OverflowThreshold)  // (false for NaN)
    throw OverflowToInfinity("downcast: |" + std::to_string(x) + "| exceeds the binary32 range");
  return static_cast<float>(x);
}
inline std::complex<float> downcast_scalar(std::complex<double> z) {
  return {downcast_scalar(z.real()), downcast_scalar(z.imag())};
}

template <typename D>
auto downcast(const std::vector<D>& v) {
  using N = decltype(downcast_scalar(D{}));
  std::vector<N> out;
  out.reserve(v.size());
  for (const D& x : v) out.push_back(downcast_scalar(x));
  return out;
}

inline std::vector<double> upcast(const std::vector<float>& v) { return {v.begin(), v.end()}; }
inline std::vector<std::complex<double>> upcast(const std::vector<std::complex<float>>& v) {
  std::vector<std::complex<double>> out;
  out.reserve(v.size());
  for (const auto& z : v) out.emplace_back(z.real(), z.imag());
  return out;
}

// A std::vector tagged with its precision and scalar kind.
class PrecVector {
 public:
  using Storage = std::variant<std::vector<float>, std::vector<double>, std::vector<std::complex<float>>,
                               std::vector<std::complex<double>>>;
  PrecVector() : v_(std::vector<double>{}) {}
  explicit PrecVector(std::vector<float> v) : v_(std::move(v)) {}
  explicit PrecVector(std::vector<double> v) : v_(std::move(v)) {}
  explicit PrecVector(std::vector<std::complex<float>> v) : v_(std::move(v)) {}
  explicit PrecVector(std::vector<std::complex<double>> v) : v_(std::move(v)) {}

  // variant order: f32, f64, c32, c64
  Precision precision() const { return v_.index() % 2 == 0 ? Precision::F32 : Precision::F64; }
  ScalarKind kind() const { return v_.index() >= 2 ? ScalarKind::Complex : ScalarKind::Real; }
  std::size_t size() const {
    return std::visit([](const auto& v) { return v.size(); }, v_);
  }
  bool all_finite() const {
    return std::visit(
        [](const auto& v) {
          for (const auto& x : v)
            if (!std::isfinite(std::real(x)) || !std::isfinite(std::imag(x))) return false;
          return true;
        },
        v_);
  }
  PrecVector to(Precision target) const {
    if (target == precision()) return *this;
    return std::visit(
        [](const auto& v) -> PrecVector {
          using S = typename std::decay_t<decltype(v)>::value_type;
          if constexpr (std::is_same_v<S, double> || std::is_same_v<S, std::complex<double>>)
            return PrecVector(downcast(v));
          else
            return PrecVector(upcast(v));
        },
        v_);
  }
  template <typename T>
  const std::vector<T>& as() const {
    const auto* p = std::get_if<std::vector<T>>(&v_);
    if (!p) throw Error("PrecVector: payload does not hold the requested scalar type");
    return *p;
  }
  const Storage& storage() const { return v_; }

 private:
  Storage v_;
};

}  // namespace mprk
