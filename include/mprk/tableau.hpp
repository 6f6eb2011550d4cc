// mprk drop-in (B200): split Butcher tableaus
// (/root/reference/proj/include/mprk/tableau.hpp:8-44).  The coefficients come
// from libmprk_b200 (parsed from the same published decimals); validation and
// JSON I/O are host-side.
#pragma once

#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "mprk/b200.hpp"
#include "mprk/errors.hpp"

namespace mprk {

using CoeffMatrix = std::vector<std::vector<double>>;

enum class Method { M4s3pA, M4s3pB, M4s3pC };

struct ButcherTableau {
  std::string name;
  int q = 0;
  std::vector<double> c;
  CoeffMatrix a_high;
  CoeffMatrix a_eps;
  std::vector<double> b;
};

namespace b200 {
inline ButcherTableau library_tableau(const std::string& name) {
  constexpr int cap = 64;
  std::vector<double> ah(cap * cap), ae(cap * cap), b(cap), c(cap);
  int q = 0;
  check(mprkb_builtin_tableau(name.c_str(), cap * cap, &q, ah.data(), ae.data(), b.data(), c.data()));
  ButcherTableau t;
  t.name = name;
  t.q = q;
  t.b.assign(b.begin(), b.begin() + q);
  t.c.assign(c.begin(), c.begin() + q);
  t.a_high.assign(q, std::vector<double>(q));
  t.a_eps.assign(q, std::vector<double>(q));
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j) {
      t.a_high[i][j] = ah[static_cast<std::size_t>(i) * q + j];
      t.a_eps[i][j] = ae[static_cast<std::size_t>(i) * q + j];
    }
  return t;
}
inline std::vector<double> row_sums(const CoeffMatrix& a, const CoeffMatrix& e) {
  std::vector<double> c(a.size(), 0.0);
  for (std::size_t i = 0; i < a.size(); ++i)
    for (std::size_t j = 0; j < a[i].size() && j < e[i].size(); ++j) c[i] += a[i][j] + e[i][j];
  return c;
}
}  // namespace b200

inline const ButcherTableau& builtin_tableau(Method m) {
  static const ButcherTableau tabs[3] = {b200::library_tableau("4s3pA"), b200::library_tableau("4s3pB"),
                                         b200::library_tableau("4s3pC")};
  return tabs[static_cast<int>(m)];
}

inline Method method_from_name(const std::string& name) {
  if (name == "4s3pA") return Method::M4s3pA;
  if (name == "4s3pB") return Method::M4s3pB;
  if (name == "4s3pC") return Method::M4s3pC;
  throw Error("unknown method name: " + name);
}

inline ButcherTableau midpoint_corrected(int p) {
  if (p < 0) throw Error("midpoint_corrected: corrector count must be non-negative");
  return b200::library_tableau("midpoint" + std::to_string(p));
}

// Structural checks (tableau.cpp:146-190): one line per violated invariant.
inline std::vector<std::string> validate(const ButcherTableau& t) {
  std::vector<std::string> bad;
  const int q = t.q;
  auto square = [q](const CoeffMatrix& m) {
    if ((int)m.size() != q) return false;
    for (const auto& r : m)
      if ((int)r.size() != q) return false;
    return true;
  };
  if (q <= 0) bad.push_back("stage count must be positive");
  if (!square(t.a_high) || !square(t.a_eps) || (int)t.b.size() != q || (int)t.c.size() != q) {
    bad.push_back("coefficient blocks must all be q-by-q and q-long");
    return bad;
  }
  const auto c = b200::row_sums(t.a_high, t.a_eps);
  for (int i = 0; i < q; ++i)
    if (std::fabs(c[i] - t.c[i]) > 1e-13)
      bad.push_back("c[" + std::to_string(i) + "] does not match the row sum of A_high + A_eps");
  double w = 0.0;
  for (double x : t.b) w += x;
  if (std::fabs(w - 1.0) > 1e-13) bad.push_back("sum(b) must be 1");
  bool lower = true, diag_eps = true;
  for (int i = 0; i < q; ++i) {
    if (t.a_high[i][i] != 0.0) diag_eps = false;
    for (int j = i + 1; j < q; ++j) lower = lower && t.a_high[i][j] == 0.0 && t.a_eps[i][j] == 0.0;
  }
  if (!lower) bad.push_back("A_high + A_eps must be lower triangular");
  if (!diag_eps) bad.push_back("diagonal (implicit) coefficients must live in A_eps only");
  return bad;
}

// ---- JSON (tableau.cpp:192-233): {"name","q","c","A_high","A_eps","b"} ----
namespace b200 {
struct Json {
  enum Kind { Null, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
};

class JsonReader {
 public:
  explicit JsonReader(const std::string& s) : s_(s) {}
  Json document() {
    Json v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) { throw Error(std::string("tableau JSON does not parse: ") + what); }
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  std::string string_lit() {
    if (!eat('"')) fail("expected a string");
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\' && i_ + 1 < s_.size()) ++i_;
      out += s_[i_++];
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    Json v;
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      v.kind = Json::Obj;
      if (eat('}')) return v;
      do {
        const std::string k = string_lit();
        if (!eat(':')) fail("expected ':'");
        v.obj[k] = value();
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
    } else if (c == '[') {
      ++i_;
      v.kind = Json::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ']'");
    } else if (c == '"') {
      v.kind = Json::Str;
      v.str = string_lit();
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else {
      const char* b = s_.c_str() + i_;
      char* e = nullptr;
      v.num = std::strtod(b, &e);
      if (e == b) fail("unexpected character");
      v.kind = Json::Num;
      i_ += static_cast<std::size_t>(e - b);
    }
    return v;
  }
  const std::string& s_;
  std::size_t i_ = 0;
};

inline const Json& field(const Json& o, const char* k) {
  const auto it = o.obj.find(k);
  if (it == o.obj.end()) throw Error(std::string("tableau JSON has a wrong field: missing ") + k);
  return it->second;
}
inline std::vector<double> numbers(const Json& j, const char* what) {
  if (j.kind != Json::Arr) throw Error(std::string("tableau JSON has a wrong field: ") + what + " is not an array");
  std::vector<double> v;
  for (const Json& e : j.arr) {
    if (e.kind != Json::Num) throw Error(std::string("tableau JSON has a wrong field: ") + what + " holds a non-number");
    v.push_back(e.num);
  }
  return v;
}
inline CoeffMatrix matrix(const Json& j, const char* what) {
  if (j.kind != Json::Arr) throw Error(std::string("tableau JSON has a wrong field: ") + what + " is not an array");
  CoeffMatrix m;
  for (const Json& r : j.arr) m.push_back(numbers(r, what));
  return m;
}
inline void put_num(std::string& out, double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  out += buf;
  if (std::string(buf).find_first_of(".eEn") == std::string::npos) out += ".0";
}
inline void put_vec(std::string& out, const std::vector<double>& v) {
  out += "[";
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) out += ", ";
    put_num(out, v[i]);
  }
  out += "]";
}
inline void put_mat(std::string& out, const CoeffMatrix& m) {
  out += "[";
  for (std::size_t i = 0; i < m.size(); ++i) {
    out += i ? ",\n    " : "\n    ";
    put_vec(out, m[i]);
  }
  out += "\n  ]";
}
}  // namespace b200

inline std::string tableau_to_json(const ButcherTableau& t) {
  std::string s = "{\n  \"name\": \"" + t.name + "\",\n  \"q\": " + std::to_string(t.q) + ",\n  \"c\": ";
  b200::put_vec(s, t.c);
  s += ",\n  \"A_high\": ";
  b200::put_mat(s, t.a_high);
  s += ",\n  \"A_eps\": ";
  b200::put_mat(s, t.a_eps);
  s += ",\n  \"b\": ";
  b200::put_vec(s, t.b);
  s += "\n}";
  return s;
}

inline ButcherTableau tableau_from_json(const std::string& text) {
  const b200::Json j = b200::JsonReader(text).document();
  if (j.kind != b200::Json::Obj) throw Error("tableau JSON does not parse: not an object");
  ButcherTableau t;
  const b200::Json& nm = b200::field(j, "name");
  const b200::Json& q = b200::field(j, "q");
  if (nm.kind != b200::Json::Str || q.kind != b200::Json::Num || q.num != std::floor(q.num))
    throw Error("tableau JSON has a wrong field: name / q");
  t.name = nm.str;
  t.q = static_cast<int>(q.num);
  t.a_high = b200::matrix(b200::field(j, "A_high"), "A_high");
  t.a_eps = b200::matrix(b200::field(j, "A_eps"), "A_eps");
  t.b = b200::numbers(b200::field(j, "b"), "b");
  t.c = j.obj.count("c") ? b200::numbers(j.obj.at("c"), "c") : b200::row_sums(t.a_high, t.a_eps);
  const auto q_ = static_cast<std::size_t>(t.q > 0 ? t.q : 0);
  if (t.q <= 0 || t.b.size() != q_ || t.a_high.size() != q_ || t.a_eps.size() != q_)
    throw Error("tableau JSON dimensions are inconsistent with q");
  for (const auto* m : {&t.a_high, &t.a_eps})
    for (const auto& r : *m)
      if (r.size() != q_) throw Error("tableau JSON: coefficient rows must have length q");
  if (t.c.size() != q_) throw Error("tableau JSON: c must have length q");
  return t;
}

}  // namespace mprk
