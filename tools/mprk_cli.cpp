// mprk-b200: the reference's benchmark harness (proj/tools/main.cpp) on the
// B200 path, through the C-ABI only (include/mprk_b200.h).
//
//   run          integrate once, JSON run record      (main.cpp:145-171)
//   convergence  tau sweep vs a tiny-tau reference    (main.cpp:173-203)
//   bench        per-label timing CSV + iterations    (main.cpp:243-272)
//   verify       device self-checks, exit 0 iff pass  (report format of main.cpp:274-370)
//
// Same option names, defaults, output formats (ordered JSON keys, CSV
// headers, shortest round-trip numbers) and exit codes (0 ok, 2 solver
// failure, 1 usage/library error, 3 verify failure).  `stability` (region
// scans of the stability function) is not part of the B200 hot path and
// answers with a usage error.  --threads is accepted for compatibility; the
// kernels run on the GPU.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "mprk_b200.h"

namespace {

struct Fail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(int rc) {
  if (rc != MPRKB_OK) throw Fail(mprkb_last_error());
}

// shortest decimal that reads back to the same double (the reference's
// output number format); NaN prints as "nan"
std::string fmt(double v) {
  if (std::isnan(v)) return "nan";
  std::string s(32, '\0');
  s.resize(std::to_chars(s.data(), s.data() + s.size(), v).ptr - s.data());
  return s;
}

// text goes to stdout, or replaces the file named by --out
void write_out(const std::string& path, const std::string& text) {
  std::ostream* os = &std::cout;
  std::ofstream file;
  if (!path.empty()) {
    file.open(path, std::ios::out | std::ios::trunc);
    if (!file.is_open()) throw Fail("cannot open output file: " + path);
    os = &file;
  }
  (*os) << text;
}

// "0.1,0.05,,0.025" -> {0.1, 0.05, 0.025}; a field that is not entirely a
// number is an error
std::vector<double> number_list(const std::string& text) {
  std::vector<double> vals;
  size_t pos = 0;
  while (pos <= text.size()) {
    size_t comma = text.find(',', pos);
    if (comma == std::string::npos) comma = text.size();
    const std::string field = text.substr(pos, comma - pos);
    if (!field.empty()) {
      char* stop = nullptr;
      const double v = std::strtod(field.c_str(), &stop);
      if (stop != field.c_str() + field.size()) throw Fail("malformed number in list: " + field);
      vals.push_back(v);
    }
    pos = comma + 1;
  }
  return vals;
}

// ---- ordered JSON (the layout of nlohmann::ordered_json::dump(2)) ------------------
struct JVal {
  enum Kind { Null, Bool, Int, Num, Str, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<std::pair<std::string, JVal>> obj;
  static JVal num(double v) { JVal j; j.kind = Num; j.d = v; return j; }
  static JVal integer(long long v) { JVal j; j.kind = Int; j.i = v; return j; }
  static JVal str(std::string v) { JVal j; j.kind = Str; j.s = std::move(v); return j; }
  static JVal boolean(bool v) { JVal j; j.kind = Bool; j.b = v; return j; }
  static JVal object() { JVal j; j.kind = Obj; return j; }
  JVal& add(const std::string& k, JVal v) {
    obj.emplace_back(k, std::move(v));
    return *this;
  }
  void dump(std::string& out, int indent) const {
    switch (kind) {
      case Null: out += "null"; break;
      case Bool: out += b ? "true" : "false"; break;
      case Int: out += std::to_string(i); break;
      case Num: out += std::isfinite(d) ? fmt(d) : "null"; break;
      case Str: out += "\"" + s + "\""; break;
      case Obj:
        if (obj.empty()) {
          out += "{}";
          break;
        }
        out += "{\n";
        for (size_t k = 0; k < obj.size(); ++k) {
          out += std::string(indent + 2, ' ') + "\"" + obj[k].first + "\": ";
          obj[k].second.dump(out, indent + 2);
          out += k + 1 < obj.size() ? ",\n" : "\n";
        }
        out += std::string(indent, ' ') + "}";
        break;
    }
  }
};

// ---- options ----------------------------------------------------------------------------
struct CommonOpts {
  std::string eq = "heat";
  std::string method;
  int n = 16;
  double tau = 0.025;
  double tend = 0.1;
  double tol = 1e-6;
  std::string prec = "f64";
  std::string out;
  int threads = 0;
  bool force = false;
};

struct Tab {
  std::string name;
  int q = 0;
  std::vector<double> ah, ae, b;
};

Tab tableau_for(const std::string& name) {
  Tab t;
  t.name = name;
  if (name.rfind("midpoint", 0) == 0) {
    const std::string suffix = name.substr(8);
    int p = 0;
    const auto res = std::from_chars(suffix.data(), suffix.data() + suffix.size(), p);
    if (suffix.empty() || res.ec != std::errc{} || res.ptr != suffix.data() + suffix.size() || p < 0)
      throw Fail("bad corrector count in method name: " + name);
  } else if (name != "4s3pA" && name != "4s3pB" && name != "4s3pC") {
    throw Fail("unknown method name: " + name);
  }
  const int cap = 64;
  t.ah.resize(cap * cap);
  t.ae.resize(cap * cap);
  t.b.resize(cap);
  std::vector<double> c(cap);
  check(mprkb_builtin_tableau(name.c_str(), cap * cap, &t.q, t.ah.data(), t.ae.data(), t.b.data(), c.data()));
  t.ah.resize((size_t)t.q * t.q);
  t.ae.resize((size_t)t.q * t.q);
  t.b.resize(t.q);
  return t;
}

mprkb_config make_config(const CommonOpts& o, const Tab& t) {
  mprkb_config c;
  mprkb_config_init(&c);
  c.equation = o.eq == "heat" ? MPRKB_HEAT : MPRKB_ADVECTION;
  c.n = o.n;
  c.q = t.q;
  c.a_high = t.ah.data();
  c.a_eps = t.ae.data();
  c.b = t.b.data();
  c.tau = o.tau;
  c.t_end = o.tend;
  c.tol = o.tol;
  c.implicit_precision = o.prec == "f32" ? MPRKB_F32 : MPRKB_F64;
  c.record_timings = 1;
  return c;
}

bool refuse_unstable(const CommonOpts& o, const Tab& t) {
  if (o.eq == "heat" && t.name == "4s3pA" && !o.force) {
    std::cerr << "4s3pA is unstable on the heat problem; pass --force to run it anyway\n";
    return true;
  }
  return false;
}

struct Run {
  mprkb_result res{};
  std::vector<std::pair<std::string, std::pair<long long, double>>> timings;  // label -> count, seconds
};

Run integrate_once(const mprkb_config& cfg) {
  mprkb_stepper* s = nullptr;
  check(mprkb_stepper_create(&cfg, &s));
  Run r;
  std::vector<int> its(1 << 16);
  r.res.solve_iterations = its.data();
  r.res.solve_iterations_capacity = (int)its.size();
  const int rc = mprkb_stepper_integrate(s, nullptr, 0, nullptr, &r.res);
  if (rc != MPRKB_OK) {
    const std::string msg = mprkb_last_error();
    mprkb_stepper_destroy(s);
    throw Fail(msg);
  }
  const int nl = mprkb_stepper_timing(s, -1, nullptr, nullptr, nullptr);
  for (int i = 0; i < nl; ++i) {
    const char* label = nullptr;
    long long cnt = 0;
    double sec = 0.0;
    mprkb_stepper_timing(s, i, &label, &cnt, &sec);
    r.timings.push_back({label, {cnt, sec}});
  }
  mprkb_stepper_destroy(s);
  r.res.solve_iterations = nullptr;
  return r;
}

// ---- subcommands ---------------------------------------------------------------------------
int cmd_run(const CommonOpts& o) {
  const Tab t = tableau_for(o.method);
  if (refuse_unstable(o, t)) return 1;
  const mprkb_config cfg = make_config(o, t);
  const Run r = integrate_once(cfg);
  JVal rec = JVal::object();
  rec.add("method", JVal::str(t.name));
  rec.add("equation", JVal::str(o.eq));
  rec.add("n", JVal::integer(o.n));
  rec.add("tau", JVal::num(o.tau));
  rec.add("tend", JVal::num(o.tend));
  rec.add("tol", JVal::num(o.tol));
  rec.add("implicit_precision", JVal::str(o.prec));
  rec.add("failed", JVal::boolean(r.res.solver_failure != 0));
  rec.add("final_error_max", std::isnan(r.res.error_max) ? JVal() : JVal::num(r.res.error_max));
  rec.add("final_error_l2", std::isnan(r.res.error_l2) ? JVal() : JVal::num(r.res.error_l2));
  rec.add("mean_iterations", JVal::num(r.res.mean_iterations));
  rec.add("total_iterations", JVal::integer(r.res.total_iterations));
  rec.add("steps", JVal::integer(r.res.steps));
  rec.add("wall_seconds", JVal::num(r.res.wall_seconds));
  JVal tm = JVal::object();
  for (const auto& [label, e] : r.timings) {
    JVal x = JVal::object();
    x.add("count", JVal::integer(e.first));
    x.add("total_seconds", JVal::num(e.second));
    x.add("seconds_per_call", JVal::num(e.first ? e.second / (double)e.first : 0.0));
    tm.add(label, std::move(x));
  }
  rec.add("timings", std::move(tm));
  std::string text;
  rec.dump(text, 0);
  write_out(o.out, text + "\n");
  return r.res.solver_failure ? 2 : 0;
}

int cmd_convergence(const CommonOpts& o, const std::string& taus_csv) {
  const Tab t = tableau_for(o.method);
  if (refuse_unstable(o, t)) return 1;
  std::vector<double> taus;
  if (!taus_csv.empty()) {
    taus = number_list(taus_csv);
  } else {
    for (int k = 0; k < 4; ++k) taus.push_back(o.tau / std::pow(2.0, k));
  }
  if (taus.empty()) {
    std::cerr << "convergence: the tau list is empty\n";
    return 1;
  }
  const mprkb_config cfg = make_config(o, t);
  std::vector<double> em(taus.size()), el(taus.size());
  double slope = 0.0;
  int failed = 0;
  check(mprkb_temporal_order(&cfg, taus.data(), (int)taus.size(), em.data(), el.data(), &slope, &failed));
  std::string csv = "tau,error_max,error_l2,order_running\n";
  for (size_t i = 0; i < taus.size(); ++i) {
    const double order = i == 0 ? std::nan("") : std::log(em[i - 1] / em[i]) / std::log(taus[i - 1] / taus[i]);
    csv += fmt(taus[i]) + "," + fmt(em[i]) + "," + fmt(el[i]) + "," + fmt(order) + "\n";
  }
  write_out(o.out, csv);
  return failed ? 2 : 0;
}

int cmd_bench(const CommonOpts& o, int repeat) {
  const Tab t = tableau_for(o.method);
  if (refuse_unstable(o, t)) return 1;
  const mprkb_config cfg = make_config(o, t);
  std::vector<std::string> order;
  std::map<std::string, std::pair<long long, double>> agg;
  long long iterations = 0;
  double wall = 0.0;
  bool failed = false;
  for (int r = 0; r < repeat; ++r) {
    const Run run = integrate_once(cfg);
    for (const auto& [label, e] : run.timings) {
      if (!agg.count(label)) order.push_back(label);
      agg[label].first += e.first;
      agg[label].second += e.second;
    }
    iterations += run.res.total_iterations;
    wall += run.res.wall_seconds;
    failed = failed || run.res.solver_failure;
  }
  std::sort(order.begin(), order.end());  // TimingRegistry is an ordered map (timing.hpp:40)
  std::string csv = "label,count,total_seconds,seconds_per_call\n";
  for (const auto& label : order) {
    const auto& e = agg[label];
    csv += label + "," + std::to_string(e.first) + "," + fmt(e.second) + "," +
           fmt(e.first ? e.second / (double)e.first : 0.0) + "\n";
  }
  // run time normalised over the total number of solver iterations
  csv += "iterations," + std::to_string(iterations) + "," + fmt(wall) + "," +
         fmt(iterations > 0 ? wall / (double)iterations : 0.0) + "\n";
  write_out(o.out, csv);
  return failed ? 2 : 0;
}

// verify: device self-checks of the pieces a time step is built from; each
// prints one PASS/FAIL line (the reference's `verify` report format) and the
// exit code is 3 when any fails.  --corrupt perturbs one input so that the
// failure path itself can be exercised.
struct DevVec {
  void* p = nullptr;
  explicit DevVec(size_t bytes) { check(mprkb_malloc(&p, bytes)); }
  ~DevVec() { mprkb_free(p); }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
};

// y = M x for a dense row-major matrix
std::vector<double> matvec(const std::vector<double>& M, const std::vector<double>& x) {
  const size_t m = x.size();
  std::vector<double> y(m, 0.0);
  for (size_t r = 0; r < m; ++r)
    for (size_t c = 0; c < m; ++c) y[r] += M[r * m + c] * x[c];
  return y;
}

// dense Kronecker product of row-major square matrices A (p x p) and B (q x q)
std::vector<double> kron(const std::vector<double>& A, int p, const std::vector<double>& B, int q) {
  const int m = p * q;
  std::vector<double> K((size_t)m * m, 0.0);
  for (int ar = 0; ar < p; ++ar)
    for (int ac = 0; ac < p; ++ac)
      for (int br = 0; br < q; ++br)
        for (int bc = 0; bc < q; ++bc)
          K[(size_t)(ar * q + br) * m + (ac * q + bc)] = A[(size_t)ar * p + ac] * B[(size_t)br * q + bc];
  return K;
}

double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b, double* scale) {
  double d = 0.0, s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    d = std::max(d, std::abs(a[i] - b[i]));
    s = std::max(s, std::abs(b[i]));
  }
  if (scale) *scale = s;
  return d;
}

std::vector<double> run_op_f64(mprkb_op* op, const std::vector<double>& x) {
  const size_t bytes = x.size() * sizeof(double);
  DevVec dx(bytes), dy(bytes);
  std::vector<double> y(x.size());
  check(mprkb_memcpy_h2d(dx.p, x.data(), bytes, nullptr));
  check(mprkb_op_apply(op, dx.p, dy.p, nullptr));
  check(mprkb_memcpy_d2h(y.data(), dy.p, bytes, nullptr));
  check(mprkb_stream_synchronize(nullptr));
  return y;
}

int cmd_verify(bool corrupt) {
  std::vector<std::pair<std::string, bool>> report;

  // (1) built-in tableaus: weights sum to one, strictly lower A_high,
  // lower-triangular A_eps (tableau.cpp:146-190)
  {
    bool ok = true;
    for (const std::string name : {"4s3pA", "4s3pB", "4s3pC", "midpoint1"}) {
      Tab t = tableau_for(name);
      if (corrupt && name == "4s3pB") t.b.back() -= 2e-3;
      const double wsum = std::accumulate(t.b.begin(), t.b.end(), 0.0);
      ok &= std::abs(wsum - 1.0) <= 1e-13;
      for (int r = 0; r < t.q; ++r)
        for (int c = r; c < t.q; ++c) {
          ok &= t.ah[(size_t)r * t.q + c] == 0.0;
          if (c > r) ok &= t.ae[(size_t)r * t.q + c] == 0.0;
        }
    }
    report.emplace_back("tableau-validate", ok);
  }

  // (2) the device stencil equals the explicit Kronecker sum
  //     sigma I + gamma (T (x) I (x) I + I (x) T (x) I + I (x) I (x) T)
  //     with T the 1D Dirichlet Laplacian or periodic central difference
  {
    const int n = 4, m = n * n * n;
    uint64_t state = 0x9E3779B97F4A7C15ull;  // splitmix64 stream
    auto uniform = [&](double lo, double hi) {
      uint64_t z = (state += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      return lo + (hi - lo) * ((double)(z >> 11) * 0x1.0p-53);
    };
    bool ok = true;
    for (const int kind : {MPRKB_DIRICHLET_LAPLACE, MPRKB_PERIODIC_CENTRAL}) {
      std::vector<double> T((size_t)n * n, 0.0), I((size_t)n * n, 0.0);
      for (int i = 0; i < n; ++i) {
        I[(size_t)i * n + i] = 1.0;
        if (kind == MPRKB_DIRICHLET_LAPLACE) {
          T[(size_t)i * n + i] = 2.0;
          if (i > 0) T[(size_t)i * n + i - 1] = -1.0;
          if (i + 1 < n) T[(size_t)i * n + i + 1] = -1.0;
        } else {
          T[(size_t)i * n + (i + 1) % n] += 1.0;
          T[(size_t)i * n + (i + n - 1) % n] -= 1.0;
        }
      }
      // index i + n j + n^2 k: the k factor is the outermost Kronecker factor
      const auto Tk = kron(kron(T, n, I, n), n * n, I, n);
      const auto Tj = kron(kron(I, n, T, n), n * n, I, n);
      const auto Ti = kron(kron(I, n, I, n), n * n, T, n);
      const double sigma = uniform(-1.5, 1.5), gam = uniform(-1.5, 1.5);
      std::vector<double> A((size_t)m * m);
      for (size_t e = 0; e < A.size(); ++e)
        A[e] = gam * (Tk[e] + Tj[e] + Ti[e]) + ((e / m == e % m) ? sigma : 0.0);
      std::vector<double> x(m);
      for (double& v : x) v = uniform(-1.0, 1.0);
      mprkb_op* op = nullptr;
      check(mprkb_op_stencil(MPRKB_F64, n, kind, sigma + (corrupt ? 1e-6 : 0.0), gam, &op));
      const auto got = run_op_f64(op, x);
      mprkb_op_destroy(op);
      double scale = 0.0;
      const double err = max_abs_diff(got, matvec(A, x), &scale);
      ok &= err <= 1e-13 * std::max(1.0, scale);
    }
    report.emplace_back("kronecker-oracle", ok);
  }

  // (3) the stage FastDiag preconditioner inverts the stage operator:
  //     P (A x) = x for the heat stage system (precond.hpp:153-186)
  {
    const int n = 12, m = n * n * n;
    const double tau = 0.01, a = 0.5;
    mprkb_op *A = nullptr, *P = nullptr;
    check(mprkb_op_stage_operator(MPRKB_F64, MPRKB_HEAT, n, 0.0, tau, a, &A));
    check(mprkb_op_fastdiag_stage(MPRKB_F64, MPRKB_HEAT, n, tau, a, MPRKB_FAST, &P));
    std::vector<double> x(m);
    for (int i = 0; i < m; ++i) x[i] = std::cos(0.37 * i) + (corrupt && i == 5 ? 1.0 : 0.0);
    const auto y = run_op_f64(A, x);
    auto z = run_op_f64(P, y);
    if (corrupt) z[5] -= 1.0;
    mprkb_op_destroy(A);
    mprkb_op_destroy(P);
    double scale = 0.0;
    const double err = max_abs_diff(z, x, &scale);
    report.emplace_back("fastdiag-inverse", err <= 1e-10 * std::max(1.0, scale) && !corrupt);
  }

  int failed = 0;
  for (const auto& [name, pass] : report) {
    std::printf("%-24s %s\n", name.c_str(), pass ? "PASS" : "FAIL");
    failed += pass ? 0 : 1;
  }
  return failed ? 3 : 0;
}

[[noreturn]] void usage(const std::string& msg) {
  std::cerr << msg << "\n"
            << "usage: mprk-b200 {run|convergence|bench|verify} [--eq heat|advection] --method M [--n N]\n"
               "                 [--tau T] [--tend T] [--tol X] [--prec f32|f64] [--out FILE] [--threads K]\n"
               "                 [--force] [--taus a,b,c (convergence)] [--repeat R (bench)]\n";
  std::exit(1);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage("a subcommand is required");
  const std::string sub = argv[1];
  CommonOpts o;
  std::string taus;
  int repeat = 1;
  bool corrupt = false, have_method = false;
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) usage(a + " needs a value");
        return argv[++i];
      };
      if (a == "--eq") {
        o.eq = val();
        if (o.eq != "heat" && o.eq != "advection") usage("--eq: heat or advection");
      } else if (a == "--method") {
        o.method = val();
        have_method = true;
      } else if (a == "--n") {
        o.n = std::stoi(val());
        if (o.n <= 0) usage("--n must be positive");
      } else if (a == "--tau") {
        o.tau = std::stod(val());
        if (!(o.tau > 0)) usage("--tau must be positive");
      } else if (a == "--tend") {
        o.tend = std::stod(val());
        if (!(o.tend > 0)) usage("--tend must be positive");
      } else if (a == "--tol") {
        o.tol = std::stod(val());
        if (!(o.tol > 0)) usage("--tol must be positive");
      } else if (a == "--prec") {
        o.prec = val();
        if (o.prec != "f32" && o.prec != "f64") usage("--prec: f32 or f64");
      } else if (a == "--out") {
        o.out = val();
      } else if (a == "--threads") {
        o.threads = std::stoi(val());
      } else if (a == "--force") {
        o.force = true;
      } else if (a == "--taus" && sub == "convergence") {
        taus = val();
      } else if (a == "--repeat" && sub == "bench") {
        repeat = std::stoi(val());
        if (repeat <= 0) usage("--repeat must be positive");
      } else if (a == "--corrupt" && sub == "verify") {
        corrupt = true;
      } else {
        usage("unknown option " + a);
      }
    }
  } catch (const std::exception&) {
    usage("malformed option value");
  }
  try {
    if (sub == "verify") return cmd_verify(corrupt);
    if (sub == "stability")
      usage("stability: region scans of the stability function are outside the B200 hot path "
            "(use the reference mprk tool)");
    if (sub != "run" && sub != "convergence" && sub != "bench") usage("unknown subcommand " + sub);
    if (!have_method) usage("--method is required");
    if (sub == "run") return cmd_run(o);
    if (sub == "convergence") return cmd_convergence(o, taus);
    return cmd_bench(o, repeat);
  } catch (const std::exception& e) {
    std::cerr << e.what() << "\n";
    return 1;
  }
}
