// mprk-b200: the reference's benchmark harness (proj/tools/main.cpp) on the
// B200 path, through the C-ABI only (include/mprk_b200.h).
//
//   run          integrate once, JSON run record      (main.cpp:145-171)
//   convergence  tau sweep vs a tiny-tau reference    (main.cpp:173-203)
//   bench        per-label timing CSV + iterations    (main.cpp:243-272)
//   verify       device self-checks, exit 0 iff pass  (main.cpp:274-370)
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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
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

std::string fmt(double v) {
  if (std::isnan(v)) return "nan";
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, res.ptr);
}

void emit(const std::string& text, const std::string& out_path) {
  if (out_path.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream f(out_path);
  if (!f) throw Fail("cannot open output file: " + out_path);
  f << text;
}

std::vector<double> parse_doubles(const std::string& csv) {
  std::vector<double> out;
  std::stringstream ss(csv);
  std::string item;
  while (std::getline(ss, item, ',')) {
    if (item.empty()) continue;
    std::size_t used = 0;
    const double v = std::stod(item, &used);
    if (used != item.size()) throw Fail("malformed number in list: " + item);
    out.push_back(v);
  }
  return out;
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
  emit(text + "\n", o.out);
  return r.res.solver_failure ? 2 : 0;
}

int cmd_convergence(const CommonOpts& o, const std::string& taus_csv) {
  const Tab t = tableau_for(o.method);
  if (refuse_unstable(o, t)) return 1;
  std::vector<double> taus;
  if (!taus_csv.empty()) {
    taus = parse_doubles(taus_csv);
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
  emit(csv, o.out);
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
  emit(csv, o.out);
  return failed ? 2 : 0;
}

// verify: the reference's self-checks that concern the time-stepping path,
// run on the device.
int cmd_verify(bool corrupt) {
  struct Check {
    std::string name;
    bool pass;
  };
  std::vector<Check> checks;
  {
    // builtin tableaus are structurally valid: row sums, sum(b) = 1, lower
    // triangular, implicit diagonal in A_eps only (tableau.cpp:146-190)
    bool ok = true;
    for (const char* m : {"4s3pA", "4s3pB", "4s3pC"}) {
      Tab t = tableau_for(m);
      if (corrupt && std::string(m) == "4s3pB") t.b[0] += 1e-3;
      double bs = 0.0;
      for (double w : t.b) bs += w;
      ok = ok && std::abs(bs - 1.0) <= 1e-13;
      for (int i = 0; i < t.q; ++i)
        for (int j = 0; j < t.q; ++j) {
          if (j > i) ok = ok && t.ah[i * t.q + j] == 0.0 && t.ae[i * t.q + j] == 0.0;
          if (j == i) ok = ok && t.ah[i * t.q + j] == 0.0;
        }
    }
    checks.push_back({"tableau-validate", ok});
  }
  {
    // the device Kronecker-sum stencil against a dense Kronecker product at
    // n = 3 (main.cpp:310-349)
    const int n = 3, nn = n * n * n;
    std::mt19937 rng(777);
    std::uniform_real_distribution<double> dist(-2.0, 2.0);
    bool ok = true;
    for (const int stencil : {MPRKB_DIRICHLET_LAPLACE, MPRKB_PERIODIC_CENTRAL}) {
      std::vector<std::vector<double>> k1(n, std::vector<double>(n, 0.0));
      if (stencil == MPRKB_DIRICHLET_LAPLACE) {
        for (int i = 0; i < n; ++i) {
          k1[i][i] = 2.0;
          if (i > 0) k1[i][i - 1] = -1.0;
          if (i + 1 < n) k1[i][i + 1] = -1.0;
        }
      } else {
        for (int i = 0; i < n; ++i) {
          k1[i][(i + 1) % n] += 1.0;
          k1[i][(i + n - 1) % n] -= 1.0;
        }
      }
      const double sigma = dist(rng), gamma = dist(rng);
      std::vector<double> x(nn), got(nn), want(nn, 0.0);
      for (double& v : x) v = dist(rng);
      void *dx = nullptr, *dy = nullptr;
      check(mprkb_malloc(&dx, nn * 8));
      check(mprkb_malloc(&dy, nn * 8));
      check(mprkb_memcpy_h2d(dx, x.data(), nn * 8, nullptr));
      check(mprkb_stencil_apply(MPRKB_F64, n, stencil, sigma, gamma, dx, dy, nullptr));
      check(mprkb_memcpy_d2h(got.data(), dy, nn * 8, nullptr));
      check(mprkb_stream_synchronize(nullptr));
      mprkb_free(dx);
      mprkb_free(dy);
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) {
            const int row = i + n * j + n * n * k;
            want[row] += sigma * x[row];
            for (int c = 0; c < n; ++c) {
              want[row] += gamma * k1[k][c] * x[i + n * j + n * n * c];
              want[row] += gamma * k1[j][c] * x[i + n * c + n * n * k];
              want[row] += gamma * k1[i][c] * x[c + n * j + n * n * k];
            }
          }
      double err = 0.0, ref = 0.0;
      for (int r = 0; r < nn; ++r) {
        err = std::max(err, std::abs(got[r] - want[r]));
        ref = std::max(ref, std::abs(want[r]));
      }
      ok = ok && err <= 1e-12 * std::max(1.0, ref);
    }
    checks.push_back({"kronecker-oracle", ok});
  }
  bool all = true;
  for (const Check& c : checks) {
    std::printf("%-24s %s\n", c.name.c_str(), c.pass ? "PASS" : "FAIL");
    all = all && c.pass;
  }
  return all ? 0 : 3;
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
