// ssam_cli.cpp -- the `ssam` command line, routed to the B200 engine.
//
// Mirrors the reference front-end (proj/tools/ssam_cli.cpp) for the hot-path
// commands:
//   ssam run conv1d|conv2d|stencil2d|stencil3d|scan [options]   (:138-246)
//   ssam bench --suite conv-sweep|table3 [options]              (:364-482)
// Every kernel runs through the C ABI (libssam_b200.so) on the GPU and is
// checked against the direct-gather kernels (oracle summation order and
// arithmetic, ssam_b200_gather_*; a plain double running sum for scan).
// Same exit codes (0 pass, 1 mismatch or runtime failure, 2 usage /
// invalid_argument / length_error, :25-27, :664-680), same --corrupt
// fault-injection hook (:131-134), same inputs (grid seed S, filter seed
// S+1, rng.hpp SplitMix64), and one JSON record per line in --out, with no
// timestamps in `run` records so identical flags give identical bytes
// (acceptance criterion 8).  `cost` and `halo` are the reference's analytical
// model and blocking diagnostics, which are not part of the B200 engine: they
// exit 2.  CLI11 / nlohmann::json are not needed: the option grammar is the
// reference's flat `--name value` form.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <vector>

#include "ssam_b200.h"

namespace {

constexpr int kExitPass = 0, kExitMismatch = 1, kExitUsage = 2;

struct Usage {
  std::string msg;
};

// ---- inputs: SplitMix64 exactly as rng.hpp:11-53 ------------------------------
struct SplitMix64 {
  std::uint64_t s;
  explicit SplitMix64(std::uint64_t seed) : s(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  long long next_int(long long lo, long long hi) {
    return lo + static_cast<long long>(next() % static_cast<std::uint64_t>(hi - lo + 1));
  }
  double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-52 - 1.0; }
  template <class T> T scalar() {
    if constexpr (std::is_integral_v<T>) return static_cast<T>(next_int(-100, 100));
    else return static_cast<T>(next_unit());
  }
  template <class T> T coeff() {
    if constexpr (std::is_integral_v<T>) return static_cast<T>(next_int(-9, 9));
    else return static_cast<T>(next_unit());
  }
};

template <class T> std::vector<T> draws(size_t n, std::uint64_t seed, bool coeff) {
  SplitMix64 r(seed);
  std::vector<T> v(n);
  for (T& x : v) x = coeff ? r.template coeff<T>() : r.template scalar<T>();
  return v;
}

// ---- deterministic JSON records (keys sorted, %.17g doubles) ----------------------
struct Json {
  std::map<std::string, std::string> kv;
  Json& s(const std::string& k, const std::string& v) {
    std::string e = "\"";
    for (char c : v) e += (c == '"' || c == '\\') ? std::string("\\") + c : std::string(1, c);
    kv[k] = e + "\"";
    return *this;
  }
  Json& i(const std::string& k, long long v) { kv[k] = std::to_string(v); return *this; }
  Json& u(const std::string& k, unsigned long long v) { kv[k] = std::to_string(v); return *this; }
  Json& b(const std::string& k, bool v) { kv[k] = v ? "true" : "false"; return *this; }
  Json& d(const std::string& k, double v) {
    char buf[40];
    if (std::isfinite(v)) std::snprintf(buf, sizeof buf, "%.17g", v);
    else std::snprintf(buf, sizeof buf, "null");
    kv[k] = buf;
    return *this;
  }
  Json& o(const std::string& k, const Json& v) { kv[k] = v.dump(); return *this; }
  std::string dump() const {
    std::string out = "{";
    for (const auto& [k, v] : kv) out += (out.size() > 1 ? "," : "") + ("\"" + k + "\":" + v);
    return out + "}";
  }
};

Json counters_json(const ssam_op_counters& c) {
  return Json().u("mads", c.mads).u("shuffles", c.shuffles).u("broadcast_reads", c.broadcast_reads)
      .u("global_loads", c.global_loads).u("global_stores", c.global_stores);
}

struct Sink {
  std::string path;
  std::vector<std::string> lines;
  void flush() const {
    if (path.empty()) return;
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open --out file: " + path);
    for (const auto& l : lines) std::fprintf(f, "%s\n", l.c_str());
    std::fclose(f);
  }
};

// Engine status -> the reference's exception classes -> exit codes.
struct EngineError {
  int status;
  std::string msg;
};
void check(int st) {
  if (st != SSAM_OK) throw EngineError{st, ssam_b200_last_error()};
}

struct Err {
  double max_abs = 0, max_rel = 0;
  template <class T> static Err of(const std::vector<T>& got, const std::vector<T>& want) {
    Err e;
    for (size_t k = 0; k < got.size(); ++k) {
      const double a = std::abs(static_cast<double>(got[k]) - static_cast<double>(want[k]));
      e.max_abs = std::max(e.max_abs, a);
      e.max_rel = std::max(e.max_rel, a / std::max(1.0, std::abs(static_cast<double>(want[k]))));
    }
    return e;
  }
};

// ---- options -------------------------------------------------------------------
struct Opts {
  std::map<std::string, std::string> v;
  std::vector<std::string> pos;
  bool has(const std::string& k) const { return v.count(k) > 0; }
  std::string str(const std::string& k, const std::string& d) const {
    auto it = v.find(k);
    return it == v.end() ? d : it->second;
  }
  long long num(const std::string& k, long long d) const {
    auto it = v.find(k);
    if (it == v.end()) return d;
    char* end = nullptr;
    const long long x = std::strtoll(it->second.c_str(), &end, 10);
    if (!end || *end) throw Usage{"--" + k + ": not an integer: " + it->second};
    return x;
  }
};

Opts parse(int argc, char** argv, int first, const std::vector<std::string>& flags,
           const std::vector<std::string>& valued) {
  Opts o;
  for (int a = first; a < argc; ++a) {
    std::string t = argv[a];
    if (t.rfind("--", 0) == 0) {
      const std::string k = t.substr(2);
      bool is_flag = false, is_val = false;
      for (const auto& f : flags) is_flag |= f == k;
      for (const auto& f : valued) is_val |= f == k;
      if (is_flag) {
        o.v[k] = "1";
      } else if (is_val) {
        if (a + 1 >= argc) throw Usage{"--" + k + " needs a value"};
        o.v[k] = argv[++a];
      } else {
        throw Usage{"unknown option " + t};
      }
    } else {
      o.pos.push_back(t);
    }
  }
  return o;
}

int precision_code(const std::string& p) {
  if (p == "f32") return SSAM_DTYPE_F32;
  if (p == "f64") return SSAM_DTYPE_F64;
  if (p == "int") return SSAM_DTYPE_I64;
  throw Usage{"--precision: must be one of f32, f64, int"};
}
const char* precision_name(int d) { return d == 0 ? "f32" : (d == 1 ? "f64" : "int"); }
double tolerance_for(int d) { return d == 0 ? 1e-5 : (d == 1 ? 1e-12 : 0.0); }

template <class T>
struct Stencil {
  int dims = 2, order = 0, fpp = 0;
  std::vector<int> offs;
  std::vector<T> coeffs;
  ssam_stencil c{};
  explicit Stencil(const std::string& name) {
    int o3[3 * 125];
    double cf[125];
    const int t = ssam_b200_benchmark_stencil(name.c_str(), &dims, &order, &fpp, o3, cf, 125);
    if (t < 0) throw Usage{"unknown stencil benchmark: " + name};
    offs.assign(o3, o3 + 3 * t);
    for (int j = 0; j < t; ++j) coeffs.push_back(static_cast<T>(cf[j]));  // convert_stencil
    c = ssam_stencil{dims, order, t, offs.data(), coeffs.data()};
  }
};

// ---- run (ssam_cli.cpp:138-246) ------------------------------------------------------
template <class T>
int run_typed(const Opts& o, const std::string& kernel, int dt, Sink& sink) {
  const std::uint64_t seed = static_cast<std::uint64_t>(o.num("seed", 0));
  const bool repl = o.str("boundary", "zero") == "replicate";
  const bool corrupt = o.has("corrupt");
  ssam_kernel_config cfg;
  ssam_b200_default_config(&cfg);
  cfg.boundary = repl ? SSAM_BOUNDARY_REPLICATE : SSAM_BOUNDARY_ZERO;
  cfg.threads = static_cast<int>(o.num("threads", 0));
  auto set_pb = [&](int order, bool is3d) {
    const long long p = o.num("p", -1), b = o.num("b", -1);
    cfg.p = p > 0 ? static_cast<int>(p) : (is3d ? 2 : 4);
    cfg.b = b > 0 ? static_cast<int>(b) : (is3d ? std::max(128, 32 * (2 * order + 1)) : 128);
  };
  Json rec;
  rec.s("cmd", "run").s("kernel", kernel).s("precision", precision_name(dt)).u("seed", seed)
      .s("boundary", repl ? "replicate" : "zero").s("engine", "b200");
  ssam_op_counters cnt{};
  Err err;
  std::vector<T> got, want;
  int gw = 0, gh = 0;
  auto load2d = [&](int w, int h) {
    const std::string in = o.str("input", "");
    if (in.empty()) {
      gw = w;
      gh = h;
      return draws<T>(static_cast<size_t>(w) * h, seed, false);
    }
    int rank = 0, fdt = 0, dims[3];
    check(ssam_b200_sgrd_info(in.c_str(), &rank, &fdt, dims));
    std::vector<T> g(static_cast<size_t>(dims[0]) * dims[1]);
    check(ssam_b200_sgrd_read(in.c_str(), dt, 2, dims, g.data(), g.size(), 0, nullptr));
    gw = dims[0];
    gh = dims[1];
    return g;
  };
  auto corrupt_one = [&](std::vector<T>& v) {
    if (corrupt && !v.empty()) v[v.size() / 2] += T(1);
  };
  auto dump = [&](int rank, int d0, int d1, int d2) {
    const std::string p = o.str("dump-output", "");
    if (p.empty()) return;
    const int dims[3] = {d0, d1, d2};
    check(ssam_b200_sgrd_write(p.c_str(), dt, rank, dims, got.data(), 0, nullptr));
  };
  if (kernel == "conv2d") {
    set_pb(0, false);
    auto grid = load2d(static_cast<int>(o.num("w", 128)), static_cast<int>(o.num("h", 128)));
    const int m = static_cast<int>(o.num("m", 3)), n = static_cast<int>(o.num("n", 3));
    if (m < 1 || n < 1) throw EngineError{SSAM_ERR_INVALID_ARGUMENT, "filter: taps must be >= 1"};
    auto w = draws<T>(static_cast<size_t>(m) * n, seed + 1, true);
    got.resize(grid.size());
    want.resize(grid.size());
    check(ssam_b200_conv2d(dt, grid.data(), gw, gh, w.data(), m, n, &cfg, got.data(), &cnt));
    corrupt_one(got);
    check(ssam_b200_gather_conv2d(dt, grid.data(), gw, gh, w.data(), m, n, cfg.boundary,
                                  want.data()));
    rec.i("w", gw).i("h", gh).i("m", m).i("n", n).i("p", cfg.p).i("b", cfg.b);
    err = Err::of(got, want);
    dump(2, gw, gh, 1);
  } else if (kernel == "conv1d") {
    set_pb(0, false);
    const int len = static_cast<int>(o.num("len", 1024)), m = static_cast<int>(o.num("m", 3));
    auto sig = draws<T>(static_cast<size_t>(std::max(len, 0)), seed, false);
    auto f = draws<T>(static_cast<size_t>(std::max(m, 0)), seed + 1, true);
    got.resize(sig.size());
    want.resize(sig.size());
    check(ssam_b200_conv1d(dt, sig.data(), len, f.data(), m, &cfg, got.data(), &cnt));
    corrupt_one(got);
    check(ssam_b200_gather_conv2d(dt, sig.data(), len, 1, f.data(), m, 1, cfg.boundary,
                                  want.data()));
    rec.i("len", len).i("m", m);
    err = Err::of(got, want);
  } else if (kernel == "scan") {
    const long long len = o.num("len", 1024);
    auto v = draws<T>(static_cast<size_t>(std::max(len, 0LL)), seed, false);
    got.resize(v.size());
    check(ssam_b200_scan(dt, v.data(), static_cast<unsigned long long>(std::max(len, 0LL)), 32,
                         got.data(), &cnt));
    corrupt_one(got);
    // oracle.hpp:118-127: running sum in double (native int64), rounded per element
    using A = std::conditional_t<std::is_integral_v<T>, long long, double>;
    A run = 0;
    want.resize(v.size());
    for (size_t k = 0; k < v.size(); ++k) want[k] = static_cast<T>(run += static_cast<A>(v[k]));
    rec.i("len", len);
    err = Err::of(got, want);
  } else if (kernel == "stencil2d" || kernel == "stencil3d") {
    const bool is3d = kernel == "stencil3d";
    Stencil<T> st(o.str("stencil", "2d5pt"));
    set_pb(st.order, is3d);
    const int iters = static_cast<int>(o.num("iters", -1) > 0 ? o.num("iters", -1) : (is3d ? 2 : 4));
    if (!is3d) {
      auto grid = load2d(static_cast<int>(o.num("w", 128)), static_cast<int>(o.num("h", 128)));
      got.resize(grid.size());
      want.resize(grid.size());
      check(ssam_b200_stencil2d(dt, grid.data(), gw, gh, &st.c, &cfg, iters, got.data(), &cnt));
      corrupt_one(got);
      check(ssam_b200_gather_stencil(dt, grid.data(), gw, gh, 1, &st.c, iters, want.data()));
      rec.i("w", gw).i("h", gh);
      dump(2, gw, gh, 1);
    } else {
      const int nx = static_cast<int>(o.num("nx", 64)), ny = static_cast<int>(o.num("ny", 64)),
                nz = static_cast<int>(o.num("nz", 64));
      auto grid = draws<T>(static_cast<size_t>(nx) * ny * nz, seed, false);
      got.resize(grid.size());
      want.resize(grid.size());
      check(ssam_b200_stencil3d(dt, grid.data(), nx, ny, nz, &st.c, &cfg, iters, got.data(),
                                &cnt));
      corrupt_one(got);
      check(ssam_b200_gather_stencil(dt, grid.data(), nx, ny, nz, &st.c, iters, want.data()));
      rec.i("nx", nx).i("ny", ny).i("nz", nz);
      dump(3, nx, ny, nz);
    }
    rec.s("stencil", o.str("stencil", "2d5pt")).i("iters", iters).i("p", cfg.p).i("b", cfg.b);
    err = Err::of(got, want);
  }
  const double tol = tolerance_for(dt);
  const bool pass = err.max_rel <= tol;
  rec.d("max_abs_err", err.max_abs).d("max_rel_err", err.max_rel).d("tolerance", tol)
      .o("counters", counters_json(cnt)).b("pass", pass);
  sink.lines.push_back(rec.dump());
  std::printf("run %s precision=%s seed=%llu (B200)\n", kernel.c_str(), precision_name(dt),
              static_cast<unsigned long long>(seed));
  std::printf("  max_abs_err=%.3g max_rel_err=%.3g (tolerance %.0e)\n", err.max_abs, err.max_rel,
              tol);
  std::printf("  counters: mads=%llu shuffles=%llu broadcasts=%llu loads=%llu stores=%llu\n",
              (unsigned long long)cnt.mads, (unsigned long long)cnt.shuffles,
              (unsigned long long)cnt.broadcast_reads, (unsigned long long)cnt.global_loads,
              (unsigned long long)cnt.global_stores);
  std::printf("  result: %s\n", pass ? "PASS" : "FAIL");
  return pass ? kExitPass : kExitMismatch;
}

int cmd_run(int argc, char** argv, Sink& sink) {
  Opts o = parse(argc, argv, 2, {"corrupt"},
                 {"w", "h", "nx", "ny", "nz", "len", "m", "n", "stencil", "iters", "seed", "p", "b",
                  "precision", "boundary", "threads", "profile", "out", "input", "dump-output"});
  if (o.pos.size() != 1) throw Usage{"run: expected one kernel (conv1d|conv2d|stencil2d|stencil3d|scan)"};
  const std::string kernel = o.pos[0];
  if (kernel != "conv1d" && kernel != "conv2d" && kernel != "stencil2d" &&
      kernel != "stencil3d" && kernel != "scan")
    throw Usage{"kernel: unknown kernel " + kernel};
  const std::string b = o.str("boundary", "zero");
  if (b != "zero" && b != "replicate") throw Usage{"--boundary: must be zero or replicate"};
  const int dt = precision_code(o.str("precision", "f64"));
  if ((kernel == "stencil2d" || kernel == "stencil3d") && dt == SSAM_DTYPE_I64)
    throw Usage{"--precision: catalog stencils have fractional coefficients; use f32/f64"};
  sink.path = o.str("out", "");
  switch (dt) {
    case SSAM_DTYPE_F32: return run_typed<float>(o, kernel, dt, sink);
    case SSAM_DTYPE_F64: return run_typed<double>(o, kernel, dt, sink);
    default: return run_typed<long long>(o, kernel, dt, sink);
  }
}

// ---- bench (ssam_cli.cpp:364-482), with measured B200 time ---------------------------
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class T>
bool bench_conv_row(const Opts& o, int k, int dt, Sink& sink) {
  const int size = static_cast<int>(o.num("size", 512));
  const std::uint64_t seed = static_cast<std::uint64_t>(o.num("seed", 0));
  auto grid = draws<T>(static_cast<size_t>(size) * size, seed + k, false);
  auto w = draws<T>(static_cast<size_t>(k) * k, seed + 1000 + k, true);
  std::vector<T> got(grid.size()), want(grid.size());
  ssam_kernel_config cfg;
  ssam_b200_default_config(&cfg);
  ssam_op_counters cnt{};
  const double t0 = now_ms();
  check(ssam_b200_conv2d(dt, grid.data(), size, size, w.data(), k, k, &cfg, got.data(), &cnt));
  const double ms = now_ms() - t0;
  check(ssam_b200_gather_conv2d(dt, grid.data(), size, size, w.data(), k, k, 0, want.data()));
  const Err e = Err::of(got, want);
  const bool pass = e.max_rel <= tolerance_for(dt);
  std::printf("%4dx%-4d %10.3f ms (host call) %10llu %10llu  %s\n", k, k, ms,
              (unsigned long long)cnt.mads, (unsigned long long)cnt.shuffles, pass ? "PASS" : "FAIL");
  sink.lines.push_back(Json().s("cmd", "bench").s("suite", "conv-sweep").i("m", k).i("n", k)
                           .i("size", size).s("precision", precision_name(dt)).u("seed", seed)
                           .s("engine", "b200").d("host_call_ms", ms).d("max_rel_err", e.max_rel)
                           .o("counters", counters_json(cnt)).b("verified", pass).dump());
  return pass;
}

template <class T>
bool bench_table3_row(const Opts& o, const std::string& name, int dt, Sink& sink) {
  Stencil<T> st(name);
  const bool is3d = st.dims == 3;
  const std::uint64_t seed = static_cast<std::uint64_t>(o.num("seed", 0));
  const int size = static_cast<int>(is3d ? o.num("size3d", 64) : o.num("size", 256));
  const int iters = static_cast<int>(is3d ? o.num("iters3d", 2) : o.num("iters2d", 4));
  const size_t cells = is3d ? static_cast<size_t>(size) * size * size : static_cast<size_t>(size) * size;
  auto grid = draws<T>(cells, seed, false);
  std::vector<T> got(cells), want(cells);
  ssam_kernel_config cfg;
  ssam_b200_default_config(&cfg);
  if (is3d) {
    cfg.p = 2;
    cfg.b = std::max(256, 32 * (2 * st.order + 1));
  }
  ssam_op_counters cnt{};
  const double t0 = now_ms();
  if (is3d)
    check(ssam_b200_stencil3d(dt, grid.data(), size, size, size, &st.c, &cfg, iters, got.data(), &cnt));
  else
    check(ssam_b200_stencil2d(dt, grid.data(), size, size, &st.c, &cfg, iters, got.data(), &cnt));
  const double ms = now_ms() - t0;
  check(ssam_b200_gather_stencil(dt, grid.data(), size, size, is3d ? size : 1, &st.c, iters,
                                 want.data()));
  const Err e = Err::of(got, want);
  const bool pass = e.max_rel <= tolerance_for(dt);
  std::printf("%-10s k=%d fpp=%-4d %6d^%d iters=%d rel=%.3g %9.3f ms  %s\n", name.c_str(),
              st.order, st.fpp, size, is3d ? 3 : 2, iters, e.max_rel, ms, pass ? "PASS" : "FAIL");
  sink.lines.push_back(Json().s("cmd", "bench").s("suite", "table3").s("benchmark", name)
                           .i("order", st.order).i("fpp", st.fpp).i("dims", is3d ? 3 : 2)
                           .i("size", size).i("iters", iters).s("precision", precision_name(dt))
                           .u("seed", seed).s("engine", "b200").d("host_call_ms", ms)
                           .d("max_rel_err", e.max_rel).o("counters", counters_json(cnt))
                           .b("verified", pass).dump());
  return pass;
}

int cmd_bench(int argc, char** argv, Sink& sink) {
  Opts o = parse(argc, argv, 2, {},
                 {"suite", "size", "size3d", "iters2d", "iters3d", "precision", "seed", "profile",
                  "threads", "out"});
  if (!o.pos.empty()) throw Usage{"bench: unexpected argument " + o.pos[0]};
  const std::string suite = o.str("suite", "conv-sweep");
  if (suite != "conv-sweep" && suite != "table3") throw Usage{"--suite: must be conv-sweep or table3"};
  const int dt = precision_code(o.str("precision", suite == "table3" ? "f64" : "int"));
  sink.path = o.str("out", "");
  bool all = true;
  if (suite == "conv-sweep") {
    for (int k = 2; k <= 20; ++k)
      all &= dt == 0 ? bench_conv_row<float>(o, k, dt, sink)
                     : (dt == 1 ? bench_conv_row<double>(o, k, dt, sink)
                                : bench_conv_row<long long>(o, k, dt, sink));
  } else {
    if (dt == SSAM_DTYPE_I64)
      throw Usage{"--precision: catalog stencils have fractional coefficients; use f32/f64"};
    for (int i = 0; i < ssam_b200_benchmark_count(); ++i) {
      const std::string name = ssam_b200_benchmark_name(i);
      all &= dt == 0 ? bench_table3_row<float>(o, name, dt, sink)
                     : bench_table3_row<double>(o, name, dt, sink);
    }
  }
  std::printf("bench %s: %s\n", suite.c_str(), all ? "PASS" : "FAIL");
  return all ? kExitPass : kExitMismatch;
}

void usage() {
  std::fprintf(stderr,
               "usage: ssam run conv1d|conv2d|stencil2d|stencil3d|scan [--w W --h H --nx --ny --nz\n"
               "                --len L --m M --n N --stencil NAME --iters I --seed S --p P --b B\n"
               "                --precision f32|f64|int --boundary zero|replicate --out FILE\n"
               "                --input GRID.sgrd --dump-output GRID.sgrd]\n"
               "       ssam bench --suite conv-sweep|table3 [--size --size3d --iters2d --iters3d\n"
               "                --precision --seed --out FILE]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help")) {
    usage();
    return argc < 2 ? kExitUsage : kExitPass;
  }
  const std::string cmd = argv[1];
  Sink sink;
  try {
    int code = kExitUsage;
    if (cmd == "run") {
      code = cmd_run(argc, argv, sink);
    } else if (cmd == "bench") {
      code = cmd_bench(argc, argv, sink);
    } else if (cmd == "cost" || cmd == "halo") {
      throw Usage{cmd + ": the analytical cost model and blocking diagnostics are not part of "
                        "the B200 engine"};
    } else {
      throw Usage{"unknown command " + cmd};
    }
    sink.flush();
    return code;
  } catch (const Usage& u) {
    std::fprintf(stderr, "error: %s\n", u.msg.c_str());
    return kExitUsage;
  } catch (const EngineError& e) {
    if (e.status == SSAM_ERR_INVALID_ARGUMENT) {
      std::fprintf(stderr, "error: %s\n", e.msg.c_str());
      return kExitUsage;
    }
    if (e.status == SSAM_ERR_LENGTH) {
      std::fprintf(stderr, "resource error: %s\n", e.msg.c_str());
      return kExitUsage;
    }
    std::fprintf(stderr, "error: %s\n", e.msg.c_str());
    return kExitMismatch;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitMismatch;
  }
}
