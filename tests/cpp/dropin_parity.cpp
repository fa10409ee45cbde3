// dropin_parity.cpp -- the reference's own hot-path tests, re-run against the
// B200 drop-in (include/ssam_b200/kernels.hpp) instead of the CPU simulator.
//
// Only the #include of the kernels changes: the cases, inputs and oracle are
// the reference's (proj/tests/test_kernels_conv.cpp, test_kernels_stencil.cpp,
// acceptance.cpp criteria 1-2), with oracle.hpp as ground truth.  Built by
// the top-level Makefile against the reference headers in /root/reference
// (types + oracle) and oracle/_ref (make_benchmark_stencil); needs a GPU.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "ssam/oracle.hpp"
#include "ssam/rng.hpp"
#include "ssam_b200/kernels.hpp"  // <- instead of "ssam/kernels.hpp"

using namespace ssam;

namespace {

int g_checks = 0, g_fail = 0;
std::string g_case;

#define CHECK(cond)                                                                      \
  do {                                                                                   \
    ++g_checks;                                                                          \
    if (!(cond)) {                                                                       \
      ++g_fail;                                                                          \
      std::printf("  FAIL %s: %s (line %d)\n", g_case.c_str(), #cond, __LINE__);        \
    }                                                                                    \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

template <class G>
double max_rel_err(const G& got, const G& want) {
  double worst = 0;
  for (std::size_t i = 0; i < got.data.size(); ++i) {
    const double denom = std::max(1.0, std::abs(static_cast<double>(want.data[i])));
    worst = std::max(worst, std::abs(static_cast<double>(got.data[i]) -
                                     static_cast<double>(want.data[i])) / denom);
  }
  return worst;
}

void run(const char* name, const std::function<void()>& fn) {
  g_case = name;
  const int before = g_fail;
  fn();
  std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

}  // namespace

int main() {
  // ---- proj/tests/test_kernels_conv.cpp ----------------------------------------
  run("conv2d identity filter returns the input", [] {
    auto g = random_grid2d<long long>(64, 40, 1);
    Filter2D<long long> ident;
    CHECK(conv2d(g, ident, KernelConfig{}).data == g.data);
  });
  run("conv2d constant grid times weight sum on the interior", [] {
    Grid2D<long long> g(64, 33, 5);
    Filter2D<long long> f(3, 3, {2, 0, 1, -1, 3, 1, 0, 2, 2});
    auto out = conv2d(g, f, KernelConfig{});
    bool ok = true;
    for (int y = 1; y < 32; ++y)
      for (int x = 1; x < 63; ++x) ok = ok && out.at(x, y) == 50;
    CHECK(ok);
  });
  run("conv2d equals the oracle bit-for-bit in integer mode", [] {
    struct Shape { int m, n; };
    const Shape shapes[] = {{2, 2}, {3, 3}, {5, 5}, {8, 8}, {13, 13}, {20, 20},
                            {3, 5}, {5, 3}, {2, 7}, {1, 4}, {7, 1}};
    for (auto boundary : {Boundary::zero, Boundary::replicate}) {
      SplitMix64 seeds(42);
      for (const auto& sh : shapes) {
        auto g = random_grid2d<long long>(97, 61, seeds.next());
        auto f = random_filter<long long>(sh.m, sh.n, seeds.next());
        KernelConfig cfg;
        cfg.boundary = boundary;
        CHECK(conv2d(g, f, cfg).data == oracle::conv2d_naive(g, f, boundary).data);
      }
    }
  });
  run("conv2d double precision stays within 1e-12 of the double oracle", [] {
    auto g = random_grid2d<double>(96, 48, 9);
    auto f = random_filter<double>(5, 4, 10);
    CHECK(max_rel_err(conv2d(g, f, KernelConfig{}), oracle::conv2d_naive(g, f, Boundary::zero)) <
          1e-12);
  });
  run("conv2d totals are tiles times the per-warp law", [] {
    auto g = random_grid2d<long long>(100, 50, 3);
    auto f = random_filter<long long>(3, 3, 4);
    OpCounters totals;
    conv2d(g, f, KernelConfig{}, &totals);
    const std::uint64_t tiles = 52;  // plan_blocks(100, 50, 3x3, p=4, b=128)
    CHECK(totals.mads == tiles * 9 * 4);
    CHECK(totals.shuffles == tiles * 2 * 4);
    CHECK(totals.broadcast_reads == tiles * 9 * 4);
    CHECK(totals.global_loads == tiles * 32 * 6);
    CHECK(totals.global_stores == 100ULL * 50);
  });
  run("conv2d error paths", [] {
    KernelConfig cfg;
    auto f = random_filter<long long>(3, 3, 1);
    CHECK(throws<std::invalid_argument>([&] { conv2d(random_grid2d<long long>(16, 64, 1), f, cfg); }));
    CHECK(throws<std::invalid_argument>([&] { conv2d(random_grid2d<long long>(64, 4, 1), f, cfg); }));
    auto big = random_filter<long long>(21, 3, 1);
    CHECK(throws<std::invalid_argument>([&] { conv2d(random_grid2d<long long>(64, 64, 1), big, cfg); }));
    KernelConfig huge;
    huge.p = 250;
    CHECK(throws<std::length_error>(
        [&] { conv2d(random_grid2d<long long>(64, 300, 1), random_filter<long long>(3, 8, 1), huge); }));
  });
  run("conv2d equals the oracle across randomized configurations", [] {
    SplitMix64 rng(4096);
    for (int rep = 0; rep < 30; ++rep) {
      const int m = static_cast<int>(rng.next_int(1, 20));
      const int n = static_cast<int>(rng.next_int(1, 20));
      KernelConfig cfg;
      cfg.p = static_cast<int>(rng.next_int(1, 8));
      cfg.b = 32 * static_cast<int>(rng.next_int(1, 6));
      cfg.boundary = rng.next_int(0, 1) ? Boundary::replicate : Boundary::zero;
      const int c = n + cfg.p - 1;
      const int w = static_cast<int>(rng.next_int(32, 200));
      const int h = static_cast<int>(rng.next_int(c, 150));
      auto g = random_grid2d<long long>(w, h, rng.next());
      auto f = random_filter<long long>(m, n, rng.next());
      CHECK(conv2d(g, f, cfg).data == oracle::conv2d_naive(g, f, cfg.boundary).data);
    }
  });
  run("kernels work at non-default lane counts", [] {
    KernelConfig cfg;
    cfg.lane_count = 16;
    cfg.b = 32;
    auto g = random_grid2d<long long>(48, 24, 5);
    auto f = random_filter<long long>(4, 3, 6);
    CHECK(conv2d(g, f, cfg).data == oracle::conv2d_naive(g, f, cfg.boundary).data);
  });

  // ---- proj/tests/test_kernels_stencil.cpp ------------------------------------
  run("stencil2d identity stencil is a fixed point", [] {
    auto g = random_grid2d<long long>(64, 40, 1);
    Stencil<long long> ident;
    ident.order = 0;
    ident.taps = {{{0, 0, 0}, 1}};
    for (int iters : {1, 3}) CHECK(stencil2d(g, ident, KernelConfig{}, iters).data == g.data);
  });
  run("stencil2d single off-center taps catch orientation mistakes", [] {
    auto g = random_grid2d<long long>(64, 48, 7);
    struct Case { int dx, dy; };
    for (auto c : {Case{1, 0}, Case{-1, 0}, Case{0, 1}, Case{0, -1}, Case{1, -1}}) {
      Stencil<long long> st;
      st.order = 1;
      st.taps = {{{c.dx, c.dy, 0}, 1}};
      auto out = stencil2d(g, st, KernelConfig{}, 1);
      bool ok = true;
      for (int y = 1; y < 47; ++y)
        for (int x = 1; x < 63; ++x) ok = ok && out.at(x, y) == g.at(x + c.dx, y + c.dy);
      CHECK(ok);
    }
  });
  run("stencil2d integer stencils are bit-exact against the oracle", [] {
    auto g = random_grid2d<long long>(80, 52, 12);
    Stencil<long long> st;
    st.order = 2;
    st.taps = {{{0, 0, 0}, 3},  {{-1, 0, 0}, 2}, {{2, 0, 0}, -1},
               {{0, -2, 0}, 4}, {{1, 1, 0}, 5},  {{-2, 2, 0}, 1}};
    for (int iters : {1, 2, 4})
      CHECK(stencil2d(g, st, KernelConfig{}, iters).data ==
            oracle::stencil2d_naive(g, st, iters).data);
  });
  run("stencil2d matches the Jacobi oracle on every 2D benchmark", [] {
    for (const auto& name : benchmark_stencil_names()) {
      if (is_3d_benchmark(name)) continue;
      auto st = make_benchmark_stencil(name);
      auto g = random_grid2d<double>(64, 64, 1234);
      CHECK(max_rel_err(stencil2d(g, st, KernelConfig{}, 4), oracle::stencil2d_naive(g, st, 4)) <
            1e-12);
    }
  });
  run("stencil2d preserves the boundary ring exactly", [] {
    auto st = make_benchmark_stencil("2d13pt");
    auto g = random_grid2d<double>(72, 40, 5);
    auto out = stencil2d(g, st, KernelConfig{}, 3);
    const int k = st.order;
    bool ok = true;
    for (int y = 0; y < 40; ++y)
      for (int x = 0; x < 72; ++x)
        if (x < k || x >= 72 - k || y < k || y >= 40 - k) ok = ok && out.at(x, y) == g.at(x, y);
    CHECK(ok);
  });
  run("stencil2d error paths", [] {
    KernelConfig cfg;
    auto st = make_benchmark_stencil("2d5pt");
    CHECK(throws<std::invalid_argument>([&] { stencil2d(random_grid2d<double>(2, 2, 1), st, cfg, 1); }));
    auto g = random_grid2d<double>(64, 64, 1);
    CHECK(throws<std::invalid_argument>([&] { stencil2d(g, st, cfg, 0); }));
    Stencil<double> dup;
    dup.order = 1;
    dup.taps = {{{0, 0, 0}, 1.0}, {{0, 0, 0}, 2.0}};
    CHECK(throws<std::invalid_argument>([&] { stencil2d(g, dup, cfg, 1); }));
    CHECK(throws<std::invalid_argument>([&] { stencil2d(g, make_benchmark_stencil("3d7pt"), cfg, 1); }));
  });
  run("stencil3d matches the Jacobi oracle on every 3D benchmark", [] {
    for (const auto& name : benchmark_stencil_names()) {
      if (!is_3d_benchmark(name)) continue;
      auto st = make_benchmark_stencil(name);
      auto g = random_grid3d<double>(32, 32, 32, 4321);
      KernelConfig cfg;
      cfg.p = 2;
      cfg.b = 32 * (2 * st.order + 2);
      CHECK(max_rel_err(stencil3d(g, st, cfg, 2), oracle::stencil3d_naive(g, st, 2)) < 1e-12);
    }
  });
  run("stencil3d integer exactness", [] {
    auto g = random_grid3d<long long>(36, 10, 9, 31);
    Stencil<long long> st;
    st.dims = 3;
    st.order = 1;
    st.taps = {{{0, 0, 0}, 2}, {{1, 0, 0}, -3}, {{0, -1, 0}, 1}, {{0, 0, 1}, 4}, {{0, 0, -1}, 5}};
    KernelConfig cfg;
    cfg.p = 2;
    CHECK(stencil3d(g, st, cfg, 2).data == oracle::stencil3d_naive(g, st, 2).data);
  });
  run("stencil3d error paths", [] {
    auto st = make_benchmark_stencil("3d13pt");
    auto g = random_grid3d<double>(32, 12, 10, 1);
    KernelConfig cfg;
    cfg.p = 2;
    cfg.b = 128;
    CHECK(throws<std::invalid_argument>([&] { stencil3d(g, st, cfg, 1); }));
    KernelConfig ok;
    ok.p = 2;
    ok.b = 256;
    CHECK(throws<std::invalid_argument>([&] { stencil3d(g, make_benchmark_stencil("2d5pt"), ok, 1); }));
    CHECK(throws<std::invalid_argument>(
        [&] { stencil3d(random_grid3d<double>(32, 12, 3, 1), make_benchmark_stencil("3d13pt"), ok, 1); }));
  });

  // ---- device-set overloads (multi.cpp): slabs sharing device 0 here ----------
  run("stencil3d on a device set equals the one-device call bit for bit", [] {
    for (const char* name : {"3d7pt", "3d13pt", "3d27pt", "poisson"}) {
      auto st = convert_stencil<float>(make_benchmark_stencil(name));
      auto g = random_grid3d<float>(64, 24, 50, 77);
      KernelConfig cfg;
      cfg.p = 2;
      cfg.b = 32 * (2 * st.order + 2);
      OpCounters c1, c2;
      auto one = stencil3d(g, st, cfg, 5, &c1);
      auto many = stencil3d(g, st, cfg, 5, std::vector<int>{0, 0, 0}, &c2);
      CHECK(one.data == many.data);
      CHECK(c1.mads == c2.mads && c1.shuffles == c2.shuffles);
    }
    CHECK(throws<std::invalid_argument>([&] {
      stencil3d(random_grid3d<double>(32, 32, 32, 1), make_benchmark_stencil("3d7pt"),
                KernelConfig{}, 1, std::vector<int>{});
    }));
  });
  run("stencil2d on a device set equals the one-device call bit for bit", [] {
    for (const char* name : {"2d5pt", "2d9pt", "2ds25pt"}) {
      auto st = make_benchmark_stencil(name);
      auto g = random_grid2d<double>(200, 160, 5);
      KernelConfig cfg;
      CHECK(stencil2d(g, st, cfg, 7).data ==
            stencil2d(g, st, cfg, 7, std::vector<int>{0, 0}).data);
    }
  });

  // ---- proj/tests/acceptance.cpp criteria 1 and 2 ------------------------------
  run("acceptance: oracle-equivalence-convolution", [] {
    std::vector<std::pair<int, int>> shapes;
    for (int k = 2; k <= 20; ++k) shapes.push_back({k, k});
    shapes.push_back({3, 5});
    shapes.push_back({5, 3});
    shapes.push_back({2, 7});
    KernelConfig cfg;
    for (std::uint64_t seed = 0; seed <= 9; ++seed) {
      auto grid = random_grid2d<long long>(128, 128, seed);
      for (const auto& [m, n] : shapes) {
        auto filter = random_filter<long long>(m, n, seed * 1000 + m * 31 + n);
        CHECK(conv2d(grid, filter, cfg).data == oracle::conv2d_naive(grid, filter, cfg.boundary).data);
      }
    }
  });
  run("acceptance: oracle-equivalence-stencils", [] {
    for (const auto& name : benchmark_stencil_names()) {
      auto st64 = make_benchmark_stencil(name);
      auto st32 = convert_stencil<float>(st64);
      if (st64.dims == 2) {
        auto g64 = random_grid2d<double>(256, 256, 11);
        auto g32 = random_grid2d<float>(256, 256, 11);
        CHECK(max_rel_err(stencil2d(g64, st64, KernelConfig{}, 4), oracle::stencil2d_naive(g64, st64, 4)) <= 1e-12);
        CHECK(max_rel_err(stencil2d(g32, st32, KernelConfig{}, 4), oracle::stencil2d_naive(g32, st32, 4)) <= 1e-5);
      } else {
        KernelConfig cfg;
        cfg.p = 2;
        cfg.b = std::max(256, 32 * (2 * st64.order + 1));
        auto g64 = random_grid3d<double>(64, 64, 64, 13);
        auto g32 = random_grid3d<float>(64, 64, 64, 13);
        CHECK(max_rel_err(stencil3d(g64, st64, cfg, 2), oracle::stencil3d_naive(g64, st64, 2)) <= 1e-12);
        CHECK(max_rel_err(stencil3d(g32, st32, cfg, 2), oracle::stencil3d_naive(g32, st32, 2)) <= 1e-5);
      }
    }
  });

  // ---- proj/tests/test_kernels_conv.cpp:136-187, :210-221; acceptance criterion 3 ----
  run("conv1d identity, box-on-ramp, and oracle equality", [] {
    std::vector<long long> ramp(100);
    for (int i = 0; i < 100; ++i) ramp[i] = i;
    KernelConfig cfg;
    std::vector<long long> ident = {1};
    CHECK(conv1d(ramp, ident, cfg) == ramp);
    std::vector<long long> box(5, 1);
    auto out = conv1d(ramp, box, cfg);
    for (int i = 2; i < 98; ++i) CHECK(out[i] == 5 * i);
    SplitMix64 rng(8);
    for (int m : {2, 3, 9, 32}) {
      std::vector<long long> f(m), sig(211);
      for (auto& v : f) v = rng.next_int(-9, 9);
      for (auto& v : sig) v = rng.next_int(-100, 100);
      CHECK(conv1d(sig, f, cfg) == oracle::conv1d_naive(sig, f, Boundary::zero));
      KernelConfig repl = cfg;
      repl.boundary = Boundary::replicate;
      CHECK(conv1d(sig, f, repl) == oracle::conv1d_naive(sig, f, Boundary::replicate));
    }
    std::vector<long long> shorty(10, 1);
    CHECK(throws<std::invalid_argument>([&] { conv1d(shorty, box, cfg); }));
    std::vector<long long> wide(33, 1);
    CHECK(throws<std::invalid_argument>([&] { conv1d(ramp, wide, cfg); }));
  });

  run("scan matches prefix sums and uses 5 shuffles per 32-lane tile", [] {
    std::vector<long long> ones(96, 1);
    OpCounters counters;
    auto out = scan(ones, 32, &counters);
    for (int i = 0; i < 96; ++i) CHECK(out[i] == i + 1);
    CHECK(counters.shuffles == 3 * 5);
    std::vector<long long> alt(64);
    for (int i = 0; i < 64; ++i) alt[i] = i % 2 == 0 ? 1 : -1;
    auto alt_out = scan(alt);
    for (int i = 0; i < 64; ++i) CHECK(alt_out[i] == (i % 2 == 0 ? 1 : 0));
    SplitMix64 rng(55);
    for (int tiles : {1, 3, 7}) {
      std::vector<long long> v(32 * tiles);
      for (auto& x : v) x = rng.next_int(-1000, 1000);
      CHECK(scan(v) == oracle::scan_naive(v));
    }
    std::vector<long long> ragged(33, 1);
    CHECK(throws<std::invalid_argument>([&] { scan(ragged); }));
    CHECK(scan(std::vector<long long>{}).empty());
  });

  run("scan at lane_count 16", [] {
    std::vector<long long> v(48);
    SplitMix64 rng(9);
    for (auto& x : v) x = rng.next_int(-50, 50);
    OpCounters counters;
    CHECK(scan(v, 16, &counters) == oracle::scan_naive(v));
    CHECK(counters.shuffles == 3 * 4);
  });

  run("acceptance: scan-prefix-sums", [] {
    SplitMix64 rng(100);
    for (int rep = 0; rep < 1000; ++rep) {
      const int tiles = static_cast<int>(rng.next_int(1, 128));
      std::vector<long long> v(static_cast<std::size_t>(tiles) * 32);
      for (auto& x : v) x = rng.next_int(-1000000, 1000000);
      CHECK(scan(v) == oracle::scan_naive(v));
    }
    OpCounters counters;
    std::vector<long long> one_tile(32, 3);
    scan(one_tile, 32, &counters);
    CHECK(counters.shuffles == 5);
  });

  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
