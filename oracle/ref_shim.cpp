// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (builds oracle/_ref/libssam_ref.so).
//
// A thin extern "C" wrapper over the UNMODIFIED reference, compiled straight
// from /root/reference/proj/{include,src} by oracle/Makefile with the
// reference's own Release flags (-O3 -DNDEBUG -fopenmp, proj/CMakeLists.txt:5-11).
// No reference source is copied into this repo; this file only adapts the
// reference's C++ templates to plain pointers so Python can drive them.
//
// Exposed:
//   * the reference's CPU SSAM path (ssam::conv2d/stencil2d/stencil3d,
//     proj/include/ssam/kernels.hpp:189,231,283) -- the CPU baseline that
//     bench.py --impl reference times, and the source of OpCounters truth;
//   * the reference oracle (proj/include/ssam/oracle.hpp:44-116) and input
//     generators (grid.hpp:52-66, filter.hpp:41-47) -- used to pin
//     oracle/ssam_oracle.c through tests/golden/.
//
// Status codes mirror the C ABI: 0 ok, 1 std::invalid_argument,
// 2 std::length_error, 9 anything else.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ssam/filter.hpp"
#include "ssam/grid.hpp"
#include "ssam/kernels.hpp"
#include "ssam/oracle.hpp"
#include "ssam/grid_io.hpp"
#include "ssam/perf_model.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace ssam;

namespace {

enum { F32 = 0, F64 = 1, I64 = 2 };

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::length_error&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::runtime_error&) {
    return 3;
  } catch (...) {
    return 9;
  }
}

KernelConfig make_cfg(int p, int b, int boundary, int lane_count, int threads) {
  KernelConfig cfg;
  cfg.p = p;
  cfg.b = b;
  cfg.boundary = boundary ? Boundary::replicate : Boundary::zero;
  cfg.lane_count = lane_count;
  cfg.threads = threads;
  return cfg;
}

void put_counters(const OpCounters& c, std::uint64_t* out) {
  if (!out) return;
  out[0] = c.mads;
  out[1] = c.shuffles;
  out[2] = c.broadcast_reads;
  out[3] = c.global_loads;
  out[4] = c.global_stores;
}

template <class T>
Stencil<T> make_stencil(int dims, int order, const int* offsets, const void* coeffs, int ntaps) {
  Stencil<T> st;
  st.name = "abi";
  st.dims = dims;
  st.order = order;
  const T* c = static_cast<const T*>(coeffs);
  for (int j = 0; j < ntaps; ++j)
    st.taps.push_back({{offsets[3 * j], offsets[3 * j + 1], offsets[3 * j + 2]}, c[j]});
  return st;
}

template <class T>
int conv2d_t(const void* in, int w, int h, const void* wts, int m, int n, const KernelConfig& cfg,
             void* out, std::uint64_t* counters, bool naive) {
  return guarded([&] {
    Grid2D<T> g(w, h);
    std::memcpy(g.data.data(), in, sizeof(T) * g.data.size());
    const T* wp = static_cast<const T*>(wts);
    Filter2D<T> f(m, n, std::vector<T>(wp, wp + static_cast<std::size_t>(m) * n));
    OpCounters c;
    Grid2D<T> r = naive ? oracle::conv2d_naive(g, f, cfg.boundary) : conv2d(g, f, cfg, &c);
    std::memcpy(out, r.data.data(), sizeof(T) * r.data.size());
    put_counters(c, counters);
  });
}

template <class T>
int stencil2d_t(const void* in, int w, int h, const Stencil<T>& st, const KernelConfig& cfg,
                int iters, void* out, std::uint64_t* counters, bool naive) {
  return guarded([&] {
    Grid2D<T> g(w, h);
    std::memcpy(g.data.data(), in, sizeof(T) * g.data.size());
    OpCounters c;
    Grid2D<T> r = naive ? oracle::stencil2d_naive(g, st, iters) : stencil2d(g, st, cfg, iters, &c);
    std::memcpy(out, r.data.data(), sizeof(T) * r.data.size());
    put_counters(c, counters);
  });
}

template <class T>
int stencil3d_t(const void* in, int nx, int ny, int nz, const Stencil<T>& st,
                const KernelConfig& cfg, int iters, void* out, std::uint64_t* counters,
                bool naive) {
  return guarded([&] {
    Grid3D<T> g(nx, ny, nz);
    std::memcpy(g.data.data(), in, sizeof(T) * g.data.size());
    OpCounters c;
    Grid3D<T> r = naive ? oracle::stencil3d_naive(g, st, iters) : stencil3d(g, st, cfg, iters, &c);
    std::memcpy(out, r.data.data(), sizeof(T) * r.data.size());
    put_counters(c, counters);
  });
}

template <class T>
int conv1d_t(const void* in, int len, const void* wts, int m, const KernelConfig& cfg, void* out,
             std::uint64_t* counters, bool naive) {
  return guarded([&] {
    const T* ip = static_cast<const T*>(in);
    const T* wp = static_cast<const T*>(wts);
    std::vector<T> sig(ip, ip + len), f(wp, wp + m);
    OpCounters c;
    std::vector<T> r = naive ? oracle::conv1d_naive(sig, f, cfg.boundary) : conv1d(sig, f, cfg, &c);
    std::memcpy(out, r.data(), sizeof(T) * r.size());
    put_counters(c, counters);
  });
}

template <class T>
int scan_t(const void* in, int len, int lane_count, void* out, std::uint64_t* counters,
           bool naive) {
  return guarded([&] {
    const T* ip = static_cast<const T*>(in);
    std::vector<T> v(ip, ip + len);
    OpCounters c;
    std::vector<T> r = naive ? oracle::scan_naive(v) : scan(v, lane_count, &c);
    if (!r.empty()) std::memcpy(out, r.data(), sizeof(T) * r.size());
    put_counters(c, counters);
  });
}

// SGRD files through the reference's own writer / readers (grid_io.hpp).
template <class T>
int sgrd_write_t(const char* path, int rank, const int* dims, const void* data) {
  return guarded([&] {
    const T* p = static_cast<const T*>(data);
    if (rank == 1) {
      write_grid_file<T>(path, std::vector<T>(p, p + dims[0]));
    } else if (rank == 2) {
      Grid2D<T> g(dims[0], dims[1]);
      std::memcpy(g.data.data(), p, sizeof(T) * g.data.size());
      write_grid_file<T>(path, g);
    } else {
      Grid3D<T> g(dims[0], dims[1], dims[2]);
      std::memcpy(g.data.data(), p, sizeof(T) * g.data.size());
      write_grid_file<T>(path, g);
    }
  });
}

template <class T>
int sgrd_read_t(const char* path, int rank, int* dims, void* out, long long cap) {
  return guarded([&] {
    std::ifstream is(path, std::ios::binary);
    std::vector<T> v;
    if (rank == 1) {
      v = read_vector<T>(is);
      dims[0] = static_cast<int>(v.size()); dims[1] = dims[2] = 1;
    } else if (rank == 2) {
      Grid2D<T> g = read_grid2d<T>(is);
      v = g.data; dims[0] = g.width; dims[1] = g.height; dims[2] = 1;
    } else {
      Grid3D<T> g = read_grid3d<T>(is);
      v = g.data; dims[0] = g.nx; dims[1] = g.ny; dims[2] = g.nz;
    }
    if (static_cast<long long>(v.size()) <= cap && !v.empty())
      std::memcpy(out, v.data(), sizeof(T) * v.size());
  });
}

}  // namespace

extern "C" {

int ssam_ref_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// naive != 0 runs oracle::conv2d_naive instead of the SSAM simulator.
int ssam_ref_conv2d(int dtype, const void* in, int w, int h, const void* wts, int m, int n,
                    int p, int b, int boundary, int lane_count, int threads, void* out,
                    std::uint64_t* counters, int naive) {
  const KernelConfig cfg = make_cfg(p, b, boundary, lane_count, threads);
  switch (dtype) {
    case F32: return conv2d_t<float>(in, w, h, wts, m, n, cfg, out, counters, naive);
    case F64: return conv2d_t<double>(in, w, h, wts, m, n, cfg, out, counters, naive);
    case I64: return conv2d_t<long long>(in, w, h, wts, m, n, cfg, out, counters, naive);
  }
  return 9;
}

int ssam_ref_stencil2d(int dtype, const void* in, int w, int h, int dims, int order,
                       const int* offsets, const void* coeffs, int ntaps, int p, int b,
                       int lane_count, int threads, int iters, void* out,
                       std::uint64_t* counters, int naive) {
  const KernelConfig cfg = make_cfg(p, b, 0, lane_count, threads);
  switch (dtype) {
    case F32:
      return stencil2d_t<float>(in, w, h, make_stencil<float>(dims, order, offsets, coeffs, ntaps),
                                cfg, iters, out, counters, naive);
    case F64:
      return stencil2d_t<double>(in, w, h,
                                 make_stencil<double>(dims, order, offsets, coeffs, ntaps), cfg,
                                 iters, out, counters, naive);
    case I64:
      return stencil2d_t<long long>(
          in, w, h, make_stencil<long long>(dims, order, offsets, coeffs, ntaps), cfg, iters, out,
          counters, naive);
  }
  return 9;
}

int ssam_ref_stencil3d(int dtype, const void* in, int nx, int ny, int nz, int dims, int order,
                       const int* offsets, const void* coeffs, int ntaps, int p, int b,
                       int lane_count, int threads, int iters, void* out,
                       std::uint64_t* counters, int naive) {
  const KernelConfig cfg = make_cfg(p, b, 0, lane_count, threads);
  switch (dtype) {
    case F32:
      return stencil3d_t<float>(in, nx, ny, nz,
                                make_stencil<float>(dims, order, offsets, coeffs, ntaps), cfg,
                                iters, out, counters, naive);
    case F64:
      return stencil3d_t<double>(in, nx, ny, nz,
                                 make_stencil<double>(dims, order, offsets, coeffs, ntaps), cfg,
                                 iters, out, counters, naive);
    case I64:
      return stencil3d_t<long long>(in, nx, ny, nz,
                                    make_stencil<long long>(dims, order, offsets, coeffs, ntaps),
                                    cfg, iters, out, counters, naive);
  }
  return 9;
}

// random_grid2d<T>(count, 1, seed) draws the same stream as random_grid3d.
int ssam_ref_random_grid(int dtype, void* out, int count, std::uint64_t seed) {
  return guarded([&] {
    switch (dtype) {
      case F32: { auto g = random_grid2d<float>(count, 1, seed); std::memcpy(out, g.data.data(), 4ul * count); break; }
      case F64: { auto g = random_grid2d<double>(count, 1, seed); std::memcpy(out, g.data.data(), 8ul * count); break; }
      default: { auto g = random_grid2d<long long>(count, 1, seed); std::memcpy(out, g.data.data(), 8ul * count); break; }
    }
  });
}

int ssam_ref_random_filter(int dtype, void* out, int m, int n, std::uint64_t seed) {
  return guarded([&] {
    const std::size_t cnt = static_cast<std::size_t>(m) * n;
    switch (dtype) {
      case F32: { auto f = random_filter<float>(m, n, seed); std::memcpy(out, f.w.data(), 4 * cnt); break; }
      case F64: { auto f = random_filter<double>(m, n, seed); std::memcpy(out, f.w.data(), 8 * cnt); break; }
      default: { auto f = random_filter<long long>(m, n, seed); std::memcpy(out, f.w.data(), 8 * cnt); break; }
    }
  });
}

int ssam_ref_benchmark_stencil(const char* name, int* dims, int* order, int* fpp, int* offsets,
                               double* coeffs, int cap) {
  try {
    Stencil<double> st = make_benchmark_stencil(name);
    if (static_cast<int>(st.taps.size()) > cap) return -2;
    for (std::size_t j = 0; j < st.taps.size(); ++j) {
      offsets[3 * j] = st.taps[j].offset[0];
      offsets[3 * j + 1] = st.taps[j].offset[1];
      offsets[3 * j + 2] = st.taps[j].offset[2];
      coeffs[j] = st.taps[j].coeff;
    }
    *dims = st.dims;
    *order = st.order;
    *fpp = st.fpp;
    return static_cast<int>(st.taps.size());
  } catch (...) {
    return -1;
  }
}

int ssam_ref_conv1d(int dtype, const void* in, int len, const void* wts, int m, int boundary,
                    int lane_count, void* out, std::uint64_t* counters, int naive) {
  const KernelConfig cfg = make_cfg(4, 128, boundary, lane_count, 0);
  switch (dtype) {
    case F32: return conv1d_t<float>(in, len, wts, m, cfg, out, counters, naive != 0);
    case F64: return conv1d_t<double>(in, len, wts, m, cfg, out, counters, naive != 0);
    case I64: return conv1d_t<long long>(in, len, wts, m, cfg, out, counters, naive != 0);
  }
  return 1;
}

int ssam_ref_scan(int dtype, const void* in, int len, int lane_count, void* out,
                  std::uint64_t* counters, int naive) {
  switch (dtype) {
    case F32: return scan_t<float>(in, len, lane_count, out, counters, naive != 0);
    case F64: return scan_t<double>(in, len, lane_count, out, counters, naive != 0);
    case I64: return scan_t<long long>(in, len, lane_count, out, counters, naive != 0);
  }
  return 1;
}

int ssam_ref_sgrd_write(int dtype, const char* path, int rank, const int* dims, const void* data) {
  switch (dtype) {
    case F32: return sgrd_write_t<float>(path, rank, dims, data);
    case F64: return sgrd_write_t<double>(path, rank, dims, data);
    case I64: return sgrd_write_t<long long>(path, rank, dims, data);
  }
  return 1;
}

int ssam_ref_sgrd_read(int dtype, const char* path, int rank, int* dims, void* out, long long cap) {
  switch (dtype) {
    case F32: return sgrd_read_t<float>(path, rank, dims, out, cap);
    case F64: return sgrd_read_t<double>(path, rank, dims, out, cap);
    case I64: return sgrd_read_t<long long>(path, rank, dims, out, cap);
  }
  return 1;
}

// ssam::resolve_profile (perf_model.cpp:89-97: builtin name, then
// $SSAM_PROFILE_DIR/<name>.profile, then a path) -> the six latencies as
// doubles, the profile name, and the model's latency_reg / latency_smem
// (perf_model.hpp:38-44) at m x n.
int ssam_ref_profile(const char* name_or_path, char* name, int name_cap, double* vals, int m,
                     int n, double* l_reg_smem) {
  return guarded([&] {
    const LatencyProfile p = resolve_profile(name_or_path);
    std::snprintf(name, static_cast<size_t>(name_cap), "%s", p.name.c_str());
    const Rational* r[6] = {&p.t_shfl, &p.t_mad, &p.t_smem_read, &p.t_reg, &p.t_gmem_read,
                            &p.t_gmem_write};
    for (int i = 0; i < 6; ++i) vals[i] = r[i]->to_double();
    l_reg_smem[0] = latency_reg(m, n, p).to_double();
    l_reg_smem[1] = latency_smem(m, n, p).to_double();
  });
}

}  // extern "C"
