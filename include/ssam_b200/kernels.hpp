// ssam_b200/kernels.hpp -- C++ drop-in for the reference's hot path.
//
// Replaces the three entry points of proj/include/ssam/kernels.hpp
// (relative to /root/reference) with the same signatures, argument meaning
// and exception behaviour, running on the B200 engine through the C ABI in
// ssam_b200.h:
//
//   conv2d     kernels.hpp:189-225  ->  ssam_b200_conv2d
//   stencil2d  kernels.hpp:231-277  ->  ssam_b200_stencil2d
//   stencil3d  kernels.hpp:283-384  ->  ssam_b200_stencil3d
//   (+ device-set overloads of both -> ssam_b200_stencil2d_multi / _3d_multi)
//
// The argument types stay the reference's own (Grid2D/Grid3D, Filter2D,
// Stencil, KernelConfig, OpCounters from ssam/grid.hpp, ssam/filter.hpp,
// ssam/warp.hpp), so calling code compiles unchanged: include this header
// instead of "ssam/kernels.hpp" and link libssam_b200.so.
//
// Errors: std::invalid_argument and std::length_error under exactly the
// reference's conditions (checked before any device work); CUDA failures and
// a missing device raise std::runtime_error -- there is no CPU fallback.
// OpCounters are accumulated (+=) with the reference simulator's counts.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ssam/filter.hpp"
#include "ssam/grid.hpp"
#include "ssam/warp.hpp"
#include "ssam_b200.h"

namespace ssam {

namespace b200_detail {

template <class T>
struct Dtype;
template <>
struct Dtype<float> {
  static constexpr int value = SSAM_DTYPE_F32;
};
template <>
struct Dtype<double> {
  static constexpr int value = SSAM_DTYPE_F64;
};
template <>
struct Dtype<long long> {
  static constexpr int value = SSAM_DTYPE_I64;
};

inline void check(int status) {
  if (status == SSAM_OK) return;
  const std::string msg = ssam_b200_last_error();
  if (status == SSAM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (status == SSAM_ERR_LENGTH) throw std::length_error(msg);
  throw std::runtime_error("ssam_b200: " + msg);
}

inline ssam_kernel_config to_c(const KernelConfig& cfg) {
  ssam_kernel_config c;
  c.p = cfg.p;
  c.b = cfg.b;
  c.boundary = cfg.boundary == Boundary::replicate ? SSAM_BOUNDARY_REPLICATE : SSAM_BOUNDARY_ZERO;
  c.lane_count = cfg.lane_count;
  c.threads = cfg.threads;
  return c;
}

template <class T>
struct StencilArgs {
  std::vector<int> offsets;
  std::vector<T> coeffs;
  ssam_stencil s{};
  explicit StencilArgs(const Stencil<T>& st) {
    for (const auto& tap : st.taps) {
      offsets.insert(offsets.end(), tap.offset.begin(), tap.offset.end());
      coeffs.push_back(tap.coeff);
    }
    s.dims = st.dims;
    s.order = st.order;
    s.ntaps = static_cast<int>(st.taps.size());
    s.offsets = offsets.empty() ? nullptr : offsets.data();
    s.coeffs = coeffs.empty() ? nullptr : coeffs.data();
  }
};

inline ssam_op_counters to_c(const OpCounters* c) {
  ssam_op_counters o{};
  if (c) {
    o.mads = c->mads;
    o.shuffles = c->shuffles;
    o.broadcast_reads = c->broadcast_reads;
    o.global_loads = c->global_loads;
    o.global_stores = c->global_stores;
  }
  return o;
}

inline void from_c(const ssam_op_counters& o, OpCounters* c) {
  if (!c) return;
  c->mads = o.mads;
  c->shuffles = o.shuffles;
  c->broadcast_reads = o.broadcast_reads;
  c->global_loads = o.global_loads;
  c->global_stores = o.global_stores;
}

}  // namespace b200_detail

// kernels.hpp:189 -- true 2D convolution, every cell, cfg.boundary outside.
template <class T>
Grid2D<T> conv2d(const Grid2D<T>& in, const Filter2D<T>& f, const KernelConfig& cfg,
                 OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  b200_detail::check(ssam_b200_check_conv2d(in.width, in.height, f.m, f.n, &c));
  Grid2D<T> out(in.width, in.height);
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_conv2d(b200_detail::Dtype<T>::value, in.data.data(), in.width,
                                      in.height, f.w.data(), f.m, f.n, &c, out.data.data(),
                                      counters ? &oc : nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

// kernels.hpp:231 -- iters Jacobi sweeps; the ring of width st.order carries over.
template <class T>
Grid2D<T> stencil2d(const Grid2D<T>& in, const Stencil<T>& st, const KernelConfig& cfg,
                    int iters, OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  b200_detail::StencilArgs<T> sa(st);
  b200_detail::check(ssam_b200_check_stencil2d(in.width, in.height, &sa.s, &c, iters));
  Grid2D<T> out(in.width, in.height);
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_stencil2d(b200_detail::Dtype<T>::value, in.data.data(), in.width,
                                         in.height, &sa.s, &c, iters, out.data.data(),
                                         counters ? &oc : nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

// kernels.hpp:283 -- iters 3D Jacobi sweeps.
template <class T>
Grid3D<T> stencil3d(const Grid3D<T>& in, const Stencil<T>& st, const KernelConfig& cfg,
                    int iters, OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  b200_detail::StencilArgs<T> sa(st);
  b200_detail::check(ssam_b200_check_stencil3d(in.nx, in.ny, in.nz, &sa.s, &c, iters));
  Grid3D<T> out(in.nx, in.ny, in.nz);
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_stencil3d(b200_detail::Dtype<T>::value, in.data.data(), in.nx,
                                         in.ny, in.nz, &sa.s, &c, iters, out.data.data(),
                                         counters ? &oc : nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

// Multi-GPU extensions (not in the reference): the same calls on a device
// set from one process -- slabs along the slowest axis, slab g on
// devices[g], halos peer-copied between fused launches
// (ssam_b200_stencil2d_multi / _3d_multi).  Results are bit-identical to the
// one-device calls above; errors and counters are theirs.
template <class T>
Grid2D<T> stencil2d(const Grid2D<T>& in, const Stencil<T>& st, const KernelConfig& cfg,
                    int iters, const std::vector<int>& devices, OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  b200_detail::StencilArgs<T> sa(st);
  b200_detail::check(ssam_b200_check_stencil2d(in.width, in.height, &sa.s, &c, iters));
  Grid2D<T> out(in.width, in.height);
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_stencil2d_multi(
      b200_detail::Dtype<T>::value, in.data.data(), in.width, in.height, &sa.s, &c, iters,
      devices.data(), static_cast<int>(devices.size()), out.data.data(),
      counters ? &oc : nullptr, nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

template <class T>
Grid3D<T> stencil3d(const Grid3D<T>& in, const Stencil<T>& st, const KernelConfig& cfg,
                    int iters, const std::vector<int>& devices, OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  b200_detail::StencilArgs<T> sa(st);
  b200_detail::check(ssam_b200_check_stencil3d(in.nx, in.ny, in.nz, &sa.s, &c, iters));
  Grid3D<T> out(in.nx, in.ny, in.nz);
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_stencil3d_multi(
      b200_detail::Dtype<T>::value, in.data.data(), in.nx, in.ny, in.nz, &sa.s, &c, iters,
      devices.data(), static_cast<int>(devices.size()), out.data.data(),
      counters ? &oc : nullptr, nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

// kernels.hpp:390 -- 1D convolution out(i) = sum_s in(i + (m-1)/2 - s) * f[s].
template <class T>
std::vector<T> conv1d(const std::vector<T>& signal, const std::vector<T>& filter,
                      const KernelConfig& cfg, OpCounters* counters = nullptr) {
  const ssam_kernel_config c = b200_detail::to_c(cfg);
  const long long len = static_cast<long long>(signal.size());
  const int m = static_cast<int>(filter.size());
  b200_detail::check(ssam_b200_check_conv1d(len, m, &c));
  std::vector<T> out(signal.size());
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_conv1d(b200_detail::Dtype<T>::value, signal.data(), len,
                                      filter.data(), m, &c, out.data(),
                                      counters ? &oc : nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

// kernels.hpp:422 -- inclusive prefix sum in lane_count tiles.
template <class T>
std::vector<T> scan(const std::vector<T>& values, int lane_count = 32,
                    OpCounters* counters = nullptr) {
  const unsigned long long len = values.size();
  b200_detail::check(ssam_b200_check_scan(len, lane_count));
  if (values.empty()) return {};
  std::vector<T> out(values.size());
  ssam_op_counters oc = b200_detail::to_c(counters);
  b200_detail::check(ssam_b200_scan(b200_detail::Dtype<T>::value, values.data(), len, lane_count,
                                    out.data(), counters ? &oc : nullptr));
  b200_detail::from_c(oc, counters);
  return out;
}

}  // namespace ssam
