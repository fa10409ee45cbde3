// conv2d_impl.cuh -- conv2d dispatch onto the 2D SSAM engine.
//
// Reference: ssam::conv2d, proj/include/ssam/kernels.hpp:189-225 with the
// window plans of :74-102 (weights flipped: stage (j, t) reads
// w[(m-1-j)*n + (n-1-t)]) and the boundary sampling of :23-28.
#pragma once

#include <vector>

#include "launch.cuh"

namespace ssam_b200 {

// Prefetch depth (rows in flight beyond the register cache) by window height.
__host__ __device__ constexpr int pf_rows(int nr) { return nr <= 3 ? 4 : (nr <= 8 ? 3 : 2); }

template <class T>
std::vector<T> conv_coef(const T* w, int m, int n) {
  std::vector<T> c(static_cast<size_t>(m) * n);
  for (int j = 0; j < m; ++j)
    for (int t = 0; t < n; ++t)
      c[static_cast<size_t>(j) * n + t] = w[static_cast<size_t>(m - 1 - j) * n + (n - 1 - t)];
  return c;
}

// Columns per lane: two 16-byte chunks for short fp32 filters (halves the
// per-cell shuffle and loop overhead), one chunk otherwise.
template <class T>
constexpr int conv_q(int n) {
  return sizeof(T) == 4 ? (n <= 4 ? 8 : 4) : 2;
}

template <class T, int Q, int N>
cudaError_t conv_rt(const Engine2DArgs<T>& a, cudaStream_t s) {
  return launch_ssam2d<T, Q, N, 0, DenseMask, pf_rows(N), 20 * N>(a, s);
}
template <class T, int Q, int K>
cudaError_t conv_sq(const Engine2DArgs<T>& a, cudaStream_t s) {
  return launch_ssam2d<T, Q, K, K, DenseMask, pf_rows(K), K * K>(a, s);
}

#define SSAM_CONV_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) \
  X(18) X(19) X(20)

// Runtime-width engine for every (m, n); compile-time square kernels when
// SQUARE is true (the fp32 benchmark path: fully unrolled, weights as
// constant-bank operands).
template <class T, int Q, bool SQUARE>
cudaError_t conv2d_dispatch(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                            const T* h_w, int m, int n, int boundary, cudaStream_t s) {
  const std::vector<T> coef = conv_coef(h_w, m, n);
  Engine2DArgs<T> a{d_in, d_out, W, H, m, n, coef.data(),
                    boundary ? kBndReplicate : kBndZero, 0, std::max(0, y_begin),
                    std::min(H, y_end)};
  if constexpr (SQUARE) {
    if (m == n) {
      switch (n) {
#define X(K) \
  case K: return conv_sq<T, conv_q<T>(K), K>(a, s);
        SSAM_CONV_CASES(X)
#undef X
      }
    }
  }
  switch (n) {
#define X(N) \
  case N: return conv_rt<T, conv_q<T>(N), N>(a, s);
    SSAM_CONV_CASES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

}  // namespace ssam_b200
