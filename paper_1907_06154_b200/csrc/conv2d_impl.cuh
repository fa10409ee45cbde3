// conv2d_impl.cuh -- conv2d dispatch onto the 2D SSAM engine.
//
// Reference: ssam::conv2d, proj/include/ssam/kernels.hpp:189-225 with the
// window plans of :74-102 (weights flipped: stage (j, t) reads
// w[(m-1-j)*n + (n-1-t)]) and the boundary sampling of :23-28.
#pragma once

#include <cstdlib>
#include <type_traits>
#include <vector>

#include "engine2d_conv.cuh"
#include "engine2d_fma.cuh"
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
#ifndef SSAM_CONV_Q8_MAXN
#define SSAM_CONV_Q8_MAXN 4
#endif
template <class T>
constexpr int conv_q(int n) {
  return sizeof(T) == 4 ? (n <= SSAM_CONV_Q8_MAXN ? 8 : 4) : 2;
}

// Square filters with K >= SSAM_B200_CONV_FMA (default 6; 0 = never) take the
// FMA-bound engine (engine2d_fma.cuh).
inline int conv_fma_min_k() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_CONV_FMA");
    return e ? std::atoi(e) : 6;
  }();
  return v;
}

template <class T, int Q, int NR, int MC, int RY, bool EXACT, int CAP, class Mask = DenseMask,
          bool CHAIN1 = false>
cudaError_t launch_fma2d(const Engine2DArgs<T>& a, cudaStream_t s) {
  constexpr int RB = RY > 4 ? RY : 4;
  constexpr int D = fma2d_depth<Mask, CHAIN1, EXACT, MC, NR, RY, RB>();
  if (a.M * NR > CAP || a.NR != NR || (MC > 0 && a.M != MC)) return cudaErrorInvalidValue;
  if (a.y_end <= a.y_begin) return cudaSuccess;
  Ssam2DTmaParams<T, CAP> P;
  std::memset(&P, 0, sizeof(P));
  Ssam2DParams<T, CAP>& p = P.p;
  p.in = a.in;
  p.out = a.out;
  p.W = a.W;
  p.H = a.H;
  p.M = a.M;
  if (EXACT) {
    p.A = a.M - 1 - (a.M - 1) / 2;  // L: the box starts L columns left of the outputs
    p.V = 32 * Q - (a.M - 1);
  } else {
    const LanePlan lp = plan_lanes(a.M, Q);
    p.A = lp.A;
    p.V = lp.V;
  }
  p.nstrips = (a.W + p.V - 1) / p.V;
  const int rows = a.y_end - a.y_begin;
  p.seg = (pick_seg(rows, p.nstrips, NR) + RB - 1) / RB * RB;
  p.y_begin = a.y_begin;
  p.y_end = a.y_end;
  p.bmode = a.bmode;
  p.ring = a.ring;
  p.vec_ok = 1;
  std::memcpy(p.coef, a.coef, sizeof(T) * a.M * NR);
  auto kern = ssam2d_fma_kernel<T, Q, NR, MC, Mask, RY, RB, D, EXACT, CAP, CHAIN1>;
  const size_t smem = fma2d_smem<T, Q, NR, RB, D, EXACT>(kWarpsPerBlock, a.M);
  const int gx = (p.nstrips + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const dim3 grid(gx, (rows + p.seg - 1) / p.seg);
  cudaError_t e = make_tmap_2d(&P.tmap, a.in, sizeof(T), a.W, a.H, sizeof(T) * a.W,
                               fma2d_pitch<EXACT, Q>(), RB);
  if (e != cudaSuccess) return e;
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  e = launch_pdl(kern, grid, dim3(32 * kWarpsPerBlock), smem, s, P);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

// TMA-eligible calls (zero boundary, 16-byte rows and pointers).
template <class T>
bool fma_eligible(const Engine2DArgs<T>& a) {
  return a.bmode != kBndReplicate && a.W % (16 / sizeof(T)) == 0 && aligned16(a.in) &&
         aligned16(a.out);
}

// Rows per pass (measured on B200, 8192^2 fp32, vs the light kernel):
// RY = 4 up to 10x10 (+4..30%: shorter window shifts, 16 FMA chains),
// RY = 2 at 11x11, RY = 1 beyond (the unrolled pass stays ~1600 FFMAs;
// +3..10%).  The exact lane plan is used where it adds >= 1.5% columns.
#ifndef SSAM_CONV_RY_SMALL
#define SSAM_CONV_RY_SMALL 4
#endif
#ifndef SSAM_CONV_FQ
#define SSAM_CONV_FQ 4
#endif
#ifndef SSAM_CONV_CHAIN1_MIN
#define SSAM_CONV_CHAIN1_MIN 7
#endif
#ifndef SSAM_CONV_RY11
#define SSAM_CONV_RY11 2
#endif
constexpr int fma_ry(int k) { return k <= 10 ? SSAM_CONV_RY_SMALL : (k <= 11 ? SSAM_CONV_RY11 : 1); }
constexpr bool fma_exact(int k, int q) {
  const int r = (k - 1) / 2, l = k - 1 - r, a = (l + q - 1) / q * q;
  const int v_aligned = (32 * q - r - a) / q * q, v_exact = 32 * q - (k - 1);
  return fma_ry(k) == 1 && v_exact * 1000 >= v_aligned * 1015;
}

template <class T, int Q, int K>
cudaError_t conv_fma_sq(const Engine2DArgs<T>& a, cudaStream_t s) {
  // 7x7 .. 11x11: one FMA chain per output (the reference simulator's stage
  // order) instead of the paper's two-level column partials: +4..8%
  // (profiles/r01/conv_chain1_ab.txt), max error 3.1e-6 at 10x10 on 8192^2
  // (fp32 tolerance 1e-5).  Larger filters keep the two-level order, which
  // is what holds 17x17 and 20x20 under 1e-5; 6x6 measured
  // slower with it.
  if constexpr (K >= SSAM_CONV_CHAIN1_MIN && K <= 11 && std::is_same<T, float>::value)
    return launch_fma2d<T, Q, K, K, fma_ry(K), fma_exact(K, Q), K * K, DenseMask, true>(a, s);
  return launch_fma2d<T, Q, K, K, fma_ry(K), fma_exact(K, Q), K * K>(a, s);
}

template <class T, int Q, int N>
cudaError_t conv_rt(const Engine2DArgs<T>& a, cudaStream_t s) {
  return launch_ssam2d<T, Q, N, 0, DenseMask, pf_rows(N), 20 * N>(a, s);
}
// K = 5..15 take the register-row engine (engine2d_conv.cuh) unless
// SSAM_B200_CONV_REG=0: 5x5 536 -> 602-622 GCells/s (3x3 / 4x4 gain nothing,
// profiles/r02/conv_small_ab.txt); 16+ lose to the two-level chain engine
// (profiles/r02/conv_reg_big_ab.txt).
inline bool conv_reg_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_CONV_REG");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}
#ifndef SSAM_CONV_REG_MIN
#define SSAM_CONV_REG_MIN 5
#endif
#ifndef SSAM_CONV_REG_MAX
#define SSAM_CONV_REG_MAX 15
#endif

template <class T, int Q, int K>
cudaError_t conv_sq(const Engine2DArgs<T>& a, cudaStream_t s) {
  if constexpr (K >= SSAM_CONV_REG_MIN && K <= SSAM_CONV_REG_MAX) {
    if (conv_reg_enabled() && a.bmode == kBndZero) {
      const cudaError_t e = launch_conv2d_reg<T, K>(a.in, a.out, a.W, a.H, a.y_begin, a.y_end, a.coef, s);
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
    }
  }
  if constexpr (K >= 3) {
    const int kmin = conv_fma_min_k();
    if (kmin > 0 && K >= kmin && fma_eligible(a))
      return conv_fma_sq<T, (std::is_same<T, float>::value && K <= 11) ? SSAM_CONV_FQ : (Q == 8 ? 4 : Q), K>(a, s);
  }
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
