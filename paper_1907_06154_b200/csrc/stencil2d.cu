// stencil2d.cu -- one 2D Jacobi sweep on the SSAM engine.
//
// Reference: ssam::stencil2d, proj/include/ssam/kernels.hpp:231-277 with the
// sparse window plans of :111-159 (taps bucketed by column, immediates as
// coefficients, empty columns folded into the next shift).  Here the tap
// footprint is a compile-time mask (StarMask2D for the star benchmarks
// 2d5pt/2d9pt/.../2ds25pt, DenseMask otherwise) so empty cells cost nothing
// and every coefficient is a constant-bank operand.  Orders above 6 use the
// direct-gather kernel.
#include <type_traits>

#include "conv2d_impl.cuh"

namespace ssam_b200 {

template <class T>
std::vector<T> dense2d_coef(const StencilDesc<T>& st) {
  const int k = st.order, M = 2 * k + 1;
  std::vector<T> c(static_cast<size_t>(M) * M, T(0));
  for (size_t i = 0; i < st.taps.size(); ++i)
    c[static_cast<size_t>(st.taps[i].dx + k) * M + (st.taps[i].dy + k)] = st.coeffs[i];
  return c;
}

// Columns per lane: 32 bytes for low orders, 16 bytes (one chunk) otherwise;
// int64 (tests only) stays at one chunk.
template <class T>
constexpr int st_q(int k) {
  return sizeof(T) == 4 ? (k <= 3 ? 8 : 4) : (std::is_same<T, double>::value && k <= 3 ? 4 : 2);
}

// Tall footprints (order >= 4: 9+ rows) take the FMA engine's RY-row
// passes (engine2d_fma.cuh) when the rows are TMA-eligible; SSAM_B200_ST2D_FMA=0
// keeps them on the light kernel.
inline bool st2d_fma_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_ST2D_FMA");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

// Tall stencils accumulate in one FMA chain per output (CHAIN1, the
// reference simulator's stage order); SSAM_B200_ST2D_CHAIN1=0 keeps the
// conv-style two-level order.
inline bool st2d_chain1() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_ST2D_CHAIN1");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

// Orders >= 4 (2d17pt, 2d21pt, 2ds25pt, 2d121pt) take the register-row
// engine (engine2d_conv.cuh) with the stencil's tap mask when the rows are
// TMA-eligible; SSAM_B200_ST2D_REG=0 keeps them on the FMA engine.
inline bool st2d_reg_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_ST2D_REG");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

template <class T, int Q, int K, class Mask>
cudaError_t st2d(const Engine2DArgs<T>& a, cudaStream_t s) {
  constexpr int M = 2 * K + 1;
  constexpr int QQ = st_q<T>(K);
  if constexpr (K >= 4 && !std::is_same<T, long long>::value) {
    if (st2d_reg_enabled()) {
      const cudaError_t e = launch_conv2d_reg<T, M, Mask>(a.in, a.out, a.W, a.H, a.y_begin,
                                                          a.y_end, a.coef, s, a.ring);
      if (e != cudaErrorNotSupported) return e;
      cudaGetLastError();
    }
  }
  if constexpr (K >= 4 && !std::is_same<T, long long>::value) {
    if (st2d_fma_enabled() && fma_eligible(a)) {
      constexpr int QW = QQ, RYW = 4;  // Q = 8 / RY = 2 measured no better (higher registers)
      if (st2d_chain1())
        return launch_fma2d<T, QW, M, M, RYW, false, M * M, Mask, true>(a, s);
      return launch_fma2d<T, QW, M, M, RYW, false, M * M, Mask, false>(a, s);
    }
  }
  return launch_ssam2d<T, QQ, M, M, Mask, pf_rows(M), M * M>(a, s);
}

template <class T, bool STAR>
cudaError_t stencil2d_dispatch(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                               const StencilDesc<T>& st, cudaStream_t s) {
  constexpr int Q = Lanes<T>::Q;
  const int k = st.order;
  y_begin = std::max(y_begin, k);
  y_end = std::min(y_end, H - k);
  if (y_end <= y_begin || W - 2 * k <= 0) return cudaSuccess;
  if (k > 6) return stencil2d_direct<T>(d_in, d_out, W, H, y_begin, y_end, st, s);
  const std::vector<T> coef = dense2d_coef(st);
  Engine2DArgs<T> a{d_in, d_out, W, H, 2 * k + 1, 2 * k + 1, coef.data(), kBndStencil, k,
                    y_begin, y_end};
  if constexpr (STAR) {
    if (k >= 1 && classify2d(st.taps, k) == Shape2D::star) {
      switch (k) {
        case 1: return st2d<T, Q, 1, StarMask2D<1>>(a, s);
        case 2: return st2d<T, Q, 2, StarMask2D<2>>(a, s);
        case 3: return st2d<T, Q, 3, StarMask2D<3>>(a, s);
        case 4: return st2d<T, Q, 4, StarMask2D<4>>(a, s);
        case 5: return st2d<T, Q, 5, StarMask2D<5>>(a, s);
        case 6: return st2d<T, Q, 6, StarMask2D<6>>(a, s);
      }
    }
  }
  switch (k) {
    case 0: return st2d<T, Q, 0, DenseMask>(a, s);
    case 1: return st2d<T, Q, 1, DenseMask>(a, s);
    case 2: return st2d<T, Q, 2, DenseMask>(a, s);
    case 3: return st2d<T, Q, 3, DenseMask>(a, s);
    case 4: return st2d<T, Q, 4, DenseMask>(a, s);
    case 5: return st2d<T, Q, 5, DenseMask>(a, s);
    case 6: return st2d<T, Q, 6, DenseMask>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <>
cudaError_t stencil2d_sweep<float>(const float* i, float* o, int W, int H, int yb, int ye,
                                   const StencilDesc<float>& st, cudaStream_t s) {
  return stencil2d_dispatch<float, true>(i, o, W, H, yb, ye, st, s);
}
template <>
cudaError_t stencil2d_sweep<double>(const double* i, double* o, int W, int H, int yb, int ye,
                                    const StencilDesc<double>& st, cudaStream_t s) {
  return stencil2d_dispatch<double, true>(i, o, W, H, yb, ye, st, s);
}
template <>
cudaError_t stencil2d_sweep<long long>(const long long* i, long long* o, int W, int H, int yb, int ye,
                                       const StencilDesc<long long>& st, cudaStream_t s) {
  return stencil2d_dispatch<long long, false>(i, o, W, H, yb, ye, st, s);
}

}  // namespace ssam_b200
