// stencil3d.cu -- one 3D Jacobi sweep on the z-streaming SSAM engine.
//
// Reference: ssam::stencil3d, proj/include/ssam/kernels.hpp:283-384 (per-dz
// plane plans summed through InterWarpBuffer).  Shapes with a compile-time
// mask: 3d7pt (star K=1), 3d13pt (star K=2), 3d27pt (box K=1), poisson
// (3x3x3 minus corners); any other tap set of order <= 2 runs the dense
// engine with zero cells, larger orders the direct-gather kernel.
#include "launch.cuh"

namespace ssam_b200 {

template <class T>
std::vector<T> dense3d_coef(const StencilDesc<T>& st) {
  const int k = st.order, M = 2 * k + 1;
  std::vector<T> c(static_cast<size_t>(M) * M * M, T(0));
  for (size_t i = 0; i < st.taps.size(); ++i) {
    const Tap& tp = st.taps[i];
    c[(static_cast<size_t>(tp.dz + k) * M + (tp.dx + k)) * M + (tp.dy + k)] = st.coeffs[i];
  }
  return c;
}

// Rows per warp and z-prefetch by (dtype, order): keeps the register cache
// (2K+1 planes x (RY+2K) rows x Q columns) within ~100 registers.
template <class T, int K> struct Cfg3D;
template <> struct Cfg3D<float, 0> { static constexpr int RY = 4; };
template <> struct Cfg3D<float, 1> { static constexpr int RY = 4; };
template <> struct Cfg3D<float, 2> { static constexpr int RY = 2; };
template <> struct Cfg3D<double, 0> { static constexpr int RY = 4; };
template <> struct Cfg3D<double, 1> { static constexpr int RY = 4; };
template <> struct Cfg3D<double, 2> { static constexpr int RY = 2; };
template <> struct Cfg3D<long long, 0> { static constexpr int RY = 4; };
template <> struct Cfg3D<long long, 1> { static constexpr int RY = 4; };
template <> struct Cfg3D<long long, 2> { static constexpr int RY = 2; };

template <class T, int K, class Mask, int RY = Cfg3D<T, K>::RY>
cudaError_t st3d(const Engine3DArgs<T>& a, cudaStream_t s) {
  constexpr int M = 2 * K + 1;
  return launch_ssam3d<T, Lanes<T>::Q, K, Mask, RY, M * M * M>(a, s);
}

template <class T, bool SHAPES>
cudaError_t stencil3d_dispatch(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                               int z_end, const StencilDesc<T>& st, cudaStream_t s) {
  const int k = st.order;
  // int64 (tests only) keeps the register engine to order 1; larger int64
  // footprints would spill, so they take the direct kernel.
  if (k > 2 || (!SHAPES && k > 1))
    return stencil3d_direct<T>(d_in, d_out, nx, ny, nz, z_begin, z_end, st, s);
  const std::vector<T> coef = dense3d_coef(st);
  Engine3DArgs<T> a{d_in, d_out, nx, ny, nz, k, coef.data(), z_begin, z_end};
  if constexpr (SHAPES) {
    const Shape3D sh = classify3d(st.taps, k);
    if (k == 1 && sh == Shape3D::star) return st3d<T, 1, StarMask3<1>>(a, s);
    if (k == 2 && sh == Shape3D::star) return st3d<T, 2, StarMask3<2>>(a, s);
    if (k == 1 && sh == Shape3D::poisson) return st3d<T, 1, PoissonMask3>(a, s);
    // box K=1 (3d27pt) and box K=2 (3d125pt) are the dense kernels.
  }
  switch (k) {
    case 0: return st3d<T, 0, DenseMask3>(a, s);
    case 1: return st3d<T, 1, DenseMask3>(a, s);
  }
  if constexpr (SHAPES) {
    if (k == 2) return st3d<T, 2, DenseMask3, 1>(a, s);  // 125 taps: one row per warp
  }
  return cudaErrorInvalidValue;
}

template <>
cudaError_t stencil3d_sweep<float>(const float* i, float* o, int nx, int ny, int nz, int zb,
                                   int ze, const StencilDesc<float>& st, cudaStream_t s) {
  return stencil3d_dispatch<float, true>(i, o, nx, ny, nz, zb, ze, st, s);
}
template <>
cudaError_t stencil3d_sweep<double>(const double* i, double* o, int nx, int ny, int nz, int zb,
                                    int ze, const StencilDesc<double>& st, cudaStream_t s) {
  return stencil3d_dispatch<double, true>(i, o, nx, ny, nz, zb, ze, st, s);
}
template <>
cudaError_t stencil3d_sweep<long long>(const long long* i, long long* o, int nx, int ny, int nz,
                                       int zb, int ze, const StencilDesc<long long>& st,
                                       cudaStream_t s) {
  return stencil3d_dispatch<long long, false>(i, o, nx, ny, nz, zb, ze, st, s);
}

}  // namespace ssam_b200
