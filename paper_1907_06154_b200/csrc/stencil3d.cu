// stencil3d.cu -- one 3D Jacobi sweep on the z-streaming SSAM engine.
//
// Reference: ssam::stencil3d, proj/include/ssam/kernels.hpp:283-384 (per-dz
// plane plans summed through InterWarpBuffer).  Shapes with a compile-time
// mask: 3d7pt (star K=1), 3d13pt (star K=2), 3d27pt (box K=1), poisson
// (3x3x3 minus corners); any other tap set of order <= 2 runs the dense
// engine with zero cells, larger orders the direct-gather kernel.
#include "engine3d.cuh"
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
// fp32 order 2 (3d13pt, halo-lane kernel): RY = 4 measured +5% at 512^3 and
// +13% at 2048^2 over RY = 2 (255 registers, no spills).
template <> struct Cfg3D<float, 2> { static constexpr int RY = 4; };
template <> struct Cfg3D<double, 0> { static constexpr int RY = 4; };
template <> struct Cfg3D<double, 1> { static constexpr int RY = 4; };
template <> struct Cfg3D<double, 2> { static constexpr int RY = 2; };
template <> struct Cfg3D<long long, 0> { static constexpr int RY = 4; };
template <> struct Cfg3D<long long, 1> { static constexpr int RY = 4; };
template <> struct Cfg3D<long long, 2> { static constexpr int RY = 2; };

// SSAM_B200_STAR1_HALO=0 sends 3d7pt single sweeps to the pipeline kernel (TB = 1).
inline bool star1_halo_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_STAR1_HALO");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

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
    if (pipe3d_enabled()) {  // the pipeline engine (engine3d_pipe.cuh)
      if (k == 1 && sh == Shape3D::star) {
        // single sweeps of the 7-point star: the halo-lane kernel runs the
        // pipeline's per-cell chain (bit-identical to the fused launches)
        // and streams faster at TB = 1 (profiles/r02/pipe_tb1_ab.txt:
        // 2048^2 x 514 f32 776 vs 635-665 GCells/s, f64 382 vs 322-335)
        constexpr int VQ = 16 / sizeof(T);
        if (star1_halo_enabled() && halo_mode_3d() != 0 && nx % VQ == 0 && aligned16(d_in) &&
            aligned16(d_out))
          return st3d<T, 1, StarMask3<1>>(a, s);
        return pipe3d_star1<T>(d_in, d_out, nx, ny, nz, z_begin, z_end, 1, nz - 1, coef.data(), 1, s);
      }
      if (k == 2 && sh == Shape3D::star)
        return pipe3d_star2<T>(d_in, d_out, nx, ny, nz, z_begin, z_end, 2, nz - 2, coef.data(), 1, s);
      if (k == 1)  // poisson, the 27-point box and any other order-1 tap set (dense)
        return pipe3d_box<T>(sh == Shape3D::poisson, d_in, d_out, nx, ny, nz, z_begin, z_end, 1,
                             nz - 1, coef.data(), 1, s);
    }
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

bool stencil3d_peer_fused(int dtype, int order) { return order <= (dtype == 2 ? 1 : 2); }

// ---- temporal blocking: the pipeline engine (engine3d_pipe.cuh) ---------------

// SSAM_B200_PIPE=0 routes single sweeps of every 3D shape back to the
// generic z-streaming engine (engine3d.cuh) for A/B runs, without fusion.
bool pipe3d_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_PIPE");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

// Fused depth per shape (B200, pipeline engine, GCells/s at 512^3, single
// sweep / Tb = 2; profiles/r02/pipe_shapes.txt): 3d7pt f32 660 / 996, f64
// 341 / 610; 3d13pt f32 614 / 643, f64 355 / 334; 3d27pt and poisson lose
// 30-50% fused (compute-bound, one CTA per SM).  SSAM_B200_3D_TB asks for a
// depth (clamped to the compiled ones).
int stencil3d_tb_max(int dtype, int order, Shape3D shape) {
  if (dtype == 2) return 1;
  const bool star1 = order == 1 && shape == Shape3D::star;
  const char* e = std::getenv("SSAM_B200_3D_TB");
  if (!pipe3d_enabled()) return 1;
  const int most = star1 ? 4 : (order == 1 || (order == 2 && shape == Shape3D::star)) ? 2 : 1;
  const bool star2 = order == 2 && shape == Shape3D::star;
  // (3d13pt: single sweeps with 8 planes in flight beat the fused pair at
  // 512^3, 656 vs 627-645 GCells/s f32; the fused pair runs one CTA per SM)
  (void)star2;
  const int want = e ? std::atoi(e) : (star1 ? 2 : 1);
  return std::max(1, std::min(want, most));
}

template <class T>
cudaError_t stencil3d_tb_impl(const T* d_in, T* d_out, int nx, int ny, int nz, int zb, int ze,
                              int rlo, int rhi, const StencilDesc<T>& st, int tb, cudaStream_t s) {
  if (tb < 2 || st.order < 1 || st.order > 2 || std::is_same<T, long long>::value)
    return cudaErrorNotSupported;
  const std::vector<T> coef = dense3d_coef(st);
  const Shape3D sh = classify3d(st.taps, st.order);
  if (!pipe3d_enabled()) return cudaErrorNotSupported;
  if (st.order == 2)
    return sh == Shape3D::star
               ? pipe3d_star2<T>(d_in, d_out, nx, ny, nz, zb, ze, rlo, rhi, coef.data(), tb, s)
               : cudaErrorNotSupported;
  return sh == Shape3D::star
             ? pipe3d_star1<T>(d_in, d_out, nx, ny, nz, zb, ze, rlo, rhi, coef.data(), tb, s)
             : pipe3d_box<T>(sh == Shape3D::poisson, d_in, d_out, nx, ny, nz, zb, ze, rlo, rhi,
                             coef.data(), tb, s);
}

template <>
cudaError_t stencil3d_tb<float>(const float* i, float* o, int nx, int ny, int nz, int zb, int ze,
                                int rlo, int rhi, const StencilDesc<float>& st, int tb,
                                cudaStream_t s) {
  return stencil3d_tb_impl<float>(i, o, nx, ny, nz, zb, ze, rlo, rhi, st, tb, s);
}
template <>
cudaError_t stencil3d_tb<double>(const double* i, double* o, int nx, int ny, int nz, int zb,
                                 int ze, int rlo, int rhi, const StencilDesc<double>& st, int tb,
                                 cudaStream_t s) {
  return stencil3d_tb_impl<double>(i, o, nx, ny, nz, zb, ze, rlo, rhi, st, tb, s);
}
template <>
cudaError_t stencil3d_tb<long long>(const long long*, long long*, int, int, int, int, int, int,
                                    int, const StencilDesc<long long>&, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace ssam_b200
