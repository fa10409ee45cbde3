// pipe3d_box.cu -- the order-1 box family (3d27pt, Poisson 3d19pt) on the
// pipeline engine: column partials of dx = -1 / 0 / +1 joined by one shfl_up
// and one shfl_down per row (the paper's systolic shift).
#include "pipe3d_launch.cuh"

namespace ssam_b200 {

template <class T, class Mask>
cudaError_t pipe3d_box_m(const T* i, T* o, int nx, int ny, int nz, int zb, int ze, int rlo, int rhi,
                         const T* coef, int tb, cudaStream_t s) {
  using Sh = PipeBox<Mask>;
  switch (tb) {
    case 1: return pipe3d_sweep_sh<T, Sh>(i, o, nx, ny, nz, zb, ze, coef, s);
    case 2: return launch_pipe3d<T, Sh, 2>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, s);
  }
  return cudaErrorNotSupported;
}

template <class T>
cudaError_t pipe3d_box(bool poisson, const T* i, T* o, int nx, int ny, int nz, int zb, int ze,
                       int rlo, int rhi, const T* coef, int tb, cudaStream_t s) {
  return poisson ? pipe3d_box_m<T, PoissonMask3>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, tb, s)
                 : pipe3d_box_m<T, DenseMask3>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, tb, s);
}
template cudaError_t pipe3d_box<float>(bool, const float*, float*, int, int, int, int, int, int, int, const float*, int, cudaStream_t);
template cudaError_t pipe3d_box<double>(bool, const double*, double*, int, int, int, int, int, int, int, const double*, int, cudaStream_t);

}  // namespace ssam_b200
