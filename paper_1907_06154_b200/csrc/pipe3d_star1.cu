// pipe3d_star1.cu -- the order-1 star (3d7pt) on the pipeline engine:
// single sweeps and TB = 2..4 fused sweeps (engine3d_pipe.cuh).
#include "pipe3d_launch.cuh"

namespace ssam_b200 {

template <class T>
cudaError_t pipe3d_star1(const T* i, T* o, int nx, int ny, int nz, int zb, int ze, int rlo, int rhi,
                         const T* coef, int tb, cudaStream_t s) {
  using Sh = PipeStar<1>;
  switch (tb) {
    case 1: return pipe3d_sweep_sh<T, Sh>(i, o, nx, ny, nz, zb, ze, coef, s);
    case 2: return launch_pipe3d<T, Sh, 2>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, s);
    case 3: return launch_pipe3d<T, Sh, 3>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, s);
    case 4: return launch_pipe3d<T, Sh, 4>(i, o, nx, ny, nz, zb, ze, rlo, rhi, coef, s);
  }
  return cudaErrorNotSupported;
}
template cudaError_t pipe3d_star1<float>(const float*, float*, int, int, int, int, int, int, int, const float*, int, cudaStream_t);
template cudaError_t pipe3d_star1<double>(const double*, double*, int, int, int, int, int, int, int, const double*, int, cudaStream_t);

}  // namespace ssam_b200
