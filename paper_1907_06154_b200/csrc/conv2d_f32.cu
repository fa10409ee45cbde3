// fp32 conv2d: fully unrolled square kernels (K = 1..20) + runtime-width engine.
#include "conv2d_impl.cuh"

namespace ssam_b200 {

template <>
cudaError_t conv2d_device<float>(const float* d_in, float* d_out, int W, int H, int yb, int ye,
                                 const float* h_w, int m, int n, int boundary,
                                 cudaStream_t s) {
  return conv2d_dispatch<float, Lanes<float>::Q, true>(d_in, d_out, W, H, yb, ye, h_w, m, n,
                                                       boundary, s);
}

}  // namespace ssam_b200
