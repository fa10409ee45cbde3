// fp64 and int64 conv2d on the runtime-width SSAM engine (Q = 2: one 128-bit
// access per lane per row; 64-bit shuffles are two SHFL each).
#include "conv2d_impl.cuh"

namespace ssam_b200 {

template <>
cudaError_t conv2d_device<double>(const double* d_in, double* d_out, int W, int H, int yb, int ye,
                                  const double* h_w, int m, int n, int boundary, cudaStream_t s) {
  return conv2d_dispatch<double, Lanes<double>::Q, false>(d_in, d_out, W, H, yb, ye, h_w, m, n,
                                                          boundary, s);
}

template <>
cudaError_t conv2d_device<long long>(const long long* d_in, long long* d_out, int W, int H,
                                     int yb, int ye, const long long* h_w, int m, int n,
                                     int boundary, cudaStream_t s) {
  return conv2d_dispatch<long long, Lanes<long long>::Q, false>(d_in, d_out, W, H, yb, ye, h_w,
                                                                m, n, boundary, s);
}

}  // namespace ssam_b200
