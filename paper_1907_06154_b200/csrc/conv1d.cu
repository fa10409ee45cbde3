// conv1d.cu -- 1D convolution (ssam::conv1d, proj/include/ssam/kernels.hpp:390-418).
//
// The reference's 1D plan (plan.hpp:166-190) is the 2D window plan with one
// cache row: M broadcast-weight MAD stages with a one-lane shift between
// them.  A signal is therefore a one-row grid for the 2D SSAM engine
// (engine2d.cuh): each warp loads 32 x Q consecutive samples with 128-bit
// loads, runs the bidirectional shuffle chain over the M taps and stores
// its own Q outputs; consecutive warps overlap by the M-1 halo samples.
// The weights are flipped exactly as for conv2d (w[s] -> coef[M-1-s]), so
// out(i) = sum_s in(i + (m-1)/2 - s) * w[s] (oracle.hpp:61-73).  Filters up
// to the reference's lane_count cap (32 taps) run on the register engine.
#include "conv2d_impl.cuh"

namespace ssam_b200 {

namespace {

template <class T>
cudaError_t conv1d_impl(const T* d_in, T* d_out, int len, const T* h_w, int m, int boundary,
                        cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  if (m < 1 || m > 32) return cudaErrorInvalidValue;
  const std::vector<T> coef = conv_coef(h_w, m, 1);
  Engine2DArgs<T> a{d_in, d_out, len, 1, m, 1, coef.data(),
                    boundary ? kBndReplicate : kBndZero, 0, 0, 1};
  a.direct = true;
  return launch_ssam2d<T, Lanes<T>::Q, 1, 0, DenseMask, 1, 32>(a, s);
}

}  // namespace

template <>
cudaError_t conv1d_device<float>(const float* i, float* o, int len, const float* w, int m,
                                 int b, cudaStream_t s) {
  return conv1d_impl<float>(i, o, len, w, m, b, s);
}
template <>
cudaError_t conv1d_device<double>(const double* i, double* o, int len, const double* w, int m,
                                  int b, cudaStream_t s) {
  return conv1d_impl<double>(i, o, len, w, m, b, s);
}
template <>
cudaError_t conv1d_device<long long>(const long long* i, long long* o, int len,
                                     const long long* w, int m, int b, cudaStream_t s) {
  return conv1d_impl<long long>(i, o, len, w, m, b, s);
}

}  // namespace ssam_b200
