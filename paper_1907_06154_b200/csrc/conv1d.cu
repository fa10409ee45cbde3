// conv1d.cu -- 1D convolution (ssam::conv1d, proj/include/ssam/kernels.hpp:390-418).
//
// The reference's 1D plan (plan.hpp:166-190) is the 2D window plan with one
// cache row: M broadcast-weight MAD stages with a one-lane shift between
// them.  A signal is therefore a one-row grid for the 2D SSAM engine
// (engine2d.cuh): a warp walks CH consecutive windows of 32 x Q samples
// (256-bit loads), runs the bidirectional shuffle chain over the M taps and
// stores its own Q outputs per window; consecutive windows overlap by the
// M-1 halo samples.
// The weights are flipped exactly as for conv2d (w[s] -> coef[M-1-s]), so
// out(i) = sum_s in(i + (m-1)/2 - s) * w[s] (oracle.hpp:61-73).  Filters up
// to the reference's lane_count cap (32 taps) run on the register engine.
#include "conv2d_impl.cuh"

namespace ssam_b200 {

namespace {

// Samples per lane: 32 bytes (one 256-bit load, sm_100).  At 2^28, m = 9:
// fp32 Q 4 -> 8 0.375 -> 0.336 ms, fp64 Q 2 -> 4 0.811 -> 0.661 ms; m = 32
// 0.80 -> 0.51 / 2.36 -> 1.09 ms -- fewer shuffles per output and a smaller
// window overlap; bit-identical (profiles/r02/conv1d_q_ab.txt).
#ifndef SSAM_C1D_Q32
#define SSAM_C1D_Q32 8
#endif
#ifndef SSAM_C1D_Q64
#define SSAM_C1D_Q64 4
#endif
template <class T>
constexpr int c1d_q() { return sizeof(T) == 4 ? SSAM_C1D_Q32 : SSAM_C1D_Q64; }

// A lane's Q samples as one 256-bit load when they span 32 bytes.
template <class T, int Q>
__device__ __forceinline__ void ldg_q256(const T* __restrict__ p, T (&out)[Q]) {
  static_assert(sizeof(T) * Q == 32, "256-bit vectors only");
  unsigned long long r[4];
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3])
               : "l"(p));
  memcpy(out, r, 32);
}

// One warp per run of CH consecutive chunks of V outputs: every chunk is one
// 32 x Q window (256-bit loads; the M-1 overlap with the previous chunk hits
// L1), the bidirectional chain of engine2d.cuh, and the lane's own Q stores.
template <class T, int Q, int CH, int CAP>
__global__ void __launch_bounds__(128) conv1d_kernel(const __grid_constant__ Ssam2DParams<T, CAP> p) {
  const int lane = threadIdx.x & 31;
  const long long first = (static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) +
                           (threadIdx.x >> 5)) * CH;
#pragma unroll 2
  for (int c = 0; c < CH; ++c) {
    const long long strip = first + c;
    if (strip >= p.nstrips) return;
    const int x_out0 = static_cast<int>(strip) * p.V;
    const int col0 = x_out0 - p.A + Q * lane;
    const bool fast = p.vec_ok && x_out0 - p.A >= 0 && x_out0 - p.A + 32 * Q <= p.W;
    T buf[1][Q];
    if constexpr (sizeof(T) * Q == 32) {
      if (fast)
        ldg_q256<T, Q>(p.in + col0, buf[0]);
      else
        load_row<T, Q>(p.in, p.W, 1, 0, col0, false, p.bmode, buf[0]);
    } else {
      load_row<T, Q>(p.in, p.W, 1, 0, col0, fast, p.bmode, buf[0]);
    }
    T acc[Q];
    ssam_row<T, Q, 1, 0, DenseMask, 1, CAP>(buf, 0, p, acc);
    store_row<T, Q, CAP>(p, store_plan<T, Q, CAP>(p, x_out0, col0, p.vec_ok != 0), 0, acc);
  }
}

template <class T>
cudaError_t conv1d_impl(const T* d_in, T* d_out, int len, const T* h_w, int m, int boundary,
                        cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  if (m < 1 || m > 32) return cudaErrorInvalidValue;
  constexpr int Q = c1d_q<T>(), CH = 8, CAP = 32;
  const std::vector<T> coef = conv_coef(h_w, m, 1);
  Ssam2DParams<T, CAP> p;
  std::memset(&p, 0, sizeof(p));
  p.in = d_in;
  p.out = d_out;
  p.W = len;
  p.H = 1;
  p.M = m;
  const LanePlan lp = plan_lanes(m, Q);
  p.A = lp.A;
  p.V = lp.V;
  p.nstrips = (len + lp.V - 1) / lp.V;
  p.seg = 1;
  p.y_begin = 0;
  p.y_end = 1;
  p.bmode = boundary ? kBndReplicate : kBndZero;
  const uintptr_t amask = sizeof(T) * Q == 32 ? 31 : 15;  // 256-bit loads need 32 B
  p.vec_ok = (len % Q == 0) && (reinterpret_cast<uintptr_t>(d_in) & amask) == 0 &&
             aligned16(d_out);
  std::memcpy(p.coef, coef.data(), sizeof(T) * m);
  const long long warps = (p.nstrips + CH - 1) / CH;
  const unsigned blocks = static_cast<unsigned>((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
  conv1d_kernel<T, Q, CH, CAP><<<blocks, 32 * kWarpsPerBlock, 0, s>>>(p);
  note_launch();
  return cudaGetLastError();
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
