// direct.cu -- direct-gather kernels: the generic GPU path for tap sets the
// SSAM engines do not specialise (2D order > 6, 3D order > 2).
//
// One thread per output cell, taps read from a small device table in the
// oracle's order with the oracle's arithmetic: double accumulation for
// floating types using explicitly rounded mul/add (no FMA contraction) and
// native int64 otherwise -- oracle.hpp:44-116.  For f32/f64 this reproduces
// the oracle bit-for-bit; it is still a CUDA kernel, never a CPU fallback.
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace ssam_b200 {

template <class T> struct Acc { using type = double; };
template <> struct Acc<long long> { using type = long long; };

__device__ __forceinline__ double mac(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}
__device__ __forceinline__ long long mac(long long acc, long long a, long long b) {
  return acc + a * b;
}

template <class T>
__global__ void conv2d_direct_kernel(const T* __restrict__ in, T* __restrict__ out, int W, int H,
                                     const int* __restrict__ offs, const T* __restrict__ w,
                                     int ntaps, int boundary) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  typename Acc<T>::type sum = 0;
  for (int j = 0; j < ntaps; ++j) {
    int xx = x + offs[2 * j], yy = y + offs[2 * j + 1];
    T v;
    if (xx >= 0 && xx < W && yy >= 0 && yy < H) {
      v = in[static_cast<size_t>(yy) * W + xx];
    } else if (boundary == 0) {
      v = T(0);
    } else {
      v = in[static_cast<size_t>(clampi(yy, H)) * W + clampi(xx, W)];
    }
    sum = mac(sum, static_cast<typename Acc<T>::type>(v), static_cast<typename Acc<T>::type>(w[j]));
  }
  out[static_cast<size_t>(y) * W + x] = static_cast<T>(sum);
}

template <class T>
__global__ void stencil3d_direct_kernel(const T* __restrict__ in, T* __restrict__ out, int nx,
                                        int ny, int nz, int k, int z_begin,
                                        const int* __restrict__ offs, const T* __restrict__ c,
                                        int ntaps) {
  const int x = k + blockIdx.x * blockDim.x + threadIdx.x;
  const int y = k + blockIdx.y;
  const int z = z_begin + blockIdx.z;
  if (x >= nx - k) return;
  typename Acc<T>::type sum = 0;
  for (int j = 0; j < ntaps; ++j) {
    const size_t idx = (static_cast<size_t>(z + offs[3 * j + 2]) * ny + (y + offs[3 * j + 1])) * nx +
                       (x + offs[3 * j]);
    sum = mac(sum, static_cast<typename Acc<T>::type>(in[idx]),
              static_cast<typename Acc<T>::type>(c[j]));
  }
  out[(static_cast<size_t>(z) * ny + y) * nx + x] = static_cast<T>(sum);
}

namespace {

// Stream-ordered scratch for the tap tables.
template <class T>
cudaError_t upload_taps(const std::vector<int>& offs, const std::vector<T>& c, int** d_offs,
                        T** d_c, cudaStream_t s) {
  cudaError_t e = engine_alloc(reinterpret_cast<void**>(d_offs), offs.size() * sizeof(int), s);
  if (e != cudaSuccess) return e;
  e = engine_alloc(reinterpret_cast<void**>(d_c), c.size() * sizeof(T), s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(*d_offs, offs.data(), offs.size() * sizeof(int), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(*d_c, c.data(), c.size() * sizeof(T), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  // pageable sources: make sure the staging copies completed before the
  // host vectors go out of scope.
  return cudaStreamSynchronize(s);
}

}  // namespace

template <class T>
cudaError_t conv2d_direct(const T* d_in, T* d_out, int W, int H, const T* h_w, int m, int n,
                          int boundary, cudaStream_t s) {
  const int ax = (m - 1) / 2, ay = (n - 1) / 2;
  std::vector<int> offs;
  std::vector<T> w;
  for (int sx = 0; sx < m; ++sx)
    for (int t = 0; t < n; ++t) {
      offs.push_back(ax - sx);
      offs.push_back(ay - t);
      w.push_back(h_w[static_cast<size_t>(sx) * n + t]);
    }
  int* d_offs = nullptr;
  T* d_w = nullptr;
  cudaError_t e = upload_taps(offs, w, &d_offs, &d_w, s);
  if (e == cudaSuccess) {
    const dim3 grid((W + 127) / 128, H);
    conv2d_direct_kernel<T><<<grid, 128, 0, s>>>(d_in, d_out, W, H, d_offs, d_w, m * n, boundary);
    note_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_offs, s);
  cudaFreeAsync(d_w, s);
  return e;
}

template <class T>
cudaError_t stencil3d_direct(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                             int z_end, const StencilDesc<T>& st, cudaStream_t s) {
  const int k = st.order;
  const int zb = z_begin > k ? z_begin : k;
  const int ze = z_end < nz - k ? z_end : nz - k;
  if (ze <= zb || nx - 2 * k <= 0 || ny - 2 * k <= 0) return cudaSuccess;
  std::vector<int> offs;
  for (const Tap& t : st.taps) {
    offs.push_back(t.dx);
    offs.push_back(t.dy);
    offs.push_back(t.dz);
  }
  int* d_offs = nullptr;
  T* d_c = nullptr;
  cudaError_t e = upload_taps(offs, st.coeffs, &d_offs, &d_c, s);
  if (e == cudaSuccess) {
    const dim3 grid((nx - 2 * k + 127) / 128, ny - 2 * k, ze - zb);
    stencil3d_direct_kernel<T><<<grid, 128, 0, s>>>(d_in, d_out, nx, ny, nz, k, zb, d_offs, d_c,
                                                    static_cast<int>(st.taps.size()));
    note_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_offs, s);
  cudaFreeAsync(d_c, s);
  return e;
}

// A 2D stencil is the nz = 1 slice of the 3D direct kernel with dz = 0.
template <class T>
cudaError_t stencil2d_direct(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                             const StencilDesc<T>& st, cudaStream_t s) {
  const int k = st.order;
  y_begin = y_begin > k ? y_begin : k;
  y_end = y_end < H - k ? y_end : H - k;
  if (W - 2 * k <= 0 || y_end <= y_begin) return cudaSuccess;
  std::vector<int> offs;
  for (const Tap& t : st.taps) {
    offs.push_back(t.dx);
    offs.push_back(t.dy);
    offs.push_back(0);
  }
  int* d_offs = nullptr;
  T* d_c = nullptr;
  cudaError_t e = upload_taps(offs, st.coeffs, &d_offs, &d_c, s);
  if (e == cudaSuccess) {
    // The nz = 1 slice of the 3D kernel: rows start at y_begin (passed via
    // the ring argument's y origin by offsetting the input/output rows).
    const dim3 grid((W - 2 * k + 127) / 128, y_end - y_begin, 1);
    const size_t shift = static_cast<size_t>(y_begin - k) * W;
    stencil3d_direct_kernel<T><<<grid, 128, 0, s>>>(d_in + shift, d_out + shift, W, H, 1, k, 0,
                                                    d_offs, d_c,
                                                    static_cast<int>(st.taps.size()));
    note_launch();
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_offs, s);
  cudaFreeAsync(d_c, s);
  return e;
}

#define SSAM_DIRECT_INST(T)                                                                   \
  template cudaError_t conv2d_direct<T>(const T*, T*, int, int, const T*, int, int, int,      \
                                        cudaStream_t);                                        \
  template cudaError_t stencil2d_direct<T>(const T*, T*, int, int, int, int,                 \
                                           const StencilDesc<T>&, cudaStream_t);              \
  template cudaError_t stencil3d_direct<T>(const T*, T*, int, int, int, int, int,             \
                                           const StencilDesc<T>&, cudaStream_t);
SSAM_DIRECT_INST(float)
SSAM_DIRECT_INST(double)
SSAM_DIRECT_INST(long long)

}  // namespace ssam_b200
