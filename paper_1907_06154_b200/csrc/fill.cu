// fill.cu -- device-side synthetic inputs and on-device error metrics.
//
// fill_random: SplitMix64 is index-addressable -- draw i of a stream seeded
// with S is mix(S + (i+1)*gamma) (rng.hpp:15-20) -- so every thread computes
// its own element and the device grid is bit-identical to the reference's
// random_grid2d/3d (grid.hpp:52-66) without a host copy.  Needed for the
// 2048^2 x 512N slabs, which do not fit in host RAM at N = 8.
//
// max_rel_err: max |a-b| / max(1,|b|) (acceptance.cpp:35-44), reduced on the
// device for full-size self-consistency checks.
#include <cmath>

#include "common.cuh"
#include "internal.hpp"

namespace ssam_b200 {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <class T>
__device__ __forceinline__ T draw(unsigned long long z);
template <>
__device__ __forceinline__ double draw<double>(unsigned long long z) {
  return static_cast<double>(z >> 11) * 0x1.0p-52 - 1.0;
}
template <>
__device__ __forceinline__ float draw<float>(unsigned long long z) {
  return static_cast<float>(draw<double>(z));  // round-to-nearest, like static_cast<float>
}
template <>
__device__ __forceinline__ long long draw<long long>(unsigned long long z) {
  return -100 + static_cast<long long>(z % 201ULL);
}

template <class T>
__global__ void fill_kernel(T* __restrict__ out, size_t count, unsigned long long seed,
                            unsigned long long first) {
  const unsigned long long gamma = 0x9e3779b97f4a7c15ULL;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = draw<T>(mix64(seed + (first + i + 1) * gamma));
}

cudaError_t fill_random(int dtype, void* d, size_t count, uint64_t seed, uint64_t first,
                        cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 32));
  switch (dtype) {
    case 0: fill_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float*>(d), count, seed, first); break;
    case 1: fill_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(d), count, seed, first); break;
    case 2: fill_kernel<long long><<<blocks, 256, 0, s>>>(static_cast<long long*>(d), count, seed, first); break;
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

template <class T>
__global__ void max_err_kernel(const T* __restrict__ a, const T* __restrict__ b, size_t count,
                               unsigned long long* out /* [rel_bits, abs_bits] */) {
  double rel = 0.0, ab = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double got = static_cast<double>(a[i]), want = static_cast<double>(b[i]);
    double d = fabs(got - want);
    if (isnan(d)) d = INFINITY;
    ab = fmax(ab, d);
    rel = fmax(rel, d / fmax(1.0, fabs(want)));
  }
  for (int o = 16; o > 0; o >>= 1) {
    rel = fmax(rel, __shfl_xor_sync(kFull, rel, o));
    ab = fmax(ab, __shfl_xor_sync(kFull, ab, o));
  }
  if ((threadIdx.x & 31) == 0) {
    // non-negative doubles order like their bit patterns
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(rel)));
    atomicMax(out + 1, static_cast<unsigned long long>(__double_as_longlong(ab)));
  }
}

cudaError_t max_rel_err(int dtype, const void* d_a, const void* d_b, size_t count, double* h_rel,
                        double* h_abs, cudaStream_t s) {
  unsigned long long* d_out = nullptr;
  cudaError_t e = engine_alloc(reinterpret_cast<void**>(&d_out), 16, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(d_out, 0, 16, s);
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256 + 1, 148 * 16));
  switch (dtype) {
    case 0: max_err_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(d_a), static_cast<const float*>(d_b), count, d_out); break;
    case 1: max_err_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(d_a), static_cast<const double*>(d_b), count, d_out); break;
    case 2: max_err_kernel<long long><<<blocks, 256, 0, s>>>(static_cast<const long long*>(d_a), static_cast<const long long*>(d_b), count, d_out); break;
    default: cudaFreeAsync(d_out, s); return cudaErrorInvalidValue;
  }
  note_launch();
  unsigned long long h[2] = {0, 0};
  e = cudaMemcpyAsync(h, d_out, 16, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_out, s);
  if (e != cudaSuccess) return e;
  double r, a;
  memcpy(&r, &h[0], 8);
  memcpy(&a, &h[1], 8);
  *h_rel = r;
  *h_abs = a;
  return cudaGetLastError();
}

}  // namespace ssam_b200
