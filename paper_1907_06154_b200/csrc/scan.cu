// scan.cu -- inclusive prefix sum (ssam::scan, proj/include/ssam/kernels.hpp:420-447).
//
// The reference scans lane_count-sized tiles with the Kogge-Stone warp plan
// (plan.hpp:196-218: log2(S) shfl_up stages, lanes below the shift distance
// keep their value) and carries each tile's last element into the next on
// the host.  Its result is the plain inclusive prefix sum of the input
// (oracle::scan_naive, oracle.hpp:118-127) -- exact for int64, the only type
// its tests scan.
//
// B200 shape: reduce-then-scan over 32 KiB tiles (256 threads x rows of 4
// elements per lane).
//   1. scan_reduce_kernel: one CTA per tile sums it (read n).
//   2. scan_carry_kernel: one CTA turns the tile sums into exclusive tile
//      prefixes (32 serial sums per thread, one block ladder per 32 K tiles).
//   3. scan_tile_kernel: one CTA per tile scans it from its prefix (read n,
//      write n).
// Within a tile every warp owns rows of 32 x 4 elements (coalesced 512-byte /
// 1 KiB loads and stores); per row each lane scans its 4 elements serially and the
// 32 lane totals run the same Kogge-Stone shfl_up ladder the reference
// simulates (5 shuffles), warp totals one more ladder.  A single-pass
// decoupled look-back (measured here at 2.0-2.5 TB/s on B200: the
// inclusive-prefix chain across ~600 co-resident tiles, not HBM, bound it)
// would also make floating-point results depend on timing; this order is
// fixed, so every run is bit-identical.  Traffic is 3 x n element moves
// against the 2 x n minimum.
#include <cstdint>

#include "common.cuh"
#include "internal.hpp"

namespace ssam_b200 {

namespace {

constexpr int kScanThreads = 256;
constexpr int kCarryThreads = 1024;

// Each lane owns VQ = 4 consecutive elements per row (one 16-byte load for
// fp32, two for 64-bit types), so the 5-step shuffle ladder is paid per 4
// elements.  64-bit at 2^28: 2 per lane 2917 GB/s, 4 per lane 3921 (fp64) /
// 3885 (int64), 8 per lane 3799 / 3930.
#ifndef SSAM_SCAN_VQ64
#define SSAM_SCAN_VQ64 4
#endif
template <class T>
struct ScanTile {
  static constexpr int VQ = sizeof(T) == 4 ? 4 : SSAM_SCAN_VQ64;
  static constexpr int ROWS = sizeof(T) == 4 ? 8 : 16 / VQ;  // 32 KiB tiles
  static constexpr int TILE = kScanThreads * ROWS * VQ;
};

// Loads warp `wid`'s rows of tile `tile` (zeros past n); returns whether the
// tile is whole and 16-byte aligned (vector path).
template <class T>
__device__ __forceinline__ bool load_rows(const T* __restrict__ in, size_t n, int tile, int wid,
                                          int lane, T (&v)[ScanTile<T>::ROWS][ScanTile<T>::VQ],
                                          size_t& wbase) {
  constexpr int VQ = ScanTile<T>::VQ, ROWS = ScanTile<T>::ROWS, TILE = ScanTile<T>::TILE;
  wbase = static_cast<size_t>(tile) * TILE + static_cast<size_t>(wid) * ROWS * 32 * VQ;
  const bool full = static_cast<size_t>(tile + 1) * TILE <= n &&
                    (reinterpret_cast<uintptr_t>(in) & 15) == 0;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const size_t at = wbase + static_cast<size_t>(r) * 32 * VQ + lane * VQ;
    if (full) {
      ldg_q<T, VQ>(in + at, v[r]);
    } else {
#pragma unroll
      for (int q = 0; q < VQ; ++q) v[r][q] = at + q < n ? in[at + q] : T(0);
    }
  }
  return full;
}

template <class T>
__global__ void __launch_bounds__(kScanThreads)
    scan_reduce_kernel(const T* __restrict__ in, size_t n, T* __restrict__ tile_sum) {
  constexpr int VQ = ScanTile<T>::VQ, ROWS = ScanTile<T>::ROWS;
  __shared__ T s_warp[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T v[ROWS][VQ];
  size_t wbase;
  load_rows<T>(in, n, blockIdx.x, wid, lane, v, wbase);
  T x = T(0);
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int q = 0; q < VQ; ++q) x += v[r][q];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(kFull, x, off);
  if (lane == 0) s_warp[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = T(0);
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) t += s_warp[w];
    tile_sum[blockIdx.x] = t;
  }
}

// Exclusive prefix of the tile sums: each of the 1024 threads scans
// kCarryItems consecutive sums serially, one block-wide ladder joins the
// thread totals, and a running carry links chunks of 1024 * kCarryItems sums
// (16 items for 64-bit types keeps them in registers).
template <class T>
constexpr int carry_items() { return sizeof(T) == 4 ? 32 : 16; }

template <class T>
__global__ void __launch_bounds__(kCarryThreads)
    scan_carry_kernel(const T* __restrict__ tile_sum, T* __restrict__ tile_prefix, int tiles) {
  __shared__ T s_warp[kCarryThreads / 32];
  __shared__ T s_carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = T(0);
  __syncthreads();
  constexpr int kCarryItems = carry_items<T>();
  for (long long base = 0; base < tiles; base += static_cast<long long>(kCarryThreads) * kCarryItems) {
    const long long i0 = base + static_cast<long long>(threadIdx.x) * kCarryItems;
    T v[kCarryItems];
    T run = T(0);
#pragma unroll
    for (int k = 0; k < kCarryItems; ++k) {
      v[k] = run;  // exclusive within the thread
      run += i0 + k < tiles ? tile_sum[i0 + k] : T(0);
    }
    T t = run;
#pragma unroll
    for (int d = 1; d < 32; d *= 2) {
      const T u = __shfl_up_sync(kFull, t, d);
      if (lane >= d) t += u;
    }
    if (lane == 31) s_warp[wid] = t;
    __syncthreads();
    if (wid == 0) {
      T w = s_warp[lane];
#pragma unroll
      for (int d = 1; d < 32; d *= 2) {
        const T u = __shfl_up_sync(kFull, w, d);
        if (lane >= d) w += u;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    T ex = __shfl_up_sync(kFull, t, 1);
    if (lane == 0) ex = T(0);
    const T pre = s_carry + ((wid > 0 ? s_warp[wid - 1] : T(0)) + ex);
#pragma unroll
    for (int k = 0; k < kCarryItems; ++k)
      if (i0 + k < tiles) tile_prefix[i0 + k] = pre + v[k];
    __syncthreads();
    if (threadIdx.x == kCarryThreads - 1) s_carry = pre + run;
    __syncthreads();
  }
}

template <class T>
__global__ void __launch_bounds__(kScanThreads)
    scan_tile_kernel(const T* __restrict__ in, T* __restrict__ out, size_t n,
                     const T* __restrict__ tile_prefix) {
  constexpr int VQ = ScanTile<T>::VQ, ROWS = ScanTile<T>::ROWS, NW = kScanThreads / 32;
  __shared__ T s_warp[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T v[ROWS][VQ];
  size_t wbase;
  const bool full = load_rows<T>(in, n, blockIdx.x, wid, lane, v, wbase) &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  T carry = T(0);  // running total of the warp's earlier rows
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
#pragma unroll
    for (int q = 1; q < VQ; ++q) v[r][q] += v[r][q - 1];
    T t = v[r][VQ - 1];
#pragma unroll
    for (int d = 1; d < 32; d *= 2) {
      const T u = __shfl_up_sync(kFull, t, d);
      if (lane >= d) t += u;
    }
    T ex = __shfl_up_sync(kFull, t, 1);  // exclusive lane prefix within the row
    if (lane == 0) ex = T(0);
    ex += carry;
#pragma unroll
    for (int q = 0; q < VQ; ++q) v[r][q] += ex;
    carry += __shfl_sync(kFull, t, 31);
  }
  if (lane == 0) s_warp[wid] = carry;
  __syncthreads();
  T add = tile_prefix[blockIdx.x];
  for (int w = 0; w < wid; ++w) add += s_warp[w];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const size_t at = wbase + static_cast<size_t>(r) * 32 * VQ + lane * VQ;
#pragma unroll
    for (int q = 0; q < VQ; ++q) v[r][q] += add;
    if (full) {
      st_q<T, VQ>(out + at, v[r]);
    } else {
#pragma unroll
      for (int q = 0; q < VQ; ++q)
        if (at + q < n) out[at + q] = v[r][q];
    }
  }
}

template <class T>
cudaError_t scan_impl(const T* d_in, T* d_out, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  constexpr size_t TILE = ScanTile<T>::TILE;
  const size_t tiles = (n + TILE - 1) / TILE;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  T* scratch = nullptr;  // tile sums, then tile prefixes (stream-ordered pool)
  cudaError_t e = engine_alloc(reinterpret_cast<void**>(&scratch), 2 * tiles * sizeof(T), s);
  if (e != cudaSuccess) return e;
  const unsigned g = static_cast<unsigned>(tiles);
  scan_reduce_kernel<T><<<g, kScanThreads, 0, s>>>(d_in, n, scratch);
  scan_carry_kernel<T><<<1, kCarryThreads, 0, s>>>(scratch, scratch + tiles,
                                                    static_cast<int>(tiles));
  scan_tile_kernel<T><<<g, kScanThreads, 0, s>>>(d_in, d_out, n, scratch + tiles);
  for (int k = 0; k < 3; ++k) note_launch();
  e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e;
}

}  // namespace

template <>
cudaError_t scan_device<float>(const float* i, float* o, size_t n, cudaStream_t s) {
  return scan_impl<float>(i, o, n, s);
}
template <>
cudaError_t scan_device<double>(const double* i, double* o, size_t n, cudaStream_t s) {
  return scan_impl<double>(i, o, n, s);
}
template <>
cudaError_t scan_device<long long>(const long long* i, long long* o, size_t n, cudaStream_t s) {
  return scan_impl<long long>(i, o, n, s);
}

}  // namespace ssam_b200
