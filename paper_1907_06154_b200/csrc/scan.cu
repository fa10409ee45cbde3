// scan.cu -- inclusive prefix sum (ssam::scan, proj/include/ssam/kernels.hpp:420-447).
//
// The reference scans lane_count-sized tiles with the Kogge-Stone warp plan
// (plan.hpp:196-218: log2(S) shfl_up stages, lanes below the shift distance
// keep their value) and carries each tile's last element into the next on
// the host.  Its result is the plain inclusive prefix sum of the input
// (oracle::scan_naive, oracle.hpp:118-127) -- exact for int64, the only type
// its tests scan.
//
// B200 shape: an L2-chunked reduce-then-scan over 32 KiB tiles (256 threads x
// rows of 4 elements per lane), one launch ("step") per chunk of CHUNK = 384
// tiles (12 MiB of input).  Step c scans chunk c -- reduced by step c-1, so
// its second read hits L2 -- and reduces chunk c+1.  HBM traffic is 2 x n
// element moves (a 3-pass reduce/carry/scan moves 3 x n).
//   * reduce blocks sum a tile of chunk c+1 into sums[] (input loads marked
//     L2 evict_last: they are read again next step);
//   * scan blocks scan their tile in registers, then form its exclusive
//     prefix themselves: carry[c] + the chunk's earlier tile sums, in a fixed
//     thread / tree order; block 0 also writes carry[c+1] = carry[c] +
//     total(c).  Their loads and stores are marked evict_first.
// Steps 0.. are programmatic-dependent launches with the reduce blocks first:
// those read only the input, so they start while step c-1 drains; the scan
// blocks griddep_wait for it.  Within a tile every warp owns rows of 32 x 4
// elements (coalesced 512-byte / 1 KiB loads and stores); per row each lane
// scans its 4 elements serially and the 32 lane totals run the same
// Kogge-Stone shfl_up ladder the reference simulates (5 shuffles).  Every
// association is fixed, so every run is bit-identical (a decoupled look-back
// would make floating-point results depend on timing).  A/B against the
// 3-pass form, plain launches, ready flags, a bulk-copy step and one
// persistent kernel:
// profiles/r02/scan_chunk_ab.txt.
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "internal.hpp"
#include "launch.cuh"

namespace ssam_b200 {

namespace {

constexpr int kScanThreads = 256;
// Tiles per L2 chunk, 12 MiB (profiles/r02/scan_chunk_ab.txt: 296..2048 tiles
// span 0.494..0.403 ms for fp32 at 2^28, the minimum at 384; fp64 with 256-bit
// accesses 0.813 ms at 384, 0.865 at 512).
#ifndef SSAM_SCAN_CHUNK
#define SSAM_SCAN_CHUNK 384
#endif
#ifndef SSAM_SCAN_V256
#define SSAM_SCAN_V256 1
#endif
#ifndef SSAM_SCAN_HINTS
#define SSAM_SCAN_HINTS 1
#endif

// Each lane owns VQ = 4 consecutive elements per row (one 16-byte access for
// fp32, one 256-bit access for 64-bit types), so the 5-step shuffle ladder is
// paid per 4 elements.  Measured: 64-bit VQ 2 / 8 lose (3-pass form and the
// chunked one), fp32 VQ 8 (256-bit) is within 1%.
#ifndef SSAM_SCAN_VQ32
#define SSAM_SCAN_VQ32 4
#endif
#ifndef SSAM_SCAN_VQ64
#define SSAM_SCAN_VQ64 4
#endif
template <class T>
struct ScanTile {
  static constexpr int VQ = sizeof(T) == 4 ? SSAM_SCAN_VQ32 : SSAM_SCAN_VQ64;
  static constexpr int ROWS = 128 / (VQ * sizeof(T));  // 32 KiB tiles
  static constexpr int TILE = kScanThreads * ROWS * VQ;
  static constexpr int CHUNK = SSAM_SCAN_CHUNK;
  // base-address alignment the vector path needs (256-bit for 64-bit types)
  static constexpr uintptr_t ALIGN = (sizeof(T) * VQ == 32 && SSAM_SCAN_V256) ? 31 : 15;
};

__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// A lane's Q elements with an L2 eviction-priority hint: one 256-bit access
// when they span 32 bytes (64-bit types, Q = 4: a warp row is one fully
// coalesced 1 KiB request instead of two half-used 16-byte ones), else
// 16-byte chunks.
template <class T, int Q>
__device__ __forceinline__ void ldg_q_hint(const T* __restrict__ p, T (&out)[Q], uint64_t pol) {
  if constexpr (sizeof(T) * Q == 32 && SSAM_SCAN_V256) {
    unsigned long long r[4];
    asm volatile("ld.global.nc.L2::cache_hint.v4.b64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3])
                 : "l"(p), "l"(pol));
    memcpy(out, r, 32);
  } else {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int c = 0; c < Q / V; ++c) {
      int4 r;
      asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                   : "l"(p + c * V), "l"(pol));
      T tmp[V];
      memcpy(tmp, &r, 16);
#pragma unroll
      for (int q = 0; q < V; ++q) out[c * V + q] = tmp[q];
    }
  }
}
template <class T, int Q>
__device__ __forceinline__ void st_q_hint(T* p, const T (&in)[Q], uint64_t pol) {
  if constexpr (sizeof(T) * Q == 32 && SSAM_SCAN_V256) {
    unsigned long long r[4];
    memcpy(r, in, 32);
    asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "l"(r[0]),
                 "l"(r[1]), "l"(r[2]), "l"(r[3]), "l"(pol)
                 : "memory");
  } else {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int c = 0; c < Q / V; ++c) {
      int4 r;
      memcpy(&r, in + c * V, 16);
      asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p + c * V),
                   "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "l"(pol)
                   : "memory");
    }
  }
}

// Loads warp `wid`'s rows of tile `tile` (zeros past n) with L2 policy
// `pol`; returns whether the tile is whole and 16-byte aligned (vector path).
template <class T>
__device__ __forceinline__ bool load_rows(const T* __restrict__ in, size_t n, size_t tile,
                                          int wid, int lane,
                                          T (&v)[ScanTile<T>::ROWS][ScanTile<T>::VQ],
                                          size_t& wbase, uint64_t pol) {
  constexpr int VQ = ScanTile<T>::VQ, ROWS = ScanTile<T>::ROWS, TILE = ScanTile<T>::TILE;
  wbase = tile * TILE + static_cast<size_t>(wid) * ROWS * 32 * VQ;
  const bool full =
      (tile + 1) * TILE <= n && (reinterpret_cast<uintptr_t>(in) & ScanTile<T>::ALIGN) == 0;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const size_t at = wbase + static_cast<size_t>(r) * 32 * VQ + lane * VQ;
    if (full) {
#if SSAM_SCAN_HINTS
      ldg_q_hint<T, VQ>(in + at, v[r], pol);
#else
      ldg_q<T, VQ>(in + at, v[r]);
#endif
    } else {
#pragma unroll
      for (int q = 0; q < VQ; ++q) v[r][q] = at + q < n ? in[at + q] : T(0);
    }
  }
  return full;
}

// Fixed-order sum of s[0 .. cnt) over the block (every thread gets it).
template <class T>
__device__ __forceinline__ T block_sum_prefix(const T* __restrict__ s, int cnt, T* s_red,
                                              int lane, int wid) {
  constexpr int NW = kScanThreads / 32;
  T acc = T(0);
  for (int j = threadIdx.x; j < cnt; j += kScanThreads) acc += __ldcg(s + j);  // written this grid
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(kFull, acc, off);
  if (lane == 0) s_red[wid] = acc;
  __syncthreads();
  T t = T(0);
#pragma unroll
  for (int w = 0; w < NW; ++w) t += s_red[w];
  return t;
}

// Step c (c = -1 .. chunks-1): blocks [0, rc) reduce chunk c+1, blocks
// [rc, gridDim.x) scan chunk c.
// 4 CTAs per SM (<= 64 registers): the step is latency-bound, and 93-108
// registers (3 CTAs) cost 25-30%, 5 CTAs spill (profiles/r02/scan_chunk_ab.txt).
template <class T>
__global__ void __launch_bounds__(kScanThreads, 4)
    scan_step_kernel(const T* __restrict__ in, T* __restrict__ out, size_t n,
                     T* __restrict__ sums, T* __restrict__ carry, int c, int rc, int last_chunk) {
  constexpr int VQ = ScanTile<T>::VQ, ROWS = ScanTile<T>::ROWS, NW = kScanThreads / 32;
  __shared__ T s_warp[NW];
  __shared__ T s_red[NW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T v[ROWS][VQ];
  size_t wbase;
  griddep_launch();  // step c+1's reduce blocks may fill SMs as this grid drains
  if (static_cast<int>(blockIdx.x) < rc) {  // reduce a tile of chunk c+1
    const int b = blockIdx.x;
    const size_t tile = static_cast<size_t>(c + 1) * ScanTile<T>::CHUNK + b;
    load_rows<T>(in, n, tile, wid, lane, v, wbase, l2_policy_last());
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
      for (int w = 0; w < NW; ++w) t += s_warp[w];
      sums[tile] = t;
      if (c < 0 && b == 0) carry[0] = T(0);
    }
    return;
  }
  // scan tile b of chunk c
  const int b = blockIdx.x - rc, sc = gridDim.x - rc;
  const size_t tile = static_cast<size_t>(c) * ScanTile<T>::CHUNK + b;
  const uint64_t pol_first = l2_policy_first();
  const bool full = load_rows<T>(in, n, tile, wid, lane, v, wbase, pol_first) &&
                    (reinterpret_cast<uintptr_t>(out) & ScanTile<T>::ALIGN) == 0;
  T run = T(0);  // running total of the warp's earlier rows
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
    ex += run;
#pragma unroll
    for (int q = 0; q < VQ; ++q) v[r][q] += ex;
    run += __shfl_sync(kFull, t, 31);
  }
  if (lane == 0) s_warp[wid] = run;
  griddep_wait();  // step c-1 (sums of chunk c, carry[c]) complete
  const T* cs = sums + static_cast<size_t>(c) * ScanTile<T>::CHUNK;
  const T cin = __ldcg(carry + c);
  const T pre = cin + block_sum_prefix<T>(cs, b, s_red, lane, wid);  // syncs s_warp too
  if (b == 0 && c < last_chunk) {
    __syncthreads();  // s_red reuse
    const T tot = block_sum_prefix<T>(cs, sc, s_red, lane, wid);
    if (threadIdx.x == 0) carry[c + 1] = cin + tot;
  }
  T add = pre;
  for (int w = 0; w < wid; ++w) add += s_warp[w];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const size_t at = wbase + static_cast<size_t>(r) * 32 * VQ + lane * VQ;
#pragma unroll
    for (int q = 0; q < VQ; ++q) v[r][q] += add;
    if (full) {
#if SSAM_SCAN_HINTS
      st_q_hint<T, VQ>(out + at, v[r], pol_first);
#else
      st_q<T, VQ>(out + at, v[r]);
#endif
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
  const size_t chunks = (tiles + ScanTile<T>::CHUNK - 1) / ScanTile<T>::CHUNK;
  T* scratch = nullptr;  // tile sums, then the chunk carries (stream-ordered pool)
  cudaError_t e = engine_alloc(reinterpret_cast<void**>(&scratch),
                               (tiles + chunks) * sizeof(T), s);
  if (e != cudaSuccess) return e;
  T* carry = scratch + tiles;
  const int last = static_cast<int>(chunks) - 1;
  constexpr size_t CH = ScanTile<T>::CHUNK;
  auto count = [&](long long c) -> unsigned {
    if (c < 0 || c > last) return 0u;
    return static_cast<unsigned>(std::min<size_t>(CH, tiles - c * CH));
  };
  for (int c = -1; c <= last && e == cudaSuccess; ++c) {
    const unsigned sc = count(c), rc = count(c + 1);
    if (c < 0) {  // an ordinary launch: orders the chain after d_in's producer
      scan_step_kernel<T><<<rc, kScanThreads, 0, s>>>(d_in, d_out, n, scratch, carry, c,
                                                       static_cast<int>(rc), last);
    } else {
      e = launch_pdl(scan_step_kernel<T>, dim3(sc + rc), dim3(kScanThreads), 0, s, d_in, d_out,
                     n, scratch, carry, c, static_cast<int>(rc), last);
    }
    note_launch();
  }
  if (e == cudaSuccess) e = cudaGetLastError();
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
