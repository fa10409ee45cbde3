// scan.cu -- inclusive prefix sum (ssam::scan, proj/include/ssam/kernels.hpp:420-447).
//
// The reference scans lane_count-sized tiles with the Kogge-Stone warp plan
// (plan.hpp:196-218: log2(S) shfl_up stages, lanes below the shift distance
// keep their value) and carries each tile's last element into the next on
// the host.  Its result is the plain inclusive prefix sum of the input
// (oracle::scan_naive, oracle.hpp:118-127) -- exact for int64, the only type
// its tests scan.
//
// B200 shape: one pass over HBM (read once, write once).  A CTA of 256
// threads owns a tile of 256 x ITEMS elements (128 contiguous bytes per
// thread, 32 KiB per tile): each thread scans its ITEMS serially, the 32
// thread totals of a warp are combined by the same Kogge-Stone shfl_up
// ladder the reference simulates (5 shuffles), warp totals by one more
// ladder, and tiles are chained with decoupled look-back: every tile
// publishes its aggregate as soon as it is known and its inclusive prefix
// once its predecessor's is, so the grid never waits for a second pass.
// The look-back is warp-wide: 32 predecessors are inspected per step.
// Tile order is taken from an atomic ticket so a tile only ever waits on
// tiles that are already running.
#include <cstdint>

#include "common.cuh"
#include "internal.hpp"

namespace ssam_b200 {

namespace {

constexpr int kScanThreads = 256;

template <class T>
struct ScanState {
  int* ticket;      // next tile to hand out
  int* flag;        // per tile: 0 nothing, 1 aggregate, 2 inclusive prefix
  T* agg;
  T* incl;
};

template <class T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}

template <class T, int ITEMS>
__global__ void __launch_bounds__(kScanThreads)
    scan_kernel(const T* __restrict__ in, T* __restrict__ out, size_t n, ScanState<T> st) {
  constexpr int TILE = kScanThreads * ITEMS;
  constexpr int NW = kScanThreads / 32;
  __shared__ int s_tile;
  __shared__ T s_warp[NW];
  __shared__ T s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(st.ticket, 1);
  __syncthreads();
  const int tile = s_tile;
  const size_t base = static_cast<size_t>(tile) * TILE + static_cast<size_t>(tid) * ITEMS;

  // thread-serial inclusive scan of ITEMS contiguous elements
  T v[ITEMS];
  constexpr int VQ = 16 / sizeof(T);
  const bool full = base + ITEMS <= n && (reinterpret_cast<uintptr_t>(in + base) & 15) == 0;
  if (full) {
#pragma unroll
    for (int c = 0; c < ITEMS / VQ; ++c) {
      T tmp[VQ];
      ldg_q<T, VQ>(in + base + c * VQ, tmp);
#pragma unroll
      for (int q = 0; q < VQ; ++q) v[c * VQ + q] = tmp[q];
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) v[i] = base + i < n ? in[base + i] : T(0);
  }
#pragma unroll
  for (int i = 1; i < ITEMS; ++i) v[i] += v[i - 1];

  // Kogge-Stone over the warp's thread totals (shift 1, 2, 4, 8, 16)
  T t = v[ITEMS - 1];
#pragma unroll
  for (int d = 1; d < 32; d *= 2) {
    const T u = __shfl_up_sync(kFull, t, d);
    if (lane >= d) t += u;
  }
  if (lane == 31) s_warp[wid] = t;
  __syncthreads();
  if (wid == 0) {
    T w = lane < NW ? s_warp[lane] : T(0);
#pragma unroll
    for (int d = 1; d < NW; d *= 2) {
      const T u = __shfl_up_sync(kFull, w, d);
      if (lane >= d) w += u;
    }
    if (lane < NW) s_warp[lane] = w;  // inclusive warp prefixes
  }
  __syncthreads();
  const T aggregate = s_warp[NW - 1];

  // Decoupled look-back by warp 0: publish the aggregate, then inspect 32
  // predecessors per step (one per lane) and sum aggregates down to the
  // nearest published inclusive prefix.
  if (wid == 0) {
    T excl = T(0);
    if (tile == 0) {
      if (lane == 0) {
        st.incl[0] = aggregate;
        __threadfence();
        atomicExch(&st.flag[0], 2);
      }
    } else {
      if (lane == 0) {
        st.agg[tile] = aggregate;
        __threadfence();
        atomicExch(&st.flag[tile], 1);
      }
      for (int base = tile - 1;; base -= 32) {
        const int j = base - lane;  // lane 0 = nearest predecessor
        int f = 2;
        T v = T(0);
        if (j >= 0) {
          do {
            f = ld_volatile(&st.flag[j]);
          } while (f == 0);
          __threadfence();
          v = f == 2 ? ld_volatile(&st.incl[j]) : ld_volatile(&st.agg[j]);
        }
        const unsigned inc = __ballot_sync(kFull, f == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // lanes 0..stop contribute
        T c = lane <= stop ? v : T(0);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) c += __shfl_down_sync(kFull, c, off);
        excl += __shfl_sync(kFull, c, 0);
        if (inc) break;
      }
      if (lane == 0) {
        st.incl[tile] = excl + aggregate;
        __threadfence();
        atomicExch(&st.flag[tile], 2);
      }
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  T add = s_prefix;
  if (wid > 0) add += s_warp[wid - 1];
  const T tprev = __shfl_up_sync(kFull, t, 1);
  if (lane > 0) add += tprev;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) v[i] += add;
  if (full) {
#pragma unroll
    for (int c = 0; c < ITEMS / VQ; ++c) {
      T tmp[VQ];
#pragma unroll
      for (int q = 0; q < VQ; ++q) tmp[q] = v[c * VQ + q];
      st_q<T, VQ>(out + base + c * VQ, tmp);
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (base + i < n) out[base + i] = v[i];
  }
}

template <class T>
cudaError_t scan_impl(const T* d_in, T* d_out, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  constexpr int ITEMS = sizeof(T) == 4 ? 32 : 16;  // 128 contiguous bytes per thread
  constexpr size_t TILE = static_cast<size_t>(kScanThreads) * ITEMS;
  const size_t tiles = (n + TILE - 1) / TILE;
  if (tiles > 0x7fffffff) return cudaErrorInvalidValue;
  // scratch: ticket + flags, then the two value arrays (stream-ordered pool)
  const size_t fbytes = (tiles + 1) * sizeof(int);
  const size_t voff = (fbytes + 15) / 16 * 16;
  const size_t bytes = voff + 2 * tiles * sizeof(T);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, bytes, s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(scratch, 0, fbytes, s);
  if (e == cudaSuccess) {
    ScanState<T> st;
    st.ticket = static_cast<int*>(scratch);
    st.flag = st.ticket + 1;
    st.agg = reinterpret_cast<T*>(static_cast<char*>(scratch) + voff);
    st.incl = st.agg + tiles;
    scan_kernel<T, ITEMS><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(d_in, d_out, n,
                                                                                st);
    note_launch();
    e = cudaGetLastError();
  }
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
