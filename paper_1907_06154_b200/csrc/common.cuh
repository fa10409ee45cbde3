// common.cuh -- device helpers shared by the SSAM engines (sm_100a).
//
// The SSAM execution model of arXiv 1907.06154 maps onto Blackwell as:
//   * a warp is the systolic array: 32 lanes, each owning Q consecutive grid
//     columns (Q*sizeof(T) = 16 B, one 128-bit load per row per lane);
//   * the register file is the cache: each lane keeps a sliding window of
//     rows (2D) or planes (3D) of its Q columns in registers;
//   * partial sums travel lane to lane with __shfl_up_sync -- a one-column
//     shift is Q-1 register renames plus ONE shuffle of the lane's last
//     element, so the shuffle cost per output is 1/Q of the paper's;
//   * there is no shared-memory round trip per tap.
// Reference semantics: proj/include/ssam/plan.hpp:103-159 (PE update rule
// s <- ctrl(r (x) x) (+) shift(s)), warp.hpp:59-77 (shfl_up keeps low lanes).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace ssam_b200 {

constexpr unsigned kFull = 0xffffffffu;

// Q columns per lane so one row segment is one 16-byte access per lane.
template <class T> struct Lanes { static constexpr int Q = 16 / sizeof(T); };

// 16-byte aligned Q-vector used for 128-bit global loads/stores.
template <class T, int Q>
struct alignas(sizeof(T) * Q) VecT {
  T v[Q];
};

template <class T>
__device__ __forceinline__ T fma_t(T a, T b, T c) { return a * b + c; }
template <>
__device__ __forceinline__ float fma_t<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_t<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

// Explicitly rounded multiply / add: never contracted into an FMA, so a
// chain written with mul_t / fma_t / add_t has ONE rounding sequence in
// every kernel that uses it (bit-identical results across engines).
template <class T>
__device__ __forceinline__ T mul_t(T a, T b) { return a * b; }
template <>
__device__ __forceinline__ float mul_t<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_t<double>(double a, double b) { return __dmul_rn(a, b); }
template <class T>
__device__ __forceinline__ T add_t(T a, T b) { return a + b; }
template <>
__device__ __forceinline__ float add_t<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_t<double>(double a, double b) { return __dadd_rn(a, b); }

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) { return __shfl_up_sync(kFull, v, d); }

// Shift a lane-distributed row of 32*Q values one column toward higher x:
// element i takes element i-1.  Lane 0's first element keeps its own value
// (shfl_up semantics, warp.hpp:59-77); it only ever feeds invalid outputs.
template <class T, int Q>
__device__ __forceinline__ void shift_up1(T (&a)[Q]) {
  const T top = shfl_up(a[Q - 1], 1);
#pragma unroll
  for (int q = Q - 1; q > 0; --q) a[q] = a[q - 1];
  a[0] = top;
}

// The mirror image: element i takes element i+1 (shfl_down; lane 31's last
// element keeps its own value and only feeds invalid outputs).
template <class T, int Q>
__device__ __forceinline__ void shift_down1(T (&a)[Q]) {
  const T bot = __shfl_down_sync(kFull, a[0], 1);
#pragma unroll
  for (int q = 0; q < Q - 1; ++q) a[q] = a[q + 1];
  a[Q - 1] = bot;
}

// Read-only 128-bit load through the non-coherent path.
template <class T, int Q>
__device__ __forceinline__ void ld_vec(const T* __restrict__ p, T (&out)[Q]) {
  static_assert(sizeof(T) * Q == 16, "128-bit vectors only");
  const int4 r = __ldg(reinterpret_cast<const int4*>(p));
  VecT<T, Q> v;
  memcpy(&v, &r, sizeof(r));
#pragma unroll
  for (int q = 0; q < Q; ++q) out[q] = v.v[q];
}

template <class T, int Q>
__device__ __forceinline__ void st_vec(T* p, const T (&in)[Q]) {
  VecT<T, Q> v;
#pragma unroll
  for (int q = 0; q < Q; ++q) v.v[q] = in[q];
  *reinterpret_cast<VecT<T, Q>*>(p) = v;
}

__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }

// ---------------------------------------------------------------------------
// TMA bulk-copy staging (sm_90+/sm_100a): cp.async.bulk global -> shared,
// completion tracked by a transaction-counting mbarrier per ring slot.  One
// lane issues; the copy engine moves the bytes while the warp computes, so a
// ring of D slots keeps D row loads in flight without holding registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// Makes mbarrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Orders this thread's prior generic-proxy shared accesses (and those made
// visible to it by an acquiring mbarrier wait) before its subsequent
// async-proxy ops: the WAR hand-off when a consumed slot is refilled by TMA.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

#ifndef SSAM_MBAR_HINT_NS
#define SSAM_MBAR_HINT_NS 2000
#endif
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
#if SSAM_MBAR_HINT_NS > 0
  // suspend-time hint: a waiting warp sleeps (up to the hint) instead of
  // re-issuing the probe, leaving issue slots to the warps that compute
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "n"(SSAM_MBAR_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#ifdef SSAM_DEBUG_HANG
  // debug builds (make debug): a wait that never completes reports and traps
  long long n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++n == (1ll << 20)) {
      printf("mbar_wait stuck: block (%d,%d,%d) thread %d bar 0x%x parity %u\n", blockIdx.x,
             blockIdx.y, blockIdx.z, threadIdx.x, bar, parity);
      __trap();
    }
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}

// 2D tiled TMA load of one box at element coordinates (x, y) of the tensor
// map; out-of-bounds cells arrive as zeros.  The map lives in the kernel's
// __grid_constant__ parameter block.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// Programmatic dependent launch (sm_90+): a grid launched with the
// programmatic-serialization attribute may start while its predecessor
// drains.  griddep_wait() blocks until the predecessor grid has completed
// and its memory is visible -- every kernel calls it before its first
// global read or write; griddep_launch() lets the next grid be scheduled
// into SMs this grid frees.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// TMA ring protocols (PTX memory model).  A slot read with LDS (generic
// proxy) may only be refilled by TMA (async proxy) once every read is
// ordered before the refill:
//  * rings shared by several warps (engine3d.cuh, engine3d_pipe.cuh): each
//    consumer lane arrives on the slot's EMPTY mbarrier (release); the
//    producer waits on it (acquire), executes fence.proxy.async and issues
//    the copy -- the producer/consumer mbarrier pipeline;
//  * warp-private rings (engine2d.cuh, engine2d_fma.cuh, tb2d.cu):
//    ring_release_warp() -- every lane executes fence.proxy.async after its
//    reads, then the warp barrier orders all lanes before lane 0's copy (the
//    fence-then-barrier-then-issue pattern of TMA stores, mirrored).  A/B on
//    the 2D fused kernels: as fast as an unsynchronised hand-back, 4% faster
//    than the mbarrier protocol (profiles/r02/ring_protocol_ab.txt).
__device__ __forceinline__ void ring_release_warp() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
}

// Q-vector shared load / global store as 16-byte chunks (Q*sizeof(T) in {16, 32}).
template <class T, int Q>
__device__ __forceinline__ void lds_q(const T* p, T (&out)[Q]) {
  constexpr int V = 16 / sizeof(T);
  static_assert(Q % V == 0, "whole 16-byte chunks");
#pragma unroll
  for (int c = 0; c < Q / V; ++c) {
    const int4 r = *reinterpret_cast<const int4*>(p + c * V);
    T tmp[V];
    memcpy(tmp, &r, 16);
#pragma unroll
    for (int q = 0; q < V; ++q) out[c * V + q] = tmp[q];
  }
}

template <class T, int Q>
__device__ __forceinline__ void st_q(T* p, const T (&in)[Q]) {
  constexpr int V = 16 / sizeof(T);
  static_assert(Q % V == 0, "whole 16-byte chunks");
#pragma unroll
  for (int c = 0; c < Q / V; ++c) {
    int4 r;
    memcpy(&r, in + c * V, 16);
    *reinterpret_cast<int4*>(p + c * V) = r;
  }
}

template <class T, int Q>
__device__ __forceinline__ void ldg_q(const T* __restrict__ p, T (&out)[Q]) {
  constexpr int V = 16 / sizeof(T);
  static_assert(Q % V == 0, "whole 16-byte chunks");
#pragma unroll
  for (int c = 0; c < Q / V; ++c) {
    const int4 r = __ldg(reinterpret_cast<const int4*>(p + c * V));
    T tmp[V];
    memcpy(tmp, &r, 16);
#pragma unroll
    for (int q = 0; q < V; ++q) out[c * V + q] = tmp[q];
  }
}

// 128-bit shared load of one lane's Q-vector.
template <class T, int Q>
__device__ __forceinline__ void lds_vec(const T* p, T (&out)[Q]) {
  static_assert(sizeof(T) * Q == 16, "128-bit vectors only");
  const int4 r = *reinterpret_cast<const int4*>(p);
  VecT<T, Q> v;
  memcpy(&v, &r, sizeof(r));
#pragma unroll
  for (int q = 0; q < Q; ++q) out[q] = v.v[q];
}

}  // namespace ssam_b200
