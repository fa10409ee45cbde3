// engine2d.cuh -- the 2D SSAM engine (conv2d and 2D stencil sweeps), sm_100a.
//
// One warp owns a vertical strip of the grid: 32 lanes x Q columns of input
// (base .. base+32Q-1) and streams DOWN the strip, one output row per step
// (the "y-streaming window" of SURVEY Appendix B).  Per lane the register
// file holds NR+PF rows of its Q columns: NR rows for the current output row
// (the register cache, C = NR in the paper's notation) plus PF rows of
// prefetch so PF+1 128-bit loads per lane are always in flight.
//
// Per output row the warp runs the systolic chain of the reference's window
// plans (kernels.hpp:74-102 for dense filters, :111-159 for sparse taps):
//   for filter column j = 0..M-1:
//       colpart = sum_t coef[j][t] * row[t]        (register cache x broadcast r)
//       acc     = shift1(acc) + colpart            (shfl_up systolic transfer)
// i.e. the paper's two-level accumulation: an NR-tap
// column partial, then one add per column.  This order is what keeps fp32
// conv within 1e-5 up to 20x20.  After the chain (plus E extra
// shifts so results land 16-byte aligned) lane position i holds output column
// base + i - G for i >= M-1+E.
//
// Everything is expressed as a correlation
//     out(x, y) = sum_{j,t} coef[j*NR+t] * in(x + j - L, y + t - U)
// with R = (M-1)/2, L = M-1-R, D = (NR-1)/2, U = NR-1-D.  conv2d maps to it
// with coef[j][t] = w[(m-1-j)*n + (n-1-t)] -- the flipped filter exactly as
// the reference builds it (kernels.hpp:90) -- and stencils with
// coef[j][t] = c(dx=j-k, dy=t-k) (unflipped taps, oracle.hpp:88-90).
#pragma once

#include "common.cuh"

namespace ssam_b200 {

enum : int { kBndZero = 0, kBndReplicate = 1, kBndStencil = 2 };

template <class T, int CAP>
struct Ssam2DParams {
  const T* in;
  T* out;
  int W, H;
  int M;           // filter columns (runtime copy; equals MC when compile-time)
  int e, G, A, V;  // lane plan, see plan_lanes() in launch2d.cuh
  int nstrips;     // warps across x
  int seg;         // output rows streamed per warp
  int y_begin, y_end;
  int bmode;       // kBndZero / kBndReplicate (conv) or kBndStencil
  int ring;        // stencil: only [ring, W-ring) x [ring, H-ring) is written
  int vec_ok;      // W % Q == 0 and both pointers 16-byte aligned
  T coef[CAP];     // coef[j*NR + t]
};

// Dense mask: every (j, t) cell carries a coefficient (conv filters, generic taps).
struct DenseMask {
  __host__ __device__ static constexpr bool has(int, int) { return true; }
};
// Star stencil of order K: centre column j == K or centre row t == K.
template <int K>
struct StarMask2D {
  __host__ __device__ static constexpr bool has(int j, int t) { return j == K || t == K; }
};

template <class T, int Q>
__device__ __forceinline__ void load_row(const T* __restrict__ in, int W, int H, int y, int col0,
                                         bool fast, int bmode, T (&dst)[Q]) {
  if (y < 0 || y >= H) {
    if (bmode != kBndReplicate) {
#pragma unroll
      for (int q = 0; q < Q; ++q) dst[q] = T(0);
      return;
    }
    y = clampi(y, H);
  }
  const T* row = in + static_cast<size_t>(y) * W;
  if (fast) {
    ld_vec<T, Q>(row + col0, dst);
    return;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int x = col0 + q;
    if (x >= 0 && x < W)
      dst[q] = __ldg(row + x);
    else if (bmode == kBndReplicate)
      dst[q] = __ldg(row + clampi(x, W));
    else
      dst[q] = T(0);
  }
}

// One output row, compile-time filter footprint (MC x NR) and tap mask.
template <class T, int Q, int NR, int MC, class Mask, int NB, int CAP>
__device__ __forceinline__ void ssam_row_ct(const T (&buf)[NB][Q],
                                            const Ssam2DParams<T, CAP>& p, T (&acc)[Q]) {
#pragma unroll
  for (int j = 0; j < MC; ++j) {
    T cp[Q];
    bool any = false;
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      if (Mask::has(j, t)) {
        const T c = p.coef[j * NR + t];
#pragma unroll
        for (int q = 0; q < Q; ++q) cp[q] = any ? fma_t(c, buf[t][q], cp[q]) : c * buf[t][q];
        any = true;
      }
    }
    if (j == 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) acc[q] = any ? cp[q] : T(0);
    } else {
      shift1<T, Q>(acc);
      if (any) {
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[q] += cp[q];
      }
    }
  }
  constexpr int R = (MC - 1) / 2;
  constexpr int E = (Q - R % Q) % Q;
#pragma unroll
  for (int s = 0; s < E; ++s) shift1<T, Q>(acc);
}

// One output row, runtime filter width p.M (dense); NR rows compile-time.
template <class T, int Q, int NR, int NB, int CAP>
__device__ __forceinline__ void ssam_row_rt(const T (&buf)[NB][Q],
                                            const Ssam2DParams<T, CAP>& p, T (&acc)[Q]) {
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = T(0);
#pragma unroll 2
  for (int j = 0; j < p.M; ++j) {
    T cp[Q];
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const T c = p.coef[j * NR + t];
#pragma unroll
      for (int q = 0; q < Q; ++q) cp[q] = t == 0 ? c * buf[t][q] : fma_t(c, buf[t][q], cp[q]);
    }
    shift1<T, Q>(acc);  // the j == 0 shift moves zeros: harmless
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] += cp[q];
  }
  for (int s = 0; s < p.e; ++s) shift1<T, Q>(acc);
}

template <class T, int Q, int CAP>
__device__ __forceinline__ void store_row(const Ssam2DParams<T, CAP>& p, int y, int x_out0,
                                          int xres, const T (&acc)[Q]) {
  if (xres < x_out0 || xres >= x_out0 + p.V) return;  // not owned by this warp
  int xlo = 0, xhi = p.W;
  if (p.bmode == kBndStencil) {
    if (y < p.ring || y >= p.H - p.ring) return;  // boundary ring carries over
    xlo = p.ring;
    xhi = p.W - p.ring;
  }
  T* row = p.out + static_cast<size_t>(y) * p.W;
  if (p.vec_ok && xres >= xlo && xres + Q <= xhi) {
    st_vec<T, Q>(row + xres, acc);
    return;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (xres + q >= xlo && xres + q < xhi) row[xres + q] = acc[q];
}

template <class T, int Q, int NR, int MC, class Mask, int NB, int CAP>
__device__ __forceinline__ void ssam_row(const T (&buf)[NB][Q], const Ssam2DParams<T, CAP>& p,
                                         T (&acc)[Q]) {
  if constexpr (MC > 0)
    ssam_row_ct<T, Q, NR, MC, Mask, NB, CAP>(buf, p, acc);
  else
    ssam_row_rt<T, Q, NR, NB, CAP>(buf, p, acc);
}

// Dynamic shared memory of the TMA path: per warp D row slots + D mbarriers.
template <class T, int Q, int D>
__host__ __device__ constexpr size_t ring2d_bytes(int warps) {
  return static_cast<size_t>(warps) * D * (32 * Q * sizeof(T) + 8);
}

// MC > 0: compile-time footprint with Mask; MC == 0: runtime p.M, dense.
//
// Two load paths, chosen per launch (warp-uniform):
//  * TMA ring (aligned grids, the benchmark path): lane 0 keeps D row copies
//    in flight with cp.async.bulk into a per-warp shared ring; lanes read
//    their 16-byte Q-vector with one LDS.128 and push it into the register
//    window.  D rows of prefetch cost no registers.
//  * direct loads (unaligned widths): 128-bit / scalar LDG with PF rows of
//    register prefetch.
template <class T, int Q, int NR, int MC, class Mask, int PF, int CAP, int D>
__global__ void __launch_bounds__(128) ssam2d_kernel(const __grid_constant__ Ssam2DParams<T, CAP> p) {
  constexpr int U = NR - 1 - (NR - 1) / 2;
  constexpr int ROW = 32 * Q;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int strip = blockIdx.x * (blockDim.x >> 5) + wib;
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;
  const int col0 = base + Q * lane;
  const int xres = col0 - p.G;

  if (p.vec_ok) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * D * ROW;
    uint64_t* bars = reinterpret_cast<uint64_t*>(
                         smem_raw + static_cast<size_t>(blockDim.x >> 5) * D * ROW * sizeof(T)) +
                     wib * D;
    const bool interior_x = base >= 0 && base + ROW <= p.W;
    const int cbeg = max(base, 0), cend = min(base + ROW, p.W);
    const uint32_t bytes = static_cast<uint32_t>(cend - cbeg) * sizeof(T);
    const int doff = cbeg - base;
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < D; ++s) mbar_init(smem_u32(&bars[s]), 1);
      fence_mbar_init();
    }
    __syncwarp();
    const int count = (y1 - y0) + NR - 1;
    auto issue = [&](int i) {
      const int s = i % D;
      const int r = clampi(y0 - U + i, p.H);
      fence_proxy_async();
      mbar_arrive_expect_tx(smem_u32(&bars[s]), bytes);
      tma_load_1d(smem_u32(ring + s * ROW + doff), p.in + static_cast<size_t>(r) * p.W + cbeg,
                  bytes, smem_u32(&bars[s]));
    };
    if (lane == 0)
      for (int i = 0; i < min(D, count); ++i) issue(i);

    T win[NR][Q];
    for (int i = 0; i < count; ++i) {
      const int s = i % D;
      mbar_wait(smem_u32(&bars[s]), (i / D) & 1);
#pragma unroll
      for (int t = 0; t < NR - 1; ++t)
#pragma unroll
        for (int q = 0; q < Q; ++q) win[t][q] = win[t + 1][q];
      const T* slot = ring + s * ROW;
      lds_vec<T, Q>(slot + Q * lane, win[NR - 1]);
      const int r = y0 - U + i;
      if (p.bmode == kBndZero && (r < 0 || r >= p.H)) {
#pragma unroll
        for (int q = 0; q < Q; ++q) win[NR - 1][q] = T(0);
      } else if (p.bmode != kBndStencil && !interior_x) {
        // conv edge strips: outside columns are zero or the clamped edge cell
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int x = col0 + q;
          if (x < 0 || x >= p.W)
            win[NR - 1][q] = p.bmode == kBndZero ? T(0) : slot[clampi(x, p.W) - base];
        }
      }
      __syncwarp();
      if (lane == 0 && i + D < count) issue(i + D);
      if (i >= NR - 1) {
        T acc[Q];
        ssam_row<T, Q, NR, MC, Mask, NR, CAP>(win, p, acc);
        store_row<T, Q, CAP>(p, y0 + i - (NR - 1), x_out0, xres, acc);
      }
    }
    return;
  }

  constexpr int NB = NR + PF;
  const bool fast = false;  // unaligned grids: scalar loads
  T buf[NB][Q];
#pragma unroll
  for (int t = 0; t < NB - 1; ++t)
    load_row<T, Q>(p.in, p.W, p.H, y0 - U + t, col0, fast, p.bmode, buf[t]);

  for (int y = y0; y < y1; ++y) {
    load_row<T, Q>(p.in, p.W, p.H, y - U + NB - 1, col0, fast, p.bmode, buf[NB - 1]);
    T acc[Q];
    ssam_row<T, Q, NR, MC, Mask, NB, CAP>(buf, p, acc);
    store_row<T, Q, CAP>(p, y, x_out0, xres, acc);
#pragma unroll
    for (int t = 0; t < NB - 1; ++t)
#pragma unroll
      for (int q = 0; q < Q; ++q) buf[t][q] = buf[t + 1][q];
  }
}

}  // namespace ssam_b200
