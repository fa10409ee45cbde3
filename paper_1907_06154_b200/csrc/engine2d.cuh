// engine2d.cuh -- the 2D SSAM engine (conv2d and 2D stencil sweeps), sm_100a.
//
// One warp owns a vertical strip of the grid: 32 lanes x Q columns of input
// and streams DOWN the strip, one output row per step (the "y-streaming
// window" of SURVEY Appendix B).  Per lane the register file holds the NR
// rows of its Q columns that the current output row needs -- the paper's
// register cache -- and nothing is re-read from memory per tap.
//
// Per output row the warp runs the systolic chain of the reference's window
// plans (kernels.hpp:74-102 for dense filters, :111-159 for sparse taps):
//     colpart_j = sum_t coef[j][t] * row[t]       (register cache x broadcast r)
//     acc       = shift(acc) + colpart_j          (shuffle systolic transfer)
// i.e. the paper's two-level accumulation: an NR-tap
// column partial, then one add per column -- the order that keeps fp32 conv
// within 1e-5 up to 20x20.
//
// Blackwell twist -- a BIDIRECTIONAL chain.  The paper's single shfl_up chain
// lands each result R columns to the right of its output, which for 16-byte
// vector stores costs (-R mod Q) extra shuffles per row.  Here the L left
// columns flow up (shfl_up, as in the paper) and the R right columns flow
// down (shfl_down); the two partial sums meet in the output's own lane:
//     out(x) = [ sum_{j<=L} left chain ] + [ sum_{j>L} right chain ]
// Same M-1 shuffles, no re-alignment, every lane stores its own Q columns.
//
// Everything is expressed as a correlation
//     out(x, y) = sum_{j,t} coef[j*NR+t] * in(x + j - L, y + t - U)
// with R = (M-1)/2, L = M-1-R, D = (NR-1)/2, U = NR-1-D.  conv2d maps to it
// with coef[j][t] = w[(m-1-j)*n + (n-1-t)] -- the flipped filter exactly as
// the reference builds it (kernels.hpp:90) -- and stencils with
// coef[j][t] = c(dx=j-k, dy=t-k) (unflipped taps, oracle.hpp:88-90).
//
// Two kernels share the row computation:
//  * ssam2d_tma_kernel (16-byte aligned rows, zero boundary / stencils -- the
//    benchmark path): rows arrive as RB-row TMA boxes (cp.async.bulk.tensor,
//    one mbarrier per box, D boxes in flight per warp).  The TMA unit's
//    out-of-bounds zero fill IS the zero boundary.
//  * ssam2d_kernel (replicate boundary, unaligned widths): direct loads with
//    PF rows of register prefetch.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"

namespace ssam_b200 {

enum : int { kBndZero = 0, kBndReplicate = 1, kBndStencil = 2 };

template <class T, int CAP>
struct Ssam2DParams {
  const T* in;
  T* out;
  int W, H;
  int M;        // filter columns (runtime copy; equals MC when compile-time)
  int A, V;     // lane plan: lane 0 starts at x_out0 - A; V outputs per warp row
  int nstrips;  // warps across x
  int seg;      // output rows streamed per warp
  int y_begin, y_end;
  int bmode;    // kBndZero / kBndReplicate (conv) or kBndStencil
  int ring;     // stencil: only [ring, W-ring) x [ring, H-ring) is written
  int vec_ok;   // Q-vector loads/stores usable (LDG kernel)
  T coef[CAP];  // coef[j*NR + t]
};

template <class T, int CAP>
struct alignas(64) Ssam2DTmaParams {
  CUtensorMap tmap;  // (W, H) row-major, box 32Q x RB
  Ssam2DParams<T, CAP> p;
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
template <class Mask> struct IsStar2D { static constexpr bool value = false; };
template <int K> struct IsStar2D<StarMask2D<K>> { static constexpr bool value = true; };

// Column-chain form of the star row (left chain up, right chain down).
template <class T, int Q, int K, int NB, class CF>
__device__ __forceinline__ void star_row_colchain(const T (&buf)[NB][Q], int rot, CF coef,
                                               T (&acc)[Q]) {
  constexpr int NR = 2 * K + 1;
  {
    const T c = coef(0, K);
    const int b = (rot + K) % NB;
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = mul_t(c, buf[b][q]);
  }
#pragma unroll
  for (int j = 1; j <= K; ++j) {
    shift_up1<T, Q>(acc);
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      if (!StarMask2D<K>::has(j, t)) continue;
      const T c = coef(j, t);
      const int b = (rot + t) % NB;
#pragma unroll
      for (int q = 0; q < Q; ++q) acc[q] = fma_t(c, buf[b][q], acc[q]);
    }
  }
  if constexpr (K > 0) {
    T accr[Q];
    {
      const T c = coef(NR - 1, K);
      const int b = (rot + K) % NB;
#pragma unroll
      for (int q = 0; q < Q; ++q) accr[q] = mul_t(c, buf[b][q]);
    }
#pragma unroll
    for (int j = NR - 2; j > K; --j) {
      shift_down1<T, Q>(accr);
      const T c = coef(j, K);  // off-centre columns of a star: the centre row only
      const int b = (rot + K) % NB;
#pragma unroll
      for (int q = 0; q < Q; ++q) accr[q] = fma_t(c, buf[b][q], accr[q]);
    }
    shift_down1<T, Q>(accr);
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = add_t(acc[q], accr[q]);
  }
}

// One output row of an order-K star as ONE FMA chain per output: the
// centre tap's rounded product, then the x taps (dx = -K..-1, 1..K), then
// the y taps (dy = -K..-1, 1..K) -- the 3D pipeline's order
// (pipe_star_cell).  The x neighbours are the centre row's own values: a
// lane's Q columns plus K columns shuffled in from each neighbour lane (K
// SHFL up, K down per row), so every tap is one FFMA (2d5pt: 1 FMUL + 4
// FFMA per cell).  Window row t (dy = t - K) is buf[(rot + t) % NB];
// coef(j, t) returns the tap's coefficient.  Written with mul_t / fma_t only
// (no contraction freedom), so the single-sweep engines and every
// temporal-blocking stage produce bit-identical rows.  (fp64, int64: the
// column-chain order above.)
template <class T, int Q, int K, int NB, class CF>
__device__ __forceinline__ void star_row_chain(const T (&buf)[NB][Q], int rot, CF coef,
                                               T (&acc)[Q]) {
  // fp32: 2d5pt Tb 4 1750 -> 1935, 2d9pt Tb 2 1135 -> 1182 GCells/s; fp64
  // measured 4% slower at 2d5pt Tb 4 and keeps the column chain
  // (profiles/r02/star2d_chain_ab.txt)
  if constexpr (K >= 1 && K <= Q && std::is_same<T, float>::value) {
    const T(&cr)[Q] = buf[(rot + K) % NB];
    T lft[K], rgt[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      lft[i] = shfl_up(cr[Q - K + i], 1);
      rgt[i] = __shfl_down_sync(kFull, cr[i], 1);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      auto xs = [&](int qq) { return qq < 0 ? lft[K + qq] : (qq >= Q ? rgt[qq - Q] : cr[qq]); };
      T v = mul_t(coef(K, K), cr[q]);
#pragma unroll
      for (int d = -K; d <= K; ++d)
        if (d != 0) v = fma_t(coef(K + d, K), xs(q + d), v);
#pragma unroll
      for (int d = -K; d <= K; ++d)
        if (d != 0) v = fma_t(coef(K, K + d), buf[(rot + K + d) % NB][q], v);
      acc[q] = v;
    }
  } else {
    star_row_colchain<T, Q, K, NB>(buf, rot, coef, acc);
  }
}

// Column partial of filter column j: window row t is buf[(rot + t) % NB].
template <class T, int Q, int NR, class Mask, int NB, int CAP>
__device__ __forceinline__ bool colpart_ct(const T (&buf)[NB][Q], int rot, int j,
                                           const Ssam2DParams<T, CAP>& p, T (&cp)[Q]) {
  bool any = false;
#pragma unroll
  for (int t = 0; t < NR; ++t) {
    if (Mask::has(j, t)) {
      const T c = p.coef[j * NR + t];
      const int b = (rot + t) % NB;
#pragma unroll
      for (int q = 0; q < Q; ++q) cp[q] = any ? fma_t(c, buf[b][q], cp[q]) : c * buf[b][q];
      any = true;
    }
  }
  return any;
}

// One output row, compile-time footprint (MC x NR) and tap mask.  `rot` must
// fold to a constant after unrolling (it indexes registers).
template <class T, int Q, int NR, int MC, class Mask, int NB, int CAP>
__device__ __forceinline__ void ssam_row_ct(const T (&buf)[NB][Q], int rot,
                                            const Ssam2DParams<T, CAP>& p, T (&acc)[Q]) {
  if constexpr (IsStar2D<Mask>::value && MC == NR) {
    star_row_chain<T, Q, (NR - 1) / 2, NB>(buf, rot,
                                           [&](int j, int t) { return p.coef[j * NR + t]; }, acc);
    return;
  }
  constexpr int R = (MC - 1) / 2, L = MC - 1 - R;
  // left chain: columns j = 0..L flow up into the centre lane
#pragma unroll
  for (int j = 0; j <= L; ++j) {
    T cp[Q];
    const bool any = colpart_ct<T, Q, NR, Mask, NB, CAP>(buf, rot, j, p, cp);
    if (j == 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) acc[q] = any ? cp[q] : T(0);
    } else {
      shift_up1<T, Q>(acc);
      if (any) {
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[q] += cp[q];
      }
    }
  }
  if constexpr (R > 0) {
    // right chain: columns j = MC-1..L+1 flow down, one more step lands it
    T accr[Q];
#pragma unroll
    for (int j = MC - 1; j > L; --j) {
      T cp[Q];
      const bool any = colpart_ct<T, Q, NR, Mask, NB, CAP>(buf, rot, j, p, cp);
      if (j == MC - 1) {
#pragma unroll
        for (int q = 0; q < Q; ++q) accr[q] = any ? cp[q] : T(0);
      } else {
        shift_down1<T, Q>(accr);
        if (any) {
#pragma unroll
          for (int q = 0; q < Q; ++q) accr[q] += cp[q];
        }
      }
    }
    shift_down1<T, Q>(accr);
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] += accr[q];
  }
}

// One output row, runtime filter width p.M (dense); NR rows compile-time.
template <class T, int Q, int NR, int NB, int CAP>
__device__ __forceinline__ void ssam_row_rt(const T (&buf)[NB][Q], int rot,
                                            const Ssam2DParams<T, CAP>& p, T (&acc)[Q]) {
  const int R = (p.M - 1) / 2, L = p.M - 1 - R;
  auto colpart = [&](int j, T (&cp)[Q]) {
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const T c = p.coef[j * NR + t];
      const int b = (rot + t) % NB;
#pragma unroll
      for (int q = 0; q < Q; ++q) cp[q] = t == 0 ? c * buf[b][q] : fma_t(c, buf[b][q], cp[q]);
    }
  };
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = T(0);
  for (int j = 0; j <= L; ++j) {
    T cp[Q];
    colpart(j, cp);
    shift_up1<T, Q>(acc);  // the j == 0 shift moves zeros: harmless
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] += cp[q];
  }
  if (R > 0) {
    T accr[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) accr[q] = T(0);
    for (int j = p.M - 1; j > L; --j) {
      T cp[Q];
      colpart(j, cp);
      shift_down1<T, Q>(accr);
#pragma unroll
      for (int q = 0; q < Q; ++q) accr[q] += cp[q];
    }
    shift_down1<T, Q>(accr);
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] += accr[q];
  }
}

template <class T, int Q, int NR, int MC, class Mask, int NB, int CAP>
__device__ __forceinline__ void ssam_row(const T (&buf)[NB][Q], int rot,
                                         const Ssam2DParams<T, CAP>& p, T (&acc)[Q]) {
  if constexpr (MC > 0)
    ssam_row_ct<T, Q, NR, MC, Mask, NB, CAP>(buf, rot, p, acc);
  else
    ssam_row_rt<T, Q, NR, NB, CAP>(buf, rot, p, acc);
}

// Per-lane store plan, fixed for the whole strip: each lane stores its own Q
// columns [x0, x0+Q) when they belong to the warp's [x_out0, x_out0+V).
struct StorePlan {
  int x0;
  bool own;
  bool whole;    // all Q outputs writable as 16-byte vectors
  int xlo, xhi;  // writable column range
};

template <class T, int Q, int CAP>
__device__ __forceinline__ StorePlan store_plan(const Ssam2DParams<T, CAP>& p, int x_out0,
                                                int x0, bool vec) {
  StorePlan s;
  s.x0 = x0;
  s.own = x0 >= x_out0 && x0 < x_out0 + p.V;
  s.xlo = p.bmode == kBndStencil ? p.ring : 0;
  s.xhi = p.bmode == kBndStencil ? p.W - p.ring : p.W;
  s.whole = vec && x0 >= s.xlo && x0 + Q <= s.xhi;
  return s;
}

template <class T, int Q, int CAP>
__device__ __forceinline__ void store_row(const Ssam2DParams<T, CAP>& p, const StorePlan& sp,
                                          int y, const T (&acc)[Q]) {
  if (!sp.own) return;
  if (p.bmode == kBndStencil && (y < p.ring || y >= p.H - p.ring)) return;  // ring carries over
  T* row = p.out + static_cast<size_t>(y) * p.W + sp.x0;
  if (sp.whole) {
    st_q<T, Q>(row, acc);
    return;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (sp.x0 + q >= sp.xlo && sp.x0 + q < sp.xhi) row[q] = acc[q];
}

// Shared memory of the TMA kernel: per warp D boxes of RB rows, D mbarriers
// and a spare 128-byte line.
template <class T, int Q, int RB, int D>
__host__ __device__ constexpr size_t tma2d_smem(int warps) {
  return static_cast<size_t>(warps) *
         (D * (static_cast<size_t>(RB) * 32 * Q * sizeof(T) + 8) + 128);
}

template <class T, int Q, int NR, int MC, class Mask, int RB, int D, int CAP>
__global__ void __launch_bounds__(128)
    ssam2d_tma_kernel(const __grid_constant__ Ssam2DTmaParams<T, CAP> P) {
  const Ssam2DParams<T, CAP>& p = P.p;
  constexpr int U = NR - 1 - (NR - 1) / 2;
  constexpr int ROW = 32 * Q;
  constexpr uint32_t BOX_BYTES = RB * ROW * sizeof(T);
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int strip = blockIdx.x * (blockDim.x >> 5) + wib;
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;  // 16-byte aligned box origin
  const StorePlan sp = store_plan<T, Q, CAP>(p, x_out0, base + Q * lane, true);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * D * RB * ROW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
                       smem_raw + static_cast<size_t>(blockDim.x >> 5) * D * BOX_BYTES) +
                   wib * D;
  if (lane == 0) {
    prefetch_tmap(&P.tmap);
#pragma unroll
    for (int s = 0; s < D; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains
  const int count = (y1 - y0) + NR - 1;  // stream rows y0-U .. y1-1+D
  const int nbox = (count + RB - 1) / RB;
  auto issue = [&](int j) {
    const int s = j % D;
    const uint32_t bar = smem_u32(&bars[s]);
    mbar_arrive_expect_tx(bar, BOX_BYTES);
    tma_load_2d(smem_u32(ring + s * RB * ROW), &P.tmap, base, y0 - U + j * RB, bar);
  };
  if (lane == 0)
    for (int j = 0; j < min(D, nbox); ++j) issue(j);
  // Ring hand-back after the warp's last read of box j (common.cuh
  // ring_release_warp): the slot is refilled with box j + D.
  auto recycle = [&](int j) {
    ring_release_warp();
    if (lane == 0 && j + D < nbox) issue(j + D);
  };

  if constexpr (RB == NR) {
    // Whole-window boxes: box j's NR rows are read into one half of a
    // 2*NR-row register window in one burst of LDS (latency overlapped), then
    // NR output rows are computed from the previous box's rows plus these.
    // Two boxes per loop trip swap the halves' roles: no register moves.
    T win[2 * NR][Q];
    auto box = [&](int j, int cur) {
      const int s = j % D;
      mbar_wait(smem_u32(&bars[s]), (j / D) & 1);
      const T* slot = ring + s * RB * ROW + Q * lane;
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) lds_q<T, Q>(slot + rr * ROW, win[cur + rr]);
      recycle(j);  // slot s is in registers: refill it while the rows compute
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const int i = j * NR + rr;
        if (i >= count) break;
        if (i >= NR - 1) {
          T acc[Q];
          // window row t = stream row i-NR+1+t: rows of the previous box sit
          // in the other half, so it is win[(cur + NR + rr + 1 + t) % 2NR]
          ssam_row<T, Q, NR, MC, Mask, 2 * NR, CAP>(win, cur + NR + rr + 1, p, acc);
          store_row<T, Q, CAP>(p, sp, y0 + i - (NR - 1), acc);
        }
      }
    };
    for (int j = 0; j < nbox; j += 2) {
      box(j, 0);
      if (j + 1 < nbox) box(j + 1, NR);
    }
  } else {
    // Tall windows: the window shifts down one row per step and exactly one
    // row body is emitted (a large filter's row is thousands of FMAs; more
    // unrolling only thrashes the instruction cache).  A slot is handed back
    // after its last row was read.
    T win[NR][Q];
    for (int j = 0; j < nbox; ++j) {
      const int s = j % D;
      mbar_wait(smem_u32(&bars[s]), (j / D) & 1);
      const T* slot = ring + s * RB * ROW + Q * lane;
      const int rows = min(RB, count - j * RB);
#pragma unroll 1
      for (int rr = 0; rr < rows; ++rr) {
        const int i = j * RB + rr;
#pragma unroll
        for (int t = 0; t < NR - 1; ++t)
#pragma unroll
          for (int q = 0; q < Q; ++q) win[t][q] = win[t + 1][q];
        lds_q<T, Q>(slot + rr * ROW, win[NR - 1]);
        if (i >= NR - 1) {
          T acc[Q];
          ssam_row<T, Q, NR, MC, Mask, NR, CAP>(win, 0, p, acc);
          store_row<T, Q, CAP>(p, sp, y0 + i - (NR - 1), acc);
        }
      }
      recycle(j);
    }
  }
}

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
    ldg_q<T, Q>(row + col0, dst);
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

// Direct-load kernel: replicate boundary and unaligned widths.
template <class T, int Q, int NR, int MC, class Mask, int PF, int CAP>
__global__ void __launch_bounds__(128) ssam2d_kernel(const __grid_constant__ Ssam2DParams<T, CAP> p) {
  constexpr int U = NR - 1 - (NR - 1) / 2;
  constexpr int NB = NR + PF;
  const int lane = threadIdx.x & 31;
  const int strip = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;
  const int col0 = base + Q * lane;
  const bool fast = p.vec_ok && base >= 0 && base + 32 * Q <= p.W;
  const StorePlan sp = store_plan<T, Q, CAP>(p, x_out0, col0, p.vec_ok != 0);

  T buf[NB][Q];
#pragma unroll
  for (int t = 0; t < NB - 1; ++t)
    load_row<T, Q>(p.in, p.W, p.H, y0 - U + t, col0, fast, p.bmode, buf[t]);

  for (int y = y0; y < y1; ++y) {
    load_row<T, Q>(p.in, p.W, p.H, y - U + NB - 1, col0, fast, p.bmode, buf[NB - 1]);
    T acc[Q];
    ssam_row<T, Q, NR, MC, Mask, NB, CAP>(buf, 0, p, acc);
    store_row<T, Q, CAP>(p, sp, y, acc);
#pragma unroll
    for (int t = 0; t < NB - 1; ++t)
#pragma unroll
      for (int q = 0; q < Q; ++q) buf[t][q] = buf[t + 1][q];
  }
}

}  // namespace ssam_b200
