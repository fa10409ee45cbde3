// engine3d_pipe.cuh -- the 3D SSAM engine as a TB-stage warp pipeline:
// TB Jacobi sweeps per pass over HBM, sm_100a.
//
// Reference semantics: ssam::stencil3d (proj/include/ssam/kernels.hpp:283-384)
// applied TB times (temporal blocking is Tb consecutive sweeps):
// every sweep writes the interior [K, n-K) per axis and carries the ring.
// Shapes: the order-K star (3d7pt K = 1, 3d13pt K = 2; any coefficients) and
// the order-1 box family (3d27pt, Poisson 3d19pt: any 3x3x3 mask).
//
// One CTA owns an x-strip (32 lanes x Q columns; lane plan A/V for a
// 2 K TB + 1 column footprint), ROWS output rows and a z-segment.  Its warps
// form TB stages plus one producer warp:
//
//   producer   TMA: input plane boxes (strip x (rows + 2 K TB)) into a ring of
//              DZ slots (full = transaction count, empty = stage-1 lanes);
//   stage s    streams the planes of stage s-1 (stage 0 = the TMA ring) and
//              computes sweep s for its band: ROWS + 2 K (TB - s) rows, each
//              warp RY(s) of them.  Stages < TB write their planes to a
//              shared-memory ring (DI slots, full = producer lanes, empty =
//              consumer lanes); stage TB stores the interior to HBM.
//
// Per output row a lane holds its Q columns of the 2K+1 source planes in
// registers (z-streaming).  Stars keep only the RY centre rows of the
// off-centre planes (a star never reads their y neighbours); a plane's 2K
// halo rows are read from its slot when it becomes the centre.  Boxes keep
// all RY + 2 rows.  x neighbours come from shuffles of the centre row
// (stars: K up, K down) or of the dx = -1 / +1 column partials (boxes:
// one up, one down -- the systolic shift of the paper's dataflow).  Each
// cell is ONE fixed chain of FMAs (pipe_star_cell / pipe_box_cell), so every
// kernel of a shape -- any TB, aligned or direct-load -- gives bit-identical
// results for the same number of sweeps.
//
// Ring protocol (PTX memory model): a consumer lane reads a slot with LDS,
// consumes the values in FMAs, then arrives (release) on the slot's empty
// barrier; the producer waits (acquire) on it and, for TMA refills, issues
// fence.proxy.async before the bulk copy (generic-proxy reads ordered before
// async-proxy writes).  Every lane arrives itself -- no __syncwarp hand-off.
#pragma once

#include "engine3d.cuh"

namespace ssam_b200 {

template <int K_>
struct PipeStar {
  static constexpr int K = K_;
  static constexpr bool STAR = true;
  using Mask = StarMask3<K_>;
};
template <class Mask_>
struct PipeBox {
  static constexpr int K = 1;
  static constexpr bool STAR = false;
  using Mask = Mask_;
};

// Geometry of one (T, shape, TB) pipeline.  Stage s (1..TB) has sy(s)
// warps of ry(s) rows; sy(s) * ry(s) >= nr(s) = ROWS + 2 K (TB - s).
template <class T, class Sh, int TB_>
struct PipeGeom {
  static constexpr int TB = TB_;
  static constexpr int K = Sh::K;
  static constexpr bool STAR = Sh::STAR;
  static constexpr int Q = 16 / static_cast<int>(sizeof(T));
  static constexpr int BW = 32 * Q;  // strip / box / slot row width
  // Tb = 2 order-1 star, stage geometry per element type (profiles/r02/
  // pipe_stage_ab.txt, sustained_ab2.txt).  Round 1's 6 x 3 / 4 x 4 split
  // left stage 1 waiting on the intermediate ring's EMPTY barriers (26% of
  // ncu's stall samples): stage 2, which also stores to HBM, was the slower
  // stage.  fp32 (the headline): 18 output rows, stage 1 5 warps x 4 rows
  // (20 = 18 + 2 halo), stage 2 6 x 3 -- no idle rows; under the bench's
  // sustained, power-capped load 1203 -> 1295 GCells/s (6 x 3 / 6 x 3: 1247).
  // fp64: 16 rows, 6 x 3 / 6 x 3 (2048^2 x 258 660 -> 720 in short runs).
#ifndef SSAM_P2_ROWS
#define SSAM_P2_ROWS (sizeof(T) == 4 ? 18 : 16)
#endif
#ifndef SSAM_P2_SY1
#define SSAM_P2_SY1 (sizeof(T) == 4 ? 5 : 6)
#define SSAM_P2_RY1 (sizeof(T) == 4 ? 4 : 3)
#define SSAM_P2_SY2 6
#define SSAM_P2_RY2 3
#endif
  static constexpr int ROWS = (TB == 2 && K == 1) ? static_cast<int>(SSAM_P2_ROWS) : 16;
  static constexpr int sy(int s) {
    if (K == 2) return TB == 1 ? 8 : (s == 1 ? 10 : 8);
    return TB == 1 ? 4
         : TB == 2 ? (s == 1 ? SSAM_P2_SY1 : SSAM_P2_SY2)
         : TB == 3 ? (s == 1 ? 5 : s == 2 ? 6 : 4)
                   : (s == 1 ? 4 : s == 2 ? 5 : s == 3 ? 6 : 4);
  }
  static constexpr int ry(int s) {
    if (K == 2) return 2;
    return TB == 1 ? 4
         : TB == 2 ? (s == 1 ? SSAM_P2_RY1 : SSAM_P2_RY2)
         : TB == 3 ? (s == 1 ? 4 : s == 2 ? 3 : 4)
                   : (s == 1 ? 6 : s == 2 ? 4 : s == 3 ? 3 : 4);
  }
  static constexpr int nr(int s) { return ROWS + 2 * K * (TB - s); }
  static constexpr int first_warp(int s) {
    int w = 0;
    for (int i = 1; i < s; ++i) w += sy(i);
    return w;
  }
  static constexpr int CWARPS = first_warp(TB + 1);
  static constexpr int THREADS = 32 * (CWARPS + 1);  // + the TMA producer warp
#ifndef SSAM_STAR_DZ
#define SSAM_STAR_DZ 6
#endif
#ifndef SSAM_STAR_DI
#define SSAM_STAR_DI 3
#endif
  // input / intermediate ring depth: a stage holds the 2K+1 planes of its
  // first step before it releases any, so a ring needs at least 2K+1 slots
#ifndef SSAM_STAR_DZ1
#define SSAM_STAR_DZ1 SSAM_STAR_DZ
#endif
  // single sweeps of the order-2 star keep 8 planes in flight (3d13pt
  // 512^3 f32 612 -> 656, f64 360 -> 370; profiles/r02/dz1_ab.txt)
  static constexpr int DZW = TB == 1 ? (K == 2 ? 8 : SSAM_STAR_DZ1) : SSAM_STAR_DZ;
  static constexpr int DZ = DZW > 2 * K + 2 ? DZW : 2 * K + 2;
  static constexpr int DI = SSAM_STAR_DI > 2 * K + 1 ? SSAM_STAR_DI : 2 * K + 1;
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int IN_ROWS = cmax(sy(1) * ry(1) + 2 * K, nr(1) + 2 * K);
  // slot rows of the ring between stage s and s+1: written by s, read by s+1
  static constexpr int mid_rows(int s) {
    return cmax(sy(s) * ry(s), sy(s + 1) * ry(s + 1) + 2 * K);
  }
  static constexpr size_t al(size_t b) { return (b + 127) / 128 * 128; }
  static constexpr size_t IN_SLOT = al(size_t(IN_ROWS) * BW * sizeof(T));
  static constexpr size_t mid_slot(int s) { return al(size_t(mid_rows(s)) * BW * sizeof(T)); }
  static constexpr size_t mid_off(int s) {
    size_t o = DZ * IN_SLOT;
    for (int i = 1; i < s; ++i) o += DI * mid_slot(i);
    return o;
  }
  static constexpr size_t BAR_OFF = mid_off(TB);
  static constexpr size_t SMEM = BAR_OFF + (2 * DZ + 2 * DI * (TB - 1)) * 8;
#ifndef SSAM_STAR_MINB2
#define SSAM_STAR_MINB2 2
#endif
  // resident CTAs per SM the register budget is planned for
  // (the box family holds all RY + 2 rows of three planes: one CTA per SM
  // when fused)
  static constexpr int MINB = !STAR && TB > 1 ? 1
                            : THREADS <= 160 ? 3
                            : (THREADS <= 352 ? (TB == 2 ? SSAM_STAR_MINB2 : 2)
                                              : (TB == 2 && K == 1 && THREADS <= 512 ? SSAM_STAR_MINB2 : 1));
  static constexpr int CAP = (2 * K + 1) * (2 * K + 1) * (2 * K + 1);
  static_assert(IN_ROWS <= 256, "TMA box rows");
  static_assert(K <= Q, "x halo within one neighbour lane");
};

struct PipeCtx {
  unsigned char* smem;
  int lane;
  int x0, base, x_out0;  // this lane's first column, strip box origin, owned columns start
  int y_cta0;            // first output row of the CTA
  int z0, nseg;          // first output plane, planes in this segment
  bool edge;             // the CTA's bands touch the x or y ring
};

template <class G>
__device__ __forceinline__ uint64_t* pipe_bar(unsigned char* smem, int idx) {
  return reinterpret_cast<uint64_t*>(smem + G::BAR_OFF) + idx;
}
// barrier indices: in_full [0,DZ), in_empty [DZ,2DZ), then per ring s = 1..TB-1:
// full [2DZ + 2DI(s-1), +DI), empty [+DI, +2DI)
template <class G> __device__ __forceinline__ int bi_full(int s) {
  return s == 0 ? 0 : 2 * G::DZ + 2 * G::DI * (s - 1);
}
template <class G> __device__ __forceinline__ int bi_empty(int s) {
  return s == 0 ? G::DZ : 2 * G::DZ + 2 * G::DI * (s - 1) + G::DI;
}

// ---- the per-cell chains (shared by the pipeline and the direct kernel) ----

// Box-family column partial j (dx = j-1) of order 1: the mask's taps of that
// column, dz outer, dy inner, first product rounded.  sv(l, t) returns the
// sample at dz = l-1, dy = t-1 in that column.
template <class T, class Mask, class P, class FS>
__device__ __forceinline__ T pipe_box_col(const P& p, int j, FS sv) {
  T v = T(0);
  bool first = true;
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int t = 0; t < 3; ++t)
      if (Mask::has(j, t, l)) {
        const T c = p.coef[(l * 3 + j) * 3 + t];
        v = first ? mul_t(c, sv(l, t)) : fma_t(c, sv(l, t), v);
        first = false;
      }
  return v;
}
#ifndef SSAM_BOX_JOIN
#define SSAM_BOX_JOIN 1
#endif
// out(x) = L(x-1), then the dx = 0 column's taps FMA'd into it, then
// + R(x+1) (L / R the dx = -1 / +1 column partials, shifted across lanes):
// 28 FP instructions per 27-point cell instead of 29 for (C + L) + R.
// sv(l, t) returns the sample at dz = l-1, dy = t-1 of the centre column.
template <class T, class Mask, class P, class FS>
__device__ __forceinline__ T pipe_box_cell(const P& p, T lft, T rgt, FS sv) {
#if SSAM_BOX_JOIN
  T v = lft;
#pragma unroll
  for (int l = 0; l < 3; ++l)
#pragma unroll
    for (int t = 0; t < 3; ++t)
      if (Mask::has(1, t, l)) v = fma_t(p.coef[(l * 3 + 1) * 3 + t], sv(l, t), v);
  return add_t(v, rgt);
#else
  return add_t(add_t(pipe_box_col<T, Mask>(p, 1, sv), lft), rgt);
#endif
}

// One stage of the pipeline (sweep S of TB) for warp w of the stage.
template <class T, class Sh, int TB, int S, bool PEER, class Par>
__device__ __forceinline__ void pipe_stage(const Par& p, const PipeCtx& c, int w) {
  using G = PipeGeom<T, Sh, TB>;
  constexpr int K = Sh::K, NPL = 2 * K + 1;
  constexpr int Q = G::Q, BW = G::BW, RY = G::ry(S), NROW = RY + 2 * K;
  constexpr int D = S == 1 ? G::DZ : G::DI;  // source ring depth
  constexpr size_t SLOT = S == 1 ? G::IN_SLOT : G::mid_slot(S > 1 ? S - 1 : 1);
  constexpr bool LAZY = Sh::STAR;  // stars read the halo rows of the centre plane late
  const int lane = c.lane;
  const unsigned char* src = c.smem + (S == 1 ? 0 : G::mid_off(S > 1 ? S - 1 : 1));
  uint64_t* sfull = pipe_bar<G>(c.smem, bi_full<G>(S - 1));
  uint64_t* sempty = pipe_bar<G>(c.smem, bi_empty<G>(S - 1));
  const int n_out = c.nseg + 2 * K * (TB - S);  // planes this stage produces
  const int zfirst = c.z0 - K * (TB - S);       // plane of output m = zfirst + m
  const int band0 = -K * (TB - S);              // band row b <-> y = y_cta0 + band0 + b
  const int row0 = w * RY;                      // this warp's first band row

  auto slot_ptr = [&](int j) -> const T* {
    return reinterpret_cast<const T*>(src + static_cast<size_t>(j % D) * SLOT) + row0 * BW +
           Q * lane;
  };
  // plane j arrives: wait for it, read its rows (stars: the RY centre rows)
  auto take = [&](int j, T (&dst)[NROW][Q]) {
    mbar_wait(smem_u32(&sfull[j % D]), (j / D) & 1);
    const T* sp = slot_ptr(j);
#pragma unroll
    for (int r = LAZY ? K : 0; r < (LAZY ? K + RY : NROW); ++r) lds_q<T, Q>(sp + r * BW, dst[r]);
  };
  auto halo = [&](int j, T (&dst)[NROW][Q]) {
    if constexpr (LAZY) {
      const T* sp = slot_ptr(j);
#pragma unroll
      for (int r = 0; r < K; ++r) {
        lds_q<T, Q>(sp + r * BW, dst[r]);
        lds_q<T, Q>(sp + (RY + K + r) * BW, dst[RY + K + r]);
      }
    }
  };
  auto release = [&](int j) { mbar_arrive(smem_u32(&sempty[j % D])); };

  // destination
  [[maybe_unused]] T* dst_ring = nullptr;
  [[maybe_unused]] uint64_t* dfull = nullptr;
  [[maybe_unused]] uint64_t* dempty = nullptr;
  if constexpr (S < TB) {
    dst_ring = reinterpret_cast<T*>(c.smem + G::mid_off(S));
    dfull = pipe_bar<G>(c.smem, bi_full<G>(S));
    dempty = pipe_bar<G>(c.smem, bi_empty<G>(S));
  }
  const int xlo = K, xhi = p.nx - K, ylo = K, yhi = p.ny - K;
  const bool owner = c.x0 >= c.x_out0 && c.x0 < c.x_out0 + p.V;
  const bool vec = c.x0 >= xlo && c.x0 + Q <= xhi;

  T pl[NPL][NROW][Q];
#pragma unroll
  for (int i = 0; i < 2 * K; ++i) take(i, pl[i]);

  for (int mb = 0; mb < n_out; mb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int m = mb + ph;
      if (m >= n_out) break;
      take(m + 2 * K, pl[(ph + 2 * K) % NPL]);
      T(&cen)[NROW][Q] = pl[(ph + K) % NPL];
      halo(m + K, cen);
      const int z = zfirst + m;
      if constexpr (S < TB) {
        if (m >= G::DI) mbar_wait(smem_u32(&dempty[m % G::DI]), ((m / G::DI) - 1) & 1);
      }
      const bool zring = z < p.zr_lo || z >= p.zr_hi;
      [[maybe_unused]] const bool mirror = PEER && S == TB && mirrored3(p, z);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const T(&cr)[Q] = cen[r + K];
        T out[Q];
        if constexpr (Sh::STAR) {
          T lft[K], rgt[K];
#pragma unroll
          for (int i = 0; i < K; ++i) {
            lft[i] = shfl_up(cr[Q - K + i], 1);
            rgt[i] = __shfl_down_sync(kFull, cr[i], 1);
          }
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            auto xv = [&](int d) {
              const int qq = q + d;
              return qq < 0 ? lft[K + qq] : (qq >= Q ? rgt[qq - Q] : cr[qq]);
            };
            auto yv = [&](int d) { return cen[r + K + d][q]; };
            auto zv = [&](int d) { return pl[(ph + K + d) % NPL][r + K][q]; };
            out[q] = pipe_star_cell<T, K>(p, cr[q], xv, yv, zv);
          }
        } else {
          T L[Q], R[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            auto sv = [&](int l, int t) { return pl[(ph + l) % NPL][r + t][q]; };
            L[q] = pipe_box_col<T, typename Sh::Mask>(p, 0, sv);
            R[q] = pipe_box_col<T, typename Sh::Mask>(p, 2, sv);
          }
          const T lL = shfl_up(L[Q - 1], 1);
          const T rR = __shfl_down_sync(kFull, R[0], 1);
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            auto sv = [&](int l, int t) { return pl[(ph + l) % NPL][r + t][q]; };
            out[q] = pipe_box_cell<T, typename Sh::Mask>(p, q == 0 ? lL : L[q - 1],
                                                         q == Q - 1 ? rR : R[q + 1], sv);
          }
        }
        const int y = c.y_cta0 + band0 + row0 + r;
        if constexpr (S < TB) {
          // the global ring keeps its value through every sweep
          if (zring || c.edge) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              const int x = c.x0 + q;
              if (zring || y < ylo || y >= yhi || x < xlo || x >= xhi) out[q] = cr[q];
            }
          }
          st_q<T, Q>(dst_ring + static_cast<size_t>(m % G::DI) * (G::mid_slot(S) / sizeof(T)) +
                         (row0 + r) * BW + Q * lane,
                     out);
        } else {
          if (owner && y < yhi && (G::sy(S) * RY == G::ROWS || row0 + r < G::ROWS))
            store_row3<T, Q>(p, z, y, c.x0, out, vec, xlo, xhi, mirror);
        }
      }
      if constexpr (S < TB) mbar_arrive(smem_u32(&dfull[m % G::DI]));
      if constexpr (LAZY) {
        release(m + K);  // its halo rows fed this step's FMAs; the slot may refill
        if (m < K) release(m);  // planes 0..K-1 are never the centre
      } else {
        release(m + 2 * K);  // every row of the new plane fed this step's FMAs
        if (m == 0) {
#pragma unroll
          for (int i = 0; i < 2 * K; ++i) release(i);
        }
      }
    }
  }
  if constexpr (LAZY) {
#pragma unroll
    for (int i = 0; i < K; ++i) release(n_out + K + i);  // only ever z+ planes
  }
}

template <class T, class Sh, int TB, int S, bool PEER, class Par>
__device__ __forceinline__ void pipe_dispatch(const Par& p, const PipeCtx& c, int wib) {
  using G = PipeGeom<T, Sh, TB>;
  if constexpr (S <= TB) {
    if (wib < G::first_warp(S + 1)) {
      pipe_stage<T, Sh, TB, S, PEER>(p, c, wib - G::first_warp(S));
      return;
    }
    pipe_dispatch<T, Sh, TB, S + 1, PEER>(p, c, wib);
  }
}

template <class T, class Sh, int TB, bool PEER>
__global__ void __launch_bounds__(PipeGeom<T, Sh, TB>::THREADS, PipeGeom<T, Sh, TB>::MINB)
    pipe3d_kernel(const __grid_constant__ Ssam3DTmaParams<T, PipeGeom<T, Sh, TB>::CAP> P) {
  using G = PipeGeom<T, Sh, TB>;
  constexpr int K = Sh::K;
  const auto& p = P.p;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  // warp index via a shuffle so the compiler treats the role branches as
  // warp-uniform (coefficients then stay uniform-register FFMA operands)
  const int wib = __shfl_sync(kFull, static_cast<int>(threadIdx.x >> 5), 0);

  PipeCtx c;
  c.smem = smem_raw;
  c.lane = lane;
  c.x_out0 = blockIdx.x * p.V;
  c.base = c.x_out0 - p.A;
  c.x0 = c.base + G::Q * lane;
  c.y_cta0 = K + blockIdx.y * G::ROWS;
  c.z0 = p.z_begin + blockIdx.z * p.zseg;
  c.nseg = min(p.zseg, p.z_end - c.z0);
  // (generous in y: rows a stage computes past its band feed nothing)
  c.edge = c.base < K || c.base + G::BW > p.nx - K || c.y_cta0 - K * TB < K ||
           c.y_cta0 + G::ROWS + 2 * K * TB + 8 > p.ny - K;

  if (threadIdx.x == 0) {
    prefetch_tmap(&P.tmap);
    for (int s = 0; s < G::DZ; ++s) {
      mbar_init(smem_u32(pipe_bar<G>(smem_raw, s)), 1);
      mbar_init(smem_u32(pipe_bar<G>(smem_raw, G::DZ + s)), 32 * G::sy(1));
    }
    for (int r = 1; r < TB; ++r)
      for (int s = 0; s < G::DI; ++s) {
        mbar_init(smem_u32(pipe_bar<G>(smem_raw, bi_full<G>(r) + s)), 32 * G::sy(r));
        mbar_init(smem_u32(pipe_bar<G>(smem_raw, bi_empty<G>(r) + s)), 32 * G::sy(r + 1));
      }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains

  if (wib == G::CWARPS) {
    // TMA producer: input plane i <-> z = z0 - K TB + i, box rows from y_cta0 - K TB
    if (lane != 0) return;
    const int n_in = c.nseg + 2 * K * TB;
    const uint32_t bytes = static_cast<uint32_t>(G::IN_ROWS * G::BW * sizeof(T));
    for (int i = 0; i < n_in; ++i) {
      const int s = i % G::DZ;
      if (i >= G::DZ) {
        mbar_wait(smem_u32(pipe_bar<G>(smem_raw, G::DZ + s)), ((i / G::DZ) - 1) & 1);
        fence_proxy_async();
      }
      const uint32_t bar = smem_u32(pipe_bar<G>(smem_raw, s));
      const int z = c.z0 - K * TB + i;
      const int row = (z >= 0 && z < p.nz) ? z * p.ny + (c.y_cta0 - K * TB) : -G::IN_ROWS;
      mbar_arrive_expect_tx(bar, bytes);
      tma_load_2d(smem_u32(smem_raw + s * G::IN_SLOT), &P.tmap, c.base, row, bar);
    }
    return;
  }
  pipe_dispatch<T, Sh, TB, 1, PEER>(p, c, wib);
}

// Direct-load single sweep (rows not 16-byte aligned): one cell per thread,
// the same per-cell chains.
template <class T, class Sh, bool PEER, int CAP>
__global__ void __launch_bounds__(128) pipe3d_direct_kernel(const __grid_constant__ Ssam3DParams<T, CAP> p) {
  constexpr int K = Sh::K;
  const int x = K + blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= p.nx - K) return;
  const long long sy = p.nx, sz = static_cast<long long>(p.nx) * p.ny;
  const T* in = p.in;
  for (int z = p.z_begin + blockIdx.z; z < p.z_end; z += gridDim.z)
    for (int y = K + blockIdx.y; y < p.ny - K; y += gridDim.y) {
      const long long i = (static_cast<long long>(z) * p.ny + y) * p.nx + x;
      T v;
      if constexpr (Sh::STAR) {
        v = pipe_star_cell<T, K>(
            p, __ldg(in + i), [&](int d) { return __ldg(in + i + d); },
            [&](int d) { return __ldg(in + i + d * sy); },
            [&](int d) { return __ldg(in + i + d * sz); });
      } else {
        auto col = [&](int j) {
          return pipe_box_col<T, typename Sh::Mask>(
              p, j, [&](int l, int t) { return __ldg(in + i + (j - 1) + (l - 1) * sz + (t - 1) * sy); });
        };
        v = pipe_box_cell<T, typename Sh::Mask>(
            p, col(0), col(2), [&](int l, int t) { return __ldg(in + i + (l - 1) * sz + (t - 1) * sy); });
      }
      p.out[i] = v;
      if (PEER) {
        if (p.peer_lo != nullptr && z < p.peer_lo_end) p.peer_lo[i + p.peer_lo_shift] = v;
        if (p.peer_hi != nullptr && z >= p.peer_hi_begin) p.peer_hi[i + p.peer_hi_shift] = v;
      }
    }
}

}  // namespace ssam_b200
