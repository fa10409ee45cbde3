// engine3d_star.cuh -- the order-1 3D star (3d7pt) as a TB-stage warp
// pipeline: TB Jacobi sweeps per pass over HBM, sm_100a.
//
// Reference semantics: ssam::stencil3d (proj/include/ssam/kernels.hpp:283-384)
// applied TB times (temporal blocking is Tb consecutive sweeps):
// every sweep writes the interior [1, n-1) per axis and carries the ring.
//
// One CTA owns an x-strip (32 lanes x Q columns, lane plan A/V as the other
// engines), ROWS output rows and a z-segment.  Its warps form TB stages plus
// one producer warp:
//
//   producer   TMA: input plane boxes (strip x (rows + 2 TB)) into a ring of
//              DZ slots (full = transaction count, empty = stage-1 lanes);
//   stage s    streams the planes of stage s-1 (stage 0 = the TMA ring) and
//              computes sweep s for its band: ROWS + 2 (TB - s) rows, each
//              warp RY(s) of them.  Stages < TB write their planes to a
//              shared-memory ring (DI slots, full = producer lanes, empty =
//              consumer lanes); stage TB stores the interior to HBM.
//
// Per output row a lane holds its Q columns of three source planes in
// registers (z-streaming): the centre plane's RY + 2 rows, only the RY
// centre rows of the z-1 / z+1 planes (the star never reads their y
// neighbours; a plane's two halo rows are read from its slot when it
// becomes the centre).  x neighbours at the lane's ends come from one
// shfl_up and one shfl_down of the centre row; nothing else moves between
// lanes.  Each cell is ONE fixed FMA chain (star7_cell), so every kernel of
// this family -- any TB, aligned or direct-load -- gives bit-identical
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

// out = c0*c + cxm*xm + cxp*xp + cym*ym + cyp*yp + czm*zm + czp*zp as one
// chain (first product rounded, then six FMAs).  coef index (l*3+j)*3+t with
// l = dz+1, j = dx+1, t = dy+1 (engine3d.cuh).
template <class T, class P>
__device__ __forceinline__ T star7_cell(const P& p, T c, T xm, T xp, T ym, T yp, T zm, T zp) {
  T v = p.coef[13] * c;
  v = fma_t(p.coef[10], xm, v);
  v = fma_t(p.coef[16], xp, v);
  v = fma_t(p.coef[12], ym, v);
  v = fma_t(p.coef[14], yp, v);
  v = fma_t(p.coef[4], zm, v);
  v = fma_t(p.coef[22], zp, v);
  return v;
}

// Geometry of one (T, TB) pipeline.  Stage s (1..TB) has sy(s) warps of
// ry(s) rows; sy(s) * ry(s) >= nr(s) = ROWS + 2 (TB - s).
template <class T, int TB_>
struct StarGeom {
  static constexpr int TB = TB_;
  static constexpr int Q = 16 / static_cast<int>(sizeof(T));
  static constexpr int BW = 32 * Q;  // strip / box / slot row width
  static constexpr int ROWS = 16;
  // (warps, rows) per stage, chosen so each stage's band is covered exactly
  static constexpr int sy(int s) {
    return TB == 1 ? 4
         : TB == 2 ? (s == 1 ? 6 : 4)
         : TB == 3 ? (s == 1 ? 5 : s == 2 ? 6 : 4)
                   : (s == 1 ? 4 : s == 2 ? 5 : s == 3 ? 6 : 4);
  }
  static constexpr int ry(int s) {
    return TB == 1 ? 4
         : TB == 2 ? (s == 1 ? 3 : 4)
         : TB == 3 ? (s == 1 ? 4 : s == 2 ? 3 : 4)
                   : (s == 1 ? 6 : s == 2 ? 4 : s == 3 ? 3 : 4);
  }
  static constexpr int nr(int s) { return ROWS + 2 * (TB - s); }
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
  static constexpr int DZ = SSAM_STAR_DZ, DI = SSAM_STAR_DI;  // input / intermediate ring depth
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int IN_ROWS = cmax(sy(1) * ry(1) + 2, nr(1) + 2);
  // slot rows of the ring between stage s and s+1: written by s, read by s+1
  static constexpr int mid_rows(int s) { return cmax(sy(s) * ry(s), sy(s + 1) * ry(s + 1) + 2); }
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
  static constexpr int MINB = TB == 1 ? 3 : (TB == 2 ? SSAM_STAR_MINB2 : 1);
  static_assert(IN_ROWS <= 256, "TMA box rows");
};

template <class T, int TB>
struct StarCtx {
  unsigned char* smem;
  int lane;
  int x0, base, x_out0;  // this lane's first column, strip box origin, owned columns start
  int y_cta0;            // first output row of the CTA
  int z0, nseg;          // first output plane, planes in this segment
  bool edge;             // the CTA's bands touch the x or y ring
};

template <class T, int TB>
__device__ __forceinline__ uint64_t* star_bar(unsigned char* smem, int idx) {
  return reinterpret_cast<uint64_t*>(smem + StarGeom<T, TB>::BAR_OFF) + idx;
}
// barrier indices: in_full [0,DZ), in_empty [DZ,2DZ), then per ring s = 1..TB-1:
// full [2DZ + 2DI(s-1), +DI), empty [+DI, +2DI)
template <class T, int TB> __device__ __forceinline__ int bi_full(int s) {
  using G = StarGeom<T, TB>;
  return s == 0 ? 0 : 2 * G::DZ + 2 * G::DI * (s - 1);
}
template <class T, int TB> __device__ __forceinline__ int bi_empty(int s) {
  using G = StarGeom<T, TB>;
  return s == 0 ? G::DZ : 2 * G::DZ + 2 * G::DI * (s - 1) + G::DI;
}

// One stage of the pipeline (sweep S of TB) for warp w of the stage.
template <class T, int TB, int S, bool PEER, class Par>
__device__ __forceinline__ void star_stage(const Par& p, const StarCtx<T, TB>& c, int w) {
  using G = StarGeom<T, TB>;
  constexpr int Q = G::Q, BW = G::BW, RY = G::ry(S), NROW = RY + 2;
  constexpr int D = S == 1 ? G::DZ : G::DI;  // source ring depth
  constexpr size_t SLOT = S == 1 ? G::IN_SLOT : G::mid_slot(S > 1 ? S - 1 : 1);
  const int lane = c.lane;
  const unsigned char* src = c.smem + (S == 1 ? 0 : G::mid_off(S > 1 ? S - 1 : 1));
  uint64_t* sfull = star_bar<T, TB>(c.smem, bi_full<T, TB>(S - 1));
  uint64_t* sempty = star_bar<T, TB>(c.smem, bi_empty<T, TB>(S - 1));
  const int n_out = c.nseg + 2 * (TB - S);   // planes this stage produces
  const int zfirst = c.z0 - (TB - S);        // plane of output m = zfirst + m
  const int band0 = -(TB - S);               // band row b <-> y = y_cta0 + band0 + b
  const int row0 = w * RY;                   // this warp's first band row

  auto slot_ptr = [&](int j) -> const T* {
    return reinterpret_cast<const T*>(src + static_cast<size_t>(j % D) * SLOT) + row0 * BW + Q * lane;
  };
  // plane j arrives: wait for it, read its RY centre rows (rows 1..RY)
#ifndef SSAM_STAR_EAGER
#define SSAM_STAR_EAGER 0
#endif
  // EAGER: all RY + 2 rows at arrival (slot released one step earlier, two
  // more rows of registers per plane); lazy: halo rows when centre.
  constexpr bool EAGER = SSAM_STAR_EAGER != 0;
  auto take = [&](int j, T (&dst)[NROW][Q]) {
    mbar_wait(smem_u32(&sfull[j % D]), (j / D) & 1);
    const T* sp = slot_ptr(j);
#pragma unroll
    for (int r = EAGER ? 0 : 1; r <= (EAGER ? RY + 1 : RY); ++r) lds_q<T, Q>(sp + r * BW, dst[r]);
  };
  auto halo = [&](int j, T (&dst)[NROW][Q]) {
    if constexpr (!EAGER) {
      const T* sp = slot_ptr(j);
      lds_q<T, Q>(sp, dst[0]);
      lds_q<T, Q>(sp + (RY + 1) * BW, dst[RY + 1]);
    }
  };
  auto release = [&](int j) { mbar_arrive(smem_u32(&sempty[j % D])); };

  // destination
  [[maybe_unused]] T* dst_ring = nullptr;
  [[maybe_unused]] uint64_t* dfull = nullptr;
  [[maybe_unused]] uint64_t* dempty = nullptr;
  if constexpr (S < TB) {
    dst_ring = reinterpret_cast<T*>(c.smem + G::mid_off(S));
    dfull = star_bar<T, TB>(c.smem, bi_full<T, TB>(S));
    dempty = star_bar<T, TB>(c.smem, bi_empty<T, TB>(S));
  }
  const int xlo = 1, xhi = p.nx - 1, ylo = 1, yhi = p.ny - 1;
  const bool owner = c.x0 >= c.x_out0 && c.x0 < c.x_out0 + p.V;
  const bool vec = c.x0 >= xlo && c.x0 + Q <= xhi;

  T pl[3][NROW][Q];
  take(0, pl[0]);
  take(1, pl[1]);

  auto step = [&](int m, const T (&zm)[NROW][Q], T (&cen)[NROW][Q], const T (&zp)[NROW][Q]) {
    halo(m + 1, cen);
    const int z = zfirst + m;
    if constexpr (S < TB) {
      const int s = m % G::DI;
      if (m >= G::DI) mbar_wait(smem_u32(&dempty[s]), ((m / G::DI) - 1) & 1);
    }
    const bool zring = z < p.zr_lo || z >= p.zr_hi;
    [[maybe_unused]] const bool mirror = PEER && S == TB && mirrored3(p, z);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const T(&cr)[Q] = cen[r + 1];
      const T xl = shfl_up(cr[Q - 1], 1);
      const T xr = __shfl_down_sync(kFull, cr[0], 1);
      T out[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const T xm = q == 0 ? xl : cr[q - 1];
        const T xp = q == Q - 1 ? xr : cr[q + 1];
        out[q] = star7_cell<T>(p, cr[q], xm, xp, cen[r][q], cen[r + 2][q], zm[r + 1][q],
                               zp[r + 1][q]);
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
    if constexpr (EAGER) {
      release(m + 2);  // every row of the new plane fed this step's FMAs
      if (m == 0) {
        release(0);
        release(1);
      }
    } else {
      release(m + 1);  // its halo rows fed this step's FMAs; the slot may refill
      if (m == 0) release(0);
    }
  };

  for (int mb = 0; mb < n_out; mb += 3) {
    take(mb + 2, pl[2]);
    step(mb, pl[0], pl[1], pl[2]);
    if (mb + 1 >= n_out) break;
    take(mb + 3, pl[0]);
    step(mb + 1, pl[1], pl[2], pl[0]);
    if (mb + 2 >= n_out) break;
    take(mb + 4, pl[1]);
    step(mb + 2, pl[2], pl[0], pl[1]);
  }
  if constexpr (!EAGER) release(n_out + 1);  // the last plane was only ever a z+1 plane
}

template <class T, int TB, int S, bool PEER, class Par>
__device__ __forceinline__ void star_dispatch(const Par& p, const StarCtx<T, TB>& c, int wib) {
  using G = StarGeom<T, TB>;
  if constexpr (S <= TB) {
    if (wib < G::first_warp(S + 1)) {
      star_stage<T, TB, S, PEER>(p, c, wib - G::first_warp(S));
      return;
    }
    star_dispatch<T, TB, S + 1, PEER>(p, c, wib);
  }
}

template <class T, int TB, bool PEER>
__global__ void __launch_bounds__(StarGeom<T, TB>::THREADS, StarGeom<T, TB>::MINB)
    star3d_kernel(const __grid_constant__ Ssam3DTmaParams<T, 27> P) {
  using G = StarGeom<T, TB>;
  const Ssam3DParams<T, 27>& p = P.p;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  // warp index via a shuffle so the compiler treats the role branches as
  // warp-uniform (coefficients then stay uniform-register FFMA operands)
  const int wib = __shfl_sync(kFull, static_cast<int>(threadIdx.x >> 5), 0);

  StarCtx<T, TB> c;
  c.smem = smem_raw;
  c.lane = lane;
  c.x_out0 = blockIdx.x * p.V;
  c.base = c.x_out0 - p.A;
  c.x0 = c.base + G::Q * lane;
  c.y_cta0 = 1 + blockIdx.y * G::ROWS;
  c.z0 = p.z_begin + blockIdx.z * p.zseg;
  c.nseg = min(p.zseg, p.z_end - c.z0);
  // (generous in y: rows a stage computes past its band feed nothing)
  c.edge = c.base < 1 || c.base + G::BW > p.nx - 1 || c.y_cta0 - TB < 1 ||
           c.y_cta0 + G::ROWS + 2 * TB + 8 > p.ny - 1;

  if (threadIdx.x == 0) {
    prefetch_tmap(&P.tmap);
    for (int s = 0; s < G::DZ; ++s) {
      mbar_init(smem_u32(star_bar<T, TB>(smem_raw, s)), 1);
      mbar_init(smem_u32(star_bar<T, TB>(smem_raw, G::DZ + s)), 32 * G::sy(1));
    }
    for (int r = 1; r < TB; ++r)
      for (int s = 0; s < G::DI; ++s) {
        mbar_init(smem_u32(star_bar<T, TB>(smem_raw, bi_full<T, TB>(r) + s)), 32 * G::sy(r));
        mbar_init(smem_u32(star_bar<T, TB>(smem_raw, bi_empty<T, TB>(r) + s)), 32 * G::sy(r + 1));
      }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains

  if (wib == G::CWARPS) {
    // TMA producer: input plane i <-> z = z0 - TB + i, box rows from y_cta0 - TB
    if (lane != 0) return;
    const int n_in = c.nseg + 2 * TB;
    const uint32_t bytes = static_cast<uint32_t>(G::IN_ROWS * G::BW * sizeof(T));
    for (int i = 0; i < n_in; ++i) {
      const int s = i % G::DZ;
      if (i >= G::DZ) {
        mbar_wait(smem_u32(star_bar<T, TB>(smem_raw, G::DZ + s)), ((i / G::DZ) - 1) & 1);
        fence_proxy_async();
      }
      const uint32_t bar = smem_u32(star_bar<T, TB>(smem_raw, s));
      const int z = c.z0 - TB + i;
      const int row = (z >= 0 && z < p.nz) ? z * p.ny + (c.y_cta0 - TB) : -G::IN_ROWS;
      mbar_arrive_expect_tx(bar, bytes);
      tma_load_2d(smem_u32(smem_raw + s * G::IN_SLOT), &P.tmap, c.base, row, bar);
    }
    return;
  }
  star_dispatch<T, TB, 1, PEER>(p, c, wib);
}

// Direct-load single sweep (rows not 16-byte aligned): one cell per thread,
// the same star7_cell chain.
template <class T, bool PEER>
__global__ void __launch_bounds__(128) star3d_direct_kernel(const __grid_constant__ Ssam3DParams<T, 27> p) {
  const int x = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= p.nx - 1) return;
  const size_t sxy = static_cast<size_t>(p.nx) * p.ny;
  const T* in = p.in;
  for (int z = p.z_begin + blockIdx.z; z < p.z_end; z += gridDim.z)
    for (int y = 1 + blockIdx.y; y < p.ny - 1; y += gridDim.y) {
      const size_t i = (static_cast<size_t>(z) * p.ny + y) * p.nx + x;
      const T v = star7_cell<T>(p, __ldg(in + i), __ldg(in + i - 1), __ldg(in + i + 1),
                                __ldg(in + i - p.nx), __ldg(in + i + p.nx), __ldg(in + i - sxy),
                                __ldg(in + i + sxy));
      p.out[i] = v;
      if (PEER) {
        if (p.peer_lo != nullptr && z < p.peer_lo_end) p.peer_lo[i + p.peer_lo_shift] = v;
        if (p.peer_hi != nullptr && z >= p.peer_hi_begin) p.peer_hi[i + p.peer_hi_shift] = v;
      }
    }
}

}  // namespace ssam_b200
