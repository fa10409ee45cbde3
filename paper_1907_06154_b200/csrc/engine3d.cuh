// engine3d.cuh -- the 3D SSAM engine (3D stencil Jacobi sweeps), sm_100a.
//
// The reference maps one warp to one x-y plane and sums the per-dz partials
// through a block-shared InterWarpBuffer (kernels.hpp:283-384,
// blocking.hpp:82-97).  On Blackwell that smem round trip
// and the 2k/warp_count plane re-loads are unnecessary: each warp owns an
// x-strip (32 lanes x Q columns) x RY output rows and STREAMS along z,
// keeping the 2K+1 most recent input planes of its (RY+2K) x Q footprint in
// registers (z-streaming).  Per output row the chain is
// the systolic one of the 2D engine (bidirectional, see engine2d.cuh) with
// the column partial now folding every (dy, dz) tap of that dx column:
//     colpart_j = sum_{l,t} c(dx=j-K, dy=t-K, dz=l-K) * plane[l][row+t]
// Planes arrive as 2D TMA boxes (one per plane, DZ planes in flight per
// warp) from a (nx, ny*nz) view of the grid; unaligned grids fall back to
// direct loads.  Only interior cells [K, n-K) per axis are written; the ring
// of width K is carried by both ping-pong buffers (set up once per call) --
// the reference's next = cur copy (kernels.hpp:323) without a per-sweep copy.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "engine2d.cuh"

namespace ssam_b200 {

template <class T, int CAP>
struct Ssam3DParams {
  const T* in;
  T* out;
  int nx, ny, nz;
  int A, V;         // lane plan (as in 2D, M = 2K+1)
  int nstrips;
  int ygroups;      // groups of RY interior rows
  int zseg;         // output planes streamed per warp
  int z_begin, z_end;
  int ring;         // = K
  int vec_ok;
  int cta_sx;       // TMA kernel: adjacent x-strips per CTA (sharing one box)
  int zfast;        // TMA kernels: grid is (x, z-segment, y-group) instead of (x, y, z)
  int zr_lo, zr_hi; // fused (Tb > 1) kernel: planes outside [zr_lo, zr_hi) are global ring
  // Peer-memory halo (slab runs, ssam_peer_halo): output planes z < peer_lo_end
  // are also stored to peer_lo at element offset + peer_lo_shift, planes
  // z >= peer_hi_begin to peer_hi (the neighbours' ghost slots).
  T* peer_lo;
  T* peer_hi;
  long long peer_lo_shift, peer_hi_shift;
  int peer_lo_end, peer_hi_begin;
  T coef[CAP];      // coef[(l*M + j)*M + t], l = dz+K, j = dx+K, t = dy+K
};

template <class T, int CAP>
struct alignas(64) Ssam3DTmaParams {
  CUtensorMap tmap;  // (nx, ny*nz) row-major view, box 32Q x (RY+2K)
  Ssam3DParams<T, CAP> p;
};

struct DenseMask3 {
  __host__ __device__ static constexpr bool has(int, int, int) { return true; }
};
// Star: at most one of dx, dy, dz is non-zero.
template <int K>
struct StarMask3 {
  __host__ __device__ static constexpr bool has(int j, int t, int l) {
    return (j == K && t == K) || (j == K && l == K) || (t == K && l == K);
  }
};
// Poisson 19-point: |dx| + |dy| + |dz| <= 2 on the 3x3x3 box (stencil_catalog.cpp:70-75).
struct PoissonMask3 {
  __host__ __device__ static constexpr bool has(int j, int t, int l) {
    return (j != 1) + (t != 1) + (l != 1) <= 2;
  }
};

// coef[(l*M + j)*M + t] with l = dz+K, j = dx+K, t = dy+K (engine3d.cuh)
template <int K>
__host__ __device__ constexpr int cidx(int dx, int dy, int dz) {
  return ((dz + K) * (2 * K + 1) + (dx + K)) * (2 * K + 1) + (dy + K);
}

// ---- the star's per-cell chain (shared by every 3D star kernel: the
// pipeline engine, its direct-load kernel and the halo-lane kernel, so all
// of them give bit-identical results for the same number of sweeps) --------

// Star of order K: centre, then the x taps (dx = -K..-1, 1..K), the y taps,
// the z taps -- first product rounded, then one FMA per tap.  xv/yv/zv(d)
// return the sample at offset d on that axis.
template <class T, int K, class P, class FX, class FY, class FZ>
__device__ __forceinline__ T pipe_star_cell(const P& p, T c, FX xv, FY yv, FZ zv) {
  T v = mul_t(p.coef[cidx<K>(0, 0, 0)], c);
#pragma unroll
  for (int d = -K; d <= K; ++d)
    if (d != 0) v = fma_t(p.coef[cidx<K>(d, 0, 0)], xv(d), v);
#pragma unroll
  for (int d = -K; d <= K; ++d)
    if (d != 0) v = fma_t(p.coef[cidx<K>(0, d, 0)], yv(d), v);
#pragma unroll
  for (int d = -K; d <= K; ++d)
    if (d != 0) v = fma_t(p.coef[cidx<K>(0, 0, d)], zv(d), v);
  return v;
}


// Stores one lane's Q outputs of row (z, y) at column x0 (vector when `vec`,
// else only the columns inside [xlo, xhi)), and mirrors planes a neighbour
// keeps as ghost slots into its buffer over peer memory.
template <class T, int Q>
__device__ __forceinline__ void put_q3(T* row, const T (&v)[Q], bool vec, int x0, int xlo, int xhi) {
  if (vec) {
    st_q<T, Q>(row, v);
  } else {
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (x0 + q >= xlo && x0 + q < xhi) row[q] = v[q];
  }
}
// Whether output plane z is mirrored into a neighbour's ghost slots (uniform
// per plane; false outside peer-halo slab runs).
template <class P>
__device__ __forceinline__ bool mirrored3(const P& p, int z) {
  return (p.peer_lo != nullptr && z < p.peer_lo_end) ||
         (p.peer_hi != nullptr && z >= p.peer_hi_begin);
}
template <class T, int Q, class P>
__device__ __forceinline__ void store_row3(const P& p, int z, int y, int x0, const T (&v)[Q],
                                           bool vec, int xlo, int xhi, bool mirror) {
  T* row = p.out + (static_cast<size_t>(z) * p.ny + y) * p.nx + x0;
  put_q3<T, Q>(row, v, vec, x0, xlo, xhi);
  if (mirror) {
    const long long off = row - p.out;
    if (p.peer_lo != nullptr && z < p.peer_lo_end)
      put_q3<T, Q>(p.peer_lo + (off + p.peer_lo_shift), v, vec, x0, xlo, xhi);
    if (p.peer_hi != nullptr && z >= p.peer_hi_begin)
      put_q3<T, Q>(p.peer_hi + (off + p.peer_hi_shift), v, vec, x0, xlo, xhi);
  }
}

// One ring slot: a brows x bcols box, padded to the 128-byte alignment TMA
// requires of every destination.
template <class T>
__host__ __device__ constexpr size_t box_slot_elems(int brows, int bcols) {
  return (static_cast<size_t>(brows) * bcols * sizeof(T) + 127) / 128 * 128 / sizeof(T);
}

// Shared memory of the TMA kernel: DZ plane boxes shared by the CTA's warps
// (sx strips x sy row groups), a full and an empty mbarrier per slot (the
// empty barrier counts one arrive per consumer lane), and 128 B per warp.
template <class T, int Q, int RY, int K, int DZ>
__host__ __device__ constexpr size_t ring3d_bytes(int sx, int sy, int v) {
  return static_cast<size_t>(DZ) *
             (box_slot_elems<T>(sy * RY + 2 * K, (sx - 1) * v + 32 * Q) * sizeof(T) + 16) +
         static_cast<size_t>(sx * sy) * 128;
}

template <class T, int Q, int NROW>
__device__ __forceinline__ void load_plane(const T* __restrict__ in, int nx, int ny, int nz, int z,
                                           int yr0, int col0, T (&dst)[NROW][Q]) {
  const bool zin = z >= 0 && z < nz;
#pragma unroll
  for (int r = 0; r < NROW; ++r) {
    const int y = yr0 + r;
    if (!zin || y < 0 || y >= ny) {
#pragma unroll
      for (int q = 0; q < Q; ++q) dst[r][q] = T(0);
      continue;
    }
    const T* row = in + (static_cast<size_t>(z) * ny + y) * nx;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int x = col0 + q;
      dst[r][q] = (x >= 0 && x < nx) ? __ldg(row + x) : T(0);
    }
  }
}

// Column partial j of output row r; plane slot of dz = l-K is (ph + l) % NPL.
template <class T, int Q, int K, class Mask, int RY, int NPL, int CAP>
__device__ __forceinline__ bool colpart3(const T (&pl)[NPL][RY + 2 * K][Q], int ph, int r, int j,
                                         const Ssam3DParams<T, CAP>& p, T (&cp)[Q]) {
  constexpr int M = 2 * K + 1;
  bool any = false;
#pragma unroll
  for (int l = 0; l < M; ++l)
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (Mask::has(j, t, l)) {
        const T c = p.coef[(l * M + j) * M + t];
        const int s = (ph + l) % NPL;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          cp[q] = any ? fma_t(c, pl[s][r + t][q], cp[q]) : c * pl[s][r + t][q];
        any = true;
      }
    }
  return any;
}

// Column partials of filter column j for RG consecutive output rows r0..:
// taps outer, rows inner, so each weight is fetched once per RG rows (fp64
// weights are LDC.64 loads, not DFMA operands); per row the tap order -- and
// so the result -- is exactly colpart3's.
#ifndef SSAM_HALO_RG
#define SSAM_HALO_RG 1
#endif
#ifndef SSAM_3D_RG
#define SSAM_3D_RG 2  // measured: fp64 27pt / poisson / 7pt +5..6%, fp32 27pt +1.5%; 4 is worse
#endif
template <class T, int Q, int K, class Mask, int NROW, int NPL, int RG, int CAP>
__device__ __forceinline__ bool colpart3_rows(const T (&pl)[NPL][NROW][Q], int ph, int r0, int j,
                                              const Ssam3DParams<T, CAP>& p, T (&cp)[RG][Q]) {
  constexpr int M = 2 * K + 1;
  bool any = false;
#pragma unroll
  for (int l = 0; l < M; ++l)
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (Mask::has(j, t, l)) {
        const T c = p.coef[(l * M + j) * M + t];
        const int s = (ph + l) % NPL;
#pragma unroll
        for (int g = 0; g < RG; ++g)
#pragma unroll
          for (int q = 0; q < Q; ++q)
            cp[g][q] = any ? fma_t(c, pl[s][r0 + g + t][q], cp[g][q]) : c * pl[s][r0 + g + t][q];
        any = true;
      }
    }
  return any;
}

// Single-chain accumulation: the taps of filter column j are FMAs straight
// into the running chain value -- no separate column partial, so no FMUL to
// start it and no FADD to join it.  Fewer FP ops, but one long dependent
// chain instead of independent column partials; measured per shape at 512^3
// (two-level -> single chain, GCells/s): 3d13pt f32 445 -> 460, poisson f64
// 275 -> 306, but 3d7pt f64 371 -> 359, 3d13pt f64 221 -> 210, and the fused
// Tb = 2 3d7pt f32 1047 -> 955.  So only those two shapes take it.  Every 3D
// kernel of one (type, mask) -- aligned, halo-lane, direct, fused Tb = 2 and
// the halo lanes' mini-chains -- uses the same order, so they stay
// bit-identical.
template <class T, class Mask>
constexpr bool chain1_3d() {
  return (sizeof(T) == 8 && std::is_same<Mask, PoissonMask3>::value && !std::is_integral<T>::value) ||
         (sizeof(T) == 4 && std::is_same<Mask, StarMask3<2>>::value);
}
template <class T, int Q, int K, class Mask, int NROW, int NPL, int RG, int CAP>
__device__ __forceinline__ void colfma3_rows(const T (&pl)[NPL][NROW][Q], int ph, int r0, int j,
                                             const Ssam3DParams<T, CAP>& p, T (&acc)[RG][Q]) {
  constexpr int M = 2 * K + 1;
#pragma unroll
  for (int l = 0; l < M; ++l)
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (Mask::has(j, t, l)) {
        const T c = p.coef[(l * M + j) * M + t];
        const int s = (ph + l) % NPL;
#pragma unroll
        for (int g = 0; g < RG; ++g)
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[g][q] = fma_t(c, pl[s][r0 + g + t][q], acc[g][q]);
      }
    }
}

// RY output rows of plane z from the register planes (bidirectional chain),
// RG rows at a time.
template <class T, int Q, int K, class Mask, int RY, int NPL, int CAP, bool PEER>
__device__ __forceinline__ void compute_rows(const T (&pl)[NPL][RY + 2 * K][Q], int ph,
                                             const Ssam3DParams<T, CAP>& p, int z, int y_out0,
                                             int x0, bool owner) {
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int RG = (RY % SSAM_3D_RG == 0) ? SSAM_3D_RG : 1;
  const int xlo = p.ring, xhi = p.nx - p.ring;
  const int yhi = p.ny - p.ring;
  const bool mirror = PEER && mirrored3(p, z);
#pragma unroll
  for (int r0 = 0; r0 < RY; r0 += RG) {
    T acc[RG][Q];
    if constexpr (chain1_3d<T, Mask>()) {
#pragma unroll
      for (int g = 0; g < RG; ++g)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[g][q] = T(0);
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        if (j > 0) {
#pragma unroll
          for (int g = 0; g < RG; ++g) shift_up1<T, Q>(acc[g]);
        }
        colfma3_rows<T, Q, K, Mask, NROW, NPL, RG, CAP>(pl, ph, r0, j, p, acc);
      }
      if constexpr (K > 0) {
        T accr[RG][Q];
#pragma unroll
        for (int g = 0; g < RG; ++g)
#pragma unroll
          for (int q = 0; q < Q; ++q) accr[g][q] = T(0);
#pragma unroll
        for (int j = M - 1; j > K; --j) {
          if (j < M - 1) {
#pragma unroll
            for (int g = 0; g < RG; ++g) shift_down1<T, Q>(accr[g]);
          }
          colfma3_rows<T, Q, K, Mask, NROW, NPL, RG, CAP>(pl, ph, r0, j, p, accr);
        }
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          shift_down1<T, Q>(accr[g]);
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[g][q] += accr[g][q];
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j <= K; ++j) {
        T cp[RG][Q];
        const bool any = colpart3_rows<T, Q, K, Mask, NROW, NPL, RG, CAP>(pl, ph, r0, j, p, cp);
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          if (j == 0) {
#pragma unroll
            for (int q = 0; q < Q; ++q) acc[g][q] = any ? cp[g][q] : T(0);
          } else {
            shift_up1<T, Q>(acc[g]);
            if (any) {
#pragma unroll
              for (int q = 0; q < Q; ++q) acc[g][q] += cp[g][q];
            }
          }
        }
      }
      if constexpr (K > 0) {
        T accr[RG][Q];
#pragma unroll
        for (int j = M - 1; j > K; --j) {
          T cp[RG][Q];
          const bool any = colpart3_rows<T, Q, K, Mask, NROW, NPL, RG, CAP>(pl, ph, r0, j, p, cp);
#pragma unroll
          for (int g = 0; g < RG; ++g) {
            if (j == M - 1) {
#pragma unroll
              for (int q = 0; q < Q; ++q) accr[g][q] = any ? cp[g][q] : T(0);
            } else {
              shift_down1<T, Q>(accr[g]);
              if (any) {
#pragma unroll
                for (int q = 0; q < Q; ++q) accr[g][q] += cp[g][q];
              }
            }
          }
        }
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          shift_down1<T, Q>(accr[g]);
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[g][q] += accr[g][q];
        }
      }
    }
#pragma unroll
    for (int g = 0; g < RG; ++g) {
      const int y = y_out0 + r0 + g;
      if (owner && y < yhi)
        store_row3<T, Q>(p, z, y, x0, acc[g], p.vec_ok && x0 >= xlo && x0 + Q <= xhi, xlo, xhi,
                         mirror);
    }
  }
}

// TMA kernel (16-byte aligned rows).  The CTA's WPB warps cover WPB*RY
// consecutive output rows of one x-strip and share one 2D tensor-map box of
// WPB*RY + 2K rows per input plane (the y halo is fetched once per CTA, not
// once per warp).  DZ plane slots form a ring guarded by a full barrier
// (TMA transaction count) and an empty barrier (one arrival per warp).
// Thread 0 produces: after consuming plane i it refills the slot of plane
// i-1 -- one plane of slack so it rarely waits on the slowest warp.
// Out-of-range rows, planes and columns arrive as zeros (interior outputs
// never read them).
template <class T, int Q, int K, class Mask, int RY, int DZ, int CAP, bool PEER = false>
__global__ void __launch_bounds__(256)
    ssam3d_tma_kernel(const __grid_constant__ Ssam3DTmaParams<T, CAP> P) {
  const Ssam3DParams<T, CAP>& p = P.p;
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int NPL = M;
  constexpr int ROW = 32 * Q;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  // CTA = sx adjacent x-strips x sy row groups; one box spans all of them.
  const int sx = p.cta_sx, sy = wpb / p.cta_sx;
  const int wx = wib % sx, wy = wib / sx;
  const int brows = sy * RY + 2 * K;
  const int bcols = (sx - 1) * p.V + ROW;
  const uint32_t box_bytes = static_cast<uint32_t>(brows) * bcols * sizeof(T);
  const size_t slot_elems = box_slot_elems<T>(brows, bcols);
  const int y_cta0 = p.ring + (p.zfast ? blockIdx.z : blockIdx.y) * sy * RY;
  const int y_out0 = y_cta0 + wy * RY;
  const int z0 = p.z_begin + (p.zfast ? blockIdx.y : blockIdx.z) * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int base = blockIdx.x * sx * p.V - p.A;  // box origin (16-byte aligned)
  const int x_out0 = (blockIdx.x * sx + wx) * p.V;
  const int x0 = base + wx * p.V + Q * lane;
  const bool owner = x0 >= x_out0 && x0 < x_out0 + p.V;
  const int count = (z1 - z0) + 2 * K;  // input planes z0-K .. z1-1+K

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + DZ * slot_elems * sizeof(T));
  uint64_t* empty = full + DZ;
  if (threadIdx.x == 0) {
    prefetch_tmap(&P.tmap);
#pragma unroll
    for (int s = 0; s < DZ; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 32 * wpb);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains
  // Plane i of the stream (z = z0 - K + i): rows y_cta0-K .. of the
  // flattened (ny*nz)-row view; planes outside [0, nz) land outside -> zeros.
  auto issue = [&](int i) {
    const int s = i % DZ;
    if (i >= DZ) {
      mbar_wait(smem_u32(&empty[s]), ((i / DZ) - 1) & 1);  // acquire: every lane's reads done
      fence_proxy_async();  // generic-proxy reads before the async-proxy refill
    }
    const uint32_t bar = smem_u32(&full[s]);
    const int z = z0 - K + i;
    const int row = (z >= 0 && z < p.nz) ? z * p.ny + (y_cta0 - K) : -brows;
    mbar_arrive_expect_tx(bar, box_bytes);
    tma_load_2d(smem_u32(ring + s * slot_elems), &P.tmap, base, row, bar);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < min(DZ, count); ++i) issue(i);
  auto take = [&](int i, T (&dst)[NROW][Q]) {
    const int s = i % DZ;
    mbar_wait(smem_u32(&full[s]), (i / DZ) & 1);
    const T* slot = ring + s * slot_elems + static_cast<size_t>(wy * RY) * bcols + wx * p.V +
                    Q * lane;
#pragma unroll
    for (int r = 0; r < NROW; ++r) lds_q<T, Q>(slot + r * bcols, dst[r]);
    mbar_arrive(smem_u32(&empty[s]));  // release: this lane's reads of slot s are done
    if (threadIdx.x == 0 && i >= 1 && i - 1 + DZ < count) issue(i - 1 + DZ);
  };

  T pl[NPL][NROW][Q];
#pragma unroll
  for (int i = 0; i < NPL - 1; ++i) take(i, pl[i]);
  for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int z = zb + ph;
      if (z >= z1) break;
      take(z - z0 + 2 * K, pl[(ph + NPL - 1) % NPL]);
      compute_rows<T, Q, K, Mask, RY, NPL, CAP, PEER>(pl, ph, p, z, y_out0, x0, owner);
    }
  }
}

// Direct-load kernel (rows not 16-byte aligned).
template <class T, int Q, int K, class Mask, int RY, int CAP, bool PEER = false>
__global__ void __launch_bounds__(128) ssam3d_kernel(const __grid_constant__ Ssam3DParams<T, CAP> p) {
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int NPL = M;
  const int lane = threadIdx.x & 31;
  const int group = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (group >= p.ygroups) return;
  const int y_out0 = p.ring + group * RY;
  const int z0 = p.z_begin + blockIdx.z * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int x_out0 = blockIdx.x * p.V;
  const int x0 = x_out0 - p.A + Q * lane;
  const bool owner = x0 >= x_out0 && x0 < x_out0 + p.V;

  T pl[NPL][NROW][Q];
#pragma unroll
  for (int s = 0; s < NPL - 1; ++s)
    load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z0 - K + s, y_out0 - K, x0, pl[s]);
  for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int z = zb + ph;
      if (z >= z1) break;
      load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z + K, y_out0 - K, x0,
                             pl[(ph + NPL - 1) % NPL]);
      compute_rows<T, Q, K, Mask, RY, NPL, CAP, PEER>(pl, ph, p, z, y_out0, x0, owner);
    }
  }
}


// ===========================================================================
// Full-warp lane plan with halo lanes (ssam3d_halo_kernel).
//
// The kernels above follow the paper's lane plan: a warp loads 32Q columns
// and emits the ~32Q-2K whose chains stay inside the warp, rounded down to
// whole Q-vectors (120 of 128 for K = 1).  On a 512-wide grid that is five
// strips for 512 columns -- 15% of every load and FMA spent on columns
// another warp also computes.  Here EVERY lane owns its Q columns (a warp
// emits all 32Q) and the chain's missing inputs at the warp's two ends come
// from halo lanes: lane 0 additionally holds the K columns left of the
// strip, lane 31 the K columns right of it, read from a box that is VQ
// columns wider on each side.  Each lane runs one short halo chain over
// those K columns with its own coefficient set (lane 0: the left chain's
// dx < 0 columns, lane 31: the mirrored right chain's dx > 0 columns --
// the masks are x-symmetric) and the results are injected into the
// systolic chain where shfl_up / shfl_down would have brought them in from
// a lane outside the warp.  The injected sums are formed in exactly the
// order the main chain uses (h_m(c) = h_{m-1}(c-1) + colpart_m(c), colpart
// over (dz, dy) in the same tap order), so results are bit-identical to
// the kernels above.
// ===========================================================================

// Window rows whose halo columns feed a dx != 0 tap (compile-time).
template <int K, class Mask, int RY>
__host__ __device__ constexpr bool halo_row_needed(int w) {
  constexpr int M = 2 * K + 1;
  for (int m = 0; m < K; ++m)
    for (int l = 0; l < M; ++l)
      for (int t = 0; t < M; ++t)
        if (Mask::has(m, t, l) && w - t >= 0 && w - t < RY) return true;
  return false;
}

// Shared memory of the halo kernel: DZ plane slots of sx per-strip boxes.
template <class T, int Q, int RY, int K, int DZ>
__host__ __device__ constexpr size_t halo3d_bytes(int sx, int sy) {
  constexpr int VQ = 16 / sizeof(T);
  return static_cast<size_t>(DZ) *
             (sx * box_slot_elems<T>(sy * RY + 2 * K, 32 * Q + 2 * VQ) * sizeof(T) + 16) +
         static_cast<size_t>(sx * sy) * 128;
}

// CTA size / residency targets of the halo kernel: two 256-thread CTAs per SM
// for the light fp32 star (fits 128 registers without spills); the heavier
// footprints run 128-thread CTAs, three per SM for fp32 order 1 (<= 170
// registers).
template <class T, int K, class Mask>
__host__ __device__ constexpr bool halo3d_light() {
  return sizeof(T) == 4 && K == 1 && Mask::has(0, 1, 1) && !Mask::has(0, 0, 1);
}
template <class T, int K, class Mask>
__host__ __device__ constexpr int halo3d_max_threads() {
  return halo3d_light<T, K, Mask>() ? 256 : 128;
}
template <class T, int K, class Mask>
__host__ __device__ constexpr int halo3d_min_blocks() {
  return halo3d_light<T, K, Mask>() ? 2 : (sizeof(T) == 4 && K == 1 ? 3 : 1);
}

template <class T, int Q, int K, class Mask, int RY, int DZ, int CAP, bool PEER = false>
__global__ void __launch_bounds__((halo3d_max_threads<T, K, Mask>()),
                                  (halo3d_min_blocks<T, K, Mask>()))
    ssam3d_halo_kernel(const __grid_constant__ Ssam3DTmaParams<T, CAP> P) {
  static_assert(K >= 1, "order-0 stencils have no chain");
  const Ssam3DParams<T, CAP>& p = P.p;
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int HRG = (RY % SSAM_HALO_RG == 0) ? SSAM_HALO_RG : 1;  // rows per weight fetch
  constexpr int NPL = M;
  constexpr int VQ = 16 / sizeof(T);
  constexpr int BW = 32 * Q + 2 * VQ;  // box width: the strip plus VQ columns each side
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int sx = p.cta_sx, sy = wpb / p.cta_sx;
  const int wx = wib % sx, wy = wib / sx;
  const int brows = sy * RY + 2 * K;
  const uint32_t box_bytes = static_cast<uint32_t>(brows) * BW * sizeof(T);
  const size_t sub_elems = box_slot_elems<T>(brows, BW);
  const size_t slot_elems = sx * sub_elems;
  const int y_cta0 = p.ring + (p.zfast ? blockIdx.z : blockIdx.y) * sy * RY;
  const int y_out0 = y_cta0 + wy * RY;
  const int z0 = p.z_begin + (p.zfast ? blockIdx.y : blockIdx.z) * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int x_cta0 = blockIdx.x * sx * 32 * Q;
  const int x0 = x_cta0 + wx * 32 * Q + Q * lane;
  const int count = (z1 - z0) + 2 * K;
  const bool is_r = lane == 31;


  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + DZ * slot_elems * sizeof(T));
  uint64_t* empty = full + DZ;
  if (threadIdx.x == 0) {
    prefetch_tmap(&P.tmap);
#pragma unroll
    for (int s = 0; s < DZ; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 32 * wpb);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains
  auto issue = [&](int i) {
    const int s = i % DZ;
    if (i >= DZ) {
      mbar_wait(smem_u32(&empty[s]), ((i / DZ) - 1) & 1);  // acquire: every lane's reads done
      fence_proxy_async();  // generic-proxy reads before the async-proxy refill
    }
    const uint32_t bar = smem_u32(&full[s]);
    const int z = z0 - K + i;
    const int row = (z >= 0 && z < p.nz) ? z * p.ny + (y_cta0 - K) : -brows;
    mbar_arrive_expect_tx(bar, box_bytes * sx);
    for (int w = 0; w < sx; ++w)
      tma_load_2d(smem_u32(ring + s * slot_elems + w * sub_elems), &P.tmap,
                  x_cta0 + w * 32 * Q - VQ, row, bar);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < min(DZ, count); ++i) issue(i);
  // halo column c of this lane: lane 0 -> x_strip0 - K + c, lane 31 -> x_strip_end + K - 1 - c
  const int hoff0 = is_r ? VQ + 32 * Q + K - 1 : VQ - K;
  const int hstep = is_r ? -1 : 1;
  auto take = [&](int i, T (&dst)[NROW][Q], T (&hdst)[NROW][K]) {
    const int s = i % DZ;
    mbar_wait(smem_u32(&full[s]), (i / DZ) & 1);
    const T* slot = ring + s * slot_elems + wx * sub_elems + static_cast<size_t>(wy * RY) * BW;
#pragma unroll
    for (int r = 0; r < NROW; ++r) lds_q<T, Q>(slot + r * BW + VQ + Q * lane, dst[r]);
#pragma unroll
    for (int r = 0; r < NROW; ++r) {
      if (!halo_row_needed<K, Mask, RY>(r)) continue;
#pragma unroll
      for (int c = 0; c < K; ++c) hdst[r][c] = slot[r * BW + hoff0 + hstep * c];
    }
    mbar_arrive(smem_u32(&empty[s]));  // release: this lane's reads of slot s are done
    if (threadIdx.x == 0 && i >= 1 && i - 1 + DZ < count) issue(i - 1 + DZ);
  };

  const int xlo = p.ring, xhi = p.nx - p.ring;
  const int yhi = p.ny - p.ring;
  const bool vec = x0 >= xlo && x0 + Q <= xhi;
  T pl[NPL][NROW][Q];
  T hp[NPL][NROW][K];
#pragma unroll
  for (int i = 0; i < NPL - 1; ++i) take(i, pl[i], hp[i]);
  for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int z = zb + ph;
      if (z >= z1) break;
      take(z - z0 + 2 * K, pl[(ph + NPL - 1) % NPL], hp[(ph + NPL - 1) % NPL]);
      const bool mirror = PEER && mirrored3(p, z);
      if constexpr (std::is_same<Mask, StarMask3<1>>::value) {
        // the 7-point star: the pipeline engine's per-cell chain
        // (pipe_star_cell), so single sweeps here equal the fused pipeline
        // kernels bit for bit; x neighbours from the neighbour lanes, and
        // at the warp's ends from the halo lanes' columns
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const T(&cr)[Q] = pl[(ph + K) % NPL][r + K];
          const T hc = hp[(ph + K) % NPL][r + K][0];
          const T up = shfl_up(cr[Q - 1], 1);
          const T dn = __shfl_down_sync(kFull, cr[0], 1);
          const T lft = lane == 0 ? hc : up;
          const T rgt = is_r ? hc : dn;
          T acc1[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            auto xv = [&](int d) { return q + d < 0 ? lft : (q + d >= Q ? rgt : cr[q + d]); };
            auto yv = [&](int d) { return pl[(ph + K) % NPL][r + K + d][q]; };
            auto zv = [&](int d) { return pl[(ph + K + d) % NPL][r + K][q]; };
            acc1[q] = pipe_star_cell<T, 1>(p, cr[q], xv, yv, zv);
          }
          const int y = y_out0 + r;
          if (y < yhi) store_row3<T, Q>(p, z, y, x0, acc1, vec, xlo, xhi, mirror);
        }
        continue;
      }
#pragma unroll
      for (int r0 = 0; r0 < RY; r0 += HRG) {
        // halo chains: inj[g][m] = h_m(K-1), h_m(c) = h_{m-1}(c-1) + colpart_m(c)
        T inj[HRG][K];
#pragma unroll
        for (int g = 0; g < HRG; ++g) {
          const int r = r0 + g;
          T h[K];
#pragma unroll
          for (int m = 0; m < K; ++m) {
#pragma unroll
            for (int c = K - 1; c >= m; --c) {
              // both sides' colparts with constant-bank weights (lane 31
              // mirrors dx -> -dx); each lane keeps its own side's
              if constexpr (chain1_3d<T, Mask>()) {
                T cl = m == 0 ? T(0) : h[c - 1];
                T cr = cl;
#pragma unroll
                for (int l = 0; l < M; ++l)
#pragma unroll
                  for (int t = 0; t < M; ++t)
                    if (Mask::has(m, t, l)) {
                      const T v = hp[(ph + l) % NPL][r + t][c];
                      cl = fma_t(p.coef[(l * M + m) * M + t], v, cl);
                      cr = fma_t(p.coef[(l * M + (M - 1 - m)) * M + t], v, cr);
                    }
                h[c] = is_r ? cr : cl;
              } else {
                T cl = T(0), cr = T(0);
                bool any = false;
#pragma unroll
                for (int l = 0; l < M; ++l)
#pragma unroll
                  for (int t = 0; t < M; ++t)
                    if (Mask::has(m, t, l)) {
                      const T v = hp[(ph + l) % NPL][r + t][c];
                      const T wl = p.coef[(l * M + m) * M + t];
                      const T wr = p.coef[(l * M + (M - 1 - m)) * M + t];
                      cl = any ? fma_t(wl, v, cl) : wl * v;
                      cr = any ? fma_t(wr, v, cr) : wr * v;
                      any = true;
                    }
                const T cp = is_r ? cr : cl;
                if (m == 0)
                  h[c] = any ? cp : T(0);
                else
                  h[c] = any ? h[c - 1] + cp : h[c - 1];
              }
            }
            inj[g][m] = h[K - 1];
          }
        }
        T acc[HRG][Q];
        T accr[HRG][Q];
        if constexpr (chain1_3d<T, Mask>()) {
#pragma unroll
          for (int j = 0; j <= K; ++j) {
#pragma unroll
            for (int g = 0; g < HRG; ++g) {
              if (j == 0) {
#pragma unroll
                for (int q = 0; q < Q; ++q) acc[g][q] = T(0);
              } else {
                shift_up1<T, Q>(acc[g]);
                if (lane == 0) acc[g][0] = inj[g][j - 1];
              }
            }
            colfma3_rows<T, Q, K, Mask, NROW, NPL, HRG, CAP>(pl, ph, r0, j, p, acc);
          }
#pragma unroll
          for (int j = M - 1; j > K; --j) {
#pragma unroll
            for (int g = 0; g < HRG; ++g) {
              if (j == M - 1) {
#pragma unroll
                for (int q = 0; q < Q; ++q) accr[g][q] = T(0);
              } else {
                shift_down1<T, Q>(accr[g]);
                if (is_r) accr[g][Q - 1] = inj[g][M - 2 - j];
              }
            }
            colfma3_rows<T, Q, K, Mask, NROW, NPL, HRG, CAP>(pl, ph, r0, j, p, accr);
          }
        } else {
#pragma unroll
          for (int j = 0; j <= K; ++j) {
            T cp[HRG][Q];
            const bool any = colpart3_rows<T, Q, K, Mask, NROW, NPL, HRG, CAP>(pl, ph, r0, j, p, cp);
#pragma unroll
            for (int g = 0; g < HRG; ++g) {
              if (j == 0) {
#pragma unroll
                for (int q = 0; q < Q; ++q) acc[g][q] = any ? cp[g][q] : T(0);
              } else {
                shift_up1<T, Q>(acc[g]);
                if (lane == 0) acc[g][0] = inj[g][j - 1];
                if (any) {
#pragma unroll
                  for (int q = 0; q < Q; ++q) acc[g][q] += cp[g][q];
                }
              }
            }
          }
#pragma unroll
          for (int j = M - 1; j > K; --j) {
            T cp[HRG][Q];
            const bool any = colpart3_rows<T, Q, K, Mask, NROW, NPL, HRG, CAP>(pl, ph, r0, j, p, cp);
#pragma unroll
            for (int g = 0; g < HRG; ++g) {
              if (j == M - 1) {
#pragma unroll
                for (int q = 0; q < Q; ++q) accr[g][q] = any ? cp[g][q] : T(0);
              } else {
                shift_down1<T, Q>(accr[g]);
                if (is_r) accr[g][Q - 1] = inj[g][M - 2 - j];
                if (any) {
#pragma unroll
                  for (int q = 0; q < Q; ++q) accr[g][q] += cp[g][q];
                }
              }
            }
          }
        }
#pragma unroll
        for (int g = 0; g < HRG; ++g) {
          const int r = r0 + g;
          T acc1[Q];
          shift_down1<T, Q>(accr[g]);
          if (is_r) accr[g][Q - 1] = inj[g][K - 1];
#pragma unroll
          for (int q = 0; q < Q; ++q) acc1[q] = acc[g][q] + accr[g][q];
          const int y = y_out0 + r;
          if (y < yhi) store_row3<T, Q>(p, z, y, x0, acc1, vec, xlo, xhi, mirror);
        }
      }
    }
  }
}

}  // namespace ssam_b200
