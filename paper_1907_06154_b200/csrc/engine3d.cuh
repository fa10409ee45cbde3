// engine3d.cuh -- the 3D SSAM engine (3D stencil Jacobi sweeps), sm_100a.
//
// The reference maps one warp to one x-y plane and sums the per-dz partials
// through a block-shared InterWarpBuffer (kernels.hpp:283-384,
// blocking.hpp:82-97).  On Blackwell that smem round trip
// and the 2k/warp_count plane re-loads are unnecessary: each warp owns an
// x-strip (32 lanes x Q columns) x RY output rows and STREAMS along z,
// keeping the 2K+1 most recent input planes of its (RY+2K) x Q footprint in
// registers (z-streaming).  Per output row the chain is
// the same systolic one as in 2D, with the column partial now folding every
// (dy, dz) tap of that dx column:
//     colpart_j = sum_{l,t} c(dx=j-K, dy=t-K, dz=l-K) * plane[l][row+t]
//     acc       = shift1(acc) + colpart_j
// Planes arrive through a per-warp TMA ring (cp.async.bulk, one row copy per
// lane, DZ planes in flight); unaligned grids fall back to direct loads.
// Only interior cells [K, n-K) per axis are written; the ring of width K is
// carried by both ping-pong buffers (set up once per call), which is the
// reference's next = cur copy (kernels.hpp:323) without the per-sweep copy.
#pragma once

#include "common.cuh"
#include "engine2d.cuh"

namespace ssam_b200 {

template <class T, int CAP>
struct Ssam3DParams {
  const T* in;
  T* out;
  int nx, ny, nz;
  int e, G, A, V;   // lane plan (as in 2D, M = 2K+1)
  int nstrips;
  int ygroups;      // groups of RY interior rows
  int zseg;         // output planes streamed per warp
  int z_begin, z_end;
  int ring;         // = K
  int vec_ok;
  T coef[CAP];      // coef[(l*M + j)*M + t], l = dz+K, j = dx+K, t = dy+K
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

template <class T, int Q, int RY, int K, int DZ>
__host__ __device__ constexpr size_t ring3d_bytes(int warps) {
  return static_cast<size_t>(warps) * DZ * ((RY + 2 * K) * 32 * Q * sizeof(T) + 8);
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

// RY output rows of plane z from the register planes; slot s of plane
// (output plane + l - K) is (ph + l) % NPL.
template <class T, int Q, int K, class Mask, int RY, int NPL, int CAP>
__device__ __forceinline__ void compute_rows(const T (&pl)[NPL][RY + 2 * K][Q], int ph,
                                             const Ssam3DParams<T, CAP>& p, int z, int y_out0,
                                             int xres, bool owner) {
  constexpr int M = 2 * K + 1;
  constexpr int E = (Q - K % Q) % Q;
  const int xlo = p.ring, xhi = p.nx - p.ring;
  const int yhi = p.ny - p.ring;
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    T acc[Q];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      T cp[Q];
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
#pragma unroll
    for (int s = 0; s < E; ++s) shift1<T, Q>(acc);
    const int y = y_out0 + r;
    if (owner && y < yhi) {
      T* row = p.out + (static_cast<size_t>(z) * p.ny + y) * p.nx;
      if (p.vec_ok && xres >= xlo && xres + Q <= xhi) {
        st_vec<T, Q>(row + xres, acc);
      } else {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (xres + q >= xlo && xres + q < xhi) row[xres + q] = acc[q];
      }
    }
  }
}

template <class T, int Q, int K, class Mask, int RY, int DZ, int CAP>
__global__ void __launch_bounds__(128) ssam3d_kernel(const __grid_constant__ Ssam3DParams<T, CAP> p) {
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int NPL = M;  // planes resident in registers
  constexpr int ROW = 32 * Q;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int strip = blockIdx.x;
  const int group = blockIdx.y * (blockDim.x >> 5) + wib;
  if (group >= p.ygroups) return;
  const int y_out0 = p.ring + group * RY;
  const int z0 = p.z_begin + blockIdx.z * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;
  const int col0 = base + Q * lane;
  const int xres = col0 - p.G;
  const bool owner = xres >= x_out0 && xres < x_out0 + p.V;
  const int count = (z1 - z0) + 2 * K;  // input planes z0-K .. z1-1+K

  T pl[NPL][NROW][Q];

  if (p.vec_ok) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * DZ * NROW * ROW;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(blockDim.x >> 5) *
                                                                DZ * NROW * ROW * sizeof(T)) +
                     wib * DZ;
    const int cbeg = max(base, 0), cend = min(base + ROW, p.nx);
    const uint32_t bytes = static_cast<uint32_t>(cend - cbeg) * sizeof(T);
    const int doff = cbeg - base;
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < DZ; ++s) mbar_init(smem_u32(&bars[s]), 1);
      fence_mbar_init();
    }
    __syncwarp();
    // Plane i of the stream (z = z0 - K + i) lands in ring slot i % DZ: lane 0
    // arms the slot's barrier for NROW row copies, lanes 0..NROW-1 issue one
    // row each.  Rows/planes outside the grid are fetched clamped -- interior
    // outputs never read them.
    auto issue = [&](int i) {
      const int s = i % DZ;
      const uint32_t bar = smem_u32(&bars[s]);
      fence_proxy_async();
      if (lane == 0) mbar_arrive_expect_tx(bar, bytes * NROW);
      __syncwarp();
      if (lane < NROW) {
        const int z = clampi(z0 - K + i, p.nz);
        const int y = clampi(y_out0 - K + lane, p.ny);
        tma_load_1d(smem_u32(ring + (s * NROW + lane) * ROW + doff),
                    p.in + (static_cast<size_t>(z) * p.ny + y) * p.nx + cbeg, bytes, bar);
      }
    };
    for (int i = 0; i < min(DZ, count); ++i) issue(i);
    auto take = [&](int i, T (&dst)[NROW][Q]) {
      const int s = i % DZ;
      mbar_wait(smem_u32(&bars[s]), (i / DZ) & 1);
#pragma unroll
      for (int r = 0; r < NROW; ++r) lds_vec<T, Q>(ring + (s * NROW + r) * ROW + Q * lane, dst[r]);
      __syncwarp();
      if (i + DZ < count) issue(i + DZ);
    };
#pragma unroll
    for (int i = 0; i < NPL - 1; ++i) take(i, pl[i]);
    for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
      for (int ph = 0; ph < NPL; ++ph) {
        const int z = zb + ph;
        if (z >= z1) break;
        take(z - z0 + 2 * K, pl[(ph + NPL - 1) % NPL]);
        compute_rows<T, Q, K, Mask, RY, NPL, CAP>(pl, ph, p, z, y_out0, xres, owner);
      }
    }
    return;
  }

  // Direct-load path (grids whose rows are not 16-byte aligned).
#pragma unroll
  for (int s = 0; s < NPL - 1; ++s)
    load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z0 - K + s, y_out0 - K, col0, pl[s]);
  for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int z = zb + ph;
      if (z >= z1) break;
      load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z + K, y_out0 - K, col0,
                             pl[(ph + NPL - 1) % NPL]);
      compute_rows<T, Q, K, Mask, RY, NPL, CAP>(pl, ph, p, z, y_out0, xres, owner);
    }
  }
}

}  // namespace ssam_b200
