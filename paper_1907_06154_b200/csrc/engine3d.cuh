// engine3d.cuh -- the 3D SSAM engine (3D stencil Jacobi sweeps), sm_100a.
//
// The reference maps one warp to one x-y plane and sums the per-dz partials
// through a block-shared InterWarpBuffer (kernels.hpp:283-384,
// blocking.hpp:82-97).  On Blackwell that smem round trip
// and the 2k/warp_count plane re-loads are unnecessary: each warp owns an
// x-strip (32 lanes x Q columns) x RY output rows and STREAMS along z,
// keeping the 2K+1(+PFZ) most recent input planes of its (RY+2K) x Q
// footprint in registers (z-streaming).  Per output row
// the chain is the same systolic one as in 2D, with the column partial now
// folding every (dy, dz) tap of that dx column:
//     colpart_j = sum_{l,t} c(dx=j-K, dy=t-K, dz=l-K) * plane[l][row+t]
//     acc       = shift1(acc) + colpart_j
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

template <class T, int Q, int NROW>
__device__ __forceinline__ void load_plane(const T* __restrict__ in, int nx, int ny, int nz, int z,
                                           int yr0, int col0, bool fast, T (&dst)[NROW][Q]) {
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
    if (fast) {
      ld_vec<T, Q>(row + col0, dst[r]);
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int x = col0 + q;
        dst[r][q] = (x >= 0 && x < nx) ? __ldg(row + x) : T(0);
      }
    }
  }
}

template <class T, int Q, int K, class Mask, int RY, int PFZ, int CAP>
__global__ void __launch_bounds__(128) ssam3d_kernel(const __grid_constant__ Ssam3DParams<T, CAP> p) {
  constexpr int M = 2 * K + 1;
  constexpr int NROW = RY + 2 * K;
  constexpr int NPL = M + PFZ;  // planes resident in registers
  constexpr int E = (Q - K % Q) % Q;
  const int lane = threadIdx.x & 31;
  const int strip = blockIdx.x;
  const int group = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (group >= p.ygroups) return;
  const int y_out0 = p.ring + group * RY;
  const int z0 = p.z_begin + blockIdx.z * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;
  const int col0 = base + Q * lane;
  const int xres = col0 - p.G;
  const bool fast = p.vec_ok && base >= 0 && base + 32 * Q <= p.nx;
  const bool owner = xres >= x_out0 && xres < x_out0 + p.V;
  const int xlo = p.ring, xhi = p.nx - p.ring;
  const int yhi = p.ny - p.ring;

  // slot(plane zz) = (zz - (z0 - K)) mod NPL
  T pl[NPL][NROW][Q];
#pragma unroll
  for (int s = 0; s < NPL - 1; ++s)
    load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z0 - K + s, y_out0 - K, col0, fast, pl[s]);

  for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
    for (int ph = 0; ph < NPL; ++ph) {
      const int z = zb + ph;
      if (z >= z1) break;
      // Bring in plane z + K + PFZ (PFZ planes ahead of first use).
      load_plane<T, Q, NROW>(p.in, p.nx, p.ny, p.nz, z + K + PFZ, y_out0 - K, col0, fast,
                             pl[(ph + NPL - 1) % NPL]);
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
  }
}

}  // namespace ssam_b200
