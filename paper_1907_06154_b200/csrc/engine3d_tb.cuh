// engine3d_tb.cuh -- two fused 3D Jacobi sweeps per pass over HBM (temporal
// blocking, Tb = 2) on the z-streaming SSAM engine, sm_100a.
//
// The reference has no temporal blocking: its semantics
// are just Tb consecutive sweeps of stencil3d (kernels.hpp:283-384), each
// writing the interior and carrying the ring of width K.  Two sweeps read and
// write HBM once here, so the per-update traffic halves (4 B / cell-update
// for fp32).
//
// Warp-specialised CTA, one x-strip wide (32 x Q columns, aligned lane plan
// for an effective footprint of 2*(2K)+1 columns):
//   * 4 "stage-1" warps stream the input planes from the TMA ring (as
//     ssam3d_tma_kernel does) and compute the FIRST sweep for the CTA's
//     sy*RY output rows plus K rows above and below (each warp RY1 rows of
//     that band), for every plane z0-K .. z1-1+K.  Cells of the global ring
//     keep their input value, exactly as a sweep leaves them.  The rows land
//     in a shared-memory ring of intermediate planes.
//   * 4 "stage-2" warps stream those intermediate planes into their register
//     windows and compute the SECOND sweep for planes z0 .. z1-1, storing the
//     interior to HBM.
// Both stages run the same per-row systolic chain (colpart over (dy, dz),
// bidirectional shuffle chain over dx, engine2d.cuh / engine3d.cuh) with the
// same coefficients and order as one ssam3d sweep, so two fused sweeps are
// bit-identical to two calls of the single-sweep kernels.
//
// Rings: input TMA slots (full: transaction count, empty: 4 stage-1 arrivals)
// and intermediate slots (full: 4 stage-1 arrivals, empty: 4 stage-2
// arrivals), both with mbarrier phase parity.
#pragma once

#include "engine3d.cuh"

namespace ssam_b200 {

// The chain of one output row (engine3d.cuh compute_rows, without the store).
template <class T, int Q, int K, class Mask, int NROW, int NPL, int CAP>
__device__ __forceinline__ void row_chain(const T (&pl)[NPL][NROW][Q], int ph, int r,
                                          const Ssam3DParams<T, CAP>& p, T (&acc)[Q]) {
  constexpr int M = 2 * K + 1;
  T accr[Q];
  if constexpr (chain1_3d<T, Mask>()) {
    // single chain, exactly compute_rows' order (RG = 1)
    T a2[1][Q], r2[1][Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) a2[0][q] = r2[0][q] = T(0);
#pragma unroll
    for (int j = 0; j <= K; ++j) {
      if (j > 0) shift_up1<T, Q>(a2[0]);
      colfma3_rows<T, Q, K, Mask, NROW, NPL, 1, CAP>(pl, ph, r, j, p, a2);
    }
#pragma unroll
    for (int j = M - 1; j > K; --j) {
      if (j < M - 1) shift_down1<T, Q>(r2[0]);
      colfma3_rows<T, Q, K, Mask, NROW, NPL, 1, CAP>(pl, ph, r, j, p, r2);
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      acc[q] = a2[0][q];
      accr[q] = r2[0][q];
    }
  } else {
    auto colpart = [&](int j, T (&cp)[Q]) {
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
    };
#pragma unroll
    for (int j = 0; j <= K; ++j) {
      T cp[Q];
      const bool any = colpart(j, cp);
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
#pragma unroll
    for (int j = M - 1; j > K; --j) {
      T cp[Q];
      const bool any = colpart(j, cp);
      if (j == M - 1) {
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
  }
  shift_down1<T, Q>(accr);
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] += accr[q];
}

// Geometry shared by host and device.
template <class T, int Q, int K, int RY, int SY_ = 4>
struct Tb3Geom {
  static constexpr int SY = SY_;                      // stage-2 warps (row groups)
  static constexpr int ROWS2 = SY * RY;               // output rows per CTA
  static constexpr int IROWS = ROWS2 + 2 * K;         // intermediate rows (sweep-1 band)
  static constexpr int RY1 = (IROWS + SY - 1) / SY;   // sweep-1 rows per stage-1 warp
  static constexpr int BROWS = SY * RY1 + 2 * K;      // input box rows
  static constexpr int BW = 32 * Q;                   // box / strip width
  static constexpr int DZ = 4, DI = 4;                // input / intermediate ring depth
  static constexpr size_t IN_SLOT = (size_t(BROWS) * BW * sizeof(T) + 127) / 128 * 128;
  static constexpr size_t MID_SLOT = (size_t(IROWS) * BW * sizeof(T) + 127) / 128 * 128;
  static constexpr int THREADS = 2 * SY * 32;          // SY sweep-1 + SY sweep-2 warps
  static constexpr size_t SMEM =
      DZ * IN_SLOT + DI * MID_SLOT + (2 * DZ + 2 * DI) * 8 + THREADS * 4;
};

template <class T, int Q, int K, class Mask, int RY, int CAP, int SY = 4, bool PEER = false>
__global__ void __launch_bounds__(2 * SY * 32)
    ssam3d_tb2_kernel(const __grid_constant__ Ssam3DTmaParams<T, CAP> P) {
  using G = Tb3Geom<T, Q, K, RY, SY>;
  constexpr int M = 2 * K + 1, NPL = M;
  constexpr int NROW1 = G::RY1 + 2 * K, NROW2 = RY + 2 * K;
  constexpr int BW = G::BW, DZ = G::DZ, DI = G::DI;
  const Ssam3DParams<T, CAP>& p = P.p;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const bool stage1 = wib < G::SY;
  const int w = stage1 ? wib : wib - G::SY;
  const int y_cta0 = p.ring + blockIdx.y * G::ROWS2;
  const int z0 = p.z_begin + blockIdx.z * p.zseg;
  const int z1 = min(z0 + p.zseg, p.z_end);
  const int x_out0 = blockIdx.x * p.V;
  const int base = x_out0 - p.A;  // 16-byte aligned box origin
  const int x0 = base + Q * lane;
  const int n_in = (z1 - z0) + 4 * K;   // input planes z0-2K .. z1-1+2K
  const int n_mid = (z1 - z0) + 2 * K;  // intermediate planes z0-K .. z1-1+K

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* in_ring = reinterpret_cast<T*>(smem_raw);
  T* mid_ring = reinterpret_cast<T*>(smem_raw + DZ * G::IN_SLOT);
  uint64_t* in_full = reinterpret_cast<uint64_t*>(smem_raw + DZ * G::IN_SLOT + DI * G::MID_SLOT);
  uint64_t* in_empty = in_full + DZ;
  uint64_t* mid_full = in_empty + DZ;
  uint64_t* mid_empty = mid_full + DI;
  const uint32_t scratch = smem_u32(mid_empty + DI) + threadIdx.x * 4;
  if (threadIdx.x == 0) {
    prefetch_tmap(&P.tmap);
#pragma unroll
    for (int s = 0; s < DZ; ++s) {
      mbar_init(smem_u32(&in_full[s]), 1);
      mbar_init(smem_u32(&in_empty[s]), G::SY);
    }
#pragma unroll
    for (int s = 0; s < DI; ++s) {
      mbar_init(smem_u32(&mid_full[s]), G::SY);
      mbar_init(smem_u32(&mid_empty[s]), G::SY);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains

  if (stage1) {
    // ---- sweep 1: input planes -> intermediate band rows y_cta0-K .. ------
    const int box_y0 = y_cta0 - 2 * K;
    auto issue = [&](int i) {
      const int s = i % DZ;
      if (i >= DZ) mbar_wait(smem_u32(&in_empty[s]), ((i / DZ) - 1) & 1);
      const uint32_t bar = smem_u32(&in_full[s]);
      const int z = z0 - 2 * K + i;
      const int row = (z >= 0 && z < p.nz) ? z * p.ny + box_y0 : -G::BROWS;
      mbar_arrive_expect_tx(bar, static_cast<uint32_t>(G::BROWS * BW * sizeof(T)));
      tma_load_2d(smem_u32(in_ring + s * (G::IN_SLOT / sizeof(T))), &P.tmap, base, row, bar);
    };
    if (threadIdx.x == 0)
      for (int i = 0; i < min(DZ, n_in); ++i) issue(i);
    auto take = [&](int i, T (&dst)[NROW1][Q]) {
      const int s = i % DZ;
      mbar_wait(smem_u32(&in_full[s]), (i / DZ) & 1);
      const T* slot = in_ring + s * (G::IN_SLOT / sizeof(T)) + (w * G::RY1) * BW + Q * lane;
#pragma unroll
      for (int r = 0; r < NROW1; ++r) lds_q<T, Q>(slot + r * BW, dst[r]);
      wait_loaded<T, Q, NROW1>(dst, 0, NROW1, scratch);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&in_empty[s]));
      if (threadIdx.x == 0 && i >= 1 && i - 1 + DZ < n_in) issue(i - 1 + DZ);
    };
    const int xlo = p.ring, xhi = p.nx - p.ring;
    const int band0 = w * G::RY1;  // this warp's first band row (band row 0 = y_cta0-K)
    T pl[NPL][NROW1][Q];
#pragma unroll
    for (int i = 0; i < NPL - 1; ++i) take(i, pl[i]);
    for (int mb = 0; mb < n_mid; mb += NPL) {
#pragma unroll
      for (int ph = 0; ph < NPL; ++ph) {
        const int m = mb + ph;  // intermediate plane index: z = z0 - K + m
        if (m >= n_mid) break;
        take(m + 2 * K, pl[(ph + NPL - 1) % NPL]);
        const int z = z0 - K + m;
        const bool zring = z < p.zr_lo || z >= p.zr_hi;
        const int s = m % DI;
        if (m >= DI) mbar_wait(smem_u32(&mid_empty[s]), ((m / DI) - 1) & 1);
        T* dst = mid_ring + s * (G::MID_SLOT / sizeof(T)) + Q * lane;
#pragma unroll
        for (int r = 0; r < G::RY1; ++r) {
          const int br = band0 + r;
          if (br >= G::IROWS) break;
          T acc[Q];
          row_chain<T, Q, K, Mask, NROW1, NPL, CAP>(pl, ph, r, p, acc);
          // the global ring keeps its input value through a sweep
          const int y = y_cta0 - K + br;
          const bool yring = y < p.ring || y >= p.ny - p.ring;
          const T(&cen)[Q] = pl[(ph + K) % NPL][r + K];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int x = x0 + q;
            if (zring || yring || x < xlo || x >= xhi) acc[q] = cen[q];
          }
          st_q<T, Q>(dst + br * BW, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&mid_full[s]));
      }
    }
  } else {
    // ---- sweep 2: intermediate planes -> HBM ------------------------------
    const int y_out0 = y_cta0 + w * RY;
    const int xlo = p.ring, xhi = p.nx - p.ring;
    const int yhi = p.ny - p.ring;
    const bool owner = x0 >= x_out0 && x0 < x_out0 + p.V;
    const bool vec = p.vec_ok && x0 >= xlo && x0 + Q <= xhi;
    auto take = [&](int m, T (&dst)[NROW2][Q]) {
      const int s = m % DI;
      mbar_wait(smem_u32(&mid_full[s]), (m / DI) & 1);
      const T* slot = mid_ring + s * (G::MID_SLOT / sizeof(T)) + (w * RY) * BW + Q * lane;
#pragma unroll
      for (int r = 0; r < NROW2; ++r) lds_q<T, Q>(slot + r * BW, dst[r]);
      wait_loaded<T, Q, NROW2>(dst, 0, NROW2, scratch);
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&mid_empty[s]));
    };
    T pl[NPL][NROW2][Q];
#pragma unroll
    for (int i = 0; i < NPL - 1; ++i) take(i, pl[i]);
    for (int zb = z0; zb < z1; zb += NPL) {
#pragma unroll
      for (int ph = 0; ph < NPL; ++ph) {
        const int z = zb + ph;
        if (z >= z1) break;
        take(z - z0 + 2 * K, pl[(ph + NPL - 1) % NPL]);
        const bool mirror = PEER && mirrored3(p, z);
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          T acc[Q];
          row_chain<T, Q, K, Mask, NROW2, NPL, CAP>(pl, ph, r, p, acc);
          const int y = y_out0 + r;
          if (owner && y < yhi) store_row3<T, Q>(p, z, y, x0, acc, vec, xlo, xhi, mirror);
        }
      }
    }
  }
}

}  // namespace ssam_b200
