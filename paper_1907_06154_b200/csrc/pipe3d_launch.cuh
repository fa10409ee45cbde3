// pipe3d_launch.cuh -- host launchers of the 3D pipeline engine
// (engine3d_pipe.cuh): single sweeps (TB = 1), TB fused sweeps per HBM pass,
// and the direct-load kernel for grids whose rows are not 16-byte aligned.
//
// Reference: ssam::stencil3d (proj/include/ssam/kernels.hpp:283-384).
#pragma once

#include "engine3d_pipe.cuh"
#include "launch.cuh"

namespace ssam_b200 {

template <class T, class Sh, int TB>
cudaError_t launch_pipe3d(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                          int zr_lo, int zr_hi, const T* coef, cudaStream_t s) {
  using G = PipeGeom<T, Sh, TB>;
  constexpr int K = Sh::K, Q = G::Q, VQ = 16 / sizeof(T), CAP = G::CAP;
  if (nx % VQ != 0 || !aligned16(d_in) || !aligned16(d_out)) return cudaErrorNotSupported;
  // outputs [z_begin, z_end) inside the buffer's interior and the global
  // interior [zr_lo, zr_hi); the pipeline reads planes z_begin-K TB .. z_end-1+K TB
  const int zb = std::max({z_begin, zr_lo, K}), ze = std::min({z_end, zr_hi, nz - K});
  if (ze <= zb || ny <= 2 * K || nx <= 2 * K) return cudaSuccess;
  Ssam3DTmaParams<T, CAP> P;
  std::memset(&P, 0, sizeof(P));
  Ssam3DParams<T, CAP>& p = P.p;
  apply_peer_halo(p);
  p.in = d_in;
  p.out = d_out;
  p.nx = nx;
  p.ny = ny;
  p.nz = nz;
  const LanePlan lp = plan_lanes(2 * K * TB + 1, Q);  // TB sweeps: K TB columns each side
  p.A = lp.A;
  p.V = lp.V;
  p.nstrips = (nx - K + lp.V - 1) / lp.V;
  p.ring = K;
  p.vec_ok = 1;
  const int yrows = ny - 2 * K, zrows = ze - zb;
  const int ybands = (yrows + G::ROWS - 1) / G::ROWS;
  // Long z-segments amortise the 2 K TB prologue planes of a segment while
  // the grid keeps ~4 waves of CTAs; SSAM_B200_3D_TB_ZSEG overrides.
  const long long xy_ctas = static_cast<long long>(p.nstrips) * ybands;
  int zseg = std::min(zrows, 128);
  while (zseg > 16 && xy_ctas * ((zrows + zseg - 1) / zseg) < 4LL * G::MINB * kSMs) zseg /= 2;
  if (const char* e = std::getenv("SSAM_B200_3D_TB_ZSEG")) zseg = std::max(4, std::atoi(e));
  p.zseg = zseg;
  p.z_begin = zb;
  p.z_end = ze;
  p.zr_lo = zr_lo;
  p.zr_hi = zr_hi;
  std::memcpy(p.coef, coef, sizeof(T) * CAP);
  const dim3 grid(p.nstrips, ybands, (zrows + zseg - 1) / zseg);
  if (grid.y > 65535 || grid.z > 65535) return cudaErrorNotSupported;
  cudaError_t e = make_tmap_2d(&P.tmap, d_in, sizeof(T), nx, static_cast<uint64_t>(ny) * nz,
                               sizeof(T) * nx, G::BW, G::IN_ROWS);
  if (e != cudaSuccess) return e;
  auto kern = peer_halo_slot() ? pipe3d_kernel<T, Sh, TB, true> : pipe3d_kernel<T, Sh, TB, false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, grid, dim3(G::THREADS), G::SMEM, s, P);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

template <class T, class Sh>
cudaError_t launch_pipe3d_direct(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                                 int z_end, const T* coef, cudaStream_t s) {
  constexpr int K = Sh::K, CAP = (2 * K + 1) * (2 * K + 1) * (2 * K + 1);
  const int zb = std::max(z_begin, K), ze = std::min(z_end, nz - K);
  if (ze <= zb || ny <= 2 * K || nx <= 2 * K) return cudaSuccess;
  Ssam3DParams<T, CAP> p;
  std::memset(&p, 0, sizeof(p));
  apply_peer_halo(p);
  p.in = d_in;
  p.out = d_out;
  p.nx = nx;
  p.ny = ny;
  p.nz = nz;
  p.z_begin = zb;
  p.z_end = ze;
  std::memcpy(p.coef, coef, sizeof(T) * CAP);
  const dim3 grid((nx - 2 * K + 127) / 128, std::min(ny - 2 * K, 65535), std::min(ze - zb, 65535));
  if (peer_halo_slot())
    pipe3d_direct_kernel<T, Sh, true, CAP><<<grid, 128, 0, s>>>(p);
  else
    pipe3d_direct_kernel<T, Sh, false, CAP><<<grid, 128, 0, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

// One sweep: the aligned pipeline (TB = 1), else the direct-load kernel.
template <class T, class Sh>
cudaError_t pipe3d_sweep_sh(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                            int z_end, const T* coef, cudaStream_t s) {
  constexpr int K = Sh::K;
  cudaError_t e = launch_pipe3d<T, Sh, 1>(d_in, d_out, nx, ny, nz, z_begin, z_end, K, nz - K, coef, s);
  if (e != cudaErrorNotSupported) return e;
  cudaGetLastError();
  return launch_pipe3d_direct<T, Sh>(d_in, d_out, nx, ny, nz, z_begin, z_end, coef, s);
}

}  // namespace ssam_b200
