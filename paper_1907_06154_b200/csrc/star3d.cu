// star3d.cu -- launchers of the order-1 3D star pipeline (engine3d_star.cuh):
// single sweeps (TB = 1) and TB = 2..4 fused sweeps per HBM pass.
//
// Reference: ssam::stencil3d (proj/include/ssam/kernels.hpp:283-384) for the
// 7-point star of the catalog (stencil_catalog.cpp:47-52, any coefficients).
#include "engine3d_star.cuh"
#include "launch.cuh"

namespace ssam_b200 {

// SSAM_B200_STAR=0 routes the star back to the generic 3D engines (A/B).
bool star3d_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_STAR");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

template <class T, int TB>
cudaError_t launch_star3d(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                          int zr_lo, int zr_hi, const T* coef27, cudaStream_t s) {
  using G = StarGeom<T, TB>;
  constexpr int Q = G::Q, VQ = 16 / sizeof(T);
  if (nx % VQ != 0 || !aligned16(d_in) || !aligned16(d_out)) return cudaErrorNotSupported;
  // outputs [z_begin, z_end) inside the buffer's interior and the global
  // interior [zr_lo, zr_hi); the pipeline reads planes z_begin-TB .. z_end-1+TB
  const int zb = std::max({z_begin, zr_lo, 1}), ze = std::min({z_end, zr_hi, nz - 1});
  if (ze <= zb || ny < 3 || nx < 3) return cudaSuccess;
  Ssam3DTmaParams<T, 27> P;
  std::memset(&P, 0, sizeof(P));
  Ssam3DParams<T, 27>& p = P.p;
  apply_peer_halo(p);
  p.in = d_in;
  p.out = d_out;
  p.nx = nx;
  p.ny = ny;
  p.nz = nz;
  const LanePlan lp = plan_lanes(2 * TB + 1, Q);  // TB sweeps: TB columns each side
  p.A = lp.A;
  p.V = lp.V;
  p.nstrips = (nx - 1 + lp.V - 1) / lp.V;
  p.ring = 1;
  p.vec_ok = 1;
  const int yrows = ny - 2, zrows = ze - zb;
  const int ybands = (yrows + G::ROWS - 1) / G::ROWS;
  // Long z-segments amortise the 2 TB prologue planes of a segment while the
  // grid keeps ~4 waves of CTAs; SSAM_B200_3D_TB_ZSEG overrides.
  const long long xy_ctas = static_cast<long long>(p.nstrips) * ybands;
  int zseg = std::min(zrows, 128);
  while (zseg > 16 && xy_ctas * ((zrows + zseg - 1) / zseg) < 4LL * G::MINB * kSMs) zseg /= 2;
  if (const char* e = std::getenv("SSAM_B200_3D_TB_ZSEG")) zseg = std::max(4, std::atoi(e));
  p.zseg = zseg;
  p.z_begin = zb;
  p.z_end = ze;
  p.zr_lo = zr_lo;
  p.zr_hi = zr_hi;
  std::memcpy(p.coef, coef27, sizeof(T) * 27);
  const dim3 grid(p.nstrips, ybands, (zrows + zseg - 1) / zseg);
  if (grid.y > 65535 || grid.z > 65535) return cudaErrorNotSupported;
  cudaError_t e = make_tmap_2d(&P.tmap, d_in, sizeof(T), nx, static_cast<uint64_t>(ny) * nz,
                               sizeof(T) * nx, G::BW, G::IN_ROWS);
  if (e != cudaSuccess) return e;
  auto kern = peer_halo_slot() ? star3d_kernel<T, TB, true> : star3d_kernel<T, TB, false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, grid, dim3(G::THREADS), G::SMEM, s, P);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

template <class T>
cudaError_t star3d_direct(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                          const T* coef27, cudaStream_t s) {
  const int zb = std::max(z_begin, 1), ze = std::min(z_end, nz - 1);
  if (ze <= zb || ny < 3 || nx < 3) return cudaSuccess;
  Ssam3DParams<T, 27> p;
  std::memset(&p, 0, sizeof(p));
  apply_peer_halo(p);
  p.in = d_in;
  p.out = d_out;
  p.nx = nx;
  p.ny = ny;
  p.nz = nz;
  p.z_begin = zb;
  p.z_end = ze;
  std::memcpy(p.coef, coef27, sizeof(T) * 27);
  const dim3 grid((nx - 2 + 127) / 128, std::min(ny - 2, 65535), std::min(ze - zb, 65535));
  if (peer_halo_slot())
    star3d_direct_kernel<T, true><<<grid, 128, 0, s>>>(p);
  else
    star3d_direct_kernel<T, false><<<grid, 128, 0, s>>>(p);
  note_launch();
  return cudaGetLastError();
}

template <class T>
cudaError_t star3d_sweep(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                         const T* coef27, cudaStream_t s) {
  cudaError_t e = launch_star3d<T, 1>(d_in, d_out, nx, ny, nz, z_begin, z_end, 1, nz - 1, coef27, s);
  if (e != cudaErrorNotSupported) return e;
  cudaGetLastError();
  return star3d_direct<T>(d_in, d_out, nx, ny, nz, z_begin, z_end, coef27, s);
}

template <class T>
cudaError_t star3d_tb(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                      int zr_lo, int zr_hi, const T* coef27, int tb, cudaStream_t s) {
  switch (tb) {
    case 2: return launch_star3d<T, 2>(d_in, d_out, nx, ny, nz, z_begin, z_end, zr_lo, zr_hi, coef27, s);
    case 3: return launch_star3d<T, 3>(d_in, d_out, nx, ny, nz, z_begin, z_end, zr_lo, zr_hi, coef27, s);
    case 4: return launch_star3d<T, 4>(d_in, d_out, nx, ny, nz, z_begin, z_end, zr_lo, zr_hi, coef27, s);
  }
  return cudaErrorNotSupported;
}

template cudaError_t star3d_sweep<float>(const float*, float*, int, int, int, int, int, const float*, cudaStream_t);
template cudaError_t star3d_sweep<double>(const double*, double*, int, int, int, int, int, const double*, cudaStream_t);
template cudaError_t star3d_tb<float>(const float*, float*, int, int, int, int, int, int, int, const float*, int, cudaStream_t);
template cudaError_t star3d_tb<double>(const double*, double*, int, int, int, int, int, int, int, const double*, int, cudaStream_t);

}  // namespace ssam_b200
