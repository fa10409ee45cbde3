// launch.cuh -- host-side launch planning for the SSAM engines.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "engine2d.cuh"
#include "engine3d.cuh"
#include "internal.hpp"
#include "tmap.hpp"

namespace ssam_b200 {

constexpr int kSMs = 148;          // B200: 2 dies x 74 SMs
constexpr int kWarpsPerBlock = 4;  // 128-thread blocks

// Launches with programmatic stream serialization (PDL) for the TMA kernels,
// which all start with griddep_wait(): back-to-back sweeps overlap one
// launch's ramp-up with the previous one's tail.  SSAM_B200_PDL=0 disables.
inline bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SSAM_B200_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return v;
}
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Lane plan for an M-column footprint, Q columns per lane (engine2d.cuh).
// R = (M-1)/2, L = M-1-R.  Lane 0 starts at the Q-aligned column
// x_out0 - A; with the bidirectional chain every lane's result sits in its
// own columns, valid where the L columns to the left and the R to the right
// are inside the warp: [origin + L, origin + 32Q - R).  The warp owns the
// Q-aligned run [x_out0, x_out0 + V) of that range.
struct LanePlan {
  int A, V;
};
inline LanePlan plan_lanes(int M, int Q) {
  const int R = (M - 1) / 2, L = M - 1 - R;
  LanePlan lp;
  lp.A = (L + Q - 1) / Q * Q;
  lp.V = (32 * Q - R - lp.A) / Q * Q;
  return lp;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

// Rows streamed per warp: enough warps for ~2 waves of ~24 resident warps/SM,
// but long enough that the NR-1 prologue rows stay a small overhead.
inline int seg_warps_per_sm() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_2D_WARPS_PER_SM");
    return e ? std::max(1, std::atoi(e)) : 48;
  }();
  return v;
}
inline int pick_seg(int rows, int nstrips, int nr) {
  const long long target_warps = static_cast<long long>(kSMs) * seg_warps_per_sm();
  long long segs = (target_warps + nstrips - 1) / nstrips;
  segs = std::max<long long>(1, std::min<long long>(segs, rows));
  int seg = static_cast<int>((rows + segs - 1) / segs);
  seg = std::max(seg, std::min(rows, 8 * nr));
  return std::max(seg, 1);
}

template <class T>
struct Engine2DArgs {
  const T* in;
  T* out;
  int W, H;
  int M, NR;
  const T* coef;  // host, [M][NR]
  int bmode, ring;
  int y_begin, y_end;
  bool direct = false;  // force the direct-load kernel (1-row grids: conv1d)
};

// Taps of a compile-time footprint (MC == 0: runtime width, count as dense 20).
template <class Mask>
constexpr int mask_taps(int mc, int nr) {
  int n = 0;
  for (int j = 0; j < (mc > 0 ? mc : 20); ++j)
    for (int t = 0; t < nr; ++t) n += Mask::has(j, t) ? 1 : 0;
  return n;
}
// TMA box depth: whole-window boxes (ping-pong register windows, fully
// unrolled) when the window is short and a row is light; otherwise 4-row
// boxes with one row body per loop trip.  About 6-10 rows in flight per warp.
constexpr int box_rows(int nr, int row_fmas) { return (nr <= 8 && row_fmas <= 256) ? nr : 4; }
constexpr int box_ring(int rb, int q, int tsize) {
  return std::max(2, ((q * tsize >= 32 ? 6 : 10) + rb - 1) / rb);
}

template <class T, int Q, int NR, int MC, class Mask, int PF, int CAP>
cudaError_t launch_ssam2d(const Engine2DArgs<T>& a, cudaStream_t s) {
  static_assert(MC == 0 || MC * NR <= CAP, "coefficient capacity");
  if (a.M * NR > CAP || a.NR != NR || (MC > 0 && a.M != MC)) return cudaErrorInvalidValue;
  if (a.y_end <= a.y_begin) return cudaSuccess;
  constexpr int VQ = 16 / sizeof(T);
  const bool tma = !a.direct && a.bmode != kBndReplicate && a.W % VQ == 0 && aligned16(a.in) &&
                   aligned16(a.out);
  Ssam2DTmaParams<T, CAP> P;
  std::memset(&P, 0, sizeof(P));
  Ssam2DParams<T, CAP>& p = P.p;
  p.in = a.in;
  p.out = a.out;
  p.W = a.W;
  p.H = a.H;
  p.M = a.M;
  const LanePlan lp = plan_lanes(a.M, Q);
  p.A = lp.A;
  p.V = lp.V;
  p.nstrips = (a.W + lp.V - 1) / lp.V;
  const int rows = a.y_end - a.y_begin;
  p.seg = pick_seg(rows, p.nstrips, NR);
  p.y_begin = a.y_begin;
  p.y_end = a.y_end;
  p.bmode = a.bmode;
  p.ring = a.ring;
  p.vec_ok = (a.W % Q == 0) && aligned16(a.in) && aligned16(a.out);
  std::memcpy(p.coef, a.coef, sizeof(T) * a.M * NR);
  const dim3 grid((p.nstrips + kWarpsPerBlock - 1) / kWarpsPerBlock, (rows + p.seg - 1) / p.seg);
  if (tma) {
    constexpr int RB = box_rows(NR, mask_taps<Mask>(MC, NR) * Q);
    constexpr int D = box_ring(RB, Q, sizeof(T));
    cudaError_t e = make_tmap_2d(&P.tmap, a.in, sizeof(T), a.W, a.H, sizeof(T) * a.W, 32 * Q, RB);
    if (e != cudaSuccess) return e;
    auto kern = ssam2d_tma_kernel<T, Q, NR, MC, Mask, RB, D, CAP>;
    const size_t smem = tma2d_smem<T, Q, RB, D>(kWarpsPerBlock);
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    e = launch_pdl(kern, grid, dim3(32 * kWarpsPerBlock), smem, s, P);
    if (e != cudaSuccess) return e;
  } else {
    ssam2d_kernel<T, Q, NR, MC, Mask, PF, CAP><<<grid, 32 * kWarpsPerBlock, 0, s>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

template <class T>
struct Engine3DArgs {
  const T* in;
  T* out;
  int nx, ny, nz;
  int K;
  const T* coef;  // host, [(2K+1)^3] as coef[(l*M + j)*M + t]
  int z_begin, z_end;
};

template <class P>
inline void apply_peer_halo(P& p) {
  using T = typename std::remove_pointer<decltype(p.out)>::type;
  if (const PeerHalo* h = peer_halo_slot()) {
    p.peer_lo = static_cast<T*>(h->lo);
    p.peer_lo_shift = h->lo_shift;
    p.peer_lo_end = h->lo_end;
    p.peer_hi = static_cast<T*>(h->hi);
    p.peer_hi_shift = h->hi_shift;
    p.peer_hi_begin = h->hi_begin;
  }
}

constexpr int kRing3D = 4;  // TMA plane slots per CTA ring (3D engine)

// Warps per 3D CTA (each RY rows); SSAM_B200_3D_WPB overrides (4 or 8).
inline int cta_warps_3d() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_3D_WPB");
    const int w = e ? std::atoi(e) : 0;  // 0: per-stencil default
    return w >= 8 ? 8 : (w >= 4 ? 4 : 0);
  }();
  return v;
}
// Adjacent x-strips per 3D CTA (1 or 2); SSAM_B200_3D_SX overrides.
inline int cta_strips_3d() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_3D_SX");
    return e ? std::atoi(e) : 0;  // 0: per-stencil default
  }();
  return v;
}

// The halo-lane 3D kernel (engine3d.cuh) exists for order >= 1 x-symmetric
// masks except the 125-tap box.  Measured (B200, 512^3 and 2048^2x514, vs
// the aligned-plan kernel, bit-identical): fp32 3d7pt +12% / +1.3%, 3d13pt
// fp32 +22%, fp64 +8%, fp32 Poisson +7% (halo weights as constant-bank
// operands, 3 CTAs/SM); the fp32 27-point box is even and the fp64 order-1
// footprints lose 8-17% (registers), so they keep the aligned plan.  SSAM_B200_3D_HALO=0/1 forces it off/on where it exists.
inline int halo_mode_3d() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_3D_HALO");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
template <class T, int K, class Mask>
constexpr bool halo_default_3d() {
  return std::is_same<Mask, StarMask3<2>>::value || std::is_same<Mask, StarMask3<1>>::value ||
         (sizeof(T) == 4 && std::is_same<Mask, PoissonMask3>::value);
}

// CTA order of the TMA kernels.  The hardware launches blockIdx.x fastest,
// then y, then z.  (x, y-group, z-segment) re-reads each segment's 2K halo
// planes long after the neighbouring segment read them (HBM, not L2);
// (x, z-segment, y-group) makes z-neighbours concurrent instead.  Measured on
// B200 the second order is SLOWER everywhere (3d7pt 2048^2x514: 774 -> 718
// GCells/s; 512^3 cases -3..6%), so (x, y, z) stays the default;
// SSAM_B200_3D_ZFAST=1 selects the other.
inline int zfast_3d() {
  static const int v = [] {
    const char* e = std::getenv("SSAM_B200_3D_ZFAST");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
template <class P3>
dim3 grid3d(P3& p, int gx, int gy, int gz) {
  p.zfast = zfast_3d() != 0 && gz <= 65535;
  return p.zfast ? dim3(gx, gz, gy) : dim3(gx, gy, gz);
}

template <class T, int Q, int K, class Mask, int RY, int CAP, int RYH = RY>
cudaError_t launch_ssam3d(const Engine3DArgs<T>& a, cudaStream_t s) {
  constexpr int M = 2 * K + 1;
  static_assert(M * M * M <= CAP, "coefficient capacity");
  if (a.K != K) return cudaErrorInvalidValue;
  const int zb = std::max(a.z_begin, K), ze = std::min(a.z_end, a.nz - K);
  const int yrows = a.ny - 2 * K;
  if (ze <= zb || yrows <= 0 || a.nx - 2 * K <= 0) return cudaSuccess;
  constexpr int VQ = 16 / sizeof(T);
  const bool tma = a.nx % VQ == 0 && aligned16(a.in) && aligned16(a.out);
  Ssam3DTmaParams<T, CAP> P;
  std::memset(&P, 0, sizeof(P));
  Ssam3DParams<T, CAP>& p = P.p;
  apply_peer_halo(p);
  p.in = a.in;
  p.out = a.out;
  p.nx = a.nx;
  p.ny = a.ny;
  p.nz = a.nz;
  const LanePlan lp = plan_lanes(M, Q);
  p.A = lp.A;
  p.V = lp.V;
  p.nstrips = (a.nx + lp.V - 1) / lp.V;
  p.ygroups = (yrows + RY - 1) / RY;
  p.ring = K;
  p.vec_ok = (a.nx % Q == 0) && aligned16(a.in) && aligned16(a.out);
  const int zrows = ze - zb;
  // Short z-segments (measured: 608 -> 726 GCells/s for 3d7pt at 2048^2x514
  // going from whole-z CTAs to 32 planes): many short CTAs keep the machine
  // evenly loaded to the end and keep vertically adjacent CTAs in step, so
  // their shared halo rows still hit in L2.  The 2K-plane prologue per
  // segment is the price; SSAM_B200_3D_ZSEG overrides.
  // Sweep at 2048^2 x 514 f32: 3d7pt best at 16-24 planes, the heavier
  // poisson / 3d27pt / 3d13pt (compute-bound) at 48-64.
  const bool light7 = std::is_same<Mask, StarMask3<1>>::value;
  int zseg = std::min(zrows, light7 ? 24 : 32 * std::max(1, K) + 16);
  if (const char* zs = std::getenv("SSAM_B200_3D_ZSEG")) zseg = std::max(4, std::atoi(zs));
  p.zseg = zseg;
  p.z_begin = zb;
  p.z_end = ze;
  std::memcpy(p.coef, a.coef, sizeof(T) * M * M * M);
  bool launched = false;
  if constexpr (K >= 1 && !(K >= 2 && std::is_same<Mask, DenseMask3>::value)) {
    const int hm = halo_mode_3d();
    if (tma && (hm > 0 || (hm < 0 && halo_default_3d<T, K, Mask>()))) {
      // Full-warp lane plan with halo lanes (ssam3d_halo_kernel): every warp
      // emits 32Q columns; CTA = sx strips x sy row groups, one box per strip.
      constexpr int DZ = kRing3D;
      constexpr int VQ = 16 / sizeof(T);
      p.A = 0;
      p.V = 32 * Q;
      p.nstrips = (a.nx - K + p.V - 1) / p.V;
      const bool light = std::is_same<Mask, StarMask3<1>>::value;
      int wpb = cta_warps_3d() ? cta_warps_3d() : (light ? 8 : 4);
      wpb = std::min(wpb, halo3d_max_threads<T, K, Mask>() / 32);  // the kernel's launch bound
      const int want_sx = cta_strips_3d() ? cta_strips_3d() : (light ? 2 : 1);
      int sx = (want_sx >= 2 && p.nstrips >= 2) ? 2 : 1;
      auto fits = [&](int w, int x) {
        const int yy = w / x;
        return yy * RYH + 2 * K <= 256 && halo3d_bytes<T, Q, RYH, K, DZ>(x, yy) <= 200 * 1024;
      };
      while (wpb > sx * 2 && !fits(wpb, sx)) wpb /= 2;
      const int sy = wpb / sx;
      p.cta_sx = sx;
      p.ygroups = (yrows + RYH - 1) / RYH;
      const dim3 grid = grid3d(p, (p.nstrips + sx - 1) / sx, (p.ygroups + sy - 1) / sy,
                               (zrows + zseg - 1) / zseg);
      cudaError_t e = make_tmap_2d(&P.tmap, a.in, sizeof(T), a.nx,
                                   static_cast<uint64_t>(a.ny) * a.nz, sizeof(T) * a.nx,
                                   32 * Q + 2 * VQ, sy * RYH + 2 * K);
      if (e != cudaSuccess) return e;
      auto kern = peer_halo_slot() ? ssam3d_halo_kernel<T, Q, K, Mask, RYH, DZ, CAP, true>
                                   : ssam3d_halo_kernel<T, Q, K, Mask, RYH, DZ, CAP, false>;
      const size_t smem = halo3d_bytes<T, Q, RYH, K, DZ>(sx, sy);
      if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      e = launch_pdl(kern, grid, dim3(32 * wpb), smem, s, P);
      if (e != cudaSuccess) return e;
      launched = true;
    }
  }
  if (launched) {
    // halo kernel above
  } else if (tma) {
    // Taller CTAs share more of the y halo (2K rows per wpb*RY); the box
    // must stay within TMA's 256-row limit and the ring within shared memory.
    // CTA = sx adjacent strips x sy row groups sharing one plane box: wider
    // boxes halve the x-halo re-reads and make each row fetch ~1 KB
    // contiguous.  Box limits: 256 elements per dimension, shared memory.
    constexpr int DZ = kRing3D;
    // Measured defaults: the light 7-point star streams best from 2-strip x
    // 4-row-group CTAs; heavier footprints from 1 x 4.
    const bool light = std::is_same<Mask, StarMask3<1>>::value;
    int wpb = cta_warps_3d() ? cta_warps_3d() : (light ? 8 : 4);
    const int want_sx = cta_strips_3d() ? cta_strips_3d() : (light ? 2 : 1);
    int sx = (want_sx >= 2 && lp.V + 32 * Q <= 256 && p.nstrips >= 2) ? 2 : 1;
    auto fits = [&](int w, int x) {
      const int yy = w / x;
      return yy * RY + 2 * K <= 256 && ring3d_bytes<T, Q, RY, K, DZ>(x, yy, lp.V) <= 200 * 1024;
    };
    while (wpb > sx * 2 && !fits(wpb, sx)) wpb /= 2;
    const int sy = wpb / sx;
    p.cta_sx = sx;
    const dim3 grid = grid3d(p, (p.nstrips + sx - 1) / sx, (p.ygroups + sy - 1) / sy,
                             (zrows + zseg - 1) / zseg);
    cudaError_t e = make_tmap_2d(&P.tmap, a.in, sizeof(T), a.nx,
                                 static_cast<uint64_t>(a.ny) * a.nz, sizeof(T) * a.nx,
                                 (sx - 1) * lp.V + 32 * Q, sy * RY + 2 * K);
    if (e != cudaSuccess) return e;
    auto kern = peer_halo_slot() ? ssam3d_tma_kernel<T, Q, K, Mask, RY, DZ, CAP, true>
                                 : ssam3d_tma_kernel<T, Q, K, Mask, RY, DZ, CAP, false>;
    const size_t smem = ring3d_bytes<T, Q, RY, K, DZ>(sx, sy, lp.V);
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    e = launch_pdl(kern, grid, dim3(32 * wpb), smem, s, P);
    if (e != cudaSuccess) return e;
  } else {
    const dim3 grid(p.nstrips, (p.ygroups + kWarpsPerBlock - 1) / kWarpsPerBlock,
                    (zrows + zseg - 1) / zseg);
    auto kern = peer_halo_slot() ? ssam3d_kernel<T, Q, K, Mask, RY, CAP, true>
                                 : ssam3d_kernel<T, Q, K, Mask, RY, CAP, false>;
    kern<<<grid, 32 * kWarpsPerBlock, 0, s>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace ssam_b200
