// internal.hpp -- host-side contracts between the C ABI (abi.cpp) and the
// kernel launchers (*.cu).  No reference or torch types; plain pointers.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace ssam_b200 {

enum class Shape2D { other, star };
enum class Shape3D { other, star, box, poisson };

struct Tap {
  int dx, dy, dz;
};

// Tap-set classification used for kernel selection; the coefficients are
// always the caller's (any values), only the offset set is matched.
Shape2D classify2d(const std::vector<Tap>& taps, int order);
Shape3D classify3d(const std::vector<Tap>& taps, int order);

template <class T>
struct StencilDesc {
  int dims = 2;
  int order = 0;
  std::vector<Tap> taps;
  std::vector<T> coeffs;
};

// ---- conv2d: out = sum_{s,t} in(x+ax-s, y+ay-t) * w[s*n+t] -----------------
// d_in/d_out device pointers (distinct); h_w host pointer to m*n weights.
// Output rows [y_begin, y_end); rows outside [0, H) are the image boundary.
template <class T>
cudaError_t conv2d_device(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                          const T* h_w, int m, int n, int boundary, cudaStream_t s);

// ---- one Jacobi sweep (2D), interior cells only ---------------------------
// Writes next(x,y) for k <= x < W-k and y in [y_begin, y_end) ∩ [k, H-k).
// Ring cells of d_out are left untouched (callers keep them equal to the
// input ring).
template <class T>
cudaError_t stencil2d_sweep(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                            const StencilDesc<T>& st, cudaStream_t s);

// Tb fused sweeps (temporal blocking).  Returns cudaErrorNotSupported when no
// fused kernel exists for this stencil/dtype/Tb (the caller then sweeps).
template <class T>
cudaError_t stencil2d_tb(const T* d_in, T* d_out, int W, int H, const StencilDesc<T>& st, int tb,
                         cudaStream_t s);
int stencil2d_tb_max(int dtype, int order, bool star);
// stencil2d_tb over output rows [y_begin, y_end) with the global ring outside
// rows [yr_lo, yr_hi) (row slabs pass local bounds).
template <class T>
cudaError_t stencil2d_tb_range(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                               int yr_lo, int yr_hi, const StencilDesc<T>& st, int tb,
                               cudaStream_t s);

// ---- one Jacobi sweep (3D) over output planes [z_begin, z_end) ------------
// Plane indices are global to the (nz-plane) buffer; the ring test uses
// ring_lo/ring_hi for z so a slab can place the true domain faces.
template <class T>
cudaError_t stencil3d_sweep(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                            int z_end, const StencilDesc<T>& st, cudaStream_t s);

// Tb fused 3D sweeps (temporal blocking) writing planes [z_begin, z_end) of
// the interior; planes outside [zr_lo, zr_hi) are the global ring (kept
// fixed), so a z-slab with k*Tb ghost planes passes its local bounds.
// Returns cudaErrorNotSupported when no fused kernel exists.
template <class T>
cudaError_t stencil3d_tb(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                         int zr_lo, int zr_hi, const StencilDesc<T>& st, int tb, cudaStream_t s);

// ---- the 3D pipeline engine (engine3d_pipe.cuh, pipe3d_*.cu) -------------
// coef: host, the dense (2K+1)^3 layout coef[(l*M + j)*M + t] (l = dz+K,
// j = dx+K, t = dy+K).  tb = 1 is one sweep over output planes [z_begin,
// z_end) (aligned: the pipeline; otherwise the direct-load kernel); tb >= 2
// fuses tb sweeps (order-1 star: 2..4; order-2 star and the box family: 2)
// with the global ring outside planes [zr_lo, zr_hi); cudaErrorNotSupported
// for unaligned grids or depths without a kernel.
bool pipe3d_enabled();
template <class T>
cudaError_t pipe3d_star1(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                         int zr_lo, int zr_hi, const T* coef, int tb, cudaStream_t s);
template <class T>
cudaError_t pipe3d_star2(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin, int z_end,
                         int zr_lo, int zr_hi, const T* coef, int tb, cudaStream_t s);
template <class T>
cudaError_t pipe3d_box(bool poisson, const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                       int z_end, int zr_lo, int zr_hi, const T* coef, int tb, cudaStream_t s);
// The fused depth stencil3d_run uses for a (dtype, order, shape): measured
// per shape; SSAM_B200_3D_TB caps it (1 = single sweeps).
int stencil3d_tb_max(int dtype, int order, Shape3D shape);

// ---- one process, several devices (multi.cpp) --------------------------------
// Host grid in -> `iters` sweeps on slabs along the slowest axis (rows in 2D,
// nz = 1; z-planes in 3D), slab g on devices[g] with k*tb ghost planes per
// shared face, halos by cudaMemcpyPeerAsync overlapped with the interior ->
// host grid out.  Bit-identical to the one-device run.  *used = the number
// of slabs (fewer than ndev when a slab would own fewer than k*tb planes).
template <class T>
cudaError_t multi_stencil(const T* h_in, T* h_out, int nx, int ny, int nz, const StencilDesc<T>& st,
                          int iters, int tb, const int* devices, int ndev, int* used);

// ---- direct-gather kernels (generic path: any order / tap set) -------------
// Bit-faithful to the oracle's summation order (double accumulation for FP,
// no FMA contraction), used where no SSAM specialisation applies.
template <class T>
cudaError_t conv2d_direct(const T* d_in, T* d_out, int W, int H, const T* h_w, int m, int n,
                          int boundary, cudaStream_t s);
template <class T>
cudaError_t stencil2d_direct(const T* d_in, T* d_out, int W, int H, int y_begin, int y_end,
                             const StencilDesc<T>& st, cudaStream_t s);
template <class T>
cudaError_t stencil3d_direct(const T* d_in, T* d_out, int nx, int ny, int nz, int z_begin,
                             int z_end, const StencilDesc<T>& st, cudaStream_t s);

// ---- 1D: conv1d and scan (kernels.hpp:390-447) -------------------------------
// conv1d: out(i) = sum_{s<m} in(i + (m-1)/2 - s) * w[s], m <= 32 (the
// reference's lane_count cap), boundary zero or replicate.
template <class T>
cudaError_t conv1d_device(const T* d_in, T* d_out, int len, const T* h_w, int m, int boundary,
                          cudaStream_t s);
// Inclusive prefix sum of n elements (reduce, carry, scan: fixed order).
template <class T>
cudaError_t scan_device(const T* d_in, T* d_out, size_t n, cudaStream_t s);

// ---- latency micro-benchmarks (latency.cu): t[0..7] = t_shfl, t_mad,
// t_smem_read, t_reg, t_gmem_read, t_gmem_write, t_l2_read (cycles), SM MHz
cudaError_t measure_latency(double* t, cudaStream_t s);

// ---- utilities --------------------------------------------------------------
// Stream-ordered scratch from the engine's private per-device pool (freed
// blocks stay cached; the device's default pool is never touched).  Free
// with cudaFreeAsync.
cudaError_t engine_alloc(void** p, std::size_t bytes, cudaStream_t s);
cudaError_t fill_random(int dtype, void* d, std::size_t count, std::uint64_t seed,
                        std::uint64_t first, cudaStream_t s);
// max |a-b| / max(1,|b|) and max |a-b| over count elements, into host doubles.
cudaError_t max_rel_err(int dtype, const void* d_a, const void* d_b, std::size_t count,
                        double* h_rel, double* h_abs, cudaStream_t s);

// Peer-memory halo of the 3D sweep being launched on this thread (slab runs,
// ssam_peer_halo in ssam_b200.h): the z-streaming kernels also store output
// planes z < lo_end to `lo` (+ lo_shift elements) and z >= hi_begin to `hi`.
struct PeerHalo {
  void* lo;
  long long lo_shift;
  int lo_end;
  void* hi;
  long long hi_shift;
  int hi_begin;
};
const PeerHalo*& peer_halo_slot();
// Whether stencil3d_sweep / stencil3d_tb of this stencil run a kernel that
// honours the peer halo (the register engines; the direct kernel does not).
bool stencil3d_peer_fused(int dtype, int order);

// How many launches of our kernels the last host call issued (bench evidence).
void note_launch();
std::uint64_t launches();

}  // namespace ssam_b200
