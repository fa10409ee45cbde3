// multi.cpp -- one process, several GPUs: the slab engine behind
// ssam_b200_stencil2d_multi / ssam_b200_stencil3d_multi.
//
// Reference: ssam::stencil2d / ssam::stencil3d (proj/include/ssam/
// kernels.hpp:231-277, :283-384) -- the same Jacobi semantics, the grid cut
// into slabs along its slowest axis (rows in 2D, z-planes in 3D; SURVEY
// §8(e)).  Slab g lives on devices[g] with G = k * Tb ghost planes on each
// face it shares with a neighbour (none on the true domain faces), so one
// fused launch of Tb sweeps needs no data from outside the slab.
//
// Per round (Tb sweeps, or the remainder), for every slab:
//   compute stream: wait for the neighbours' (and its own) halo copies of
//                   the previous round; launch the two boundary bands (the
//                   G owned planes next to each shared face), record `bnd`;
//                   launch the interior.
//   copy stream:    wait `bnd`; cudaMemcpyPeerAsync the boundary bands into
//                   the neighbours' ghost planes of the buffer they read in
//                   the next round (NVLink P2P with peer access enabled);
//                   record `cp`.
// The copies overlap the interior launch.  Ghost planes are read only by
// the boundary launches and owned planes only written by their own slab,
// so the event graph above orders every read before the write that
// replaces it.  Every launch is the single-device kernel on a
// local buffer with the global ring passed in local coordinates, and fused
// launches equal single sweeps bit for bit, so the result equals the
// one-device call bit for bit for any slab count.
#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "internal.hpp"

namespace ssam_b200 {

namespace {

template <class T>
struct Slab {
  int dev = 0;
  int z0 = 0, z1 = 0;    // owned global planes [z0, z1)
  int glo = 0, ghi = 0;  // ghost planes below / above
  int nl = 0;            // local planes = glo + owned + ghi
  T* buf[2] = {nullptr, nullptr};
  cudaStream_t cs = nullptr, xs = nullptr;
  cudaEvent_t bnd = nullptr, cp = nullptr;
  int owned() const { return z1 - z0; }
};

struct DeviceGuard {
  int dev = 0;
  DeviceGuard() { cudaGetDevice(&dev); }
  ~DeviceGuard() { cudaSetDevice(dev); }
};

template <class T>
cudaError_t launch_band(int dims, const T* in, T* out, int nx, int ny, int nl, int zb, int ze,
                        int zr_lo, int zr_hi, const StencilDesc<T>& st, int depth,
                        cudaStream_t s) {
  if (ze <= zb) return cudaSuccess;
  if (dims == 3) {
    if (depth > 1) return stencil3d_tb<T>(in, out, nx, ny, nl, zb, ze, zr_lo, zr_hi, st, depth, s);
    return stencil3d_sweep<T>(in, out, nx, ny, nl, zb, ze, st, s);
  }
  if (depth > 1) return stencil2d_tb_range<T>(in, out, nx, nl, zb, ze, zr_lo, zr_hi, st, depth, s);
  return stencil2d_sweep<T>(in, out, nx, nl, zb, ze, st, s);
}

}  // namespace

template <class T>
cudaError_t multi_stencil(const T* h_in, T* h_out, int nx, int ny, int nz, const StencilDesc<T>& st,
                          int iters, int tb, const int* devices, int ndev, int* used) {
  const int dims = st.dims;
  // 2D: a "plane" is one row of nx cells, nplanes = ny
  const int nplanes = dims == 3 ? nz : ny;
  const size_t pe = dims == 3 ? static_cast<size_t>(nx) * ny : static_cast<size_t>(nx);
  const int k = st.order;
  tb = std::max(1, tb);
  const int G = std::max(1, k * tb);
  // slabs must own at least G planes (a neighbour's ghosts come from one slab)
  int n = std::max(1, std::min(ndev, nplanes / std::max(G, 2 * k + 1)));
  if (used) *used = n;

  DeviceGuard guard;
  std::vector<Slab<T>> sl(n);
  cudaError_t e = cudaSuccess;
  auto cleanup = [&]() {
    for (auto& s : sl) {
      if (cudaSetDevice(s.dev) != cudaSuccess) continue;
      if (s.cs) cudaStreamSynchronize(s.cs);
      if (s.xs) cudaStreamSynchronize(s.xs);
      for (T* b : s.buf)
        if (b) cudaFree(b);
      if (s.bnd) cudaEventDestroy(s.bnd);
      if (s.cp) cudaEventDestroy(s.cp);
      if (s.cs) cudaStreamDestroy(s.cs);
      if (s.xs) cudaStreamDestroy(s.xs);
    }
  };
#define SSAM_TRY(x)        \
  do {                     \
    e = (x);               \
    if (e != cudaSuccess) { \
      cleanup();           \
      return e;            \
    }                      \
  } while (0)

  for (int g = 0; g < n; ++g) {
    Slab<T>& s = sl[g];
    s.dev = devices[g];
    s.z0 = static_cast<int>(static_cast<long long>(nplanes) * g / n);
    s.z1 = static_cast<int>(static_cast<long long>(nplanes) * (g + 1) / n);
    s.glo = g > 0 ? G : 0;
    s.ghi = g < n - 1 ? G : 0;
    s.nl = s.owned() + s.glo + s.ghi;
    SSAM_TRY(cudaSetDevice(s.dev));
    SSAM_TRY(cudaStreamCreateWithFlags(&s.cs, cudaStreamNonBlocking));
    SSAM_TRY(cudaStreamCreateWithFlags(&s.xs, cudaStreamNonBlocking));
    SSAM_TRY(cudaEventCreateWithFlags(&s.bnd, cudaEventDisableTiming));
    SSAM_TRY(cudaEventCreateWithFlags(&s.cp, cudaEventDisableTiming));
    const size_t bytes = static_cast<size_t>(s.nl) * pe * sizeof(T);
    // plain allocations: peers copy into them (pool memory would need
    // per-peer access descriptors)
    SSAM_TRY(cudaMalloc(&s.buf[0], bytes));
    SSAM_TRY(cudaMalloc(&s.buf[1], bytes));
  }
  // NVLink P2P between neighbouring devices (copies stage through the host
  // otherwise; same-device slabs copy on the device)
  for (int g = 0; g + 1 < n; ++g) {
    const int a = sl[g].dev, b = sl[g + 1].dev;
    if (a == b) continue;
    for (auto [x, y] : {std::pair<int, int>{a, b}, {b, a}}) {
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, x, y) == cudaSuccess && ok) {
        cudaSetDevice(x);
        const cudaError_t pe2 = cudaDeviceEnablePeerAccess(y, 0);
        if (pe2 != cudaSuccess && pe2 != cudaErrorPeerAccessAlreadyEnabled) {
          e = pe2;
          cleanup();
          return e;
        }
        cudaGetLastError();
      }
    }
  }
  // load: every local plane (ghosts included) into buf[0], then buf[1] = buf[0]
  // so both carry the ring
  for (auto& s : sl) {
    SSAM_TRY(cudaSetDevice(s.dev));
    const size_t bytes = static_cast<size_t>(s.nl) * pe * sizeof(T);
    SSAM_TRY(cudaMemcpyAsync(s.buf[0], h_in + static_cast<size_t>(s.z0 - s.glo) * pe, bytes,
                             cudaMemcpyHostToDevice, s.cs));
    SSAM_TRY(cudaMemcpyAsync(s.buf[1], s.buf[0], bytes, cudaMemcpyDeviceToDevice, s.cs));
  }
  // Every slab's buffers are initialised before any neighbour's halo copy
  // (on that neighbour's copy stream) may write into their ghost planes.
  for (auto& s : sl) {
    SSAM_TRY(cudaSetDevice(s.dev));
    SSAM_TRY(cudaStreamSynchronize(s.cs));
  }

  // Is a fused launch of this depth compiled for the stencil / dtype /
  // alignment?  (An empty output range validates without launching.)
  auto fused_ok = [&](int depth) {
    if (depth < 2) return false;
    cudaSetDevice(sl[0].dev);
    const T* a = sl[0].buf[0];
    T* b = sl[0].buf[1];
    const cudaError_t pr =
        dims == 3 ? stencil3d_tb<T>(a, b, nx, ny, sl[0].nl, 0, 0, 0, sl[0].nl, st, depth, sl[0].cs)
                  : stencil2d_tb_range<T>(a, b, nx, sl[0].nl, 0, 0, 0, sl[0].nl, st, depth, sl[0].cs);
    cudaGetLastError();
    return pr == cudaSuccess;
  };

  int cur = 0, done = 0;
  bool first = true;
  while (done < iters) {
    // full-depth fused rounds, the remainder fused where a kernel of that
    // depth exists, else single sweeps (fused == single sweeps bit for bit)
    int depth = std::min(tb, iters - done);
    if (!fused_ok(depth)) depth = 1;
    // phase A: compute
    for (int g = 0; g < n; ++g) {
      Slab<T>& s = sl[g];
      SSAM_TRY(cudaSetDevice(s.dev));
      if (!first) {
        SSAM_TRY(cudaStreamWaitEvent(s.cs, s.cp, 0));
        if (g > 0) SSAM_TRY(cudaStreamWaitEvent(s.cs, sl[g - 1].cp, 0));
        if (g + 1 < n) SSAM_TRY(cudaStreamWaitEvent(s.cs, sl[g + 1].cp, 0));
      }
      const int zoff = s.z0 - s.glo;  // global plane of local plane 0
      const int rlo = k - zoff, rhi = nplanes - k - zoff;
      const int ob = s.glo, oe = s.glo + s.owned();  // owned local planes
      const T* in = s.buf[cur];
      T* out = s.buf[cur ^ 1];
      // boundary bands first (only faces shared with a neighbour), then the interior
      const int lo_e = s.glo > 0 ? std::min(oe, ob + G) : ob;
      const int hi_b = s.ghi > 0 ? std::max(lo_e, oe - G) : oe;
      SSAM_TRY(launch_band<T>(dims, in, out, nx, ny, s.nl, ob, lo_e, rlo, rhi, st, depth, s.cs));
      SSAM_TRY(launch_band<T>(dims, in, out, nx, ny, s.nl, hi_b, oe, rlo, rhi, st, depth, s.cs));
      SSAM_TRY(cudaEventRecord(s.bnd, s.cs));
      SSAM_TRY(launch_band<T>(dims, in, out, nx, ny, s.nl, lo_e, hi_b, rlo, rhi, st, depth, s.cs));
    }
    // phase B: halo copies into the neighbours' next-round input buffer
    for (int g = 0; g < n; ++g) {
      Slab<T>& s = sl[g];
      SSAM_TRY(cudaSetDevice(s.dev));
      SSAM_TRY(cudaStreamWaitEvent(s.xs, s.bnd, 0));
      const size_t band = static_cast<size_t>(G) * pe * sizeof(T);
      if (g > 0) {  // my lowest G owned planes -> the lower neighbour's upper ghosts
        Slab<T>& d = sl[g - 1];
        SSAM_TRY(cudaMemcpyPeerAsync(d.buf[cur ^ 1] + static_cast<size_t>(d.glo + d.owned()) * pe,
                                     d.dev, s.buf[cur ^ 1] + static_cast<size_t>(s.glo) * pe,
                                     s.dev, band, s.xs));
      }
      if (g + 1 < n) {  // my highest G owned planes -> the upper neighbour's lower ghosts
        Slab<T>& d = sl[g + 1];
        SSAM_TRY(cudaMemcpyPeerAsync(d.buf[cur ^ 1], d.dev,
                                     s.buf[cur ^ 1] + static_cast<size_t>(s.glo + s.owned() - G) * pe,
                                     s.dev, band, s.xs));
      }
      SSAM_TRY(cudaEventRecord(s.cp, s.xs));
    }
    cur ^= 1;
    done += depth;
    first = false;
  }
  // store the owned planes
  for (auto& s : sl) {
    SSAM_TRY(cudaSetDevice(s.dev));
    SSAM_TRY(cudaStreamWaitEvent(s.cs, s.cp, 0));
    SSAM_TRY(cudaMemcpyAsync(h_out + static_cast<size_t>(s.z0) * pe,
                             s.buf[cur] + static_cast<size_t>(s.glo) * pe,
                             static_cast<size_t>(s.owned()) * pe * sizeof(T),
                             cudaMemcpyDeviceToHost, s.cs));
  }
  for (auto& s : sl) {
    SSAM_TRY(cudaSetDevice(s.dev));
    SSAM_TRY(cudaStreamSynchronize(s.cs));
    SSAM_TRY(cudaStreamSynchronize(s.xs));
  }
#undef SSAM_TRY
  cleanup();
  return cudaSuccess;
}

template cudaError_t multi_stencil<float>(const float*, float*, int, int, int,
                                          const StencilDesc<float>&, int, int, const int*, int,
                                          int*);
template cudaError_t multi_stencil<double>(const double*, double*, int, int, int,
                                           const StencilDesc<double>&, int, int, const int*, int,
                                           int*);
template cudaError_t multi_stencil<long long>(const long long*, long long*, int, int, int,
                                              const StencilDesc<long long>&, int, int, const int*,
                                              int, int*);

}  // namespace ssam_b200
