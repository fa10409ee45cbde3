// tb2d.cu -- temporal blocking for 2D stencils: TB Jacobi sweeps per pass.
//
// The reference has no temporal blocking; its semantics are
// pinned only as "TB fused steps == TB sweeps of oracle::stencil2d_naive"
// (oracle.hpp:80-96).  Here one warp streams down its strip exactly as in
// the single-sweep engine, but carries a PIPELINE of TB stages in registers:
//
//     input row r  ->  stage 1 window (rows r-2k..r)  ->  gen-1 row r-k
//                  ->  stage 2 window                 ->  gen-2 row r-2k ...
//                  ->  stage TB                       ->  gen-TB row r-TB*k  (stored)
//
// Each stage is the SSAM row computation (bidirectional shuffle chain, taps
// as constant operands).  Only the input row is read and only the last
// generation is written, so HBM traffic per cell-update drops TB-fold.
// Every stage shrinks the valid x-range by k columns per side (overlapped /
// trapezoidal tiling in x); in y there is no redundancy except the 2*TB*k
// rows at each segment's ends.  Ring cells (width k, every generation equal
// to the input) pass through: a stage's output at a ring cell is the centre
// value of its own input window, which sits in the same lane.
#include <algorithm>
#include <cstring>
#include <type_traits>
#include <vector>

#include "launch.cuh"

namespace ssam_b200 {

template <class T, int CAP>
struct alignas(64) Tb2DParams {
  CUtensorMap tmap;  // (W, H), box 32Q x RB
  const T* in;
  T* out;
  int W, H;
  int A, V, nstrips, seg, y_begin, y_end;
  int ring;          // x ring (k)
  int yr_lo, yr_hi;  // rows outside [yr_lo, yr_hi) are the global ring (a row slab passes
                     // its local bounds, which may lie outside the buffer)
  T coef[CAP];
};

// One stage's output row from its NR-row window: the single-sweep engines'
// star chain (engine2d.cuh star_row_chain), so Tb fused sweeps are
// bit-identical to Tb single sweeps.  Window row t lives in register slot
// (rot + t) % NR (rotation by index, `rot` folds to a constant after
// unrolling).
template <class T, int Q, int K, class Mask, int CAP>
__device__ __forceinline__ void tb_stage_row(const T (&w)[2 * K + 1][Q], int rot,
                                             const Tb2DParams<T, CAP>& p, T (&acc)[Q]) {
  static_assert(IsStar2D<Mask>::value, "temporal blocking is compiled for star stencils");
  constexpr int NR = 2 * K + 1;
  star_row_chain<T, Q, K, NR>(w, rot, [&](int j, int t) { return p.coef[j * NR + t]; }, acc);
}

template <class T, int Q, int K, class Mask, int TB, int RB, int D, int CAP>
__global__ void __launch_bounds__(128) tb2d_kernel(const __grid_constant__ Tb2DParams<T, CAP> p) {
  constexpr int NR = 2 * K + 1;
  constexpr int ROW = 32 * Q;
  constexpr uint32_t BOX_BYTES = RB * ROW * sizeof(T);
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int strip = blockIdx.x * (blockDim.x >> 5) + wib;
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * p.V;
  const int base = x_out0 - p.A;
  const int x0 = base + Q * lane;
  const bool own = x0 >= x_out0 && x0 < x_out0 + p.V;
  const int xlo = p.ring, xhi = p.W - p.ring;
  const bool whole = x0 >= xlo && x0 + Q <= xhi;
  // Does any stage row of this warp fall on the ring (columns of the window,
  // or rows y0 - TB*K .. y1 + TB*K)?  Warp-uniform.
  const bool edge = base < xlo || base + 32 * Q > xhi || y0 - TB * K < p.yr_lo ||
                    y1 + TB * K > p.yr_hi;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * D * RB * ROW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
                       smem_raw + static_cast<size_t>(blockDim.x >> 5) * D * BOX_BYTES) +
                   wib * D;
  if (lane == 0) {
    prefetch_tmap(&p.tmap);
#pragma unroll
    for (int s = 0; s < D; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains
  const int yin0 = y0 - TB * K;                // first input row of the stream
  const int count = (y1 - y0) + 2 * TB * K;    // input rows yin0 .. y1-1+TB*K
  const int nbox = (count + RB - 1) / RB;
  auto issue = [&](int j) {
    const int s = j % D;
    const uint32_t bar = smem_u32(&bars[s]);
    mbar_arrive_expect_tx(bar, BOX_BYTES);
    tma_load_2d(smem_u32(ring + s * RB * ROW), &p.tmap, base, yin0 + j * RB, bar);
  };
  if (lane == 0)
    for (int j = 0; j < min(D, nbox); ++j) issue(j);

  // Per stage: the NR rows of its input generation; window row t <-> dy = t-K.
  T win[TB][NR][Q];
  for (int j = 0; j < nbox; ++j) {
    const int s = j % D;
    mbar_wait(smem_u32(&bars[s]), (j / D) & 1);
    const T* slot = ring + s * RB * ROW + Q * lane;
    // RB == NR: stream row i lands in register slot i % NR = rr of every
    // stage's window, and window row t is slot (rr + 1 + t) % NR -- the
    // windows rotate by renaming, one fully unrolled box per loop trip.
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      const int i = j * RB + rr;
      if (i >= count) break;
      const int r = yin0 + i;  // input row entering stage 1
      T in_row[Q];
      lds_q<T, Q>(slot + rr * ROW, in_row);
#pragma unroll
      for (int st = 0; st < TB; ++st) {
        // push the stage input row, then compute gen-(st+1) row r - (st+1)K
#pragma unroll
        for (int q = 0; q < Q; ++q) win[st][rr][q] = in_row[q];
        const int y = r - (st + 1) * K;
        T acc[Q];
        tb_stage_row<T, Q, K, Mask, CAP>(win[st], rr + 1, p, acc);
        // ring cells keep their (generation-invariant) value; only warps
        // whose window touches the ring pay for the selects
        if (edge) {
          const bool row_ring = y < p.yr_lo || y >= p.yr_hi;
          const int c = (rr + 1 + K) % NR;  // centre row slot
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int x = x0 + q;
            if (row_ring || x < xlo || x >= xhi) acc[q] = win[st][c][q];
          }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) in_row[q] = acc[q];
      }
      // in_row now holds generation TB of row r - TB*K
      const int y = r - TB * K;
      if (own && y >= y0 && y < y1 && y >= p.yr_lo && y < p.yr_hi) {
        T* row = p.out + static_cast<size_t>(y) * p.W + x0;
        if (whole) {
          st_q<T, Q>(row, in_row);
        } else {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (x0 + q >= xlo && x0 + q < xhi) row[q] = in_row[q];
        }
      }
    }
    // ring hand-back (PTX memory model): every lane orders its reads of the
    // slot before later async-proxy writes (fence.proxy.async), the warp
    // barrier orders all lanes before lane 0, which then refills the slot
    ring_release_warp();
    if (lane == 0 && j + D < nbox) issue(j + D);
  }
}

namespace {

template <class T>
std::vector<T> dense_coef(const StencilDesc<T>& st) {
  const int k = st.order, M = 2 * k + 1;
  std::vector<T> c(static_cast<size_t>(M) * M, T(0));
  for (size_t i = 0; i < st.taps.size(); ++i)
    c[static_cast<size_t>(st.taps[i].dx + k) * M + (st.taps[i].dy + k)] = st.coeffs[i];
  return c;
}

template <class T, int Q, int K, class Mask, int TB>
cudaError_t launch_tb(const T* in, T* out, int W, int H, int yb, int ye, int rlo, int rhi,
                      const StencilDesc<T>& st, cudaStream_t s) {
  constexpr int NR = 2 * K + 1;
  constexpr int RB = NR;                 // whole-window boxes (rotation by renaming)
  constexpr int D = (12 + RB - 1) / RB;  // ~12 rows in flight per warp
  constexpr int CAP = NR * NR;
  Tb2DParams<T, CAP> p;
  std::memset(&p, 0, sizeof(p));
  p.in = in;
  p.out = out;
  p.W = W;
  p.H = H;
  const LanePlan lp = plan_lanes(2 * TB * K + 1, Q);  // TB stages of halo
  p.A = lp.A;
  p.V = lp.V;
  if (p.V <= 0) return cudaErrorNotSupported;
  p.nstrips = (W + lp.V - 1) / lp.V;
  p.ring = K;
  p.yr_lo = rlo;
  p.yr_hi = rhi;
  p.y_begin = std::max(std::max(yb, rlo), 0);
  p.y_end = std::min(std::min(ye, rhi), H);
  const int rows = p.y_end - p.y_begin;
  if (rows <= 0 || W - 2 * K <= 0) return cudaSuccess;
  p.seg = std::max(pick_seg(rows, p.nstrips, NR), std::min(rows, 16 * TB * K));
  const std::vector<T> c = dense_coef(st);
  std::memcpy(p.coef, c.data(), sizeof(T) * CAP);
  cudaError_t e = make_tmap_2d(&p.tmap, in, sizeof(T), W, H, sizeof(T) * W, 32 * Q, RB);
  if (e != cudaSuccess) return e;
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * D * (RB * 32 * Q * sizeof(T) + 8);
  const dim3 grid((p.nstrips + kWarpsPerBlock - 1) / kWarpsPerBlock, (rows + p.seg - 1) / p.seg);
  e = launch_pdl(tb2d_kernel<T, Q, K, Mask, TB, RB, D, CAP>, grid, dim3(32 * kWarpsPerBlock), smem,
                 s, p);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

// Fused depths compiled per (dtype, star order); the memory-bound star
// stencils gain from TB, the compute-heavy ones (k >= 3) do not.
template <class T, int K>
cudaError_t tb_dispatch(const T* in, T* out, int W, int H, int yb, int ye, int rlo, int rhi,
                        const StencilDesc<T>& st, int tb, cudaStream_t s) {
  constexpr int Q = 16 / sizeof(T);
  switch (tb) {
    case 2: return launch_tb<T, Q, K, StarMask2D<K>, 2>(in, out, W, H, yb, ye, rlo, rhi, st, s);
    case 4: return launch_tb<T, Q, K, StarMask2D<K>, 4>(in, out, W, H, yb, ye, rlo, rhi, st, s);
    case 8:
      if constexpr (K == 1)
        return launch_tb<T, Q, K, StarMask2D<K>, 8>(in, out, W, H, yb, ye, rlo, rhi, st, s);
      return cudaErrorNotSupported;
  }
  return cudaErrorNotSupported;
}

}  // namespace

template <class T>
cudaError_t stencil2d_tb_range(const T* in, T* out, int W, int H, int y_begin, int y_end,
                               int yr_lo, int yr_hi, const StencilDesc<T>& st, int tb,
                               cudaStream_t s) {
  if constexpr (std::is_same<T, long long>::value) {
    return cudaErrorNotSupported;
  } else {
    constexpr int VQ = 16 / sizeof(T);
    if (W % VQ != 0 || (reinterpret_cast<std::uintptr_t>(in) & 15u) ||
        (reinterpret_cast<std::uintptr_t>(out) & 15u))
      return cudaErrorNotSupported;
    if (classify2d(st.taps, st.order) != Shape2D::star) return cudaErrorNotSupported;
    switch (st.order) {
      case 1: return tb_dispatch<T, 1>(in, out, W, H, y_begin, y_end, yr_lo, yr_hi, st, tb, s);
      case 2: return tb_dispatch<T, 2>(in, out, W, H, y_begin, y_end, yr_lo, yr_hi, st, tb, s);
    }
    return cudaErrorNotSupported;
  }
}

template <class T>
cudaError_t stencil2d_tb(const T* in, T* out, int W, int H, const StencilDesc<T>& st, int tb,
                         cudaStream_t s) {
  return stencil2d_tb_range<T>(in, out, W, H, st.order, H - st.order, st.order, H - st.order,
                               st, tb, s);
}

template cudaError_t stencil2d_tb<float>(const float*, float*, int, int, const StencilDesc<float>&,
                                         int, cudaStream_t);
template cudaError_t stencil2d_tb_range<float>(const float*, float*, int, int, int, int, int, int,
                                               const StencilDesc<float>&, int, cudaStream_t);
template cudaError_t stencil2d_tb_range<double>(const double*, double*, int, int, int, int, int,
                                                int, const StencilDesc<double>&, int,
                                                cudaStream_t);
template cudaError_t stencil2d_tb_range<long long>(const long long*, long long*, int, int, int,
                                                   int, int, int, const StencilDesc<long long>&,
                                                   int, cudaStream_t);
template cudaError_t stencil2d_tb<double>(const double*, double*, int, int,
                                          const StencilDesc<double>&, int, cudaStream_t);
template cudaError_t stencil2d_tb<long long>(const long long*, long long*, int, int,
                                             const StencilDesc<long long>&, int, cudaStream_t);

// Deepest fused depth for automatic scheduling (1 = none).
int stencil2d_tb_max(int dtype, int order, bool star) {
  if (dtype == 2 || !star) return 1;
  // Measured x100 on 8192^2 (GCells/s, Tb = 1/2/4/8; single FMA chain, ring
  // selects only in edge warps): 2d5pt f32 676/767/1768/1582, f64
  // 351/441/933/654; 2d9pt f32 675/1166/1009/-, f64 355/590/486/-.
  if (order == 1) return 4;  // TB=8 is compiled but slower (register pressure)
  if (order == 2) return 2;
  return 1;
}

}  // namespace ssam_b200
