// engine2d_conv.cuh -- the register-row engine: conv2d with square filters
// K = 5..15 and the 2D stencils of order 4..6 (with their tap mask), sm_100a.
//
// Reference: ssam::conv2d (proj/include/ssam/kernels.hpp:189-225), the true
// convolution out(x,y) = sum_{s,t} in(x+ax-s, y+ay-t) * w[s*n+t]
// (oracle.hpp:40-56), written as the correlation
//     out(x, y) = sum_{j,t} coef[j*K+t] * in(x + j - L, y + t - U)
// with coef[j][t] = w[(K-1-j)*K + (K-1-t)] (conv_coef, kernels.hpp:90).
//
// Why not the shuffle chain here: from K ~ 6 the conv is FMA-bound (2K^2
// flop per output), and in the systolic chain every
// column step costs a SHFL plus Q-1 register moves per output vector, the
// chain's first/last lanes hold no valid output, and the window shift adds
// more moves -- ncu on the chain engine: 74-81% of issued instructions are
// FFMA, FMA pipe 62-71% busy (profiles/r02/ncu_conv_*_v1.txt).  B200's
// shared memory has bandwidth to spare at this arithmetic intensity, so each
// lane instead reads its Q + K - 1 input columns of a row straight from the
// TMA-staged box (three 16-byte LDS for fp32 Q = 4) and keeps the register
// cache for the ROWS: per pass of RY output rows it streams the RY + K - 1
// input rows once, and every input row feeds K x Q FFMAs into each of the
// (up to K) output rows it belongs to -- ~96% of the issued instructions
// are FFMAs with the weights as constant-bank operands, every lane's Q
// columns are outputs, and no shuffles are needed.
//
// Per output the sum is ONE FMA chain, rows t outer, columns j inner (a
// fixed order, so results are deterministic; fp32 within 1e-5 of the
// double-accumulated oracle); from 12x12 each input row's K taps are summed
// first and the row partials added (two-level, SURVEY §8(c) caveat 1).
#pragma once

#include <type_traits>

#include "launch.cuh"

#ifndef SSAM_CONVREG_TWO_MIN
#define SSAM_CONVREG_TWO_MIN 12
#endif

namespace ssam_b200 {

template <class T, int K, int Q>
struct ConvRegGeom {
  static constexpr int V = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte chunk
  static constexpr int R = (K - 1) / 2, L = K - 1 - R;         // columns right / left of an output
  static constexpr int HL = (L + V - 1) / V * V;               // box pad left (whole chunks)
  static constexpr int HR = (R + V - 1) / V * V;               // box pad right
  // a TMA box is at most 256 elements wide: a warp strip of 32 Q columns
  // is staged as NSUB overlapping sub-boxes, each serving SUBL lanes
  static constexpr int NSUB = (HL + 32 * Q + HR) <= 256 ? 1 : 2;
  static constexpr int SUBL = 32 / NSUB;
  static constexpr int BW = HL + SUBL * Q + HR;                // sub-box / smem row width
  static constexpr int OFF = HL - L;                           // lane's first column in its chunks
  static constexpr int NC = (OFF + Q + K - 1 + V - 1) / V;     // chunks a lane reads per row
  // one sub-box of RB rows, padded to TMA's 128-byte destination alignment;
  // a ring slot holds NSUB of them
  template <int RB>
  static constexpr int sub_elems() {
    return static_cast<int>((RB * BW * sizeof(T) + 127) / 128 * 128 / sizeof(T));
  }
  template <int RB>
  static constexpr int slot_elems() { return NSUB * sub_elems<RB>(); }
  static_assert(BW <= 256, "TMA box width");
  static_assert(Q % V == 0, "whole chunks per lane");
};

template <class T, int CAP>
struct alignas(64) ConvRegParams {
  CUtensorMap tmap;  // (W, H), box BW x RB
  T* out;
  int W, H;
  int nstrips, seg, y_begin, y_end;
  int xlo, xhi;  // written columns (stencils: the interior [k, W-k))
  T coef[CAP];   // coef[j*K + t]
};

// Does input row i of a pass (RY output rows, K-row footprint) need chunk c
// of the lane's columns?  (A chunk is read only if some tap of the mask
// lands in it -- a star's off-centre rows need just the lane's own columns.)
template <class Mask, int K, int Q, int RY, int OFF, int V>
__host__ __device__ constexpr bool row_needs_chunk(int i, int c) {
  for (int r = 0; r < RY; ++r) {
    const int t = i - r;
    if (t < 0 || t >= K) continue;
    for (int j = 0; j < K; ++j) {
      if (!Mask::has(j, t)) continue;
      for (int q = 0; q < Q; ++q) {
        const int col = OFF + q + j;
        if (col >= c * V && col < c * V + V) return true;
      }
    }
  }
  return false;
}

template <class T, int K, int Q, int RY, int RB, int D, int CAP, class Mask = DenseMask>
__global__ void __launch_bounds__(128)
    conv2d_reg_kernel(const __grid_constant__ ConvRegParams<T, CAP> p) {
  using G = ConvRegGeom<T, K, Q>;
  constexpr int V = G::V, BW = G::BW, NC = G::NC, OFF = G::OFF;
  constexpr int U = K - 1 - (K - 1) / 2;  // rows above an output
  constexpr int NIN = RY + K - 1;         // input rows per pass
  constexpr uint32_t BOX_BYTES = RB * BW * sizeof(T);
  constexpr int SLOT = G::template slot_elems<RB>();
  static_assert(RB == RY, "pass p starts at the first row of box p");
  // large filters sum each input row's K taps first, then add the row
  // partials -- the paper's two-level order transposed,
  // which is what keeps fp32 within 1e-5 at 17x17 .. 20x20
  constexpr bool TWO = K >= SSAM_CONVREG_TWO_MIN && std::is_same<Mask, DenseMask>::value;
  constexpr int NB = (NIN - 1) / RB + 1;  // boxes a pass reads
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int strip = blockIdx.x * (blockDim.x >> 5) + wib;
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * 32 * Q;
  const int xb = x_out0 - G::HL;  // box origin (16-byte aligned)
  const int x0 = x_out0 + Q * lane;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * D * SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
                       smem_raw + static_cast<size_t>(blockDim.x >> 5) * D * SLOT * sizeof(T)) +
                   wib * D;
  if (lane == 0) {
    prefetch_tmap(&p.tmap);
#pragma unroll
    for (int s = 0; s < D; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  griddep_launch();
  // stream row i = image row y0 - U + i; pass p reads rows p*RY .. p*RY + NIN - 1
  const int npass = (y1 - y0 + RY - 1) / RY;
  const int nrows = npass * RY + K - 1;
  const int nbox = (nrows + RB - 1) / RB;
  auto issue = [&](int b) {
    const int s = b % D;
    const uint32_t bar = smem_u32(&bars[s]);
    mbar_arrive_expect_tx(bar, BOX_BYTES * G::NSUB);
#pragma unroll
    for (int k = 0; k < G::NSUB; ++k)
      tma_load_2d(smem_u32(ring + s * SLOT + k * G::template sub_elems<RB>()), &p.tmap,
                  xb + k * G::SUBL * Q, y0 - U + b * RB, bar);
  };
  if (lane == 0)
    for (int b = 0; b < min(D, nbox); ++b) issue(b);
  int ready = 0;  // boxes waited for
  // a lane's chunks start at column Q * (lane % SUBL) of its sub-box
  const T* lane_base =
      ring + (lane / G::SUBL) * G::template sub_elems<RB>() + Q * (lane % G::SUBL);
  int cslot = 0;                         // ring slot of box `pass`

  for (int pass = 0; pass < npass; ++pass) {
    const int s0 = pass * RY;
    // every box holding rows s0 .. s0 + NIN - 1 has landed
    const int need = min(nbox, (s0 + NIN - 1) / RB + 1);
    while (ready < need) {
      mbar_wait(smem_u32(&bars[ready % D]), (ready / D) & 1);
      ++ready;
    }
    T acc[RY][Q];
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) acc[r][q] = T(0);
    const T* bp[NB];
    {
      int sl = cslot;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        bp[k] = lane_base + sl * SLOT;
        sl = sl + 1 == D ? 0 : sl + 1;
      }
    }
#pragma unroll
    for (int i = 0; i < NIN; ++i) {
      const T* rowp = bp[i / RB] + (i % RB) * BW;
      T x[NC * V];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (!row_needs_chunk<Mask, K, Q, RY, OFF, V>(i, c)) continue;
        const int4 w = *reinterpret_cast<const int4*>(rowp + c * V);
        memcpy(&x[c * V], &w, 16);
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int t = i - r;  // filter row of input row i for output row r
        if (t < 0 || t >= K) continue;
        if constexpr (TWO) {
          // two-level: the row's K-tap partial, then one add into the output
          static_assert(std::is_same<Mask, DenseMask>::value, "two-level order: dense filters");
          T rp[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) rp[q] = p.coef[t] * x[OFF + q];
#pragma unroll
          for (int j = 1; j < K; ++j) {
            const T c = p.coef[j * K + t];
#pragma unroll
            for (int q = 0; q < Q; ++q) rp[q] = fma_t(c, x[OFF + q + j], rp[q]);
          }
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[r][q] += rp[q];
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j) {
            if (!Mask::has(j, t)) continue;
            const T c = p.coef[j * K + t];
#pragma unroll
            for (int q = 0; q < Q; ++q) acc[r][q] = fma_t(c, x[OFF + q + j], acc[r][q]);
          }
        }
      }
    }
    const int y = y0 + s0;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (y + r >= y1) break;
      T* o = p.out + static_cast<size_t>(y + r) * p.W + x0;
      if (x0 >= p.xlo && x0 + Q <= p.xhi) {
        st_q<T, Q>(o, acc[r]);
      } else {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (x0 + q >= p.xlo && x0 + q < p.xhi) o[q] = acc[r][q];
      }
    }
    // box `pass` lies wholly above the next pass's first row: hand it back
    ring_release_warp();
    if (lane == 0 && pass + D < nbox) issue(pass + D);
    cslot = cslot + 1 == D ? 0 : cslot + 1;
  }
}

template <class Mask, int K>
constexpr int mask_tap_count() {
  int n = 0;
  for (int j = 0; j < K; ++j)
    for (int t = 0; t < K; ++t) n += Mask::has(j, t) ? 1 : 0;
  return n;
}

template <class T, int K, class Mask = DenseMask>
struct ConvRegCfg {
#ifndef SSAM_CONVREG_Q32
#define SSAM_CONVREG_Q32 4
#endif
#ifndef SSAM_CONVREG_Q64
#define SSAM_CONVREG_Q64 2
#endif
  static constexpr int Q = sizeof(T) == 4 ? SSAM_CONVREG_Q32 : SSAM_CONVREG_Q64;
#ifndef SSAM_CONVREG_RY
#define SSAM_CONVREG_RY 4
#endif
#ifndef SSAM_CONVREG_RY_BIG
#define SSAM_CONVREG_RY_BIG 2
#endif
#ifndef SSAM_CONVREG_RY_STAR
#define SSAM_CONVREG_RY_STAR 6
#endif
  // star stencils: 6 rows per pass (2ds25pt f32 609 -> 652 GCells/s, 2d21pt
  // / 2d17pt +3%; dense filters keep 4 -- profiles/r02/st2d_ry_ab.txt)
  static constexpr int RY = IsStar2D<Mask>::value ? SSAM_CONVREG_RY_STAR
                          : mask_tap_count<Mask, K>() <= 121 ? SSAM_CONVREG_RY : SSAM_CONVREG_RY_BIG;
  static constexpr int RB = RY;
  // rows kept for the window (K - 1) + one pass in flight + prefetch
  static constexpr int D = (K - 1 + RB - 1) / RB + 3;
};

// conv2d (Mask = DenseMask, every column written) and 2D stencils (a tap
// mask, only the interior [ring, W - ring) written; rows are clamped by the
// caller).
template <class T, int K, class Mask = DenseMask>
cudaError_t launch_conv2d_reg(const T* in, T* out, int W, int H, int y_begin, int y_end,
                              const T* coef, cudaStream_t s, int ring = 0) {
  using C = ConvRegCfg<T, K, Mask>;
  using G = ConvRegGeom<T, K, C::Q>;
  constexpr int CAP = K * K;
  if (W % G::V != 0 || !aligned16(in) || !aligned16(out)) return cudaErrorNotSupported;
  if (y_end <= y_begin) return cudaSuccess;
  ConvRegParams<T, CAP> p;
  std::memset(&p, 0, sizeof(p));
  p.out = out;
  p.W = W;
  p.H = H;
  p.nstrips = (W + 32 * C::Q - 1) / (32 * C::Q);
  const int rows = y_end - y_begin;
  p.seg = (pick_seg(rows, p.nstrips, K) + C::RY - 1) / C::RY * C::RY;
  p.y_begin = y_begin;
  p.y_end = y_end;
  p.xlo = ring;
  p.xhi = W - ring;
  std::memcpy(p.coef, coef, sizeof(T) * CAP);
  cudaError_t e = make_tmap_2d(&p.tmap, in, sizeof(T), W, H, sizeof(T) * W, G::BW, C::RB);
  if (e != cudaSuccess) return e;
  auto kern = conv2d_reg_kernel<T, K, C::Q, C::RY, C::RB, C::D, CAP, Mask>;
  const size_t smem =
      static_cast<size_t>(kWarpsPerBlock) * C::D * (G::template slot_elems<C::RB>() * sizeof(T) + 8);
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid((p.nstrips + kWarpsPerBlock - 1) / kWarpsPerBlock, (rows + p.seg - 1) / p.seg);
  e = launch_pdl(kern, grid, dim3(32 * kWarpsPerBlock), smem, s, p);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

}  // namespace ssam_b200
