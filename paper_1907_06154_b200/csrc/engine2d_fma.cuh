// engine2d_fma.cuh -- the FMA-bound 2D SSAM engine (dense conv2d, K >= 5).
//
// Same systolic model as engine2d.cuh (one warp = one 32 x Q column strip
// streaming down the rows, the window rows in registers, partial sums moved
// lane to lane by the bidirectional shuffle chain, two-level accumulation of
// PAPER.md:491-497), re-shaped for filters whose arithmetic, not HBM, bounds
// the kernel (2K^2 flop per 8 bytes: K >= 6 on B200).  What changes:
//
//  * RY output rows per pass.  The window holds NR+RY-1 rows; each pass
//    takes RY new rows and emits RY rows: RY*Q independent FMA chains, and
//    the window shift costs (NR-1)*Q moves per RY rows instead of per row.
//  * The unrolled body is ONE pass, never the 2*NR-row ping-pong body of the
//    light kernel (for 7x7 that body is ~56 KB of SASS, and ncu showed the
//    light kernel stalled on instruction fetch).
//  * Exact lane plan (EXACT): lane 0 starts at x_out0 - L, unaligned, so each
//    warp emits 32Q - (M-1) columns instead of the 16-byte-rounded plan
//    (104 -> 109 of 128 at 20x20).  TMA box origins must be 16-byte aligned,
//    so the box starts at the aligned column below and is Q columns wider;
//    lanes read their Q columns at the misalignment d (LDS.128 / 2x LDS.64 /
//    Q x LDS.32) and store them as predicated scalars.
//  * Boxes are aligned to passes: the stream is padded by OFF rows in front
//    so that every pass's rows sit in one box (one mbarrier test per pass,
//    no per-row bookkeeping).
//  * Compile-time widths unroll the column loop with the weights as
//    constant-bank operands; run-time widths (MC = 0) loop over columns with
//    each column's NR weights broadcast from shared memory.
//
// Stencils use it too (compile-time tap masks, interior-only stores): the
// tall star footprints (2ds25pt) otherwise spend a quarter of their issue
// slots on the light kernel's one-row window shifts.
//
// Arithmetic per output is that of the light kernel's compile-time path
// (engine2d.cuh ssam_row_ct): colpart_j is the serial FMA chain over the
// column's taps in t order starting with a multiply; acc = colpart_0, then
// acc = shift_up(acc) + colpart_j; accr likewise from the right; then
// acc += shift_down(accr).  Results are bit-identical to that kernel.
//
// Rows arrive as RB-row TMA boxes (zero fill = zero boundary) in a per-warp
// ring of D slots.  A box is handed back once its rows have fed a pass's
// FFMAs (so its LDS have returned); in the prologue, where the window is
// taller than the ring, as soon as its rows were read (common.cuh
// ring_release_warp before lane 0 refills the slot).
#pragma once

#include "engine2d.cuh"

namespace ssam_b200 {

// Front padding of the row stream so that pass boundaries fall on box
// boundaries: (OFF + NR - 1) % RB == 0.
__host__ __device__ constexpr int fma2d_off(int nr, int rb) { return (rb - (nr - 1) % rb) % rb; }

template <bool EXACT, int Q>
__host__ __device__ constexpr int fma2d_pitch() { return 32 * Q + (EXACT ? Q : 0); }

// One ring slot: RB rows of the box, padded to TMA's 128-byte destination alignment.
template <class T, int Q, int RB, bool EXACT>
__host__ __device__ constexpr size_t fma2d_slot_bytes() {
  return (static_cast<size_t>(RB) * fma2d_pitch<EXACT, Q>() * sizeof(T) + 127) / 128 * 128;
}

template <class T, int Q, int NR, int RB, int D, bool EXACT>
__host__ __device__ constexpr size_t fma2d_smem(int warps, int m) {
  return 128 +  // guard in front of the ring (STARX reads up to K' columns left of a row)
         static_cast<size_t>(warps) * (D * (fma2d_slot_bytes<T, Q, RB, EXACT>() + 8)) +
         static_cast<size_t>(warps) * 128 +
         static_cast<size_t>(m) * ((NR * sizeof(T) + 15) / 16 * 16);
}

// Star footprints (StarMask2D<K>) on the single-chain path take their K
// horizontal taps on each side straight from the centre row in shared memory
// (STARX): per output row a lane reads Q + 2K' columns (K' = K rounded up to
// 16 bytes) with vector LDS instead of running the shuffle chain (one SHFL
// and Q-1 register moves per column step).  The vertical arm stays in the
// register window.  The ring then keeps a box until the passes that use its
// rows as centre rows (K rows behind the window front) are done, so it is
// deeper (fma2d_depth).  Measured at 8192^2 (chain -> STARX, GCells/s):
// 2ds25pt (K=6) f32 407 -> 443, f64 236 -> 268; 2d21pt (K=5) f32 477 -> 487,
// f64 249 -> 270; but 2d17pt (K=4) f32 544 -> 505, f64 319 -> 296 -- so K >= 5.
template <class Mask> struct StarK2D { static constexpr int value = -1; };
template <int K> struct StarK2D<StarMask2D<K>> { static constexpr int value = K; };
#ifndef SSAM_ST2D_STARX
#define SSAM_ST2D_STARX 1
#endif
template <class Mask, bool CHAIN1, bool EXACT, int MC>
__host__ __device__ constexpr bool fma2d_starx() {
  return SSAM_ST2D_STARX && CHAIN1 && !EXACT && MC > 0 && StarK2D<Mask>::value >= 5;
}
// Ring depth: 3 boxes, or for STARX every box of the prologue and first pass plus one.
template <class Mask, bool CHAIN1, bool EXACT, int MC, int NR, int RY, int RB>
__host__ __device__ constexpr int fma2d_depth() {
  return fma2d_starx<Mask, CHAIN1, EXACT, MC>()
             ? (fma2d_off(NR, RB) + NR - 1 + RY + RB - 1) / RB + 1
             : 3;
}

template <class T, int Q, int NR, int MC, class Mask, int RY, int RB, int D, bool EXACT, int CAP,
          bool CHAIN1 = false>
__global__ void __launch_bounds__(128)
    ssam2d_fma_kernel(const __grid_constant__ Ssam2DTmaParams<T, CAP> P) {
  static_assert(RB % RY == 0, "passes never straddle boxes");
  constexpr bool UNROLL = MC > 0;
  constexpr bool STARX = fma2d_starx<Mask, CHAIN1, EXACT, MC>();
  constexpr int SK = StarK2D<Mask>::value;
  const Ssam2DParams<T, CAP>& p = P.p;
  constexpr int U = NR - 1 - (NR - 1) / 2;
  constexpr int ROW = fma2d_pitch<EXACT, Q>();  // smem row pitch = box width
  constexpr int NW = NR + RY - 1;               // window rows
  constexpr int CV = 16 / sizeof(T);            // coefficients per 16-byte chunk
  constexpr int NRP = (NR + CV - 1) / CV * CV;  // padded column of weights
  constexpr int OFF = fma2d_off(NR, RB);
  constexpr uint32_t BOX_BYTES = RB * ROW * sizeof(T);
  constexpr uint32_t SLOT_BYTES = fma2d_slot_bytes<T, Q, RB, EXACT>();
  constexpr int SLOT = SLOT_BYTES / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int M = UNROLL ? MC : p.M;

  extern __shared__ __align__(128) unsigned char smem_all[];
  unsigned char* smem_raw = smem_all + 128;
  T* ring = reinterpret_cast<T*>(smem_raw) + static_cast<size_t>(wib) * D * SLOT;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem_raw + static_cast<size_t>(nwarps) * D * SLOT_BYTES) +
      wib * D;
  T* scoef = reinterpret_cast<T*>(smem_raw +
                                  static_cast<size_t>(nwarps) * (D * (SLOT_BYTES + 8) + 128));
  if constexpr (!UNROLL) {
    // weights of column j at scoef[j*NRP .. j*NRP+NR), zero padded
    for (int idx = threadIdx.x; idx < M * NRP; idx += blockDim.x) {
      const int j = idx / NRP, t = idx - j * NRP;
      scoef[idx] = t < NR ? p.coef[j * NR + t] : T(0);
    }
    __syncthreads();
  }

  const int strip = blockIdx.x * nwarps + wib;
  if (strip >= p.nstrips) return;
  const int y0 = p.y_begin + blockIdx.y * p.seg;
  const int y1 = min(y0 + p.seg, p.y_end);
  const int x_out0 = strip * p.V;
  const int xl = x_out0 - p.A;  // lane 0's first column (any column when EXACT)
  constexpr int VQ = 16 / sizeof(T);
  const int base = EXACT ? (xl >= 0 ? xl / VQ * VQ : -((-xl + VQ - 1) / VQ) * VQ) : xl;
  const int dmis = xl - base;  // EXACT: misalignment of the lanes in the box (warp-uniform)
  const int x0 = xl + Q * lane;
  // columns of this lane that are outputs of this warp and of the image
  // (stencils: only the interior [ring, W-ring) is written; rows are clamped by the caller)
  const int xlo = max(x_out0, p.bmode == kBndStencil ? p.ring : 0);
  const int xhi = min(x_out0 + p.V, p.bmode == kBndStencil ? p.W - p.ring : p.W);
  uint32_t qmask = 0;
#pragma unroll
  for (int q = 0; q < Q; ++q) qmask |= (x0 + q >= xlo && x0 + q < xhi) ? 1u << q : 0u;
  const bool whole = qmask == (1u << Q) - 1 && dmis == 0;

  if (lane == 0) {
    prefetch_tmap(&P.tmap);
#pragma unroll
    for (int s = 0; s < D; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();    // predecessor grid done (PDL launch)
  griddep_launch();  // let the next grid fill SMs as this one drains
  const int npass = (y1 - y0 + RY - 1) / RY;
  const int nbox = (OFF + NR - 1) / RB + npass * RY / RB + ((npass * RY) % RB ? 1 : 0);
  // stream row s is image row y0 - U - OFF + s
  auto issue = [&](int b) {
    const int s = b % D;
    const uint32_t bar = smem_u32(&bars[s]);
    mbar_arrive_expect_tx(bar, BOX_BYTES);
    tma_load_2d(smem_u32(ring + s * SLOT), &P.tmap, base, y0 - U - OFF + b * RB, bar);
  };
  if (lane == 0)
    for (int b = 0; b < min(D, nbox); ++b) issue(b);
  // Ring hand-back after the warp's last read of box b (common.cuh
  // ring_release_warp): the slot is refilled with box b + D.
  auto recycle = [&](int b) {
    ring_release_warp();
    if (lane == 0 && b + D < nbox) issue(b + D);
  };
  auto row_ptr = [&](int s) -> const T* {
    const int b = s / RB;
    return ring + (b % D) * SLOT + (s - b * RB) * ROW + dmis + Q * lane;
  };
  // a lane's Q columns of a smem row (16-byte aligned unless EXACT)
  auto lds_row = [&](const T* src, T (&dst)[Q]) {
    if (!EXACT || dmis == 0) {
      lds_q<T, Q>(src, dst);
    } else if (sizeof(T) == 4 && Q % 2 == 0 && (dmis & 1) == 0) {
#pragma unroll
      for (int q = 0; q < Q; q += 2) {
        const float2 v = *reinterpret_cast<const float2*>(src + q);
        memcpy(&dst[q], &v, 8);
      }
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) dst[q] = src[q];
    }
  };
  auto wait_box = [&](int b) { mbar_wait(smem_u32(&bars[b % D]), (b / D) & 1); };

  auto load_col = [&](int j, T (&c)[NRP]) {
    if constexpr (UNROLL) {
#pragma unroll
      for (int t = 0; t < NR; ++t) c[t] = p.coef[j * NR + t];
    } else {
      const int4* src = reinterpret_cast<const int4*>(scoef + j * NRP);
#pragma unroll
      for (int v = 0; v < NRP / CV; ++v) {
        const int4 w = src[v];
        memcpy(&c[v * CV], &w, 16);
      }
    }
  };
  // Column partial of filter column j (weights c) for output row r: the
  // serial FMA chain over the column's taps (Mask), first tap a multiply.
  auto colpart = [&](const T (&win)[NW][Q], const T (&c)[NRP], int j, int r, T (&cp)[Q]) {
    bool any = false;
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      if (Mask::has(j, t)) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
          cp[q] = any ? fma_t(c[t], win[r + t][q], cp[q]) : c[t] * win[r + t][q];
        any = true;
      }
    }
    if (!any) {
#pragma unroll
      for (int q = 0; q < Q; ++q) cp[q] = T(0);
    }
    return any;
  };

  // Prologue: stream rows OFF .. OFF+NR-2 into window rows 0 .. NR-2.
  T win[NW][Q];
#pragma unroll
  for (int t = 0; t < NR - 1; ++t) {
    const int s = OFF + t;
    if (t == 0 || s % RB == 0) wait_box(s / RB);
    lds_row(row_ptr(s), win[t]);
    if (!STARX && (s + 1) % RB == 0) recycle(s / RB);  // box s/RB fully read
  }

  T* outp = p.out + static_cast<size_t>(y0) * p.W + x0;
  const size_t W = static_cast<size_t>(p.W);
  int s = OFF + NR - 1;  // first stream row of the pass (a multiple of RY; box-aligned per RB)
  int rel = 0;           // STARX: next box to hand back
  // STARX: centre row of the pass's first output row (stream row s - SK) as
  // (ring slot, row in box); a lane's reads start K' columns left of its own
  // (lanes reading across a row edge only feed columns the lane plan drops,
  // and the guard in front of the ring keeps lane 0 of slot 0 in bounds)
  int cslot = ((s - SK) / RB) % D, cw = (s - SK) % RB;
  const int hoff = Q * lane - (SK + VQ - 1) / VQ * VQ;
  for (int pass = 0; pass < npass; ++pass, s += RY) {
    if (s % RB == 0) wait_box(s / RB);
    const T* rp = row_ptr(s);
#pragma unroll
    for (int r = 0; r < RY; ++r) lds_row(rp + r * ROW, win[NR - 1 + r]);

    T acc[RY][Q];
    const int R = (M - 1) / 2, L = M - 1 - R;
    if constexpr (STARX) {
      // vertical arm: filter column SK over the register window
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[r][q] = T(0);
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        const T c = p.coef[SK * NR + t];
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[r][q] = fma_t(c, win[r + t][q], acc[r][q]);
      }
      // horizontal arm: the centre row (stream row s + r - SK) from the ring;
      // lanes whose reads are clamped at the box edge only feed columns the
      // lane plan discards
      constexpr int KP = (SK + VQ - 1) / VQ * VQ, NH = Q + 2 * KP;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const bool nxt = cw + r >= RB;  // centre row in the following box
        const T* rowp = ring + (nxt ? (cslot + 1 == D ? 0 : cslot + 1) : cslot) * SLOT +
                        (cw + r - (nxt ? RB : 0)) * ROW + hoff;
        T hx[NH];
#pragma unroll
        for (int v = 0; v < NH / VQ; ++v) {
          const int4 w = *reinterpret_cast<const int4*>(rowp + v * VQ);
          memcpy(&hx[v * VQ], &w, 16);
        }
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          if (j == SK) continue;
          const T c = p.coef[j * NR + SK];
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[r][q] = fma_t(c, hx[KP + q + j - SK], acc[r][q]);
        }
      }
    } else if constexpr (CHAIN1) {
      // Single chain (stencils): every tap FMAs straight into the shifted
      // partial sum -- the reference simulator's own stage order (one MAD per
      // tap, a shift between columns, kernels.hpp:111-159) without the
      // column-partial FMUL / FADD pair, which for 1-tap star columns doubled
      // the work.
      auto colfma = [&](const T (&c)[NRP], int j, int r, T (&a)[Q]) {
#pragma unroll
        for (int t = 0; t < NR; ++t)
          if (Mask::has(j, t)) {
#pragma unroll
            for (int q = 0; q < Q; ++q) a[q] = fma_t(c[t], win[r + t][q], a[q]);
          }
      };
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[r][q] = T(0);
#pragma unroll(UNROLL ? 20 : 1)
      for (int j = 0; j <= L; ++j) {
        T c[NRP];
        load_col(j, c);
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          if (j > 0) shift_up1<T, Q>(acc[r]);
          colfma(c, j, r, acc[r]);
        }
      }
      if (R > 0) {
        T accr[RY][Q];
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int q = 0; q < Q; ++q) accr[r][q] = T(0);
#pragma unroll(UNROLL ? 20 : 1)
        for (int j = M - 1; j > L; --j) {
          T c[NRP];
          load_col(j, c);
#pragma unroll
          for (int r = 0; r < RY; ++r) {
            if (j < M - 1) shift_down1<T, Q>(accr[r]);
            colfma(c, j, r, accr[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          shift_down1<T, Q>(accr[r]);
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[r][q] += accr[r][q];
        }
      }
    } else {
    // left chain: columns 0..L flow up (shfl_up) into the output lane
    {
      T c[NRP];
      load_col(0, c);
#pragma unroll
      for (int r = 0; r < RY; ++r) colpart(win, c, 0, r, acc[r]);
    }
#pragma unroll(UNROLL ? 20 : 1)
    for (int j = 1; j <= L; ++j) {
      T c[NRP];
      load_col(j, c);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        T cp[Q];
        const bool any = colpart(win, c, j, r, cp);
        shift_up1<T, Q>(acc[r]);
        if (any) {
#pragma unroll
          for (int q = 0; q < Q; ++q) acc[r][q] += cp[q];
        }
      }
    }
    if (R > 0) {
      T accr[RY][Q];
      {
        T c[NRP];
        load_col(M - 1, c);
#pragma unroll
        for (int r = 0; r < RY; ++r) colpart(win, c, M - 1, r, accr[r]);
      }
      // right chain: columns M-2..L+1 flow down (shfl_down)
#pragma unroll(UNROLL ? 20 : 1)
      for (int j = M - 2; j > L; --j) {
        T c[NRP];
        load_col(j, c);
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          T cp[Q];
          const bool any = colpart(win, c, j, r, cp);
          shift_down1<T, Q>(accr[r]);
          if (any) {
#pragma unroll
            for (int q = 0; q < Q; ++q) accr[r][q] += cp[q];
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        shift_down1<T, Q>(accr[r]);
#pragma unroll
        for (int q = 0; q < Q; ++q) acc[r][q] += accr[r][q];
      }
    }
    }  // two-level chain
    const int y = y0 + pass * RY;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      if (y + r < y1) {
        T* o = outp + (pass * RY + r) * W;
        if (whole) {
          st_q<T, Q>(o, acc[r]);
        } else if (qmask) {
#pragma unroll
          for (int q = 0; q < Q; ++q)
            if (qmask & (1u << q)) o[q] = acc[r][q];
        }
      }
    }
    if constexpr (STARX) {
      // centre rows below s + RY - SK are done: boxes wholly below are free
      while ((rel + 1) * RB <= s + RY - SK) recycle(rel++);
    } else if ((s + RY) % RB == 0) {
      recycle(s / RB);  // the pass read the last row of box s/RB
    }
    if constexpr (STARX) {
      cw += RY;
      if (cw >= RB) {
        cw -= RB;
        cslot = cslot + 1 == D ? 0 : cslot + 1;
      }
    }
#pragma unroll
    for (int t = 0; t < NR - 1; ++t)
#pragma unroll
      for (int q = 0; q < Q; ++q) win[t][q] = win[t + RY][q];
  }
}

}  // namespace ssam_b200
