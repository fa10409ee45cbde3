/*
 * ssam_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU ground truth for the SSAM hot
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker.  The
 * product path (paper_1907_06154_b200/libssam_b200.so) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function here
 * against (a) the hand-computed fixtures of proj/tests/test_oracle.cpp and
 * (b) golden digests produced by the reference's own oracle.hpp, compiled
 * from /root/reference by oracle/Makefile into oracle/_ref/ and captured by
 * tests/golden/make_golden.py.
 *
 * Semantics restated (file:line relative to /root/reference):
 *   SplitMix64 ............ proj/include/ssam/rng.hpp:15-49
 *   random_grid2d/3d ...... proj/include/ssam/grid.hpp:52-66   (next_scalar, storage order)
 *   random_filter ......... proj/include/ssam/filter.hpp:41-47 (next_coeff)
 *   conv2d_naive .......... proj/include/ssam/oracle.hpp:44-59 (double acc for FP, s-major then t)
 *   stencil2d_naive ....... proj/include/ssam/oracle.hpp:80-96 (Jacobi, ring of width k fixed)
 *   stencil3d_naive ....... proj/include/ssam/oracle.hpp:98-116
 *   conv1d_naive .......... proj/include/ssam/oracle.hpp:61-73 (sample1d :30-36)
 *   scan_naive ............ proj/include/ssam/oracle.hpp:118-127
 *   benchmark catalog ..... proj/src/stencil_catalog.cpp:21-112
 *
 * Accumulation: double for f32/f64 inputs, native int64 for i64, one rounding
 * to the element type per cell per sweep (oracle.hpp:17-19).  Built with
 * -ffp-contract=off so no FMA contraction changes the double sums.  The
 * OpenMP loops only split independent output rows; each cell's summation
 * order is exactly the reference's, so results do not depend on threads.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SSAM_F32 0
#define SSAM_F64 1
#define SSAM_I64 2

static const uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:15-20 -- state advances by gamma before each draw. */
uint64_t ssam_oracle_splitmix_next(uint64_t* state) {
  *state += kGamma;
  return mix64(*state);
}

static inline double unit_from(uint64_t z) { /* rng.hpp:28-30 */
  return (double)(z >> 11) * 0x1.0p-52 - 1.0;
}

/* Fill count values of the reference's next_scalar (kind 0) or next_coeff
 * (kind 1) stream, starting at stream position `first` (0 = first draw). */
static void fill_stream(int dtype, void* out, size_t count, uint64_t seed, uint64_t first,
                        int coeff) {
  const int64_t lo = coeff ? -9 : -100;
  const uint64_t span = coeff ? 19u : 201u;
  for (size_t i = 0; i < count; ++i) {
    const uint64_t z = mix64(seed + (first + i + 1) * kGamma);
    switch (dtype) {
      case SSAM_F32: ((float*)out)[i] = (float)unit_from(z); break;
      case SSAM_F64: ((double*)out)[i] = unit_from(z); break;
      default: ((int64_t*)out)[i] = lo + (int64_t)(z % span); break;
    }
  }
}

/* grid.hpp:52-66: random_grid2d/3d draw next_scalar in storage order. */
void ssam_oracle_random_grid(int dtype, void* out, size_t count, uint64_t seed, uint64_t first) {
  fill_stream(dtype, out, count, seed, first, 0);
}

/* filter.hpp:41-47: random_filter draws next_coeff for w[s*n+t]. */
void ssam_oracle_random_filter(int dtype, void* out, size_t count, uint64_t seed) {
  fill_stream(dtype, out, count, seed, 0, 1);
}

static inline int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }

/* oracle.hpp:21-28 */
#define SAMPLE2D(T, g, w, h, x, y, bnd, dst)                                 \
  do {                                                                       \
    int xx_ = (x), yy_ = (y);                                                \
    if (xx_ >= 0 && xx_ < (w) && yy_ >= 0 && yy_ < (h))                      \
      dst = (g)[(size_t)yy_ * (w) + xx_];                                    \
    else if ((bnd) == 0)                                                     \
      dst = (T)0;                                                            \
    else                                                                     \
      dst = (g)[(size_t)clampi(yy_, (h)) * (w) + clampi(xx_, (w))];          \
  } while (0)

/* oracle.hpp:44-59:  out(x,y) = sum_{s<m} sum_{t<n} in(x+ax-s, y+ay-t) * w[s*n+t] */
#define CONV2D_BODY(T, ACC)                                                  \
  {                                                                          \
    const T* g = (const T*)in;                                               \
    const T* f = (const T*)wts;                                              \
    T* o = (T*)out;                                                          \
    const int ax = (m - 1) / 2, ay = (n - 1) / 2;                            \
    _Pragma("omp parallel for schedule(static)")                             \
    for (int y = 0; y < h; ++y)                                              \
      for (int x = 0; x < w; ++x) {                                          \
        ACC sum = 0;                                                         \
        for (int s = 0; s < m; ++s)                                          \
          for (int t = 0; t < n; ++t) {                                      \
            T v;                                                             \
            SAMPLE2D(T, g, w, h, x + ax - s, y + ay - t, boundary, v);       \
            sum += (ACC)v * (ACC)f[(size_t)s * n + t];                       \
          }                                                                  \
        o[(size_t)y * w + x] = (T)sum;                                       \
      }                                                                      \
  }

int ssam_oracle_conv2d(int dtype, const void* in, int w, int h, const void* wts, int m, int n,
                       int boundary, void* out) {
  if (w < 1 || h < 1 || m < 1 || n < 1) return 1;
  switch (dtype) {
    case SSAM_F32: CONV2D_BODY(float, double) break;
    case SSAM_F64: CONV2D_BODY(double, double) break;
    case SSAM_I64: CONV2D_BODY(int64_t, int64_t) break;
    default: return 1;
  }
  return 0;
}

/* oracle.hpp:61-73: out(i) = sum_{s<m} in(i+ax-s) * f[s], ax = (m-1)/2,
 * sample1d (:30-36) zero or clamp-replicate. */
#define CONV1D_BODY(T, ACC)                                                  \
  {                                                                          \
    const T* g = (const T*)in;                                               \
    const T* f = (const T*)wts;                                              \
    T* o = (T*)out;                                                          \
    const int ax = (m - 1) / 2;                                              \
    for (int i = 0; i < len; ++i) {                                          \
      ACC sum = 0;                                                           \
      for (int s = 0; s < m; ++s) {                                          \
        int j = i + ax - s;                                                  \
        T v;                                                                 \
        if (j >= 0 && j < len) v = g[j];                                     \
        else if (boundary == 0) v = (T)0;                                    \
        else v = g[clampi(j, len)];                                          \
        sum += (ACC)v * (ACC)f[s];                                           \
      }                                                                      \
      o[i] = (T)sum;                                                         \
    }                                                                        \
  }

int ssam_oracle_conv1d(int dtype, const void* in, int len, const void* wts, int m, int boundary,
                       void* out) {
  if (len < 0 || m < 1) return 1;
  switch (dtype) {
    case SSAM_F32: CONV1D_BODY(float, double) break;
    case SSAM_F64: CONV1D_BODY(double, double) break;
    case SSAM_I64: CONV1D_BODY(int64_t, int64_t) break;
    default: return 1;
  }
  return 0;
}

/* oracle.hpp:118-127: running sum in Acc<T>, rounded to T per element. */
#define SCAN_BODY(T, ACC)                                                    \
  {                                                                          \
    const T* g = (const T*)in;                                               \
    T* o = (T*)out;                                                          \
    ACC run = 0;                                                             \
    for (size_t i = 0; i < len; ++i) {                                       \
      run += (ACC)g[i];                                                      \
      o[i] = (T)run;                                                         \
    }                                                                        \
  }

int ssam_oracle_scan(int dtype, const void* in, size_t len, void* out) {
  switch (dtype) {
    case SSAM_F32: SCAN_BODY(float, double) break;
    case SSAM_F64: SCAN_BODY(double, double) break;
    case SSAM_I64: SCAN_BODY(int64_t, int64_t) break;
    default: return 1;
  }
  return 0;
}

/* oracle.hpp:80-96: Jacobi sweeps over k <= x < W-k, k <= y < H-k; taps in
 * the caller's order; the ring of width k (= declared order) carries over. */
#define STENCIL2D_BODY(T, ACC)                                               \
  {                                                                          \
    const T* c = (const T*)coeffs;                                           \
    T* cur = (T*)malloc(sizeof(T) * cells);                                  \
    T* nxt = (T*)malloc(sizeof(T) * cells);                                  \
    if (!cur || !nxt) { free(cur); free(nxt); return 2; }                    \
    memcpy(cur, in, sizeof(T) * cells);                                      \
    memcpy(nxt, in, sizeof(T) * cells);                                      \
    for (int it = 0; it < iters; ++it) {                                     \
      _Pragma("omp parallel for schedule(static)")                           \
      for (int y = k; y < h - k; ++y)                                        \
        for (int x = k; x < w - k; ++x) {                                    \
          ACC sum = 0;                                                       \
          for (int j = 0; j < ntaps; ++j)                                    \
            sum += (ACC)cur[(size_t)(y + offsets[3 * j + 1]) * w +           \
                            (x + offsets[3 * j])] * (ACC)c[j];               \
          nxt[(size_t)y * w + x] = (T)sum;                                   \
        }                                                                    \
      T* tmp = cur; cur = nxt; nxt = tmp;                                    \
    }                                                                        \
    memcpy(out, cur, sizeof(T) * cells);                                     \
    free(cur); free(nxt);                                                    \
  }

int ssam_oracle_stencil2d(int dtype, const void* in, int w, int h, const int* offsets,
                          const void* coeffs, int ntaps, int order, int iters, void* out) {
  if (w < 1 || h < 1 || ntaps < 0 || iters < 0) return 1;
  const size_t cells = (size_t)w * h;
  const int k = order;
  switch (dtype) {
    case SSAM_F32: STENCIL2D_BODY(float, double) break;
    case SSAM_F64: STENCIL2D_BODY(double, double) break;
    case SSAM_I64: STENCIL2D_BODY(int64_t, int64_t) break;
    default: return 1;
  }
  return 0;
}

/* oracle.hpp:98-116 */
#define STENCIL3D_BODY(T, ACC)                                               \
  {                                                                          \
    const T* c = (const T*)coeffs;                                           \
    T* cur = (T*)malloc(sizeof(T) * cells);                                  \
    T* nxt = (T*)malloc(sizeof(T) * cells);                                  \
    if (!cur || !nxt) { free(cur); free(nxt); return 2; }                    \
    memcpy(cur, in, sizeof(T) * cells);                                      \
    memcpy(nxt, in, sizeof(T) * cells);                                      \
    for (int it = 0; it < iters; ++it) {                                     \
      _Pragma("omp parallel for schedule(static) collapse(2)")               \
      for (int z = k; z < nz - k; ++z)                                       \
        for (int y = k; y < ny - k; ++y)                                     \
          for (int x = k; x < nx - k; ++x) {                                 \
            ACC sum = 0;                                                     \
            for (int j = 0; j < ntaps; ++j) {                                \
              const size_t idx =                                             \
                  ((size_t)(z + offsets[3 * j + 2]) * ny +                   \
                   (size_t)(y + offsets[3 * j + 1])) * nx +                  \
                  (size_t)(x + offsets[3 * j]);                              \
              sum += (ACC)cur[idx] * (ACC)c[j];                              \
            }                                                                \
            nxt[((size_t)z * ny + y) * nx + x] = (T)sum;                     \
          }                                                                  \
      T* tmp = cur; cur = nxt; nxt = tmp;                                    \
    }                                                                        \
    memcpy(out, cur, sizeof(T) * cells);                                     \
    free(cur); free(nxt);                                                    \
  }

int ssam_oracle_stencil3d(int dtype, const void* in, int nx, int ny, int nz, const int* offsets,
                          const void* coeffs, int ntaps, int order, int iters, void* out) {
  if (nx < 1 || ny < 1 || nz < 1 || ntaps < 0 || iters < 0) return 1;
  const size_t cells = (size_t)nx * ny * nz;
  const int k = order;
  switch (dtype) {
    case SSAM_F32: STENCIL3D_BODY(float, double) break;
    case SSAM_F64: STENCIL3D_BODY(double, double) break;
    case SSAM_I64: STENCIL3D_BODY(int64_t, int64_t) break;
    default: return 1;
  }
  return 0;
}

/* ------------------------------------------------------------------------
 * Benchmark catalog -- proj/src/stencil_catalog.cpp:21-112.
 * Shapes: star (centre + arms of length k per axis), box ((2k+1)^dims),
 * box_even (8x8, offsets [-4,3]), poisson19 (3x3x3 minus corners).
 * Canonical order: (dz, dy, dx) ascending with the centre pulled out last;
 * off-centre tap j (1-based) of t weighs j / (2 * t(t+1)/2), centre 0.5
 * (1.0 when it is the only tap).
 * ---------------------------------------------------------------------- */
enum { SHAPE_STAR, SHAPE_BOX, SHAPE_BOX_EVEN, SHAPE_POISSON19 };
typedef struct {
  const char* name;
  int dims, order, fpp, shape;
} bench_def;

static const bench_def kBench[] = {
    {"2d5pt", 2, 1, 9, SHAPE_STAR},     {"2d9pt", 2, 2, 17, SHAPE_STAR},
    {"2d13pt", 2, 3, 25, SHAPE_STAR},   {"2d17pt", 2, 4, 33, SHAPE_STAR},
    {"2d21pt", 2, 5, 41, SHAPE_STAR},   {"2ds25pt", 2, 6, 49, SHAPE_STAR},
    {"2d25pt", 2, 2, 33, SHAPE_BOX},    {"2d64pt", 2, 4, 73, SHAPE_BOX_EVEN},
    {"2d81pt", 2, 4, 95, SHAPE_BOX},    {"2d121pt", 2, 5, 241, SHAPE_BOX},
    {"3d7pt", 3, 1, 13, SHAPE_STAR},    {"3d13pt", 3, 2, 25, SHAPE_STAR},
    {"3d27pt", 3, 1, 30, SHAPE_BOX},    {"3d125pt", 3, 2, 130, SHAPE_BOX},
    {"poisson", 3, 1, 21, SHAPE_POISSON19},
};
#define NBENCH ((int)(sizeof(kBench) / sizeof(kBench[0])))

int ssam_oracle_benchmark_count(void) { return NBENCH; }
const char* ssam_oracle_benchmark_name(int i) { return (i >= 0 && i < NBENCH) ? kBench[i].name : 0; }

static int cmp_zyx(const void* a, const void* b) {
  const int* p = (const int*)a;
  const int* q = (const int*)b;
  if (p[2] != q[2]) return p[2] < q[2] ? -1 : 1;
  if (p[1] != q[1]) return p[1] < q[1] ? -1 : 1;
  if (p[0] != q[0]) return p[0] < q[0] ? -1 : 1;
  return 0;
}

/* Writes up to cap taps; returns the tap count, or -1 for an unknown name. */
int ssam_oracle_benchmark_stencil(const char* name, int* dims, int* order, int* fpp,
                                  int* offsets, double* coeffs, int cap) {
  const bench_def* d = 0;
  for (int i = 0; i < NBENCH; ++i)
    if (strcmp(name, kBench[i].name) == 0) d = &kBench[i];
  if (!d) return -1;
  int offs[125 * 3];
  int n = 0;
  const int k = d->order;
#define PUSH(a, b, c) do { offs[3 * n] = (a); offs[3 * n + 1] = (b); offs[3 * n + 2] = (c); ++n; } while (0)
  switch (d->shape) {
    case SHAPE_STAR:
      PUSH(0, 0, 0);
      for (int i = 1; i <= k; ++i) {
        PUSH(-i, 0, 0); PUSH(i, 0, 0); PUSH(0, -i, 0); PUSH(0, i, 0);
        if (d->dims == 3) { PUSH(0, 0, -i); PUSH(0, 0, i); }
      }
      break;
    case SHAPE_BOX: {
      const int zlo = d->dims == 3 ? -k : 0, zhi = d->dims == 3 ? k : 0;
      for (int dz = zlo; dz <= zhi; ++dz)
        for (int dy = -k; dy <= k; ++dy)
          for (int dx = -k; dx <= k; ++dx) PUSH(dx, dy, dz);
      break;
    }
    case SHAPE_BOX_EVEN:
      for (int dy = -4; dy <= 3; ++dy)
        for (int dx = -4; dx <= 3; ++dx) PUSH(dx, dy, 0);
      break;
    default:
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx)
            if (abs(dx) + abs(dy) + abs(dz) <= 2) PUSH(dx, dy, dz);
      break;
  }
#undef PUSH
  qsort(offs, (size_t)n, 3 * sizeof(int), cmp_zyx);
  if (n > cap) return -2;
  const int t = n - 1;
  const double denom = 2.0 * ((double)t * (t + 1) / 2.0);
  int out = 0, j = 0;
  for (int i = 0; i < n; ++i) {
    const int* o = &offs[3 * i];
    if (o[0] == 0 && o[1] == 0 && o[2] == 0) continue;
    ++j;
    offsets[3 * out] = o[0]; offsets[3 * out + 1] = o[1]; offsets[3 * out + 2] = o[2];
    coeffs[out] = t > 0 ? (double)j / denom : 0.0;
    ++out;
  }
  offsets[3 * out] = 0; offsets[3 * out + 1] = 0; offsets[3 * out + 2] = 0;
  coeffs[out] = 0.5 + (t == 0 ? 0.5 : 0.0);
  ++out;
  *dims = d->dims;
  *order = d->order;
  *fpp = d->fpp;
  return out;
}
