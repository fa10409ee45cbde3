// abi.cpp -- the C ABI (include/ssam_b200.h): the reference's error contract,
// closed-form OpCounters, the benchmark catalog, buffer management and
// dispatch onto the CUDA engines.
//
// Every compute entry point ends on the GPU; there is no host compute path.

#include "ssam_b200.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include <cuda_runtime.h>

#include "internal.hpp"

namespace ssam_b200 {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
std::uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// Shape classification (kernel selection only).
// ---------------------------------------------------------------------------
namespace {
bool same_set(std::vector<std::array<int, 3>> a, std::vector<std::array<int, 3>> b) {
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  return a == b;
}
std::vector<std::array<int, 3>> as_arrays(const std::vector<Tap>& taps) {
  std::vector<std::array<int, 3>> v;
  v.reserve(taps.size());
  for (const Tap& t : taps) v.push_back({t.dx, t.dy, t.dz});
  return v;
}
std::vector<std::array<int, 3>> star_set(int k, int dims) {
  std::vector<std::array<int, 3>> v{{0, 0, 0}};
  for (int i = 1; i <= k; ++i) {
    v.push_back({-i, 0, 0});
    v.push_back({i, 0, 0});
    v.push_back({0, -i, 0});
    v.push_back({0, i, 0});
    if (dims == 3) {
      v.push_back({0, 0, -i});
      v.push_back({0, 0, i});
    }
  }
  return v;
}
std::vector<std::array<int, 3>> box_set(int k, int dims) {
  std::vector<std::array<int, 3>> v;
  const int zk = dims == 3 ? k : 0;
  for (int dz = -zk; dz <= zk; ++dz)
    for (int dy = -k; dy <= k; ++dy)
      for (int dx = -k; dx <= k; ++dx) v.push_back({dx, dy, dz});
  return v;
}
std::vector<std::array<int, 3>> poisson_set() {
  std::vector<std::array<int, 3>> v;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx)
        if (std::abs(dx) + std::abs(dy) + std::abs(dz) <= 2) v.push_back({dx, dy, dz});
  return v;
}
}  // namespace

Shape2D classify2d(const std::vector<Tap>& taps, int order) {
  return same_set(as_arrays(taps), star_set(order, 2)) ? Shape2D::star : Shape2D::other;
}
Shape3D classify3d(const std::vector<Tap>& taps, int order) {
  const auto t = as_arrays(taps);
  if (same_set(t, star_set(order, 3))) return Shape3D::star;
  if (same_set(t, box_set(order, 3))) return Shape3D::box;
  if (order == 1 && same_set(t, poisson_set())) return Shape3D::poisson;
  return Shape3D::other;
}

}  // namespace ssam_b200

using namespace ssam_b200;

namespace {

thread_local std::string g_err;

int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation)
    return fail(SSAM_ERR_OUT_OF_MEMORY, std::string(where) + ": " + cudaGetErrorString(e));
  return fail(SSAM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool dtype_ok(int dtype) { return dtype >= 0 && dtype <= 2; }

ssam_kernel_config cfg_or_default(const ssam_kernel_config* c) {
  ssam_kernel_config d;
  ssam_b200_default_config(&d);
  return c ? *c : d;
}

// KernelConfig::check(filter_n) -- proj/include/ssam/filter.hpp:130-138.
int check_cfg(const ssam_kernel_config& c, int filter_n) {
  if (c.p < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "config: p must be >= 1");
  if (c.lane_count < 2 || c.lane_count > 64 || (c.lane_count & (c.lane_count - 1)) != 0)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "config: lane_count must be a power of two in [2, 64]");
  if (c.b < c.lane_count || c.b % c.lane_count != 0)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "config: b must be a positive multiple of lane_count");
  if (static_cast<long long>(filter_n) + c.p - 1 > 255)
    return fail(SSAM_ERR_LENGTH, "config: register cache C = n + p - 1 exceeds the cap");
  return SSAM_OK;
}

// validate_stencil -- filter.hpp:76-94.
int validate_stencil(const ssam_stencil* st) {
  if (!st) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: null descriptor");
  if (st->dims != 2 && st->dims != 3)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: dims must be 2 or 3");
  if (st->ntaps <= 0 || !st->offsets) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: no taps");
  if (!st->coeffs) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: null coefficients");
  int k = 0;
  for (int i = 0; i < st->ntaps; ++i) {
    const int* o = st->offsets + 3 * i;
    if (st->dims == 2 && o[2] != 0)
      return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: 2D stencil has a z offset");
    for (int c = 0; c < 3; ++c) {
      if (std::abs(o[c]) > st->order)
        return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: offset outside declared order");
      k = std::max(k, std::abs(o[c]));
    }
  }
  if (k != st->order)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: declared order does not match taps");
  for (int i = 0; i < st->ntaps; ++i)
    for (int j = i + 1; j < st->ntaps; ++j)
      if (std::memcmp(st->offsets + 3 * i, st->offsets + 3 * j, 3 * sizeof(int)) == 0)
        return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil: duplicate tap offset");
  return SSAM_OK;
}

// conv2d preconditions, in the reference's order: Filter2D ctor
// (filter.hpp:28-31), kernels.hpp:192-198, plan_blocks (blocking.cpp:10-16).
int check_conv2d(int w, int h, int m, int n, const ssam_kernel_config& c) {
  if (m < 1 || n < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "filter: taps must be >= 1");
  if (w < 1 || h < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "grid2d: dimensions must be >= 1");
  if (m > 20 || n > 20)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "conv2d: filter larger than the supported 20x20 range");
  if (int s = check_cfg(c, n)) return s;
  if (w < c.lane_count) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv2d: grid narrower than one warp");
  if (h < n + c.p - 1)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "conv2d: grid shorter than one cache block");
  if (m > c.lane_count) return fail(SSAM_ERR_INVALID_ARGUMENT, "plan_blocks: m exceeds lane_count");
  return SSAM_OK;
}

// kernels.hpp:234-245 (+ plan_blocks / stencil_window_plans lane checks).
int check_stencil2d(int w, int h, const ssam_stencil* st, const ssam_kernel_config& c, int iters) {
  if (w < 1 || h < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "grid2d: dimensions must be >= 1");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 2) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: needs a 2D stencil");
  if (iters < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: iters must be >= 1");
  const int m = 2 * st->order + 1;
  if (w < m || h < m)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: domain smaller than the stencil diameter");
  if (int s = check_cfg(c, m)) return s;
  if (m > c.lane_count) return fail(SSAM_ERR_INVALID_ARGUMENT, "plan_blocks: m exceeds lane_count");
  return SSAM_OK;
}

// kernels.hpp:286-299 (+ stencil_window_plans lane check).
int check_stencil3d(int nx, int ny, int nz, const ssam_stencil* st, const ssam_kernel_config& c,
                    int iters) {
  if (nx < 1 || ny < 1 || nz < 1)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "grid3d: dimensions must be >= 1");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 3) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: needs a 3D stencil");
  if (iters < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: iters must be >= 1");
  const int m = 2 * st->order + 1;
  if (nx < m || ny < m || nz < m)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: domain smaller than the stencil diameter");
  if (int s = check_cfg(c, m)) return s;
  if (c.b / c.lane_count < m)
    return fail(SSAM_ERR_INVALID_ARGUMENT,
                "stencil3d: block must hold at least 2k+1 warps; raise b");
  if (m > c.lane_count)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil plans: order too high for the warp");
  return SSAM_OK;
}

// ---- closed-form OpCounters ---------------------------------------------------
// One window plan's (mads, shuffles) for a 2D tap slice -- the stage list
// stencil_window_plans builds (kernels.hpp:111-159): one mad per tap, one
// shuffle at the first tap of every column reached after a shift, plus a
// trailing copy stage if a shift is left over.
struct WindowStats {
  std::uint64_t mads = 0, shuffles = 0;
};
WindowStats window_stats(const std::vector<int>& column_counts) {
  WindowStats ws;
  int pending = 0;
  for (size_t j = 0; j < column_counts.size(); ++j) {
    if (j > 0) pending += 1;
    for (int c = 0; c < column_counts[j]; ++c) {
      ws.mads += 1;
      if (pending > 0) ws.shuffles += 1;
      pending = 0;
    }
  }
  if (pending > 0) ws.shuffles += 1;
  return ws;
}

std::uint64_t ceil_div(std::uint64_t a, std::uint64_t b) { return (a + b - 1) / b; }

// conv2d: tiles x per-warp law (test_kernels_conv.cpp:70-103).
void counters_conv2d(int w, int h, int m, int n, const ssam_kernel_config& c,
                     ssam_op_counters* out) {
  const std::uint64_t S = c.lane_count, C = static_cast<std::uint64_t>(n) + c.p - 1;
  const std::uint64_t tiles = ceil_div(h, c.p) * ceil_div(w, S - m + 1);
  out->mads += tiles * m * n * c.p;
  out->shuffles += tiles * (m - 1) * c.p;
  out->broadcast_reads += tiles * m * n * c.p;
  out->global_loads += tiles * S * C;
  out->global_stores += static_cast<std::uint64_t>(w) * h;
}

void counters_stencil2d(int w, int h, const ssam_stencil* st, const ssam_kernel_config& c,
                        int iters, ssam_op_counters* out) {
  const int k = st->order, m = 2 * k + 1;
  std::vector<int> cols(m, 0);
  for (int i = 0; i < st->ntaps; ++i) cols[st->offsets[3 * i] + k] += 1;
  const WindowStats ws = window_stats(cols);
  const std::uint64_t S = c.lane_count, C = static_cast<std::uint64_t>(m) + c.p - 1;
  const std::uint64_t tiles = ceil_div(h, c.p) * ceil_div(w, S - m + 1);
  const std::uint64_t it = iters;
  out->mads += it * tiles * ws.mads * c.p;
  out->shuffles += it * tiles * ws.shuffles * c.p;
  out->global_loads += it * tiles * S * C;
  out->global_stores += it * static_cast<std::uint64_t>(w - 2 * k) * (h - 2 * k);
}

void counters_stencil3d(int nx, int ny, int nz, const ssam_stencil* st,
                        const ssam_kernel_config& c, int iters, ssam_op_counters* out) {
  const int k = st->order, m = 2 * k + 1;
  const std::uint64_t S = c.lane_count, C = static_cast<std::uint64_t>(m) + c.p - 1;
  const int warp_count = c.b / c.lane_count;
  const int valid_z = warp_count - 2 * k;
  const std::uint64_t blocks =
      ceil_div(nx, S - m + 1) * ceil_div(ny, c.p) * ceil_div(nz, valid_z);
  std::uint64_t mads = 0, shuffles = 0;
  for (int dz = -k; dz <= k; ++dz) {
    std::vector<int> cols(m, 0);
    bool any = false;
    for (int i = 0; i < st->ntaps; ++i)
      if (st->offsets[3 * i + 2] == dz) {
        cols[st->offsets[3 * i] + k] += 1;
        any = true;
      }
    if (!any) continue;
    const WindowStats ws = window_stats(cols);
    mads += ws.mads * c.p;
    shuffles += ws.shuffles * c.p;
  }
  const std::uint64_t it = iters, wc = warp_count;
  out->mads += it * blocks * wc * mads;
  out->shuffles += it * blocks * wc * shuffles;
  out->global_loads += it * blocks * wc * S * C;
  out->global_stores +=
      it * static_cast<std::uint64_t>(nx - 2 * k) * (ny - 2 * k) * (nz - 2 * k);
}

// ---- benchmark catalog (stencil_catalog.cpp:21-112 semantics) ----------------
struct BenchDef {
  const char* name;
  int dims, order, fpp;
  char shape;  // 's' star, 'b' box, 'e' 8x8 even box, 'p' poisson19
};
constexpr BenchDef kBench[] = {
    {"2d5pt", 2, 1, 9, 's'},    {"2d9pt", 2, 2, 17, 's'},    {"2d13pt", 2, 3, 25, 's'},
    {"2d17pt", 2, 4, 33, 's'},  {"2d21pt", 2, 5, 41, 's'},   {"2ds25pt", 2, 6, 49, 's'},
    {"2d25pt", 2, 2, 33, 'b'},  {"2d64pt", 2, 4, 73, 'e'},   {"2d81pt", 2, 4, 95, 'b'},
    {"2d121pt", 2, 5, 241, 'b'}, {"3d7pt", 3, 1, 13, 's'},   {"3d13pt", 3, 2, 25, 's'},
    {"3d27pt", 3, 1, 30, 'b'},  {"3d125pt", 3, 2, 130, 'b'}, {"poisson", 3, 1, 21, 'p'},
};
constexpr int kNumBench = sizeof(kBench) / sizeof(kBench[0]);

// ---- device + buffers ----------------------------------------------------------
int device_ready() {
  static std::once_flag once;
  static int count = 0;
  std::call_once(once, [] {
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
      count = 0;
      cudaGetLastError();
    }
  });
  if (count <= 0) return fail(SSAM_ERR_NO_DEVICE, "no CUDA device available");
  return SSAM_OK;
}

// The engine's own stream-ordered pool per device: freed staging buffers of
// the host-grid calls stay cached (repeated calls reuse them instead of
// re-mapping memory) without touching the device's default pool, which torch
// and other cudaMallocAsync users share.  ssam_b200_trim_cache() returns the
// cached memory.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
cudaMemPool_t engine_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::uint64_t thr = std::numeric_limits<std::uint64_t>::max();
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pools[dev] = pool;
  }
  return g_pools[dev];
}

}  // namespace

namespace ssam_b200 {
cudaError_t engine_alloc(void** p, std::size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = engine_pool();
  return pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
}
}  // namespace ssam_b200

namespace {

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) {
    cudaMemPool_t pool = engine_pool();
    return pool ? cudaMallocFromPoolAsync(&p, bytes, pool, s) : cudaMallocAsync(&p, bytes, s);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

template <class T>
StencilDesc<T> make_desc(const ssam_stencil* st) {
  StencilDesc<T> d;
  d.dims = st->dims;
  d.order = st->order;
  const T* c = static_cast<const T*>(st->coeffs);
  for (int i = 0; i < st->ntaps; ++i) {
    d.taps.push_back({st->offsets[3 * i], st->offsets[3 * i + 1], st->offsets[3 * i + 2]});
    d.coeffs.push_back(c[i]);
  }
  return d;
}

// Temporal-block schedule: full tb-deep fused launches, then single sweeps.
template <class T>
cudaError_t run2d(T* a, T* b, int W, int H, const StencilDesc<T>& d, int iters, int tb,
                  cudaStream_t s, T** result) {
  const size_t bytes = static_cast<size_t>(W) * H * sizeof(T);
  cudaError_t e = cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, s);  // ring in both
  if (e != cudaSuccess) return e;
  T* cur = a;
  T* nxt = b;
  int done = 0;
  while (done < iters) {
    const int left = iters - done;
    int depth = 1;
    if (tb > 1 && left >= 2) {
      depth = std::min(tb, left);
      e = stencil2d_tb<T>(cur, nxt, W, H, d, depth, s);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        depth = 1;
      } else if (e != cudaSuccess) {
        return e;
      }
    }
    if (depth == 1) {
      e = stencil2d_sweep<T>(cur, nxt, W, H, 0, H, d, s);
      if (e != cudaSuccess) return e;
    }
    std::swap(cur, nxt);
    done += depth;
  }
  *result = cur;
  return cudaSuccess;
}

template <class T>
cudaError_t run3d(T* a, T* b, int nx, int ny, int nz, const StencilDesc<T>& d, int iters,
                  cudaStream_t s, T** result) {
  const size_t bytes = static_cast<size_t>(nx) * ny * nz * sizeof(T);
  cudaError_t e = cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return e;
  T* cur = a;
  T* nxt = b;
  const int dtype = sizeof(T) == 4 ? 0 : (std::is_same<T, double>::value ? 1 : 2);
  const int tb = stencil3d_tb_max(dtype, d.order, classify3d(d.taps, d.order));
  int done = 0;
  while (done < iters) {
    // full-depth fused launches, then the remainder as one shorter fused
    // launch where a kernel exists, else single sweeps
    int depth = std::min(tb, iters - done);
    if (depth > 1) {
      e = stencil3d_tb<T>(cur, nxt, nx, ny, nz, 0, nz, d.order, nz - d.order, d, depth, s);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        depth = 1;
      } else if (e != cudaSuccess) {
        return e;
      }
    }
    if (depth == 1) {
      e = stencil3d_sweep<T>(cur, nxt, nx, ny, nz, 0, nz, d, s);
      if (e != cudaSuccess) return e;
    }
    std::swap(cur, nxt);
    done += depth;
  }
  *result = cur;
  return cudaSuccess;
}

int default_tb(int dtype, const ssam_stencil* st) {
  return ssam_b200_stencil2d_tb_max(dtype, st);
}

// Host-grid calls: H2D -> GPU engine -> D2H on the per-thread stream.
template <class T>
int host_conv2d(const void* in, int w, int h, const void* wts, int m, int n, int boundary,
                void* out) {
  cudaStream_t s = cudaStreamPerThread;
  const size_t bytes = static_cast<size_t>(w) * h * sizeof(T);
  DevBuf din(s), dout(s);
  cudaError_t e;
  if ((e = din.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "conv2d alloc");
  if ((e = dout.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "conv2d alloc");
  if ((e = cudaMemcpyAsync(din.p, in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "conv2d H2D");
  if ((e = conv2d_device<T>(static_cast<const T*>(din.p), static_cast<T*>(dout.p), w, h, 0, h,
                            static_cast<const T*>(wts), m, n, boundary, s)) != cudaSuccess)
    return cuda_fail(e, "conv2d kernel");
  if ((e = cudaMemcpyAsync(out, dout.p, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "conv2d D2H");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "conv2d sync");
  return SSAM_OK;
}

template <class T>
int host_stencil(const void* in, int nx, int ny, int nz, const ssam_stencil* st, int iters,
                 void* out) {
  cudaStream_t s = cudaStreamPerThread;
  const size_t bytes = static_cast<size_t>(nx) * ny * nz * sizeof(T);
  DevBuf a(s), b(s);
  cudaError_t e;
  if ((e = a.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "stencil alloc");
  if ((e = b.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "stencil alloc");
  if ((e = cudaMemcpyAsync(a.p, in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "stencil H2D");
  const StencilDesc<T> d = make_desc<T>(st);
  T* res = nullptr;
  if (st->dims == 2) {
    const int dtype = sizeof(T) == 4 ? SSAM_DTYPE_F32 : (std::is_same<T, double>::value ? 1 : 2);
    e = run2d<T>(static_cast<T*>(a.p), static_cast<T*>(b.p), nx, ny, d, iters,
                 default_tb(dtype, st), s, &res);
  } else {
    e = run3d<T>(static_cast<T*>(a.p), static_cast<T*>(b.p), nx, ny, nz, d, iters, s, &res);
  }
  if (e != cudaSuccess) return cuda_fail(e, "stencil kernel");
  if ((e = cudaMemcpyAsync(out, res, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "stencil D2H");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "stencil sync");
  return SSAM_OK;
}

template <template <class> class F, class... Args>
int by_dtype(int dtype, Args&&... args) {
  switch (dtype) {
    case SSAM_DTYPE_F32: return F<float>::run(args...);
    case SSAM_DTYPE_F64: return F<double>::run(args...);
    case SSAM_DTYPE_I64: return F<long long>::run(args...);
  }
  return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
}

template <class T> struct HostConv {
  template <class... A> static int run(A... a) { return host_conv2d<T>(a...); }
};
template <class T> struct HostStencil {
  template <class... A> static int run(A... a) { return host_stencil<T>(a...); }
};

// Multi-device host calls (multi.cpp): same validation and counters as the
// one-device entry points, the device list checked against the runtime.
template <class T>
int host_stencil_multi(const void* in, int nx, int ny, int nz, const ssam_stencil* st, int iters,
                       const int* devices, int ndev, void* out, int* used) {
  const StencilDesc<T> d = make_desc<T>(st);
  const int dtype = sizeof(T) == 4 ? SSAM_DTYPE_F32 : (std::is_same<T, double>::value ? 1 : 2);
  const int tb = st->dims == 2 ? default_tb(dtype, st)
                               : stencil3d_tb_max(dtype, d.order, classify3d(d.taps, d.order));
  const cudaError_t e = multi_stencil<T>(static_cast<const T*>(in), static_cast<T*>(out), nx, ny,
                                         st->dims == 2 ? 1 : nz, d, iters, tb, devices, ndev, used);
  if (e != cudaSuccess) return cuda_fail(e, "stencil multi");
  return SSAM_OK;
}
template <class T> struct HostStencilMulti {
  template <class... A> static int run(A... a) { return host_stencil_multi<T>(a...); }
};

int check_devices(const int* devices, int ndev) {
  if (!devices || ndev < 1) return fail(SSAM_ERR_INVALID_ARGUMENT, "multi: empty device list");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    count = 0;
  }
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count)
      return fail(SSAM_ERR_INVALID_ARGUMENT, "multi: device index out of range");
  return SSAM_OK;
}

// ---- 1D: conv1d / scan (kernels.hpp:390-447) -----------------------------------
bool pow2_lanes(int s) { return s >= 2 && s <= 64 && (s & (s - 1)) == 0; }

// ssam::conv1d's checks in its order (kernels.hpp:393-397, then the
// WarpState constructor, warp.hpp:36-38, on the first tile).
int check_conv1d(long long len, int m, const ssam_kernel_config& c) {
  const int s = c.lane_count;
  if (m < 1 || m > s)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "conv1d: filter length must be in [1, lane_count]");
  if (len < s) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv1d: signal shorter than one warp");
  if (!pow2_lanes(s))
    return fail(SSAM_ERR_INVALID_ARGUMENT, "warp: lane_count must be a power of two in [2, 64]");
  return SSAM_OK;
}

// ssam::scan's checks (kernels.hpp:425-429, make_scan_plan plan.hpp:199-201).
// An empty input returns before the plan is built, so any lane_count > 0 is
// accepted for it; lane_count <= 0 (undefined in the reference) is rejected.
int check_scan(unsigned long long len, int s) {
  if (s <= 0) return fail(SSAM_ERR_INVALID_ARGUMENT, "scan: lane_count must be positive");
  if (len % static_cast<unsigned long long>(s) != 0)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "scan: length must be a multiple of lane_count");
  if (len == 0) return SSAM_OK;
  if (!pow2_lanes(s))
    return fail(SSAM_ERR_INVALID_ARGUMENT,
                "scan plan: lane_count must be a power of two in [2, 64]");
  return SSAM_OK;
}

// Closed forms of the simulator's counts: conv1d tiles of valid_w = S-m+1
// outputs, each m MAD stages (broadcast weight), m-1 shifts, S loads;
// scan tiles of S, each log2(S) MAD + shuffle stages (immediate 1), S loads
// and S stores.
void counters_conv1d(long long len, int m, const ssam_kernel_config& c, ssam_op_counters* o) {
  const std::uint64_t s = c.lane_count;
  const std::uint64_t tiles = ceil_div(static_cast<std::uint64_t>(len), s - m + 1);
  o->mads += tiles * m;
  o->shuffles += tiles * (m - 1);
  o->broadcast_reads += tiles * m;
  o->global_loads += tiles * s;
  o->global_stores += static_cast<std::uint64_t>(len);
}
void counters_scan(unsigned long long len, int s, ssam_op_counters* o) {
  if (len == 0) return;
  const std::uint64_t tiles = len / s;
  std::uint64_t lg = 0;
  while ((1 << lg) < s) ++lg;
  o->mads += tiles * lg;
  o->shuffles += tiles * lg;
  o->global_loads += len;
  o->global_stores += len;
}

template <class T>
int host_conv1d(const void* in, int len, const void* wts, int m, int boundary, void* out) {
  cudaStream_t s = cudaStreamPerThread;
  const size_t bytes = static_cast<size_t>(len) * sizeof(T);
  DevBuf din(s), dout(s);
  cudaError_t e;
  if ((e = din.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "conv1d alloc");
  if ((e = dout.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "conv1d alloc");
  if ((e = cudaMemcpyAsync(din.p, in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "conv1d H2D");
  if ((e = conv1d_device<T>(static_cast<const T*>(din.p), static_cast<T*>(dout.p), len,
                            static_cast<const T*>(wts), m, boundary, s)) != cudaSuccess)
    return cuda_fail(e, "conv1d kernel");
  if ((e = cudaMemcpyAsync(out, dout.p, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "conv1d D2H");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "conv1d sync");
  return SSAM_OK;
}

template <class T>
int host_scan(const void* in, size_t len, void* out) {
  cudaStream_t s = cudaStreamPerThread;
  const size_t bytes = len * sizeof(T);
  DevBuf din(s), dout(s);
  cudaError_t e;
  if ((e = din.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "scan alloc");
  if ((e = dout.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "scan alloc");
  if ((e = cudaMemcpyAsync(din.p, in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "scan H2D");
  if ((e = scan_device<T>(static_cast<const T*>(din.p), static_cast<T*>(dout.p), len, s)) !=
      cudaSuccess)
    return cuda_fail(e, "scan kernel");
  if ((e = cudaMemcpyAsync(out, dout.p, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "scan D2H");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "scan sync");
  return SSAM_OK;
}

template <class T> struct HostConv1 {
  template <class... A> static int run(A... a) { return host_conv1d<T>(a...); }
};
template <class T> struct HostScan {
  template <class... A> static int run(A... a) { return host_scan<T>(a...); }
};

// Direct-gather runs (oracle summation order and arithmetic, direct.cu) on
// host buffers: the GPU-side verifier the CLI compares the engine against.
template <class T>
int host_gather(int kind, const void* in, int nx, int ny, int nz, const void* wts, int m, int n,
                int boundary, const ssam_stencil* st, int iters, void* out) {
  cudaStream_t s = cudaStreamPerThread;
  const size_t bytes = static_cast<size_t>(nx) * ny * nz * sizeof(T);
  DevBuf a(s), b(s);
  cudaError_t e;
  if ((e = a.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "gather alloc");
  if ((e = b.alloc(bytes)) != cudaSuccess) return cuda_fail(e, "gather alloc");
  if ((e = cudaMemcpyAsync(a.p, in, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "gather H2D");
  T* cur = static_cast<T*>(a.p);
  T* nxt = static_cast<T*>(b.p);
  if (kind == 0) {
    e = conv2d_direct<T>(cur, nxt, nx, ny, static_cast<const T*>(wts), m, n, boundary, s);
    std::swap(cur, nxt);
  } else {
    const StencilDesc<T> d = make_desc<T>(st);
    e = cudaMemcpyAsync(nxt, cur, bytes, cudaMemcpyDeviceToDevice, s);  // the ring
    for (int it = 0; e == cudaSuccess && it < iters; ++it) {
      e = st->dims == 2 ? stencil2d_direct<T>(cur, nxt, nx, ny, 0, ny, d, s)
                        : stencil3d_direct<T>(cur, nxt, nx, ny, nz, 0, nz, d, s);
      std::swap(cur, nxt);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "gather kernel");
  if ((e = cudaMemcpyAsync(out, cur, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "gather D2H");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "gather sync");
  return SSAM_OK;
}
template <class T> struct HostGather {
  template <class... A> static int run(A... a) { return host_gather<T>(a...); }
};

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

namespace ssam_b200 {
// Status + message for the other host-side units (grid_io.cpp).
int set_error(int status, const std::string& msg) { return fail(status, msg); }

const PeerHalo*& peer_halo_slot() {
  thread_local const PeerHalo* h = nullptr;
  return h;
}
}  // namespace ssam_b200

namespace {

PeerHalo to_peer(const ssam_peer_halo* p) {
  return PeerHalo{p->lo, p->lo_shift, p->lo_end, p->hi, p->hi_shift, p->hi_begin};
}

// Makes the launches of one ABI call store the peer halo (launch.cuh, apply_peer_halo).
struct PeerScope {
  explicit PeerScope(const PeerHalo* h) { peer_halo_slot() = h; }
  ~PeerScope() { peer_halo_slot() = nullptr; }
  PeerScope(const PeerScope&) = delete;
  PeerScope& operator=(const PeerScope&) = delete;
};

// Copies the written planes [z0, z1) a neighbour mirrors into its buffer
// (whole planes: ring cells equal on both sides) -- for kernels that do not
// store the peer halo themselves.
int push_planes(int dtype, void* d_out, int nx, int ny, int z0, int z1, const PeerHalo& h,
                cudaStream_t s) {
  const size_t es = dtype == 0 ? 4 : 8, plane = static_cast<size_t>(nx) * ny * es;
  char* base = static_cast<char*>(d_out);
  auto push = [&](void* peer, long long shift, int a, int b) -> cudaError_t {
    if (!peer || b <= a) return cudaSuccess;
    char* dst = static_cast<char*>(peer) + (static_cast<long long>(a) * nx * ny + shift) * static_cast<long long>(es);
    return cudaMemcpyAsync(dst, base + a * plane, (b - a) * plane, cudaMemcpyDefault, s);
  };
  cudaError_t e = push(h.lo, h.lo_shift, z0, std::min(z1, h.lo_end));
  if (e == cudaSuccess) e = push(h.hi, h.hi_shift, std::max(z0, h.hi_begin), z1);
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil3d_sweep_peer: push");
}

}  // namespace

// ===========================================================================
namespace {
// Device-resident direct-gather sweeps (the oracle's order and arithmetic):
// the per-cell verifier of full-size device runs (bench max_rel, GPU tests).
template <class T>
cudaError_t gather_run(T* a, T* b, int nx, int ny, int nz, const StencilDesc<T>& d, int iters,
                       cudaStream_t s, T** result) {
  const size_t bytes = static_cast<size_t>(nx) * ny * nz * sizeof(T);
  cudaError_t e = cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice, s);  // the ring
  T* cur = a;
  T* nxt = b;
  for (int it = 0; e == cudaSuccess && it < iters; ++it) {
    e = d.dims == 2 ? stencil2d_direct<T>(cur, nxt, nx, ny, 0, ny, d, s)
                    : stencil3d_direct<T>(cur, nxt, nx, ny, nz, 0, nz, d, s);
    std::swap(cur, nxt);
  }
  *result = cur;
  return e;
}

}  // namespace

namespace {
// Many independent grids through the engine with the copies overlapped:
// grid k's H2D (copy stream), sweeps (compute stream) and D2H (copy-back
// stream) run while grid k-1 is being computed / copied back, `depth` grids
// in flight, each with its own pair of device buffers.
template <class T>
int host_stencil_batch(int count, const void* const* in, void* const* out, int nx, int ny, int nz,
                       const ssam_stencil* st, int iters, int depth) {
  const size_t bytes = static_cast<size_t>(nx) * ny * nz * sizeof(T);
  const StencilDesc<T> d = make_desc<T>(st);
  const int dtype = sizeof(T) == 4 ? SSAM_DTYPE_F32 : (std::is_same<T, double>::value ? 1 : 2);
  depth = std::max(1, std::min(depth, count));
  struct Res {
    cudaStream_t s[3] = {};
    std::vector<cudaEvent_t> ev;
    std::vector<void*> buf;
    ~Res() {
      for (cudaStream_t x : s)
        if (x) cudaStreamSynchronize(x);
      for (void* p : buf)
        if (p) cudaFreeAsync(p, s[1]);
      if (s[1]) cudaStreamSynchronize(s[1]);
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
      for (cudaStream_t x : s)
        if (x) cudaStreamDestroy(x);
    }
  } r;
  cudaError_t e = cudaSuccess;
  for (cudaStream_t& x : r.s)
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  r.ev.assign(3 * depth, nullptr);
  for (cudaEvent_t& x : r.ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  r.buf.assign(2 * depth, nullptr);
  cudaMemPool_t pool = engine_pool();
  for (void*& p : r.buf)
    if (e == cudaSuccess)
      e = pool ? cudaMallocFromPoolAsync(&p, bytes, pool, r.s[1]) : cudaMallocAsync(&p, bytes, r.s[1]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(r.s[1]);
  if (e != cudaSuccess) return cuda_fail(e, "stencil batch setup");
  cudaEvent_t* ev_in = r.ev.data();            // input landed
  cudaEvent_t* ev_done = r.ev.data() + depth;  // result computed
  cudaEvent_t* ev_out = r.ev.data() + 2 * depth;  // result copied back (slot free)
  for (int k = 0; k < count && e == cudaSuccess; ++k) {
    const int sl = k % depth;
    T* a = static_cast<T*>(r.buf[2 * sl]);
    T* b = static_cast<T*>(r.buf[2 * sl + 1]);
    if (k >= depth) e = cudaStreamWaitEvent(r.s[0], ev_out[sl], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(a, in[k], bytes, cudaMemcpyHostToDevice, r.s[0]);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[sl], r.s[0]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(r.s[1], ev_in[sl], 0);
    T* res = nullptr;
    if (e == cudaSuccess)
      e = st->dims == 2 ? run2d<T>(a, b, nx, ny, d, iters, default_tb(dtype, st), r.s[1], &res)
                        : run3d<T>(a, b, nx, ny, nz, d, iters, r.s[1], &res);
    if (e == cudaSuccess) e = cudaEventRecord(ev_done[sl], r.s[1]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(r.s[2], ev_done[sl], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out[k], res, bytes, cudaMemcpyDeviceToHost, r.s[2]);
    if (e == cudaSuccess) e = cudaEventRecord(ev_out[sl], r.s[2]);
  }
  for (cudaStream_t x : r.s)
    if (e == cudaSuccess) e = cudaStreamSynchronize(x);
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil batch");
}
template <class T> struct HostBatch {
  template <class... A> static int run(A... a) { return host_stencil_batch<T>(a...); }
};
}  // namespace

extern "C" {

int ssam_b200_abi_version(void) { return SSAM_B200_ABI_VERSION; }
const char* ssam_b200_last_error(void) { return g_err.c_str(); }
uint64_t ssam_b200_launch_count(void) { return launches(); }

int ssam_b200_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void ssam_b200_default_config(ssam_kernel_config* cfg) {
  if (!cfg) return;
  cfg->p = 4;
  cfg->b = 128;
  cfg->boundary = SSAM_BOUNDARY_ZERO;
  cfg->lane_count = 32;
  cfg->threads = 0;
}

int ssam_b200_check_conv2d(int w, int h, int m, int n, const ssam_kernel_config* cfg) {
  g_err.clear();
  return check_conv2d(w, h, m, n, cfg_or_default(cfg));
}
int ssam_b200_check_stencil2d(int w, int h, const ssam_stencil* st, const ssam_kernel_config* cfg,
                              int iters) {
  g_err.clear();
  return check_stencil2d(w, h, st, cfg_or_default(cfg), iters);
}
int ssam_b200_check_stencil3d(int nx, int ny, int nz, const ssam_stencil* st,
                              const ssam_kernel_config* cfg, int iters) {
  g_err.clear();
  return check_stencil3d(nx, ny, nz, st, cfg_or_default(cfg), iters);
}

int ssam_b200_counters_conv2d(int w, int h, int m, int n, const ssam_kernel_config* cfg,
                              ssam_op_counters* counters) {
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_conv2d(w, h, m, n, c)) return s;
  if (counters) counters_conv2d(w, h, m, n, c, counters);
  return SSAM_OK;
}
int ssam_b200_counters_stencil2d(int w, int h, const ssam_stencil* st,
                                 const ssam_kernel_config* cfg, int iters,
                                 ssam_op_counters* counters) {
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil2d(w, h, st, c, iters)) return s;
  if (counters) counters_stencil2d(w, h, st, c, iters, counters);
  return SSAM_OK;
}
int ssam_b200_counters_stencil3d(int nx, int ny, int nz, const ssam_stencil* st,
                                 const ssam_kernel_config* cfg, int iters,
                                 ssam_op_counters* counters) {
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil3d(nx, ny, nz, st, c, iters)) return s;
  if (counters) counters_stencil3d(nx, ny, nz, st, c, iters, counters);
  return SSAM_OK;
}

int ssam_b200_conv2d(int dtype, const void* in, int w, int h, const void* weights, int m, int n,
                     const ssam_kernel_config* cfg, void* out, ssam_op_counters* counters) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_conv2d(w, h, m, n, c)) return s;
  if (!in || !out || !weights) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv2d: null pointer");
  if (int s = device_ready()) return s;
  const int b = c.boundary == SSAM_BOUNDARY_REPLICATE ? 1 : 0;
  if (int s = by_dtype<HostConv>(dtype, in, w, h, weights, m, n, b, out)) return s;
  if (counters) counters_conv2d(w, h, m, n, c, counters);
  return SSAM_OK;
}

int ssam_b200_stencil2d(int dtype, const void* in, int w, int h, const ssam_stencil* st,
                        const ssam_kernel_config* cfg, int iters, void* out,
                        ssam_op_counters* counters) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil2d(w, h, st, c, iters)) return s;
  if (!in || !out) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: null pointer");
  if (int s = device_ready()) return s;
  if (int s = by_dtype<HostStencil>(dtype, in, w, h, 1, st, iters, out)) return s;
  if (counters) counters_stencil2d(w, h, st, c, iters, counters);
  return SSAM_OK;
}

int ssam_b200_stencil3d(int dtype, const void* in, int nx, int ny, int nz, const ssam_stencil* st,
                        const ssam_kernel_config* cfg, int iters, void* out,
                        ssam_op_counters* counters) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil3d(nx, ny, nz, st, c, iters)) return s;
  if (!in || !out) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: null pointer");
  if (int s = device_ready()) return s;
  if (int s = by_dtype<HostStencil>(dtype, in, nx, ny, nz, st, iters, out)) return s;
  if (counters) counters_stencil3d(nx, ny, nz, st, c, iters, counters);
  return SSAM_OK;
}

int ssam_b200_measure_latency(ssam_latency_profile* out) {
  g_err.clear();
  if (!out) return fail(SSAM_ERR_INVALID_ARGUMENT, "measure_latency: null output");
  if (int s = device_ready()) return s;
  double t[8];
  const cudaError_t e = measure_latency(t, cudaStreamPerThread);
  if (e != cudaSuccess) return cuda_fail(e, "measure_latency");
  out->t_shfl = t[0];
  out->t_mad = t[1];
  out->t_smem_read = t[2];
  out->t_reg = t[3];
  out->t_gmem_read = t[4];
  out->t_gmem_write = t[5];
  out->t_l2_read = t[6];
  out->sm_clock_mhz = t[7];
  return SSAM_OK;
}

int ssam_b200_stencil2d_multi(int dtype, const void* in, int w, int h, const ssam_stencil* st,
                              const ssam_kernel_config* cfg, int iters, const int* devices,
                              int ndev, void* out, ssam_op_counters* counters, int* used) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil2d(w, h, st, c, iters)) return s;
  if (!in || !out) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: null pointer");
  if (int s = device_ready()) return s;
  if (int s = check_devices(devices, ndev)) return s;
  if (int s = by_dtype<HostStencilMulti>(dtype, in, w, h, 1, st, iters, devices, ndev, out, used))
    return s;
  if (counters) counters_stencil2d(w, h, st, c, iters, counters);
  return SSAM_OK;
}

int ssam_b200_stencil3d_multi(int dtype, const void* in, int nx, int ny, int nz,
                              const ssam_stencil* st, const ssam_kernel_config* cfg, int iters,
                              const int* devices, int ndev, void* out, ssam_op_counters* counters,
                              int* used) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_stencil3d(nx, ny, nz, st, c, iters)) return s;
  if (!in || !out) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: null pointer");
  if (int s = device_ready()) return s;
  if (int s = check_devices(devices, ndev)) return s;
  if (int s = by_dtype<HostStencilMulti>(dtype, in, nx, ny, nz, st, iters, devices, ndev, out, used))
    return s;
  if (counters) counters_stencil3d(nx, ny, nz, st, c, iters, counters);
  return SSAM_OK;
}

int ssam_b200_stencil_batch(int dtype, int count, const void* const* in, void* const* out, int nx,
                            int ny, int nz, const ssam_stencil* st, int iters, int depth) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims == 2) nz = 1;
  const int m = 2 * st->order + 1;
  if (count < 0 || !in || !out || iters < 0 || nx < m || ny < m || (st->dims == 3 && nz < m))
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil_batch: bad arguments");
  for (int k = 0; k < count; ++k)
    if (!in[k] || !out[k]) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil_batch: null grid");
  if (count == 0) return SSAM_OK;
  if (int s = device_ready()) return s;
  return by_dtype<HostBatch>(dtype, count, in, out, nx, ny, nz, st, iters, depth <= 0 ? 2 : depth);
}

int ssam_b200_benchmark_count(void) { return kNumBench; }
const char* ssam_b200_benchmark_name(int i) {
  return (i >= 0 && i < kNumBench) ? kBench[i].name : nullptr;
}

int ssam_b200_benchmark_stencil(const char* name, int* dims, int* order, int* fpp, int* offsets,
                                double* coeffs, int cap) {
  const BenchDef* d = nullptr;
  for (const BenchDef& b : kBench)
    if (name && std::strcmp(name, b.name) == 0) d = &b;
  if (!d) {
    g_err = std::string("unknown stencil benchmark: ") + (name ? name : "(null)");
    return -1;
  }
  std::vector<std::array<int, 3>> offs;
  switch (d->shape) {
    case 's': offs = star_set(d->order, d->dims); break;
    case 'b': offs = box_set(d->order, d->dims); break;
    case 'p': offs = poisson_set(); break;
    default:
      for (int dy = -4; dy <= 3; ++dy)
        for (int dx = -4; dx <= 3; ++dx) offs.push_back({dx, dy, 0});
  }
  // Canonical order: (dz, dy, dx) ascending; the centre goes last.
  std::sort(offs.begin(), offs.end(), [](const auto& a, const auto& b) {
    return std::make_tuple(a[2], a[1], a[0]) < std::make_tuple(b[2], b[1], b[0]);
  });
  const int n = static_cast<int>(offs.size());
  if (n > cap) return -2;
  const int t = n - 1;
  const double denom = 2.0 * (static_cast<double>(t) * (t + 1) / 2.0);
  int out = 0, j = 0;
  for (const auto& o : offs) {
    if (o == std::array<int, 3>{0, 0, 0}) continue;
    ++j;
    std::memcpy(offsets + 3 * out, o.data(), 3 * sizeof(int));
    coeffs[out++] = t > 0 ? static_cast<double>(j) / denom : 0.0;
  }
  offsets[3 * out] = offsets[3 * out + 1] = offsets[3 * out + 2] = 0;
  coeffs[out++] = 0.5 + (t == 0 ? 0.5 : 0.0);
  *dims = d->dims;
  *order = d->order;
  *fpp = d->fpp;
  return out;
}

// ---- device-resident entry points ------------------------------------------------

int ssam_b200_conv2d_device(int dtype, const void* d_in, void* d_out, int w, int h, int y_begin,
                            int y_end, const void* h_weights, int m, int n, int boundary,
                            void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (m < 1 || n < 1 || m > 20 || n > 20 || w < 1 || h < 1)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "conv2d_device: bad shape");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = conv2d_device<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), w, h, y_begin, y_end, static_cast<const float*>(h_weights), m, n, boundary, s); break;
    case 1: e = conv2d_device<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), w, h, y_begin, y_end, static_cast<const double*>(h_weights), m, n, boundary, s); break;
    case 2: e = conv2d_device<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), w, h, y_begin, y_end, static_cast<const long long*>(h_weights), m, n, boundary, s); break;
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "conv2d_device");
}

int ssam_b200_stencil2d_sweep(int dtype, const void* d_in, void* d_out, int w, int h, int y_begin,
                              int y_end, const ssam_stencil* st, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 2) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: needs a 2D stencil");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = stencil2d_sweep<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), w, h, y_begin, y_end, make_desc<float>(st), s); break;
    case 1: e = stencil2d_sweep<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), w, h, y_begin, y_end, make_desc<double>(st), s); break;
    case 2: e = stencil2d_sweep<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), w, h, y_begin, y_end, make_desc<long long>(st), s); break;
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil2d_sweep");
}

int ssam_b200_stencil2d_tb(int dtype, const void* d_in, void* d_out, int w, int h,
                           const ssam_stencil* st, int tb, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 2) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: needs a 2D stencil");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = stencil2d_tb<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), w, h, make_desc<float>(st), tb, s); break;
    case 1: e = stencil2d_tb<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), w, h, make_desc<double>(st), tb, s); break;
    case 2: e = stencil2d_tb<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), w, h, make_desc<long long>(st), tb, s); break;
  }
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d_tb: no fused kernel for this case");
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil2d_tb");
}

int ssam_b200_stencil2d_tb_range(int dtype, const void* d_in, void* d_out, int w, int h,
                                 int y_begin, int y_end, int y_ring_lo, int y_ring_hi,
                                 const ssam_stencil* st, int tb, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 2) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: needs a 2D stencil");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = stencil2d_tb_range<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), w, h, y_begin, y_end, y_ring_lo, y_ring_hi, make_desc<float>(st), tb, s); break;
    case 1: e = stencil2d_tb_range<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), w, h, y_begin, y_end, y_ring_lo, y_ring_hi, make_desc<double>(st), tb, s); break;
    case 2: e = stencil2d_tb_range<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), w, h, y_begin, y_end, y_ring_lo, y_ring_hi, make_desc<long long>(st), tb, s); break;
  }
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d_tb_range: no fused kernel for this case");
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil2d_tb_range");
}

int ssam_b200_stencil2d_tb_max(int dtype, const ssam_stencil* st) {
  if (!st || st->dims != 2 || !dtype_ok(dtype)) return 1;
  std::vector<Tap> taps;
  for (int i = 0; i < st->ntaps; ++i)
    taps.push_back({st->offsets[3 * i], st->offsets[3 * i + 1], st->offsets[3 * i + 2]});
  return stencil2d_tb_max(dtype, st->order, classify2d(taps, st->order) == Shape2D::star);
}

int ssam_b200_stencil3d_sweep(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                              int z_begin, int z_end, const ssam_stencil* st, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 3) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: needs a 3D stencil");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = stencil3d_sweep<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), nx, ny, nz, z_begin, z_end, make_desc<float>(st), s); break;
    case 1: e = stencil3d_sweep<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), nx, ny, nz, z_begin, z_end, make_desc<double>(st), s); break;
    case 2: e = stencil3d_sweep<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), nx, ny, nz, z_begin, z_end, make_desc<long long>(st), s); break;
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil3d_sweep");
}

int ssam_b200_stencil2d_run(int dtype, void* d_a, void* d_b, int w, int h, const ssam_stencil* st,
                            int iters, int tb, void* stream, void** d_result) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 2) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: needs a 2D stencil");
  if (iters < 0) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d: iters must be >= 0");
  if (!d_a || !d_b || !d_result || d_a == d_b)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d_run: null or aliased buffer");
  if (w < 2 * st->order + 1 || h < 2 * st->order + 1)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil2d_run: domain smaller than 2k+1");
  if (int s = device_ready()) return s;
  if (tb <= 0) tb = default_tb(dtype, st);
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  void* r = nullptr;
  switch (dtype) {
    case 0: { float* q = nullptr; e = run2d<float>(static_cast<float*>(d_a), static_cast<float*>(d_b), w, h, make_desc<float>(st), iters, tb, s, &q); r = q; break; }
    case 1: { double* q = nullptr; e = run2d<double>(static_cast<double*>(d_a), static_cast<double*>(d_b), w, h, make_desc<double>(st), iters, tb, s, &q); r = q; break; }
    case 2: { long long* q = nullptr; e = run2d<long long>(static_cast<long long*>(d_a), static_cast<long long*>(d_b), w, h, make_desc<long long>(st), iters, tb, s, &q); r = q; break; }
  }
  if (e != cudaSuccess) return cuda_fail(e, "stencil2d_run");
  *d_result = r;
  return SSAM_OK;
}

int ssam_b200_stencil3d_run(int dtype, void* d_a, void* d_b, int nx, int ny, int nz,
                            const ssam_stencil* st, int iters, void* stream, void** d_result) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 3) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: needs a 3D stencil");
  if (iters < 0) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: iters must be >= 0");
  if (!d_a || !d_b || !d_result || d_a == d_b)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d_run: null or aliased buffer");
  const int m = 2 * st->order + 1;
  if (nx < m || ny < m || nz < m)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d_run: domain smaller than 2k+1");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  void* r = nullptr;
  switch (dtype) {
    case 0: { float* q = nullptr; e = run3d<float>(static_cast<float*>(d_a), static_cast<float*>(d_b), nx, ny, nz, make_desc<float>(st), iters, s, &q); r = q; break; }
    case 1: { double* q = nullptr; e = run3d<double>(static_cast<double*>(d_a), static_cast<double*>(d_b), nx, ny, nz, make_desc<double>(st), iters, s, &q); r = q; break; }
    case 2: { long long* q = nullptr; e = run3d<long long>(static_cast<long long*>(d_a), static_cast<long long*>(d_b), nx, ny, nz, make_desc<long long>(st), iters, s, &q); r = q; break; }
  }
  if (e != cudaSuccess) return cuda_fail(e, "stencil3d_run");
  *d_result = r;
  return SSAM_OK;
}

int ssam_b200_gather_stencil_run(int dtype, void* d_a, void* d_b, int nx, int ny, int nz,
                                 const ssam_stencil* st, int iters, void* stream,
                                 void** d_result) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims == 2) nz = 1;
  if (nx < 1 || ny < 1 || nz < 1 || iters < 0 || !d_a || !d_b || !d_result || d_a == d_b)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "gather_stencil_run: bad arguments");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  void* r = nullptr;
  switch (dtype) {
    case 0: { float* q = nullptr; e = gather_run<float>(static_cast<float*>(d_a), static_cast<float*>(d_b), nx, ny, nz, make_desc<float>(st), iters, s, &q); r = q; break; }
    case 1: { double* q = nullptr; e = gather_run<double>(static_cast<double*>(d_a), static_cast<double*>(d_b), nx, ny, nz, make_desc<double>(st), iters, s, &q); r = q; break; }
    case 2: { long long* q = nullptr; e = gather_run<long long>(static_cast<long long*>(d_a), static_cast<long long*>(d_b), nx, ny, nz, make_desc<long long>(st), iters, s, &q); r = q; break; }
  }
  if (e != cudaSuccess) return cuda_fail(e, "gather_stencil_run");
  *d_result = r;
  return SSAM_OK;
}

int ssam_b200_trim_cache(void) {
  g_err.clear();
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (cudaMemPool_t p : g_pools)
    if (p && cudaMemPoolTrimTo(p, 0) != cudaSuccess) return cuda_fail(cudaGetLastError(), "trim_cache");
  return SSAM_OK;
}

int ssam_b200_fill_random(int dtype, void* d_out, size_t count, uint64_t seed, uint64_t first,
                          void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = device_ready()) return s;
  const cudaError_t e = fill_random(dtype, d_out, count, seed, first, as_stream(stream));
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "fill_random");
}

int ssam_b200_max_rel_err(int dtype, const void* d_a, const void* d_b, size_t count,
                          double* max_rel, double* max_abs, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = device_ready()) return s;
  double r = 0, a = 0;
  const cudaError_t e = max_rel_err(dtype, d_a, d_b, count, &r, &a, as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "max_rel_err");
  if (max_rel) *max_rel = r;
  if (max_abs) *max_abs = a;
  return SSAM_OK;
}

// ---- 1D entry points (kernels.hpp:390-447) ----------------------------------------
int ssam_b200_check_conv1d(long long len, int m, const ssam_kernel_config* cfg) {
  g_err.clear();
  return check_conv1d(len, m, cfg_or_default(cfg));
}
int ssam_b200_check_scan(unsigned long long len, int lane_count) {
  g_err.clear();
  return check_scan(len, lane_count);
}
int ssam_b200_counters_conv1d(long long len, int m, const ssam_kernel_config* cfg,
                              ssam_op_counters* counters) {
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_conv1d(len, m, c)) return s;
  if (counters) counters_conv1d(len, m, c, counters);
  return SSAM_OK;
}
int ssam_b200_counters_scan(unsigned long long len, int lane_count, ssam_op_counters* counters) {
  if (int s = check_scan(len, lane_count)) return s;
  if (counters) counters_scan(len, lane_count, counters);
  return SSAM_OK;
}

int ssam_b200_conv1d(int dtype, const void* in, long long len, const void* weights, int m,
                     const ssam_kernel_config* cfg, void* out, ssam_op_counters* counters) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  const ssam_kernel_config c = cfg_or_default(cfg);
  if (int s = check_conv1d(len, m, c)) return s;
  if (len > 0x7fffffffLL) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv1d: signal too long");
  if (!in || !out || !weights) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv1d: null pointer");
  if (int s = device_ready()) return s;
  const int b = c.boundary == SSAM_BOUNDARY_REPLICATE ? 1 : 0;
  if (int s = by_dtype<HostConv1>(dtype, in, static_cast<int>(len), weights, m, b, out)) return s;
  if (counters) counters_conv1d(len, m, c, counters);
  return SSAM_OK;
}

int ssam_b200_scan(int dtype, const void* in, unsigned long long len, int lane_count, void* out,
                   ssam_op_counters* counters) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = check_scan(len, lane_count)) return s;
  if (len == 0) return SSAM_OK;
  if (!in || !out) return fail(SSAM_ERR_INVALID_ARGUMENT, "scan: null pointer");
  if (int s = device_ready()) return s;
  if (int s = by_dtype<HostScan>(dtype, in, static_cast<size_t>(len), out)) return s;
  if (counters) counters_scan(len, lane_count, counters);
  return SSAM_OK;
}

int ssam_b200_conv1d_device(int dtype, const void* d_in, void* d_out, int len,
                            const void* h_weights, int m, int boundary, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (m < 1 || m > 32 || len < 0) return fail(SSAM_ERR_INVALID_ARGUMENT, "conv1d_device: bad shape");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = conv1d_device<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), len, static_cast<const float*>(h_weights), m, boundary, s); break;
    case 1: e = conv1d_device<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), len, static_cast<const double*>(h_weights), m, boundary, s); break;
    case 2: e = conv1d_device<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), len, static_cast<const long long*>(h_weights), m, boundary, s); break;
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "conv1d_device");
}

int ssam_b200_scan_device(int dtype, const void* d_in, void* d_out, size_t len, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorInvalidValue;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = scan_device<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), len, s); break;
    case 1: e = scan_device<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), len, s); break;
    case 2: e = scan_device<long long>(static_cast<const long long*>(d_in), static_cast<long long*>(d_out), len, s); break;
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "scan_device");
}

// ---- direct-gather verifier (oracle arithmetic on the GPU) -----------------------
int ssam_b200_gather_conv2d(int dtype, const void* in, int w, int h, const void* weights, int m,
                            int n, int boundary, void* out) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (w < 1 || h < 1 || m < 1 || n < 1 || !in || !out || !weights)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "gather_conv2d: bad arguments");
  if (int s = device_ready()) return s;
  return by_dtype<HostGather>(dtype, 0, in, w, h, 1, weights, m, n, boundary,
                              static_cast<const ssam_stencil*>(nullptr), 0, out);
}

int ssam_b200_gather_stencil(int dtype, const void* in, int nx, int ny, int nz,
                             const ssam_stencil* st, int iters, void* out) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (nx < 1 || ny < 1 || nz < 1 || iters < 0 || !in || !out)
    return fail(SSAM_ERR_INVALID_ARGUMENT, "gather_stencil: bad arguments");
  if (int s = device_ready()) return s;
  return by_dtype<HostGather>(dtype, 1, in, nx, ny, st->dims == 2 ? 1 : nz,
                              static_cast<const void*>(nullptr), 0, 0, 0, st, iters, out);
}

int ssam_b200_stencil3d_tb(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                           int z_begin, int z_end, int z_ring_lo, int z_ring_hi,
                           const ssam_stencil* st, int tb, void* stream) {
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  if (st->dims != 3) return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d: needs a 3D stencil");
  if (int s = device_ready()) return s;
  cudaError_t e = cudaErrorNotSupported;
  const cudaStream_t s = as_stream(stream);
  switch (dtype) {
    case 0: e = stencil3d_tb<float>(static_cast<const float*>(d_in), static_cast<float*>(d_out), nx, ny, nz, z_begin, z_end, z_ring_lo, z_ring_hi, make_desc<float>(st), tb, s); break;
    case 1: e = stencil3d_tb<double>(static_cast<const double*>(d_in), static_cast<double*>(d_out), nx, ny, nz, z_begin, z_end, z_ring_lo, z_ring_hi, make_desc<double>(st), tb, s); break;
    default: break;
  }
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    return fail(SSAM_ERR_INVALID_ARGUMENT, "stencil3d_tb: no fused kernel for this case");
  }
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "stencil3d_tb");
}

int ssam_b200_stencil3d_tb_max(int dtype, const ssam_stencil* st) {
  if (!st || st->dims != 3 || !dtype_ok(dtype)) return 1;
  std::vector<Tap> taps;
  for (int i = 0; i < st->ntaps; ++i)
    taps.push_back({st->offsets[3 * i], st->offsets[3 * i + 1], st->offsets[3 * i + 2]});
  return stencil3d_tb_max(dtype, st->order, classify3d(taps, st->order));
}

int ssam_b200_stencil3d_sweep_peer(int dtype, const void* d_in, void* d_out, int nx, int ny,
                                   int nz, int z_begin, int z_end, const ssam_stencil* st,
                                   const ssam_peer_halo* peer, void* stream) {
  if (!peer) return ssam_b200_stencil3d_sweep(dtype, d_in, d_out, nx, ny, nz, z_begin, z_end, st, stream);
  g_err.clear();
  if (!dtype_ok(dtype)) return fail(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (int s = validate_stencil(st)) return s;
  const PeerHalo h = to_peer(peer);
  int rc;
  {
    PeerScope scope(&h);
    rc = ssam_b200_stencil3d_sweep(dtype, d_in, d_out, nx, ny, nz, z_begin, z_end, st, stream);
  }
  if (rc != SSAM_OK || stencil3d_peer_fused(dtype, st->order)) return rc;
  // direct-gather kernel (order > 2): push the boundary planes after it
  return push_planes(dtype, d_out, nx, ny, std::max(z_begin, st->order),
                     std::min(z_end, nz - st->order), h, as_stream(stream));
}

int ssam_b200_stencil3d_tb_peer(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                                int z_begin, int z_end, int z_ring_lo, int z_ring_hi,
                                const ssam_stencil* st, int tb, const ssam_peer_halo* peer,
                                void* stream) {
  if (!peer)
    return ssam_b200_stencil3d_tb(dtype, d_in, d_out, nx, ny, nz, z_begin, z_end, z_ring_lo,
                                  z_ring_hi, st, tb, stream);
  const PeerHalo h = to_peer(peer);
  PeerScope scope(&h);
  return ssam_b200_stencil3d_tb(dtype, d_in, d_out, nx, ny, nz, z_begin, z_end, z_ring_lo,
                                z_ring_hi, st, tb, stream);
}

static_assert(sizeof(cudaIpcMemHandle_t) == SSAM_IPC_HANDLE_BYTES, "IPC handle size");

int ssam_b200_ipc_alloc(size_t bytes, void** d_ptr, void* handle) {
  g_err.clear();
  if (!d_ptr || !handle || bytes == 0) return fail(SSAM_ERR_INVALID_ARGUMENT, "ipc_alloc: bad argument");
  if (int s = device_ready()) return s;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "ipc_alloc");
  cudaIpcMemHandle_t hd;
  e = cudaIpcGetMemHandle(&hd, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "ipc_alloc: handle");
  }
  std::memcpy(handle, &hd, sizeof(hd));
  *d_ptr = p;
  return SSAM_OK;
}

int ssam_b200_ipc_free(void* d_ptr) {
  g_err.clear();
  const cudaError_t e = cudaFree(d_ptr);
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "ipc_free");
}

int ssam_b200_ipc_open(const void* handle, void** d_ptr) {
  g_err.clear();
  if (!d_ptr || !handle) return fail(SSAM_ERR_INVALID_ARGUMENT, "ipc_open: bad argument");
  if (int s = device_ready()) return s;
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  const cudaError_t e = cudaIpcOpenMemHandle(d_ptr, hd, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "ipc_open");
}

int ssam_b200_ipc_close(void* d_ptr) {
  g_err.clear();
  const cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? SSAM_OK : cuda_fail(e, "ipc_close");
}

// ---- stream memory operations (peer-halo generation flags) -------------------
// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry points: the GPU front end performs the write after the stream's
// prior work (with a memory barrier, so the kernel's peer stores are visible
// first) and holds the stream until a 32-bit word reaches a value -- no SM
// and no host round trip.
}  // extern "C"
namespace {
using WriteValueFn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
using WaitValueFn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<F>(p);
}
WriteValueFn write_value_fn() {
  static WriteValueFn f = driver_fn<WriteValueFn>("cuStreamWriteValue32");
  return f;
}
WaitValueFn wait_value_fn() {
  static WaitValueFn f = driver_fn<WaitValueFn>("cuStreamWaitValue32");
  return f;
}
constexpr unsigned kWaitGeq = 0x0;  // CU_STREAM_WAIT_VALUE_GEQ
}  // namespace
extern "C" {

int ssam_b200_stream_write_u32(void* d_addr, uint32_t value, void* stream) {
  g_err.clear();
  if (!d_addr) return fail(SSAM_ERR_INVALID_ARGUMENT, "stream_write_u32: null address");
  if (int s = device_ready()) return s;
  WriteValueFn f = write_value_fn();
  if (!f) return fail(SSAM_ERR_CUDA, "stream_write_u32: cuStreamWriteValue32 unavailable");
  const int r = f(as_stream(stream), reinterpret_cast<unsigned long long>(d_addr), value, 0);
  return r == 0 ? SSAM_OK : fail(SSAM_ERR_CUDA, "cuStreamWriteValue32 failed: " + std::to_string(r));
}

int ssam_b200_stream_wait_u32(const void* d_addr, uint32_t value, void* stream) {
  g_err.clear();
  if (!d_addr) return fail(SSAM_ERR_INVALID_ARGUMENT, "stream_wait_u32: null address");
  if (int s = device_ready()) return s;
  WaitValueFn f = wait_value_fn();
  if (!f) return fail(SSAM_ERR_CUDA, "stream_wait_u32: cuStreamWaitValue32 unavailable");
  const int r = f(as_stream(stream), reinterpret_cast<unsigned long long>(d_addr), value, kWaitGeq);
  return r == 0 ? SSAM_OK : fail(SSAM_ERR_CUDA, "cuStreamWaitValue32 failed: " + std::to_string(r));
}

}  // extern "C"
