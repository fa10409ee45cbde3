// latency.cu -- a measured B200 LatencyProfile for the reference's perf
// model (proj/include/ssam/perf_model.hpp:14-26, builtin P100/V100 values at
// proj/src/perf_model.cpp:22-39, "from micro-benchmark measurements").
//
// Each field is the latency in SM cycles of one warp instruction on a
// dependent chain (one warp, clock64 around 64 x 256 chained operations):
//   t_mad        fma.rn.f32 x = x * a + b
//   t_shfl       shfl.sync.idx.b32 of the value just shuffled
//   t_smem_read  ld.shared.u32 pointer chase (each lane its own bank)
//   t_reg        not measurable in isolation; the reference's 1
//   t_gmem_read  ld.global.cg pointer chase, each step one coalesced 128-byte
//                line (lane l reads word l), random lines over a 256 MiB
//                buffer (> the 126 MB L2: HBM latency)
//   t_gmem_write st.global.wt + fence.acq_rel.gpu per step (the store
//                reaching device scope)
// plus, for reference, t_l2_read: the same chase over 16 MiB (L2 hits).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace ssam_b200 {

namespace {

constexpr int kUnroll = 64;
constexpr int kIters = 256;
constexpr int kOps = kUnroll * kIters;

#define SSAM_REP64(X) X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X \
                      X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X X

__global__ void lat_alu_kernel(float a, float b, long long* cycles, float* sink) {
  float x = threadIdx.x;
  int y = threadIdx.x;
  __shared__ uint32_t chase[32 * 64];
  // smem chain: lane l walks words l, l+32, ... (no bank conflicts)
  for (int i = threadIdx.x; i < 32 * 64; i += 32)
    chase[i] = static_cast<uint32_t>(__cvta_generic_to_shared(&chase[(i + 32) % (32 * 64)]));
  __syncwarp();
  uint32_t p = static_cast<uint32_t>(__cvta_generic_to_shared(&chase[threadIdx.x]));

  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
    SSAM_REP64(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(b));)
  }
  long long t1 = clock64();
  for (int i = 0; i < kIters; ++i) {
    SSAM_REP64(asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(y) : "r"(31 - (int)threadIdx.x));)
  }
  long long t2 = clock64();
  for (int i = 0; i < kIters; ++i) {
    SSAM_REP64(asm volatile("ld.shared.u32 %0, [%0];" : "+r"(p) : : "memory");)
  }
  long long t3 = clock64();
  if (threadIdx.x == 0) {
    cycles[0] = t1 - t0;
    cycles[1] = t2 - t1;
    cycles[2] = t3 - t2;
  }
  sink[threadIdx.x] = x + static_cast<float>(y) + static_cast<float>(p);
}

// Global chase: node k occupies words [32 k, 32 k + 32); word 32 k + l holds
// the element index of lane l's word in the next node.
__global__ void lat_gmem_kernel(const uint32_t* __restrict__ next, int steps, long long* cycles,
                                uint32_t* sink) {
  uint32_t i = threadIdx.x;
  // warm the TLB / first touch of the start line
  i = __ldcg(next + i);
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  sink[threadIdx.x] = i;
}

__global__ void lat_store_kernel(uint32_t* buf, int steps, long long* cycles) {
  uint32_t* q = buf + threadIdx.x;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    asm volatile("st.global.wt.u32 [%0], %1;" ::"l"(q), "r"(s) : "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

cudaError_t chase_latency(size_t bytes, int steps, uint64_t seed, cudaStream_t s, double* out) {
  const size_t nodes = bytes / 128;
  std::vector<uint32_t> order(nodes);
  std::iota(order.begin(), order.end(), 0u);
  std::mt19937_64 rng(seed);
  std::shuffle(order.begin(), order.end(), rng);
  std::vector<uint32_t> h(nodes * 32);
  for (size_t k = 0; k < nodes; ++k) {
    const uint32_t from = order[k], to = order[(k + 1) % nodes];
    for (uint32_t l = 0; l < 32; ++l) h[static_cast<size_t>(from) * 32 + l] = to * 32 + l;
  }
  uint32_t* d = nullptr;
  long long* dc = nullptr;
  uint32_t* sink = nullptr;
  cudaError_t e = cudaMalloc(&d, h.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&dc, sizeof(long long));
  if (e == cudaSuccess) e = cudaMalloc(&sink, 32 * sizeof(uint32_t));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
  long long cyc = 0;
  if (e == cudaSuccess) {
    lat_gmem_kernel<<<1, 32, 0, s>>>(d, steps, dc, sink);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (d) cudaFree(d);
  if (dc) cudaFree(dc);
  if (sink) cudaFree(sink);
  *out = static_cast<double>(cyc) / steps;
  return e;
}

}  // namespace

cudaError_t measure_latency(double* t /* [8] */, cudaStream_t s) {
  long long* dc = nullptr;
  float* sink = nullptr;
  uint32_t* buf = nullptr;
  cudaError_t e = cudaMalloc(&dc, 4 * sizeof(long long));
  if (e == cudaSuccess) e = cudaMalloc(&sink, 32 * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&buf, 32 * sizeof(uint32_t));
  long long c[4] = {0, 0, 0, 0};
  if (e == cudaSuccess) {
    // warm-up launch, then the measured one
    for (int rep = 0; rep < 2 && e == cudaSuccess; ++rep) {
      lat_alu_kernel<<<1, 32, 0, s>>>(1.0000001f, 1e-7f, dc, sink);
      note_launch();
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(c, dc, 3 * sizeof(long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  const int wsteps = 4096;
  if (e == cudaSuccess) {
    for (int rep = 0; rep < 2 && e == cudaSuccess; ++rep) {
      lat_store_kernel<<<1, 32, 0, s>>>(buf, wsteps, dc + 3);
      note_launch();
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(c + 3, dc + 3, sizeof(long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  double hbm = 0, l2 = 0;
  if (e == cudaSuccess) e = chase_latency(size_t(256) << 20, 8192, 7, s, &hbm);
  if (e == cudaSuccess) e = chase_latency(size_t(16) << 20, 8192, 9, s, &l2);
  if (dc) cudaFree(dc);
  if (sink) cudaFree(sink);
  if (buf) cudaFree(buf);
  if (e != cudaSuccess) return e;
  t[0] = static_cast<double>(c[1]) / kOps;  // t_shfl
  t[1] = static_cast<double>(c[0]) / kOps;  // t_mad
  t[2] = static_cast<double>(c[2]) / kOps;  // t_smem_read
  t[3] = 1.0;                               // t_reg
  t[4] = hbm;                               // t_gmem_read
  t[5] = static_cast<double>(c[3]) / wsteps;  // t_gmem_write
  t[6] = l2;                                // t_l2_read
  int dev = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  t[7] = khz / 1000.0;
  return cudaSuccess;
}

}  // namespace ssam_b200
