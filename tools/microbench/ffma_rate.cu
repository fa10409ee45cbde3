// FP32 FMA issue-rate micro-benchmark (B200): 3-register FFMA, FFMA with a
// uniform-register (kernel-parameter) operand, and packed FFMA2.  Each
// thread runs 8 independent chains; 4 warps per SMSP; prints FMAs per clock
// per SM.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma_rate.cu -o /tmp/ffma && /tmp/ffma
#include <cstdio>
#include <cstring>
constexpr int ITERS = 4096;

__global__ void ffma_reg(float* out, float a0, float b0) {
  float x[8], a = a0 + threadIdx.x * 1e-9f, b = b0 - threadIdx.x * 1e-9f;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(a), "f"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
__global__ void ffma_ur(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);  // a, b uniform (kernel params)
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}
__global__ void ffma2(float* out, float a0, float b0) {
  unsigned long long x[4], a, b;
  float2 af = make_float2(a0, a0), bf = make_float2(b0, b0);
  memcpy(&a, &af, 8); memcpy(&b, &bf, 8);
  for (int i = 0; i < 4; ++i) { float2 v = make_float2(threadIdx.x + i, threadIdx.x - i); memcpy(&x[i], &v, 8); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(a), "l"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 4; ++i) { float2 v; memcpy(&v, &x[i], 8); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (float)(t1 - t0);
}

int main() {
  float* d; cudaMalloc(&d, (1 << 20) * 4 + 64);
  const int blocks = 148, threads = 512;  // 16 warps per SM
  auto run = [&](auto kern, const char* name) {
    kern<<<blocks, threads>>>(d, 1.0000001f, 1e-7f);
    kern<<<blocks, threads>>>(d, 1.0000001f, 1e-7f);
    cudaDeviceSynchronize();
    float cyc; cudaMemcpy(&cyc, d + (1 << 20), 4, cudaMemcpyDeviceToHost);
    const double fmas = double(threads) * ITERS * 8;  // per SM (one block per SM)
    printf("%-10s %.1f FMA/clk/SM (%.0f cycles)\n", name, fmas / cyc, cyc);
  };
  run(ffma_reg, "FFMA-reg");
  run(ffma_ur, "FFMA-ur");
  run(ffma2, "FFMA2");
  return 0;
}
