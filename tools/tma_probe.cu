// Standalone probe of 2D tiled TMA behaviours the SSAM loaders rely on:
// tensor map in a __grid_constant__ parameter, unaligned / negative box
// origins, out-of-bounds zero fill.  nvcc -arch=sm_100a tools/tma_probe.cu -o /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_1907_06154_b200/csrc/common.cuh"

using namespace ssam_b200;

struct alignas(64) P {
  CUtensorMap map;
  float* out;
  int x, y, prefetch;
};

__global__ void probe(const __grid_constant__ P p) {
  __shared__ __align__(128) float buf[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    if (p.prefetch) prefetch_tmap(&p.map);
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar), sizeof(buf));
    tma_load_2d(smem_u32(buf), &p.map, p.x, p.y, smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  for (int i = threadIdx.x; i < 4 * 64; i += blockDim.x) p.out[i] = buf[i];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int W = 256, H = 16;
  std::vector<float> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  float *d, *o;
  cudaMalloc(&d, W * H * 4);
  cudaMalloc(&o, 4 * 64 * 4);
  cudaMemcpy(d, h.data(), W * H * 4, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn fn = (EncodeFn)fnp;
  P p;
  memset(&p, 0, sizeof(p));
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {64, 4};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&p.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d\n", (int)r);
  p.out = o;
  struct Case { int x, y, pf; } cases[] = {{0, 0, 0}, {0, 0, 1}, {4, 2, 0}, {3, 2, 0}, {-7, 0, 0},
                                          {-1, -2, 0}, {250, 14, 0}};
  for (auto c : cases) {
    p.x = c.x;
    p.y = c.y;
    p.prefetch = c.pf;
    probe<<<1, 128>>>(p);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(256);
    if (e == cudaSuccess) cudaMemcpy(got.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 4 && e == cudaSuccess; ++rr)
      for (int cc = 0; cc < 64; ++cc) {
        const int x = c.x + cc, y = c.y + rr;
        const float want = (x >= 0 && x < W && y >= 0 && y < H) ? h[y * W + x] : 0.f;
        bad += got[rr * 64 + cc] != want;
      }
    printf("x=%d y=%d pf=%d -> %s bad=%d\n", c.x, c.y, c.pf, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
