// grid_io.cpp -- SGRD grid files straight to / from device buffers.
//
// The format is the reference's (proj/include/ssam/grid_io.hpp:14-23): a
// 16-byte header -- "SGRD", version 1, rank (1..3), scalar code (1 f32,
// 2 f64, 3 i64), reserved, three little-endian u16 dims (d0 fastest, unused
// = 1), reserved -- then the raw little-endian scalars in storage order.
// Error conditions follow its readers and writers: dims > 65535 is an
// invalid_argument (write_header, :45-47); bad magic / truncated header,
// version, rank, scalar type and truncated payload are runtime_errors
// (read_header :58-66, read_scalars :81-85), as is an unopenable file.
//
// B200 side: a grid of a 2048 x 2048 x 512 slab is 8 GiB, so the payload is
// streamed through two pinned staging buffers: while one chunk is copied
// host->device (or device->host) on the caller's stream, the next one is
// read from (written to) the file.  Host destinations skip the staging.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "ssam_b200.h"

namespace ssam_b200 {
int set_error(int status, const std::string& msg);  // abi.cpp
}

namespace {

using ssam_b200::set_error;

constexpr size_t kChunk = size_t(64) << 20;  // 64 MiB per staging buffer

int elem_size(int dtype) { return dtype == SSAM_DTYPE_F32 ? 4 : 8; }
int scalar_code(int dtype) { return dtype + 1; }  // f32 1, f64 2, i64 3

struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(path ? std::fopen(path, mode) : nullptr) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaError_t init() {
    for (int i = 0; i < 2; ++i) {
      cudaError_t e = cudaMallocHost(&p[i], kChunk);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
};

int read_header(FILE* f, int& rank, int& dtype, int dims[3]) {
  unsigned char h[16];
  if (std::fread(h, 1, 16, f) != 16 || std::memcmp(h, "SGRD", 4) != 0)
    return set_error(SSAM_ERR_RUNTIME, "grid io: bad magic or truncated header");
  if (h[4] != 1) return set_error(SSAM_ERR_RUNTIME, "grid io: unsupported format version");
  rank = h[5];
  dtype = static_cast<int>(h[6]) - 1;
  for (int i = 0; i < 3; ++i) dims[i] = h[8 + 2 * i] | (h[9 + 2 * i] << 8);
  return SSAM_OK;
}

}  // namespace

extern "C" {

int ssam_b200_sgrd_info(const char* path, int* rank, int* dtype, int* dims) {
  File f(path, "rb");
  if (!f.f) return set_error(SSAM_ERR_RUNTIME, std::string("grid io: cannot open ") + (path ? path : ""));
  int r = 0, d = 0, dm[3];
  if (int s = read_header(f.f, r, d, dm)) return s;
  if (rank) *rank = r;
  if (dtype) *dtype = d;
  if (dims) std::memcpy(dims, dm, sizeof dm);
  return SSAM_OK;
}

int ssam_b200_sgrd_read(const char* path, int dtype, int rank, int* dims, void* dst,
                        size_t capacity, int on_device, void* stream) {
  if (dtype < 0 || dtype > 2) return set_error(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  File f(path, "rb");
  if (!f.f) return set_error(SSAM_ERR_RUNTIME, std::string("grid io: cannot open ") + (path ? path : ""));
  int r = 0, d = 0, dm[3];
  if (int s = read_header(f.f, r, d, dm)) return s;
  if (r != rank) return set_error(SSAM_ERR_RUNTIME, "grid io: rank mismatch");
  if (d != dtype) return set_error(SSAM_ERR_RUNTIME, "grid io: scalar type mismatch");
  if (dims) std::memcpy(dims, dm, sizeof dm);
  // read_grid2d / read_grid3d construct the grid before the payload, and the
  // Grid2D / Grid3D constructors reject empty dimensions (grid.hpp:20, :38)
  if (rank == 2 && (dm[0] < 1 || dm[1] < 1))
    return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid2d: dimensions must be >= 1");
  if (rank == 3 && (dm[0] < 1 || dm[1] < 1 || dm[2] < 1))
    return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid3d: dimensions must be >= 1");
  const size_t count = size_t(dm[0]) * (rank >= 2 ? dm[1] : 1) * (rank >= 3 ? dm[2] : 1);
  if (!dst) return count == 0 ? SSAM_OK : set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: null buffer");
  if (count > capacity)
    return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: buffer smaller than the grid");
  const size_t bytes = count * elem_size(dtype);
  if (!on_device) {
    if (std::fread(dst, 1, bytes, f.f) != bytes)
      return set_error(SSAM_ERR_RUNTIME, "grid io: truncated payload");
    return SSAM_OK;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Pinned pin;
  cudaError_t e = pin.init();
  if (e != cudaSuccess) return set_error(SSAM_ERR_CUDA, cudaGetErrorString(e));
  size_t off = 0;
  for (int k = 0; off < bytes; ++k) {
    const int b = k & 1;
    const size_t n = std::min(kChunk, bytes - off);
    if (k >= 2 && (e = cudaEventSynchronize(pin.ev[b])) != cudaSuccess) break;
    if (std::fread(pin.p[b], 1, n, f.f) != n) {
      cudaStreamSynchronize(s);
      return set_error(SSAM_ERR_RUNTIME, "grid io: truncated payload");
    }
    if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, pin.p[b], n, cudaMemcpyHostToDevice,
                             s)) != cudaSuccess)
      break;
    if ((e = cudaEventRecord(pin.ev[b], s)) != cudaSuccess) break;
    off += n;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? SSAM_OK : set_error(SSAM_ERR_CUDA, cudaGetErrorString(e));
}

int ssam_b200_sgrd_write(const char* path, int dtype, int rank, const int* dims, const void* src,
                         int on_device, void* stream) {
  if (dtype < 0 || dtype > 2) return set_error(SSAM_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (rank < 1 || rank > 3 || !dims) return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: bad rank");
  int dm[3] = {dims[0], rank >= 2 ? dims[1] : 1, rank >= 3 ? dims[2] : 1};
  // write_grid_file (grid_io.hpp:129-134) opens -- and truncates -- the file
  // first, then write_header rejects oversize dimensions (:43-46)
  File f(path, "wb");
  if (!f.f) return set_error(SSAM_ERR_RUNTIME, std::string("grid io: cannot open ") + (path ? path : "") + " for writing");
  for (int i = 0; i < 3; ++i)
    if (dm[i] > 0xffff)
      return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: dimension exceeds format limit (65535)");
  for (int i = 0; i < 3; ++i)
    if (dm[i] < 0) return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: negative dimension");
  unsigned char h[16] = {'S', 'G', 'R', 'D', 1, static_cast<unsigned char>(rank),
                         static_cast<unsigned char>(scalar_code(dtype)), 0};
  for (int i = 0; i < 3; ++i) {
    h[8 + 2 * i] = static_cast<unsigned char>(dm[i] & 0xff);
    h[9 + 2 * i] = static_cast<unsigned char>(dm[i] >> 8);
  }
  if (std::fwrite(h, 1, 16, f.f) != 16) return set_error(SSAM_ERR_RUNTIME, "grid io: write failed");
  const size_t bytes = size_t(dm[0]) * dm[1] * dm[2] * elem_size(dtype);
  if (bytes == 0) return SSAM_OK;
  if (!src) return set_error(SSAM_ERR_INVALID_ARGUMENT, "grid io: null buffer");
  if (!on_device) {
    return std::fwrite(src, 1, bytes, f.f) == bytes ? SSAM_OK
                                                   : set_error(SSAM_ERR_RUNTIME, "grid io: write failed");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Pinned pin;
  cudaError_t e = pin.init();
  if (e != cudaSuccess) return set_error(SSAM_ERR_CUDA, cudaGetErrorString(e));
  // D2H of chunk k+1 runs while chunk k is written to the file.
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t k) -> cudaError_t {
    const size_t off = k * kChunk, n = std::min(kChunk, bytes - off);
    cudaError_t r = cudaMemcpyAsync(pin.p[k & 1], static_cast<const char*>(src) + off, n,
                                    cudaMemcpyDeviceToHost, s);
    return r == cudaSuccess ? cudaEventRecord(pin.ev[k & 1], s) : r;
  };
  if ((e = issue(0)) != cudaSuccess) return set_error(SSAM_ERR_CUDA, cudaGetErrorString(e));
  for (size_t k = 0; k < nchunks; ++k) {
    if ((e = cudaEventSynchronize(pin.ev[k & 1])) != cudaSuccess) break;
    if (k + 1 < nchunks && (e = issue(k + 1)) != cudaSuccess) break;
    const size_t n = std::min(kChunk, bytes - k * kChunk);
    if (std::fwrite(pin.p[k & 1], 1, n, f.f) != n) {
      cudaStreamSynchronize(s);
      return set_error(SSAM_ERR_RUNTIME, "grid io: write failed");
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? SSAM_OK : set_error(SSAM_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
