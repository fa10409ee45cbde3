/*
 * ssam_b200.h -- C ABI of the B200-native SSAM engine (libssam_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * has no FFI layer: its boundary is the three C++ templates of
 * proj/include/ssam/kernels.hpp (relative to /root/reference):
 *
 *   Grid2D<T> conv2d   (const Grid2D<T>&, const Filter2D<T>&, const KernelConfig&,
 *                       OpCounters* = nullptr);                            // kernels.hpp:189
 *   Grid2D<T> stencil2d(const Grid2D<T>&, const Stencil<T>&, const KernelConfig&,
 *                       int iters, OpCounters* = nullptr);                 // kernels.hpp:231
 *   Grid3D<T> stencil3d(const Grid3D<T>&, const Stencil<T>&, const KernelConfig&,
 *                       int iters, OpCounters* = nullptr);                 // kernels.hpp:283
 *
 * with T in {float, double, long long} (proj/tools/ssam_cli.cpp:241-243), and the
 * 1D entry points of the same header:
 *
 *   std::vector<T> conv1d(const std::vector<T>&, const std::vector<T>&,
 *                         const KernelConfig&, OpCounters* = nullptr);  // kernels.hpp:390
 *   std::vector<T> scan  (const std::vector<T>&, int lane_count = 32,
 *                         OpCounters* = nullptr);                       // kernels.hpp:422
 * Each entry point below replaces one of them; include/ssam_b200/kernels.hpp
 * re-exposes the exact C++ signatures on top of this ABI and re-raises the
 * reference's exception types from the status codes.
 *
 * Plain pointers and sizes only: no C++, torch or reference types cross it.
 * Grids are dense, row-major, x fastest: 2D data[y*W + x] (grid.hpp:11-28),
 * 3D data[(z*ny + y)*nx + x] (grid.hpp:30-49).
 *
 * Every call runs on the GPU.  There is no CPU fallback: without a CUDA
 * device the compute entry points return SSAM_ERR_NO_DEVICE.  Validation
 * happens first and needs no device, so the error contract is testable on
 * any host.
 */
#ifndef SSAM_B200_H
#define SSAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSAM_B200_ABI_VERSION 2

/* Element type of a call: float, double, long long (int64). */
typedef enum { SSAM_DTYPE_F32 = 0, SSAM_DTYPE_F64 = 1, SSAM_DTYPE_I64 = 2 } ssam_dtype;

/* ssam::Boundary (filter.hpp:15): zero padding or clamp-replicate. */
typedef enum { SSAM_BOUNDARY_ZERO = 0, SSAM_BOUNDARY_REPLICATE = 1 } ssam_boundary;

typedef enum {
  SSAM_OK = 0,
  SSAM_ERR_INVALID_ARGUMENT = 1, /* the reference throws std::invalid_argument */
  SSAM_ERR_LENGTH = 2,           /* the reference throws std::length_error (C > 255) */
  SSAM_ERR_CUDA = 3,             /* CUDA runtime failure; see ssam_b200_last_error() */
  SSAM_ERR_NO_DEVICE = 4,        /* no usable CUDA device */
  SSAM_ERR_OUT_OF_MEMORY = 5,    /* device allocation failed */
  SSAM_ERR_RUNTIME = 6           /* the reference throws std::runtime_error (grid I/O) */
} ssam_status;

/* ssam::KernelConfig (filter.hpp:117-139).  Validated exactly like
 * KernelConfig::check(); after validation p, b, lane_count and threads are
 * tuning hints only -- results never depend on them. */
typedef struct {
  int p;          /* outputs per lane per tile (reference default 4) */
  int b;          /* threads per block (reference default 128) */
  int boundary;   /* ssam_boundary; conv2d only */
  int lane_count; /* simulated warp width, power of two in [2, 64] */
  int threads;    /* CPU worker threads in the reference; ignored */
} ssam_kernel_config;

/* ssam::OpCounters (warp.hpp:12-28).  Filled with exactly what the
 * reference's simulator counts for the same call (closed forms), and
 * ACCUMULATED into (+=), as kernels.hpp:50-54 does. */
typedef struct {
  uint64_t mads;
  uint64_t shuffles;
  uint64_t broadcast_reads;
  uint64_t global_loads;
  uint64_t global_stores;
} ssam_op_counters;

/* ssam::Stencil<T> (filter.hpp:52-68): ntaps (dx, dy, dz) offsets and their
 * coefficients, stored as elements of the call's dtype. */
typedef struct {
  int dims;           /* 2 or 3 */
  int order;          /* k: largest |offset| component */
  int ntaps;
  const int* offsets; /* 3 * ntaps ints: dx, dy, dz per tap */
  const void* coeffs; /* ntaps elements of the call's dtype */
} ssam_stencil;

/* ssam::LatencyProfile (perf_model.hpp:14-26) measured on this device, in SM
 * cycles of one warp instruction on a dependent chain; t_l2_read and the SM
 * clock are extra (see csrc/latency.cu for each micro-benchmark). */
typedef struct {
  double t_shfl;
  double t_mad;
  double t_smem_read;
  double t_reg;
  double t_gmem_read;  /* HBM: coalesced 128-byte lines, random over 256 MiB */
  double t_gmem_write; /* st.global.wt + fence.acq_rel.gpu */
  double t_l2_read;    /* same chase over 16 MiB (L2 hits) */
  double sm_clock_mhz;
} ssam_latency_profile;

/* ---- library ------------------------------------------------------------ */
int ssam_b200_abi_version(void);
/* Message for the last non-OK status on the calling thread ("" if none). */
const char* ssam_b200_last_error(void);
/* Number of CUDA devices (0 when none is usable). */
int ssam_b200_device_count(void);
/* KernelConfig defaults: p=4, b=128, zero boundary, lane_count=32, threads=0. */
void ssam_b200_default_config(ssam_kernel_config* cfg);
/* Kernel launches issued by this process so far (evidence for benchmarks). */
uint64_t ssam_b200_launch_count(void);

/* ---- host-grid entry points (replace kernels.hpp:189 / :231 / :283) -----
 * in/out are host pointers of width*height (or nx*ny*nz) elements; they may
 * not alias.  Synchronous.  Pinned host memory gives full-speed copies. */
int ssam_b200_conv2d(int dtype, const void* in, int width, int height, const void* weights, int m,
                     int n, const ssam_kernel_config* cfg, void* out, ssam_op_counters* counters);

int ssam_b200_stencil2d(int dtype, const void* in, int width, int height, const ssam_stencil* st,
                        const ssam_kernel_config* cfg, int iters, void* out,
                        ssam_op_counters* counters);

int ssam_b200_stencil3d(int dtype, const void* in, int nx, int ny, int nz, const ssam_stencil* st,
                        const ssam_kernel_config* cfg, int iters, void* out,
                        ssam_op_counters* counters);

/* Runs the latency micro-benchmarks on the current device (a few ms). */
int ssam_b200_measure_latency(ssam_latency_profile* out);

/* Multi-GPU from one process (the drop-in's device-set variant of
 * kernels.hpp:231 / :283).  The grid is cut into `ndev` slabs along its
 * slowest axis (rows in 2D, z-planes in 3D); slab g runs on CUDA device
 * devices[g] (repeats allowed: two slabs may share a device) with k*Tb ghost
 * planes on every face shared with a neighbour.  After each fused launch of
 * Tb sweeps the boundary planes go to the neighbours' ghost planes by
 * cudaMemcpyPeerAsync (NVLink P2P, peer access enabled on demand), on a copy
 * stream overlapped with the interior launch.  Results are bit-identical to
 * ssam_b200_stencil2d / ssam_b200_stencil3d; errors and counters are
 * theirs, plus SSAM_ERR_INVALID_ARGUMENT for an empty list or a device index
 * out of range.  *used (optional) receives the number of slabs actually run
 * (fewer than ndev when a slab would own fewer than k*Tb planes). */
int ssam_b200_stencil2d_multi(int dtype, const void* in, int width, int height,
                              const ssam_stencil* st, const ssam_kernel_config* cfg, int iters,
                              const int* devices, int ndev, void* out, ssam_op_counters* counters,
                              int* used);
int ssam_b200_stencil3d_multi(int dtype, const void* in, int nx, int ny, int nz,
                              const ssam_stencil* st, const ssam_kernel_config* cfg, int iters,
                              const int* devices, int ndev, void* out, ssam_op_counters* counters,
                              int* used);

/* A batch of independent grids (same shape and stencil) through the engine
 * with the PCIe copies overlapped: grid k's host->device copy, sweeps and
 * device->host copy run on three streams while neighbouring grids are in
 * other stages, `depth` grids in flight (0: 2; bench.py uses 3, which
 * keeps both neighbours' copies under a step's sweeps), each with two device
 * buffers.  Results equal `count` calls of ssam_b200_stencil2d/3d (no
 * config checks, no counters); pinned host buffers give the overlap.  2D
 * stencils pass nz = 1.  Blocks until every result is on the host. */
int ssam_b200_stencil_batch(int dtype, int count, const void* const* in, void* const* out, int nx,
                            int ny, int nz, const ssam_stencil* st, int iters, int depth);

/* Validation only (no device needed): the status the call above would
 * return for these arguments before touching the GPU. */
int ssam_b200_check_conv2d(int width, int height, int m, int n, const ssam_kernel_config* cfg);
int ssam_b200_check_stencil2d(int width, int height, const ssam_stencil* st,
                              const ssam_kernel_config* cfg, int iters);
int ssam_b200_check_stencil3d(int nx, int ny, int nz, const ssam_stencil* st,
                              const ssam_kernel_config* cfg, int iters);

/* Closed-form OpCounters of the reference simulator for a call (no device). */
int ssam_b200_counters_conv2d(int width, int height, int m, int n, const ssam_kernel_config* cfg,
                              ssam_op_counters* counters);
int ssam_b200_counters_stencil2d(int width, int height, const ssam_stencil* st,
                                 const ssam_kernel_config* cfg, int iters,
                                 ssam_op_counters* counters);
int ssam_b200_counters_stencil3d(int nx, int ny, int nz, const ssam_stencil* st,
                                 const ssam_kernel_config* cfg, int iters,
                                 ssam_op_counters* counters);

/* ---- benchmark catalog (proj/src/stencil_catalog.cpp:81-127) ------------- */
int ssam_b200_benchmark_count(void);
const char* ssam_b200_benchmark_name(int index);
/* make_benchmark_stencil(name): writes up to cap taps (offsets 3*cap ints,
 * coeffs cap doubles); returns the tap count, or -1 for an unknown name
 * (the reference throws std::invalid_argument). */
int ssam_b200_benchmark_stencil(const char* name, int* dims, int* order, int* fpp, int* offsets,
                                double* coeffs, int cap);

/* ---- device-resident entry points (benchmarks, multi-GPU) -----------------
 * Pointers are device memory of the current device, 16-byte alignment and
 * width % (16/sizeof(T)) == 0 give the vectorised path.  stream is a
 * cudaStream_t (NULL = legacy default stream).  Asynchronous. */

/* conv2d over output rows [y_begin, y_end) of a width x height buffer.  A
 * row slab of a larger image passes only the rows it holds: rows outside
 * the buffer are the image boundary (zero or replicate). */
int ssam_b200_conv2d_device(int dtype, const void* d_in, void* d_out, int width, int height,
                            int y_begin, int y_end, const void* h_weights, int m, int n,
                            int boundary, void* stream);

/* One Jacobi sweep over output rows [y_begin, y_end) ∩ [k, height-k).  Only
 * interior cells are written: d_out's ring must already equal d_in's. */
int ssam_b200_stencil2d_sweep(int dtype, const void* d_in, void* d_out, int width, int height,
                              int y_begin, int y_end, const ssam_stencil* st, void* stream);

/* tb fused sweeps (temporal blocking) over the whole grid; returns
 * SSAM_ERR_INVALID_ARGUMENT if no fused kernel exists for this case. */
int ssam_b200_stencil2d_tb(int dtype, const void* d_in, void* d_out, int width, int height,
                           const ssam_stencil* st, int tb, void* stream);
/* Deepest fused temporal block available for (dtype, stencil); 1 = none. */
int ssam_b200_stencil2d_tb_max(int dtype, const ssam_stencil* st);
/* stencil2d_tb over output rows [y_begin, y_end) only; rows outside
 * [y_ring_lo, y_ring_hi) are the global ring and stay fixed (a row slab with
 * k*tb ghost rows passes its local bounds, which may lie outside the buffer).
 * Reads rows y_begin-k*tb .. y_end-1+k*tb. */
int ssam_b200_stencil2d_tb_range(int dtype, const void* d_in, void* d_out, int width, int height,
                                 int y_begin, int y_end, int y_ring_lo, int y_ring_hi,
                                 const ssam_stencil* st, int tb, void* stream);

/* One Jacobi sweep over output planes [z_begin, z_end) ∩ [k, nz-k) of an
 * nx x ny x nz buffer (a z-slab with ghost planes passes local indices). */
int ssam_b200_stencil3d_sweep(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                              int z_begin, int z_end, const ssam_stencil* st, void* stream);

/* tb fused 3D sweeps (temporal blocking, tb = 2 for order-1 stencils):
 * writes planes [z_begin, z_end) of the interior; planes outside
 * [z_ring_lo, z_ring_hi) are the global ring and stay fixed (a whole grid
 * passes k, nz-k; a z-slab with k*tb ghost planes its local bounds, which
 * may lie outside the buffer).  Reads planes z_begin-k*tb .. z_end-1+k*tb.
 * SSAM_ERR_INVALID_ARGUMENT if no fused kernel exists.  d_out's ring must
 * equal d_in's.  _tb_max: deepest fused block (1 = none). */
int ssam_b200_stencil3d_tb(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                           int z_begin, int z_end, int z_ring_lo, int z_ring_hi,
                           const ssam_stencil* st, int tb, void* stream);
int ssam_b200_stencil3d_tb_max(int dtype, const ssam_stencil* st);

/* Peer-memory halo for z-slab runs (one process per GPU, buffers shared with
 * CUDA IPC; NVLink P2P across GPUs).  The sweep kernel itself stores the
 * output planes a neighbour keeps as ghost slots into that neighbour's
 * buffer, so no separate exchange runs: planes z < lo_end also go to `lo` at
 * element offset (index + lo_shift), planes z >= hi_begin to `hi` at
 * (index + hi_shift).  NULL lo / hi: no neighbour on that side.  The caller
 * orders the sweeps across ranks (neighbours' previous sweep finished before
 * this one starts, e.g. with IPC events).  Replaces the send/recv pair of the
 * NCCL path (paper_1907_06154_b200/slab.py); the reference is single-node
 * single-GPU. */
typedef struct ssam_peer_halo {
  void* lo;
  long long lo_shift;
  int lo_end;
  void* hi;
  long long hi_shift;
  int hi_begin;
} ssam_peer_halo;

int ssam_b200_stencil3d_sweep_peer(int dtype, const void* d_in, void* d_out, int nx, int ny,
                                   int nz, int z_begin, int z_end, const ssam_stencil* st,
                                   const ssam_peer_halo* peer, void* stream);
int ssam_b200_stencil3d_tb_peer(int dtype, const void* d_in, void* d_out, int nx, int ny, int nz,
                                int z_begin, int z_end, int z_ring_lo, int z_ring_hi,
                                const ssam_stencil* st, int tb, const ssam_peer_halo* peer,
                                void* stream);

/* Device buffers shareable across processes (cudaMalloc + CUDA IPC handle of
 * SSAM_IPC_HANDLE_BYTES bytes).  _open maps a handle exported by another
 * process (same GPU, or a peer GPU with P2P access); _close unmaps it. */
#define SSAM_IPC_HANDLE_BYTES 64
int ssam_b200_ipc_alloc(size_t bytes, void** d_ptr, void* handle);
int ssam_b200_ipc_free(void* d_ptr);
int ssam_b200_ipc_open(const void* handle, void** d_ptr);
int ssam_b200_ipc_close(void* d_ptr);
/* Device-side generation flags for the peer path (no host barrier per
 * sweep): write_u32 stores `value` to the 32-bit word at d_addr (local or
 * IPC-mapped peer memory) once the stream's prior work is done and visible;
 * wait_u32 holds the stream until the word is >= value.  Both are stream
 * memory operations (cuStreamWriteValue32 / cuStreamWaitValue32). */
int ssam_b200_stream_write_u32(void* d_addr, uint32_t value, void* stream);
int ssam_b200_stream_wait_u32(const void* d_addr, uint32_t value, void* stream);

/* iters sweeps with ping-pong buffers.  d_a holds the input; d_b is scratch
 * of the same size whose ring this call initialises.  *d_result receives
 * d_a or d_b, whichever holds the final generation.  tb: temporal block
 * depth (0 = automatic, 1 = none). */
int ssam_b200_stencil2d_run(int dtype, void* d_a, void* d_b, int width, int height,
                            const ssam_stencil* st, int iters, int tb, void* stream,
                            void** d_result);
int ssam_b200_stencil3d_run(int dtype, void* d_a, void* d_b, int nx, int ny, int nz,
                            const ssam_stencil* st, int iters, void* stream, void** d_result);
/* (stencil3d_run fuses sweeps in pairs with ssam_b200_stencil3d_tb where
 * available: same results, half the HBM passes.) */

/* Device SplitMix64 fill, bit-identical to the reference's random_grid2d/3d:
 * element i receives stream draw (first + i) of seed (rng.hpp, grid.hpp:52-66). */
int ssam_b200_fill_random(int dtype, void* d_out, size_t count, uint64_t seed, uint64_t first,
                          void* stream);

/* max_i |a_i - b_i| / max(1, |b_i|) and max |a_i - b_i| (acceptance.cpp:35-44),
 * reduced on the device; synchronises the stream. */
int ssam_b200_max_rel_err(int dtype, const void* d_a, const void* d_b, size_t count,
                          double* max_rel, double* max_abs, void* stream);

/* ---- 1D: conv1d and scan (replace kernels.hpp:390 / :422) ----------------
 * conv1d: out(i) = sum_{s<m} in(i + (m-1)/2 - s) * w[s] (oracle.hpp:61-73),
 * cfg->boundary zero or replicate; the reference's checks: m in
 * [1, lane_count], len >= lane_count, lane_count a power of two in [2, 64]
 * (all std::invalid_argument).  scan: inclusive prefix sum; len must be a
 * multiple of lane_count (empty input is returned as is).  Host buffers,
 * synchronous; counters accumulate the simulator's tallies. */
int ssam_b200_conv1d(int dtype, const void* in, long long len, const void* weights, int m,
                     const ssam_kernel_config* cfg, void* out, ssam_op_counters* counters);
int ssam_b200_scan(int dtype, const void* in, unsigned long long len, int lane_count, void* out,
                   ssam_op_counters* counters);
int ssam_b200_check_conv1d(long long len, int m, const ssam_kernel_config* cfg);
int ssam_b200_check_scan(unsigned long long len, int lane_count);
int ssam_b200_counters_conv1d(long long len, int m, const ssam_kernel_config* cfg,
                              ssam_op_counters* counters);
int ssam_b200_counters_scan(unsigned long long len, int lane_count, ssam_op_counters* counters);
/* Device-resident, stream-ordered: conv1d (m <= 32; d_in and d_out may not
 * overlap) and the scan (an L2-chunked reduce-then-scan, one launch per
 * 12 MiB of input; d_out == d_in scans in place). */
int ssam_b200_conv1d_device(int dtype, const void* d_in, void* d_out, int len,
                            const void* h_weights, int m, int boundary, void* stream);
int ssam_b200_scan_device(int dtype, const void* d_in, void* d_out, size_t len, void* stream);

/* ---- SGRD grid files (proj/include/ssam/grid_io.hpp:14-158) ---------------
 * The reference's binary format: "SGRD", version 1, rank, scalar code
 * (f32 1 / f64 2 / i64 3), u16 dims (d0 fastest, unused = 1), raw
 * little-endian scalars.  dims > 65535 -> SSAM_ERR_INVALID_ARGUMENT; bad
 * magic, version, rank or scalar type, truncation and unopenable files ->
 * SSAM_ERR_RUNTIME (std::runtime_error in the reference).  on_device != 0:
 * the buffer is device memory and the payload streams through pinned
 * staging buffers on `stream` (disk I/O overlapped with the PCIe copies);
 * both calls return when the data has landed. */
int ssam_b200_sgrd_info(const char* path, int* rank, int* dtype, int* dims /* [3] */);
int ssam_b200_sgrd_read(const char* path, int dtype, int rank, int* dims /* [3], out */, void* dst,
                        size_t capacity_elems, int on_device, void* stream);
int ssam_b200_sgrd_write(const char* path, int dtype, int rank, const int* dims /* [3] */,
                         const void* src, int on_device, void* stream);

/* ---- direct-gather verifier -----------------------------------------------
 * The same operators computed by one-thread-per-cell gather kernels in the
 * oracle's summation order and arithmetic (oracle.hpp:44-116: double
 * accumulation, no FMA contraction; native int64) -- the GPU-side check the
 * CLI (`ssam run`, proj/tools/ssam_cli.cpp:138-230) compares the SSAM engine
 * against.  Host buffers, synchronous, no validation beyond shapes.  A 2D
 * stencil passes nz = 1; conv1d is conv2d with h = 1, n = 1. */
int ssam_b200_gather_conv2d(int dtype, const void* in, int width, int height, const void* weights,
                            int m, int n, int boundary, void* out);
int ssam_b200_gather_stencil(int dtype, const void* in, int nx, int ny, int nz,
                             const ssam_stencil* st, int iters, void* out);
/* The same gather sweeps on DEVICE buffers (d_a holds the input, d_b is
 * scratch; *d_result is whichever holds the result), stream-ordered: the
 * per-cell check of full-size device-resident runs (bench max_rel). */
int ssam_b200_gather_stencil_run(int dtype, void* d_a, void* d_b, int nx, int ny, int nz,
                                 const ssam_stencil* st, int iters, void* stream,
                                 void** d_result);

/* Returns the device memory the host-grid calls keep cached in the engine's
 * own stream-ordered pool (one per device; the default pool is untouched). */
int ssam_b200_trim_cache(void);

#ifdef __cplusplus
}
#endif

#endif /* SSAM_B200_H */
