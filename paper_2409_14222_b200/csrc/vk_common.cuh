// Shared plumbing for the Vanka/MG C ABI: error state, handle layouts.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/vanka_b200.h"

#ifndef VK_PDL_MB_DEFAULT
#define VK_PDL_MB_DEFAULT 0
#endif

namespace vk {

void set_error(const char* fmt, ...);

// Device-side CSR (scipy csr_matrix with sorted indices, int32 indexing).
struct Csr {
  int32_t nrows = 0, ncols = 0;
  int64_t nnz = 0;
  int32_t* indptr = nullptr;
  int32_t* indices = nullptr;
  double* data = nullptr;
  double mean_row = 0.0;
  double warp_max_mean = 0.0;  // mean over 32-row groups of the longest row
  int32_t max_row = 0;
  // CSR-stream schedule: row blocks of <= kStreamNnz nonzeros / kStreamRows rows
  int32_t nblocks = 0;
  int2* blk = nullptr;         // [nblocks+1] (first row, first nonzero) of each block
  uint64_t uid = 0;            // process-unique id of this (immutable) sparsity pattern
};

#ifndef VK_STREAM_THREADS
#define VK_STREAM_THREADS 256
#endif
#ifndef VK_STREAM_U
#define VK_STREAM_U 8
#endif
constexpr int kStreamThreads = VK_STREAM_THREADS;
constexpr int kStreamU = VK_STREAM_U;
constexpr int kStreamNnz = kStreamThreads * kStreamU;   // 2048 nonzeros per block
constexpr int kStreamRows = 2 * kStreamThreads;

// Patch set: CSR-like layout of patch DoF lists + explicit inverses.
struct Patches {
  int32_t npatch = 0;       // kept patches
  int32_t ndof = 0;
  int32_t smax = 0;
  int64_t total = 0;        // sum of patch sizes
  int32_t weighting = 0;
  // device arrays
  int64_t* off = nullptr;       // [npatch+1] offsets into idx / weights / zbuf
  int32_t* idx = nullptr;       // [total] velocity dofs then pressure dofs
  int32_t* nvel = nullptr;      // [npatch]
  double* w = nullptr;          // [total]
  int32_t* mult = nullptr;      // [ndof] multiplicity (integer)
  int32_t* cand = nullptr;      // [npatch] candidate index of kept patch
  int64_t* opoff = nullptr;     // [npatch+1] offsets (doubles) into inv
  double* inv = nullptr;        // explicit inverses, column-major per patch
  int64_t inv_total = 0;
  int32_t* dptr = nullptr;      // [ndof+1] DoF -> slot map offsets
  int32_t* dslot = nullptr;     // [total] slots (flat patch entry ids), patch order
  double* zbuf = nullptr;       // [total] weighted local corrections
  bool mixed_sizes = false;     // >25% of patches need fewer row slots than the largest
  bool factored = false;
  // host copies of the schedule (sizes) for bucketing
  std::vector<int64_t> h_off;
  // factor schedule, built by the first factorization (sizes never change):
  // patch ids grouped by size class, and (smax, first, count) per class
  int32_t* fac_ids = nullptr;
  int32_t* fac_status = nullptr;  // [npatch]
  // extraction map, built by the first factorisation against a matrix: for
  // every (patch row, stored CSR entry of that row) the local column (-1 if
  // the column is not in the patch); keyed by the CSR handle (its pattern)
  int64_t* fac_eoff = nullptr;    // [total+1] offsets into fac_emap per patch row (flat idx position)
  int16_t* fac_emap = nullptr;
  uint64_t fac_emap_key = 0;      // Csr::uid the map was built for (0 = none)
  std::vector<std::tuple<int, int, int>> fac_classes;
};

}  // namespace vk

struct vk_csr_s : public vk::Csr {};
struct vk_patches_s : public vk::Patches {};

#define VK_CHECK_CUDA(call)                                                      \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      vk::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                  \
                    cudaGetErrorString(e_));                                     \
      return VK_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define VK_CHECK_LAUNCH()                                                        \
  do {                                                                           \
    cudaError_t e_ = cudaGetLastError();                                         \
    if (e_ != cudaSuccess) {                                                     \
      vk::set_error("%s:%d launch: %s", __FILE__, __LINE__,                     \
                    cudaGetErrorString(e_));                                     \
      return VK_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define VK_REQUIRE(cond, ...)                                                    \
  do {                                                                           \
    if (!(cond)) {                                                               \
      vk::set_error(__VA_ARGS__);                                                \
      return VK_ERR_ARG;                                                         \
    }                                                                            \
  } while (0)

static inline cudaStream_t vk_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static inline int vk_grid(int64_t work, int block, int cap = 148 * 16) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// Blocks of `kernel` that are resident on the whole device at once (SM count
// x occupancy), cached per (kernel, block size, dynamic shared memory).
// Persistent grid-stride kernels launch exactly this many so there is no
// partial last wave.
static inline int vk_current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

static inline int vk_resident_blocks(const void* kernel, int block, size_t smem = 0) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const int dev = vk_current_device();   // occupancy is cached per device
  const auto key = std::make_tuple(kernel, block, smem, dev);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int n = per_sm * sms;
  cache.emplace(key, n);
  return n;
}

// Opt `kernel` into `bytes` of dynamic shared memory on the CURRENT device
// (a function attribute is per device: a process driving a second GPU must
// set it there too).  Done once per (kernel, device, bytes).
static inline cudaError_t vk_smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(kernel, vk_current_device());
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

// TMA 1-D bulk copies (cp.async.bulk) completed on an mbarrier.
// ---- programmatic dependent launch (PDL) for the latency-bound coarse
// levels.  Every kernel on the V-cycle path triggers its dependents at entry
// (griddepcontrol.launch_dependents) and waits for its predecessor
// (griddepcontrol.wait, a no-op without a programmatic predecessor) before
// touching anything an earlier kernel in the stream produced; what it reads
// before the wait is setup-time data (matrix / patch structure, operators).
// The launch side opts in per launch: only launches that move less than
// vk_pdl_bytes() (small, one-wave kernels) get the programmatic-serialisation
// attribute, so big multi-wave kernels never share SMs with waiting CTAs.
static __device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
static __device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// bytes below which a launch may overlap its predecessor (VK_PDL_MB, MB;
// 0 disables PDL)
static inline int64_t vk_pdl_bytes() {
  static const int64_t v = [] {
    const char* e = getenv("VK_PDL_MB");
    return int64_t(e ? atof(e) : VK_PDL_MB_DEFAULT) * (int64_t(1) << 20);
  }();
  return v;
}

template <typename... KArgs, typename... Args>
static cudaError_t vk_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, int64_t bytes, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (bytes < vk_pdl_bytes()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static __device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
static __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
static __device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}


