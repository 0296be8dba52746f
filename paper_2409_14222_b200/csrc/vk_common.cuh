// Shared plumbing for the Vanka/MG C ABI: error state, handle layouts.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/vanka_b200.h"

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
  int32_t max_row = 0;
  // CSR-stream schedule: row blocks of <= kStreamNnz nonzeros / kStreamRows rows
  int32_t nblocks = 0;
  int32_t* rowblk = nullptr;   // [nblocks+1]
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
// x occupancy), cached per kernel.  Persistent grid-stride kernels launch
// exactly this many so there is no partial last wave.
static inline int vk_resident_blocks(const void* kernel, int block, size_t smem = 0) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(kernel);
  if (it != cache.end()) return it->second;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int n = per_sm * sms;
  cache.emplace(kernel, n);
  return n;
}
