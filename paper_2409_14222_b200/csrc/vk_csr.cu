#include <atomic>
// K5/K6: CSR matrices on the device, SpMV / fused residual / transfers.
//
// Replaces scipy csr_matvec at reference sparsela.py:45-47 (spmv),
// mg.py:41-45 (TransferPair.prolong / restrict — restrict through an explicit
// transposed CSR), mg.py:270, 294 (residual b - A x).
//
// CSR-stream kernel (HBM-bound, 0.17 flop/B): the rows are cut on the host
// into blocks of <= 2048 nonzeros / 512 rows.  A 256-thread CTA owns one
// block: every thread issues 8 independent coalesced (col, val) loads plus
// the 8 x-gathers (x is L2-resident), and stores the products in shared
// memory; then each row is summed sequentially, left to right, without FMA
// contraction: y_i = ((0 + a_i0 x_0) + a_i1 x_1) + ...  — the exact
// operation order of scipy's csr_matvec (and, through the ascending-source
// transpose, of csc_matvec for masked.T), so SpMV / residual / transfers are
// bit-identical to the reference.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include <cooperative_groups.h>

#include "vk_common.cuh"

namespace cg = cooperative_groups;

#ifndef VK_CSR_SHORT  // thread-per-row kernel when the mean over 32-row groups of
#define VK_CSR_SHORT 11  // the longest row is <= this (measured: transfers P of cfg2/3)
#endif

namespace vk {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace vk

extern "C" const char* vk_last_error(void) { return vk::g_err; }
extern "C" int vk_version(void) { return 1; }
extern "C" int vk_device_sync(void) {
  VK_CHECK_CUDA(cudaDeviceSynchronize());
  return VK_OK;
}

namespace {

using vk::kStreamNnz;
using vk::kStreamRows;
using vk::kStreamThreads;
using vk::kStreamU;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// MODE 0: y = alpha*Ax + beta*y (beta == 0: y not read);  MODE 1: y = b - A x
//
// Latency chain per CTA (what bounds the one-wave transfers): the block table
// holds (first row, first nonzero) pairs, so the (col, val) loads of the first
// chunk, the row-pointer loads and the epilogue operand (b or y) are all in
// flight together; only the x gathers wait for col.
// x / b loads: through the read-only path (NC) when the data comes from an
// earlier kernel; coherent loads when an earlier phase of the same
// cooperative kernel wrote them (vk_residual_restrict / vk_prolong_residual)
template <bool NC>
__device__ __forceinline__ double ld_x(const double* p) {
  if (NC) return __ldg(p);
  return *p;
}

// One row block (block table entry `bi`) of the CSR-stream SpMV; shared
// arrays passed in by the kernel.
template <int MODE, bool PDL, bool NC>
__device__ __forceinline__ void stream_block(int bi, const int2* __restrict__ blk,
                                             const int* __restrict__ ptr,
                                             const int* __restrict__ col,
                                             const double* __restrict__ val, const double* x,
                                             double* y, double alpha, double beta,
                                             const double* b, double* prod, int* sptr,
                                             double& carry) {
  const int t = threadIdx.x;
  const int2 e0 = blk[bi], e1 = blk[bi + 1];
  const int r0 = e0.x, k0 = e0.y, k1 = e1.y;
  const int nr = e1.x - r0;
  const bool single = (nr == 1);
  // epilogue operand (b or y) of each row, read after its sum
#define VK_PRE(i) ((MODE == 1) ? b[r0 + (i)] : y[r0 + (i)])
  for (int i = t; i <= nr; i += kStreamThreads) cp_async4(sptr + i, ptr + r0 + i);
  // block table and row pointers (setup data) are in flight; x and b / y
  // come from the preceding kernel
  if (PDL) pdl_wait();
  if (t == 0) carry = 0.0;
  for (int kc = k0; kc < k1 || (kc == k0 && k0 == k1); kc += kStreamNnz) {
    const int kend = min(k1, kc + kStreamNnz);
    int c[kStreamU];
    double v[kStreamU];
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const int k = kc + t + u * kStreamThreads;
      c[u] = (k < kend) ? __ldcs(col + k) : 0;
      v[u] = (k < kend) ? __ldcs(val + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kStreamU; ++u) {
      const int k = kc + t + u * kStreamThreads;
      if (k < kend) prod[k - kc] = __dmul_rn(v[u], ld_x<NC>(x + c[u]));
    }
    cp_async_wait_all();
    __syncthreads();
    if (single) {
      // a row longer than one chunk: thread 0 carries the sequential sum
      if (t == 0) {
        double s = carry;
        for (int k = kc; k < kend; ++k) s = __dadd_rn(s, prod[k - kc]);
        carry = s;
      }
    } else {
      // One thread per row, each row summed left to right.  Lane l starts
      // d = (a - l) mod 16 steps late, so at every step the half-warp reads
      // 16 distinct 8-byte bank slots ((a + k) mod 16 == (step + l) mod 16)
      // instead of colliding whenever row starts agree mod 16.  (A cheaper
      // skew — d = rank among the lanes sharing a start slot — and no skew
      // measured slower.)
      for (int i0 = 0; i0 < nr; i0 += kStreamThreads) {
        const int i = i0 + t;
        const int lane = t & 31;
        int a = 0, len = 0;
        if (i < nr) {
          a = sptr[i] - kc;
          len = sptr[i + 1] - kc - a;
        }
        const int d = len > 0 ? (a - lane) & 15 : 0;
        const int steps = __reduce_max_sync(0xffffffffu, len > 0 ? len + d : 0);
        double s = 0.0;
#pragma unroll 4
        for (int st = 0; st < steps; ++st) {
          const int k = st - d;
          if (k >= 0 && k < len) s = __dadd_rn(s, prod[a + k]);
        }
        if (i >= nr) continue;
        const int row = r0 + i;
        if (MODE == 1) {
          y[row] = __dsub_rn(VK_PRE(i), s);
        } else {
          double out = (alpha == 1.0) ? s : __dmul_rn(alpha, s);
          if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? VK_PRE(i) : __dmul_rn(beta, VK_PRE(i)), out);
          y[row] = out;
        }
      }
    }
    __syncthreads();
    if (k0 == k1) break;
  }
  if (single && t == 0) {
    const double s = carry;
    if (MODE == 1) {
      y[r0] = __dsub_rn(VK_PRE(0), s);
    } else {
      double out = (alpha == 1.0) ? s : __dmul_rn(alpha, s);
      if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? VK_PRE(0) : __dmul_rn(beta, VK_PRE(0)), out);
      y[r0] = out;
    }
  }
}

#undef VK_PRE

template <int MODE>
__global__ void __launch_bounds__(kStreamThreads) csr_stream_kernel(
    const int2* __restrict__ blk, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
    double alpha, double beta, const double* __restrict__ b) {
  __shared__ double prod[kStreamNnz];
  __shared__ int sptr[kStreamRows + 1];
  __shared__ double carry;
  pdl_trigger();
  stream_block<MODE, true, true>(blockIdx.x, blk, ptr, col, val, x, y, alpha, beta, b, prod, sptr,
                                 carry);
}

// Short-row kernel (thread per row): for matrices with a few nonzeros per
// row (prolongations) the shared-memory staging of the stream kernel costs
// more than it saves.  Same per-row operation order (sequential, FMA-free).
template <int MODE, bool PDL, bool NC>
__device__ __forceinline__ void row_work(int row, const int* __restrict__ ptr,
                                         const int* __restrict__ col,
                                         const double* __restrict__ val, const double* x,
                                         double* y, double alpha, double beta, const double* b) {
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  if (PDL) pdl_wait();
  double pre = 0.0;
  if (MODE == 1) pre = __ldg(b + row);
  else if (beta != 0.0) pre = y[row];
  double s = 0.0;
  int k = k0;
  for (; k + 4 <= k1; k += 4) {
    int c[4];
    double v[4], p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = __ldg(col + k + u);
      v[u] = __ldg(val + k + u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = __dmul_rn(v[u], ld_x<NC>(x + c[u]));
#pragma unroll
    for (int u = 0; u < 4; ++u) s = __dadd_rn(s, p[u]);
  }
  for (; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(val + k), ld_x<NC>(x + __ldg(col + k))));
  if (MODE == 1) {
    y[row] = __dsub_rn(pre, s);
  } else {
    double out = (alpha == 1.0) ? s : __dmul_rn(alpha, s);
    if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? pre : __dmul_rn(beta, pre), out);
    y[row] = out;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) csr_row_kernel(
    int nrows, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
    double alpha, double beta, const double* __restrict__ b) {
  pdl_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) {
    pdl_wait();
    return;
  }
  row_work<MODE, true, true>(row, ptr, col, val, x, y, alpha, beta, b);
}

// Two SpMV phases in ONE cooperative launch with a grid barrier between
// them: the V-cycle's residual + restriction (r = b - A x; rc = P^T r,
// mg.py:294-295) and prolongation + the next residual (x += P xc;
// r = b - A x, mg.py:296-297).  Each phase runs the same per-row code as the
// standalone kernels (persistent CTAs walk the row blocks / rows), so the
// results are bit-identical; the barrier replaces a kernel boundary, and
// phase B reads phase A's output with coherent loads.
struct CsrPhase {
  const int2* blk;
  int nblocks, nrows;
  const int* ptr;
  const int* col;
  const double* val;
  const double* x;
  double* y;
  double alpha, beta;
  const double* b;
};

template <int MODE, bool SHORT, bool NC>
__device__ __forceinline__ void run_phase(const CsrPhase& p, double* prod, int* sptr,
                                          double& carry) {
  if (SHORT) {
    for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < p.nrows;
         row += gridDim.x * blockDim.x)
      row_work<MODE, false, NC>(row, p.ptr, p.col, p.val, p.x, p.y, p.alpha, p.beta, p.b);
  } else {
    for (int bi = blockIdx.x; bi < p.nblocks; bi += gridDim.x) {
      __syncthreads();
      stream_block<MODE, false, NC>(bi, p.blk, p.ptr, p.col, p.val, p.x, p.y, p.alpha, p.beta,
                                    p.b, prod, sptr, carry);
    }
  }
}

template <int MA, bool SA, int MB, bool SB>
__global__ void __launch_bounds__(kStreamThreads) csr_two_phase_kernel(CsrPhase A, CsrPhase B) {
  __shared__ double prod[kStreamNnz];
  __shared__ int sptr[kStreamRows + 1];
  __shared__ double carry;
  run_phase<MA, SA, true>(A, prod, sptr, carry);
  cg::this_grid().sync();
  run_phase<MB, SB, false>(B, prod, sptr, carry);
}

// Opt-in tree-reduction kernel (VK_SPMV_TREE=1, NOT bit-exact): G lanes
// per row stride over its entries with FMA and combine by a shuffle tree —
// the usual vector-CSR SpMV.  It trades scipy's sequential, FMA-free row
// order (hence bit-identity with the reference) for parallel row sums; it
// exists to measure what that order costs.  The bit-exact kernels above stay
// the default everywhere.
template <int MODE, int G>
__global__ void __launch_bounds__(256) csr_tree_kernel(
    int nrows, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
    double alpha, double beta, const double* __restrict__ b) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int rows_per_cta = blockDim.x / G;
  for (int row0 = blockIdx.x * rows_per_cta; row0 < nrows; row0 += gridDim.x * rows_per_cta) {
    const int row = row0 + threadIdx.x / G;
    double s = 0.0;
    if (row < nrows) {
      const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
      for (int k = k0 + sub; k < k1; k += G) s = fma(__ldcs(val + k), __ldg(x + __ldcs(col + k)), s);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, G);
    if (row < nrows && sub == 0) {
      if (MODE == 1) {
        y[row] = b[row] - s;
      } else {
        double out = alpha * s;
        if (beta != 0.0) out += beta * y[row];
        y[row] = out;
      }
    }
  }
}

static bool tree_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_SPMV_TREE");
    return e && e[0] == '1';
  }();
  return v;
}

template <int MODE>
cudaError_t launch_tree(const vk::Csr& a, const double* x, double* y, double alpha, double beta,
                        const double* b, cudaStream_t st) {
  const double m = a.mean_row;
  const int64_t bytes = 12 * a.nnz + 24 * int64_t(a.nrows);
#define VK_TREE(G_)                                                                             \
  return vk_launch(csr_tree_kernel<MODE, G_>, dim3(std::min<int64_t>((a.nrows + 256 / G_ - 1) /  \
                                                                     (256 / G_), 148 * 16)),     \
                   dim3(256), 0, st, bytes, a.nrows, a.indptr, a.indices, a.data, x, y, alpha,    \
                   beta, b)
  if (m <= 12) VK_TREE(4);
  if (m <= 24) VK_TREE(8);
  if (m <= 48) VK_TREE(16);
  VK_TREE(32);
#undef VK_TREE
}

template <int MODE>
cudaError_t launch_spmv(const vk::Csr& a, const double* x, double* y, double alpha, double beta,
                        const double* b, cudaStream_t st) {
  if (a.nblocks == 0) return cudaSuccess;
  if (tree_enabled()) return launch_tree<MODE>(a, x, y, alpha, beta, b, st);
  if (a.warp_max_mean <= VK_CSR_SHORT) {
    return vk_launch(csr_row_kernel<MODE>, dim3((a.nrows + 255) / 256), dim3(256), 0, st,
                     12 * a.nnz + 24 * int64_t(a.nrows), a.nrows, a.indptr, a.indices, a.data,
                     x, y, alpha, beta, b);
  }
  return vk_launch(csr_stream_kernel<MODE>, dim3(a.nblocks), dim3(kStreamThreads), 0, st,
                   12 * a.nnz + 24 * int64_t(a.nrows), a.blk, a.indptr, a.indices, a.data, x, y,
                   alpha, beta, b);
}

CsrPhase phase_of(const vk::Csr& a, const double* x, double* y, double alpha, double beta,
                  const double* b) {
  CsrPhase p;
  p.blk = a.blk;
  p.nblocks = a.nblocks;
  p.nrows = a.nrows;
  p.ptr = a.indptr;
  p.col = a.indices;
  p.val = a.data;
  p.x = x;
  p.y = y;
  p.alpha = alpha;
  p.beta = beta;
  p.b = b;
  return p;
}

template <int MA, int MB>
cudaError_t launch_two_phase(const vk::Csr& a, CsrPhase A, const vk::Csr& bm, CsrPhase B,
                             cudaStream_t st) {
  const bool sa = a.warp_max_mean <= VK_CSR_SHORT, sb = bm.warp_max_mean <= VK_CSR_SHORT;
  const void* k;
  if (sa && sb) k = (const void*)csr_two_phase_kernel<MA, true, MB, true>;
  else if (sa) k = (const void*)csr_two_phase_kernel<MA, true, MB, false>;
  else if (sb) k = (const void*)csr_two_phase_kernel<MA, false, MB, true>;
  else k = (const void*)csr_two_phase_kernel<MA, false, MB, false>;
  const int grid = vk_resident_blocks(k, kStreamThreads, 0);
  void* args[] = {&A, &B};
  return cudaLaunchCooperativeKernel(k, dim3(grid), dim3(kStreamThreads), args, 0, st);
}

__global__ void csr_to_dense_kernel(int nrows, int ncols, const int* __restrict__ ptr,
                                    const int* __restrict__ col, const double* __restrict__ val,
                                    double* __restrict__ dense) {
  for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
    double* drow = dense + static_cast<int64_t>(row) * ncols;
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) drow[j] = 0.0;
    __syncthreads();
    for (int k = ptr[row] + threadIdx.x; k < ptr[row + 1]; k += blockDim.x) drow[col[k]] = val[k];
    __syncthreads();
  }
}

// (col * nrows + row, value) of every stored entry, one thread per row
__global__ void transpose_keys_kernel(int nrows, const int* __restrict__ ptr,
                                      const int* __restrict__ col, const double* __restrict__ val,
                                      unsigned long long* __restrict__ keys,
                                      double* __restrict__ vals) {
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrows;
       row += gridDim.x * blockDim.x)
    for (int k = ptr[row]; k < ptr[row + 1]; ++k) {
      keys[k] = (unsigned long long)col[k] * (unsigned long long)nrows + row;
      vals[k] = val[k];
    }
}

// greedy row blocks: <= kStreamNnz nonzeros and <= kStreamRows rows; a row
// longer than kStreamNnz gets a block of its own
std::vector<int32_t> make_row_blocks(const std::vector<int32_t>& p) {
  const int32_t n = static_cast<int32_t>(p.size()) - 1;
  std::vector<int32_t> rb;
  rb.push_back(0);
  int32_t r = 0;
  while (r < n) {
    int32_t start = r;
    int64_t nnz = 0;
    while (r < n && r - start < kStreamRows) {
      const int64_t len = p[r + 1] - p[r];
      if (r > start && nnz + len > kStreamNnz) break;
      nnz += len;
      ++r;
      if (nnz > kStreamNnz) break;  // single long row
    }
    rb.push_back(r);
  }
  return rb;
}

}  // namespace

extern "C" int vk_csr_create(const int32_t* indptr, const int32_t* indices, const double* data,
                             int32_t nrows, int32_t ncols, int64_t nnz, vk_csr_t* out) {
  VK_REQUIRE(out != nullptr && nrows >= 0 && ncols >= 0 && nnz >= 0, "vk_csr_create: bad args");
  VK_REQUIRE(nnz < (int64_t(1) << 31), "vk_csr_create: nnz exceeds int32 indexing");
  std::vector<int32_t> hp(nrows + 1);
  cudaError_t e = cudaMemcpy(hp.data(), indptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDefault);
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_create: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  VK_REQUIRE(hp[0] == 0 && hp[nrows] == nnz, "vk_csr_create: indptr does not match nnz");
  auto rb = make_row_blocks(hp);
  static std::atomic<uint64_t> next_uid{1};
  auto* a = new vk_csr_s();
  a->uid = next_uid.fetch_add(1);
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = nnz;
  a->nblocks = static_cast<int32_t>(rb.size()) - 1;
  e = cudaMalloc(&a->indptr, sizeof(int32_t) * (nrows + 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->indices, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->data, sizeof(double) * std::max<int64_t>(nnz, 1));
  std::vector<int2> bt(rb.size());
  for (size_t i = 0; i < rb.size(); ++i) bt[i] = make_int2(rb[i], hp[rb[i]]);
  if (e == cudaSuccess) e = cudaMalloc(&a->blk, sizeof(int2) * bt.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(a->indptr, hp.data(), sizeof(int32_t) * (nrows + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->blk, bt.data(), sizeof(int2) * bt.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpy(a->indices, indices, sizeof(int32_t) * nnz, cudaMemcpyDefault);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(a->data, data, sizeof(double) * nnz, cudaMemcpyDefault);
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_create: %s", cudaGetErrorString(e));
    cudaFree(a->indptr);
    cudaFree(a->indices);
    cudaFree(a->data);
    cudaFree(a->blk);
    delete a;
    return VK_ERR_CUDA;
  }
  int32_t mx = 0;
  for (int32_t i = 0; i < nrows; ++i) mx = std::max(mx, hp[i + 1] - hp[i]);
  a->max_row = mx;
  a->mean_row = nrows ? double(nnz) / nrows : 0.0;
  // divergence measure of a thread-per-row schedule: mean over 32-row groups
  // of the longest row in the group
  double wsum = 0.0;
  int32_t ng = 0;
  for (int32_t g = 0; g < nrows; g += 32, ++ng) {
    int32_t m = 0;
    for (int32_t i = g; i < std::min(nrows, g + 32); ++i) m = std::max(m, hp[i + 1] - hp[i]);
    wsum += m;
  }
  a->warp_max_mean = ng ? wsum / ng : 0.0;
  *out = a;
  return VK_OK;
}

extern "C" int vk_csr_transpose(vk_csr_t a, vk_csr_t* out) {
  VK_REQUIRE(a && out, "vk_csr_transpose: null handle");
  // Deterministic transpose on the device: entry (i, j) gets the key
  // j * nrows + i and the keys are radix-sorted (vk_coo_to_csr), so the
  // entries of each output row come in ascending source-row order — the
  // accumulation order of scipy's csc_matvec on masked.T (mg.py:44-45).
  // Every stored entry is kept (explicit zeros included: drop_abs < 0).
  const int64_t nnz = a->nnz;
  unsigned long long* keys = nullptr;
  double* vals = nullptr;
  cudaError_t e = cudaMalloc(&keys, sizeof(unsigned long long) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&vals, sizeof(double) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess && a->nrows > 0) {
    transpose_keys_kernel<<<vk_grid(a->nrows, 256, 148 * 16), 256>>>(a->nrows, a->indptr,
                                                                     a->indices, a->data, keys, vals);
    e = cudaGetLastError();
  }
  int rc = VK_OK;
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_transpose: %s", cudaGetErrorString(e));
    rc = VK_ERR_CUDA;
  } else {
    rc = vk_coo_to_csr(nnz, reinterpret_cast<int64_t*>(keys), vals, a->ncols, a->nrows, 0, -1.0,
                       nullptr, nullptr, nullptr, out);
  }
  cudaFree(keys);
  cudaFree(vals);
  return rc;
}

extern "C" int vk_csr_info(vk_csr_t a, int32_t* nrows, int32_t* ncols, int64_t* nnz) {
  VK_REQUIRE(a, "vk_csr_info: null handle");
  if (nrows) *nrows = a->nrows;
  if (ncols) *ncols = a->ncols;
  if (nnz) *nnz = a->nnz;
  return VK_OK;
}

extern "C" int vk_csr_destroy(vk_csr_t a) {
  if (!a) return VK_OK;
  cudaFree(a->indptr);
  cudaFree(a->indices);
  cudaFree(a->data);
  cudaFree(a->blk);
  delete a;
  return VK_OK;
}

extern "C" int vk_spmv(vk_csr_t a, const double* x, double* y, double alpha, double beta,
                       void* stream) {
  VK_REQUIRE(a, "vk_spmv: null matrix");
  if (a->nrows == 0) return VK_OK;  // empty output: nothing to touch
  VK_REQUIRE((x || a->ncols == 0) && y, "vk_spmv: null argument");
  cudaError_t e = launch_spmv<0>(*a, x, y, alpha, beta, nullptr, vk_stream(stream));
  if (e != cudaSuccess) {
    vk::set_error("vk_spmv: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

extern "C" int vk_residual(vk_csr_t a, const double* b, const double* x, double* r, void* stream) {
  VK_REQUIRE(a, "vk_residual: null matrix");
  VK_REQUIRE(a->nrows == a->ncols, "vk_residual: matrix must be square");
  if (a->nrows == 0) return VK_OK;
  VK_REQUIRE(b && x && r, "vk_residual: null argument");
  cudaError_t e = launch_spmv<1>(*a, x, r, 1.0, 0.0, b, vk_stream(stream));
  if (e != cudaSuccess) {
    vk::set_error("vk_residual: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

extern "C" int vk_csr_to_dense(vk_csr_t a, double* dense, void* stream) {
  VK_REQUIRE(a && dense, "vk_csr_to_dense: null argument");
  if (a->nrows == 0) return VK_OK;
  int grid = std::min(a->nrows, 148 * 8);
  csr_to_dense_kernel<<<grid, 256, 0, vk_stream(stream)>>>(a->nrows, a->ncols, a->indptr,
                                                          a->indices, a->data, dense);
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_residual_restrict(vk_csr_t a, const double* b, const double* x, double* r,
                                    vk_csr_t pt, double* rc, void* stream) {
  VK_REQUIRE(a && pt && b && x && r && rc, "vk_residual_restrict: null argument");
  VK_REQUIRE(a->nrows == a->ncols && pt->ncols == a->nrows,
             "vk_residual_restrict: shape mismatch");
  if (tree_enabled() || a->nblocks == 0 || pt->nblocks == 0) {   // plain two launches
    if (int st = vk_residual(a, b, x, r, stream)) return st;
    return vk_spmv(pt, r, rc, 1.0, 0.0, stream);
  }
  const cudaError_t e = launch_two_phase<1, 0>(*a, phase_of(*a, x, r, 1.0, 0.0, b), *pt,
                                               phase_of(*pt, r, rc, 1.0, 0.0, nullptr),
                                               vk_stream(stream));
  if (e != cudaSuccess) {
    vk::set_error("vk_residual_restrict: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

extern "C" int vk_prolong_residual(vk_csr_t p, const double* xc, double* x, vk_csr_t a,
                                   const double* b, double* r, void* stream) {
  VK_REQUIRE(a && p && b && x && r && xc, "vk_prolong_residual: null argument");
  VK_REQUIRE(a->nrows == a->ncols && p->nrows == a->nrows, "vk_prolong_residual: shape mismatch");
  if (tree_enabled() || a->nblocks == 0 || p->nblocks == 0) {
    if (int st = vk_spmv(p, xc, x, 1.0, 1.0, stream)) return st;
    return vk_residual(a, b, x, r, stream);
  }
  const cudaError_t e = launch_two_phase<0, 1>(*p, phase_of(*p, xc, x, 1.0, 1.0, nullptr), *a,
                                               phase_of(*a, x, r, 1.0, 0.0, b),
                                               vk_stream(stream));
  if (e != cudaSuccess) {
    vk::set_error("vk_prolong_residual: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

extern "C" int vk_csr_max_abs(vk_csr_t a, double* out_host) {
  VK_REQUIRE(a && out_host, "vk_csr_max_abs: null argument");
  std::vector<double> d(a->nnz);
  if (a->nnz)
    VK_CHECK_CUDA(cudaMemcpy(d.data(), a->data, sizeof(double) * a->nnz, cudaMemcpyDeviceToHost));
  double m = 0.0;
  for (double v : d) m = std::max(m, std::fabs(v));
  *out_host = m;
  return VK_OK;
}

extern "C" int vk_csr_export(vk_csr_t a, int32_t* indptr, int32_t* indices, double* data) {
  VK_REQUIRE(a, "vk_csr_export: null handle");
  if (indptr)
    VK_CHECK_CUDA(cudaMemcpy(indptr, a->indptr, sizeof(int32_t) * (a->nrows + 1),
                             cudaMemcpyDeviceToHost));
  if (indices && a->nnz)
    VK_CHECK_CUDA(cudaMemcpy(indices, a->indices, sizeof(int32_t) * a->nnz, cudaMemcpyDeviceToHost));
  if (data && a->nnz)
    VK_CHECK_CUDA(cudaMemcpy(data, a->data, sizeof(double) * a->nnz, cudaMemcpyDeviceToHost));
  return VK_OK;
}
