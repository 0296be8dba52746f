// K5/K6: CSR matrices on the device, SpMV / fused residual / transfers.
//
// Replaces scipy csr_matvec at reference sparsela.py:45-47 (spmv),
// mg.py:41-45 (TransferPair.prolong / restrict, restrict via an explicit
// transposed CSR), mg.py:270, 294 (residual b - A x).
//
// HBM-bound (0.17 flop/B): a sub-warp of VPR lanes owns a row; each lane
// streams UNROLL (col, val) pairs per batch with evict-first loads so the
// L2-resident x / b vectors (<= 5.4 MB) are not displaced by the matrix
// stream; sub-warp shuffle reduction.
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>

#include "vk_common.cuh"

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

__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }

// mode 0: y = alpha*Ax + beta*y   (beta == 0: y not read)
// mode 1: y = b - A x
template <int VPR, int UNROLL, int MODE>
__global__ void __launch_bounds__(256) spmv_kernel(int nrows, const int* __restrict__ ptr,
                                                   const int* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, double alpha,
                                                   double beta, const double* __restrict__ b) {
  const int lane = threadIdx.x & (VPR - 1);
  constexpr int ROWS_PER_WARP = 32 / VPR;
  const int warps_per_block = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int sub = (threadIdx.x & 31) / VPR;
  const int64_t step = int64_t(gridDim.x) * warps_per_block * ROWS_PER_WARP;
  // warp-uniform trip count so every lane reaches the shuffles
  for (int64_t base = (int64_t(blockIdx.x) * warps_per_block + warp) * ROWS_PER_WARP; base < nrows;
       base += step) {
    const int row = static_cast<int>(base) + sub;
    const bool active = row < nrows;
    const int start = active ? __ldg(ptr + row) : 0;
    const int end = active ? __ldg(ptr + row + 1) : 0;
    double sum = 0.0;
    for (int k0 = start + lane; k0 < end; k0 += VPR * UNROLL) {
      int c[UNROLL];
      double v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int k = k0 + u * VPR;
        if (k < end) {
          c[u] = ld_stream(col + k);
          v[u] = ld_stream(val + k);
        } else {
          c[u] = -1;
          v[u] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (c[u] >= 0) sum = fma(v[u], __ldg(x + c[u]), sum);
    }
#pragma unroll
    for (int off = VPR / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off, VPR);
    if (lane == 0 && active) {
      if (MODE == 1) {
        y[row] = __dsub_rn(b[row], sum);
      } else {
        double out = (alpha == 1.0) ? sum : __dmul_rn(alpha, sum);
        if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? y[row] : __dmul_rn(beta, y[row]), out);
        y[row] = out;
      }
    }
  }
}

template <int MODE>
cudaError_t launch_spmv(const vk::Csr& a, const double* x, double* y, double alpha, double beta,
                        const double* b, cudaStream_t st) {
  const int block = 256;
  // lanes per row from the mean row length (P2 ~26, P4/Q3/BDM3 ~60-70,
  // transfers 2-39)
  const double m = a.mean_row;
  int vpr = m > 48 ? 32 : (m > 20 ? 16 : (m > 10 ? 8 : 4));
  const int64_t groups = a.nrows;
  const int per_block = block / vpr;
  int grid = static_cast<int>(std::min<int64_t>((groups + per_block - 1) / per_block, 148 * 64));
  if (grid < 1) grid = 1;
  switch (vpr) {
    case 32:
      spmv_kernel<32, 2, MODE><<<grid, block, 0, st>>>(a.nrows, a.indptr, a.indices, a.data, x, y,
                                                       alpha, beta, b);
      break;
    case 16:
      spmv_kernel<16, 2, MODE><<<grid, block, 0, st>>>(a.nrows, a.indptr, a.indices, a.data, x, y,
                                                       alpha, beta, b);
      break;
    case 8:
      spmv_kernel<8, 2, MODE><<<grid, block, 0, st>>>(a.nrows, a.indptr, a.indices, a.data, x, y,
                                                      alpha, beta, b);
      break;
    default:
      spmv_kernel<4, 2, MODE><<<grid, block, 0, st>>>(a.nrows, a.indptr, a.indices, a.data, x, y,
                                                      alpha, beta, b);
      break;
  }
  return cudaGetLastError();
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

}  // namespace

extern "C" int vk_csr_create(const int32_t* indptr, const int32_t* indices, const double* data,
                             int32_t nrows, int32_t ncols, int64_t nnz, vk_csr_t* out) {
  VK_REQUIRE(out != nullptr && nrows >= 0 && ncols >= 0 && nnz >= 0, "vk_csr_create: bad args");
  VK_REQUIRE(nnz < (int64_t(1) << 31), "vk_csr_create: nnz exceeds int32 indexing");
  auto* a = new vk_csr_s();
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = nnz;
  cudaError_t e = cudaMalloc(&a->indptr, sizeof(int32_t) * (nrows + 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->indices, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->data, sizeof(double) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess)
    e = cudaMemcpy(a->indptr, indptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDefault);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpy(a->indices, indices, sizeof(int32_t) * nnz, cudaMemcpyDefault);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(a->data, data, sizeof(double) * nnz, cudaMemcpyDefault);
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_create: %s", cudaGetErrorString(e));
    cudaFree(a->indptr);
    cudaFree(a->indices);
    cudaFree(a->data);
    delete a;
    return VK_ERR_CUDA;
  }
  // row statistics for the launch heuristic
  std::vector<int32_t> hp(nrows + 1);
  cudaMemcpy(hp.data(), a->indptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDeviceToHost);
  int32_t mx = 0;
  for (int32_t i = 0; i < nrows; ++i) mx = std::max(mx, hp[i + 1] - hp[i]);
  a->max_row = mx;
  a->mean_row = nrows ? double(nnz) / nrows : 0.0;
  *out = a;
  return VK_OK;
}

extern "C" int vk_csr_transpose(vk_csr_t a, vk_csr_t* out) {
  VK_REQUIRE(a && out, "vk_csr_transpose: null handle");
  // Deterministic counting transpose (entries of each output row in
  // ascending source-row order, i.e. the summation order of scipy's
  // csc_matvec on masked.T).  Setup-only; done on the host.
  const int64_t nnz = a->nnz;
  std::vector<int32_t> p(a->nrows + 1), c(nnz);
  std::vector<double> v(nnz);
  VK_CHECK_CUDA(cudaMemcpy(p.data(), a->indptr, sizeof(int32_t) * (a->nrows + 1), cudaMemcpyDeviceToHost));
  if (nnz) {
    VK_CHECK_CUDA(cudaMemcpy(c.data(), a->indices, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
    VK_CHECK_CUDA(cudaMemcpy(v.data(), a->data, sizeof(double) * nnz, cudaMemcpyDeviceToHost));
  }
  std::vector<int32_t> tp(a->ncols + 1, 0), tc(nnz);
  std::vector<double> tv(nnz);
  for (int64_t k = 0; k < nnz; ++k) tp[c[k] + 1]++;
  for (int32_t j = 0; j < a->ncols; ++j) tp[j + 1] += tp[j];
  std::vector<int32_t> cur(tp.begin(), tp.end() - 1);
  for (int32_t i = 0; i < a->nrows; ++i)
    for (int32_t k = p[i]; k < p[i + 1]; ++k) {
      const int32_t dst = cur[c[k]]++;
      tc[dst] = i;
      tv[dst] = v[k];
    }
  return vk_csr_create(tp.data(), tc.data(), tv.data(), a->ncols, a->nrows, nnz, out);
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
  delete a;
  return VK_OK;
}

extern "C" int vk_spmv(vk_csr_t a, const double* x, double* y, double alpha, double beta,
                       void* stream) {
  VK_REQUIRE(a && x && y, "vk_spmv: null argument");
  if (a->nrows == 0) return VK_OK;
  cudaError_t e = launch_spmv<0>(*a, x, y, alpha, beta, nullptr, vk_stream(stream));
  if (e != cudaSuccess) {
    vk::set_error("vk_spmv: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

extern "C" int vk_residual(vk_csr_t a, const double* b, const double* x, double* r, void* stream) {
  VK_REQUIRE(a && b && x && r, "vk_residual: null argument");
  VK_REQUIRE(a->nrows == a->ncols, "vk_residual: matrix must be square");
  if (a->nrows == 0) return VK_OK;
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
