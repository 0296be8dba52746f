// K5/K6: CSR matrices on the device, SpMV / fused residual / transfers.
//
// Replaces scipy csr_matvec at reference sparsela.py:45-47 (spmv),
// mg.py:41-45 (TransferPair.prolong / restrict — restrict through an explicit
// transposed CSR), mg.py:270, 294 (residual b - A x).
//
// HBM-bound (0.17 flop/B).  Rows are cut on the host into blocks of <= 2040
// nonzeros / 512 rows, and each block gets a *block-local column
// compression*: the sorted unique columns it touches plus a 16-bit local
// index per nonzero (10 instead of 12 streamed bytes per nonzero, and one
// x-gather per unique column instead of one per nonzero — neighbouring FE
// rows share most columns).  Persistent CTAs stream the blocks through a
// three-deep register pipeline (128-bit value / index loads of block i+2,
// x gathers of block i+1, row sums of block i), see csr_pipe_kernel.  Each
// row is summed sequentially, left to right, without FMA:
// y_i = ((0 + a_i0 x_0) + a_i1 x_1) + ... — the exact operation order of
// scipy's csr_matvec (and, through the ascending-source transpose, of
// csc_matvec for masked.T), so SpMV, residual and transfers are
// bit-identical to the reference.
#include <algorithm>
#include <cstdarg>
#include <cstring>
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

using vk::kStreamNnz;
using vk::kStreamRows;
using vk::kStreamThreads;

// MODE 0: y = alpha*Ax + beta*y (beta == 0: y not read);  MODE 1: y = b - A x
template <int MODE>
__device__ __forceinline__ void store_row(int row, double s, double* __restrict__ y, double alpha,
                                          double beta, const double* __restrict__ b) {
  if (MODE == 1) {
    y[row] = __dsub_rn(b[row], s);
  } else {
    double out = (alpha == 1.0) ? s : __dmul_rn(alpha, s);
    if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? y[row] : __dmul_rn(beta, y[row]), out);
    y[row] = out;
  }
}

constexpr int kMaxU = 8;   // unique columns per thread: nu <= 2048

// One row block ("chunk") held in registers while it is in flight.  Thread t
// owns the 16-byte-aligned group of 8 nonzeros starting at (k0 & ~7) + 8t:
// one 128-bit load of local indices and four 128-bit loads of values.
struct ChunkRegs {
  int4 info;           // r0, nrows, k0, nnz   (nnz = 0: no chunk)
  int2 uu;             // u0, nu
  uint4 lid;
  double2 v[4];
  int uc[kMaxU];
  int p0, p1;          // row pointers of rows t and t + 256
};

__device__ __forceinline__ void load_chunk(int blk, int nblk, ChunkRegs& c, const int4* __restrict__ info,
                                           const int2* __restrict__ uinfo, const int* __restrict__ ptr,
                                           const double* __restrict__ val,
                                           const uint16_t* __restrict__ lidx,
                                           const int* __restrict__ ucol) {
  const int t = threadIdx.x;
  if (blk >= nblk) {
    c.info = make_int4(0, 0, 0, 0);
    c.uu = make_int2(0, 0);
    return;
  }
  c.info = __ldg(info + blk);
  c.uu = __ldg(uinfo + blk);
  const int k0 = c.info.z, nnz = c.info.w;
  if (nnz > kStreamNnz) {      // a single long row: csr_longrow_kernel
    c.info.w = 0;
    c.info.y = 0;
    c.uu.y = 0;
    return;
  }
  const int e = (k0 & ~7) + 8 * t;
  if (e < k0 + nnz) {
    c.lid = __ldcs(reinterpret_cast<const uint4*>(lidx + e));
    const double2* vp = reinterpret_cast<const double2*>(val + e);
#pragma unroll
    for (int q = 0; q < 4; ++q) c.v[q] = __ldcs(vp + q);
  }
#pragma unroll
  for (int j = 0; j < kMaxU; ++j) {
    const int u = t + kStreamThreads * j;
    c.uc[j] = (u < c.uu.y) ? __ldg(ucol + c.uu.x + u) : 0;
  }
  c.p0 = (t <= c.info.y) ? __ldg(ptr + c.info.x + t) : 0;
  c.p1 = (t + kStreamThreads <= c.info.y) ? __ldg(ptr + c.info.x + t + kStreamThreads) : 0;
}

__device__ __forceinline__ int lid_of(const uint4& l, int j) {
  const unsigned w = (j < 2) ? l.x : (j < 4) ? l.y : (j < 6) ? l.z : l.w;
  return (j & 1) ? int(w >> 16) : int(w & 0xffffu);
}

// One 256-thread CTA per row block (up to 8 resident per SM):
//   (1) 128-bit loads of the block's local indices / values and the
//       unique-column list, one group of 8 nonzeros per thread;
//   (2) one x-gather per unique column (L2-resident x) into shared memory;
//   (3) products a_k * x_col(k) from the shared x table;
//   (4) sequential, FMA-free row sums (scipy's order).
template <int MODE>
__global__ void __launch_bounds__(kStreamThreads) csr_blk_kernel(
    int nblk, const int4* __restrict__ info, const int2* __restrict__ uinfo,
    const int* __restrict__ ptr, const double* __restrict__ val, const uint16_t* __restrict__ lidx,
    const int* __restrict__ ucol, const double* __restrict__ x, double* __restrict__ y,
    double alpha, double beta, const double* __restrict__ b) {
  __shared__ double prod[kStreamNnz + 8];
  __shared__ double xl[kStreamThreads * kMaxU];
  __shared__ int sptr[kStreamRows + 1];
  const int t = threadIdx.x;
  const int blk = blockIdx.x;
  ChunkRegs c;
  load_chunk(blk, nblk, c, info, uinfo, ptr, val, lidx, ucol);
  double xv[kMaxU];
#pragma unroll
  for (int j = 0; j < kMaxU; ++j) {
    const int u = t + kStreamThreads * j;
    xv[j] = (u < c.uu.y) ? __ldg(x + c.uc[j]) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < kMaxU; ++j) {
    const int u = t + kStreamThreads * j;
    if (u < c.uu.y) xl[u] = xv[j];
  }
  if (t <= c.info.y) sptr[t] = c.p0;
  if (t + kStreamThreads <= c.info.y) sptr[t + kStreamThreads] = c.p1;
  __syncthreads();
  if (c.info.w > 0) {
    const int k0 = c.info.z;
    const int e = (k0 & ~7) + 8 * t;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = e + j - k0;
      if (k >= 0 && k < c.info.w) {
        const double vj = (j & 1) ? c.v[j >> 1].y : c.v[j >> 1].x;
        prod[k] = __dmul_rn(vj, xl[lid_of(c.lid, j)]);
      }
    }
  }
  __syncthreads();
  const int4 ci = c.info;
  if (__ldg(&info[blk].w) > kStreamNnz) return;     // long row: csr_longrow_kernel
  for (int i = t; i < ci.y; i += kStreamThreads) {
    const int a = sptr[i] - ci.z, e = sptr[i + 1] - ci.z;
    double sum = 0.0;
    for (int k = a; k < e; ++k) sum = __dadd_rn(sum, prod[k]);
    store_row<MODE>(ci.x + i, sum, y, alpha, beta, b);
  }
}

// rows longer than one block (never in the FE operators, kept for generality)
template <int MODE>
__global__ void csr_longrow_kernel(const int* __restrict__ rows, int nlong, const int* __restrict__ ptr,
                                   const int* __restrict__ col, const double* __restrict__ val,
                                   const double* __restrict__ x, double* __restrict__ y, double alpha,
                                   double beta, const double* __restrict__ b) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nlong; q += gridDim.x * blockDim.x) {
    const int row = rows[q];
    double s = 0.0;
    for (int k = ptr[row]; k < ptr[row + 1]; ++k) s = __dadd_rn(s, __dmul_rn(val[k], x[col[k]]));
    store_row<MODE>(row, s, y, alpha, beta, b);
  }
}

template <int MODE>
cudaError_t launch_spmv(const vk::Csr& a, const double* x, double* y, double alpha, double beta,
                        const double* b, cudaStream_t st) {
  if (a.nblocks > 0)
    csr_blk_kernel<MODE><<<a.nblocks, kStreamThreads, 0, st>>>(a.nblocks, a.blkinfo, a.blkucol, a.indptr,
                                                              a.data, a.lidx, a.ucol, x, y, alpha, beta, b);
  if (a.nlong > 0)
    csr_longrow_kernel<MODE><<<std::min((a.nlong + 127) / 128, 148), 128, 0, st>>>(
        a.longrows, a.nlong, a.indptr, a.indices, a.data, x, y, alpha, beta, b);
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

// Row blocks: <= kStreamNnz nonzeros and <= kStreamRows rows.  A row longer
// than kStreamNnz is diverted to the long-row list.
void make_row_blocks(const std::vector<int32_t>& p, std::vector<int32_t>& rb,
                     std::vector<int32_t>& longrows) {
  const int32_t n = static_cast<int32_t>(p.size()) - 1;
  rb.assign(1, 0);
  int32_t r = 0;
  while (r < n) {
    const int32_t start = r;
    int64_t nnz = 0;
    // <= 511 rows: the 512 row pointers of a block are two per thread
    while (r < n && r - start < kStreamRows - 1) {
      const int64_t len = p[r + 1] - p[r];
      if (len > kStreamNnz) break;
      if (nnz + len > kStreamNnz) break;
      nnz += len;
      ++r;
    }
    if (r == start) {  // a long row: its own block, skipped by the block kernel
      longrows.push_back(r);
      ++r;
      rb.push_back(r);
      continue;
    }
    rb.push_back(r);
  }
}

}  // namespace

extern "C" int vk_csr_create(const int32_t* indptr, const int32_t* indices, const double* data,
                             int32_t nrows, int32_t ncols, int64_t nnz, vk_csr_t* out) {
  VK_REQUIRE(out != nullptr && nrows >= 0 && ncols >= 0 && nnz >= 0, "vk_csr_create: bad args");
  VK_REQUIRE(nnz < (int64_t(1) << 31), "vk_csr_create: nnz exceeds int32 indexing");
  std::vector<int32_t> hp(nrows + 1), hc(nnz);
  cudaError_t e = cudaMemcpy(hp.data(), indptr, sizeof(int32_t) * (nrows + 1), cudaMemcpyDefault);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(hc.data(), indices, sizeof(int32_t) * nnz, cudaMemcpyDefault);
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_create: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  VK_REQUIRE(hp[0] == 0 && hp[nrows] == nnz, "vk_csr_create: indptr does not match nnz");
  for (int32_t i = 0; i < nrows; ++i) {
    VK_REQUIRE(hp[i + 1] >= hp[i], "vk_csr_create: indptr must be nondecreasing");
    for (int32_t k = hp[i]; k < hp[i + 1]; ++k)
      VK_REQUIRE(hc[k] >= 0 && hc[k] < ncols && (k == hp[i] || hc[k] > hc[k - 1]),
                 "vk_csr_create: row %d column indices must be sorted, unique and in range", i);
  }
  std::vector<int32_t> rb, longrows;
  make_row_blocks(hp, rb, longrows);
  // block-local column compression
  const int32_t nb = static_cast<int32_t>(rb.size()) - 1;
  std::vector<int32_t> up(nb + 1, 0), uc;
  std::vector<uint16_t> li(nnz + 16, 0);
  std::vector<int32_t> tmp;
  for (int32_t bk = 0; bk < nb; ++bk) {
    const int32_t a = hp[rb[bk]], z = hp[rb[bk + 1]];
    if (z - a <= kStreamNnz) {
      tmp.assign(hc.begin() + a, hc.begin() + z);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      for (int32_t k = a; k < z; ++k)
        li[k] = static_cast<uint16_t>(std::lower_bound(tmp.begin(), tmp.end(), hc[k]) - tmp.begin());
      uc.insert(uc.end(), tmp.begin(), tmp.end());
    }
    up[bk + 1] = static_cast<int32_t>(uc.size());
  }
  std::vector<int4> info(std::max(nb, 1));
  std::vector<int2> uinfo(std::max(nb, 1));
  int32_t max_nu = 0, max_nr = 0;
  for (int32_t bk = 0; bk < nb; ++bk) {
    info[bk] = make_int4(rb[bk], rb[bk + 1] - rb[bk], hp[rb[bk]], hp[rb[bk + 1]] - hp[rb[bk]]);
    uinfo[bk] = make_int2(up[bk], up[bk + 1] - up[bk]);
    max_nu = std::max(max_nu, up[bk + 1] - up[bk]);
    max_nr = std::max(max_nr, rb[bk + 1] - rb[bk]);
  }
  auto* a = new vk_csr_s();
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = nnz;
  a->nblocks = nb;
  a->nucol = static_cast<int64_t>(uc.size());
  a->nlong = static_cast<int32_t>(longrows.size());
  a->max_nu = max_nu;
  a->max_nr = max_nr;
  // +16 B slack on every TMA-streamed array (16-byte aligned superset copies)
  hp.resize(nrows + 1 + 4, hp[nrows]);
  uc.resize(uc.size() + 4, 0);
  e = cudaMalloc(&a->indptr, sizeof(int32_t) * hp.size());
  if (e == cudaSuccess) e = cudaMalloc(&a->blkinfo, sizeof(int4) * info.size());
  if (e == cudaSuccess) e = cudaMalloc(&a->blkucol, sizeof(int2) * uinfo.size());
  if (e == cudaSuccess) e = cudaMemcpy(a->blkinfo, info.data(), sizeof(int4) * info.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->blkucol, uinfo.data(), sizeof(int2) * uinfo.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&a->indices, sizeof(int32_t) * std::max<int64_t>(nnz, 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->data, sizeof(double) * (nnz + 8));
  if (e == cudaSuccess) e = cudaMalloc(&a->rowblk, sizeof(int32_t) * rb.size());
  if (e == cudaSuccess) e = cudaMalloc(&a->ucolptr, sizeof(int32_t) * up.size());
  if (e == cudaSuccess) e = cudaMalloc(&a->ucol, sizeof(int32_t) * std::max<size_t>(uc.size(), 1));
  if (e == cudaSuccess) e = cudaMalloc(&a->lidx, sizeof(uint16_t) * li.size());
  if (e == cudaSuccess && !longrows.empty())
    e = cudaMalloc(&a->longrows, sizeof(int32_t) * longrows.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(a->indptr, hp.data(), sizeof(int32_t) * hp.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->rowblk, rb.data(), sizeof(int32_t) * rb.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->ucolptr, up.data(), sizeof(int32_t) * up.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !uc.empty())
    e = cudaMemcpy(a->ucol, uc.data(), sizeof(int32_t) * uc.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->lidx, li.data(), sizeof(uint16_t) * li.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !longrows.empty())
    e = cudaMemcpy(a->longrows, longrows.data(), sizeof(int32_t) * longrows.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpy(a->indices, hc.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(a->data, data, sizeof(double) * nnz, cudaMemcpyDefault);
  if (e == cudaSuccess) e = cudaMemset(a->data + nnz, 0, sizeof(double) * 8);
  if (e != cudaSuccess) {
    vk::set_error("vk_csr_create: %s", cudaGetErrorString(e));
    vk_csr_destroy(a);
    return VK_ERR_CUDA;
  }
  int32_t mx = 0;
  for (int32_t i = 0; i < nrows; ++i) mx = std::max(mx, hp[i + 1] - hp[i]);
  a->max_row = mx;
  a->mean_row = nrows ? double(nnz) / nrows : 0.0;
  *out = a;
  return VK_OK;
}

extern "C" int vk_csr_transpose(vk_csr_t a, vk_csr_t* out) {
  VK_REQUIRE(a && out, "vk_csr_transpose: null handle");
  // Deterministic counting transpose: the entries of each output row come in
  // ascending source-row order, i.e. the accumulation order of scipy's
  // csc_matvec on masked.T (mg.py:44-45).  Setup-only; done on the host.
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
  cudaFree(a->rowblk);
  cudaFree(a->ucolptr);
  cudaFree(a->ucol);
  cudaFree(a->lidx);
  cudaFree(a->longrows);
  cudaFree(a->blkinfo);
  cudaFree(a->blkucol);
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
