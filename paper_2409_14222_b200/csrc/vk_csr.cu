// K5/K6: CSR matrices on the device, SpMV / fused residual / transfers.
//
// Replaces scipy csr_matvec at reference sparsela.py:45-47 (spmv),
// mg.py:41-45 (TransferPair.prolong / restrict — restrict through an explicit
// transposed CSR), mg.py:270, 294 (residual b - A x).
//
// HBM-bound (0.17 flop/B).  Rows are cut on the host into blocks of <= 2040
// nonzeros / 511 rows, and each block gets a *block-local column
// compression*: the sorted unique columns it touches plus a 16-bit local
// index per nonzero (10 instead of 12 streamed bytes per nonzero, and one
// x-gather per unique column instead of one per nonzero — neighbouring FE
// rows share most columns).  A warp-specialised persistent kernel streams the
// blocks through a TMA ring (csr_ws_kernel).  Each
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

// ---- TMA bulk copy / mbarrier helpers (PTX, sm_90+; compiled for sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Warp-specialised, persistent CSR kernel:
//   warp 0      : one elected thread streams each row block's value,
//                 local-index, unique-column and row-pointer ranges into a
//                 kStages-deep shared-memory ring with cp.async.bulk (TMA),
//                 completion on a per-stage mbarrier;
//   warps 1..4  : gather warps — x at the block's unique columns (L2-resident)
//                 into the stage's x table;
//   warps 5..12 : row warps — one row per thread, summed sequentially left to
//                 right as fl(sum + fl(a_k * x_col(k))) straight out of shared
//                 memory (scipy's order, no FMA), epilogue, release the stage.
// TMA streaming, gathers and the serial row sums of different blocks run
// concurrently; products are never written back, which keeps shared-memory
// traffic at ~28 B per nonzero.
constexpr int kStages = 3;
constexpr int kGatherWarps = 4;
constexpr int kRowWarps = 8;
constexpr int kPipeThreads = 32 * (1 + kGatherWarps + kRowWarps);   // 416

struct PipeLayout {
  int stage_bytes, off_lid, off_ucol, off_ptr, off_xl;
};

template <int MODE>
__global__ void __launch_bounds__(kPipeThreads) csr_ws_kernel(
    int nblk, const int4* __restrict__ info, const int2* __restrict__ uinfo,
    const int* __restrict__ ptr, const double* __restrict__ val, const uint16_t* __restrict__ lidx,
    const int* __restrict__ ucol, const double* __restrict__ x, double* __restrict__ y,
    double alpha, double beta, const double* __restrict__ b, PipeLayout L) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[kStages], xl_bar[kStages], empty_bar[kStages];
  const int warp = threadIdx.x >> 5;
  const int G = gridDim.x;
  auto lo16 = [](int64_t v) { return v & ~int64_t(15); };
  auto hi16 = [](int64_t v) { return (v + 15) & ~int64_t(15); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&xl_bar[s], 32 * kGatherWarps);
      mbar_init(&empty_bar[s], 32 * kRowWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      int c = 0;
      for (int blk = blockIdx.x; blk < nblk; blk += G, ++c) {
        const int s = c % kStages;
        if (c >= kStages) mbar_wait(&empty_bar[s], ((c / kStages) - 1) & 1);
        const int4 in = __ldg(info + blk);
        const int2 uu = __ldg(uinfo + blk);
        unsigned char* st = smem + s * L.stage_bytes;
        if (in.w == 0 || in.w > kStreamNnz) {
          mbar_expect_tx(&full_bar[s], 0);
          continue;
        }
        const int64_t v0 = lo16(int64_t(in.z) * 8), v1 = hi16(int64_t(in.z + in.w) * 8);
        const int64_t l0 = lo16(int64_t(in.z) * 2), l1 = hi16(int64_t(in.z + in.w) * 2);
        const int64_t c0 = lo16(int64_t(uu.x) * 4), c1 = hi16(int64_t(uu.x + uu.y) * 4);
        const int64_t p0 = lo16(int64_t(in.x) * 4), p1 = hi16(int64_t(in.x + in.y + 1) * 4);
        fence_proxy_async();
        mbar_expect_tx(&full_bar[s],
                       static_cast<uint32_t>((v1 - v0) + (l1 - l0) + (c1 - c0) + (p1 - p0)));
        bulk_g2s(st, reinterpret_cast<const char*>(val) + v0, uint32_t(v1 - v0), &full_bar[s], pol);
        bulk_g2s(st + L.off_lid, reinterpret_cast<const char*>(lidx) + l0, uint32_t(l1 - l0),
                 &full_bar[s], pol);
        if (c1 > c0)
          bulk_g2s(st + L.off_ucol, reinterpret_cast<const char*>(ucol) + c0, uint32_t(c1 - c0),
                   &full_bar[s], pol);
        bulk_g2s(st + L.off_ptr, reinterpret_cast<const char*>(ptr) + p0, uint32_t(p1 - p0),
                 &full_bar[s], pol);
      }
    }
  } else if (warp <= kGatherWarps) {
    // ------------------------------------------------------ gather warps
    const int t = threadIdx.x - 32;
    constexpr int NT = 32 * kGatherWarps;
    constexpr int UPT = (kStreamNnz + NT - 1) / NT;
    int c = 0;
    for (int blk = blockIdx.x; blk < nblk; blk += G, ++c) {
      const int s = c % kStages;
      mbar_wait(&full_bar[s], (c / kStages) & 1);
      const int4 in = __ldg(info + blk);
      const int2 uu = __ldg(uinfo + blk);
      if (in.w > 0 && in.w <= kStreamNnz) {
        unsigned char* st = smem + s * L.stage_bytes;
        const int* sucol = reinterpret_cast<const int*>(st + L.off_ucol) + ((int64_t(uu.x) * 4) & 15) / 4;
        double* xl = reinterpret_cast<double*>(st + L.off_xl);
        double xv[UPT];
#pragma unroll
        for (int j = 0; j < UPT; ++j) {
          const int u = t + NT * j;
          xv[j] = (u < uu.y) ? __ldg(x + sucol[u]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < UPT; ++j) {
          const int u = t + NT * j;
          if (u < uu.y) xl[u] = xv[j];
        }
      }
      mbar_arrive(&xl_bar[s]);
    }
  } else {
    // ------------------------------------------------------ row warps
    const int t = threadIdx.x - 32 * (1 + kGatherWarps);
    constexpr int NT = 32 * kRowWarps;
    int c = 0;
    for (int blk = blockIdx.x; blk < nblk; blk += G, ++c) {
      const int s = c % kStages;
      mbar_wait(&xl_bar[s], (c / kStages) & 1);
      const int4 in = __ldg(info + blk);
      if (in.w <= kStreamNnz) {
        unsigned char* st = smem + s * L.stage_bytes;
        const double* sv = reinterpret_cast<const double*>(st) + ((int64_t(in.z) * 8) & 15) / 8;
        const uint16_t* sl = reinterpret_cast<const uint16_t*>(st + L.off_lid) + ((int64_t(in.z) * 2) & 15) / 2;
        const int* sp = reinterpret_cast<const int*>(st + L.off_ptr) + ((int64_t(in.x) * 4) & 15) / 4;
        const double* xl = reinterpret_cast<const double*>(st + L.off_xl);
        for (int i = t; i < in.y; i += NT) {
          const int row = in.x + i;
          // epilogue operand first: its load overlaps the serial sum
          const double pre = (MODE == 1) ? __ldg(b + row) : (beta != 0.0 ? y[row] : 0.0);
          double sum = 0.0;
          if (in.w > 0) {
            const int a = sp[i] - in.z, e = sp[i + 1] - in.z;
            // groups of 8: all shared-memory loads and products first, then
            // the 8 dependent adds (the last group predicated, no tail loop)
            for (int k = a; k < e; k += 8) {
              int l[8];
              double v[8], p[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                l[q] = (k + q < e) ? sl[k + q] : 0;
                v[q] = (k + q < e) ? sv[k + q] : 0.0;
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) p[q] = __dmul_rn(v[q], xl[l[q]]);
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (k + q < e) sum = __dadd_rn(sum, p[q]);
            }
          }
          if (MODE == 1) {
            y[row] = __dsub_rn(pre, sum);
          } else {
            double out = (alpha == 1.0) ? sum : __dmul_rn(alpha, sum);
            if (beta != 0.0) out = __dadd_rn(beta == 1.0 ? pre : __dmul_rn(beta, pre), out);
            y[row] = out;
          }
        }
      }
      mbar_arrive(&empty_bar[s]);
    }
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
  if (a.nblocks > 0) {
    auto r16 = [](int v) { return (v + 15) & ~15; };
    PipeLayout L;
    const int vbytes = r16(8 * (kStreamNnz + 2));
    const int lbytes = r16(2 * (kStreamNnz + 16));
    const int cbytes = r16(4 * (a.max_nu + 8));
    const int pbytes = r16(4 * (a.max_nr + 1 + 8));
    const int xbytes = r16(8 * std::max(a.max_nu, 2));
    L.off_lid = vbytes;
    L.off_ucol = vbytes + lbytes;
    L.off_ptr = vbytes + lbytes + cbytes;
    L.off_xl = vbytes + lbytes + cbytes + pbytes;
    L.stage_bytes = L.off_xl + xbytes;
    const int smem = kStages * L.stage_bytes;
    static int attr_bytes[2] = {48 * 1024, 48 * 1024};
    if (smem > attr_bytes[MODE]) {
      cudaError_t e = cudaFuncSetAttribute(csr_ws_kernel<MODE>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr_bytes[MODE] = smem;
    }
    int nsm = 148, per_sm = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_ws_kernel<MODE>, kPipeThreads, smem);
    const int grid = std::max(1, std::min(a.nblocks, nsm * std::max(per_sm, 1)));
    csr_ws_kernel<MODE><<<grid, kPipeThreads, smem, st>>>(a.nblocks, a.blkinfo, a.blkucol, a.indptr,
                                                          a.data, a.lidx, a.ucol, x, y, alpha, beta,
                                                          b, L);
  }
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
