// Vector / dense helpers for the device-resident FGMRES and V-cycle
// (reference sparsela.fgmres, sparsela.py:117-191; NullspaceProjector,
// sparsela.py:99-114; coarse_solve, mg.py:274-279; v_cycle bc copy,
// mg.py:298-300).  Reductions are deterministic: fixed grid, fixed
// per-thread order, tree in shared memory, last-arriving block combines the
// block partials in index order (one launch, graph-capturable; the arrival
// counter resets itself).  The block partials and the arrival counter live in
// a caller-owned scratch buffer (VK_REDUCE_SCRATCH doubles, zero-filled once):
// reductions in flight on different streams never share state, so the calls
// are re-entrant across streams as the header promises.
#include <algorithm>

#include "vk_common.cuh"

namespace {

constexpr int kRedBlock = 256;
constexpr int kRedGrid = 296;

static_assert(kRedGrid + 2 <= VK_REDUCE_SCRATCH, "scratch too small");

// scratch layout: [0, kRedGrid) block partials, [kRedGrid] arrival counter
// (as an unsigned int), [kRedGrid + 1] a spare scalar (vk_project's q.x)
__device__ __forceinline__ unsigned int* arrive_of(double* scratch) {
  return reinterpret_cast<unsigned int*>(scratch + kRedGrid);
}

// last-arriving block combines the partials in block order
__device__ __forceinline__ void grid_finish(double bs, double* sh, double* scratch, double* out,
                                            bool fin_sqrt) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    scratch[blockIdx.x] = bs;
    __threadfence();
    const unsigned int ticket = atomicAdd(arrive_of(scratch), 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double v = 0.0;
    for (int b = threadIdx.x; b < gridDim.x; b += kRedBlock)
      v = __dadd_rn(v, *((volatile double*)&scratch[b]));
    __syncthreads();
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = kRedBlock / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *out = fin_sqrt ? sqrt(sh[0]) : sh[0];
      *arrive_of(scratch) = 0u;
    }
  }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int t = threadIdx.x;
  sh[t] = v;
  __syncthreads();
  for (int o = kRedBlock / 2; o > 0; o >>= 1) {
    if (t < o) sh[t] = __dadd_rn(sh[t], sh[t + o]);
    __syncthreads();
  }
  return sh[0];
}

// FIN: 0 = dot, 1 = sqrt(dot)
template <int FIN>
__global__ void __launch_bounds__(kRedBlock) dot_kernel(int64_t n, const double* __restrict__ x,
                                                        const double* __restrict__ y,
                                                        double* __restrict__ out,
                                                        double* scratch) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sh[kRedBlock];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * int64_t(kRedBlock) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kRedBlock)
    acc = fma(x[i], y[i], acc);
  const double bs = block_sum(acc, sh);
  grid_finish(bs, sh, scratch, out, FIN != 0);
}

// y -= a x, then the dot of x2 with the updated y: element i is owned by the
// same thread as in dot_kernel (grid kRedGrid x kRedBlock, grid-stride), so
// the per-thread fma order and the reduction are those of dot_kernel.
template <int FIN>
__global__ void __launch_bounds__(kRedBlock) axpy_dot_kernel(int64_t n, const double* __restrict__ a,
                                                             const double* __restrict__ x,
                                                             double* y, const double* x2,
                                                             double* __restrict__ out,
                                                             double* scratch) {
  pdl_trigger();
  pdl_wait();
  __shared__ double sh[kRedBlock];
  const double av = *a;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * int64_t(kRedBlock) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * kRedBlock) {
    const double yn = __dsub_rn(y[i], __dmul_rn(av, x[i]));
    y[i] = yn;
    acc = fma(x2 == y ? yn : x2[i], yn, acc);
  }
  const double bs = block_sum(acc, sh);
  grid_finish(bs, sh, scratch, out, FIN != 0);
}

__global__ void axpy_dev_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ x,
                                double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const double av = *a;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __dsub_rn(y[i], __dmul_rn(av, x[i]));
}

__global__ void axpy_kernel(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

__global__ void div_dev_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ d,
                               double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const double dv = *d;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __ddiv_rn(x[i], dv);
}

__global__ void copy_index_kernel(int64_t m, const int* __restrict__ idx, const double* __restrict__ src,
                                  double* __restrict__ dst) {
  pdl_trigger();
  pdl_wait();
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m; k += int64_t(gridDim.x) * blockDim.x) {
    const int i = idx[k];
    dst[i] = src[i];
  }
}

// y = M x, dense row-major: one warp per row, 128-bit loads where aligned.
__global__ void __launch_bounds__(256) gemv_kernel(int m, int n, const double* __restrict__ mat,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < m; row += nw) {
    const double* a = mat + int64_t(row) * n;
    double acc = 0.0;
    if ((n & 1) == 0) {
      const double2* a2 = reinterpret_cast<const double2*>(a);
      const double2* x2 = reinterpret_cast<const double2*>(x);
      for (int j = lane; j < n / 2; j += 32) {
        const double2 av = __ldcs(a2 + j);
        const double2 xv = __ldg(x2 + j);
        acc = fma(av.x, xv.x, acc);
        acc = fma(av.y, xv.y, acc);
      }
    } else {
      for (int j = lane; j < n; j += 32) acc = fma(__ldcs(a + j), __ldg(x + j), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = acc;
  }
}

// x += sum_k c[k] * Z[k, :]  in ascending k
__global__ void combine_kernel(int64_t n, int count, const double* __restrict__ z, const double* __restrict__ c,
                               double* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int k = 0; k < count; ++k) acc = fma(c[k], z[int64_t(k) * n + i], acc);
    x[i] = __dadd_rn(x[i], acc);
  }
}

// Chebyshev vector update (reference mg.py:246-254): first: d = z / c2,
// else d = c1 * d + c2 * z; then x = x + d (elementwise, reference order)
__global__ void cheb_update_kernel(int64_t n, const double* __restrict__ z, double* __restrict__ d,
                                   double* __restrict__ x, double c1, double c2, int first) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double dn = first ? __ddiv_rn(z[i], c2) : __dadd_rn(__dmul_rn(c1, d[i]), __dmul_rn(c2, z[i]));
    d[i] = dn;
    x[i] = __dadd_rn(x[i], dn);
  }
}

__global__ void project_apply_kernel(int64_t n, const double* __restrict__ q, const double* __restrict__ s,
                                     double* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
  const double sv = *s;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = __dsub_rn(x[i], __dmul_rn(q[i], sv));
}

}  // namespace

#define VK_VEC_GRID(n) vk_grid((n), 256, 148 * 8)

extern "C" int vk_dot(int64_t n, const double* x, const double* y, double* out_dev,
                      double* scratch_dev, void* stream) {
  VK_REQUIRE(out_dev && scratch_dev && n >= 0 && (n == 0 || (x && y)), "vk_dot: bad argument");
  VK_CHECK_CUDA(vk_launch(dot_kernel<0>, dim3(kRedGrid), dim3(kRedBlock), 0, vk_stream(stream), 16 * n, n, x, y, out_dev, scratch_dev));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_nrm2(int64_t n, const double* x, double* out_dev, double* scratch_dev,
                       void* stream) {
  VK_REQUIRE(out_dev && scratch_dev && n >= 0 && (n == 0 || x), "vk_nrm2: bad argument");
  VK_CHECK_CUDA(vk_launch(dot_kernel<1>, dim3(kRedGrid), dim3(kRedBlock), 0, vk_stream(stream), 8 * n, n, x, x, out_dev, scratch_dev));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_axpy_dev(int64_t n, const double* a_dev, const double* x, double* y, void* stream) {
  VK_REQUIRE(a_dev && (n == 0 || (x && y)), "vk_axpy_dev: null argument");
  if (n == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(axpy_dev_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 24 * n, n, a_dev, x, y));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_axpy_dot(int64_t n, const double* a_dev, const double* x, double* y, const double* x2,
                           double* out_dev, int32_t sqrt_out, double* scratch_dev, void* stream) {
  VK_REQUIRE(a_dev && out_dev && scratch_dev && n >= 0 && (n == 0 || (x && y && x2)),
             "vk_axpy_dot: bad argument");
  if (sqrt_out)
    VK_CHECK_CUDA(vk_launch(axpy_dot_kernel<1>, dim3(kRedGrid), dim3(kRedBlock), 0, vk_stream(stream), 8 * n, n, a_dev, x, y, x2, out_dev, scratch_dev));
  else
    VK_CHECK_CUDA(vk_launch(axpy_dot_kernel<0>, dim3(kRedGrid), dim3(kRedBlock), 0, vk_stream(stream), 16 * n, n, a_dev, x, y, x2, out_dev, scratch_dev));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_axpy(int64_t n, double a, const double* x, double* y, void* stream) {
  VK_REQUIRE(x && y, "vk_axpy: null argument");
  if (n == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(axpy_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 24 * n, n, a, x, y));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_div_dev(int64_t n, const double* x, const double* d_dev, double* y, void* stream) {
  VK_REQUIRE(x && d_dev && y, "vk_div_dev: null argument");
  if (n == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(div_dev_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 16 * n, n, x, d_dev, y));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_project(int64_t n, const double* q, double* x, double* scratch_dev, void* stream) {
  VK_REQUIRE(q && x && scratch_dev, "vk_project: null argument");
  if (n == 0) return VK_OK;
  double* qx = scratch_dev + kRedGrid + 1;
  VK_CHECK_CUDA(vk_launch(dot_kernel<0>, dim3(kRedGrid), dim3(kRedBlock), 0, vk_stream(stream), 16 * n, n, q, x, qx, scratch_dev));
  VK_CHECK_CUDA(vk_launch(project_apply_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 24 * n, n, q, (const double*)qx, x));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_copy_index(int64_t m, const int32_t* idx, const double* src, double* dst, void* stream) {
  VK_REQUIRE(idx && src && dst, "vk_copy_index: null argument");
  if (m == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(copy_index_kernel, dim3(VK_VEC_GRID(m)), dim3(256), 0, vk_stream(stream), 20 * m, m, idx, src, dst));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_gemv(int32_t m, int32_t n, const double* mat, const double* x, double* y, void* stream) {
  VK_REQUIRE(mat && x && y && m >= 0 && n >= 0, "vk_gemv: bad argument");
  if (m == 0) return VK_OK;
  const int grid = std::min((m + 7) / 8, 148 * 8);
  VK_CHECK_CUDA(vk_launch(gemv_kernel, dim3(grid), dim3(256), 0, vk_stream(stream), 8 * int64_t(m) * n, m, n, mat, x, y));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_combine(int64_t n, int32_t count, const double* z, const double* coef_dev, double* x,
                          void* stream) {
  VK_REQUIRE(z && coef_dev && x, "vk_combine: null argument");
  if (n == 0 || count == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(combine_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 8 * n * (int64_t(count) + 2), n, count, z, coef_dev, x));
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_cheb_update(int64_t n, const double* z, double* d, double* x, double c1,
                              double c2, int32_t first, void* stream) {
  VK_REQUIRE(z && d && x, "vk_cheb_update: null argument");
  if (n == 0) return VK_OK;
  VK_CHECK_CUDA(vk_launch(cheb_update_kernel, dim3(VK_VEC_GRID(n)), dim3(256), 0, vk_stream(stream), 32 * n, n, z, d, x, c1, c2, int(first != 0)));
  VK_CHECK_LAUNCH();
  return VK_OK;
}
