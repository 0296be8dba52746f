// Discretisation-error measurement of a solved system against the
// manufactured enclosed-flow solution (reference bench.py:95-164,
// `error_norms`): broken-H1 velocity error and its base, largest pointwise
// divergence, mean-free pressure L2 error, and for H(div) pairs the
// tangential-jump seminorm over the interior edges.
//
// One thread per (cell, quadrature point) evaluates u_h, grad u_h and p_h from
// the reference tabulation pushed forward by that point's Jacobian (identity
// or Piola, as in assembly) and the exact velocity / gradient at the mapped
// point (assembly.py:65-81); one thread per (interior edge, point) the jump of
// the tangential trace.  The per-point terms go to scratch arrays and ONE CTA
// reduces them in a fixed order (deterministic), the pressure in two passes
// like the reference (mean first, then sum w (p - mean)^2).
#include "vk_common.cuh"
#include "vk_fem.cuh"

namespace {

constexpr int kPointThreads = 128;
constexpr int kReduceThreads = 1024;

struct ErrArgs {
  int ncells, nq, nv, np, quad, piola, nvert, poffset;
  const double *w, *pts, *rv, *rg, *pv;   // w[nq], pts[nq][2], rv[nq][nv][2], rg[nq][nv][2][2],
                                          // pv[nq][np]
  const double* cell_xy;                  // [ncells][nvert][2]
  const int *vdofs, *pdofs;
  const double *vscale, *pscale;
  const double* x;                        // the solution vector
  double* work;                           // [5][ncells*nq]: e2, b2, |div|, p, w det
};

__global__ void __launch_bounds__(kPointThreads) error_points_kernel(ErrArgs a) {
  const int64_t total = int64_t(a.ncells) * a.nq;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(t / a.nq), q = int(t % a.nq);
    const double* xy = a.cell_xy + int64_t(c) * a.nvert * 2;
    const double xi = a.pts[2 * q], eta = a.pts[2 * q + 1];
    double J[2][2], det, inv[2][2];
    jacobian(a.quad, xy, xi, eta, J, det, inv);
    double uh[2] = {0.0, 0.0}, gh[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int* gv = a.vdofs + int64_t(c) * a.nv;
    const double* sv = a.vscale + int64_t(c) * a.nv;
    for (int i = 0; i < a.nv; ++i) {
      const double* rv = a.rv + (int64_t(q) * a.nv + i) * 2;
      const double* rg = a.rg + (int64_t(q) * a.nv + i) * 4;
      const double rvv[2] = {__ldg(rv), __ldg(rv + 1)};
      const double rgg[2][2] = {{__ldg(rg), __ldg(rg + 1)}, {__ldg(rg + 2), __ldg(rg + 3)}};
      double pv[2], pg[2][2];
      push(a.piola, J, det, inv, rvv, rgg, pv, pg);
      const double coef = sv[i] * a.x[gv[i]];                   // bench.py:129
      uh[0] += pv[0] * coef;
      uh[1] += pv[1] * coef;
      gh[0][0] += pg[0][0] * coef;
      gh[0][1] += pg[0][1] * coef;
      gh[1][0] += pg[1][0] * coef;
      gh[1][1] += pg[1][1] * coef;
    }
    double ph = 0.0;
    if (a.np) {
      const int* gq = a.pdofs + int64_t(c) * a.np;
      const double* sq = a.pscale + int64_t(c) * a.np;
      for (int p = 0; p < a.np; ++p)
        ph += __ldg(a.pv + int64_t(q) * a.np + p) * (sq[p] * a.x[int64_t(a.poffset) + gq[p]]);
    }
    double px, py;
    map_point(a.quad, xy, xi, eta, px, py);
    double sx, cx, sy, cy;
    sincos(M_PI * px, &sx, &cx);
    sincos(M_PI * py, &sy, &cy);
    const double ue[2] = {sx * cy, -(cx * sy)};                 // assembly.py:65-69
    const double ge[2][2] = {{M_PI * cx * cy, -(M_PI * sx * sy)},
                             {M_PI * sx * sy, -(M_PI * cx * cy)}};   // assembly.py:72-80
    double e2 = 0.0, b2 = 0.0;
    for (int v = 0; v < 2; ++v) {
      e2 += (uh[v] - ue[v]) * (uh[v] - ue[v]);
      b2 += ue[v] * ue[v];
    }
    double g2 = 0.0, gb2 = 0.0;
    for (int v = 0; v < 2; ++v)
      for (int d = 0; d < 2; ++d) {
        g2 += (gh[v][d] - ge[v][d]) * (gh[v][d] - ge[v][d]);
        gb2 += ge[v][d] * ge[v][d];
      }
    const double wd = a.w[q] * det;
    a.work[t] = wd * (e2 + g2);
    a.work[total + t] = wd * (b2 + gb2);
    a.work[2 * total + t] = fabs(gh[0][0] + gh[1][1]);
    a.work[3 * total + t] = ph;
    a.work[4 * total + t] = wd;
  }
}

struct JumpArgs {
  int nedges, nq, nv;
  const double* w;           // [nq] interval weights
  const double* rv;          // [6][nq][nv][2]: (slot, aligned) reference tables
  const int* info;           // [nedges][6]: c1, c2, slot1, aligned1, slot2, aligned2
  const double* geo;         // [nedges][5]: tx, ty, n1x, n1y, h_e
  const double* cell_xy;     // [ncells][3][2]
  const int* vdofs;
  const double* vscale;
  const double* x;
  double* work;              // [nedges*nq]: w_q h_e [v.t]^2 / (2 h_e)
};

__global__ void __launch_bounds__(kPointThreads) error_jump_kernel(JumpArgs a) {
  const int64_t total = int64_t(a.nedges) * a.nq;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(t / a.nq), q = int(t % a.nq);
    const int* inf = a.info + int64_t(e) * 6;
    const double* g = a.geo + int64_t(e) * 5;
    const double t0 = g[0], t1 = g[1], h = g[4];
    double trace[2];
    for (int s = 0; s < 2; ++s) {
      const int cell = inf[s], tab = inf[2 + 2 * s] * 2 + inf[3 + 2 * s];
      const double* xy = a.cell_xy + int64_t(cell) * 6;
      double J[2][2], det, inv[2][2];
      jacobian(0, xy, 0.0, 0.0, J, det, inv);
      const int* gv = a.vdofs + int64_t(cell) * a.nv;
      const double* sv = a.vscale + int64_t(cell) * a.nv;
      double acc = 0.0;
      for (int i = 0; i < a.nv; ++i) {
        const double* rv = a.rv + ((int64_t(tab) * a.nq + q) * a.nv + i) * 2;
        const double r0 = __ldg(rv), r1 = __ldg(rv + 1);
        const double p0 = (J[0][0] * r0 + J[0][1] * r1) / det;
        const double p1 = (J[1][0] * r0 + J[1][1] * r1) / det;
        acc += (p0 * t0 + p1 * t1) * (sv[i] * a.x[gv[i]]);      // bench.py:151-154
      }
      trace[s] = acc;
    }
    const double dvt = trace[0] - trace[1];
    a.work[t] = (a.w[q] * h) * (dvt * dvt) * 0.5 / h;           // bench.py:157
  }
}

// fixed-order block reduction: thread-strided partials, then a shared tree
template <bool MAX>
__device__ double block_reduce(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = kReduceThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      sh[threadIdx.x] = MAX ? fmax(sh[threadIdx.x], sh[threadIdx.x + s])
                            : sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// out[0..5] = sum e2, sum b2, max |div|, sum w (p - mean)^2, sum jump terms, mean
__global__ void __launch_bounds__(kReduceThreads) error_reduce_kernel(
    int64_t ncq, const double* __restrict__ work, int64_t neq, const double* __restrict__ jump,
    double* __restrict__ out) {
  __shared__ double sh[kReduceThreads];
  double e2 = 0.0, b2 = 0.0, dv = 0.0, wp = 0.0, ws = 0.0;
  for (int64_t t = threadIdx.x; t < ncq; t += kReduceThreads) {
    e2 += work[t];
    b2 += work[ncq + t];
    dv = fmax(dv, work[2 * ncq + t]);
    wp += work[4 * ncq + t] * work[3 * ncq + t];
    ws += work[4 * ncq + t];
  }
  e2 = block_reduce<false>(e2, sh);
  b2 = block_reduce<false>(b2, sh);
  dv = block_reduce<true>(dv, sh);
  wp = block_reduce<false>(wp, sh);
  ws = block_reduce<false>(ws, sh);
  const double mean = ws != 0.0 ? wp / ws : 0.0;                // bench.py:138
  double pe = 0.0;
  for (int64_t t = threadIdx.x; t < ncq; t += kReduceThreads) {
    const double d = work[3 * ncq + t] - mean;
    pe += work[4 * ncq + t] * (d * d);                          // bench.py:139
  }
  pe = block_reduce<false>(pe, sh);
  double jp = 0.0;
  for (int64_t t = threadIdx.x; t < neq; t += kReduceThreads) jp += jump[t];
  jp = block_reduce<false>(jp, sh);
  if (threadIdx.x == 0) {
    out[0] = e2;
    out[1] = b2;
    out[2] = dv;
    out[3] = pe;
    out[4] = jp;
    out[5] = mean;
  }
}

}  // namespace

extern "C" int vk_error_cells(int32_t ncells, int32_t nq, int32_t nv, int32_t np, int32_t quad,
                              int32_t piola, const double* w, const double* pts, const double* rv,
                              const double* rg, const double* pv, const double* cell_xy,
                              const int32_t* vdofs, const double* vscale, const int32_t* pdofs,
                              const double* pscale, int32_t poffset, const double* x,
                              double* work, void* stream) {
  VK_REQUIRE(ncells >= 0 && nq > 0 && nv > 0 && np >= 0 && w && pts && rv && rg && cell_xy &&
                 vdofs && vscale && x && work && (np == 0 || (pv && pdofs && pscale)),
             "vk_error_cells: bad argument");
  if (ncells == 0) return VK_OK;
  ErrArgs a{ncells, nq, nv, np, quad, piola, quad ? 4 : 3, poffset, w, pts, rv, rg, pv, cell_xy,
            vdofs, pdofs, vscale, pscale, x, work};
  error_points_kernel<<<vk_grid(int64_t(ncells) * nq, kPointThreads, 148 * 16), kPointThreads, 0,
                        vk_stream(stream)>>>(a);
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_error_jump(int32_t nedges, int32_t nq, int32_t nv, const double* w,
                             const double* rv, const int32_t* info, const double* geo,
                             const double* cell_xy, const int32_t* vdofs, const double* vscale,
                             const double* x, double* work, void* stream) {
  VK_REQUIRE(nedges >= 0 && nq > 0 && nv > 0 && w && rv && info && geo && cell_xy && vdofs &&
                 vscale && x && work,
             "vk_error_jump: bad argument");
  if (nedges == 0) return VK_OK;
  JumpArgs a{nedges, nq, nv, w, rv, info, geo, cell_xy, vdofs, vscale, x, work};
  error_jump_kernel<<<vk_grid(int64_t(nedges) * nq, kPointThreads, 148 * 16), kPointThreads, 0,
                      vk_stream(stream)>>>(a);
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_error_reduce(int64_t ncq, const double* work, int64_t neq, const double* jump,
                               double* out, void* stream) {
  VK_REQUIRE(ncq >= 0 && neq >= 0 && out && (ncq == 0 || work) && (neq == 0 || jump),
             "vk_error_reduce: bad argument");
  error_reduce_kernel<<<1, kReduceThreads, 0, vk_stream(stream)>>>(ncq, work, neq, jump, out);
  VK_CHECK_LAUNCH();
  return VK_OK;
}
