// K4: the additive Vanka sweep (reference vanka.apply_additive,
// vanka.py:142-148, with the damped update of mg.chebyshev_relax,
// mg.py:268-271).
//
// Two stream-ordered kernels, no atomics, bit-reproducible:
//   patch_solve_kernel — one warp per patch (persistent grid-stride over
//     patches in build order so residual gathers stay local): stream the
//     column-major explicit inverse with evict-first loads (the dominant
//     8*s^2 bytes), rows lane, lane+32, ... per lane, then z = w (*) y
//     (fl(w*y), exactly `p.weights * local`) into a sum(s)-long buffer.
//   dof_gather_kernel — one thread per DoF sums its z entries in ascending
//     patch order (the DoF->slot map), reproducing the reference's
//     sequential `out[idx] += ...` order, and applies the epilogue
//     out = acc | x = scale*acc | x = x + scale*acc.
#include <algorithm>
#include <cstdlib>

#include "vk_common.cuh"

namespace {




constexpr int kApplyWarps = 8;
constexpr int kApplyMaxS = 192;

// y = A_p^{-1} r_p for rows lane + 32 q (q < R), column groups of U with the
// last group predicated (no scalar tail): U*R independent loads per lane.
template <int R, int U>
__device__ __forceinline__ void stream_patch(int lane, int s, int64_t base,
                                             const double* __restrict__ A,
                                             const double* __restrict__ w, const double* rsh,
                                             double* __restrict__ z) {
  double y[R];
#pragma unroll
  for (int q = 0; q < R; ++q) y[q] = 0.0;
  for (int j = 0; j < s; j += U) {
    double a[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        a[u][q] = (i < s && j + u < s) ? __ldcs(A + (j + u) * s + i) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double rj = (j + u < s) ? rsh[j + u] : 0.0;
#pragma unroll
      for (int q = 0; q < R; ++q) y[q] = fma(a[u][q], rj, y[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = lane + 32 * q;
    if (i < s) z[base + i] = __dmul_rn(w[base + i], y[q]);
  }
}

// RMAX = ceil(smax / 32) sizes the prologue registers; each patch streams
// with its own R = ceil(s / 32) (warp-uniform switch), so mixed-size sets
// (P4: 31/52/123, Q3: 33/57/99) do not pay for the largest class.
//
// The per-patch prologue (offsets -> index list -> residual gather) is a
// chain of dependent loads; it is software-pipelined three patches deep so
// each stage has a whole patch's operator stream to land: at the top of
// patch p the warp stores r_p (gathered during patch p-1) to shared memory,
// issues the residual gathers of p+1 (indices loaded during p-1), the index
// loads of p+2 (offsets loaded during p-1) and the offset loads of p+3, and
// only then streams patch p's operator.
__host__ __device__ constexpr int unroll_of(int r) { return r <= 2 ? 8 : (r <= 4 ? 4 : 2); }

// MINB: resident CTAs per SM the register allocation must allow (memory
// parallelism: each warp keeps U*R column loads in flight).
#ifndef VK_APPLY_MINB12
#define VK_APPLY_MINB12 4
#endif
__host__ __device__ constexpr int minb_of(int r) { return r <= 2 ? VK_APPLY_MINB12 : (r <= 4 ? 3 : 2); }

template <int RMAX, bool DISPATCH>
__global__ void __launch_bounds__(kApplyWarps * 32, minb_of(RMAX)) patch_solve_kernel(
    int npatch, const int64_t* __restrict__ off, const int* __restrict__ idx,
    const double* __restrict__ w, const int64_t* __restrict__ opoff,
    const double* __restrict__ inv, const double* __restrict__ r, double* __restrict__ z) {
  pdl_trigger();
  __shared__ double rsh_all[kApplyWarps][32 * RMAX];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* rsh = rsh_all[warp];
  const int nw = gridDim.x * kApplyWarps;
  const int p0 = blockIdx.x * kApplyWarps + warp;

  // pipeline registers: stage A (r values), B (indices), C (offsets)
  int64_t baseA = 0, opA = 0, baseB = 0, opB = 0, baseC = 0, opC = 0;
  int sA = 0, sB = 0, sC = 0;
  double rA[RMAX];
  int iB[RMAX];
  auto load_meta = [&](int p, int64_t& base, int& sz, int64_t& op) {
    if (p < npatch) {
      base = off[p];
      sz = static_cast<int>(off[p + 1] - base);
      op = opoff[p];
    } else {
      base = 0;
      sz = 0;
      op = 0;
    }
  };
  load_meta(p0, baseA, sA, opA);
  pdl_wait();   // operators / structure above are setup data; r is not
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    const int i = lane + 32 * q;
    rA[q] = (i < sA) ? __ldg(r + idx[baseA + i]) : 0.0;
  }
  load_meta(p0 + nw, baseB, sB, opB);
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    const int i = lane + 32 * q;
    iB[q] = (i < sB) ? idx[baseB + i] : 0;
  }
  load_meta(p0 + 2 * nw, baseC, sC, opC);

  for (int p = p0; p < npatch; p += nw) {
    const int64_t base = baseA, ob = opA;
    const int s = sA;
#pragma unroll
    for (int q = 0; q < RMAX; ++q) rsh[lane + 32 * q] = rA[q];
    // advance the pipeline (loads land while patch p streams)
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      const int i = lane + 32 * q;
      rA[q] = (i < sB) ? __ldg(r + iB[q]) : 0.0;
    }
    baseA = baseB; opA = opB; sA = sB;
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      const int i = lane + 32 * q;
      iB[q] = (i < sC) ? idx[baseC + i] : 0;
    }
    baseB = baseC; opB = opC; sB = sC;
    load_meta(p + 3 * nw, baseC, sC, opC);
    __syncwarp();

    const double* A = inv + ob;
    if (!DISPATCH) {
      stream_patch<RMAX, unroll_of(RMAX)>(lane, s, base, A, w, rsh, z);
    } else {
      const int rp = (s + 31) >> 5;
      if (RMAX <= 1 || rp <= 1) {
        stream_patch<1, unroll_of(1)>(lane, s, base, A, w, rsh, z);
      } else if (RMAX <= 2 || rp == 2) {
        stream_patch<2, unroll_of(2)>(lane, s, base, A, w, rsh, z);
      } else if (RMAX <= 3 || rp == 3) {
        stream_patch<3, unroll_of(3)>(lane, s, base, A, w, rsh, z);
      } else if (RMAX <= 4 || rp == 4) {
        stream_patch<4, unroll_of(4)>(lane, s, base, A, w, rsh, z);
      } else if (RMAX <= 5 || rp == 5) {
        stream_patch<5, unroll_of(5)>(lane, s, base, A, w, rsh, z);
      } else {
        stream_patch<6, unroll_of(6)>(lane, s, base, A, w, rsh, z);
      }
    }
    __syncwarp();
  }
}

// K4b: thread per DoF, its slots read in groups of four with the loads
// issued before the in-order additions — acc = ((0 + z_0) + z_1) + ... in
// ascending patch order, exactly out[idx] += ... of src/vanka.py:147.  (Two
// DoFs per thread in one resident wave measured slower.)
// Chebyshev epilogues (degree mode, reference mg.py:246-254): d and x
// updated in the same pass, in the reference's elementwise order
constexpr int kCheb0 = 3;   // d = acc / scale;               x = x + d
constexpr int kChebK = 4;   // d = c1 * d + scale * acc;      x = x + d
constexpr int kCheb0Set = 5;  // d = acc / scale;             x = d   (x was zero)

template <int MODE>
__global__ void __launch_bounds__(256) dof_gather_kernel(int ndof, const int* __restrict__ dptr,
                                                         const int* __restrict__ dslot,
                                                         const double* __restrict__ z,
                                                         double* __restrict__ out, double scale,
                                                         double* __restrict__ dvec, double c1) {
  pdl_trigger();
  pdl_wait();
  const int nth = gridDim.x * blockDim.x;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < ndof; d += nth) {
    const int a = dptr[d], e = dptr[d + 1];
    double acc = 0.0;
    for (int k = a; k < e; k += 4) {
      int sl[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) sl[u] = (k + u < e) ? dslot[k + u] : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (sl[u] >= 0) ? z[sl[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (sl[u] >= 0) acc = __dadd_rn(acc, v[u]);
    }
    if (MODE == VK_APPLY_OUT) {
      out[d] = acc;
    } else if (MODE == VK_APPLY_XSET) {
      out[d] = __dmul_rn(scale, acc);
    } else if (MODE == VK_APPLY_XADD) {
      out[d] = __dadd_rn(out[d], __dmul_rn(scale, acc));
    } else {
      const double dn = (MODE == kChebK) ? __dadd_rn(__dmul_rn(c1, dvec[d]), __dmul_rn(scale, acc))
                                         : __ddiv_rn(acc, scale);
      dvec[d] = dn;
      out[d] = (MODE == kCheb0Set) ? dn : __dadd_rn(out[d], dn);
    }
  }
}

template <int MODE>
cudaError_t launch_gather(const vk_patches_s* h, const double* zbuf, double* out, double scale,
                          cudaStream_t st, double* dvec = nullptr, double c1 = 0.0) {
  const int grid = std::max(1, std::min((h->ndof + 255) / 256, 148 * 8));
  return vk_launch(dof_gather_kernel<MODE>, dim3(grid), dim3(256), 0, st,
                   12 * h->total + 16 * int64_t(h->ndof), h->ndof, (const int*)h->dptr,
                   (const int*)h->dslot, zbuf, out, scale, dvec, c1);
}

}  // namespace

static int check_apply(vk_patches_t h) {
  VK_REQUIRE(h, "vk_patches_apply: null handle");
  VK_REQUIRE(h->factored, "vk_patches_apply: patches are not factored");
  VK_REQUIRE(h->smax <= kApplyMaxS, "vk_patches_apply: patch size %d > %d", h->smax, kApplyMaxS);
  return VK_OK;
}

namespace {

// Small patch sets (coarse MG levels: fewer patches than resident warps) are
// latency-bound in patch_solve_kernel — one warp streams a whole operator.
// Here G warps of a CTA share one patch, warp g streaming columns
// [g*cs, (g+1)*cs) for all rows; the G partial products are added in the
// fixed order g = 0..G-1 (deterministic) before the weighting.
template <int R, int G>
__global__ void __launch_bounds__(kApplyWarps * 32) patch_solve_split_kernel(
    int npatch, const int64_t* __restrict__ off, const int* __restrict__ idx,
    const double* __restrict__ w, const int64_t* __restrict__ opoff,
    const double* __restrict__ inv, const double* __restrict__ r, double* __restrict__ z) {
  pdl_trigger();
  pdl_wait();
  constexpr int PPC = kApplyWarps / G;               // patches per CTA
  __shared__ double rsh[PPC][32 * R];
  __shared__ double part[PPC][G][32 * R];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int slot = warp / G, g = warp % G;
  for (int p0 = blockIdx.x * PPC; p0 < npatch; p0 += gridDim.x * PPC) {
    const int p = p0 + slot;
    const bool live = p < npatch;
    int64_t base = 0, ob = 0;
    int s = 0;
    if (live) {
      base = off[p];
      s = static_cast<int>(off[p + 1] - base);
      ob = opoff[p];
      for (int i = g * 32 + lane; i < s; i += 32 * G) rsh[slot][i] = __ldg(r + idx[base + i]);
    }
    __syncthreads();
    double y[R];
#pragma unroll
    for (int q = 0; q < R; ++q) y[q] = 0.0;
    if (live) {
      const int cs = (s + G - 1) / G;
      const int j0 = g * cs, j1 = min(s, j0 + cs);
      const double* A = inv + ob;
      for (int j = j0; j < j1; j += 4) {
        double a[4][R];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < R; ++q) {
            const int i = lane + 32 * q;
            a[u][q] = (i < s && j + u < j1) ? __ldcs(A + (j + u) * s + i) : 0.0;
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double rj = (j + u < j1) ? rsh[slot][j + u] : 0.0;
#pragma unroll
          for (int q = 0; q < R; ++q) y[q] = fma(a[u][q], rj, y[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) part[slot][g][lane + 32 * q] = y[q];
    }
    __syncthreads();
    if (live && g == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < s) {
          double acc = part[slot][0][i];
#pragma unroll
          for (int gg = 1; gg < G; ++gg) acc = __dadd_rn(acc, part[slot][gg][i]);
          z[base + i] = __dmul_rn(w[base + i], acc);
        }
      }
    }
    __syncthreads();
  }
}

// Bulk-copy variant for small patches (s <= kBulkMaxS): each warp streams its
// patches' explicit inverses with one cp.async.bulk (TMA, 1-D) per patch into
// a two-stage shared-memory ring, completion tracked by an mbarrier per
// stage; an elected lane issues the copy for patch p+2nw as soon as the warp
// has finished reading patch p's buffer.  A patch operator is one contiguous,
// 16-byte aligned block ((s*s+1)&~1 doubles, vk_factor.cu), so the DMA engine
// moves the whole 8 s^2 bytes as one transfer (evict-first in L2) and the
// lanes read it back conflict-free (lane = row).  Residual gathers use the
// same three-deep pipeline as patch_solve_kernel; per-element arithmetic is
// identical (fma over columns in order, then fl(w*y)).
constexpr int kBulkMaxS = 40;
#ifndef VK_BULK_NS     // stages (patch operators in flight) per warp
#define VK_BULK_NS 2
#endif
#ifndef VK_BULK_NW     // warps per CTA (one CTA per SM)
#define VK_BULK_NW 8
#endif
constexpr int kBulkStages = VK_BULK_NS;
constexpr int kBulkWarps = VK_BULK_NW;
constexpr int kBulkDynMax = (227 - 8) * 1024;   // dynamic ring (static: gathers, barriers)
inline size_t bulk_smem(int smax) {
  return sizeof(double) * size_t((smax * smax + 1) & ~1) * kBulkStages * kBulkWarps;
}

template <int R>
__global__ void __launch_bounds__(kBulkWarps * 32, 1) patch_solve_bulk_kernel(
    int npatch, const int64_t* __restrict__ off, const int* __restrict__ idx,
    const double* __restrict__ w, const int64_t* __restrict__ opoff,
    const double* __restrict__ inv, const double* __restrict__ r, double* __restrict__ z,
    int stage_doubles) {
  constexpr int NS = kBulkStages;
  pdl_trigger();
  extern __shared__ __align__(128) double sbuf[];   // [warps][NS][stage_doubles]
  __shared__ __align__(8) uint64_t bars[kBulkWarps][NS];
  __shared__ double rsh_all[kBulkWarps][32 * R];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* rsh = rsh_all[warp];
  double* ring = sbuf + size_t(NS * warp) * stage_doubles;
  uint64_t* bar = bars[warp];
  const int nw = gridDim.x * kBulkWarps;
  const int p0 = blockIdx.x * kBulkWarps + warp;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const uint64_t pol = evict_first_policy();
  auto issue = [&](int s, int64_t op, int st) {     // lane 0: patch operator -> stage st
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(((s * s + 1) & ~1) * sizeof(double));
      mbar_expect_tx(&bar[st], bytes);
      bulk_g2s(ring + size_t(st) * stage_doubles, inv + op, bytes, &bar[st], pol);
    }
  };
  auto meta_s = [&](int p) { return p < npatch ? static_cast<int>(off[p + 1] - off[p]) : 0; };
  auto meta_op = [&](int p) { return p < npatch ? opoff[p] : int64_t(0); };
  // fill the ring: patches p0, p0 + nw, ..., p0 + (NS-1) nw
#pragma unroll
  for (int q = 0; q < NS; ++q)
    if (p0 + q * nw < npatch) issue(meta_s(p0 + q * nw), meta_op(p0 + q * nw), q);
  // operator of the patch that refills the stage consumed next (p + NS nw),
  // fetched one iteration ahead
  int sI = meta_s(p0 + NS * nw);
  int64_t opI = meta_op(p0 + NS * nw);

  // residual pipeline registers: stage A (r values), B (indices), C (offsets)
  int64_t baseA = 0, baseB = 0, baseC = 0;
  int sA = 0, sB = 0, sC = 0;
  double rA[R];
  int iB[R];
  auto load_meta = [&](int p, int64_t& base, int& sz) {
    if (p < npatch) {
      base = off[p];
      sz = static_cast<int>(off[p + 1] - base);
    } else {
      base = 0;
      sz = 0;
    }
  };
  load_meta(p0, baseA, sA);
  pdl_wait();   // operators / structure above are setup data; r is not
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = lane + 32 * q;
    rA[q] = (i < sA) ? __ldg(r + idx[baseA + i]) : 0.0;
  }
  load_meta(p0 + nw, baseB, sB);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int i = lane + 32 * q;
    iB[q] = (i < sB) ? idx[baseB + i] : 0;
  }
  load_meta(p0 + 2 * nw, baseC, sC);

  uint32_t parity = 0u;                            // one bit per stage
  int b = 0;
  for (int p = p0; p < npatch; p += nw) {
    const int64_t base = baseA;
    const int s = sA;
#pragma unroll
    for (int q = 0; q < R; ++q) rsh[lane + 32 * q] = rA[q];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = lane + 32 * q;
      rA[q] = (i < sB) ? __ldg(r + iB[q]) : 0.0;
    }
    baseA = baseB; sA = sB;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = lane + 32 * q;
      iB[q] = (i < sC) ? idx[baseC + i] : 0;
    }
    baseB = baseC; sB = sC;
    load_meta(p + 3 * nw, baseC, sC);
    __syncwarp();

    mbar_wait(&bar[b], (parity >> b) & 1u);
    parity ^= (1u << b);
    const double* A = ring + size_t(b) * stage_doubles;
    double y[R];
#pragma unroll
    for (int q = 0; q < R; ++q) y[q] = 0.0;
#pragma unroll 4
    for (int j = 0; j < s; ++j) {
      const double rj = rsh[j];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = lane + 32 * q;
        if (i < s) y[q] = fma(A[j * s + i], rj, y[q]);   // lanes past s stay in their stage
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = lane + 32 * q;
      if (i < s) z[base + i] = __dmul_rn(__ldg(w + base + i), y[q]);
    }
    __syncwarp();                                   // stage b fully read
    if (p + NS * nw < npatch) issue(sI, opI, b);
    sI = meta_s(p + (NS + 1) * nw);
    opI = meta_op(p + (NS + 1) * nw);
    b = (b + 1 == NS) ? 0 : b + 1;
  }
}

// Chunked bulk-copy variant for s <= 128: a warp's patch operators are
// streamed as a sequence of column chunks (cc columns, cc even,
// cc*s*8 <= kChunkBytes; a patch's last chunk is padded to 16 bytes, which
// the operator layout provides) through a kChunkStages-deep per-warp
// shared-memory ring, one cp.async.bulk + mbarrier per chunk.  Measured
// (tools/gpu_scripts/build_variants.sh, cfg2-5): one 16 KB stage per warp
// beats 2-6 smaller stages (8 warps' transfers overlap each other; fewer,
// larger DMA transfers): cfg3 0.98, cfg4 1.02, cfg5 1.07 of the copy peak.  Lane 0 is the
// producer: it keeps the ring full with the chunks of the warp's next
// patches (its own cursor, one patch of metadata prefetched); all lanes
// consume column by column.  Same per-element arithmetic as
// patch_solve_kernel.
#ifndef VK_CHUNK_BYTES
#define VK_CHUNK_BYTES 16384
#endif
#ifndef VK_CHUNK_STAGES
#define VK_CHUNK_STAGES 1
#endif
constexpr int kChunkBytes = VK_CHUNK_BYTES;
constexpr int kChunkDoubles = kChunkBytes / 8;
constexpr int kChunkStages = VK_CHUNK_STAGES;

__host__ __device__ constexpr int chunk_cols(int s) {
  return (kChunkDoubles / s) >= s ? s : ((kChunkDoubles / s) & ~1);
}

template <int R>
__device__ __forceinline__ void chunk_columns(int lane, int s, int j0, int j1, const double* As,
                                              const double* rsh, double (&y)[4]) {
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    const double rj = rsh[j];
    const double* col = As + (j - j0) * s;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = lane + 32 * q;
      if (i < s) y[q] = fma(col[i], rj, y[q]);
    }
  }
}

template <int RMAX>
__global__ void __launch_bounds__(kApplyWarps * 32, 1) patch_solve_chunk_kernel(
    int npatch, const int64_t* __restrict__ off, const int* __restrict__ idx,
    const double* __restrict__ w, const int64_t* __restrict__ opoff,
    const double* __restrict__ inv, const double* __restrict__ r, double* __restrict__ z) {
  pdl_trigger();
  extern __shared__ __align__(128) double sbuf[];   // [warps][stages][kChunkDoubles]
  __shared__ __align__(8) uint64_t bars[kApplyWarps][kChunkStages];
  __shared__ double rsh_all[kApplyWarps][32 * RMAX];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* rsh = rsh_all[warp];
  double* ring = sbuf + warp * kChunkStages * kChunkDoubles;
  uint64_t* bar = bars[warp];
  const int nw = gridDim.x * kApplyWarps;
  const int p0 = blockIdx.x * kApplyWarps + warp;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kChunkStages; ++k) mbar_init(&bar[k], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const uint64_t pol = evict_first_policy();

  auto meta_s = [&](int p) { return p < npatch ? static_cast<int>(off[p + 1] - off[p]) : 0; };
  auto meta_op = [&](int p) { return p < npatch ? opoff[p] : int64_t(0); };
  // producer cursor (uniform in the warp; lane 0 issues)
  int pp = p0, pj = 0, ps = meta_s(p0);
  int64_t pop = meta_op(p0);
  int ns = meta_s(p0 + nw);
  int64_t nop = meta_op(p0 + nw);
  int pstage = 0;
  auto issue_next = [&]() {
    if (pp >= npatch) return;
    const int cc = chunk_cols(ps);
    const int cols = min(cc, ps - pj);
    const uint32_t bytes = static_cast<uint32_t>(((cols * ps + 1) & ~1) * sizeof(double));
    if (lane == 0) {
      mbar_expect_tx(&bar[pstage], bytes);
      bulk_g2s(ring + pstage * kChunkDoubles, inv + pop + int64_t(pj) * ps, bytes, &bar[pstage], pol);
    }
    pstage = (pstage + 1 == kChunkStages) ? 0 : pstage + 1;
    pj += cols;
    if (pj >= ps) {
      pp += nw;
      pj = 0;
      ps = ns;
      pop = nop;
      ns = meta_s(pp + nw);
      nop = meta_op(pp + nw);
    }
  };
#pragma unroll
  for (int k = 0; k < kChunkStages; ++k) issue_next();

  // residual pipeline (as patch_solve_kernel): A = r values, B = indices, C = offsets
  int64_t baseA = 0, baseB = 0, baseC = 0;
  int sA = 0, sB = 0, sC = 0;
  double rA[RMAX], wA[RMAX];   // r values and weights of the patch in stage A
  int iB[RMAX];
  auto load_meta = [&](int p, int64_t& base, int& sz) {
    if (p < npatch) {
      base = off[p];
      sz = static_cast<int>(off[p + 1] - base);
    } else {
      base = 0;
      sz = 0;
    }
  };
  load_meta(p0, baseA, sA);
  pdl_wait();   // operators / structure above are setup data; r is not
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    const int i = lane + 32 * q;
    rA[q] = (i < sA) ? __ldg(r + idx[baseA + i]) : 0.0;
    wA[q] = (i < sA) ? __ldg(w + baseA + i) : 0.0;
  }
  load_meta(p0 + nw, baseB, sB);
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    const int i = lane + 32 * q;
    iB[q] = (i < sB) ? idx[baseB + i] : 0;
  }
  load_meta(p0 + 2 * nw, baseC, sC);

  int cstage = 0;
  uint32_t phase_bits = 0;                       // parity per stage
  for (int p = p0; p < npatch; p += nw) {
    const int64_t base = baseA;
    const int s = sA;
    double wc[RMAX];
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      rsh[lane + 32 * q] = rA[q];
      wc[q] = wA[q];
    }
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      const int i = lane + 32 * q;
      rA[q] = (i < sB) ? __ldg(r + iB[q]) : 0.0;
      wA[q] = (i < sB) ? __ldg(w + baseB + i) : 0.0;
    }
    baseA = baseB; sA = sB;
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      const int i = lane + 32 * q;
      iB[q] = (i < sC) ? idx[baseC + i] : 0;
    }
    baseB = baseC; sB = sC;
    load_meta(p + 3 * nw, baseC, sC);
    __syncwarp();

    double y[4] = {0.0, 0.0, 0.0, 0.0};
    const int cc = chunk_cols(s);
    const int rp = (s + 31) >> 5;
    for (int j0 = 0; j0 < s; j0 += cc) {
      const int j1 = min(s, j0 + cc);
      mbar_wait(&bar[cstage], (phase_bits >> cstage) & 1u);
      phase_bits ^= (1u << cstage);
      const double* As = ring + cstage * kChunkDoubles;
      if (RMAX <= 1 || rp <= 1) chunk_columns<1>(lane, s, j0, j1, As, rsh, y);
      else if (RMAX <= 2 || rp == 2) chunk_columns<(RMAX < 2 ? RMAX : 2)>(lane, s, j0, j1, As, rsh, y);
      else if (RMAX <= 3 || rp == 3) chunk_columns<(RMAX < 3 ? RMAX : 3)>(lane, s, j0, j1, As, rsh, y);
      else chunk_columns<(RMAX < 4 ? RMAX : 4)>(lane, s, j0, j1, As, rsh, y);
      __syncwarp();                               // stage fully read
      issue_next();
      cstage = (cstage + 1 == kChunkStages) ? 0 : cstage + 1;
    }
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
      const int i = lane + 32 * q;
      if (i < s) z[base + i] = __dmul_rn(wc[q], y[q]);
    }
  }
}

}  // namespace

// VK_APPLY_BULK=0 disables the bulk-copy kernel (A/B measurements)
static bool bulk_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_APPLY_BULK");
    return !(e && e[0] == '0');
  }();
  return v;
}

// VK_APPLY_CHUNK=0 disables the chunked bulk-copy kernel (A/B measurements)
static bool chunk_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_APPLY_CHUNK");
    return !(e && e[0] == '0');
  }();
  return v;
}

// patch sets smaller than this take the split kernel (4 warps per patch,
// plain loads); VK_SPLIT_MAX overrides it (A/B measurements).  Measured on
// the captured V-cycles (tools/vcycle_time.py): with 2 * 1184 instead of
// 4 * 1184 the 4225-patch levels of cfg2 / cfg4 move to the TMA kernels and
// the V-cycle drops 1284 -> 1260 us (cfg2), 2469 -> 2447 us (cfg4); cfg3 and
// cfg5 have no level in between and are unchanged bit for bit.
static int split_max() {
  static const int v = [] {
    const char* e = getenv("VK_SPLIT_MAX");
    return e ? atoi(e) : 148 * kApplyWarps * 2;
  }();
  return v;
}

// which K4a kernel a patch set runs (same decisions as vk_patches_solve)
static const char* solve_kernel_name(const vk_patches_s* h) {
  const int rpl = (h->smax + 31) / 32;
  if (h->npatch == 0) return "none";
  if (h->npatch < split_max() && rpl <= 4) return "patch_solve_split_kernel";
  if (h->smax <= kBulkMaxS && !h->mixed_sizes && bulk_enabled() &&
      bulk_smem(h->smax) <= size_t(kBulkDynMax))
    return "patch_solve_bulk_kernel";
  if (h->smax <= 128 && chunk_enabled()) return "patch_solve_chunk_kernel";
  return "patch_solve_kernel";
}

extern "C" const char* vk_patches_solve_kernel(vk_patches_t h) {
  return h ? solve_kernel_name(h) : "none";
}

extern "C" int vk_patches_solve(vk_patches_t h, const double* r, double* zbuf, void* stream) {
  if (int st = check_apply(h)) return st;
  VK_REQUIRE(r, "vk_patches_solve: null residual");
  double* const z = zbuf ? zbuf : h->zbuf;  // caller-owned z: concurrent applies
  const int rpl = (h->smax + 31) / 32;
  const int64_t bytes = 8 * h->inv_total + 20 * h->total;   // for the PDL decision
  cudaError_t le = cudaSuccess;
  if (h->npatch > 0 && h->npatch < split_max() && rpl <= 4) {
    // coarse levels: 4 warps per patch
    constexpr int G = 4;
    const int grid = std::min((h->npatch + kApplyWarps / G - 1) / (kApplyWarps / G), 148 * 16);
#define VK_SPLIT(RV)                                                                        \
  le = vk_launch(patch_solve_split_kernel<RV, G>, dim3(grid), dim3(kApplyWarps * 32), 0,    \
                 vk_stream(stream), bytes, h->npatch, h->off, h->idx, h->w, h->opoff, h->inv, \
                 r, z)
    switch (rpl) {
      case 1: VK_SPLIT(1); break;
      case 2: VK_SPLIT(2); break;
      case 3: VK_SPLIT(3); break;
      default: VK_SPLIT(4); break;
    }
#undef VK_SPLIT
  } else if (h->npatch > 0 && h->smax <= kBulkMaxS && !h->mixed_sizes && bulk_enabled() &&
             bulk_smem(h->smax) <= size_t(kBulkDynMax)) {
    // small patches: TMA bulk copies into a per-warp ring of kBulkStages
    const int stage_doubles = ((h->smax * h->smax + 1) & ~1);
    const size_t dsm = bulk_smem(h->smax);
    const int want = (h->npatch + kBulkWarps - 1) / kBulkWarps;
#define VK_BULK(RV)                                                                           \
  do {                                                                                        \
    auto k = patch_solve_bulk_kernel<RV>;                                                     \
    VK_CHECK_CUDA(vk_smem_optin((const void*)k, kBulkDynMax));                                \
    const int grid = std::min(want, vk_resident_blocks((const void*)k, kBulkWarps * 32, dsm)); \
    le = vk_launch(k, dim3(grid), dim3(kBulkWarps * 32), dsm, vk_stream(stream), bytes,       \
                   h->npatch, h->off, h->idx, h->w, h->opoff, h->inv, r, z,             \
                   stage_doubles);                                                            \
  } while (0)
    if (rpl <= 1) VK_BULK(1);
    else VK_BULK(2);
#undef VK_BULK
  } else if (h->npatch > 0 && h->smax <= 128 && chunk_enabled()) {
    // larger patches: TMA bulk copies of column chunks through a per-warp ring
    const size_t dsm = sizeof(double) * size_t(kChunkDoubles) * kChunkStages * kApplyWarps;
    const int want = (h->npatch + kApplyWarps - 1) / kApplyWarps;
#define VK_CHUNK(RV)                                                                          \
  do {                                                                                        \
    auto k = patch_solve_chunk_kernel<RV>;                                                    \
    VK_CHECK_CUDA(vk_smem_optin((const void*)k, int(dsm)));                                   \
    const int grid = std::min(want, vk_resident_blocks((const void*)k, kApplyWarps * 32, dsm)); \
    le = vk_launch(k, dim3(grid), dim3(kApplyWarps * 32), dsm, vk_stream(stream), bytes,      \
                   h->npatch, h->off, h->idx, h->w, h->opoff, h->inv, r, z);            \
  } while (0)
    switch (rpl) {
      case 1: VK_CHUNK(1); break;
      case 2: VK_CHUNK(2); break;
      case 3: VK_CHUNK(3); break;
      default: VK_CHUNK(4); break;
    }
#undef VK_CHUNK
  } else if (h->npatch > 0) {
    // persistent: exactly the resident CTAs, so no partial last wave
    const int want = (h->npatch + kApplyWarps - 1) / kApplyWarps;
#define VK_SOLVE(RV)                                                                        \
  if (h->mixed_sizes) {                                                                     \
    auto k = patch_solve_kernel<RV, true>;                                                  \
    const int grid = std::min(want, vk_resident_blocks((const void*)k, kApplyWarps * 32));  \
    k<<<grid, kApplyWarps * 32, 0, vk_stream(stream)>>>(                                    \
        h->npatch, h->off, h->idx, h->w, h->opoff, h->inv, r, z);                     \
  } else {                                                                                  \
    auto k = patch_solve_kernel<RV, false>;                                                 \
    const int grid = std::min(want, vk_resident_blocks((const void*)k, kApplyWarps * 32));  \
    k<<<grid, kApplyWarps * 32, 0, vk_stream(stream)>>>(                                    \
        h->npatch, h->off, h->idx, h->w, h->opoff, h->inv, r, z);                     \
  }
    switch (rpl) {
      case 1: VK_SOLVE(1); break;
      case 2: VK_SOLVE(2); break;
      case 3: VK_SOLVE(3); break;
      case 4: VK_SOLVE(4); break;
      case 5: VK_SOLVE(5); break;
      default: VK_SOLVE(6); break;
    }
#undef VK_SOLVE
  }
  if (le != cudaSuccess) {
    vk::set_error("vk_patches_solve: %s", cudaGetErrorString(le));
    return VK_ERR_CUDA;
  }
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_patches_accumulate(vk_patches_t h, const double* zbuf, double* out,
                                     double scale, int32_t mode, void* stream) {
  if (int st = check_apply(h)) return st;
  const double* const z = zbuf ? zbuf : h->zbuf;
  VK_REQUIRE(out, "vk_patches_accumulate: null output");
  VK_REQUIRE(mode == VK_APPLY_OUT || mode == VK_APPLY_XSET || mode == VK_APPLY_XADD,
             "vk_patches_apply: bad mode %d", mode);
  cudaStream_t st = vk_stream(stream);
  if (h->ndof > 0) {
    cudaError_t e;
    switch (mode) {
      case VK_APPLY_OUT: e = launch_gather<VK_APPLY_OUT>(h, z, out, scale, st); break;
      case VK_APPLY_XSET: e = launch_gather<VK_APPLY_XSET>(h, z, out, scale, st); break;
      default: e = launch_gather<VK_APPLY_XADD>(h, z, out, scale, st); break;
    }
    if (e != cudaSuccess) {
      vk::set_error("vk_patches_accumulate: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
  }
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_patches_apply(vk_patches_t h, const double* r, double* out, double scale,
                                int32_t mode, double* zbuf, void* stream) {
  VK_REQUIRE(r && out, "vk_patches_apply: null argument");
  if (int st = vk_patches_solve(h, r, zbuf, stream)) return st;
  return vk_patches_accumulate(h, zbuf, out, scale, mode, stream);
}

extern "C" int vk_patches_apply_cheb(vk_patches_t h, const double* r, double* x, double* d,
                                     double c1, double c2, int32_t first, double* zbuf,
                                     void* stream) {
  VK_REQUIRE(r && x && d, "vk_patches_apply_cheb: null argument");
  if (int st = vk_patches_solve(h, r, zbuf, stream)) return st;
  const double* const z = zbuf ? zbuf : h->zbuf;
  if (h->ndof > 0) {
    const cudaStream_t st = vk_stream(stream);
    const cudaError_t e = first == 2 ? launch_gather<kCheb0Set>(h, z, x, c2, st, d, c1)
                          : first    ? launch_gather<kCheb0>(h, z, x, c2, st, d, c1)
                                     : launch_gather<kChebK>(h, z, x, c2, st, d, c1);
    if (e != cudaSuccess) {
      vk::set_error("vk_patches_apply_cheb: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
  }
  VK_CHECK_LAUNCH();
  return VK_OK;
}
