// K2 + K3: patch submatrix extraction fused with a batched fp64 inverse.
//
// Reference: vanka.factor_patches (vanka.py:129-139) =
//   extract_submatrix (sparsela.py:50-60)  -> dense A[idx, idx]
//   lu_factor         (sparsela.py:63-84)  -> getrf + row-scale pivot guard
// and the apply-time lu_solve (sparsela.py:87-90).
//
// One CTA per patch, block resident in shared memory (row-major, odd leading
// dimension => conflict-free column access for 64-bit words):
//   1. extraction: warp per block row, each lane binary-searches a CSR column
//      of row idx[i] in the sorted patch index list; stored entries are copied
//      verbatim (bit-exact), absent ones are +0.0.
//   2. guard: row scale = max |A_ij| (all-zero row -> VK_PATCH_ZERO_ROW).
//   3. in-place Gauss-Jordan with partial pivoting.  Pivot search breaks ties
//      to the lowest row like LAPACK idamax; the pivot taken at step k is U_kk
//      of the LU with partial pivoting, checked against 1e-12 * rowscale of
//      its source row (VK_PATCH_SMALL_PIVOT) exactly like sparsela.py:79-83.
//   4. the explicit inverse (same bytes as L\U, no triangular dependency at
//      apply time) is written column-major with the column permutation undone.
// Size classes: patches are bucketed by size; classes up to 128 run the
// register-tiled kernel (factor_tile_kernel), larger ones the shared-memory
// kernel (factor_kernel, also used for the extraction-only export).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include <cub/cub.cuh>

#include "vk_common.cuh"

namespace {

constexpr int kMaxPatch = 164;  // s*(s|1)*8 + 20 s bytes <= 227 KB

__host__ __device__ inline int lda_of(int s) { return s | 1; }

inline size_t factor_smem_bytes(int s) {
  return sizeof(double) * (size_t(s) * lda_of(s) + s) + sizeof(int) * (5 * size_t(s) + 1);
}

// One warp: rowoff[i+1] holds row i's length on entry, the exclusive prefix
// (row offsets into the flattened entry list) on exit.
__device__ __forceinline__ void warp_scan_rows(int lane, int s, int* rowoff) {
  int carry = 0;
  for (int base = 0; base < s; base += 32) {
    const int i = base + lane;
    int v = (i < s) ? rowoff[i + 1] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (i < s) rowoff[i + 1] = v + carry;
    carry += __shfl_sync(0xffffffffu, v, 31);
  }
  if (lane == 0) rowoff[0] = 0;
}

// position of A[i][j] in a staged block (see extract_blocks_kernel)
__host__ __device__ __forceinline__ int blk_at(int i, int j, int s) {
  int c = j;
  if (!(s & 1)) {
    c = j + i;
    if (c >= s) c -= s;
  }
  return i * s + c;
}

// Extraction of the dense patch block A[idx, idx] from the CSR with every
// (row, stored entry) pair as an independent work item: thread t takes
// entries t, t + nth, ..., four in flight, finds its row by binary search in
// the row offsets and its column by binary search in the sorted patch list,
// and copies the stored value verbatim (absent entries stay +0.0).
__device__ __forceinline__ void extract_entries(int tid, int nth, int s, int ld, const int* sidx,
                                                const int* rowoff, const int* rowk0,
                                                const int* __restrict__ col,
                                                const double* __restrict__ val, double* A) {
  const int E = rowoff[s];
  for (int e0 = tid; e0 < E; e0 += 4 * nth) {
    int rw[4], c[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * nth;
      rw[u] = -1;
      if (e < E) {
        int lo = 0, hi = s - 1;           // last row with rowoff[row] <= e
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (rowoff[mid] <= e) lo = mid; else hi = mid - 1;
        }
        const int k = rowk0[lo] + (e - rowoff[lo]);
        rw[u] = lo;
        c[u] = __ldg(col + k);
        v[u] = __ldg(val + k);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (rw[u] < 0) continue;
      int lo = 0, hi = s - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sidx[mid] < c[u]) lo = mid + 1; else hi = mid;
      }
      if (sidx[lo] == c[u]) A[rw[u] * ld + lo] = v[u];
    }
  }
}

// Extraction through the cached map (re-factorisations): warp per patch row,
// lanes over the row's stored entries; the local column comes from the map,
// so no searches — a streaming gather of the values (bit-exact copy).
__device__ __forceinline__ void extract_rows_mapped(int warp, int lane, int nw, int s, int ld,
                                                    const int* rowoff, const int* rowk0,
                                                    const double* __restrict__ val,
                                                    const int16_t* __restrict__ emap,
                                                    double* A) {
  for (int i = warp; i < s; i += nw) {
    const int e0 = rowoff[i], len = rowoff[i + 1] - e0, k0 = rowk0[i];
    for (int kk = lane; kk < len; kk += 64) {
      const int j0 = __ldg(emap + e0 + kk);
      const double v0 = __ldg(val + k0 + kk);
      const bool two = kk + 32 < len;
      const int j1 = two ? __ldg(emap + e0 + kk + 32) : -1;
      const double v1 = two ? __ldg(val + k0 + kk + 32) : 0.0;
      if (j0 >= 0) A[i * ld + j0] = v0;
      if (j1 >= 0) A[i * ld + j1] = v1;
    }
  }
}

// per patch row (flat position g in idx): number of stored CSR entries (map
// size); the inclusive scan gives the map offset of every patch row
__global__ void entry_count_kernel(int64_t total, const int* __restrict__ idx,
                                   const int* __restrict__ ptr, int64_t* __restrict__ cnt) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x)
    cnt[g + 1] = ptr[idx[g] + 1] - ptr[idx[g]];
}

// per patch (one warp): the local column of every stored entry of its rows
// (binary search in the sorted patch list, as extract_entries), or -1
__global__ void __launch_bounds__(128) emap_fill_kernel(int npatch, const int64_t* __restrict__ off,
                                                        const int* __restrict__ idx,
                                                        const int* __restrict__ ptr,
                                                        const int* __restrict__ col,
                                                        const int64_t* __restrict__ eoff,
                                                        int16_t* __restrict__ emap) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < npatch; p += nw) {
    const int64_t base = off[p];
    const int s = static_cast<int>(off[p + 1] - base);
    const int* sidx = idx + base;
    int64_t e = eoff[base];
    for (int i = 0; i < s; ++i) {
      const int r = __ldg(sidx + i);
      const int a0 = __ldg(ptr + r), len = __ldg(ptr + r + 1) - a0;
      for (int kk = lane; kk < len; kk += 32) {
        const int c = __ldg(col + a0 + kk);
        int lo = 0, hi = s - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(sidx + mid) < c) lo = mid + 1; else hi = mid;
        }
        emap[e + kk] = (__ldg(sidx + lo) == c) ? static_cast<int16_t>(lo) : int16_t(-1);
      }
      e += len;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) factor_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int* __restrict__ idx, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const int64_t* __restrict__ opoff, double* __restrict__ inv,
    int* __restrict__ status, double* __restrict__ blocks_out, const int64_t* __restrict__ blk_off,
    int extract_only) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_piv;
  __shared__ int s_status;
  constexpr int NW = NT / 32;
  constexpr int QMAX = (kMaxPatch + 31) / 32;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  for (int b = blockIdx.x; b < count; b += gridDim.x) {
    const int p = plist[b];
    const int64_t base = off[p];
    const int s = static_cast<int>(off[p + 1] - base);
    const int ld = lda_of(s);
    double* A = smem;
    double* rs = A + size_t(s) * ld;
    int* sidx = reinterpret_cast<int*>(rs + s);
    int* perm = sidx + s;
    int* iperm = perm + s;
    int* rowoff = iperm + s;      // s + 1
    int* rowk0 = rowoff + s + 1;  // s

    for (int i = threadIdx.x; i < s; i += NT) {
      const int r = idx[base + i];
      sidx[i] = r;
      perm[i] = i;
      const int a = ptr[r];
      rowk0[i] = a;
      rowoff[i + 1] = ptr[r + 1] - a;
    }
    for (int e = threadIdx.x; e < s * ld; e += NT) A[e] = 0.0;
    if (threadIdx.x == 0) s_status = 0;
    __syncthreads();
    if (warp == 0) warp_scan_rows(lane, s, rowoff);
    __syncthreads();

    // 1. extraction (bit-exact copy of stored entries)
    extract_entries(threadIdx.x, NT, s, ld, sidx, rowoff, rowk0, col, val, A);
    __syncthreads();
    if (blocks_out) {
      double* dst = blocks_out + blk_off[b];
      for (int e = threadIdx.x; e < s * s; e += NT) dst[e] = A[(e / s) * ld + (e % s)];
      if (extract_only) {
        __syncthreads();
        continue;
      }
    }

    // 2. row scales and the all-zero-row guard (sparsela.py:76-78)
    for (int i = warp; i < s; i += NW) {
      double m = 0.0;
      for (int j = lane; j < s; j += 32) m = fmax(m, fabs(A[i * ld + j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        rs[i] = m;
        if (m == 0.0) s_status = VK_PATCH_ZERO_ROW;
      }
    }
    __syncthreads();
    if (s_status != 0) {
      if (threadIdx.x == 0) status[p] = s_status;
      __syncthreads();
      continue;
    }

    // 3. Gauss-Jordan with partial pivoting
    for (int k = 0; k < s; ++k) {
      if (warp == 0) {
        double best = -1.0;
        int bi = s;
        for (int i = k + lane; i < s; i += 32) {
          const double v = fabs(A[i * ld + k]);
          if (v > best) {  // strict: first (lowest) row wins ties, like idamax
            best = v;
            bi = i;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) {
          s_piv = bi;
          if (bi != k) {
            const int t = perm[k];
            perm[k] = perm[bi];
            perm[bi] = t;
          }
        }
      }
      __syncthreads();
      const int pr = s_piv;
      if (pr != k) {
        for (int j = threadIdx.x; j < s; j += NT) {
          const double t = A[k * ld + j];
          A[k * ld + j] = A[pr * ld + j];
          A[pr * ld + j] = t;
        }
        __syncthreads();
      }
      const double piv = A[k * ld + k];
      if (!(fabs(piv) >= 1e-12 * rs[perm[k]])) {  // also catches NaN
        if (threadIdx.x == 0) s_status = VK_PATCH_SMALL_PIVOT;
        break;  // block-uniform: every thread sees the same piv
      }
      const double rinv = 1.0 / piv;
      // scaled pivot row in registers (columns lane + 32 q); row k itself is
      // rewritten only after every warp has finished this step
      double pk[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        const int j = lane + 32 * q;
        pk[q] = (j < s) ? ((j == k) ? rinv : A[k * ld + j] * rinv) : 0.0;
      }
      for (int i = warp; i < s; i += NW) {
        if (i == k) continue;
        const double f = A[i * ld + k];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const int j = lane + 32 * q;
          if (j < s) A[i * ld + j] = (j == k) ? -f * rinv : fma(-f, pk[q], A[i * ld + j]);
        }
      }
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          const int j = lane + 32 * q;
          if (j < s) A[k * ld + j] = pk[q];
        }
      }
    }
    __syncthreads();
    if (s_status != 0) {
      if (threadIdx.x == 0) status[p] = s_status;
      __syncthreads();
      continue;
    }
    // 4. inverse of A = X P (X = inverse of the row-permuted block):
    //    Ainv[i][j] = X[i][iperm[j]], written column-major.
    for (int q = threadIdx.x; q < s; q += NT) iperm[perm[q]] = q;
    __syncthreads();
    double* dst = inv + opoff[p];
    for (int e = threadIdx.x; e < s * s; e += NT) {
      const int j = e / s, i = e - j * s;
      dst[e] = A[i * ld + iperm[j]];
    }
    if (threadIdx.x == 0) status[p] = VK_PATCH_OK;
    __syncthreads();
  }
}

// generic A[rows, cols]: warp per output row, binary search of each stored
// column in the sorted `cols` list; stored values copied verbatim.
__global__ void extract_kernel(const int* __restrict__ ptr, const int* __restrict__ col,
                               const double* __restrict__ val, const int* __restrict__ rows, int nr,
                               const int* __restrict__ cols, int nc, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += nw) {
    double* o = out + int64_t(i) * nc;
    for (int j = lane; j < nc; j += 32) o[j] = 0.0;
    __syncwarp();
    const int r = rows[i];
    for (int k = ptr[r] + lane; k < ptr[r + 1]; k += 32) {
      const int c = col[k];
      int lo = 0, hi = nc - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < c) lo = mid + 1; else hi = mid;
      }
      if (cols[lo] == c) o[lo] = val[k];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Blocked Gauss-Jordan with FP64 tensor-core (DMMA) updates and look-ahead for
// the large classes, 64 < s <= S (S = 80 / 96 / 104 / 112 / 128).  The block
// lives in shared memory, padded to S with an identity tail (which stays
// decoupled); the columns are processed in panels of 8:
//   * panel factorisation (warp 0, registers; rows lane + 32q): the 8
//     Gauss-Jordan steps on the panel columns of ALL rows — pivot search over
//     the open positions with LAPACK's first-maximum tie-break (redux.sync on
//     the |value| bits, then the lowest position), the reference guard
//     |pivot| >= 1e-12 rowscale (sparsela.py:79-83), pivot-row broadcast by
//     shuffles and the per-element step of the unblocked kernels (scaled
//     pivot row, fma(-f, p_j, a), -f/pivot in the pivot column); rows never
//     move: warp 0 keeps every row's position in registers for the patch;
//   * panel update: every other column tile becomes
//     C = (pivot row of the panel ? 0 : C) + Pn R, R = the panel's 8 pivot
//     rows before the update — the in-place Gauss-Jordan elimination of 8
//     columns in GEMM form (2 S^2 8 flops), on DMMA m8n8k4 (mma.sync .f64),
//     8 x 8 tiles;
//   * look-ahead: while warps 1..7 update the block with panel p, warp 0
//     updates panel p+1's own column tile with panel p and factors panel p+1,
//     so the latency chain of the pivot steps overlaps the tensor-core
//     updates.  Two CTA barriers per 8 columns (vs two per column).
// Results agree with the unblocked kernels to rounding (the elimination is
// associated per panel); pivots and guard verdicts are those of getrf up to
// exact near-ties.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int S>
__host__ __device__ constexpr size_t dmma_smem_bytes() {
  // W, two panel buffers, two pivot-row buffers, row scales; ints: sidx,
  // rowoff, rowk0, perm, posof, two isp flag arrays
  return sizeof(double) * (size_t(S) * (S + 1) + 2 * size_t(S) * 8 + 2 * 8 * size_t(S + 1) + S) +
         sizeof(int) * (7 * size_t(S) + 1);
}

// up to B 8x8 tiles of the panel update at once (all shared-memory loads
// first, then the 8 DMMAs, then the stores: the tiles' dependency chains
// overlap instead of running back to back); tiles (ti[u], tj[u]), u < n
template <int B>
__device__ __forceinline__ void panel_update_tiles(double* W, int LD, const double* Pb,
                                                   const double* Rb, const int* isp,
                                                   const int (&ti)[B], const int (&tj)[B],
                                                   const bool (&ok)[B], int lane) {
  double c0[B], c1[B], a0[B], a1[B], b0[B], b1[B];
  int row[B], cc[B];
#pragma unroll
  for (int u = 0; u < B; ++u) {
    row[u] = ti[u] * 8 + (lane >> 2);
    cc[u] = tj[u] * 8 + 2 * (lane & 3);
    if (ok[u]) {
      const bool zr = isp[row[u]] != 0;
      c0[u] = zr ? 0.0 : W[row[u] * LD + cc[u]];
      c1[u] = zr ? 0.0 : W[row[u] * LD + cc[u] + 1];
      a0[u] = Pb[row[u] * 8 + (lane & 3)];
      a1[u] = Pb[row[u] * 8 + 4 + (lane & 3)];
      b0[u] = Rb[(lane & 3) * LD + tj[u] * 8 + (lane >> 2)];
      b1[u] = Rb[(4 + (lane & 3)) * LD + tj[u] * 8 + (lane >> 2)];
    }
  }
#pragma unroll
  for (int u = 0; u < B; ++u)
    if (ok[u]) dmma_8x8x4(c0[u], c1[u], a0[u], b0[u]);
#pragma unroll
  for (int u = 0; u < B; ++u)
    if (ok[u]) dmma_8x8x4(c0[u], c1[u], a1[u], b1[u]);
#pragma unroll
  for (int u = 0; u < B; ++u)
    if (ok[u]) {
      W[row[u] * LD + cc[u]] = c0[u];
      W[row[u] * LD + cc[u] + 1] = c1[u];
    }
}

// warp 0: the 8 Gauss-Jordan steps of the panel at k0 (columns k0..k0+7 of
// all S rows, in registers); the pivot row and the row at position k are
// found by warp reductions over the positions held in registers.  Writes the
// factored panel to W and Pb, the pivot rows to pids / isp.  Returns
// VK_PATCH_SMALL_PIVOT on a failed guard.
template <int S, int R>
__device__ __forceinline__ int factor_panel(double* W, double* Pb, int (&pos)[R], int* isp,
                                            int* pids, const double* rs, int k0, int lane) {
  constexpr int LD = S + 1, NB = 8;
  bool bad = false;   // no early exit: the 8 steps stay straight-line code, so
                      // the compiler can overlap step k+1's reductions with
                      // the tail of step k (a failed guard only flags the patch)
  double pan[R][NB];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int r = lane + 32 * q;
#pragma unroll
    for (int c = 0; c < NB; ++c) pan[q][c] = (r < S) ? W[r * LD + k0 + c] : 0.0;
  }
#pragma unroll
  for (int kk = 0; kk < NB; ++kk) {
    const int k = k0 + kk;
    double best = -1.0;
    int bpos = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const double v = fabs(pan[q][kk]);
      if (pos[q] >= k && pos[q] < S && (v > best || (v == best && pos[q] < bpos))) {
        best = v;
        bpos = pos[q];
      }
    }
    const unsigned long long key =
        best >= 0.0 ? static_cast<unsigned long long>(__double_as_longlong(best)) : 0ull;
    const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const int ppos = static_cast<int>(__reduce_min_sync(
        0xffffffffu, (hi == mhi && lo == mlo) ? static_cast<unsigned>(bpos) : 0x7fffffffu));
    unsigned mine_p = 0xffffffffu, mine_k = 0xffffffffu;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const unsigned r = static_cast<unsigned>(lane + 32 * q);
      if (pos[q] == ppos) mine_p = r;
      if (pos[q] == k) mine_k = r;
    }
    const int rp = static_cast<int>(__reduce_min_sync(0xffffffffu, mine_p));   // pivot row
    const int rk = static_cast<int>(__reduce_min_sync(0xffffffffu, mine_k));   // row at k
    const int owner = rp & 31, qp = rp >> 5;
    double prow[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double sel = pan[0][c];
#pragma unroll
      for (int q = 1; q < R; ++q) sel = (qp == q) ? pan[q][c] : sel;
      prow[c] = __shfl_sync(0xffffffffu, sel, owner);
    }
    const double piv = prow[kk];
    bad |= !(fabs(piv) >= 1e-12 * rs[rp]);           // warp-uniform
    const double rinv = __drcp_rn(piv);              // == 1.0 / piv (correctly rounded)
#pragma unroll
    for (int c = 0; c < NB; ++c) prow[c] = (c == kk) ? rinv : prow[c] * rinv;
    // branch-free: the pivot row takes the scaled row, every other row the
    // elimination (no divergence between the owner lane and the rest)
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int r = lane + 32 * q;
      const bool isp_row = (r == rp);
      const double f = pan[q][kk];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const double e = (c == kk) ? -f * rinv : fma(-f, prow[c], pan[q][c]);
        pan[q][c] = isp_row ? prow[c] : e;
      }
      pos[q] = isp_row ? k : ((r == rk) ? ppos : pos[q]);
    }
    if (lane == 0) pids[kk] = rp;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int r = lane + 32 * q;
    if (r < S) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        W[r * LD + k0 + c] = pan[q][c];
        Pb[r * NB + c] = pan[q][c];
      }
    }
  }
  __syncwarp();
  if (bad) return VK_PATCH_SMALL_PIVOT;
  if (lane < NB) isp[pids[lane]] = 1;
  return VK_PATCH_OK;
}

#ifdef VK_FACTOR_TRACE
#define VK_TRACE_ADD(slot, t0) (trc[slot] += clock64() - (t0))
#else
#define VK_TRACE_ADD(slot, t0)
#endif

template <int S>
__global__ void __launch_bounds__(256, (S <= 96) ? 2 : 1) factor_dmma_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int* __restrict__ idx, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const int64_t* __restrict__ opoff, double* __restrict__ inv,
    int* __restrict__ status, const int64_t* __restrict__ eoff,
    const int16_t* __restrict__ emap) {
  constexpr int NT = 256, NW = NT / 32, LD = S + 1, NB = 8, TT = S / 8, R = (S + 31) / 32;
  constexpr int TB = (S <= 96) ? 1 : 4;              // tiles per batch (register budget:
                                                     // 2 CTAs / SM below 97)
  static_assert(S % 8 == 0, "8x8 tiles");
  extern __shared__ __align__(16) double smem[];
  double* W = smem;                                  // S x LD
  double* Pb0 = W + S * LD;                          // 2 x (S x NB)  factored panels
  double* Rb0 = Pb0 + 2 * S * NB;                    // 2 x (NB x LD) pivot rows
  double* rs = Rb0 + 2 * NB * LD;                    // S row scales
  int* sidx = reinterpret_cast<int*>(rs + S);        // S
  int* rowoff = sidx + S;                            // S + 1
  int* rowk0 = rowoff + S + 1;                       // S
  int* perm = rowk0 + S;                             // S  position -> row
  int* posof = perm + S;                             // S  row -> position
  int* isp0 = posof + S;                             // 2 x S pivot-row flags
  __shared__ int pids0[2][NB];
  __shared__ int s_bad;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#ifdef VK_FACTOR_TRACE
  long long trc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tt0;
#endif

  for (int bb = blockIdx.x; bb < count; bb += gridDim.x) {
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    const int p = plist[bb];
    const int64_t base = off[p];
    const int s = static_cast<int>(off[p + 1] - base);
    const int np = (s + NB - 1) / NB;
    for (int i = t; i < S; i += NT) {
      if (i < s) {
        const int r = idx[base + i];
        sidx[i] = r;
        const int a0 = ptr[r];
        rowk0[i] = a0;
        rowoff[i + 1] = ptr[r + 1] - a0;
      }
      isp0[i] = 0;
      isp0[S + i] = 0;
    }
    for (int e = t; e < S * LD; e += NT) W[e] = 0.0;
    if (t == 0) s_bad = 0;
    __syncthreads();
    if (warp == 0) warp_scan_rows(lane, s, rowoff);
    __syncthreads();
    if (emap)
      extract_rows_mapped(warp, lane, NW, s, LD, rowoff, rowk0, val, emap + eoff[base], W);
    else
      extract_entries(t, NT, s, LD, sidx, rowoff, rowk0, col, val, W);
    for (int i = s + t; i < S; i += NT) W[i * LD + i] = 1.0;       // identity tail
    __syncthreads();
    for (int i = warp; i < S; i += NW) {                           // row scales, zero-row guard
      double m = 0.0;
      for (int j = lane; j < S; j += 32) m = fmax(m, fabs(W[i * LD + j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        rs[i] = m;
        if (i < s && m == 0.0) s_bad = VK_PATCH_ZERO_ROW;
      }
    }
    __syncthreads();
    VK_TRACE_ADD(0, tt0);
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      __syncthreads();
      continue;
    }
    // positions of rows lane + 32q, kept by warp 0 for the whole patch
    int pos[R];
#pragma unroll
    for (int q = 0; q < R; ++q) pos[q] = (lane + 32 * q < S) ? lane + 32 * q : 0x7fffffff;
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    // prologue: panel 0, its pivot rows
    if (warp == 0) {
      const int st = factor_panel<S, R>(W, Pb0, pos, isp0, pids0[0], rs, 0, lane);
      if (st && lane == 0) s_bad = st;
    }
    __syncthreads();
    if (!s_bad)
      for (int e = t; e < NB * S; e += NT) Rb0[(e / S) * LD + e % S] = W[pids0[0][e / S] * LD + e % S];
    __syncthreads();
    VK_TRACE_ADD(1, tt0);
    for (int pp = 0; pp < np && !s_bad; ++pp) {
      const int cur = pp & 1, nxt = cur ^ 1;
      const double* Pb = Pb0 + cur * S * NB;
      const double* Rb = Rb0 + cur * NB * LD;
      const int* isp = isp0 + cur * S;
      const bool ahead = pp + 1 < np;
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      if (warp == 0) {
        if (ahead) {
          // look-ahead: panel pp+1's own column tile first, then factor it
          for (int t0 = 0; t0 < TT; t0 += TB) {
            int ti[TB], tj[TB];
            bool ok[TB];
#pragma unroll
            for (int u = 0; u < TB; ++u) {
              ti[u] = t0 + u;
              tj[u] = pp + 1;
              ok[u] = t0 + u < TT;
            }
            panel_update_tiles<TB>(W, LD, Pb, Rb, isp, ti, tj, ok, lane);
          }
          __syncwarp();
          VK_TRACE_ADD(2, tt0);
#ifdef VK_FACTOR_TRACE
          tt0 = clock64();
#endif
          const int st = factor_panel<S, R>(W, Pb0 + nxt * S * NB, pos, isp0 + nxt * S,
                                            pids0[nxt], rs, (pp + 1) * NB, lane);
          if (st && lane == 0) s_bad = st;
          VK_TRACE_ADD(3, tt0);
        }
      } else {
        // warps 1..7: every other column tile except panels pp and pp+1
        if constexpr (TB == 1) {
          for (int tile = warp - 1; tile < TT * TT; tile += NW - 1) {
            const int ti[1] = {tile % TT}, tj[1] = {tile / TT};
            if (tj[0] == pp || (ahead && tj[0] == pp + 1)) continue;
            const bool ok[1] = {true};
            panel_update_tiles<1>(W, LD, Pb, Rb, isp, ti, tj, ok, lane);
          }
        } else
        for (int m0 = warp - 1; m0 < TT * TT; m0 += TB * (NW - 1)) {
          int ti[TB], tj[TB];
          bool ok[TB];
#pragma unroll
          for (int u = 0; u < TB; ++u) {
            const int tile = m0 + u * (NW - 1);
            ti[u] = tile % TT;
            tj[u] = tile / TT;
            ok[u] = tile < TT * TT && tj[u] != pp && !(ahead && tj[u] == pp + 1);
          }
          panel_update_tiles<TB>(W, LD, Pb, Rb, isp, ti, tj, ok, lane);
        }
        VK_TRACE_ADD(4, tt0);
      }
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      __syncthreads();
      VK_TRACE_ADD(5, tt0);
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      if (s_bad) break;                                // block-uniform
      if (t < NB) isp0[cur * S + pids0[cur][t]] = 0;   // panel pp done
      if (ahead)                                       // pivot rows of pp+1, fully updated
        for (int e = t; e < NB * S; e += NT)
          Rb0[nxt * NB * LD + (e / S) * LD + e % S] = W[pids0[nxt][e / S] * LD + e % S];
      __syncthreads();
      VK_TRACE_ADD(6, tt0);
    }
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      __syncthreads();
      continue;
    }
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (warp == 0) {                                   // row <-> position maps
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = lane + 32 * q;
        if (r < S) {
          posof[r] = pos[q];
          perm[pos[q]] = r;
        }
      }
    }
    __syncthreads();
    // inverse, column-major, coalesced: Ainv[i][j] = W[perm[i]][posof[j]]
    // (the mapping of the unblocked kernels, dst[perm[pc] s + posof[pr]])
    double* dst = inv + opoff[p];
    for (int e = t; e < s * s; e += NT) {
      const int j = e / s, i = e % s;
      dst[e] = W[perm[i] * LD + posof[j]];
    }
    if (t == 0) status[p] = VK_PATCH_OK;
    __syncthreads();
    VK_TRACE_ADD(7, tt0);
  }
#ifdef VK_FACTOR_TRACE
  if (blockIdx.x == 0 && (t == 0 || t == 32))
    printf("[dmma S=%d t=%d] init+extract %lld prologue %lld w0-tile %lld w0-panel %lld "
           "upd %lld bar1 %lld rcopy+bar2 %lld scatter %lld (cycles, summed over patches)\n",
           S, t, trc[0], trc[1], trc[2], trc[3], trc[4], trc[5], trc[6], trc[7]);
#endif
}

// ---------------------------------------------------------------------------
// Blocked Gauss-Jordan with FP64 DMMA updates for the large classes
// (96 < s <= 128 by default), round-3 form of factor_dmma_kernel:
//   * the block arrives from the K2 pass (staged slot, coalesced loads; the
//     next patch's slot is prefetched into L2 while this one is factored);
//   * panel factorisation (warp 0, registers, rows lane + 32q): per column a
//     redux.sync on the high word of |a| plus a ballot (ties resolved exactly,
//     lowest position first), the winner lane scales its row in registers and
//     publishes it through shared memory; row scales live in registers; no
//     select chains over the panel;
//   * look-ahead: warps 1..7 update panel p+1's column tile first, a named
//     barrier hands it to warp 0, which factors panel p+1 while warps 1..7
//     apply panel p to the rest of the block (8x8 DMMA tiles,
//     C = (pivot row ? 0 : C) + Pn R as in factor_dmma_kernel).
template <int S, int R>
__device__ __forceinline__ int factor_panel2(double* W, double* Pb, int (&pos)[R],
                                             const double (&rsc)[R], int* isp, int* pids,
                                             double* pbuf, int k0, int lane) {
  constexpr int LD = S + 1, NB = 8;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NONE = 0x7fffffff;
  double pan[R][NB];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int r = lane + 32 * q;
#pragma unroll
    for (int c = 0; c < NB; ++c) pan[q][c] = (r < S) ? W[r * LD + k0 + c] : 0.0;
  }
  int okall = 1;
  // rotated panel: register 0 always holds the pivot column (the update
  // writes column c into register c-1 and the pivot column into register
  // NB-1), so the 8 steps are one compact runtime loop; after NB steps the
  // frame is the identity again
#pragma unroll 1
  for (int kk = 0; kk < NB; ++kk) {
    const int k = k0 + kk;
    // this lane's best open row (branch-free): largest |a|, lowest position
    double bv = -1.0;
    int bpos = NONE, bq = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const double v = fabs(pan[q][0]);
      const bool open = pos[q] >= k && pos[q] < S;
      const bool better = open && (v > bv || (v == bv && pos[q] < bpos));
      bv = better ? v : bv;
      bpos = better ? pos[q] : bpos;
      bq = better ? q : bq;
    }
    const bool any = bpos != NONE;
    const unsigned long long key =
        any ? static_cast<unsigned long long>(__double_as_longlong(bv)) : 0ull;
    const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
    const unsigned mhi = __reduce_max_sync(FULL, hi);
    unsigned eq = __ballot_sync(FULL, any && hi == mhi);
    if (__popc(eq) > 1) {
      const unsigned mlo = __reduce_max_sync(FULL, (eq >> lane) & 1u ? lo : 0u);
      eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && lo == mlo);
      if (__popc(eq) > 1) {
        const unsigned pm = __reduce_min_sync(
            FULL, (eq >> lane) & 1u ? static_cast<unsigned>(bpos) : 0x7fffffffu);
        eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && static_cast<unsigned>(bpos) == pm);
      }
    }
    const int wl = __ffs(eq) - 1;
    // the winner publishes its raw panel row (rotated frame), position, slot
    // and guard verdict; every lane forms 1/pivot and the scaled row itself
    // (same operations as the unblocked kernels, so the values are identical)
    double* pb = pbuf + (kk & 1) * (NB + 2);
    if (lane == wl) {
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q != bq) continue;
#pragma unroll
        for (int c = 0; c < NB; c += 2)
          *reinterpret_cast<double2*>(pb + c) = make_double2(pan[q][c], pan[q][c + 1]);
        const int ok = fabs(pan[q][0]) >= 1e-12 * rsc[q];    // sparsela.py:79-83
        reinterpret_cast<int*>(pb + NB)[0] = bpos;
        reinterpret_cast<int*>(pb + NB)[1] = q;
        reinterpret_cast<int*>(pb + NB + 1)[0] = ok;
      }
    }
    __syncwarp();
    double prow[NB];
#pragma unroll
    for (int c = 0; c < NB; c += 2) {
      const double2 v = *reinterpret_cast<const double2*>(pb + c);
      prow[c] = v.x;
      prow[c + 1] = v.y;
    }
    const int ppos = reinterpret_cast<const int*>(pb + NB)[0];
    const int qw = reinterpret_cast<const int*>(pb + NB)[1];
    okall &= reinterpret_cast<const int*>(pb + NB + 1)[0];
    const double rinv = __drcp_rn(prow[0]);            // == 1.0 / pivot (correctly rounded)
#pragma unroll
    for (int c = 1; c < NB; ++c) prow[c] = prow[c] * rinv;
    prow[0] = rinv;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const double f = pan[q][0];
#pragma unroll
      for (int c = 1; c < NB; ++c) pan[q][c - 1] = fma(-f, prow[c], pan[q][c]);
      pan[q][NB - 1] = -f * rinv;
    }
    if (lane == wl) {                                  // the pivot row: the scaled row
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == qw) {
#pragma unroll
          for (int c = 1; c < NB; ++c) pan[q][c - 1] = prow[c];
          pan[q][NB - 1] = rinv;
        }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const bool isp = (lane == wl && q == qw);
      pos[q] = isp ? k : ((pos[q] == k) ? ppos : pos[q]);
    }
    if (lane == 0) pids[kk] = wl + 32 * qw;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int r = lane + 32 * q;
    if (r < S) {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        W[r * LD + k0 + c] = pan[q][c];
        Pb[r * NB + c] = pan[q][c];
      }
    }
  }
  __syncwarp();
  if (!okall) return VK_PATCH_SMALL_PIVOT;
  if (lane < NB) isp[pids[lane]] = 1;
  return VK_PATCH_OK;
}

// warps 1..7 of factor_blk_kernel: the rank-8 Gauss-Jordan update of the
// block by panel pp (C = (pivot row ? 0 : C) + Pn R on 8x8 DMMA tiles) for
// every column tile except pp (already final) and pp+1 when `skip1` (done
// first by the look-ahead).  Work units are (tile row, half of the column
// tiles), dealt round-robin to the 7 warps; the A fragments and pivot-row
// flags of a tile row are loaded once per unit, four tiles are in flight.
template <int S>
__device__ __forceinline__ void blk_update(double* W, const double* Pb, const double* Rb,
                                           const int* isp, int pp, bool skip1, int w, int nw,
                                           int lane) {
  constexpr int LD = S + 1, TT = S / 8, H0 = (TT + 1) / 2;
  const int g = lane >> 2, m = lane & 3;
  for (int u = w; u < 2 * TT; u += nw) {
    const int ti = u >> 1, half = u & 1;
    const int t0 = half ? H0 : 0, t1 = half ? TT : H0;
    const int row = ti * 8 + g;
    const double a0 = Pb[row * 8 + m], a1 = Pb[row * 8 + 4 + m];
    const bool zr = isp[row] != 0;
    double* Wr = W + row * LD + 2 * m;
    const double* R0 = Rb + m * LD + g;
    const double* R1 = Rb + (4 + m) * LD + g;
    for (int tj0 = t0; tj0 < t1; tj0 += 4) {
      double c0[4], c1[4], b0[4], b1[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int tj = min(tj0 + v, t1 - 1);
        c0[v] = zr ? 0.0 : Wr[tj * 8];
        c1[v] = zr ? 0.0 : Wr[tj * 8 + 1];
        b0[v] = R0[tj * 8];
        b1[v] = R1[tj * 8];
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) dmma_8x8x4(c0[v], c1[v], a0, b0[v]);
#pragma unroll
      for (int v = 0; v < 4; ++v) dmma_8x8x4(c0[v], c1[v], a1, b1[v]);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int tj = tj0 + v;
        if (tj < t1 && tj != pp && !(skip1 && tj == pp + 1)) {
          Wr[tj * 8] = c0[v];
          Wr[tj * 8 + 1] = c1[v];
        }
      }
    }
  }
}

template <int S>
__host__ __device__ constexpr size_t blk_smem_bytes() {
  // W, two panel buffers, two pivot-row buffers, row scales, panel pivot-row
  // buffer; ints: perm, posof, two isp flag arrays
  return sizeof(double) * (size_t(S) * (S + 1) + 2 * size_t(S) * 8 + 2 * 8 * size_t(S + 1) + S + 20) +
         sizeof(int) * (4 * size_t(S));
}

#ifndef VK_BLK_THREADS
#define VK_BLK_THREADS 256      // threads of factor_blk_kernel (a multiple of 32)
#endif

template <int S>
__global__ void __launch_bounds__(VK_BLK_THREADS, 1) factor_blk_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int64_t* __restrict__ opoff, double* __restrict__ inv, int* __restrict__ status) {
  constexpr int NT = VK_BLK_THREADS, NW = NT / 32, LD = S + 1, NB = 8, TT = S / 8, R = (S + 31) / 32;
  constexpr int NONE = 0x7fffffff;
  static_assert(S % 8 == 0, "8x8 tiles");
  extern __shared__ __align__(16) double smem[];
  double* W = smem;                                  // S x LD
  double* Pb0 = W + S * LD;                          // 2 x (S x NB)  factored panels
  double* Rb0 = Pb0 + 2 * S * NB;                    // 2 x (NB x LD) pivot rows
  double* rs = Rb0 + 2 * NB * LD;                    // S row scales
  double* pbuf = rs + S;                             // 2 x (NB + 2) panel pivot row + info
  int* perm = reinterpret_cast<int*>(pbuf + 2 * (NB + 2)); // S  position -> row
  int* posof = perm + S;                             // S  row -> position
  int* isp0 = posof + S;                             // 2 x S pivot-row flags
  __shared__ int pids0[2][NB];
  __shared__ int s_bad;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#ifdef VK_FACTOR_TRACE
  long long trc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tt0;
#endif

  for (int bb = blockIdx.x; bb < count; bb += gridDim.x) {
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    const int p = plist[bb];
    const int s = static_cast<int>(off[p + 1] - off[p]);
    const int np = (s + NB - 1) / NB;
    if (t == 0 && bb + static_cast<int>(gridDim.x) < count) {   // next block -> L2
      const int pn = plist[bb + gridDim.x];
      const int sn = static_cast<int>(off[pn + 1] - off[pn]);
      const uint32_t bytes = static_cast<uint32_t>(((sn * sn + 1) & ~1) * sizeof(double));
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(inv + opoff[pn]), "r"(bytes)
                   : "memory");
    }
    const double* src = inv + opoff[p];
    for (int i0 = warp; i0 < S; i0 += 4 * NW) {        // 4 rows x S/32 loads in flight
      double v[4][(S + 31) / 32];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int jj = 0; jj < (S + 31) / 32; ++jj) {
          const int i = i0 + u * NW, j = lane + 32 * jj;
          v[u][jj] = (i < s && j < s) ? __ldg(src + blk_at(i, j, s)) : (i == j ? 1.0 : 0.0);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int jj = 0; jj < (S + 31) / 32; ++jj) {
          const int i = i0 + u * NW, j = lane + 32 * jj;
          if (i < S && j < S) W[i * LD + j] = v[u][jj];
        }
    }
    for (int i = t; i < 2 * S; i += NT) isp0[i] = 0;
    if (t == 0) s_bad = 0;
    __syncthreads();
    for (int i = warp; i < S; i += NW) {                           // row scales, zero-row guard
      double m = 0.0;
      for (int j = lane; j < S; j += 32) m = fmax(m, fabs(W[i * LD + j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) {
        rs[i] = m;
        if (i < s && m == 0.0) s_bad = VK_PATCH_ZERO_ROW;
      }
    }
    __syncthreads();
    VK_TRACE_ADD(0, tt0);
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      __syncthreads();
      continue;
    }
    int pos[R];
    double rsc[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int r = lane + 32 * q;
      pos[q] = (r < S) ? r : NONE;
      rsc[q] = (r < S) ? rs[r] : 0.0;
    }
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (warp == 0) {
      const int st = factor_panel2<S, R>(W, Pb0, pos, rsc, isp0, pids0[0], pbuf, 0, lane);
      if (st && lane == 0) s_bad = st;
    }
    __syncthreads();
    if (!s_bad)
      for (int e = t; e < NB * S; e += NT) Rb0[(e / S) * LD + e % S] = W[pids0[0][e / S] * LD + e % S];
    __syncthreads();
    VK_TRACE_ADD(1, tt0);
    for (int pp = 0; pp < np && !s_bad; ++pp) {
      const int cur = pp & 1, nxt = cur ^ 1;
      const double* Pb = Pb0 + cur * S * NB;
      const double* Rb = Rb0 + cur * NB * LD;
      const int* isp = isp0 + cur * S;
      const bool ahead = pp + 1 < np;
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      if (ahead) {
        if (warp > 0) {                              // panel pp+1's own column tile first
          for (int ti = warp - 1; ti < TT; ti += NW - 1) {
            const int tia[1] = {ti}, tja[1] = {pp + 1};
            const bool ok[1] = {true};
            panel_update_tiles<1>(W, LD, Pb, Rb, isp, tia, tja, ok, lane);
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");   // ... handed to warp 0
      }
      VK_TRACE_ADD(2, tt0);
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      if (warp == 0) {
        if (ahead) {
          const int st = factor_panel2<S, R>(W, Pb0 + nxt * S * NB, pos, rsc, isp0 + nxt * S,
                                             pids0[nxt], pbuf, (pp + 1) * NB, lane);
          if (st && lane == 0) s_bad = st;
        }
        VK_TRACE_ADD(3, tt0);
      } else {
        // warps 1..7: every other column tile except panels pp and pp+1
#ifndef VK_BLK_NOUPD
#ifndef VK_BLK_ALL_WARPS
        // the warps that share warp 0's scheduler (warp id mod 4 == 0) sit this
        // phase out: the panel chain, which bounds the class, gets the issue slots of
        // its SMSP to itself while six warps on the other three SMSPs update
        // (same units, same results; measured: 128-class 12.98 -> 11.87 ms,
        // 104-class 9.06 -> 8.45 ms)
        if (warp & 3)
          blk_update<S>(W, Pb, Rb, isp, pp, ahead, warp - 1 - (warp >> 2), NW - (NW + 3) / 4, lane);
#else
        blk_update<S>(W, Pb, Rb, isp, pp, ahead, warp - 1, NW - 1, lane);
#endif
#endif
        VK_TRACE_ADD(4, tt0);
      }
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      __syncthreads();
      VK_TRACE_ADD(5, tt0);
#ifdef VK_FACTOR_TRACE
      tt0 = clock64();
#endif
      if (s_bad) break;                                // block-uniform
      if (t < NB) isp0[cur * S + pids0[cur][t]] = 0;   // panel pp done
      if (ahead)                                       // pivot rows of pp+1, fully updated
        for (int e = t; e < NB * S; e += NT)
          Rb0[nxt * NB * LD + (e / S) * LD + e % S] = W[pids0[nxt][e / S] * LD + e % S];
      __syncthreads();
      VK_TRACE_ADD(6, tt0);
    }
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      __syncthreads();
      continue;
    }
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (warp == 0) {                                   // row <-> position maps
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = lane + 32 * q;
        if (r < S) {
          posof[r] = pos[q];
          perm[pos[q]] = r;
        }
      }
    }
    __syncthreads();
    // inverse, column-major, coalesced: Ainv[x][y] = W[perm[x]][posof[y]]
    double* dst = inv + opoff[p];
    for (int y = warp; y < s; y += NW) {
      const int cy = posof[y];
      for (int x = lane; x < s; x += 32) dst[y * s + x] = W[perm[x] * LD + cy];
    }
    if (t == 0) status[p] = VK_PATCH_OK;
    __syncthreads();
    VK_TRACE_ADD(7, tt0);
  }
#ifdef VK_FACTOR_TRACE
  if (blockIdx.x == 0 && (t == 0 || t == 32))
    printf("[blk S=%d t=%d] load+scales %lld prologue %lld coltile+handoff %lld w0-panel %lld "
           "upd %lld bar1 %lld rcopy+bar2 %lld output %lld (cycles, summed over patches)\n",
           S, t, trc[0], trc[1], trc[2], trc[3], trc[4], trc[5], trc[6], trc[7]);
#endif
}

// VK_FACTOR_BLK=0 keeps factor_dmma_kernel (in-kernel extraction) for the large classes
bool blk_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_FACTOR_BLK");
    return !(e && e[0] == '0');
  }();
  return v;
}

// VK_FACTOR_DMMA=0 keeps the register-tiled kernel for the large classes
bool dmma_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_FACTOR_DMMA");
    return !(e && e[0] == '0');
  }();
  return v;
}

struct Bucket {
  int smax;
  std::vector<int> ids;
};

std::vector<Bucket> make_buckets(const std::vector<int64_t>& off, int first, int count) {
  static const int edges[] = {16, 24, 32, 40, 48, 56, 64, 80, 96, 104, 112, 128, 144, kMaxPatch};
  std::vector<Bucket> b(sizeof(edges) / sizeof(int));
  for (size_t i = 0; i < b.size(); ++i) b[i].smax = edges[i];
  for (int p = first; p < first + count; ++p) {
    const int s = static_cast<int>(off[p + 1] - off[p]);
    for (auto& bk : b)
      if (s <= bk.smax) {
        bk.ids.push_back(p);
        break;
      }
  }
  return b;
}

// Register-tiled Gauss-Jordan for s <= TR*RA (= TC*CB): a CTA of TR x TC
// threads holds the whole block in registers, thread (tr, tc) owning rows
// tr + TR*ra and columns tc + TC*cb.  Rows are never moved: LAPACK's row
// interchanges are tracked as the position->row map `perm` (so the pivot
// search, its lowest-position tie-break and the guard are those of getrf).
//
// Step k (two CTA barriers):
//   * every warp runs the pivot search over positions k..s-1 of the
//     published column k itself (redux.sync argmax, lowest position on ties)
//     and swaps its own copy of `perm` -- no barrier between search and use;
//   * the owners of the pivot row scale it in registers and publish it;
//     barrier;
//   * every thread applies the rank-1 update to its tile; the owners of
//     column k+1 publish it for the next search; barrier.
// The column loop is split as k = kb*TC + kt with kb unrolled, so the pivot
// column's register block index is a compile-time constant (no select chains
// over the tile).  Per-element arithmetic is unchanged: row scaling
// a*rinv (rinv in the pivot column), update fma(-f, p_j, a) (-f*rinv in the
// pivot column).  The inverse Ainv[i][j] = Y[perm[i]][iperm[j]] is scattered
// straight from the registers to the column-major operator.
template <int TR, int TC, int RA, int CB, int MB>
__global__ void __launch_bounds__(TR * TC, MB) factor_tile_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int* __restrict__ idx, const int* __restrict__ ptr, const int* __restrict__ col,
    const double* __restrict__ val, const int64_t* __restrict__ opoff, double* __restrict__ inv,
    int* __restrict__ status, const int64_t* __restrict__ eoff,
    const int16_t* __restrict__ emap) {
  constexpr int NT = TR * TC;
  constexpr int NW = NT / 32;
  constexpr int SM = TR * RA;              // largest block (rows)
  constexpr int SMC = TC * CB;             // column capacity (>= rows)
  static_assert(SMC >= SM, "the column tiling must cover the rows");
  static_assert(NT % 32 == 0, "whole warps");
  extern __shared__ __align__(16) double A[];   // SM x (SM|1) extraction staging
  __shared__ double rs[SM];
  __shared__ double colk[2][SM];
  __shared__ double prow[2][SMC];
  __shared__ int sidx[SM], posof[SM], rowoff[SM + 1], rowk0[SM];
  __shared__ int wperm[NW][SM];            // per-warp copies of the position->row map
  __shared__ int wpos[NW][SM];             // ... and of the row->position map
  __shared__ int s_bad;
  const int t = threadIdx.x;
  const int tr = t / TC, tc = t % TC;
  const int lane = t & 31;
  const int warp = t >> 5;

  for (int bb = blockIdx.x; bb < count; bb += gridDim.x) {
    const int p = plist[bb];
    const int64_t base = off[p];
    const int s = static_cast<int>(off[p + 1] - base);
    const int ld = s | 1;
    for (int i = t; i < s; i += NT) {
      const int r = idx[base + i];
      sidx[i] = r;
      const int a0 = ptr[r];
      rowk0[i] = a0;
      rowoff[i + 1] = ptr[r + 1] - a0;
    }
    for (int i = lane; i < s; i += 32) {
      wperm[warp][i] = i;
      wpos[warp][i] = i;
    }
    for (int e = t; e < s * ld; e += NT) A[e] = 0.0;
    if (t == 0) s_bad = 0;
    __syncthreads();
    if (t < 32) warp_scan_rows(lane, s, rowoff);
    __syncthreads();
    if (emap)
      extract_rows_mapped(warp, lane, NW, s, ld, rowoff, rowk0, val, emap + eoff[base], A);
    else
      extract_entries(t, NT, s, ld, sidx, rowoff, rowk0, col, val, A);
    __syncthreads();
    for (int i = t; i < s; i += NT) {           // row scales, zero-row guard
      double m = 0.0;
      for (int j = 0; j < s; ++j) m = fmax(m, fabs(A[i * ld + j]));
      rs[i] = m;
      if (m == 0.0) s_bad = VK_PATCH_ZERO_ROW;
    }
    double a[RA][CB];
#pragma unroll
    for (int ra = 0; ra < RA; ++ra)
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        const int i = tr + TR * ra, j = tc + TC * cb;
        a[ra][cb] = (i < s && j < s) ? A[i * ld + j] : 0.0;
      }
    if (tc == 0) {                               // publish column 0
#pragma unroll
      for (int ra = 0; ra < RA; ++ra) {
        const int i = tr + TR * ra;
        if (i < s) colk[0][i] = a[ra][0];
      }
    }
    __syncthreads();
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      __syncthreads();
      continue;
    }
    int bad = 0;
#pragma unroll
    for (int kb = 0; kb < CB; ++kb) {
      for (int kt = 0; kt < TC; ++kt) {
        const int k = kb * TC + kt;
        if (k >= s || bad) break;
        const int buf = k & 1;
        // pivot search (every warp): first max |colk| over positions k..s-1,
        // as a scan over rows (independent loads of position and value,
        // lowest position kept among equal maxima — idamax's first max)
        // (small blocks; large ones scan only the s - k open positions)
        double best = -1.0;
        int bi = s;
        if constexpr (SM <= 64) {
          for (int i = lane; i < s; i += 32) {
            const int pi = wpos[warp][i];
            const double v = fabs(colk[buf][i]);
            if (pi >= k && (v > best || (v == best && pi < bi))) {
              best = v;
              bi = pi;
            }
          }
        } else {
          for (int q = k + lane; q < s; q += 32) {
            const double v = fabs(colk[buf][wperm[warp][q]]);
            if (v > best) {
              best = v;
              bi = q;
            }
          }
        }
        const unsigned long long key =
            best >= 0.0 ? static_cast<unsigned long long>(__double_as_longlong(best)) : 0ull;
        const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const int pos = __reduce_min_sync(
            0xffffffffu, (hi == mhi && lo == mlo) ? bi : 0x7fffffff);
        const int r = wperm[warp][pos];
        const int rk = wperm[warp][k];
        __syncwarp();
        if (lane == 0) {
          wperm[warp][k] = r;
          wperm[warp][pos] = rk;
          wpos[warp][r] = k;
          wpos[warp][rk] = pos;
        }
        __syncwarp();
        const double piv = colk[buf][r];
        if (!(fabs(piv) >= 1e-12 * rs[r])) {     // uniform: same data in every thread
          bad = VK_PATCH_SMALL_PIVOT;
          break;
        }
        const double rinv = 1.0 / piv;
        const bool own_row = (tr == r % TR);
        const int rb = r / TR;
        // scaled pivot row (owners: tr == r % TR); register block rb matched
        // against the unrolled ra so every access is static
        if (own_row) {
#pragma unroll
          for (int ra = 0; ra < RA; ++ra) {
            if (ra == rb) {
#pragma unroll
              for (int cb = 0; cb < CB; ++cb) {
                const int j = tc + TC * cb;
                const double v = (cb == kb && tc == kt) ? rinv : a[ra][cb] * rinv;
                if (j < s) prow[buf][j] = v;
              }
            }
          }
        }
        __syncthreads();
        double pj[CB];
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) pj[cb] = prow[buf][tc + TC * cb];
        // rank-1 update of the whole tile, branch-free (rows >= s are never
        // read back; the pivot row is overwritten with its scaled copy below)
        const bool own_k = (tc == kt);
#pragma unroll
        for (int ra = 0; ra < RA; ++ra) {
          const double f = colk[buf][tr + TR * ra];
#pragma unroll
          for (int cb = 0; cb < CB; ++cb) {
            if (cb == kb) {
              const double g = fma(-f, pj[cb], a[ra][cb]);
              const double h = -f * rinv;
              a[ra][cb] = own_k ? h : g;
            } else {
              a[ra][cb] = fma(-f, pj[cb], a[ra][cb]);
            }
          }
        }
        if (own_row) {
#pragma unroll
          for (int ra = 0; ra < RA; ++ra)
            if (ra == rb) {
#pragma unroll
              for (int cb = 0; cb < CB; ++cb) a[ra][cb] = pj[cb];
            }
        }
        // publish column k+1 (block kb, or kb+1 after the last kt)
        if (k + 1 < s) {
          if (kt + 1 < TC) {
            if (tc == kt + 1) {
#pragma unroll
              for (int ra = 0; ra < RA; ++ra) colk[buf ^ 1][tr + TR * ra] = a[ra][kb];
            }
          } else if (kb + 1 < CB) {
            if (tc == 0) {
#pragma unroll
              for (int ra = 0; ra < RA; ++ra)
                colk[buf ^ 1][tr + TR * ra] = a[ra][kb + 1 < CB ? kb + 1 : kb];
            }
          }
        }
        __syncthreads();
      }
    }
    if (bad) {
      if (t == 0) status[p] = bad;
      __syncthreads();
      continue;
    }
    const int* perm0 = wperm[0];
    for (int q = t; q < s; q += NT) posof[perm0[q]] = q;
    __syncthreads();
    double* dst = inv + opoff[p];
#pragma unroll
    for (int ra = 0; ra < RA; ++ra)
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        const int pr = tr + TR * ra, pc = tc + TC * cb;
        if (pr < s && pc < s) dst[int64_t(perm0[pc]) * s + posof[pr]] = a[ra][cb];
      }
    if (t == 0) status[p] = VK_PATCH_OK;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2 as its own pass (default path): the dense patch blocks A[idx, idx] are
// gathered once into the operator slots (inv + opoff[p]) that their inverses
// will overwrite; K3 then streams each block into shared memory with one bulk
// copy, prefetched while the previous patch is factored, so the extraction's
// dependent global loads are off the factorisation's critical path.
// Staged layout: row-major with stride s; for even s row i is rotated by i
// (A[i][j] at i s + (j + i) mod s) so that lanes reading one column of
// consecutive rows hit distinct banks (odd effective stride) in both cases.

constexpr int kXRows = 8;     // patch rows per warp pass in the extraction
constexpr int kXCols = 128;   // largest block the staged (rows / warp) kernels take

// one warp per patch, kXRows rows at a time: row metadata for the pass, the
// stored entries of every row loaded before any is placed (two per lane per
// row in flight; longer rows finish in a second loop), the local column from
// the extraction map, verbatim values, zeros elsewhere; rows written
// coalesced in the staged layout.  Patches larger than kXCols are skipped
// (their kernel extracts itself).
__global__ void __launch_bounds__(256) extract_blocks_kernel(
    int p0, int p1, int scut, const int64_t* __restrict__ off, const int* __restrict__ idx,
    const int* __restrict__ ptr, const double* __restrict__ val,
    const int64_t* __restrict__ eoff, const int16_t* __restrict__ emap,
    const int64_t* __restrict__ opoff, int64_t obase, double* __restrict__ out) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double xbuf[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* B = xbuf + warp * kXRows * kXCols;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int p = p0 + blockIdx.x * (blockDim.x >> 5) + warp; p < p1; p += nw) {
    const int64_t base = off[p];
    const int s = static_cast<int>(off[p + 1] - base);
    if (s > scut) continue;
    double* o = out + (opoff[p] - obase);
    // row metadata of pass i0 (lane u < nr: row i0 + u); the next pass's is
    // fetched while this pass's entries are in flight
    auto meta = [&](int i0, int& a0, int& len, int64_t& e0) {
      a0 = 0;
      len = 0;
      e0 = 0;
      if (lane < min(kXRows, s - i0)) {
        const int r = idx[base + i0 + lane];
        e0 = eoff[base + i0 + lane];
        a0 = ptr[r];
        len = ptr[r + 1] - a0;
      }
    };
    int a0, len;
    int64_t e0;
    meta(0, a0, len, e0);
    for (int i0 = 0; i0 < s; i0 += kXRows) {
      const int nr = min(kXRows, s - i0);
#pragma unroll
      for (int u = 0; u < kXRows; ++u)
        if (u < nr)
          for (int j = lane; j < s; j += 32) B[u * kXCols + j] = 0.0;
      int jv[kXRows][2];
      double vv[kXRows][2];
#pragma unroll
      for (int u = 0; u < kXRows; ++u) {
        const int lu = __shfl_sync(FULL, len, u), au = __shfl_sync(FULL, a0, u);
        const int64_t eu = __shfl_sync(FULL, e0, u);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int kk = lane + 32 * hh;
          const bool ok = u < nr && kk < lu;
          jv[u][hh] = ok ? __ldg(emap + eu + kk) : -1;
          vv[u][hh] = ok ? __ldg(val + au + kk) : 0.0;
        }
      }
      int na0 = 0, nlen = 0;
      int64_t ne0 = 0;
      if (i0 + kXRows < s) meta(i0 + kXRows, na0, nlen, ne0);
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kXRows; ++u)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          if (jv[u][hh] >= 0) B[u * kXCols + jv[u][hh]] = vv[u][hh];
      for (int u = 0; u < nr; ++u) {                  // rows with more than 64 entries
        const int lu = __shfl_sync(FULL, len, u), au = __shfl_sync(FULL, a0, u);
        const int64_t eu = __shfl_sync(FULL, e0, u);
        for (int kk = 64 + lane; kk < lu; kk += 32) {
          const int j = __ldg(emap + eu + kk);
          if (j >= 0) B[u * kXCols + j] = __ldg(val + au + kk);
        }
      }
      __syncwarp();
      for (int u = 0; u < nr; ++u) {
        const int i = i0 + u;
        for (int j = lane; j < s; j += 32) o[blk_at(i, j, s)] = B[u * kXCols + j];
      }
      __syncwarp();
      a0 = na0;
      len = nlen;
      e0 = ne0;
    }
  }
}

// bulk copy of patch p's staged block (opoff slots are 16-byte aligned and
// hold s^2 rounded up to even doubles)
__device__ __forceinline__ void stage_block(int p, const int64_t* off, const int64_t* opoff,
                                            const double* inv, double* stage, uint64_t* bar,
                                            uint64_t pol) {
  const int s = static_cast<int>(off[p + 1] - off[p]);
  const uint32_t bytes = static_cast<uint32_t>(((s * s + 1) & ~1) * sizeof(double));
  mbar_expect_tx(bar, bytes);
  bulk_g2s(stage, inv + opoff[p], bytes, bar, pol);
}

// ---------------------------------------------------------------------------
// Rows-in-lanes Gauss-Jordan (K3, default for s <= 128).  A group of
// NWR x CH warps factors one patch: lane l of row-warp wr owns block row
// i = 32 wr + l, column half ch of it (C = S / CH columns) in registers, so
// the multiplier of a row is its own register and the whole rank-1 update is
// register DFMA with the pivot row broadcast from shared memory (LDS.128,
// no bank conflicts).  Several patches per SM (one group per CTA) hide the
// latency of the pivot-step chain, which the one-CTA-per-patch kernels could
// not.
//   * rotated columns: in the half that holds pivot column k the registers are
//     renamed by one per step (register 0 is always column k), so the loop
//     over k is a plain runtime loop with static register indices;
//   * step k: the warps holding column k pick their candidate (first maximum
//     of |a_ik| over the open positions, LAPACK idamax order, via redux.sync)
//     and publish it with its guard verdict |a_ik| >= 1e-12 rowscale_i
//     (sparsela.py:79-83); barrier; every warp selects the same winner, the
//     lanes of the pivot row publish the scaled row a_r * (1/pivot); barrier;
//     every lane updates fma(-f, p_j, a_ij) (-f/pivot in column k);
//   * rows never move: each lane keeps its row's LAPACK position.
// Per-element arithmetic equals the register-tiled and shared-memory kernels
// (bit-identical inverses); the inverse is staged by position and written
// column-major, coalesced.

template <int C, int NWR, int CH, int MB>
__global__ void __launch_bounds__(32 * NWR * CH, MB) factor_rows_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int64_t* __restrict__ opoff, double* __restrict__ inv, int* __restrict__ status) {
  constexpr int S = C * CH, NR = 32 * NWR;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NONE = 0x7fffffff;
  static_assert(C % 2 == 0 && NR >= S, "rows per group / column pairs");
  extern __shared__ __align__(16) double stage[];     // the staged block (blk_at layout)
  __shared__ __align__(16) double cb[2][NWR][C];      // candidates' scaled rows (own half)
  __shared__ __align__(16) double ob[CH > 1 ? S : 2]; // pivot row, the other column groups
  __shared__ double fcol[2][CH > 1 ? NR : 1];         // column k for the other groups
  __shared__ double rsh[CH][NR];
  __shared__ double cabs[2][NWR];                     // candidates: |value|, position, row, guard
  __shared__ int cpos[2][NWR], crow[2][NWR], cok[2][NWR];
  __shared__ int perm[S];
  __shared__ int s_bad;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wr = warp % NWR, ch = warp / NWR;
  const int i = 32 * wr + lane;                       // block row of this lane
  const uint64_t pol = evict_first_policy();          // each block is read once
  if (t == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (t == 0 && static_cast<int>(blockIdx.x) < count)
    stage_block(plist[blockIdx.x], off, opoff, inv, stage, &bar, pol);
  uint32_t phase = 0;
#ifdef VK_FACTOR_TRACE
  long long trc[4] = {0, 0, 0, 0}, tt0 = clock64();
#endif

  for (int bb = blockIdx.x; bb < count; bb += gridDim.x) {
    const int p = plist[bb];
    const int s = static_cast<int>(off[p + 1] - off[p]);
    mbar_wait(&bar, phase);
    phase ^= 1;
    double a[C];
    double m = 0.0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int c = ch * C + j;
      a[j] = (i < s && c < s) ? stage[blk_at(i, c, s)] : 0.0;
      m = fmax(m, fabs(a[j]));
    }
    rsh[ch][i] = m;
    if (t == 0) s_bad = 0;
    __syncthreads();                                  // stage consumed: prefetch the next block
    if (t == 0 && bb + static_cast<int>(gridDim.x) < count)
      stage_block(plist[bb + gridDim.x], off, opoff, inv, stage, &bar, pol);
    double rsc = rsh[0][i];
#pragma unroll
    for (int c = 1; c < CH; ++c) rsc = fmax(rsc, rsh[c][i]);
    if (ch == 0 && i < s && rsc == 0.0) s_bad = VK_PATCH_ZERO_ROW;   // sparsela.py:74-77
    __syncthreads();
    VK_TRACE_ADD(0, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (s_bad) {
      if (t == 0) status[p] = s_bad;
      continue;
    }
    int pos = (i < s) ? i : NONE;                     // LAPACK position of this row

    // candidate of this row-warp for step k (warps holding column k): first
    // maximum |a_ik| over the open positions, published with |value|,
    // position, row and guard verdict (and, for two column halves, its row
    // scaled by its own reciprocal: the other half waits only for the winner)
    auto candidate = [&](int k) {
      const int b = k & 1;
      const double f = a[0];
      if (CH > 1) fcol[b][i] = f;
      const bool open = pos >= k && pos < s;
      const unsigned long long key =
          open ? static_cast<unsigned long long>(__double_as_longlong(fabs(f))) : 0ull;
      const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
      const unsigned mhi = __reduce_max_sync(FULL, hi);
      unsigned eq = __ballot_sync(FULL, open && hi == mhi);
      if (__popc(eq) > 1) {                             // tie on the high word (rare)
        const unsigned mlo = __reduce_max_sync(FULL, (eq >> lane) & 1u ? lo : 0u);
        eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && lo == mlo);
        if (__popc(eq) > 1) {                           // exact tie: lowest position
          const unsigned pm = __reduce_min_sync(
              FULL, (eq >> lane) & 1u ? static_cast<unsigned>(pos) : 0x7fffffffu);
          eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && static_cast<unsigned>(pos) == pm);
        }
      }
      if (eq == 0u) {
        if (lane == 0) cpos[b][wr] = NONE;
      } else if (lane == __ffs(eq) - 1) {
        if (CH > 1) {
          const double rc = __drcp_rn(f);               // == 1.0 / f (correctly rounded)
          double* dst = cb[b][wr];
          dst[0] = rc;
#pragma unroll
          for (int j = 1; j < C; ++j) dst[j] = a[j] * rc;
        }
        cabs[b][wr] = fabs(f);
        cpos[b][wr] = pos;
        crow[b][wr] = i;
        cok[b][wr] = fabs(f) >= 1e-12 * rsc;            // sparsela.py:79-83
      }
    };

    int bad = 0;
    if (ch == 0) candidate(0);
    for (int k = 0; k < s; ++k) {
      const int b = k & 1;
      const bool own = (CH == 1) || ch == k / C;        // warp-uniform
      __syncthreads();
      // the same winner in every warp: largest |value|, lowest position on ties
      int bw = 0;
      if (NWR > 1) {
        double best = -1.0;
        int bp = NONE;
#pragma unroll
        for (int w = 0; w < NWR; ++w) {
          const int ps = cpos[b][w];
          const double av = cabs[b][w];
          if (ps != NONE && (av > best || (av == best && ps < bp))) {
            best = av;
            bp = ps;
            bw = w;
          }
        }
      }
      if (!cok[b][bw]) {                                // block-uniform
        bad = VK_PATCH_SMALL_PIVOT;
        break;
      }
      const int ppos = cpos[b][bw], r = crow[b][bw];
      const bool isp = (i == r);
      const double* P = cb[b][bw];
      double rinv;
      if (CH == 1) {                                    // the winner scales and publishes
        if (isp) {                                      // (one lane; its registers become
          rinv = __drcp_rn(a[0]);                       //  the scaled row)
          double2* P2w = reinterpret_cast<double2*>(cb[b][0]);
#pragma unroll
          for (int jj = 0; jj < C / 2; ++jj) {
            const double x = (jj == 0) ? rinv : a[2 * jj] * rinv;
            const double y = a[2 * jj + 1] * rinv;
            if (jj > 0) a[2 * jj] = x;
            a[2 * jj + 1] = y;
            P2w[jj] = make_double2(x, y);
          }
        }
        __syncthreads();
        P = cb[b][0];
        rinv = P[0];
      } else {
        rinv = P[0];
      }
      if (own) {
        const double f = a[0];
        if (CH > 1 && isp) {                            // its registers become the scaled row
#pragma unroll
          for (int j = 1; j < C; ++j) a[j] *= rinv;
        }
        const double g = isp ? 0.0 : f;                 // fma(-0, p, a) == a exactly
        const double2* P2 = reinterpret_cast<const double2*>(P);
        // rotate: register j-1 <- column j
#pragma unroll
        for (int jj = 0; jj < C / 2; ++jj) {
          const double2 q = P2[jj];
          if (jj > 0) a[2 * jj - 1] = fma(-g, q.x, a[2 * jj]);
          a[2 * jj] = fma(-g, q.y, a[2 * jj + 1]);
        }
        a[C - 1] = isp ? rinv : -f * rinv;
      } else {
        const double f = fcol[b][i];
        if (isp) {                                      // the pivot row, this column group
#pragma unroll
          for (int j = 0; j < C; ++j) {
            a[j] *= rinv;
            ob[ch * C + j] = a[j];
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * NWR * (CH - 1)) : "memory");   // other groups
        const double g = isp ? 0.0 : f;
        const double2* P2 = reinterpret_cast<const double2*>(ob + ch * C);
#pragma unroll
        for (int jj = 0; jj < C / 2; ++jj) {
          const double2 q = P2[jj];
          a[2 * jj] = fma(-g, q.x, a[2 * jj]);
          a[2 * jj + 1] = fma(-g, q.y, a[2 * jj + 1]);
        }
      }
      pos = isp ? k : ((pos == k) ? ppos : pos);
      if (k + 1 < s && ((CH == 1) || ch == (k + 1) / C)) candidate(k + 1);
    }
    VK_TRACE_ADD(1, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (bad) {
      if (t == 0) status[p] = bad;
      continue;
    }
    if (ch == 0 && i < s) perm[pos] = i;
    __syncthreads();
    // Ainv[x][y] = W[perm x][posof y]: row i (position pos), column c goes
    // to column-major dst[perm[c] s + pos]
    if (i < s) {
      double* dst = inv + opoff[p];
      const int n = min(max(s - ch * C, 0), C);         // rotations of this half
#pragma unroll
      for (int j = 0; j < C; ++j) {
        int c = j + n;
        c = (c >= C ? c - C : c) + ch * C;
        if (c < s) dst[perm[c] * s + pos] = a[j];
      }
    }
    if (t == 0) status[p] = VK_PATCH_OK;
    __syncthreads();                                  // perm reuse
    VK_TRACE_ADD(2, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
  }
#ifdef VK_FACTOR_TRACE
  if (blockIdx.x == 0 && t == 0)
    printf("[rows C=%d NWR=%d CH=%d] load %lld steps %lld output %lld (cycles, %d patches)\n",
           C, NWR, CH, trc[0], trc[1], trc[2], (count + gridDim.x - 1) / gridDim.x);
#endif
}

// ---------------------------------------------------------------------------
// One warp per patch (K3 for s <= 48): R block rows per lane (i = lane + 32q),
// all C columns in registers, rotated like factor_rows_kernel.  No CTA
// barriers: the pivot search is a warp vote, the winner lane scales its row in
// registers and publishes it through a per-warp double buffer, one __syncwarp
// per step.  Same pivots, guard and per-element arithmetic as the other K3
// kernels (bit-identical inverses).  Blocks arrive by bulk copy (staged by
// extract_blocks_kernel), the next one while this one is factored.
template <int C, int R, int MB>
__global__ void __launch_bounds__(32, MB) factor_warp_kernel(
    const int* __restrict__ plist, int count, const int64_t* __restrict__ off,
    const int64_t* __restrict__ opoff, double* __restrict__ inv, int* __restrict__ status) {
  constexpr int S = C;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NONE = 0x7fffffff;
  static_assert(C % 2 == 0 && 32 * R >= S, "rows per lane / column pairs");
  extern __shared__ __align__(16) double stage[];     // the staged block (blk_at layout)
  __shared__ __align__(16) double prow[2][C];         // scaled pivot row (rotated frame)
  __shared__ int perm[S];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  const uint64_t pol = evict_first_policy();
  if (lane == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (lane == 0 && static_cast<int>(blockIdx.x) < count)
    stage_block(plist[blockIdx.x], off, opoff, inv, stage, &bar, pol);
  uint32_t phase = 0;
#ifdef VK_FACTOR_TRACE
  long long trc[4] = {0, 0, 0, 0}, tt0 = clock64();
#endif

  for (int bb = blockIdx.x; bb < count; bb += gridDim.x) {
    const int p = plist[bb];
    const int s = static_cast<int>(off[p + 1] - off[p]);
    mbar_wait(&bar, phase);
    phase ^= 1;
    double a[R][C], rsc[R];
    int pos[R];
    bool zero = false;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = lane + 32 * q;
      double m = 0.0;
#pragma unroll
      for (int j = 0; j < C; ++j) {
        a[q][j] = (i < s && j < s) ? stage[blk_at(i, j, s)] : 0.0;
        m = fmax(m, fabs(a[q][j]));
      }
      rsc[q] = m;
      pos[q] = (i < s) ? i : NONE;
      zero |= (i < s && m == 0.0);
    }
    __syncwarp();                                      // stage consumed: prefetch the next block
    if (lane == 0 && bb + static_cast<int>(gridDim.x) < count)
      stage_block(plist[bb + gridDim.x], off, opoff, inv, stage, &bar, pol);
    VK_TRACE_ADD(0, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (__any_sync(FULL, zero)) {                      // sparsela.py:74-77
      if (lane == 0) status[p] = VK_PATCH_ZERO_ROW;
      continue;
    }
    int bad = 0;
    for (int k = 0; k < s; ++k) {
      const int b = k & 1;
      // this lane's best open row: largest |a_i,k|, lowest position on ties
      unsigned long long bkey = 0ull;
      int bpos = NONE, bq = 0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const unsigned long long key =
            static_cast<unsigned long long>(__double_as_longlong(fabs(a[q][0])));
        const bool open = pos[q] >= k && pos[q] < s;
        if (open && (bpos == NONE || key > bkey || (key == bkey && pos[q] < bpos))) {
          bkey = key;
          bpos = pos[q];
          bq = q;
        }
      }
      const bool any = bpos != NONE;
      const unsigned hi = static_cast<unsigned>(bkey >> 32), lo = static_cast<unsigned>(bkey);
      const unsigned mhi = __reduce_max_sync(FULL, any ? hi : 0u);
      unsigned eq = __ballot_sync(FULL, any && hi == mhi);
      if (__popc(eq) > 1) {                            // tie on the high word (rare)
        const unsigned mlo = __reduce_max_sync(FULL, (eq >> lane) & 1u ? lo : 0u);
        eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && lo == mlo);
        if (__popc(eq) > 1) {                          // exact tie: lowest position
          const unsigned pm = __reduce_min_sync(
              FULL, (eq >> lane) & 1u ? static_cast<unsigned>(bpos) : 0x7fffffffu);
          eq = __ballot_sync(FULL, ((eq >> lane) & 1u) && static_cast<unsigned>(bpos) == pm);
        }
      }
      const int wl = __ffs(eq) - 1;
      const int ppos = __shfl_sync(FULL, bpos, wl);
      const int qw = __shfl_sync(FULL, bq, wl);
      int ok = 1;
      if (lane == wl) {                                // scale and publish the pivot row
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q != qw) continue;
          const double f = a[q][0];
          ok = fabs(f) >= 1e-12 * rsc[q];              // sparsela.py:79-83
          const double rinv = __drcp_rn(f);            // == 1.0 / f (correctly rounded)
          double2* P2w = reinterpret_cast<double2*>(prow[b]);
#pragma unroll
          for (int jj = 0; jj < C / 2; ++jj) {
            const double x = (jj == 0) ? rinv : a[q][2 * jj] * rinv;
            const double y = a[q][2 * jj + 1] * rinv;
            if (jj > 0) a[q][2 * jj] = x;
            a[q][2 * jj + 1] = y;
            P2w[jj] = make_double2(x, y);
          }
        }
      }
      if (!__shfl_sync(FULL, ok, wl)) {                // warp-uniform
        bad = VK_PATCH_SMALL_PIVOT;
        break;
      }
      __syncwarp();
      const double2* P2 = reinterpret_cast<const double2*>(prow[b]);
      double g[R], fq[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        fq[q] = a[q][0];
        g[q] = (lane == wl && q == qw) ? 0.0 : fq[q];  // fma(-0, p, a) == a exactly
      }
      double rinv = 0.0;
      // rotate: register j-1 <- column j
#pragma unroll
      for (int jj = 0; jj < C / 2; ++jj) {
        const double2 pq = P2[jj];
        if (jj == 0) rinv = pq.x;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (jj > 0) a[q][2 * jj - 1] = fma(-g[q], pq.x, a[q][2 * jj]);
          a[q][2 * jj] = fma(-g[q], pq.y, a[q][2 * jj + 1]);
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const bool isp = (lane == wl && q == qw);
        a[q][C - 1] = isp ? rinv : -fq[q] * rinv;
        pos[q] = isp ? k : ((pos[q] == k) ? ppos : pos[q]);
      }
    }
    VK_TRACE_ADD(1, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
    if (bad) {
      if (lane == 0) status[p] = bad;
      continue;
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (lane + 32 * q < s) perm[pos[q]] = lane + 32 * q;
    __syncwarp();
    // row i (position pos), column c -> column-major dst[perm[c] s + pos]
    // (s rotations: register j holds column (j + s) mod C)
    double* dst = inv + opoff[p];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (lane + 32 * q < s) {
#pragma unroll
        for (int j = 0; j < C; ++j) {
          int c = j + s;
          c = c >= C ? c - C : c;
          if (c < s) dst[perm[c] * s + pos[q]] = a[q][j];
        }
      }
    }
    if (lane == 0) status[p] = VK_PATCH_OK;
    __syncwarp();                                      // perm reuse
    VK_TRACE_ADD(2, tt0);
#ifdef VK_FACTOR_TRACE
    tt0 = clock64();
#endif
  }
#ifdef VK_FACTOR_TRACE
  if (blockIdx.x == 0 && lane == 0)
    printf("[warp C=%d R=%d] load %lld steps %lld output %lld (cycles, %d patches)\n", C, R,
           trc[0], trc[1], trc[2], (count + gridDim.x - 1) / gridDim.x);
#endif
}

template <int C, int R, int MB>
cudaError_t launch_warp(const int* d_ids, int count, const vk_patches_s* h, int* d_status,
                        cudaStream_t st) {
  auto kern = factor_warp_kernel<C, R, MB>;
  const size_t dsm = sizeof(double) * size_t((C * C + 1) & ~1);
  cudaError_t e = vk_smem_optin((const void*)kern, int(dsm));
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min(count, vk_resident_blocks((const void*)kern, 32, dsm)));
  kern<<<grid, 32, dsm, st>>>(d_ids, count, h->off, h->opoff, h->inv, d_status);
  return cudaGetLastError();
}

// VK_FACTOR_ROWS=0 keeps the round-2 kernels (register tiles / DMMA)
bool rows_enabled() {
  static const bool v = [] {
    const char* e = getenv("VK_FACTOR_ROWS");
    return !(e && e[0] == '0');
  }();
  return v;
}

// largest patch size factored by the staged kernels (rows / warp); the
// classes above run the DMMA kernel (VK_FACTOR_ROWS_MAX overrides, <= 128)
int rows_max() {
  static const int v = [] {
    const char* e = getenv("VK_FACTOR_ROWS_MAX");
    return e ? std::max(0, std::min(kXCols, atoi(e))) : 96;
  }();
  return rows_enabled() ? v : 0;
}

template <int C, int NWR, int CH, int MB>
cudaError_t launch_rows(const int* d_ids, int count, const vk_patches_s* h, int* d_status,
                        cudaStream_t st) {
  auto kern = factor_rows_kernel<C, NWR, CH, MB>;
  constexpr int NT = 32 * NWR * CH;
  const size_t dsm = sizeof(double) * size_t((C * CH * C * CH + 1) & ~1);
  cudaError_t e = vk_smem_optin((const void*)kern, int(dsm));
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min(count, vk_resident_blocks((const void*)kern, NT, dsm)));
  kern<<<grid, NT, dsm, st>>>(d_ids, count, h->off, h->opoff, h->inv, d_status);
  return cudaGetLastError();
}

// One size class: d_ids (device) lists its patches.  Asynchronous on st.
int launch_class(int smax, const int* d_ids, int count, const vk_patches_s* h, const vk::Csr* a,
                 int* d_status, double* blocks, const int64_t* d_boff, int extract_only,
                 cudaStream_t st) {
  if (count == 0) return VK_OK;
  const size_t smem = factor_smem_bytes(smax);
  if (!extract_only && smax <= rows_max()) {
    cudaError_t e;
    if (smax <= 16) e = launch_warp<16, 1, 24>(d_ids, count, h, d_status, st);
    else if (smax <= 24) e = launch_warp<24, 1, 20>(d_ids, count, h, d_status, st);
    else if (smax <= 32) e = launch_warp<32, 1, 16>(d_ids, count, h, d_status, st);
    else if (smax <= 40) e = launch_warp<40, 2, 8>(d_ids, count, h, d_status, st);
    else if (smax <= 48) e = launch_warp<48, 2, 8>(d_ids, count, h, d_status, st);
    else if (smax <= 56) e = launch_rows<56, 2, 1, 6>(d_ids, count, h, d_status, st);
    else if (smax <= 64) e = launch_rows<64, 2, 1, 5>(d_ids, count, h, d_status, st);
    else if (smax <= 80) e = launch_rows<40, 3, 2, 2>(d_ids, count, h, d_status, st);
    else if (smax <= 96) e = launch_rows<48, 3, 2, 2>(d_ids, count, h, d_status, st);
    else if (smax <= 104) e = launch_rows<26, 4, 4, 1>(d_ids, count, h, d_status, st);
    else if (smax <= 112) e = launch_rows<28, 4, 4, 1>(d_ids, count, h, d_status, st);
    else e = launch_rows<32, 4, 4, 1>(d_ids, count, h, d_status, st);
    if (e != cudaSuccess) {
      vk::set_error("factor_rows_kernel: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
    return VK_OK;
  }
  if (!extract_only && smax > 64 && smax <= 128 && dmma_enabled() && blk_enabled()) {
    cudaError_t e = cudaSuccess;
#define VK_BLK(S_)                                                                              \
  do {                                                                                          \
    auto kern = factor_blk_kernel<S_>;                                                          \
    const size_t dsm = blk_smem_bytes<S_>();                                                    \
    e = vk_smem_optin((const void*)kern, int(dsm));                                             \
    const int grid = std::max(1, std::min(count, vk_resident_blocks((const void*)kern,          \
                                                                    VK_BLK_THREADS, dsm)));     \
    if (e == cudaSuccess)                                                                       \
      kern<<<grid, VK_BLK_THREADS, dsm, st>>>(d_ids, count, h->off, h->opoff, h->inv, d_status); \
  } while (0)
    if (smax <= 80) VK_BLK(80);
    else if (smax <= 96) VK_BLK(96);
    else if (smax <= 104) VK_BLK(104);
    else if (smax <= 112) VK_BLK(112);
    else VK_BLK(128);
#undef VK_BLK
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
      vk::set_error("factor_blk_kernel: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
    return VK_OK;
  }
  if (!extract_only && smax > 64 && smax <= 128 && dmma_enabled()) {
    cudaError_t e = cudaSuccess;
#define VK_DMMA(S_)                                                                             \
  do {                                                                                          \
    auto kern = factor_dmma_kernel<S_>;                                                         \
    const size_t dsm = dmma_smem_bytes<S_>();                                                   \
    e = vk_smem_optin((const void*)kern, int(dsm));                                             \
    const int grid = std::max(1, std::min(count, vk_resident_blocks((const void*)kern, 256, dsm))); \
    if (e == cudaSuccess)                                                                       \
      kern<<<grid, 256, dsm, st>>>(d_ids, count, h->off, h->idx, a->indptr, a->indices,          \
                                   a->data, h->opoff, h->inv, d_status, h->fac_eoff,            \
                                   h->fac_emap);                                                \
  } while (0)
    if (smax <= 80) VK_DMMA(80);
    else if (smax <= 96) VK_DMMA(96);
    else if (smax <= 104) VK_DMMA(104);
    else if (smax <= 112) VK_DMMA(112);
    else VK_DMMA(128);
#undef VK_DMMA
    if (e != cudaSuccess) {
      vk::set_error("factor_dmma_kernel: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
  } else if (!extract_only && smax <= 128) {
    // register-tiled classes: (TR x TC threads, RA x CB tile per thread)
    cudaError_t e = cudaSuccess;
#define VK_TILE(TR_, TC_, RA_, CB_, MB_)                                                         \
  do {                                                                                         \
    auto kern = factor_tile_kernel<TR_, TC_, RA_, CB_, MB_>;                                      \
    const size_t dsm = sizeof(double) * size_t(TR_ * RA_) * size_t((TR_ * RA_) | 1);          \
    e = vk_smem_optin((const void*)kern, int(dsm));                                            \
    int per_sm = 1;                                                                            \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TR_ * TC_, dsm);              \
    const int grid = std::max(1, std::min(count, 148 * std::max(per_sm, 1)));                 \
    if (e == cudaSuccess)                                                                      \
      kern<<<grid, TR_ * TC_, dsm, st>>>(d_ids, count, h->off, h->idx, a->indptr, a->indices,  \
                                         a->data, h->opoff, h->inv, d_status, h->fac_eoff,     \
                                         h->fac_emap);                                         \
  } while (0)
    // MB: CTAs per SM the register budget must allow (occupancy vs. spills,
    // measured per class)
    if (smax <= 16) VK_TILE(8, 8, 2, 2, 8);
    else if (smax <= 24) VK_TILE(8, 8, 3, 3, 8);
    else if (smax <= 32) VK_TILE(8, 8, 4, 4, 8);
    else if (smax <= 40) VK_TILE(8, 8, 5, 5, 8);   // 8x16 x 5x3, 8x4 x 5x10: slower
    else if (smax <= 48) VK_TILE(8, 8, 6, 6, 8);
    else if (smax <= 56) VK_TILE(8, 8, 7, 7, 6);
    else if (smax <= 64) VK_TILE(8, 16, 8, 4, 4);
    else if (smax <= 80) VK_TILE(16, 16, 5, 5, 2);
    else if (smax <= 96) VK_TILE(16, 16, 6, 6, 2);
    else if (smax <= 112) VK_TILE(16, 16, 7, 7, 1);
    else VK_TILE(16, 16, 8, 8, 1);
#undef VK_TILE
    if (e != cudaSuccess) {
      vk::set_error("factor_tile_kernel: %s", cudaGetErrorString(e));
      return VK_ERR_CUDA;
    }
  } else if (smax <= 32) {
    VK_CHECK_CUDA(vk_smem_optin((const void*)factor_kernel<128>, int(smem)));
    factor_kernel<128><<<std::min(count, 148 * 32), 128, smem, st>>>(
        d_ids, count, h->off, h->idx, a->indptr, a->indices, a->data, h->opoff, h->inv, d_status,
        blocks, d_boff, extract_only);
  } else if (smax <= 64) {
    VK_CHECK_CUDA(vk_smem_optin((const void*)factor_kernel<256>, int(smem)));
    factor_kernel<256><<<std::min(count, 148 * 16), 256, smem, st>>>(
        d_ids, count, h->off, h->idx, a->indptr, a->indices, a->data, h->opoff, h->inv, d_status,
        blocks, d_boff, extract_only);
  } else {
    VK_CHECK_CUDA(vk_smem_optin((const void*)factor_kernel<512>, int(smem)));
    factor_kernel<512><<<std::min(count, 148 * 8), 512, smem, st>>>(
        d_ids, count, h->off, h->idx, a->indptr, a->indices, a->data, h->opoff, h->inv, d_status,
        blocks, d_boff, extract_only);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    vk::set_error("factor_kernel: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

// extraction-only export path: upload the class lists, launch, wait
int launch_bucket_sync(const Bucket& bk, const vk_patches_s* h, const vk::Csr* a, int* d_status,
                       double* blocks, const std::vector<int64_t>& blk_off_host) {
  if (bk.ids.empty()) return VK_OK;
  int* d_ids = nullptr;
  int64_t* d_boff = nullptr;
  VK_CHECK_CUDA(cudaMalloc(&d_ids, sizeof(int) * bk.ids.size()));
  VK_CHECK_CUDA(cudaMalloc(&d_boff, sizeof(int64_t) * blk_off_host.size()));
  VK_CHECK_CUDA(cudaMemcpy(d_ids, bk.ids.data(), sizeof(int) * bk.ids.size(), cudaMemcpyHostToDevice));
  VK_CHECK_CUDA(cudaMemcpy(d_boff, blk_off_host.data(), sizeof(int64_t) * blk_off_host.size(),
                           cudaMemcpyHostToDevice));
  int st = launch_class(bk.smax, d_ids, static_cast<int>(bk.ids.size()), h, a, d_status, blocks,
                        d_boff, 1, 0);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(d_ids);
  cudaFree(d_boff);
  if (!st && e != cudaSuccess) {
    vk::set_error("factor_kernel: %s", cudaGetErrorString(e));
    st = VK_ERR_CUDA;
  }
  return st;
}

std::mutex g_factor_mutex;   // factorisations / extractions (shared streams, handle maps)

// extraction map for matrix a (built by the first factorisation against it,
// kept in the handle): for every patch row and stored CSR entry of that row,
// the local column in the patch (-1 if absent) -- later extractions gather
// without searching
int ensure_emap(vk_patches_s* h, const vk::Csr* a) {
  if (h->fac_emap_key != a->uid && h->npatch > 0) {
    cudaFree(h->fac_emap);
    h->fac_emap = nullptr;
    h->fac_emap_key = 0;
    if (!h->fac_eoff) VK_CHECK_CUDA(cudaMalloc(&h->fac_eoff, sizeof(int64_t) * (h->total + 1)));
    VK_CHECK_CUDA(cudaMemset(h->fac_eoff, 0, sizeof(int64_t) * (h->total + 1)));
    entry_count_kernel<<<vk_grid(h->total, 256), 256>>>(h->total, h->idx, a->indptr, h->fac_eoff);
    VK_CHECK_LAUNCH();
    size_t tb = 0;
    VK_CHECK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, h->fac_eoff, h->fac_eoff,
                                                h->total + 1));
    void* tmp = nullptr;
    VK_CHECK_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
    cudaError_t se = cub::DeviceScan::InclusiveSum(tmp, tb, h->fac_eoff, h->fac_eoff,
                                                   h->total + 1);
    cudaFree(tmp);
    VK_CHECK_CUDA(se);
    int64_t etotal = 0;
    VK_CHECK_CUDA(cudaMemcpy(&etotal, h->fac_eoff + h->total, sizeof(int64_t),
                             cudaMemcpyDeviceToHost));
    VK_CHECK_CUDA(cudaMalloc(&h->fac_emap, sizeof(int16_t) * std::max<int64_t>(etotal, 1)));
    emap_fill_kernel<<<vk_grid(int64_t(h->npatch) * 32, 128, 148 * 16), 128>>>(
        h->npatch, h->off, h->idx, a->indptr, a->indices, h->fac_eoff, h->fac_emap);
    VK_CHECK_LAUNCH();
    h->fac_emap_key = a->uid;
  }
  return VK_OK;
}

// K2 for every patch of [p0, p1) with s <= kXCols into out (slot offsets
// opoff - obase), staged layout blk_at; stream st
int launch_extract(vk_patches_s* h, const vk::Csr* a, int p0, int p1, int scut,
                   const int64_t* opoff, int64_t obase, double* out, cudaStream_t st) {
  if (p1 <= p0) return VK_OK;
  const size_t xs = sizeof(double) * size_t(8 * kXRows * kXCols);
  VK_CHECK_CUDA(vk_smem_optin((const void*)extract_blocks_kernel, int(xs)));
  const int grid = std::max(1, std::min((p1 - p0 + 7) / 8,
                                        vk_resident_blocks((const void*)extract_blocks_kernel, 256, xs)));
  extract_blocks_kernel<<<grid, 256, xs, st>>>(p0, p1, std::min(scut, kXCols), h->off, h->idx, a->indptr, a->data,
                                               h->fac_eoff, h->fac_emap, opoff, obase, out);
  VK_CHECK_LAUNCH();
  return VK_OK;
}

}  // namespace

extern "C" int vk_extract(vk_csr_t a, const int32_t* rows, int32_t nrows, const int32_t* cols,
                          int32_t ncols, double* out_dev, void* stream) {
  VK_REQUIRE(a && rows && cols && out_dev && nrows > 0 && ncols > 0, "vk_extract: bad argument");
  const int grid = std::min((nrows + 7) / 8, 148 * 8);
  extract_kernel<<<grid, 256, 0, vk_stream(stream)>>>(a->indptr, a->indices, a->data, rows, nrows, cols,
                                                      ncols, out_dev);
  VK_CHECK_LAUNCH();
  return VK_OK;
}

extern "C" int vk_patches_extract(vk_patches_t h, vk_csr_t a, int32_t first, int32_t count,
                                  double* blocks_host) {
  VK_REQUIRE(h && a && blocks_host, "vk_patches_extract: null argument");
  VK_REQUIRE(first >= 0 && count >= 0 && first + count <= h->npatch, "vk_patches_extract: range");
  VK_REQUIRE(a->nrows == h->ndof && a->ncols == h->ndof, "vk_patches_extract: matrix is %dx%d, patches need %d",
             a->nrows, a->ncols, h->ndof);
  if (count == 0) return VK_OK;
  VK_REQUIRE(h->smax <= kMaxPatch, "patch size %d exceeds %d", h->smax, kMaxPatch);
  std::lock_guard<std::mutex> lock(g_factor_mutex);   // the extraction map lives in the handle
  // blocks of up to kXCols rows: the production K2 pass (extract_blocks_kernel,
  // staged layout) into a scratch laid out like the operator slots; larger
  // blocks: the shared-memory kernel's extraction (row-major)
  std::vector<int64_t> rel(count + 1, 0), oo(h->npatch + 1, 0);
  for (int q = 0; q < count; ++q) {
    const int64_t s = h->h_off[first + q + 1] - h->h_off[first + q];
    rel[q + 1] = rel[q] + s * s;
    oo[first + q + 1] = oo[first + q] + ((s * s + 1) & ~int64_t(1));
  }
  for (int p = first + count + 1; p <= h->npatch; ++p) oo[p] = oo[first + count];
  {
    const int est = ensure_emap(h, a);
    if (est) return est;
  }
  double* d_blocks = nullptr;
  double* d_stage = nullptr;
  int64_t* d_oo = nullptr;
  int* d_status = nullptr;
  VK_CHECK_CUDA(cudaMalloc(&d_blocks, sizeof(double) * std::max<int64_t>(rel[count], 1)));
  VK_CHECK_CUDA(cudaMalloc(&d_stage, sizeof(double) * std::max<int64_t>(oo[h->npatch], 2)));
  VK_CHECK_CUDA(cudaMalloc(&d_oo, sizeof(int64_t) * (h->npatch + 1)));
  VK_CHECK_CUDA(cudaMalloc(&d_status, sizeof(int) * h->npatch));
  VK_CHECK_CUDA(cudaMemcpy(d_oo, oo.data(), sizeof(int64_t) * (h->npatch + 1), cudaMemcpyHostToDevice));
  int st = launch_extract(h, a, first, first + count, kXCols, d_oo, 0, d_stage, 0);
  auto buckets = make_buckets(h->h_off, first, count);
  for (auto& bk : buckets) {
    if (st || bk.smax <= kXCols) continue;
    std::vector<int64_t> boff(bk.ids.size());
    for (size_t q = 0; q < bk.ids.size(); ++q) boff[q] = rel[bk.ids[q] - first];
    st = launch_bucket_sync(bk, h, a, d_status, d_blocks, boff);
  }
  std::vector<double> staged(oo[h->npatch]);
  if (!st) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
      e = cudaMemcpy(blocks_host, d_blocks, sizeof(double) * rel[count], cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
      e = cudaMemcpy(staged.data(), d_stage, sizeof(double) * oo[h->npatch], cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      vk::set_error("vk_patches_extract: %s", cudaGetErrorString(e));
      st = VK_ERR_CUDA;
    }
  }
  if (!st)
    for (int q = 0; q < count; ++q) {                 // un-stage into row-major blocks
      const int s = static_cast<int>(h->h_off[first + q + 1] - h->h_off[first + q]);
      if (s > kXCols) continue;
      const double* src = staged.data() + oo[first + q];
      double* dst = blocks_host + rel[q];
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) dst[i * s + j] = src[blk_at(i, j, s)];
    }
  cudaFree(d_blocks);
  cudaFree(d_stage);
  cudaFree(d_oo);
  cudaFree(d_status);
  return st;
}

extern "C" int vk_patches_factor(vk_patches_t h, vk_csr_t a, int32_t* status_host, int32_t* first_bad) {
  VK_REQUIRE(h && a, "vk_patches_factor: null argument");
  // setup-time call: serialised, because the auxiliary stream and its
  // fork/join events below are shared by all handles
  std::lock_guard<std::mutex> lock(g_factor_mutex);
  VK_REQUIRE(a->nrows == h->ndof && a->ncols == h->ndof,
             "vk_patches_factor: matrix is %dx%d, patches need %d", a->nrows, a->ncols, h->ndof);
  if (h->smax > kMaxPatch) {
    vk::set_error("vk_patches_factor: patch size %d exceeds the shared-memory limit %d", h->smax,
                  kMaxPatch);
    return VK_ERR_UNSUPPORTED;
  }
  if (!h->fac_status) {
    // first factorization: operator storage (s^2 rounded to even, 16-byte
    // aligned per patch) and the size-class schedule, kept in the handle
    std::vector<int64_t> oo(h->npatch + 1, 0);
    for (int p = 0; p < h->npatch; ++p) {
      const int64_t s = h->h_off[p + 1] - h->h_off[p];
      oo[p + 1] = oo[p] + ((s * s + 1) & ~int64_t(1));
    }
    if (!h->opoff) VK_CHECK_CUDA(cudaMalloc(&h->opoff, sizeof(int64_t) * (h->npatch + 1)));
    VK_CHECK_CUDA(cudaMemcpy(h->opoff, oo.data(), sizeof(int64_t) * (h->npatch + 1), cudaMemcpyHostToDevice));
    if (h->inv && h->inv_total != oo[h->npatch]) {
      cudaFree(h->inv);
      h->inv = nullptr;
    }
    if (!h->inv) {
      VK_CHECK_CUDA(cudaMalloc(&h->inv, sizeof(double) * std::max<int64_t>(oo[h->npatch], 2)));
      h->inv_total = oo[h->npatch];
    }
    auto buckets = make_buckets(h->h_off, 0, h->npatch);
    std::vector<int32_t> ids;
    std::vector<std::pair<double, std::tuple<int, int, int>>> cls;
    for (auto& bk : buckets) {
      if (bk.ids.empty()) continue;
      double work = 0.0;
      for (int q : bk.ids) work += std::pow(double(h->h_off[q + 1] - h->h_off[q]), 3);
      cls.push_back({work, {bk.smax, int(ids.size()), int(bk.ids.size())}});
      ids.insert(ids.end(), bk.ids.begin(), bk.ids.end());
    }
    std::sort(cls.begin(), cls.end(), [](auto& x, auto& y) { return x.first > y.first; });
    h->fac_classes.clear();
    for (auto& c : cls) h->fac_classes.push_back(c.second);
    VK_CHECK_CUDA(cudaMalloc(&h->fac_ids, sizeof(int32_t) * std::max<size_t>(ids.size(), 1)));
    if (!ids.empty())
      VK_CHECK_CUDA(cudaMemcpy(h->fac_ids, ids.data(), sizeof(int32_t) * ids.size(), cudaMemcpyHostToDevice));
    VK_CHECK_CUDA(cudaMalloc(&h->fac_status, sizeof(int32_t) * std::max(h->npatch, 1)));
  }
  int* d_status = h->fac_status;
  {
    const int est = ensure_emap(h, a);
    if (est) return est;
  }
  // K2: every block of the staged classes into its operator slot (the staged
  // K3 kernels stream them from there)
  if (rows_max() > 0 || blk_enabled()) {
    static const bool timing_x = getenv("VK_FACTOR_TIMING") != nullptr;
    cudaEvent_t x0 = nullptr, x1 = nullptr;
    if (timing_x) {
      cudaEventCreate(&x0);
      cudaEventCreate(&x1);
      cudaEventRecord(x0, 0);
    }
    const int xst = launch_extract(h, a, 0, h->npatch, blk_enabled() ? kXCols : rows_max(),
                                   h->opoff, 0, h->inv, 0);
    if (xst) return xst;
    if (timing_x) {
      cudaEventRecord(x1, 0);
      cudaEventSynchronize(x1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, x0, x1);
      fprintf(stderr, "[vk_factor] extraction (K2): %d patches, %.3f ms\n", h->npatch, ms);
      cudaEventDestroy(x0);
      cudaEventDestroy(x1);
    }
  }
  // The largest class (most work) runs on the legacy stream, the small ones
  // (boundary / coarse patches) beside it on an auxiliary stream; one join.
  struct AuxStream {                 // one per device (streams belong to a device)
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaError_t err = cudaSuccess;
    AuxStream() {
      err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      if (err == cudaSuccess) err = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      if (err == cudaSuccess) err = cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    }
  };
  static std::mutex aux_mu;
  static std::map<int, AuxStream*> aux_by_dev;
  AuxStream* aux_p;
  {
    std::lock_guard<std::mutex> lock(aux_mu);
    AuxStream*& slot = aux_by_dev[vk_current_device()];
    if (!slot) slot = new AuxStream();
    aux_p = slot;
  }
  AuxStream& aux_streams = *aux_p;
  VK_CHECK_CUDA(aux_streams.err);
  cudaStream_t aux = aux_streams.s;
  cudaEvent_t ev_fork = aux_streams.fork, ev_join = aux_streams.join;
  VK_CHECK_CUDA(cudaMemsetAsync(d_status, 0, sizeof(int) * std::max(h->npatch, 1), 0));
  VK_CHECK_CUDA(cudaEventRecord(ev_fork, 0));
  VK_CHECK_CUDA(cudaStreamWaitEvent(aux, ev_fork, 0));
  int st = VK_OK;
  // VK_FACTOR_TIMING=1 runs the classes one after another and prints the
  // device time of each
  static const bool timing = getenv("VK_FACTOR_TIMING") != nullptr;
  for (size_t c = 0; c < h->fac_classes.size() && !st; ++c) {
    const int smax = std::get<0>(h->fac_classes[c]), first = std::get<1>(h->fac_classes[c]);
    const int count = std::get<2>(h->fac_classes[c]);
    cudaStream_t cs = (c == 0 || timing) ? cudaStream_t(0) : aux;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, 0);
    }
    st = launch_class(smax, h->fac_ids + first, count, h, a, d_status, nullptr, nullptr, 0, cs);
    if (e0) {
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<int32_t> hid(count);
      cudaMemcpy(hid.data(), h->fac_ids + first, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
      double f = 0.0;
      for (int q : hid) f += 2.0 * std::pow(double(h->h_off[q + 1] - h->h_off[q]), 3) / 3.0;
      fprintf(stderr, "[vk_factor] class <=%d: %d patches, %.3f ms, %.1f GFLOP/s LU-equiv\n",
              smax, count, ms, f / (ms * 1e-3) / 1e9);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
  if (!st) {
    VK_CHECK_CUDA(cudaEventRecord(ev_join, aux));
    VK_CHECK_CUDA(cudaStreamWaitEvent(0, ev_join, 0));
  }
  std::vector<int32_t> hs(h->npatch);
  if (!st && h->npatch) {
    cudaError_t e = cudaMemcpy(hs.data(), d_status, sizeof(int) * h->npatch, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      vk::set_error("vk_patches_factor: %s", cudaGetErrorString(e));
      st = VK_ERR_CUDA;
    }
  }
  if (st) return st;
  if (status_host) std::copy(hs.begin(), hs.end(), status_host);
  int bad = -1;
  for (int p = 0; p < h->npatch; ++p)
    if (hs[p] != VK_PATCH_OK) {
      bad = p;
      break;
    }
  if (first_bad) *first_bad = bad;
  h->factored = (bad < 0);
  // apply schedule: per-patch row-slot dispatch pays off for mixed size
  // classes (P4: 31/52/123, Q3: 33/57/99), not for uniform ones (P2, BDM3)
  {
    const int rmax = (h->smax + 31) / 32;
    int64_t small = 0;
    for (int p = 0; p < h->npatch; ++p)
      if ((h->h_off[p + 1] - h->h_off[p] + 31) / 32 < rmax) ++small;
    h->mixed_sizes = (4 * small > h->npatch);
  }
  if (bad >= 0) {
    vk::set_error("singular patch block at patch %d (status %d)", bad, hs[bad]);
    return VK_SINGULAR;
  }
  return VK_OK;
}

extern "C" int vk_patches_export_inverse(vk_patches_t h, int32_t first, int32_t count, double* inv_host) {
  VK_REQUIRE(h && inv_host, "vk_patches_export_inverse: null argument");
  VK_REQUIRE(h->factored, "vk_patches_export_inverse: patches not factored");
  VK_REQUIRE(first >= 0 && count >= 0 && first + count <= h->npatch, "vk_patches_export_inverse: range");
  std::vector<int64_t> oo(h->npatch + 1);
  VK_CHECK_CUDA(cudaMemcpy(oo.data(), h->opoff, sizeof(int64_t) * (h->npatch + 1), cudaMemcpyDeviceToHost));
  int64_t w = 0;
  for (int p = first; p < first + count; ++p) {
    const int64_t s = h->h_off[p + 1] - h->h_off[p];
    std::vector<double> cm(s * s);
    if (s) VK_CHECK_CUDA(cudaMemcpy(cm.data(), h->inv + oo[p], sizeof(double) * s * s, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < s; ++i)
      for (int64_t j = 0; j < s; ++j) inv_host[w + i * s + j] = cm[j * s + i];
    w += s * s;
  }
  return VK_OK;
}
