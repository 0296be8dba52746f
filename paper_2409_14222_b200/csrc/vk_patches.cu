// K1: device patch construction (reference vanka.py:49-126).
//
// One warp per candidate patch: gather the cell_dofs rows of the patch's
// incident cells into a shared-memory array, bitonic-sort it, drop
// duplicates and constrained DoFs with a ballot compaction, append the
// sorted pressure DoFs.  Multiplicities are integer atomics (exact and
// order-free), weights 1.0/mult are IEEE divisions — both bit-exact with the
// reference's float64 `mult[idx] += 1.0; 1.0 / mult` (vanka.py:67-73).
//
// Also builds the DoF -> (patch entry) transpose map used by the
// deterministic, atomic-free accumulation of the additive apply: for every
// DoF its slots are listed in ascending patch order, which is exactly the
// order of the reference's sequential `out[idx] += ...` (vanka.py:145-147).
#include <algorithm>
#include <climits>
#include <vector>

#include "vk_common.cuh"

namespace {

constexpr int kMaxCap = 1024;

template <int CAP>
__global__ void __launch_bounds__(128) build_stage_kernel(
    const int* __restrict__ cell_dofs, int nloc, const int* __restrict__ e2c_ptr,
    const int* __restrict__ e2c, int ncand, const int* __restrict__ pptr,
    const int* __restrict__ pdofs, const unsigned char* __restrict__ constrained,
    int* __restrict__ stage, int* __restrict__ nv_out, int* __restrict__ cnt_out,
    int* __restrict__ err) {
  constexpr int WARPS = 4;
  __shared__ int buf[WARPS][CAP];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* a = buf[warp];
  for (int cand = blockIdx.x * WARPS + warp; cand < ncand; cand += gridDim.x * WARPS) {
    const int c0 = e2c_ptr[cand], c1 = e2c_ptr[cand + 1];
    const int nc = (c1 - c0) * nloc;
    if (nc > CAP) {
      if (lane == 0) atomicExch(err, cand + 1);
      continue;
    }
    for (int t = lane; t < CAP; t += 32) {
      int v = INT_MAX;
      if (t < nc) {
        const int cell = e2c[c0 + t / nloc];
        v = cell_dofs[static_cast<int64_t>(cell) * nloc + t % nloc];
      }
      a[t] = v;
    }
    __syncwarp();
    // bitonic sort (ascending) of CAP entries
    for (int k = 2; k <= CAP; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = lane; t < CAP; t += 32) {
          const int partner = t ^ j;
          if (partner > t) {
            const int x = a[t], y = a[partner];
            const bool up = (t & k) == 0;
            if ((x > y) == up) {
              a[t] = y;
              a[partner] = x;
            }
          }
        }
        __syncwarp();
      }
    }
    // unique + unconstrained, compacted in order
    int* out = stage + static_cast<int64_t>(cand) * CAP;
    int count = 0;
    for (int t0 = 0; t0 < nc; t0 += 32) {
      const int t = t0 + lane;
      bool keep = false;
      int v = 0;
      if (t < nc) {
        v = a[t];
        keep = (t == 0 || a[t - 1] != v) && !constrained[v];
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) out[count + __popc(m & ((1u << lane) - 1u))] = v;
      count += __popc(m);
    }
    // pressure dofs: rank sort (distinct values)
    const int p0 = pptr[cand], np = pptr[cand + 1] - p0;
    if (count + np > CAP) {
      if (lane == 0) atomicExch(err, cand + 1);
      continue;
    }
    for (int i = lane; i < np; i += 32) {
      const int v = pdofs[p0 + i];
      int rank = 0;
      for (int q = 0; q < np; ++q) {
        const int u = pdofs[p0 + q];
        rank += (u < v) || (u == v && q < i);
      }
      out[count + rank] = v;
    }
    if (lane == 0) {
      nv_out[cand] = count;
      cnt_out[cand] = count + np;
    }
    __syncwarp();
  }
}

__global__ void fill_kernel(int npatch, int cap, const int* __restrict__ cand,
                            const int* __restrict__ stage, const int64_t* __restrict__ off,
                            int* __restrict__ idx, int* __restrict__ mult) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p = warp; p < npatch; p += nwarps) {
    const int c = cand[p];
    const int64_t o = off[p];
    const int s = static_cast<int>(off[p + 1] - o);
    const int* src = stage + static_cast<int64_t>(c) * cap;
    for (int i = lane; i < s; i += 32) {
      const int d = src[i];
      idx[o + i] = d;
      atomicAdd(mult + d, 1);
    }
  }
}

__global__ void weights_kernel(int npatch, int invmult, const int64_t* __restrict__ off,
                               const int* __restrict__ nvel, const int* __restrict__ idx,
                               const int* __restrict__ mult, double* __restrict__ w) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p = warp; p < npatch; p += nwarps) {
    const int64_t o = off[p];
    const int s = static_cast<int>(off[p + 1] - o);
    const int nv = nvel[p];
    for (int i = lane; i < s; i += 32) {
      double v = 1.0;
      if (invmult && i < nv) v = 1.0 / static_cast<double>(mult[idx[o + i]]);
      w[o + i] = v;
    }
  }
}

// DoF -> slot map: scatter with atomics, then sort each (short) segment so
// slots appear in ascending flat order == ascending patch order.
__global__ void slot_scatter_kernel(int64_t total, const int* __restrict__ idx,
                                    const int* __restrict__ dptr, int* __restrict__ cursor,
                                    int* __restrict__ dslot) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
       k += int64_t(gridDim.x) * blockDim.x) {
    const int d = idx[k];
    const int pos = atomicAdd(cursor + d, 1);
    dslot[dptr[d] + pos] = static_cast<int>(k);
  }
}

__global__ void slot_sort_kernel(int ndof, const int* __restrict__ dptr, int* __restrict__ dslot) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < ndof; d += gridDim.x * blockDim.x) {
    const int a = dptr[d], b = dptr[d + 1];
    for (int i = a + 1; i < b; ++i) {
      const int v = dslot[i];
      int j = i - 1;
      while (j >= a && dslot[j] > v) {
        dslot[j + 1] = dslot[j];
        --j;
      }
      dslot[j + 1] = v;
    }
  }
}

template <typename T>
int upload(T** dst, const T* src, size_t n) {
  cudaError_t e = cudaMalloc(dst, sizeof(T) * std::max<size_t>(n, 1));
  if (e == cudaSuccess && n) e = cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyDefault);
  if (e != cudaSuccess) {
    vk::set_error("upload: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}


// DoF -> slot transpose map (ascending patch order per DoF).
int build_slot_map(vk_patches_s* h) {
  const int ndof = h->ndof;
  std::vector<int32_t> hm(std::max(ndof, 1)), hd(ndof + 1, 0);
  if (ndof) VK_CHECK_CUDA(cudaMemcpy(hm.data(), h->mult, sizeof(int) * ndof, cudaMemcpyDeviceToHost));
  for (int d = 0; d < ndof; ++d) hd[d + 1] = hd[d] + hm[d];
  int* cursor = nullptr;
  VK_CHECK_CUDA(cudaMalloc(&h->dslot, sizeof(int) * std::max<int64_t>(h->total, 1)));
  VK_CHECK_CUDA(cudaMalloc(&cursor, sizeof(int) * std::max(ndof, 1)));
  VK_CHECK_CUDA(cudaMemset(cursor, 0, sizeof(int) * std::max(ndof, 1)));
  int st = upload(&h->dptr, hd.data(), ndof + 1);
  if (st) {
    cudaFree(cursor);
    return st;
  }
  if (h->total > 0) {
    slot_scatter_kernel<<<vk_grid(h->total, 256), 256>>>(h->total, h->idx, h->dptr, cursor, h->dslot);
    slot_sort_kernel<<<vk_grid(ndof, 256), 256>>>(ndof, h->dptr, h->dslot);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(cursor);
  if (e != cudaSuccess) {
    vk::set_error("slot map: %s", cudaGetErrorString(e));
    return VK_ERR_CUDA;
  }
  return VK_OK;
}

__global__ void count_kernel(int64_t total, const int* __restrict__ idx, int* __restrict__ mult) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(mult + idx[k], 1);
}

}  // namespace

void vk_patches_free(vk_patches_s* h);

void vk_patches_free(vk_patches_s* h) {
  if (!h) return;
  cudaFree(h->off);
  cudaFree(h->idx);
  cudaFree(h->nvel);
  cudaFree(h->w);
  cudaFree(h->mult);
  cudaFree(h->cand);
  cudaFree(h->opoff);
  cudaFree(h->inv);
  cudaFree(h->dptr);
  cudaFree(h->dslot);
  cudaFree(h->zbuf);
  cudaFree(h->fac_ids);
  cudaFree(h->fac_status);
  cudaFree(h->fac_eoff);
  cudaFree(h->fac_emap);
  delete h;
}

extern "C" int vk_patches_build(const int32_t* cell_dofs, int32_t ncells, int32_t nloc,
                                const int32_t* ent2cell_ptr, const int32_t* ent2cell,
                                int32_t ncand, const int32_t* pdof_ptr, const int32_t* pdofs,
                                const uint8_t* constrained, int32_t ndof, int32_t weighting,
                                vk_patches_t* out) {
  VK_REQUIRE(out && cell_dofs && ent2cell_ptr && ent2cell && pdof_ptr && constrained,
             "vk_patches_build: null argument");
  VK_REQUIRE(weighting == VK_WEIGHT_INVMULT || weighting == VK_WEIGHT_UNIT,
             "unknown weighting %d", weighting);
  VK_REQUIRE(ncells >= 0 && nloc > 0 && ncand >= 0 && ndof >= 0, "vk_patches_build: bad sizes");

  // host views of the small pointer arrays (sizes, capacity)
  std::vector<int32_t> he(ncand + 1), hp(ncand + 1);
  VK_CHECK_CUDA(cudaMemcpy(he.data(), ent2cell_ptr, sizeof(int32_t) * (ncand + 1), cudaMemcpyDefault));
  VK_CHECK_CUDA(cudaMemcpy(hp.data(), pdof_ptr, sizeof(int32_t) * (ncand + 1), cudaMemcpyDefault));
  int maxcand = 0;
  for (int i = 0; i < ncand; ++i)
    maxcand = std::max(maxcand, (he[i + 1] - he[i]) * nloc + (hp[i + 1] - hp[i]));
  int cap = 32;
  while (cap < maxcand) cap <<= 1;
  if (cap > kMaxCap) {
    vk::set_error("vk_patches_build: patch candidate list of %d exceeds %d", maxcand, kMaxCap);
    return VK_ERR_UNSUPPORTED;
  }

  int *d_cd = nullptr, *d_e2cp = nullptr, *d_e2c = nullptr, *d_pp = nullptr, *d_pd = nullptr;
  unsigned char* d_con = nullptr;
  int *stage = nullptr, *nv = nullptr, *cnt = nullptr, *err = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_cd);
    cudaFree(d_e2cp);
    cudaFree(d_e2c);
    cudaFree(d_pp);
    cudaFree(d_pd);
    cudaFree(d_con);
    cudaFree(stage);
    cudaFree(nv);
    cudaFree(cnt);
    cudaFree(err);
  };
  int st = upload(&d_cd, cell_dofs, size_t(ncells) * nloc);
  if (!st) st = upload(&d_e2cp, ent2cell_ptr, ncand + 1);
  if (!st) st = upload(&d_e2c, ent2cell, size_t(he[ncand]));
  if (!st) st = upload(&d_pp, pdof_ptr, ncand + 1);
  if (!st) st = upload(&d_pd, pdofs, size_t(hp[ncand]));
  if (!st) st = upload(&d_con, reinterpret_cast<const unsigned char*>(constrained), size_t(ndof));
  if (st) {
    cleanup();
    return st;
  }
  cudaError_t e = cudaMalloc(&stage, sizeof(int) * std::max<size_t>(size_t(ncand) * cap, 1));
  if (e == cudaSuccess) e = cudaMalloc(&nv, sizeof(int) * std::max(ncand, 1));
  if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(int) * std::max(ncand, 1));
  if (e == cudaSuccess) e = cudaMalloc(&err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(err, 0, sizeof(int));
  if (e != cudaSuccess) {
    vk::set_error("vk_patches_build: %s", cudaGetErrorString(e));
    cleanup();
    return VK_ERR_CUDA;
  }
  if (ncand > 0) {
    const int grid = std::min((ncand + 3) / 4, 148 * 16);
#define VK_BUILD(CAPV)                                                                      \
  build_stage_kernel<CAPV><<<grid, 128>>>(d_cd, nloc, d_e2cp, d_e2c, ncand, d_pp, d_pd, d_con, \
                                          stage, nv, cnt, err)
    switch (cap) {
      case 32: VK_BUILD(32); break;
      case 64: VK_BUILD(64); break;
      case 128: VK_BUILD(128); break;
      case 256: VK_BUILD(256); break;
      case 512: VK_BUILD(512); break;
      default: VK_BUILD(1024); break;
    }
#undef VK_BUILD
  }
  std::vector<int32_t> hcnt(ncand), hnv(ncand);
  int herr = 0;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ncand)
    e = cudaMemcpy(hcnt.data(), cnt, sizeof(int) * ncand, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ncand)
    e = cudaMemcpy(hnv.data(), nv, sizeof(int) * ncand, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess || herr) {
    if (e != cudaSuccess)
      vk::set_error("vk_patches_build: %s", cudaGetErrorString(e));
    else
      vk::set_error("vk_patches_build: candidate %d overflows its stage", herr - 1);
    cleanup();
    return e != cudaSuccess ? VK_ERR_CUDA : VK_ERR_ARG;
  }

  // keep non-empty patches (vanka.py:64-65), offsets on the host
  auto* h = new vk_patches_s();
  h->ndof = ndof;
  h->weighting = weighting;
  std::vector<int32_t> kept, keptnv;
  kept.reserve(ncand);
  for (int i = 0; i < ncand; ++i)
    if (hcnt[i] > 0) {
      kept.push_back(i);
      keptnv.push_back(hnv[i]);
    }
  h->npatch = static_cast<int32_t>(kept.size());
  h->h_off.assign(h->npatch + 1, 0);
  int smax = 0;
  for (int p = 0; p < h->npatch; ++p) {
    h->h_off[p + 1] = h->h_off[p] + hcnt[kept[p]];
    smax = std::max(smax, hcnt[kept[p]]);
  }
  h->smax = smax;
  h->total = h->h_off[h->npatch];

  st = upload(&h->off, h->h_off.data(), h->npatch + 1);
  if (!st) st = upload(&h->cand, kept.data(), kept.size());
  if (!st) st = upload(&h->nvel, keptnv.data(), keptnv.size());
  e = cudaSuccess;
  if (!st) {
    e = cudaMalloc(&h->idx, sizeof(int) * std::max<int64_t>(h->total, 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->w, sizeof(double) * std::max<int64_t>(h->total, 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->zbuf, sizeof(double) * std::max<int64_t>(h->total, 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->mult, sizeof(int) * std::max(ndof, 1));
    if (e == cudaSuccess) e = cudaMemset(h->mult, 0, sizeof(int) * std::max(ndof, 1));
  }
  if (st || e != cudaSuccess) {
    if (e != cudaSuccess) vk::set_error("vk_patches_build: %s", cudaGetErrorString(e));
    cleanup();
    vk_patches_free(h);
    return st ? st : VK_ERR_CUDA;
  }
  if (h->npatch > 0) {
    const int grid = std::min((h->npatch + 7) / 8, 148 * 16);
    fill_kernel<<<grid, 256>>>(h->npatch, cap, h->cand, stage, h->off, h->idx, h->mult);
    weights_kernel<<<grid, 256>>>(h->npatch, weighting == VK_WEIGHT_INVMULT, h->off, h->nvel,
                                  h->idx, h->mult, h->w);
  }
  e = cudaGetLastError();
  cleanup();
  if (e != cudaSuccess) {
    vk::set_error("vk_patches_build: %s", cudaGetErrorString(e));
    vk_patches_free(h);
    return VK_ERR_CUDA;
  }
  st = build_slot_map(h);
  if (st) {
    vk_patches_free(h);
    return st;
  }
  *out = h;
  return VK_OK;
}

extern "C" int vk_patches_from_lists(const int64_t* offsets, const int32_t* indices,
                                     const int32_t* num_velocity, const double* weights,
                                     int32_t npatch, int32_t ndof, vk_patches_t* out) {
  VK_REQUIRE(out && offsets && num_velocity && npatch >= 0 && ndof >= 0,
             "vk_patches_from_lists: bad argument");
  for (int p = 0; p < npatch; ++p)
    VK_REQUIRE(offsets[p + 1] >= offsets[p], "vk_patches_from_lists: offsets must be nondecreasing");
  const int64_t in_total = offsets[npatch] - offsets[0];
  VK_REQUIRE(in_total == 0 || indices, "vk_patches_from_lists: null indices");
  // size-0 patches contribute nothing to the sweep and have no block to
  // factor: they are dropped like the reference's _finish drops empty
  // patches (vanka.py:64-65); cand_of_patch maps kept -> input position
  std::vector<int32_t> cand, nv;
  std::vector<int64_t> koff(1, 0);
  std::vector<int32_t> hi;
  std::vector<double> kw;
  hi.reserve(in_total);
  for (int p = 0; p < npatch; ++p) {
    const int64_t a = offsets[p], b = offsets[p + 1];
    if (b == a) continue;
    cand.push_back(p);
    nv.push_back(num_velocity[p]);
    hi.insert(hi.end(), indices + (a - offsets[0]), indices + (b - offsets[0]));
    if (weights) kw.insert(kw.end(), weights + (a - offsets[0]), weights + (b - offsets[0]));
    koff.push_back(koff.back() + (b - a));
  }
  auto* h = new vk_patches_s();
  h->ndof = ndof;
  h->npatch = static_cast<int32_t>(cand.size());
  h->weighting = weights ? VK_WEIGHT_INVMULT : VK_WEIGHT_UNIT;
  h->h_off = koff;
  h->total = koff.back();
  int smax = 0;
  for (int p = 0; p < h->npatch; ++p)
    smax = std::max<int>(smax, static_cast<int>(koff[p + 1] - koff[p]));
  h->smax = smax;
  for (int64_t k = 0; k < h->total; ++k)
    if (hi[k] < 0 || hi[k] >= ndof) {
      vk_patches_free(h);
      vk::set_error("vk_patches_from_lists: index %d out of range", hi[k]);
      return VK_ERR_ARG;
    }
  for (int p = 0; p < h->npatch; ++p)
    for (int64_t k = koff[p] + 1; k < koff[p + 1]; ++k)
      if (hi[k - 1] >= hi[k]) {
        vk_patches_free(h);
        vk::set_error("vk_patches_from_lists: patch %d indices must be sorted and duplicate-free",
                      cand[p]);
        return VK_ERR_ARG;
      }
  npatch = h->npatch;
  const int32_t* num_velocity_k = nv.data();
  const double* weights_k = weights ? kw.data() : nullptr;
  std::vector<double> hw;
  if (!weights_k) hw.assign(std::max<int64_t>(h->total, 1), 1.0);
  int st = upload(&h->off, h->h_off.data(), npatch + 1);
  if (!st) st = upload(&h->idx, hi.data(), h->total);
  if (!st) st = upload(&h->nvel, num_velocity_k, npatch);
  if (!st) st = upload(&h->w, weights_k ? weights_k : hw.data(), h->total);
  if (!st) st = upload(&h->cand, cand.data(), npatch);
  if (st) {
    vk_patches_free(h);
    return st;
  }
  cudaError_t e = cudaMalloc(&h->zbuf, sizeof(double) * std::max<int64_t>(h->total, 1));
  if (e == cudaSuccess) e = cudaMalloc(&h->mult, sizeof(int) * std::max(ndof, 1));
  if (e == cudaSuccess) e = cudaMemset(h->mult, 0, sizeof(int) * std::max(ndof, 1));
  if (e == cudaSuccess && h->total) {
    count_kernel<<<vk_grid(h->total, 256), 256>>>(h->total, h->idx, h->mult);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    vk::set_error("vk_patches_from_lists: %s", cudaGetErrorString(e));
    vk_patches_free(h);
    return VK_ERR_CUDA;
  }
  st = build_slot_map(h);
  if (st) {
    vk_patches_free(h);
    return st;
  }
  *out = h;
  return VK_OK;
}

extern "C" int vk_patches_info(vk_patches_t h, int32_t* npatch, int64_t* total, int32_t* smax) {
  VK_REQUIRE(h, "vk_patches_info: null handle");
  if (npatch) *npatch = h->npatch;
  if (total) *total = h->total;
  if (smax) *smax = h->smax;
  return VK_OK;
}

extern "C" int vk_patches_export(vk_patches_t h, int64_t* offsets, int32_t* indices,
                                 int32_t* num_velocity, double* weights, double* multiplicity,
                                 int32_t* cand_of_patch) {
  VK_REQUIRE(h, "vk_patches_export: null handle");
  if (offsets) std::copy(h->h_off.begin(), h->h_off.end(), offsets);
  if (indices && h->total)
    VK_CHECK_CUDA(cudaMemcpy(indices, h->idx, sizeof(int) * h->total, cudaMemcpyDeviceToHost));
  if (num_velocity && h->npatch)
    VK_CHECK_CUDA(cudaMemcpy(num_velocity, h->nvel, sizeof(int) * h->npatch, cudaMemcpyDeviceToHost));
  if (weights && h->total)
    VK_CHECK_CUDA(cudaMemcpy(weights, h->w, sizeof(double) * h->total, cudaMemcpyDeviceToHost));
  if (cand_of_patch && h->npatch)
    VK_CHECK_CUDA(cudaMemcpy(cand_of_patch, h->cand, sizeof(int) * h->npatch, cudaMemcpyDeviceToHost));
  if (multiplicity && h->ndof) {
    std::vector<int32_t> m(h->ndof);
    VK_CHECK_CUDA(cudaMemcpy(m.data(), h->mult, sizeof(int) * h->ndof, cudaMemcpyDeviceToHost));
    for (int d = 0; d < h->ndof; ++d) multiplicity[d] = static_cast<double>(m[d]);
  }
  return VK_OK;
}

extern "C" int vk_patches_destroy(vk_patches_t h) {
  vk_patches_free(h);
  return VK_OK;
}
