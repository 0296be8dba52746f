/* Plain-C client of libvanka_b200.so (include/vanka_b200.h): builds a small
 * 1-D Laplacian, three overlapping patches, factors them, applies one
 * additive sweep and one residual on the device, and checks the results
 * against a CPU computation.  Device buffers come from the CUDA runtime
 * directly; no Python, no torch.  Exit 0 on success.
 *   gcc -O2 -Iinclude tests/c/abi_demo.c -Lpaper_2409_14222_b200 -lvanka_b200 \
 *       -L/usr/local/cuda/lib64 -lcudart -o /tmp/abi_demo */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "vanka_b200.h"

#define N 8
#define CK(x)                                                           \
  do {                                                                  \
    int rc_ = (x);                                                      \
    if (rc_ != VK_OK) {                                                 \
      fprintf(stderr, "%s -> %d: %s\n", #x, rc_, vk_last_error());     \
      return 1;                                                         \
    }                                                                   \
  } while (0)

static void solve_dense(int s, double* a, double* b) { /* Gaussian elimination, no pivoting (SPD) */
  for (int k = 0; k < s; ++k)
    for (int i = k + 1; i < s; ++i) {
      double f = a[i * s + k] / a[k * s + k];
      for (int j = k; j < s; ++j) a[i * s + j] -= f * a[k * s + j];
      b[i] -= f * b[k];
    }
  for (int i = s - 1; i >= 0; --i) {
    double t = b[i];
    for (int j = i + 1; j < s; ++j) t -= a[i * s + j] * b[j];
    b[i] = t / a[i * s + i];
  }
}

int main(void) {
  /* A = tridiag(-1, 2, -1) */
  int32_t indptr[N + 1], indices[3 * N];
  double data[3 * N], dense[N * N];
  int nnz = 0;
  memset(dense, 0, sizeof dense);
  for (int i = 0; i < N; ++i) {
    indptr[i] = nnz;
    for (int j = i - 1; j <= i + 1; ++j)
      if (j >= 0 && j < N) {
        indices[nnz] = j;
        data[nnz] = (i == j) ? 2.0 : -1.0;
        dense[i * N + j] = data[nnz];
        ++nnz;
      }
  }
  indptr[N] = nnz;
  vk_csr_t A;
  CK(vk_csr_create(indptr, indices, data, N, N, nnz, &A));

  /* patches {0..3}, {2..5}, {4..7}, inverse-multiplicity weights */
  int64_t offs[4] = {0, 4, 8, 12};
  int32_t idx[12] = {0, 1, 2, 3, 2, 3, 4, 5, 4, 5, 6, 7};
  int32_t nvel[3] = {4, 4, 4};
  double mult[N] = {0}, w[12];
  for (int k = 0; k < 12; ++k) mult[idx[k]] += 1.0;
  for (int k = 0; k < 12; ++k) w[k] = 1.0 / mult[idx[k]];
  vk_patches_t P;
  CK(vk_patches_from_lists(offs, idx, nvel, w, 3, N, &P));
  int32_t status[3], bad = -1;
  CK(vk_patches_factor(P, A, status, &bad));

  double r[N], out[N], ref[N];
  for (int i = 0; i < N; ++i) r[i] = sin(1.0 + i);
  double *dr, *dout, *dres;
  if (cudaMalloc((void**)&dr, sizeof r) || cudaMalloc((void**)&dout, sizeof out) ||
      cudaMalloc((void**)&dres, sizeof out))
    return 2;
  cudaMemcpy(dr, r, sizeof r, cudaMemcpyHostToDevice);
  CK(vk_patches_apply(P, dr, dout, 1.0, VK_APPLY_OUT, NULL, NULL));
  CK(vk_device_sync());
  cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);

  /* CPU reference: out = sum_p R^T W A_p^{-1} R r (reference vanka.py:142-148) */
  memset(ref, 0, sizeof ref);
  for (int p = 0; p < 3; ++p) {
    double a[16], b[4];
    for (int i = 0; i < 4; ++i) {
      b[i] = r[idx[4 * p + i]];
      for (int j = 0; j < 4; ++j) a[i * 4 + j] = dense[idx[4 * p + i] * N + idx[4 * p + j]];
    }
    solve_dense(4, a, b);
    for (int i = 0; i < 4; ++i) ref[idx[4 * p + i]] += w[4 * p + i] * b[i];
  }
  double err = 0.0;
  for (int i = 0; i < N; ++i) err = fmax(err, fabs(out[i] - ref[i]));

  /* residual r - A x with x = out */
  CK(vk_residual(A, dr, dout, dres, NULL));
  CK(vk_device_sync());
  double res[N], rerr = 0.0;
  cudaMemcpy(res, dres, sizeof res, cudaMemcpyDeviceToHost);
  for (int i = 0; i < N; ++i) {
    double ax = 0.0;
    for (int k = indptr[i]; k < indptr[i + 1]; ++k) ax += data[k] * out[indices[k]];
    rerr = fmax(rerr, fabs(res[i] - (r[i] - ax)));
  }
  printf("abi_demo: sweep max err %.3e, residual max err %.3e\n", err, rerr);
  vk_patches_destroy(P);
  vk_csr_destroy(A);
  cudaFree(dr);
  cudaFree(dout);
  cudaFree(dres);
  return (err < 1e-13 && rerr == 0.0) ? 0 : 3;
}
