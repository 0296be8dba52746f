// Per-point geometry shared by the assembly and error-norm kernels: the
// Jacobian of the affine (triangle) / bilinear (quadrilateral) cell map and
// the push-forward of reference basis data (reference elements.py:487-570).
#pragma once

namespace {

// per-quadrature-point Jacobian of the affine (tri) / bilinear (quad) map
__device__ __forceinline__ void jacobian(int quad, const double* __restrict__ xy, double x,
                                         double y, double J[2][2], double& det, double inv[2][2]) {
  const double x0 = xy[0], y0 = xy[1];
  J[0][0] = xy[2] - x0;
  J[1][0] = xy[3] - y0;
  J[0][1] = xy[4] - x0;
  J[1][1] = xy[5] - y0;
  if (quad) {
    const double tx = x0 - xy[2] - xy[4] + xy[6], ty = y0 - xy[3] - xy[5] + xy[7];
    J[0][0] += y * tx;
    J[1][0] += y * ty;
    J[0][1] += x * tx;
    J[1][1] += x * ty;
  }
  det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  inv[0][0] = J[1][1] / det;
  inv[0][1] = -J[0][1] / det;
  inv[1][0] = -J[1][0] / det;
  inv[1][1] = J[0][0] / det;
}

// physical gradient (c, a) and value (c) of reference basis function data
// rv[c], rg[c][d] under the identity (gradients by J^-T) or Piola map
__device__ __forceinline__ void push(int piola, const double J[2][2], double det,
                                     const double inv[2][2], const double rv[2],
                                     const double rg[2][2], double pv[2], double pg[2][2]) {
  if (!piola) {
    pv[0] = rv[0];
    pv[1] = rv[1];
    for (int c = 0; c < 2; ++c)
      for (int a = 0; a < 2; ++a) pg[c][a] = rg[c][0] * inv[0][a] + rg[c][1] * inv[1][a];
    return;
  }
  for (int c = 0; c < 2; ++c) pv[c] = (J[c][0] * rv[0] + J[c][1] * rv[1]) / det;
  double jg[2][2];
  for (int c = 0; c < 2; ++c)
    for (int b = 0; b < 2; ++b) jg[c][b] = J[c][0] * rg[0][b] + J[c][1] * rg[1][b];
  for (int c = 0; c < 2; ++c)
    for (int a = 0; a < 2; ++a) pg[c][a] = (jg[c][0] * inv[0][a] + jg[c][1] * inv[1][a]) / det;
}

// physical point of reference (xi, eta): v0 + [v1 - v0, v2 - v0] (xi, eta)
// (+ xi eta (v0 - v1 - v2 + v3) on quadrilaterals)
__device__ __forceinline__ void map_point(int quad, const double* __restrict__ xy, double xi,
                                          double eta, double& x, double& y) {
  x = xy[0] + (xi * (xy[2] - xy[0]) + eta * (xy[4] - xy[0]));
  y = xy[1] + (xi * (xy[3] - xy[1]) + eta * (xy[5] - xy[1]));
  if (quad) {
    x += xi * eta * (xy[0] - xy[2] - xy[4] + xy[6]);
    y += xi * eta * (xy[1] - xy[3] - xy[5] + xy[7]);
  }
}

}  // namespace
