// Adjoint at scattered points (favest/scalar.py:120-128 with ylm_table,
// favest/legendre.py:106-123): f(x_p) = sum_{l,m} g_{l,m} sigma_m Pbar_l^|m|(z_p) e^{i m phi_p}.
//
// One thread per point.  Orders are walked in sequence so the diagonal seed is
// a running product (extended range), the l-recurrence runs in registers, and
// the merged coefficient rows (sigma applied, m-major) are read as warp-uniform
// broadcasts.  The per-point recurrence cannot be shared between points, so
// this kernel is FP64-pipe bound on the recurrence plus 12*nfields FMA per
// (l, m, point).
#pragma once
#include "common.cuh"

namespace fv {

struct PtsArgs {
  const double* xyz;        // (M, 3) unit points
  long long M;
  const double* Grow;       // rows at rowofs[m] + (l - m), 12*nfields doubles: col 12b+4c+2s+ri
  const long long* rowofs;
  const double2* ab;
  const long long* abofs;
  double2* T;               // (B_total, M, 3)
  int Lt, B_total, b0;
};

template <int NF>
__global__ void __launch_bounds__(128) adjoint_points_kernel(PtsArgs a) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.M) return;
  const double x = a.xyz[3 * p], y = a.xyz[3 * p + 1], zr = a.xyz[3 * p + 2];
  const double t = fmin(1.0, fmax(-1.0, zr));
  const double s = sqrt(fmax(0.0, 1.0 - t * t));
  double phi = atan2(y, x);
  if (phi < 0.0) phi += 6.283185307179586;  // np.mod(atan2, 2*pi) (favest/core.py:82)
  constexpr int NC = 12 * NF;
  double out[NF][6];
#pragma unroll
  for (int b = 0; b < NF; ++b)
#pragma unroll
    for (int c = 0; c < 6; ++c) out[b][c] = 0.0;
  double seed = 0.28209479177387814;
  int se = 0;
  const int Lt = a.Lt;
  for (int m = 0; m <= Lt; ++m) {
    if (m > 0) {
      const double c = sqrt((2 * m + 1) / (2.0 * m));
      seed = __dmul_rn(__dmul_rn(-c, s), seed);
      if (fabs(seed) < 0x1p-512 && seed != 0.0) {
        seed *= 0x1p512;
        se -= XR_SHIFT;
      }
    }
    double acc[NF][12];
#pragma unroll
    for (int b = 0; b < NF; ++b)
#pragma unroll
      for (int c = 0; c < 12; ++c) acc[b][c] = 0.0;
    const double* rows = a.Grow + (size_t)a.rowofs[m] * NC;
    double p2 = seed, p1 = __dmul_rn(__dmul_rn(sqrt(2 * m + 3.0), t), seed);
    int e = se;
    const double2* abm = a.ab + a.abofs[m];
    for (int l = m; l <= Lt; ++l) {
      double v;
      if (l == m) {
        v = p2;
      } else if (l == m + 1) {
        v = p1;
      } else {
        const double2 abv = abm[l - m - 2];  // (a_l, a_l * b_l)
        const double pn = fma(abv.x * t, p1, -(abv.y * p2));
        p2 = p1;
        p1 = pn;
        if (e < 0 && fabs(p1) >= 0x1p512) {
          p1 *= 0x1p-512;
          p2 *= 0x1p-512;
          e += XR_SHIFT;
        }
        v = p1;
      }
      if (e < 0) v = xr_value(v, e);
      const double* row = rows + (size_t)(l - m) * NC;
#pragma unroll
      for (int b = 0; b < NF; ++b)
#pragma unroll
        for (int c = 0; c < 12; c += 2) {
          const double2 g = __ldg(reinterpret_cast<const double2*>(row + 12 * b + c));
          acc[b][c] = fma(v, g.x, acc[b][c]);
          acc[b][c + 1] = fma(v, g.y, acc[b][c + 1]);
        }
    }
    double sn, cs;
    sincos(phi * m, &sn, &cs);
#pragma unroll
    for (int b = 0; b < NF; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // + order: e^{i m phi} * acc_+
        const double pr = acc[b][4 * c + 0], pi = acc[b][4 * c + 1];
        out[b][2 * c] += cs * pr - sn * pi;
        out[b][2 * c + 1] += cs * pi + sn * pr;
        if (m > 0) {  // - order: e^{-i m phi} * acc_-
          const double nr = acc[b][4 * c + 2], ni = acc[b][4 * c + 3];
          out[b][2 * c] += cs * nr + sn * ni;
          out[b][2 * c + 1] += cs * ni - sn * nr;
        }
      }
  }
#pragma unroll
  for (int b = 0; b < NF; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      a.T[((size_t)(a.b0 + b) * a.M + p) * 3 + c] = make_double2(out[b][2 * c], out[b][2 * c + 1]);
}

}  // namespace fv
