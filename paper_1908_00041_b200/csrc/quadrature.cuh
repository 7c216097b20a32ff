// Gauss-Legendre rule on the device (favest/quadrature.py:29-48 obtains the
// rule from scipy.special.roots_legendre on the host).
//
// One thread per root pair (+-x): Newton's method on the colatitude theta of
// P_n(cos theta) = 0, from Tricomi's asymptotic guess
//   theta_k ~ pi (4k - 1) / (4n + 2),  cos theta_k (1 - (n - 1) / (8 n^3)),
// with P_n, P_{n-1} by the three-term recurrence at z = cos(theta) and
//   d/dtheta P_n(cos theta) = n (z P_n - P_{n-1}) / sin(theta),
// the recurrence run in difference form on u = 1 - cos(theta) = 2 sin^2(theta/2)
// (see legendre_pair_u), and the weight
//   w = 2 sin^2(theta) / (n P_{n-1}(cos theta))^2.
// Outputs are ring colatitudes (ascending) and Gauss weights, i.e. the
// reference's arccos(nodes[::-1]) and gauss_w[::-1] without the arccos.
// This is a deliberate deviation from the reference's scipy weights when used
// (gen_gl_tensor(..., on_device=True)): more accurate polar weights, not
// bitwise the reference's; the default path keeps scipy's.
#pragma once
#include <cuda_runtime.h>

namespace fv {

// P_n, P_{n-1} and D_n = P_n - P_{n-1} at z = 1 - u, by the recurrence in
// difference form (D_j = ((j - 1) D_{j-1} - (2j - 1) u P_{j-1}) / j,
// P_j = P_{j-1} + D_j, an exact rearrangement of the three-term recurrence):
// near the pole z = cos(theta) itself carries only ~eps / u relative information
// about u = 1 - z = 2 sin^2(theta / 2), which costs the polar weights 1e-9 ..
// 1e-7 (what scipy's rule shows); with u computed from theta directly they stay
// at rounding level.
__device__ __forceinline__ void legendre_pair_u(int n, double u, double& pn, double& pn1, double& dn) {
  double p = 1.0, d = 0.0, pprev = 0.0;  // P_0, D_0 (unused), P_{-1}
  for (int j = 1; j <= n; ++j) {
    const double dj = (j == 1) ? -u : fma((double)(j - 1), d, -(2.0 * j - 1.0) * u * p) / j;
    pprev = p;
    p += dj;
    d = dj;
  }
  pn = p;
  pn1 = pprev;
  dn = d;
}

__global__ void gauss_legendre_kernel(int n, double* theta, double* w) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;  // root pair k: the (k+1)-th smallest colatitude
  const int half = (n + 1) / 2;
  if (k >= half) return;
  const double pi = 3.141592653589793238462643383279502884;
  double th;
  if ((n & 1) && k == half - 1) {
    th = 0.5 * pi;  // the middle root of an odd rule: exactly the equator
  } else {
    const double nd = (double)n;
    const double t0 = pi * (4.0 * (k + 1) - 1.0) / (4.0 * nd + 2.0);
    th = acos(cos(t0) * (1.0 - (nd - 1.0) / (8.0 * nd * nd * nd)));
    // Newton on f(theta) = P_n(cos theta): f' = n (z P_n - P_{n-1}) / sin(theta)
    //                                         = n (D_n - u P_n) / sin(theta)
    for (int it = 0; it < 30; ++it) {
      const double sh = sin(0.5 * th), u = 2.0 * sh * sh, s = sin(th);
      double pn, pn1, dn;
      legendre_pair_u(n, u, pn, pn1, dn);
      const double dth = pn * s / (nd * (dn - u * pn));
      th -= dth;
      if (fabs(dth) <= 4e-16 * th) break;
    }
  }
  const double sh = sin(0.5 * th), u = 2.0 * sh * sh, s = sin(th);
  double pn, pn1, dn;
  legendre_pair_u(n, u, pn, pn1, dn);
  const double wk = 2.0 * s * s / ((double)n * pn1 * ((double)n * pn1));
  theta[k] = th;
  w[k] = wk;
  if (n - 1 - k != k) {
    theta[n - 1 - k] = pi - th;
    w[n - 1 - k] = wk;
  }
}

}  // namespace fv
