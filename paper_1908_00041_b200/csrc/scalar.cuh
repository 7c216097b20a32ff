// Scalar spherical harmonic transforms (favest/scalar.py:94-128, 146-184:
// forward_sht_fast / adjoint_sht_fast / forward_sht_direct / adjoint_sht_direct)
// through the vector machinery: B scalar fields ride as the three Cartesian
// components of ceil(B / 3) pseudo fields (scalar field s = component s % 3 of
// pseudo field s / 3), so the ring DFTs, the folded Legendre contractions and
// the scattered-point kernels run unchanged.  The forward Legendre output rows F
// already hold the scalar coefficients of every component (sigma and the ring
// weights applied); the Clebsch-Gordan stage is replaced by an unpack, and on
// the adjoint side the coupling by a pack of the scalar coefficients into the
// same G layouts (fragment tiles with gamma_l for the grid, plain rows for
// points).
#pragma once
#include "common.cuh"

namespace fv {

// f [B][n] -> Tp [K][n][3] (zeros for the padding components of the last pseudo field)
__global__ void scalar_to_pseudo_kernel(const double2* __restrict__ f, long long n, int B, double2* __restrict__ Tp,
                                        long long total) {
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(idx % 3);
    const long long r = idx / 3;
    const long long i = r % n, k = r / n;
    const long long s = 3 * k + c;
    Tp[idx] = s < B ? f[s * n + i] : make_double2(0.0, 0.0);
  }
}

// Tp [K][n][3] -> f [B][n]
__global__ void pseudo_to_scalar_kernel(const double2* __restrict__ Tp, long long n, int B, double2* __restrict__ f) {
  const long long total = (long long)B * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long s = idx / n, i = idx % n;
    f[idx] = Tp[((s / 3) * n + i) * 3 + s % 3];
  }
}

// forward Legendre rows of pseudo fields pf0 .. pf0 + nfp - 1 (F rows tri(l, |m|),
// ncol doubles: col 12 b + 4 c + 2 sign + re/im) -> flat scalar coefficients
// out[s][l^2 + l + m], l <= lmax (favest/core.py:23-37)
__global__ void scalar_unpack_kernel(const double* __restrict__ F, int ncol, int lmax, int pf0, int nfp, int B,
                                     double2* __restrict__ out) {
  const int l = blockIdx.y;
  const int am = blockIdx.x * blockDim.x + threadIdx.x;
  if (am > l) return;
  const double* row = F + ((size_t)l * (l + 1) / 2 + am) * ncol;
  const long long K = (long long)(lmax + 1) * (lmax + 1);
  for (int b = 0; b < nfp; ++b)
    for (int c = 0; c < 3; ++c) {
      const int s = 3 * (pf0 + b) + c;
      if (s >= B) return;
      const double* v = row + 12 * b + 4 * c;
      double2* o = out + s * K + (long long)l * l + l;
      o[am] = make_double2(v[0], v[1]);
      if (am > 0) o[-am] = make_double2(v[2], v[3]);
    }
}

struct ScalarPackArgs {
  const double2* g;         // [B][(lmax + 1)^2] flat scalar coefficients
  int lmax, B, pf0, nfp;    // pseudo fields pf0 .. pf0 + nfp - 1 of this group
  double* G;                // grid: fragment tiles (gofs), points: rows (rowofs)
  const long long* gofs;
  const long long* rowofs;
  const double2* dg;        // grid mode: gamma_l (the Legendre adjoint's block rescaling)
  const long long* dgofs;
  int Lt, NT, rows_mode, m_begin;
};

// Merged-coefficient layout of cg_adj_kernel (aux_kernels.cuh) with the scalar
// coefficients of each component in place of the coupled g^X, g^Y, g^Z:
// column 12 b + 4 c + 2 sign + re/im = sigma_M (gamma_l) g_{3 (pf0 + b) + c}[l, M].
__global__ void scalar_pack_kernel(ScalarPackArgs a) {
  const int mi = blockIdx.y;
  const long long am = a.m_begin + mi;
  const int nrows = a.Lt + 1 - (int)am;
  constexpr int LC = 32, KS = LC / 8;  // legendre.cuh ADJ_LC / ADJ_KS
  const int nlc = (nrows + LC - 1) / LC;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (a.rows_mode ? nrows : LC * nlc)) return;
  const long long l = am + row;
  const int lc = row / LC, idx = row % LC;
  const int par = idx & 1, k = idx >> 1, ks = k >> 2, q = k & 3;
  double* Gt = a.rows_mode ? a.G + (size_t)(a.rowofs[am] + row) * (12 * a.nfp)
                           : a.G + (size_t)(a.gofs[am] + lc) * (2 * KS * a.NT * 32);
  auto put = [&](int n, double v) {
    if (a.rows_mode)
      Gt[n] = v;
    else
      Gt[((size_t)(par * KS + ks) * a.NT + (n >> 3)) * 32 + ((n & 7) << 2) + q] = v;
  };
  if (!a.rows_mode)
    for (int n = 12 * a.nfp; n < 8 * a.NT; ++n) put(n, 0.0);
  const bool live = l <= a.Lt;
  double gam = 1.0;
  if (!a.rows_mode && live) gam = a.dg[a.dgofs[am] + (l - am)].y;  // gamma_l (legendre.cuh)
  const long long K = (long long)(a.lmax + 1) * (a.lmax + 1);
  for (int b = 0; b < a.nfp; ++b)
    for (int c = 0; c < 3; ++c) {
      const int s = 3 * (a.pf0 + b) + c;
      for (int sg = 0; sg < 2; ++sg) {
        double2 v = make_double2(0.0, 0.0);
        if (live && s < a.B && l <= a.lmax && !(sg == 1 && am == 0)) {
          const long long M = sg ? -am : am;
          v = a.g[s * K + l * l + l + M];
          const double sig = ((M < 0 && (am & 1)) ? -1.0 : 1.0) * gam;  // favest/legendre.py:101-103
          v.x *= sig;
          v.y *= sig;
        }
        const int n0 = 12 * b + 4 * c + 2 * sg;
        put(n0, v.x);
        put(n0 + 1, v.y);
      }
    }
}

}  // namespace fv
