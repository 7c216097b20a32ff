// Setup, layout and Clebsch-Gordan kernels around the Legendre contraction.
//
//   seeds_kernel      Pbar_m^m(t_p) for every order and ring pair, extended
//                     range (favest/legendre.py:60-65)
//   ab_kernel         recurrence coefficients a_lm, b_lm (favest/legendre.py:70-71)
//   fold_fwd_kernel   ring spectra -> folded, weighted Cartesian components in
//                     DMMA fragment order (favest/scalar.py:149-152); used by
//                     the order-sharded path, the grid path fuses it into the
//                     FFT (fft2.cuh fft_fold_kernel)
//   cg_fwd_kernel     F^x, F^y, F^z -> combos F^U, F^V, F^W
//                     (favest/transforms.py:109-112, applied after the linear
//                     scalar transform) -> a_lm, b_lm (favest/transforms.py:120-146)
//   cg_adj_kernel     a_lm, b_lm -> merged g^X, g^Y, g^Z in fragment order
//                     (favest/coupling.py:200-240, favest/transforms.py:165-175)
#pragma once
#include "common.cuh"

namespace fv {

constexpr double INV_SQRT_4PI_D = 0.28209479177387814;  // 1/sqrt(4*pi), favest/legendre.py:24

// One thread per ring pair; sequential over m exactly like the reference's
// diagonal loop, renormalising by 2^512 below 2^-512 (oracle.seed_table).
__global__ void seeds_kernel(const double* __restrict__ pair_s, int nPpad, int Lt, double* seed_x,
                             int* seed_e) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nPpad) return;
  const double s = pair_s[p];
  double cur = INV_SQRT_4PI_D;
  int e = 0;
  seed_x[p] = cur;
  seed_e[p] = 0;
  for (int m = 1; m <= Lt; ++m) {
    const double c = sqrt((2 * m + 1) / (2.0 * m));
    cur = __dmul_rn(__dmul_rn(-c, s), cur);
    if (fabs(cur) < 0x1p-512 && cur != 0.0) {
      cur *= 0x1p512;
      e -= XR_SHIFT;
    }
    seed_x[(size_t)m * nPpad + p] = cur;
    seed_e[(size_t)m * nPpad + p] = e;
  }
}

// Polar start (legendre.cuh): per (order m, ring pair p) the first degree
// l_s >= m with |Pbar_{l_s}^m(t_p)| >= 2^-100 and the values (P_ls, P_ls+1),
// found by running the recurrence in extended range from the diagonal seed.
// l_s = Lt+1 when no degree <= Lt reaches the threshold (and for padding pairs).
// Uses the same FMA-form step as the hot loop (legendre.cuh rec_step).
__device__ __forceinline__ bool xr_significant(double x, int e) {
  return e == 0 ? fabs(x) >= 0x1p-100 : (e == -XR_SHIFT ? fabs(x) >= 0x1p412 : false);
}

__global__ void start_kernel(const double* __restrict__ seed_x, const int* __restrict__ seed_e,
                             const double* __restrict__ pair_t, const int* __restrict__ pair_n,
                             const double2* __restrict__ ab, const long long* __restrict__ abofs,
                             const double2* __restrict__ dg, const long long* __restrict__ dgofs, int nPpad,
                             int Lt, int* start_l, double2* start_v) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (p >= nPpad) return;
  const size_t o = (size_t)m * nPpad + p;
  int ls = Lt + 1;
  double A = 0.0, B = 0.0;
  if (pair_n[p] >= 0) {
    const double t = pair_t[p];
    const double2* abm = ab + abofs[m];
    int e = seed_e[o];
    double p2 = seed_x[o];                                        // P_m^m
    double p1 = (m < Lt) ? (sqrt(2 * m + 3.0) * t) * p2 : 0.0;   // P_{m+1}^m
    auto step = [&](int l, double q1, double q2) {                // P_l from P_{l-1}, P_{l-2}
      const double2 ac = abm[l - m - 2];
      return fma(ac.x * t, q1, -(ac.y * q2));
    };
    if (xr_significant(p2, e)) {
      ls = m;
      A = xr_value(p2, e);
      B = (m < Lt) ? xr_value(p1, e) : 0.0;
    } else if (m < Lt && xr_significant(p1, e)) {
      ls = m + 1;
      A = xr_value(p1, e);
      B = (m + 2 <= Lt) ? xr_value(step(m + 2, p1, p2), e) : 0.0;
    } else {
      for (int l = m + 2; l <= Lt; ++l) {
        const double pn = step(l, p1, p2);
        p2 = p1;
        p1 = pn;
        if (e < 0 && fabs(p1) >= 0x1p512) {
          p1 *= 0x1p-512;
          p2 *= 0x1p-512;
          e += XR_SHIFT;
        }
        if (xr_significant(p1, e)) {
          ls = l;
          A = xr_value(p1, e);
          B = (l + 1 <= Lt) ? xr_value(step(l + 1, p1, p2), e) : 0.0;
          break;
        }
      }
    }
  }
  // injected in block-rescaled units R = P / gamma (legendre.cuh)
  if (ls <= Lt) {
    const double2* dgm = dg + dgofs[m];
    A = A / dgm[ls - m].y;
    B = (ls + 1 <= Lt) ? B / dgm[ls + 1 - m].y : 0.0;
  }
  start_l[o] = ls;
  start_v[o] = make_double2(A, B);
}

// Block-rescaled recurrence coefficients (legendre.cuh): for each order m the
// degrees are cut into 32-blocks starting at l = m; inside a block
//   P_l = gamma_l R_l,  R_l = t R_{l-1} - d_l R_{l-2},
//   gamma_l = gamma_{l-1} a_l, d_l = b_l / a_{l-1}        (interior rows)
//   gamma_l = a_l, d_l = b_l                              (first recurrence row of a block:
//                                                          l = m+2 or (l-m) % 32 == 0)
// with a_l, b_l of favest/legendre.py:70-71; rows l = m, m+1 (seeds) have
// (d, gamma) = (0, 1).  At block ends the state is converted back to P.
// One thread per (m, block).  dg[dgofs[m] + (l - m)] = (d_l, gamma_l).
__global__ void dg_kernel(int Lt, const long long* __restrict__ dgofs, double2* dg) {
  const int m = blockIdx.y;
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  const int l0 = m + 32 * blk;
  if (l0 > Lt) return;
  double2* out = dg + dgofs[m];
  auto ab_of = [&](int l, double& a, double& b) {
    const long long L2 = (long long)l * l, M2 = (long long)m * m;
    const double lf = (double)l;
    a = sqrt((4.0 * lf * lf - 1.0) / (double)(L2 - M2));
    const double lm1 = lf - 1.0;
    b = sqrt((lm1 * lm1 - (double)M2) / (4.0 * (lm1 * lm1) - 1.0));
  };
  double gam = 1.0;
  for (int l = l0; l <= min(Lt, l0 + 31); ++l) {
    if (l < m + 2) {
      out[l - m] = make_double2(0.0, 1.0);
      continue;
    }
    double a, b;
    ab_of(l, a, b);
    if (l == m + 2 || l == l0) {
      gam = a;
      out[l - m] = make_double2(b, gam);
    } else {
      double ap, bp;
      ab_of(l - 1, ap, bp);
      gam *= a;
      out[l - m] = make_double2(b / ap, gam);
    }
  }
}

// (a_l, a_l * b_l) for l = m+2..Lt, stored m-major at abofs[m] + (l - m - 2).
__global__ void ab_kernel(int Lt, const long long* __restrict__ abofs, double2* ab) {
  const int m = blockIdx.y;
  const int l = m + 2 + blockIdx.x * blockDim.x + threadIdx.x;
  if (l > Lt) return;
  const long long L2 = (long long)l * l, M2 = (long long)m * m;
  const double lf = (double)l;
  const double a = sqrt((4.0 * lf * lf - 1.0) / (double)(L2 - M2));
  const double lm1 = lf - 1.0;
  const double b = sqrt((lm1 * lm1 - (double)M2) / (4.0 * (lm1 * lm1) - 1.0));
  ab[abofs[m] + (l - m - 2)] = make_double2(a, a * b);  // FMA-form recurrence (legendre.cuh)
}

// Forward fold.  Thread per (local order mi, pair p, field b, component c):
//   E = w_n S_n + w_s S_s, O = w_n S_n - w_s S_s of the Cartesian ring spectra
//   at bins +m and -m (times sigma_{-m} on the -m bin), written as the four
//   columns 12 b + 4 c + (2 sign + re/im) of
//   X[mi][chunk][par][ks][nt][n_hi 2][k 4][n_lo 4] (B operand tiles; the
//   consumer lane (k = lane & 3, n = lane >> 2) reads 16 n_hi + 4 k + n_lo),
//   one aligned 32-byte sector per parity.  The U/V/W combos of
//   favest/transforms.py:112 are formed after the (linear) scalar transform, in
//   the CG stage.  blockIdx.z == 3 nfields zeroes the padding columns.  The
//   grid path fuses this into the ring FFT (fft2.cuh fft_fold_kernel).
// per (order m, chunk c of `width` pairs): the smallest polar start among the
// chunk's pairs (legendre.cuh: the forward skips all-zero leading chunk tiles
// of each l-block, the adjoint all-zero leading stages of each item)
__global__ void chunk_start_kernel(const int* __restrict__ start_l, int nPpad, int nchunks, int width, int* cmin) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (c >= nchunks) return;
  const int* s = start_l + (size_t)m * nPpad + (size_t)c * width;
  int v = s[0];
  for (int i = 1; i < width; ++i) v = min(v, s[i]);
  cmin[(size_t)m * nchunks + c] = v;
}

struct FoldArgs {
  const double2* S;     // ring spectra, layout lay (common.cuh SLayout)
  double* X;
  const int* pair_n;
  const int* pair_s;
  const double* ring_w;
  int n_phi, n_theta, B_total, b0, nfields, NT, nPpad, nchunks, m_begin, m_count;
  SLayout lay;
};

__global__ void fold_fwd_kernel(FoldArgs a) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int mi = blockIdx.y;
  const int z = blockIdx.z;  // 3 b + c, or 3 nfields: padding columns
  if (p >= a.nPpad) return;
  const int m = a.m_begin + mi;
  const int chunk = p >> 5, ks = (p >> 2) & 7, q = p & 3;
  double* xt = a.X + ((size_t)mi * a.nchunks + chunk) * (2 * 8 * a.NT * 32) + (size_t)ks * a.NT * 32 + q * 4;
  const size_t par_stride = (size_t)8 * a.NT * 32;
  auto put4 = [&](int col, double2 v0, double2 v1, double2 o0, double2 o1) {  // col % 4 == 0
    const int off = (col >> 3) * 32 + ((col >> 2) & 1) * 16;
    st_global_v4(xt + off, v0, v1);
    st_global_v4(xt + par_stride + off, o0, o1);
  };
  const double2 zero = make_double2(0.0, 0.0);
  if (z == 3 * a.nfields) {  // padding columns 12 nf .. 8 NT - 1 (at most one group of 4)
    if (12 * a.nfields < 8 * a.NT) put4(12 * a.nfields, zero, zero, zero, zero);
    return;
  }
  const int b = z / 3, c = z % 3;
  const int rn = a.pair_n[p], rs = a.pair_s[p];
  double2 E[2] = {zero, zero}, O[2] = {zero, zero};
  if (rn >= 0) {
    const double wn = a.ring_w[rn];
    const double ws = rs >= 0 ? a.ring_w[rs] : 0.0;
    const long long rb = (long long)(a.b0 + b) * a.n_theta;
    const double2* base_n = a.S + spec_cr(a.lay, c, rb + rn);
    const double2* base_s = rs >= 0 ? a.S + spec_cr(a.lay, c, rb + rs) : base_n;
    for (int sgn = 0; sgn < 2; ++sgn) {
      if (sgn == 1 && m == 0) break;
      const long long bin = spec_bin(a.lay, m, sgn, a.n_phi);
      const double sig = (sgn == 1 && (m & 1)) ? -1.0 : 1.0;
      const double2 Tn = base_n[bin * a.lay.bs];
      const double nr = wn * Tn.x, ni = wn * Tn.y;
      if (rs >= 0) {
        const double2 Ts = base_s[bin * a.lay.bs];
        const double sr = ws * Ts.x, si = ws * Ts.y;
        E[sgn] = make_double2(sig * (nr + sr), sig * (ni + si));
        O[sgn] = make_double2(sig * (nr - sr), sig * (ni - si));
      } else {  // unpaired ring: both parities see the ring itself
        E[sgn] = O[sgn] = make_double2(sig * nr, sig * ni);
      }
    }
  }
  put4(12 * b + 4 * c, E[0], E[1], O[0], O[1]);
}

// ---------------------------------------------------------------------------
// Clebsch-Gordan factor table: xi^1..6, mu^1..3 (favest/coupling.py:143-170) at
// every flat position k = l*l + l + m, l <= L+1, stored as 9 arrays of K_t
// doubles (plan time; same closed forms, so bitwise the reference's values).
// ---------------------------------------------------------------------------
__global__ void cg_table_kernel(int Lt, double* cgt) {
  const long long Kt = (long long)(Lt + 1) * (Lt + 1);
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Kt) return;
  long long l = (long long)sqrt((double)k);
  while (l * l > k) --l;
  while ((l + 1) * (l + 1) <= k) ++l;
  const long long m = k - l * l - l;
#pragma unroll
  for (int i = 1; i <= 6; ++i) cgt[(i - 1) * Kt + k] = xi_coef(i, l, m);
#pragma unroll
  for (int i = 1; i <= 3; ++i) cgt[(5 + i) * Kt + k] = mu_coef(i, l, m);
}

// ---------------------------------------------------------------------------
// forward Clebsch-Gordan assembly: favest/transforms.py:120-146
// ---------------------------------------------------------------------------
struct CgFwdArgs {
  const double* F;      // rows tri(l, |m|), ncolF doubles: col 12b + 4c + 2s + ri
  double2* A;           // (B_total, K) div coefficients
  double2* Bc;          // (B_total, K) curl coefficients
  const double* cgt;    // cg_table_kernel: 9 x K_t (xi1..6, mu1..3)
  int L, ncolF, B_total, b0, nfields;
  int c_lo, c_hi;       // orders |m| written: [c_lo, c_hi) (F rows of c_lo-1 .. c_hi must be current)
  // pair-chunk split of the forward Legendre launch (legendre.cuh FwdArgs::ksplit): F
  // is the sum of nsplit partial buffers, F then Fx + (s - 1) * fx_stride for s = 1..,
  // added in this order (pointer arithmetic: an indexed pointer array would go to local memory)
  int nsplit;
  const double* Fx;
  long long fx_stride;
  // several 4-field groups in one launch (grid.z = group): F of group g at + g * fg_stride, fields b0 + 4 g ..
  long long fg_stride;
};

// U = -x + i y, V = x + i y, W = z (favest/transforms.py:112) from the
// Cartesian scalar coefficients (the scalar transform is linear)
__device__ __forceinline__ double2 combo_uvw(int comp, double2 x, double2 y, double2 z) {
  if (comp == 0) return make_double2(-x.x - y.y, -x.y + y.x);
  if (comp == 1) return make_double2(x.x - y.y, x.y + y.x);
  return z;
}

// One output (a_lm, b_lm) from its nine factors x = (xi1..6, mu1..3) and the U / V / W
// coefficients at degrees l-1 (a), l+1 (b), l (c): favest/transforms.py:137-144 in the
// reference's association order with every product and sum rounded separately, as
// numpy evaluates it (no FMA contraction), shared by all forward CG kernels so they
// agree bitwise.
__device__ __forceinline__ void cg_fwd_combine(const double (&x)[9], double2 ua, double2 ub, double2 uc, double2 va,
                                               double2 vb, double2 vc, double2 wa, double2 wb, double2 wc,
                                               double2& A, double2& B) {
  const double is2 = 0.7071067811865475;  // favest/transforms.py:46 (1/np.sqrt(2.0))
  auto part = [&](double p1, double p2, double p3, double p4, double p5, double p6) {
    const double s4 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(x[0], p1), __dmul_rn(x[1], p2)), __dmul_rn(x[2], p3)),
                                __dmul_rn(x[3], p4));
    return __dadd_rn(__dadd_rn(__dmul_rn(is2, s4), __dmul_rn(x[4], p5)), __dmul_rn(x[5], p6));
  };
  A = make_double2(part(ua.x, ub.x, va.x, vb.x, wa.x, wb.x), part(ua.y, ub.y, va.y, vb.y, wa.y, wb.y));
  // b = -i/sqrt2 (mu1 fu + mu3 fv) - i mu2 fw
  const double sr = __dadd_rn(__dmul_rn(x[6], uc.x), __dmul_rn(x[8], vc.x));
  const double si = __dadd_rn(__dmul_rn(x[6], uc.y), __dmul_rn(x[8], vc.y));
  B = make_double2(__dadd_rn(__dmul_rn(is2, si), __dmul_rn(x[7], wc.y)),
                   __dsub_rn(-__dmul_rn(is2, sr), __dmul_rn(x[7], wc.x)));
}

__device__ __forceinline__ double2 f_read(const CgFwdArgs& a, int b, int comp, long long l, long long m) {
  // scalar coefficient F^comp_{l,m} (comp 0 U, 1 V, 2 W), zero outside 0 <= l <= L+1, |m| <= l
  if (l < 0 || l > a.L + 1 || llabs(m) > l) return make_double2(0.0, 0.0);
  const long long am = llabs(m);
  const int sgn = (m < 0) ? 1 : 0;
  const double* row = a.F + ((size_t)l * (l + 1) / 2 + am) * a.ncolF + 12 * b + 2 * sgn;
  const double2 x = *reinterpret_cast<const double2*>(row);
  const double2 y = *reinterpret_cast<const double2*>(row + 4);
  const double2 z = *reinterpret_cast<const double2*>(row + 8);
  return combo_uvw(comp, x, y, z);
}

__global__ void cg_fwd_kernel(CgFwdArgs a) {
  const long long l = blockIdx.y;
  const long long am = blockIdx.x * blockDim.x + threadIdx.x;
  if (am > l) return;
  const long long K = (long long)(a.L + 1) * (a.L + 1);
  for (int sg = 0; sg < (am == 0 ? 1 : 2); ++sg) {
    const long long M = sg ? -am : am;
    // table values at the source positions (l+dl, M+dm); zero if out of range
    const long long Kt = (long long)(a.L + 2) * (a.L + 2);
    auto xi_at = [&](int i, long long ls, long long ms) -> double {
      if (ls < 0 || ls > a.L + 1 || llabs(ms) > ls) return 0.0;
      return __ldg(&a.cgt[(i - 1) * Kt + ls * ls + ls + ms]);
    };
    auto mu_at = [&](int i, long long ls, long long ms) -> double {
      if (ls < 0 || ls > a.L + 1 || llabs(ms) > ls) return 0.0;
      return __ldg(&a.cgt[(5 + i) * Kt + ls * ls + ls + ms]);
    };
    const double x1 = xi_at(1, l - 1, M - 1), x2 = xi_at(2, l + 1, M - 1);
    const double x3 = xi_at(3, l - 1, M + 1), x4 = xi_at(4, l + 1, M + 1);
    const double x5 = xi_at(5, l - 1, M), x6 = xi_at(6, l + 1, M);
    const double u1 = mu_at(1, l, M - 1), u2 = mu_at(2, l, M), u3 = mu_at(3, l, M + 1);
    for (int b = 0; b < a.nfields; ++b) {
      const double2 fu_a = f_read(a, b, 0, l - 1, M - 1), fu_b = f_read(a, b, 0, l + 1, M - 1);
      const double2 fv_a = f_read(a, b, 1, l - 1, M + 1), fv_b = f_read(a, b, 1, l + 1, M + 1);
      const double2 fw_a = f_read(a, b, 2, l - 1, M), fw_b = f_read(a, b, 2, l + 1, M);
      const double2 fu_c = f_read(a, b, 0, l, M - 1), fv_c = f_read(a, b, 1, l, M + 1);
      const double2 fw_c = f_read(a, b, 2, l, M);
      const double xs[9] = {x1, x2, x3, x4, x5, x6, u1, u2, u3};
      double2 ca, cb;
      cg_fwd_combine(xs, fu_a, fu_b, fu_c, fv_a, fv_b, fv_c, fw_a, fw_b, fw_c, ca, cb);
      double ar = ca.x, ai = ca.y, br = cb.x, bi = cb.y;
      if (l == 0) ar = ai = br = bi = 0.0;  // favest/transforms.py:145-146
      const size_t o = (size_t)(a.b0 + b) * K + l * l + l + M;
      a.A[o] = make_double2(ar, ai);
      a.Bc[o] = make_double2(br, bi);
    }
  }
}

// 16-byte cp.async global -> shared; ok == false zero-fills (src-size 0; src must still be a valid address)
__device__ __forceinline__ void cgs_cp16(void* dst_smem, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst_smem)), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}

// Tiled forward CG: CTA per (degree l, block of 32 orders |m|).  The F rows it
// reads (degrees l-1, l, l+1; orders m0-1 .. m0+32, contiguous in the tri
// layout) are staged in shared memory with coalesced 16-byte loads; thread per
// (order, field, sign).  Same arithmetic as cg_fwd_kernel (bitwise equal).
// NF (fields in the group) is a template parameter so that every index
// division is by a compile-time constant; all indices fit 32 bits.
constexpr int CGF_THREADS = 256, CGF_MB = 32;
// orders per CTA: 32 at three or four fields (one (order, field, sign) output per thread); a
// one-field launch (C4) takes 128 orders and a two-field launch 64, so every thread has an output
__host__ __device__ constexpr int cgf_mb(int nf) { return nf == 1 ? 128 : nf == 2 ? 64 : CGF_MB; }
__host__ __device__ constexpr int cgf_nt(int nf) { return (12 * nf + 7) / 8; }
__host__ __device__ constexpr int cgf_rs(int nf) { return 4 * cgf_nt(nf) + 1; }  // odd double2 row stride
template <int NF, bool SPLIT = false, bool GROUPS = false>
__global__ void __launch_bounds__(CGF_THREADS) cg_fwd_tile_kernel(CgFwdArgs a) {
  constexpr int MB = cgf_mb(NF);
  constexpr int NV = 4 * cgf_nt(NF), RS = cgf_rs(NF), ROWS = MB + 2;
  const int l = blockIdx.y;
  const int m0 = (blockIdx.x + a.c_lo / MB) * MB;  // the grid starts at the first written block
  if (m0 > l) return;
  // field group of this CTA (grid.z = 1: group 0); locals, not writes to the parameter struct
  // (a mutated kernel parameter is copied out of the constant bank: +29 us at C3)
  // (GROUPS instantiation only: the one-group kernel keeps its 80 registers and three CTAs per SM)
  const double* const Fg = GROUPS ? a.F + blockIdx.z * a.fg_stride : a.F;
  const int b0g = GROUPS ? a.b0 + 4 * blockIdx.z : a.b0;
  extern __shared__ __align__(16) double2 cgf_smem[];  // [3][ROWS][RS]
  const int Lt = a.L + 1;
  const int K = (a.L + 1) * (a.L + 1), Kt = (Lt + 1) * (Lt + 1);
  // this thread's output (order m0 + mi, field b, sign sg); its nine factors are
  // loaded together with the staging loads (one memory round trip, not one more
  // after the barrier)
  constexpr int NW = MB * NF * 2;
  static_assert(NW <= CGF_THREADS, "one (order, field, sign) output per thread");
  const int w = threadIdx.x;
  const int mi = w % MB, b = (w / MB) % NF, sg = w / (MB * NF);
  const int am = m0 + mi;
  const bool work = w < NW && am <= l && !(sg == 1 && am == 0) && am >= a.c_lo && am < a.c_hi;
  const int M = sg ? -am : am;
  auto tab = [&](int i, int ls, int ms) -> double {
    if (!work || ls < 0 || ls > Lt || abs(ms) > ls) return 0.0;
    return __ldg(&a.cgt[i * Kt + ls * ls + ls + ms]);
  };
  const double x1 = tab(0, l - 1, M - 1), x2 = tab(1, l + 1, M - 1);
  const double x3 = tab(2, l - 1, M + 1), x4 = tab(3, l + 1, M + 1);
  const double x5 = tab(4, l - 1, M), x6 = tab(5, l + 1, M);
  const double u1 = tab(6, l, M - 1), u2 = tab(7, l, M), u3 = tab(8, l, M + 1);
  // staging: the ROWS x NV entries of one degree are contiguous in the tri layout, so thread
  // t < ST (row r0 = t / NV, column v = t % NV) reads entry t + ST u of each degree's segment
  // in pass u (row r0 + RPP u, same column): no per-entry index arithmetic (the divisions of
  // a flat entry index were two thirds of the kernel's instructions, which was issue bound)
  constexpr int RPP = CGF_THREADS / NV, ST = RPP * NV, PASSES = (ROWS + RPP - 1) / RPP;
  const int r0 = threadIdx.x / NV, v = threadIdx.x - r0 * NV;
  const bool stager = threadIdx.x < ST;
  const double2* const F2 = reinterpret_cast<const double2*>(Fg);
  if constexpr (!SPLIT) {
    // 16-byte cp.async straight into the padded rows (zero fill outside the table): nothing
    // passes through registers, every copy of the thread is in flight at once
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int lp = l - 1 + i;
      const bool rowok = lp >= 0 && lp <= Lt;
      const int base = (lp * (lp + 1) / 2 + m0 - 1) * NV + (int)threadIdx.x;
#pragma unroll
      for (int u = 0; u < PASSES; ++u) {
        const int rr = r0 + RPP * u, mp = m0 - 1 + rr;
        const bool ok = rowok && mp >= 0 && mp <= lp;
        // (an unsigned 32-bit index select, not a pointer select: no 64-bit select / sign extension)
        if (stager && rr < ROWS) cgs_cp16(&cgf_smem[(i * ROWS + rr) * RS + v], F2 + (ok ? (unsigned)(base + ST * u) : 0u), ok);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // split forward launches: the partial F buffers 1.. are added in split order on the way
    double2 x[3 * PASSES];
    unsigned okmask = 0;  // bit i * PASSES + u: entry inside the table
#pragma unroll
    for (int i = 0; i < 3; ++i) {  // all loads of the thread in flight before the stores
      const int lp = l - 1 + i;
      const bool rowok = stager && lp >= 0 && lp <= Lt;
      const int base = (lp * (lp + 1) / 2 + m0 - 1) * NV + (int)threadIdx.x;
#pragma unroll
      for (int u = 0; u < PASSES; ++u) {
        const int mp = m0 - 1 + r0 + RPP * u;
        const bool ok = rowok && r0 + RPP * u < ROWS && mp >= 0 && mp <= lp;
        x[i * PASSES + u] = make_double2(0.0, 0.0);
        if (ok) {
          x[i * PASSES + u] = __ldg(F2 + base + ST * u);
          okmask |= 1u << (i * PASSES + u);
        }
      }
    }
    for (int sp = 1; sp < a.nsplit; ++sp) {
      const double2* Fp = reinterpret_cast<const double2*>(a.Fx + (sp - 1) * a.fx_stride);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int lp = l - 1 + i;
        const int base = (lp * (lp + 1) / 2 + m0 - 1) * NV + (int)threadIdx.x;
#pragma unroll
        for (int u = 0; u < PASSES; ++u) {
          if (okmask >> (i * PASSES + u) & 1u) {
            const double2 y = __ldg(Fp + base + ST * u);
            x[i * PASSES + u].x += y.x;
            x[i * PASSES + u].y += y.y;
          }
        }
      }
    }
    if (stager) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int u = 0; u < PASSES; ++u)
          if (r0 + RPP * u < ROWS) cgf_smem[(i * ROWS + r0 + RPP * u) * RS + v] = x[i * PASSES + u];
    }
  }
  __syncthreads();
  if (!work) return;
  // staged F^{x,y,z}_{l+dl, mm}: row |mm| - (m0 - 1); out-of-range rows were staged as 0;
  // combo comp of favest/transforms.py:112 formed on read
  auto f = [&](int comp, int dl, int mm) -> double2 {
    const double2* r = cgf_smem + ((dl + 1) * ROWS + abs(mm) - (m0 - 1)) * RS + 6 * b + (mm < 0 ? 1 : 0);
    return combo_uvw(comp, r[0], r[2], r[4]);
  };
  const double2 fu_a = f(0, -1, M - 1), fu_b = f(0, 1, M - 1);
  const double2 fv_a = f(1, -1, M + 1), fv_b = f(1, 1, M + 1);
  const double2 fw_a = f(2, -1, M), fw_b = f(2, 1, M);
  const double2 fu_c = f(0, 0, M - 1), fv_c = f(1, 0, M + 1);
  const double2 fw_c = f(2, 0, M);
  const double xs[9] = {x1, x2, x3, x4, x5, x6, u1, u2, u3};
  double2 ca, cb;
  cg_fwd_combine(xs, fu_a, fu_b, fu_c, fv_a, fv_b, fv_c, fw_a, fw_b, fw_c, ca, cb);
  double ar = ca.x, ai = ca.y, br = cb.x, bi = cb.y;
  if (l == 0) ar = ai = br = bi = 0.0;  // favest/transforms.py:145-146
  const size_t o = (size_t)(b0g + b) * K + (l * l + l + M);
  a.A[o] = make_double2(ar, ai);
  a.Bc[o] = make_double2(br, bi);
}

// ---------------------------------------------------------------------------
// adjoint Clebsch-Gordan: favest/coupling.py:227-239 and transforms.py:168-175.
// Thread per (table degree l <= L+1, order |m|) and row slot; writes sigma_m * g
// into the fragment-ordered G tiles of order |m| (padding rows / columns -> 0).
// ---------------------------------------------------------------------------
struct CgAdjArgs {
  const double2* A;     // (B_total, K) div
  const double2* Bc;    // (B_total, K) curl
  const double2* dg;    // grid mode: (d, gamma) of the block-rescaled recurrence, G is scaled by gamma_l
  const long long* dgofs;
  const double* cgt;    // cg_table_kernel: 9 x K_t (xi1..6, mu1..3)
  double* G;
  const long long* gofs;    // fragment mode: tile offset (units of 512*NT doubles) per order
  const long long* rowofs;  // row mode: row offset per order (rows of 12*nfields doubles)
  int L, NT, B_total, b0, nfields, m_begin;
  int rows_mode;            // 0: DMMA fragment tiles (grid path), 1: plain rows (points path)
  const double* cga;        // cg_adj_tile_kernel: factors in G-row order ((i * 2 + sign) * nrow + row)
  long long nrow;
  // cg_adj_multi_kernel, several 4-field groups in one launch (grid.z = group): G of group g at
  // + g * gg_stride, fields b0 + 4 g ..
  long long gg_stride;
};

// cgt -> G-row order: row (gofs[|m|] + chunk) * 32 + idx holds degree
// l = |m| + 32 chunk + idx; entry (i, sign) = factor i at (l, +-|m|), zero for
// l > L+1 and for the duplicate m = 0 sign.
__global__ void cga_table_kernel(int Lt, const long long* __restrict__ gofs, const double* __restrict__ cgt,
                                 double* cga, long long nrow) {
  const int am = blockIdx.y, c = blockIdx.x, idx = threadIdx.x;
  if (c * 32 >= Lt + 1 - am) return;
  const long long l = am + 32LL * c + idx;
  const long long row = (gofs[am] + c) * 32 + idx;
  const long long Kt = (long long)(Lt + 1) * (Lt + 1);
  for (int sg = 0; sg < 2; ++sg) {
    const bool on = l <= Lt && !(sg == 1 && am == 0);
    const long long k = l * l + l + (sg ? -am : am);
    for (int i = 0; i < 9; ++i) cga[(i * 2 + sg) * nrow + row] = on ? cgt[i * Kt + k] : 0.0;
  }
}

__device__ __forceinline__ double2 c_read(const double2* t, const CgAdjArgs& a, int b, long long l, long long m) {
  if (l < 0 || l > a.L || llabs(m) > l) return make_double2(0.0, 0.0);
  return t[(size_t)(a.b0 + b) * (a.L + 1) * (a.L + 1) + l * l + l + m];
}

__global__ void cg_adj_kernel(CgAdjArgs a) {
  const int mi = blockIdx.y;
  const long long am = a.m_begin + mi;
  const int Lt = a.L + 1;
  const int nrows = Lt + 1 - (int)am;
  constexpr int LC = 32, KS = LC / 8;  // legendre.cuh ADJ_LC / ADJ_KS
  const int nlc = (nrows + LC - 1) / LC;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. LC*nlc-1
  if (row >= (a.rows_mode ? nrows : LC * nlc)) return;
  const long long l = am + row;
  const int lc = row / LC, idx = row % LC;
  const int par = idx & 1, k = idx >> 1, ks = k >> 2, q = k & 3;
  double* Gt = a.rows_mode ? a.G + (size_t)(a.rowofs[am] + row) * (12 * a.nfields)
                           : a.G + (size_t)(a.gofs[am] + lc) * (2 * KS * a.NT * 32);
  auto put = [&](int n, double v) {
    if (a.rows_mode)
      Gt[n] = v;
    else
      Gt[((size_t)(par * KS + ks) * a.NT + (n >> 3)) * 32 + ((n & 7) << 2) + q] = v;
  };
  if (!a.rows_mode)
    for (int n = 12 * a.nfields; n < 8 * a.NT; ++n) put(n, 0.0);
  const bool live = l <= Lt;
  const double is2 = 0.7071067811865475;
  for (int sg = 0; sg < 2; ++sg) {
    const long long m = sg ? -am : am;
    const bool on = live && !(sg == 1 && am == 0);
    double x1 = 0, x2 = 0, x3 = 0, x4 = 0, x5 = 0, x6 = 0, u1 = 0, u2 = 0, u3 = 0;
    if (on) {
      const long long Kt = (long long)(Lt + 1) * (Lt + 1), k = l * l + l + m;
      x1 = __ldg(&a.cgt[0 * Kt + k]); x2 = __ldg(&a.cgt[1 * Kt + k]); x3 = __ldg(&a.cgt[2 * Kt + k]);
      x4 = __ldg(&a.cgt[3 * Kt + k]); x5 = __ldg(&a.cgt[4 * Kt + k]); x6 = __ldg(&a.cgt[5 * Kt + k]);
      u1 = __ldg(&a.cgt[6 * Kt + k]); u2 = __ldg(&a.cgt[7 * Kt + k]); u3 = __ldg(&a.cgt[8 * Kt + k]);
    }
    double sig = (m < 0 && (am & 1)) ? -1.0 : 1.0;  // favest/legendre.py:101-103
    if (!a.rows_mode && live) sig *= a.dg[a.dgofs[am] + (l - am)].y;  // gamma_l (legendre.cuh)
    for (int b = 0; b < a.nfields; ++b) {
      double2 gx = make_double2(0, 0), gy = make_double2(0, 0), gz = make_double2(0, 0);
      if (on) {
        const double2 ap1p = c_read(a.A, a, b, l + 1, m + 1), ap1m = c_read(a.A, a, b, l + 1, m - 1);
        const double2 am1p = c_read(a.A, a, b, l - 1, m + 1), am1m = c_read(a.A, a, b, l - 1, m - 1);
        const double2 ap10 = c_read(a.A, a, b, l + 1, m), am10 = c_read(a.A, a, b, l - 1, m);
        const double2 bp = c_read(a.Bc, a, b, l, m + 1), bm = c_read(a.Bc, a, b, l, m - 1);
        const double2 b0 = c_read(a.Bc, a, b, l, m);
        // nu1..nu6, eta1..eta3 (favest/coupling.py:227-239)
        const double2 nu1 = make_double2(ap1p.x * x1 - ap1m.x * x3, ap1p.y * x1 - ap1m.y * x3);
        const double2 nu2 = make_double2(am1p.x * x2 - am1m.x * x4, am1p.y * x2 - am1m.y * x4);
        const double2 s3 = make_double2(ap1p.x * x1 + ap1m.x * x3, ap1p.y * x1 + ap1m.y * x3);
        const double2 nu3 = make_double2(-s3.y, s3.x);
        const double2 s4 = make_double2(am1p.x * x2 + am1m.x * x4, am1p.y * x2 + am1m.y * x4);
        const double2 nu4 = make_double2(-s4.y, s4.x);
        const double2 nu5 = make_double2(ap10.x * x5, ap10.y * x5);
        const double2 nu6 = make_double2(am10.x * x6, am10.y * x6);
        const double2 d1 = make_double2(bp.x * u1 - bm.x * u3, bp.y * u1 - bm.y * u3);
        const double2 eta1 = make_double2(-d1.y, d1.x);
        const double2 eta2 = make_double2(bp.x * u1 + bm.x * u3, bp.y * u1 + bm.y * u3);
        const double2 eta3 = make_double2(-(b0.y * u2), b0.x * u2);
        // merge (favest/transforms.py:168-175)
        gx = make_double2(-is2 * ((nu1.x + nu2.x) + eta1.x), -is2 * ((nu1.y + nu2.y) + eta1.y));
        gy = make_double2(-is2 * ((nu3.x + nu4.x) - eta2.x), -is2 * ((nu3.y + nu4.y) - eta2.y));
        gz = make_double2((nu5.x + nu6.x) + eta3.x, (nu5.y + nu6.y) + eta3.y);
      }
      const int n0 = 12 * b + 2 * sg;
      put(n0 + 0, sig * gx.x); put(n0 + 1, sig * gx.y);
      put(n0 + 4, sig * gy.x); put(n0 + 5, sig * gy.y);
      put(n0 + 8, sig * gz.x); put(n0 + 9, sig * gz.y);
    }
  }
}

// Grid-path adjoint CG, tiled: CTA per (order |m|, 32-row chunk) of the DMMA
// G tiles.  The A / B entries the chunk needs (rows l0-1 .. l0+32, orders
// +-|m|-1 .. +-|m|+1, all NF fields of the group) are staged in shared memory,
// the chunk is assembled in shared memory in fragment order (padded blocks,
// conflict-free stores) and written out as one contiguous block.  The nine
// factors come from cga (G-row order, coalesced).  Same arithmetic as
// cg_adj_kernel (bitwise equal results).
constexpr int CGA_THREADS = 256;
__host__ __device__ constexpr int cga_bstride(int nf) { return cgf_nt(nf) * 32 + 4; }
template <int NF>
__global__ void __launch_bounds__(CGA_THREADS) cg_adj_tile_kernel(CgAdjArgs a) {
  constexpr int LC = 32, KS = LC / 8, NT = cgf_nt(NF), BS = cga_bstride(NF);
  constexpr int TILE = 2 * KS * NT * 32;  // doubles
  static_assert(LC * NF * 2 <= CGA_THREADS, "one (row, field, sign) per thread");
  const int am = a.m_begin + blockIdx.y;
  const int Lt = a.L + 1;
  const int c = blockIdx.x;
  if (c * LC >= Lt + 1 - am) return;
  const int l0 = am + c * LC;
  extern __shared__ __align__(16) double cga_smem[];
  double* Gs = cga_smem;                                           // 2 KS padded blocks
  double2* As = reinterpret_cast<double2*>(Gs + 2 * KS * BS);      // [NF][34][7] (odd stride)
  double2* Bs = As + NF * 34 * 7;
  // this thread's output (row idx, field b, sign sg); its nine factors and
  // gamma are loaded together with the staging loads (one memory round trip)
  const int w = threadIdx.x;
  const int idx = w % LC, b = (w / LC) % NF, sg = w / (LC * NF);
  const int l = l0 + idx;
  const bool work = w < LC * NF * 2 && l <= Lt && !(sg == 1 && am == 0);
  double cfv[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double gam = 0.0;
  if (work) {
    const double* cf = a.cga + (a.gofs[am] + c) * 32 + sg * a.nrow + idx;  // coalesced over idx
#pragma unroll
    for (int i = 0; i < 9; ++i) cfv[i] = __ldg(cf + 2 * i * a.nrow);
    gam = a.dg[a.dgofs[am] + (l - am)].y;
  }
  constexpr int NE = NF * 34 * 6, PER = (NE + CGA_THREADS - 1) / CGA_THREADS;
  const int K = (a.L + 1) * (a.L + 1);
  double2 va[PER], vb[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * CGA_THREADS;
    va[u] = vb[u] = make_double2(0.0, 0.0);
    if (e < NE) {
      const int bb = e / (34 * 6), r = (e / 6) % 34, j = e % 6;
      const int lp = l0 - 1 + r;
      const int mp = (j < 3 ? am : -am) + (j % 3) - 1;
      if (lp >= 0 && lp <= a.L && abs(mp) <= lp) {
        const size_t o = (size_t)(a.b0 + bb) * K + (lp * lp + lp + mp);
        va[u] = __ldg(&a.A[o]);
        vb[u] = __ldg(&a.Bc[o]);
      }
    }
  }
  for (int i = threadIdx.x; i < 2 * KS * BS; i += CGA_THREADS) Gs[i] = 0.0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * CGA_THREADS;
    if (e < NE) {
      As[e / 6 * 7 + e % 6] = va[u];
      Bs[e / 6 * 7 + e % 6] = vb[u];
    }
  }
  __syncthreads();
  if (work) {
    const int m = sg ? -am : am;
    double sig = (m < 0 && (am & 1)) ? -1.0 : 1.0;  // favest/legendre.py:101-103
    sig *= gam;                                      // gamma_l (legendre.cuh)
    // staged entries: row r = l - l0 + 1 (+-1), j = 3 sg + (M' - m + 1)
    auto at = [&](const double2* t, int dr, int dm) { return t[(b * 34 + idx + 1 + dr) * 7 + 3 * sg + dm + 1]; };
    CgAdjIn v;
    v.ap1p = at(As, 1, 1); v.ap1m = at(As, 1, -1); v.am1p = at(As, -1, 1); v.am1m = at(As, -1, -1);
    v.ap10 = at(As, 1, 0); v.am10 = at(As, -1, 0);
    v.bp = at(Bs, 0, 1); v.bm = at(Bs, 0, -1); v.b0 = at(Bs, 0, 0);
    double2 gx, gy, gz;
    cg_adj_merge(cfv, v, gx, gy, gz);
    const int par = idx & 1, kk = idx >> 1, ks = kk >> 2, q = kk & 3;
    double* gb = Gs + (par * KS + ks) * BS + q;
    auto put = [&](int n, double v) { gb[(n >> 3) * 32 + ((n & 7) << 2)] = v; };
    const int n0 = 12 * b + 2 * sg;
    put(n0 + 0, sig * gx.x); put(n0 + 1, sig * gx.y);
    put(n0 + 4, sig * gy.x); put(n0 + 5, sig * gy.y);
    put(n0 + 8, sig * gz.x); put(n0 + 9, sig * gz.y);
  }
  __syncthreads();
  double2* dst = reinterpret_cast<double2*>(a.G + (size_t)(a.gofs[am] + c) * TILE);
  constexpr int BH = NT * 16;  // double2 per block
  for (int i = threadIdx.x; i < TILE / 2; i += CGA_THREADS) {
    const int blk = i / BH, o = i - blk * BH;
    dst[i] = reinterpret_cast<const double2*>(Gs + blk * BS)[o];
  }
}

// Grid-path adjoint CG over runs of NO consecutive orders: CTA per (run of orders
// am0 .. am0 + NO - 1, 32-row chunk c).  cg_adj_tile_kernel stages, per (order, chunk),
// the orders m-1 .. m+1 of both signs: every a / b entry is read by three CTAs, in
// 48-byte pieces that straddle sectors, ~780 MB of L2 -> SM traffic at C3 for 437 MB of
// HBM traffic.  Here the a / b window of the whole run (degrees l0-1 .. l0+NO+32, orders
// am0-1 .. am0+NO of both signs: (NO+2) x 16-byte contiguous pieces) is staged once,
// together with the run's factor and gamma rows, all by 16-byte cp.async (nothing passes
// through registers), and the NO tiles are assembled one after the other in two
// alternating padded buffers (the copy-out of tile o overlaps the assembly of tile o+1;
// one CTA barrier per tile).  Same arithmetic as cg_adj_kernel (cg_adj_merge: bitwise equal).
template <int NF, int NO>
struct CgaMulti {
  static constexpr int LC = 32, KS = LC / 8, NT = cgf_nt(NF), BS = cga_bstride(NF);
  static constexpr int R = NO + LC + 1;     // staged degrees
  static constexpr int NC = NO + 2;         // staged orders per sign block
  static constexpr int CS = 2 * NC + 1;     // odd row stride (double2): conflict-free LDS.128 over rows
  static constexpr int GBUF = 2 * KS * BS;  // doubles per padded tile buffer
  static constexpr size_t bytes =
      (size_t)2 * GBUF * 8 + (size_t)2 * NF * R * CS * 16 + (size_t)NO * 18 * 32 * 8 + (size_t)NO * 32 * 16;
};
template <int NF, int NO>
__global__ void __launch_bounds__(CGA_THREADS) cg_adj_multi_kernel(CgAdjArgs a, int m_count) {
  using C = CgaMulti<NF, NO>;
  constexpr int LC = C::LC, KS = C::KS, NT = C::NT, BS = C::BS, R = C::R, NC = C::NC, CS = C::CS;
  constexpr int TILE = 2 * KS * NT * 32;  // doubles
  static_assert(LC * NF * 2 <= CGA_THREADS, "one (row, field, sign) per thread");
  const int Lt = a.L + 1;
  const int o0 = blockIdx.y * NO;
  const int am0 = a.m_begin + o0;
  const int c = blockIdx.x;
  if (c * LC >= Lt + 1 - am0) return;
  // field group of this CTA (grid.z = 1: group 0); locals, not writes to the parameter struct
  double* const Gg = a.G + blockIdx.z * a.gg_stride;
  const int b0g = a.b0 + 4 * blockIdx.z;
  const int no = min(NO, m_count - o0);
  extern __shared__ __align__(16) double cgm_smem[];
  double* Gs = cgm_smem;                                          // [2][GBUF]
  double2* As = reinterpret_cast<double2*>(Gs + 2 * C::GBUF);     // [NF][R][CS]
  double2* Bs = As + NF * R * CS;
  double* Fs = reinterpret_cast<double*>(Bs + NF * R * CS);       // factors [NO][9 x 2 signs][32 rows]
  double2* Ds = reinterpret_cast<double2*>(Fs + NO * 18 * 32);    // (d, gamma) [NO][32 rows]
  const int K = (a.L + 1) * (a.L + 1);
  const int lp0 = am0 + c * LC - 1;
  if constexpr (CGA_THREADS % (2 * NC) == 0 && CGA_THREADS / (2 * NC) <= R) {
    // thread t: column j = t % 2NC (fixed order mp), staged rows t / 2NC + RP u of the NF x R
    // (field, degree) rows; (field, degree) advance incrementally (no per-entry divisions)
    constexpr int RP = CGA_THREADS / (2 * NC), NROW = NF * R;
    const int j = threadIdx.x % (2 * NC);
    const int mp = j < NC ? am0 - 1 + j : -(am0 + NO) + (j - NC);
    const int amp = abs(mp);
    int row = threadIdx.x / (2 * NC), r = row, bb = 0;  // RP <= R: the first row is in field 0
    for (; row < NROW; row += RP) {
      const int lp = lp0 + r;
      const bool ok = lp >= 0 && lp <= a.L && amp <= lp;
      const size_t o = ok ? (size_t)(b0g + bb) * K + (lp * lp + lp + mp) : 0;
      cgs_cp16(&As[row * CS + j], a.A + o, ok);
      cgs_cp16(&Bs[row * CS + j], a.Bc + o, ok);
      r += RP;
      if (r >= R) { r -= R; ++bb; }
    }
  } else {
    constexpr int NE = NF * R * 2 * NC;
    for (int e = threadIdx.x; e < NE; e += CGA_THREADS) {
      const int j = e % (2 * NC), r = (e / (2 * NC)) % R, bb = e / (2 * NC * R);
      const int lp = lp0 + r;
      const int mp = j < NC ? am0 - 1 + j : -(am0 + NO) + (j - NC);
      const bool ok = lp >= 0 && lp <= a.L && abs(mp) <= lp;
      const size_t o = ok ? (size_t)(b0g + bb) * K + (lp * lp + lp + mp) : 0;
      cgs_cp16(&As[(bb * R + r) * CS + j], a.A + o, ok);
      cgs_cp16(&Bs[(bb * R + r) * CS + j], a.Bc + o, ok);
    }
  }
  for (int e = threadIdx.x; e < NO * 18 * 16; e += CGA_THREADS) {
    const int h = e % 16, k = (e / 16) % 18, o = e / (16 * 18);
    const int am = am0 + o;
    const bool ok = o < no && c * LC < Lt + 1 - am;
    cgs_cp16(&Fs[(o * 18 + k) * 32 + 2 * h], a.cga + (ok ? (a.gofs[am] + c) * 32 + (long long)k * a.nrow + 2 * h : 0), ok);
  }
  for (int e = threadIdx.x; e < NO * 32; e += CGA_THREADS) {
    const int idx = e % 32, o = e / 32;
    const int am = am0 + o;
    const bool ok = o < no && am + c * LC + idx <= Lt;
    cgs_cp16(&Ds[e], a.dg + (ok ? a.dgofs[am] + c * LC + idx : 0), ok);
  }
  // padding columns 12 NF .. 8 NT - 1 are never written below: zero the buffers once (with
  // 12 NF a multiple of 8 the (row, field, sign) threads write every copied-out entry of a
  // tile for every order, zeros included)
  if constexpr ((12 * NF) % 8 != 0)
    for (int i = threadIdx.x; i < 2 * C::GBUF; i += CGA_THREADS) Gs[i] = 0.0;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int w = threadIdx.x;
  const int idx = w % LC, b = (w / LC) % NF, sg = w / (LC * NF);
  const int par = idx & 1, kk = idx >> 1, ks = kk >> 2, q = kk & 3;
  const int n0 = 12 * b + 2 * sg;
  for (int o = 0; o < no; ++o) {
    const int am = am0 + o;
    if (c * LC >= Lt + 1 - am) break;  // the higher orders of the run have no chunk c either
    double* G = Gs + (o & 1) * C::GBUF;
    if (w < LC * NF * 2) {
      const int l = am + c * LC + idx;
      const bool work = l <= Lt && !(sg == 1 && am == 0);
      double2 gx = make_double2(0.0, 0.0), gy = gx, gz = gx;
      double sig = 0.0;
      if (work) {
        double cfv[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) cfv[i] = Fs[(o * 18 + 2 * i + sg) * 32 + idx];
        sig = (sg && (am & 1)) ? -1.0 : 1.0;  // favest/legendre.py:101-103
        sig *= Ds[o * 32 + idx].y;             // gamma_l (legendre.cuh)
        // staged row of degree l + dr: o + idx + 1 + dr; column of order +-am + dm
        const int col = sg ? NC + NO - o : o + 1;
        auto at = [&](const double2* t, int dr, int dm) { return t[(b * R + o + idx + 1 + dr) * CS + col + dm]; };
        CgAdjIn v;
        v.ap1p = at(As, 1, 1); v.ap1m = at(As, 1, -1); v.am1p = at(As, -1, 1); v.am1m = at(As, -1, -1);
        v.ap10 = at(As, 1, 0); v.am10 = at(As, -1, 0);
        v.bp = at(Bs, 0, 1); v.bm = at(Bs, 0, -1); v.b0 = at(Bs, 0, 0);
        cg_adj_merge(cfv, v, gx, gy, gz);
      }
      double* gb = G + (par * KS + ks) * BS + q;
      auto put = [&](int n, double v) { gb[(n >> 3) * 32 + ((n & 7) << 2)] = work ? v : 0.0; };
      put(n0 + 0, sig * gx.x); put(n0 + 1, sig * gx.y);
      put(n0 + 4, sig * gy.x); put(n0 + 5, sig * gy.y);
      put(n0 + 8, sig * gz.x); put(n0 + 9, sig * gz.y);
    }
    __syncthreads();
    double2* dst = reinterpret_cast<double2*>(Gg + (size_t)(a.gofs[am] + c) * TILE);
    constexpr int BH = NT * 16;  // double2 per block
    for (int i = threadIdx.x; i < TILE / 2; i += CGA_THREADS) {
      const int blk = i / BH, oo = i - blk * BH;
      dst[i] = reinterpret_cast<const double2*>(G + blk * BS)[oo];
    }
  }
}

}  // namespace fv
