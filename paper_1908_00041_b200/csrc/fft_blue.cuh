// Ring DFTs of lengths with a prime factor P > 19 and no Rader plan
// (fft_rader.cuh): C2's n_phi = 516 = 12 * 43 and other small primes (P <= 64)
// by direct conjugate-pair residue DFTs in one CTA per ring (smallp_kernel),
// larger primes by batched cuFFT sub-DFTs of length P plus the R-point combine
// (rp_combine_kernel).  favest/scalar.py:149 (np.fft.fft along a ring) and
// :178 (np.fft.ifft * n_phi, i.e. the unnormalised inverse).
//
// n = R * P.  Decimation in time over the R residues:
//   X[k + P s] = sum_r w_R^{r s} ( w_n^{r k} Y_r[k] ),   Y_r = DFT_P(x[r + R q], q < P)
// The inverse direction is conj(DFT(conj(x))).  Tables are exactly rounded from
// long double on the host.  (A Bluestein chirp-z variant of the residue DFTs was
// measured slower than cuFFT's sub-DFTs at C4 and removed; the Rader kernels
// replaced both there.)
#pragma once
#include "fft2.cuh"

namespace fv {

constexpr int BLUE_T = 256;

// factorisation and tables of the cuFFT sub-DFT path (ring_fft_rp)
struct BlueArgs {
  const double2* rootN;   // exp(-2 pi i j / n), j < n
  const double2* rootR;   // exp(-2 pi i j / R), j < R
  int n, R, P;
};

__device__ __forceinline__ double2 bl_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 bl_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 bl_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i
__device__ __forceinline__ double2 bl_mi(double2 a) { return make_double2(a.y, -a.x); }

// ---------------------------------------------------------------------------
// Small prime factor (P <= 64, e.g. C2's 516 = 12 * 43): one CTA per
// (ring, component) does the whole ring in shared memory with direct
// conjugate-pair DFTs (no Bluestein):
//   Y_r[k] = x_0 + sum_{q=1}^{(P-1)/2} (x_q + x_{P-q}) cos(2 pi q k / P)
//                - i (x_q - x_{P-q}) sin(2 pi q k / P)        (and k -> P - k: + i)
// on the residue subsequences x_q = x[r + R q], then w_n^{r k} and the direct
// R-point DFTs X[k + P s] = sum_r w_R^{r s} Y'_r[k] (output index = thread
// index: coalesced stores).  ~2P + 8R flops per point.
// ---------------------------------------------------------------------------
constexpr int SMALLP_MAX = 64;
// 8 warps (288 threads -- one stage-1 pass fewer and a one-pass fold epilogue at
// C2 -- measured 6 % slower: 72 registers, one CTA per SM fewer)
constexpr int SMALLP_T = 256;

struct SmallPArgs {
  const double2* in;
  long long in_cs, in_rs, in_es;
  double2* out;
  long long out_cs, out_rs, out_es;
  const double2* rootN;  // exp(-2 pi i j / n), j < n
  const double2* WR;     // [r][s] = exp(-2 pi i (r s mod R) / R), R x R
  const double2* WP;     // [q - 1][k] = (cos, sin)(2 pi (q k mod P) / P), q = 1..H, k = 0..H, H = (P - 1) / 2
  int n, R, P, nrings, inverse;
  int in_rblk;           // blocked input rings (common.cuh SLayout rblk), 0: in_rs apart
  int ahead;             // L2 prefetch of the input of item blockIdx.x + ahead (fft2.cuh), 0: off
};

// residue DFTs of nr rings: xs[ring][n] -> ys[ring][R][P] (twiddled by w_n^{r k})
__device__ __forceinline__ void smallp_stage1(const SmallPArgs& a, const double2* xs, double2* ys,
                                              const double2* wp, int nr) {
  const int H = (a.P - 1) / 2;
  const int per = a.R * (H + 1);
  for (int it = threadIdx.x; it < nr * per; it += SMALLP_T) {
    const int ring = it / per, j = it - ring * per;
    const int r = j / (H + 1), k = j - r * (H + 1);
    const double2* x = xs + ring * a.n + r;
    double2* y = ys + ring * a.n + r * a.P;
    double2 A = x[0], Bv = make_double2(0.0, 0.0);
    const double2* w = wp + k;
#pragma unroll 4
    for (int q = 1; q <= H; ++q) {
      const double2 u = x[q * a.R], v = x[(a.P - q) * a.R];
      const double2 t = w[(q - 1) * (H + 1)];
      A.x = fma(u.x + v.x, t.x, A.x);
      A.y = fma(u.y + v.y, t.x, A.y);
      Bv.x = fma(u.x - v.x, t.y, Bv.x);
      Bv.y = fma(u.y - v.y, t.y, Bv.y);
    }
    // X_k = A - i B, X_{P-k} = A + i B; then the twiddle w_n^{r k}
    y[k] = bl_mul(make_double2(A.x + Bv.y, A.y - Bv.x), __ldg(&a.rootN[(long long)r * k]));
    if (k > 0) y[a.P - k] = bl_mul(make_double2(A.x - Bv.y, A.y + Bv.x), __ldg(&a.rootN[(long long)r * (a.P - k)]));
  }
}

// Stage 2, thread per (ring, bin k, group of SG consecutive outputs s): each
// residue value of bin k is read once and feeds the group's SG accumulators
// (the generic per-output loop re-read all R of them per output).  Per output
// the sum still runs over r = 0, 1, ..., R-1 in order: same arithmetic.
constexpr int SP_SGMAX = 8;
__host__ __device__ inline int smallp_sg(int P, int R) {  // outputs per thread of stage 2 (two rings)
  int sg = (2 * P * R + SMALLP_T - 1) / SMALLP_T;
  while (2 * P * ((R + sg - 1) / sg) > SMALLP_T) ++sg;
  return sg;
}
template <class Store>
__device__ __forceinline__ void smallp_stage2(const SmallPArgs& a, const double2* ys, const double2* wr, int nr,
                                              Store st) {
  const int P = a.P, R = a.R;
  const int per = nr * P;
  int SG = (per * R + SMALLP_T - 1) / SMALLP_T;  // outputs per thread: the fewest that give one pass
  while (per * ((R + SG - 1) / SG) > SMALLP_T) ++SG;
  const int ngr = (R + SG - 1) / SG;
  for (int it = threadIdx.x; it < per * ngr; it += SMALLP_T) {
    const int sgi = it / per, rk = it - sgi * per;
    const int ring = rk / P, k = rk - ring * P;
    const double2* yr = ys + ring * a.n + k;
    const int s0 = sgi * SG, ns = min(R, s0 + SG) - s0;
    double2 acc[SP_SGMAX];
    const double2 z0 = yr[0];
#pragma unroll
    for (int u = 0; u < SP_SGMAX; ++u) acc[u] = z0;
    for (int r = 1; r < R; ++r) {
      const double2 z = yr[r * P];
      const double2* w = wr + r * R + s0;
#pragma unroll
      for (int u = 0; u < SP_SGMAX; ++u)
        if (u < ns) acc[u] = bl_add(acc[u], bl_mul(z, w[u]));
    }
#pragma unroll
    for (int u = 0; u < SP_SGMAX; ++u)
      if (u < ns) st(ring, (s0 + u) * P + k, acc[u]);
  }
}

// R-point DFT of output o = s P + k of one ring's residue spectra
__device__ __forceinline__ double2 smallp_out(const SmallPArgs& a, const double2* ys, const double2* wr, int o) {
  const int s = o / a.P, k = o - s * a.P;
  double2 acc = ys[k];
  const double2* w = wr + s;
  for (int r = 1; r < a.R; ++r) acc = bl_add(acc, bl_mul(ys[r * a.P + k], w[r * a.R]));
  return acc;
}

// Plain transform: CTA per (component, ring pair) -- both rings' items keep all
// 256 threads busy through both stages, and in the adjoint's ring-pair spectrum
// layout the two rings' bins are one contiguous stream.
__global__ void __launch_bounds__(SMALLP_T) smallp_kernel(SmallPArgs a) {
  extern __shared__ __align__(16) double2 sp_smem[];
  const int H = (a.P - 1) / 2;
  const int n = a.n;
  double2* xs = sp_smem;                  // [2][n] rings
  double2* ys = sp_smem + 2 * n;          // [2][R][P] twiddled residue DFTs
  double2* wp = ys + 2 * n;               // [H][H + 1] (cos, sin): lane k reads [q][k], conflict free
  double2* wr = wp + H * (H + 1);         // [R][R]
  const int c = blockIdx.x % 3, r0 = 2 * (blockIdx.x / 3);
  const int nr = min(2, a.nrings - r0);
  const double cj = a.inverse ? -1.0 : 1.0;
  auto ring_base = [&](int ring) {
    return a.in_rblk ? (long long)(ring >> (31 - __clz(a.in_rblk))) * a.in_rs + (ring & (a.in_rblk - 1))
                     : (long long)ring * a.in_rs;
  };
  if (a.ahead && a.in_rblk == 2 && threadIdx.x == 0 && blockIdx.x + a.ahead < gridDim.x) {
    const int it2 = blockIdx.x + a.ahead, c2 = it2 % 3, q0 = 2 * (it2 / 3);
    if (a.nrings - q0 >= 2) f2_prefetch_l2(a.in + c2 * a.in_cs + ring_base(q0), (unsigned)(2 * n * sizeof(double2)));
  }
  const double2* src0 = a.in + c * a.in_cs + ring_base(r0);
  const double2* src1 = a.in + c * a.in_cs + ring_base(r0 + nr - 1);
  for (int i = threadIdx.x; i < nr * n; i += SMALLP_T) {
    const int ring = i / n, j = i - ring * n;
    double2 v = (ring ? src1 : src0)[(long long)j * a.in_es];
    v.y *= cj;
    xs[i] = v;
  }
  for (int i = threadIdx.x; i < H * (H + 1); i += SMALLP_T) wp[i] = __ldg(&a.WP[i]);
  for (int i = threadIdx.x; i < a.R * a.R; i += SMALLP_T) wr[i] = __ldg(&a.WR[i]);
  __syncthreads();
  smallp_stage1(a, xs, ys, wp, nr);
  __syncthreads();
  if (smallp_sg(a.P, a.R) <= SP_SGMAX) {
    smallp_stage2(a, ys, wr, nr, [&](int ring, int o, double2 v) {  // consecutive k: coalesced
      a.out[c * a.out_cs + (long long)(r0 + ring) * a.out_rs + (long long)o * a.out_es] = make_double2(v.x, cj * v.y);
    });
    return;
  }
  for (int i = threadIdx.x; i < nr * n; i += SMALLP_T) {
    const int ring = i / n, o = i - ring * n;
    const double2 v = smallp_out(a, ys + ring * n, wr, o);  // output index = thread index: coalesced
    a.out[c * a.out_cs + (long long)(r0 + ring) * a.out_rs + (long long)o * a.out_es] = make_double2(v.x, cj * v.y);
  }
}

// Forward with the equatorial fold fused (C2: n_phi = 516), the small-prime
// counterpart of fft2.cuh fft_fold_kernel: CTA per (ring pair, field,
// component), both rings' spectra kept in shared memory, epilogue writes the
// Legendre B operand X exactly as fft_fold_kernel does.
__global__ void __launch_bounds__(SMALLP_T) smallp_fold_kernel(SmallPArgs a, Fft2Args f) {
  extern __shared__ __align__(16) double2 sp_smem[];
  const int H = (a.P - 1) / 2;
  const int n = a.n;
  double2* xs = sp_smem;                  // [2][n] rings, then their spectra
  double2* ys = sp_smem + 2 * n;          // [2][R][P]
  double2* wp = ys + 2 * n;
  double2* wr = wp + H * (H + 1);
  const int item = blockIdx.x;
  const int c = item % 3, b = (item / 3) % f.nfields, p = item / (3 * f.nfields);
  if (f.ahead && c == 0 && threadIdx.x == 0 && item + f.ahead < (int)gridDim.x) {
    const int it2 = item + f.ahead, b2 = (it2 / 3) % f.nfields, p2 = it2 / (3 * f.nfields);
    const int rn2 = f.pair_n[p2], rs2 = f.pair_s[p2];
    const double2* base2 = f.in + (long long)b2 * f.field_stride;
    const unsigned ring_bytes = (unsigned)(3 * n * sizeof(double2));
    if (rn2 >= 0) f2_prefetch_l2(base2 + (long long)rn2 * f.in_rs, ring_bytes);
    if (rs2 >= 0) f2_prefetch_l2(base2 + (long long)rs2 * f.in_rs, ring_bytes);
  }
  const int rn = f.pair_n[p], rs = f.pair_s[p];
  const int nr = (rn >= 0) + (rs >= 0);
  if (nr > 0) {
    const double2* base = f.in + (long long)b * f.field_stride + c;
    for (int i = threadIdx.x; i < nr * n; i += SMALLP_T) {
      const int ring = i / n, j = i - ring * n;
      xs[i] = base[(long long)(ring ? rs : rn) * f.in_rs + (long long)j * f.in_es];
    }
    for (int i = threadIdx.x; i < H * (H + 1); i += SMALLP_T) wp[i] = __ldg(&a.WP[i]);
    for (int i = threadIdx.x; i < a.R * a.R; i += SMALLP_T) wr[i] = __ldg(&a.WR[i]);
    __syncthreads();
    smallp_stage1(a, xs, ys, wp, nr);
    __syncthreads();
    if (smallp_sg(a.P, a.R) <= SP_SGMAX) {
      smallp_stage2(a, ys, wr, nr, [&](int ring, int o, double2 v) { xs[ring * n + o] = v; });
    } else {
      for (int i = threadIdx.x; i < nr * n; i += SMALLP_T) {
        const int ring = i / n, o = i - ring * n;
        xs[i] = smallp_out(a, ys + ring * n, wr, o);
      }
    }
    __syncthreads();
  }
  // epilogue (fft2.cuh fft_fold_kernel): thread per order m
  const int chunk = p >> 5, ks = (p >> 2) & 7, kq = p & 3;
  const int col = 12 * b + 4 * c;
  const size_t tile = (size_t)2 * 8 * f.NT * 32;
  const size_t par_stride = (size_t)8 * f.NT * 32;
  const size_t off = ((size_t)ks * f.NT + (col >> 3)) * 32 + ((col >> 2) & 1) * 16 + kq * 4;
  const bool padcols = (b == f.nfields - 1) && c == 2 && ((12 * f.nfields) & 7) == 4;
  const int pcol = 12 * f.nfields;
  const size_t poff = ((size_t)ks * f.NT + (pcol >> 3)) * 32 + ((pcol >> 2) & 1) * 16 + kq * 4;
  const double wn = rn >= 0 ? f.ring_w[rn] : 0.0;
  const double ws = rs >= 0 ? f.ring_w[rs] : 0.0;
  const double2* Sn = xs;
  const double2* Ss = xs + n;
  for (int m = threadIdx.x; m <= f.Lt; m += SMALLP_T) {
    double2 Ep = make_double2(0.0, 0.0), Em = Ep, Op = Ep, Om = Ep;
    if (nr > 0) {
      const int bm = m ? n - m : 0;
      const double2 np = Sn[m], nm = Sn[bm];
      const double sg = (m & 1) ? -1.0 : 1.0;  // sigma_{-m} on the -m bin
      if (rs >= 0) {
        const double2 sp = Ss[m], sm = Ss[bm];
        Ep = make_double2(wn * np.x + ws * sp.x, wn * np.y + ws * sp.y);
        Op = make_double2(wn * np.x - ws * sp.x, wn * np.y - ws * sp.y);
        Em = make_double2(sg * (wn * nm.x + ws * sm.x), sg * (wn * nm.y + ws * sm.y));
        Om = make_double2(sg * (wn * nm.x - ws * sm.x), sg * (wn * nm.y - ws * sm.y));
      } else {  // unpaired ring: both parities see the ring itself
        Ep = Op = make_double2(wn * np.x, wn * np.y);
        Em = Om = make_double2(sg * (wn * nm.x), sg * (wn * nm.y));
      }
      if (m == 0) Em = Om = make_double2(0.0, 0.0);
    }
    double* xt = f.X + ((size_t)m * f.nchunks + chunk) * tile;
    st_global_v4(xt + off, Ep, Em);
    st_global_v4(xt + par_stride + off, Op, Om);
    if (padcols) {
      const double2 z = make_double2(0.0, 0.0);
      st_global_v4(xt + poff, z, z);
      st_global_v4(xt + par_stride + poff, z, z);
    }
  }
}

// ---------------------------------------------------------------------------
// Large prime factor (C4: 8196 = 12 * 683): the P-point DFTs of the R residue
// subsequences run as batched cuFFT plans of length P (3 R strided plans of
// nrings transforms: 2.6-3.2 ms for C4's 147k transforms, against 8.2 ms for
// cuFFT's own length-8196 plan), then this kernel applies the twiddles
// w_n^{r k} and the R-point DFTs:  X[k + P s] = sum_r w_R^{r s} w_n^{r k} Y_r[k].
// Y is the scratch [comp][r][ring][k]; thread per (comp, ring, k), loads
// coalesced over k.
// ---------------------------------------------------------------------------
struct RpArgs {
  const double2* Y;      // [3][R][nrings][P]
  double2* out;
  long long out_cs, out_rs, out_es;
  const double2* rootN;  // exp(-2 pi i j / n), j < n
  const double2* rootR;  // exp(-2 pi i j / R), j < R
  int n, P, nrings, inverse;
};

template <int RR>
__global__ void __launch_bounds__(BLUE_T) rp_combine_kernel(RpArgs a) {
  const long long idx = (long long)blockIdx.x * BLUE_T + threadIdx.x;
  const long long per_c = (long long)a.nrings * a.P;
  if (idx >= 3 * per_c) return;
  const int c = (int)(idx / per_c);
  const long long rem = idx - c * per_c;
  const int ring = (int)(rem / a.P), k = (int)(rem - (long long)ring * a.P);
  const double cj = a.inverse ? -1.0 : 1.0;
  const double2* y = a.Y + (size_t)c * RR * per_c + rem;
  double2 z[RR];
  z[0] = y[0];
#pragma unroll
  for (int r = 1; r < RR; ++r) {
    double2 w = __ldg(&a.rootN[(long long)r * k]);
    w.y *= cj;
    z[r] = bl_mul(y[(size_t)r * per_c], w);
  }
  double2* dst = a.out + c * a.out_cs + (long long)ring * a.out_rs;
#pragma unroll 1
  for (int s = 0; s < RR; ++s) {
    double2 acc = z[0];
#pragma unroll
    for (int r = 1; r < RR; ++r) {
      double2 w = __ldg(&a.rootR[(r * s) % RR]);
      w.y *= cj;
      acc = bl_add(acc, bl_mul(z[r], w));
    }
    dst[(long long)(k + (long long)a.P * s) * a.out_es] = acc;
  }
}

}  // namespace fv
