// Ring DFTs of lengths with a prime factor P > 19 (C2: n_phi = 516 = 12 * 43,
// C4: n_phi = 8196 = 12 * 683), replacing the cuFFT Bluestein plans (7.4 ms
// per direction at C4).  favest/scalar.py:149 (np.fft.fft along a ring) and
// :178 (np.fft.ifft * n_phi, i.e. the unnormalised inverse).
//
// n = R * P.  Decimation in time over the R residues:
//   X[k + P s] = sum_r w_R^{r s} ( w_n^{r k} Y_r[k] ),   Y_r = DFT_P(x[r + R q], q < P)
// * blue_p_kernel: one CTA per (component, ring, residue r) computes Y_r by
//   Bluestein's chirp-z identity q k = (q^2 + k^2 - (k - q)^2) / 2:
//   Y_r[k] = c_k * sum_q (x_q c_q) conj(c_{k-q}),  c_j = exp(-pi i j^2 / P),
//   a cyclic convolution of length M >= 2P - 1 (M = 2^a 3^b) done as
//   FFT_M -> x FFT_M(conj c) / M (plan-time table) -> inverse FFT_M, all in
//   shared memory with a Stockham radix-{2,3,4,8} loop; then applies w_n^{r k}
//   and stores Y'_r contiguously in a scratch buffer.
// * blue_r_kernel: thread per (component, ring, k) forms the R outputs
//   X[k + P s] from the R scratch values (direct R-point DFT) and writes them
//   with the caller's strides.
// The inverse direction is conj(DFT(conj(x))): conjugate on load (K1) and on
// store (K2).  Tables (chirps, roots, FFT_M of the chirp) are exactly rounded
// from long double on the host.
#pragma once
#include "fft2.cuh"

namespace fv {

constexpr int BLUE_T = 256;
constexpr int BLUE_MAXST = 12;

struct BlueArgs {
  const double2* in;
  long long in_cs, in_rs, in_es;
  double2* out;
  long long out_cs, out_rs, out_es;
  double2* S1;            // scratch [3 * nrings][R][P]
  const double2* rootM;   // exp(-2 pi i j / M), j < M
  const double2* chirp;   // exp(-pi i q^2 / P), q < P
  const double2* FB;      // FFT_M(b) / M, b_j = conj(chirp_|j|) wrapped cyclically
  const double2* rootN;   // exp(-2 pi i j / n), j < n
  const double2* rootR;   // exp(-2 pi i j / R), j < R
  int n, R, P, M, nrings, inverse;
  int nst;
  int radix[BLUE_MAXST];  // M = prod radix (each 2, 3, 4 or 8)
};

__device__ __forceinline__ double2 bl_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 bl_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 bl_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i
__device__ __forceinline__ double2 bl_mi(double2 a) { return make_double2(a.y, -a.x); }

// forward-sign (exp(-2 pi i / R)) DFT codelets
template <int R>
__device__ __forceinline__ void bl_dft(double2 (&v)[8]);

template <>
__device__ __forceinline__ void bl_dft<2>(double2 (&v)[8]) {
  const double2 a = v[0], b = v[1];
  v[0] = bl_add(a, b);
  v[1] = bl_sub(a, b);
}

template <>
__device__ __forceinline__ void bl_dft<3>(double2 (&v)[8]) {
  const double s3 = 0.86602540378443864676;  // sin(2 pi / 3)
  const double2 t1 = bl_add(v[1], v[2]);
  const double2 t2 = make_double2(v[0].x - 0.5 * t1.x, v[0].y - 0.5 * t1.y);
  const double2 d = bl_sub(v[1], v[2]);
  const double2 t3 = make_double2(s3 * d.y, -s3 * d.x);  // -i sin(2pi/3) (v1 - v2)
  v[0] = bl_add(v[0], t1);
  v[1] = bl_add(t2, t3);
  v[2] = bl_sub(t2, t3);
}

template <>
__device__ __forceinline__ void bl_dft<4>(double2 (&v)[8]) {
  const double2 a = bl_add(v[0], v[2]), b = bl_sub(v[0], v[2]);
  const double2 c = bl_add(v[1], v[3]), d = bl_mi(bl_sub(v[1], v[3]));
  v[0] = bl_add(a, c);
  v[2] = bl_sub(a, c);
  v[1] = bl_add(b, d);
  v[3] = bl_sub(b, d);
}

template <>
__device__ __forceinline__ void bl_dft<8>(double2 (&v)[8]) {
  const double h = 0.70710678118654752440;  // sqrt(2) / 2
  double2 e[8] = {v[0], v[2], v[4], v[6]}, o[8] = {v[1], v[3], v[5], v[7]};
  bl_dft<4>(e);
  bl_dft<4>(o);
  // w8^k o_k, w8 = exp(-i pi / 4)
  const double2 o1 = make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
  const double2 o2 = bl_mi(o[2]);
  const double2 o3 = make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
  v[0] = bl_add(e[0], o[0]);
  v[4] = bl_sub(e[0], o[0]);
  v[1] = bl_add(e[1], o1);
  v[5] = bl_sub(e[1], o1);
  v[2] = bl_add(e[2], o2);
  v[6] = bl_sub(e[2], o2);
  v[3] = bl_add(e[3], o3);
  v[7] = bl_sub(e[3], o3);
}

// One Stockham stage x -> y of the length-M transform with sub-transform span Ns.
template <int R>
__device__ __forceinline__ void bl_stage(const double2* x, double2* y, const double2* __restrict__ rootM, int M,
                                         int Ns) {
  const int nb = M / R;
  const int tstep = M / (Ns * R);
  for (int j = threadIdx.x; j < nb; j += BLUE_T) {
    const int k = j % Ns;
    double2 v[8];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = x[j + i * nb];
    if (Ns > 1) {
#pragma unroll
      for (int i = 1; i < R; ++i) v[i] = bl_mul(v[i], __ldg(&rootM[i * k * tstep]));
    }
    bl_dft<R>(v);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int i = 0; i < R; ++i) y[base + i * Ns] = v[i];
  }
}

// forward FFT_M of buf[0..M) (ping-pong with tmp); returns the buffer holding the result
__device__ __forceinline__ double2* bl_fft(double2* buf, double2* tmp, const BlueArgs& a) {
  int Ns = 1;
  for (int s = 0; s < a.nst; ++s) {
    const int R = a.radix[s];
    switch (R) {
      case 2: bl_stage<2>(buf, tmp, a.rootM, a.M, Ns); break;
      case 3: bl_stage<3>(buf, tmp, a.rootM, a.M, Ns); break;
      case 4: bl_stage<4>(buf, tmp, a.rootM, a.M, Ns); break;
      default: bl_stage<8>(buf, tmp, a.rootM, a.M, Ns); break;
    }
    __syncthreads();
    double2* t = buf;
    buf = tmp;
    tmp = t;
    Ns *= R;
  }
  return buf;
}

__global__ void __launch_bounds__(BLUE_T) blue_p_kernel(BlueArgs a) {
  extern __shared__ __align__(16) double2 bl_smem[];  // 2 x M
  double2* b0 = bl_smem;
  double2* b1 = bl_smem + a.M;
  const int r = blockIdx.x % a.R;
  const long long rc = blockIdx.x / a.R;  // c * nrings + ring
  const int c = (int)(rc / a.nrings), ring = (int)(rc % a.nrings);
  const double2* src = a.in + c * a.in_cs + ring * a.in_rs;
  const double cj = a.inverse ? -1.0 : 1.0;
  for (int q = threadIdx.x; q < a.M; q += BLUE_T) {
    double2 v = make_double2(0.0, 0.0);
    if (q < a.P) {
      double2 x = src[(long long)(r + (long long)a.R * q) * a.in_es];
      x.y *= cj;
      v = bl_mul(x, __ldg(&a.chirp[q]));
    }
    b0[q] = v;
  }
  __syncthreads();
  double2* X = bl_fft(b0, b1, a);
  double2* T = (X == b0) ? b1 : b0;
  // convolution with the chirp in the frequency domain; the inverse FFT_M as
  // conj(FFT(conj(.))) (the 1 / M is folded into FB)
  for (int q = threadIdx.x; q < a.M; q += BLUE_T) {
    const double2 v = bl_mul(X[q], __ldg(&a.FB[q]));
    X[q] = make_double2(v.x, -v.y);
  }
  __syncthreads();
  double2* Y = bl_fft(X, T, a);
  double2* dst = a.S1 + (rc * a.R + r) * (long long)a.P;
  for (int k = threadIdx.x; k < a.P; k += BLUE_T) {
    const double2 y = make_double2(Y[k].x, -Y[k].y);
    const double2 v = bl_mul(bl_mul(y, __ldg(&a.chirp[k])), __ldg(&a.rootN[(long long)r * k]));
    dst[k] = v;
  }
}

template <int RR>
__global__ void __launch_bounds__(BLUE_T) blue_r_kernel(BlueArgs a) {
  const long long idx = (long long)blockIdx.x * BLUE_T + threadIdx.x;
  const long long total = 3LL * a.nrings * a.P;
  if (idx >= total) return;
  const long long rc = idx / a.P;
  const int k = (int)(idx - rc * a.P);
  const int c = (int)(rc / a.nrings), ring = (int)(rc % a.nrings);
  const double2* src = a.S1 + rc * RR * (long long)a.P + k;
  double2 z[RR];
#pragma unroll
  for (int r = 0; r < RR; ++r) z[r] = src[(long long)r * a.P];
  double2* dst = a.out + c * a.out_cs + ring * a.out_rs;
  const double cj = a.inverse ? -1.0 : 1.0;
#pragma unroll 1
  for (int s = 0; s < RR; ++s) {
    double2 acc = z[0];
#pragma unroll
    for (int r = 1; r < RR; ++r) acc = bl_add(acc, bl_mul(z[r], __ldg(&a.rootR[(r * s) % RR])));
    dst[(long long)(k + (long long)a.P * s) * a.out_es] = make_double2(acc.x, cj * acc.y);
  }
}

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
