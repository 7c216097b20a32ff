// Ring DFTs of length n = R * P with a large prime P (C4: n_phi = 8196 =
// 12 * 683) by Rader's algorithm, one ring of one component per CTA, the
// whole ring resident in shared memory.
//
// Reference semantics: favest/scalar.py:149 (np.fft.fft along longitude) and
// :178 (np.fft.ifft * n_phi); the inverse is conj(DFT(conj(x))).  The
// forward variant fuses the equatorial fold of favest/scalar.py:150-152 (the
// Legendre B operand X, exactly as fft2.cuh fft_fold_kernel writes it) through
// a two-CTA cluster: the north and south rings of a mirror pair are
// transformed by the two CTAs and each writes half of the orders, reading the
// partner's spectrum through distributed shared memory.
//
// Algorithm (Cooley-Tukey over n = R * P, residues x_r[q] = x[r + R q]):
//   Y_r[k] = DFT_P(x_r)[k] * w_n^{r k},   X[k + P s] = sum_r w_R^{r s} Y_r[k].
// DFT_P by Rader: with g a primitive root mod P,
//   X_r[g^j] = x_r[0] + (a (*) b)[j],  a[i] = x_r[g^-i],  b[m] = w_P^{g^m},
// a cyclic convolution of length P - 1 = F1 * F2 (683: 682 = 31 * 22) done as
// DFT_{P-1}(a) . DFT_{P-1}(b) / (P - 1) -> inverse DFT_{P-1}, with x_r[0]
// added to the product's zero bin (it then reaches every output).
//
// In place, no scratch: residue r's slots q = 1..P-1 (addresses r + R q of the
// ring buffer) hold the P - 1 convolution values; logical position p lives in
// slot sig[p] = g^-p mod P, which is exactly where a[p] = x_r[g^-p] already
// sits, so the gather is free.  The forward DFT_{P-1} is two in-place passes
// (radix F1 over stride F2 with the w_{P-1}^{n2 k1} twiddle, then radix F2 over
// contiguous positions) and leaves frequency k1 + F1 k2 at position F2 k1 + k2;
// the second pass also multiplies by the transformed kernel and runs the first
// inverse pass in registers (radix F2, twiddle w_{P-1}^-(k1 j2)); the last pass
// (inverse radix F1 over stride F2) leaves c[j] + x_r[0] = X_r[g^j] at logical
// position j, i.e. slot g^-j: slot q holds X_r[q^-1].  The R-point combine
// reads Y_r[k] from slot inv[k] (the twelve residues of one k are one 192-byte
// run) and writes X[k + P s].  Each pass reads and writes only its own
// butterfly's slots, so the passes need one barrier each and no register
// staging across a barrier.
//
// Cost per ring: 2 * R * F2 radix-F1 and R * F1 radix-F2 (x2) butterflies +
// P radix-R: ~1.8 MFLOP at n = 8196; shared memory 16 n bytes (131 KB), one
// CTA per SM; inputs of the next wave are prefetched into L2.
#pragma once
#include <cooperative_groups.h>

#include "fft2.cuh"

namespace fv {

constexpr int RD_T = 384;

struct RaderArgs {
  const double2* in;
  long long in_cs, in_rs, in_es;
  int in_rblk;                // blocked input rings (common.cuh SLayout rblk), 0 = in_rs apart
  double2* out;
  long long out_cs, out_rs, out_es;
  const short* sig;           // [P-1] slot of logical position p: g^-p mod P, then [P] inverses (inv[0] = 0)
  const double2* tab;         // RaderTab: [P-1] exp(-2 pi i e / (P-1)), [P-1] DFT_{P-1}(b) / (P-1) with
                              // b[m] = exp(-2 pi i g^m / P), [128] exp(-2 pi i j / n), [ceil(n / 128)]
                              // exp(-2 pi i 128 j / n); copied to shared memory by every CTA
  int nrings, inverse;
  int ahead;                  // L2 prefetch distance in CTAs (0: off)
};

// R-point DFT of a prime R by conjugate pairs with each output pair stored as
// soon as it is formed (live set: the R - 1 sums / differences).
template <int R, class Store>
__device__ __forceinline__ void dft_prime_put(const double2 (&v)[R], Store put) {
  constexpr int H = (R - 1) / 2;
  constexpr int O = root_offset(R);
  double2 s[H + 1], d[H + 1];
  const double2 x0 = v[0];
  double2 X0 = x0;
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    s[j] = cadd(v[j], v[R - j]);
    d[j] = csub(v[j], v[R - j]);
    X0 = cadd(X0, s[j]);
  }
  put(0, X0);
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double ar = x0.x, ai = x0.y, br = 0.0, bi = 0.0;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int m = (j * k) % R;
      const double c = kRootCos[O + m], sn = kRootSin[O + m];
      ar = fma(c, s[j].x, ar);
      ai = fma(c, s[j].y, ai);
      br = fma(sn, d[j].x, br);
      bi = fma(sn, d[j].y, bi);
    }
    put(k, make_double2(ar + bi, ai - br));
    put(R - k, make_double2(ar - bi, ai + br));
  }
}

// the inverse (sign +) prime DFT: conj(DFT(conj v))
template <int R, class Store>
__device__ __forceinline__ void idft_prime_put(double2 (&v)[R], Store put) {
#pragma unroll
  for (int j = 0; j < R; ++j) v[j].y = -v[j].y;
  dft_prime_put<R>(v, [&](int k, double2 x) { put(k, make_double2(x.x, -x.y)); });
}

// shared-memory layout of one CTA: the ring, the tables, the index arrays
template <int R, int P, int NRG = 1>
struct RaderSmem {
  static constexpr int N = R * P, M = P - 1;
  static constexpr int NHI = (N + 127) / 128;
  static constexpr int TAB = 2 * M + 128 + NHI;  // double2 entries of RaderArgs::tab
  static constexpr size_t bytes = (size_t)(NRG * N + TAB) * 16 + (size_t)(M + P) * 2;
  double2* buf;  // NRG rings of N
  const double2 *tw, *Bn, *lo, *hi;
  const short *sig, *inv;
  __device__ explicit RaderSmem(double2* base) {
    buf = base;
    tw = base + NRG * N;
    Bn = tw + M;
    lo = Bn + M;
    hi = lo + 128;
    sig = reinterpret_cast<const short*>(hi + NHI);
    inv = sig + M;
  }
  // exp(-2 pi i e / n), e < n: two table entries, one complex product
  __device__ __forceinline__ double2 rootN(int e) const { return cmul(lo[e & 127], hi[e >> 7]); }
};

// copy the tables (RaderArgs::tab, sig, inv) into shared memory
template <int R, int P, int NRG = 1>
__device__ __forceinline__ void rader_tables(const RaderSmem<R, P, NRG>& sm, const RaderArgs& a) {
  using S = RaderSmem<R, P, NRG>;
  double2* dt = const_cast<double2*>(sm.tw);
  for (int i = threadIdx.x; i < S::TAB; i += RD_T) dt[i] = __ldg(a.tab + i);
  short* di = const_cast<short*>(sm.sig);
  for (int i = threadIdx.x; i < S::M + P; i += RD_T) di[i] = a.sig[i];
}

// Rader DFTs of the R residues of one ring held in buf[n]; on exit slot q of
// residue r (buf[r + R q]) holds X_r[q^-1] (q >= 1) and slot 0 holds X_r[0].
template <int R, int P, int F1, int F2, int NRG = 1>
__device__ __forceinline__ void rader_residues(const RaderSmem<R, P, NRG>& sm) {
  const short* sig = sm.sig;
  static_assert(F1 * F2 == P - 1, "P - 1 = F1 * F2");
  // pass 1: radix F1 over stride F2 (logical p = F2 n1 + n2), twiddle w^(n2 k1)
  for (int itg = threadIdx.x; itg < NRG * R * F2; itg += RD_T) {
    const int it = NRG > 1 ? itg % (R * F2) : itg;
    double2* buf = sm.buf + (NRG > 1 ? itg / (R * F2) : 0) * (R * P);
    const int r = it % R, n2 = it / R;
    double2 v[F1];
#pragma unroll
    for (int n1 = 0; n1 < F1; ++n1) v[n1] = buf[r + R * sig[F2 * n1 + n2]];
    dft_prime_put<F1>(v, [&](int k1, double2 x) {
      if (k1 && n2) x = cmul(x, sm.tw[n2 * k1]);
      buf[r + R * sig[F2 * k1 + n2]] = x;
    });
  }
  __syncthreads();
  // pass 2: radix F2 over contiguous positions F2 k1 + k2 (frequency k1 + F1 k2),
  // times the transformed kernel, x_r[0] into the zero bin, then the first inverse
  // pass (radix F2, twiddle w^-(k1 j2)) in registers
  for (int itg = threadIdx.x; itg < NRG * R * F1; itg += RD_T) {
    const int it = NRG > 1 ? itg % (R * F1) : itg;
    double2* buf = sm.buf + (NRG > 1 ? itg / (R * F1) : 0) * (R * P);
    const int r = it % R, k1 = it / R;
    double2 v[F2];
    const short* sg = sig + F2 * k1;
#pragma unroll
    for (int k2 = 0; k2 < F2; ++k2) v[k2] = buf[r + R * sg[k2]];
    dft<F2, false>(v);
    double2 x0 = make_double2(0.0, 0.0);
    if (k1 == 0) {  // frequency 0: X_r[0] = x_r[0] + sum_q x_r[q] into slot 0 (only this thread's)
      x0 = buf[r];
      buf[r] = cadd(x0, v[0]);
    }
#pragma unroll
    for (int k2 = 0; k2 < F2; ++k2) v[k2] = cmul(v[k2], sm.Bn[k1 + F1 * k2]);
    if (k1 == 0) v[0] = cadd(v[0], x0);  // x_r[0] joins every convolution output
    dft<F2, true>(v);
#pragma unroll
    for (int j2 = 0; j2 < F2; ++j2) {
      double2 x = v[j2];
      if (k1 && j2) {
        double2 w = sm.tw[k1 * j2];
        w.y = -w.y;
        x = cmul(x, w);
      }
      buf[r + R * sg[j2]] = x;
    }
  }
  __syncthreads();
  // pass 3: inverse radix F1 over stride F2: logical j = F2 j1 + j2 <- c[j] + x_r[0]
  for (int itg = threadIdx.x; itg < NRG * R * F2; itg += RD_T) {
    const int it = NRG > 1 ? itg % (R * F2) : itg;
    double2* buf = sm.buf + (NRG > 1 ? itg / (R * F2) : 0) * (R * P);
    const int r = it % R, j2 = it / R;
    double2 v[F1];
#pragma unroll
    for (int k1 = 0; k1 < F1; ++k1) v[k1] = buf[r + R * sig[F2 * k1 + j2]];
    idft_prime_put<F1>(v, [&](int j1, double2 x) { buf[r + R * sig[F2 * j1 + j2]] = x; });
  }
}

// the R-point combine of output bin k: Y_r[k] from slot inv[k], twiddles w_n^{r k}
template <int R, int P, int NRG = 1>
__device__ __forceinline__ void rader_combine(const RaderSmem<R, P, NRG>& sm, int k, double2 (&y)[R], int ring = 0) {
  const int q = sm.inv[k];
  const double2* src = sm.buf + ring * (R * P) + R * q;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    y[r] = src[r];
    if (r && k) y[r] = cmul(y[r], sm.rootN(r * k));
  }
  dft<R, false>(y);
}

// load one ring (element stride es) into buf, conjugated for the inverse; all of a
// thread's loads of a batch are in flight together
template <int N>
__device__ __forceinline__ void rader_load(double2* buf, const double2* src, long long es, bool conj) {
  constexpr int PER = (N + RD_T - 1) / RD_T, BATCH = 8;
#pragma unroll
  for (int u = 0; u < PER; u += BATCH) {
    double2 t[BATCH];
#pragma unroll
    for (int i = 0; i < BATCH; ++i) {
      const int j = threadIdx.x + (u + i) * RD_T;
      if (u + i < PER && j < N) t[i] = __ldg(src + (long long)j * es);
    }
#pragma unroll
    for (int i = 0; i < BATCH; ++i) {
      const int j = threadIdx.x + (u + i) * RD_T;
      if (u + i < PER && j < N) buf[j] = make_double2(t[i].x, conj ? -t[i].y : t[i].y);
    }
  }
}

// Plain transform (the inverse of the adjoint, and the order-sharded path's
// ring DFTs): CTA per (ring, component), component fastest.
template <int R, int P, int F1, int F2>
__global__ void __launch_bounds__(RD_T, 1) rader_fft_kernel(RaderArgs a) {
  extern __shared__ __align__(16) double2 rd_smem[];
  constexpr int N = R * P;
  const RaderSmem<R, P> sm(rd_smem);
  double2* buf = sm.buf;
  const int c = blockIdx.x % 3, ring = blockIdx.x / 3;
  auto ring_base = [&](int rg) {
    return a.in_rblk ? (long long)(rg >> (31 - __clz(a.in_rblk))) * a.in_rs + (rg & (a.in_rblk - 1))
                     : (long long)rg * a.in_rs;
  };
  if (a.ahead && threadIdx.x == 0 && blockIdx.x + a.ahead < gridDim.x) {
    const int it2 = blockIdx.x + a.ahead, c2 = it2 % 3, rg2 = it2 / 3;
    if (a.in_es == 1 && !a.in_rblk) f2_prefetch_l2(a.in + c2 * a.in_cs + ring_base(rg2), (unsigned)(N * 16));
    else if (a.in_rblk == 2 && a.in_es == 2 && (rg2 & 1) == 0 && rg2 + 1 < a.nrings)  // the pair's block
      f2_prefetch_l2(a.in + c2 * a.in_cs + ring_base(rg2), (unsigned)(2 * N * 16));
  }
  const bool inv = a.inverse != 0;
  rader_tables<R, P>(sm, a);
  rader_load<N>(buf, a.in + c * a.in_cs + ring_base(ring), a.in_es, inv);
  __syncthreads();
  rader_residues<R, P, F1, F2>(sm);
  __syncthreads();
  double2* dst = a.out + c * a.out_cs + (long long)ring * a.out_rs;
  for (int k = threadIdx.x; k < P; k += RD_T) {
    double2 y[R];
    rader_combine<R, P>(sm, k, y);
#pragma unroll
    for (int s = 0; s < R; ++s) dst[(long long)(k + P * s) * a.out_es] = make_double2(y[s].x, inv ? -y[s].y : y[s].y);
  }
}

// Forward with the equatorial fold (fft2.cuh fft_fold_kernel's epilogue): a
// cluster of two CTAs per (ring pair, field, component), rank 0 the north
// ring, rank 1 the south ring; each writes the X sectors of half of the orders.
template <int R, int P, int F1, int F2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RD_T, 1) rader_fold_kernel(RaderArgs a, Fft2Args f) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double2 rd_smem[];
  constexpr int N = R * P;
  const RaderSmem<R, P> sm(rd_smem);
  double2* buf = sm.buf;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int item = blockIdx.x >> 1;
  const int c = item % 3, b = (item / 3) % f.nfields, p = item / (3 * f.nfields);
  const int rn = f.pair_n[p], rs = f.pair_s[p];
  const int my_ring = rank ? rs : rn;
  if (f.ahead && c == 0 && threadIdx.x == 0 && item + f.ahead < (int)(gridDim.x >> 1)) {
    const int it2 = item + f.ahead, b2 = (it2 / 3) % f.nfields, p2 = it2 / (3 * f.nfields);
    const int rg2 = rank ? f.pair_s[p2] : f.pair_n[p2];
    if (rg2 >= 0)
      f2_prefetch_l2(f.in + (long long)b2 * f.field_stride + (long long)rg2 * f.in_rs, (unsigned)(3 * N * 16));
  }
  if (my_ring >= 0) {
    rader_tables<R, P>(sm, a);
    rader_load<N>(buf, f.in + (long long)b * f.field_stride + c + (long long)my_ring * f.in_rs, f.in_es, false);
    __syncthreads();
    rader_residues<R, P, F1, F2>(sm);
    __syncthreads();
    // combine in place: every thread holds its bins' outputs across one barrier
    constexpr int KPT = (P + RD_T - 1) / RD_T;
    double2 y[KPT][R];
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = threadIdx.x + i * RD_T;
      if (k < P) rader_combine<R, P>(sm, k, y[i]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = threadIdx.x + i * RD_T;
      if (k < P) {
#pragma unroll
        for (int s = 0; s < R; ++s) buf[k + P * s] = y[i][s];
      }
    }
  }
  cluster.sync();  // both spectra complete (an absent south ring leaves its CTA's buffer unused)
  const double2* Sn = cluster.map_shared_rank(buf, 0);
  const double2* Ss = cluster.map_shared_rank(buf, 1);
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
  const int nr = (rn >= 0) + (rs >= 0);
  const int half = (f.Lt + 2) / 2;
  const int m0 = rank ? half : 0, m1 = rank ? f.Lt + 1 : half;
  for (int m = m0 + threadIdx.x; m < m1; m += RD_T) {
    double2 Ep = make_double2(0.0, 0.0), Em = Ep, Op = Ep, Om = Ep;
    if (nr > 0) {
      const int bm = m ? N - m : 0;
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
  cluster.sync();  // the partner may still read this CTA's spectrum
}

// ---------------------------------------------------------------------------
// Short rings (C2: n_phi = 516 = 12 * 43, P - 1 = 7 * 6): NRG rings per CTA so the
// passes fill the CTA (one ring has 72 / 84 butterflies and 43 combine bins for 384
// threads), two CTAs per SM.  The forward variant takes ring PAIRS (north ring 2 i,
// south ring 2 i + 1 of item i in the same CTA), so the fold needs no cluster.
// Replaces the direct 43-point DFTs of fft_blue.cuh smallp_kernel (~2 P flops per
// point, issue bound).
// ---------------------------------------------------------------------------
template <int R, int P, int F1, int F2, int NRG>
__global__ void __launch_bounds__(RD_T, 2) rader_multi_fft_kernel(RaderArgs a) {
  extern __shared__ __align__(16) double2 rd_smem[];
  constexpr int N = R * P;
  const RaderSmem<R, P, NRG> sm(rd_smem);
  const int nitems = 3 * a.nrings, item0 = blockIdx.x * NRG;
  auto ring_base = [&](int rg) {
    return a.in_rblk ? (long long)(rg >> (31 - __clz(a.in_rblk))) * a.in_rs + (rg & (a.in_rblk - 1))
                     : (long long)rg * a.in_rs;
  };
  const bool inv = a.inverse != 0;
  rader_tables<R, P, NRG>(sm, a);
#pragma unroll
  for (int i = 0; i < NRG; ++i) {
    const int item = min(item0 + i, nitems - 1);  // a short last CTA repeats its last ring (never stored)
    rader_load<N>(sm.buf + i * N, a.in + (item % 3) * a.in_cs + ring_base(item / 3), a.in_es, inv);
  }
  __syncthreads();
  rader_residues<R, P, F1, F2, NRG>(sm);
  __syncthreads();
  for (int w = threadIdx.x; w < NRG * P; w += RD_T) {
    const int i = w / P, k = w - i * P, item = item0 + i;
    if (item >= nitems) continue;
    double2 y[R];
    rader_combine<R, P, NRG>(sm, k, y, i);
    double2* dst = a.out + (item % 3) * a.out_cs + (long long)(item / 3) * a.out_rs;
#pragma unroll
    for (int s = 0; s < R; ++s) dst[(long long)(k + P * s) * a.out_es] = make_double2(y[s].x, inv ? -y[s].y : y[s].y);
  }
}

template <int R, int P, int F1, int F2, int NPR>
__global__ void __launch_bounds__(RD_T, 2) rader_multi_fold_kernel(RaderArgs a, Fft2Args f, int nitems) {
  extern __shared__ __align__(16) double2 rd_smem[];
  constexpr int N = R * P, NRG = 2 * NPR;
  static_assert(NRG * P <= RD_T, "one combine bin per thread");
  const RaderSmem<R, P, NRG> sm(rd_smem);
  const int item0 = blockIdx.x * NPR;
  rader_tables<R, P, NRG>(sm, a);
#pragma unroll
  for (int i = 0; i < NPR; ++i) {
    const int item = min(item0 + i, nitems - 1);
    const int c = item % 3, b = (item / 3) % f.nfields, p = item / (3 * f.nfields);
    const int rn = f.pair_n[p], rs = f.pair_s[p];
    const double2* base = f.in + (long long)b * f.field_stride + c;
    // an absent ring's buffer is transformed as it is and never read by the epilogue
    if (rn >= 0) rader_load<N>(sm.buf + (2 * i) * N, base + (long long)rn * f.in_rs, f.in_es, false);
    if (rs >= 0) rader_load<N>(sm.buf + (2 * i + 1) * N, base + (long long)rs * f.in_rs, f.in_es, false);
  }
  __syncthreads();
  rader_residues<R, P, F1, F2, NRG>(sm);
  __syncthreads();
  {  // combine in place: every thread holds its bin's outputs across one barrier
    const int w = threadIdx.x, i = w / P, k = w - i * P;
    double2 y[R];
    if (w < NRG * P) rader_combine<R, P, NRG>(sm, k, y, i);
    __syncthreads();
    if (w < NRG * P) {
#pragma unroll
      for (int s = 0; s < R; ++s) sm.buf[i * N + k + P * s] = y[s];
    }
  }
  __syncthreads();
  // epilogue (fft2.cuh fft_fold_kernel's): thread per (item, order m)
  const size_t tile = (size_t)2 * 8 * f.NT * 32;
  const size_t par_stride = (size_t)8 * f.NT * 32;
  for (int w = threadIdx.x; w < NPR * (f.Lt + 1); w += RD_T) {
    const int i = w / (f.Lt + 1), m = w - i * (f.Lt + 1), item = item0 + i;
    if (item >= nitems) continue;
    const int c = item % 3, bg = (item / 3) % f.nfields, p = item / (3 * f.nfields);
    const int nfg = f.gfields ? f.gfields : f.nfields;  // fields per X buffer
    const int b = bg % nfg;
    double* const X = f.X + (size_t)(bg / nfg) * f.x_gstride;
    const int rn = f.pair_n[p], rs = f.pair_s[p];
    const int chunk = p >> 5, ks = (p >> 2) & 7, kq = p & 3;
    const int col = 12 * b + 4 * c;
    const size_t off = ((size_t)ks * f.NT + (col >> 3)) * 32 + ((col >> 2) & 1) * 16 + kq * 4;
    const bool padcols = (b == nfg - 1) && c == 2 && ((12 * nfg) & 7) == 4;
    const int pcol = 12 * nfg;
    const size_t poff = ((size_t)ks * f.NT + (pcol >> 3)) * 32 + ((pcol >> 2) & 1) * 16 + kq * 4;
    const double wn = rn >= 0 ? f.ring_w[rn] : 0.0;
    const double ws = rs >= 0 ? f.ring_w[rs] : 0.0;
    const double2* Sn = sm.buf + (2 * i) * N;
    const double2* Ss = Sn + N;
    double2 Ep = make_double2(0.0, 0.0), Em = Ep, Op = Ep, Om = Ep;
    if (rn >= 0) {
      const int bm = m ? N - m : 0;
      const double2 np = Sn[m], nm = Sn[bm];
      const double sg = (m & 1) ? -1.0 : 1.0;  // sigma_{-m} on the -m bin
      if (rs >= 0) {
        const double2 sp = Ss[m], sm2 = Ss[bm];
        Ep = make_double2(wn * np.x + ws * sp.x, wn * np.y + ws * sp.y);
        Op = make_double2(wn * np.x - ws * sp.x, wn * np.y - ws * sp.y);
        Em = make_double2(sg * (wn * nm.x + ws * sm2.x), sg * (wn * nm.y + ws * sm2.y));
        Om = make_double2(sg * (wn * nm.x - ws * sm2.x), sg * (wn * nm.y - ws * sm2.y));
      } else {  // unpaired ring: both parities see the ring itself
        Ep = Op = make_double2(wn * np.x, wn * np.y);
        Em = Om = make_double2(sg * (wn * nm.x), sg * (wn * nm.y));
      }
      if (m == 0) Em = Om = make_double2(0.0, 0.0);
    }
    double* xt = X + ((size_t)m * f.nchunks + chunk) * tile;
    st_global_v4(xt + off, Ep, Em);
    st_global_v4(xt + par_stride + off, Op, Om);
    if (padcols) {
      const double2 z = make_double2(0.0, 0.0);
      st_global_v4(xt + poff, z, z);
      st_global_v4(xt + par_stride + poff, z, z);
    }
  }
}

}  // namespace fv
