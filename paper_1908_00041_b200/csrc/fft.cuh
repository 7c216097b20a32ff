// Ring DFTs along longitude (favest/scalar.py:149 forward np.fft.fft, :178
// inverse np.fft.ifft * n_phi, i.e. unnormalised), hand-written for sm_100a.
//
// One CTA per (ring, Cartesian component): the ring (n <= FFT_NMAX complex
// doubles) lives in shared memory (two ping-pong buffers, 66 KB at n = 2052 ->
// three CTAs per SM) and is transformed by a mixed-radix Stockham sequence
// (self-sorting, no bit reversal).  The first stage reads the field straight
// from HBM (any element stride, e.g. the [B][N][3] AoS field), the last stage
// writes straight to HBM, so HBM sees exactly one read and one write per value.
//
// Radices: 4 and 2 (multiplier-free), odd primes 3..19 with the conjugate
// symmetric DFT (pairs X[k], X[R-k] share the cosine sums), whose roots are
// __constant__ operands of the DFMAs.  Lengths with a prime factor > 19 use
// cuFFT (plan.cu).  Inter-stage twiddles exp(-+2 pi i k/n) come from a
// per-plan table computed in long double on the host.
#pragma once
#include "common.cuh"

namespace fv {

constexpr int FFT_THREADS = 256;
constexpr int FFT_NMAX = 4104;   // covers n_phi = 2L+4 for L <= 2050
constexpr int FFT_MAXST = 16;
constexpr int FFT_TWLO = 64;     // twiddle w^k = hi[k / 64] * lo[k % 64] (two small smem tables)
constexpr int FFT_TWN = FFT_TWLO + (FFT_NMAX + FFT_TWLO - 1) / FFT_TWLO;

// cos / sin(2 pi m / R) for the odd primes R = 3..19 and 31 (the Rader stage,
// fft_rader.cuh), packed: offset of R below
constexpr int kRootR[8] = {3, 5, 7, 11, 13, 17, 19, 31};
__constant__ double kRootCos[3 + 5 + 7 + 11 + 13 + 17 + 19 + 31];
__constant__ double kRootSin[3 + 5 + 7 + 11 + 13 + 17 + 19 + 31];

__host__ __device__ constexpr int root_offset(int R) {
  return R == 3 ? 0 : R == 5 ? 3 : R == 7 ? 8 : R == 11 ? 15 : R == 13 ? 26 : R == 17 ? 39 : R == 19 ? 56 : 75;
}

struct RingFftArgs {
  const double2* in;
  double2* out;
  long long in_cs, in_rs;           // strides (complex units): component, ring
  long long out_cs, out_rs;
  int in_es, out_es;                // element strides (complex units)
  const double2* tw;                // FFT_TWLO entries exp(-2 pi i k / n), k < 64, then exp(-2 pi i 64 j / n)
  int n, nst;
  int nrings;                       // rings (all fields) -> 3 * nrings items
  int radix[FFT_MAXST];
  int ns[FFT_MAXST];                // product of the previous radices
  unsigned nsmagic[FFT_MAXST];      // ceil(2^32 / ns): j / ns = umulhi(j, magic) for j < 2^16
  int tstride[FFT_MAXST];           // n / (ns * radix)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// exp(-2 pi i e / R) for the composite radices' internal twiddles, packed by R
// (offsets below; filled per device by plan.cu).
constexpr int kCompR[12] = {4, 6, 8, 9, 10, 12, 14, 15, 16, 18, 20, 22};
__constant__ double kCompCos[4 + 6 + 8 + 9 + 10 + 12 + 14 + 15 + 16 + 18 + 20 + 22];
__constant__ double kCompSin[4 + 6 + 8 + 9 + 10 + 12 + 14 + 15 + 16 + 18 + 20 + 22];
__host__ __device__ constexpr int comp_offset(int R) {
  return R == 4 ? 0 : R == 6 ? 4 : R == 8 ? 10 : R == 9 ? 18 : R == 10 ? 27 : R == 12 ? 37 : R == 14 ? 49
       : R == 15 ? 63 : R == 16 ? 78 : R == 18 ? 94 : R == 20 ? 112 : 132;
}
__host__ __device__ constexpr int first_factor(int R) {
  return R % 4 == 0 ? 4 : R % 2 == 0 ? 2 : R % 3 == 0 ? 3 : R % 5 == 0 ? 5 : R % 7 == 0 ? 7 : R;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// v * exp(-+2 pi i e / R); e is a constant after unrolling (j2 * k1 in dft):
// multiples of a quarter turn are exact swaps / negations, the rest one complex
// multiply by a constant-bank operand.
template <int R, bool INV>
__device__ __forceinline__ double2 rot_dyn(double2 v, int e) {
  e %= R;
  if (e == 0) return v;
  if ((4 * e) % R == 0) {
    const int q = 4 * e / R;
    if (q == 2) return make_double2(-v.x, -v.y);
    if ((q == 1) != INV) return make_double2(v.y, -v.x);
    return make_double2(-v.y, v.x);
  }
  const double c = kCompCos[comp_offset(R) + e], sn = kCompSin[comp_offset(R) + e];
  const double si = INV ? sn : -sn;
  return make_double2(fma(v.x, c, -v.y * si), fma(v.x, si, v.y * c));
}

// In-register DFT of size R (natural order in and out).  Primes 2, 3, 5, 7
// direct; R = 4 multiplier-free; composites R = A * B by one Cooley-Tukey split
// (A DFTs over the stride-B subsequences, constant twiddles, B DFTs).
template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&v)[R]);

template <int R, bool INV>
__device__ __forceinline__ void dft_prime(double2 (&v)[R]) {
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
  v[0] = X0;
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
    if (INV) {
      v[k] = make_double2(ar - bi, ai + br);
      v[R - k] = make_double2(ar + bi, ai - br);
    } else {
      v[k] = make_double2(ar + bi, ai - br);
      v[R - k] = make_double2(ar - bi, ai + br);
    }
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&v)[R]) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    const double2 s0 = cadd(v[0], v[2]), d0 = csub(v[0], v[2]);
    const double2 s1 = cadd(v[1], v[3]), d1 = csub(v[1], v[3]);
    v[0] = cadd(s0, s1);
    v[2] = csub(s0, s1);
    if (INV) {
      v[1] = make_double2(d0.x - d1.y, d0.y + d1.x);
      v[3] = make_double2(d0.x + d1.y, d0.y - d1.x);
    } else {
      v[1] = make_double2(d0.x + d1.y, d0.y - d1.x);
      v[3] = make_double2(d0.x - d1.y, d0.y + d1.x);
    }
  } else if constexpr (first_factor(R) == R) {
    dft_prime<R, INV>(v);
  } else {
    constexpr int A = first_factor(R), B = R / A;
    double2 y[R];
#pragma unroll
    for (int j2 = 0; j2 < B; ++j2) {  // x[B j1 + j2] -> A-point DFT over j1
      double2 t[A];
#pragma unroll
      for (int j1 = 0; j1 < A; ++j1) t[j1] = v[B * j1 + j2];
      dft<A, INV>(t);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) y[k1 * B + j2] = t[k1];
#pragma unroll
      for (int k1 = 1; k1 < A; ++k1) {
        // twiddle W_R^(j2 k1): unrolled constant exponent via a small switch on j2*k1
        y[k1 * B + j2] = rot_dyn<R, INV>(y[k1 * B + j2], j2 * k1);
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {  // B-point DFT over j2 -> X[k1 + A k2]
      double2 t[B];
#pragma unroll
      for (int j2 = 0; j2 < B; ++j2) t[j2] = y[k1 * B + j2];
      dft<B, INV>(t);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = t[k2];
    }
  }
}

// R-point DFT of v for the large primes (11, 13, 17, 19), results stored to
// dst[(base + k*Ns) * des] as soon as each pair X[k], X[R-k] is formed (keeps
// the live set to the R-1 sums / differences).
template <int R, bool INV>
__device__ __forceinline__ void prime_store(const double2 (&v)[R], double2* __restrict__ dst, int base, int Ns,
                                            int des) {
  auto put = [&](int k, double2 x) { dst[(base + k * Ns) * des] = x; };
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
    // X[k] = A + i sgn B, X[R-k] = A - i sgn B with B = sum sin * d (sgn = -1 forward)
    if (INV) {
      put(k, make_double2(ar - bi, ai + br));
      put(R - k, make_double2(ar + bi, ai - br));
    } else {
      put(k, make_double2(ar + bi, ai - br));
      put(R - k, make_double2(ar - bi, ai + br));
    }
  }
}

// w^k (k < n) from the factored smem tables; conjugated for the inverse.
template <bool INV>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int k) {
  double2 w = cmul(tw[FFT_TWLO + (k >> 6)], tw[k & (FFT_TWLO - 1)]);
  if (INV) w.y = -w.y;
  return w;
}

// One Stockham stage of radix R (Ns = product of the previous radices):
// butterfly j reads src[j + r*n/R], twiddles by w^(r*(j%Ns)*n/(Ns*R)) (the
// exponent is < n, no modulo), writes dst[(j/Ns)*Ns*R + j%Ns + r*Ns].  src is
// shared memory; dst is the other ping-pong buffer or, for the last stage, HBM
// (element stride des).
template <int R, bool INV>
__device__ __forceinline__ void fft_stage(const double2* __restrict__ src, double2* __restrict__ dst, int des,
                                          const double2* __restrict__ tw, int n, int Ns, unsigned magic,
                                          int tstride) {
  const int nb = n / R;
  for (int j = threadIdx.x; j < nb; j += FFT_THREADS) {
    const int q = Ns == 1 ? j : (int)__umulhi((unsigned)j, magic);  // j / Ns
    const int k = j - q * Ns;                                        // j % Ns
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
    if (Ns > 1) {
      const int step = k * tstride;
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twiddle<INV>(tw, r * step));
    }
    const int base = q * Ns * R + k;
    if constexpr (R >= 11 && first_factor(R) == R) {  // large primes
      prime_store<R, INV>(v, dst, base, Ns, des);
    } else {
      dft<R, INV>(v);
#pragma unroll
      for (int r = 0; r < R; ++r) dst[(base + r * Ns) * des] = v[r];
    }
  }
}

template <bool INV>
__device__ __forceinline__ void fft_stage_dispatch(int R, const double2* src, double2* dst, int des,
                                                   const double2* tw, int n, int Ns, unsigned magic, int ts) {
  switch (R) {
#define FV_FFT_CASE(r) \
  case r: fft_stage<r, INV>(src, dst, des, tw, n, Ns, magic, ts); break;
    FV_FFT_CASE(2) FV_FFT_CASE(3) FV_FFT_CASE(4) FV_FFT_CASE(5) FV_FFT_CASE(6) FV_FFT_CASE(7)
    FV_FFT_CASE(8) FV_FFT_CASE(9) FV_FFT_CASE(10) FV_FFT_CASE(11) FV_FFT_CASE(12) FV_FFT_CASE(13)
    FV_FFT_CASE(14) FV_FFT_CASE(15) FV_FFT_CASE(16) FV_FFT_CASE(17)
#undef FV_FFT_CASE
    default: fft_stage<19, INV>(src, dst, des, tw, n, Ns, magic, ts); break;
  }
}

__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}

// Persistent: 2 CTAs per SM walk the (ring, component) items, component fastest
// (the three components of a ring stream the same interleaved [N][3] lines
// through L2 together).  Each item's input is staged into shared memory with
// cp.async (every element in flight at once), and the next item's staging is
// issued as soon as stage 0 has consumed the buffer, so it overlaps the
// remaining in-smem stages.  Dynamic smem: 3 n complex doubles (ping-pong +
// staging) + the twiddle tables.
template <bool INV>
__global__ void __launch_bounds__(FFT_THREADS, 2) ring_fft_kernel(RingFftArgs a) {
  extern __shared__ __align__(16) double2 buf[];
  const int n = a.n, nst = a.nst;
  double2* stg = buf + 2 * n;
  double2* tw = buf + 3 * n;
  const int nitems = 3 * a.nrings;
  const int ntw = FFT_TWLO + (n + FFT_TWLO - 1) / FFT_TWLO;
  for (int i = threadIdx.x; i < ntw; i += FFT_THREADS) tw[i] = a.tw[i];
  auto stage_in = [&](int item) {
    const int c = item % 3, ring = item / 3;
    const double2* src = a.in + c * a.in_cs + ring * a.in_rs;
    for (int i = threadIdx.x; i < n; i += FFT_THREADS) cp_async16(&stg[i], &src[(long long)i * a.in_es]);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int item = blockIdx.x;
  if (item < nitems) stage_in(item);
  for (; item < nitems; item += gridDim.x) {
    const int c = item % 3, ring = item / 3;
    double2* gout = a.out + c * a.out_cs + ring * a.out_rs;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (nst == 1) {
      fft_stage_dispatch<INV>(a.radix[0], stg, gout, a.out_es, tw, n, 1, a.nsmagic[0],
                                           a.tstride[0]);
      __syncthreads();
      if (item + gridDim.x < nitems) stage_in(item + gridDim.x);
      continue;
    }
    // stage s reads buffer (s & 1) (stage 0: the staging buffer) and writes ((s + 1) & 1)
    fft_stage_dispatch<INV>(a.radix[0], stg, buf + n, 1, tw, n, 1, a.nsmagic[0], a.tstride[0]);
    __syncthreads();
    if (item + gridDim.x < nitems) stage_in(item + gridDim.x);  // staging buffer is free again
    for (int s = 1; s < nst - 1; ++s) {
      fft_stage_dispatch<INV>(a.radix[s], buf + (s & 1) * n, buf + ((s + 1) & 1) * n, 1, tw, n,
                                            a.ns[s], a.nsmagic[s], a.tstride[s]);
      __syncthreads();
    }
    const int s = nst - 1;
    fft_stage_dispatch<INV>(a.radix[s], buf + (s & 1) * n, gout, a.out_es, tw, n, a.ns[s],
                                         a.nsmagic[s], a.tstride[s]);
    __syncthreads();  // the next item's stage 0 overwrites the ping-pong buffers
  }
}

}  // namespace fv
