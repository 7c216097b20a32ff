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

// cos / sin(2 pi m / R) for the odd primes R = 3..19, packed: offset of R below
__constant__ double kRootCos[3 + 5 + 7 + 11 + 13 + 17 + 19];
__constant__ double kRootSin[3 + 5 + 7 + 11 + 13 + 17 + 19];

__host__ __device__ constexpr int root_offset(int R) {
  return R == 3 ? 0 : R == 5 ? 3 : R == 7 ? 8 : R == 11 ? 15 : R == 13 ? 26 : R == 17 ? 39 : 56;
}

struct RingFftArgs {
  const double2* in;
  double2* out;
  long long in_cs, in_rs;           // strides (complex units): component, ring
  long long out_cs, out_rs;
  int in_es, out_es;                // element strides (complex units)
  const double2* tw;                // tw[k] = exp(-2 pi i k / n), k < n
  int n, nst;
  int radix[FFT_MAXST];
  int ns[FFT_MAXST];                // product of the previous radices
  unsigned nsmagic[FFT_MAXST];      // ceil(2^32 / ns): j / ns = umulhi(j, magic) for j < 2^16
  int tstride[FFT_MAXST];           // n / (ns * radix)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// R-point DFT of v, results stored to dst[(base + k*Ns) * des]; forward uses
// exp(-2 pi i jk/R), inverse exp(+...).  Odd primes: conjugate-symmetric form,
// outputs are stored as soon as each pair X[k], X[R-k] is formed (keeps the
// live set to the R-1 sums/differences).
template <int R, bool INV>
__device__ __forceinline__ void butterfly_store(const double2 (&v)[R], double2* __restrict__ dst, int base, int Ns,
                                                int des) {
  auto put = [&](int k, double2 x) { dst[(base + k * Ns) * des] = x; };
  if constexpr (R == 2) {
    put(0, make_double2(v[0].x + v[1].x, v[0].y + v[1].y));
    put(1, make_double2(v[0].x - v[1].x, v[0].y - v[1].y));
  } else if constexpr (R == 4) {
    const double2 a = v[0], b = v[1], c = v[2], d = v[3];
    const double2 s0 = make_double2(a.x + c.x, a.y + c.y), d0 = make_double2(a.x - c.x, a.y - c.y);
    const double2 s1 = make_double2(b.x + d.x, b.y + d.y), d1 = make_double2(b.x - d.x, b.y - d.y);
    put(0, make_double2(s0.x + s1.x, s0.y + s1.y));
    put(2, make_double2(s0.x - s1.x, s0.y - s1.y));
    // forward: X1 = d0 - i d1, X3 = d0 + i d1
    if (INV) {
      put(1, make_double2(d0.x - d1.y, d0.y + d1.x));
      put(3, make_double2(d0.x + d1.y, d0.y - d1.x));
    } else {
      put(1, make_double2(d0.x + d1.y, d0.y - d1.x));
      put(3, make_double2(d0.x - d1.y, d0.y + d1.x));
    }
  } else {
    constexpr int H = (R - 1) / 2;
    constexpr int O = root_offset(R);
    double2 s[H + 1], d[H + 1];
    const double2 x0 = v[0];
    double2 X0 = x0;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      s[j] = make_double2(v[j].x + v[R - j].x, v[j].y + v[R - j].y);
      d[j] = make_double2(v[j].x - v[R - j].x, v[j].y - v[R - j].y);
      X0 = make_double2(X0.x + s[j].x, X0.y + s[j].y);
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
}

// One Stockham stage of radix R (Ns = product of the previous radices):
// butterfly j reads src[j + r*n/R], twiddles by w^(r*(j%Ns)*n/(Ns*R)) (the
// exponent is < n, no modulo), writes dst[(j/Ns)*Ns*R + j%Ns + r*Ns].  src and
// dst are distinct (ping-pong smem buffers, or global for the first / last
// stage; GSRC / GDST select the address space at compile time), so a thread
// keeps only the R values of the butterfly it is working on.
template <int R, bool INV, bool GSRC, bool GDST>
__device__ __forceinline__ void fft_stage(const double2* __restrict__ src, int ses, double2* __restrict__ dst, int des,
                                          const double2* __restrict__ tw, int n, int Ns, unsigned magic,
                                          int tstride) {
  const int nb = n / R;
  for (int j = threadIdx.x; j < nb; j += FFT_THREADS) {
    const int q = Ns == 1 ? j : (int)__umulhi((unsigned)j, magic);  // j / Ns
    const int k = j - q * Ns;                           // j % Ns
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = GSRC ? __ldg(&src[(j + r * nb) * ses]) : src[j + r * nb];
    if (Ns > 1) {
      const int step = k * tstride;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        double2 w = __ldg(&tw[r * step]);
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    butterfly_store<R, INV>(v, dst, q * Ns * R + k, Ns, GDST ? des : 1);
  }
}

template <bool INV, bool GSRC, bool GDST>
__device__ __forceinline__ void fft_stage_dispatch(int R, const double2* src, int ses, double2* dst, int des,
                                                   const double2* tw, int n, int Ns, unsigned magic, int ts) {
  switch (R) {
    case 2: fft_stage<2, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 3: fft_stage<3, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 4: fft_stage<4, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 5: fft_stage<5, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 7: fft_stage<7, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 11: fft_stage<11, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 13: fft_stage<13, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    case 17: fft_stage<17, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
    default: fft_stage<19, INV, GSRC, GDST>(src, ses, dst, des, tw, n, Ns, magic, ts); break;
  }
}

// grid (3 components, rings): the three components of a ring are adjacent
// CTAs, so they stream the same interleaved [N][3] lines through L2 together.
// Dynamic smem: 2 n complex doubles (ping-pong).
template <bool INV>
__global__ void __launch_bounds__(FFT_THREADS, 2) ring_fft_kernel(RingFftArgs a) {
  extern __shared__ __align__(16) double2 buf[];
  const int c = blockIdx.x, ring = blockIdx.y;
  const double2* gin = a.in + c * a.in_cs + ring * a.in_rs;
  double2* gout = a.out + c * a.out_cs + ring * a.out_rs;
  const int n = a.n, nst = a.nst;
  if (nst == 1) {
    fft_stage_dispatch<INV, true, true>(a.radix[0], gin, a.in_es, gout, a.out_es, a.tw, n, 1, a.nsmagic[0],
                                        a.tstride[0]);
    return;
  }
  // stage s reads buffer (s & 1) and writes buffer ((s + 1) & 1)
  fft_stage_dispatch<INV, true, false>(a.radix[0], gin, a.in_es, buf + n, 1, a.tw, n, 1, a.nsmagic[0], a.tstride[0]);
  __syncthreads();
  for (int s = 1; s < nst - 1; ++s) {
    fft_stage_dispatch<INV, false, false>(a.radix[s], buf + (s & 1) * n, 1, buf + ((s + 1) & 1) * n, 1, a.tw, n,
                                          a.ns[s], a.nsmagic[s], a.tstride[s]);
    __syncthreads();
  }
  const int s = nst - 1;
  fft_stage_dispatch<INV, false, true>(a.radix[s], buf + (s & 1) * n, 1, gout, a.out_es, a.tw, n, a.ns[s],
                                       a.nsmagic[s], a.tstride[s]);
}

}  // namespace fv
