// Ring DFTs, second generation: two rings per CTA, in-place stages, direct
// global I/O, and (forward) the equatorial fold fused into the epilogue.
//
// Reference semantics: favest/scalar.py:149 (np.fft.fft along longitude, sign
// -1) and :178 (np.fft.ifft * n_phi, i.e. the unnormalised sign +1 DFT); the
// fused forward epilogue is the gather / weighting of favest/scalar.py:150-152
// restated with equatorial folding (see fold_fwd_kernel in aux_kernels.cuh,
// which it replaces on the grid path).
//
// Design (B200): the previous kernel (fft.cuh ring_fft_kernel) staged one ring
// per CTA through a cp.async buffer and two ping-pong buffers (100 KB per CTA)
// and was latency / issue bound at 2.1-2.4 TB/s.  Here
//   * one CTA transforms NR = 2 rings of one component at once (the two halves
//     of every stage run side by side, so a radix-19 first stage keeps 216 of
//     256 threads busy instead of 108);
//   * the first stage loads its butterfly inputs straight from HBM into
//     registers (all R loads of a thread in flight), so there is no staging
//     buffer; middle stages are in place (inputs -> registers, barrier,
//     outputs -> the same buffer), so the CTA needs only NR * n complex
//     doubles of shared memory (64 KB at n = 2052, two CTAs per SM);
//   * inter-stage twiddles come from a per-stage table in global memory
//     (L1-resident, exactly rounded, entry (k, r) = w^(r k n / (Ns R)) for the
//     R-1 non-trivial rows), one 16-byte load per twiddle and no product;
//   * the radix plan is chosen for the two-ring thread mapping (plan.cu
//     fft2_factor) and compiled in: n = 2052 runs 19 x 18 x 6 with 216 / 228 /
//     684 butterflies on 256 threads, every index division is by a constant
//     (a runtime radix switch made ptxas spill kilobytes per thread); lengths
//     without an instantiated plan use fft.cuh + the separate fold kernel;
//   * forward on a mirror-symmetric grid: the CTA takes the mirror pair
//     (north ring, south ring) of one (field, component) and its epilogue
//     writes the folded, weighted, sigma_m-signed B operand of the Legendre
//     kernel directly: for every order m and parity, the four values
//     (+m re, +m im, -m re, -m im) of the component are one aligned 32-byte
//     sector of X (X columns are Cartesian, [k][n] inside each fragment tile),
//     so the fold kernel and the spectrum round trip through HBM disappear.
#pragma once
#include "fft.cuh"

namespace fv {

constexpr int F2_T = 256;
constexpr int F2_NR = 2;       // rings per CTA
constexpr int F2_MAXREG = 20;  // complex values a thread holds across an in-place stage barrier

template <int R>
__host__ __device__ constexpr int f2_kb() {
  return F2_MAXREG / R > 0 ? F2_MAXREG / R : 1;
}
// rings / threads per CTA of the plain transform (stage templates take both;
// one ring per 128-thread CTA, four CTAs per SM, measured 4% slower at n = 2052)
constexpr int F2P_NR = 2, F2P_T = 256;
__host__ __device__ constexpr int f2_kb_rt(int R) { return F2_MAXREG / R > 0 ? F2_MAXREG / R : 1; }

// threadIdx.x re-read per stage: an opaque value stops the compiler from
// hoisting every stage's per-thread index math out of the persistent item
// loop (which keeps it live across all stages and spills the radix-19 stage)
__device__ __forceinline__ int opaque_tid() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

struct Fft2Args {
  const double2* in;
  double2* out;                      // plain epilogue
  long long in_cs, in_rs, out_cs, out_rs;  // component / ring strides (complex units)
  int in_es, out_es;                 // element strides
  int in_rblk;                       // plain: blocked input rings (common.cuh SLayout rblk), 0 = in_rs apart
  const double2* tw;                 // twiddle tables (forward sign): stage 1 then stage 2, entry [k][r - 1]
  int nrings;                        // plain: rings per component
  // fused forward fold
  double* X;
  const int* pair_n;
  const int* pair_s;
  const double* ring_w;
  long long field_stride;            // complex units between fields of the input
  int nchunks, NT, nfields, Lt;
  int ahead;                         // L2 prefetch of the input of item blockIdx.x + ahead (0: off)
  // rader_multi_fold_kernel: nfields spans several groups of gfields fields, the X of group g at
  // + g * x_gstride (0: one group)
  int gfields;
  long long x_gstride;
};

// cp.async.bulk.prefetch.L2: one instruction per contiguous block (16-byte
// aligned address and size); no completion, no register or shared state
__device__ __forceinline__ void f2_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// compile-time plan: up to three stages R0 x R1 x R2 (0 = absent), largest first
template <int R0, int R1, int R2>
struct F2Plan {
  static constexpr int N = R0 * (R1 ? R1 : 1) * (R2 ? R2 : 1);
  static constexpr int NST = 1 + (R1 != 0) + (R2 != 0);
  static constexpr int TW2 = R1 ? (R1 - 1) * R0 : 0;  // offset of stage 2's table
};

template <int R, bool INV>
__device__ __forceinline__ void f2_twiddle(double2 (&v)[R], const double2* __restrict__ t) {
#pragma unroll
  for (int r = 1; r < R; ++r) {
    double2 w = __ldg(t + r - 1);
    if (INV) w.y = -w.y;
    v[r] = cmul(v[r], w);
  }
}

// First stage (Ns = 1): inputs straight from global memory (per-ring base
// pointers, element stride es), outputs to shared memory or, for a one-stage
// plan, to global memory (element stride des).
template <int R, int N, bool INV, bool LAST, int NR, int T>
__device__ __forceinline__ void f2_first(const double2* const (&src)[NR], int es, int nr, double2* buf,
                                         double2* const (&dst)[NR], int des) {
  constexpr int KB = f2_kb<R>(), NB = N / R;  // plan.cu fft2_factor: <= KB butterflies per thread at T / NR = 128
  const int tot = nr * NB;
  const int tid = threadIdx.x;
  double2 v[KB][R];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int j = tid + k * T;
    if (j < tot) {
      const int ring = j / NB, jj = j - ring * NB;
      const double2* s = (NR > 1 && ring) ? src[NR - 1] : src[0];
#pragma unroll
      for (int r = 0; r < R; ++r) v[k][r] = __ldg(s + (long long)(jj + r * NB) * es);
    }
  }
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int j = tid + k * T;
    if (j < tot) {
      const int ring = j / NB, jj = j - ring * NB;
      dft<R, INV>(v[k]);
      if (LAST) {
        double2* d = (NR > 1 && ring) ? dst[NR - 1] : dst[0];
#pragma unroll
        for (int r = 0; r < R; ++r) d[(long long)(jj + r * NB) * des] = v[k][r];
      } else {
        double2* d = buf + ring * N + jj * R;
#pragma unroll
        for (int r = 0; r < R; ++r) d[r] = v[k][r];
      }
    }
  }
}

// Middle stage (or the last stage of the fused epilogue): in place in shared memory.
template <int R, int NS, int N, bool INV, int T>
__device__ __forceinline__ void f2_mid(const double2* __restrict__ tw, int nr, double2* buf) {
  constexpr int KB = f2_kb<R>(), NB = N / R;  // plan.cu fft2_factor: <= KB butterflies per thread at T / NR = 128
  const int tot = nr * NB;
  const int tid = threadIdx.x;
  double2 v[KB][R];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int j = tid + k * T;
    if (j < tot) {
      const int ring = j / NB, jj = j - ring * NB;
      const double2* src = buf + ring * N;
#pragma unroll
      for (int r = 0; r < R; ++r) v[k][r] = src[jj + r * NB];
      f2_twiddle<R, INV>(v[k], tw + (jj % NS) * (R - 1));
      dft<R, INV>(v[k]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int j = tid + k * T;
    if (j < tot) {
      const int ring = j / NB, jj = j - ring * NB;
      double2* d = buf + ring * N + (jj / NS) * NS * R + jj % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) d[r * NS] = v[k][r];
    }
  }
  __syncthreads();
}

// Last stage of the plain transform: shared memory -> global (element stride des).
template <int R, int NS, int N, bool INV, int NR, int T>
__device__ __forceinline__ void f2_last(const double2* __restrict__ tw, int nr, const double2* buf,
                                        double2* const (&dst)[NR], int des) {
  constexpr int KB = f2_kb<R>(), NB = N / R;  // plan.cu fft2_factor: <= KB butterflies per thread at T / NR = 128
  const int tot = nr * NB;
  const int tid = threadIdx.x;
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int j = tid + k * T;
    if (j < tot) {
      const int ring = j / NB, jj = j - ring * NB;
      const double2* src = buf + ring * N;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = src[jj + r * NB];
      const int kk = jj % NS;
      f2_twiddle<R, INV>(v, tw + kk * (R - 1));
      const int base = (jj / NS) * NS * R + kk;
      double2* d = (NR > 1 && ring) ? dst[NR - 1] : dst[0];
      if constexpr (R >= 11 && first_factor(R) == R) {
        prime_store<R, INV>(v, d, base, NS, des);
      } else {
        dft<R, INV>(v);
#pragma unroll
        for (int r = 0; r < R; ++r) d[(long long)(base + r * NS) * des] = v[r];
      }
    }
  }
}

// nr rings (<= 2) of length N: global src -> ... -> shared memory (KEEP: the
// spectrum stays in buf for the fused epilogue) or -> global dst.
template <int R0, int R1, int R2, bool INV, bool KEEP, int NR, int T>
__device__ __forceinline__ void f2_run(const double2* tw, const double2* const (&src)[NR], int es, int nr,
                                       double2* buf, double2* const (&dst)[NR], int des) {
  using P = F2Plan<R0, R1, R2>;
  constexpr int N = P::N;
  if constexpr (P::NST == 1) {
    f2_first<R0, N, INV, !KEEP, NR, T>(src, es, nr, buf, dst, des);
    if (KEEP) __syncthreads();
  } else if constexpr (P::NST == 2) {
    f2_first<R0, N, INV, false, NR, T>(src, es, nr, buf, dst, des);
    __syncthreads();
    if constexpr (KEEP) f2_mid<R1, R0, N, INV, T>(tw, nr, buf);
    else f2_last<R1, R0, N, INV, NR, T>(tw, nr, buf, dst, des);
  } else {
    f2_first<R0, N, INV, false, NR, T>(src, es, nr, buf, dst, des);
    __syncthreads();
    f2_mid<R1, R0, N, INV, T>(tw, nr, buf);
    if constexpr (KEEP) f2_mid<R2, R0 * R1, N, INV, T>(tw + P::TW2, nr, buf);
    else f2_last<R2, R0 * R1, N, INV, NR, T>(tw + P::TW2, nr, buf, dst, des);
  }
}

// Plain transform: item = (group of F2P_NR consecutive rings, component),
// component fastest; one CTA per item.  (Persistent CTAs with an L2 prefetch of the next
// item were measured slower: the item loop made ptxas hoist per-thread index
// math across stages and spill.)
template <bool INV, int R0, int R1, int R2>
__global__ void __launch_bounds__(F2P_T, 2) ring_fft2_kernel(Fft2Args a, int nitems) {
  extern __shared__ __align__(16) double2 f2buf[];
  const int item = blockIdx.x;
  if (item >= nitems) return;
  const int c = item % 3, g = item / 3;
  const int r0 = g * F2P_NR;
  if (a.ahead && a.in_rblk == F2P_NR && threadIdx.x == 0 && item + a.ahead < nitems) {
    // the item one wave ahead: its two rings of one component are one
    // contiguous block of the ring-pair spectrum layout
    const int it2 = item + a.ahead, c2 = it2 % 3, q0 = (it2 / 3) * F2P_NR;
    if (a.nrings - q0 >= F2P_NR)
      f2_prefetch_l2(a.in + c2 * a.in_cs + (long long)(q0 / F2P_NR) * a.in_rs,
                     (unsigned)(F2P_NR * F2Plan<R0, R1, R2>::N * sizeof(double2)));
  }
  const int nr = min(F2P_NR, a.nrings - r0);
  const double2* src[F2P_NR];
  double2* dst[F2P_NR];
#pragma unroll
  for (int i = 0; i < F2P_NR; ++i) {
    const int r = min(r0 + i, a.nrings - 1);
    src[i] = a.in + c * a.in_cs +
             (a.in_rblk ? (long long)(r >> (31 - __clz(a.in_rblk))) * a.in_rs + (r & (a.in_rblk - 1)) : r * a.in_rs);
    dst[i] = a.out + c * a.out_cs + r * a.out_rs;
  }
  f2_run<R0, R1, R2, INV, false, F2P_NR, F2P_T>(a.tw, src, a.in_es, nr, f2buf, dst, a.out_es);
}

// Fused forward: item = (pair p < nchunks * 32, field b < nfields, component c),
// c fastest.  Input T is the (B, N, 3) field (element stride 3, ring stride
// 3 n, field stride field_stride); X receives, for every order m = 0..Lt and
// parity,  E/O = sigma * (w_n S_n[+-m] +/- w_s S_s[+-m])  at columns
// 12 b + 4 c + (2 sign + re/im) (Cartesian component c), rows ordered
// [m][chunk][par][ks][nt][n_hi 2][k 4][n_lo 4] (the Legendre consumers' B
// fragments; a component's four columns share n_hi, so they are one sector).
template <int R0, int R1, int R2>
__global__ void __launch_bounds__(F2_T, 2) fft_fold_kernel(Fft2Args a, int nitems) {
  extern __shared__ __align__(16) double2 f2buf[];
  constexpr int n = F2Plan<R0, R1, R2>::N;
  const int item = blockIdx.x;
  if (item >= nitems) return;
  const int c = item % 3, b = (item / 3) % a.nfields, p = item / (3 * a.nfields);
  if (a.ahead && c == 0 && threadIdx.x == 0 && item + a.ahead < nitems) {
    // the ring pair of the item one wave ahead (whole rings: all three
    // components are interleaved), once per (pair, field)
    const int it2 = item + a.ahead, b2 = (it2 / 3) % a.nfields, p2 = it2 / (3 * a.nfields);
    const int rn2 = a.pair_n[p2], rs2 = a.pair_s[p2];
    const double2* base2 = a.in + (long long)b2 * a.field_stride;
    constexpr unsigned ring_bytes = 3u * n * sizeof(double2);
    if (rn2 >= 0) f2_prefetch_l2(base2 + (long long)rn2 * a.in_rs, ring_bytes);
    if (rs2 >= 0) f2_prefetch_l2(base2 + (long long)rs2 * a.in_rs, ring_bytes);
  }
  const int rn = a.pair_n[p], rs = a.pair_s[p];
  const int nr = (rn >= 0) + (rs >= 0);
  if (nr > 0) {
    const double2* base = a.in + (long long)b * a.field_stride + c;
    const double2* src[F2_NR] = {base + (long long)rn * a.in_rs, base + (long long)(rs >= 0 ? rs : rn) * a.in_rs};
    double2* dst[F2_NR] = {nullptr, nullptr};
    f2_run<R0, R1, R2, false, true, F2_NR, F2_T>(a.tw, src, a.in_es, nr, f2buf, dst, 0);
  }
  // epilogue: thread per order m
  const int chunk = p >> 5, ks = (p >> 2) & 7, kq = p & 3;
  const int col = 12 * b + 4 * c;
  const size_t tile = (size_t)2 * 8 * a.NT * 32;
  const size_t par_stride = (size_t)8 * a.NT * 32;
  const size_t off = ((size_t)ks * a.NT + (col >> 3)) * 32 + ((col >> 2) & 1) * 16 + kq * 4;
  // padding columns 12 nf .. 8 NT - 1 (when 12 nf is not a multiple of 8): the
  // last (field, component) item zeroes them
  const bool padcols = (b == a.nfields - 1) && c == 2 && ((12 * a.nfields) & 7) == 4;
  const int pcol = 12 * a.nfields;
  const size_t poff = ((size_t)ks * a.NT + (pcol >> 3)) * 32 + ((pcol >> 2) & 1) * 16 + kq * 4;
  const double wn = rn >= 0 ? a.ring_w[rn] : 0.0;
  const double ws = rs >= 0 ? a.ring_w[rs] : 0.0;
  const double2* Sn = f2buf;
  const double2* Ss = f2buf + n;
  for (int m = threadIdx.x; m <= a.Lt; m += F2_T) {
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
    double* xt = a.X + ((size_t)m * a.nchunks + chunk) * tile;
    st_global_v4(xt + off, Ep, Em);
    st_global_v4(xt + par_stride + off, Op, Om);
    if (padcols) {
      const double2 z = make_double2(0.0, 0.0);
      st_global_v4(xt + poff, z, z);
      st_global_v4(xt + par_stride + poff, z, z);
    }
  }
}

// Instantiated plans (n_phi = 2L + 4 of the benchmark grids and the test
// lengths); plan.cu fft2_factor must produce exactly these radix triples.
#define FV_F2_PLANS(X) \
  X(19, 18, 6)         /* 2052: L = 1024 */ \
  X(17, 4, 0)          /* 68: L = 32 */ \
  X(19, 6, 3)          /* 342 */ \
  X(13, 11, 2)         /* 286 */ \
  X(8, 4, 4)           /* 128 */ \
  X(8, 8, 0)           /* 64 */ \
  X(8, 6, 0)           /* 48 */ \
  X(6, 6, 0)           /* 36 */ \
  X(6, 4, 0)           /* 24 */

}  // namespace fv
