// Adjoint at scattered points (favest/scalar.py:120-128 with ylm_table,
// favest/legendre.py:106-123): f(x_p) = sum_{l,m} g_{l,m} sigma_m Pbar_l^|m|(z_p) e^{i m phi_p}.
//
// One thread per point.  Orders are walked in sequence so the diagonal seed is
// a running product (extended range), the l-recurrence runs in registers, and
// the merged coefficient rows (sigma applied, m-major) are staged per order in
// shared memory and read as broadcasts.  The per-point recurrence cannot be shared between points, so
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

constexpr int PTS_THREADS = 256;

// Coefficient rows of order m (rows rowofs[m] .. + Lt - m, NC doubles each) into
// shared memory with cp.async (16-byte pieces); one commit group per order.
template <int NC>
__device__ __forceinline__ void pts_stage_rows(const PtsArgs& a, int m, double* dst) {
  if (m <= a.Lt) {
    const double2* src = reinterpret_cast<const double2*>(a.Grow + (size_t)a.rowofs[m] * NC);
    const int n2 = (a.Lt + 1 - m) * NC / 2;
    for (int i = threadIdx.x; i < n2; i += PTS_THREADS)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 2 * i)), "l"(src + i) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// The block's points walk the orders together; order m's coefficient rows are
// staged in shared memory (double-buffered: the rows of m + 1 are in flight
// while m is consumed) and read as broadcasts, the next row prefetched into
// registers one degree ahead of its FMAs.  STAGE = false (degrees whose two
// row buffers exceed shared memory) reads the rows from global memory instead.
template <int NF, bool STAGE>
__global__ void __launch_bounds__(PTS_THREADS) adjoint_points_kernel(PtsArgs a) {
  constexpr int NC = 12 * NF;
  extern __shared__ __align__(16) double pts_rows[];  // 2 x (Lt + 1) x NC
  const int Lt = a.Lt;
  const size_t bufsz = (size_t)(Lt + 1) * NC;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p < a.M;
  const long long pc = live ? p : a.M - 1;
  const double x = a.xyz[3 * pc], y = a.xyz[3 * pc + 1], zr = a.xyz[3 * pc + 2];
  const double t = fmin(1.0, fmax(-1.0, zr));
  const double s = sqrt(fmax(0.0, 1.0 - t * t));
  double phi = atan2(y, x);
  if (phi < 0.0) phi += 6.283185307179586;  // np.mod(atan2, 2*pi) (favest/core.py:82)
  double out[NF][6];
#pragma unroll
  for (int b = 0; b < NF; ++b)
#pragma unroll
    for (int c = 0; c < 6; ++c) out[b][c] = 0.0;
  double seed = 0.28209479177387814;
  int se = 0;
  if (STAGE) pts_stage_rows<NC>(a, 0, pts_rows);
  for (int m = 0; m <= Lt; ++m) {
    const double* rows = STAGE ? pts_rows + (m & 1) * bufsz : a.Grow + (size_t)a.rowofs[m] * NC;
    if (STAGE) {
      pts_stage_rows<NC>(a, m + 1, pts_rows + ((m + 1) & 1) * bufsz);
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // order m's rows have landed
      __syncthreads();
    }
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
    double p2 = seed, p1 = __dmul_rn(__dmul_rn(sqrt(2 * m + 3.0), t), seed);
    int e = se;
    const double2* abm = a.ab + a.abofs[m];
    double2 gnext[NF][6];
#pragma unroll
    for (int b = 0; b < NF; ++b)
#pragma unroll
      for (int c = 0; c < 6; ++c) gnext[b][c] = reinterpret_cast<const double2*>(rows)[6 * b + c];
    double2 abn = (m + 2 <= Lt) ? __ldg(abm) : make_double2(0.0, 0.0);
    for (int l = m; l <= Lt; ++l) {
      double2 g[NF][6];
#pragma unroll
      for (int b = 0; b < NF; ++b)
#pragma unroll
        for (int c = 0; c < 6; ++c) g[b][c] = gnext[b][c];
      if (l < Lt) {
        const double2* nrow = reinterpret_cast<const double2*>(rows + (size_t)(l + 1 - m) * NC);
#pragma unroll
        for (int b = 0; b < NF; ++b)
#pragma unroll
          for (int c = 0; c < 6; ++c) gnext[b][c] = nrow[6 * b + c];
      }
      double v;
      if (l == m) {
        v = p2;
      } else if (l == m + 1) {
        v = p1;
      } else {
        const double2 abv = abn;  // (a_l, a_l * b_l)
        if (l + 1 <= Lt) abn = __ldg(abm + (l + 1 - m - 2));
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
#pragma unroll
      for (int b = 0; b < NF; ++b)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          acc[b][2 * c] = fma(v, g[b][c].x, acc[b][2 * c]);
          acc[b][2 * c + 1] = fma(v, g[b][c].y, acc[b][2 * c + 1]);
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
    if (STAGE) __syncthreads();  // buffer (m & 1) is refilled with order m + 2 next
  }
  if (!live) return;
#pragma unroll
  for (int b = 0; b < NF; ++b)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      a.T[((size_t)(a.b0 + b) * a.M + p) * 3 + c] = make_double2(out[b][2 * c], out[b][2 * c + 1]);
}

// ---------------------------------------------------------------------------
// Tensor-core form of the scattered adjoint.  For each order m the block
// computes C_m = P_m G_m with P_m[p][l] = Pbar_l^m(z_p) (points x degrees) and
// G_m[l][col] the merged coefficient rows (degrees x 12 NF columns), on
// DMMA.8x8x4: a warp owns 32 points = 4 M-tiles, k-steps are 4 degrees.  Each
// lane runs the recurrence of its own point (extended range as above); the
// four values of a k-step go through a 1 KB per-warp shared buffer into A
// fragments (lane (row r, k) reads point 8 i + r, degree k).  The rows of
// order m are staged in shared memory with a padded stride (RS = 4 mod 16:
// B-fragment reads are conflict free) and double-buffered across orders.
// After the last degree of m the accumulators (point, column pair) are rotated
// by e^{+-i m phi} of their point and added to the output accumulators; the
// +m / -m column pairs of one (field, component) sit in lanes q and q ^ 1 and
// are combined once at the end.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ptsd_nt(int nf) { return (12 * nf + 7) / 8; }
__host__ __device__ constexpr int ptsd_rs(int nf) { return ((8 * ptsd_nt(nf) + 11) / 16) * 16 + 4; }

template <int NF>
__device__ __forceinline__ void ptsd_stage_rows(const PtsArgs& a, int m, double* dst, double2* abdst) {
  constexpr int NC = 12 * NF, RS = ptsd_rs(NF);
  if (m <= a.Lt) {
    // recurrence coefficients (a_l, a_l b_l), l = m + 2 .. Lt
    const double2* abs = a.ab + a.abofs[m];
    for (int i = threadIdx.x; i < a.Lt - m - 1; i += PTS_THREADS)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(abdst + i)), "l"(abs + i) : "memory");
    const double2* src = reinterpret_cast<const double2*>(a.Grow + (size_t)a.rowofs[m] * NC);
    const int nrow = a.Lt + 1 - m;
    const int n2 = nrow * (NC / 2);
    for (int i = threadIdx.x; i < n2; i += PTS_THREADS) {
      const int r = i / (NC / 2), c = i - r * (NC / 2);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + r * RS + 2 * c)), "l"(src + i)
                   : "memory");
    }
    // zero rows up to the next multiple of 4 and the padding columns 12 NF .. 8 NT - 1
    const int nr4 = (nrow + 3) & ~3;
    for (int i = threadIdx.x; i < nr4 * (RS - NC); i += PTS_THREADS) {
      const int r = i / (RS - NC), c = NC + i % (RS - NC);
      dst[r * RS + c] = 0.0;
    }
    for (int i = threadIdx.x; i < (nr4 - nrow) * NC; i += PTS_THREADS) dst[(nrow + i / NC) * RS + i % NC] = 0.0;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int NF>
__global__ void __launch_bounds__(PTS_THREADS, NF == 1 ? 2 : 1) adjoint_points_dmma_kernel(PtsArgs a) {
  constexpr int NT = ptsd_nt(NF), RS = ptsd_rs(NF);
  extern __shared__ __align__(16) double ptsd_smem[];
  const int Lt = a.Lt;
  const int nrows4 = (Lt + 1 + 3) & ~3;
  const size_t bufsz = (size_t)nrows4 * RS + 2 * (Lt + 1);  // rows, then (a_l, a_l b_l)
  double* rowbuf = ptsd_smem;                       // 2 x bufsz
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* pbuf = ptsd_smem + 2 * bufsz + warp * 128;  // [32 points][4 degrees]
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = p < a.M;
  const long long pc = live ? p : a.M - 1;
  const double x = a.xyz[3 * pc], y = a.xyz[3 * pc + 1], zr = a.xyz[3 * pc + 2];
  const double t = fmin(1.0, fmax(-1.0, zr));
  const double s = sqrt(fmax(0.0, 1.0 - t * t));
  double phi = atan2(y, x);
  if (phi < 0.0) phi += 6.283185307179586;  // np.mod(atan2, 2*pi) (favest/core.py:82)
  const int g = lane >> 2, q = lane & 3;
  // phi of the four points this lane holds accumulators for (M-tile i, row g)
  double phi_i[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) phi_i[i] = __shfl_sync(0xffffffffu, phi, 8 * i + g);
  double out[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) out[i][j][0] = out[i][j][1] = 0.0;
  double seed = 0.28209479177387814;
  int se = 0;
  auto abuf = [&](int k) { return reinterpret_cast<double2*>(rowbuf + k * bufsz + (size_t)nrows4 * RS); };
  ptsd_stage_rows<NF>(a, 0, rowbuf, abuf(0));
  for (int m = 0; m <= Lt; ++m) {
    const double* rows = rowbuf + (m & 1) * bufsz;
    const double2* abm = abuf(m & 1);
    ptsd_stage_rows<NF>(a, m + 1, rowbuf + ((m + 1) & 1) * bufsz, abuf((m + 1) & 1));
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // order m's rows have landed
    __syncthreads();
    if (m > 0) {
      const double c = sqrt((2 * m + 1) / (2.0 * m));
      seed = __dmul_rn(__dmul_rn(-c, s), seed);
      if (fabs(seed) < 0x1p-512 && seed != 0.0) {
        seed *= 0x1p512;
        se -= XR_SHIFT;
      }
    }
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double p2 = seed, p1 = __dmul_rn(__dmul_rn(sqrt(2 * m + 3.0), t), seed);
    int e = se;
    // one recurrence step (degree m + 2 + number of steps so far), value in P units;
    // the k-step's four coefficient pairs are loaded one k-step ahead (the shared
    // memory latency otherwise sits on every step of the dependent chain)
    const double2* abp = abm;  // (a_l, a_l b_l), l = m + 2 .., staged
    auto step = [&](double2 abv) -> double {
      const double pn = fma(abv.x * t, p1, -(abv.y * p2));
      p2 = p1;
      p1 = pn;
      if (e < 0 && fabs(p1) >= 0x1p512) {
        p1 *= 0x1p-512;
        p2 *= 0x1p-512;
        e += XR_SHIFT;
      }
      return e < 0 ? xr_value(p1, e) : p1;
    };
    double2 abn[4];  // coefficients of the next k-step's plain steps
#pragma unroll
    for (int k = 0; k < 4; ++k) abn[k] = abp[k];  // (past the order's end: stale rows, never used)
    const double* brow = rows + (size_t)q * RS + g;  // B fragment row q of the k-step's four degrees
    for (int l0 = m; l0 <= Lt; l0 += 4, brow += 4 * RS) {
      // warp-uniform cases: the order's first k-step starts from the seeds, the
      // last may run past Lt; every other k-step is four plain recurrence steps
      double v[4];
      double2 ab[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) ab[k] = abn[k];
      if (l0 == m) {
        v[0] = e < 0 ? xr_value(p2, e) : p2;
        v[1] = m + 1 <= Lt ? (e < 0 ? xr_value(p1, e) : p1) : 0.0;
        abp += 2;
#pragma unroll
        for (int k = 0; k < 4; ++k) abn[k] = abp[k];
        v[2] = m + 2 <= Lt ? step(ab[0]) : 0.0;
        v[3] = m + 3 <= Lt ? step(ab[1]) : 0.0;
      } else {
        abp += 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) abn[k] = abp[k];
        if (l0 + 3 <= Lt) {
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = step(ab[k]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = l0 + k <= Lt ? step(ab[k]) : 0.0;
        }
      }
      __syncwarp();
      reinterpret_cast<double2*>(pbuf)[2 * lane] = make_double2(v[0], v[1]);
      reinterpret_cast<double2*>(pbuf)[2 * lane + 1] = make_double2(v[2], v[3]);
      __syncwarp();
      double af[4], bf[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = pbuf[(8 * i + g) * 4 + q];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = brow[8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    // rotate by e^{+i m phi} (sign 0 columns) / e^{-i m phi} (sign 1 columns) and accumulate
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double sn, cs;
      sincos(phi_i[i] * m, &sn, &cs);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int cp = 4 * j + q;  // column pair: 6 b + 2 c + sign
        const double sg = (cp & 1) ? -sn : sn;
        if ((cp & 1) && m == 0) continue;  // the -0 order is not a separate coefficient
        const double re = acc[i][j][0], im = acc[i][j][1];
        out[i][j][0] += cs * re - sg * im;
        out[i][j][1] += cs * im + sg * re;
      }
    }
    __syncthreads();  // buffer (m & 1) is refilled with order m + 2 next
  }
  // combine the +m / -m column pairs (lanes q, q ^ 1) and write T
  const long long pbase = (long long)blockIdx.x * blockDim.x + warp * 32;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double r = out[i][j][0] + __shfl_xor_sync(0xffffffffu, out[i][j][0], 1);
      const double im = out[i][j][1] + __shfl_xor_sync(0xffffffffu, out[i][j][1], 1);
      const int cp = 4 * j + q;
      const long long pt = pbase + 8 * i + g;
      if ((q & 1) == 0 && cp < 6 * NF && pt < a.M) {
        const int b = cp / 6, c = (cp % 6) >> 1;
        a.T[((size_t)(a.b0 + b) * a.M + pt) * 3 + c] = make_double2(r, im);
      }
    }
}

// ---------------------------------------------------------------------------
// Forward at weighted scattered points — the direct route of forward_favest
// (favest/scalar.py:94-105: sum_k w_k f_k conj(Y_lm(x_k)), conj(Y_lm) =
// sigma_m Pbar_l^|m|(z) e^{-i m phi}, favest/legendre.py:101-123).  Output is
// the forward Legendre row block F[tri(l, m)][col] (col 12 b + 4 c + 2 s + ri,
// s = 0: +m, s = 1: -m, Cartesian c) that cg_fwd_tile_kernel consumes, the
// same rows the grid path produces.
//
// Per order m: F_m[l][col] = sum_k Pbar_l^m(z_k) Y_k[col] with
// Y_k[(b, c, +m)] = w_k T_bc(x_k) e^{-i m phi_k} and
// Y_k[(b, c, -m)] = (-1)^m w_k T_bc(x_k) e^{+i m phi_k}: a DMMA.8x8x4 product
// with degrees as M, points as K (the reduction) and columns as N.
//
// Work item = (order m, 128-degree window, point range r).  The CTA walks its
// point range in chunks of 256 (one point per thread): each thread forms its
// point's Y row in shared memory, seeds Pbar_m^m directly in extended range
// (K_m (-s)^m by square-and-multiply, no per-order running product) and runs
// the three-term recurrence across the window, 32 degrees at a time into a
// shared P block; then warp (mi, h) contracts M-tile mi of the block over the
// chunk's points h*128 .. h*128+127 into register accumulators that live for
// the whole item.  At the end the two K halves are summed in a fixed order and
// the item's rows are written to its range slice of the partial workspace;
// fpart_reduce_kernel adds the R slices in range order (deterministic).
// ---------------------------------------------------------------------------
struct FptsArgs {
  const double* xyz;      // (M, 3) unit points
  const double* w;        // (M) weights
  long long M;
  const double2* T;       // (B_total, M, 3)
  double* Fpart;          // [R][tri(Lt)][ncol]
  long long part_stride;  // doubles per range slice
  const double2* ab;      // recurrence (a_l, a_l b_l) per order (ab_kernel)
  const long long* abofs;
  const double* seedk;    // K_m = Pbar_m^m(t) / (-s)^m
  const int2* items;      // (m, window), heaviest first
  int Lt, B_total, b0, R, ncol;
};

constexpr int FPD_THREADS = 256, FPD_CHUNK = 256, FPD_DB = 32, FPD_PS = FPD_CHUNK + 4, FPD_MT = 4;
constexpr int FPD_WIN = FPD_MT * FPD_DB;  // degrees per window

__host__ __device__ constexpr size_t fpd_smem_bytes(int nf, int Lt) {
  return ((size_t)FPD_DB * FPD_PS + (size_t)FPD_CHUNK * ptsd_rs(nf)) * sizeof(double) +
         (size_t)(Lt + 3) * sizeof(double2);  // l = m+2..Lt, plus the two-ahead prefetch
}

// Pbar_m^m(t) = (-1)^m K_m s^m as x * 2^e (e a multiple of 512, e <= 0), with
// s^m = r 2^E from square-and-multiply on frexp-normalised factors (exact range)
__device__ __forceinline__ void fpd_seed(int m, double s, double km, double& x, int& e) {
  e = 0;
  if (m == 0) {
    x = km;
    return;
  }
  if (s == 0.0) {
    x = 0.0;
    return;
  }
  int ks;
  const double f = frexp(s, &ks);
  double r = 1.0, bb = f;
  long long er = 0, eb = 0;
  for (int n = m;;) {
    int tt;
    if (n & 1) {
      r = frexp(r * bb, &tt);
      er += eb + tt;
    }
    n >>= 1;
    if (!n) break;
    bb = frexp(bb * bb, &tt);
    eb = 2 * eb + tt;
  }
  const long long E = er + (long long)ks * m;
  const double v = (m & 1) ? -km * r : km * r;
  const long long qq = E > 0 ? 0 : (-E) / XR_SHIFT;
  e = (int)(-XR_SHIFT * qq);
  x = ldexp(v, (int)(E + XR_SHIFT * qq));
}

template <int NF>
__global__ void __launch_bounds__(FPD_THREADS, NF == 1 ? 2 : 1) forward_points_dmma_kernel(FptsArgs a) {
  constexpr int NT = ptsd_nt(NF), RS = ptsd_rs(NF), NCOL = 8 * NT;
  extern __shared__ __align__(16) double fpd_smem[];
  double* Ps = fpd_smem;                                                    // [FPD_DB][FPD_PS]
  double* Ys = Ps + FPD_DB * FPD_PS;                                        // [FPD_CHUNK][RS]
  double2* abs_ = reinterpret_cast<double2*>(Ys + (size_t)FPD_CHUNK * RS);  // (a_l, a_l b_l), l = m+2..Lt
  const int item = blockIdx.x / a.R, r = blockIdx.x - item * a.R;
  const int2 it = a.items[item];
  const int m = it.x, Lt = a.Lt;
  const int lw0 = m + it.y * FPD_WIN, lw1 = min(Lt + 1, lw0 + FPD_WIN);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int mi = warp & 3, h = warp >> 2;
  for (int i = threadIdx.x; i < Lt - m - 1; i += FPD_THREADS) abs_[i] = a.ab[a.abofs[m] + i];
  const long long p_begin = a.M * r / a.R, p_end = a.M * (r + 1) / a.R;
  const double km = a.seedk[m], c1 = sqrt(2 * m + 3.0);
  const double sgm = (m & 1) ? -1.0 : 1.0;
  double acc[FPD_MT][NT][2];
#pragma unroll
  for (int j = 0; j < FPD_MT; ++j)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[j][n][0] = acc[j][n][1] = 0.0;
  __syncthreads();  // recurrence coefficients staged
  for (long long c0 = p_begin; c0 < p_end; c0 += FPD_CHUNK) {
    const long long p = c0 + threadIdx.x;
    const bool live = p < p_end;
    double t = 0.0, s = 0.0;
    double* yrow = Ys + threadIdx.x * RS;
    if (live) {
      const double x = a.xyz[3 * p], y = a.xyz[3 * p + 1], zr = a.xyz[3 * p + 2];
      t = fmin(1.0, fmax(-1.0, zr));
      s = sqrt(fmax(0.0, 1.0 - t * t));
      double phi = atan2(y, x);
      if (phi < 0.0) phi += 6.283185307179586;  // np.mod(atan2, 2*pi) (favest/core.py:82)
      const double wk = a.w[p];
      double sn, cs;
      sincos(phi * m, &sn, &cs);  // favest/legendre.py:121: exp(i * (phi * m))
#pragma unroll
      for (int b = 0; b < NF; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double2 v = a.T[((size_t)(a.b0 + b) * a.M + p) * 3 + c];
          const double vr = wk * v.x, vi = wk * v.y;
          // +m: e^{-i m phi} (w T);  -m: (-1)^m e^{+i m phi} (w T), absent at m = 0
          reinterpret_cast<double2*>(yrow)[6 * b + 2 * c] = make_double2(cs * vr + sn * vi, cs * vi - sn * vr);
          reinterpret_cast<double2*>(yrow)[6 * b + 2 * c + 1] =
              m == 0 ? make_double2(0.0, 0.0) : make_double2(sgm * (cs * vr - sn * vi), sgm * (cs * vi + sn * vr));
        }
#pragma unroll
      for (int c = 12 * NF; c < NCOL; ++c) yrow[c] = 0.0;
    } else {
#pragma unroll
      for (int c = 0; c < NCOL; ++c) yrow[c] = 0.0;
    }
    // recurrence state of this thread's point, seeded at degree m
    double p2, p1;
    int e;
    fpd_seed(m, s, km, p2, e);
    p1 = __dmul_rn(__dmul_rn(c1, t), p2);  // favest/legendre.py:66-67
    // plain recurrence step: the next degree m + 2 + (steps so far), in P units; the
    // coefficients are read two steps ahead (shared-memory latency off the chain;
    // the two reads past the order's last degree are padding, never used)
    const double2* abp = abs_ + 2;
    double2 ab0 = abs_[0], ab1 = abs_[1];
    auto step = [&]() -> double {
      const double2 abv = ab0;
      ab0 = ab1;
      ab1 = *abp++;
      const double pn = fma(abv.x * t, p1, -(abv.y * p2));
      p2 = p1;
      p1 = pn;
      if (e < 0 && fabs(p1) >= 0x1p512) {
        p1 *= 0x1p-512;
        p2 *= 0x1p-512;
        e += XR_SHIFT;
      }
      return e < 0 ? xr_value(p1, e) : p1;
    };
    for (int l = m + 2; l < lw0; ++l) step();  // degrees below this item's window
#pragma unroll
    for (int j = 0; j < FPD_MT; ++j) {
      const int d0 = lw0 + j * FPD_DB;
      if (d0 >= lw1) break;
      // warp-uniform cases: the order's first block starts from the seeds, the
      // window's last block may end early; otherwise 32 plain steps
      double* pcol = Ps + threadIdx.x;
      int k0 = 0;
      if (d0 == m) {
        pcol[0] = e < 0 ? xr_value(p2, e) : p2;
        pcol[FPD_PS] = m + 1 < lw1 ? (e < 0 ? xr_value(p1, e) : p1) : 0.0;
        k0 = 2;
      }
      if (d0 + FPD_DB <= lw1) {
#pragma unroll 4
        for (int k = k0; k < FPD_DB; ++k) pcol[k * FPD_PS] = step();
      } else {
        for (int k = k0; k < FPD_DB; ++k) pcol[k * FPD_PS] = d0 + k < lw1 ? step() : 0.0;
      }
      __syncthreads();
      if (d0 + 8 * mi < lw1) {
        const double* pa = Ps + (8 * mi + g) * FPD_PS + h * (FPD_CHUNK / 2) + q;
        const double* pb = Ys + (size_t)(h * (FPD_CHUNK / 2) + q) * RS + g;
#pragma unroll 8
        for (int ks = 0; ks < FPD_CHUNK / 8; ++ks) {
          const double af = pa[4 * ks];
          double bf[NT];
#pragma unroll
          for (int n = 0; n < NT; ++n) bf[n] = pb[(size_t)4 * ks * RS + 8 * n];
#pragma unroll
          for (int n = 0; n < NT; ++n) dmma_m8n8k4(acc[j][n][0], acc[j][n][1], af, bf[n]);
        }
      }
      __syncthreads();  // P block (and, after the last block, the Y tile) free again
    }
  }
  // sum the two point halves (h = 0 + h = 1, fixed order) and store the item's rows
  double* red = Ps;  // [4 M-tile warps][FPD_MT][NT][2][32]
  if (h == 1) {
#pragma unroll
    for (int j = 0; j < FPD_MT; ++j)
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        red[(((mi * FPD_MT + j) * NT + n) * 2 + 0) * 32 + lane] = acc[j][n][0];
        red[(((mi * FPD_MT + j) * NT + n) * 2 + 1) * 32 + lane] = acc[j][n][1];
      }
  }
  __syncthreads();
  if (h == 0) {
    double* out = a.Fpart + (size_t)r * a.part_stride;
#pragma unroll
    for (int j = 0; j < FPD_MT; ++j) {
      const int lr = lw0 + j * FPD_DB + 8 * mi + g;
      if (lr < lw1) {
        double* row = out + ((size_t)lr * (lr + 1) / 2 + m) * a.ncol;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const double v0 = acc[j][n][0] + red[(((mi * FPD_MT + j) * NT + n) * 2 + 0) * 32 + lane];
          const double v1 = acc[j][n][1] + red[(((mi * FPD_MT + j) * NT + n) * 2 + 1) * 32 + lane];
          *reinterpret_cast<double2*>(row + 8 * n + 2 * q) = make_double2(v0, v1);
        }
      }
    }
  }
}

// F = sum over the R point-range slices, in range order (bitwise reproducible)
__global__ void fpart_reduce_kernel(const double2* __restrict__ part, long long n2, int R, double2* __restrict__ F) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x) {
    double2 s = part[i];
    for (int r = 1; r < R; ++r) {
      const double2 v = part[(size_t)r * n2 + i];
      s.x += v.x;
      s.y += v.y;
    }
    F[i] = s;
  }
}

}  // namespace fv
