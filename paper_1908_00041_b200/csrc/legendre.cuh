// Per-order associated-Legendre contraction kernels (the hot path).
//
// Forward (analysis), favest/scalar.py:146-154 restated per order m >= 0 with
// equatorial folding:
//   F[l, col] = sum_{pairs p} Pbar_l^m(t_p) * X_{par(l-m)}[p, col]
// Adjoint (synthesis), favest/scalar.py:170-179:
//   E/O[p, col] = sum_{l: par(l-m)} Pbar_l^m(t_p) * G[l, col]
//   north = E + O, south = E - O.
//
// Columns: col = 12*field + 4*component + 2*sign + re/im (sign 0: +m, 1: -m);
// 8-column n-tiles, NT of them per launch (<= 4 fields per launch).
//
// Both kernels: one CTA owns one order m (forward) or one (m, 64-pair chunk)
// (adjoint).  Two producer warps run the normalized three-term recurrence
// (favest/legendre.py:60-74, identical operation order, extended range) one
// ring pair per lane and write Pbar tiles into shared memory directly in the
// mma.m8n8k4.f64 fragment order (XOR-swizzled, bank-conflict free); lane 0 of
// the producer also bulk-copies the matching ring-data / coefficient tile
// (pre-arranged in fragment order in HBM) with cp.async.bulk.  Eight consumer
// warps issue DMMA.8x8x4.  Stages are handed over with mbarriers.
#pragma once
#include "common.cuh"

namespace fv {

constexpr int kConsumerWarps = 8;
constexpr int kProducerWarps = 2;
constexpr int kThreads = 32 * (kConsumerWarps + kProducerWarps);

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
constexpr int FWD_LB = 64;       // l rows per l-block (32 per parity)
constexpr int FWD_RC = 32;       // ring pairs per chunk (8 k-steps)
constexpr int FWD_STAGES = 4;
constexpr int FWD_PTILE = 2 * 4 * 8 * 32;  // doubles: [par][Mtile 4][ks 8][lane]

struct FwdArgs {
  const double* X;          // [m][chunk][par][ks 8][NT][32]
  double* F;                // rows tri(l, m) (l-major), 8*NT doubles each
  const double* seed_x;     // [m][nPpad]
  const int* seed_e;        // [m][nPpad]
  const double2* ab;        // recurrence (a_l, b_l), m-major: abofs[m] + (l - m - 2)
  const long long* abofs;
  const double* pair_t;     // [nPpad] cos(theta) of the north ring of each pair
  int Lt, nPpad, nchunks, m_begin;
};

template <int NT>
struct FwdSmem {
  static constexpr int XTILE = 2 * 8 * NT * 32;
  static constexpr int STAGE = FWD_PTILE + XTILE;
  static constexpr size_t bytes(int nPpad) {
    return (size_t)FWD_STAGES * STAGE * 8 + 2 * FWD_STAGES * 8 + (size_t)nPpad * 24;
  }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_fwd_kernel(FwdArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = FwdSmem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FWD_STAGES * SM::STAGE);
  uint64_t* empty = full + FWD_STAGES;
  double* st_p1 = reinterpret_cast<double*>(empty + FWD_STAGES);
  double* st_p2 = st_p1 + args.nPpad;
  int* st_e = reinterpret_cast<int*>(st_p2 + args.nPpad);

  const int m = args.m_begin + blockIdx.x;
  const int Lt = args.Lt;
  const int nrows = Lt + 1 - m;
  const int nlb = (nrows + FWD_LB - 1) / FWD_LB;
  const int nchunks = args.nchunks;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < FWD_STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], 32 * kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    const int pw = warp - kConsumerWarps;
    const double sq = sqrt(2 * m + 3.0);
    const double2* abm = args.ab + args.abofs[m];
    for (int j = 0; j < nlb; ++j) {
      const int l0 = m + FWD_LB * j;
      // this warp's recurrence coefficients for rows l0..l0+63 (2 per lane)
      double2 abr0 = make_double2(0.0, 0.0), abr1 = make_double2(0.0, 0.0);
      {
        int la = l0 + lane, lb = l0 + 32 + lane;
        if (la >= m + 2 && la <= Lt) abr0 = abm[la - m - 2];
        if (lb >= m + 2 && lb <= Lt) abr1 = abm[lb - m - 2];
      }
      for (int c = pw; c < nchunks; c += kProducerWarps) {
        const int t = j * nchunks + c;
        const int stage = t % FWD_STAGES;
        const uint32_t round = t / FWD_STAGES;
        mbar_wait(&empty[stage], (round & 1) ^ 1);
        double* Ps = smem + stage * SM::STAGE;
        double* Xs = Ps + FWD_PTILE;
        if (lane == 0) {
          asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])),
                       "r"((uint32_t)(SM::XTILE * 8))
                       : "memory");
          bulk_g2s(Xs, args.X + ((size_t)(m - args.m_begin) * nchunks + c) * SM::XTILE,
                   SM::XTILE * 8, &full[stage]);
        }
        const int p = c * FWD_RC + lane;
        const double tt = args.pair_t[p];
        double p1, p2;
        int e;
        if (j == 0) {
          p2 = args.seed_x[(size_t)m * args.nPpad + p];
          e = args.seed_e[(size_t)m * args.nPpad + p];
          p1 = __dmul_rn(__dmul_rn(sq, tt), p2);
        } else {
          p1 = st_p1[p];
          p2 = st_p2[p];
          e = st_e[p];
        }
        const int s = lane >> 2, q = lane & 3;
        const bool scaled = __any_sync(0xffffffffu, e < 0);
#pragma unroll 8
        for (int idx = 0; idx < FWD_LB; ++idx) {
          const int l = l0 + idx;
          double v;
          if (j == 0 && idx < 2) {
            v = (idx == 0) ? p2 : p1;
          } else {
            const double2 abv = (idx < 32) ? make_double2(__shfl_sync(0xffffffffu, abr0.x, idx),
                                                          __shfl_sync(0xffffffffu, abr0.y, idx))
                                           : make_double2(__shfl_sync(0xffffffffu, abr1.x, idx - 32),
                                                          __shfl_sync(0xffffffffu, abr1.y, idx - 32));
            // favest/legendre.py:72-74: a * (t * P_{l-1} - b * P_{l-2}), no contraction
            const double pn = __dmul_rn(abv.x, __dsub_rn(__dmul_rn(tt, p1), __dmul_rn(abv.y, p2)));
            p2 = p1;
            p1 = pn;
            if (scaled && e < 0 && fabs(p1) >= 0x1p512) {
              p1 *= 0x1p-512;
              p2 *= 0x1p-512;
              e += XR_SHIFT;
            }
            v = p1;
          }
          if (scaled) v = xr_value(v, e);
          if (l > Lt) v = 0.0;
          const int par = idx & 1, rp = idx >> 1, i = rp >> 3, g = rp & 7;
          Ps[((par * 4 + i) * 8 + s) * 32 + ((g ^ (s & 3)) << 2) + q] = v;
        }
        if (j + 1 < nlb) {
          st_p1[p] = p1;
          st_p2[p] = p2;
          st_e[p] = e;
        }
        mbar_arrive(&full[stage]);
      }
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  constexpr int NTW = (NT + 1) / 2;
  const int par = warp >> 2;
  const int mh = (warp >> 1) & 1;
  const int nh = warp & 1;
  const int nt0 = nh * NTW;
  const int g = lane >> 2, q = lane & 3;
  const int ncolF = 8 * NT;
  double acc[2][NTW][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NTW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int j = 0; j < nlb; ++j) {
    for (int c = 0; c < nchunks; ++c) {
      const int t = j * nchunks + c;
      const int stage = t % FWD_STAGES;
      const uint32_t round = t / FWD_STAGES;
      mbar_wait(&full[stage], round & 1);
      const double* Ps = smem + stage * SM::STAGE;
      const double* Xs = Ps + FWD_PTILE;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int sw = ((g ^ (ks & 3)) << 2) + q;
        const double a0 = Ps[((par * 4 + 2 * mh + 0) * 8 + ks) * 32 + sw];
        const double a1 = Ps[((par * 4 + 2 * mh + 1) * 8 + ks) * 32 + sw];
#pragma unroll
        for (int jn = 0; jn < NTW; ++jn) {
          if (nt0 + jn < NT) {
            const double b = Xs[((par * 8 + ks) * NT + nt0 + jn) * 32 + lane];
            dmma_m8n8k4(acc[0][jn][0], acc[0][jn][1], a0, b);
            dmma_m8n8k4(acc[1][jn][0], acc[1][jn][1], a1, b);
          }
        }
      }
      mbar_arrive(&empty[stage]);
    }
    // epilogue for this l-block: rows l = l0 + 2*(8*i + g) + par
    const int l0 = m + FWD_LB * j;
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int i = 2 * mh + ii;
      const int l = l0 + 2 * (8 * i + g) + par;
      if (l <= Lt) {
        double* row = args.F + ((size_t)l * (l + 1) / 2 + m) * ncolF;
#pragma unroll
        for (int jn = 0; jn < NTW; ++jn) {
          if (nt0 + jn < NT) {
            *reinterpret_cast<double2*>(row + (nt0 + jn) * 8 + 2 * q) =
                make_double2(acc[ii][jn][0], acc[ii][jn][1]);
          }
        }
      }
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) acc[ii][jn][0] = acc[ii][jn][1] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// adjoint
// ---------------------------------------------------------------------------
constexpr int ADJ_LC = 64;       // l values per stage (32 per parity, 8 k-steps each)
constexpr int ADJ_RC = 64;       // ring pairs per CTA (8 M-tiles)
constexpr int ADJ_STAGES = 3;
constexpr int ADJ_PTILE = 2 * 8 * 8 * 32;  // doubles: [par][ks 8][Mtile 8][lane]

struct AdjArgs {
  const double* G;          // per m: (gofs[m] + lc) * GTILE, [par][ks 8][NT][32]
  const long long* gofs;
  double2* S;               // spectrum [comp][field][ring][n_phi] (all fields)
  const double* seed_x;
  const int* seed_e;
  const double2* ab;
  const long long* abofs;
  const double* pair_t;
  const int* pair_n;        // north ring of each pair (-1: padding)
  const int* pair_s;        // south ring (-1: unpaired)
  int Lt, nPpad, nrc, n_phi, n_theta, B_total, b0, nfields, m_begin;
};

template <int NT>
struct AdjSmem {
  static constexpr int GTILE = 2 * 8 * NT * 32;
  static constexpr int STAGE = ADJ_PTILE + GTILE;
  static constexpr size_t bytes() { return (size_t)ADJ_STAGES * STAGE * 8 + 2 * ADJ_STAGES * 8; }
};

__device__ __forceinline__ int adj_swz(int g, int q, int i) {
  return (g << 2) + (q ^ ((g >> 2) | ((i & 1) << 1)));
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_adj_kernel(AdjArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = AdjSmem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ADJ_STAGES * SM::STAGE);
  uint64_t* empty = full + ADJ_STAGES;

  const int m = args.m_begin + blockIdx.x / args.nrc;
  const int rc = blockIdx.x % args.nrc;
  const int Lt = args.Lt;
  const int nrows = Lt + 1 - m;
  const int nlc = (nrows + ADJ_LC - 1) / ADJ_LC;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ADJ_STAGES; ++s) {
      mbar_init(&full[s], 64);
      mbar_init(&empty[s], 32 * kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    const int pw = warp - kConsumerWarps;
    const int rho = 32 * pw + lane;            // pair within the CTA's chunk
    const int p = rc * ADJ_RC + rho;
    const int i = rho >> 3, g = rho & 7;
    const double tt = args.pair_t[p];
    double p2 = args.seed_x[(size_t)m * args.nPpad + p];
    int e = args.seed_e[(size_t)m * args.nPpad + p];
    double p1 = __dmul_rn(__dmul_rn(sqrt(2 * m + 3.0), tt), p2);
    const double2* abm = args.ab + args.abofs[m];
    const double* Gm = args.G + (size_t)args.gofs[m] * SM::GTILE;
    for (int lc = 0; lc < nlc; ++lc) {
      const int stage = lc % ADJ_STAGES;
      const uint32_t round = lc / ADJ_STAGES;
      mbar_wait(&empty[stage], (round & 1) ^ 1);
      double* Ps = smem + stage * SM::STAGE;
      double* Gs = Ps + ADJ_PTILE;
      if (pw == 0 && lane == 0) {
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])),
                     "r"((uint32_t)(SM::GTILE * 8))
                     : "memory");
        bulk_g2s(Gs, Gm + (size_t)lc * SM::GTILE, SM::GTILE * 8, &full[stage]);
      }
      const int l0 = m + ADJ_LC * lc;
      double2 abr0 = make_double2(0.0, 0.0), abr1 = make_double2(0.0, 0.0);
      {
        int la = l0 + lane, lb = l0 + 32 + lane;
        if (la >= m + 2 && la <= Lt) abr0 = abm[la - m - 2];
        if (lb >= m + 2 && lb <= Lt) abr1 = abm[lb - m - 2];
      }
      const bool scaled = __any_sync(0xffffffffu, e < 0);
#pragma unroll 8
      for (int idx = 0; idx < ADJ_LC; ++idx) {
        const int l = l0 + idx;
        double v;
        if (lc == 0 && idx < 2) {
          v = (idx == 0) ? p2 : p1;
        } else {
          const double2 abv = (idx < 32) ? make_double2(__shfl_sync(0xffffffffu, abr0.x, idx),
                                                        __shfl_sync(0xffffffffu, abr0.y, idx))
                                         : make_double2(__shfl_sync(0xffffffffu, abr1.x, idx - 32),
                                                        __shfl_sync(0xffffffffu, abr1.y, idx - 32));
          const double pn = __dmul_rn(abv.x, __dsub_rn(__dmul_rn(tt, p1), __dmul_rn(abv.y, p2)));
          p2 = p1;
          p1 = pn;
          if (scaled && e < 0 && fabs(p1) >= 0x1p512) {
            p1 *= 0x1p-512;
            p2 *= 0x1p-512;
            e += XR_SHIFT;
          }
          v = p1;
        }
        if (scaled) v = xr_value(v, e);
        if (l > Lt) v = 0.0;
        const int par = idx & 1, k = idx >> 1, ks = k >> 2, q = k & 3;
        Ps[((par * 8 + ks) * 8 + i) * 32 + adj_swz(g, q, i)] = v;
      }
      mbar_arrive(&full[stage]);
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  constexpr int NTW = (NT + 1) / 2;
  const int par = warp >> 2;
  const int mh = (warp >> 1) & 1;
  const int nh = warp & 1;
  const int nt0 = nh * NTW;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][NTW][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NTW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int lc = 0; lc < nlc; ++lc) {
    const int stage = lc % ADJ_STAGES;
    const uint32_t round = lc / ADJ_STAGES;
    mbar_wait(&full[stage], round & 1);
    const double* Ps = smem + stage * SM::STAGE;
    const double* Gs = Ps + ADJ_PTILE;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      double a[4];
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = 4 * mh + ii;
        a[ii] = Ps[((par * 8 + ks) * 8 + i) * 32 + adj_swz(g, q, i)];
      }
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) {
        if (nt0 + jn < NT) {
          const double b = Gs[((par * 8 + ks) * NT + nt0 + jn) * 32 + lane];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii) dmma_m8n8k4(acc[ii][jn][0], acc[ii][jn][1], a[ii], b);
        }
      }
    }
    mbar_arrive(&empty[stage]);
  }

  // epilogue: combine parities through shared memory (odd warps publish, even warps finish)
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps));
  double* xch = smem;  // reuse stage buffers: [mh][nh][ii][jn][lane][2]
  const int slot = ((mh * 2 + nh) * 4) * NTW;
  if (par == 1) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) {
        double* d = xch + ((size_t)(slot + ii * NTW + jn) * 32 + lane) * 2;
        d[0] = acc[ii][jn][0];
        d[1] = acc[ii][jn][1];
      }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps));
  if (par == 0) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int rho = (4 * mh + ii) * 8 + g;
      const int p = rc * ADJ_RC + rho;
      const int rn = args.pair_n[p];
      const int rs = args.pair_s[p];
      if (rn < 0) continue;
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) {
        if (nt0 + jn >= NT) continue;
        const double* d = xch + ((size_t)(slot + ii * NTW + jn) * 32 + lane) * 2;
        const int ser = ((nt0 + jn) * 8 + 2 * q) >> 1;  // 6*field + 2*comp + sign
        const int b = ser / 6, comp = (ser % 6) >> 1, sgn = ser & 1;
        if (b >= args.nfields) continue;
        if (sgn == 1 && m == 0) continue;
        const int bin = sgn ? (args.n_phi - m) % args.n_phi : m;
        const double er = acc[ii][jn][0], ei = acc[ii][jn][1];
        const double orr = d[0], oi = d[1];
        const size_t base = ((size_t)comp * args.B_total + args.b0 + b) * args.n_theta;
        args.S[(base + rn) * args.n_phi + bin] = make_double2(er + orr, ei + oi);
        if (rs >= 0) args.S[(base + rs) * args.n_phi + bin] = make_double2(er - orr, ei - oi);
      }
    }
  }
}

}  // namespace fv
