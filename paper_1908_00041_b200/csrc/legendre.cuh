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
// Both kernels are warp specialised.  Four producer warps (one per SMSP) run
// the normalized three-term recurrence (favest/legendre.py:66-74) one ring
// pair per lane and write Pbar tiles into shared memory directly in the
// mma.m8n8k4.f64 fragment order (XOR swizzled, bank-conflict free); the
// matching ring-data / coefficient tile, pre-arranged in fragment order in
// HBM, is bulk-copied by the TMA engine (cp.async.bulk).  Eight consumer warps
// issue DMMA.8x8x4.  Stages are handed over with mbarriers.
//
// Polar start: the plan precomputes, per (m, pair), the first degree
// l_s >= m with |Pbar_{l_s}^m| >= 2^-100 and the values at l_s, l_s + 1
// (extended-range recurrence, aux_kernels.cuh start_kernel).  Below l_s the
// values are < 2^-100 ~ 7.9e-31 (they underflow to 0/NaN in the reference for
// L >~ 1900) and are taken as exact zeros, so the hot loop needs no extended
// range arithmetic and tiles / k-steps / M-tiles that are entirely below
// their start are skipped by producers and consumers alike.
#pragma once
#include "common.cuh"

namespace fv {

constexpr int kConsumerWarps = 8;
constexpr int kProducerWarps = 4;  // one per SMSP: the recurrence chain is latency bound
constexpr int kThreads = 32 * (kConsumerWarps + kProducerWarps);

// Recurrence step in FMA form: with (a_l, c_l = a_l * b_l) precomputed,
//   P_l = a_l t P_{l-1} - c_l P_{l-2} = fma(a_l t, P_{l-1}, -(c_l P_{l-2})).
// Only the FMA is on the loop-carried chain (a_l t and c_l P_{l-2} are known one
// step early).  Rounding differs from the reference's a*(t*P1 - b*P2) by an ulp
// per step (checked against the oracle at 1e-11 relative; typically 1e-15..1e-13).
// MIXED tiles inject the polar-start values: P = A at l == l_s, B at l_s + 1; before
// l_s the state is (0, 0) and the recurrence yields exact zeros.
struct Inject {
  int ls;
  double A, B;
};

template <bool MIXED>
__device__ __forceinline__ double rec_step(double& p1, double& p2, double at, double c, int l, const Inject& in) {
  double pn = fma(at, p1, -(c * p2));
  if (MIXED) {
    pn = (l == in.ls) ? in.A : pn;
    pn = (l == in.ls + 1) ? in.B : pn;
  }
  p2 = p1;
  p1 = pn;
  return pn;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
constexpr int FWD_LB = 64;       // l rows per l-block (32 per parity)
constexpr int FWD_RC = 32;       // ring pairs per chunk (8 k-steps)
constexpr int FWD_STAGES = 5;
constexpr int FWD_PTILE = 2 * 4 * 8 * 32;  // doubles: [par][Mtile 4][ks 8][lane]

struct FwdArgs {
  const double* X;          // [m][chunk][par][ks 8][NT][32]
  double* F;                // rows tri(l, m) (l-major), 8*NT doubles each
  const int* start_l;       // [m][nPpad] polar start degree (Lt+1: never)
  const double2* start_v;   // [m][nPpad] (P_ls, P_ls+1)
  const double2* ab;        // (a_l, a_l*b_l), m-major: abofs[m] + (l - m - 2)
  const long long* abofs;
  const double* pair_t;     // [nPpad] cos(theta) of the north ring of each pair
  int Lt, nP, nPpad, nchunks, m_begin;
  int dbg;  // 0 normal; 1: consumers skip MMAs; 2: producers skip the recurrence; 3: both
};

struct StageMeta {
  int zero;     // 1: every Pbar in the tile is below the polar threshold
  int kmin[8];  // per k-step: smallest polar start among its four pairs
  int pad[7];
};

template <int NT>
struct FwdSmem {
  static constexpr int XTILE = 2 * 8 * NT * 32;
  static constexpr int STAGE = FWD_PTILE + XTILE;
  static constexpr size_t bytes(int nPx) {
    return (size_t)FWD_STAGES * STAGE * 8 + 2 * FWD_STAGES * 8 + FWD_STAGES * sizeof(StageMeta) +
           kProducerWarps * FWD_LB * 16 + (size_t)nPx * 28;
  }
};

// rows idx = 0..63 of one (l-block, chunk) tile; lane = ring pair 4s+q of the chunk.
// Coefficients are pulled from shared memory 8 steps at a time and a_l*t is
// formed off the loop-carried chain.
template <bool MIXED>
__device__ __forceinline__ void fwd_produce(double* Ps, const double2* abw, double tt, double& p1, double& p2,
                                            int lane, int l0, const Inject& in) {
  const int s = lane >> 2, q = lane & 3, sx = s & 3;
  double* bp[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) bp[g] = Ps + s * 32 + q + ((g ^ sx) << 2);
#pragma unroll
  for (int b0 = 0; b0 < FWD_LB; b0 += 8) {
    double at[8], cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 ac = abw[b0 + k];
      at[k] = ac.x * tt;
      cc[k] = ac.y;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double v = rec_step<MIXED>(p1, p2, at[k], cc[k], l0 + idx, in);
      const int par = idx & 1, rp = idx >> 1, i = rp >> 3, g = rp & 7;
      bp[g][(par * 4 + i) * 8 * 32] = v;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_fwd_kernel(FwdArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = FwdSmem<NT>;
  const int nPx = args.nchunks * FWD_RC;  // pairs covered by the forward chunks
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FWD_STAGES * SM::STAGE);
  uint64_t* empty = full + FWD_STAGES;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + FWD_STAGES);
  double2* abw_all = reinterpret_cast<double2*>(meta + FWD_STAGES);
  double* st_p1 = reinterpret_cast<double*>(abw_all + kProducerWarps * FWD_LB);
  double* st_p2 = st_p1 + nPx;
  double* st_t = st_p2 + nPx;
  int* st_ls = reinterpret_cast<int*>(st_t + nPx);

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
  for (int p = threadIdx.x; p < nPx; p += blockDim.x) {
    st_t[p] = args.pair_t[p];
    st_ls[p] = args.start_l[(size_t)m * args.nPpad + p];
    st_p1[p] = 0.0;
    st_p2[p] = 0.0;
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    const int pw = warp - kConsumerWarps;
    double2* abw = abw_all + pw * FWD_LB;
    const double2* abm = args.ab + args.abofs[m];
    for (int j = 0; j < nlb; ++j) {
      const int l0 = m + FWD_LB * j;
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // (a, a*b) for rows l0..l0+63; zero past Lt (rows become 0)
        const int l = l0 + 32 * h + lane;
        abw[32 * h + lane] = (l >= m + 2 && l <= Lt) ? abm[l - m - 2] : make_double2(0.0, 0.0);
      }
      __syncwarp();
      for (int c = pw; c < nchunks; c += kProducerWarps) {
        const int t = j * nchunks + c;
        const int stage = t % FWD_STAGES;
        const uint32_t round = t / FWD_STAGES;
        const int p = c * FWD_RC + lane;
        const double tt = st_t[p];
        Inject in;
        in.ls = st_ls[p];
        const bool before = in.ls > l0 + FWD_LB - 1;             // tile entirely below start
        const bool inject = !before && in.ls + 1 >= l0;           // start value(s) land in this tile
        const bool zero = __all_sync(0xffffffffu, before);
        const bool mixed = __any_sync(0xffffffffu, inject);
        in.A = in.B = 0.0;
        if (mixed) {
          const double2 v = args.start_v[(size_t)m * args.nPpad + p];
          in.A = v.x;
          in.B = v.y;
        }
        double p1 = st_p1[p], p2 = st_p2[p];
        // smallest polar start of the k-step (4 consecutive lanes)
        int km = min(in.ls, __shfl_xor_sync(0xffffffffu, in.ls, 1));
        km = min(km, __shfl_xor_sync(0xffffffffu, km, 2));
        mbar_wait(&empty[stage], (round & 1) ^ 1);
        double* Ps = smem + stage * SM::STAGE;
        double* Xs = Ps + FWD_PTILE;
        if (lane == 0) meta[stage].zero = zero;
        if ((lane & 3) == 0) meta[stage].kmin[lane >> 2] = km;
        if (!zero) {
          if (lane == 0) {
            asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])),
                         "r"((uint32_t)(SM::XTILE * 8))
                         : "memory");
            bulk_g2s(Xs, args.X + ((size_t)(m - args.m_begin) * nchunks + c) * SM::XTILE, SM::XTILE * 8,
                     &full[stage]);
          }
          if (args.dbg & 2) {
          } else if (mixed) {
            fwd_produce<true>(Ps, abw, tt, p1, p2, lane, l0, in);
          } else {
            fwd_produce<false>(Ps, abw, tt, p1, p2, lane, l0, in);
          }
          if (j + 1 < nlb) {
            st_p1[p] = p1;
            st_p2[p] = p2;
          }
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
    const int l0 = m + FWD_LB * j;
    const int lhi = l0 + 32 * mh + 31;  // last row of this warp's two M-tiles
    for (int c = 0; c < nchunks; ++c) {
      const int t = j * nchunks + c;
      const int stage = t % FWD_STAGES;
      const uint32_t round = t / FWD_STAGES;
      mbar_wait(&full[stage], round & 1);
      const double* Ps = smem + stage * SM::STAGE;
      const double* Xs = Ps + FWD_PTILE;
      if (!meta[stage].zero && !(args.dbg & 1)) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (meta[stage].kmin[ks] <= lhi) {
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
        }
      }
      mbar_arrive(&empty[stage]);
    }
    // epilogue for this l-block: rows l = l0 + 2*(8*i + g) + par
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
constexpr int ADJ_LC = 32;       // l values per stage (16 per parity, 4 k-steps each)
constexpr int ADJ_KS = ADJ_LC / 8;
constexpr int ADJ_RC = 128;      // ring pairs per CTA (16 M-tiles, one per producer lane)
constexpr int ADJ_MT = ADJ_RC / 8;
constexpr int ADJ_STAGES = 4;
constexpr int ADJ_PTILE = 2 * ADJ_KS * ADJ_MT * 32;  // doubles: [par][ks][Mtile][lane]

struct AdjArgs {
  const double* G;          // per m: (gofs[m] + lc) * GTILE, [par][ks ADJ_KS][NT][32]
  const long long* gofs;
  double2* S;               // spectrum [comp][field][ring][n_phi] (all fields)
  const int* start_l;
  const double2* start_v;
  const double2* ab;
  const long long* abofs;
  const double* pair_t;
  const int* pair_n;        // north ring of each pair (-1: padding)
  const int* pair_s;        // south ring (-1: unpaired)
  int Lt, nP, nPpad, nrc, n_phi, n_theta, B_total, b0, nfields, m_begin;
  int dbg;
};

template <int NT>
struct AdjSmem {
  static constexpr int GTILE = 2 * ADJ_KS * NT * 32;
  static constexpr int STAGE = ADJ_PTILE + GTILE;
  static constexpr size_t bytes() {
    return (size_t)ADJ_STAGES * STAGE * 8 + 2 * ADJ_STAGES * 8 + kProducerWarps * ADJ_LC * 16;
  }
};

__device__ __forceinline__ int adj_swz(int g, int q, int i) {
  return (g << 2) + (q ^ ((g >> 2) | ((i & 1) << 1)));
}

// l values idx = 0..ADJ_LC-1 of one stage for the lane's pair (M-tile i, row g)
template <bool MIXED>
__device__ __forceinline__ void adj_produce(double* Ps, const double2* abw, double tt, double& p1, double& p2,
                                            int i, int g, int l0, const Inject& in) {
  const int cx = (g >> 2) | ((i & 1) << 1);
  double* bp[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) bp[q] = Ps + i * 32 + (g << 2) + (q ^ cx);
#pragma unroll
  for (int b0 = 0; b0 < ADJ_LC; b0 += 8) {
    double at[8], cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 ac = abw[b0 + k];
      at[k] = ac.x * tt;
      cc[k] = ac.y;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double v = rec_step<MIXED>(p1, p2, at[k], cc[k], l0 + idx, in);
      const int par = idx & 1, kk = idx >> 1, ks = kk >> 2, q = kk & 3;
      bp[q][(par * ADJ_KS + ks) * ADJ_MT * 32] = v;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_adj_kernel(AdjArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = AdjSmem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ADJ_STAGES * SM::STAGE);
  uint64_t* empty = full + ADJ_STAGES;
  double2* abw_all = reinterpret_cast<double2*>(empty + ADJ_STAGES);

  const int m = args.m_begin + blockIdx.x / args.nrc;
  const int rc = blockIdx.x % args.nrc;
  const int Lt = args.Lt;
  const int nrows = Lt + 1 - m;
  const int nlc = (nrows + ADJ_LC - 1) / ADJ_LC;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ADJ_STAGES; ++s) {
      mbar_init(&full[s], 32 * kProducerWarps);
      mbar_init(&empty[s], 32 * kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp >= kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    const int pw = warp - kConsumerWarps;
    double2* abw = abw_all + pw * ADJ_LC;
    const int rho = 32 * pw + lane;            // pair within the CTA's chunk
    const int p = rc * ADJ_RC + rho;
    const int i = rho >> 3, g = rho & 7;
    const double tt = args.pair_t[p];
    Inject in;
    in.ls = args.start_l[(size_t)m * args.nPpad + p];
    {
      const double2 v = args.start_v[(size_t)m * args.nPpad + p];
      in.A = v.x;
      in.B = v.y;
    }
    double p1 = 0.0, p2 = 0.0;
    const double2* abm = args.ab + args.abofs[m];
    const double* Gm = args.G + (size_t)args.gofs[m] * SM::GTILE;
    for (int lc = 0; lc < nlc; ++lc) {
      const int stage = lc % ADJ_STAGES;
      const uint32_t round = lc / ADJ_STAGES;
      const int l0 = m + ADJ_LC * lc;
      const bool before = in.ls > l0 + ADJ_LC - 1;
      const bool zero = __all_sync(0xffffffffu, before);
      const bool mixed = __any_sync(0xffffffffu, !before && in.ls + 1 >= l0);
      if (!zero) {
        __syncwarp();
        const int l = l0 + lane;
        abw[lane] = (l >= m + 2 && l <= Lt) ? abm[l - m - 2] : make_double2(0.0, 0.0);
        __syncwarp();
      }
      mbar_wait(&empty[stage], (round & 1) ^ 1);
      double* Ps = smem + stage * SM::STAGE;
      double* Gs = Ps + ADJ_PTILE;
      if (pw == 0 && lane == 0) {
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])),
                     "r"((uint32_t)(SM::GTILE * 8))
                     : "memory");
        bulk_g2s(Gs, Gm + (size_t)lc * SM::GTILE, SM::GTILE * 8, &full[stage]);
      }
      // all-zero warps write nothing: the consumers skip their M-tiles (polar start)
      if (zero || (args.dbg & 2)) {
      } else if (mixed) {
        adj_produce<true>(Ps, abw, tt, p1, p2, i, g, l0, in);
      } else {
        adj_produce<false>(Ps, abw, tt, p1, p2, i, g, l0, in);
      }
      mbar_arrive(&full[stage]);
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  // warp (par, mq): M-tiles 4mq..4mq+3 (32 pairs) x all NT n-tiles of parity par
  const int par = warp >> 2;
  const int mq = warp & 3;
  const int g = lane >> 2, q = lane & 3;
  // first degree at which each of the warp's M-tiles has a pair above the polar threshold
  int mt_start[4];
  {
    int v = args.start_l[(size_t)m * args.nPpad + rc * ADJ_RC + 32 * mq + lane];
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) mt_start[ii] = __shfl_sync(0xffffffffu, v, 8 * ii);
  }
  double acc[4][NT][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int lc = 0; lc < nlc; ++lc) {
    const int stage = lc % ADJ_STAGES;
    const uint32_t round = lc / ADJ_STAGES;
    const int lhi = m + ADJ_LC * lc + ADJ_LC - 1;
    mbar_wait(&full[stage], round & 1);
    const double* Ps = smem + stage * SM::STAGE;
    const double* Gs = Ps + ADJ_PTILE;
    bool act[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) act[ii] = mt_start[ii] <= lhi;
    if (!(args.dbg & 1) && (act[0] || act[1] || act[2] || act[3])) {
#pragma unroll
      for (int ks = 0; ks < ADJ_KS; ++ks) {
        double a[4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const int i = 4 * mq + ii;
          a[ii] = act[ii] ? Ps[((par * ADJ_KS + ks) * ADJ_MT + i) * 32 + adj_swz(g, q, i)] : 0.0;
        }
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) {
          const double b = Gs[((par * ADJ_KS + ks) * NT + jn) * 32 + lane];
#pragma unroll
          for (int ii = 0; ii < 4; ++ii)
            if (act[ii]) dmma_m8n8k4(acc[ii][jn][0], acc[ii][jn][1], a[ii], b);
        }
      }
    }
    mbar_arrive(&empty[stage]);
  }

  // epilogue: combine parities through shared memory (odd warps publish, even warps finish)
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps));
  double* xch = smem;  // reuse stage buffers: [mq][ii][jn][lane][2]
  if (par == 1) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        double* d = xch + ((size_t)((mq * 4 + ii) * NT + jn) * 32 + lane) * 2;
        d[0] = acc[ii][jn][0];
        d[1] = acc[ii][jn][1];
      }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps));
  if (par == 0 && rc * ADJ_RC + 32 * mq < args.nP) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int rho = (4 * mq + ii) * 8 + g;
      const int p = rc * ADJ_RC + rho;
      const int rn = args.pair_n[p];
      const int rs = args.pair_s[p];
      if (rn < 0) continue;
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        const double* d = xch + ((size_t)((mq * 4 + ii) * NT + jn) * 32 + lane) * 2;
        const int ser = (jn * 8 + 2 * q) >> 1;  // 6*field + 2*comp + sign
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
