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
// forward columns are the Cartesian components x, y, z (the U/V/W combos are
// formed in the CG stage), adjoint columns the merged g^X, g^Y, g^Z;
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
#ifndef FV_PRODUCERS_FIRST
#define FV_PRODUCERS_FIRST 0
#endif
// warp roles: producers take warps 0..3 (one per SMSP) when FV_PRODUCERS_FIRST,
// otherwise the last four warps; the issue arbiter's warp ordering decides how
// the producer's FP64 ops interleave with the consumers' DMMAs.
__device__ __forceinline__ bool is_producer(int warp) {
  return FV_PRODUCERS_FIRST ? warp < kProducerWarps : warp >= kConsumerWarps;
}
__device__ __forceinline__ int producer_index(int warp) {
  return FV_PRODUCERS_FIRST ? warp : warp - kConsumerWarps;
}
__device__ __forceinline__ int consumer_index(int warp) {
  return FV_PRODUCERS_FIRST ? warp - kProducerWarps : warp;
}

// Block-rescaled recurrence (two FP64 ops per step, one on the loop-carried
// chain): inside 32-degree blocks P_l = gamma_l R_l with
//   R_l = fma(t, R_{l-1}, -(d_l R_{l-2}))
// (d_l, gamma_l from aux_kernels.cuh dg_kernel); the state is converted back to
// P at each block end.  gamma is folded into the consumers instead of the
// producer: the forward scales its output rows by gamma_l, the adjoint's
// coefficient tiles are pre-scaled by gamma_l (cg_adj_kernel).  The producer
// shares the SM sub-partition's FP64 datapath with the DMMA warps, so its op
// count per step bounds how far ahead of them it can run.  Rounding differs from
// the reference's a*(t*P1 - b*P2) at the ulp level per step (checked against the
// oracle at 1e-11 relative; typically 1e-15..1e-13).
// MIXED tiles inject the polar-start values (pre-divided by gamma): R = A at
// l == l_s, B at l_s + 1; before l_s the state is (0, 0) and stays exactly zero.
struct Inject {
  int ls;
  double A, B;
};

template <bool MIXED>
__device__ __forceinline__ double rec_step(double& p1, double& p2, double tt, double d, int l, const Inject& in) {
  double pn = fma(tt, p1, -(d * p2));
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

struct __align__(16) StageMeta {
  int kmin[8];  // per k-step: smallest polar start among its four pairs (16-byte aligned for LDS.128)
  int zero;     // 1: every Pbar in the tile is below the polar threshold
  int pad[7];
};

struct FwdArgs {
  const double* X;          // [m][chunk][par][ks 8][NT][n_hi 2][k 4][n_lo 4]
  double* F;                // rows tri(l, m) (l-major), 8*NT doubles each
  const int* start_l;       // [m][nPpad] polar start degree (Lt+1: never)
  const double2* start_v;   // [m][nPpad] (P_ls, P_ls+1)
  const double2* dg;        // (d_l, gamma_l), m-major: dgofs[m] + (l - m)
  const long long* dgofs;
  const double* pair_t;     // [nPpad] cos(theta) of the north ring of each pair
  int Lt, nP, nPpad, nchunks, m_begin;
  // timing isolation (FV_DEBUG_MODE): 1 consumers skip MMAs, 2 producers skip the recurrence, 4 no adjoint
  // epilogue, 8 single-field consumers skip their fragment loads, 32 one elected mbarrier arrival per warp
  int dbg;
  int m_count;  // orders m_begin .. m_begin + m_count - 1 (persistent CTAs walk them)
  long long* trace;  // optional pipeline timeline of CTA trace_cta (clock64 stamps), normally null
  int trace_cta;
  // table mode (plan-time Legendre tiles, ptab_fwd_kernel): null -> on-the-fly producer
  const double* ptab;         // [tile][FWD_PTILE], tile = tofs[m] + j * nchunks + c
  const StageMeta* mtab;
  const long long* tofs;
  // per (order, chunk): smallest polar start of the chunk's 32 pairs (plan-time);
  // the leading chunks of an l-block whose start lies past the block are skipped
  // by producers and consumers alike (no pipeline stage for an all-zero tile)
  const int* cmin;
  // several 4-field groups in one launch (small problems: more CTAs per launch):
  // CTA b works on group b % ngroups, X / F of group g at + g * x_gstride / f_gstride
  int ngroups;
  long long x_gstride, f_gstride;
  // pair-chunk split (launches with few orders: the order-sharded chunks): split s
  // of ksplit contracts the chunks c = s (mod ksplit) of every order into its own
  // partial F buffer (s = 0: F, s > 0: Fx + (s - 1) * f_gstride); the forward CG
  // adds them in split order
  int ksplit;
  double* Fx;
  // legendre_fwd2_kernel: plan-time recurrence state (P_{l0-1}, P_{l0-2}) of every pair at every
  // tile start (fseed_kernel), [tofs[m] + j * nchunks + c][lane]; null -> legendre_fwd_kernel
  const double2* seed;
  // real k-steps (groups of four pairs) of the last, padded chunk: ceil((nP - 32 (nchunks - 1)) / 4)
  int klast;
};

// chunk starts of one order held across the warp (chunk 32 g + lane in v[g])
struct ChunkStarts {
  int v[4];
  int ng;  // 0: no skipping (more than 128 chunks)
};

__device__ __forceinline__ ChunkStarts load_chunk_starts(const int* cmin_m, int nchunks, int lane, int split = 0,
                                                         int S = 1) {
  // the chunks of one split: u = 0 .. nu-1 is chunk split + S u
  const int nu = (nchunks - split + S - 1) / S;
  ChunkStarts cs;
  cs.ng = nu <= 128 ? (nu + 31) / 32 : 0;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int u = 32 * g + lane;
    cs.v[g] = (g < cs.ng && u < nu) ? __ldg(&cmin_m[split + S * u]) : 0x7fffffff;
  }
  return cs;
}

// first chunk of the l-block [l0, l0 + FWD_LB) with a started pair (chunks before it are all-zero tiles)
// (a pair that never starts has l_s = Lt + 1: the bound is clamped to Lt, or every chunk of an
// order's last l-block, whose padding rows reach past Lt + 1, would count as live)
__device__ __forceinline__ int first_live_chunk(const ChunkStarts& cs, int l0, int Lt, int nchunks) {
  if (cs.ng == 0) return 0;
  const int lhi = min(l0 + FWD_LB - 1, Lt);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (g >= cs.ng) break;
    const unsigned b = __ballot_sync(0xffffffffu, cs.v[g] <= lhi);
    if (b) return min(32 * g + __ffs(b) - 1, nchunks);
  }
  return nchunks;
}



template <int NT>
struct FwdSmem {
  static constexpr int XTILE = 2 * 8 * NT * 32;
  static constexpr int STAGE = FWD_PTILE + XTILE;
  // K-split consumers (NT <= 2): partial sums of k-quarters 1..3 [par][3][Mtile 4][NT][2][lane]
  static constexpr int KRED = NT <= 2 ? 2 * 3 * 4 * NT * 2 * 32 : 0;
  static constexpr size_t bytes(int nPx) {
    return (size_t)FWD_STAGES * STAGE * 8 + 2 * FWD_STAGES * 8 + 16 + FWD_STAGES * sizeof(StageMeta) +
           kProducerWarps * FWD_LB * 16 + (size_t)nPx * 28 + (size_t)KRED * 8;
  }
};

// rows idx = 0..63 of one (l-block, chunk) tile; lane = ring pair 4s+q of the chunk.
// (d, gamma) for the 64 rows are staged in shared memory and pulled 8 at a time;
// rows 31 and 63 end a 32-degree block: the state goes back to P units there.
template <bool MIXED, bool SCALE = false>
__device__ __forceinline__ void fwd_produce(double* Ps, const double2* dgw, double tt, double& p1, double& p2,
                                            int lane, int l0, const Inject& in) {
  const int s = lane >> 2, q = lane & 3, sx = s & 3;
  double* bp[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) bp[g] = Ps + s * 32 + q + ((g ^ sx) << 2);
#pragma unroll
  for (int b0 = 0; b0 < FWD_LB; b0 += 8) {
    double dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[k] = dgw[b0 + k].x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double v = rec_step<MIXED>(p1, p2, tt, dd[k], l0 + idx, in);
      const int par = idx & 1, rp = idx >> 1, i = rp >> 3, g = rp & 7;
      bp[g][(par * 4 + i) * 8 * 32] = SCALE ? v * dgw[idx].y : v;  // SCALE: Pbar itself (plan tables)
      if ((idx & 31) == 31) {
        p1 *= dgw[idx].y;
        p2 *= dgw[idx - 1].y;
      }
    }
  }
}

// Per-CTA producer state of the forward (one order m): pair cos(theta), polar
// start, recurrence state carried across l-blocks.
struct FwdState {
  double* p1;
  double* p2;
  const double* t;
  const int* ls;
};

struct TileClass {
  bool zero, mixed;
  int km;  // smallest polar start of the lane's k-step
};

__device__ __forceinline__ TileClass fwd_classify_ls(int ls, int l0) {
  TileClass tc;
  const bool before = ls > l0 + FWD_LB - 1;          // tile entirely below start
  const bool inject = !before && ls + 1 >= l0;        // start value(s) land in this tile
  tc.zero = __all_sync(0xffffffffu, before);
  tc.mixed = __any_sync(0xffffffffu, inject);
  int km = min(ls, __shfl_xor_sync(0xffffffffu, ls, 1));
  tc.km = min(km, __shfl_xor_sync(0xffffffffu, km, 2));
  return tc;
}

__device__ __forceinline__ TileClass fwd_classify(const FwdState& st, int p, int l0, int lane) {
  return fwd_classify_ls(st.ls[p], l0);
}

// rows of one (l-block j, chunk c) tile into Ps (shared or global), state update
template <bool SCALE = false>
__device__ __forceinline__ void fwd_compute(const FwdArgs& args, const FwdState& st, const TileClass& tc, double* Ps,
                                            const double2* abw, int m, int j, int nlb, int p, int l0, int lane) {
  Inject in;
  in.ls = st.ls[p];
  in.A = in.B = 0.0;
  if (tc.mixed) {
    const double2 v = args.start_v[(size_t)m * args.nPpad + p];
    in.A = v.x;
    in.B = v.y;
  }
  double p1 = st.p1[p], p2 = st.p2[p];
  const double tt = st.t[p];
  if (tc.mixed) fwd_produce<true, SCALE>(Ps, abw, tt, p1, p2, lane, l0, in);
  else fwd_produce<false, SCALE>(Ps, abw, tt, p1, p2, lane, l0, in);
  if (j + 1 < nlb) {
    st.p1[p] = p1;
    st.p2[p] = p2;
  }
}

__device__ __forceinline__ void fwd_stage_coefs(double2* abw, const FwdArgs& args, int m, int l0, int lane) {
  const double2* dgm = args.dg + args.dgofs[m];
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // (d, gamma) for rows l0..l0+63; rows past Lt are never stored
    const int l = l0 + 32 * h + lane;
    abw[32 * h + lane] = (l <= args.Lt) ? dgm[l - m] : make_double2(0.0, 1.0);
  }
  __syncwarp();
}

// Plan-time table of forward Legendre tiles (table mode): exactly the tiles the
// on-the-fly producer would build, in the same shared-memory fragment layout,
// plus their StageMeta.  One CTA (4 producer warps) per order m.
__global__ void __launch_bounds__(32 * kProducerWarps) ptab_fwd_kernel(FwdArgs args, double* ptab, StageMeta* mtab) {
  extern __shared__ __align__(128) double smem[];
  const int nPx = args.nchunks * FWD_RC;
  double2* abw_all = reinterpret_cast<double2*>(smem);
  FwdState st;
  double* sp1 = reinterpret_cast<double*>(abw_all + kProducerWarps * FWD_LB);
  st.p1 = sp1;
  st.p2 = sp1 + nPx;
  double* st_t = sp1 + 2 * nPx;
  int* st_ls = reinterpret_cast<int*>(st_t + nPx);
  st.t = st_t;
  st.ls = st_ls;
  const int m = args.m_begin + blockIdx.x;
  const int nlb = (args.Lt + 1 - m + FWD_LB - 1) / FWD_LB;
  for (int p = threadIdx.x; p < nPx; p += blockDim.x) {
    st_t[p] = args.pair_t[p];
    st_ls[p] = args.start_l[(size_t)m * args.nPpad + p];
    st.p1[p] = 0.0;
    st.p2[p] = 0.0;
  }
  __syncthreads();
  const int pw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* abw = abw_all + pw * FWD_LB;
  const long long base = args.tofs[m];
  for (int j = 0; j < nlb; ++j) {
    const int l0 = m + FWD_LB * j;
    fwd_stage_coefs(abw, args, m, l0, lane);
    for (int c = pw; c < args.nchunks; c += kProducerWarps) {
      const long long tile = base + (long long)j * args.nchunks + c;
      const int p = c * FWD_RC + lane;
      const TileClass tc = fwd_classify(st, p, l0, lane);
      if (lane == 0) mtab[tile].zero = tc.zero;
      if ((lane & 3) == 0) mtab[tile].kmin[lane >> 2] = tc.km;
      // table tiles hold Pbar = gamma_l R_l itself: the table-mode epilogue needs no gamma
      if (!tc.zero) fwd_compute<true>(args, st, tc, ptab + tile * FWD_PTILE, abw, m, j, nlb, p, l0, lane);
    }
  }
}

template <int KS0, int NTW, int NT, int KS1 = 8>
__device__ __forceinline__ void fwd_mtile_run(int nt0, double (&acc)[NTW][2], const double (&a)[8],
                                              const double (&bb)[8][NTW]) {
  // odd NT: the second column half holds one n-tile fewer; two unguarded instantiations
  // selected by one branch (a per-DMMA guard would make every mma.sync predicated)
  auto run = [&](auto nj) {
#pragma unroll
    for (int ks = KS0; ks < KS1; ++ks)
#pragma unroll
      for (int jn = 0; jn < decltype(nj)::value; ++jn) dmma_m8n8k4(acc[jn][0], acc[jn][1], a[ks], bb[ks][jn]);
  };
  if constexpr (NT % 2 == 0) {
    run(std::integral_constant<int, NTW>{});
  } else {
    if (nt0 == 0) run(std::integral_constant<int, NTW>{});
    else run(std::integral_constant<int, NTW - 1>{});
  }
}

// DMMAs of one M-tile from its first active k-step on (switch = real branch)
template <int NTW, int NT>
__device__ __forceinline__ void fwd_mtile_dmma(int kfirst, int nt0, double (&acc)[NTW][2], const double (&a)[8],
                                               const double (&bb)[8][NTW]) {
  switch (kfirst) {
    case 0: fwd_mtile_run<0, NTW, NT>(nt0, acc, a, bb); break;
    case 1: fwd_mtile_run<1, NTW, NT>(nt0, acc, a, bb); break;
    case 2: fwd_mtile_run<2, NTW, NT>(nt0, acc, a, bb); break;
    case 3: fwd_mtile_run<3, NTW, NT>(nt0, acc, a, bb); break;
    case 4: fwd_mtile_run<4, NTW, NT>(nt0, acc, a, bb); break;
    case 5: fwd_mtile_run<5, NTW, NT>(nt0, acc, a, bb); break;
    case 6: fwd_mtile_run<6, NTW, NT>(nt0, acc, a, bb); break;
    case 7: fwd_mtile_run<7, NTW, NT>(nt0, acc, a, bb); break;
    default: break;
  }
}

// Persistent forward: CTA b walks orders in snake order over rounds of gridDim
// (m ascending = work descending), which balances the per-order work (L+2-m).
__device__ __forceinline__ int fwd_item(int k, int b, int G) { return (k & 1) ? k * G + (G - 1 - b) : k * G + b; }

template <int NT, bool SPLIT = false>
__global__ void __launch_bounds__(kThreads, 1) legendre_fwd_kernel(FwdArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = FwdSmem<NT>;
  const int nPx = args.nchunks * FWD_RC;  // pairs covered by the forward chunks
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FWD_STAGES * SM::STAGE);
  uint64_t* empty = full + FWD_STAGES;
  // consumer warp 0's count of finished tiles (the producers' aliasing guard)
  volatile int* cons0 = reinterpret_cast<volatile int*>(empty + FWD_STAGES);
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + FWD_STAGES + 2);
  double2* abw_all = reinterpret_cast<double2*>(meta + FWD_STAGES);
  double* st_p1 = reinterpret_cast<double*>(abw_all + kProducerWarps * FWD_LB);
  double* st_p2 = st_p1 + nPx;
  double* st_t = st_p2 + nPx;
  int* st_ls = reinterpret_cast<int*>(st_t + nPx);

  const int Lt = args.Lt;
  const int nchunks = args.nchunks;
  const int S = (SPLIT && args.ksplit > 1) ? args.ksplit : 1;  // compile-time 1 in the unsplit kernel
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // field group of this CTA (blocks interleave the groups: heavy orders of every group first);
  // locals, not writes to the kernel parameter struct (a mutated parameter is copied out of the
  // constant bank)
  const int gi_ = blockIdx.x % (args.ngroups > 0 ? args.ngroups : 1);
  const double* const Xg = args.X + gi_ * args.x_gstride;
  double* const Fg = args.F + gi_ * args.f_gstride;
  const int bxg = blockIdx.x / (args.ngroups > 0 ? args.ngroups : 1);
  const int gdg = gridDim.x / (args.ngroups > 0 ? args.ngroups : 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < FWD_STAGES; ++s) {
      mbar_init(&full[s], (args.dbg & 32) ? 1 : 32);
      mbar_init(&empty[s], (args.dbg & 32) ? kConsumerWarps : 32 * kConsumerWarps);
    }
    *cons0 = 0;
    fence_barrier_init();
  }
  unsigned long long gt0 = 0;
  if (args.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  __syncthreads();

  if (is_producer(warp)) {
    // ------------------------------ producer ------------------------------
    const int pw = producer_index(warp);
    double2* abw = abw_all + pw * FWD_LB;
    FwdState st{st_p1, st_p2, st_t, st_ls};
    const bool table = args.ptab != nullptr;
    const uint64_t pol_first = l2_evict_first(), pol_last = l2_evict_last();
    uint32_t tbase = 0;  // tile counter across this CTA's orders
    for (int k = 0;; ++k) {
      const int it = fwd_item(k, bxg, gdg);
      if (it >= args.m_count * S) break;
      const int item = it / S, split = it - item * S;
      const int nu = (nchunks - split + S - 1) / S;  // this split's chunks c = split + S u
      const int m = args.m_begin + item;
      const int nlb = (Lt + 1 - m + FWD_LB - 1) / FWD_LB;
      // Tile ownership (u: the split's chunk index, c = split + S u).  Warp pw owns the chunks c = pw (mod 4) (their recurrence
      // state never changes hands).  Each l-block's leading all-zero chunks
      // (polar start past the block) are skipped by producers and consumers
      // alike, so tile t of the pipeline is the t-th live tile.  A producer
      // waits for its slot with a parity wait, which aliases once the slot is
      // two rounds behind; a warp's consecutive tiles can be up to ~2 rounds
      // apart here, so it first waits until consumer warp 0 has finished tile
      // t - 5 (which implies every consumer has finished tile t - 10).
      if (!table) {
        for (int u = pw; u < nu; u += kProducerWarps) {
          const int p = (split + S * u) * FWD_RC + lane;
          st_t[p] = args.pair_t[p];
          st_ls[p] = args.start_l[(size_t)m * args.nPpad + p];
          st_p1[p] = 0.0;
          st_p2[p] = 0.0;
        }
        __syncwarp();
      }
      const ChunkStarts cst = load_chunk_starts(args.cmin + (size_t)m * nchunks, nchunks, lane, split, S);
      uint32_t tb = tbase;
      for (int j = 0; j < nlb; ++j) {
        const int l0 = m + FWD_LB * j;
        const int u0 = first_live_chunk(cst, l0, Lt, nu);
        const int ufirst = u0 + ((pw - u0) & (kProducerWarps - 1));
        if (!table && ufirst < nu) fwd_stage_coefs(abw, args, m, l0, lane);
        for (int u = ufirst; u < nu; u += kProducerWarps) {
          const int c = split + S * u;
          const int tl = j * nchunks + c;  // table tile index (all chunks)
          const uint32_t t = tb + (u - u0);
          if (t >= 2 * FWD_STAGES)
            while (*cons0 < (int)t - (FWD_STAGES - 1)) __nanosleep(32);
        {
          const int stage = t % FWD_STAGES;
          const uint32_t round = t / FWD_STAGES;
          const int p = c * FWD_RC + lane;
          const TileClass tc =
              fwd_classify_ls(table ? __ldg(&args.start_l[(size_t)m * args.nPpad + p]) : st_ls[p], l0);
          const bool tr = args.trace && blockIdx.x == args.trace_cta && lane == 0 && t < 4096;
          if (tr) args.trace[t * 8 + 0] = clock64();
          mbar_wait(&empty[stage], (round & 1) ^ 1);
          if (tr) args.trace[t * 8 + 1] = clock64();
          double* Ps = smem + stage * SM::STAGE;
          double* Xs = Ps + FWD_PTILE;
          if (tc.zero || !table) {
            if (lane == 0) meta[stage].zero = tc.zero;
            if ((lane & 3) == 0) meta[stage].kmin[lane >> 2] = tc.km;
          }
          if (!tc.zero) {
            // The padded last chunk with at most four real pairs (the benchmark grids: one):
            // only k-step 0 is ever read (the consumers' ke = 1 path), so only its blocks are
            // copied, 3 + 2 KB instead of 24.6 + 16 KB per tile.  NT > 2 only: the single-field
            // consumers split the k-steps over warps and load every k-step's fragments.
            const bool lone = NT > 2 && args.klast == 1 && c == nchunks - 1;
            if (lane == 0 && lone) {
              const uint32_t xb = NT * 32 * 8;  // one k-step of one parity of the X tile
              const uint32_t bytes = 2 * xb + (table ? 8 * 256 + (uint32_t)sizeof(StageMeta) : 0u);
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(bytes)
                           : "memory");
              const double* xsrc = Xg + ((size_t)(m - args.m_begin) * nchunks + c) * SM::XTILE;
#pragma unroll
              for (int par = 0; par < 2; ++par)
                bulk_g2s_hint(Xs + par * 8 * NT * 32, xsrc + par * 8 * NT * 32, xb, &full[stage], pol_last);
              if (table) {
                const long long tile = args.tofs[m] + tl;
#pragma unroll
                for (int b = 0; b < 8; ++b)  // (parity, M-tile) blocks of k-step 0
                  bulk_g2s_hint(Ps + b * 8 * 32, args.ptab + tile * FWD_PTILE + b * 8 * 32, 256, &full[stage],
                                pol_first);
                bulk_g2s_hint(&meta[stage], args.mtab + tile, sizeof(StageMeta), &full[stage], pol_first);
              }
            } else if (lane == 0) {
              const uint32_t bytes = SM::XTILE * 8 + (table ? FWD_PTILE * 8 + (uint32_t)sizeof(StageMeta) : 0u);
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(bytes)
                           : "memory");
              // X chunks are re-read by every l-block of the order: keep them in L2;
              // the table tiles are read once: let them go first
              bulk_g2s_hint(Xs, Xg + ((size_t)(m - args.m_begin) * nchunks + c) * SM::XTILE, SM::XTILE * 8,
                            &full[stage], pol_last);
              if (table) {
                const long long tile = args.tofs[m] + tl;
                bulk_g2s_hint(Ps, args.ptab + tile * FWD_PTILE, FWD_PTILE * 8, &full[stage], pol_first);
                bulk_g2s_hint(&meta[stage], args.mtab + tile, sizeof(StageMeta), &full[stage], pol_first);
              }
            }
            if (!table && !(args.dbg & 2)) fwd_compute(args, st, tc, Ps, abw, m, j, nlb, p, l0, lane);
          }
          if (tr) args.trace[t * 8 + 2] = clock64() | ((long long)tc.zero << 62) | ((long long)tc.mixed << 61);
          if (args.dbg & 32) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stage]);
          } else {
            mbar_arrive(&full[stage]);
          }
        }
        }
        tb += nu - u0;
      }
      tbase = tb;
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  if constexpr (NT <= 2) {
    // Single-field launches (NT <= 2: 12 columns): with the (parity, row half,
    // column half) split below every warp would hold one n-tile, 1.5 fragment
    // loads per DMMA, and the consumers become shared-memory-issue bound (C4:
    // 30.7 of 32.7 ms with the recurrence switched off).  K-split instead: warp
    // (par, kq) takes all four M-tiles x NT n-tiles of its parity over k-steps
    // 2 kq, 2 kq + 1 (0.75 loads per DMMA); the four k-quarter partial sums are
    // added in a fixed order (kq 0, 1, 2, 3) at each l-block's epilogue.
    const int cw = consumer_index(warp);
    const int par = cw >> 2, kq = cw & 3;
    const int g = lane >> 2, q = lane & 3;
    const int xq = (g >> 2) * 16 + q * 4 + (g & 3);
    const int ncolF = 8 * NT;
    double* red = reinterpret_cast<double*>(st_ls + nPx);
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
    uint32_t tbase = 0;
    for (int k = 0;; ++k) {
      const int it = fwd_item(k, bxg, gdg);
      if (it >= args.m_count * S) break;
      const int item = it / S, split = it - item * S;
      const int nu = (nchunks - split + S - 1) / S;
      double* const Fout = split ? args.Fx + (size_t)(split - 1) * args.f_gstride : Fg;
      const int m = args.m_begin + item;
      const int nlb = (Lt + 1 - m + FWD_LB - 1) / FWD_LB;
      const double2* dgm = args.dg + args.dgofs[m];
      const ChunkStarts cst = load_chunk_starts(args.cmin + (size_t)m * nchunks, nchunks, lane, split, S);
      for (int j = 0; j < nlb; ++j) {
        const int l0 = m + FWD_LB * j;
        const int u0 = first_live_chunk(cst, l0, Lt, nu);
        // gamma of this warp's epilogue rows, loaded before the tiles (not after them)
        double gam4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int l = l0 + 2 * (8 * i + g) + par;
          gam4[i] = (args.ptab || l > Lt) ? 1.0 : __ldg(&dgm[l - m].y);
        }
        // Tiles of the l-block software-pipelined by one: the DMMAs of tile t are
        // issued, tile t is released, then tile t + 1 is awaited and its fragments
        // loaded while those DMMAs execute (without this both consumer warps of an
        // SMSP woke on the same barrier and loaded together, leaving the DMMA pipe
        // idle for the load latency of every tile).
        struct Frag {
          double a[2][4], bb[2][NT];
          int km0, km1;
          bool live;
        };
        auto fetch = [&](uint32_t t, Frag& f) {
          const int stage = t % FWD_STAGES;
#ifdef FV_TRACE_CONSUMERS
          const bool tr = args.trace && blockIdx.x == args.trace_cta && lane == 0 && cw == 0 && t < 4096;
          if (tr) args.trace[t * 8 + 3] = clock64();
#endif
          mbar_wait(&full[stage], (t / FWD_STAGES) & 1);
#ifdef FV_TRACE_CONSUMERS
          if (tr) args.trace[t * 8 + 4] = clock64();
#endif
          const double* Ps = smem + stage * SM::STAGE;
          const double* Xs = Ps + FWD_PTILE;
          f.km0 = meta[stage].kmin[2 * kq];
          f.km1 = meta[stage].kmin[2 * kq + 1];
          f.live = !meta[stage].zero && !(args.dbg & 1);
          if (f.live && !(args.dbg & 8)) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int ks = 2 * kq + kk;
              const int sw = ((g ^ (ks & 3)) << 2) + q;
#pragma unroll
              for (int i = 0; i < 4; ++i) f.a[kk][i] = lds_f64(&Ps[((par * 4 + i) * 8 + ks) * 32 + sw]);
#pragma unroll
              for (int jn = 0; jn < NT; ++jn) f.bb[kk][jn] = lds_f64(&Xs[((par * 8 + ks) * NT + jn) * 32 + xq]);
            }
          }
        };
        // M-tile i (rows l0 + 16 i .. + 15) runs k-step ks once some pair of it has
        // started (kmin[ks] <= last row) and it is not padding past Lt; real branches
        auto mma = [&](const Frag& f) {
          if (!f.live) return;
          if (l0 + 48 <= Lt && max(f.km0, f.km1) <= l0 + 15) {
            // every M-tile runs both k-steps (all but the tiles on the polar-start boundary and
            // the last l-block): one straight-line run.  A guarded mma.sync costs a WARPSYNC and
            // a predicate wait per guard (ncu: as many stall samples as the DMMAs themselves)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[kk][i], f.bb[kk][jn]);
            }
            return;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r0 = l0 + 16 * i;
            if (r0 > Lt) continue;
            if (f.km0 <= r0 + 15) {
#pragma unroll
              for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[0][i], f.bb[0][jn]);
            }
            if (f.km1 <= r0 + 15) {
#pragma unroll
              for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[1][i], f.bb[1][jn]);
            }
          }
        };
        auto release = [&](uint32_t t) {
#ifdef FV_TRACE_CONSUMERS
          if (args.trace && blockIdx.x == args.trace_cta && lane == 0 && cw == 0 && t < 4096)
            args.trace[t * 8 + 5] = clock64();  // DMMAs of tile t issued
#endif
          if (!(args.dbg & 32) || lane == 0) mbar_arrive(&empty[t % FWD_STAGES]);  // the fragments are in registers
          if (cw == 0 && lane == 0) *cons0 = (int)t + 1;
        };
        // two register sets alternate: tile t + 1 is awaited and loaded into the
        // other set while tile t's DMMAs execute
        Frag f0, f1;
        const uint32_t tend = tbase + (uint32_t)(nu - u0);
        if (tbase < tend) fetch(tbase, f0);
        for (uint32_t t = tbase; t < tend; t += 2) {
          mma(f0);
          release(t);
          if (t + 1 >= tend) break;
          fetch(t + 1, f1);
          mma(f1);
          release(t + 1);
          if (t + 2 < tend) fetch(t + 2, f0);
        }
        tbase += nu - u0;
        // epilogue of the l-block: k-quarters 1..3 park their partial sums, quarter 0
        // adds them in order and writes rows l = l0 + 2 (8 i + g) + par
        double* rp = red + (size_t)(par * 3) * 4 * NT * 64;
        if (kq > 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
              double* r = rp + (((kq - 1) * 4 + i) * NT + jn) * 64;
              r[lane] = acc[i][jn][0];
              r[32 + lane] = acc[i][jn][1];
            }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(32 * kConsumerWarps) : "memory");
        if (kq == 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int l = l0 + 2 * (8 * i + g) + par;
            double v[NT][2];
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) {
              v[jn][0] = acc[i][jn][0];
              v[jn][1] = acc[i][jn][1];
#pragma unroll
              for (int w = 0; w < 3; ++w) {
                const double* r = rp + ((w * 4 + i) * NT + jn) * 64;
                v[jn][0] += r[lane];
                v[jn][1] += r[32 + lane];
              }
            }
            if (l <= Lt) {
              double* row = Fout + ((size_t)l * (l + 1) / 2 + m) * ncolF;
              const double gam = gam4[i];  // P_l = gamma_l R_l
#pragma unroll
              for (int jn = 0; jn < NT; ++jn)
                *reinterpret_cast<double2*>(row + jn * 8 + 2 * q) = make_double2(gam * v[jn][0], gam * v[jn][1]);
            }
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(32 * kConsumerWarps) : "memory");
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
      }
    }
    return;
  }
  constexpr int NTW = (NT + 1) / 2;
  const int cw = consumer_index(warp);
  const int par = cw >> 2;
  const int mh = (cw >> 1) & 1;
  const int nh = cw & 1;
  const int nt0 = nh * NTW;
  const int g = lane >> 2, q = lane & 3;
  // B element (k = q, n = g) of an [n_hi 2][k 4][n_lo 4] X tile: each half-warp (g < 4, g >= 4) reads 16
  // consecutive doubles (conflict free; an [k][n] order would be 2-way conflicted per half-warp)
  const int xq = (g >> 2) * 16 + q * 4 + (g & 3);
  const int ncolF = 8 * NT;
  double acc[2][NTW][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NTW; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  uint32_t tbase = 0;
  for (int k = 0;; ++k) {
  const int it = fwd_item(k, bxg, gdg);
  if (it >= args.m_count * S) break;
  const int item = it / S, split = it - item * S;
  const int nu = (nchunks - split + S - 1) / S;
  double* const Fout = split ? args.Fx + (size_t)(split - 1) * args.f_gstride : Fg;
  const int m = args.m_begin + item;
  const int nlb = (Lt + 1 - m + FWD_LB - 1) / FWD_LB;
  const ChunkStarts cst = load_chunk_starts(args.cmin + (size_t)m * nchunks, nchunks, lane, split, S);
  for (int j = 0; j < nlb; ++j) {
    const int l0 = m + FWD_LB * j;
    const int u0 = first_live_chunk(cst, l0, Lt, nu);
    for (int u = u0; u < nu; ++u) {
      const uint32_t t = tbase + (u - u0);
      const int stage = t % FWD_STAGES;
      const uint32_t round = t / FWD_STAGES;
      const bool tr = args.trace && blockIdx.x == args.trace_cta && lane == 0 && cw == 0 && t < 4096;
      if (tr) args.trace[t * 8 + 3] = clock64();
      mbar_wait(&full[stage], round & 1);
      if (tr) args.trace[t * 8 + 4] = clock64();
      const double* Ps = smem + stage * SM::STAGE;
      const double* Xs = Ps + FWD_PTILE;
      const int4 km0 = *reinterpret_cast<const int4*>(&meta[stage].kmin[0]);
      const int4 km1 = *reinterpret_cast<const int4*>(&meta[stage].kmin[4]);
      const int kmin[8] = {km0.x, km0.y, km0.z, km0.w, km1.x, km1.y, km1.z, km1.w};
      // M-tile i = 2*mh + ii holds rows l0 + 16 i .. l0 + 16 i + 15 (one parity); its
      // k-steps below the polar start form a prefix (pairs further from the pole start
      // earlier) and M-tiles past Lt are padding, so each M-tile runs its DMMAs from its
      // first active k-step on.  A warp whose two M-tiles are both inactive (the rows past
      // Lt of an order's last l-block, the polar-start boundary) skips the tile's fragment
      // loads too: those tiles cost their 40 LDS.64 per warp and nothing else (traced: the
      // one-row order m = Lt spent 1150 cycles per tile on them).
      // The bound is clamped to Lt: padding pairs (the last chunk holds n_theta / 2 mod 32
      // real pairs: ONE on the benchmark grids) and pairs that never start have l_s = Lt + 1.
      // ke = 1: only k-step 0 is active (that last chunk), and only it is run.
      const int r0 = l0 + 32 * mh, r1 = r0 + 16;
      const int h0 = min(r0 + 15, Lt), h1 = min(r1 + 15, Lt);
      int kf0 = 8, kf1 = 8, ke0 = 0, ke1 = 0;
#pragma unroll
      for (int ks = 7; ks >= 0; --ks) {
        if (r0 <= Lt && kmin[ks] <= h0) {
          kf0 = ks;
          ke0 = max(ke0, ks + 1);
        }
        if (r1 <= Lt && kmin[ks] <= h1) {
          kf1 = ks;
          ke1 = max(ke1, ks + 1);
        }
      }
      if (!meta[stage].zero && !(args.dbg & 1) && (kf0 < 8 || kf1 < 8)) {
        // all fragments of the tile first (loads hoisted), then the DMMAs, selected with
        // real branches (a predicated-off DMMA still occupies the FP64 tensor pipe)
        double a0[8], a1[8], bb[8][NTW];
        const int kload = max(ke0, ke1) == 1 ? 1 : 8;  // the padded last chunk: only k-step 0 was copied
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (ks >= kload) break;
          const int sw = ((g ^ (ks & 3)) << 2) + q;
          a0[ks] = lds_f64(&Ps[((par * 4 + 2 * mh + 0) * 8 + ks) * 32 + sw]);
          a1[ks] = lds_f64(&Ps[((par * 4 + 2 * mh + 1) * 8 + ks) * 32 + sw]);
#pragma unroll
          for (int jn = 0; jn < NTW; ++jn)
            bb[ks][jn] = (nt0 + jn < NT) ? lds_f64(&Xs[((par * 8 + ks) * NT + nt0 + jn) * 32 + xq]) : 0.0;
        }
        if (kf0 == 0 && kf1 == 0 && ke0 == 8 && ke1 == 8) {
          // both M-tiles fully active (all but boundary tiles): one straight-line run, one
          // convergence point instead of one per M-tile
          fwd_mtile_run<0, NTW, NT>(nt0, acc[0], a0, bb);
          fwd_mtile_run<0, NTW, NT>(nt0, acc[1], a1, bb);
        } else if (max(ke0, ke1) == 1) {
          // the padded last chunk: one real k-step
          if (kf0 == 0) fwd_mtile_run<0, NTW, NT, 1>(nt0, acc[0], a0, bb);
          if (kf1 == 0) fwd_mtile_run<0, NTW, NT, 1>(nt0, acc[1], a1, bb);
        } else {
          fwd_mtile_dmma<NTW, NT>(kf0, nt0, acc[0], a0, bb);
          fwd_mtile_dmma<NTW, NT>(kf1, nt0, acc[1], a1, bb);
        }
      }
      if (tr) args.trace[t * 8 + 5] = clock64();
      if (!(args.dbg & 32) || lane == 0) mbar_arrive(&empty[stage]);
      if (cw == 0 && lane == 0) *cons0 = (int)t + 1;
    }
    tbase += nu - u0;
    // epilogue for this l-block: rows l = l0 + 2*(8*i + g) + par
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int i = 2 * mh + ii;
      const int l = l0 + 2 * (8 * i + g) + par;
      if (l <= Lt) {
        double* row = Fout + ((size_t)l * (l + 1) / 2 + m) * ncolF;
        const double gam = args.ptab ? 1.0 : args.dg[args.dgofs[m] + (l - m)].y;  // P_l = gamma_l R_l
#pragma unroll
        for (int jn = 0; jn < NTW; ++jn) {
          if (nt0 + jn < NT) {
            *reinterpret_cast<double2*>(row + (nt0 + jn) * 8 + 2 * q) =
                make_double2(gam * acc[ii][jn][0], gam * acc[ii][jn][1]);
          }
        }
      }
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) acc[ii][jn][0] = acc[ii][jn][1] = 0.0;
    }
  }
  }
  if (args.trace && cw == 0 && lane == 0 && blockIdx.x < 4096) {
    unsigned long long gt1;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long* ct = args.trace + 4096 * 8 + blockIdx.x * 4;
    ct[0] = (long long)gt0;
    ct[1] = (long long)gt1;
    ct[2] = smid;
  }
}

// ---------------------------------------------------------------------------
// forward, single field, on the fly: two recurrence chains per producer lane
// ---------------------------------------------------------------------------
// With the guard-free consumers the single-field forward (C4) is bound by its producers:
// a lane runs ONE dependent chain (one DFMA per degree on the chain) whose latency the
// consumers' DMMAs stretch on the shared FP64 datapath (10 -> 20-30 cycles per step), and
// the recurrence state carried from l-block to l-block ties every chunk to one warp and
// takes 58 KB of shared memory.  Here the plan stores the state of every pair at every tile
// start (fseed_kernel: 16 bytes per (order, l-block, pair), 4.4 GB at L = 4096, exactly the
// carried state, so results are bitwise those of legendre_fwd_kernel).  Tiles are then
// independent: no state in shared memory, EIGHT 24 KB stages, and a producer warp fills
// TWO tiles at once (adjacent live chunks of one l-block), its lanes running the two
// chains interleaved.  Warp pw owns the slots 2 pw, 2 pw + 1 for good (pairs are aligned
// to even pipeline positions; an l-block with an odd live count gets one dummy zero tile),
// so its parity waits are exact and the aliasing guard of legendre_fwd_kernel is gone.
// Consumers are those of legendre_fwd_kernel's single-field path.
constexpr int FWD2_STAGES = 8;

template <int NT>
struct Fwd2Smem {
  static constexpr int XTILE = 2 * 8 * NT * 32;
  static constexpr int STAGE = FWD_PTILE + XTILE;
  static constexpr int KRED = 2 * 3 * 4 * NT * 2 * 32;  // k-quarter partial sums (as FwdSmem)
  static constexpr size_t bytes = (size_t)FWD2_STAGES * STAGE * 8 + 2 * FWD2_STAGES * 8 +
                                  FWD2_STAGES * sizeof(StageMeta) + kProducerWarps * FWD_LB * 16 + (size_t)KRED * 8;
};

// Plan time: the recurrence state of every pair at the start of every (l-block, chunk)
// tile, walking the tiles exactly as the on-the-fly producer does (one CTA per order).
__global__ void __launch_bounds__(32 * kProducerWarps) fseed_kernel(FwdArgs args, double2* seed) {
  extern __shared__ __align__(128) double smem[];
  const int nPx = args.nchunks * FWD_RC;
  double* scratch = smem;  // [producer warp][FWD_PTILE]: the tiles themselves are not kept
  double2* abw_all = reinterpret_cast<double2*>(scratch + kProducerWarps * FWD_PTILE);
  FwdState st;
  double* sp1 = reinterpret_cast<double*>(abw_all + kProducerWarps * FWD_LB);
  st.p1 = sp1;
  st.p2 = sp1 + nPx;
  double* st_t = sp1 + 2 * nPx;
  int* st_ls = reinterpret_cast<int*>(st_t + nPx);
  st.t = st_t;
  st.ls = st_ls;
  const int m = args.m_begin + blockIdx.x;
  const int nlb = (args.Lt + 1 - m + FWD_LB - 1) / FWD_LB;
  for (int p = threadIdx.x; p < nPx; p += blockDim.x) {
    st_t[p] = args.pair_t[p];
    st_ls[p] = args.start_l[(size_t)m * args.nPpad + p];
    st.p1[p] = 0.0;
    st.p2[p] = 0.0;
  }
  __syncthreads();
  const int pw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* abw = abw_all + pw * FWD_LB;
  const long long base = args.tofs[m];
  for (int j = 0; j < nlb; ++j) {
    const int l0 = m + FWD_LB * j;
    fwd_stage_coefs(abw, args, m, l0, lane);
    for (int c = pw; c < args.nchunks; c += kProducerWarps) {
      const long long tile = base + (long long)j * args.nchunks + c;
      const int p = c * FWD_RC + lane;
      const TileClass tc = fwd_classify(st, p, l0, lane);
      seed[tile * 32 + lane] = make_double2(st.p1[p], st.p2[p]);
      if (!tc.zero) fwd_compute(args, st, tc, scratch + pw * FWD_PTILE, abw, m, j, nlb, p, l0, lane);
    }
  }
}

// rows 0..63 of two tiles of one l-block at once (lane = the same pair slot in both
// chunks): fwd_produce's arithmetic, the two chains interleaved
__device__ __forceinline__ void fwd_produce2(double* PsA, double* PsB, const double2* dgw, double ttA, double ttB,
                                             double a1, double a2, double b1, double b2, int lane) {
  const int s = lane >> 2, q = lane & 3, sx = s & 3;
  int off[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) off[g] = s * 32 + q + ((g ^ sx) << 2);
#pragma unroll
  for (int b0 = 0; b0 < FWD_LB; b0 += 8) {
    double dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[k] = dgw[b0 + k].x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double va = fma(ttA, a1, -(dd[k] * a2));
      const double vb = fma(ttB, b1, -(dd[k] * b2));
      a2 = a1;
      a1 = va;
      b2 = b1;
      b1 = vb;
      const int par = idx & 1, rp = idx >> 1, i = rp >> 3, g = rp & 7;
      const int o = off[g] + (par * 4 + i) * 8 * 32;
      PsA[o] = va;
      PsB[o] = vb;
      if ((idx & 31) == 31) {
        const double g1 = dgw[idx].y, g2 = dgw[idx - 1].y;
        a1 *= g1;
        a2 *= g2;
        b1 *= g1;
        b2 *= g2;
      }
    }
  }
}

template <int NT, bool SPLIT = false>
__global__ void __launch_bounds__(kThreads, 1) legendre_fwd2_kernel(FwdArgs args) {
  static_assert(NT <= 2, "single-field forward");
  extern __shared__ __align__(128) double smem[];
  using SM = Fwd2Smem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FWD2_STAGES * SM::STAGE);
  uint64_t* empty = full + FWD2_STAGES;
  StageMeta* meta = reinterpret_cast<StageMeta*>(empty + FWD2_STAGES);
  double2* abw_all = reinterpret_cast<double2*>(meta + FWD2_STAGES);
  double* red_base = reinterpret_cast<double*>(abw_all + kProducerWarps * FWD_LB);

  const int Lt = args.Lt;
  const int nchunks = args.nchunks;
  const int S = (SPLIT && args.ksplit > 1) ? args.ksplit : 1;  // compile-time 1 in the unsplit kernel
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // field group of this CTA (blocks interleave the groups: heavy orders of every group first);
  // locals, not writes to the kernel parameter struct (a mutated parameter is copied out of the
  // constant bank)
  const int gi_ = blockIdx.x % (args.ngroups > 0 ? args.ngroups : 1);
  const double* const Xg = args.X + gi_ * args.x_gstride;
  double* const Fg = args.F + gi_ * args.f_gstride;
  const int bxg = blockIdx.x / (args.ngroups > 0 ? args.ngroups : 1);
  const int gdg = gridDim.x / (args.ngroups > 0 ? args.ngroups : 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < FWD2_STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], 32 * kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (is_producer(warp)) {
    // ------------------------------ producer ------------------------------
    const int pw = producer_index(warp);
    double2* abw = abw_all + pw * FWD_LB;
    const uint64_t pol_last = l2_evict_last();
    const int sA = 2 * pw, sB = 2 * pw + 1;  // this warp's stage slots
    double* const PsA = smem + sA * SM::STAGE;
    double* const PsB = smem + sB * SM::STAGE;
    uint32_t tbase = 0;  // pipeline position of the l-block's first tile (always even)
    for (int k = 0;; ++k) {
      const int it = fwd_item(k, bxg, gdg);
      if (it >= args.m_count * S) break;
      const int item = it / S, split = it - item * S;
      const int nu = (nchunks - split + S - 1) / S;  // this split's chunks c = split + S u
      const int m = args.m_begin + item;
      const int nlb = (Lt + 1 - m + FWD_LB - 1) / FWD_LB;
      const int* ls_m = args.start_l + (size_t)m * args.nPpad;
      const ChunkStarts cst = load_chunk_starts(args.cmin + (size_t)m * nchunks, nchunks, lane, split, S);
      for (int j = 0; j < nlb; ++j) {
        const int l0 = m + FWD_LB * j;
        const int u0 = first_live_chunk(cst, l0, Lt, nu);
        const int npairs = (nu - u0 + 1) >> 1;
        // pair q of the l-block sits at pipeline positions tbase + 2 q, + 1: owner ((tbase >> 1) + q) & 3
        const int q0 = (pw - (int)(tbase >> 1)) & (kProducerWarps - 1);
        if (q0 < npairs) fwd_stage_coefs(abw, args, m, l0, lane);
        for (int q = q0; q < npairs; q += kProducerWarps) {
          const int uA = u0 + 2 * q;
          const bool hasB = uA + 1 < nu;  // an odd live count: the last pair's second tile is a dummy
          const int cA = split + S * uA, cB = split + S * (uA + 1);
          const int pA = cA * FWD_RC + lane, pB = cB * FWD_RC + lane;
          const int lsA = __ldg(&ls_m[pA]);
          const int lsB = hasB ? __ldg(&ls_m[pB]) : 0x7fffffff;
          const long long tl = args.tofs[m] + (long long)j * nchunks;
          const double2 sdA = __ldg(&args.seed[(tl + cA) * 32 + lane]);
          const double2 sdB = hasB ? __ldg(&args.seed[(tl + cB) * 32 + lane]) : make_double2(0.0, 0.0);
          const double ttA = __ldg(&args.pair_t[pA]);
          const double ttB = hasB ? __ldg(&args.pair_t[pB]) : 0.0;
          const TileClass tcA = fwd_classify_ls(lsA, l0);
          TileClass tcB = fwd_classify_ls(lsB, l0);  // a dummy classifies as zero
          const uint32_t round = (tbase + 2u * (uint32_t)q) / FWD2_STAGES;
          mbar_wait(&empty[sA], (round & 1) ^ 1);
          mbar_wait(&empty[sB], (round & 1) ^ 1);
          if (lane == 0) {
            meta[sA].zero = tcA.zero;
            meta[sB].zero = tcB.zero;
          }
          if ((lane & 3) == 0) {
            meta[sA].kmin[lane >> 2] = tcA.km;
            meta[sB].kmin[lane >> 2] = tcB.km;
          }
          if (lane == 0) {
            if (!tcA.zero) {
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[sA])),
                           "r"((uint32_t)(SM::XTILE * 8))
                           : "memory");
              bulk_g2s_hint(PsA + FWD_PTILE, Xg + ((size_t)(m - args.m_begin) * nchunks + cA) * SM::XTILE,
                            SM::XTILE * 8, &full[sA], pol_last);
            }
            if (!tcB.zero) {
              asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[sB])),
                           "r"((uint32_t)(SM::XTILE * 8))
                           : "memory");
              bulk_g2s_hint(PsB + FWD_PTILE, Xg + ((size_t)(m - args.m_begin) * nchunks + cB) * SM::XTILE,
                            SM::XTILE * 8, &full[sB], pol_last);
            }
          }
          if (!(args.dbg & 2)) {
            if (!tcA.zero && !tcB.zero && !tcA.mixed && !tcB.mixed) {
              fwd_produce2(PsA, PsB, abw, ttA, ttB, sdA.x, sdA.y, sdB.x, sdB.y, lane);
            } else {
              // boundary tiles (a polar start inside the tile) and lone tiles: one chain at a time
              auto one = [&](const TileClass& tc, double* Ps, int ls, int p, double tt, double2 sd) {
                if (tc.zero) return;
                Inject in;
                in.ls = ls;
                in.A = in.B = 0.0;
                if (tc.mixed) {
                  const double2 v = args.start_v[(size_t)m * args.nPpad + p];
                  in.A = v.x;
                  in.B = v.y;
                }
                double p1 = sd.x, p2 = sd.y;
                if (tc.mixed) fwd_produce<true>(Ps, abw, tt, p1, p2, lane, l0, in);
                else fwd_produce<false>(Ps, abw, tt, p1, p2, lane, l0, in);
              };
              one(tcA, PsA, lsA, pA, ttA, sdA);
              one(tcB, PsB, lsB, pB, ttB, sdB);
            }
          }
          mbar_arrive(&full[sA]);
          mbar_arrive(&full[sB]);
        }
        tbase += 2u * (uint32_t)npairs;
      }
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  // (legendre_fwd_kernel's single-field consumers on eight stages)
  // Single-field launches (NT <= 2: 12 columns): with the (parity, row half,
  // column half) split below every warp would hold one n-tile, 1.5 fragment
  // loads per DMMA, and the consumers become shared-memory-issue bound (C4:
  // 30.7 of 32.7 ms with the recurrence switched off).  K-split instead: warp
  // (par, kq) takes all four M-tiles x NT n-tiles of its parity over k-steps
  // 2 kq, 2 kq + 1 (0.75 loads per DMMA); the four k-quarter partial sums are
  // added in a fixed order (kq 0, 1, 2, 3) at each l-block's epilogue.
  const int cw = consumer_index(warp);
  const int par = cw >> 2, kq = cw & 3;
  const int g = lane >> 2, q = lane & 3;
  const int xq = (g >> 2) * 16 + q * 4 + (g & 3);
  const int ncolF = 8 * NT;
  double* red = red_base;
  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
  uint32_t tbase = 0;
  for (int k = 0;; ++k) {
    const int it = fwd_item(k, bxg, gdg);
    if (it >= args.m_count * S) break;
    const int item = it / S, split = it - item * S;
    const int nu = (nchunks - split + S - 1) / S;
    double* const Fout = split ? args.Fx + (size_t)(split - 1) * args.f_gstride : Fg;
    const int m = args.m_begin + item;
    const int nlb = (Lt + 1 - m + FWD_LB - 1) / FWD_LB;
    const double2* dgm = args.dg + args.dgofs[m];
    const ChunkStarts cst = load_chunk_starts(args.cmin + (size_t)m * nchunks, nchunks, lane, split, S);
    for (int j = 0; j < nlb; ++j) {
      const int l0 = m + FWD_LB * j;
      const int u0 = first_live_chunk(cst, l0, Lt, nu);
      // gamma of this warp's epilogue rows, loaded before the tiles (not after them)
      double gam4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int l = l0 + 2 * (8 * i + g) + par;
        gam4[i] = (args.ptab || l > Lt) ? 1.0 : __ldg(&dgm[l - m].y);
      }
      // Tiles of the l-block software-pipelined by one: the DMMAs of tile t are
      // issued, tile t is released, then tile t + 1 is awaited and its fragments
      // loaded while those DMMAs execute (without this both consumer warps of an
      // SMSP woke on the same barrier and loaded together, leaving the DMMA pipe
      // idle for the load latency of every tile).
      struct Frag {
        double a[2][4], bb[2][NT];
        int km0, km1;
        bool live;
      };
      auto fetch = [&](uint32_t t, Frag& f) {
        const int stage = t % FWD2_STAGES;
#ifdef FV_TRACE_CONSUMERS
        const bool tr = args.trace && blockIdx.x == args.trace_cta && lane == 0 && cw == 0 && t < 4096;
        if (tr) args.trace[t * 8 + 3] = clock64();
#endif
        mbar_wait(&full[stage], (t / FWD2_STAGES) & 1);
#ifdef FV_TRACE_CONSUMERS
        if (tr) args.trace[t * 8 + 4] = clock64();
#endif
        const double* Ps = smem + stage * SM::STAGE;
        const double* Xs = Ps + FWD_PTILE;
        f.km0 = meta[stage].kmin[2 * kq];
        f.km1 = meta[stage].kmin[2 * kq + 1];
        f.live = !meta[stage].zero && !(args.dbg & 1);
        if (f.live && !(args.dbg & 8)) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int ks = 2 * kq + kk;
            const int sw = ((g ^ (ks & 3)) << 2) + q;
#pragma unroll
            for (int i = 0; i < 4; ++i) f.a[kk][i] = lds_f64(&Ps[((par * 4 + i) * 8 + ks) * 32 + sw]);
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) f.bb[kk][jn] = lds_f64(&Xs[((par * 8 + ks) * NT + jn) * 32 + xq]);
          }
        }
      };
      // M-tile i (rows l0 + 16 i .. + 15) runs k-step ks once some pair of it has
      // started (kmin[ks] <= last row) and it is not padding past Lt; real branches
      auto mma = [&](const Frag& f) {
        if (!f.live) return;
        if (l0 + 48 <= Lt && max(f.km0, f.km1) <= l0 + 15) {
          // every M-tile runs both k-steps (all but the tiles on the polar-start boundary and
          // the last l-block): one straight-line run.  A guarded mma.sync costs a WARPSYNC and
          // a predicate wait per guard (ncu: as many stall samples as the DMMAs themselves)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[kk][i], f.bb[kk][jn]);
          }
          return;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r0 = l0 + 16 * i;
          if (r0 > Lt) continue;
          if (f.km0 <= r0 + 15) {
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[0][i], f.bb[0][jn]);
          }
          if (f.km1 <= r0 + 15) {
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) dmma_m8n8k4(acc[i][jn][0], acc[i][jn][1], f.a[1][i], f.bb[1][jn]);
          }
        }
      };
      auto release = [&](uint32_t t) {
#ifdef FV_TRACE_CONSUMERS
        if (args.trace && blockIdx.x == args.trace_cta && lane == 0 && cw == 0 && t < 4096)
          args.trace[t * 8 + 5] = clock64();  // DMMAs of tile t issued
#endif
        mbar_arrive(&empty[t % FWD2_STAGES]);  // the fragments are in registers
      };
      // two register sets alternate: tile t + 1 is awaited and loaded into the
      // other set while tile t's DMMAs execute
      Frag f0, f1;
      // an odd live count is padded with one dummy zero tile so that pairs never span l-blocks
      const uint32_t tend = tbase + 2u * (uint32_t)((nu - u0 + 1) >> 1);
      if (tbase < tend) fetch(tbase, f0);
      for (uint32_t t = tbase; t < tend; t += 2) {
        mma(f0);
        release(t);
        if (t + 1 >= tend) break;
        fetch(t + 1, f1);
        mma(f1);
        release(t + 1);
        if (t + 2 < tend) fetch(t + 2, f0);
      }
      tbase = tend;
      // epilogue of the l-block: k-quarters 1..3 park their partial sums, quarter 0
      // adds them in order and writes rows l = l0 + 2 (8 i + g) + par
      double* rp = red + (size_t)(par * 3) * 4 * NT * 64;
      if (kq > 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) {
            double* r = rp + (((kq - 1) * 4 + i) * NT + jn) * 64;
            r[lane] = acc[i][jn][0];
            r[32 + lane] = acc[i][jn][1];
          }
      }
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kConsumerWarps) : "memory");
      if (kq == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int l = l0 + 2 * (8 * i + g) + par;
          double v[NT][2];
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) {
            v[jn][0] = acc[i][jn][0];
            v[jn][1] = acc[i][jn][1];
#pragma unroll
            for (int w = 0; w < 3; ++w) {
              const double* r = rp + ((w * 4 + i) * NT + jn) * 64;
              v[jn][0] += r[lane];
              v[jn][1] += r[32 + lane];
            }
          }
          if (l <= Lt) {
            double* row = Fout + ((size_t)l * (l + 1) / 2 + m) * ncolF;
            const double gam = gam4[i];  // P_l = gamma_l R_l
#pragma unroll
            for (int jn = 0; jn < NT; ++jn)
              *reinterpret_cast<double2*>(row + jn * 8 + 2 * q) = make_double2(gam * v[jn][0], gam * v[jn][1]);
          }
        }
      }
      asm volatile("bar.sync 2, %0;" ::"n"(32 * kConsumerWarps) : "memory");
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
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
#ifndef FV_ADJ_STAGES
#define FV_ADJ_STAGES 5
#endif
constexpr int ADJ_STAGES = FV_ADJ_STAGES;
constexpr int ADJ_MTILE = 2 * ADJ_KS * 32;           // doubles per M-tile: [par][ks][lane]
constexpr int ADJ_PTILE = ADJ_MT * ADJ_MTILE;         // doubles: [Mtile][par][ks][lane] (M-tile major, so
                                                      // any run of M-tiles is one contiguous bulk copy)

struct AdjArgs {
  const double* G;          // per m: (gofs[m] + lc) * GTILE, [par][ks ADJ_KS][NT][32]
  const long long* gofs;
  double2* S;               // ring spectra, layout lay (common.cuh SLayout)
  const int* start_l;
  const double2* start_v;
  const double2* dg;
  const long long* dgofs;
  const double* pair_t;
  const int* pair_n;        // north ring of each pair (-1: padding)
  const int* pair_s;        // south ring (-1: unpaired)
  int Lt, nP, nPpad, nrc, n_phi, n_theta, B_total, b0, nfields, m_begin;
  int dbg;
  int m_count;  // orders m_begin .. m_begin + m_count - 1
  // table mode: P^T stage tiles [aofs[m] + rc * nlc(m) + lc][ADJ_PTILE] (ptab_adj_kernel)
  const double* ptab;
  const long long* aofs;
  long long* trace;  // optional pipeline timeline of CTA trace_cta (clock64 stamps), normally null
  int trace_cta;
  SLayout lay;
  const int* cmin;   // per (order, 128-pair chunk): smallest polar start (the leading all-zero stages are skipped)
  // several 4-field groups in one launch: item i works on group i % ngroups (G of group g
  // at + g * g_gstride, its fields from b0 + 4 g)
  int ngroups;
  long long g_gstride;
};

// first 32-degree stage of item (m, rc) in which some pair of the chunk has started
__device__ __forceinline__ int adj_first_stage(const AdjArgs& a, int m, int rc) {
  const int cm = __ldg(&a.cmin[(size_t)m * a.nrc + rc]);
  const int nlc = (a.Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
  if (cm > a.Lt) return nlc;
  const int x = cm - m - (ADJ_LC - 1);
  return x > 0 ? (x + ADJ_LC - 1) / ADJ_LC : 0;
}

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

// l values idx = 0..ADJ_LC-1 of one stage (= one 32-degree block) for the lane's
// pair (M-tile i, row g); the state goes back to P units after the last row.
template <bool MIXED>
__device__ __forceinline__ void adj_produce(double* Ps, const double2* dgw, double tt, double& p1, double& p2,
                                            int i, int g, int l0, const Inject& in) {
  const int cx = (g >> 2) | ((i & 1) << 1);
  double* bp[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) bp[q] = Ps + i * ADJ_MTILE + (g << 2) + (q ^ cx);
#pragma unroll
  for (int b0 = 0; b0 < ADJ_LC; b0 += 8) {
    double dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[k] = dgw[b0 + k].x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double v = rec_step<MIXED>(p1, p2, tt, dd[k], l0 + idx, in);
      const int par = idx & 1, kk = idx >> 1, ks = kk >> 2, q = kk & 3;
      bp[q][(par * ADJ_KS + ks) * 32] = v;
    }
  }
  p1 *= dgw[ADJ_LC - 1].y;
  p2 *= dgw[ADJ_LC - 2].y;
}

// Plan-time table of adjoint P^T stage tiles (table mode); all-zero warps leave
// their M-tiles unwritten, exactly as the on-the-fly producer does.
__global__ void __launch_bounds__(32 * kProducerWarps) ptab_adj_kernel(AdjArgs args, double* ptab) {
  __shared__ double2 abw_all[kProducerWarps * ADJ_LC];
  const int m = args.m_begin + blockIdx.x / args.nrc;
  const int rc = blockIdx.x % args.nrc;
  const int Lt = args.Lt;
  const int nlc = (Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
  const int pw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* abw = abw_all + pw * ADJ_LC;
  const int rho = 32 * pw + lane;
  const int p = rc * ADJ_RC + rho;
  const int i = rho >> 3, g = rho & 7;
  const double tt = args.pair_t[p];
  Inject in;
  in.ls = args.start_l[(size_t)m * args.nPpad + p];
  const double2 v = args.start_v[(size_t)m * args.nPpad + p];
  in.A = v.x;
  in.B = v.y;
  double p1 = 0.0, p2 = 0.0;
  const double2* dgm = args.dg + args.dgofs[m];
  double* base = ptab + (size_t)(args.aofs[m] + (long long)rc * nlc) * ADJ_PTILE;
  for (int lc = 0; lc < nlc; ++lc) {
    const int l0 = m + ADJ_LC * lc;
    const bool before = in.ls > l0 + ADJ_LC - 1;
    const bool zero = __all_sync(0xffffffffu, before);
    const bool mixed = __any_sync(0xffffffffu, !before && in.ls + 1 >= l0);
    if (zero) continue;
    __syncwarp();
    const int l = l0 + lane;
    abw[lane] = (l <= Lt) ? dgm[l - m] : make_double2(0.0, 1.0);
    __syncwarp();
    double* Ps = base + (size_t)lc * ADJ_PTILE;
    if (mixed) adj_produce<true>(Ps, abw, tt, p1, p2, i, g, l0, in);
    else adj_produce<false>(Ps, abw, tt, p1, p2, i, g, l0, in);
  }
}

// DMMAs of one (k-step, parity) for a consumer warp: M-tiles ii >= I0 of its two
template <int I0, int NT, int I1 = 2>
__device__ __forceinline__ void adj_ks_run(double (&acc)[2][NT][2], const double (&a)[2], const double (&b)[NT]) {
#pragma unroll
  for (int jn = 0; jn < NT; ++jn)
#pragma unroll
    for (int ii = I0; ii < I1; ++ii) dmma_m8n8k4(acc[ii][jn][0], acc[ii][jn][1], a[ii], b[jn]);
}

// A chunk that holds a single M-tile of real pairs (the benchmark grids: n_theta / 2 = 1 mod 128,
// so every order's last chunk is ONE pair): with the regular split only consumer warp 0 has work,
// 48 DMMAs per stage on one sub-partition.  Here the item's six (NT) n-tiles go to NT warps, both
// parities each, eight DMMAs per stage and warp (every k-step that lies within Lt is run; before
// the polar start the Legendre values are zeros).  Kept out of line: the item runs once per order
// and must not add registers to legendre_adj_kernel's main loop.
// (scalar arguments, not the AdjArgs struct: a reference to the kernel's parameter struct would
// force a stack copy of it in the caller)
struct AdjSoloOut {
  double2* S;
  SLayout lay;
  int n_phi, n_theta, nfields, dbg;
};
template <int NT>
__device__ __noinline__ uint32_t adj_solo_item(AdjSoloOut args, const int* pair_n, const int* pair_s, int Lt,
                                               const double* smem, int stage_doubles, uint64_t* full, uint64_t* empty,
                                               uint32_t sc, int m, int rc, int fb0, int lc0, int nlc, int cw,
                                               int lane) {
  const int g = lane >> 2, q = lane & 3;
  const bool mine = cw < NT && !(args.dbg & 1);
  const int p = rc * ADJ_RC + g;  // M-tile 0, row g
  const int rn = __ldg(&pair_n[p]), rs = __ldg(&pair_s[p]);
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [parity][re/im] of n-tile cw
  for (int lc = lc0; lc < nlc; ++lc, ++sc) {
    const int stage = sc % ADJ_STAGES;
    const int l0s = m + ADJ_LC * lc;
    mbar_wait(&full[stage], (sc / ADJ_STAGES) & 1);
    if (mine) {
      const double* Ps = smem + (size_t)stage * stage_doubles;
      const double* Gs = Ps + ADJ_PTILE;
#pragma unroll
      for (int t = 0; t < 2 * ADJ_KS; ++t) {
        const int ks = t >> 1, par = t & 1;
        if (l0s + 8 * ks <= Lt) {
          const double a = lds_f64(&Ps[(par * ADJ_KS + ks) * 32 + adj_swz(g, q, 0)]);
          const double b = lds_f64(&Gs[((par * ADJ_KS + ks) * NT + cw) * 32 + lane]);
          dmma_m8n8k4(acc[par][0], acc[par][1], a, b);
        }
      }
    }
    mbar_arrive(&empty[stage]);
  }
  if (mine && !(args.dbg & 4) && rn >= 0) {
    const int ser = 4 * cw + q;  // 6*field + 2*comp + sign
    const int b = ser / 6, comp = (ser % 6) >> 1, sgn = ser & 1;
    if (b < args.nfields && !(sgn == 1 && m == 0)) {
      double2* dst = args.S + spec_bin(args.lay, m, sgn, args.n_phi) * args.lay.bs;
      const long long rbase = (long long)(fb0 + b) * args.n_theta;
      const double er = acc[0][0], ei = acc[0][1], orr = acc[1][0], oi = acc[1][1];
      dst[spec_cr(args.lay, comp, rbase + rn)] = make_double2(er + orr, ei + oi);
      if (rs >= 0) dst[spec_cr(args.lay, comp, rbase + rs)] = make_double2(er - orr, ei - oi);
    }
  }
  return sc;
}

// Persistent: one CTA per SM walks the (order m, 128-pair chunk) items in
// descending-work order (item = blockIdx.x + k * gridDim.x; m ascending), with
// one stage counter across items, so the producers fill the next item's stages
// while the consumers run the previous item's epilogue.  Each consumer warp owns
// both parities of its M-tiles, so the epilogue (north = E + O, south = E - O)
// is register-local: no exchange buffer and no CTA barrier, and the shared
// memory goes to a fifth stage.
template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_adj_kernel(AdjArgs args) {
  extern __shared__ __align__(128) double smem[];
  using SM = AdjSmem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ADJ_STAGES * SM::STAGE);
  uint64_t* empty = full + ADJ_STAGES;
  double2* abw_all = reinterpret_cast<double2*>(empty + ADJ_STAGES);

  const int Lt = args.Lt;
  const int ngr = args.ngroups > 0 ? args.ngroups : 1;
  const int nitems = args.m_count * args.nrc * ngr;
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

  if (is_producer(warp)) {
    // ------------------------------ producer ------------------------------
    const int pw = producer_index(warp);
    double2* abw = abw_all + pw * ADJ_LC;
    const int rho = 32 * pw + lane;            // pair within the item's chunk
    const int i = rho >> 3, g = rho & 7;
    const bool table = args.ptab != nullptr;
    const uint64_t pol_first = l2_evict_first(), pol_last = l2_evict_last();
    uint32_t sc = 0;                           // stage counter across items
    for (int itg = blockIdx.x; itg < nitems; itg += gridDim.x) {
      const int gi = itg % ngr, item = itg / ngr;
      const int m = args.m_begin + item / args.nrc;
      const int rc = item % args.nrc;
      const int nlc = (Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
      const int p = rc * ADJ_RC + rho;
      const double tt = args.pair_t[p];
      Inject in;
      in.ls = args.start_l[(size_t)m * args.nPpad + p];
      {
        const double2 v = args.start_v[(size_t)m * args.nPpad + p];
        in.A = v.x;
        in.B = v.y;
      }
      double p1 = 0.0, p2 = 0.0;
      const double2* dgm = args.dg + args.dgofs[m];
      const double* Gm = args.G + gi * args.g_gstride + (size_t)args.gofs[m] * SM::GTILE;
      // (d, gamma) of the stage's 32 degrees, one per lane, loaded one stage ahead
      // (an L2 round trip on the recurrence's critical path otherwise)
      auto dg_at = [&](int lcx) {
        const int l = m + ADJ_LC * lcx + lane;
        return (l <= Lt) ? __ldg(&dgm[l - m]) : make_double2(0.0, 1.0);
      };
      const int lc0 = adj_first_stage(args, m, rc);  // leading all-zero stages are skipped
      double2 dg_next = table ? make_double2(0.0, 1.0) : dg_at(lc0);
      for (int lc = lc0; lc < nlc; ++lc, ++sc) {
        const int stage = sc % ADJ_STAGES;
        const uint32_t round = sc / ADJ_STAGES;
        const int l0 = m + ADJ_LC * lc;
        const bool before = in.ls > l0 + ADJ_LC - 1;
        const bool zero = __all_sync(0xffffffffu, before);
        const bool mixed = __any_sync(0xffffffffu, !before && in.ls + 1 >= l0);
        if (!table) {
          const double2 dg_cur = dg_next;
          if (lc + 1 < nlc) dg_next = dg_at(lc + 1);
          if (!zero) {
            __syncwarp();
            abw[lane] = dg_cur;
            __syncwarp();
          }
        }
        // table mode: each producer warp copies the run of its four M-tiles that
        // holds a started pair in this stage (polar start, padding pairs) -- the
        // consumers never read the others
        uint32_t act = 0;
        if (table) {
          const unsigned bal = __ballot_sync(0xffffffffu, in.ls <= l0 + ADJ_LC - 1 && l0 <= Lt);
#pragma unroll
          for (int t = 0; t < 4; ++t) act |= ((bal >> (8 * t)) & 0xffu) ? (1u << t) : 0u;
        }
        const bool tr = args.trace && blockIdx.x == args.trace_cta && pw == 0 && lane == 0 && sc < 4096;
        if (tr) args.trace[sc * 8 + 0] = clock64();
        mbar_wait(&empty[stage], (round & 1) ^ 1);
        if (tr) args.trace[sc * 8 + 1] = clock64();
        double* Ps = smem + stage * SM::STAGE;
        double* Gs = Ps + ADJ_PTILE;
        if (lane == 0) {
          const int lo = act ? __ffs(act) - 1 : 0, hi = act ? 32 - __clz(act) : 0;
          const uint32_t bytes = (pw == 0 ? SM::GTILE * 8 : 0u) + (uint32_t)(hi - lo) * ADJ_MTILE * 8;
          if (bytes) {
            asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(bytes)
                         : "memory");
            // G tiles are shared by the order's ring chunks (kept in L2), table tiles are read once
            if (pw == 0) bulk_g2s_hint(Gs, Gm + (size_t)lc * SM::GTILE, SM::GTILE * 8, &full[stage], pol_last);
            if (hi > lo)
              bulk_g2s_hint(Ps + (4 * pw + lo) * ADJ_MTILE,
                            args.ptab + (size_t)(args.aofs[m] + (long long)rc * nlc + lc) * ADJ_PTILE +
                                (4 * pw + lo) * ADJ_MTILE,
                            (uint32_t)(hi - lo) * ADJ_MTILE * 8, &full[stage], pol_first);
          }
        }
        // all-zero warps write nothing: the consumers skip their M-tiles (polar start)
        if (zero || table || (args.dbg & 2)) {
        } else if (mixed) {
          adj_produce<true>(Ps, abw, tt, p1, p2, i, g, l0, in);
        } else {
          adj_produce<false>(Ps, abw, tt, p1, p2, i, g, l0, in);
        }
        mbar_arrive(&full[stage]);
        if (tr) args.trace[sc * 8 + 2] = clock64() | ((long long)item << 40);
      }
    }
    return;
  }

  // -------------------------------- consumers --------------------------------
  // warp cw owns M-tiles cw and cw + 8 (pairs 8 cw .. 8 cw + 7 and 64 + 8 cw ..)
  // for both parities and all NT n-tiles; the SM sub-partition cw % 4 thus sees
  // M-tiles {s, s + 4, s + 8, s + 12}, the same mix of polar and equatorial
  // pairs on every sub-partition, so the polar skip shortens the stage instead
  // of idling one sub-partition's DMMA pipe.
  const int cw = consumer_index(warp);
  const int g = lane >> 2, q = lane & 3;
  uint32_t sc = 0;
  const int l16 = lane & 15;
  const int soff = 8 * cw + 64 * (l16 >> 3) + (l16 & 7);
  // polar starts of the warp's pairs, loaded one item ahead (a global-memory round
  // trip at every item start otherwise, with the stages already filled)
  auto start_of = [&](int itg) {
    const int it = itg / ngr;
    return itg < nitems ? __ldg(&args.start_l[(size_t)(args.m_begin + it / args.nrc) * args.nPpad +
                                              (it % args.nrc) * ADJ_RC + soff])
                        : 0;
  };
  int v_next = start_of(blockIdx.x);
  for (int itg = blockIdx.x; itg < nitems; itg += gridDim.x) {
    const int gi = itg % ngr, item = itg / ngr;
    const int m = args.m_begin + item / args.nrc;
    const int rc = item % args.nrc;
    const int fb0 = args.b0 + 4 * gi;  // first field of this item's group
    const int nlc = (Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
    // first degree at which each of the warp's M-tiles has a pair above the polar threshold
    int mt_start[2];
    {
      int v = v_next;
      v_next = start_of(itg + gridDim.x);
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) mt_start[ii] = __shfl_sync(0xffffffffu, v, 8 * ii);
    }
    if (NT > 2 && args.nP - rc * ADJ_RC <= 8 && !args.trace) {
      // a chunk with one M-tile of real pairs: its n-tiles over NT warps (adj_solo_item)
      const AdjSoloOut so{args.S, args.lay, args.n_phi, args.n_theta, args.nfields, args.dbg};
      sc = adj_solo_item<NT>(so, args.pair_n, args.pair_s, Lt, smem, SM::STAGE, full, empty, sc, m, rc, fb0,
                             adj_first_stage(args, m, rc), nlc, cw, lane);
      continue;
    }
    // the epilogue's ring indices, loaded now (their latency hides behind the item's
    // stages instead of sitting between the last DMMA and the stores)
    int ring_n[2], ring_s[2];
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int p = rc * ADJ_RC + (cw + 8 * ii) * 8 + g;
      ring_n[ii] = __ldg(&args.pair_n[p]);
      ring_s[ii] = __ldg(&args.pair_s[p]);
    }
    double acc[2][2][NT][2];  // [parity][M-tile][n-tile][re/im]
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int p2 = 0; p2 < 2; ++p2)
#pragma unroll
        for (int b = 0; b < NT; ++b) acc[a][p2][b][0] = acc[a][p2][b][1] = 0.0;

    for (int lc = adj_first_stage(args, m, rc); lc < nlc; ++lc, ++sc) {
      const int stage = sc % ADJ_STAGES;
      const uint32_t round = sc / ADJ_STAGES;
      const int l0s = m + ADJ_LC * lc;
      const bool tr = args.trace && blockIdx.x == args.trace_cta && (cw == 0 || cw == 3) && lane == 0 && sc < 4096;
      if (tr) args.trace[sc * 8 + (cw == 0 ? 3 : 6)] = clock64();
      mbar_wait(&full[stage], round & 1);
      if (tr && cw == 0) args.trace[sc * 8 + 4] = clock64();
      const double* Ps = smem + stage * SM::STAGE;
      const double* Gs = Ps + ADJ_PTILE;
      const int mts = min(mt_start[0], mt_start[1]);
      if (!(args.dbg & 1) && mts <= min(l0s + ADJ_LC - 1, Lt) && l0s <= Lt) {
        // half-steps t = (k-step ks = t / 2, parity t % 2), fragments double-buffered
        // in registers: the loads of half-step t + 1 are in flight while the DMMAs
        // of half-step t issue
        double a[2][2], b[2][NT];
        auto load = [&](int t, int bufi) {
          const int ks = t >> 1, par = t & 1;
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int i = cw + 8 * ii;
            a[bufi][ii] = lds_f64(&Ps[i * ADJ_MTILE + (par * ADJ_KS + ks) * 32 + adj_swz(g, q, i)]);
          }
#pragma unroll
          for (int jn = 0; jn < NT; ++jn) b[bufi][jn] = lds_f64(&Gs[((par * ADJ_KS + ks) * NT + jn) * 32 + lane]);
        };
        load(0, 0);
        if (mt_start[0] <= l0s + 7 && mt_start[1] <= l0s + 7 && l0s + 8 * (ADJ_KS - 1) <= Lt) {
          // both M-tiles run every k-step (all but the stages on the polar-start boundary
          // and the last degrees): one straight-line run without guarded mma.sync groups
          // (each guard costs a WARPSYNC and a predicate wait)
#pragma unroll
          for (int t = 0; t < 2 * ADJ_KS; ++t) {
            if (t + 1 < 2 * ADJ_KS) load(t + 1, (t + 1) & 1);
            adj_ks_run<0, NT>(acc[t & 1], a[t & 1], b[t & 1]);
          }
        } else
#pragma unroll
        for (int t = 0; t < 2 * ADJ_KS; ++t) {
          if (t + 1 < 2 * ADJ_KS) load(t + 1, (t + 1) & 1);
          // k-step ks holds degrees l0s + 8 ks .. + 7 of both parities.  The active
          // M-tile set is a suffix of {cw, cw + 8} (pairs nearer the equator start
          // earlier); k-steps past Lt hold zero coefficient rows.  Real branches:
          // a predicated-off DMMA still occupies the pipe.
          const int ks = t >> 1, par = t & 1;
          const int khi = min(l0s + 8 * ks + 7, Lt);  // never-started and padding pairs have l_s = Lt + 1
          if (l0s + 8 * ks <= Lt) {
            const bool on0 = mt_start[0] <= khi, on1 = mt_start[1] <= khi;
            if (on0 && on1) adj_ks_run<0, NT>(acc[par], a[t & 1], b[t & 1]);
            else if (on1) adj_ks_run<1, NT>(acc[par], a[t & 1], b[t & 1]);
            else if (on0) adj_ks_run<0, NT, 1>(acc[par], a[t & 1], b[t & 1]);  // the padded last chunk
          }
        }
      }
      if (tr) args.trace[sc * 8 + (cw == 0 ? 5 : 7)] = clock64();
      mbar_arrive(&empty[stage]);
    }

    // epilogue, register-local: north = E + O, south = E - O (bin-major layout:
    // lanes g are 8 consecutive pairs -> 8 consecutive north (south) rings, i.e.
    // 128-byte runs of one bin row).  Column -> (field, comp, sign) and the bin
    // rows depend only on jn and q.
    if (rc * ADJ_RC + 8 * cw < args.nP && !(args.dbg & 4)) {
      const long long bin0 = spec_bin(args.lay, m, 0, args.n_phi), bin1 = spec_bin(args.lay, m, 1, args.n_phi);
      double2* dst[NT];
      long long rbase[NT];
      int comps[NT];
      bool ok[NT];
#pragma unroll
      for (int jn = 0; jn < NT; ++jn) {
        const int ser = 4 * jn + q;  // 6*field + 2*comp + sign
        const int b = ser / 6, comp = (ser % 6) >> 1, sgn = ser & 1;
        ok[jn] = b < args.nfields && !(sgn == 1 && m == 0);
        dst[jn] = args.S + (sgn ? bin1 : bin0) * args.lay.bs;
        comps[jn] = comp;
        rbase[jn] = (long long)(fb0 + b) * args.n_theta;
      }
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        const int rn = ring_n[ii], rs = ring_s[ii];
        if (rn < 0) continue;
#pragma unroll
        for (int jn = 0; jn < NT; ++jn) {
          if (!ok[jn]) continue;
          const double er = acc[0][ii][jn][0], ei = acc[0][ii][jn][1];
          const double orr = acc[1][ii][jn][0], oi = acc[1][ii][jn][1];
          dst[jn][spec_cr(args.lay, comps[jn], rbase[jn] + rn)] = make_double2(er + orr, ei + oi);
          if (rs >= 0) dst[jn][spec_cr(args.lay, comps[jn], rbase[jn] + rs)] = make_double2(er - orr, ei - oi);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Single-field on-the-fly adjoint (NT <= 2: C4, and any one-field call whose
// plan tables do not fit).  With one field the DMMA work per stage is a third
// of C3's, and the producers' recurrence (one dependent chain per lane, ~30
// cycles per step while DMMAs hold the SM sub-partition's FP64 datapath) was
// the critical path: C4 adjoint Legendre 25.6 ms against 18.4 ms for the
// consumers alone.  Here a work item is a PAIR of 128-pair chunks (A, B) of
// one order: every producer lane runs two independent chains (its pair in A
// and in B), and the stage slots alternate A, B, A, B ... (all producer warps
// still touch every slot, so the parity slot waits stay exact); consumers keep
// an accumulator set per chunk and write both epilogues at the item's end.
// ---------------------------------------------------------------------------
template <bool MIXED>
__device__ __forceinline__ void adj_produce2(double* PsA, double* PsB, const double2* dgw, double ttA, double ttB,
                                             double& p1A, double& p2A, double& p1B, double& p2B, int i, int g, int l0,
                                             const Inject& inA, const Inject& inB) {
  const int cx = (g >> 2) | ((i & 1) << 1);
  double* bA[4];
  double* bB[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    bA[q] = PsA + i * ADJ_MTILE + (g << 2) + (q ^ cx);
    bB[q] = PsB + i * ADJ_MTILE + (g << 2) + (q ^ cx);
  }
#pragma unroll
  for (int b0 = 0; b0 < ADJ_LC; b0 += 8) {
    double dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[k] = dgw[b0 + k].x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k;
      const double vA = rec_step<MIXED>(p1A, p2A, ttA, dd[k], l0 + idx, inA);
      const double vB = rec_step<MIXED>(p1B, p2B, ttB, dd[k], l0 + idx, inB);
      const int par = idx & 1, kk = idx >> 1, ks = kk >> 2, q = kk & 3;
      bA[q][(par * ADJ_KS + ks) * 32] = vA;
      bB[q][(par * ADJ_KS + ks) * 32] = vB;
    }
  }
  const double g1 = dgw[ADJ_LC - 1].y, g2 = dgw[ADJ_LC - 2].y;
  p1A *= g1;
  p2A *= g2;
  p1B *= g1;
  p2B *= g2;
}

// one consumer stage (the warp's M-tiles {cw, cw + 8}, both parities), as in legendre_adj_kernel
template <int NT>
__device__ __forceinline__ void adj_consume(const double* Ps, const double* Gs, double (&acc)[2][2][NT][2],
                                            const int (&mt_start)[2], int l0s, int Lt, int cw, int g, int q,
                                            int lane) {
  const int mts = min(mt_start[0], mt_start[1]);
  if (!(mts <= min(l0s + ADJ_LC - 1, Lt) && l0s <= Lt)) return;
  double a[2][2], b[2][NT];
  auto load = [&](int t, int bufi) {
    const int ks = t >> 1, par = t & 1;
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int i = cw + 8 * ii;
      a[bufi][ii] = lds_f64(&Ps[i * ADJ_MTILE + (par * ADJ_KS + ks) * 32 + adj_swz(g, q, i)]);
    }
#pragma unroll
    for (int jn = 0; jn < NT; ++jn) b[bufi][jn] = lds_f64(&Gs[((par * ADJ_KS + ks) * NT + jn) * 32 + lane]);
  };
  load(0, 0);
  if (mt_start[0] <= l0s + 7 && mt_start[1] <= l0s + 7 && l0s + 8 * (ADJ_KS - 1) <= Lt) {
    // both M-tiles run every k-step (all but the stages on the polar-start boundary and the
    // last degrees): one straight-line run, no guarded mma.sync (WARPSYNC + predicate wait each)
#pragma unroll
    for (int t = 0; t < 2 * ADJ_KS; ++t) {
      if (t + 1 < 2 * ADJ_KS) load(t + 1, (t + 1) & 1);
      adj_ks_run<0, NT>(acc[t & 1], a[t & 1], b[t & 1]);
    }
    return;
  }
#pragma unroll
  for (int t = 0; t < 2 * ADJ_KS; ++t) {
    if (t + 1 < 2 * ADJ_KS) load(t + 1, (t + 1) & 1);
    const int ks = t >> 1, par = t & 1;
    const int khi = min(l0s + 8 * ks + 7, Lt);  // never-started and padding pairs have l_s = Lt + 1
    if (l0s + 8 * ks <= Lt) {
      const bool on0 = mt_start[0] <= khi, on1 = mt_start[1] <= khi;
      if (on0 && on1) adj_ks_run<0, NT>(acc[par], a[t & 1], b[t & 1]);
      else if (on1) adj_ks_run<1, NT>(acc[par], a[t & 1], b[t & 1]);
      else if (on0) adj_ks_run<0, NT, 1>(acc[par], a[t & 1], b[t & 1]);  // the padded last chunk
    }
  }
}

// epilogue of one chunk: north = E + O, south = E - O into the spectrum (as in legendre_adj_kernel)
template <int NT>
__device__ __forceinline__ void adj_store(const AdjArgs& args, const double (&acc)[2][2][NT][2], const int (&ring_n)[2],
                                          const int (&ring_s)[2], int m, int q) {
  const long long bin0 = spec_bin(args.lay, m, 0, args.n_phi), bin1 = spec_bin(args.lay, m, 1, args.n_phi);
#pragma unroll
  for (int jn = 0; jn < NT; ++jn) {
    const int ser = 4 * jn + q;  // 6*field + 2*comp + sign
    const int b = ser / 6, comp = (ser % 6) >> 1, sgn = ser & 1;
    if (!(b < args.nfields && !(sgn == 1 && m == 0))) continue;
    double2* dst = args.S + (sgn ? bin1 : bin0) * args.lay.bs;
    const long long rbase = (long long)(args.b0 + b) * args.n_theta;
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int rn = ring_n[ii], rs = ring_s[ii];
      if (rn < 0) continue;
      const double er = acc[0][ii][jn][0], ei = acc[0][ii][jn][1];
      const double orr = acc[1][ii][jn][0], oi = acc[1][ii][jn][1];
      dst[spec_cr(args.lay, comp, rbase + rn)] = make_double2(er + orr, ei + oi);
      if (rs >= 0) dst[spec_cr(args.lay, comp, rbase + rs)] = make_double2(er - orr, ei - oi);
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) legendre_adj_dual_kernel(AdjArgs args) {
  static_assert(NT <= 2, "dual-chunk items are for single-field launches");
  extern __shared__ __align__(128) double smem[];
  using SM = AdjSmem<NT>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ADJ_STAGES * SM::STAGE);
  uint64_t* empty = full + ADJ_STAGES;
  double2* abw_all = reinterpret_cast<double2*>(empty + ADJ_STAGES);
  const int Lt = args.Lt;
  const int nrcp = (args.nrc + 1) / 2;  // chunk pairs per order
  const int nitems = args.m_count * nrcp;
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

  if (is_producer(warp)) {
    const int pw = producer_index(warp);
    double2* abw = abw_all + pw * ADJ_LC;
    const int rho = 32 * pw + lane;
    const int i = rho >> 3, g = rho & 7;
    const uint64_t pol_last = l2_evict_last();
    uint32_t sc = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const int m = args.m_begin + item / nrcp;
      const int rcA = 2 * (item % nrcp);
      const bool hasB = rcA + 1 < args.nrc;
      const int nlc = (Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
      const int pA = rcA * ADJ_RC + rho, pB = hasB ? pA + ADJ_RC : pA;
      const double ttA = args.pair_t[pA], ttB = args.pair_t[pB];
      Inject inA, inB;
      inA.ls = args.start_l[(size_t)m * args.nPpad + pA];
      inB.ls = hasB ? args.start_l[(size_t)m * args.nPpad + pB] : Lt + ADJ_LC + 1;  // absent: never starts
      {
        const double2 vA = args.start_v[(size_t)m * args.nPpad + pA];
        const double2 vB = args.start_v[(size_t)m * args.nPpad + pB];
        inA.A = vA.x;
        inA.B = vA.y;
        inB.A = vB.x;
        inB.B = vB.y;
      }
      double p1A = 0.0, p2A = 0.0, p1B = 0.0, p2B = 0.0;
      const double2* dgm = args.dg + args.dgofs[m];
      const double* Gm = args.G + (size_t)args.gofs[m] * SM::GTILE;
      auto dg_at = [&](int lcx) {
        const int l = m + ADJ_LC * lcx + lane;
        return (l <= Lt) ? __ldg(&dgm[l - m]) : make_double2(0.0, 1.0);
      };
      const int lc0 = hasB ? min(adj_first_stage(args, m, rcA), adj_first_stage(args, m, rcA + 1))
                           : adj_first_stage(args, m, rcA);
      double2 dg_next = dg_at(lc0);
      for (int lc = lc0; lc < nlc; ++lc) {
        const int l0 = m + ADJ_LC * lc;
        const bool beforeA = inA.ls > l0 + ADJ_LC - 1, beforeB = inB.ls > l0 + ADJ_LC - 1;
        const bool zeroA = __all_sync(0xffffffffu, beforeA), zeroB = __all_sync(0xffffffffu, beforeB);
        const bool mixed = __any_sync(0xffffffffu, (!beforeA && inA.ls + 1 >= l0) || (!beforeB && inB.ls + 1 >= l0));
        const double2 dg_cur = dg_next;
        if (lc + 1 < nlc) dg_next = dg_at(lc + 1);
        if (!zeroA || !zeroB) {
          __syncwarp();
          abw[lane] = dg_cur;
          __syncwarp();
        }
        const int sA = sc % ADJ_STAGES;
        mbar_wait(&empty[sA], ((sc / ADJ_STAGES) & 1) ^ 1);
        const uint32_t scB = sc + 1;
        const int sB = scB % ADJ_STAGES;
        if (hasB) mbar_wait(&empty[sB], ((scB / ADJ_STAGES) & 1) ^ 1);
        double* PsA = smem + sA * SM::STAGE;
        double* PsB = smem + sB * SM::STAGE;
        if (lane == 0 && pw == 0) {
          // the order's coefficient tile of this degree block, once per chunk slot
          asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[sA])),
                       "r"((uint32_t)(SM::GTILE * 8))
                       : "memory");
          bulk_g2s_hint(PsA + ADJ_PTILE, Gm + (size_t)lc * SM::GTILE, SM::GTILE * 8, &full[sA], pol_last);
          if (hasB) {
            asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[sB])),
                         "r"((uint32_t)(SM::GTILE * 8))
                         : "memory");
            bulk_g2s_hint(PsB + ADJ_PTILE, Gm + (size_t)lc * SM::GTILE, SM::GTILE * 8, &full[sB], pol_last);
          }
        }
        if (!(args.dbg & 2)) {
          if (!zeroA && !zeroB) {
            if (mixed) adj_produce2<true>(PsA, PsB, abw, ttA, ttB, p1A, p2A, p1B, p2B, i, g, l0, inA, inB);
            else adj_produce2<false>(PsA, PsB, abw, ttA, ttB, p1A, p2A, p1B, p2B, i, g, l0, inA, inB);
          } else if (!zeroA) {
            if (mixed) adj_produce<true>(PsA, abw, ttA, p1A, p2A, i, g, l0, inA);
            else adj_produce<false>(PsA, abw, ttA, p1A, p2A, i, g, l0, inA);
          } else if (!zeroB) {
            if (mixed) adj_produce<true>(PsB, abw, ttB, p1B, p2B, i, g, l0, inB);
            else adj_produce<false>(PsB, abw, ttB, p1B, p2B, i, g, l0, inB);
          }
        }
        mbar_arrive(&full[sA]);
        if (hasB) mbar_arrive(&full[sB]);
        sc += hasB ? 2 : 1;
      }
    }
    return;
  }

  const int cw = consumer_index(warp);
  const int g = lane >> 2, q = lane & 3;
  uint32_t sc = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int m = args.m_begin + item / nrcp;
    const int rcA = 2 * (item % nrcp);
    const bool hasB = rcA + 1 < args.nrc;
    const int nlc = (Lt + 1 - m + ADJ_LC - 1) / ADJ_LC;
    int mtA[2], mtB[2], rnA[2], rsA[2], rnB[2], rsB[2];
    {
      const int l16 = lane & 15;
      const int off = 8 * cw + 64 * (l16 >> 3) + (l16 & 7);
      int vA = args.start_l[(size_t)m * args.nPpad + rcA * ADJ_RC + off];
      int vB = hasB ? args.start_l[(size_t)m * args.nPpad + (rcA + 1) * ADJ_RC + off] : Lt + ADJ_LC + 1;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        vA = min(vA, __shfl_xor_sync(0xffffffffu, vA, o));
        vB = min(vB, __shfl_xor_sync(0xffffffffu, vB, o));
      }
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        mtA[ii] = __shfl_sync(0xffffffffu, vA, 8 * ii);
        mtB[ii] = __shfl_sync(0xffffffffu, vB, 8 * ii);
      }
    }
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int p = rcA * ADJ_RC + (cw + 8 * ii) * 8 + g;
      rnA[ii] = __ldg(&args.pair_n[p]);
      rsA[ii] = __ldg(&args.pair_s[p]);
      rnB[ii] = hasB ? __ldg(&args.pair_n[p + ADJ_RC]) : -1;
      rsB[ii] = hasB ? __ldg(&args.pair_s[p + ADJ_RC]) : -1;
    }
    double accA[2][2][NT][2], accB[2][2][NT][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int p2 = 0; p2 < 2; ++p2)
#pragma unroll
        for (int b = 0; b < NT; ++b) accA[a][p2][b][0] = accA[a][p2][b][1] = accB[a][p2][b][0] = accB[a][p2][b][1] = 0.0;
    const int lc0 = hasB ? min(adj_first_stage(args, m, rcA), adj_first_stage(args, m, rcA + 1))
                         : adj_first_stage(args, m, rcA);
    for (int lc = lc0; lc < nlc; ++lc) {
      const int l0s = m + ADJ_LC * lc;
      {
        const int stage = sc % ADJ_STAGES;
        mbar_wait(&full[stage], (sc / ADJ_STAGES) & 1);
        const double* Ps = smem + stage * SM::STAGE;
        if (!(args.dbg & 1)) adj_consume<NT>(Ps, Ps + ADJ_PTILE, accA, mtA, l0s, Lt, cw, g, q, lane);
        mbar_arrive(&empty[stage]);
        ++sc;
      }
      if (hasB) {
        const int stage = sc % ADJ_STAGES;
        mbar_wait(&full[stage], (sc / ADJ_STAGES) & 1);
        const double* Ps = smem + stage * SM::STAGE;
        if (!(args.dbg & 1)) adj_consume<NT>(Ps, Ps + ADJ_PTILE, accB, mtB, l0s, Lt, cw, g, q, lane);
        mbar_arrive(&empty[stage]);
        ++sc;
      }
    }
    if (!(args.dbg & 4)) {
      if (rcA * ADJ_RC + 8 * cw < args.nP) adj_store<NT>(args, accA, rnA, rsA, m, q);
      if (hasB && (rcA + 1) * ADJ_RC + 8 * cw < args.nP) adj_store<NT>(args, accB, rnB, rsB, m, q);
    }
  }
}

}  // namespace fv
