// C ABI (include/favest_b200.h): plans, workspaces, cuFFT and the kernel
// sequence of the forward / adjoint VSHT on B200 (sm_100a).
#include <cuda_runtime.h>
#include <cufft.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <type_traits>
#include <map>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "../../include/favest_b200.h"
#include "../../include/favest_io.h"
#include "aux_kernels.cuh"
#include "fft.cuh"
#include "fft2.cuh"
#include "fft_blue.cuh"
#include "fft_rader.cuh"
#include "legendre.cuh"
#include "points.cuh"
#include "quadrature.cuh"
#include "scalar.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define FV_CUDA(x)                                                                            \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? FV_ENOMEM : FV_ECUDA,                    \
                  std::string("CUDA error in ") + #x + ": " + cudaGetErrorString(e_));        \
    }                                                                                         \
  } while (0)

#define FV_CUFFT(x)                                                                           \
  do {                                                                                        \
    cufftResult r_ = (x);                                                                     \
    if (r_ != CUFFT_SUCCESS) {                                                                \
      return fail(r_ == CUFFT_ALLOC_FAILED ? FV_ENOMEM : FV_ECUDA,                            \
                  std::string("cuFFT error ") + std::to_string((int)r_) + " in " + #x);       \
    }                                                                                         \
  } while (0)

#define FV_TRY(x)          \
  do {                     \
    int rc_ = (x);         \
    if (rc_ != FV_OK) return rc_; \
  } while (0)

// FV_DEBUG_MODE=1/2 isolates the consumer / producer halves of the Legendre kernels (timing only)
int dbg_mode() {
  static int v = [] { const char* e = std::getenv("FV_DEBUG_MODE"); return e ? std::atoi(e) : 0; }();
  return v;
}

// FV_TRACE_CTA=<m> records the forward pipeline timeline of that CTA (tools/trace_fwd.py)
long long* g_trace = nullptr;
int trace_cta() {
  static int v = [] { const char* e = std::getenv("FV_TRACE_CTA"); return e ? std::atoi(e) : -1; }();
  return v;
}
long long* trace_buf() {
  if (trace_cta() < 0) return nullptr;
  if (!g_trace) {
    cudaMalloc(&g_trace, 4096 * 12 * sizeof(long long));
    cudaMemset(g_trace, 0, 4096 * 12 * sizeof(long long));  // forward: 4096 x 8 + CTA records; adjoint: 4096 x 8 + 4096 x 2
  }
  return g_trace;
}

inline int ntiles_for(int nfields) { return (12 * nfields + 7) / 8; }

}  // namespace

struct fvPlan {
  int kind = 0;  // 0 grid, 1 points
  int L = 0, Lt = 0, n_theta = 0, n_phi = 0, nP = 0, nPpad = 0, nchunks = 0, nrc = 0;
  int max_batch = 0, device = 0, paired = 0, num_sms = 148;
  fv::SLayout lay_f{}, lay_a{};  // ring-spectrum layouts of the forward / adjoint (fixed for any B <= max_batch)
  // grid tables
  double* pair_t = nullptr;
  double* pair_sin = nullptr;
  int* pair_n = nullptr;
  int* pair_s = nullptr;
  double* ring_w = nullptr;
  double* seed_x = nullptr;  // plan-time only (freed after the polar-start tables)
  int* seed_e = nullptr;
  int* start_l = nullptr;
  int* cmin = nullptr;          // [m][forward chunk] smallest polar start of the chunk's pairs
  int* cmin_a = nullptr;        // [m][adjoint 128-pair chunk]
  double2* start_v = nullptr;
  double2* ab = nullptr;
  long long* abofs = nullptr;
  double* cgt = nullptr;        // Clebsch-Gordan factors xi1..6, mu1..3 (9 x K_t)
  double* cga = nullptr;        // the same factors in G-row order for the adjoint (9 x 2 signs x 32 g_tiles)
  double2* dg = nullptr;        // block-rescaled recurrence (d, gamma) (grid plans)
  long long* dgofs = nullptr;
  // table mode: plan-time Legendre tiles streamed by TMA instead of the on-the-fly producer
  double* ptab_f = nullptr;
  double2* fseed = nullptr;   // legendre_fwd2_kernel: recurrence state at every forward tile start (fseed_tables)
  fv::StageMeta* mtab_f = nullptr;
  long long* tofs = nullptr;
  double* ptab_a = nullptr;
  long long* aofs = nullptr;
  size_t ptab_bytes = 0;
  long long* gofs = nullptr;    // tile offsets per order (grid G layout)
  long long* rowofs = nullptr;  // row offsets per order (points G layout)
  // direct forward at points (points plans, allocated on the first fv_forward_points)
  double* seedk = nullptr;      // K_m = Pbar_m^m / (-s)^m
  int2* fitems = nullptr;       // (order, 128-degree window), heaviest first
  int n_fitems = 0;
  double* Fpart = nullptr;      // point-range partial rows [R][tri(Lt)][ncol]
  double* Tp = nullptr;         // scalar transforms: pseudo fields [K][n][3]
  size_t Tp_cap = 0;
  size_t Fpart_cap = 0, F_cap = 0;
  long long g_tiles = 0;
  // workspaces
  double2* Sf = nullptr;        // ring spectra [comp][bin][ring of all max_batch fields] (ring fastest)
  double2* Sa = nullptr;
  double* X = nullptr;
  double* F = nullptr;
  double* Fx = nullptr;  // partial F buffers 1..3 of split forward launches (lazily, 3 x f_gstride)
  double* G = nullptr;
  int ngroups_buf = 1;                            // 4-field groups whose X / F / G fit side by side
  size_t x_gstride = 0, f_gstride = 0, g_gstride = 0;  // doubles per group
  std::map<std::tuple<long long, long long, long long, long long, int>, cufftHandle> ffts;  // strided cuFFT plans
  // hand-written ring FFT (fft.cuh) when every prime factor of n_phi is <= 19
  bool custom_fft = false;
  // Bluestein ring FFT (fft_blue.cuh) for n_phi = R * P with a prime P > 19
  bool smallp = false, rpfft = false;
  bool rader = false;        // n_phi = R * P by Rader's algorithm (fft_rader.cuh), tables in blue_tab
  int rader_R = 0, rader_P = 0;
  fv::RaderArgs rd_args{};
  std::map<std::tuple<long long, long long, int>, cufftHandle> subffts;  // length-P sub-DFT plans (rpfft)
  fv::BlueArgs blue_args{};  // tables and factorisation (pointers owned below)
  fv::SmallPArgs sp_args{};
  double2* blue_tab = nullptr;
  double2* blue_s1 = nullptr;
  size_t blue_s1_cap = 0;
  int fft_nst = 0;
  int fft_radix[fv::FFT_MAXST] = {};
  double2* fft_tw = nullptr;
  // two-ring FFT (fft2.cuh): radix plan, per-stage twiddle tables; fused forward fold
  bool fft2 = false, fused_fold = false;
  int f2_nst = 0;
  int f2_radix[fv::FFT_MAXST] = {};
  double2* f2_tw = nullptr;
  // profiling
  bool profiling = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace {

template <typename T>
int dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  FV_CUDA(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  return FV_OK;
}

void free_plan(fvPlan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  void* ptrs[] = {p->pair_t, p->pair_sin, p->pair_n, p->pair_s, p->ring_w, p->seed_x,
                  p->seed_e, p->start_l,  p->start_v, p->ab,   p->abofs,  p->gofs,
                  p->dg,     p->dgofs,  p->cgt,     p->cga,     p->ptab_f,  p->mtab_f, p->tofs,   p->ptab_a, p->aofs, p->fseed,
                  p->rowofs, p->Sf,       p->Sa,      p->X,    p->F,      p->Fx,     p->G,
                  p->seedk,  p->fitems,   p->Fpart,   p->blue_tab, p->blue_s1, p->cmin, p->cmin_a, p->Tp,
                  p->fft_tw, p->f2_tw};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (auto& kv : p->ffts) cufftDestroy(kv.second);
  for (auto& kv : p->subffts) cufftDestroy(kv.second);
  for (auto e : p->ev_pool) cudaEventDestroy(e);
  delete p;
}

int ab_tables(fvPlan* p) {
  const int Lt = p->Lt;
  std::vector<long long> abofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m) abofs[m + 1] = abofs[m] + std::max(0, Lt - m - 1);
  FV_TRY(dalloc(&p->abofs, Lt + 1));
  FV_TRY(dalloc(&p->ab, abofs[Lt + 1]));
  FV_CUDA(cudaMemcpy(p->abofs, abofs.data(), (Lt + 1) * sizeof(long long), cudaMemcpyHostToDevice));
  if (Lt >= 2) {
    dim3 grid((Lt + 127) / 128, Lt + 1);
    fv::ab_kernel<<<grid, 128>>>(Lt, p->abofs, p->ab);
    FV_CUDA(cudaGetLastError());
  }
  return FV_OK;
}

int cg_tables(fvPlan* p) {
  const long long Kt = (long long)(p->Lt + 1) * (p->Lt + 1);
  FV_TRY(dalloc(&p->cgt, (size_t)(9 * Kt)));
  fv::cg_table_kernel<<<(unsigned)((Kt + 255) / 256), 256>>>(p->Lt, p->cgt);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

int dg_tables(fvPlan* p) {
  const int Lt = p->Lt;
  std::vector<long long> ofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m) ofs[m + 1] = ofs[m] + (Lt + 1 - m);
  FV_TRY(dalloc(&p->dgofs, Lt + 1));
  FV_TRY(dalloc(&p->dg, ofs[Lt + 1]));
  FV_CUDA(cudaMemcpy(p->dgofs, ofs.data(), (Lt + 1) * sizeof(long long), cudaMemcpyHostToDevice));
  dim3 grid((Lt + 1 + 31) / 32, Lt + 1);
  fv::dg_kernel<<<grid, 32>>>(Lt, p->dgofs, p->dg);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

// Table mode (legendre.cuh): precompute every forward tile and adjoint stage tile
// once per plan when they fit the budget FV_PTAB_GB (default 32 GB; FV_PTAB=0
// disables).  At L=1024 this is ~5 GB; at L=4096 it would be ~250 GB, so large
// degrees keep the on-the-fly recurrence producer.
int ptab_tables(fvPlan* p) {
  const char* en = std::getenv("FV_PTAB");
  if (en && std::atoi(en) == 0) return FV_OK;
  const char* gb = std::getenv("FV_PTAB_GB");
  const double budget = (gb ? std::atof(gb) : 32.0) * 1e9;
  const int Lt = p->Lt;
  std::vector<long long> tofs(Lt + 2, 0), aofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m) {
    tofs[m + 1] = tofs[m] + (long long)((Lt + 1 - m + fv::FWD_LB - 1) / fv::FWD_LB) * p->nchunks;
    aofs[m + 1] = aofs[m] + (long long)((Lt + 1 - m + fv::ADJ_LC - 1) / fv::ADJ_LC) * p->nrc;
  }
  const size_t bytes = (size_t)tofs[Lt + 1] * (fv::FWD_PTILE * 8 + sizeof(fv::StageMeta)) +
                       (size_t)aofs[Lt + 1] * fv::ADJ_PTILE * 8;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  if ((double)bytes > budget || bytes > free_b / 2) return FV_OK;
  FV_TRY(dalloc(&p->tofs, Lt + 1));
  FV_TRY(dalloc(&p->aofs, Lt + 1));
  FV_TRY(dalloc(&p->ptab_f, (size_t)tofs[Lt + 1] * fv::FWD_PTILE));
  FV_TRY(dalloc(&p->mtab_f, (size_t)tofs[Lt + 1]));
  FV_TRY(dalloc(&p->ptab_a, (size_t)aofs[Lt + 1] * fv::ADJ_PTILE));
  FV_CUDA(cudaMemcpy(p->tofs, tofs.data(), (Lt + 1) * 8, cudaMemcpyHostToDevice));
  FV_CUDA(cudaMemcpy(p->aofs, aofs.data(), (Lt + 1) * 8, cudaMemcpyHostToDevice));
  fv::FwdArgs fa{};
  fa.start_l = p->start_l;
  fa.start_v = p->start_v;
  fa.dg = p->dg;
  fa.dgofs = p->dgofs;
  fa.pair_t = p->pair_t;
  fa.Lt = Lt;
  fa.nP = p->nP;
  fa.nPpad = p->nPpad;
  fa.nchunks = p->nchunks;
  fa.tofs = p->tofs;
  const size_t smem_f = fv::kProducerWarps * fv::FWD_LB * 16 + (size_t)p->nchunks * fv::FWD_RC * 28;
  FV_CUDA(cudaFuncSetAttribute(fv::ptab_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f));
  fv::ptab_fwd_kernel<<<Lt + 1, 32 * fv::kProducerWarps, smem_f>>>(fa, p->ptab_f, p->mtab_f);
  FV_CUDA(cudaGetLastError());
  fv::AdjArgs aa{};
  aa.start_l = p->start_l;
  aa.start_v = p->start_v;
  aa.dg = p->dg;
  aa.dgofs = p->dgofs;
  aa.pair_t = p->pair_t;
  aa.Lt = Lt;
  aa.nP = p->nP;
  aa.nPpad = p->nPpad;
  aa.nrc = p->nrc;
  aa.aofs = p->aofs;
  fv::ptab_adj_kernel<<<(Lt + 1) * p->nrc, 32 * fv::kProducerWarps>>>(aa, p->ptab_a);
  FV_CUDA(cudaGetLastError());
  p->ptab_bytes = bytes;
  return FV_OK;
}

// On-the-fly plans (no Legendre tables: large L): the recurrence state of every pair at
// every forward tile start, for the single-field forward with two chains per producer lane
// (legendre.cuh legendre_fwd2_kernel).  16 bytes per (order, l-block, pair): 4.4 GB at
// L = 4096; skipped past FV_FSEED_GB (default 16) or half of the free memory, and with
// FV_FWD2=0.
int fseed_tables(fvPlan* p) {
  if (p->ptab_f) return FV_OK;
  const char* en = std::getenv("FV_FWD2");
  if (en && std::atoi(en) == 0) return FV_OK;
  const char* gb = std::getenv("FV_FSEED_GB");
  const double budget = (gb ? std::atof(gb) : 16.0) * 1e9;
  const int Lt = p->Lt;
  std::vector<long long> tofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m)
    tofs[m + 1] = tofs[m] + (long long)((Lt + 1 - m + fv::FWD_LB - 1) / fv::FWD_LB) * p->nchunks;
  const size_t bytes = (size_t)tofs[Lt + 1] * 32 * sizeof(double2);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  if ((double)bytes > budget || bytes > free_b / 2) return FV_OK;
  const size_t smem = (size_t)fv::kProducerWarps * fv::FWD_PTILE * 8 + fv::kProducerWarps * fv::FWD_LB * 16 +
                      (size_t)p->nchunks * fv::FWD_RC * 28;
  if (smem > 227 * 1024) return FV_OK;
  if (!p->tofs) {
    FV_TRY(dalloc(&p->tofs, Lt + 1));
    FV_CUDA(cudaMemcpy(p->tofs, tofs.data(), (Lt + 1) * 8, cudaMemcpyHostToDevice));
  }
  FV_TRY(dalloc(&p->fseed, (size_t)tofs[Lt + 1] * 32));
  fv::FwdArgs fa{};
  fa.start_l = p->start_l;
  fa.start_v = p->start_v;
  fa.dg = p->dg;
  fa.dgofs = p->dgofs;
  fa.pair_t = p->pair_t;
  fa.Lt = Lt;
  fa.nP = p->nP;
  fa.nPpad = p->nPpad;
  fa.nchunks = p->nchunks;
  fa.tofs = p->tofs;
  FV_CUDA(cudaFuncSetAttribute(fv::fseed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fv::fseed_kernel<<<Lt + 1, 32 * fv::kProducerWarps, smem>>>(fa, p->fseed);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

cudaEvent_t next_event(fvPlan* p) {
  if (p->ev_used == p->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p->ev_pool.push_back(e);
  }
  return p->ev_pool[p->ev_used++];
}

// One pipeline stage's launches: an NVTX range on the host (fv:fft, fv:fold,
// fv:legendre, fv:cg -- visible in nsys / ncu --nvtx timelines; a no-op without a
// tool attached) and, with profiling on, CUDA events on the stream.
struct StageMark {
  fvPlan* p;
  int stage;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr;
  StageMark(fvPlan* p_, int st, cudaStream_t s_) : p(p_), stage(st), s(s_) {
    static const char* const names[] = {"fv:fft", "fv:fold", "fv:legendre", "fv:cg"};
    nvtxRangePushA(names[st & 3]);
    if (p->profiling) {
      e0 = next_event(p);
      cudaEventRecord(e0, s);
    }
  }
  ~StageMark() {
    if (p->profiling) {
      cudaEvent_t e1 = next_event(p);
      cudaEventRecord(e1, s);
      p->marks.push_back({stage, {e0, e1}});
    }
    nvtxRangePop();
  }
};

// cuFFT fallback (lengths with a prime factor > 19): one strided batched plan per
// (strides, ring count), cached in the plan; components are separate executions
int get_fft_strided(fvPlan* p, long long irs, long long ies, long long ors, long long oes, int nrings, cufftHandle* h) {
  const auto key = std::make_tuple(irs, ies, ors, oes, nrings);
  auto it = p->ffts.find(key);
  if (it == p->ffts.end()) {
    int n = p->n_phi;
    cufftHandle hh;
    FV_CUFFT(cufftPlanMany(&hh, 1, &n, &n, (int)ies, (int)irs, &n, (int)oes, (int)ors, CUFFT_Z2Z, nrings));
    it = p->ffts.emplace(key, hh).first;
  }
  *h = it->second;
  return FV_OK;
}

// Opt a kernel into 227 KB of dynamic shared memory once per (kernel
// instantiation, device).  The device's bit is published only after the
// attribute call succeeded (a failure is retried by the next launch), and with
// release / acquire ordering, so a second host thread never launches before
// the attribute is set; two threads racing on the first launch both make the
// (idempotent) call.
template <class K>
cudaError_t smem_optin_once(std::atomic<unsigned long long>* mask, int device, K kernel) {
  const unsigned long long bit = 1ull << (device & 63);
  if (mask->load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) mask->fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int NT>
int launch_fwd(fvPlan* p, const fv::FwdArgs& args, int m_count, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0}, attr_split{0};
  const size_t bytes = fv::FwdSmem<NT>::bytes(p->nchunks * fv::FWD_RC);
  if (bytes > 227 * 1024) return fail(FV_EINVAL, "grid too large for the forward kernel's shared memory");
  fv::FwdArgs a2 = args;
  a2.m_count = m_count;
  // one CTA per order (and split): the hardware block scheduler hands out orders in
  // ascending m (descending work) dynamically, which balances better than a static
  // persistent split
  const unsigned grid = (unsigned)(m_count * std::max(1, a2.ngroups) * std::max(1, a2.ksplit));
  if constexpr (NT <= 2) {
    // single field on the fly with plan-time seeds: two recurrence chains per producer lane
    if (!a2.ptab && p->fseed) {
      static std::atomic<unsigned long long> attr2{0}, attr2_split{0};
      a2.seed = p->fseed;
      a2.tofs = p->tofs;
      const size_t b2 = fv::Fwd2Smem<NT>::bytes;
      if (a2.ksplit > 1) {
        FV_CUDA(smem_optin_once(&attr2_split, p->device, fv::legendre_fwd2_kernel<NT, true>));
        fv::legendre_fwd2_kernel<NT, true><<<grid, fv::kThreads, b2, s>>>(a2);
      } else {
        FV_CUDA(smem_optin_once(&attr2, p->device, fv::legendre_fwd2_kernel<NT, false>));
        fv::legendre_fwd2_kernel<NT, false><<<grid, fv::kThreads, b2, s>>>(a2);
      }
      FV_CUDA(cudaGetLastError());
      return FV_OK;
    }
  }
  if (a2.ksplit > 1) {
    FV_CUDA(smem_optin_once(&attr_split, p->device, fv::legendre_fwd_kernel<NT, true>));
    fv::legendre_fwd_kernel<NT, true><<<grid, fv::kThreads, bytes, s>>>(a2);
  } else {
    FV_CUDA(smem_optin_once(&attr, p->device, fv::legendre_fwd_kernel<NT, false>));
    fv::legendre_fwd_kernel<NT, false><<<grid, fv::kThreads, bytes, s>>>(a2);
  }
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

template <int NT>
int launch_adj(fvPlan* p, const fv::AdjArgs& args, int m_count, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  const size_t bytes = fv::AdjSmem<NT>::bytes();
  FV_CUDA(smem_optin_once(&attr, p->device, fv::legendre_adj_kernel<NT>));
  if (bytes > 227 * 1024) return fail(FV_EINVAL, "adjoint kernel shared memory exceeds 227 KB");
  fv::AdjArgs a2 = args;
  a2.m_count = m_count;
  if constexpr (NT <= 2) {
    // single field on the fly: items of two ring chunks, two recurrence chains per producer lane
    // (FV_ADJ_DUAL=0 keeps one chunk per item)
    static const bool dual = [] { const char* e = std::getenv("FV_ADJ_DUAL"); return !(e && std::atoi(e) == 0); }();
    if (dual && !args.ptab) {
      static std::atomic<unsigned long long> attr2{0};
      FV_CUDA(smem_optin_once(&attr2, p->device, fv::legendre_adj_dual_kernel<NT>));
      const int items2 = m_count * ((p->nrc + 1) / 2);
      fv::legendre_adj_dual_kernel<NT><<<std::min(items2, p->num_sms), fv::kThreads, bytes, s>>>(a2);
      FV_CUDA(cudaGetLastError());
      return FV_OK;
    }
  }
  const int items = m_count * p->nrc * std::max(1, a2.ngroups);
  fv::legendre_adj_kernel<NT><<<std::min(items, p->num_sms), fv::kThreads, bytes, s>>>(a2);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

int dispatch_fwd(fvPlan* p, int NT, const fv::FwdArgs& a, int mc, cudaStream_t s) {
  switch (NT) {
    case 2: return launch_fwd<2>(p, a, mc, s);
    case 3: return launch_fwd<3>(p, a, mc, s);
    case 5: return launch_fwd<5>(p, a, mc, s);
    case 6: return launch_fwd<6>(p, a, mc, s);
  }
  return fail(FV_EINVAL, "unsupported field group");
}

int dispatch_adj(fvPlan* p, int NT, const fv::AdjArgs& a, int mc, cudaStream_t s) {
  switch (NT) {
    case 2: return launch_adj<2>(p, a, mc, s);
    case 3: return launch_adj<3>(p, a, mc, s);
    case 5: return launch_adj<5>(p, a, mc, s);
    case 6: return launch_adj<6>(p, a, mc, s);
  }
  return fail(FV_EINVAL, "unsupported field group");
}

// radix sequence for the hand-written FFT: each prime 11..19 is its own stage;
// the small primes (2, 3, 5, 7) are packed greedily into composite radices
// <= 16 (fewer, fatter stages: fewer shared-memory passes and barriers).
// Largest radix first: the first stage has no twiddles.
bool fft_factor(int n, int* radix, int* nst) {
  if (n < 2 || n > fv::FFT_NMAX) return false;
  std::vector<int> small, out;
  for (int p : {2, 3, 5, 7, 11, 13, 17, 19})
    while (n % p == 0) {
      (p <= 7 ? small : out).push_back(p);
      n /= p;
    }
  if (n != 1) return false;
  std::sort(small.begin(), small.end(), std::greater<int>());
  while (!small.empty()) {
    int r = small.front();
    small.erase(small.begin());
    for (bool grew = true; grew;) {
      grew = false;
      for (size_t i = 0; i < small.size(); ++i)
        if (r * small[i] <= 16) {
          r *= small[i];
          small.erase(small.begin() + i);
          grew = true;
          break;
        }
    }
    out.push_back(r);
  }
  std::sort(out.begin(), out.end(), std::greater<int>());
  if ((int)out.size() > fv::FFT_MAXST) return false;
  for (size_t i = 0; i < out.size(); ++i) radix[i] = out[i];
  *nst = (int)out.size();
  return true;
}

// roots of the odd-prime butterflies and the composites' internal twiddles
// (per device: __constant__ lives in each context)
int fill_root_tables() {
  double rc[sizeof(fv::kRootCos) / sizeof(double)], rs[sizeof(fv::kRootSin) / sizeof(double)];
  for (int R : fv::kRootR)
    for (int m = 0; m < R; ++m) {
      const long double a = 2.0L * 3.141592653589793238462643383279502884L * m / R;
      rc[fv::root_offset(R) + m] = (double)cosl(a);
      rs[fv::root_offset(R) + m] = (double)sinl(a);
    }
  FV_CUDA(cudaMemcpyToSymbol(fv::kRootCos, rc, sizeof(rc)));
  FV_CUDA(cudaMemcpyToSymbol(fv::kRootSin, rs, sizeof(rs)));
  double cc[sizeof(fv::kCompCos) / sizeof(double)], cs[sizeof(fv::kCompSin) / sizeof(double)];
  for (int R : fv::kCompR)
    for (int e = 0; e < R; ++e) {
      const long double a = 2.0L * 3.141592653589793238462643383279502884L * e / R;
      cc[fv::comp_offset(R) + e] = (double)cosl(a);
      cs[fv::comp_offset(R) + e] = (double)sinl(a);
    }
  FV_CUDA(cudaMemcpyToSymbol(fv::kCompCos, cc, sizeof(cc)));
  FV_CUDA(cudaMemcpyToSymbol(fv::kCompSin, cs, sizeof(cs)));
  return FV_OK;
}

int setup_fft(fvPlan* p) {
  const char* env = std::getenv("FV_FFT");
  const bool force_cufft = env && std::string(env) == "cufft";
  if (force_cufft || !fft_factor(p->n_phi, p->fft_radix, &p->fft_nst)) return FV_OK;
  FV_TRY(fill_root_tables());
  // factored twiddles: lo[k] = w^k (k < 64), hi[j] = w^(64 j)
  const int nhi = (p->n_phi + fv::FFT_TWLO - 1) / fv::FFT_TWLO;
  std::vector<double2> tw(fv::FFT_TWLO + nhi);
  for (int k = 0; k < (int)tw.size(); ++k) {
    const long long e = k < fv::FFT_TWLO ? k : (long long)fv::FFT_TWLO * (k - fv::FFT_TWLO);
    const long double a = 2.0L * 3.141592653589793238462643383279502884L * e / p->n_phi;
    tw[k] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  FV_TRY(dalloc(&p->fft_tw, tw.size()));
  FV_CUDA(cudaMemcpy(p->fft_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  const size_t smem = (3 * (size_t)p->n_phi + fv::FFT_TWN) * sizeof(double2);
  FV_CUDA(cudaFuncSetAttribute(fv::ring_fft_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  FV_CUDA(cudaFuncSetAttribute(fv::ring_fft_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  p->custom_fft = true;
  return FV_OK;
}

// Radix plan of the two-ring kernel (fft2.cuh): radices 2..20, each stage's
// butterflies (2 n / R of them) spread over F2_T threads with at most f2_kb(R)
// per thread (they are held in registers across the in-place barrier).  Cost
// model: per-thread butterfly work  sum_s ceil(2n / (R_s T)) R_s (2 + log2 R_s)
// plus a fixed cost per stage (barrier, shared-memory pass); minimised by DP over
// the divisors of n.  Largest radix first (the first stage has no twiddles).
bool fft2_factor(int n, int* radix, int* nst) {
  if (n < 2 || 2 * (size_t)n * sizeof(double2) > 110 * 1024) return false;
  std::map<int, std::pair<double, int>> best;  // remaining length -> (cost, first radix)
  std::function<double(int)> solve = [&](int m) -> double {
    if (m == 1) return 0.0;
    auto it = best.find(m);
    if (it != best.end()) return it->second.first;
    double bc = 1e300;
    int br = 0;
    for (int R = 2; R <= 20; ++R) {
      if (m % R) continue;
      const int kb = (2 * n / R + fv::F2_T - 1) / fv::F2_T;
      if (kb > fv::f2_kb_rt(R)) continue;
      const double c = kb * R * (2.0 + std::log2((double)R)) + 40.0 + solve(m / R);
      if (c < bc) {
        bc = c;
        br = R;
      }
    }
    best[m] = {bc, br};
    return bc;
  };
  if (solve(n) >= 1e299) return false;
  std::vector<int> out;
  for (int m = n; m > 1; m /= best[m].second) out.push_back(best[m].second);
  if ((int)out.size() > fv::FFT_MAXST) return false;
  std::sort(out.begin(), out.end(), std::greater<int>());
  for (size_t i = 0; i < out.size(); ++i) radix[i] = out[i];
  *nst = (int)out.size();
  return true;
}

bool f2_instantiated(const int* r, int nst) {
  const int r1 = nst > 1 ? r[1] : 0, r2 = nst > 2 ? r[2] : 0;
#define FV_F2_HAS(a, b, c) \
  if (r[0] == a && r1 == b && r2 == c) return true;
  FV_F2_PLANS(FV_F2_HAS)
#undef FV_F2_HAS
  return false;
}

template <typename F>
int f2_dispatch(const fvPlan* p, F&& f) {
  const int r0 = p->f2_radix[0], r1 = p->f2_nst > 1 ? p->f2_radix[1] : 0, r2 = p->f2_nst > 2 ? p->f2_radix[2] : 0;
#define FV_F2_CALL(a, b, c) \
  if (r0 == a && r1 == b && r2 == c) return f(std::integral_constant<int, a>{}, std::integral_constant<int, b>{}, std::integral_constant<int, c>{});
  FV_F2_PLANS(FV_F2_CALL)
#undef FV_F2_CALL
  return fail(FV_EINVAL, "no compiled two-ring FFT plan");
}

int setup_fft2(fvPlan* p) {
  const char* env = std::getenv("FV_FFT");
  if (env && (std::string(env) == "cufft" || std::string(env) == "v1")) return FV_OK;
  if (!fft2_factor(p->n_phi, p->f2_radix, &p->f2_nst) || p->f2_nst > 3 || !f2_instantiated(p->f2_radix, p->f2_nst))
    return FV_OK;
  const int n = p->n_phi;
  // twiddles of stages 1.. (stage 0 has none): entry [k < Ns][r - 1 < R - 1] = w^(r k n / (Ns R))
  std::vector<double2> tw;
  int ns = p->f2_radix[0];
  for (int s = 1; s < p->f2_nst; ++s) {
    const int R = p->f2_radix[s];
    const long long ts = n / (ns * R);
    for (int k = 0; k < ns; ++k)
      for (int r = 1; r < R; ++r) {
        const long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)(r * k * ts) / n;
        tw.push_back(make_double2((double)cosl(a), -(double)sinl(a)));
      }
    ns *= R;
  }
  FV_TRY(dalloc(&p->f2_tw, tw.size()));
  if (!tw.empty())
    FV_CUDA(cudaMemcpy(p->f2_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
  const int smem = (int)(fv::F2_NR * (size_t)n * sizeof(double2));
  FV_TRY(f2_dispatch(p, [&](auto A, auto B, auto C) -> int {
    FV_CUDA(cudaFuncSetAttribute(fv::ring_fft2_kernel<false, A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FV_CUDA(cudaFuncSetAttribute(fv::ring_fft2_kernel<true, A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FV_CUDA(cudaFuncSetAttribute(fv::fft_fold_kernel<A, B, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return FV_OK;
  }));
  p->fft2 = true;
  const char* ff = std::getenv("FV_FUSED_FOLD");
  p->fused_fold = !(ff && std::atoi(ff) == 0);
  return FV_OK;
}

// Bluestein ring FFT plan (fft_blue.cuh): n = R * P with P the largest prime
// factor (> 19, which the radix kernels do not cover), every prime of R <= 19
// Rader plans instantiated in fft_rader.cuh: (R, P, F1, F2) with P - 1 = F1 * F2,
// F1 an odd prime with constant-bank roots, F2 a composite of dft<>.
#define FV_RADER_PLANS(X)                  \
  X(12, 683, 31, 22) /* 8196: L = 4096 */ \
  X(12, 43, 7, 6)    /* 516: L = 256 */

// rings of at most kRaderMultiMaxN points go kRaderMultiRings to a CTA (fft_rader.cuh
// rader_multi_*_kernel: the forward takes kRaderMultiRings / 2 mirror pairs)
constexpr int kRaderMultiMaxN = 1024, kRaderMultiRings = 4;

template <class F>
int rader_dispatch(int R, int P, F f) {
#define FV_RD_CASE(R_, P_, F1_, F2_) \
  if (R == R_ && P == P_)            \
    return f(std::integral_constant<int, R_>{}, std::integral_constant<int, P_>{}, \
             std::integral_constant<int, F1_>{}, std::integral_constant<int, F2_>{});
  FV_RADER_PLANS(FV_RD_CASE)
#undef FV_RD_CASE
  return fail(FV_EINVAL, "no Rader plan for this length");
}

bool rader_instantiated(int R, int P) {
  bool ok = false;
#define FV_RD_HAVE(R_, P_, F1_, F2_) ok |= (R == R_ && P == P_);
  FV_RADER_PLANS(FV_RD_HAVE)
#undef FV_RD_HAVE
  return ok;
}

// Rader tables for n = R * P: primitive root g, slot table g^-p, modular inverses,
// the P-1 roots, the transformed kernel DFT_{P-1}(w_P^{g^m}) / (P-1) (long double
// sums), the n roots of the combine.  Packed into p->blue_tab.
int setup_rader(fvPlan* p, int R, int P) {
  const int n = R * P, M = P - 1;
  auto powmod = [](long long b, long long e, long long m) {
    long long r = 1;
    b %= m;
    while (e) {
      if (e & 1) r = r * b % m;
      b = b * b % m;
      e >>= 1;
    }
    return r;
  };
  std::vector<int> pf;
  for (int f = 2, rem = M; rem > 1; ++f)
    if (rem % f == 0) {
      pf.push_back(f);
      while (rem % f == 0) rem /= f;
    }
  int g = 2;
  for (;; ++g) {
    bool prim = true;
    for (int f : pf) prim &= powmod(g, M / f, P) != 1;
    if (prim) break;
  }
  const long long ginv = powmod(g, P - 2, P);
  const long double PI_ = 3.141592653589793238462643383279502884L;
  const int nhi = (n + 127) / 128;
  const size_t o_tw = 0, o_Bn = o_tw + M, o_lo = o_Bn + M, o_hi = o_lo + 128, o_idx = o_hi + nhi;
  const size_t n_idx = ((size_t)(M + P) * sizeof(short) + sizeof(double2) - 1) / sizeof(double2);
  std::vector<double2> tab(o_idx + n_idx);
  for (int e = 0; e < M; ++e) {
    const long double a = 2.0L * PI_ * e / M;
    tab[o_tw + e] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  std::vector<long double> br(M), bi(M);
  for (int m = 0; m < M; ++m) {
    const long double a = 2.0L * PI_ * (long double)powmod(g, m, P) / P;
    br[m] = cosl(a);
    bi[m] = -sinl(a);
  }
  for (int f = 0; f < M; ++f) {
    long double re = 0.0L, im = 0.0L;
    for (int m = 0; m < M; ++m) {
      const long double a = 2.0L * PI_ * (long double)(((long long)m * f) % M) / M;
      const long double c = cosl(a), sn = -sinl(a);
      re += br[m] * c - bi[m] * sn;
      im += br[m] * sn + bi[m] * c;
    }
    tab[o_Bn + f] = make_double2((double)(re / M), (double)(im / M));
  }
  for (int j = 0; j < 128; ++j) {
    const long double a = 2.0L * PI_ * j / n;
    tab[o_lo + j] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  for (int j = 0; j < nhi; ++j) {
    const long double a = 2.0L * PI_ * (128.0L * j) / n;
    tab[o_hi + j] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  short* idx = reinterpret_cast<short*>(tab.data() + o_idx);
  for (int q = 0; q < M; ++q) idx[q] = (short)powmod(ginv, q, P);  // sig[p] = g^-p
  idx[M] = 0;                                                      // inv[0]
  for (int k = 1; k < P; ++k) idx[M + k] = (short)powmod(k, P - 2, P);
  FV_TRY(fill_root_tables());
  FV_TRY(dalloc(&p->blue_tab, tab.size()));
  FV_CUDA(cudaMemcpy(p->blue_tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
  fv::RaderArgs& a = p->rd_args;
  a.tab = p->blue_tab + o_tw;
  a.sig = reinterpret_cast<const short*>(p->blue_tab + o_idx);
  FV_TRY(rader_dispatch(R, P, [&](auto R_, auto P_, auto F1_, auto F2_) -> int {
    constexpr int bytes = (int)fv::RaderSmem<R_, P_>::bytes;
    FV_CUDA(cudaFuncSetAttribute(fv::rader_fft_kernel<R_, P_, F1_, F2_>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    FV_CUDA(cudaFuncSetAttribute(fv::rader_fold_kernel<R_, P_, F1_, F2_>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if constexpr (R_ * P_ <= kRaderMultiMaxN) {  // short rings: several per CTA
      constexpr int mbytes = (int)fv::RaderSmem<R_, P_, kRaderMultiRings>::bytes;
      FV_CUDA(cudaFuncSetAttribute(fv::rader_multi_fft_kernel<R_, P_, F1_, F2_, kRaderMultiRings>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mbytes));
      FV_CUDA(cudaFuncSetAttribute(fv::rader_multi_fold_kernel<R_, P_, F1_, F2_, kRaderMultiRings / 2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, mbytes));
    }
    return FV_OK;
  }));
  p->rader_R = R;
  p->rader_P = P;
  const char* ff = std::getenv("FV_FUSED_FOLD");
  p->fused_fold = !(ff && std::atoi(ff) == 0);
  p->rader = true;
  return FV_OK;
}

// Lengths n = R * P with a prime P > 19: the small-prime kernels (P <= 64), a Rader
// plan, or cuFFT sub-DFTs + rp_combine_kernel for R one of these (R = 1: cuFFT's own
// plan for a prime length).  FV_FFT=rp forces the cuFFT sub-DFT path.
constexpr int kBlueR[] = {1, 2, 3, 4, 6, 8, 12, 16, 24};

int setup_blue(fvPlan* p) {
  const char* env = std::getenv("FV_FFT");
  if (env && std::string(env) == "cufft") return FV_OK;
  const int n = p->n_phi;
  int P = 1, rem = n;
  for (int f = 2; (long long)f * f <= rem; ++f)
    while (rem % f == 0) {
      P = std::max(P, f);
      rem /= f;
    }
  P = std::max(P, rem);
  if (P <= 19) return FV_OK;
  const int R = n / P;
  const long double PI_ = 3.141592653589793238462643383279502884L;
  // a Rader plan, where instantiated, replaces the direct small-prime DFTs (C2: forward
  // FFT + fold 0.237 -> 0.183 ms, inverse 0.165 -> 0.109 ms); FV_FFT=smallp keeps them
  const bool want_rader = rader_instantiated(R, P) && !(env && std::string(env) == "smallp");
  if (P <= fv::SMALLP_MAX && R <= 64 && !(env && std::string(env) == "rp") && !want_rader) {
    // direct conjugate-pair DFTs in one CTA per ring (smallp_kernel)
    const int H = (P - 1) / 2;
    std::vector<double2> tab((size_t)n + R * R + H * (H + 1));
    for (int j = 0; j < n; ++j) {
      const long double g = 2.0L * PI_ * j / n;
      tab[j] = make_double2((double)cosl(g), -(double)sinl(g));
    }
    for (int r = 0; r < R; ++r)
      for (int s2 = 0; s2 < R; ++s2) {
        const long double g = 2.0L * PI_ * ((r * s2) % R) / R;
        tab[n + r * R + s2] = make_double2((double)cosl(g), -(double)sinl(g));
      }
    for (int q = 1; q <= H; ++q)
      for (int k = 0; k <= H; ++k) {
        const long double g = 2.0L * PI_ * ((q * k) % P) / P;
        tab[n + R * R + (q - 1) * (H + 1) + k] = make_double2((double)cosl(g), (double)sinl(g));
      }
    FV_TRY(dalloc(&p->blue_tab, tab.size()));
    FV_CUDA(cudaMemcpy(p->blue_tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
    fv::SmallPArgs& s = p->sp_args;
    s.n = n;
    s.R = R;
    s.P = P;
    s.rootN = p->blue_tab;
    s.WR = p->blue_tab + n;
    s.WP = p->blue_tab + n + R * R;
    const size_t smem_f = (size_t)(4 * n + R * R + H * (H + 1)) * sizeof(double2);  // two rings per CTA
    if (smem_f > 200 * 1024) return FV_OK;
    FV_CUDA(cudaFuncSetAttribute(fv::smallp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f));
    FV_CUDA(cudaFuncSetAttribute(fv::smallp_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f));
    const char* ff = std::getenv("FV_FUSED_FOLD");
    p->fused_fold = !(ff && std::atoi(ff) == 0);
    p->smallp = true;
    return FV_OK;
  }
  // hand-written Rader DFTs (fft_rader.cuh) where a plan is instantiated (FV_FFT=rp: the
  // cuFFT sub-DFT path below)
  if (rader_instantiated(R, P) && !(env && std::string(env) == "rp"))
    return setup_rader(p, R, P);
  bool ok = false;
  for (int x : kBlueR) ok |= (x == R);
  if (!ok) return FV_OK;
  // large P without a Rader plan: batched cuFFT sub-DFTs of length P + the combine
  // kernel (rp_combine_kernel)
  {
    if (R == 1) return FV_OK;  // a prime length: cuFFT's own plan
    std::vector<double2> tab(n + R);
    for (int j = 0; j < n; ++j) {
      const long double g = 2.0L * PI_ * j / n;
      tab[j] = make_double2((double)cosl(g), -(double)sinl(g));
    }
    for (int j = 0; j < R; ++j) {
      const long double g = 2.0L * PI_ * j / R;
      tab[n + j] = make_double2((double)cosl(g), -(double)sinl(g));
    }
    FV_TRY(dalloc(&p->blue_tab, tab.size()));
    FV_CUDA(cudaMemcpy(p->blue_tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice));
    p->blue_args.n = n;
    p->blue_args.R = R;
    p->blue_args.P = P;
    p->blue_args.rootN = p->blue_tab;
    p->blue_args.rootR = p->blue_tab + n;
    p->rpfft = true;
    return FV_OK;
  }
  return FV_OK;
}

// FFT input prefetch distance in items (FV_FFT_PREFETCH; 0 disables).  C3
// sweep (fft stage per step, 4 fields): off 0.527 ms, 74 / 110 / 148 / 200 /
// 296 / 444 items ahead 0.509 / 0.508 / 0.510 / 0.512 / 0.520 / 0.535 ms:
// default one item per SM
int fft_prefetch_ahead() {
  static const int v = [] {
    const char* e = std::getenv("FV_FFT_PREFETCH");
    if (e) return std::max(0, std::atoi(e));
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return v;
}

int ring_fft_smallp(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
                    double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s,
                    int in_rblk = 0) {
  fv::SmallPArgs a = p->sp_args;
  a.in_rblk = in_rblk;
  a.in = in;
  a.in_cs = in_cs;
  a.in_rs = in_rs;
  a.in_es = in_es;
  a.out = out;
  a.out_cs = out_cs;
  a.out_rs = out_rs;
  a.out_es = out_es;
  a.nrings = nrings;
  a.inverse = inverse ? 1 : 0;
  a.ahead = fft_prefetch_ahead();
  const int H = (a.P - 1) / 2;
  const size_t smem = (size_t)(4 * a.n + a.R * a.R + H * (H + 1)) * sizeof(double2);  // two rings per CTA
  fv::smallp_kernel<<<(unsigned)(3LL * ((nrings + 1) / 2)), fv::SMALLP_T, smem, s>>>(a);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

int ring_fft_rader(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
                   double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s,
                   int in_rblk = 0) {
  fv::RaderArgs a = p->rd_args;
  a.in = in;
  a.in_cs = in_cs;
  a.in_rs = in_rs;
  a.in_es = in_es;
  a.in_rblk = in_rblk;
  a.out = out;
  a.out_cs = out_cs;
  a.out_rs = out_rs;
  a.out_es = out_es;
  a.nrings = nrings;
  a.inverse = inverse ? 1 : 0;
  a.ahead = fft_prefetch_ahead();
  return rader_dispatch(p->rader_R, p->rader_P, [&](auto R_, auto P_, auto F1_, auto F2_) -> int {
    if constexpr (R_ * P_ <= kRaderMultiMaxN) {
      const unsigned grid = (unsigned)((3LL * nrings + kRaderMultiRings - 1) / kRaderMultiRings);
      fv::rader_multi_fft_kernel<R_, P_, F1_, F2_, kRaderMultiRings>
          <<<grid, fv::RD_T, fv::RaderSmem<R_, P_, kRaderMultiRings>::bytes, s>>>(a);
    } else {
      fv::rader_fft_kernel<R_, P_, F1_, F2_>
          <<<(unsigned)(3LL * nrings), fv::RD_T, fv::RaderSmem<R_, P_>::bytes, s>>>(a);
    }
    FV_CUDA(cudaGetLastError());
    return FV_OK;
  });
}

int ring_fft_rp(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
                double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s) {
  const fv::BlueArgs& ba = p->blue_args;
  const int R = ba.R, P = ba.P;
  const size_t need = (size_t)3 * nrings * ba.n;
  if (p->blue_s1_cap < need) {
    if (p->blue_s1) {
      FV_CUDA(cudaDeviceSynchronize());
      cudaFree(p->blue_s1);
      p->blue_s1 = nullptr;
      p->blue_s1_cap = 0;
    }
    FV_TRY(dalloc(&p->blue_s1, need));
    p->blue_s1_cap = need;
  }
  // sub-DFT plan: element q of residue r at in + r * es + q * (R es), transform b at + b * rs
  const long long istride = (long long)R * in_es;
  const auto key = std::make_tuple(istride, in_rs, nrings);
  auto it = p->subffts.find(key);
  if (it == p->subffts.end()) {
    if (istride > INT32_MAX || in_rs > INT32_MAX) return fail(FV_EINVAL, "ring stride too large for cuFFT");
    int nP = P;
    cufftHandle hh;
    FV_CUFFT(cufftPlanMany(&hh, 1, &nP, &nP, (int)istride, (int)in_rs, &nP, 1, P, CUFFT_Z2Z, nrings));
    it = p->subffts.emplace(key, hh).first;
  }
  FV_CUFFT(cufftSetStream(it->second, s));
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < R; ++r) {
      auto* ip = reinterpret_cast<cufftDoubleComplex*>(const_cast<double2*>(in + c * in_cs + r * in_es));
      auto* op = reinterpret_cast<cufftDoubleComplex*>(p->blue_s1 + ((size_t)(c * R + r) * nrings) * P);
      FV_CUFFT(cufftExecZ2Z(it->second, ip, op, inverse ? CUFFT_INVERSE : CUFFT_FORWARD));
    }
  fv::RpArgs a{p->blue_s1, out, out_cs, out_rs, out_es, ba.rootN, ba.rootR, ba.n, P, nrings, inverse ? 1 : 0};
  const unsigned g = (unsigned)((3LL * nrings * P + fv::BLUE_T - 1) / fv::BLUE_T);
  switch (R) {
    case 2: fv::rp_combine_kernel<2><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 3: fv::rp_combine_kernel<3><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 4: fv::rp_combine_kernel<4><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 6: fv::rp_combine_kernel<6><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 8: fv::rp_combine_kernel<8><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 12: fv::rp_combine_kernel<12><<<g, fv::BLUE_T, 0, s>>>(a); break;
    case 16: fv::rp_combine_kernel<16><<<g, fv::BLUE_T, 0, s>>>(a); break;
    default: fv::rp_combine_kernel<24><<<g, fv::BLUE_T, 0, s>>>(a); break;
  }
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}


int ring_fft2_raw(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
                  double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s,
                  int in_rblk = 0) {
  fv::Fft2Args a{};
  a.in_rblk = in_rblk;
  a.tw = p->f2_tw;
  a.in = in;
  a.out = out;
  a.in_cs = in_cs; a.in_rs = in_rs; a.in_es = (int)in_es;
  a.out_cs = out_cs; a.out_rs = out_rs; a.out_es = (int)out_es;
  a.nrings = nrings;
  a.ahead = fft_prefetch_ahead();
  const int grid = 3 * ((nrings + fv::F2P_NR - 1) / fv::F2P_NR);
  const size_t smem = fv::F2P_NR * (size_t)p->n_phi * sizeof(double2);
  return f2_dispatch(p, [&](auto A, auto B, auto C) -> int {
    if (inverse) fv::ring_fft2_kernel<true, A, B, C><<<grid, fv::F2P_T, smem, s>>>(a, grid);
    else fv::ring_fft2_kernel<false, A, B, C><<<grid, fv::F2P_T, smem, s>>>(a, grid);
    FV_CUDA(cudaGetLastError());
    return FV_OK;
  });
}

// fused forward FFT + fold of fields b0 .. b0 + nf - 1 of T (B, N, 3) into X (all orders)
// (ngroups > 1: that many full 4-field groups in one launch, X buffers x_gstride apart; only the
// several-rings-per-CTA Rader kernel takes it, see fft_fold_groups)
int fft_fold(fvPlan* p, const double2* T, int b0, int nf, cudaStream_t s, double* X, int ngroups = 1) {
  fv::Fft2Args a{};
  if (p->rader) {  // Rader ring DFT, north / south ring of a pair on a two-CTA cluster (fft_rader.cuh)
    const long long n = p->n_phi;
    a.in_rs = 3 * n;
    a.in_es = 3;
    a.field_stride = 3 * n * p->n_theta;
    a.in = T + (long long)b0 * a.field_stride;
    a.X = X;
    a.pair_n = p->pair_n;
    a.pair_s = p->pair_s;
    a.ring_w = p->ring_w;
    a.nchunks = p->nchunks;
    a.NT = ntiles_for(nf);
    a.nfields = nf * ngroups;
    a.gfields = ngroups > 1 ? nf : 0;
    a.x_gstride = (long long)p->x_gstride;
    a.Lt = p->Lt;
    a.ahead = fft_prefetch_ahead() / 2;
    const int nitems = p->nchunks * fv::FWD_RC * nf * ngroups * 3;  // (pair, field, component)
    return rader_dispatch(p->rader_R, p->rader_P, [&](auto R_, auto P_, auto F1_, auto F2_) -> int {
      if constexpr (R_ * P_ <= kRaderMultiMaxN) {
        constexpr int NPR = kRaderMultiRings / 2;
        fv::rader_multi_fold_kernel<R_, P_, F1_, F2_, NPR>
            <<<(unsigned)((nitems + NPR - 1) / NPR), fv::RD_T, fv::RaderSmem<R_, P_, kRaderMultiRings>::bytes, s>>>(
                p->rd_args, a, nitems);
      } else {
        fv::rader_fold_kernel<R_, P_, F1_, F2_>
            <<<2u * (unsigned)nitems, fv::RD_T, fv::RaderSmem<R_, P_>::bytes, s>>>(p->rd_args, a);
      }
      FV_CUDA(cudaGetLastError());
      return FV_OK;
    });
  }
  if (p->smallp) {  // small-prime ring DFT (fft_blue.cuh smallp_fold_kernel)
    const long long n = p->n_phi;
    a.in_rs = 3 * n;
    a.in_es = 3;
    a.field_stride = 3 * n * p->n_theta;
    a.in = T + (long long)b0 * a.field_stride;
    a.X = X;
    a.pair_n = p->pair_n;
    a.pair_s = p->pair_s;
    a.ring_w = p->ring_w;
    a.nchunks = p->nchunks;
    a.NT = ntiles_for(nf);
    a.nfields = nf;
    a.Lt = p->Lt;
    a.ahead = fft_prefetch_ahead();
    const fv::SmallPArgs& sp = p->sp_args;
    const int H = (sp.P - 1) / 2;
    const size_t smem = (size_t)(4 * sp.n + sp.R * sp.R + H * (H + 1)) * sizeof(double2);
    fv::smallp_fold_kernel<<<p->nchunks * fv::FWD_RC * nf * 3, fv::SMALLP_T, smem, s>>>(sp, a);
    FV_CUDA(cudaGetLastError());
    return FV_OK;
  }
  const long long n = p->n_phi;
  a.tw = p->f2_tw;
  a.in_rs = 3 * n;
  a.in_es = 3;
  a.field_stride = 3 * n * p->n_theta;
  a.in = T + (long long)b0 * a.field_stride;
  a.X = X;
  a.pair_n = p->pair_n;
  a.pair_s = p->pair_s;
  a.ring_w = p->ring_w;
  a.nchunks = p->nchunks;
  a.NT = ntiles_for(nf);
  a.nfields = nf;
  a.Lt = p->Lt;
  a.ahead = fft_prefetch_ahead();
  const int grid = p->nchunks * fv::FWD_RC * nf * 3;
  const size_t smem = fv::F2_NR * (size_t)p->n_phi * sizeof(double2);
  return f2_dispatch(p, [&](auto A, auto B, auto C) -> int {
    fv::fft_fold_kernel<A, B, C><<<grid, fv::F2_T, smem, s>>>(a, grid);
    FV_CUDA(cudaGetLastError());
    return FV_OK;
  });
}

// 3 components x nrings ring DFTs with the hand-written kernel; element (c, ring, q) at
// c * cs + ring * rs + q * es (complex units) on both sides
int ring_fft_raw(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
                 double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s) {
  fv::RingFftArgs a{};
  a.in = in;
  a.out = out;
  a.in_cs = in_cs; a.in_rs = in_rs; a.in_es = (int)in_es;
  a.out_cs = out_cs; a.out_rs = out_rs; a.out_es = (int)out_es;
  a.tw = p->fft_tw;
  a.n = p->n_phi;
  a.nst = p->fft_nst;
  int ns = 1;
  for (int i = 0; i < p->fft_nst; ++i) {
    a.radix[i] = p->fft_radix[i];
    a.ns[i] = ns;
    a.nsmagic[i] = ns == 1 ? 0u : (unsigned)((0x100000000ull + ns - 1) / ns);  // exact j/ns for j < 2^16
    a.tstride[i] = p->n_phi / (ns * p->fft_radix[i]);
    ns *= p->fft_radix[i];
  }
  a.nrings = nrings;
  const int grid = std::min(3 * a.nrings, 2 * p->num_sms);
  const size_t smem = (3 * (size_t)p->n_phi + fv::FFT_TWN) * sizeof(double2);
  if (inverse) fv::ring_fft_kernel<true><<<grid, fv::FFT_THREADS, smem, s>>>(a);
  else fv::ring_fft_kernel<false><<<grid, fv::FFT_THREADS, smem, s>>>(a);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

int begin_call(fvPlan* p) {
  if (!p) return fail(FV_EINVAL, "null plan");
  FV_CUDA(cudaSetDevice(p->device));
  g_err.clear();
  return FV_OK;
}

}  // namespace

extern "C" {

const char* fv_version(void) { return "favest_b200 0.1.0 sm_100a"; }

int fv_gauss_legendre(int n, double* thetas, double* weights, int device) {
  if (n < 1) return fail(FV_EINVAL, "Gauss-Legendre rule needs at least one node, got " + std::to_string(n));
  if (!thetas || !weights) return fail(FV_EINVAL, "null output");
  int prev = 0;
  FV_CUDA(cudaGetDevice(&prev));
  FV_CUDA(cudaSetDevice(device));
  double* d = nullptr;
  int rc = FV_OK;
  if (cudaMalloc(&d, 2 * (size_t)n * sizeof(double)) != cudaSuccess) {
    cudaSetDevice(prev);
    return fail(FV_ENOMEM, "device allocation failed");
  }
  const int half = (n + 1) / 2;
  fv::gauss_legendre_kernel<<<(half + 127) / 128, 128>>>(n, d, d + n);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(thetas, d, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(weights, d + n, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) rc = fail(FV_ECUDA, std::string("Gauss-Legendre rule: ") + cudaGetErrorString(e));
  cudaFree(d);
  cudaSetDevice(prev);
  return rc;
}

// debug: copy the forward pipeline trace (4096 tiles x 8 stamps) to the host
int fv_debug_trace(long long* host) {
  if (!g_trace) return FV_EINVAL;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_trace, 4096 * 12 * sizeof(long long), cudaMemcpyDeviceToHost);
  return FV_OK;
}

const char* fv_last_error(void) { return g_err.c_str(); }

int fv_plan_create_grid(fvPlan** out, int L, int n_theta, int n_phi, const double* ring_theta_host,
                        const double* ring_weight_host, int max_batch, int device) {
  if (!out) return fail(FV_EINVAL, "null output pointer");
  *out = nullptr;
  if (L < 1) return fail(FV_EINVAL, "vector transforms need lmax >= 1, got " + std::to_string(L));
  if (n_theta < 1) return fail(FV_EINVAL, "grid needs at least one ring");
  if (n_phi < 1) return fail(FV_EINVAL, "n_phi must be positive, got " + std::to_string(n_phi));
  const int needed = 2 * (L + 1) + 1;  // favest/transforms.py:63
  if (n_phi < needed)
    return fail(FV_EINVAL, "fast-scalar path needs n_phi >= " + std::to_string(needed) + " for degree " +
                               std::to_string(L) + ", grid has n_phi=" + std::to_string(n_phi));
  if (max_batch < 1) return fail(FV_EINVAL, "max_batch must be positive");
  for (int r = 0; r < n_theta; ++r) {
    if (!(ring_theta_host[r] > 0.0 && ring_theta_host[r] < M_PI))
      return fail(FV_EINVAL, "ring colatitudes must lie strictly inside (0, pi)");
    if (r > 0 && !(ring_theta_host[r] > ring_theta_host[r - 1]))
      return fail(FV_EINVAL, "ring colatitudes must be strictly increasing");
  }
  fvPlan* p = new fvPlan();
  p->kind = 0;
  p->L = L;
  p->Lt = L + 1;
  p->n_theta = n_theta;
  p->n_phi = n_phi;
  p->max_batch = max_batch;
  p->device = device;
  auto bail = [&](int rc) {
    free_plan(p);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(FV_ECUDA, "cannot select device"));
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);

  // ring cosines exactly as favest/scalar.py:133 + favest/legendre.py:53-57
  std::vector<double> t(n_theta), w(ring_weight_host, ring_weight_host + n_theta);
  for (int r = 0; r < n_theta; ++r) t[r] = std::min(1.0, std::max(-1.0, std::cos(ring_theta_host[r])));
  // equatorial folding when the grid is mirror symmetric (GL: cos mirrors to 3e-16, weights bitwise)
  bool sym = true;
  for (int r = 0; r < n_theta / 2 && sym; ++r) {
    const int r2 = n_theta - 1 - r;
    if (std::fabs(t[r] + t[r2]) > 1e-13) sym = false;
    if (std::fabs(w[r] - w[r2]) > 1e-13 * std::fabs(w[r])) sym = false;
  }
  std::vector<int> pn, ps;
  if (sym) {
    for (int r = 0; r < n_theta / 2; ++r) {
      pn.push_back(r);
      ps.push_back(n_theta - 1 - r);
    }
    if (n_theta & 1) {
      pn.push_back(n_theta / 2);
      ps.push_back(-1);
    }
  } else {
    for (int r = 0; r < n_theta; ++r) {
      pn.push_back(r);
      ps.push_back(-1);
    }
  }
  p->paired = sym ? 1 : 0;
  p->nP = (int)pn.size();
  p->nPpad = (p->nP + fv::ADJ_RC - 1) / fv::ADJ_RC * fv::ADJ_RC;
  p->nchunks = (p->nP + fv::FWD_RC - 1) / fv::FWD_RC;  // forward chunks (pairs beyond nP are zero)
  p->nrc = p->nPpad / fv::ADJ_RC;
  std::vector<double> pt(p->nPpad, 0.0), psn(p->nPpad, 0.0);
  pn.resize(p->nPpad, -1);
  ps.resize(p->nPpad, -1);
  for (int i = 0; i < p->nP; ++i) {
    pt[i] = t[pn[i]];
    psn[i] = std::sqrt(std::max(0.0, 1.0 - pt[i] * pt[i]));
  }
  const int Lt = p->Lt;
  int rc;
  if ((rc = dalloc(&p->pair_t, p->nPpad)) || (rc = dalloc(&p->pair_sin, p->nPpad)) ||
      (rc = dalloc(&p->pair_n, p->nPpad)) || (rc = dalloc(&p->pair_s, p->nPpad)) ||
      (rc = dalloc(&p->ring_w, n_theta)) || (rc = dalloc(&p->seed_x, (size_t)(Lt + 1) * p->nPpad)) ||
      (rc = dalloc(&p->seed_e, (size_t)(Lt + 1) * p->nPpad)))
    return bail(rc);
  cudaMemcpy(p->pair_t, pt.data(), p->nPpad * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(p->pair_sin, psn.data(), p->nPpad * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(p->pair_n, pn.data(), p->nPpad * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p->pair_s, ps.data(), p->nPpad * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p->ring_w, w.data(), n_theta * 8, cudaMemcpyHostToDevice);
  fv::seeds_kernel<<<(p->nPpad + 127) / 128, 128>>>(p->pair_sin, p->nPpad, Lt, p->seed_x, p->seed_e);
  if (cudaGetLastError() != cudaSuccess) return bail(fail(FV_ECUDA, "seed kernel launch failed"));
  if ((rc = ab_tables(p)) || (rc = dg_tables(p)) || (rc = cg_tables(p))) return bail(rc);
  // polar-start tables (legendre.cuh), then the extended-range seeds are no longer needed
  if ((rc = dalloc(&p->start_l, (size_t)(Lt + 1) * p->nPpad)) ||
      (rc = dalloc(&p->start_v, (size_t)(Lt + 1) * p->nPpad)))
    return bail(rc);
  {
    dim3 grid((p->nPpad + 127) / 128, Lt + 1);
    fv::start_kernel<<<grid, 128>>>(p->seed_x, p->seed_e, p->pair_t, p->pair_n, p->ab, p->abofs, p->dg, p->dgofs,
                                    p->nPpad, Lt, p->start_l, p->start_v);
    if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(FV_ECUDA, "polar-start kernel failed"));
    cudaFree(p->seed_x);
    cudaFree(p->seed_e);
    p->seed_x = nullptr;
    p->seed_e = nullptr;
    if ((rc = dalloc(&p->cmin, (size_t)(Lt + 1) * p->nchunks))) return bail(rc);
    dim3 cg((p->nchunks + 127) / 128, Lt + 1);
    fv::chunk_start_kernel<<<cg, 128>>>(p->start_l, p->nPpad, p->nchunks, fv::FWD_RC, p->cmin);
    if ((rc = dalloc(&p->cmin_a, (size_t)(Lt + 1) * p->nrc))) return bail(rc);
    dim3 ca((p->nrc + 127) / 128, Lt + 1);
    fv::chunk_start_kernel<<<ca, 128>>>(p->start_l, p->nPpad, p->nrc, fv::ADJ_RC, p->cmin_a);
    if (cudaGetLastError() != cudaSuccess) return bail(fail(FV_ECUDA, "chunk-start kernel launch failed"));
  }
  if ((rc = ptab_tables(p))) return bail(rc);
  if ((rc = fseed_tables(p))) return bail(rc);
  // G layout tile offsets: nlc(m) = ceil((Lt+1-m)/ADJ_LC) tiles per order
  std::vector<long long> gofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m) gofs[m + 1] = gofs[m] + (Lt + 1 - m + fv::ADJ_LC - 1) / fv::ADJ_LC;
  p->g_tiles = gofs[Lt + 1];
  if ((rc = dalloc(&p->gofs, Lt + 1))) return bail(rc);
  cudaMemcpy(p->gofs, gofs.data(), (Lt + 1) * 8, cudaMemcpyHostToDevice);
  if ((rc = dalloc(&p->cga, (size_t)18 * 32 * p->g_tiles))) return bail(rc);
  {
    dim3 grid((Lt + 1 + fv::ADJ_LC - 1) / fv::ADJ_LC, Lt + 1);
    fv::cga_table_kernel<<<grid, 32>>>(Lt, p->gofs, p->cgt, p->cga, 32 * p->g_tiles);
    FV_CUDA(cudaGetLastError());
  }
  if ((rc = setup_fft(p)) || (rc = setup_fft2(p)) || (rc = setup_blue(p))) return bail(rc);
  // workspaces (field groups of <= 4 -> NT <= 6)
  const int gs = std::min(4, max_batch);
  const int NTmax = ntiles_for(gs);
  {
    // FV_SLAYOUT=<fwd><adj> digits, 0 ring-major / 1 bin-major / 2 ring pairs (default
    // 02 when the inverse ring DFT is hand-written, else 01: the forward FFT writes
    // contiguous rings, the adjoint epilogue writes 128-byte runs of one bin)
    const char* sl = std::getenv("FV_SLAYOUT");
    const bool own_fft = p->fft2 || p->smallp || p->rader;
    const char fdig = (sl && sl[0]) ? sl[0] : '0';
    char adig = (sl && sl[0] && sl[1]) ? sl[1] : (own_fft ? '2' : '1');
    if (adig == '2' && !own_fft) adig = '1';
    const char* rb = std::getenv("FV_SLAYOUT_RBLK");  // experiments: ring block of the blocked layout
    int rbsh = 1;  // ring pairs
    if (rb) rbsh = std::atoi(rb) >= 8 ? 3 : std::atoi(rb) >= 4 ? 2 : 1;
    const int rblk = 1 << rbsh;
    const long long rings = (long long)max_batch * n_theta, rings8 = (rings + 7) / 8 * 8;
    const fv::SLayout ringmajor{rings8 * n_phi, n_phi, 1, 0, 0, 0}, binmajor{rings8 * n_phi, 1, rings, 0, 0, 0},
        blocked{rings8 * n_phi, (long long)rblk * n_phi, rblk, 0, 0, rblk, rbsh};
    p->lay_f = fdig == '1' ? binmajor : ringmajor;
    p->lay_a = adig == '2' ? blocked : adig == '0' ? ringmajor : binmajor;
  }
  const size_t spec = (size_t)3 * ((max_batch * (size_t)n_theta + 7) / 8 * 8) * n_phi;
  p->x_gstride = (size_t)(Lt + 1) * p->nchunks * (2 * 8 * NTmax * 32);
  p->f_gstride = (size_t)(Lt + 1) * (Lt + 2) / 2 * 8 * NTmax;
  p->g_gstride = (size_t)p->g_tiles * (2 * fv::ADJ_KS * NTmax * 32);
  {
    // several full field groups per Legendre launch when their buffers stay small (<= 2 GB)
    const size_t per = (p->x_gstride + p->f_gstride + p->g_gstride) * sizeof(double);
    const int want = (max_batch + 3) / 4;
    p->ngroups_buf = std::max(1, std::min(want, (int)std::min<size_t>(16, (2ull << 30) / std::max<size_t>(per, 1))));
  }
  const size_t ngb = (size_t)p->ngroups_buf;
  if ((rc = dalloc(&p->Sf, spec)) || (rc = dalloc(&p->Sa, spec)) || (rc = dalloc(&p->X, ngb * p->x_gstride)) ||
      (rc = dalloc(&p->F, ngb * p->f_gstride)) || (rc = dalloc(&p->G, ngb * p->g_gstride)))
    return bail(rc);
  if (cudaMemset(p->Sa, 0, spec * sizeof(double2)) != cudaSuccess) return bail(fail(FV_ECUDA, "memset failed"));
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(FV_ECUDA, std::string("plan setup: ") + cudaGetErrorString(e)));
  *out = p;
  return FV_OK;
}

int fv_plan_create_points(fvPlan** out, int L, int max_batch, int device) {
  if (!out) return fail(FV_EINVAL, "null output pointer");
  *out = nullptr;
  if (L < 1) return fail(FV_EINVAL, "vector coefficients need lmax >= 1");
  if (max_batch < 1) return fail(FV_EINVAL, "max_batch must be positive");
  fvPlan* p = new fvPlan();
  p->kind = 1;
  p->L = L;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
  p->Lt = L + 1;
  p->max_batch = max_batch;
  p->device = device;
  auto bail = [&](int rc) {
    free_plan(p);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(FV_ECUDA, "cannot select device"));
  int rc;
  if ((rc = ab_tables(p)) || (rc = cg_tables(p))) return bail(rc);
  const int Lt = p->Lt;
  std::vector<long long> rowofs(Lt + 2, 0);
  for (int m = 0; m <= Lt; ++m) rowofs[m + 1] = rowofs[m] + (Lt + 1 - m);
  if ((rc = dalloc(&p->rowofs, Lt + 1))) return bail(rc);
  cudaMemcpy(p->rowofs, rowofs.data(), (Lt + 1) * 8, cudaMemcpyHostToDevice);
  const int gs = std::min(4, max_batch);
  if ((rc = dalloc(&p->G, (size_t)rowofs[Lt + 1] * 12 * gs))) return bail(rc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail(FV_ECUDA, std::string("plan setup: ") + cudaGetErrorString(e)));
  *out = p;
  return FV_OK;
}

void fv_plan_destroy(fvPlan* plan) { free_plan(plan); }

int fv_plan_info(const fvPlan* p, int* L, int* n_theta, int* n_phi, int* n_pairs, int* paired) {
  if (!p) return fail(FV_EINVAL, "null plan");
  if (L) *L = p->L;
  if (n_theta) *n_theta = p->n_theta;
  if (n_phi) *n_phi = p->n_phi;
  if (n_pairs) *n_pairs = p->nP;
  if (paired) *paired = p->paired;
  return FV_OK;
}

int fv_order_cost(const fvPlan* p, double* cost) {
  if (!p) return fail(FV_EINVAL, "null plan");
  if (p->kind != 0) return fail(FV_EINVAL, "order cost needs a grid plan");
  if (!cost) return fail(FV_EINVAL, "null output");
  const int Lt = p->Lt;
  std::vector<int> ls((size_t)(Lt + 1) * p->nPpad);
  FV_CUDA(cudaMemcpy(ls.data(), p->start_l, ls.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int m = 0; m <= Lt; ++m) {
    double c = 0.0;
    for (int q = 0; q < p->nP; ++q) c += std::max(0, Lt + 1 - std::max(m, ls[(size_t)m * p->nPpad + q]));
    cost[m] = c;
  }
  return FV_OK;
}

int fv_set_profiling(fvPlan* p, int enable) {
  if (!p) return fail(FV_EINVAL, "null plan");
  if (p->profiling && !p->marks.empty()) cudaEventSynchronize(p->marks.back().second.second);
  p->profiling = enable != 0;
  p->marks.clear();  // stage times accumulate over all calls until the next fv_set_profiling
  p->ev_used = 0;
  return FV_OK;
}

double fv_stage_ms(const fvPlan* p, int stage) {
  if (!p || p->marks.empty()) return -1.0;
  cudaEventSynchronize(p->marks.back().second.second);
  double tot = 0.0;
  for (auto& mk : p->marks) {
    if (mk.first != stage) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, mk.second.first, mk.second.second);
    tot += ms;
  }
  return tot;
}

int fv_stage_count(const fvPlan* p, int stage) {
  if (!p) return 0;
  int n = 0;
  for (auto& mk : p->marks) n += mk.first == stage;
  return n;
}

namespace {

int check_grid_call(fvPlan* p, int B, const void* x, const void* y, const void* z) {
  FV_TRY(begin_call(p));
  if (p->kind != 0) return fail(FV_EINVAL, "fast-scalar path requires a rule with tensor-grid structure");
  if (B < 1 || B > p->max_batch)
    return fail(FV_EINVAL, "batch " + std::to_string(B) + " outside 1.." + std::to_string(p->max_batch));
  if (!x || !y || !z) return fail(FV_EINVAL, "null data pointer");
  return FV_OK;
}

// CG assembly (favest/transforms.py:120-146) of coefficient orders [c_lo, c_hi) of fields
// b0 .. b0 + nf - 1 from the forward Legendre rows in p->F (ncol = 8 NT)
int cg_forward(fvPlan* p, double* a, double* b, int B, int b0, int nf, int NT, int c_lo, int c_hi, cudaStream_t s,
               const double* F = nullptr, int nsplit = 1, const double* Fx = nullptr, int ngroups = 1) {
  StageMark mk(p, 3, s);
  fv::CgFwdArgs ca{F ? F : p->F, reinterpret_cast<double2*>(a), reinterpret_cast<double2*>(b), p->cgt, p->L, 8 * NT, B, b0,
                   nf, c_lo, c_hi, nsplit, nsplit > 1 ? Fx : nullptr, (long long)p->f_gstride, (long long)p->f_gstride};
  // ngroups full 4-field groups (F buffers f_gstride apart) in one launch: grid.z
  const int mb = fv::cgf_mb(nf);
  dim3 grid((c_hi + mb - 1) / mb - c_lo / mb, p->L + 1, ngroups);
  const size_t smem = (size_t)3 * (mb + 2) * fv::cgf_rs(nf) * sizeof(double2);
  if (nf == 1) {  // 56 KB of staging at 128 orders per CTA
    static std::atomic<unsigned long long> attr{0}, attr_split{0};
    FV_CUDA(smem_optin_once(&attr, p->device, fv::cg_fwd_tile_kernel<1, false>));
    FV_CUDA(smem_optin_once(&attr_split, p->device, fv::cg_fwd_tile_kernel<1, true>));
  }
  auto go = [&](auto split) {
    constexpr bool SP = decltype(split)::value;
    switch (nf) {
      case 1: fv::cg_fwd_tile_kernel<1, SP><<<grid, fv::CGF_THREADS, smem, s>>>(ca); break;
      case 2: fv::cg_fwd_tile_kernel<2, SP><<<grid, fv::CGF_THREADS, smem, s>>>(ca); break;
      case 3: fv::cg_fwd_tile_kernel<3, SP><<<grid, fv::CGF_THREADS, smem, s>>>(ca); break;
      default: fv::cg_fwd_tile_kernel<4, SP><<<grid, fv::CGF_THREADS, smem, s>>>(ca); break;
    }
  };
  if (ngroups > 1 && nsplit == 1 && nf == 4) {
    fv::cg_fwd_tile_kernel<4, false, true><<<grid, fv::CGF_THREADS, smem, s>>>(ca);
  } else {
    if (ngroups > 1) return fail(FV_EINVAL, "grouped forward CG launches take full 4-field groups without splits");
    if (nsplit > 1) go(std::true_type{});
    else go(std::false_type{});
  }
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

// fold + Legendre over orders [m_lo, m_hi) and CG for orders [c_lo, c_hi), reading the
// spectra of every ring of the grid in layout `lay` (natural or compact bins)
// Scalar mode of the vector pipeline (scalar.cuh): the fields are pseudo fields
// whose components are scalar fields; the CG stages become unpack / pack.
struct ScalarIO {
  double2* out = nullptr;       // forward: flat scalar coefficients [B][(lmax + 1)^2]
  const double2* in = nullptr;  // adjoint: flat scalar coefficients
  int lmax = 0, B = 0;          // scalar degree and scalar field count
};

int scalar_unpack(const ScalarIO& io, const double* F, int NT, int pf0, int nfp, int Lt_rows, cudaStream_t s) {
  const int lm = std::min(io.lmax, Lt_rows);
  dim3 grid((lm + 1 + 127) / 128, lm + 1);
  fv::scalar_unpack_kernel<<<grid, 128, 0, s>>>(F, 8 * NT, io.lmax, pf0, nfp, io.B, io.out);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

// pair-chunk split of a forward Legendre launch of mc orders: about two CTAs per SM
// (one CTA per (order, split)), at most 4 splits and one chunk per split; 1 when the
// orders alone fill the GPU (every full-grid launch).  FV_FWD_KSPLIT=n forces n.
int fwd_ksplit(const fvPlan* p, int mc) {
  static const int forced = [] { const char* e = std::getenv("FV_FWD_KSPLIT"); return e ? std::atoi(e) : -1; }();
  int ks = forced >= 0 ? std::max(1, forced) : (int)std::lround(2.0 * p->num_sms / std::max(1, mc));
  return std::max(1, std::min({ks, 4, p->nchunks}));
}

// Fields per forward Legendre launch: up to 4, fewer when the shared memory of
// the launch's n-tile count (5 stages + per-pair recurrence state) would exceed
// 227 KB -- 4 fields (NT = 6) fit up to L ~ 1900, 2 fields (NT = 3) up to L ~ 4000.
int fwd_group_cap(const fvPlan* p) {
  const int nPx = p->nchunks * fv::FWD_RC;
  for (int nf = 4; nf > 1; --nf) {
    size_t bytes = 0;
    switch (ntiles_for(nf)) {
      case 3: bytes = fv::FwdSmem<3>::bytes(nPx); break;
      case 5: bytes = fv::FwdSmem<5>::bytes(nPx); break;
      default: bytes = fv::FwdSmem<6>::bytes(nPx); break;
    }
    if (bytes <= 227 * 1024) return nf;
  }
  return 1;
}

// the several-rings-per-CTA Rader fold kernel takes all groups of a launch at once
bool fft_fold_groups(const fvPlan* p) { return p->rader && p->rader_R * p->rader_P <= kRaderMultiMaxN; }

int forward_orders(fvPlan* p, const double2* S, const fv::SLayout& lay, double* a, double* b, int B, int m_lo,
                   int m_hi, int c_lo, int c_hi, cudaStream_t s, const double2* Tfield = nullptr,
                   const ScalarIO* sio = nullptr) {
  const int Lt = p->Lt;
  const int mc = m_hi - m_lo;
  const int cap = fwd_group_cap(p);
  for (int b0 = 0; b0 < B;) {
    // up to ngroups_buf full 4-field groups go through one Legendre launch
    const int ng = cap == 4 ? std::max(1, std::min((B - b0) / 4, p->ngroups_buf)) : 1;
    const int nf = ng > 1 ? 4 : std::min(cap, B - b0);
    const int NT = ntiles_for(nf);
    for (int g = 0; g < ng; ++g) {
      double* Xg = p->X + (size_t)g * p->x_gstride;
      const int bg = b0 + 4 * g;
      if (S) {
        StageMark mk(p, 1, s);
        fv::FoldArgs fa{S, Xg, p->pair_n, p->pair_s, p->ring_w, p->n_phi, p->n_theta, B, bg, nf, NT,
                        p->nchunks * fv::FWD_RC, p->nchunks, m_lo, mc, lay};
        dim3 grid((p->nchunks * fv::FWD_RC + 127) / 128, mc, 3 * nf + 1);
        fv::fold_fwd_kernel<<<grid, 128, 0, s>>>(fa);
        FV_CUDA(cudaGetLastError());
      } else if (ng > 1 && fft_fold_groups(p)) {  // all groups in one launch
        if (g == 0) {
          StageMark mk(p, 0, s);
          FV_TRY(fft_fold(p, Tfield, b0, nf, s, p->X, ng));
        }
      } else {  // fused FFT + fold straight from the field (fft2.cuh / fft_blue.cuh)
        StageMark mk(p, 0, s);
        FV_TRY(fft_fold(p, Tfield, bg, nf, s, Xg));
      }
    }
    // launches with few orders (the order-sharded chunks) split every order's pair
    // chunks over up to 4 CTAs, each into its own partial F buffer (the CG adds them)
    const int ks = (ng == 1 && !sio) ? fwd_ksplit(p, mc) : 1;
    if (ks > 1 && !p->Fx) FV_TRY(dalloc(&p->Fx, (size_t)3 * p->f_gstride));
    {
      StageMark mk(p, 2, s);
      fv::FwdArgs args{p->X, p->F, p->start_l, p->start_v, p->dg, p->dgofs, p->pair_t, Lt, p->nP, p->nPpad,
                       p->nchunks, m_lo, dbg_mode(), mc, trace_buf(), trace_cta(), p->ptab_f, p->mtab_f, p->tofs, p->cmin,
                       ng, (long long)p->x_gstride, (long long)p->f_gstride, ks, p->Fx};
      args.klast = (p->nP - fv::FWD_RC * (p->nchunks - 1) + 3) / 4;
      FV_TRY(dispatch_fwd(p, NT, args, mc, s));
    }
    if (sio)
      for (int g = 0; g < ng; ++g) {
        StageMark mk(p, 3, s);
        FV_TRY(scalar_unpack(*sio, p->F + (size_t)g * p->f_gstride, NT, b0 + 4 * g, nf, Lt, s));
      }
    else if (c_hi > c_lo)
      FV_TRY(cg_forward(p, a, b, B, b0, nf, NT, c_lo, c_hi, s, p->F, ks, p->Fx, ng));
    b0 += ng > 1 ? 4 * ng : nf;
  }
  return FV_OK;
}

// CG + Legendre synthesis for orders [m_lo, m_hi) into spectra of every ring (layout `lay`)
int adjoint_orders(fvPlan* p, const double* a, const double* b, double2* S, const fv::SLayout& lay, int B, int m_lo,
                   int m_hi, cudaStream_t s, const ScalarIO* sio = nullptr) {
  const int Lt = p->Lt;
  const int mc = m_hi - m_lo;
  for (int b0 = 0; b0 < B;) {
    // up to ngroups_buf full 4-field groups go through one Legendre launch
    const int ng = std::max(1, std::min((B - b0) / 4, p->ngroups_buf));
    const int nf = ng > 1 ? 4 : std::min(4, B - b0);
    const int NT = ntiles_for(nf);
    for (int g = 0; g < ng && sio; ++g) {  // scalar mode: pack the coefficients instead of coupling them
      StageMark mk(p, 3, s);
      fv::ScalarPackArgs sa{sio->in, sio->lmax, sio->B, b0 + 4 * g, nf, p->G + (size_t)g * p->g_gstride, p->gofs,
                            nullptr, p->dg, p->dgofs, Lt, NT, 0, m_lo};
      dim3 grid((Lt + 1 - m_lo + fv::ADJ_LC - 1) / fv::ADJ_LC * fv::ADJ_LC / 32, mc);
      fv::scalar_pack_kernel<<<grid, 32, 0, s>>>(sa);
      FV_CUDA(cudaGetLastError());
    }
    static const int multi = [] { const char* e = std::getenv("FV_CGA_MULTI"); return e ? std::atoi(e) : -1; }();
    // the multi-order kernel takes all ng groups in one launch (grid.z); the tile kernel one per group
    for (int g = 0; g < (multi ? 1 : ng) && !sio; ++g) {
      StageMark mk(p, 3, s);
      fv::CgAdjArgs ca{reinterpret_cast<const double2*>(a), reinterpret_cast<const double2*>(b), p->dg, p->dgofs,
                       p->cgt, p->G + (size_t)g * p->g_gstride, p->gofs, nullptr, p->L, NT, B, b0 + 4 * g, nf, m_lo,
                       0, p->cga, 32 * p->g_tiles, (long long)p->g_gstride};
      dim3 grid((Lt + 1 - m_lo + fv::ADJ_LC - 1) / fv::ADJ_LC, mc);
      const size_t smem = (size_t)2 * fv::ADJ_KS * fv::cga_bstride(nf) * sizeof(double) +
                          2 * (size_t)nf * 34 * 7 * sizeof(double2);
      // runs of consecutive orders per CTA (cg_adj_multi_kernel): two at 3-4 fields (three CTAs
      // per SM), four at 1-2 fields; FV_CGA_MULTI=0 selects the one-order tile kernel
      auto launch_multi = [&](auto nfc, auto noc) -> int {
        constexpr int NF_ = decltype(nfc)::value, NO_ = decltype(noc)::value;
        static std::atomic<unsigned long long> attr{0};
        FV_CUDA(smem_optin_once(&attr, p->device, fv::cg_adj_multi_kernel<NF_, NO_>));
        const dim3 mgrid(grid.x, (mc + NO_ - 1) / NO_, ng);
        fv::cg_adj_multi_kernel<NF_, NO_><<<mgrid, fv::CGA_THREADS, fv::CgaMulti<NF_, NO_>::bytes, s>>>(ca, mc);
        return FV_OK;
      };
      auto by_run = [&](auto nfc) -> int {
        const int run = multi > 0 ? multi : (decltype(nfc)::value >= 3 ? 2 : 4);
        if (run == 2) return launch_multi(nfc, std::integral_constant<int, 2>{});
        return launch_multi(nfc, std::integral_constant<int, 4>{});
      };
      if (multi) {
        switch (nf) {
          case 1: FV_TRY(by_run(std::integral_constant<int, 1>{})); break;
          case 2: FV_TRY(by_run(std::integral_constant<int, 2>{})); break;
          case 3: FV_TRY(by_run(std::integral_constant<int, 3>{})); break;
          default: FV_TRY(by_run(std::integral_constant<int, 4>{})); break;
        }
      } else {
        switch (nf) {
          case 1: fv::cg_adj_tile_kernel<1><<<grid, fv::CGA_THREADS, smem, s>>>(ca); break;
          case 2: fv::cg_adj_tile_kernel<2><<<grid, fv::CGA_THREADS, smem, s>>>(ca); break;
          case 3: fv::cg_adj_tile_kernel<3><<<grid, fv::CGA_THREADS, smem, s>>>(ca); break;
          default: fv::cg_adj_tile_kernel<4><<<grid, fv::CGA_THREADS, smem, s>>>(ca); break;
        }
      }
      FV_CUDA(cudaGetLastError());
    }
    {
      StageMark mk(p, 2, s);
      fv::AdjArgs args{p->G, p->gofs, S, p->start_l, p->start_v, p->dg, p->dgofs, p->pair_t, p->pair_n,
                       p->pair_s, Lt, p->nP, p->nPpad, p->nrc, p->n_phi, p->n_theta, B, b0, nf, m_lo, dbg_mode(),
                       mc, p->ptab_a, p->aofs, trace_buf(), trace_cta(), lay, p->cmin_a, ng, (long long)p->g_gstride};
      FV_TRY(dispatch_adj(p, NT, args, mc, s));
    }
    b0 += ng > 1 ? 4 * ng : nf;
  }
  return FV_OK;
}

// three components x nrings ring DFTs of length n_phi, arbitrary strides (complex units)
int ring_ffts(fvPlan* p, bool inverse, const double2* in, long long in_cs, long long in_rs, long long in_es,
              double2* out, long long out_cs, long long out_rs, long long out_es, int nrings, cudaStream_t s,
              int in_rblk = 0) {
  StageMark mk(p, 0, s);
  if (in_rblk) {  // blocked rings: only the hand-written two-ring / small-prime / Rader kernels read them
    if (p->rader)
      return ring_fft_rader(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s, in_rblk);
    if (p->fft2)
      return ring_fft2_raw(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s, in_rblk);
    if (p->smallp)
      return ring_fft_smallp(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s, in_rblk);
    return fail(FV_EINVAL, "blocked spectrum layout without a hand-written ring DFT");
  }
  if (p->fft2) return ring_fft2_raw(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s);
  if (p->custom_fft) return ring_fft_raw(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s);
  if (p->smallp) return ring_fft_smallp(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s);
  if (p->rader) return ring_fft_rader(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s);
  if (p->rpfft) return ring_fft_rp(p, inverse, in, in_cs, in_rs, in_es, out, out_cs, out_rs, out_es, nrings, s);
  cufftHandle h;
  FV_TRY(get_fft_strided(p, in_rs, in_es, out_rs, out_es, nrings, &h));
  FV_CUFFT(cufftSetStream(h, s));
  for (int c = 0; c < 3; ++c) {
    auto* i = reinterpret_cast<cufftDoubleComplex*>(const_cast<double2*>(in)) + c * in_cs;
    auto* o = reinterpret_cast<cufftDoubleComplex*>(out) + c * out_cs;
    FV_CUFFT(cufftExecZ2Z(h, i, o, inverse ? CUFFT_INVERSE : CUFFT_FORWARD));
  }
  return FV_OK;
}

}  // namespace

namespace {
int forward_grid_impl(fvPlan* p, const double2* T, double* a, double* b, int B, cudaStream_t s,
                      const ScalarIO* sio = nullptr) {
  const long long n = p->n_phi;
  if ((p->fft2 || p->smallp || p->rader) && p->fused_fold)
    return forward_orders(p, nullptr, p->lay_f, a, b, B, 0, p->Lt + 1, 0, p->L + 1, s, T, sio);
  FV_TRY(ring_ffts(p, false, T, 1, 3 * n, 3, p->Sf, p->lay_f.cs, p->lay_f.rs, p->lay_f.bs, B * p->n_theta, s));
  return forward_orders(p, p->Sf, p->lay_f, a, b, B, 0, p->Lt + 1, 0, p->L + 1, s, nullptr, sio);
}

int adjoint_grid_impl(fvPlan* p, const double* a, const double* b, double2* T, int B, cudaStream_t s,
                      const ScalarIO* sio = nullptr) {
  FV_TRY(adjoint_orders(p, a, b, p->Sa, p->lay_a, B, 0, p->Lt + 1, s, sio));
  const long long n = p->n_phi;
  return ring_ffts(p, true, p->Sa, p->lay_a.cs, p->lay_a.rs, p->lay_a.bs, T, 1, 3 * n, 3, B * p->n_theta, s,
                   p->lay_a.rblk);
}

// pseudo-field scratch for B scalar fields of n points: ceil(B / 3) x n x 3
int scalar_scratch(fvPlan* p, int B, long long n) {
  const size_t need = (size_t)((B + 2) / 3) * n * 3 * 2;  // doubles
  if (p->Tp_cap >= need) return FV_OK;
  if (p->Tp) {
    FV_CUDA(cudaDeviceSynchronize());
    cudaFree(p->Tp);
    p->Tp = nullptr;
    p->Tp_cap = 0;
  }
  FV_TRY(dalloc(&p->Tp, need));
  p->Tp_cap = need;
  return FV_OK;
}

int check_scalar_call(fvPlan* p, int B, int lmax, const void* x, const void* y) {
  if (B < 1 || B > 3 * p->max_batch)
    return fail(FV_EINVAL, "scalar batch " + std::to_string(B) + " outside 1.." + std::to_string(3 * p->max_batch));
  if (lmax < 0) return fail(FV_EINVAL, "lmax must be non-negative, got " + std::to_string(lmax));
  if (lmax > p->Lt)
    return fail(FV_EINVAL, "scalar degree " + std::to_string(lmax) + " exceeds the plan's " + std::to_string(p->Lt));
  if (!x || !y) return fail(FV_EINVAL, "null data pointer");
  return FV_OK;
}

unsigned grid_for(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16); }
}  // namespace

int fv_forward_grid(fvPlan* p, const double* T, double* a, double* b, int B, void* stream) {
  FV_TRY(check_grid_call(p, B, T, a, b));
  return forward_grid_impl(p, reinterpret_cast<const double2*>(T), a, b, B, reinterpret_cast<cudaStream_t>(stream));
}

int fv_adjoint_grid(fvPlan* p, const double* a, const double* b, double* T, int B, void* stream) {
  FV_TRY(check_grid_call(p, B, T, a, b));
  return adjoint_grid_impl(p, a, b, reinterpret_cast<double2*>(T), B, reinterpret_cast<cudaStream_t>(stream));
}

int fv_forward_scalar_grid(fvPlan* p, const double* f, double* out, int lmax, int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 0) return fail(FV_EINVAL, "fast-scalar path requires a rule with tensor-grid structure");
  FV_TRY(check_scalar_call(p, B, lmax, f, out));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const long long n = (long long)p->n_theta * p->n_phi;
  FV_TRY(scalar_scratch(p, B, n));
  const int K = (B + 2) / 3;
  const long long tot = (long long)K * n * 3;
  fv::scalar_to_pseudo_kernel<<<grid_for(tot), 256, 0, s>>>(reinterpret_cast<const double2*>(f), n, B,
                                                            reinterpret_cast<double2*>(p->Tp), tot);
  FV_CUDA(cudaGetLastError());
  ScalarIO io;
  io.out = reinterpret_cast<double2*>(out);
  io.lmax = lmax;
  io.B = B;
  return forward_grid_impl(p, reinterpret_cast<const double2*>(p->Tp), nullptr, nullptr, K, s, &io);
}

int fv_adjoint_scalar_grid(fvPlan* p, const double* g, double* f, int lmax, int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 0) return fail(FV_EINVAL, "fast-scalar path requires a rule with tensor-grid structure");
  FV_TRY(check_scalar_call(p, B, lmax, g, f));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const long long n = (long long)p->n_theta * p->n_phi;
  FV_TRY(scalar_scratch(p, B, n));
  const int K = (B + 2) / 3;
  ScalarIO io;
  io.in = reinterpret_cast<const double2*>(g);
  io.lmax = lmax;
  io.B = B;
  FV_TRY(adjoint_grid_impl(p, nullptr, nullptr, reinterpret_cast<double2*>(p->Tp), K, s, &io));
  fv::pseudo_to_scalar_kernel<<<grid_for((long long)B * n), 256, 0, s>>>(reinterpret_cast<const double2*>(p->Tp), n,
                                                                         B, reinterpret_cast<double2*>(f));
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

// ---- order-sharded building blocks (paper_1908_00041_b200/dist.py) ----
int fv_ring_fft(fvPlan* p, int inverse, const double* in, long long in_cs, long long in_rs, long long in_es,
                double* out, long long out_cs, long long out_rs, long long out_es, int nrings, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 0) return fail(FV_EINVAL, "fast-scalar path requires a rule with tensor-grid structure");
  if (!in || !out) return fail(FV_EINVAL, "null data pointer");
  if (nrings < 0) return fail(FV_EINVAL, "negative ring count");
  if (nrings == 0) return FV_OK;
  return ring_ffts(p, inverse != 0, reinterpret_cast<const double2*>(in), in_cs, in_rs, in_es,
                   reinterpret_cast<double2*>(out), out_cs, out_rs, out_es, nrings,
                   reinterpret_cast<cudaStream_t>(stream));
}

namespace {
int check_orders(fvPlan* p, long long rs, long long bs, int bin_lo, int nbins, int m_lo, int m_hi) {
  if (m_lo < 0 || m_hi > p->Lt + 1 || m_lo >= m_hi)
    return fail(FV_EINVAL, "order range [" + std::to_string(m_lo) + ", " + std::to_string(m_hi) + ") outside 0.." +
                               std::to_string(p->Lt));
  if (nbins < 0 || (nbins > 0 && (m_lo < bin_lo || m_hi > bin_lo + nbins)))
    return fail(FV_EINVAL, "compact bins do not cover the order range");
  if (rs <= 0 || bs <= 0) return fail(FV_EINVAL, "spectrum strides must be positive");
  return FV_OK;
}
}  // namespace

int fv_forward_orders(fvPlan* p, const double* S, long long cs, long long rs, long long bs, int bin_lo, int nbins,
                      double* a, double* b, int B, int m_lo, int m_hi, int c_lo, int c_hi, void* stream) {
  FV_TRY(check_grid_call(p, B, S, a, b));
  FV_TRY(check_orders(p, rs, bs, bin_lo, nbins, m_lo, m_hi));
  if (c_lo < 0 || c_hi > p->L + 1 || c_lo > c_hi) return fail(FV_EINVAL, "coefficient order range invalid");
  if (c_hi > c_lo && ((c_lo > 0 && c_lo - 1 < m_lo) || c_hi > m_hi - 1 || (c_lo == 0 && m_lo > 0)))
    return fail(FV_EINVAL, "coefficient orders need the Legendre orders c_lo-1 .. c_hi");
  const fv::SLayout lay{cs, rs, bs, bin_lo, nbins};
  return forward_orders(p, reinterpret_cast<const double2*>(S), lay, a, b, B, m_lo, m_hi, c_lo, c_hi,
                        reinterpret_cast<cudaStream_t>(stream));
}

int fv_adjoint_orders(fvPlan* p, const double* a, const double* b, int B, int m_lo, int m_hi, double* S, long long cs,
                      long long rs, long long bs, int bin_lo, int nbins, void* stream) {
  FV_TRY(check_grid_call(p, B, S, a, b));
  FV_TRY(check_orders(p, rs, bs, bin_lo, nbins, m_lo, m_hi));
  const fv::SLayout lay{cs, rs, bs, bin_lo, nbins};
  return adjoint_orders(p, a, b, reinterpret_cast<double2*>(S), lay, B, m_lo, m_hi,
                        reinterpret_cast<cudaStream_t>(stream));
}

int fv_forward_orders_packed(fvPlan* p, const double* S, const long long* ring_offsets, long long rts, int bin_lo,
                             int nbins, double* a, double* b, int B, int m_lo, int m_hi, int c_lo, int c_hi,
                             void* stream) {
  FV_TRY(check_grid_call(p, B, S, a, b));
  FV_TRY(check_orders(p, 1, 1, bin_lo, nbins, m_lo, m_hi));
  if (nbins <= 0) return fail(FV_EINVAL, "packed spectra need compact bins");
  if (!ring_offsets || rts < (long long)B * p->n_theta) return fail(FV_EINVAL, "ring-offset table too small");
  if (c_lo < 0 || c_hi > p->L + 1 || c_lo > c_hi) return fail(FV_EINVAL, "coefficient order range invalid");
  if (c_hi > c_lo && ((c_lo > 0 && c_lo - 1 < m_lo) || c_hi > m_hi - 1 || (c_lo == 0 && m_lo > 0)))
    return fail(FV_EINVAL, "coefficient orders need the Legendre orders c_lo-1 .. c_hi");
  fv::SLayout lay{0, 1, 1, bin_lo, nbins};
  lay.rtab = ring_offsets;
  lay.rts = rts;
  return forward_orders(p, reinterpret_cast<const double2*>(S), lay, a, b, B, m_lo, m_hi, c_lo, c_hi,
                        reinterpret_cast<cudaStream_t>(stream));
}

int fv_adjoint_orders_packed(fvPlan* p, const double* a, const double* b, int B, int m_lo, int m_hi, double* S,
                             const long long* ring_offsets, long long rts, int bin_lo, int nbins, void* stream) {
  FV_TRY(check_grid_call(p, B, S, a, b));
  FV_TRY(check_orders(p, 1, 1, bin_lo, nbins, m_lo, m_hi));
  if (nbins <= 0) return fail(FV_EINVAL, "packed spectra need compact bins");
  if (!ring_offsets || rts < (long long)B * p->n_theta) return fail(FV_EINVAL, "ring-offset table too small");
  fv::SLayout lay{0, 1, 1, bin_lo, nbins};
  lay.rtab = ring_offsets;
  lay.rts = rts;
  return adjoint_orders(p, a, b, reinterpret_cast<double2*>(S), lay, B, m_lo, m_hi,
                        reinterpret_cast<cudaStream_t>(stream));
}

namespace {
int adjoint_points_impl(fvPlan* p, const double* xyz, long long M, const double* a, const double* b, double* T, int B,
                        cudaStream_t s, const ScalarIO* sio = nullptr);
}  // namespace

int fv_adjoint_points(fvPlan* p, const double* xyz, long long M, const double* a, const double* b, double* T,
                      int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 1) return fail(FV_EINVAL, "plan was not created for scattered points");
  if (B < 1 || B > p->max_batch)
    return fail(FV_EINVAL, "batch " + std::to_string(B) + " outside 1.." + std::to_string(p->max_batch));
  if (M < 0) return fail(FV_EINVAL, "negative point count");
  if (M == 0) return FV_OK;
  if (!xyz || !T || !a || !b) return fail(FV_EINVAL, "null data pointer");
  return adjoint_points_impl(p, xyz, M, a, b, T, B, reinterpret_cast<cudaStream_t>(stream));
}

namespace {
int adjoint_points_impl(fvPlan* p, const double* xyz, long long M, const double* a, const double* b, double* T, int B,
                        cudaStream_t s, const ScalarIO* sio) {
  const int Lt = p->Lt;
  for (int b0 = 0; b0 < B; b0 += 4) {
    const int nf = std::min(4, B - b0);
    if (sio) {  // scalar mode: the coefficients packed into the merged rows
      StageMark mk(p, 3, s);
      fv::ScalarPackArgs sa{sio->in, sio->lmax, sio->B, b0, nf, p->G, nullptr, p->rowofs, nullptr, nullptr,
                            Lt, 0, 1, 0};
      dim3 grid((Lt + 1 + 127) / 128, Lt + 1);
      fv::scalar_pack_kernel<<<grid, 128, 0, s>>>(sa);
      FV_CUDA(cudaGetLastError());
    } else {
      StageMark mk(p, 3, s);
      fv::CgAdjArgs ca{reinterpret_cast<const double2*>(a), reinterpret_cast<const double2*>(b), nullptr, nullptr,
                       p->cgt, p->G, nullptr, p->rowofs, p->L, 0, B, b0, nf, 0, 1};
      dim3 grid((Lt + 1 + 127) / 128, Lt + 1);
      fv::cg_adj_kernel<<<grid, 128, 0, s>>>(ca);
      FV_CUDA(cudaGetLastError());
    }
    {
      StageMark mk(p, 2, s);
      fv::PtsArgs pa{xyz, M, p->G, p->rowofs, p->ab, p->abofs, reinterpret_cast<double2*>(T), Lt, B, b0};
      const unsigned grid = (unsigned)((M + fv::PTS_THREADS - 1) / fv::PTS_THREADS);
      // tensor-core kernel when its two row buffers fit shared memory (FV_PTS_DMMA=0: FMA kernel)
      {
        const char* e = std::getenv("FV_PTS_DMMA");
        const int nt = (12 * nf + 7) / 8, rs = ((8 * nt + 11) / 16) * 16 + 4;
        const size_t sd = (size_t)2 * (((Lt + 1 + 3) & ~3) * rs + 2 * (Lt + 1)) * sizeof(double) +
                          fv::PTS_THREADS / 32 * 128 * sizeof(double);
        if (!(e && std::atoi(e) == 0) && sd <= 220 * 1024) {
          auto launchd = [&](auto kern) -> int {
            FV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd));
            kern<<<grid, fv::PTS_THREADS, sd, s>>>(pa);
            return FV_OK;
          };
          switch (nf) {
            case 1: FV_TRY(launchd(fv::adjoint_points_dmma_kernel<1>)); break;
            case 2: FV_TRY(launchd(fv::adjoint_points_dmma_kernel<2>)); break;
            case 3: FV_TRY(launchd(fv::adjoint_points_dmma_kernel<3>)); break;
            default: FV_TRY(launchd(fv::adjoint_points_dmma_kernel<4>)); break;
          }
          FV_CUDA(cudaGetLastError());
          continue;
        }
      }
      const size_t smem = (size_t)2 * (Lt + 1) * 12 * nf * sizeof(double);
      const bool stage = smem <= 200 * 1024;  // else rows straight from global memory
      auto launch = [&](auto kern) -> int {
        if (stage) FV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, fv::PTS_THREADS, stage ? smem : 0, s>>>(pa);
        return FV_OK;
      };
      switch (nf * 2 + (stage ? 1 : 0)) {
        case 3: FV_TRY(launch(fv::adjoint_points_kernel<1, true>)); break;
        case 2: FV_TRY(launch(fv::adjoint_points_kernel<1, false>)); break;
        case 5: FV_TRY(launch(fv::adjoint_points_kernel<2, true>)); break;
        case 4: FV_TRY(launch(fv::adjoint_points_kernel<2, false>)); break;
        case 7: FV_TRY(launch(fv::adjoint_points_kernel<3, true>)); break;
        case 6: FV_TRY(launch(fv::adjoint_points_kernel<3, false>)); break;
        case 9: FV_TRY(launch(fv::adjoint_points_kernel<4, true>)); break;
        default: FV_TRY(launch(fv::adjoint_points_kernel<4, false>)); break;
      }
      FV_CUDA(cudaGetLastError());
    }
  }
  return FV_OK;
}
}  // namespace

}  // extern "C"

// ---- direct forward at weighted points (favest/scalar.py:94-105) ----
namespace {

// plan-time state of the direct forward: K_m seeds and the (order, window) item list
int fpts_setup(fvPlan* p) {
  if (p->seedk) return FV_OK;
  const int Lt = p->Lt;
  std::vector<double> km(Lt + 1);
  double cur = 0.28209479177387814;  // 1/sqrt(4 pi), favest/legendre.py:60
  km[0] = cur;
  for (int m = 1; m <= Lt; ++m) {
    cur *= std::sqrt((2 * m + 1) / (2.0 * m));  // |favest/legendre.py:62-65| without the s factor
    km[m] = cur;
  }
  std::vector<int2> items;
  for (int m = 0; m <= Lt; ++m)
    for (int w = 0; m + w * fv::FPD_WIN <= Lt; ++w) items.push_back(make_int2(m, w));
  // heaviest first: window rows, then the recurrence steps below the window
  auto work = [&](int2 it) {
    const int lo = it.x + it.y * fv::FPD_WIN, hi = std::min(Lt + 1, lo + fv::FPD_WIN);
    return 8.0 * (hi - lo) + (lo - it.x);
  };
  std::stable_sort(items.begin(), items.end(), [&](int2 x, int2 y) { return work(x) > work(y); });
  FV_TRY(dalloc(&p->seedk, Lt + 1));
  FV_TRY(dalloc(&p->fitems, items.size()));
  FV_CUDA(cudaMemcpy(p->seedk, km.data(), (Lt + 1) * sizeof(double), cudaMemcpyHostToDevice));
  FV_CUDA(cudaMemcpy(p->fitems, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice));
  p->n_fitems = (int)items.size();
  return FV_OK;
}

int grow(double** buf, size_t* cap, size_t n) {
  if (*cap >= n) return FV_OK;
  if (*buf) {
    FV_CUDA(cudaDeviceSynchronize());  // earlier calls may still read the old buffer
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
  }
  FV_TRY(dalloc(buf, n));
  *cap = n;
  return FV_OK;
}

template <int NF>
int launch_fpts(fvPlan* p, const fv::FptsArgs& fa, unsigned grid, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  const size_t smem = fv::fpd_smem_bytes(NF, p->Lt);
  FV_CUDA(smem_optin_once(&attr, p->device, fv::forward_points_dmma_kernel<NF>));
  fv::forward_points_dmma_kernel<NF><<<grid, fv::FPD_THREADS, smem, s>>>(fa);
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

}  // namespace

namespace {
int forward_points_impl(fvPlan* p, const double* xyz, const double* w, long long M, const double* T, double* a,
                        double* b, int B, cudaStream_t s, const ScalarIO* sio);
}  // namespace

extern "C" int fv_forward_points(fvPlan* p, const double* xyz, const double* w, long long M, const double* T,
                                 double* a, double* b, int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 1) return fail(FV_EINVAL, "plan was not created for scattered points");
  if (B < 1 || B > p->max_batch)
    return fail(FV_EINVAL, "batch " + std::to_string(B) + " outside 1.." + std::to_string(p->max_batch));
  if (M < 0) return fail(FV_EINVAL, "negative point count");
  if (!a || !b || (M > 0 && (!xyz || !w || !T))) return fail(FV_EINVAL, "null data pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const long long K = (long long)(p->L + 1) * (p->L + 1);
  if (M == 0) {  // empty rule: every coefficient is an empty sum
    FV_CUDA(cudaMemsetAsync(a, 0, (size_t)B * K * 16, s));
    FV_CUDA(cudaMemsetAsync(b, 0, (size_t)B * K * 16, s));
    return FV_OK;
  }
  return forward_points_impl(p, xyz, w, M, T, a, b, B, s, nullptr);
}

namespace {
int forward_points_impl(fvPlan* p, const double* xyz, const double* w, long long M, const double* T, double* a,
                        double* b, int B, cudaStream_t s, const ScalarIO* sio) {
  const int Lt = p->Lt;
  if (fv::fpd_smem_bytes(1, Lt) > 227 * 1024)
    return fail(FV_EINVAL, "degree " + std::to_string(p->L) + " too large for the direct forward kernel");
  FV_TRY(fpts_setup(p));
  const int gs = (fv::fpd_smem_bytes(4, Lt) <= 227 * 1024) ? 4 : 1;  // fields per launch
  const long long rows = (long long)(Lt + 1) * (Lt + 2) / 2;
  // point ranges: enough CTAs to balance the uneven items over all SMs, bounded workspace
  const long long nchunk = (M + fv::FPD_CHUNK - 1) / fv::FPD_CHUNK;
  const long long want = (16LL * p->num_sms + p->n_fitems - 1) / p->n_fitems;
  const long long cap_r = std::max(1LL, (long long)(1ull << 30) / (rows * 8 * fv::ptsd_nt(gs) * 8));
  const int R = (int)std::max(1LL, std::min({want, nchunk, 32LL, cap_r}));
  const int NTmax = fv::ptsd_nt(gs);
  FV_TRY(grow(&p->Fpart, &p->Fpart_cap, (size_t)R * rows * 8 * NTmax));
  FV_TRY(grow(&p->F, &p->F_cap, (size_t)rows * 8 * NTmax));
  for (int b0 = 0; b0 < B; b0 += gs) {
    const int nf = std::min(gs, B - b0);
    const int NT = fv::ptsd_nt(nf);
    {
      StageMark mk(p, 2, s);
      fv::FptsArgs fa{xyz, w, M, reinterpret_cast<const double2*>(T), p->Fpart, rows * 8 * NT, p->ab, p->abofs,
                      p->seedk, p->fitems, Lt, B, b0, R, 8 * NT};
      const unsigned grid = (unsigned)((long long)p->n_fitems * R);
      switch (nf) {
        case 1: FV_TRY(launch_fpts<1>(p, fa, grid, s)); break;
        case 2: FV_TRY(launch_fpts<2>(p, fa, grid, s)); break;
        case 3: FV_TRY(launch_fpts<3>(p, fa, grid, s)); break;
        default: FV_TRY(launch_fpts<4>(p, fa, grid, s)); break;
      }
      const long long n2 = rows * 4 * NT;
      fv::fpart_reduce_kernel<<<(unsigned)std::min<long long>((n2 + 255) / 256, 8LL * p->num_sms), 256, 0, s>>>(
          reinterpret_cast<const double2*>(p->Fpart), n2, R, reinterpret_cast<double2*>(p->F));
      FV_CUDA(cudaGetLastError());
    }
    if (sio) {
      StageMark mk(p, 3, s);
      FV_TRY(scalar_unpack(*sio, p->F, NT, b0, nf, Lt, s));
    } else {
      FV_TRY(cg_forward(p, a, b, B, b0, nf, NT, 0, p->L + 1, s));
    }
  }
  return FV_OK;
}
}  // namespace

extern "C" int fv_forward_scalar_points(fvPlan* p, const double* xyz, const double* w, long long M, const double* f,
                                        double* out, int lmax, int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 1) return fail(FV_EINVAL, "plan was not created for scattered points");
  FV_TRY(check_scalar_call(p, B, lmax, out, out));
  if (M < 0) return fail(FV_EINVAL, "negative point count");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (M == 0) {
    FV_CUDA(cudaMemsetAsync(out, 0, (size_t)B * (lmax + 1) * (lmax + 1) * 16, s));
    return FV_OK;
  }
  if (!xyz || !w || !f) return fail(FV_EINVAL, "null data pointer");
  FV_TRY(scalar_scratch(p, B, M));
  const int K = (B + 2) / 3;
  const long long tot = (long long)K * M * 3;
  fv::scalar_to_pseudo_kernel<<<grid_for(tot), 256, 0, s>>>(reinterpret_cast<const double2*>(f), M, B,
                                                            reinterpret_cast<double2*>(p->Tp), tot);
  FV_CUDA(cudaGetLastError());
  ScalarIO io;
  io.out = reinterpret_cast<double2*>(out);
  io.lmax = lmax;
  io.B = B;
  return forward_points_impl(p, xyz, w, M, p->Tp, nullptr, nullptr, K, s, &io);
}

extern "C" int fv_adjoint_scalar_points(fvPlan* p, const double* xyz, long long M, const double* g, double* f,
                                        int lmax, int B, void* stream) {
  FV_TRY(begin_call(p));
  if (p->kind != 1) return fail(FV_EINVAL, "plan was not created for scattered points");
  FV_TRY(check_scalar_call(p, B, lmax, g, g));
  if (M < 0) return fail(FV_EINVAL, "negative point count");
  if (M == 0) return FV_OK;
  if (!xyz || !f) return fail(FV_EINVAL, "null data pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  FV_TRY(scalar_scratch(p, B, M));
  const int K = (B + 2) / 3;
  ScalarIO io;
  io.in = reinterpret_cast<const double2*>(g);
  io.lmax = lmax;
  io.B = B;
  FV_TRY(adjoint_points_impl(p, xyz, M, nullptr, nullptr, p->Tp, K, s, &io));
  fv::pseudo_to_scalar_kernel<<<grid_for((long long)B * M), 256, 0, s>>>(reinterpret_cast<const double2*>(p->Tp), M,
                                                                         B, reinterpret_cast<double2*>(f));
  FV_CUDA(cudaGetLastError());
  return FV_OK;
}

#include "fileio.cuh"
