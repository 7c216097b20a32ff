// Shared device helpers for the FaVeST VSHT kernels (sm_100a).
//
// - FP64 tensor-core tile: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); B200 has no
//   tcgen05 kind for f64, and DMMA measured 37.0 TF/s vs DFMA 33.6 TF/s on
//   this pool (tools/fp64_microbench.cu, profiles/r01_fp64_microbench.txt).
// - mbarrier + cp.async.bulk (TMA 1-D bulk copy) producer/consumer pipeline.
// - extended-range ("X-number") scale handling for the Legendre recurrence.
// - the nine closed-form Clebsch-Gordan coefficients, same expression order as
//   the reference (favest/coupling.py:39-78), so xi/mu are bitwise equal.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace fv {

// Ring-spectrum layout: element (component c, ring R = field * n_theta + t, bin q)
// lives at c * cs + R * rs + q * bs (units of complex doubles).  Ring-major
// (rs = n_phi, bs = 1) keeps each ring's FFT contiguous; bin-major (rs = 1,
// bs = rings) makes one bin row of consecutive rings contiguous for the
// per-order kernels.  Chosen per direction by the plan.
// Compact bins (order-sharded spectra, nbins > 0): only the orders
// bin_lo .. bin_lo + nbins - 1 are held, +m at bin m - bin_lo, -m at
// nbins + m - bin_lo.  nbins == 0: natural DFT bins (m, (n_phi - m) % n_phi).
// Blocked (rblk = 2, the grid adjoint's default when its inverse ring DFT is a
// hand-written kernel): rings in pairs, [comp][ring / 2][bin][ring % 2] -- the
// two rings a ring-DFT CTA transforms are one contiguous 32-byte-per-bin
// stream (coalesced stage-0 loads), and the adjoint epilogue still writes
// whole 32-byte sectors (rs = pair stride 2 * bins, bs = 2).
struct SLayout {
  long long cs, rs, bs;
  int bin_lo, nbins;
  int rblk = 0;  // 0: ring R at R * rs; 2^k: ring R at (R >> k) * rs + (R & (2^k - 1))
  int rbsh = 0;  // k
  // ring-offset table (order-sharded transposes, dist.py): when set, element
  // (component c, ring R, bin j) is at rtab[c * rts + R] + j * bs, so a kernel
  // can read / write the per-rank blocks of an all-to-all buffer in place
  const long long* rtab = nullptr;
  long long rts = 0;
};

__host__ __device__ __forceinline__ long long spec_ring(const SLayout& l, long long R) {
  return l.rblk ? (R >> l.rbsh) * l.rs + (R & (l.rblk - 1)) : R * l.rs;
}

// offset of (component c, ring R) without the bin term
__device__ __forceinline__ long long spec_cr(const SLayout& l, int c, long long R) {
  return l.rtab ? __ldg(l.rtab + c * l.rts + R) : c * l.cs + spec_ring(l, R);
}

__device__ __forceinline__ long long spec_bin(const SLayout& l, int m, int sgn, int n_phi) {
  if (l.nbins == 0) return sgn ? (n_phi - m) % n_phi : m;
  return (sgn ? l.nbins : 0) + (m - l.bin_lo);
}

constexpr int XR_SHIFT = 512;  // value = x * 2^e, e a multiple of 512 (oracle/favest_oracle.py)

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// one 32-byte global store (sm_100 STG.256): a full sector in one instruction
__device__ __forceinline__ void st_global_v4(double* p, double2 lo, double2 hi) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(lo.x), "d"(lo.y), "d"(hi.x), "d"(hi.y)
               : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory load kept in program order with the (volatile) DMMA asm, so the
// fragment loads of a stage are all issued before its guarded DMMA groups.
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared, completion counted on an mbarrier (TMA engine).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction-priority policies for bulk copies: streamed-once tiles (the
// plan-time Legendre tables) evict first, tiles re-read by later stages / other
// CTAs (ring data, coefficient tiles) evict last.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// value of an extended-range number x * 2^e (e <= 0, multiple of 512); below
// 2^-1024 the value is flushed to zero, matching oracle._xr_value.
__device__ __forceinline__ double xr_value(double x, int e) {
  if (e == 0) return x;
  if (e == -XR_SHIFT) return x * 0x1p-512;
  if (e == -2 * XR_SHIFT) return x * 0x1p-1024;
  return 0.0;
}

// ---------------------------------------------------------------------------
// Clebsch-Gordan closed forms: favest/coupling.py:25-78 (same operation order)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double coupling_c(long long l) {  // coupling.py:25-29
  return sqrt((l + 1.0) / (2.0 * l + 1.0));
}
__device__ __forceinline__ double coupling_d(long long l) {  // coupling.py:32-36
  return sqrt(l / (2.0 * l + 1.0));
}

__device__ __forceinline__ double cg_explicit(int dl, int m2, long long l, long long m) {
  long long j1 = l + dl;
  long long m1 = m - m2;
  if (l < 0 || j1 < 0 || llabs(m) > l || llabs(m1) > j1) return 0.0;
  double lf = (double)l, mf = (double)m;
  if (dl == -1) {
    if (m2 == 1) return sqrt((double)(l + m) * (lf + mf - 1.0) / ((2.0 * lf) * (2.0 * lf - 1.0)));
    if (m2 == 0) return sqrt((double)((l + m) * (l - m)) / (lf * (2.0 * lf - 1.0)));
    return sqrt((double)(l - m) * (lf - mf - 1.0) / ((2.0 * lf) * (2.0 * lf - 1.0)));
  }
  if (dl == 1) {
    if (m2 == 1) return sqrt((lf - mf + 1.0) * (lf - mf + 2.0) / ((2.0 * lf + 2.0) * (2.0 * lf + 3.0)));
    if (m2 == 0) return -sqrt((lf - mf + 1.0) * (lf + mf + 1.0) / ((2.0 * lf + 3.0) * (lf + 1.0)));
    return sqrt((lf + mf + 1.0) * (lf + mf + 2.0) / ((2.0 * lf + 3.0) * (2.0 * lf + 2.0)));
  }
  if (l == 0) return 0.0;
  if (m2 == 1) return -sqrt((double)(l + m) * (lf - mf + 1.0) / (lf * (2.0 * lf + 2.0)));
  if (m2 == 0) return mf / sqrt(lf * (lf + 1.0));
  return sqrt((lf + mf + 1.0) * (double)(l - m) / (lf * (2.0 * lf + 2.0)));
}

// xi^1..6 and mu^1..3 at table position (l, m): favest/coupling.py:159-167.
// Only valid table positions (0 <= l <= lmax+1, |m| <= l) are ever requested;
// positions outside read as zero through the callers' range checks
// (favest/coupling.py:173-184).
__device__ __forceinline__ double xi_coef(int i, long long l, long long m) {
  switch (i) {
    case 1: return coupling_c(l + 1) * cg_explicit(-1, 1, l + 1, m + 1);
    case 2: return l >= 1 ? coupling_d(l - 1) * cg_explicit(1, 1, l - 1, m + 1) : 0.0;
    case 3: return coupling_c(l + 1) * cg_explicit(-1, -1, l + 1, m - 1);
    case 4: return l >= 1 ? coupling_d(l - 1) * cg_explicit(1, -1, l - 1, m - 1) : 0.0;
    case 5: return coupling_c(l + 1) * cg_explicit(-1, 0, l + 1, m);
    default: return l >= 1 ? coupling_d(l - 1) * cg_explicit(1, 0, l - 1, m) : 0.0;
  }
}
__device__ __forceinline__ double mu_coef(int i, long long l, long long m) {
  if (i == 1) return cg_explicit(0, 1, l, m + 1);
  if (i == 2) return cg_explicit(0, 0, l, m);
  return cg_explicit(0, -1, l, m - 1);
}

// Adjoint coupling of one (l, M, field): nu1..nu6, eta1..eta3
// (favest/coupling.py:227-239) and the merge into g^X, g^Y, g^Z
// (favest/transforms.py:168-175), from the nine factors x = (xi1..6, mu1..3) at
// (l, M) and the a / b entries at the shifted positions (zero outside range).
// One definition for every caller, so all paths are bitwise equal.
struct CgAdjIn {
  double2 ap1p, ap1m, am1p, am1m, ap10, am10;  // a at (l+1, M+1), (l+1, M-1), (l-1, M+1), (l-1, M-1), (l+1, M), (l-1, M)
  double2 bp, bm, b0;                          // b at (l, M+1), (l, M-1), (l, M)
};

__device__ __forceinline__ void cg_adj_merge(const double (&x)[9], const CgAdjIn& v, double2& gx, double2& gy,
                                             double2& gz) {
  const double is2 = 0.7071067811865475;  // favest/transforms.py:46 (1/np.sqrt(2.0))
  const double x1 = x[0], x2 = x[1], x3 = x[2], x4 = x[3], x5 = x[4], x6 = x[5], u1 = x[6], u2 = x[7], u3 = x[8];
  const double2 nu1 = make_double2(v.ap1p.x * x1 - v.ap1m.x * x3, v.ap1p.y * x1 - v.ap1m.y * x3);
  const double2 nu2 = make_double2(v.am1p.x * x2 - v.am1m.x * x4, v.am1p.y * x2 - v.am1m.y * x4);
  const double2 s3 = make_double2(v.ap1p.x * x1 + v.ap1m.x * x3, v.ap1p.y * x1 + v.ap1m.y * x3);
  const double2 nu3 = make_double2(-s3.y, s3.x);
  const double2 s4 = make_double2(v.am1p.x * x2 + v.am1m.x * x4, v.am1p.y * x2 + v.am1m.y * x4);
  const double2 nu4 = make_double2(-s4.y, s4.x);
  const double2 nu5 = make_double2(v.ap10.x * x5, v.ap10.y * x5);
  const double2 nu6 = make_double2(v.am10.x * x6, v.am10.y * x6);
  const double2 d1 = make_double2(v.bp.x * u1 - v.bm.x * u3, v.bp.y * u1 - v.bm.y * u3);
  const double2 eta1 = make_double2(-d1.y, d1.x);
  const double2 eta2 = make_double2(v.bp.x * u1 + v.bm.x * u3, v.bp.y * u1 + v.bm.y * u3);
  const double2 eta3 = make_double2(-(v.b0.y * u2), v.b0.x * u2);
  gx = make_double2(-is2 * ((nu1.x + nu2.x) + eta1.x), -is2 * ((nu1.y + nu2.y) + eta1.y));
  gy = make_double2(-is2 * ((nu3.x + nu4.x) - eta2.x), -is2 * ((nu3.y + nu4.y) - eta2.y));
  gz = make_double2((nu5.x + nu6.x) + eta3.x, (nu5.y + nu6.y) + eta3.y);
}

}  // namespace fv
