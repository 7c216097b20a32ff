/*
 * favest_b200.h — C ABI of the B200-native FaVeST forward / adjoint vector
 * spherical harmonic transforms (VSHT).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (pure Python, /root/reference/pkg/src/favest) dispatches its scalar
 * backends from two entry points; each function below replaces one of them:
 *
 *   fv_forward_grid    <- forward_favest(..., path="fast-scalar"|"auto")
 *                         favest/transforms.py:79-147, with its scalar stage
 *                         _forward_fast_values favest/scalar.py:146-154 and the
 *                         CG assembly favest/transforms.py:120-146
 *   fv_adjoint_grid    <- adjoint_favest(coeffs, rule|TensorGrid, ...)
 *                         favest/transforms.py:150-181 with
 *                         build_adjoint_coupling favest/coupling.py:200-240 and
 *                         _adjoint_fast_values favest/scalar.py:170-179
 *   fv_adjoint_points  <- adjoint_favest(coeffs, points) (direct route)
 *                         favest/transforms.py:150-181 with
 *                         _adjoint_direct_values favest/scalar.py:120-128
 *   fv_forward_points  <- forward_favest(samples, rule, ..., "direct-scalar")
 *                         favest/transforms.py:79-147 with
 *                         _forward_direct_values favest/scalar.py:94-105
 *   fv_forward_scalar_grid / fv_adjoint_scalar_grid
 *                      <- forward_sht_fast / adjoint_sht_fast favest/scalar.py:146-184
 *   fv_forward_scalar_points / fv_adjoint_scalar_points
 *                      <- forward_sht_direct / adjoint_sht_direct favest/scalar.py:94-128
 *   fv_plan_create_grid <- the per-grid state the reference rebuilds on every
 *                         call: TensorGrid (favest/scalar.py:29-84),
 *                         legendre_table (favest/legendre.py:36-75),
 *                         build_cg_tables (favest/coupling.py:143-170)
 *
 * Data layout (all device pointers, caller-owned, contiguous, float64):
 *   samples T   complex128 [B][N][3], N = n_theta * n_phi ring-major points
 *               (favest/scalar.py:66-74), components x, y, z
 *   coeffs a, b complex128 [B][(L+1)^2], flat index l*l + l + m
 *               (favest/core.py:23-37); entry 0 must be 0
 *   points      float64 [M][3] unit vectors
 * Complex numbers are interleaved (re, im) doubles.
 *
 * Semantics: pure functions of their inputs, asynchronous on `stream`
 * (a cudaStream_t, may be NULL for the legacy stream).  A plan is not safe for
 * concurrent calls; distinct plans are independent.  Reductions run in a fixed
 * order: results are bitwise reproducible run to run on the same device.
 *
 * Status codes: FV_OK; FV_EINVAL mirrors the reference's ValueError
 * conditions (message via fv_last_error(), same wording); FV_ECUDA, FV_ENOMEM
 * and FV_ENCCL are runtime failures (RuntimeError on the Python side).
 */
#ifndef FAVEST_B200_H
#define FAVEST_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define FV_OK 0
#define FV_EINVAL 1
#define FV_ECUDA 2
#define FV_ENCCL 3
#define FV_ENOMEM 4

typedef struct fvPlan fvPlan;

/* Version string of the library ("favest_b200 <version> sm_100a"). */
const char* fv_version(void);

/* Gauss-Legendre rule of n nodes computed on the device (Newton on the
 * colatitude; replaces scipy.special.roots_legendre inside
 * favest/quadrature.py:29-48 when requested): thetas[k] ascending colatitudes
 * (= arccos of the nodes, descending in cos), weights[k] the Gauss weights
 * (summing to 2), host arrays of n doubles.  Blocking.  Not bitwise scipy's
 * (more accurate polar weights). */
int fv_gauss_legendre(int n, double* thetas, double* weights, int device);

/* Message of the last failing call on this thread ("" if none). */
const char* fv_last_error(void);

/*
 * Grid plan for vector degree L on an iso-latitude tensor grid.
 * ring_theta_host / ring_weight_host: n_theta host doubles, colatitudes
 * strictly increasing in (0, pi) and per-point weights including the 2*pi/n_phi
 * factor (TensorGrid, favest/scalar.py:29-61) — passed through verbatim, never
 * recomputed.  Requires n_phi >= 2(L+1)+1
 * (favest/transforms.py:63-72).  max_batch bounds B of later calls.
 */
int fv_plan_create_grid(fvPlan** out, int L, int n_theta, int n_phi, const double* ring_theta_host,
                        const double* ring_weight_host, int max_batch, int device);

/* Plan for the scattered-point transforms (fv_adjoint_points, fv_forward_points) at vector degree L. */
int fv_plan_create_points(fvPlan** out, int L, int max_batch, int device);

void fv_plan_destroy(fvPlan* plan);

/* Plan properties: 1 if the grid was folded about the equator (mirror pairs). */
int fv_plan_info(const fvPlan* plan, int* L, int* n_theta, int* n_phi, int* n_pairs, int* paired);

/* Per-order Legendre work of a grid plan, for balancing the order-sharded
 * partition (the multi-GPU layout of paper_1908_00041_b200/dist.py): cost[m],
 * m = 0..L+1, is the number of (degree, ring pair) products the contraction of
 * order m actually runs -- pairs count from their polar start (the first degree
 * whose |Pbar| reaches 2^-100), not from l = m.  Blocking (a device -> host
 * copy).  Replaces the reference's nothing: favest has one process. */
int fv_order_cost(const fvPlan* plan, double* cost);

/* Forward VSHT of B tangent fields on the plan's grid: T -> (a, b). */
int fv_forward_grid(fvPlan* plan, const double* T, double* a, double* b, int B, void* stream);

/* Adjoint VSHT on the plan's grid: (a, b) -> T (Cartesian components). */
int fv_adjoint_grid(fvPlan* plan, const double* a, const double* b, double* T, int B, void* stream);

/* Adjoint VSHT at M scattered unit points: (a, b) -> T [B][M][3]. */
int fv_adjoint_points(fvPlan* plan, const double* xyz, long long M, const double* a, const double* b,
                      double* T, int B, void* stream);

/*
 * Forward VSHT at M weighted scattered points (the direct route: a rule without
 * tensor-grid structure, or path="direct-scalar"): T [B][M][3] -> (a, b).
 * Replaces forward_favest(..., path="direct-scalar") favest/transforms.py:79-147
 * with _forward_direct_values favest/scalar.py:94-105.  xyz: float64 [M][3] unit
 * points, w: float64 [M] weights (QuadratureRule.points / .weights, passed
 * through verbatim).  M = 0 gives zero coefficients.  Needs a points plan.
 */
int fv_forward_points(fvPlan* plan, const double* xyz, const double* w, long long M, const double* T, double* a,
                      double* b, int B, void* stream);

/*
 * Scalar spherical harmonic transforms of degree lmax <= the plan's L + 1
 * (favest/scalar.py:94-128, 146-184: forward_sht_fast, adjoint_sht_fast,
 * forward_sht_direct, adjoint_sht_direct).  B <= 3 * max_batch scalar fields
 * f [B][N] (grid) or [B][M] (points), coefficients [B][(lmax+1)^2] at
 * l*l + l + m.  They run through the vector kernels with the scalar fields as
 * the Cartesian components of pseudo fields (no Clebsch-Gordan stage).
 */
int fv_forward_scalar_grid(fvPlan* plan, const double* f, double* out, int lmax, int B, void* stream);
int fv_adjoint_scalar_grid(fvPlan* plan, const double* g, double* f, int lmax, int B, void* stream);
int fv_forward_scalar_points(fvPlan* plan, const double* xyz, const double* w, long long M, const double* f,
                             double* out, int lmax, int B, void* stream);
int fv_adjoint_scalar_points(fvPlan* plan, const double* xyz, long long M, const double* g, double* f, int lmax,
                             int B, void* stream);

/*
 * Order-sharded building blocks (ring-sharded fields,
 * m-sharded contraction, one all-to-all transpose per direction; the Python
 * driver is paper_1908_00041_b200/dist.py).  Together they are exactly
 * fv_forward_grid / fv_adjoint_grid split at the transpose:
 *   fv_forward_grid  = fv_ring_fft(forward) ; fv_forward_orders(all orders)
 *   fv_adjoint_grid  = fv_adjoint_orders(all orders) ; fv_ring_fft(inverse)
 *
 * Spectra: element (component c, ring R, bin j) at c*cs + R*rs + j*bs complex
 * units, R = field * n_theta + ring over ALL rings of the plan's grid.  nbins = 0:
 * natural DFT bins (order m at bin m, -m at (n_phi - m) % n_phi); nbins > 0:
 * compact bins holding orders bin_lo .. bin_lo + nbins - 1 (+m at m - bin_lo,
 * -m at nbins + m - bin_lo).
 */

/* 3 x nrings ring DFTs of length n_phi (favest/scalar.py:149 forward, :178
 * inverse unnormalised); element (c, ring, q) at c*cs + ring*rs + q*es. */
int fv_ring_fft(fvPlan* plan, int inverse, const double* in, long long in_cs, long long in_rs, long long in_es,
                double* out, long long out_cs, long long out_rs, long long out_es, int nrings, void* stream);

/* Forward contraction for Legendre orders [m_lo, m_hi) and CG assembly of the
 * coefficient orders [c_lo, c_hi) (favest/scalar.py:150-154 restricted to those
 * orders, favest/transforms.py:120-146); entries of a, b for other orders are
 * not touched.  Needs m_lo <= c_lo - 1 (or c_lo = 0 = m_lo) and c_hi <= m_hi - 1. */
int fv_forward_orders(fvPlan* plan, const double* S, long long cs, long long rs, long long bs, int bin_lo, int nbins,
                      double* a, double* b, int B, int m_lo, int m_hi, int c_lo, int c_hi, void* stream);

/* Adjoint coupling + synthesis of orders [m_lo, m_hi) into the spectra
 * (favest/coupling.py:227-239, favest/scalar.py:170-177 restricted to those
 * orders); reads a, b at orders m_lo - 1 .. m_hi. */
int fv_adjoint_orders(fvPlan* plan, const double* a, const double* b, int B, int m_lo, int m_hi, double* S,
                      long long cs, long long rs, long long bs, int bin_lo, int nbins, void* stream);

/* The same two stages on "packed" spectra: element (component c, ring R, bin j)
 * at ring_offsets[c * rts + R] + j complex units (ring_offsets: device int64,
 * 3 x rts entries, rts >= B * n_theta; compact bins, nbins > 0), so the blocks
 * of an all-to-all buffer -- one contiguous block per peer rank -- are read
 * (forward) or written (adjoint) in place, with no pack / unpack copies. */
int fv_forward_orders_packed(fvPlan* plan, const double* S, const long long* ring_offsets, long long rts, int bin_lo,
                             int nbins, double* a, double* b, int B, int m_lo, int m_hi, int c_lo, int c_hi,
                             void* stream);
int fv_adjoint_orders_packed(fvPlan* plan, const double* a, const double* b, int B, int m_lo, int m_hi, double* S,
                             const long long* ring_offsets, long long rts, int bin_lo, int nbins, void* stream);

/*
 * Stage timing (milliseconds, CUDA events recorded on each call's stream):
 * fv_set_profiling(plan, 1) starts accumulating over all following calls,
 * fv_stage_ms sums one stage (0 fft, 1 fold, 2 legendre, 3 cg) and the number
 * of launches of that stage is fv_stage_count.  fv_set_profiling(plan, 0)
 * stops and resets.  Returns -1 if nothing was recorded.
 */
int fv_set_profiling(fvPlan* plan, int enable);
double fv_stage_ms(const fvPlan* plan, int stage);
int fv_stage_count(const fvPlan* plan, int stage);

#ifdef __cplusplus
}
#endif
#endif /* FAVEST_B200_H */
