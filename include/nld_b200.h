/*
 * nld_b200.h -- C-ABI of the B200-native ANOVA-Laplacian hot path.
 *
 * This is the drop-in boundary for the reference package `nldenoise`
 * (/root/reference/pkg/src/nldenoise).  The reference is in-process Python,
 * so its "FFI" is its Python call surface; each entry point below replaces
 * one reference interface (file:line cited) and is bound by the Python shim
 * `paper_2407_06834_b200/_lib.py` through ctypes.
 *
 * Conventions
 *  - every function returns an int status: NLD_OK or one of NLD_ERR_*;
 *    nld_last_error() returns a thread-local message for the last failure.
 *    The codes map one-to-one onto the reference exception classes
 *    (errors.py:4-45).
 *  - vectors and features are DEVICE pointers (fp64) unless stated;
 *    `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - batched right-hand sides are row-major [nrhs][n] with leading
 *    dimension `ld` (>= n).
 *  - no torch types cross this boundary.
 */
#ifndef NLD_B200_H
#define NLD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NLD_ABI_VERSION 1

#if defined(__GNUC__)
#define NLD_API __attribute__((visibility("default")))
#else
#define NLD_API
#endif

/* status codes -> reference exceptions (errors.py) */
#define NLD_OK 0
#define NLD_ERR_DIMENSION 1   /* DimensionMismatchError (errors.py:24)      */
#define NLD_ERR_SCALING 2     /* ScalingOverflowError  (errors.py:28-29)    */
#define NLD_ERR_WINDOW 3      /* WindowSizeError       (errors.py:32-33)    */
#define NLD_ERR_DENSE_LIMIT 4 /* DenseLimitError       (errors.py:36-37)    */
#define NLD_ERR_BREAKDOWN 5   /* SolverBreakdownError  (errors.py:40-41)    */
#define NLD_ERR_VALUE 6       /* ValueError                                 */
#define NLD_ERR_CUDA 7        /* RuntimeError: CUDA failure / no device     */

/* operator kinds for nld_op_apply */
#define NLD_APPLY_GAMMA 0          /* Gamma v            kernel.py:118-127   */
#define NLD_APPLY_GAMMA_SQUARED 1  /* squared subkernels kernel.py:129-140   */
#define NLD_APPLY_SYSTEM 2         /* lam v + mu(eta v - Gamma v) linops.py:48-50 */
#define NLD_APPLY_LAPLACIAN 3      /* eta v - Gamma v    linops.py:43-46     */
#define NLD_APPLY_WINDOW_SUM 4     /* sum_l G_l v (unit diagonal kept)       */
/* OR into `kind`: batched v / out are pixel-major [n][nrhs] (rhs fastest,
 * ld ignored) -- the kernels' native layout, no transposes */
#define NLD_LAYOUT_PIXEL_MAJOR 0x100

/* preconditioners for nld_cg_solve (deflated_solve's prec, linops.py:286-293) */
#define NLD_PREC_NONE 0
#define NLD_PREC_JACOBI 1
#define NLD_PREC_L2 2

typedef struct nld_operator nld_operator;

/* Collective hook for pixel sharding.  The library calls it at
 * the plan-build reductions (torus bbox / radius / support box), once per
 * product for the per-window grid sum, and for the CG scalars.
 * dtype: 0 f64, 1 i32; op: 0 sum, 1 min, 2 max; on_device: buf is a device
 * pointer ordered on `stream` (else a host pointer).  Returns 0 on success. */
typedef int (*nld_allreduce_fn)(void* ctx, void* buf, int64_t count, int32_t dtype,
                                int32_t op, int32_t on_device, void* stream);

/* NFFT / fast-summation parameters, FastsumPlan.build (transform.py:273-283).
 * n_expansion <= 0 selects the reference's adaptive expansion_degree
 * (transform.py:254-258); mode 0 = "fast", 1 = "exact" (kernel.py:28-29).
 * no_sliced: 0 (default) runs 16k-rhs batches of 3-D m = 4 windows on the
 * integer-sliced tcgen05 kernels (exact int8 digit products, fp64 combine);
 * 1 runs them on the fp64 DMMA kernels (results agree to rounding). */
typedef struct {
  int32_t n_expansion;
  int32_t cutoff;
  double oversampling;
  double rmax;
  double truncation_eps;
  int32_t mode;
  int32_t no_sliced;
  int64_t dense_limit;
} nld_params;

/* per-window plan summary (FastsumPlan fields, transform.py:261-270) */
typedef struct {
  int32_t dim;
  int32_t bandwidth;      /* N_d                                   */
  int32_t grid;           /* oversampled n = 2 ceil(os N_d / 2)    */
  int32_t cutoff;
  double center[3];
  double scale;
  double sig_scaled;
  int32_t box_lo[3];      /* support box of the spread grid        */
  int32_t box_w[3];
  int64_t n_cells;        /* occupied stencil cells                */
  int64_t n_subproblems;  /* work items: parts of one cell, <= 2048..8192 nodes */
  int64_t n_edge;         /* nodes with 2m+1 nonzero weights       */
} nld_window_info;

/* per-call stage timings (CUDA events), last nld_op_apply */
typedef struct {
  float spread_ms;
  float assemble_ms;
  float conv_ms;
  float gather_ms;
  float epilogue_ms;
  float total_ms;
  int32_t launches;
  int32_t reserved;
} nld_stats;

NLD_API const char* nld_last_error(void);
NLD_API int nld_abi_version(void);

/* AnovaOperator.__init__ + lazy _build_plans (kernel.py:28-77,
 * transform.py:272-320).  features_dev: (n, n_features) row-major fp64 on the
 * device; windows given as CSR on the HOST: window w uses feature columns
 * window_index[window_offset[w] .. window_offset[w+1]).  Plans, node tables,
 * the cell sort and the subproblem lists are built here and owned by the
 * handle; the features are copied per window as the reference does
 * (kernel.py:73). */
NLD_API int nld_op_create(const double* features_dev, int64_t n, int32_t n_features,
                  const int32_t* window_index, const int32_t* window_offset,
                  int32_t n_windows, double sigma, const nld_params* params,
                  void* stream, nld_operator** out);
NLD_API int nld_op_destroy(nld_operator* op);

/* Make `op` one shard of a pixel-sharded operator: its nodes are a slice of
 * global_n nodes.  Must be called before the first product (plan build). */
NLD_API int nld_op_set_comm(nld_operator* op, nld_allreduce_fn fn, void* ctx,
                            int64_t global_n);

/* One fused product per right-hand side (kernel.py:79-93, linops.py:43-50).
 * coef: per-rhs (lam, mu) pairs for NLD_APPLY_SYSTEM, ignored otherwise.
 * NLD_APPLY_SYSTEM/LAPLACIAN use the cached degree (nld_op_degree).
 * Pixel-major batches (kind | NLD_LAYOUT_PIXEL_MAJOR, v/out = [n][nrhs]) are
 * the kernels' native layout; with v and out 32-byte aligned (any cudaMalloc'd
 * or torch-allocated buffer) the window sum and the degree/shift terms are
 * fused into the last window's gather, otherwise the product goes through
 * the library's aligned workspace (same result, one more pass). */
NLD_API int nld_op_apply(nld_operator* op, int32_t kind, const double* v, double* out,
                 int32_t nrhs, int64_t ld, const double* coef_host,
                 void* stream);

/* eta = Gamma 1 (kernel.py:142-146), cached on the device; squared != 0
 * gives degree_squared (kernel.py:148-154).  eta_out may be NULL (just
 * build the cache) or a device buffer of n doubles. */
NLD_API int nld_op_degree(nld_operator* op, int32_t squared, double* eta_out,
                  void* stream);

/* dense kernel matrix with zero diagonal, (n, n) row-major device buffer
 * (kernel.py:156-158); NLD_ERR_DENSE_LIMIT above params.dense_limit. */
NLD_API int nld_op_assemble_dense(nld_operator* op, int32_t squared, double* out,
                          void* stream);

NLD_API int nld_op_window_info(const nld_operator* op, int32_t window,
                       nld_window_info* out);
NLD_API int nld_op_stats(const nld_operator* op, nld_stats* out);
NLD_API int nld_op_set_timing(nld_operator* op, int32_t enabled);
/* Test hook (no reference counterpart): fill every allocated workspace
 * buffer of the operator (blocks, grids, convolution scratch, per-window
 * gathers, G digits, assemble scratch, CG vectors) with 0xFF bytes -- NaN as
 * doubles -- so a later product that read workspace it did not write first
 * would return NaN or garbage (an initcheck that needs no sanitizer). */
NLD_API int nld_op_debug_poison(nld_operator* op);

/* deflated_solve / plain_solve (linops.py:263-319) on nrhs systems
 * A_r = lam_r I + mu_r (diag eta - Gamma) sharing every Gamma application.
 * f, u: device [nrhs][ld].  lam/mu/iterations/relres/converged are HOST
 * arrays of nrhs; history (HOST, may be NULL) is [nrhs][history_cap] and
 * receives residual_history (linops.py:184-190), padded with NaN.
 * deflate != 0 -> deflated_solve (constant eigenvector split off),
 * 0 -> plain_solve. */
NLD_API int nld_cg_solve(nld_operator* op, const double* f, double* u, int32_t nrhs,
                 int64_t ld, const double* lam, const double* mu,
                 int32_t precond, int32_t deflate, double tol, int32_t maxit,
                 int32_t warm_start, int32_t* iterations, double* relres,
                 int32_t* converged, double* history, int32_t history_cap,
                 void* stream);

/* DeflatingBasis.apply / apply_adjoint (linops.py:134-176) for a device
 * vector v of length n (v[0] != 0): out = U x or U^T x. */
NLD_API int nld_basis_apply(const double* v, const double* x, double* out, int64_t n,
                    int32_t adjoint, void* stream);

/* scs_up / scs_down (linops.py:114-131) on device vectors. */
NLD_API int nld_scs(const double* x, double* out, int64_t n, int32_t down,
            void* stream);

/* small device vector kernels used by the generic pcg (linops.py:193-244):
 * out = a x + b y;   dots[k] = <x_k, y_k> for k < count (HOST result). */
NLD_API int nld_axpby(double a, const double* x, double b, const double* y,
              double* out, int64_t n, void* stream);
NLD_API int nld_dot(const double* x, const double* y, int64_t n, double* result,
            void* stream);

/* ---- general transforms (transform.py:74-333) ------------------------------
 * An NFFT plan is an nld_operator in raw-torus mode over n nodes of dimension d
 * (device, row-major) mapped by (p - center) * scale (center may be NULL = 0;
 * check_torus != 0 raises NLD_ERR_SCALING if a mapped node leaves
 * [-1/2, 1/2)^d as map_to_torus does, transform.py:310-317).  Bandwidth M is
 * the same in every dimension (even); the grid is n = 2 ceil(os M / 2).
 * Complex arrays are interleaved (re, im) fp64, coefficients C-order over
 * k = -M/2 .. M/2-1 per dimension.  Destroy with nld_op_destroy. */
NLD_API int nld_nfft_create(const double* nodes_dev, int64_t n, int32_t d,
                            int32_t bandwidth, double oversampling, int32_t cutoff,
                            const double* center, double scale, int32_t check_torus,
                            void* stream, nld_operator** out);
/* nfft_adjoint (transform.py:215-223): coeffs = deconv(ifftn(spread(values))
 * * prod(nos)), optionally times a real multiplier (kernel coefficients). */
NLD_API int nld_nfft_adjoint(nld_operator* plan, const double* values, double* coeffs,
                             const double* mult, void* stream);
/* nfft (transform.py:200-212): values = gather(fftn(embed(deconv(coeffs)))). */
NLD_API int nld_nfft_trafo(nld_operator* plan, const double* coeffs, double* values,
                           void* stream);
/* ndft / ndft_adjoint (transform.py:74-102), exact O(n M^d). */
NLD_API int nld_ndft(const double* nodes, int64_t n, int32_t d, int32_t bandwidth,
                     const double* in, double* out, int32_t adjoint, void* stream);
/* gauss_transform_direct (transform.py:231-244), exact. */
NLD_API int nld_gauss_direct(const double* targets, int64_t nt, const double* sources,
                             int64_t ns, int32_t d, const double* alpha, double sigbar,
                             double* out, void* stream);
/* FastsumPlan.build pieces (transform.py:292-307): bounding-box centre and
 * scale (HOST outputs), and kernel_coeffs (device, M^d real). */
NLD_API int nld_fastsum_geometry(const double* points, int64_t n, int32_t d, double rmax,
                                 double* center_host, double* scale_host, void* stream);
NLD_API int nld_gauss_coeffs(int32_t bandwidth, int32_t d, double sig_scaled, double* out,
                             void* stream);
/* NfftPlan.window_factors (transform.py:140-145), HOST output of M values. */
NLD_API int nld_window_factors(int32_t bandwidth, int32_t grid, int32_t cutoff,
                               double* out_host);

/* ---- feature / window preparation (features.py:20-104) ------------------
 * image: device, channel-planar [channels][h][w] fp64.  out: device
 * (h*w, channels*patch^2), columns channel-major then raster patch order,
 * value a * (v - b); mode 0 pads with zeros (the reference, a=1, b=0),
 * mode 1 reflects (BASELINE's generator, a=0.4, b=0.5). */
NLD_API int nld_extract_patches(const double* image, int64_t h, int64_t w, int32_t channels,
                                int32_t patch, int32_t mode, double a, double b,
                                double* out, void* stream);
/* plug-in mutual information (nats) of every column with column `center`,
 * 16 x 16 equal-width bins over each column's range; HOST output of d. */
NLD_API int nld_mi_scores(const double* features, int64_t n, int32_t d, int32_t center,
                          double* scores_host, void* stream);

/* fp64 FMA throughput probe (the roofline denominator of the FMA-bound
 * spread/gather kernels): 8 independent DFMA chains per thread, `iters`
 * steps, `blocks` x 256 threads (<= 0: 8 per SM).  HOST outputs. */
NLD_API int nld_probe_fp64(int64_t iters, int32_t blocks, double* tflops,
                           double* ms, void* stream);
/* the same for the fp64 tensor path (mma.sync m8n8k4 f64, DMMA). */
NLD_API int nld_probe_dmma(int64_t iters, int32_t blocks, double* tflops,
                           double* ms, void* stream);
/* half the warps DMMA, half DFMA: do the two fp64 paths share resources? */
/* int8 tensor-core (tcgen05 kind::i8, M=128 N=256 K=32) throughput probe: the
 * roofline denominator of the integer-sliced spread / gather (TOPS). */
NLD_API int nld_probe_imma(int64_t iters, int32_t blocks, double* tops, double* ms,
                           void* stream);
NLD_API int nld_probe_mixed(int64_t iters_mma, int64_t iters_fma, double* tflops,
                            double* ms, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NLD_B200_H */
