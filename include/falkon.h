/*
 * falkon.h — C ABI of the B200-native Falkon hot path (libfalkon.so).
 *
 * What the library computes (PAPER.md = arXiv 2006.10350 text, cited by line):
 *   - the Nystrom kernel product  u = Knm^T (Knm v)  in row blocks, Knm never stored
 *     ("Blockwise Knm-vector product"), summed over all ranks;
 *   - the one-sided products  w = Knm v  and  u = Knm^T w  (Alg. 1 line 9, PAPER.md:114;
 *     prediction Eq. (4));
 *   - the Falkon preconditioner  T = chol(Kmm),  A = chol(T T^T / m + lambda I)  in ONE
 *     m x m fp64 buffer (Alg. 1 lines 13-17; Eq. (7) PAPER.md:254-256;
 *     in-place layout PAPER.md:257-265 and Fig. 3);
 *   - Falkon's preconditioned CG (Alg. 1) with LinOp read as
 *     Eq. (9):  A^-T ( T^-T Knm^T Knm T^-1 A^-1 beta + lambda n A^-1 beta ).
 *
 * Kernels (`kernel` argument):
 *   FALKON_GAUSSIAN   k(x,c) = exp(-||x-c||^2 / (2 sigma^2))
 *   FALKON_LAPLACIAN  k(x,c) = exp(-||x-c|| / sigma)            (reading c7)
 *
 * Conventions (all entry points):
 *   - Matrices are ROW-MAJOR, contiguous: X is n_local x d, C is m x d (fp32).
 *   - Pointers may be CUDA device pointers on the context's device OR host pointers
 *     (pinned or pageable); host inputs are staged into the context workspace, host
 *     outputs are copied back.  If ANY output pointer is host memory the call
 *     synchronises the context stream before returning; otherwise the call is
 *     stream-ordered (asynchronous) on the context stream (see falkon_ctx_set_stream).
 *     falkon_fit and the preconditioner build always return with results ready.
 *   - Sizes are int64_t.  Arrays are caller-owned and never retained after return.
 *   - Multi-GPU: one context per process/GPU.  X, y, f are ROW SHARDS (n_local rows on
 *     this rank); C, v, u, alpha are REPLICATED.  Every call that produces an m-vector
 *     sums it over all ranks with one NCCL allreduce; lambda * n uses
 *     the GLOBAL n = sum of n_local (reading c15).
 *   - Errors: functions return FALKON_OK (0) or an error code; falkon_strerror() names
 *     it and falkon_last_error() returns a message with details.  On error, outputs are
 *     unspecified.  EINVAL is returned for NULL pointers, n_local < 0, d < 1, m < 1,
 *     sigma <= 0 or non-finite, lambda < 0, iters < 0, unknown kernel.
 *   - Not re-entrant on one context; different contexts are independent.
 */
#ifndef FALKON_H_
#define FALKON_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct falkon_ctx falkon_ctx;

enum { FALKON_GAUSSIAN = 0, FALKON_LAPLACIAN = 1 };

enum {
  FALKON_OK = 0,
  FALKON_EINVAL = 1,     /* invalid argument */
  FALKON_ENOTPD = 2,     /* Cholesky met a non-positive pivot (see falkon_fit_info) */
  FALKON_ENONFINITE = 3, /* CG: p^T A p <= 0 or non-finite (reading c9) */
  FALKON_ENOMEM = 4,     /* device allocation failed */
  FALKON_ECUDA = 5,      /* CUDA runtime error */
  FALKON_ENCCL = 6,      /* NCCL error or NCCL library not loadable */
  FALKON_EUNSUPPORTED = 7 /* no sm_100 device / feature unavailable */
};

/* Product-path selection (falkon_ctx_set_option FALKON_OPT_PATH). */
enum { FALKON_PATH_AUTO = 0, FALKON_PATH_SIMT = 1, FALKON_PATH_TENSOR = 2,
       /* fp64 throughout (reading d4): coordinates (x - mu) g in fp64 from the fp32
          inputs, fp64 exponent and exp2, fp64 contractions (~1e-15 relative kernel values; the
          FP64 pipe binds, ~4e11 n*m/s at d = 28).  Single-vector products and fits only
          (multi-output calls return FALKON_EUNSUPPORTED). */
       FALKON_PATH_F64 = 3 };

/* Options (falkon_ctx_set_option). */
enum {
  FALKON_OPT_PATH = 1,          /* FALKON_PATH_*; AUTO = tensor cores for Gaussian with d > threshold */
  FALKON_OPT_TC_MIN_D = 2,      /* AUTO: tensor path for d > this (default 4: measured crossover at
                                   n = 1e7, tensor 1.77e12 vs SIMT 1.42e12 n*m/s at d = 6) */
  FALKON_OPT_TC_TERMS = 3,      /* fp16 split terms of the tensor cross term: only 3 is built (the
                                   fp32-accurate h.h + l.h + h.l split); other values return
                                   FALKON_EUNSUPPORTED (1 and 2 terms fail the alpha bar) */
  FALKON_OPT_KERNEL_TIMING = 4, /* 1: record CUDA events around every launch (falkon_ctx_timings) */
  FALKON_OPT_EXP_OFFLOAD = 5,   /* tensor path: exp2 on the FMA pipe for 0 = none, 1 = all,
                                   2 = 1/4, 3 = 1/2 of the entries (rest on MUFU) */
  FALKON_OPT_POTRF_OUTER = 6,   /* blocked Cholesky: depth of the trailing fp64 GEMM updates in
                                   units of 128 columns (1..64; 0 = auto (default): 16 with the
                                   Ozaki GEMMs, 8 with the DMMA ones, as measured) */
  FALKON_OPT_GEMM_WARPS = 7,    /* fp64 DMMA GEMM CTA: 8 (128 x 128 tile, 8 warps), 16 (16 warps),
                                   2 (128 x 64 tiles, 2 CTAs of 8 warps per SM) or 5 (default:
                                   TMA-fed producer warp + 8 DMMA warps for the GEMMs whose A and B
                                   are the same view, 2 elsewhere) */
  FALKON_OPT_SINGLE_EVAL = 8,   /* single-vector products on the tensor path: 0 = two passes (the
                                   cross term and exp evaluated twice), 1 = single evaluation:
                                   pass A also stores k(x_i, c_j) for a strip of rows in HBM and
                                   u += strip^T w reads them back, 2 = auto
                                   (default: single evaluation when d > 190, where the fp16x3
                                   cross term costs more than the 8 B/entry strip round trip) */
  FALKON_OPT_STRIP_BYTES = 9,   /* single evaluation: device bytes of the k strip (default 16 GiB,
                                   minimum 64 MiB; rows per strip = bytes / (4 m)) */
  FALKON_OPT_TC_CLUSTER = 10,   /* tensor path: 1 = one CTA per P tile; 2 = clusters of two CTAs on
                                   consecutive P tiles, each loading half of every streamed Q box
                                   and multicasting it to both (halves the L2 -> SM traffic) */
  FALKON_OPT_LOOKAHEAD = 11,    /* blocked Cholesky: 1 (default) = the next outer panel's
                                   factorisation runs on a high-priority stream while the bulk of
                                   the trailing update runs on a low-priority one; 0 = serial */
  FALKON_OPT_ACCUM_F64 = 12,    /* precision of the two contractions (SURVEY.md §7 hard part 3):
                                   0 = fp32 v and w, fp32 partial sums flushed to fp64 per tile;
                                   1 = fp64 v and w, each exact product k(x,c) * v accumulated by
                                   DFMA in fp64 (k itself stays fp32).  Applies to the single-vector
                                   products, fits, GSC fits and predictions; multi-output calls
                                   stay fp32.  See DESIGN.md for the measured default. */
  FALKON_OPT_FIT_PRECISE = 14,  /* 1 (default): fits (falkon_fit, falkon_gsc_fit) on the AUTO path
                                   take (a) FALKON_PATH_F64 when d <= 32 and m > 25,000 (fp32
                                   kernel values put alpha past the 1e-3 bar there, DESIGN.md
                                   reading d4), else (b) the SIMT kernels when the AUTO path is
                                   the tensor kernel, d <= 32 and the mean scaled centre norm
                                   ||c~||^2/2 exceeds 4 (the tensor cores' truncating accumulation
                                   biases K, reading d3); 0 = always the AUTO path */
  FALKON_OPT_DIST_PRECOND = 13, /* 1: build the preconditioner with the distributed schedule
                                   (NEXT-1, below) even on a 1-rank NCCL communicator (tests the
                                   broadcast path on one GPU).  With world > 1 it is always used. */
  FALKON_OPT_OZAKI = 16,        /* 1 (default): the preconditioner's large fp64 GEMMs (Cholesky
                                   trailing updates with k range >= 256, the LAUUM T D T^T in k
                                   chunks of 1024) run on the int8 tensor cores by the
                                   Ozaki scheme (error-free split into 8 signed 7-bit slices per
                                   row-scaled operand, 36 exact int32 slice products, fp64
                                   recombination; ~1e-15 relative, deterministic, not bitwise equal
                                   to the DMMA GEMM); 0 = fp64 DMMA.  Measured: m = 5e4 build
                                   4.10 -> 3.06 s. */
  FALKON_OPT_SE_GEMV_SMS = 15   /* single evaluation schedule: G > 0 = split SMs (two strip
                                   buffers; the GEMV of strip s runs as a persistent grid of G CTAs
                                   on a highest-priority stream while pass A of strip s + 1 takes
                                   the other SMs; the last strip's GEMV uses the whole GPU);
                                   0 (default) = serial (pass A of a strip, then its GEMV on all
                                   SMs): measured faster on TIMIT (314 vs 352-389 ms per product,
                                   DESIGN.md §7).  0 <= G < SM count, else FALKON_EINVAL. */
};

/* Per-launch-class accumulated device times in ms (falkon_ctx_timings). */
enum {
  FALKON_T_PREP = 0,      /* a1: centering / scaling / packing / norms */
  FALKON_T_PASS_A = 1,    /* a2-a4: w = Knm v  (fused cross term + exp + contraction) */
  FALKON_T_PASS_B = 2,    /* a2,a3,a5: u = Knm^T w */
  FALKON_T_REDUCE = 3,    /* deterministic fp64 reduction of per-CTA partials */
  FALKON_T_ALLREDUCE = 4, /* a6: NCCL allreduce(m) */
  FALKON_T_PRECOND = 5,   /* a9: Kmm, POTRF, LAUUM, POTRF */
  FALKON_T_TRSV = 6,      /* a7: triangular solves */
  FALKON_T_VEC = 7,       /* a7: CG vector ops */
  FALKON_T_COUNT = 8
};

typedef struct {
  double jitter_used;      /* delta actually added to diag(Kmm) (reading c6) */
  int32_t failed_factor;   /* ENOTPD: 0 = T (Kmm), 1 = A (T T^T/m + lambda I); else -1 */
  int64_t failed_column;   /* ENOTPD: first non-positive pivot column; else -1 */
  int32_t iters_run;       /* < iters only on exact breakdown r^T r == 0 */
  int32_t failed_iter;     /* ENONFINITE: CG iteration (1-based); else -1 */
  double t_precond_s;      /* phase times (Table 1 split), device clock */
  double t_rhs_s;
  double t_cg_s;
  double t_total_s;
  int32_t product_path;    /* FALKON_PATH_SIMT / _TENSOR / _F64: the product kernels the fit used */
} falkon_fit_info;

/* ---- context ------------------------------------------------------------------------- */

/* NCCL unique id for a multi-rank context.  Call on rank 0, broadcast the 128 bytes to all
   ranks (e.g. with torch.distributed), then call falkon_ctx_create on every rank. */
int falkon_get_unique_id(unsigned char id[128]);

/* Create a context on CUDA device `device` for rank `rank` of `world` ranks.  `id` is
   required when world > 1; with world == 1 a non-NULL id creates a 1-rank NCCL communicator
   (every m-vector still goes through ncclAllReduce: used to test the collective path on one
   GPU).  Requires an sm_100 device (returns FALKON_EUNSUPPORTED otherwise).
   The context owns a CUDA stream, a device workspace and (world > 1) an NCCL communicator. */
int falkon_ctx_create(falkon_ctx **out, int device, int rank, int world, const unsigned char *id);
int falkon_ctx_destroy(falkon_ctx *ctx);

/* Make the context launch on `stream` (a cudaStream_t cast to void*; NULL = the legacy
   default stream).  Until this is called the context uses its own non-blocking stream.
   The caller keeps ownership of the stream. */
int falkon_ctx_set_stream(falkon_ctx *ctx, void *stream);
int falkon_ctx_set_option(falkon_ctx *ctx, int option, int64_t value);
/* Accumulated per-class device times (ms) since the last reset; out has FALKON_T_COUNT
   entries; launches[] (optional) receives the number of kernel launches per class. */
int falkon_ctx_timings(falkon_ctx *ctx, double *out_ms, int64_t *launches, int reset);
/* Total number of kernel launches issued by the library on this context. */
int64_t falkon_ctx_launch_count(const falkon_ctx *ctx);

/* ---- the hot path ---------------------------------------------------------------------- */

/* u = sum over ranks of Knm_r^T (Knm_r v).
   X: n_local x d fp32 (row shard).  C: m x d fp32 (replicated).  v: m fp64 (replicated;
   rounded to fp32 for the contractions).  u: m fp64 (allreduced; identical on all ranks).
   n_local == 0 is allowed (contributes zero). */
int falkon_knm_matvec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                      const float *C, int64_t m, int kernel, double sigma,
                      const double *v, double *u);

/* w = Knm v on this rank's rows (no collective).  w: n_local fp64. */
int falkon_kernel_vec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                      const float *C, int64_t m, int kernel, double sigma,
                      const double *v, double *w);

/* u = sum over ranks of Knm_r^T w_r  (Alg. 1 line 9 right-hand side).  w: n_local fp64. */
int falkon_kernel_tvec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                       const float *C, int64_t m, int kernel, double sigma,
                       const double *w, double *u);

/* ---- preconditioner (supporting machinery of the CG loop) ------------------------------ */

/* Number of fp64 elements of the `work` buffer of falkon_precond_build / _solve (the
   inverses of the 64 x 64 diagonal blocks of T^T and A^T, 2 * ceil(m/64) * 4096). */
int64_t falkon_precond_work_elems(int64_t m);

/* Build the preconditioner into the caller-owned m x m fp64 row-major buffer `P`, the
   two m-vectors diagT, diagA and `work` (falkon_precond_work_elems(m) doubles), all device
   memory (Fig. 3):
     strictly-upper(P) = strictly-upper(T),  diagT = diag(T),   T^T T = Kmm + delta I
     strictly-lower(P) = strictly-lower(A^T), diagA = diag(A),  A^T A = T T^T/m + lambda I
   (T, A upper triangular; the diagonal of P is scratch).  delta = jitter (< 0: default
   1e-8).  Replicated: every rank builds the same bits (no collective).  Returns ENOTPD with
   info->failed_factor/failed_column set when a pivot is <= 0 or non-finite. */
int falkon_precond_build(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                         double sigma, double lambda, double jitter,
                         double *P, double *diagT, double *diagA, double *work,
                         falkon_fit_info *info);

/* Distributed preconditioner build (multi-GPU Cholesky of PAPER.md:460-469,
   App. C Alg. 3/4 PAPER.md:1073-1216), here with G ranks SIMULATED in this process on the
   context's device: rank r's buffers are P[r] (m x m), diagT[r], diagA[r] (m) and work[r]
   (falkon_precond_work_elems(m)), all device memory, arrays of G host-side pointers.
   Schedule (also what falkon_fit runs across real ranks when world > 1): outer panel j of
   each factor (potrf_outer x 128 columns) belongs to rank j mod G; its owner factors it, the
   factored panel is broadcast, and every rank applies the trailing update to its own column
   panels; the LAUUM T T^T/m is split by the same column panels.  Every rank ends with the same
   bits as falkon_precond_build (same GEMM calls per element).  Errors as
   falkon_precond_build; EINVAL for G outside 1..64. */
int falkon_precond_build_sim(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                             double sigma, double lambda, double jitter, int G, double *const *P,
                             double *const *diagT, double *const *diagA, double *const *work,
                             falkon_fit_info *info);

/* In-place triangular solve x <- op(F)^-1 x with F = T (which = 0) or A (which = 1) read
   from a buffer built by falkon_precond_build (with its work buffer); op = transpose if
   trans != 0.  x: m fp64 device memory.  Stream-ordered. */
int falkon_precond_solve(falkon_ctx *ctx, const double *P, const double *diagT,
                         const double *diagA, const double *work, int64_t m, int which,
                         int trans, double *x);

/* Multi-column form of falkon_precond_solve: column c of x starts at x + c * ldx (ldx >= m),
   c < k.  One pass over the triangle per 16 columns (multi-output fits). */
int falkon_precond_solve_multi(falkon_ctx *ctx, const double *P, const double *diagT,
                               const double *diagA, const double *work, int64_t m, int which,
                               int trans, double *x, int64_t ldx, int64_t k);

/* ---- Falkon ---------------------------------------------------------------------------- */

/* alpha = Falkon(X, y, C, kernel, sigma, lambda, iters)  (Alg. 1).
   y: n_local fp32 targets (row shard).  alpha: m fp64 (replicated).  jitter < 0 -> 1e-8.
   iters == 0 -> alpha = 0.  info (host, optional) receives phase times and diagnostics.
   The m x m fp64 buffer (8 m^2 bytes) is allocated for the call and freed at return. */
int falkon_fit(falkon_ctx *ctx, const float *X, const float *y, int64_t n_local, int64_t d,
               const float *C, int64_t m, int kernel, double sigma, double lambda,
               int32_t iters, double jitter, double *alpha, falkon_fit_info *info);

/* f = k(X, C) alpha  (Eq. (4)) on this rank's rows; no collective.
   alpha: m fp64.  f: n_local fp64. */
int falkon_predict(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                   const float *C, int64_t m, int kernel, double sigma,
                   const double *alpha, double *f);

/* ---- multi-output (k outputs, e.g. TIMIT's 144 classes) -- */

/* U = sum over ranks of Knm_r^T (Knm_r V) for k vectors at once.  V, U: m x k fp64 ROW-MAJOR
   (replicated; U allreduced).  On the tensor path the vectors go through the fused kernel in
   blocks of 8 or 16 (one cross term + exp per entry for the whole block);
   on the SIMT path (Laplacian, d <= 8) each column is its own pass.  k >= 1. */
int falkon_knm_matmat(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                      const float *C, int64_t m, int kernel, double sigma,
                      const double *V, int64_t k, double *U);

/* F = k(X, C) alpha for k coefficient columns (Eq. (4)); alpha m x k, F n_local x k fp64,
   row-major; no collective. */
int falkon_predict_multi(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                         const float *C, int64_t m, int kernel, double sigma,
                         const double *alpha, int64_t k, double *F);

/* Multi-output Falkon: Alg. 1 for the k columns of Y (n_local x k fp32 row-major) at once.
   The k CGs are independent (per-column step sizes and breakdown rules, reading c9) and share
   the preconditioner and every kernel product.  alpha: m x k fp64 row-major (replicated).
   info->iters_run is the mean over columns; other fields as falkon_fit. */
int falkon_fit_multi(falkon_ctx *ctx, const float *X, const float *Y, int64_t n_local, int64_t d,
                     const float *C, int64_t m, int64_t k, int kernel, double sigma,
                     double lambda, int32_t iters, double jitter, double *alpha,
                     falkon_fit_info *info);

/* ---- GSC-Falkon / LogFalkon (Appendix B, Alg. 2) ------------------- */

/* Losses of falkon_gsc_fit (Def. 1 / Example 1). */
enum {
  FALKON_LOSS_LOGISTIC = 0, /* l(z,y) = log(1 + exp(-y z)), y in {-1,+1} (Example 1(a)) */
  FALKON_LOSS_SQUARED = 1   /* l(z,y) = (z - y)^2 / 2: one step from 0 is exactly falkon_fit */
};

/* alpha = GSC-Falkon(X, y, C, y_C, loss, path)  (Alg. 2, DESIGN.md
   readings g1-g7).  Starting from alpha = 0, runs n_steps approximate Newton steps
   ("WeightedFalkon"); step k, at level mu[k] > 0 with iters[k] >= 0 CG iterations, solves
     (Knm^T D Knm + mu n (Kmm + delta I)) alpha_new = Knm^T (D z - g)
   preconditioned by T^-1 A^-1 with A^T A = (1/m) T D~ T^T + mu I, where z = Knm alpha,
   g_i = l'(z_i, y_i), D = diag(l''(z_i, y_i)) on the rows and D~ = diag(l''((Kmm alpha)_j,
   yC_j)) on the centres.  CG runs on the correction from the warm
   start beta_0 = A T alpha (reading g4; same iterates as CG from beta_0).
   X: n_local x d fp32 (row shard).  y: n_local fp32 labels (+-1 for the logistic loss).
   C: m x d fp32, yC: m fp32 labels of the centres (replicated).  mu, iters: n_steps HOST
   arrays: the explicit level path of Alg. 2 (reading g5), built by the caller (e.g.
   synth.GSC_CONFIGS); the library does none of the schedule.
   alpha: m fp64 (replicated).  T = chol(Kmm + delta I) is built once; A is rebuilt per step
   in the same m x m fp64 buffer.  info: phase times summed over steps, iters_run = total CG
   iterations.  Errors: as falkon_fit; EINVAL also for n_steps < 1, unknown loss, mu <= 0. */
int falkon_gsc_fit(falkon_ctx *ctx, const float *X, const float *y, int64_t n_local, int64_t d,
                   const float *C, const float *yC, int64_t m, int kernel, double sigma,
                   int loss, int32_t n_steps, const double *mu, const int32_t *iters,
                   double jitter, double *alpha, falkon_fit_info *info);

const char *falkon_strerror(int code);
/* Details of the last error on this thread (static storage, valid until the next call). */
const char *falkon_last_error(void);
/* Library build info string (arch, version). */
const char *falkon_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FALKON_H_ */
