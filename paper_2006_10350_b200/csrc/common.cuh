// common.cuh — internal definitions of libfalkon (context, workspace, errors, PTX helpers).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "falkon.h"

namespace falkon {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define FK_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return ::falkon::fail(e_ == cudaErrorMemoryAllocation ? FALKON_ENOMEM : FALKON_ECUDA, \
                            std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

#define FK_TRY(call)                 \
  do {                               \
    int r_ = (call);                 \
    if (r_ != FALKON_OK) return r_;  \
  } while (0)

#define FK_LAUNCH_CHECK() FK_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ context
enum WsSlot {
  WS_CMEAN = 0,   // fp64 d: centering shift mu (mean of C)
  WS_CMEAN_PART,  // fp64 partial column sums
  WS_CP,          // packed centers (fp32 SIMT layout or fp16 split layout)
  WS_CB,          // fp32 m: center biases b_j
  WS_XP,          // packed rows
  WS_XA,          // fp32 n: row biases a_i
  WS_V32,         // fp32 m: v rounded
  WS_W32,         // fp32 n: w rounded (pass B input)
  WS_W64,         // fp64 n: w
  WS_PART,        // fp64 partials
  WS_U64,         // fp64 m scratch
  WS_STAGE_X,     // staging of host inputs
  WS_STAGE_C,
  WS_STAGE_V,
  WS_STAGE_OUT,
  WS_STAGE_Y,
  WS_CG,          // fp64 CG vectors
  WS_FLAGS,       // int flags / counters
  WS_SCALARS,     // fp64 scalars (dots)
  WS_TMAP,        // TMA descriptors (device copies)
  WS_PW,          // fp64 NB x NB inverse of the current diagonal block
  WS_CG2,         // fp64 CG scalars
  WS_TRMV,        // fp64 partials of the transposed triangular mat-vec
  WS_DW,          // fp32 n: per-row curvature weights D (GSC LinOp, Alg. 2)
  WS_Z64,         // fp64 n: predictions z = Knm alpha on the rows (GSC)
  WS_GSC,         // fp64 m vectors of the GSC outer loop
  WS_TRSV,        // fp64 m: sentinel-initialised output of the triangular solve
  WS_MCOL,        // fp32 column scratch of the SIMT multi-vector passes
  WS_MCOL64,      // fp64 + fp32 column outputs of the SIMT multi-vector passes
  WS_MV32,        // fp32 [m_pad][kv] packed vector block (multi-output)
  WS_MW32,        // fp32 [n_pad][kv] pass-A output block (multi-output)
  WS_MU64,        // fp64 [m][kv] pass-B output block (multi-output)
  WS_MULTI,       // fp64 multi-output fit state
  WS_KSTRIP,      // fp32 k strip of the single-evaluation product [rows][ldk]
  WS_SE_ACC,      // fp64 [splits][m] accumulators of the strip GEMV
  WS_V64,         // fp64 m_pad: v zero-padded (ACCUM_F64 pass-A input)
  WS_DIST_STAGE,  // fp64 m x NBO: packed A panel of the distributed preconditioner (NEXT-1)
  WS_SIM_FLAGS,   // pivot-failure words of the simulated ranks (precond_build_sim)
  WS_OZ0,         // int8 slices + row exponents of the Ozaki GEMM (base / high-priority stream)
  WS_OZ1,         // the same for the low-priority stream of the Cholesky lookahead
  WS_COUNT
};

struct TimedEvent {
  cudaEvent_t start, stop;
  int cls;
};

struct Options {
  int path = FALKON_PATH_AUTO;
  int tc_min_d = 4;   // measured SIMT/tensor crossover (profiles/r2_crossover.jsonl)
  int tc_terms = 3;
  int kernel_timing = 0;
  int exp_offload = 0;  // tensor path: share of exp2 evaluated on the FMA pipe (0..3)
  int gemm_warps = 5;   // fp64 GEMM variant: 5 = TMA-fed producer warp + 8 DMMA warps where
                        // A and B are the same view (trailing updates, LAUUM; measured m = 5e4
                        // 4.45 s, bitwise-identical factors), else 2; 2 = 128 x 64 tiles,
                        // 2 CTAs/SM (4.76 s); 8 = 128 x 128 tiles, 1 CTA/SM (4.96 s); 16 warps
  int potrf_outer = 0;  // outer POTRF block in units of NB = 128 (trailing-update depth);
                        // 0 = auto: 16 with the Ozaki GEMMs (m = 5e4: 8 -> 3.00 s, 16 -> 2.88 s,
                        // 32 -> 3.01 s), 8 with DMMA (2 -> 5.46 s, 4 -> 5.21 s, 8 -> 5.10 s)
  int lookahead = 1;    // blocked Cholesky: overlap the next panel with the trailing update
  int single_eval = 2;  // 0 two-pass, 1 single evaluation (k strip through HBM), 2 auto
  int tc_cluster = 2;   // tensor path: clusters of 2 CTAs multicasting the Q boxes (measured
                        // MSD 21.7 -> 20.9 ms, TIMIT 431 -> 424 ms), or 1 CTA
  int64_t strip_bytes = (int64_t)16 << 30;
  int accum_f64 = 0;    // FALKON_OPT_ACCUM_F64: fp64 v / w with DFMA contractions
  int dist_precond = 0; // FALKON_OPT_DIST_PRECOND: distributed build even on a 1-rank communicator
  int se_gemv_sms = 0;  // FALKON_OPT_SE_GEMV_SMS: split-SM single evaluation (0 = serial)
  int ozaki = 1;        // FALKON_OPT_OZAKI: big preconditioner GEMMs on the int8 tensor cores (ozaki.cu;
                        // measured m = 5e4: build 4.10 -> 3.06 s, factors 1e-13 from the DMMA build)
  int fit_precise = 1;  // FALKON_OPT_FIT_PRECISE: fits on small-d, large-norm data take the SIMT path
};

}  // namespace falkon

struct falkon_ctx {
  int device = 0, rank = 0, world = 1;
  int sm_count = 148;
  int cc_major = 10, cc_minor = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  void *nccl_comm = nullptr;
  void *ws[falkon::WS_COUNT] = {};
  size_t ws_bytes[falkon::WS_COUNT] = {};
  falkon::Options opt;
  // timing
  std::vector<falkon::TimedEvent> pending;
  std::vector<falkon::TimedEvent> free_events;
  double t_ms[FALKON_T_COUNT] = {};
  int64_t t_launches[FALKON_T_COUNT] = {};
  int64_t launches = 0;
  // blocked Cholesky lookahead (precond.cu): high-priority stream for the panel chain, low
  // priority for the bulk trailing update; created on first use
  cudaStream_t hi_stream = nullptr, lo_stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host-X pipeline of falkon_knm_matvec
  // split-SM single evaluation (kvp_tc.cu): highest-priority stream of the strip GEMV and the
  // events ordering pass A (strip buffer b written) / GEMV (buffer b read); created on first use
  cudaStream_t se_stream = nullptr;
  cudaEvent_t se_ev[4] = {};
  // co-resident CTAs of cluster launches, per kernel (kvp_tc.cu tc_cluster_slots)
  static constexpr int NSLOTCACHE = 8;
  const void *slot_fn[NSLOTCACHE] = {};
  int64_t slot_n[NSLOTCACHE] = {};
};

namespace falkon {

// effective outer POTRF block (FALKON_OPT_POTRF_OUTER, 0 = auto)
inline int potrf_outer(const falkon_ctx *ctx) {
  return ctx->opt.potrf_outer > 0 ? ctx->opt.potrf_outer : (ctx->opt.ozaki ? 16 : 8);
}

// Grow-only workspace slot (contents undefined after growth).  Sizes are rounded up to
// 256 B and a 256 B tail is always available so vector/bulk loads may overrun slightly.
int ws_get(falkon_ctx *ctx, int slot, size_t bytes, void **out);

// Launch accounting + optional CUDA-event timing around a launch.
struct LaunchScope {
  falkon_ctx *ctx;
  int cls;
  TimedEvent ev{};
  bool timed = false;
  LaunchScope(falkon_ctx *c, int cls_);
  ~LaunchScope();
};

int resolve_timings(falkon_ctx *ctx);

// pointer kind
bool is_device_ptr(const void *p);

// NCCL (dlopen'ed)
int nccl_get_unique_id(unsigned char id[128]);
int nccl_comm_init(falkon_ctx *ctx, const unsigned char *id);
int nccl_comm_destroy(falkon_ctx *ctx);
int nccl_allreduce_f64(falkon_ctx *ctx, double *buf, int64_t count);
int nccl_allreduce_i64(falkon_ctx *ctx, int64_t *buf, int64_t count);
int nccl_allreduce_min_u64(falkon_ctx *ctx, unsigned long long *buf, int64_t count);
int nccl_broadcast_bytes(falkon_ctx *ctx, void *buf, size_t bytes, int root);

// ------------------------------------------------------------------ product path (kvp.cu)
struct Prepared {
  // packed operands of one product call (owned by ctx workspace)
  int64_t n = 0, m = 0, d = 0;
  int kernel = 0;
  int path = FALKON_PATH_SIMT;
  int dq = 0;          // packed row stride (elements)
  const void *Xp = nullptr;
  const float *xa = nullptr;
  const void *Cp = nullptr;
  const float *cb = nullptr;
  const double *mu = nullptr;  // tensor path: centring shift (device, d)
  double g = 0.0;              // tensor path: coordinate scale sqrt(log2 e) / sigma
  // CUtensorMap x6 (tensor path): X as P, C as Q, C as P, X as Q, and the 192-row Q maps of
  // the opt-in TS kernel (C, X)
  alignas(64) unsigned char tmaps[6 * 128];
};

// X == nullptr (tensor path only): the packed-X buffer and maps are set up for n rows but no
// row is packed yet (tc_pack_rows fills row ranges, e.g. while later rows are still in flight)
int prepare_operands(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C,
                     int64_t m, int kernel, double sigma, Prepared *pp);
// w = Knm z  (pass A).  z: fp32 m (device).  w64 (n, optional) and/or w32 (n, optional).
int pass_A(falkon_ctx *ctx, const Prepared &pp, const float *z, double *w64, float *w32);
// u = Knm^T w (pass B) on this rank (no collective).  w: fp32 n (padded).  u: fp64 m.
int pass_B(falkon_ctx *ctx, const Prepared &pp, const float *w, double *u);
int f64_to_f32(falkon_ctx *ctx, const double *src, float *dst, int64_t n, int64_t n_pad);
// mean over the centres of ||c_j - mean(C)||^2 (host result; synchronises the stream)
int center_spread(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, double *mean_sq);
// FALKON_OPT_ACCUM_F64 passes: z fp64 (zero-padded to a multiple of 128), contraction by DFMA of
// the exact fp32 kernel value, fp64 output (w64: n, u: m).
int pass_A64(falkon_ctx *ctx, const Prepared &pp, const double *z, double *w64);
int pass_B64(falkon_ctx *ctx, const Prepared &pp, const double *w, double *u);
// dst[0..n) = src (times scale[i] if scale), dst[n..n_pad) = 0
int f64_pad(falkon_ctx *ctx, const double *src, double *dst, int64_t n, int64_t n_pad,
            const float *scale = nullptr);
int f32_to_f64_pad(falkon_ctx *ctx, const float *src, double *dst, int64_t n, int64_t n_pad);
// multi-vector passes: z [q][kv] fp32 (q = m for pass A, n_pad rows for pass B), outputs
// [p][kv] (fp64 and/or fp32); kv = 1, 8 or 16
int pass_A_multi(falkon_ctx *ctx, const Prepared &pp, const float *z, int kv, double *w64,
                 float *w32);
int pass_B_multi(falkon_ctx *ctx, const Prepared &pp, const float *w, int kv, double *u);
int f32_to_f32_pad(falkon_ctx *ctx, const float *src, float *dst, int64_t n, int64_t n_pad);

// tensor path (kvp_tc.cu)
bool tc_supported(const falkon_ctx *ctx, int kernel, int64_t d);
// returns FALKON_TC_RANGE (internal) when a packed coordinate or bias is out of fp16 range
int tc_prepare(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C, int64_t m,
               double sigma, const double *mu, Prepared *pp);
constexpr int FALKON_TC_RANGE = 1000;  // internal: tensor-path operands out of fp16 range
// device flag of the fp16 range guard (reset: zero it on the stream); check: read + sync
int tc_range_flag(falkon_ctx *ctx, int **flag, bool reset);
int tc_range_check(falkon_ctx *ctx, bool *bad);
// kv > 1 (8 or 16): z is [q][kv] fp32 and the outputs [p][kv] (multi-vector product)
int tc_pass(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z, double *out64,
            float *out32, int kv = 1);
// fp64 z / DFMA contraction variant (FALKON_OPT_ACCUM_F64), single vector
int tc_pass64(falkon_ctx *ctx, const Prepared &pp, bool passA, const double *z, double *out64);
// tensor path, rows [r0, r0 + nr): pack them from Xrows (nr x d fp32, device), and pass A over
// them alone (w32 + r0 receives their w).  Used by the host-X pipeline of falkon_knm_matvec.
int tc_pack_rows(falkon_ctx *ctx, const Prepared &pp, const float *Xrows, int64_t r0, int64_t nr);
int tc_pass_A_rows(falkon_ctx *ctx, const Prepared &pp, const float *z, float *w32, int64_t r0,
                   int64_t nr);
// single evaluation: true when single-vector products use the k strip
bool tc_single_eval(const falkon_ctx *ctx, const Prepared &pp);
// u = Knm^T (Knm z) on this rank with every kernel value evaluated once: per strip of rows,
// pass A stores the strip's k values (fp32, row-major) while computing w, then a streaming
// GEMV reads them back for u += strip^T w.  w32: fp32 n_pad output (w of every row).
int tc_product_single_eval(falkon_ctx *ctx, const Prepared &pp, const float *z, float *w32,
                           double *u, const float *dw = nullptr);
// the same with fp64 z / w and DFMA contractions (FALKON_OPT_ACCUM_F64); w64: fp64 n_pad
int tc_product_single_eval64(falkon_ctx *ctx, const Prepared &pp, const double *z, double *w64,
                             double *u, const float *dw = nullptr);

// ------------------------------------------------------------------ preconditioner (precond.cu)
int precond_build(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel, double sigma,
                  double lambda, double jitter, double *P, double *diagT, double *diagA,
                  double *work, falkon_fit_info *info);
int64_t precond_work_elems(int64_t m);
// Split build for GSC-Falkon (Alg. 2): T once (Kmm does not change along the Newton path),
// then A per step from M = T diag(dscale) T^T / m + lambda I (dscale NULL: D = I).
int precond_build_T(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                    double sigma, double jitter, double *P, double *diagT, double *work,
                    falkon_fit_info *info);
int precond_build_A(falkon_ctx *ctx, int64_t m, double lambda, const double *dscale, double *P,
                    double *diagT, double *diagA, double *work, double jitter,
                    falkon_fit_info *info);
// NEXT-1 test entry: the distributed (1D block-cyclic) build with G ranks simulated in this
// process, rank r's buffers P[r], diagT[r], diagA[r], work[r] (device memory)
int precond_build_sim(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                      double sigma, double lambda, double jitter, int G, double *const *P,
                      double *const *diagT, double *const *diagA, double *const *work,
                      falkon_fit_info *info);
// z = T^T (T x) = (Kmm + delta I) x from the factored buffer; tmp: m doubles
int trmv_TtT(falkon_ctx *ctx, const double *P, const double *diagT, int64_t m, const double *x,
             double *tmp, double *z);
// multi-column solve: columns x + c ldx, c < kcols (one pass over the triangle per 16 columns)
int trsv_multi(falkon_ctx *ctx, const double *P, const double *diag, const double *work, int64_t m,
               int which, int trans, double *x, int64_t ldx, int64_t kcols);
// x <- op(F)^-1 x, F = T (which 0) or A (which 1); work = the build's work buffer
int trsv(falkon_ctx *ctx, const double *P, const double *diag, const double *work, int64_t m,
         int which, int trans, double *x);

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fp32 k >= 0 (an ex2.approx.ftz result: +0 or a normal number) -> the same value in fp64,
// by re-biasing the exponent with integer ops (ACCUM_F64 contractions: the DFMA operand is the
// exact fp32 kernel value; this keeps the conversion off the F2F unit).  +0 maps to 2^-127
// (absolute error < 6e-39, far below the fp32 rounding of k itself).
__device__ __forceinline__ double k_to_f64(float k) {
  const uint32_t b = __float_as_uint(k);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
__host__ __device__ constexpr T cdiv(T a, T b) {
  return (a + b - 1) / b;
}
template <typename T>
__host__ __device__ constexpr T round_up(T a, T b) {
  return cdiv(a, b) * b;
}

}  // namespace falkon
