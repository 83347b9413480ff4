// capi.cu — the extern "C" boundary of libfalkon (include/falkon.h) and the device-side
// Falkon driver: RHS, conjugate gradient with LinOp (Alg. 1; Eq. (9)
// PAPER.md:269), final alpha, prediction (Eq. (4)).
//
// Every step of the path runs in this library's kernels on the context stream.  The CG
// loop never synchronises with the host: scalars (rho, gamma) live in device memory, the
// breakdown tests of reading c9 are evaluated on the device, and the host reads the
// diagnostics once at the end of the fit.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "common.cuh"

using namespace falkon;

namespace falkon {
const char *last_error_cstr();

// ------------------------------------------------------------------ argument checks
static int check_common(falkon_ctx *ctx, int64_t n, int64_t d, int64_t m, int kernel,
                        double sigma) {
  if (!ctx) return fail(FALKON_EINVAL, "ctx is NULL");
  if (n < 0) return fail(FALKON_EINVAL, "n_local < 0");
  if (d < 1) return fail(FALKON_EINVAL, "d < 1");
  if (m < 1) return fail(FALKON_EINVAL, "m < 1");
  if (kernel != FALKON_GAUSSIAN && kernel != FALKON_LAPLACIAN)
    return fail(FALKON_EINVAL, "unknown kernel " + std::to_string(kernel));
  if (!(sigma > 0.0) || !std::isfinite(sigma)) return fail(FALKON_EINVAL, "sigma must be > 0 and finite");
  FK_CUDA(cudaSetDevice(ctx->device));
  return FALKON_OK;
}

// Device view of a caller array: device pointers pass through; host arrays are staged.
static int stage_in(falkon_ctx *ctx, int slot, const void *p, size_t bytes, const void **out) {
  if (bytes == 0 || is_device_ptr(p)) {
    *out = p;
    return FALKON_OK;
  }
  void *w;
  FK_TRY(ws_get(ctx, slot, bytes, &w));
  FK_CUDA(cudaMemcpyAsync(w, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
  *out = w;
  return FALKON_OK;
}

// ------------------------------------------------------------------ fp64 vector kernels
constexpr int VT = 256;
constexpr int DOT_BLOCKS = 256;

// deterministic two-stage dot product: partials[b] then out = sum_b partials[b] (fixed order)
__global__ void dot_partial_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                   int64_t n, double *__restrict__ part) {
  __shared__ double s[VT];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VT)
    acc = fma(a[i], b[i], acc);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = VT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}
__global__ void dot_final_kernel(const double *__restrict__ part, int nb, double *__restrict__ out) {
  __shared__ double s[DOT_BLOCKS];
  s[threadIdx.x] = threadIdx.x < nb ? part[threadIdx.x] : 0.0;
  __syncthreads();
  for (int o = DOT_BLOCKS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// CG scalar slots
enum { S_RHO = 0, S_RHO_NEW, S_GAMMA, S_STOP, S_ITERS, S_FAIL, S_NSLOTS };

__global__ void cg_init_kernel(double *sc) {
  // called after rho = r.r has been written to sc[S_RHO]
  sc[S_STOP] = (sc[S_RHO] == 0.0) ? 1.0 : 0.0;  // reading c9: r^T r == 0 -> no iteration
  sc[S_ITERS] = 0.0;
  sc[S_FAIL] = -1.0;
}

// x += a p ; r -= a q  with a = rho / gamma; breakdown -> stop + record iteration
__global__ void cg_xr_kernel(double *__restrict__ x, double *__restrict__ r,
                             const double *__restrict__ p, const double *__restrict__ q, int64_t m,
                             double *sc, int it) {
  const double stop = sc[S_STOP];
  if (stop != 0.0) return;
  const double gamma = sc[S_GAMMA], rho = sc[S_RHO];
  if (!(gamma > 0.0) || !isfinite(gamma)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[S_FAIL] = it;
    return;
  }
  const double a = rho / gamma;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(a, p[i], x[i]);
    r[i] = fma(-a, q[i], r[i]);
  }
}
// After rho_new = r.r: p = r + (rho_new/rho) p ; rho = rho_new ; handle stop/fail flags.
// Runs as a single-CTA kernel followed by the vector update, so the flags are consistent.
__global__ void cg_flags_kernel(double *sc, int it) {
  if (sc[S_STOP] != 0.0) return;
  if (sc[S_FAIL] >= 0.0) {
    sc[S_STOP] = 2.0;
    return;
  }
  const double rn = sc[S_RHO_NEW];
  if (!isfinite(rn)) {
    sc[S_FAIL] = it;
    sc[S_STOP] = 2.0;
    return;
  }
  sc[S_ITERS] = it;
  sc[S_GAMMA] = rn / sc[S_RHO];  // beta, stored in the gamma slot for cg_p_kernel
  sc[S_RHO] = rn;
  if (rn == 0.0) sc[S_STOP] = 3.0;  // exact convergence: x is final (reading c9)
}
__global__ void cg_p_kernel(double *__restrict__ p, const double *__restrict__ r, int64_t m,
                            const double *sc) {
  if (sc[S_STOP] == 2.0) return;
  if (sc[S_STOP] == 1.0) return;
  const double beta = sc[S_GAMMA];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], r[i]);
}
// y += s x
__global__ void axpy_kernel(double *__restrict__ y, const double *__restrict__ x, double s,
                            int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(s, x[i], y[i]);
}

static unsigned vgrid(int64_t m) { return (unsigned)std::min<int64_t>(cdiv<int64_t>(m, VT), 2048); }

static int dot(falkon_ctx *ctx, const double *a, const double *b, int64_t m, double *part,
               double *out) {
  const int nb = (int)std::min<int64_t>(DOT_BLOCKS, std::max<int64_t>(1, cdiv<int64_t>(m, VT)));
  LaunchScope ls(ctx, FALKON_T_VEC);
  dot_partial_kernel<<<nb, VT, 0, ctx->stream>>>(a, b, m, part);
  dot_final_kernel<<<1, DOT_BLOCKS, 0, ctx->stream>>>(part, nb, out);
  ctx->launches++;
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}


// ------------------------------------------------------------------ GSC losses (Alg. 2)
// (l', l'') of Def. 1 / Example 1 in fp64; logistic in a stable form:
// sigma(-s) = 1 / (1 + e^s) evaluated through e^{-|s|} (no overflow), s = y z.
__device__ __forceinline__ void loss_d12(int loss, double z, double y, double &d1, double &d2) {
  if (loss == FALKON_LOSS_LOGISTIC) {
    const double s = y * z;
    const double e = exp(-fabs(s));
    const double sn = s >= 0.0 ? e / (1.0 + e) : 1.0 / (1.0 + e);  // sigma(-s)
    d1 = -y * sn;
    d2 = sn * (1.0 - sn);
  } else {
    d1 = z - y;
    d2 = 1.0;
  }
}
// rows: g (-> w, pass B input: fp32, or fp64 under ACCUM_F64) and D (-> fp32 weights) at the
// predictions z (reading g1)
template <typename G>
__global__ void gsc_row_loss_kernel(const double *__restrict__ z, const float *__restrict__ y,
                                    int64_t n, int64_t n_pad, int loss, G *__restrict__ g,
                                    float *__restrict__ dw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d1 = 0.0, d2 = 0.0;
    if (i < n) loss_d12(loss, z ? z[i] : 0.0, (double)y[i], d1, d2);
    g[i] = (G)d1;
    dw[i] = (float)d2;
  }
}
// centres: D~_j = l''((Kmm alpha)_j, yC_j) with Kmm alpha = zt - delta alpha
__global__ void gsc_center_weight_kernel(const double *__restrict__ zt,
                                         const double *__restrict__ alpha, double delta,
                                         const float *__restrict__ yC, int64_t m, int loss,
                                         double *__restrict__ dm) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    double d1, d2;
    loss_d12(loss, zt[j] - delta * alpha[j], (double)yC[j], d1, d2);
    dm[j] = d2;
  }
}
// r = -(r + s zt): the preconditioned Newton residual at the warm start, -(Knm^T g + mu n K alpha)
__global__ void gsc_rhs_kernel(double *__restrict__ r, const double *__restrict__ zt, double s,
                               int64_t m) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    r[i] = -fma(s, zt[i], r[i]);
}

// ------------------------------------------------------------------ fit-time product path
// DESIGN.md reading d3: the tensor cores accumulate fp32 by truncation, so the folded-bias
// fp16x3 cross term carries a bias of ~ulp(|partial sums|)/2 toward zero; its scale is the
// magnitude of the biases a_p = -||x~_p||^2/2.  Measured (profiles/r2_fit_golden_*): on TAXI-
// shaped data (d 9, sigma 1: mean ||c~||^2/2 = 6.5) the fit's alpha error is 7x the SIMT
// path's (1.8e-3 vs 2.4e-4 at m = 2e4, n = 2e5), on HIGGS / MSD-shaped data (1.3-1.4) the
// tensor path is as accurate or better.  So a Gaussian FIT whose AUTO path would be the tensor
// kernel runs on the SIMT kernels when d <= 32 (the packed FP32 kernel) and the mean scaled
// centre norm exceeds FIT_BIAS_MAX; products outside fits keep the tensor path.
constexpr double FIT_BIAS_MAX = 4.0;
// reading d4: fits with d <= 32 and more centres than this run on FALKON_PATH_F64
constexpr int64_t FIT_F64_MIN_M = 25000;
struct FitPathScope {  // restores the context's path option at scope exit
  falkon_ctx *ctx;
  int saved;
  int chosen = FALKON_PATH_AUTO;
  explicit FitPathScope(falkon_ctx *c) : ctx(c), saved(c->opt.path) {}
  ~FitPathScope() { ctx->opt.path = saved; }
  int choose(const float *Cd, int64_t m, int64_t d, int kernel, double sigma) {
    if (ctx->opt.path == FALKON_PATH_F64) {
      chosen = FALKON_PATH_F64;
      return FALKON_OK;
    }
    chosen = tc_supported(ctx, kernel, d) ? FALKON_PATH_TENSOR : FALKON_PATH_SIMT;
    if (!ctx->opt.fit_precise || ctx->opt.path != FALKON_PATH_AUTO || d > 32) return FALKON_OK;
    // reading d4: small-d fits at large m need fp64 kernel values for the alpha bar (measured:
    // HIGGS-shaped n = 1.05M, m = 5e4: alpha 1.4e-3 on fp32-class kernels of either pipe)
    if (m > FIT_F64_MIN_M) {
      ctx->opt.path = FALKON_PATH_F64;
      chosen = FALKON_PATH_F64;
      return FALKON_OK;
    }
    if (chosen != FALKON_PATH_TENSOR) return FALKON_OK;
    double msq = 0.0;
    FK_TRY(center_spread(ctx, Cd, m, d, &msq));
    const double bias = 0.5 * msq * 1.4426950408889634 / (sigma * sigma);  // mean |b_j|
    if (bias > FIT_BIAS_MAX) {
      ctx->opt.path = FALKON_PATH_SIMT;
      chosen = FALKON_PATH_SIMT;
    }
    return FALKON_OK;
  }
};

// ------------------------------------------------------------------ product pieces
struct Fit {
  Prepared pp;
  float *v32 = nullptr;   // m_pad
  float *w32 = nullptr;   // n_pad
  double *v64 = nullptr;  // m_pad (ACCUM_F64)
  double *w64 = nullptr;  // n_pad (ACCUM_F64)
  bool f64 = false;       // FALKON_OPT_ACCUM_F64: fp64 v / w, DFMA contractions
};

static int64_t pad128(int64_t n) { return round_up<int64_t>(std::max<int64_t>(n, 1), 128); }

// v (fp64 m, device) -> the pass-A operand of the fit's precision
static int load_v(falkon_ctx *ctx, Fit &F, const double *v) {
  if (F.f64) return f64_pad(ctx, v, F.v64, F.pp.m, pad128(F.pp.m));
  return f64_to_f32(ctx, v, F.v32, F.pp.m, pad128(F.pp.m));
}
// pass A on the loaded v: w64 (external, optional) or the fit's own w buffer
static int pass_A_fit(falkon_ctx *ctx, Fit &F, double *w64) {
  if (F.f64) return pass_A64(ctx, F.pp, F.v64, w64 ? w64 : F.w64);
  return pass_A(ctx, F.pp, F.v32, w64, w64 ? nullptr : F.w32);
}
// pass B on the fit's w buffer
static int pass_B_fit(falkon_ctx *ctx, Fit &F, double *u) {
  if (F.f64) return pass_B64(ctx, F.pp, F.w64, u);
  return pass_B(ctx, F.pp, F.w32, u);
}
// the fit's w buffer from an fp32 (y, g) or fp64 (w) n-vector
static int load_w32(falkon_ctx *ctx, Fit &F, const float *w) {
  if (F.pp.n <= 0) return FALKON_OK;
  if (F.f64) return f32_to_f64_pad(ctx, w, F.w64, F.pp.n, pad128(F.pp.n));
  return f32_to_f32_pad(ctx, w, F.w32, F.pp.n, pad128(F.pp.n));
}
static int load_w64(falkon_ctx *ctx, Fit &F, const double *w) {
  if (F.pp.n <= 0) return FALKON_OK;
  if (F.f64) return f64_pad(ctx, w, F.w64, F.pp.n, pad128(F.pp.n));
  return f64_to_f32(ctx, w, F.w32, F.pp.n, pad128(F.pp.n));
}

// w[i] *= dw[i] for the rows, 0 in the padding (GSC LinOp: Knm^T D Knm, Alg. 2 line 6)
__global__ void scale_rows_kernel(float *__restrict__ w, const float *__restrict__ dw, int64_t n,
                                  int64_t n_pad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = i < n ? w[i] * dw[i] : 0.0f;
}

// u = sum_ranks Knm^T D Knm v  (D = I when dw == NULL: Alg. 1's product)
static int product(falkon_ctx *ctx, Fit &F, const double *v, double *u,
                   const float *dw = nullptr) {
  const int64_t m = F.pp.m;
  FK_TRY(load_v(ctx, F, v));
  if (F.pp.n > 0 && tc_single_eval(ctx, F.pp)) {  // NEXT-4: one evaluation per entry
    if (F.f64) FK_TRY(tc_product_single_eval64(ctx, F.pp, F.v64, F.w64, u, dw));
    else FK_TRY(tc_product_single_eval(ctx, F.pp, F.v32, F.w32, u, dw));
    return nccl_allreduce_f64(ctx, u, m);
  }
  FK_TRY(pass_A_fit(ctx, F, nullptr));
  if (dw) {
    const int64_t n_pad = pad128(F.pp.n);
    if (F.f64) {
      FK_TRY(f64_pad(ctx, F.w64, F.w64, F.pp.n, n_pad, dw));  // w_i * D_ii in fp64, in place
    } else {
      LaunchScope ls(ctx, FALKON_T_VEC);
      scale_rows_kernel<<<vgrid(n_pad), VT, 0, ctx->stream>>>(F.w32, dw, F.pp.n, n_pad);
    }
  }
  FK_TRY(pass_B_fit(ctx, F, u));
  return nccl_allreduce_f64(ctx, u, m);
}

// CG vectors and device scalars of one solve (Alg. 1 line 10)
struct CgState {
  double *x, *r, *p, *t1, *t2, *u, *sc, *dpart;
};

// Textbook CG from x = 0 on the preconditioned operator (reading c9), with r already set to
// the right-hand side:  LinOp(p) = A^-T ( T^-T Knm^T D Knm T^-1 A^-1 p + lam_n A^-1 p )
// (Eq. (9); Alg. 2 LinOp PAPER.md:979-985 with D = diag(dw), D = I if dw NULL).
// Never synchronises with the host: breakdown flags live in sc.
static int cg_run(falkon_ctx *ctx, Fit &F, const double *P, const double *dT, const double *dA,
                  const double *pw, int64_t m, double lam_n, int iters, const float *dw,
                  const CgState &S) {
  FK_CUDA(cudaMemsetAsync(S.x, 0, sizeof(double) * m, ctx->stream));
  FK_CUDA(cudaMemcpyAsync(S.p, S.r, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  FK_TRY(dot(ctx, S.r, S.r, m, S.dpart, S.sc + S_RHO));
  {
    LaunchScope ls(ctx, FALKON_T_VEC);
    cg_init_kernel<<<1, 1, 0, ctx->stream>>>(S.sc);
  }
  for (int it = 1; it <= iters; ++it) {
    FK_CUDA(cudaMemcpyAsync(S.t1, S.p, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
    FK_TRY(trsv(ctx, P, dA, pw, m, 1, 0, S.t1));  // t1 = A^-1 p
    FK_CUDA(cudaMemcpyAsync(S.t2, S.t1, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
    FK_TRY(trsv(ctx, P, dT, pw, m, 0, 0, S.t2));  // t2 = T^-1 t1
    FK_TRY(product(ctx, F, S.t2, S.u, dw));       // u = Knm^T D Knm t2 (allreduced)
    FK_TRY(trsv(ctx, P, dT, pw, m, 0, 1, S.u));   // u = T^-T u
    {
      LaunchScope ls(ctx, FALKON_T_VEC);
      axpy_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(S.u, S.t1, lam_n, m);
    }
    FK_TRY(trsv(ctx, P, dA, pw, m, 1, 1, S.u));   // q = A^-T u
    const double *qv = S.u;
    FK_TRY(dot(ctx, S.p, qv, m, S.dpart, S.sc + S_GAMMA));
    {
      LaunchScope ls(ctx, FALKON_T_VEC);
      cg_xr_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(S.x, S.r, S.p, qv, m, S.sc, it);
    }
    FK_TRY(dot(ctx, S.r, S.r, m, S.dpart, S.sc + S_RHO_NEW));
    {
      LaunchScope ls(ctx, FALKON_T_VEC);
      cg_flags_kernel<<<1, 1, 0, ctx->stream>>>(S.sc, it);
      cg_p_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(S.p, S.r, m, S.sc);
      ctx->launches++;
    }
    FK_LAUNCH_CHECK();
  }
  return FALKON_OK;
}


// ------------------------------------------------------------------ multi-output blocks (NEXT-3)
// pack columns [c0, c0 + kcols) of a strided matrix (element (i, c) at src[i rs + c cs]) into a
// zero-padded fp32 block [rows_pad][kvb]; unpack the fp64 block [rows][kvb] back.
template <typename S>
__global__ void pack_block_kernel(const S *__restrict__ src, int64_t rs, int64_t cs, int64_t rows,
                                  int64_t c0, int kcols, int kvb, float *__restrict__ dst,
                                  int64_t rows_pad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows_pad * kvb) return;
  const int64_t i = e / kvb;
  const int j = (int)(e % kvb);
  dst[e] = (i < rows && j < kcols) ? (float)src[i * rs + (c0 + j) * cs] : 0.f;
}
__global__ void unpack_block_kernel(const double *__restrict__ src, int64_t rows, int kvb,
                                    int kcols, int64_t c0, double *__restrict__ dst, int64_t rs,
                                    int64_t cs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * kcols) return;
  const int64_t i = e / kcols;
  const int j = (int)(e % kcols);
  dst[i * rs + (c0 + j) * cs] = src[i * kvb + j];
}

// column block width of a multi-vector pass: the tensor epilogue is compiled for 8 / 16 vectors
// (padded with zero columns); the SIMT path loops over exactly the columns given
static int block_kv(const Prepared &pp, int64_t left) {
  if (left == 1) return 1;
  if (pp.path == FALKON_PATH_TENSOR) return left > 8 ? 16 : 8;
  return (int)std::min<int64_t>(left, 16);
}

template <typename S>
static int pack_block(falkon_ctx *ctx, const S *src, int64_t rs, int64_t cs, int64_t rows,
                      int64_t c0, int kcols, int kvb, float *dst, int64_t rows_pad) {
  const int64_t tot = rows_pad * kvb;
  if (tot <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  pack_block_kernel<S><<<(unsigned)cdiv<int64_t>(tot, 256), 256, 0, ctx->stream>>>(
      src, rs, cs, rows, c0, kcols, kvb, dst, rows_pad);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}
static int unpack_block(falkon_ctx *ctx, const double *src, int64_t rows, int kvb, int kcols,
                        int64_t c0, double *dst, int64_t rs, int64_t cs) {
  const int64_t tot = rows * kcols;
  if (tot <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  unpack_block_kernel<<<(unsigned)cdiv<int64_t>(tot, 256), 256, 0, ctx->stream>>>(
      src, rows, kvb, kcols, c0, dst, rs, cs);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// U = Knm^T (Knm V) for k vectors on this rank (no collective): V element (j, c) at
// V[j vrs + c vcs], U element (j, c) written at U[j urs + c ucs].
static int product_multi(falkon_ctx *ctx, Fit &F, const double *V, int64_t vrs, int64_t vcs,
                         int64_t k, double *U, int64_t urs, int64_t ucs) {
  const int64_t m = F.pp.m, n = F.pp.n;
  const int64_t m_pad = round_up<int64_t>(m, 256), n_pad = round_up<int64_t>(std::max<int64_t>(n, 1), 256);
  void *v32, *w32, *u64;
  FK_TRY(ws_get(ctx, WS_MV32, sizeof(float) * m_pad * 16, &v32));
  FK_TRY(ws_get(ctx, WS_MW32, sizeof(float) * n_pad * 16, &w32));
  FK_TRY(ws_get(ctx, WS_MU64, sizeof(double) * m * 16, &u64));
  for (int64_t c0 = 0; c0 < k; ) {
    const int kvb = block_kv(F.pp, k - c0);
    const int kc = (int)std::min<int64_t>(kvb, k - c0);
    FK_TRY(pack_block<double>(ctx, V, vrs, vcs, m, c0, kc, kvb, (float *)v32, m_pad));
    FK_TRY(pass_A_multi(ctx, F.pp, (const float *)v32, kvb, nullptr, (float *)w32));
    FK_TRY(pass_B_multi(ctx, F.pp, (const float *)w32, kvb, (double *)u64));
    FK_TRY(unpack_block(ctx, (const double *)u64, m, kvb, kc, c0, U, urs, ucs));
    c0 += kc;
  }
  return FALKON_OK;
}

static int alloc_fit_vectors(falkon_ctx *ctx, Fit &F) {
  void *a, *b;
  FK_TRY(ws_get(ctx, WS_V32, sizeof(float) * pad128(F.pp.m), &a));
  FK_TRY(ws_get(ctx, WS_W32, sizeof(float) * pad128(F.pp.n), &b));
  F.v32 = (float *)a;
  F.w32 = (float *)b;
  F.f64 = ctx->opt.accum_f64 != 0 || F.pp.path == FALKON_PATH_F64;
  if (F.f64) {
    FK_TRY(ws_get(ctx, WS_V64, sizeof(double) * pad128(F.pp.m), &a));
    FK_TRY(ws_get(ctx, WS_W64, sizeof(double) * pad128(F.pp.n), &b));
    F.v64 = (double *)a;
    F.w64 = (double *)b;
  }
  return FALKON_OK;
}

}  // namespace falkon

#define BRK_CUDA(call)                                                              \
  {                                                                                 \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      rc = fail(FALKON_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
      break;                                                                        \
    }                                                                               \
  }

// ==================================================================== extern "C"
extern "C" {

const char *falkon_strerror(int code) {
  switch (code) {
    case FALKON_OK: return "ok";
    case FALKON_EINVAL: return "invalid argument";
    case FALKON_ENOTPD: return "matrix not positive definite (Cholesky pivot <= 0)";
    case FALKON_ENONFINITE: return "non-finite value or non-positive curvature in CG";
    case FALKON_ENOMEM: return "device out of memory";
    case FALKON_ECUDA: return "CUDA error";
    case FALKON_ENCCL: return "NCCL error";
    case FALKON_EUNSUPPORTED: return "unsupported device or feature";
    default: return "unknown error";
  }
}

const char *falkon_last_error(void) { return falkon::last_error_cstr(); }

const char *falkon_version(void) {
  return "libfalkon 0.1 (sm_100a; fused SIMT FP32/MUFU + tcgen05 kernel-matvec, fp64 preconditioner)";
}

int falkon_get_unique_id(unsigned char id[128]) {
  if (!id) return fail(FALKON_EINVAL, "id is NULL");
  return nccl_get_unique_id(id);
}

int falkon_ctx_create(falkon_ctx **out, int device, int rank, int world, const unsigned char *id) {
  if (!out) return fail(FALKON_EINVAL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(FALKON_EINVAL, "bad rank/world");
  if (world > 1 && id == nullptr) return fail(FALKON_EINVAL, "id is required when world > 1");
  int ndev = 0;
  FK_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(FALKON_EINVAL, "bad device ordinal");
  cudaDeviceProp prop;
  FK_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(FALKON_EUNSUPPORTED, std::string("libfalkon is built for sm_100a only; device is ") +
                                         prop.name + " sm_" + std::to_string(prop.major) +
                                         std::to_string(prop.minor));
  FK_CUDA(cudaSetDevice(device));
  falkon_ctx *c = new falkon_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->sm_count = prop.multiProcessorCount;
  c->cc_major = prop.major;
  c->cc_minor = prop.minor;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(FALKON_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  c->stream = c->own_stream;
  if (id != nullptr) {  // world == 1 with an id: a 1-rank NCCL communicator (tests the collective path)
    int r = nccl_comm_init(c, id);
    if (r != FALKON_OK) {
      cudaStreamDestroy(c->own_stream);
      delete c;
      return r;
    }
  }
  *out = c;
  return FALKON_OK;
}

int falkon_ctx_destroy(falkon_ctx *ctx) {
  if (!ctx) return FALKON_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  nccl_comm_destroy(ctx);
  for (int i = 0; i < WS_COUNT; ++i)
    if (ctx->ws[i]) cudaFree(ctx->ws[i]);
  for (auto &e : ctx->pending) {
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.stop);
  }
  for (auto &e : ctx->free_events) {
    cudaEventDestroy(e.start);
    cudaEventDestroy(e.stop);
  }
  if (ctx->hi_stream) cudaStreamDestroy(ctx->hi_stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->lo_stream) cudaStreamDestroy(ctx->lo_stream);
  if (ctx->se_stream) cudaStreamDestroy(ctx->se_stream);
  for (auto &e : ctx->se_ev)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return FALKON_OK;
}

int falkon_ctx_set_stream(falkon_ctx *ctx, void *stream) {
  if (!ctx) return fail(FALKON_EINVAL, "ctx is NULL");
  ctx->stream = (cudaStream_t)stream;  // NULL = the legacy default stream
  return FALKON_OK;
}

int falkon_ctx_set_option(falkon_ctx *ctx, int option, int64_t value) {
  if (!ctx) return fail(FALKON_EINVAL, "ctx is NULL");
  switch (option) {
    case FALKON_OPT_PATH:
      if (value < 0 || value > 3) return fail(FALKON_EINVAL, "bad path");
      ctx->opt.path = (int)value;
      return FALKON_OK;
    case FALKON_OPT_TC_MIN_D:
      if (value < 1) return fail(FALKON_EINVAL, "bad tc_min_d");
      ctx->opt.tc_min_d = (int)value;
      return FALKON_OK;
    case FALKON_OPT_TC_TERMS:  // only the fp32-accurate 3-term split is built (reading d1)
      if (value != 3)
        return fail(FALKON_EUNSUPPORTED, "tc_terms: only the 3-term fp16 split is implemented "
                                         "(1 and 2 terms fail the alpha bar, DESIGN.md reading d1)");
      return FALKON_OK;
    case FALKON_OPT_KERNEL_TIMING:
      ctx->opt.kernel_timing = value ? 1 : 0;
      return FALKON_OK;
    case FALKON_OPT_EXP_OFFLOAD:
      if (value < 0 || value > 3) return fail(FALKON_EINVAL, "exp offload mode must be 0..3");
      ctx->opt.exp_offload = (int)value;
      return FALKON_OK;
    case FALKON_OPT_GEMM_WARPS:
      if (value != 8 && value != 16 && value != 2 && value != 5)
        return fail(FALKON_EINVAL, "gemm variant must be 8, 16 (warps, 1 CTA/SM), 2 (2 CTAs/SM) "
                                   "or 5 (TMA-fed producer warp + 8 DMMA warps where A = B)");
      ctx->opt.gemm_warps = (int)value;
      return FALKON_OK;
    case FALKON_OPT_POTRF_OUTER:
      if (value < 0 || value > 64)
        return fail(FALKON_EINVAL, "potrf outer block must be 1..64 x 128 (0 = auto)");
      ctx->opt.potrf_outer = (int)value;
      return FALKON_OK;
    case FALKON_OPT_SINGLE_EVAL:
      if (value < 0 || value > 2) return fail(FALKON_EINVAL, "single_eval must be 0, 1 or 2");
      ctx->opt.single_eval = (int)value;
      return FALKON_OK;
    case FALKON_OPT_OZAKI:
      if (value < 0 || value > 1) return fail(FALKON_EINVAL, "ozaki must be 0 or 1");
      ctx->opt.ozaki = (int)value;
      return FALKON_OK;
    case FALKON_OPT_SE_GEMV_SMS:
      if (value < 0 || value >= ctx->sm_count)
        return fail(FALKON_EINVAL, "se_gemv_sms must be in [0, SM count)");
      ctx->opt.se_gemv_sms = (int)value;
      return FALKON_OK;
    case FALKON_OPT_STRIP_BYTES:
      if (value < ((int64_t)64 << 20)) return fail(FALKON_EINVAL, "strip bytes must be >= 64 MiB");
      ctx->opt.strip_bytes = value;
      return FALKON_OK;
    case FALKON_OPT_LOOKAHEAD:
      ctx->opt.lookahead = value ? 1 : 0;
      return FALKON_OK;
    case FALKON_OPT_ACCUM_F64:
      if (value != 0 && value != 1) return fail(FALKON_EINVAL, "accum_f64 must be 0 or 1");
      ctx->opt.accum_f64 = (int)value;
      return FALKON_OK;
    case FALKON_OPT_FIT_PRECISE:
      ctx->opt.fit_precise = value ? 1 : 0;
      return FALKON_OK;
    case FALKON_OPT_DIST_PRECOND:
      ctx->opt.dist_precond = value ? 1 : 0;
      return FALKON_OK;
    case FALKON_OPT_TC_CLUSTER:
      if (value != 1 && value != 2) return fail(FALKON_EINVAL, "tc_cluster must be 1 or 2");
      ctx->opt.tc_cluster = (int)value;
      return FALKON_OK;
    default:
      return fail(FALKON_EINVAL, "unknown option");
  }
}

int falkon_ctx_timings(falkon_ctx *ctx, double *out_ms, int64_t *launches, int reset) {
  if (!ctx) return fail(FALKON_EINVAL, "ctx is NULL");
  FK_TRY(resolve_timings(ctx));
  for (int i = 0; i < FALKON_T_COUNT; ++i) {
    if (out_ms) out_ms[i] = ctx->t_ms[i];
    if (launches) launches[i] = ctx->t_launches[i];
    if (reset) {
      ctx->t_ms[i] = 0.0;
      ctx->t_launches[i] = 0;
    }
  }
  return FALKON_OK;
}

int64_t falkon_ctx_launch_count(const falkon_ctx *ctx) { return ctx ? ctx->launches : -1; }

// ------------------------------------------------------------------ products
static int matvec_common(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C,
                         int64_t m, int kernel, double sigma, Fit &F) {
  const void *Xd, *Cd;
  FK_TRY(stage_in(ctx, WS_STAGE_X, X, sizeof(float) * n * d, &Xd));
  FK_TRY(stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd));
  FK_TRY(prepare_operands(ctx, (const float *)Xd, n, d, (const float *)Cd, m, kernel, sigma, &F.pp));
  return alloc_fit_vectors(ctx, F);
}

// Host X on the two-pass tensor path: the rows go up in chunks on a copy stream, and each
// chunk is packed and run through pass A as soon as it lands, so the H2D transfer overlaps the
// product (pass B needs every w, so it follows the last chunk).  Same packing and tiles as the
// staged path; a chunk's pass A may split the centres differently, so w can differ in the fp64
// order of the per-split partials (relative 1e-16 level).
static int matvec_host_pipelined(falkon_ctx *ctx, const float *X, int64_t n, int64_t d,
                                 const float *C, int64_t m, int kernel, double sigma, Fit &F,
                                 const double *vd, double *ud) {
  const void *Cd;
  FK_TRY(stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd));
  FK_TRY(prepare_operands(ctx, nullptr, n, d, (const float *)Cd, m, kernel, sigma, &F.pp));
  if (F.pp.path != FALKON_PATH_TENSOR) return FALKON_TC_RANGE;  // C out of fp16 range: staged path
  FK_TRY(alloc_fit_vectors(ctx, F));
  void *xs;
  FK_TRY(ws_get(ctx, WS_STAGE_X, sizeof(float) * n * d, &xs));
  if (!ctx->copy_stream)
    FK_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  FK_TRY(f64_to_f32(ctx, vd, F.v32, m, round_up<int64_t>(m, 128)));
  const int nchunk = 8;
  const int64_t rows = round_up<int64_t>(cdiv<int64_t>(n, nchunk), 128);
  cudaEvent_t ev[nchunk + 1];
  for (auto &e : ev) FK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  int rc = FALKON_OK;
  // the copies may only start once the staging buffer is free (prior work on ctx->stream)
  cudaEventRecord(ev[nchunk], ctx->stream);
  cudaStreamWaitEvent(ctx->copy_stream, ev[nchunk], 0);
  int c = 0;
  for (int64_t r0 = 0; r0 < n; r0 += rows, ++c) {
    const int64_t nr = std::min<int64_t>(rows, n - r0);
    float *dst = (float *)xs + r0 * d;
    if (cudaMemcpyAsync(dst, X + r0 * d, sizeof(float) * nr * d, cudaMemcpyHostToDevice,
                        ctx->copy_stream) != cudaSuccess) {
      rc = fail(FALKON_ECUDA, "cudaMemcpyAsync (host X chunk)");
      break;
    }
    cudaEventRecord(ev[c], ctx->copy_stream);
  }
  c = 0;
  for (int64_t r0 = 0; rc == FALKON_OK && r0 < n; r0 += rows, ++c) {
    const int64_t nr = std::min<int64_t>(rows, n - r0);
    cudaStreamWaitEvent(ctx->stream, ev[c], 0);
    if ((rc = tc_pack_rows(ctx, F.pp, (const float *)xs + r0 * d, r0, nr))) break;
    if ((rc = tc_pass_A_rows(ctx, F.pp, F.v32, F.w32, r0, nr))) break;
  }
  for (auto &e : ev) cudaEventDestroy(e);
  FK_TRY(rc);
  bool bad = false;  // fp16 range guard of the packed chunks
  FK_TRY(tc_range_check(ctx, &bad));
  if (bad) {  // re-prepare from the staged rows: the range guard routes them to the SIMT path
    FK_TRY(prepare_operands(ctx, (const float *)xs, n, d, (const float *)Cd, m, kernel, sigma, &F.pp));
    FK_TRY(alloc_fit_vectors(ctx, F));
    return product(ctx, F, vd, ud);
  }
  FK_TRY(pass_B(ctx, F.pp, F.w32, ud));
  return nccl_allreduce_f64(ctx, ud, m);
}

int falkon_knm_matvec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d, const float *C,
                      int64_t m, int kernel, double sigma, const double *v, double *u) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || !C || !v || !u) return fail(FALKON_EINVAL, "NULL array");
  Fit F;
  if (n_local >= 8 * 1024 && !is_device_ptr(X) && tc_supported(ctx, kernel, d) &&
      !ctx->opt.accum_f64) {
    Prepared probe;
    probe.path = FALKON_PATH_TENSOR;
    probe.d = d;
    if (!tc_single_eval(ctx, probe)) {
      const void *vd;
      FK_TRY(stage_in(ctx, WS_STAGE_V, v, sizeof(double) * m, &vd));
      const bool host_out = !is_device_ptr(u);
      double *ud = u;
      if (host_out) {
        void *w;
        FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * m, &w));
        ud = (double *)w;
      }
      const int prc = matvec_host_pipelined(ctx, X, n_local, d, C, m, kernel, sigma, F,
                                            (const double *)vd, ud);
      if (prc == FALKON_TC_RANGE) {  // centres out of fp16 range: the staged (SIMT) path
        F = Fit();
        FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
        FK_TRY(product(ctx, F, (const double *)vd, ud));
      } else {
        FK_TRY(prc);
      }
      if (host_out) {
        FK_CUDA(cudaMemcpyAsync(u, ud, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
        FK_CUDA(cudaStreamSynchronize(ctx->stream));
      }
      return FALKON_OK;
    }
  }
  FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
  const void *vd;
  FK_TRY(stage_in(ctx, WS_STAGE_V, v, sizeof(double) * m, &vd));
  const bool host_out = !is_device_ptr(u);
  double *ud = u;
  if (host_out) {
    void *w;
    FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * m, &w));
    ud = (double *)w;
  }
  FK_TRY(product(ctx, F, (const double *)vd, ud));
  if (host_out) {
    FK_CUDA(cudaMemcpyAsync(u, ud, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FALKON_OK;
}

int falkon_kernel_vec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d, const float *C,
                      int64_t m, int kernel, double sigma, const double *v, double *w) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || !C || !v || (!w && n_local > 0)) return fail(FALKON_EINVAL, "NULL array");
  if (n_local == 0) return FALKON_OK;
  Fit F;
  FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
  const void *vd;
  FK_TRY(stage_in(ctx, WS_STAGE_V, v, sizeof(double) * m, &vd));
  const bool host_out = !is_device_ptr(w);
  double *wd = w;
  if (host_out) {
    void *p;
    FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * n_local, &p));
    wd = (double *)p;
  }
  FK_TRY(load_v(ctx, F, (const double *)vd));
  FK_TRY(pass_A_fit(ctx, F, wd));
  if (host_out) {
    FK_CUDA(cudaMemcpyAsync(w, wd, sizeof(double) * n_local, cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FALKON_OK;
}

int falkon_kernel_tvec(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d, const float *C,
                       int64_t m, int kernel, double sigma, const double *w, double *u) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || !C || (!w && n_local > 0) || !u) return fail(FALKON_EINVAL, "NULL array");
  Fit F;
  FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
  const bool host_out = !is_device_ptr(u);
  double *ud = u;
  if (host_out) {
    void *p;
    FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * m, &p));
    ud = (double *)p;
  }
  if (n_local > 0) {
    const void *wd;
    FK_TRY(stage_in(ctx, WS_STAGE_V, w, sizeof(double) * n_local, &wd));
    FK_TRY(load_w64(ctx, F, (const double *)wd));
  }
  FK_TRY(pass_B_fit(ctx, F, ud));
  FK_TRY(nccl_allreduce_f64(ctx, ud, m));
  if (host_out) {
    FK_CUDA(cudaMemcpyAsync(u, ud, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FALKON_OK;
}

int falkon_predict(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d, const float *C,
                   int64_t m, int kernel, double sigma, const double *alpha, double *f) {
  return falkon_kernel_vec(ctx, X, n_local, d, C, m, kernel, sigma, alpha, f);
}

// ------------------------------------------------------------------ preconditioner API
int64_t falkon_precond_work_elems(int64_t m) { return m > 0 ? precond_work_elems(m) : 0; }

int falkon_precond_build(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                         double sigma, double lambda, double jitter, double *P, double *diagT,
                         double *diagA, double *work, falkon_fit_info *info) {
  FK_TRY(check_common(ctx, 0, d, m, kernel, sigma));
  if (!C || !P || !diagT || !diagA || !work) return fail(FALKON_EINVAL, "NULL array");
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(FALKON_EINVAL, "lambda must be >= 0");
  if (!is_device_ptr(P) || !is_device_ptr(diagT) || !is_device_ptr(diagA) || !is_device_ptr(work))
    return fail(FALKON_EINVAL, "P, diagT, diagA, work must be device memory");
  if (jitter < 0) jitter = 1e-8;
  const void *Cd;
  FK_TRY(stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd));
  return precond_build(ctx, (const float *)Cd, m, d, kernel, sigma, lambda, jitter, P, diagT, diagA,
                       work, info);
}

int falkon_precond_build_sim(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                             double sigma, double lambda, double jitter, int G, double *const *P,
                             double *const *diagT, double *const *diagA, double *const *work,
                             falkon_fit_info *info) {
  FK_TRY(check_common(ctx, 0, d, m, kernel, sigma));
  if (!C || !P || !diagT || !diagA || !work) return fail(FALKON_EINVAL, "NULL array");
  if (G < 1 || G > 64) return fail(FALKON_EINVAL, "G must be 1..64");
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(FALKON_EINVAL, "lambda must be >= 0");
  for (int r = 0; r < G; ++r)
    if (!P[r] || !diagT[r] || !diagA[r] || !work[r] || !is_device_ptr(P[r]) ||
        !is_device_ptr(diagT[r]) || !is_device_ptr(diagA[r]) || !is_device_ptr(work[r]))
      return fail(FALKON_EINVAL, "P, diagT, diagA, work of every rank must be device memory");
  if (jitter < 0) jitter = 1e-8;
  const void *Cd;
  FK_TRY(stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd));
  return precond_build_sim(ctx, (const float *)Cd, m, d, kernel, sigma, lambda, jitter, G, P, diagT,
                           diagA, work, info);
}

int falkon_precond_solve(falkon_ctx *ctx, const double *P, const double *diagT, const double *diagA,
                         const double *work, int64_t m, int which, int trans, double *x) {
  if (!ctx || !P || !diagT || !diagA || !work || !x || m < 1 || (which != 0 && which != 1))
    return fail(FALKON_EINVAL, "bad arguments");
  FK_CUDA(cudaSetDevice(ctx->device));
  return trsv(ctx, P, which == 0 ? diagT : diagA, work, m, which, trans, x);
}

int falkon_precond_solve_multi(falkon_ctx *ctx, const double *P, const double *diagT,
                               const double *diagA, const double *work, int64_t m, int which,
                               int trans, double *x, int64_t ldx, int64_t k) {
  if (!ctx || !P || !diagT || !diagA || !work || !x || m < 1 || k < 1 || ldx < m ||
      (which != 0 && which != 1))
    return fail(FALKON_EINVAL, "bad arguments");
  FK_CUDA(cudaSetDevice(ctx->device));
  return trsv_multi(ctx, P, which == 0 ? diagT : diagA, work, m, which, trans, x, ldx, k);
}

// ------------------------------------------------------------------ Falkon fit
int falkon_fit(falkon_ctx *ctx, const float *X, const float *y, int64_t n_local, int64_t d,
               const float *C, int64_t m, int kernel, double sigma, double lambda, int32_t iters,
               double jitter, double *alpha, falkon_fit_info *info) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || (!y && n_local > 0) || !C || !alpha) return fail(FALKON_EINVAL, "NULL array");
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(FALKON_EINVAL, "lambda must be >= 0");
  if (iters < 0) return fail(FALKON_EINVAL, "iters < 0");
  if (jitter < 0) jitter = 1e-8;
  falkon_fit_info loc;
  memset(&loc, 0, sizeof(loc));
  loc.failed_factor = -1;
  loc.failed_column = -1;
  loc.failed_iter = -1;
  loc.jitter_used = jitter;
  auto t_start = std::chrono::steady_clock::now();

  const bool host_out = !is_device_ptr(alpha);
  // global n (reading c15)
  int64_t n_global = n_local;
  if (ctx->nccl_comm) {
    void *p;
    FK_TRY(ws_get(ctx, WS_SCALARS, 64, &p));
    FK_CUDA(cudaMemcpyAsync(p, &n_global, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    FK_TRY(nccl_allreduce_i64(ctx, (int64_t *)p, 1));
    FK_CUDA(cudaMemcpyAsync(&n_global, p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }

  // CG vectors: x r p q t1 t2 u (+ alpha staging) and scalars
  void *cgv, *scal;
  FK_TRY(ws_get(ctx, WS_CG, sizeof(double) * m * 8, &cgv));
  FK_TRY(ws_get(ctx, WS_CG2, sizeof(double) * (S_NSLOTS + DOT_BLOCKS + 8), &scal));
  double *x = (double *)cgv, *r = x + m, *p = r + m, *q = p + m, *t1 = q + m, *t2 = t1 + m,
         *u = t2 + m, *ares = u + m;
  double *sc = (double *)scal, *dpart = sc + S_NSLOTS + 4;

  if (iters == 0) {
    FK_CUDA(cudaMemsetAsync(ares, 0, sizeof(double) * m, ctx->stream));
  }

  cudaEvent_t ev[4];
  for (auto &e : ev) FK_CUDA(cudaEventCreate(&e));
  FK_CUDA(cudaEventRecord(ev[0], ctx->stream));

  // (1) preconditioner: one m x m fp64 buffer for this fit
  double *P = nullptr, *dT = nullptr;
  int rc = FALKON_OK;
  if (iters > 0) {
    cudaError_t e = cudaMalloc(&P, sizeof(double) * (size_t)m * (size_t)m);
    if (e != cudaSuccess) {
      cudaGetLastError();
      for (auto &ee : ev) cudaEventDestroy(ee);
      return fail(FALKON_ENOMEM, "preconditioner buffer of " + std::to_string(8.0 * m * m / 1e9) +
                                     " GB: " + cudaGetErrorString(e));
    }
    e = cudaMalloc(&dT, sizeof(double) * (2 * (size_t)m + (size_t)precond_work_elems(m)));
    if (e != cudaSuccess) {
      cudaFree(P);
      for (auto &ee : ev) cudaEventDestroy(ee);
      return fail(FALKON_ENOMEM, "diag vectors");
    }
  }
  double *dA = dT ? dT + m : nullptr;
  double *pw = dT ? dT + 2 * m : nullptr;  // inverse 64x64 diagonal blocks of T^T and A^T
  auto cleanup = [&]() {
    if (P) cudaFree(P);
    if (dT) cudaFree(dT);
    for (auto &ee : ev) cudaEventDestroy(ee);
  };
  Fit F;
  FitPathScope fps(ctx);
  do {
    if (iters == 0) break;
    const void *Xd, *yd, *Cd;
    if ((rc = stage_in(ctx, WS_STAGE_X, X, sizeof(float) * n_local * d, &Xd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_Y, y, sizeof(float) * n_local, &yd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd))) break;
    if ((rc = precond_build(ctx, (const float *)Cd, m, d, kernel, sigma, lambda, jitter, P, dT, dA,
                            pw, &loc)))
      break;
    cudaEventRecord(ev[1], ctx->stream);
    if ((rc = fps.choose((const float *)Cd, m, d, kernel, sigma))) break;
    loc.product_path = fps.chosen;
    // (2) RHS  R = A^-T T^-T Knm^T y   (Alg. 1 line 9)
    if ((rc = prepare_operands(ctx, (const float *)Xd, n_local, d, (const float *)Cd, m, kernel,
                               sigma, &F.pp)))
      break;
    if ((rc = alloc_fit_vectors(ctx, F))) break;
    if ((rc = load_w32(ctx, F, (const float *)yd))) break;
    if ((rc = pass_B_fit(ctx, F, r))) break;
    if ((rc = nccl_allreduce_f64(ctx, r, m))) break;
    if ((rc = trsv(ctx, P, dT, pw, m, 0, 1, r))) break;  // T^-T
    if ((rc = trsv(ctx, P, dA, pw, m, 1, 1, r))) break;  // A^-T
    cudaEventRecord(ev[2], ctx->stream);
    // (3) CG  (Alg. 1 line 10; reading c9)
    CgState S{x, r, p, t1, t2, u, sc, dpart};
    if ((rc = cg_run(ctx, F, P, dT, dA, pw, m, lambda * (double)n_global, iters, nullptr, S)))
      break;
    if (rc) break;
    cudaEventRecord(ev[3], ctx->stream);
    // (4) alpha = T^-1 A^-1 x   (Alg. 1 line 11)
    BRK_CUDA(cudaMemcpyAsync(ares, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
    if ((rc = trsv(ctx, P, dA, pw, m, 1, 0, ares))) break;
    if ((rc = trsv(ctx, P, dT, pw, m, 0, 0, ares))) break;
  } while (0);
  if (rc != FALKON_OK) {
    if (info) *info = loc;
    cudaStreamSynchronize(ctx->stream);
    cleanup();
    return rc;
  }
  if (host_out)
    FK_CUDA(cudaMemcpyAsync(alpha, ares, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
  else
    FK_CUDA(cudaMemcpyAsync(alpha, ares, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  double hs[S_NSLOTS] = {};
  if (iters > 0)
    FK_CUDA(cudaMemcpyAsync(hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  auto t_end = std::chrono::steady_clock::now();
  loc.t_total_s = std::chrono::duration<double>(t_end - t_start).count();
  if (iters > 0) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    loc.t_precond_s = a * 1e-3;
    loc.t_rhs_s = b * 1e-3;
    loc.t_cg_s = c * 1e-3;
    loc.iters_run = (int32_t)hs[S_ITERS];
    loc.failed_iter = (int32_t)hs[S_FAIL];
  }
  cleanup();
  if (info) *info = loc;
  if (loc.failed_iter >= 0)
    return fail(FALKON_ENONFINITE, "CG breakdown at iteration " + std::to_string(loc.failed_iter));
  return FALKON_OK;
}


// ------------------------------------------------------------------ GSC-Falkon (Alg. 2)
int falkon_gsc_fit(falkon_ctx *ctx, const float *X, const float *y, int64_t n_local, int64_t d,
                   const float *C, const float *yC, int64_t m, int kernel, double sigma,
                   int loss, int32_t n_steps, const double *mu, const int32_t *iters,
                   double jitter, double *alpha, falkon_fit_info *info) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || (!y && n_local > 0) || !C || !yC || !alpha || !mu || !iters)
    return fail(FALKON_EINVAL, "NULL array");
  if (loss != FALKON_LOSS_LOGISTIC && loss != FALKON_LOSS_SQUARED)
    return fail(FALKON_EINVAL, "unknown loss " + std::to_string(loss));
  if (n_steps < 1) return fail(FALKON_EINVAL, "n_steps < 1");
  for (int k = 0; k < n_steps; ++k) {
    if (!(mu[k] > 0.0) || !std::isfinite(mu[k])) return fail(FALKON_EINVAL, "mu[k] must be > 0");
    if (iters[k] < 0) return fail(FALKON_EINVAL, "iters[k] < 0");
  }
  if (jitter < 0) jitter = 1e-8;
  falkon_fit_info loc;
  memset(&loc, 0, sizeof(loc));
  loc.failed_factor = -1;
  loc.failed_column = -1;
  loc.failed_iter = -1;
  loc.jitter_used = jitter;
  auto t_start = std::chrono::steady_clock::now();
  int64_t n_global = n_local;
  if (ctx->nccl_comm) {
    void *p;
    FK_TRY(ws_get(ctx, WS_SCALARS, 64, &p));
    FK_CUDA(cudaMemcpyAsync(p, &n_global, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    FK_TRY(nccl_allreduce_i64(ctx, (int64_t *)p, 1));
    FK_CUDA(cudaMemcpyAsync(&n_global, p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  void *cgv, *scal, *gv;
  FK_TRY(ws_get(ctx, WS_CG, sizeof(double) * m * 8, &cgv));
  FK_TRY(ws_get(ctx, WS_CG2, sizeof(double) * (S_NSLOTS + DOT_BLOCKS + 8), &scal));
  FK_TRY(ws_get(ctx, WS_GSC, sizeof(double) * m * 4, &gv));
  double *x = (double *)cgv, *r = x + m, *p = r + m, *t1 = p + m, *t2 = t1 + m, *u = t2 + m;
  double *sc = (double *)scal, *dpart = sc + S_NSLOTS + 4;
  double *acur = (double *)gv, *zt = acur + m, *tmp = zt + m, *dm = tmp + m;

  double *P = nullptr, *dT = nullptr;
  {
    cudaError_t e = cudaMalloc(&P, sizeof(double) * (size_t)m * (size_t)m);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FALKON_ENOMEM, "preconditioner buffer of " + std::to_string(8.0 * m * m / 1e9) +
                                     " GB: " + cudaGetErrorString(e));
    }
    e = cudaMalloc(&dT, sizeof(double) * (2 * (size_t)m + (size_t)precond_work_elems(m)));
    if (e != cudaSuccess) {
      cudaFree(P);
      cudaGetLastError();
      return fail(FALKON_ENOMEM, "diag vectors");
    }
  }
  double *dA = dT + m, *pw = dT + 2 * m;
  cudaEvent_t ev[4];
  for (auto &e : ev) cudaEventCreate(&e);
  auto cleanup = [&]() {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(P);
    cudaFree(dT);
    for (auto &e : ev) cudaEventDestroy(e);
  };
  int rc = FALKON_OK;
  Fit F;
  FitPathScope fps(ctx);
  do {
    const void *Xd, *yd, *Cd, *yCd;
    if ((rc = stage_in(ctx, WS_STAGE_X, X, sizeof(float) * n_local * d, &Xd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_Y, y, sizeof(float) * n_local, &yd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_V, yC, sizeof(float) * m, &yCd))) break;
    if ((rc = fps.choose((const float *)Cd, m, d, kernel, sigma))) break;
    loc.product_path = fps.chosen;
    if ((rc = prepare_operands(ctx, (const float *)Xd, n_local, d, (const float *)Cd, m, kernel,
                               sigma, &F.pp)))
      break;
    if ((rc = alloc_fit_vectors(ctx, F))) break;
    const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n_local, 1), 128);
    void *dwp, *zp;
    if ((rc = ws_get(ctx, WS_DW, sizeof(float) * n_pad, &dwp))) break;
    if ((rc = ws_get(ctx, WS_Z64, sizeof(double) * std::max<int64_t>(n_local, 1), &zp))) break;
    float *dw = (float *)dwp;
    double *z = (double *)zp;
    // T = chol(Kmm + delta I) once: Kmm does not depend on the Newton iterate (Alg. 2 WP l.1-3)
    BRK_CUDA(cudaEventRecord(ev[0], ctx->stream));
    if ((rc = precond_build_T(ctx, (const float *)Cd, m, d, kernel, sigma, jitter, P, dT, pw, &loc)))
      break;
    BRK_CUDA(cudaEventRecord(ev[1], ctx->stream));
    BRK_CUDA(cudaStreamSynchronize(ctx->stream));
    {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      loc.t_precond_s += ms * 1e-3;
    }
    BRK_CUDA(cudaMemsetAsync(acur, 0, sizeof(double) * m, ctx->stream));
    for (int k = 0; k < n_steps && rc == FALKON_OK; ++k) {
      const double muk = mu[k];
      BRK_CUDA(cudaEventRecord(ev[0], ctx->stream));
      // WeightedPreconditioner at the current alpha:
      // zt = (Kmm + delta I) alpha = T^T T alpha;  D~ = l''(Kmm alpha, yC);  A = chol(T D~ T^T/m + mu I)
      if (k == 0) {
        BRK_CUDA(cudaMemsetAsync(zt, 0, sizeof(double) * m, ctx->stream));
      } else if ((rc = trmv_TtT(ctx, P, dT, m, acur, tmp, zt))) {
        break;
      }
      {
        LaunchScope ls(ctx, FALKON_T_VEC);
        gsc_center_weight_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(zt, acur, jitter,
                                                                     (const float *)yCd, m, loss, dm);
      }
      BRK_CUDA(cudaGetLastError());
      if ((rc = precond_build_A(ctx, m, muk, dm, P, dT, dA, pw, jitter, &loc))) break;
      BRK_CUDA(cudaEventRecord(ev[1], ctx->stream));
      // rows: z = Knm alpha, g = l'(z, y), D = l''(z, y)   (readings g1, g2)
      {
        const double *zz = nullptr;
        if (k > 0 && n_local > 0) {
          if ((rc = load_v(ctx, F, acur))) break;
          if ((rc = pass_A_fit(ctx, F, z))) break;
          zz = z;
        }
        LaunchScope ls(ctx, FALKON_T_VEC);
        if (F.f64)
          gsc_row_loss_kernel<double><<<vgrid(n_pad), VT, 0, ctx->stream>>>(
              zz, (const float *)yd, n_local, n_pad, loss, F.w64, dw);
        else
          gsc_row_loss_kernel<float><<<vgrid(n_pad), VT, 0, ctx->stream>>>(
              zz, (const float *)yd, n_local, n_pad, loss, F.w32, dw);
      }
      BRK_CUDA(cudaGetLastError());
      // residual at the warm start beta_0 = A T alpha (reading g4):
      //   R - LinOp(beta_0) = -A^-T T^-T (Knm^T g + mu n (Kmm + delta I) alpha)
      if ((rc = pass_B_fit(ctx, F, r))) break;
      if ((rc = nccl_allreduce_f64(ctx, r, m))) break;
      {
        LaunchScope ls(ctx, FALKON_T_VEC);
        gsc_rhs_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(r, zt, muk * (double)n_global, m);
      }
      BRK_CUDA(cudaGetLastError());
      if ((rc = trsv(ctx, P, dT, pw, m, 0, 1, r))) break;  // T^-T
      if ((rc = trsv(ctx, P, dA, pw, m, 1, 1, r))) break;  // A^-T
      BRK_CUDA(cudaEventRecord(ev[2], ctx->stream));
      // CG on the correction (Alg. 2 line 10), LinOp with D on the rows
      CgState S{x, r, p, t1, t2, u, sc, dpart};
      if (iters[k] > 0) {
        if ((rc = cg_run(ctx, F, P, dT, dA, pw, m, muk * (double)n_global, iters[k], dw, S))) break;
        // alpha += T^-1 A^-1 x  (Alg. 2 line 11 applied to beta_0 + x)
        BRK_CUDA(cudaMemcpyAsync(t1, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
        if ((rc = trsv(ctx, P, dA, pw, m, 1, 0, t1))) break;
        if ((rc = trsv(ctx, P, dT, pw, m, 0, 0, t1))) break;
        LaunchScope ls(ctx, FALKON_T_VEC);
        axpy_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(acur, t1, 1.0, m);
      }
      BRK_CUDA(cudaGetLastError());
      BRK_CUDA(cudaEventRecord(ev[3], ctx->stream));
      double hs[S_NSLOTS] = {};
      if (iters[k] > 0)
        BRK_CUDA(cudaMemcpyAsync(hs, sc, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
      BRK_CUDA(cudaStreamSynchronize(ctx->stream));
      float a = 0, b = 0, c = 0;
      cudaEventElapsedTime(&a, ev[0], ev[1]);
      cudaEventElapsedTime(&b, ev[1], ev[2]);
      cudaEventElapsedTime(&c, ev[2], ev[3]);
      loc.t_precond_s += a * 1e-3;
      loc.t_rhs_s += b * 1e-3;
      loc.t_cg_s += c * 1e-3;
      if (iters[k] > 0) {
        loc.iters_run += (int32_t)hs[S_ITERS];
        if (hs[S_FAIL] >= 0) {
          loc.failed_iter = (int32_t)hs[S_FAIL];
          rc = fail(FALKON_ENONFINITE, "CG breakdown at iteration " + std::to_string(loc.failed_iter) +
                                           " of Newton step " + std::to_string(k));
        }
      }
    }
    if (rc) break;
    BRK_CUDA(cudaMemcpyAsync(alpha, acur, sizeof(double) * m,
                             is_device_ptr(alpha) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             ctx->stream));
    BRK_CUDA(cudaStreamSynchronize(ctx->stream));
  } while (0);
  cleanup();
  loc.t_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  if (info) *info = loc;
  return rc;
}


// ------------------------------------------------------------------ multi-output (NEXT-3)
int falkon_knm_matmat(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d, const float *C,
                      int64_t m, int kernel, double sigma, const double *V, int64_t k, double *U) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || !C || !V || !U) return fail(FALKON_EINVAL, "NULL array");
  if (k < 1) return fail(FALKON_EINVAL, "k < 1");
  Fit F;
  FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
  const void *Vd;
  FK_TRY(stage_in(ctx, WS_STAGE_V, V, sizeof(double) * m * k, &Vd));
  const bool host_out = !is_device_ptr(U);
  double *Ud = U;
  if (host_out) {
    void *w;
    FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * m * k, &w));
    Ud = (double *)w;
  }
  FK_TRY(product_multi(ctx, F, (const double *)Vd, k, 1, k, Ud, k, 1));
  FK_TRY(nccl_allreduce_f64(ctx, Ud, m * k));
  if (host_out) {
    FK_CUDA(cudaMemcpyAsync(U, Ud, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FALKON_OK;
}

int falkon_predict_multi(falkon_ctx *ctx, const float *X, int64_t n_local, int64_t d,
                         const float *C, int64_t m, int kernel, double sigma, const double *alpha,
                         int64_t k, double *Fo) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || !C || !alpha || (!Fo && n_local > 0)) return fail(FALKON_EINVAL, "NULL array");
  if (k < 1) return fail(FALKON_EINVAL, "k < 1");
  if (n_local == 0) return FALKON_OK;
  Fit F;
  FK_TRY(matvec_common(ctx, X, n_local, d, C, m, kernel, sigma, F));
  const void *Ad;
  FK_TRY(stage_in(ctx, WS_STAGE_V, alpha, sizeof(double) * m * k, &Ad));
  const bool host_out = !is_device_ptr(Fo);
  double *Fd = Fo;
  if (host_out) {
    void *w;
    FK_TRY(ws_get(ctx, WS_STAGE_OUT, sizeof(double) * n_local * k, &w));
    Fd = (double *)w;
  }
  const int64_t m_pad = round_up<int64_t>(m, 256);
  void *v32, *f64b;
  FK_TRY(ws_get(ctx, WS_MV32, sizeof(float) * m_pad * 16, &v32));
  FK_TRY(ws_get(ctx, WS_Z64, sizeof(double) * n_local * 16, &f64b));
  for (int64_t c0 = 0; c0 < k;) {
    const int kvb = block_kv(F.pp, k - c0);
    const int kc = (int)std::min<int64_t>(kvb, k - c0);
    FK_TRY(pack_block<double>(ctx, (const double *)Ad, k, 1, m, c0, kc, kvb, (float *)v32, m_pad));
    FK_TRY(pass_A_multi(ctx, F.pp, (const float *)v32, kvb, (double *)f64b, nullptr));
    FK_TRY(unpack_block(ctx, (const double *)f64b, n_local, kvb, kc, c0, Fd, k, 1));
    c0 += kc;
  }
  if (host_out) {
    FK_CUDA(cudaMemcpyAsync(Fo, Fd, sizeof(double) * n_local * k, cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FALKON_OK;
}

// Multi-output Falkon: Alg. 1 for k right-hand sides at once (the k CGs are independent; they
// share the preconditioner and every kernel product).  CG state is column-major [k][m].
int falkon_fit_multi(falkon_ctx *ctx, const float *X, const float *Y, int64_t n_local, int64_t d,
                     const float *C, int64_t m, int64_t k, int kernel, double sigma, double lambda,
                     int32_t iters, double jitter, double *alpha, falkon_fit_info *info) {
  FK_TRY(check_common(ctx, n_local, d, m, kernel, sigma));
  if ((!X && n_local > 0) || (!Y && n_local > 0) || !C || !alpha) return fail(FALKON_EINVAL, "NULL array");
  if (k < 1) return fail(FALKON_EINVAL, "k < 1");
  if (!(lambda >= 0.0) || !std::isfinite(lambda)) return fail(FALKON_EINVAL, "lambda must be >= 0");
  if (iters < 0) return fail(FALKON_EINVAL, "iters < 0");
  if (jitter < 0) jitter = 1e-8;
  falkon_fit_info loc;
  memset(&loc, 0, sizeof(loc));
  loc.failed_factor = -1;
  loc.failed_column = -1;
  loc.failed_iter = -1;
  loc.jitter_used = jitter;
  auto t_start = std::chrono::steady_clock::now();
  int64_t n_global = n_local;
  if (ctx->nccl_comm) {
    void *p;
    FK_TRY(ws_get(ctx, WS_SCALARS, 64, &p));
    FK_CUDA(cudaMemcpyAsync(p, &n_global, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    FK_TRY(nccl_allreduce_i64(ctx, (int64_t *)p, 1));
    FK_CUDA(cudaMemcpyAsync(&n_global, p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    FK_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  const bool host_out = !is_device_ptr(alpha);
  void *st, *scal;
  FK_TRY(ws_get(ctx, WS_MULTI, sizeof(double) * m * k * 7, &st));
  const size_t nsl = S_NSLOTS + DOT_BLOCKS + 8;
  FK_TRY(ws_get(ctx, WS_CG2, sizeof(double) * nsl * k, &scal));
  double *x = (double *)st, *r = x + m * k, *p = r + m * k, *t1 = p + m * k, *t2 = t1 + m * k,
         *u = t2 + m * k, *ares = u + m * k;
  double *P = nullptr, *dT = nullptr;
  if (iters > 0) {
    cudaError_t e = cudaMalloc(&P, sizeof(double) * (size_t)m * (size_t)m);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FALKON_ENOMEM, "preconditioner buffer of " + std::to_string(8.0 * m * m / 1e9) + " GB");
    }
    e = cudaMalloc(&dT, sizeof(double) * (2 * (size_t)m + (size_t)precond_work_elems(m)));
    if (e != cudaSuccess) {
      cudaFree(P);
      cudaGetLastError();
      return fail(FALKON_ENOMEM, "diag vectors");
    }
  }
  double *dA = dT ? dT + m : nullptr, *pw = dT ? dT + 2 * m : nullptr;
  cudaEvent_t ev[4];
  for (auto &e : ev) cudaEventCreate(&e);
  int rc = FALKON_OK;
  Fit F;
  do {
    if (iters == 0) {
      BRK_CUDA(cudaMemsetAsync(ares, 0, sizeof(double) * m * k, ctx->stream));
      break;
    }
    const void *Xd, *Yd, *Cd;
    if ((rc = stage_in(ctx, WS_STAGE_X, X, sizeof(float) * n_local * d, &Xd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_Y, Y, sizeof(float) * n_local * k, &Yd))) break;
    if ((rc = stage_in(ctx, WS_STAGE_C, C, sizeof(float) * m * d, &Cd))) break;
    BRK_CUDA(cudaEventRecord(ev[0], ctx->stream));
    if ((rc = precond_build(ctx, (const float *)Cd, m, d, kernel, sigma, lambda, jitter, P, dT, dA,
                            pw, &loc)))
      break;
    BRK_CUDA(cudaEventRecord(ev[1], ctx->stream));
    if ((rc = prepare_operands(ctx, (const float *)Xd, n_local, d, (const float *)Cd, m, kernel,
                               sigma, &F.pp)))
      break;
    // RHS  R = A^-T T^-T Knm^T Y  (Alg. 1 line 9, k columns)
    {
      const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n_local, 1), 256);
      void *w32, *u64;
      if ((rc = ws_get(ctx, WS_MW32, sizeof(float) * n_pad * 16, &w32))) break;
      if ((rc = ws_get(ctx, WS_MU64, sizeof(double) * m * 16, &u64))) break;
      for (int64_t c0 = 0; c0 < k && rc == FALKON_OK;) {
        const int kvb = block_kv(F.pp, k - c0);
        const int kc = (int)std::min<int64_t>(kvb, k - c0);
        if ((rc = pack_block<float>(ctx, (const float *)Yd, k, 1, n_local, c0, kc, kvb,
                                    (float *)w32, n_pad)))
          break;
        if ((rc = pass_B_multi(ctx, F.pp, (const float *)w32, kvb, (double *)u64))) break;
        rc = unpack_block(ctx, (const double *)u64, m, kvb, kc, c0, r, 1, m);
        c0 += kc;
      }
      if (rc) break;
    }
    if ((rc = nccl_allreduce_f64(ctx, r, m * k))) break;
    if ((rc = trsv_multi(ctx, P, dT, pw, m, 0, 1, r, m, k))) break;
    if ((rc = trsv_multi(ctx, P, dA, pw, m, 1, 1, r, m, k))) break;
    BRK_CUDA(cudaEventRecord(ev[2], ctx->stream));
    // k independent CGs (reading c9 per column) sharing each block product
    BRK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * m * k, ctx->stream));
    BRK_CUDA(cudaMemcpyAsync(p, r, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, ctx->stream));
    double *scb = (double *)scal;
    for (int64_t c = 0; c < k && rc == FALKON_OK; ++c) {
      double *sc = scb + c * nsl;
      if ((rc = dot(ctx, r + c * m, r + c * m, m, sc + S_NSLOTS + 4, sc + S_RHO))) break;
      LaunchScope ls(ctx, FALKON_T_VEC);
      cg_init_kernel<<<1, 1, 0, ctx->stream>>>(sc);
    }
    const double lam_n = lambda * (double)n_global;
    for (int it = 1; it <= iters && rc == FALKON_OK; ++it) {
      BRK_CUDA(cudaMemcpyAsync(t1, p, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, ctx->stream));
      if ((rc = trsv_multi(ctx, P, dA, pw, m, 1, 0, t1, m, k))) break;  // t1 = A^-1 p
      BRK_CUDA(cudaMemcpyAsync(t2, t1, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, ctx->stream));
      if ((rc = trsv_multi(ctx, P, dT, pw, m, 0, 0, t2, m, k))) break;  // t2 = T^-1 t1
      if ((rc = product_multi(ctx, F, t2, 1, m, k, u, 1, m))) break;  // u = Knm^T Knm t2
      if ((rc = nccl_allreduce_f64(ctx, u, m * k))) break;
      if ((rc = trsv_multi(ctx, P, dT, pw, m, 0, 1, u, m, k))) break;  // u = T^-T u
      {
        LaunchScope ls(ctx, FALKON_T_VEC);
        axpy_kernel<<<vgrid(m * k), VT, 0, ctx->stream>>>(u, t1, lam_n, m * k);
      }
      if ((rc = trsv_multi(ctx, P, dA, pw, m, 1, 1, u, m, k))) break;  // q = A^-T u
      for (int64_t c = 0; c < k && rc == FALKON_OK; ++c) {
        double *uc = u + c * m, *sc = scb + c * nsl;
        if ((rc = dot(ctx, p + c * m, uc, m, sc + S_NSLOTS + 4, sc + S_GAMMA))) break;
        {
          LaunchScope ls(ctx, FALKON_T_VEC);
          cg_xr_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(x + c * m, r + c * m, p + c * m, uc, m, sc, it);
        }
        if ((rc = dot(ctx, r + c * m, r + c * m, m, sc + S_NSLOTS + 4, sc + S_RHO_NEW))) break;
        LaunchScope ls(ctx, FALKON_T_VEC);
        cg_flags_kernel<<<1, 1, 0, ctx->stream>>>(sc, it);
        cg_p_kernel<<<vgrid(m), VT, 0, ctx->stream>>>(p + c * m, r + c * m, m, sc);
        ctx->launches++;
      }
      BRK_CUDA(cudaGetLastError());
    }
    if (rc) break;
    BRK_CUDA(cudaEventRecord(ev[3], ctx->stream));
    // alpha_c = T^-1 A^-1 x_c  (Alg. 1 line 11)
    BRK_CUDA(cudaMemcpyAsync(ares, x, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, ctx->stream));
    if ((rc = trsv_multi(ctx, P, dA, pw, m, 1, 0, ares, m, k))) break;
    rc = trsv_multi(ctx, P, dT, pw, m, 0, 0, ares, m, k);
  } while (0);
  if (rc == FALKON_OK) {
    // column-major [k][m] -> caller's row-major m x k
    double *outd = alpha;
    void *stg = nullptr;
    if (host_out) {
      rc = ws_get(ctx, WS_STAGE_OUT, sizeof(double) * m * k, &stg);
      outd = (double *)stg;
    }
    if (rc == FALKON_OK) {
      LaunchScope ls(ctx, FALKON_T_VEC);
      unpack_block_kernel<<<(unsigned)cdiv<int64_t>(m * k, 256), 256, 0, ctx->stream>>>(
          ares, k, (int)m, (int)m, 0, outd, 1, k);  // src [k][m] as rows=k, cols=m
    }
    if (rc == FALKON_OK && host_out)
      cudaMemcpyAsync(alpha, outd, sizeof(double) * m * k, cudaMemcpyDeviceToHost, ctx->stream);
  }
  double hsum = 0;
  int32_t fail_it = -1;
  if (rc == FALKON_OK && iters > 0) {
    std::vector<double> hs(nsl * k);
    cudaMemcpyAsync(hs.data(), scal, sizeof(double) * nsl * k, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    for (int64_t c = 0; c < k; ++c) {
      hsum += hs[c * nsl + S_ITERS];
      if (hs[c * nsl + S_FAIL] >= 0 && fail_it < 0) fail_it = (int32_t)hs[c * nsl + S_FAIL];
    }
    float a = 0, b = 0, cc = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&cc, ev[2], ev[3]);
    loc.t_precond_s = a * 1e-3;
    loc.t_rhs_s = b * 1e-3;
    loc.t_cg_s = cc * 1e-3;
    loc.iters_run = (int32_t)(hsum / (double)k);  // mean over columns
    loc.failed_iter = fail_it;
  }
  cudaStreamSynchronize(ctx->stream);
  if (P) cudaFree(P);
  if (dT) cudaFree(dT);
  for (auto &e : ev) cudaEventDestroy(e);
  loc.t_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  if (info) *info = loc;
  if (rc == FALKON_OK && fail_it >= 0)
    return fail(FALKON_ENONFINITE, "CG breakdown at iteration " + std::to_string(fail_it));
  return rc;
}

}  // extern "C"
