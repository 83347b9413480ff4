// kvp.cu — fused kernel-vector products on the FP32 FMA + MUFU pipes (small d) and the
// operand preparation shared by both product paths.
//
// The product u = Knm^T (Knm v) is evaluated block-wise without storing Knm
// (PAPER.md:271-275).  Both passes are instances of ONE fused primitive
//
//     out[p] = sum_{q in Q} k(P_p, Q_q) z_q          ("kvp": kernel-vector product)
//
//   pass A (a2-a4):  P = rows of X, Q = centers C, z = v   -> w = Knm v
//   pass B (a2,a3,a5): P = centers C, Q = rows of X, z = w  -> u = Knm^T w
//
// A CTA owns 128*R points of P and keeps their coordinates in registers; Q is streamed
// through shared memory in tiles of TQ points by the TMA engine (1-D cp.async.bulk into a
// 2-stage mbarrier ring).  Per (p, q) the cross term, the exp2 (MUFU) and the contraction
// are fused in registers; the contraction over q is an in-thread reduction (no atomics).
// fp32 partial sums are flushed into fp64 once per tile (<= TQ terms).
// When P alone cannot fill the GPU the Q range is split across CTAs (blockIdx.y) and the
// fp64 partials are reduced in a fixed order (deterministic, bitwise-reproducible).
//
// Gaussian, norm expansion with centred, pre-scaled inputs:
//     x~ = (x - mu) * sqrt(log2 e)/sigma,  a_i = -||x~_i||^2/2,  b_j = -||c~_j||^2/2
//     k(x_i, c_j) = exp2( min(a_i + b_j + x~_i . c~_j, 0) )        (clamp: reading c8)
// Laplacian (reading c7), direct differences (never the expansion):
//     x^ = (x - mu) * log2 e / sigma,   k = exp2( -sqrt(sum_k (x^_k - c^_k)^2) )
#include <math.h>

#include <algorithm>

#include "common.cuh"

namespace falkon {

constexpr int KVP_THREADS = 128;
constexpr int KVP_TQ = 128;             // streamed Q points per tile (small-d kernel)
constexpr int KVP_TQ_G = 32;            // streamed Q points per tile (generic kernel)
constexpr double LOG2E = 1.4426950408889634;

// ------------------------------------------------------------------ centring shift mu = mean(C)
// Gaussian and Laplacian kernels are translation invariant; centring shrinks the norms
// and thus the cancellation of the norm expansion.
__global__ void colsum_partial_kernel(const float *__restrict__ C, int64_t m, int64_t d,
                                      int64_t rows_per_block, double *__restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(m, r0 + rows_per_block);
  for (int64_t k = threadIdx.x; k < d; k += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += (double)C[r * d + k];
    part[(int64_t)blockIdx.x * d + k] = s;
  }
}

__global__ void colsum_final_kernel(const double *__restrict__ part, int nblk, int64_t d,
                                    int64_t m, double *__restrict__ mu) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * d + k];
  mu[k] = s / (double)m;
}

int center_mean(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, double **mu_out) {
  const int64_t rpb = 64;
  const int nblk = (int)cdiv<int64_t>(m, rpb);
  void *part, *mu;
  FK_TRY(ws_get(ctx, WS_CMEAN_PART, sizeof(double) * nblk * d, &part));
  FK_TRY(ws_get(ctx, WS_CMEAN, sizeof(double) * d, &mu));
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    colsum_partial_kernel<<<nblk, 128, 0, ctx->stream>>>(C, m, d, rpb, (double *)part);
  }
  FK_LAUNCH_CHECK();
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    colsum_final_kernel<<<(unsigned)cdiv<int64_t>(d, 128), 128, 0, ctx->stream>>>(
        (const double *)part, nblk, d, m, (double *)mu);
  }
  FK_LAUNCH_CHECK();
  *mu_out = (double *)mu;
  return FALKON_OK;
}

// mean over the centres of ||c_j - mu||^2 (one CTA, fixed order: identical on every rank)
__global__ void center_spread_kernel(const float *__restrict__ C, int64_t m, int64_t d,
                                     const double *__restrict__ mu, double *__restrict__ out) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    double r = 0.0;
    for (int64_t k = 0; k < d; ++k) {
      const double x = (double)C[j * d + k] - mu[k];
      r += x * x;
    }
    acc += r;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0] / (double)m;
}

int center_spread(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, double *mean_sq) {
  double *mu;
  FK_TRY(center_mean(ctx, C, m, d, &mu));
  void *p;
  FK_TRY(ws_get(ctx, WS_SCALARS, 64, &p));
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    center_spread_kernel<<<1, 256, 0, ctx->stream>>>(C, m, d, mu, (double *)p);
  }
  FK_LAUNCH_CHECK();
  FK_CUDA(cudaMemcpyAsync(mean_sq, p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  return FALKON_OK;
}

// ------------------------------------------------------------------ packing (SIMT layout)
// One warp per row: out[r, k] = (in[r, k] - mu[k]) * g  (k < d), 0 for d <= k < dq;
// bias[r] = -0.5 * ||out[r, :]||^2 computed in fp64 from the ROUNDED fp32 coordinates, so
// that a_i + b_j + x~.c~ = -||x~ - c~||^2 / 2 holds for the coordinates actually used.
__global__ void pack_rows_kernel(const float *__restrict__ in, int64_t rows, int64_t d,
                                 const double *__restrict__ mu, double g, int dq,
                                 float *__restrict__ out, float *__restrict__ bias) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double s = 0.0;
    for (int k = lane; k < dq; k += 32) {
      float v = 0.f;
      if (k < d) v = (float)(((double)in[r * d + k] - mu[k]) * g);
      out[r * dq + k] = v;
      s += (double)v * (double)v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && bias) bias[r] = (float)(-0.5 * s);
  }
}

// ------------------------------------------------------------------ fused kvp, d <= 32, packed FP32x2
// Tile-transposed layout "TT": points are grouped in tiles of 128; a tile stores coordinate k
// of its 128 points contiguously ([k][128]), so (a) a Q tile is one contiguous bulk copy,
// (b) one LDS.128 yields coordinate k of 4 consecutive Q points and (c) the P-side register
// load is coalesced.  Each thread owns R P points with coordinates duplicated into float2
// pairs and evaluates 2 Q points per packed FFMA2 (fma.rn.f32x2): the FP32 pipe, not the
// issue slot, becomes the limit.  Laplacian tiles store NEGATED coordinates so the direct
// difference x - c is one packed add.
template <int D>
__device__ __forceinline__ int64_t tt_idx(int64_t p, int k) {
  return (p >> 7) * (int64_t)(128 * D) + (int64_t)k * 128 + (p & 127);
}

__global__ void pack_rows_tt_kernel(const float *__restrict__ in, int64_t rows, int64_t rows_pad,
                                    int d, int dpad, const double *__restrict__ mu, double g,
                                    int negate, float *__restrict__ out,
                                    float *__restrict__ bias) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_pad) return;
  const int64_t base = (r >> 7) * (int64_t)(128 * dpad) + (r & 127);
  double s = 0.0;
  for (int k = 0; k < dpad; ++k) {
    float v = 0.f;
    if (r < rows && k < d) v = (float)(((double)in[r * d + k] - mu[k]) * g);
    s += (double)v * (double)v;
    out[base + (int64_t)k * 128] = negate ? -v : v;
  }
  if (bias) bias[r] = r < rows ? (float)(-0.5 * s) : 0.f;
}

// ZD (FALKON_OPT_ACCUM_F64): z is fp64 and each exact product k * z is accumulated by DFMA
// in fp64 (no fp32 rounding of z, of the products or of the partial sums).
template <int KER, int D, int R, bool ZD = false>
__global__ void __launch_bounds__(KVP_THREADS)
    kvp_pk_kernel(const float *__restrict__ P, const float *__restrict__ pa, int64_t np,
                  const float *__restrict__ Q, const float *__restrict__ qb,
                  const void *__restrict__ zv, int64_t nq, int64_t q_per_split,
                  double *__restrict__ out64, float *__restrict__ out32) {
  constexpr int QF = KVP_TQ * D;  // floats of one Q tile
  constexpr int ZW = ZD ? 2 : 1;  // z element width in floats
  extern __shared__ __align__(128) float smem_f[];
  float *const SB = smem_f + 2 * QF;
  float *const SZ = SB + 2 * KVP_TQ;
  uint64_t *bar = reinterpret_cast<uint64_t *>(SZ + 2 * KVP_TQ * ZW);
  const char *z = reinterpret_cast<const char *>(zv);

  const int tid = threadIdx.x;
  const int64_t qlo = (int64_t)blockIdx.y * q_per_split;
  const int64_t qhi = lmin(nq, qlo + q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, KVP_TQ) : 0;
  auto issue = [&](int t) {
    const int64_t q0 = qlo + (int64_t)t * KVP_TQ;  // multiple of 128: one whole TT tile
    const int s = t & 1;
    const uint32_t bq = (uint32_t)QF * 4, bs = (uint32_t)KVP_TQ * 4, bz = bs * ZW;
    mbar_expect_tx(&bar[s], bq + (KER == FALKON_GAUSSIAN ? bs : 0) + bz);
    bulk_g2s(smem_f + s * QF, Q + (q0 >> 7) * (int64_t)QF, bq, &bar[s]);
    if (KER == FALKON_GAUSSIAN) bulk_g2s(SB + s * KVP_TQ, qb + q0, bs, &bar[s]);
    bulk_g2s(SZ + s * KVP_TQ * ZW, z + q0 * 4 * ZW, bz, &bar[s]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (ntiles > 0) issue(0);
    if (ntiles > 1) issue(1);
  }
  // owned points -> registers, duplicated pairs (x, x)
  float2 xd[R][D];
  float2 ad[R];
  const int64_t pbase = (int64_t)blockIdx.x * (KVP_THREADS * R) + tid;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t p = lmin(pbase + (int64_t)r * KVP_THREADS, np - 1);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float v = P[tt_idx<D>(p, k)];
      if (KER == FALKON_LAPLACIAN) v = -v;  // stored negated
      xd[r][k] = make_float2(v, v);
    }
    const float a = (KER == FALKON_GAUSSIAN) ? pa[p] : 0.f;
    ad[r] = make_float2(a, a);
  }
  double acc64[R];
  double accd[R][2];  // ZD: two fp64 DFMA chains per owned point
#pragma unroll
  for (int r = 0; r < R; ++r) acc64[r] = accd[r][0] = accd[r][1] = 0.0;

  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bar[s], (t >> 1) & 1);
    const int cnt = (int)lmin(KVP_TQ, qhi - (qlo + (int64_t)t * KVP_TQ));
    const float *q = smem_f + s * QF;
    const float4 *b4p = reinterpret_cast<const float4 *>(SB + s * KVP_TQ);
    const float4 *z4p = reinterpret_cast<const float4 *>(SZ + s * KVP_TQ);
    const double2 *z2p = reinterpret_cast<const double2 *>(SZ + s * KVP_TQ * ZW);
    float2 acc[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r][0] = acc[r][1] = make_float2(0.f, 0.f);
    for (int j4 = 0; j4 < cnt; j4 += 4) {
      float4 zz;
      double2 zd0, zd1;
      if (ZD) {
        zd0 = z2p[j4 >> 1];
        zd1 = z2p[(j4 >> 1) + 1];
        if (j4 + 4 > cnt) {
          if (j4 + 1 >= cnt) zd0.y = 0.0;
          if (j4 + 2 >= cnt) zd1.x = 0.0;
          if (j4 + 3 >= cnt) zd1.y = 0.0;
        }
      } else {
        zz = z4p[j4 >> 2];
        if (j4 + 4 > cnt) {  // ragged tail of the last tile
          if (j4 + 1 >= cnt) zz.y = 0.f;
          if (j4 + 2 >= cnt) zz.z = 0.f;
          if (j4 + 3 >= cnt) zz.w = 0.f;
        }
      }
      float2 e[R][2];
      if (KER == FALKON_GAUSSIAN) {
        const float4 bb = b4p[j4 >> 2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          e[r][0] = __fadd2_rn(ad[r], make_float2(bb.x, bb.y));
          e[r][1] = __fadd2_rn(ad[r], make_float2(bb.z, bb.w));
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4 q4 = *reinterpret_cast<const float4 *>(q + k * KVP_TQ + j4);
          const float2 qa = make_float2(q4.x, q4.y), qb2 = make_float2(q4.z, q4.w);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            e[r][0] = __ffma2_rn(xd[r][k], qa, e[r][0]);
            e[r][1] = __ffma2_rn(xd[r][k], qb2, e[r][1]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            e[r][h].x = ex2_approx(fminf(e[r][h].x, 0.f));
            e[r][h].y = ex2_approx(fminf(e[r][h].y, 0.f));
          }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) e[r][0] = e[r][1] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float4 q4 = *reinterpret_cast<const float4 *>(q + k * KVP_TQ + j4);  // -c
          const float2 qa = make_float2(q4.x, q4.y), qb2 = make_float2(q4.z, q4.w);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float2 d0 = __fadd2_rn(xd[r][k], qa), d1 = __fadd2_rn(xd[r][k], qb2);
            e[r][0] = __ffma2_rn(d0, d0, e[r][0]);
            e[r][1] = __ffma2_rn(d1, d1, e[r][1]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            e[r][h].x = ex2_approx(-sqrt_approx(e[r][h].x));
            e[r][h].y = ex2_approx(-sqrt_approx(e[r][h].y));
          }
      }
      if (ZD) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          accd[r][0] = fma(k_to_f64(e[r][0].x), zd0.x, accd[r][0]);
          accd[r][1] = fma(k_to_f64(e[r][0].y), zd0.y, accd[r][1]);
          accd[r][0] = fma(k_to_f64(e[r][1].x), zd1.x, accd[r][0]);
          accd[r][1] = fma(k_to_f64(e[r][1].y), zd1.y, accd[r][1]);
        }
      } else {
        const float2 za = make_float2(zz.x, zz.y), zb = make_float2(zz.z, zz.w);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r][0] = __ffma2_rn(e[r][0], za, acc[r][0]);
          acc[r][1] = __ffma2_rn(e[r][1], zb, acc[r][1]);
        }
      }
    }
    if (!ZD) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        acc64[r] += (double)((acc[r][0].x + acc[r][0].y) + (acc[r][1].x + acc[r][1].y));
    }
    __syncthreads();
    if (tid == 0 && t + 2 < ntiles) issue(t + 2);
  }
  if (ZD) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc64[r] = accd[r][0] + accd[r][1];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t p = pbase + (int64_t)r * KVP_THREADS;
    if (p < np) {
      if (out64) out64[(int64_t)blockIdx.y * np + p] = acc64[r];
      if (out32) out32[p] = (float)acc64[r];
    }
  }
}

// ------------------------------------------------------------------ fused kvp, any d (SIMT)
// Each thread owns one P point; a tile of 32 Q points is in shared memory; the 32 exponents
// of the tile are accumulated in registers over 32-wide chunks of the dimension.
template <int KER, bool ZD = false>
__global__ void __launch_bounds__(KVP_THREADS)
    kvp_generic_kernel(const float *__restrict__ P, const float *__restrict__ pa, int64_t np,
                       const float *__restrict__ Q, const float *__restrict__ qb,
                       const void *__restrict__ zv, int64_t nq, int64_t q_per_split, int dq,
                       double *__restrict__ out64, float *__restrict__ out32) {
  constexpr int TQ = KVP_TQ_G;
  constexpr int ZW = ZD ? 2 : 1;  // z element width in floats (ZD: fp64 z, DFMA contraction)
  extern __shared__ __align__(128) float smem_f[];
  const int QF = TQ * dq;
  float *const SB = smem_f + 2 * QF;
  float *const SZ = SB + 2 * TQ;
  uint64_t *bar = reinterpret_cast<uint64_t *>(SZ + 2 * TQ * ZW);
  const char *z = reinterpret_cast<const char *>(zv);

  const int tid = threadIdx.x;
  const int64_t qlo = (int64_t)blockIdx.y * q_per_split;
  const int64_t qhi = min(nq, qlo + q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, TQ) : 0;
  auto issue = [&](int t) {
    const int64_t q0 = qlo + (int64_t)t * TQ;
    const int cnt = (int)lmin(TQ, qhi - q0);
    const int cnt4 = (cnt + 3) & ~3;
    const int s = t & 1;
    const uint32_t bq = (uint32_t)cnt * dq * 4, bs = (uint32_t)cnt4 * 4, bz = bs * ZW;
    mbar_expect_tx(&bar[s], bq + (KER == FALKON_GAUSSIAN ? bs : 0) + bz);
    bulk_g2s(smem_f + s * QF, Q + q0 * dq, bq, &bar[s]);
    if (KER == FALKON_GAUSSIAN) bulk_g2s(SB + s * TQ, qb + q0, bs, &bar[s]);
    bulk_g2s(SZ + s * TQ * ZW, z + q0 * 4 * ZW, bz, &bar[s]);
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (ntiles > 0) issue(0);
    if (ntiles > 1) issue(1);
  }
  const int64_t p_raw = (int64_t)blockIdx.x * KVP_THREADS + tid;
  const int64_t p = min(p_raw, np - 1);
  const float *prow = P + p * dq;
  const float pav = (KER == FALKON_GAUSSIAN) ? pa[p] : 0.f;
  double acc64 = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bar[s], (t >> 1) & 1);
    const int cnt = (int)lmin(TQ, qhi - (qlo + (int64_t)t * TQ));
    const float *sqs = smem_f + s * QF;
    const float *sbs = SB + s * TQ;
    const float *szs = SZ + s * TQ;
    const double *szd = reinterpret_cast<const double *>(SZ + s * TQ * ZW);
    float e[TQ];
#pragma unroll
    for (int j = 0; j < TQ; ++j) e[j] = (KER == FALKON_GAUSSIAN) ? pav + sbs[j] : 0.f;
    for (int k0 = 0; k0 < dq; k0 += 32) {
      const int kc = min(32, dq - k0);  // multiple of 4
      float pch[32];
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (4 * k4 < kc) v4 = __ldg(reinterpret_cast<const float4 *>(prow + k0) + k4);
        pch[4 * k4 + 0] = v4.x;
        pch[4 * k4 + 1] = v4.y;
        pch[4 * k4 + 2] = v4.z;
        pch[4 * k4 + 3] = v4.w;
      }
#pragma unroll
      for (int j = 0; j < TQ; ++j) {
        const float4 *qrow = reinterpret_cast<const float4 *>(sqs + j * dq + k0);
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          if (4 * k4 < kc) {
            const float4 q4 = qrow[k4];
            if (KER == FALKON_GAUSSIAN) {
              e[j] = fmaf(pch[4 * k4 + 0], q4.x, e[j]);
              e[j] = fmaf(pch[4 * k4 + 1], q4.y, e[j]);
              e[j] = fmaf(pch[4 * k4 + 2], q4.z, e[j]);
              e[j] = fmaf(pch[4 * k4 + 3], q4.w, e[j]);
            } else {
              float df;
              df = pch[4 * k4 + 0] - q4.x; e[j] = fmaf(df, df, e[j]);
              df = pch[4 * k4 + 1] - q4.y; e[j] = fmaf(df, df, e[j]);
              df = pch[4 * k4 + 2] - q4.z; e[j] = fmaf(df, df, e[j]);
              df = pch[4 * k4 + 3] - q4.w; e[j] = fmaf(df, df, e[j]);
            }
          }
        }
      }
    }
    float acc = 0.f;
    double ad[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < TQ; ++j) {
      if (j < cnt) {
        const float kv = (KER == FALKON_GAUSSIAN) ? ex2_approx(fminf(e[j], 0.f))
                                                  : ex2_approx(-sqrt_approx(e[j]));
        if (ZD) ad[j & 1] = fma(k_to_f64(kv), szd[j], ad[j & 1]);
        else acc = fmaf(kv, szs[j], acc);
      }
    }
    acc64 += ZD ? ad[0] + ad[1] : (double)acc;
    __syncthreads();
    if (tid == 0 && t + 2 < ntiles) issue(t + 2);
  }
  if (p_raw < np) {
    if (out64) out64[(int64_t)blockIdx.y * np + p_raw] = acc64;
    if (out32) out32[p_raw] = (float)acc64;
  }
}

// ------------------------------------------------------------------ fp64 path (FALKON_PATH_F64)
// For fits whose alpha must match an fp64 reference where fp32 kernel values cannot (small d,
// large m: the CG iterate amplifies the ~1e-7 relative error of fp32 k; reading d4):
// coordinates (x - mu) g computed in fp64 from the fp32 inputs (exact upcast), the exponent,
// the exp2 and the contractions in fp64.  The FP64 pipe (~64 DFMA/clk/SM on B200) binds.
// fp64 path, d <= 64 (the fits that reading d4 routes here): register-blocked.  Both operands
// in the tile-transposed fp64 layout [tile of 128 points][k][128]; a CTA keeps its P tile in
// shared memory and streams Q tiles of 128 points (bulk copies, 2-stage ring); thread (tp, tq)
// owns 8 P rows x 8 Q columns (pairs 2tp + 32i, 2tq + 32j: conflict-free LDS.128), so per
// coordinate 8 LDS.128 feed 64 DFMA.  Q columns past the split's range get z = 0 (the padding of z
// is not guaranteed: pass B's z is pass A's output).
// The per-row sums of the 16 tq threads are reduced in a fixed order (deterministic).
constexpr int K64_T = 128;
constexpr int K64_DMAX = 64;  // multiple of 4
// exp2 in fp64 for t <= 0: range reduction t = n + f (|f| <= 1/2, n by the 1.5 * 2^52 rounding
// trick, which also leaves n in the low word), a degree-11 polynomial for 2^f in f itself
// (coefficients (ln 2)^k / k!: remainder < 1e-14 relative), and 2^n added to the exponent field
// with an integer add (no conversions, no final multiply: 14 fp64 operations).  t is clamped at
// -1000 (2^-1000 ~ 1e-301: below any contribution).  A 64-entry shared-memory table with a
// degree-5 polynomial measured slower (HIGGS / TAXI fp64 products -16 % / -21 %).
__device__ __forceinline__ double exp2_f64(double t) {  // t <= 0
  t = fmax(t, -1000.0);
  const double u = t + 6755399441055744.0;  // 1.5 * 2^52 + rint(t)
  const int ni = __double2loint(u);         // rint(t), two's complement
  const double f = t - (u - 6755399441055744.0);
  double p = 4.44553827187081e-10;  // (ln 2)^11 / 11!
  p = fma(p, f, 7.054911620801121e-09);
  p = fma(p, f, 1.0178086009239696e-07);
  p = fma(p, f, 1.3215486790144305e-06);
  p = fma(p, f, 1.5252733804059838e-05);
  p = fma(p, f, 0.00015403530393381606);
  p = fma(p, f, 0.0013333558146428441);
  p = fma(p, f, 0.009618129107628477);
  p = fma(p, f, 0.055504108664821576);
  p = fma(p, f, 0.2402265069591007);
  p = fma(p, f, 0.6931471805599453);
  p = fma(p, f, 1.0);  // in [0.70, 1.42]
  return __hiloint2double(__double2hiint(p) + (ni << 20), __double2loint(p));
}

__global__ void pack_rows64_tt_kernel(const float *__restrict__ in, int64_t rows, int64_t rows_pad,
                                      int64_t d, const double *__restrict__ mu, double g, int dq,
                                      double *__restrict__ out, double *__restrict__ bias) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_pad) return;
  double *o = out + (r / K64_T) * dq * K64_T + (r % K64_T);
  double ss = 0.0;
  for (int k = 0; k < dq; ++k) {
    const double v = (r < rows && k < d) ? ((double)in[r * d + k] - mu[k]) * g : 0.0;
    o[(int64_t)k * K64_T] = v;
    ss = fma(v, v, ss);
  }
  if (bias) bias[r] = -0.5 * ss;
}
__device__ __forceinline__ double2 lds_d2(const double *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}
template <int KER>
__global__ void __launch_bounds__(256, 1)
    kvp64t_kernel(const double *__restrict__ P, const double *__restrict__ pa, int64_t np,
                  const double *__restrict__ Q, const double *__restrict__ qb,
                  const double *__restrict__ z, int64_t nq, int64_t q_per_split, int dq,
                  double *__restrict__ out64) {
  extern __shared__ __align__(128) double sm64[];
  const int TB = dq * K64_T;  // doubles per tile
  // [3 mbarriers, padded to 128 B][P tile][2 Q tiles][2 x 128 biases][2 x 128 z]; the final
  // [16][128] row reduction reuses the data region (the host sizes it for both)
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm64);  // P, Q stage 0, Q stage 1
  double *sP = sm64 + 16, *sQ = sP + TB, *sB = sQ + 2 * TB, *sZ = sB + 2 * K64_T;
  const int tid = threadIdx.x, tp = tid >> 4, tq = tid & 15;
  const int64_t pt = blockIdx.x;  // P tile
  const int64_t qlo = (int64_t)blockIdx.y * q_per_split;
  const int64_t qhi = min(nq, qlo + q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, K64_T) : 0;
  const bool gauss = KER == FALKON_GAUSSIAN;
  auto issue = [&](int t) {
    const int64_t qt = (qlo + (int64_t)t * K64_T) / K64_T;
    const int s = t & 1;
    const uint32_t bt = (uint32_t)TB * 8, bv = K64_T * 8;
    mbar_expect_tx(&bar[1 + s], bt + bv + (gauss ? bv : 0));
    bulk_g2s(sQ + s * TB, Q + qt * TB, bt, &bar[1 + s]);
    bulk_g2s(sZ + s * K64_T, z + qt * K64_T, bv, &bar[1 + s]);
    if (gauss) bulk_g2s(sB + s * K64_T, qb + qt * K64_T, bv, &bar[1 + s]);
  };
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar[0], (uint32_t)TB * 8);
    bulk_g2s(sP, P + pt * TB, (uint32_t)TB * 8, &bar[0]);
    if (ntiles > 0) issue(0);
    if (ntiles > 1) issue(1);
  }
  double pav[8], part[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = pt * K64_T + 2 * tp + 32 * (i >> 1) + (i & 1);
    pav[i] = gauss ? pa[r] : 0.0;  // biases are padded to the tile
    part[i] = 0.0;
  }
  mbar_wait(&bar[0], 0);
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bar[1 + s], (t >> 1) & 1);
    const double *q = sQ + s * TB;
    double acc[8][8];
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
      const double2 b2 = gauss ? lds_d2(sB + s * K64_T + 2 * tq + 32 * j2) : make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[i][2 * j2] = pav[i] + b2.x;
        acc[i][2 * j2 + 1] = pav[i] + b2.y;
      }
    }
    for (int k = 0; k < dq; ++k) {
      double pv[8], qv[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 a2 = lds_d2(sP + k * K64_T + 2 * tp + 32 * h);
        const double2 c2 = lds_d2(q + k * K64_T + 2 * tq + 32 * h);
        pv[2 * h] = a2.x, pv[2 * h + 1] = a2.y;
        qv[2 * h] = c2.x, qv[2 * h + 1] = c2.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (gauss) {
            acc[i][j] = fma(pv[i], qv[j], acc[i][j]);
          } else {
            const double df = pv[i] - qv[j];
            acc[i][j] = fma(df, df, acc[i][j]);
          }
        }
    }
    const int64_t qc0 = qlo + (int64_t)t * K64_T;  // columns past nq contribute zero
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
      double2 z2 = lds_d2(sZ + s * K64_T + 2 * tq + 32 * j2);
      const int64_t c = qc0 + 2 * tq + 32 * j2;
      if (c >= qhi) z2.x = 0.0;
      if (c + 1 >= qhi) z2.y = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double k0 = gauss ? exp2_f64(fmin(acc[i][2 * j2], 0.0)) : exp2_f64(-sqrt(acc[i][2 * j2]));
        const double k1 = gauss ? exp2_f64(fmin(acc[i][2 * j2 + 1], 0.0))
                                : exp2_f64(-sqrt(acc[i][2 * j2 + 1]));
        part[i] = fma(k0, z2.x, part[i]);
        part[i] = fma(k1, z2.y, part[i]);
      }
    }
    __syncthreads();
    if (tid == 0 && t + 2 < ntiles) issue(t + 2);
  }
  // fixed-order reduction over the 16 tq threads of each row (the Q stage buffers are free)
  double *red = sP;  // [16][128]
#pragma unroll
  for (int i = 0; i < 8; ++i) red[tq * K64_T + 2 * tp + 32 * (i >> 1) + (i & 1)] = part[i];
  __syncthreads();
  if (tid < K64_T) {
    double sum = 0.0;
    for (int c = 0; c < 16; ++c) sum += red[c * K64_T + tid];
    const int64_t r = pt * K64_T + tid;
    if (r < np) out64[(int64_t)blockIdx.y * np + r] = sum;
  }
}

// fp64 path, Gaussian, d <= 64: the cross term on the FP64 tensor pipe (DMMA m8n8k4), the exp2
// and the contraction on the FP64 CUDA cores, so the two pipes work side by side.  Same
// operands, shared-memory tiles and bulk-copy ring as kvp64t_kernel; warp w computes the
// 32 x 64 block (P rows 32 (w & 3).., Q columns 64 (w >> 2)..) of a 128 x 128 tile as 4 x 8
// m8n8 accumulators (fragment: row lane/4, columns 2 (lane % 4) + {0, 1}).  The per-row sums
// are reduced over the 4 lanes of a row (shuffles) and the 2 warps of a row block (shared
// memory), in a fixed order.
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
// NWQ warps split a row block's 128 columns (2: 8 warps of 32 x 64; 4: 16 warps of 32 x 32)
template <int NWQ>
__global__ void __launch_bounds__(128 * NWQ, 1)
    kvp64m_kernel(const double *__restrict__ P, const double *__restrict__ pa, int64_t np,
                  const double *__restrict__ Q, const double *__restrict__ qb,
                  const double *__restrict__ z, int64_t nq, int64_t q_per_split, int dq,
                  double *__restrict__ out64) {
  extern __shared__ __align__(128) double sm64m[];
  const int TB = dq * K64_T;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm64m);  // P, Q stage 0, Q stage 1
  double *sP = sm64m + 16, *sQ = sP + TB, *sB = sQ + 2 * TB, *sZ = sB + 2 * K64_T;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int TJ = 16 / NWQ, WC = 128 / NWQ;  // 8-column tiles and columns per warp
  const int wp = warp & 3, wq = warp >> 2, g = lane >> 2, c = lane & 3;
  const int64_t pt = blockIdx.x;
  const int64_t qlo = (int64_t)blockIdx.y * q_per_split;
  const int64_t qhi = min(nq, qlo + q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, K64_T) : 0;
  auto issue = [&](int t) {
    const int64_t qt = (qlo + (int64_t)t * K64_T) / K64_T;
    const int s = t & 1;
    const uint32_t bt = (uint32_t)TB * 8, bv = K64_T * 8;
    mbar_expect_tx(&bar[1 + s], bt + 2 * bv);
    bulk_g2s(sQ + s * TB, Q + qt * TB, bt, &bar[1 + s]);
    bulk_g2s(sZ + s * K64_T, z + qt * K64_T, bv, &bar[1 + s]);
    bulk_g2s(sB + s * K64_T, qb + qt * K64_T, bv, &bar[1 + s]);
  };
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(&bar[0], (uint32_t)TB * 8);
    bulk_g2s(sP, P + pt * TB, (uint32_t)TB * 8, &bar[0]);
    if (ntiles > 0) issue(0);
    if (ntiles > 1) issue(1);
  }
  const int prow = 32 * wp + g;  // + 8 ti
  double pav[4], part[4];
#pragma unroll
  for (int ti = 0; ti < 4; ++ti) {
    pav[ti] = pa[pt * K64_T + prow + 8 * ti];  // biases are padded to the tile
    part[ti] = 0.0;
  }
  mbar_wait(&bar[0], 0);
  for (int t = 0; t < ntiles; ++t) {
    const int s = t & 1;
    mbar_wait(&bar[1 + s], (t >> 1) & 1);
    const double *q = sQ + s * TB;
    double acc[4][TJ][2];  // the DMMAs accumulate onto the biases a_p + b_q
#pragma unroll
    for (int tj = 0; tj < TJ; ++tj) {
      const double2 b2 = lds_d2(sB + s * K64_T + WC * wq + 8 * tj + 2 * c);
#pragma unroll
      for (int ti = 0; ti < 4; ++ti) {
        acc[ti][tj][0] = pav[ti] + b2.x;
        acc[ti][tj][1] = pav[ti] + b2.y;
      }
    }
    for (int k0 = 0; k0 < dq; k0 += 4) {
      const double *pk = sP + (k0 + c) * K64_T + prow;
      const double *qk = q + (k0 + c) * K64_T + WC * wq + g;
      double a[4], b[TJ];
#pragma unroll
      for (int ti = 0; ti < 4; ++ti) a[ti] = pk[8 * ti];
#pragma unroll
      for (int tj = 0; tj < TJ; ++tj) b[tj] = qk[8 * tj];
#pragma unroll
      for (int ti = 0; ti < 4; ++ti)
#pragma unroll
        for (int tj = 0; tj < TJ; ++tj) dmma884(acc[ti][tj], a[ti], b[tj]);
    }
    const int64_t qc0 = qlo + (int64_t)t * K64_T;
#pragma unroll
    for (int tj = 0; tj < TJ; ++tj) {
      const int col = WC * wq + 8 * tj + 2 * c;
      double2 z2 = lds_d2(sZ + s * K64_T + col);
      if (qc0 + col >= qhi) z2.x = 0.0;  // columns past the split's range contribute zero
      if (qc0 + col + 1 >= qhi) z2.y = 0.0;
#pragma unroll
      for (int ti = 0; ti < 4; ++ti) {
        const double k0 = exp2_f64(fmin(acc[ti][tj][0], 0.0));
        const double k1 = exp2_f64(fmin(acc[ti][tj][1], 0.0));
        part[ti] = fma(k0, z2.x, part[ti]);
        part[ti] = fma(k1, z2.y, part[ti]);
      }
    }
    __syncthreads();
    if (tid == 0 && t + 2 < ntiles) issue(t + 2);
  }
  // fixed-order reductions: the 4 lanes of a row (xor 1, 2), then the NWQ column-block warps
#pragma unroll
  for (int ti = 0; ti < 4; ++ti) {
    part[ti] += __shfl_xor_sync(0xffffffffu, part[ti], 1);
    part[ti] += __shfl_xor_sync(0xffffffffu, part[ti], 2);
  }
  double *red = sP;  // [NWQ][128]
  if (c == 0) {
#pragma unroll
    for (int ti = 0; ti < 4; ++ti) red[wq * K64_T + prow + 8 * ti] = part[ti];
  }
  __syncthreads();
  if (tid < K64_T) {
    const int64_t r = pt * K64_T + tid;
    double sum = red[tid];
#pragma unroll
    for (int w = 1; w < NWQ; ++w) sum += red[w * K64_T + tid];
    if (r < np) out64[(int64_t)blockIdx.y * np + r] = sum;
  }
}

// fp64 path, d > 64: the same 8 x 8 register blocking with the coordinates streamed in chunks
// of K64_KC (P and Q chunk of a Q tile per stage, 2-stage bulk-copy ring over the flattened
// (Q tile, chunk) sequence); the operands use the tile-transposed layout with dq a multiple
// of K64_KC.
constexpr int K64_KC = 32;
template <int KER>
__global__ void __launch_bounds__(256, 1)
    kvp64c_kernel(const double *__restrict__ P, const double *__restrict__ pa, int64_t np,
                  const double *__restrict__ Q, const double *__restrict__ qb,
                  const double *__restrict__ z, int64_t nq, int64_t q_per_split, int dq,
                  double *__restrict__ out64) {
  extern __shared__ __align__(128) double sm64c[];
  constexpr int CB = K64_KC * K64_T;  // doubles per chunk of one tile
  const int TB = dq * K64_T, nkc = dq / K64_KC;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm64c);  // stage 0, stage 1
  double *sS = sm64c + 16;                              // 2 stages x (P chunk, Q chunk)
  double *sB = sS + 4 * CB, *sZ = sB + 2 * K64_T;       // per Q-tile parity
  const int tid = threadIdx.x, tp = tid >> 4, tq = tid & 15;
  const int64_t pt = blockIdx.x;
  const int64_t qlo = (int64_t)blockIdx.y * q_per_split;
  const int64_t qhi = min(nq, qlo + q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, K64_T) : 0;
  const int nitems = ntiles * nkc;
  const bool gauss = KER == FALKON_GAUSSIAN;
  auto issue = [&](int it) {
    const int t = it / nkc, c = it % nkc, s = it & 1;
    const int64_t qt = (qlo + (int64_t)t * K64_T) / K64_T;
    const uint32_t bc = (uint32_t)CB * 8, bv = K64_T * 8;
    mbar_expect_tx(&bar[s], 2 * bc + (c == 0 ? bv + (gauss ? bv : 0) : 0));
    bulk_g2s(sS + (2 * s) * CB, P + pt * TB + (int64_t)c * CB, bc, &bar[s]);
    bulk_g2s(sS + (2 * s + 1) * CB, Q + qt * TB + (int64_t)c * CB, bc, &bar[s]);
    if (c == 0) {
      bulk_g2s(sZ + (t & 1) * K64_T, z + qt * K64_T, bv, &bar[s]);
      if (gauss) bulk_g2s(sB + (t & 1) * K64_T, qb + qt * K64_T, bv, &bar[s]);
    }
  };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (nitems > 0) issue(0);
    if (nitems > 1) issue(1);
  }
  double pav[8], part[8], acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = pt * K64_T + 2 * tp + 32 * (i >> 1) + (i & 1);
    pav[i] = gauss ? pa[r] : 0.0;
    part[i] = 0.0;
  }
  for (int it = 0; it < nitems; ++it) {
    const int t = it / nkc, c = it % nkc, s = it & 1;
    mbar_wait(&bar[s], (it >> 1) & 1);
    if (c == 0) {
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        const double2 b2 =
            gauss ? lds_d2(sB + (t & 1) * K64_T + 2 * tq + 32 * j2) : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i][2 * j2] = pav[i] + b2.x;
          acc[i][2 * j2 + 1] = pav[i] + b2.y;
        }
      }
    }
    const double *ps = sS + (2 * s) * CB, *qs = sS + (2 * s + 1) * CB;
    for (int k = 0; k < K64_KC; ++k) {
      double pv[8], qv[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 a2 = lds_d2(ps + k * K64_T + 2 * tp + 32 * h);
        const double2 c2 = lds_d2(qs + k * K64_T + 2 * tq + 32 * h);
        pv[2 * h] = a2.x, pv[2 * h + 1] = a2.y;
        qv[2 * h] = c2.x, qv[2 * h + 1] = c2.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (gauss) {
            acc[i][j] = fma(pv[i], qv[j], acc[i][j]);
          } else {
            const double df = pv[i] - qv[j];
            acc[i][j] = fma(df, df, acc[i][j]);
          }
        }
    }
    if (c == nkc - 1) {  // tile done: exp2 and contraction (columns past the range: z = 0)
      const int64_t qc0 = qlo + (int64_t)t * K64_T;
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        double2 z2 = lds_d2(sZ + (t & 1) * K64_T + 2 * tq + 32 * j2);
        const int64_t col = qc0 + 2 * tq + 32 * j2;
        if (col >= qhi) z2.x = 0.0;
        if (col + 1 >= qhi) z2.y = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double k0 = gauss ? exp2_f64(fmin(acc[i][2 * j2], 0.0)) : exp2_f64(-sqrt(acc[i][2 * j2]));
          const double k1 = gauss ? exp2_f64(fmin(acc[i][2 * j2 + 1], 0.0))
                                  : exp2_f64(-sqrt(acc[i][2 * j2 + 1]));
          part[i] = fma(k0, z2.x, part[i]);
          part[i] = fma(k1, z2.y, part[i]);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && it + 2 < nitems) issue(it + 2);
  }
  double *red = sS;  // [16][128] fixed-order row reduction
#pragma unroll
  for (int i = 0; i < 8; ++i) red[tq * K64_T + 2 * tp + 32 * (i >> 1) + (i & 1)] = part[i];
  __syncthreads();
  if (tid < K64_T) {
    double sum = 0.0;
    for (int c = 0; c < 16; ++c) sum += red[c * K64_T + tid];
    const int64_t r = pt * K64_T + tid;
    if (r < np) out64[(int64_t)blockIdx.y * np + r] = sum;
  }
}

// ------------------------------------------------------------------ reductions / conversions
__global__ void reduce_splits_kernel(const double *__restrict__ part, int splits, int64_t np,
                                     double *__restrict__ out64, float *__restrict__ out32) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  double s = 0.0;
  for (int i = 0; i < splits; ++i) s += part[(int64_t)i * np + p];
  if (out64) out64[p] = s;
  if (out32) out32[p] = (float)s;
}

__global__ void f64_to_f32_kernel(const double *__restrict__ s, float *__restrict__ d, int64_t n,
                                  int64_t n_pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = (float)s[i];
  else if (i < n_pad) d[i] = 0.f;
}
__global__ void f32_copy_pad_kernel(const float *__restrict__ s, float *__restrict__ d, int64_t n,
                                    int64_t n_pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = s[i];
  else if (i < n_pad) d[i] = 0.f;
}

int reduce_partials(falkon_ctx *ctx, const double *part, int64_t splits, int64_t np,
                    double *out64, float *out32) {
  LaunchScope ls(ctx, FALKON_T_REDUCE);
  reduce_splits_kernel<<<(unsigned)cdiv<int64_t>(np, 256), 256, 0, ctx->stream>>>(
      part, (int)splits, np, out64, out32);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

int f64_to_f32(falkon_ctx *ctx, const double *src, float *dst, int64_t n, int64_t n_pad) {
  if (n_pad <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  f64_to_f32_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(src, dst, n,
                                                                                    n_pad);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}
int f32_to_f32_pad(falkon_ctx *ctx, const float *src, float *dst, int64_t n, int64_t n_pad) {
  if (n_pad <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  f32_copy_pad_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(src, dst, n,
                                                                                      n_pad);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// ------------------------------------------------------------------ dispatch
typedef void (*kvp_fn)(const float *, const float *, int64_t, const float *, const float *,
                       const void *, int64_t, int64_t, double *, float *);

template <int KER, int D>
static kvp_fn pick_small_R(int R, bool zd) {
  if (zd) return R == 4 ? kvp_pk_kernel<KER, D, 4, true> : kvp_pk_kernel<KER, D, 2, true>;
  if (R == 4) return kvp_pk_kernel<KER, D, 4>;
  return kvp_pk_kernel<KER, D, 2>;
}

// exact D for d <= 16; multiples of 4 up to 32 (zero-padded coordinates add exact zeros)
static int small_D(int64_t d) {
  if (d <= 16) return (int)d;
  return (int)round_up<int64_t>(d, 4);
}
static int small_R(int D) { return D <= 12 ? 4 : 2; }

template <int KER>
static kvp_fn pick_small(int D, int R, bool zd) {
  switch (D) {
#define FK_CASE(DD) \
  case DD: return pick_small_R<KER, DD>(R, zd);
    FK_CASE(1) FK_CASE(2) FK_CASE(3) FK_CASE(4) FK_CASE(5) FK_CASE(6) FK_CASE(7) FK_CASE(8)
    FK_CASE(9) FK_CASE(10) FK_CASE(11) FK_CASE(12) FK_CASE(13) FK_CASE(14) FK_CASE(15)
    FK_CASE(16) FK_CASE(20) FK_CASE(24) FK_CASE(28) FK_CASE(32)
#undef FK_CASE
    default: return nullptr;
  }
}

static int occupancy(const void *fn, int threads, size_t smem) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return std::max(nb, 1);
}

// One kvp launch (+ split reduction).  out64 (np, optional) / out32 (np, optional).
// zd: z is fp64 and the contraction runs in fp64 (FALKON_OPT_ACCUM_F64).
static int kvp_launch(falkon_ctx *ctx, int kernel, int64_t d, int dq, const float *P,
                      const float *pa, int64_t np, const float *Q, const float *qb, const void *z,
                      int64_t nq, int cls, double *out64, float *out32, bool zd = false) {
  if (np <= 0) return FALKON_OK;
  const bool small = d <= 32;
  int D = 0, R = 1, TQ;
  const void *fn;
  size_t smem;
  if (small) {
    D = small_D(d);
    R = small_R(D);
    const int DQ = (D + 3) & ~3;
    TQ = KVP_TQ;
    fn = (const void *)(kernel == FALKON_GAUSSIAN ? pick_small<FALKON_GAUSSIAN>(D, R, zd)
                                                  : pick_small<FALKON_LAPLACIAN>(D, R, zd));
    smem = (size_t)(2 * TQ * D + (zd ? 6 : 4) * TQ) * 4 + 16;
    (void)DQ;
  } else {
    TQ = KVP_TQ_G;
    if (zd)
      fn = (const void *)(kernel == FALKON_GAUSSIAN ? kvp_generic_kernel<FALKON_GAUSSIAN, true>
                                                    : kvp_generic_kernel<FALKON_LAPLACIAN, true>);
    else
      fn = (const void *)(kernel == FALKON_GAUSSIAN ? kvp_generic_kernel<FALKON_GAUSSIAN>
                                                    : kvp_generic_kernel<FALKON_LAPLACIAN>);
    smem = (size_t)(2 * TQ * dq + (zd ? 6 : 4) * TQ) * 4 + 16;
  }
  if (!fn) return fail(FALKON_EINVAL, "no kvp kernel for d=" + std::to_string(d));
  FK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t per_cta = (int64_t)KVP_THREADS * R;
  const int64_t gx = cdiv<int64_t>(np, per_cta);
  const int64_t capacity = (int64_t)ctx->sm_count * occupancy(fn, KVP_THREADS, smem);
  int64_t splits = 1;
  if (gx < capacity) {
    splits = std::max<int64_t>(1, capacity / gx);
    const int64_t min_q = 4 * TQ;  // at least a few tiles per split
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, nq / min_q));
    splits = std::min<int64_t>(splits, 65535);
  }
  int64_t qps = round_up<int64_t>(cdiv<int64_t>(nq, splits), TQ);
  splits = std::max<int64_t>(1, cdiv<int64_t>(nq, qps));
  if (gx > 0x7fffffffLL) return fail(FALKON_EINVAL, "too many rows for one launch");

  double *part = out64;
  if (splits > 1 || !out64) {
    void *pp;
    FK_TRY(ws_get(ctx, WS_PART, sizeof(double) * splits * np, &pp));
    part = (double *)pp;
  }
  dim3 grid((unsigned)gx, (unsigned)splits);
  {
    LaunchScope ls(ctx, cls);
    if (small) {
      ((kvp_fn)fn)<<<grid, KVP_THREADS, smem, ctx->stream>>>(P, pa, np, Q, qb, z, nq, qps, part,
                                                             splits == 1 ? out32 : nullptr);
    } else {
      typedef void (*gen_fn)(const float *, const float *, int64_t, const float *, const float *,
                             const void *, int64_t, int64_t, int, double *, float *);
      ((gen_fn)fn)<<<grid, KVP_THREADS, smem, ctx->stream>>>(P, pa, np, Q, qb, z, nq, qps, dq,
                                                             part, splits == 1 ? out32 : nullptr);
    }
  }
  FK_LAUNCH_CHECK();
  if (splits > 1 || (!out64 && !out32)) {
    LaunchScope ls(ctx, FALKON_T_REDUCE);
    reduce_splits_kernel<<<(unsigned)cdiv<int64_t>(np, 256), 256, 0, ctx->stream>>>(
        part, (int)splits, np, out64, out32);
    FK_LAUNCH_CHECK();
  } else if (splits == 1 && !out64) {
    // out32 already written by the kernel
  }
  return FALKON_OK;
}

// fp64 path launch: out64[p] = sum_q k(P_p, Q_q) z_q (+ the deterministic split reduction)
static int kvp64_launch(falkon_ctx *ctx, int kernel, int dq, const double *P, const double *pa,
                        int64_t np, const double *Q, const double *qb, const double *z,
                        int64_t nq, int cls, double *out64) {
  if (np <= 0) return FALKON_OK;
  // register-blocked kernels on the tile-transposed layout: P resident (dq <= 64) or streamed
  // in chunks of K64_KC coordinates (dq a multiple of K64_KC, see prepare_operands)
  const bool resident = dq <= K64_DMAX;
  const int TQ = K64_T;
  // Gaussian, d <= 64: cross term on DMMA (FALKON_F64_DMMA=0 selects the all-DFMA kernel, A/B)
  const char *dm = getenv("FALKON_F64_DMMA");
  const bool dmma = kernel == FALKON_GAUSSIAN && resident && !(dm && atoi(dm) == 0);
  // FALKON_F64_NWQ=2 (A/B): 8 warps of 32 x 64 instead of 16 of 32 x 32
  const char *nw = getenv("FALKON_F64_NWQ");
  const bool w16 = !(nw && atoi(nw) == 2);
  const int threads = (dmma && w16) ? 512 : 256;
  const void *fn = dmma ? (w16 ? (const void *)kvp64m_kernel<4> : (const void *)kvp64m_kernel<2>)
      : resident
      ? (kernel == FALKON_GAUSSIAN ? (const void *)kvp64t_kernel<FALKON_GAUSSIAN>
                                   : (const void *)kvp64t_kernel<FALKON_LAPLACIAN>)
      : (kernel == FALKON_GAUSSIAN ? (const void *)kvp64c_kernel<FALKON_GAUSSIAN>
                                   : (const void *)kvp64c_kernel<FALKON_LAPLACIAN>);
  const size_t smem = resident
      ? (size_t)(16 + std::max(3 * dq * K64_T + 4 * K64_T, 16 * K64_T)) * 8
      : (size_t)(16 + 4 * K64_KC * K64_T + 4 * K64_T) * 8;
  if (smem > 227 * 1024) return fail(FALKON_EUNSUPPORTED, "fp64 path: d too large");
  FK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t gx = cdiv<int64_t>(np, K64_T);
  const int64_t capacity = (int64_t)ctx->sm_count * occupancy(fn, threads, smem);
  int64_t splits = 1;
  if (gx < 4 * capacity) {  // several waves: fewer tail effects
    splits = std::max<int64_t>(1, 4 * capacity / gx);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, nq / (4 * TQ)));
    splits = std::min<int64_t>(splits, 65535);
  }
  const int64_t qps = round_up<int64_t>(cdiv<int64_t>(nq, splits), TQ);
  splits = std::max<int64_t>(1, cdiv<int64_t>(nq, qps));
  if (gx > 0x7fffffffLL) return fail(FALKON_EINVAL, "too many rows for one launch");
  double *part = out64;
  if (splits > 1) {
    void *pp;
    FK_TRY(ws_get(ctx, WS_PART, sizeof(double) * splits * np, &pp));
    part = (double *)pp;
  }
  {
    LaunchScope ls(ctx, cls);
    typedef void (*f64_fn)(const double *, const double *, int64_t, const double *, const double *,
                           const double *, int64_t, int64_t, int, double *);
    ((f64_fn)fn)<<<dim3((unsigned)gx, (unsigned)splits), threads, smem, ctx->stream>>>(
        P, pa, np, Q, qb, z, nq, qps, dq, part);
  }
  FK_LAUNCH_CHECK();
  if (splits > 1) {
    LaunchScope ls(ctx, FALKON_T_REDUCE);
    reduce_splits_kernel<<<(unsigned)cdiv<int64_t>(np, 256), 256, 0, ctx->stream>>>(
        part, (int)splits, np, out64, nullptr);
    FK_LAUNCH_CHECK();
  }
  return FALKON_OK;
}

// ------------------------------------------------------------------ public-ish entry points
int prepare_operands(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C,
                     int64_t m, int kernel, double sigma, Prepared *pp) {
  pp->n = n;
  pp->m = m;
  pp->d = d;
  pp->kernel = kernel;
  double *mu;
  FK_TRY(center_mean(ctx, C, m, d, &mu));
  if (ctx->opt.path == FALKON_PATH_F64) {  // fp64 coordinates and biases (tile-transposed)
    pp->path = FALKON_PATH_F64;
    const int dq = (int)round_up<int64_t>(d, d <= K64_DMAX ? 4 : K64_KC);  // DMMA k-steps of 4
    pp->dq = dq;
    const double g = kernel == FALKON_GAUSSIAN ? std::sqrt(LOG2E) / sigma : LOG2E / sigma;
    const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n, 1), 128);
    const int64_t m_pad = round_up<int64_t>(m, 128);
    void *xp, *xa, *cp, *cb;
    FK_TRY(ws_get(ctx, WS_XP, sizeof(double) * n_pad * dq, &xp));
    FK_TRY(ws_get(ctx, WS_XA, sizeof(double) * n_pad, &xa));
    FK_TRY(ws_get(ctx, WS_CP, sizeof(double) * m_pad * dq, &cp));
    FK_TRY(ws_get(ctx, WS_CB, sizeof(double) * m_pad, &cb));
    const bool gauss = kernel == FALKON_GAUSSIAN;
    {  // tile-transposed layout [tile of 128][dq][128] of the register-blocked kernels
      LaunchScope ls(ctx, FALKON_T_PREP);
      pack_rows64_tt_kernel<<<(unsigned)cdiv<int64_t>(m_pad, 256), 256, 0, ctx->stream>>>(
          C, m, m_pad, d, mu, g, dq, (double *)cp, gauss ? (double *)cb : nullptr);
      pack_rows64_tt_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(
          X, n, n_pad, d, mu, g, dq, (double *)xp, gauss ? (double *)xa : nullptr);
    }
    FK_LAUNCH_CHECK();
    pp->Xp = xp;
    pp->xa = (const float *)xa;  // fp64 biases (reinterpreted by the fp64 passes)
    pp->Cp = cp;
    pp->cb = (const float *)cb;
    return FALKON_OK;
  }
  const bool use_tc = tc_supported(ctx, kernel, d);
  if (use_tc) {
    pp->path = FALKON_PATH_TENSOR;
    const int rc = tc_prepare(ctx, X, n, d, C, m, sigma, mu, pp);
    if (rc != FALKON_TC_RANGE) return rc;
    // operands out of the fp16 range of the tensor path's split (e.g. unstandardised data or a
    // tiny sigma): the fp32 SIMT kernels below take this product
  }
  pp->path = FALKON_PATH_SIMT;
  const bool tt = d <= 32;  // packed-FFMA2 kernel: tile-transposed layout, D = small_D(d)
  const int dq = tt ? small_D(d) : (int)round_up<int64_t>(d, 4);
  pp->dq = dq;
  const double g = kernel == FALKON_GAUSSIAN ? std::sqrt(LOG2E) / sigma : LOG2E / sigma;
  // padded to a multiple of 128 rows so tile loads may round up
  const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n, 1), 128);
  const int64_t m_pad = round_up<int64_t>(m, 128);
  void *xp, *xa, *cp, *cb;
  FK_TRY(ws_get(ctx, WS_XP, sizeof(float) * n_pad * dq, &xp));
  FK_TRY(ws_get(ctx, WS_XA, sizeof(float) * n_pad, &xa));
  FK_TRY(ws_get(ctx, WS_CP, sizeof(float) * m_pad * dq, &cp));
  FK_TRY(ws_get(ctx, WS_CB, sizeof(float) * m_pad, &cb));
  const int threads = 256;
  if (tt) {
    const int neg = kernel == FALKON_LAPLACIAN;
    {
      LaunchScope ls(ctx, FALKON_T_PREP);
      pack_rows_tt_kernel<<<(unsigned)cdiv<int64_t>(m_pad, 256), 256, 0, ctx->stream>>>(
          C, m, m_pad, (int)d, dq, mu, g, neg, (float *)cp,
          kernel == FALKON_GAUSSIAN ? (float *)cb : nullptr);
    }
    FK_LAUNCH_CHECK();
    if (n > 0) {
      LaunchScope ls(ctx, FALKON_T_PREP);
      pack_rows_tt_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(
          X, n, n_pad, (int)d, dq, mu, g, neg, (float *)xp,
          kernel == FALKON_GAUSSIAN ? (float *)xa : nullptr);
      FK_LAUNCH_CHECK();
    }
    pp->Xp = xp;
    pp->xa = (const float *)xa;
    pp->Cp = cp;
    pp->cb = (const float *)cb;
    return FALKON_OK;
  }
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    int64_t blocks = std::min<int64_t>(cdiv<int64_t>(m, threads / 32), 65535);
    pack_rows_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(
        C, m, d, mu, g, dq, (float *)cp, kernel == FALKON_GAUSSIAN ? (float *)cb : nullptr);
  }
  FK_LAUNCH_CHECK();
  if (n > 0) {
    LaunchScope ls(ctx, FALKON_T_PREP);
    int64_t blocks = std::min<int64_t>(cdiv<int64_t>(n, threads / 32), (int64_t)ctx->sm_count * 64);
    pack_rows_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(
        X, n, d, mu, g, dq, (float *)xp, kernel == FALKON_GAUSSIAN ? (float *)xa : nullptr);
    FK_LAUNCH_CHECK();
  }
  pp->Xp = xp;
  pp->xa = (const float *)xa;
  pp->Cp = cp;
  pp->cb = (const float *)cb;
  return FALKON_OK;
}

static int f64_needs_f64() {
  return fail(FALKON_EUNSUPPORTED, "FALKON_PATH_F64 products run on fp64 vectors only");
}

int pass_A(falkon_ctx *ctx, const Prepared &pp, const float *z, double *w64, float *w32) {
  if (pp.n <= 0) return FALKON_OK;
  if (pp.path == FALKON_PATH_F64) return f64_needs_f64();
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass(ctx, pp, true, z, w64, w32);
  return kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Xp, pp.xa, pp.n,
                    (const float *)pp.Cp, pp.cb, z, pp.m, FALKON_T_PASS_A, w64, w32);
}

int pass_B(falkon_ctx *ctx, const Prepared &pp, const float *w, double *u) {
  if (pp.n <= 0) {
    FK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * pp.m, ctx->stream));
    return FALKON_OK;
  }
  if (pp.path == FALKON_PATH_F64) return f64_needs_f64();
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass(ctx, pp, false, w, u, nullptr);
  return kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Cp, pp.cb, pp.m,
                    (const float *)pp.Xp, pp.xa, w, pp.n, FALKON_T_PASS_B, u, nullptr);
}

int pass_A64(falkon_ctx *ctx, const Prepared &pp, const double *z, double *w64) {
  if (pp.n <= 0) return FALKON_OK;
  if (pp.path == FALKON_PATH_F64)
    return kvp64_launch(ctx, pp.kernel, pp.dq, (const double *)pp.Xp, (const double *)pp.xa, pp.n,
                        (const double *)pp.Cp, (const double *)pp.cb, z, pp.m, FALKON_T_PASS_A, w64);
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass64(ctx, pp, true, z, w64);
  return kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Xp, pp.xa, pp.n,
                    (const float *)pp.Cp, pp.cb, z, pp.m, FALKON_T_PASS_A, w64, nullptr, true);
}

int pass_B64(falkon_ctx *ctx, const Prepared &pp, const double *w, double *u) {
  if (pp.n <= 0) {
    FK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * pp.m, ctx->stream));
    return FALKON_OK;
  }
  if (pp.path == FALKON_PATH_F64)
    return kvp64_launch(ctx, pp.kernel, pp.dq, (const double *)pp.Cp, (const double *)pp.cb, pp.m,
                        (const double *)pp.Xp, (const double *)pp.xa, w, pp.n, FALKON_T_PASS_B, u);
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass64(ctx, pp, false, w, u);
  return kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Cp, pp.cb, pp.m,
                    (const float *)pp.Xp, pp.xa, w, pp.n, FALKON_T_PASS_B, u, nullptr, true);
}

__global__ void pad_copy_f64_kernel(const double *__restrict__ s, double *__restrict__ d, int64_t n,
                                    int64_t n_pad, const float *__restrict__ scale) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = scale ? s[i] * (double)scale[i] : s[i];
  else if (i < n_pad) d[i] = 0.0;
}
__global__ void pad_copy_f32_f64_kernel(const float *__restrict__ s, double *__restrict__ d,
                                        int64_t n, int64_t n_pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = (double)s[i];
  else if (i < n_pad) d[i] = 0.0;
}

int f64_pad(falkon_ctx *ctx, const double *src, double *dst, int64_t n, int64_t n_pad,
            const float *scale) {
  if (n_pad <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  pad_copy_f64_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(src, dst, n,
                                                                                     n_pad, scale);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}
int f32_to_f64_pad(falkon_ctx *ctx, const float *src, double *dst, int64_t n, int64_t n_pad) {
  if (n_pad <= 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_PREP);
  pad_copy_f32_f64_kernel<<<(unsigned)cdiv<int64_t>(n_pad, 256), 256, 0, ctx->stream>>>(src, dst, n,
                                                                                         n_pad);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// ------------------------------------------------------------------ multi-vector passes
// Z in R^{q x kv} (k outputs, e.g. TIMIT's classes).  Tensor path: one fused
// pass with a kv-wide epilogue (tc_pass, kv = 8 or 16).  SIMT path (Laplacian, d <= 8): the
// single-vector kernel per column (the exp is recomputed per column).
__global__ void col_gather_f32_kernel(const float *__restrict__ src, int64_t rows, int kv, int c,
                                      float *__restrict__ dst, int64_t rows_pad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) dst[i] = src[i * kv + c];
  else if (i < rows_pad) dst[i] = 0.f;
}
template <typename T>
__global__ void col_scatter_kernel(const T *__restrict__ src, int64_t rows, int kv, int c,
                                   T *__restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) dst[i * kv + c] = src[i];
}

static int simt_multi(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z, int kv,
                      double *o64, float *o32) {
  const int64_t np = passA ? pp.n : pp.m, nq = passA ? pp.m : pp.n;
  const int64_t nq_pad = round_up<int64_t>(std::max<int64_t>(nq, 1), 128);
  const int64_t np_pad = round_up<int64_t>(std::max<int64_t>(np, 1), 128);
  void *zc, *oc;
  FK_TRY(ws_get(ctx, WS_MCOL, sizeof(float) * nq_pad, &zc));
  FK_TRY(ws_get(ctx, WS_MCOL64, sizeof(double) * np_pad + sizeof(float) * np_pad, &oc));
  double *c64 = (double *)oc;
  float *c32 = (float *)(c64 + np_pad);
  for (int c = 0; c < kv; ++c) {
    {
      LaunchScope ls(ctx, FALKON_T_PREP);
      col_gather_f32_kernel<<<(unsigned)cdiv<int64_t>(nq_pad, 256), 256, 0, ctx->stream>>>(
          z, nq, kv, c, (float *)zc, nq_pad);
    }
    FK_LAUNCH_CHECK();
    if (passA)
      FK_TRY(kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Xp, pp.xa, pp.n,
                        (const float *)pp.Cp, pp.cb, (const float *)zc, pp.m, FALKON_T_PASS_A,
                        o64 ? c64 : nullptr, o32 ? c32 : nullptr));
    else
      FK_TRY(kvp_launch(ctx, pp.kernel, pp.d, pp.dq, (const float *)pp.Cp, pp.cb, pp.m,
                        (const float *)pp.Xp, pp.xa, (const float *)zc, pp.n, FALKON_T_PASS_B,
                        c64, nullptr));
    LaunchScope ls(ctx, FALKON_T_PREP);
    if (o64)
      col_scatter_kernel<double><<<(unsigned)cdiv<int64_t>(np, 256), 256, 0, ctx->stream>>>(
          c64, np, kv, c, o64);
    if (o32)
      col_scatter_kernel<float><<<(unsigned)cdiv<int64_t>(np, 256), 256, 0, ctx->stream>>>(
          c32, np, kv, c, o32);
    FK_LAUNCH_CHECK();
  }
  return FALKON_OK;
}

int pass_A_multi(falkon_ctx *ctx, const Prepared &pp, const float *z, int kv, double *w64,
                 float *w32) {
  if (pp.n <= 0) return FALKON_OK;
  if (pp.path == FALKON_PATH_F64) return f64_needs_f64();
  if (kv == 1) return pass_A(ctx, pp, z, w64, w32);
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass(ctx, pp, true, z, w64, w32, kv);
  return simt_multi(ctx, pp, true, z, kv, w64, w32);
}

int pass_B_multi(falkon_ctx *ctx, const Prepared &pp, const float *w, int kv, double *u) {
  if (pp.path == FALKON_PATH_F64) return f64_needs_f64();
  if (pp.n <= 0) {
    FK_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * pp.m * kv, ctx->stream));
    return FALKON_OK;
  }
  if (kv == 1) return pass_B(ctx, pp, w, u);
  if (pp.path == FALKON_PATH_TENSOR) return tc_pass(ctx, pp, false, w, u, nullptr, kv);
  return simt_multi(ctx, pp, false, w, kv, u, nullptr);
}

}  // namespace falkon
