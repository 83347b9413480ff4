// kvp_tc.cu — fused kernel-vector product with the cross term on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), Gaussian kernel, large d (north_star: "Tensor cores
// are used only for the X.C^T distance GEMM when d is large").
//
// Same primitive as kvp.cu:  out[p] = sum_q k(P_p, Q_q) z_q,  k = exp2(min(t_pq, 0)),
//   t_pq = a_p + b_q + x~_p . c~_q = -||x~_p - c~_q||^2 / 2
//
// Precision ("fp16x3", SURVEY.md §7 hard part 2; single-pass TF32/fp16 fails parity):
// every centred, scaled fp32 coordinate is split x~ = h + l with h = fp16(x~),
// l = fp16(x~ - h), and the cross term is the sum of three fp16 MMAs with fp32
// accumulation in TMEM:   h_p.h_q + l_p.h_q + h_p.l_q   (l_p.l_q ~ 2^-22 dropped).
// The biases are folded into the same MMAs through two spare K slots per segment:
//   h-segment slots [d, d+1] = (1, 1);  l-segment slots [d, d+1] = fp16 hi/lo of (bias - 1)
// so  h.h adds 2,  l_p.h_q adds a_p - 1,  h_p.l_q adds b_q - 1:  total a_p + b_q.  The
// accumulator therefore holds the exponent t_pq itself and the epilogue is just
// clamp -> ex2 (MUFU) -> FFMA with z_q.  One symmetric packed layout [h (d16) | l (d16)]
// (d16 = round_up(d + 2, 16)) serves a point on either side of the product.
// Precision (measured, scripts/k_precision.py, profiles/r2_k_precision.jsonl): the tensor
// cores truncate (round toward zero) when accumulating in fp32 (scripts/probes/
// mma_rounding.py), so t carries a bias toward zero of ~ulp(|partial sums|)/2; at TAXI's
// scale (sigma = 1, |t| ~ 12) K is +2.2e-7 high on average (SIMT path: -4e-8), elsewhere
// -7e-8 (the ex2.approx bias).  A 3-piece bias fold was tried: no gain (the bias is the
// accumulation's, not the fold's).
//
// CTA structure (1 CTA per SM, 256 threads):
//   warp 0      TMA producer: the CTA's 128 P rows once (all K, resident in smem), then the
//               Q tiles (256 rows x 64 fp16 per box) through a 4-stage mbarrier ring;
//   warp 1      MMA issuer (one thread): per Q tile 3*d16/16 tcgen05.mma M=128,N=256,K=16
//               into one of two TMEM accumulators (2 x 256 columns, double-buffered);
//   warp 2      TMEM allocator;
//   warps 4-7   epilogue: thread i owns P row i (TMEM lane i), tcgen05.ld 32 columns at a
//               time, exp2 + contraction in registers, fp32 per tile -> fp64 per CTA.
// Q ranges are split across CTAs (blockIdx.y) with a deterministic fp64 reduction.
#include <cuda.h>
#include <cuda_fp16.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tcgen05.cuh"

namespace falkon {

constexpr int TC_M = 128;
constexpr int TC_N = 256;                         // Q rows per tile, shared-memory A (SS)
constexpr int TC_N_TS = 192;                      // Q rows per tile, A in TMEM (TS)
constexpr int TC_BK = 64;                          // fp16 per K box (128 B = one swizzle row)
#ifndef FALKON_SBK
#define FALKON_SBK 32
#endif
// streaming kernel: fp16 per K box (32: 64 B rows, SWIZZLE_64B, 48 KB stages; 64: 128 B rows,
// SWIZZLE_128B, half the TMA row requests per byte)
constexpr int TC_SBK = FALKON_SBK;
static_assert(TC_SBK == 32 || TC_SBK == 64, "streaming K box");
constexpr int TC_THREADS = 128 + 32 * 8;          // 4 control warps + 8 epilogue warps
constexpr int TC_SMEM_MAX = 227 * 1024;
constexpr int TC_A_BOX = TC_M * TC_BK * 2;         // 16 KB
constexpr int TC_B_BOX = TC_N * TC_BK * 2;         // 32 KB
constexpr int TC_MAX_D16 = 192;                    // A (all K) resident: 128 x 2*d16 fp16 <= 96 KB
constexpr double TC_LOG2E = 1.4426950408889634;

int reduce_partials(falkon_ctx *ctx, const double *part, int64_t splits, int64_t np,
                    double *out64, float *out32);
int center_mean(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, double **mu_out);

constexpr int TC_BIAS_SLOTS = 2;  // spare K slots per segment carrying the folded bias
static inline int tc_d16(int64_t d) { return (int)round_up<int64_t>(d + TC_BIAS_SLOTS, 16); }
// segment length of the packed [h | l] row: 16-aligned when the P tile stays resident in
// shared memory (2 * d16 <= 384), else 32-aligned for the streaming kernel (32-wide K boxes)
static inline bool tc_stream(int64_t d) { return tc_d16(d) > TC_MAX_D16; }
static inline int tc_seg(int64_t d) {
  return tc_stream(d) ? (int)round_up<int64_t>(d + TC_BIAS_SLOTS, TC_SBK) : tc_d16(d);
}
// TS (A operand in TMEM) needs 2 accumulators of TC_N_TS columns + 16 columns per d16/16
// chunk pair: 2*192 + 16*nk <= 512  <=>  d16 <= 128.
// Measured on B200 (MSD shape): TS is ~5% slower than SS — the MMA rate, not shared-memory
// bandwidth, binds — so it is opt-in (FALKON_TC_TS=1) and kept as a tested variant.
static bool tc_use_ts(int d16) {
  const char *e = getenv("FALKON_TC_TS");
  return e && atoi(e) != 0 && 2 * TC_N_TS + 16 * (d16 / 16) <= 512;
}

bool tc_supported(const falkon_ctx *ctx, int kernel, int64_t d) {
  if (kernel != FALKON_GAUSSIAN) return false;  // Laplacian: direct differences only (reading c7)
  if (ctx->opt.path == FALKON_PATH_SIMT || ctx->opt.path == FALKON_PATH_F64) return false;
  if (tc_seg(d) > 4096) return false;
  if (ctx->opt.path == FALKON_PATH_TENSOR) return true;
  return d > ctx->opt.tc_min_d;
}

// ------------------------------------------------------------------ packing
// One warp per row.  out row = [h_0..h_{d-1}, 1, 1, 0.. | l_0..l_{d-1}, (b-1)_hi, (b-1)_lo, 0..]
// Range guard: fp16 holds |x| < 65504; a scaled coordinate or folded bias at or above
// TC_FP16_SAFE sets *range_flag, and the caller falls back to the fp32 SIMT path.
constexpr double TC_FP16_SAFE = 32768.0;
__global__ void tc_pack_kernel(const float *__restrict__ in, int64_t rows, int64_t d,
                               const double *__restrict__ mu, double g, int d16,
                               __half *__restrict__ out, int *__restrict__ range_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double s = 0.0;
    for (int k = lane; k < d; k += 32) {
      const float x = (float)(((double)in[r * d + k] - mu[k]) * g);
      s += (double)x * (double)x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double bm1 = -0.5 * s - 1.0;  // bias - 1 (the h.h slots add 2)
    bool bad = !(fabs(bm1) < TC_FP16_SAFE);  // also catches NaN / inf inputs
    for (int k = lane; k < d; k += 32)
      bad |= !(fabs(((double)in[r * d + k] - mu[k]) * g) < TC_FP16_SAFE);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(range_flag, 1);
    const __half bh = __double2half(bm1);
    const __half bl = __double2half(bm1 - (double)__half2float(bh));
    __half *o = out + r * (int64_t)(2 * d16);
    for (int k = lane; k < d16; k += 32) {
      __half h, l;
      if (k < d) {
        const float x = (float)(((double)in[r * d + k] - mu[k]) * g);
        h = __float2half_rn(x);
        l = __float2half_rn(x - __half2float(h));
      } else if (k == d) {
        h = __float2half_rn(1.f);
        l = bh;
      } else if (k == d + 1) {
        h = __float2half_rn(1.f);
        l = bl;
      } else {
        h = __float2half_rn(0.f);
        l = h;
      }
      o[k] = h;
      o[d16 + k] = l;
    }
  }
}

// PTX wrappers (TMA, mbarrier, tcgen05 MMA / commit / TMEM loads): tcgen05.cuh

struct TcArgs {
  const float *z;
  const double *z64;  // ZD (ACCUM_F64): fp64 z instead of z
  int64_t np, nq, q_per_split;
  int nk;        // 16-wide K chunks per segment (d16 / 16)
  int nbox;      // 64-wide boxes covering one packed row (2*d16)
  int stages;    // depth of the Q-box ring
  double *out64;
  float *out32;
  int64_t p_base;  // first P row of this launch (TMA row coordinate offset; 0 = all rows)
  float *kst;      // single-evaluation strip: k values stored row-major [np][ldk] (or null)
  int64_t ldk;
  // fused strip GEMV (KST launches, warps 2-3): u (gacc, fp64 m) += previous strip^T w
  const float *gK;     // previous strip's k values (null: no fused GEMV)
  const void *gw;      // its rows' w (fp32, or fp64 when ZD)
  const float *gdw;    // GSC row weights (or null)
  int64_t grows, gm;   // rows of the previous strip, centres (= ldk)
  double *gacc;
  int gfirst;          // 1: overwrite gacc (first strip)
  int gslots;          // bulk-copy ring slots per GEMV warp
};

constexpr int TC_EPI_WARPS = 8;   // 2 per SM sub-partition: (TMEM lane group, column half)
constexpr int TC_MAX_STAGES = 8;

// exp2(x) for x <= 0 on the FMA pipe (FlashAttention-4-style MUFU offload): round-to-nearest
// split x = j + f (magic-number add), 2^f by a degree-5 near-minimax polynomial on
// [-0.5, 0.5] (max rel. error 2.3e-7 in fp32, same order as ex2.approx), 2^j by adding j to
// the exponent field.  x is clamped at -126 so the result stays normal.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;        // 1.5 * 2^23: low mantissa bits = round(x)
  const float r = t - 12582912.f;
  const float f = x - r;
  float p = 1.327646430581808e-3f;
  p = fmaf(p, f, 9.675540961325169e-3f);
  p = fmaf(p, f, 5.550713464617729e-2f);
  p = fmaf(p, f, 2.4022120237350464e-1f);
  p = fmaf(p, f, 6.931469440460205e-1f);
  p = fmaf(p, f, 1.0000001192092896f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Two entries of exp2_poly at once on the packed f32x2 pipe (FADD2/FFMA2: half the issue slots
// of the scalar form; per lane the same operations, so the same values as exp2_poly).  x <= 0.
__device__ __forceinline__ float2 exp2_poly2(float a, float b) {
  const float2 x = make_float2(fmaxf(a, -126.f), fmaxf(b, -126.f));
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);  // x - r, exact
  float2 p = make_float2(1.327646430581808e-3f, 1.327646430581808e-3f);
  p = __ffma2_rn(p, f, make_float2(9.675540961325169e-3f, 9.675540961325169e-3f));
  p = __ffma2_rn(p, f, make_float2(5.550713464617729e-2f, 5.550713464617729e-2f));
  p = __ffma2_rn(p, f, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = __ffma2_rn(p, f, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Epilogue modes (template): 0 = every exp2 on MUFU; 1 = all on the FMA pipe; 2 = one of
// four columns on the FMA pipe; 3 = two of four (2 and 3 evaluate their FMA-pipe entries in
// pairs, exp2_poly2); 8/9 = diagnostics (no exp / no TMEM read); 10/11 = no MMAs / no Q TMA;
// 12 = fault injection (a pipeline stage never fills: tests the trap of mbar_wait_safe).
template <int MODE>
__device__ __forceinline__ float tc_exp2(float t, int e) {
  t = fminf(t, 0.f);
  if (MODE == 1 || (MODE == 2 && e == 0) || (MODE == 3 && (e & 1) == 0)) return exp2_poly(t);
  if (MODE == 8) return t;
  return ex2_approx(t);
}

// 32 accumulator columns: k = exp2(min(t, 0)), acc += k * z (4 independent chains, 2 FFMA2).
// KST (single-evaluation strip): the 32 k values are also stored to kdst[j * TC_M], j < lim
// (the strip is column-major inside each 128-row tile, so each warp store is coalesced), and
// the second contraction reads them back instead of recomputing the cross term and the exp.
template <int MODE, bool MASK, bool KST = false>
__device__ __forceinline__ void tc_epi_chunk(const uint32_t (&r)[32], const float *__restrict__ z,
                                             int lim, float2 (&acc)[2], float *kdst = nullptr) {
  const float4 *zp = reinterpret_cast<const float4 *>(z);
  float kp[32];  // MODE 2/3: the FMA-pipe entries, evaluated in pairs
  if (MODE == 2 || MODE == 3) {
#pragma unroll
    for (int j = 0; j < 32; j += (MODE == 2 ? 8 : 4)) {
      const int j2 = MODE == 2 ? j + 4 : j + 2;  // (e 0 of groups g, g+1) / (e 0, e 2 of g)
      const float2 k2 = exp2_poly2(fminf(__uint_as_float(r[j]), 0.f), fminf(__uint_as_float(r[j2]), 0.f));
      kp[j] = k2.x;
      kp[j2] = k2.y;
    }
  }
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const float4 zz = __ldg(zp + g);
    float zv[4] = {zz.x, zz.y, zz.z, zz.w};
    float kv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = 4 * g + e;
      if (MASK && j >= lim) zv[e] = 0.f;
      if ((MODE == 2 && e == 0) || (MODE == 3 && (e & 1) == 0)) kv[e] = kp[j];
      else kv[e] = tc_exp2<(MODE == 2 || MODE == 3) ? 0 : MODE>(__uint_as_float(r[j]), e);
    }
    // chains e = 0..3 as two packed pairs (FFMA2: same per-lane fmaf, half the issue slots)
    acc[0] = __ffma2_rn(make_float2(kv[0], kv[1]), make_float2(zv[0], zv[1]), acc[0]);
    acc[1] = __ffma2_rn(make_float2(kv[2], kv[3]), make_float2(zv[2], zv[3]), acc[1]);
    if (KST) {  // column j of the tile: the warp's 32 rows are 128 contiguous bytes
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (!MASK || 4 * g + e < lim) __stcs(kdst + (4 * g + e) * TC_M, kv[e]);  // evict-first
    }
  }
}

// ACCUM_F64 epilogue (FALKON_OPT_ACCUM_F64): k = exp2(min(t, 0)) in fp32 on the MUFU as above,
// then acc[j & 3] += k * z_j by DFMA with fp64 z: the product of the fp32 kernel value and the
// fp64 vector entry is exact and the sum is fp64 (no fp32 rounding of z, w or partial sums;
// SURVEY.md §7 hard part 3).  KST: the fp32 k values are stored as in tc_epi_chunk.
__device__ __forceinline__ void ld256_f64(double (&v)[4], const double *p) {  // LDG.E.256
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
}
template <bool MASK, bool KST>
__device__ __forceinline__ void tc_epi_chunk_d(const uint32_t (&r)[32], const double *__restrict__ z,
                                               int lim, double (&acc)[4], float *kdst) {
  // one 256-bit load per 4 columns, issued one group ahead of its use (the loads' L1 latency
  // was the top stall: long scoreboard)
  double zc[4], zn[4];
  ld256_f64(zc, z);
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (g + 1 < 8) ld256_f64(zn, z + 4 * (g + 1));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = 4 * g + e;
      const double zv = (MASK && j >= lim) ? 0.0 : zc[e];
      const float k = ex2_approx(fminf(__uint_as_float(r[j]), 0.f));
      acc[e] = fma(k_to_f64(k), zv, acc[e]);
      if (KST && (!MASK || j < lim)) __stcs(kdst + j * TC_M, k);
    }
    if (g + 1 < 8) {
#pragma unroll
      for (int e = 0; e < 4; ++e) zc[e] = zn[e];
    }
  }
}

// one 32-column chunk c of the single-vector epilogue, fp32 (tc_epi_chunk) or fp64 (ZD) z
template <int MODE, bool MASK, bool KST, bool ZD>
__device__ __forceinline__ void tc_epi_any(const uint32_t (&r)[32], const float *zt,
                                           const double *ztd, int c, int lim, float2 (&acc)[2],
                                           double (&accd)[4], float *kdst) {
  if constexpr (ZD) tc_epi_chunk_d<MASK, KST>(r, ztd + c * 32, lim, accd, kdst);
  else tc_epi_chunk<MODE, MASK, KST>(r, zt + c * 32, lim, acc, kdst);
}

// Multi-vector epilogue (Kv for V in R^{q x KV}): 32 accumulator columns,
// k = exp2(min(t, 0)) once per entry, then acc[c] += k * z[j][c] for the KV vectors (z is
// [q][KV] fp32).  MASK: columns j >= lim are skipped (their z rows may be past the buffer).
__device__ __forceinline__ float4 lds128(const float *p) {  // explicit shared-memory load
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
template <bool MASK, int KV, bool SMEM = false>
__device__ __forceinline__ void tc_epi_chunk_kv(const uint32_t (&r)[32], const float *__restrict__ z,
                                                int lim, float2 (&acc)[KV > 1 ? KV / 2 : 1]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (MASK && j >= lim) break;
    const float k = ex2_approx(fminf(__uint_as_float(r[j]), 0.f));
    const float2 kk = make_float2(k, k);
    const float4 *zp = reinterpret_cast<const float4 *>(z + j * KV);
#pragma unroll
    for (int g = 0; g < KV / 4; ++g) {  // z in shared memory: LDS.128 broadcast per warp
      // smem (resident kernel: LDS, not a generic load) or global (streaming)
      const float4 zz = SMEM ? lds128(reinterpret_cast<const float *>(zp + g)) : zp[g];
      acc[2 * g] = __ffma2_rn(kk, make_float2(zz.x, zz.y), acc[2 * g]);
      acc[2 * g + 1] = __ffma2_rn(kk, make_float2(zz.z, zz.w), acc[2 * g + 1]);
    }
  }
}

__device__ __forceinline__ void tc_mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// smem (matrix descriptor) -> TMEM copy of one 128-row x 16-fp16 chunk (8 TMEM columns)
__device__ __forceinline__ void tc_cp_128x256b(uint32_t tmem_dst, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem_dst), "l"(sdesc));
}

// ------------------------------------------------------------------ strip GEMV pieces (NEXT-4)
constexpr int SE_WARPS = 8;
constexpr int SE_CPW = 8;                     // centres per warp
constexpr int SE_COLS = SE_WARPS * SE_CPW;    // centres per CTA
constexpr int SE_FLUSH = 32;                  // tiles per fp32 partial (4 x 32 = 128 terms)
// The rows' weights of one tile for lane l (rows r..r+3): w (fp32, or fp64 under WD) times the
// GSC row weights dw when dw != null (Knm^T D Knm, Alg. 2; as scale_rows_kernel); rows >= `rows`
// contribute 0.
__device__ __forceinline__ float4 gemv_w32(const float *__restrict__ w, const float *__restrict__ dw,
                                           int64_t r, int64_t rows) {
  float4 wv;
  if (r + 3 < rows) {
    wv = __ldg(reinterpret_cast<const float4 *>(w + r));
    if (dw) {
      const float4 dd = __ldg(reinterpret_cast<const float4 *>(dw + r));
      wv.x *= dd.x, wv.y *= dd.y, wv.z *= dd.z, wv.w *= dd.w;
    }
  } else {
    wv.x = r < rows ? w[r] * (dw ? dw[r] : 1.f) : 0.f;
    wv.y = r + 1 < rows ? w[r + 1] * (dw ? dw[r + 1] : 1.f) : 0.f;
    wv.z = r + 2 < rows ? w[r + 2] * (dw ? dw[r + 2] : 1.f) : 0.f;
    wv.w = 0.f;
  }
  return wv;
}
__device__ __forceinline__ double4 gemv_w64(const double *__restrict__ wd, const float *__restrict__ dw,
                                            int64_t r, int64_t rows) {
  const double2 wa = __ldg(reinterpret_cast<const double2 *>(wd + r));  // zero-padded to the tile
  const double2 wb = __ldg(reinterpret_cast<const double2 *>(wd + r + 2));
  double4 w4;
  w4.x = r < rows ? wa.x : 0.0;
  w4.y = r + 1 < rows ? wa.y : 0.0;
  w4.z = r + 2 < rows ? wb.x : 0.0;
  w4.w = r + 3 < rows ? wb.y : 0.0;
  if (dw) {
    w4.x *= r < rows ? (double)dw[r] : 0.0;
    w4.y *= r + 1 < rows ? (double)dw[r + 1] : 0.0;
    w4.z *= r + 2 < rows ? (double)dw[r + 2] : 0.0;
    w4.w *= r + 3 < rows ? (double)dw[r + 3] : 0.0;
  }
  return w4;
}

// One warp's share of u += strip^T w: the SE_CPW centres jb.. (clamped to m - 1; duplicates are
// discarded by the caller) over the strip's tiles [t0, t1).  Lane l reads the centre's 128
// values of a tile as one 512-byte float4 load and multiplies them by w of rows 4l..4l+3.
// PF: the next tile's loads are issued before this tile's FMAs (two tiles in flight; the
// standalone kernel; the fused warps share the pass-A kernel's register budget and do not).
// fp32 sums of <= 128 terms are flushed into fp64 (reading c12); WD: fp64 w, exact products by
// DFMA.  Returns, in lane c < SE_CPW, the fp64 sum of centre jb + c (fixed order).
template <bool WD, bool PF>
__device__ __forceinline__ double strip_gemv_group(const float *__restrict__ K, int64_t ldk,
                                                   const void *__restrict__ wv,
                                                   const float *__restrict__ dw, int64_t rows,
                                                   int64_t t0, int64_t t1, int64_t m, int64_t jb,
                                                   int lane) {
  const float *w = reinterpret_cast<const float *>(wv);
  const double *wd = reinterpret_cast<const double *>(wv);
  int jc[SE_CPW];  // centre offsets (m < 2^31)
#pragma unroll
  for (int c = 0; c < SE_CPW; ++c) jc[c] = (int)lmin(jb + c, m - 1) * TC_M;
  double a64[SE_CPW];
  float a32[SE_CPW];
#pragma unroll
  for (int c = 0; c < SE_CPW; ++c) a64[c] = 0.0, a32[c] = 0.f;
  float4 kq[SE_CPW];
  if (PF && t0 < t1) {
    const float *kt = K + t0 * ldk * TC_M + 4 * lane;
#pragma unroll
    for (int c = 0; c < SE_CPW; ++c) kq[c] = __ldcs(reinterpret_cast<const float4 *>(kt + jc[c]));
  }
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t r = t * TC_M + 4 * lane;
    float4 kn[SE_CPW];
    if (PF) {
      if (t + 1 < t1) {  // prefetch the next tile
        const float *kt = K + (t + 1) * ldk * TC_M + 4 * lane;
#pragma unroll
        for (int c = 0; c < SE_CPW; ++c) kn[c] = __ldcs(reinterpret_cast<const float4 *>(kt + jc[c]));
      }
    } else {
      const float *kt = K + t * ldk * TC_M + 4 * lane;
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) kq[c] = __ldcs(reinterpret_cast<const float4 *>(kt + jc[c]));
    }
    if (WD) {
      const double4 w4 = gemv_w64(wd, dw, r, rows);
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) {
        double s = a64[c];
        s = fma(k_to_f64(kq[c].x), w4.x, s);
        s = fma(k_to_f64(kq[c].y), w4.y, s);
        s = fma(k_to_f64(kq[c].z), w4.z, s);
        a64[c] = fma(k_to_f64(kq[c].w), w4.w, s);
      }
    } else {
      const float4 w4 = gemv_w32(w, dw, r, rows);
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) {
        float s = a32[c];
        s = fmaf(kq[c].x, w4.x, s);
        s = fmaf(kq[c].y, w4.y, s);
        s = fmaf(kq[c].z, w4.z, s);
        a32[c] = fmaf(kq[c].w, w4.w, s);
      }
      if ((t - t0) % SE_FLUSH == SE_FLUSH - 1) {
#pragma unroll
        for (int c = 0; c < SE_CPW; ++c) a64[c] += (double)a32[c], a32[c] = 0.f;
      }
    }
    if (PF && t + 1 < t1) {
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) kq[c] = kn[c];
    }
  }
  double out = 0.0;
#pragma unroll
  for (int c = 0; c < SE_CPW; ++c) {
    double v = a64[c] + (double)a32[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == c) out = v;
  }
  return out;
}

// Standalone strip GEMV: grid (centre blocks of SE_COLS) x (tile splits); one fp64 accumulator
// row per split (first: overwrite, else add).  No atomics: deterministic.
template <bool WEIGHTED, bool WD = false>
__global__ void __launch_bounds__(32 * SE_WARPS) se_gemv_kernel(const float *__restrict__ K, int64_t ldk,
                                                                const void *__restrict__ wv,
                                                                const float *__restrict__ dw, int64_t rows,
                                                                int64_t tiles_per_split, int64_t m,
                                                                double *__restrict__ acc, int first) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t jb = (int64_t)blockIdx.x * SE_COLS + warp * SE_CPW;
  if (jb >= m) return;
  const int64_t ntile = cdiv<int64_t>(rows, TC_M);
  const int64_t t0 = (int64_t)blockIdx.y * tiles_per_split;
  const int64_t t1 = lmin(ntile, t0 + tiles_per_split);
  const double v = strip_gemv_group<WD, true>(K, ldk, wv, WEIGHTED ? dw : nullptr, rows, t0, t1, m,
                                              jb, lane);
  const int64_t j = jb + lane;
  if (lane < SE_CPW && j < m) {
    double *o = acc + (int64_t)blockIdx.y * m + j;
    *o = first ? v : *o + v;
  }
}

// Split-SM strip GEMV (opt-in FALKON_OPT_SE_GEMV_SMS = G): a persistent grid of G CTAs streams
// strip s while pass A of strip s + 1 runs on the other SMs (second stream, highest priority, so
// the GEMV's CTAs take the first SMs pass A's CTAs release).  One 768-thread CTA per SM (its
// shared-memory claim keeps pass-A CTAs off the SM); every warp loops over centre groups of
// SE_CPW (strip_gemv_group: one writer per u_j, fixed order) with one tile's loads in flight per
// lane (8 x 16 B), 96 KB per SM.  Measured alone: 95 GB/s per SM on 16 SMs (the standalone GEMV
// is HBM-bound at 44 GB/s per SM on 148); beside pass A the schedule loses to the serial one
// (TIMIT 352-389 ms vs 314 ms per product, profiles/r2_split_sm_gemv.jsonl): the GEMV on G SMs
// drops to ~72 GB/s per SM and pass A loses more than its share of SMs.
constexpr int BL_WARPS = 24;
constexpr int BL_SMEM = 160 * 1024;
template <bool WEIGHTED, bool WD>
__global__ void __launch_bounds__(32 * BL_WARPS, 1)
    se_gemv_ldg_kernel(const float *__restrict__ K, int64_t m, const void *__restrict__ wv,
                       const float *__restrict__ dw, int64_t rows, double *__restrict__ acc,
                       int first) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntile = cdiv<int64_t>(rows, TC_M);
  const int64_t ng = cdiv<int64_t>(m, SE_CPW);
  for (int64_t g = (int64_t)blockIdx.x * BL_WARPS + wid; g < ng; g += (int64_t)gridDim.x * BL_WARPS) {
    const int64_t jb = g * SE_CPW;
    const double v = strip_gemv_group<WD, false>(K, m, wv, WEIGHTED ? dw : nullptr, rows, 0, ntile,
                                                 m, jb, lane);
    const int64_t j = jb + lane;
    if (lane < SE_CPW && j < m) acc[j] = first ? v : acc[j] + v;
  }
}

// Fused strip GEMV (warps 2 and 3 of a single-evaluation pass-A CTA, idle otherwise): while
// the tensor pipe evaluates strip s, these warps stream strip s - 1 (the other k buffer) from
// HBM.  The launch's CTAs partition the centres: CTA c owns centre groups [c G / N, (c+1) G / N)
// of SE_CPW centres over ALL tiles of the previous strip, so every u_j has one writer.
// The warps hold no loads in registers: lane 0 keeps FG_SLOTS bulk copies (TMA engine, one
// 4 KB k block [8 centres][128 rows] + the tile's w per slot) in flight into a shared-memory
// ring per warp, and the warp consumes a slot with LDS once its mbarrier completes (the
// register-staged loop reached only ~1.1 TB/s beside pass A: too few bytes in flight).
constexpr int FG_MAX_SLOTS = 8;                      // ring slots per GEMV warp (at most)
constexpr int FG_KB = SE_CPW * TC_M * 4;             // 4 KB of k per slot
constexpr int FG_SLOT = FG_KB + TC_M * 8;            // + w of the tile (fp64 room)
static inline int fg_ring_bytes(int slots) { return 128 + 128 + 2 * slots * FG_SLOT; }
template <bool WD>
__device__ __forceinline__ void fused_strip_gemv(const TcArgs &a, int wid, int lane,
                                                 uint8_t *ring_base) {
  const int FG_SLOTS = a.gslots;
  uint64_t *bar = reinterpret_cast<uint64_t *>(ring_base) + wid * FG_MAX_SLOTS;
  uint8_t *ring = ring_base + 128 + wid * FG_SLOTS * FG_SLOT;
  const int64_t nct = (int64_t)gridDim.x * gridDim.y;
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int64_t ng = cdiv<int64_t>(a.gm, SE_CPW);
  const int64_t g0 = cta * ng / nct, g1 = (cta + 1) * ng / nct;
  const int64_t ntile = cdiv<int64_t>(a.grows, TC_M);
  const int wb = WD ? 8 : 4;  // bytes per w element
  // this warp's items: (group g, tile t) for g = g0 + wid, g0 + wid + 2, ... and all t
  const int64_t my_groups = g1 > g0 + wid ? (g1 - g0 - wid + 1) / 2 : 0;
  const int64_t nitems = my_groups * ntile;
  if (nitems == 0) return;
  if (lane == 0)
    for (int s = 0; s < FG_SLOTS; ++s) mbar_init(&bar[s], 1);
  fence_mbar_init();
  __syncwarp();
  auto issue = [&](int64_t it) {  // lane 0
    const int64_t g = g0 + wid + 2 * (it / ntile), t = it % ntile;
    const int64_t jb = g * SE_CPW;
    const int s = (int)(it % FG_SLOTS);
    const uint32_t kb = (uint32_t)(lmin(SE_CPW, a.gm - jb) * TC_M * 4);
    const uint32_t wbytes = (uint32_t)(TC_M * wb);  // w rows are zero-padded past the strip
    mbar_expect_tx(&bar[s], kb + wbytes);
    bulk_g2s(ring + s * FG_SLOT, a.gK + (t * a.gm + jb) * TC_M, kb, &bar[s]);
    bulk_g2s(ring + s * FG_SLOT + FG_KB, (const uint8_t *)a.gw + t * TC_M * wb, wbytes, &bar[s]);
  };
  if (lane == 0)
    for (int64_t it = 0; it < lmin(FG_SLOTS, nitems); ++it) issue(it);
  double a64[SE_CPW];
  float a32[SE_CPW];
  for (int64_t it = 0; it < nitems; ++it) {
    const int64_t t = it % ntile;
    const int64_t jb = (g0 + wid + 2 * (it / ntile)) * SE_CPW;
    if (t == 0) {
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) a64[c] = 0.0, a32[c] = 0.f;
    }
    const int s = (int)(it % FG_SLOTS);
    mbar_wait_safe(&bar[s], (uint32_t)((it / FG_SLOTS) & 1));
    const uint8_t *slot = ring + s * FG_SLOT;
    const int nval = (int)lmin(SE_CPW, a.gm - jb);  // valid centres in this block
    const int64_t r = t * TC_M + 4 * lane;
    float4 kq[SE_CPW];
#pragma unroll
    for (int c = 0; c < SE_CPW; ++c)
      kq[c] = c < nval ? lds128(reinterpret_cast<const float *>(slot) + c * TC_M + 4 * lane)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    if (WD) {
      const double *ws = reinterpret_cast<const double *>(slot + FG_KB) + 4 * lane;
      double4 w4;
      w4.x = r < a.grows ? ws[0] : 0.0;
      w4.y = r + 1 < a.grows ? ws[1] : 0.0;
      w4.z = r + 2 < a.grows ? ws[2] : 0.0;
      w4.w = r + 3 < a.grows ? ws[3] : 0.0;
      if (a.gdw) {
        w4.x *= r < a.grows ? (double)a.gdw[r] : 0.0;
        w4.y *= r + 1 < a.grows ? (double)a.gdw[r + 1] : 0.0;
        w4.z *= r + 2 < a.grows ? (double)a.gdw[r + 2] : 0.0;
        w4.w *= r + 3 < a.grows ? (double)a.gdw[r + 3] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) {
        double acc = a64[c];
        acc = fma(k_to_f64(kq[c].x), w4.x, acc);
        acc = fma(k_to_f64(kq[c].y), w4.y, acc);
        acc = fma(k_to_f64(kq[c].z), w4.z, acc);
        a64[c] = fma(k_to_f64(kq[c].w), w4.w, acc);
      }
    } else {
      float4 w4 = lds128(reinterpret_cast<const float *>(slot + FG_KB) + 4 * lane);
      w4.x = r < a.grows ? w4.x : 0.f;
      w4.y = r + 1 < a.grows ? w4.y : 0.f;
      w4.z = r + 2 < a.grows ? w4.z : 0.f;
      w4.w = r + 3 < a.grows ? w4.w : 0.f;
      if (a.gdw) {
        w4.x *= r < a.grows ? a.gdw[r] : 0.f;
        w4.y *= r + 1 < a.grows ? a.gdw[r + 1] : 0.f;
        w4.z *= r + 2 < a.grows ? a.gdw[r + 2] : 0.f;
        w4.w *= r + 3 < a.grows ? a.gdw[r + 3] : 0.f;
      }
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) {
        float acc = a32[c];
        acc = fmaf(kq[c].x, w4.x, acc);
        acc = fmaf(kq[c].y, w4.y, acc);
        acc = fmaf(kq[c].z, w4.z, acc);
        a32[c] = fmaf(kq[c].w, w4.w, acc);
      }
      if (t % SE_FLUSH == SE_FLUSH - 1) {
#pragma unroll
        for (int c = 0; c < SE_CPW; ++c) a64[c] += (double)a32[c], a32[c] = 0.f;
      }
    }
    // the slot's values are consumed (used by the FMAs above): refill it
    __syncwarp();
    if (lane == 0 && it + FG_SLOTS < nitems) issue(it + FG_SLOTS);
    if (t == ntile - 1) {  // group done: fixed-order warp reduction, one writer per centre
      double out = 0.0;
#pragma unroll
      for (int c = 0; c < SE_CPW; ++c) {
        double v = a64[c] + (double)a32[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == c) out = v;
      }
      const int64_t j = jb + lane;
      if (lane < SE_CPW && j < a.gm) a.gacc[j] = a.gfirst ? out : a.gacc[j] + out;
    }
  }
}

// NT: Q rows per MMA tile (accumulator columns).  TS: the resident P tile is copied once
// into TMEM and used as the MMA's A operand (shared memory then only feeds B).
// STREAM: large d (2*d16 > 384): the P tile cannot stay resident, so each pipeline stage
// carries the matching 64-wide K box of BOTH segments of P and Q ([h|l] layout with
// 64-aligned segments): 16 + 16 + 32 + 32 KB, three MMAs per 16-wide chunk.
// CL = 2: clusters of two CTAs on consecutive P tiles (same Q range): each CTA loads one
// 128-row half of every Q box and multicasts it to both, halving the L2 -> SM traffic of the
// streamed operand; a stage is refilled only after BOTH CTAs' MMAs have released it (empty
// barriers count CL arrivals, commits are multicast).
// PAIR (STREAM, CL = 2): the two CTAs of a cluster run ONE tcgen05.mma.cta_group::2 of M = 256
// (each CTA's 128 P rows) x N = 256: each CTA stages only its own P rows and ITS HALF of the Q
// box (32 KB stages instead of 48 KB: deeper ring, more bytes in flight); the leader (rank 0)
// waits for both halves on its full barrier (the peer's TMA completes there), issues the MMAs
// and commits to both CTAs' empty / tfull barriers; both CTAs' epilogues release the
// accumulator on the leader's tempty barrier.
template <int MODE, int NT, bool TS, bool STREAM = false, int EPIW = TC_EPI_WARPS, int KV = 1,
          bool KST = false, int CL = 1, bool ZD = false, bool PAIR = false>
__global__ void __launch_bounds__(128 + 32 * EPIW, 1)
    tc_kvp_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                  TcArgs a) {
  static_assert(!(TS && STREAM), "TS needs the resident P tile");
  constexpr int SBK = STREAM ? TC_SBK : TC_BK;     // K width of the streamed boxes
  constexpr int SA_BOX = TC_M * SBK * 2;             // streaming: one P box (8 KB)
  constexpr int SQ_BOX = NT * SBK * 2;               // streaming: one Q box (16 KB)
  static_assert(!PAIR || (CL == 2 && NT == 2 * TC_M && KV == 1 && !TS), "pair MMA shape");
  // stage bytes; PAIR: this CTA's P boxes (streaming) and its 128-row half of the Q box
  constexpr int BBOX = PAIR ? (STREAM ? 4 * SA_BOX : TC_A_BOX)
                            : (STREAM ? 2 * (SA_BOX + SQ_BOX) : NT * TC_BK * 2);
  constexpr int GRP = EPIW / 4;          // column groups (epilogue warps per TMEM lane group)
  constexpr int HALF = NT / GRP;         // columns per epilogue warp
  constexpr int NCH = HALF / 32;         // 32-column chunks per epilogue warp
  static_assert(HALF % 32 == 0 && EPIW % 4 == 0, "tile");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages;
  uint8_t *sA = smem;                                  // nbox x 16 KB (resident P tile)
  uint8_t *sB = smem + (STREAM ? 0 : a.nbox * TC_A_BOX);  // S x BBOX
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + S * BBOX);
  uint64_t *full = bars, *empty = bars + TC_MAX_STAGES, *tfull = bars + 2 * TC_MAX_STAGES,
           *tempty = tfull + 2, *afull = tempty + 2, *zfull = afull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(zfull + 2);
  // [TC_M] fp64 half-row partials, 16-B aligned: the kv epilogue's z staging buffer that
  // follows is accessed as float4 / bulk-copy target (bars + slot end at byte 200 of the
  // 256-byte region)
  double *red = reinterpret_cast<double *>(
      (reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) & ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)blockIdx.x * TC_M;
  const int64_t qlo = (int64_t)blockIdx.y * a.q_per_split;
  const int64_t qhi = lmin(a.nq, qlo + a.q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, NT) : 0;
  const int nchunk = 2 * a.nk;  // valid 16-wide chunks of a packed row

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PAIR ? 1 : CL);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 2 * EPIW : EPIW);
    }
    mbar_init(afull, 1);
    mbar_init(&zfull[0], 1);
    mbar_init(&zfull[1], 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // partner's barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t crank = CL > 1 ? cluster_rank() : 0;
  constexpr uint16_t CMASK = (uint16_t)((1u << CL) - 1);
  const uint32_t tmem_a = tmem + 2 * NT;  // TS: P tile columns (8 per 16-wide chunk)

  if (warp == 0) {
    // TMA producer: the whole warp walks the ring, one elected lane issues the copies
    if (!STREAM && elect_one()) {
      if (PAIR) {  // both CTAs' P tiles complete on the leader's afull (its MMAs read both)
        if (crank == 0) mbar_expect_tx(afull, (uint32_t)(2 * a.nbox * TC_A_BOX));
        for (int b = 0; b < a.nbox; ++b)
          tma_load_2d_pair(sA + b * TC_A_BOX, &tmP, b * TC_BK, (int)(a.p_base + p0), afull);
      } else {
        mbar_expect_tx(afull, (uint32_t)(a.nbox * TC_A_BOX));
        for (int b = 0; b < a.nbox; ++b) tma_load_2d(sA + b * TC_A_BOX, &tmP, b * TC_BK, (int)(a.p_base + p0), afull);
      }
    }
    __syncwarp();
    const int segk = a.nk * 16;  // STREAM: elements per segment
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int q0 = (int)(qlo + (int64_t)t * NT);
      if (KV > 1 && !STREAM) {
        // the tile's z block ([NT][KV] fp32, contiguous) into z buffer t & 1 by one bulk copy,
        // once the epilogue has released tile t - 2 (the tempty phase the MMA warp also waits on)
        mbar_wait_safe(&tempty[t & 1], ((t >> 1) & 1) ^ 1);
        if (elect_one()) {
          float *zsm = reinterpret_cast<float *>(red + (size_t)TC_M * (KV > 3 ? KV : 3));
          const uint32_t bytes = (uint32_t)(lmin(NT, a.nq - q0) * KV * 4);
          mbar_expect_tx(&zfull[t & 1], bytes);
          bulk_g2s(zsm + (t & 1) * NT * KV, a.z + (int64_t)q0 * KV, bytes, &zfull[t & 1]);
        }
        __syncwarp();
      }
      for (int b = 0; b < a.nbox; ++b) {
        mbar_wait_safe(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if (MODE == 11) {  // diagnostic: no Q loads
            mbar_arrive(&full[stage]);
          } else if (MODE == 12) {  // fault injection: the stage never fills (mbar_wait_safe traps)
          } else if (PAIR && !STREAM) {  // this CTA's 128-row half of the Q box
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * BBOX);
            tma_load_2d_pair(sB + stage * BBOX, &tmQ, b * TC_BK, q0 + (int)crank * TC_M, &full[stage]);
          } else if (PAIR) {
            // own P rows (h, l) and own 128-row half of the Q box (h, l) into this CTA's stage;
            // completions count on the leader's full barrier, which expects both CTAs' boxes
            uint8_t *st = sB + stage * BBOX;
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * BBOX);
            const int pr = (int)(a.p_base + p0), qh = q0 + (int)crank * TC_M;
            tma_load_2d_pair(st, &tmP, b * SBK, pr, &full[stage]);                  // h_p
            tma_load_2d_pair(st + SA_BOX, &tmP, segk + b * SBK, pr, &full[stage]);  // l_p
            tma_load_2d_pair(st + 2 * SA_BOX, &tmQ, b * SBK, qh, &full[stage]);         // h_q half
            tma_load_2d_pair(st + 3 * SA_BOX, &tmQ, segk + b * SBK, qh, &full[stage]);  // l_q half
          } else if (STREAM) {
            uint8_t *st = sB + stage * BBOX;
            mbar_expect_tx(&full[stage], BBOX);
            tma_load_2d(st, &tmP, b * SBK, (int)(a.p_base + p0), &full[stage]);          // h_p
            tma_load_2d(st + SA_BOX, &tmP, segk + b * SBK, (int)(a.p_base + p0),
                        &full[stage]);  // l_p
            if (CL == 1) {
              tma_load_2d(st + 2 * SA_BOX, &tmQ, b * SBK, q0, &full[stage]);             // h_q
              tma_load_2d(st + 2 * SA_BOX + SQ_BOX, &tmQ, segk + b * SBK, q0,
                          &full[stage]);                                                 // l_q
            } else {  // this CTA's 128-row half of h_q and l_q, multicast to the cluster
              const int qh = q0 + (int)crank * TC_M;
              const uint32_t ho = crank * SA_BOX;
              tma_load_2d_mc(st + 2 * SA_BOX + ho, &tmQ, b * SBK, qh, &full[stage], CMASK);
              tma_load_2d_mc(st + 2 * SA_BOX + SQ_BOX + ho, &tmQ, segk + b * SBK, qh,
                             &full[stage], CMASK);
            }
          } else {
            mbar_expect_tx(&full[stage], BBOX);
            if (CL == 1)
              tma_load_2d(sB + stage * BBOX, &tmQ, b * TC_BK, q0, &full[stage]);
            else
              tma_load_2d_mc(sB + stage * BBOX + crank * TC_A_BOX, &tmQ, b * TC_BK,
                             q0 + (int)crank * TC_M, &full[stage], CMASK);
          }
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && !(PAIR && crank != 0)) {
    // MMA issuer: warp-uniform control flow, one elected lane issues tcgen05.mma.  The
    // descriptors are linear in the shared-memory address (start address in the low bits),
    // so chunk / stage offsets are plain integer adds on precomputed bases.  PAIR: the
    // leader's warp issues M = 256 MMAs for the CTA pair; the peer's warp 1 idles.
    const uint32_t idesc = (1u << 4) | ((uint32_t)(NT >> 3) << 17) |
                           ((uint32_t)((PAIR ? 2 : 1) * TC_M >> 4) << 24);
    const uint64_t a0 = sw128_desc(smem_u32(sA));
    const uint64_t b0 = (STREAM && TC_SBK == 32) ? sw64_desc(smem_u32(sB)) : sw128_desc(smem_u32(sB));
    const int nk = a.nk;
    auto adesc = [&](int c) -> uint64_t {
      return a0 + (uint64_t)(((c >> 2) * TC_A_BOX + (c & 3) * 32) >> 4);
    };
    if (!STREAM) mbar_wait_safe(afull, 0);
    tc_fence_after();
    if (TS) {
      if (elect_one())
        for (int c = 0; c < nchunk; ++c) tc_cp_128x256b(tmem_a + (uint32_t)(8 * c), adesc(c));
      __syncwarp();
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      mbar_wait_safe(&tempty[acc], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dtm = tmem + (uint32_t)(acc * NT);
      for (int b = 0; b < a.nbox; ++b) {
        mbar_wait_safe(&full[stage], phase);
        tc_fence_after();
        if (PAIR && STREAM && elect_one()) {
          const uint64_t ah = b0 + (uint64_t)((stage * BBOX) >> 4);
          const uint64_t al = ah + (uint64_t)(SA_BOX >> 4);
          const uint64_t bh = ah + (uint64_t)((2 * SA_BOX) >> 4);
          const uint64_t bl = ah + (uint64_t)((3 * SA_BOX) >> 4);
#pragma unroll
          for (int jj = 0; jj < SBK / 16; ++jj) {
            if (b * (SBK / 16) + jj < nk) {
              const uint64_t o = (uint64_t)(jj * 2);  // +32 B within the 64 B swizzle row
              tc_mma_f16_pair(dtm, ah + o, bh + o, idesc, (b | jj) ? 1u : 0u);  // h_p . h_q
              tc_mma_f16_pair(dtm, al + o, bh + o, idesc, 1u);                  // l_p . h_q
              tc_mma_f16_pair(dtm, ah + o, bl + o, idesc, 1u);                  // h_p . l_q
            }
          }
          tc_commit_pair(&empty[stage]);
        } else if (STREAM && !PAIR && elect_one()) {
          const uint64_t ah = b0 + (uint64_t)((stage * BBOX) >> 4);
          const uint64_t al = ah + (uint64_t)(SA_BOX >> 4);
          const uint64_t bh = ah + (uint64_t)((2 * SA_BOX) >> 4);
          const uint64_t bl = bh + (uint64_t)(SQ_BOX >> 4);
#pragma unroll
          for (int jj = 0; jj < SBK / 16; ++jj) {
            if (b * (SBK / 16) + jj < nk && MODE != 10) {
              const uint64_t o = (uint64_t)(jj * 2);  // +32 B within the 64 B swizzle row
              tc_mma_f16(dtm, ah + o, bh + o, idesc, (b | jj) ? 1u : 0u);  // h_p . h_q
              tc_mma_f16(dtm, al + o, bh + o, idesc, 1u);                  // l_p . h_q
              tc_mma_f16(dtm, ah + o, bl + o, idesc, 1u);                  // h_p . l_q
            }
          }
          if (CL == 1) tc_commit(&empty[stage]);
          else tc_commit_mc(&empty[stage], CMASK);
        } else if (!STREAM && elect_one()) {
          const uint64_t bs = b0 + (uint64_t)((stage * BBOX) >> 4);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int j = b * 4 + jj;  // chunk of the Q row held in this box
            if (j < nchunk && MODE != 10) {  // MODE 10: diagnostic without MMAs
              const uint64_t bd = bs + (uint64_t)(jj * 2);  // +32 B
              const int ca = j < nk ? j : j - nk;         // h_p chunk
              const uint32_t first = (b | jj) ? 1u : 0u;  // first MMA of the tile overwrites
              if (TS) tc_mma_f16_ts(dtm, tmem_a + (uint32_t)(8 * ca), bd, idesc, first);
              else if (PAIR) tc_mma_f16_pair(dtm, adesc(ca), bd, idesc, first);
              else tc_mma_f16(dtm, adesc(ca), bd, idesc, first);  // h_p . h_q | h_p . l_q
              if (j < nk) {                                        // l_p . h_q
                if (TS) tc_mma_f16_ts(dtm, tmem_a + (uint32_t)(8 * (nk + j)), bd, idesc, 1u);
                else if (PAIR) tc_mma_f16_pair(dtm, adesc(nk + j), bd, idesc, 1u);
                else tc_mma_f16(dtm, adesc(nk + j), bd, idesc, 1u);
              }
            }
          }
          if (PAIR) tc_commit_pair(&empty[stage]);
          else if (CL == 1) tc_commit(&empty[stage]);
          else tc_commit_mc(&empty[stage], CMASK);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) {
        if (PAIR) tc_commit_pair(&tfull[acc]);
        else tc_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else if (KST && KV == 1 && (warp == 2 || warp == 3)) {
    // fused strip GEMV of the previous strip (single evaluation): warp 2 has allocated TMEM
    // above and is otherwise idle until the dealloc at the end; warp 3 is idle
    if (a.gK) {
      uint8_t *gring = reinterpret_cast<uint8_t *>(
          (reinterpret_cast<uintptr_t>(red + TC_M * (KV > 3 ? KV : 3)) + 127) & ~uintptr_t(127));
      fused_strip_gemv<ZD>(a, warp - 2, lane, gring);
    }
  } else if (KV > 1 && warp >= 4) {
    // multi-vector epilogue: thread = P row; the Q tile's z block ([NT][KV] fp32) arrives in
    // shared memory by the producer's bulk copy (double-buffered, mbarrier per buffer), KV/2
    // packed FFMA2 chains per tile in fp32, then KV fp64 sums
    const int ew = warp - 4;
    const int lg = ew & 3;
    const int half = ew >> 2;
    const int row = lg * 32 + lane;
    const int64_t p = p0 + row;
    const int col0 = half * HALF;
    float *zsm = reinterpret_cast<float *>(red + (size_t)TC_M * (KV > 3 ? KV : 3));  // [2][NT][KV]
    double acc64[KV];
#pragma unroll
    for (int c = 0; c < KV; ++c) acc64[c] = 0.0;
    uint32_t rr[2][32];
    for (int t = 0; t < ntiles; ++t) {
      const int64_t q0 = qlo + (int64_t)t * NT;
      if (!STREAM)  // z block staged by the producer's bulk copy (streaming: read through L1)
        mbar_wait_safe(&zfull[t & 1], (t >> 1) & 1);
      const int accb = t & 1;
      mbar_wait_safe(&tfull[accb], (t >> 1) & 1);
      tc_fence_after();
      const int cnt = (int)lmin(NT, qhi - q0) - col0;
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(accb * NT + col0);
      const float *zt = STREAM ? a.z + (q0 + col0) * KV : zsm + (t & 1) * NT * KV + col0 * KV;
      float2 acc[KV > 1 ? KV / 2 : 1];
#pragma unroll
      for (int c = 0; c < KV / 2; ++c) acc[c] = make_float2(0.f, 0.f);
      if (cnt >= HALF) {
        tmem_ld32(tb, rr[0]);
        tmem_wait_ld_regs(rr[0]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c + 1 < NCH) tmem_ld32(tb + (uint32_t)((c + 1) * 32), rr[(c + 1) & 1]);
          tc_epi_chunk_kv<false, KV, !STREAM>(rr[c & 1], zt + c * 32 * KV, 32, acc);
          if (c + 1 < NCH) tmem_wait_ld_regs(rr[(c + 1) & 1]);
        }
      } else {
        for (int c = 0; c * 32 < cnt; ++c) {
          tmem_ld32(tb + (uint32_t)(c * 32), rr[0]);
          tmem_wait_ld_regs(rr[0]);
          tc_epi_chunk_kv<true, KV, !STREAM>(rr[0], zt + c * 32 * KV, cnt - c * 32, acc);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // PAIR: the leader's tempty collects both CTAs' epilogue warps
        if (PAIR && crank != 0) mbar_arrive_cluster(&tempty[accb], 0);
        else mbar_arrive(&tempty[accb]);
      }
#pragma unroll
      for (int c = 0; c < KV / 2; ++c) {
        acc64[2 * c] += (double)acc[c].x;
        acc64[2 * c + 1] += (double)acc[c].y;
      }
    }
    // combine the column groups of each row in a fixed order (deterministic)
    if (half > 0) {
#pragma unroll
      for (int c = 0; c < KV; ++c) red[((half - 1) * TC_M + row) * KV + c] = acc64[c];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EPIW) : "memory");
    if (half == 0 && p < a.np) {
#pragma unroll
      for (int c = 0; c < KV; ++c) {
        double tot = acc64[c];
        for (int g2 = 1; g2 < GRP; ++g2) tot += red[((g2 - 1) * TC_M + row) * KV + c];
        if (a.out64) a.out64[((int64_t)blockIdx.y * a.np + p) * KV + c] = tot;
        if (a.out32) a.out32[p * KV + c] = (float)tot;
      }
    }
  } else if (KV == 1 && warp >= 4) {
    const int ew = warp - 4;
    const int lg = ew & 3;        // TMEM lane group: warp % 4 == lg
    const int half = ew >> 2;     // column group of the accumulator
    const int row = lg * 32 + lane;
    const int64_t p = p0 + row;
    const int col0 = half * HALF;
    double acc64 = 0.0;
    double accd[4] = {0.0, 0.0, 0.0, 0.0};  // ZD: fp64 DFMA chains over the whole split
    uint32_t rr[2][32];
    for (int t = 0; t < ntiles; ++t) {
      const int accb = t & 1;
      mbar_wait_safe(&tfull[accb], (t >> 1) & 1);
      tc_fence_after();
      const int64_t q0 = qlo + (int64_t)t * NT;
      const int cnt = (int)lmin(NT, qhi - q0) - col0;  // valid columns of this half
      const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(accb * NT + col0);
      const float *zt = ZD ? nullptr : a.z + q0 + col0;
      const double *ztd = ZD ? a.z64 + q0 + col0 : nullptr;
      // KST: strip tile blockIdx.x, layout [tile][q][TC_M rows]; padding rows (p >= np) are
      // stored too (finite values; the GEMV weights them by w = 0)
      float *kd = KST ? a.kst + ((int64_t)blockIdx.x * a.ldk + q0 + col0) * TC_M + row : nullptr;
      const bool kok = p0 < a.np;  // a cluster's padding CTA (whole tile past the strip) stores nothing
      float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      if (KST) {
        const int cw = cnt < HALF ? cnt : HALF;  // this warp's columns
        if (cw == HALF) {  // software-pipelined as below
          tmem_ld32(tb, rr[0]);
          tmem_wait_ld_regs(rr[0]);
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            if (c + 1 < NCH) tmem_ld32(tb + (uint32_t)((c + 1) * 32), rr[(c + 1) & 1]);
            if (kok) tc_epi_any<MODE, false, true, ZD>(rr[c & 1], zt, ztd, c, 32, acc, accd, kd + c * 32 * TC_M);
            else tc_epi_any<MODE, false, false, ZD>(rr[c & 1], zt, ztd, c, 32, acc, accd, nullptr);
            if (c + 1 < NCH) tmem_wait_ld_regs(rr[(c + 1) & 1]);
          }
        } else {
          for (int c = 0; c * 32 < cw; ++c) {
            tmem_ld32(tb + (uint32_t)(c * 32), rr[0]);
            tmem_wait_ld_regs(rr[0]);
            if (kok) tc_epi_any<MODE, true, true, ZD>(rr[0], zt, ztd, c, cw - c * 32, acc, accd, kd + c * 32 * TC_M);
            else tc_epi_any<MODE, true, false, ZD>(rr[0], zt, ztd, c, cw - c * 32, acc, accd, nullptr);
          }
        }
      } else if (MODE == 9) {  // diagnostic: no TMEM traffic
#pragma unroll
        for (int j = 0; j < 32; ++j) rr[0][j] = __float_as_uint(-(float)j);
        for (int c = 0; c * 32 < cnt; ++c) tc_epi_chunk<0, true>(rr[0], zt + c * 32, cnt - c * 32, acc);
      } else if (cnt >= HALF) {
        // software-pipelined: the next 32 columns load from TMEM while these are processed
        tmem_ld32(tb, rr[0]);
        tmem_wait_ld_regs(rr[0]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (c + 1 < NCH) tmem_ld32(tb + (uint32_t)((c + 1) * 32), rr[(c + 1) & 1]);
          tc_epi_any<MODE, false, false, ZD>(rr[c & 1], zt, ztd, c, 32, acc, accd, nullptr);
          if (c + 1 < NCH) tmem_wait_ld_regs(rr[(c + 1) & 1]);
        }
      } else {
        for (int c = 0; c * 32 < cnt; ++c) {
          tmem_ld32(tb + (uint32_t)(c * 32), rr[0]);
          tmem_wait_ld_regs(rr[0]);
          tc_epi_any<MODE, true, false, ZD>(rr[0], zt, ztd, c, cnt - c * 32, acc, accd, nullptr);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // PAIR: the leader's tempty collects both CTAs' epilogue warps
        if (PAIR && crank != 0) mbar_arrive_cluster(&tempty[accb], 0);
        else mbar_arrive(&tempty[accb]);
      }
      if (!ZD) acc64 += (double)((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y));
    }
    if (ZD) acc64 = (accd[0] + accd[1]) + (accd[2] + accd[3]);
    // combine the column groups of each row in a fixed order (deterministic)
    if (half > 0) red[(half - 1) * TC_M + row] = acc64;
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EPIW) : "memory");
    if (half == 0 && p < a.np) {
      double tot = acc64;
#pragma unroll
      for (int g2 = 1; g2 < GRP; ++g2) tot += red[(g2 - 1) * TC_M + row];
      if (a.out64) a.out64[(int64_t)blockIdx.y * a.np + p] = tot;
      if (a.out32) a.out32[p] = (float)tot;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // the partner's last multicasts / commits into this CTA are done
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode() {
  static const PFN_encodeTiled_t fn = []() -> PFN_encodeTiled_t {  // thread-safe one-time lookup
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_encodeTiled_t)p;
    cudaGetLastError();
    return nullptr;
  }();
  return fn;
}

static int make_map(CUtensorMap *map, const __half *base, int64_t rows, int k_elems, int box_rows,
                    bool stream = false) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return fail(FALKON_EUNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)k_elems, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)k_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)(stream ? TC_SBK : TC_BK), (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void *)base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (stream && TC_SBK == 32) ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FALKON_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return FALKON_OK;
}

static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");

// Device int of the fp16 range guard (in the WS_FLAGS slot); reset = zero it (stream-ordered).
int tc_range_flag(falkon_ctx *ctx, int **flag, bool reset) {
  void *p;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64, &p));
  *flag = (int *)((char *)p + 32);  // bytes 0-15: the preconditioner's pivot-failure words
  if (reset) FK_CUDA(cudaMemsetAsync(*flag, 0, sizeof(int), ctx->stream));
  return FALKON_OK;
}
int tc_range_check(falkon_ctx *ctx, bool *bad) {
  int *flag, h = 0;
  FK_TRY(tc_range_flag(ctx, &flag, false));
  FK_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  *bad = h != 0;
  return FALKON_OK;
}

int tc_prepare(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C, int64_t m,
               double sigma, const double *mu, Prepared *pp) {
  const int d16 = tc_seg(d);
  const int kp = 2 * d16;
  const double g = std::sqrt(TC_LOG2E) / sigma;
  const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n, 1), TC_N);
  const int64_t m_pad = round_up<int64_t>(m, TC_N);
  void *xp, *cp;
  FK_TRY(ws_get(ctx, WS_XP, sizeof(__half) * n_pad * kp, &xp));
  FK_TRY(ws_get(ctx, WS_CP, sizeof(__half) * m_pad * kp, &cp));
  const int threads = 256;
  int *flag;
  FK_TRY(tc_range_flag(ctx, &flag, true));
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    const int64_t blocks = std::min<int64_t>(cdiv<int64_t>(m, threads / 32), 65535);
    tc_pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(C, m, d, mu, g, d16, (__half *)cp,
                                                                   flag);
  }
  FK_LAUNCH_CHECK();
  if (n > 0 && X) {
    LaunchScope ls(ctx, FALKON_T_PREP);
    const int64_t blocks = std::min<int64_t>(cdiv<int64_t>(n, threads / 32), (int64_t)ctx->sm_count * 64);
    tc_pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(X, n, d, mu, g, d16, (__half *)xp,
                                                                   flag);
    FK_LAUNCH_CHECK();
  }
  // range guard (one stream synchronisation per prepare): out of fp16 range -> the caller
  // re-prepares the operands for the fp32 SIMT path
  bool bad = false;
  FK_TRY(tc_range_check(ctx, &bad));
  if (bad) return FALKON_TC_RANGE;
  pp->mu = mu;
  pp->g = g;
  pp->dq = d16;
  pp->Xp = xp;
  pp->Cp = cp;
  pp->xa = nullptr;
  pp->cb = nullptr;
  CUtensorMap *maps = reinterpret_cast<CUtensorMap *>(pp->tmaps);
  const bool st = tc_stream(d);
  FK_TRY(make_map(&maps[0], (const __half *)xp, n, kp, TC_M, st));  // X as P (pass A)
  FK_TRY(make_map(&maps[1], (const __half *)cp, m, kp, TC_N, st));  // C as Q (pass A)
  FK_TRY(make_map(&maps[2], (const __half *)cp, m, kp, TC_M, st));  // C as P (pass B)
  FK_TRY(make_map(&maps[3], (const __half *)xp, n, kp, TC_N, st));  // X as Q (pass B)
  if (!st && tc_use_ts(d16)) {  // TS kernel (opt-in): Q boxes of TC_N_TS rows
    FK_TRY(make_map(&maps[4], (const __half *)cp, m, kp, TC_N_TS, st));
    FK_TRY(make_map(&maps[5], (const __half *)xp, n, kp, TC_N_TS, st));
  }
  return FALKON_OK;
}

// tail: fp64 row partials [TC_M][max(3, kv)] and (kv > 1) the z staging buffers [2][nt][kv] fp32
static size_t tc_tail_bytes(int nt, int kv, bool stream = false) {
  return (size_t)8 * TC_M * std::max(3, kv) + (kv > 1 && !stream ? (size_t)2 * nt * kv * 4 : 0);
}
static size_t tc_smem_bytes(int nbox, int stages, int nt, int kv = 1) {
  return 1024 + (size_t)nbox * TC_A_BOX + (size_t)stages * nt * TC_BK * 2 + 256 +
         tc_tail_bytes(nt, kv);
}
static int tc_stages(int nbox, int nt, int kv = 1) {
  int s = 8;
  while (s > 2 && tc_smem_bytes(nbox, s, nt, kv) > (size_t)TC_SMEM_MAX) --s;
  return s;
}


// Co-resident CTAs of a 2-CTA-cluster launch (2 x cudaOccupancyMaxActiveClusters; a GPC with
// an odd number of free SMs leaves one idle), cached per kernel.
static int64_t tc_cluster_slots(falkon_ctx *ctx, const void *fn, int threads, size_t smem) {
  for (int i = 0; i < falkon_ctx::NSLOTCACHE; ++i)  // per-context cache (contexts are independent)
    if (ctx->slot_fn[i] == fn && ctx->slot_n[i] > 0) return ctx->slot_n[i];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * ctx->sm_count);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) != cudaSuccess || nc <= 0) {
    cudaGetLastError();
    return ctx->sm_count;
  }
  const int64_t slots = 2 * (int64_t)nc;
  for (int i = 0; i < falkon_ctx::NSLOTCACHE; ++i)
    if (!ctx->slot_fn[i]) {
      ctx->slot_fn[i] = fn;
      ctx->slot_n[i] = slots;
      break;
    }
  return slots;
}

// One fused pass over P rows [p_begin, p_begin + p_count) (p_count < 0: all).  kst != null
// (pass A, kv = 1): the k values are also stored row-major into kst[(p - p_begin) * ldk + q].
// Fused GEMV of the previous strip (single evaluation; see fused_strip_gemv).
struct FusedGemv {
  const float *K = nullptr;  // previous strip's k values [tile][ldk][128]
  const void *w = nullptr;   // its rows' w (fp32, or fp64 with z64)
  const float *dw = nullptr;
  int64_t rows = 0;
  double *acc = nullptr;     // u (fp64 m)
  int first = 0;
};

// z64 != null: fp64 z and DFMA contractions (ACCUM_F64, kv 1, MODE 0); out64 is then required.
// fg (kst launches only): warps 2-3 also run the GEMV of the previous strip.
static int tc_launch(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z,
                     double *out64, float *out32, int kv, int64_t p_begin, int64_t p_count,
                     float *kst, int64_t ldk, const double *z64 = nullptr,
                     const FusedGemv *fg = nullptr) {
  const CUtensorMap *maps = reinterpret_cast<const CUtensorMap *>(pp.tmaps);
  const int d16 = pp.dq;
  const bool stream = tc_stream(pp.d);
  // resident: boxes of a whole packed row; streaming: boxes of one segment
  const int nbox = stream ? d16 / TC_SBK : (int)cdiv<int64_t>(2 * d16, TC_BK);
  const int64_t np = p_count >= 0 ? p_count : (passA ? pp.n : pp.m), nq = passA ? pp.m : pp.n;
  if (np <= 0) return FALKON_OK;
  if (kst && (!passA || kv != 1)) return fail(FALKON_EINVAL, "tc_launch: k strip needs pass A, kv 1");
  if (z64 && (kv != 1 || !out64)) return fail(FALKON_EINVAL, "tc_launch: fp64 z needs kv 1 and out64");
  // TS (opt-in, single vector, resident P, MODE 0 two-pass only): the same decision selects
  // the 192-row Q maps (maps[4], maps[5]) and the NT = 192 kernel
  const bool ts = kv == 1 && !stream && !kst && !z64 && tc_use_ts(d16);
  const int nt = ts ? TC_N_TS : TC_N;
  // CTA-pair MMA (cta_group::2) for the streaming kernel with 2-CTA clusters (default; measured
  // TIMIT single evaluation 355 -> 320 ms, two-pass 426 -> 407 ms per product,
  // profiles/r2_pair_ab.txt); FALKON_TC_PAIR=0 selects the multicast-only cluster kernel (A/B)
  const char *pe = getenv("FALKON_TC_PAIR");
  int mode = ctx->opt.exp_offload;
  if (const char *e = getenv("FALKON_TC_MODE")) mode = atoi(e);  // diagnostics (8-12)
  // resident-P kernels (d <= 190) keep the multicast clusters: the pair variant is correct but
  // slower there (MSD 21.4 -> 23.0 ms, HIGGS 576 -> 745 ms, TAXI 1337 -> 1810 ms per product:
  // the two CTAs' epilogues gate one shared accumulator pipeline), opt-in FALKON_TC_PAIR=2
  const int pv = pe ? atoi(pe) : 1;
  const bool pair = kv == 1 && ctx->opt.tc_cluster == 2 && pv != 0 && !ts &&
                    (stream || (pv == 2 && (mode == 0 || kst || z64)));
  const int nt_stage = (pair && !stream) ? TC_M : nt;  // resident pair: half-Q-box stages
  // streaming: stages of 48 KB (P and Q boxes of both segments, 32 wide) — 4 fit; a CTA of a
  // pair stages its P rows and its half of the Q box: 32 KB, 6 fit
  const size_t sstage = pair ? (size_t)4 * TC_M * TC_SBK * 2 : (size_t)2 * (TC_M + TC_N) * TC_SBK * 2;
  // single-evaluation launches reserve the fused GEMV's bulk-copy rings after the tail: at least
  // 3 slots per GEMV warp, the rest of shared memory beyond the pass-A ring (up to 8 slots)
  const bool fgr = kst && fg;  // fused GEMV in this launch
  const size_t gmin = fgr ? (size_t)fg_ring_bytes(3) : 0;
  int sst = TC_MAX_STAGES;
  while (sst > 2 && 1024 + sst * sstage + 256 + tc_tail_bytes(nt, kv, true) + gmin > (size_t)TC_SMEM_MAX) --sst;
  if (const char *e = getenv("FALKON_TC_SST")) sst = std::max(2, std::min(sst, atoi(e)));  // A/B
  int rst = tc_stages(nbox, nt_stage, kv);
  while (rst > 2 && tc_smem_bytes(nbox, rst, nt_stage, kv) + gmin > (size_t)TC_SMEM_MAX) --rst;
  const int stages = stream ? sst : rst;
  const size_t base = stream ? 1024 + (size_t)stages * sstage + 256 + tc_tail_bytes(nt, kv, true)
                             : tc_smem_bytes(nbox, stages, nt_stage, kv);
  int gslots = 0;
  if (fgr) {
    gslots = 3;
    while (gslots < FG_MAX_SLOTS && base + fg_ring_bytes(gslots + 1) <= (size_t)TC_SMEM_MAX) ++gslots;
  }
  const size_t smem = base + (fgr ? (size_t)fg_ring_bytes(gslots) : 0);
  if (smem > (size_t)TC_SMEM_MAX) return fail(FALKON_EUNSUPPORTED, "tc_pass: shared memory");
  typedef void (*kfn)(const CUtensorMap, const CUtensorMap, TcArgs);
  kfn fn;
  // resident-P kernel: 16 epilogue warps (4 per SM sub-partition) — measured 18-22 % faster
  // than 8 at small d (exp-bound epilogue) and 2 % at MSD; TS and streaming keep 8.
  int epiw = 16;
  if (const char *e = getenv("FALKON_TC_EPIW")) epiw = atoi(e) == 8 ? 8 : 16;
  if (ts || stream) epiw = 8;
#define FK_TC(M)                                                                   \
  case M:                                                                          \
    fn = ts ? tc_kvp_kernel<M, TC_N_TS, true>                                      \
            : (epiw == 16 ? tc_kvp_kernel<M, TC_N, false, false, 16>               \
                          : tc_kvp_kernel<M, TC_N, false>);                        \
    break;
  switch (mode) {
    FK_TC(1) FK_TC(2) FK_TC(3) FK_TC(8) FK_TC(9) FK_TC(10) FK_TC(11) FK_TC(12)
    default:
      fn = ts ? tc_kvp_kernel<0, TC_N_TS, true>
              : (epiw == 16 ? tc_kvp_kernel<0, TC_N, false, false, 16>
                            : tc_kvp_kernel<0, TC_N, false>);
      break;
  }
#undef FK_TC
  if (stream) fn = mode == 11 ? tc_kvp_kernel<11, TC_N, false, true> : tc_kvp_kernel<0, TC_N, false, true>;
  // 2-CTA clusters with Q multicast (FALKON_OPT_TC_CLUSTER): MODE 0, SS, single vector
  int cl = (ctx->opt.tc_cluster == 2 && kv == 1 && !ts && epiw == 16 &&
                  (mode <= 3 || kst)) || (ctx->opt.tc_cluster == 2 && kv == 1 && stream &&
                                          (mode == 0 || kst))
                     ? 2 : 1;
  if (cl == 2 && !kst) {
    if (stream) fn = tc_kvp_kernel<0, TC_N, false, true, 8, 1, false, 2>;
    else if (mode == 1) fn = tc_kvp_kernel<1, TC_N, false, false, 16, 1, false, 2>;
    else if (mode == 2) fn = tc_kvp_kernel<2, TC_N, false, false, 16, 1, false, 2>;
    else if (mode == 3) fn = tc_kvp_kernel<3, TC_N, false, false, 16, 1, false, 2>;
    else fn = tc_kvp_kernel<0, TC_N, false, false, 16, 1, false, 2>;
  }
  if (kst) {  // single-evaluation strip (MODE 0; exp offload modes do not apply)
    if (cl == 2)
      fn = stream ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, true, 2>
                  : tc_kvp_kernel<0, TC_N, false, false, 16, 1, true, 2>;
    else
      fn = stream ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, true>
                  : tc_kvp_kernel<0, TC_N, false, false, 16, 1, true>;
    epiw = stream ? 8 : 16;
  }
  if (pair && stream) {  // streaming, 2-CTA clusters: one M = 256 MMA per pair
    fn = z64 ? (kst ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, true, 2, true, true>
                    : tc_kvp_kernel<0, TC_N, false, true, 8, 1, false, 2, true, true>)
             : (kst ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, true, 2, false, true>
                    : tc_kvp_kernel<0, TC_N, false, true, 8, 1, false, 2, false, true>);
    epiw = 8;
    cl = 2;
  } else if (pair) {  // resident P tile, 2-CTA clusters: M = 256 MMAs over the pair
    fn = z64 ? (kst ? tc_kvp_kernel<0, TC_N, false, false, 16, 1, true, 2, true, true>
                    : tc_kvp_kernel<0, TC_N, false, false, 16, 1, false, 2, true, true>)
             : (kst ? tc_kvp_kernel<0, TC_N, false, false, 16, 1, true, 2, false, true>
                    : tc_kvp_kernel<0, TC_N, false, false, 16, 1, false, 2, false, true>);
    epiw = 16;
    cl = 2;
  } else if (z64) {  // ACCUM_F64 epilogue (MODE 0, exp on the MUFU; DFMA contraction)
    const bool c2 = ctx->opt.tc_cluster == 2;
    if (stream)
      fn = kst ? (c2 ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, true, 2, true>
                     : tc_kvp_kernel<0, TC_N, false, true, 8, 1, true, 1, true>)
               : (c2 ? tc_kvp_kernel<0, TC_N, false, true, 8, 1, false, 2, true>
                     : tc_kvp_kernel<0, TC_N, false, true, 8, 1, false, 1, true>);
    else
      fn = kst ? (c2 ? tc_kvp_kernel<0, TC_N, false, false, 16, 1, true, 2, true>
                     : tc_kvp_kernel<0, TC_N, false, false, 16, 1, true, 1, true>)
               : (c2 ? tc_kvp_kernel<0, TC_N, false, false, 16, 1, false, 2, true>
                     : tc_kvp_kernel<0, TC_N, false, false, 16, 1, false, 1, true>);
    epiw = stream ? 8 : 16;
    cl = c2 ? 2 : 1;
  }
  if (kv > 1) {  // multi-vector epilogue (8 epilogue warps: KV fp32 + KV fp64 sums per thread)
    epiw = 8;
    if (kv == 8) fn = stream ? tc_kvp_kernel<0, TC_N, false, true, 8, 8> : tc_kvp_kernel<0, TC_N, false, false, 8, 8>;
    else if (kv == 16) fn = stream ? tc_kvp_kernel<0, TC_N, false, true, 8, 16> : tc_kvp_kernel<0, TC_N, false, false, 8, 16>;
    else return fail(FALKON_EINVAL, "tc_pass: kv must be 1, 8 or 16");
  }
  const int threads = 128 + 32 * epiw;
  FK_CUDA(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               TC_SMEM_MAX));
  // grid: P tiles (a whole number of clusters) x Q splits, sized to whole waves of the
  // co-resident CTAs (one per SM; with clusters, 2 x the co-resident clusters)
  const int64_t gx = round_up<int64_t>(cdiv<int64_t>(np, TC_M), cl);
  const int64_t qt = cdiv<int64_t>(std::max<int64_t>(nq, 1), nt);
  const int64_t slots = cl == 1 ? ctx->sm_count : tc_cluster_slots(ctx, (const void *)fn, threads, smem);
  int64_t best_s = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= 32; ++s) {
    if (s > 1 && qt / s < 4) break;
    const int64_t ctas = gx * s;
    const int64_t waves = cdiv<int64_t>(ctas, slots);
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best_s = s;
    }
    if (ctas >= 8 * slots && eff > 0.9) break;
  }
  // L2-resident Q ranges: when the P tiles need several waves, every wave streams the same Q
  // range; a range larger than L2 is then re-read from HBM once per wave (MSD pass B: 2.7x the
  // algorithmic bytes, profiles/ncu_traffic.json).  Split Q so one range (packed rows of
  // 4 * d16 B) fits in FALKON_TC_L2Q_MB (default 40 MB of the 126 MB L2; 0 = off).
  {
    int64_t l2q = (int64_t)40 << 20;
    if (const char *e = getenv("FALKON_TC_L2Q_MB")) l2q = (int64_t)atoi(e) << 20;
    // resident-P kernels only: the streaming kernel (d > 190) re-reads its P boxes per Q tile,
    // and more Q splits cost it more than the L2 hits save (TIMIT 329 -> 338-346 ms, A/B x2)
    if (l2q > 0 && gx > slots && !stream) {
      const int64_t need = cdiv<int64_t>(nq * (int64_t)4 * d16, l2q);
      if (need > best_s && qt / need >= 4) best_s = need;
    }
  }
  int64_t qps = round_up<int64_t>(cdiv<int64_t>(nq, best_s), nt);
  const int64_t splits = std::max<int64_t>(1, cdiv<int64_t>(nq, qps));
  double *part = out64;
  if (splits > 1 || !out64) {
    void *pw;
    FK_TRY(ws_get(ctx, WS_PART, sizeof(double) * splits * np * kv, &pw));
    part = (double *)pw;
  }
  TcArgs args;
  args.z = z;
  args.z64 = z64;
  args.np = np;
  args.nq = nq;
  args.q_per_split = qps;
  args.nk = d16 / 16;
  args.nbox = nbox;
  args.stages = stages;
  args.out64 = part;
  args.out32 = splits == 1 ? out32 : nullptr;
  args.p_base = p_begin;
  args.kst = kst;
  args.ldk = ldk;
  args.gK = (kst && fg) ? fg->K : nullptr;
  args.gw = fg ? fg->w : nullptr;
  args.gdw = fg ? fg->dw : nullptr;
  args.grows = fg ? fg->rows : 0;
  args.gm = ldk;
  args.gacc = fg ? fg->acc : nullptr;
  args.gfirst = fg ? fg->first : 0;
  args.gslots = gslots;
  {
    LaunchScope ls(ctx, passA ? FALKON_T_PASS_A : FALKON_T_PASS_B);
    if (cl == 1) {
      fn<<<dim3((unsigned)gx, (unsigned)splits), threads, smem, ctx->stream>>>(
          passA ? maps[0] : maps[2], passA ? maps[ts ? 4 : 1] : maps[ts ? 5 : 3], args);
    } else {  // Q boxes of 128 rows (the P-shaped map of the Q operand), cluster launch
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)gx, (unsigned)splits);
      cfg.blockDim = dim3((unsigned)threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      FK_CUDA(cudaLaunchKernelEx(&cfg, fn, passA ? maps[0] : maps[2], passA ? maps[2] : maps[0], args));
    }
  }
  FK_LAUNCH_CHECK();
  if (splits > 1 || (!out64 && !out32))
    FK_TRY(reduce_partials(ctx, part, splits, np * kv, out64, out32));
  return FALKON_OK;
}

int tc_pass(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z, double *out64,
            float *out32, int kv) {
  return tc_launch(ctx, pp, passA, z, out64, out32, kv, 0, -1, nullptr, 0);
}

int tc_pass64(falkon_ctx *ctx, const Prepared &pp, bool passA, const double *z, double *out64) {
  return tc_launch(ctx, pp, passA, nullptr, out64, nullptr, 1, 0, -1, nullptr, 0, z);
}

int tc_pack_rows(falkon_ctx *ctx, const Prepared &pp, const float *Xrows, int64_t r0, int64_t nr) {
  if (nr <= 0) return FALKON_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(cdiv<int64_t>(nr, threads / 32), (int64_t)ctx->sm_count * 64);
  LaunchScope ls(ctx, FALKON_T_PREP);
  int *flag;
  FK_TRY(tc_range_flag(ctx, &flag, false));  // checked by the caller after the last chunk
  tc_pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(
      Xrows, nr, pp.d, pp.mu, pp.g, pp.dq, (__half *)pp.Xp + r0 * (int64_t)(2 * pp.dq), flag);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

int tc_pass_A_rows(falkon_ctx *ctx, const Prepared &pp, const float *z, float *w32, int64_t r0,
                   int64_t nr) {
  return tc_launch(ctx, pp, true, z, nullptr, w32 + r0, 1, r0, nr, nullptr, 0);
}

// ------------------------------------------------------------------ single evaluation (NEXT-4)
// Two-pass products evaluate every kernel value twice (pass A needs the whole row of K for
// w_i, pass B needs the finished w).  For large d the fp16x3 cross term (6 d16 flops per
// entry on the tensor pipe) costs more than writing k once and reading it back (8 B per entry
// of HBM traffic), so rows are processed in strips: pass A over the strip also stores its k
// values, then this GEMV streams them back:  acc[s][j] (+)= sum_{i in split s} k_ij w_i.
// Strip layout [tile][j][128 rows] (written coalesced by the epilogue): a warp reads centre
// j's 128 values of a tile as one 512-byte float4 load; lane l holds w of rows 4l..4l+3 of
// the tile.  A warp owns SE_CPW centres (independent loads in flight), lanes keep fp32 sums of
// <= 128 terms flushed into fp64 (reading c12), one shuffle reduction per centre at the end,
// one fp64 accumulator row per row split (no atomics: deterministic).
bool tc_single_eval(const falkon_ctx *ctx, const Prepared &pp) {
  if (pp.path != FALKON_PATH_TENSOR || ctx->opt.single_eval == 0) return false;
  if (ctx->opt.single_eval == 1) return true;
  return tc_stream(pp.d);  // auto: d16 > 192 (TIMIT d = 440: 6 * 448 flops vs 8 B per entry)
}

// z32/w32 (fp32 contractions) or z64/w64 (ACCUM_F64: DFMA contractions, fp64 w).  Per strip:
// pass A stores the strip's k values, then the standalone GEMV accumulates u += strip^T w.
// Every u_j is accumulated in strip order by one writer (deterministic).
static int single_eval_impl(falkon_ctx *ctx, const Prepared &pp, const float *z, const double *z64,
                            float *w32, double *w64, double *u, const float *dw) {
  const int64_t n = pp.n, m = pp.m;
  const int64_t ldk = m;
  // rows per strip: a whole number of 128-row P tiles within half the strip budget (two
  // buffers), the budget capped at half of the free device memory (plus the strips held)
  int64_t budget = ctx->opt.strip_bytes;
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
      budget = std::min<int64_t>(budget, (int64_t)(fr / 2 + ctx->ws_bytes[WS_KSTRIP]));
    else
      cudaGetLastError();
  }
  // FALKON_FUSED_GEMV=1 (experimental, off by default): two strip buffers, the GEMV of strip s - 1
  // runs in warps 2-3 of strip s's pass-A launch.  Measured on TIMIT (profiles/
  // r2_fused_gemv_ab.txt): 406-424 ms per product against 349-358 ms for the standalone GEMV
  // after each strip: the fused GEMV streams at ~1.1 TB/s beside the k stores whatever the
  // bulk-copy ring depth, and the pass-A CTAs wait for it.
  const char *fe = getenv("FALKON_FUSED_GEMV");
  const bool fused = fe && atoi(fe) != 0;
  // split-SM schedule (FALKON_OPT_SE_GEMV_SMS = G > 0): the GEMV of strip s runs as a
  // persistent grid of G CTAs on the highest-priority stream while pass A of strip s + 1 runs
  // on the remaining SMs; buffer b = s & 1 is rewritten by pass A(s + 2) only after GEMV(s)
  int gsm = fused ? 0 : ctx->opt.se_gemv_sms;
  if (const char *e = getenv("FALKON_SE_GEMV_SMS")) gsm = fused ? 0 : atoi(e);  // A/B
  gsm = std::max(0, std::min(gsm, ctx->sm_count - 1));
  const int nbuf = (fused || gsm > 0) ? 2 : 1;
  const int64_t tile_bytes = (int64_t)4 * TC_M * ldk;
  const int64_t ntiles = cdiv<int64_t>(n, TC_M);
  int64_t tiles = std::min<int64_t>(std::max<int64_t>(1, budget / nbuf / tile_bytes), ntiles);
  tiles = cdiv<int64_t>(ntiles, cdiv<int64_t>(ntiles, tiles));  // equal strips
  const int64_t rows = tiles * TC_M;
  const int64_t nstrips = cdiv<int64_t>(n, rows);
  void *kp;
  FK_TRY(ws_get(ctx, WS_KSTRIP, (size_t)tiles * tile_bytes * (nstrips > 1 ? nbuf : 1), &kp));
  float *Kbuf[2] = {(float *)kp, (float *)kp + (nstrips > 1 && nbuf == 2 ? tiles * TC_M * ldk : 0)};
  const void *wv = z64 ? (const void *)w64 : (const void *)w32;
  auto wrow = [&](int64_t r0) -> const void * {
    return z64 ? (const void *)(w64 + r0) : (const void *)(w32 + r0);
  };
  (void)wv;
  int64_t prev_r0 = 0, prev_nr = 0;
  auto gemv = [&](const float *K, int64_t r0g, int64_t nrg, int first) -> int {
    LaunchScope ls(ctx, FALKON_T_PASS_B);
    const dim3 grid((unsigned)cdiv<int64_t>(m, SE_COLS), 1u);
    const int64_t tl = cdiv<int64_t>(nrg, TC_M);
    const float *dwl = dw ? dw + r0g : nullptr;
    if (z64) {
      if (dw)
        se_gemv_kernel<true, true><<<grid, 32 * SE_WARPS, 0, ctx->stream>>>(K, ldk, w64 + r0g, dwl, nrg, tl, m, u, first);
      else
        se_gemv_kernel<false, true><<<grid, 32 * SE_WARPS, 0, ctx->stream>>>(K, ldk, w64 + r0g, nullptr, nrg, tl, m, u, first);
    } else if (dw) {
      se_gemv_kernel<true><<<grid, 32 * SE_WARPS, 0, ctx->stream>>>(K, ldk, w32 + r0g, dwl, nrg, tl, m, u, first);
    } else {
      se_gemv_kernel<false><<<grid, 32 * SE_WARPS, 0, ctx->stream>>>(K, ldk, w32 + r0g, nullptr, nrg, tl, m, u, first);
    }
    FK_LAUNCH_CHECK();
    return FALKON_OK;
  };
  if (gsm > 0 && nstrips > 1) {
    auto bulk = [&](const float *K, int64_t r0g, int64_t nrg, int first) -> int {
      LaunchScope ls(ctx, FALKON_T_PASS_B);
      const float *dwl = dw ? dw + r0g : nullptr;
      const void *wr = wrow(r0g);
      auto fn = z64 ? (dw ? se_gemv_ldg_kernel<true, true> : se_gemv_ldg_kernel<false, true>)
                    : (dw ? se_gemv_ldg_kernel<true, false> : se_gemv_ldg_kernel<false, false>);
      FK_CUDA(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, BL_SMEM));
      fn<<<(unsigned)gsm, 32 * BL_WARPS, BL_SMEM, ctx->stream>>>(K, m, wr, dwl, nrg, u, first);
      FK_LAUNCH_CHECK();
      return FALKON_OK;
    };
    if (!ctx->se_stream) {
      int least = 0, greatest = 0;
      FK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      FK_CUDA(cudaStreamCreateWithPriority(&ctx->se_stream, cudaStreamNonBlocking, greatest));
      for (auto &e : ctx->se_ev) FK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t base = ctx->stream, side = ctx->se_stream;
    cudaEvent_t *evA = ctx->se_ev, *evG = ctx->se_ev + 2;  // buffer b written / read
    for (int64_t s = 0; s < nstrips; ++s) {
      const int b = (int)(s & 1);
      const int64_t r0 = s * rows;
      const int64_t nr = std::min<int64_t>(rows, n - r0);
      if (s >= 2) FK_CUDA(cudaStreamWaitEvent(base, evG[b], 0));  // GEMV(s - 2) done with buffer b
      if (z64)
        FK_TRY(tc_launch(ctx, pp, true, nullptr, w64 + r0, nullptr, 1, r0, nr, Kbuf[b], ldk, z64));
      else
        FK_TRY(tc_launch(ctx, pp, true, z, nullptr, w32 + r0, 1, r0, nr, Kbuf[b], ldk));
      if (s + 1 < nstrips) {
        FK_CUDA(cudaEventRecord(evA[b], base));
        FK_CUDA(cudaStreamWaitEvent(side, evA[b], 0));
        ctx->stream = side;
        const int rc = bulk(Kbuf[b], r0, nr, s == 0 ? 1 : 0);
        ctx->stream = base;
        FK_TRY(rc);
        FK_CUDA(cudaEventRecord(evG[b], side));
      } else {  // the last strip's GEMV on the whole GPU, after GEMV(s - 1) (both write u)
        FK_CUDA(cudaStreamWaitEvent(base, evG[b ^ 1], 0));
        FK_TRY(gemv(Kbuf[b], r0, nr, 0));
      }
    }
    return FALKON_OK;
  }
  for (int64_t s = 0; s < nstrips; ++s) {
    const int64_t r0 = s * rows;
    const int64_t nr = std::min<int64_t>(rows, n - r0);
    if (!fused && s > 0) FK_TRY(gemv(Kbuf[(s - 1) & 1], prev_r0, prev_nr, s == 1 ? 1 : 0));
    FusedGemv fg;
    if (fused && s > 0) {
      fg.K = Kbuf[(s - 1) & 1];
      fg.w = wrow(prev_r0);
      fg.dw = dw ? dw + prev_r0 : nullptr;
      fg.rows = prev_nr;
      fg.acc = u;
      fg.first = s == 1 ? 1 : 0;
    }
    const FusedGemv *fgp = (fused && s > 0) ? &fg : nullptr;
    if (z64)
      FK_TRY(tc_launch(ctx, pp, true, nullptr, w64 + r0, nullptr, 1, r0, nr, Kbuf[s & 1], ldk, z64, fgp));
    else
      FK_TRY(tc_launch(ctx, pp, true, z, nullptr, w32 + r0, 1, r0, nr, Kbuf[s & 1], ldk, nullptr, fgp));
    prev_r0 = r0;
    prev_nr = nr;
  }
  // the last strip's GEMV: one split (every u_j one writer), centre blocks of SE_COLS
  return gemv(Kbuf[(nstrips - 1) & 1], prev_r0, prev_nr, nstrips == 1 ? 1 : 0);
}

int tc_product_single_eval(falkon_ctx *ctx, const Prepared &pp, const float *z, float *w32,
                           double *u, const float *dw) {
  return single_eval_impl(ctx, pp, z, nullptr, w32, nullptr, u, dw);
}

int tc_product_single_eval64(falkon_ctx *ctx, const Prepared &pp, const double *z, double *w64,
                             double *u, const float *dw) {
  return single_eval_impl(ctx, pp, nullptr, z, nullptr, w64, u, dw);
}

}  // namespace falkon
