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

#include <algorithm>

#include "common.cuh"

namespace falkon {

constexpr int TC_M = 128;
constexpr int TC_N = 256;
constexpr int TC_BK = 64;                          // fp16 per K box (128 B = one swizzle row)
constexpr int TC_STAGES = 4;
constexpr int TC_THREADS = 256;
constexpr int TC_A_BOX = TC_M * TC_BK * 2;         // 16 KB
constexpr int TC_B_BOX = TC_N * TC_BK * 2;         // 32 KB
constexpr int TC_MAX_D16 = 192;                    // A (all K) resident: 128 x 2*d16 fp16 <= 96 KB
constexpr double TC_LOG2E = 1.4426950408889634;

int reduce_partials(falkon_ctx *ctx, const double *part, int64_t splits, int64_t np,
                    double *out64, float *out32);
int center_mean(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, double **mu_out);

static inline int tc_d16(int64_t d) { return (int)round_up<int64_t>(d + 2, 16); }

bool tc_supported(const falkon_ctx *ctx, int kernel, int64_t d) {
  if (kernel != FALKON_GAUSSIAN) return false;  // Laplacian: direct differences only (reading c7)
  if (ctx->opt.path == FALKON_PATH_SIMT) return false;
  if (tc_d16(d) > TC_MAX_D16) return false;
  if (ctx->opt.path == FALKON_PATH_TENSOR) return true;
  return d > ctx->opt.tc_min_d;
}

// ------------------------------------------------------------------ packing
// One warp per row.  out row = [h_0..h_{d-1}, 1, 1, 0.. | l_0..l_{d-1}, (b-1)_hi, (b-1)_lo, 0..]
__global__ void tc_pack_kernel(const float *__restrict__ in, int64_t rows, int64_t d,
                               const double *__restrict__ mu, double g, int d16,
                               __half *__restrict__ out) {
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
    const double bm1 = -0.5 * s - 1.0;
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

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major SWIZZLE_128B shared-memory matrix descriptor (8-row groups of 128 B, SBO 1024 B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TcArgs {
  const float *z;
  int64_t np, nq, q_per_split;
  int nk;        // 16-wide K chunks per segment (d16 / 16)
  int nbox;      // 64-wide boxes covering one packed row (2*d16)
  double *out64;
  float *out32;
};

__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_kvp_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                  TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;                                  // nbox x 16 KB (resident P tile)
  uint8_t *sB = smem + a.nbox * TC_A_BOX;              // TC_STAGES x 32 KB
  uint64_t *bars = reinterpret_cast<uint64_t *>(sB + TC_STAGES * TC_B_BOX);
  uint64_t *full = bars, *empty = bars + TC_STAGES, *tfull = bars + 2 * TC_STAGES,
           *tempty = tfull + 2, *afull = tempty + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(afull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)blockIdx.x * TC_M;
  const int64_t qlo = (int64_t)blockIdx.y * a.q_per_split;
  const int64_t qhi = lmin(a.nq, qlo + a.q_per_split);
  const int ntiles = qhi > qlo ? (int)cdiv<int64_t>(qhi - qlo, TC_N) : 0;
  const int nchunk = 2 * a.nk;  // valid 16-wide chunks of a packed row

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    mbar_init(afull, 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // resident P tile (all K)
      mbar_expect_tx(afull, (uint32_t)(a.nbox * TC_A_BOX));
      for (int b = 0; b < a.nbox; ++b) tma_load_2d(sA + b * TC_A_BOX, &tmP, b * TC_BK, (int)p0, afull);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int q0 = (int)(qlo + (int64_t)t * TC_N);
        for (int b = 0; b < a.nbox; ++b) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], TC_B_BOX);
          tma_load_2d(sB + stage * TC_B_BOX, &tmQ, b * TC_BK, q0, &full[stage]);
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);
      const uint32_t sA_addr = smem_u32(sA), sB_addr = smem_u32(sB);
      auto adesc = [&](int c) {  // 16-wide chunk c of the resident A row block
        return sw128_desc(sA_addr + (uint32_t)((c >> 2) * TC_A_BOX + (c & 3) * 32));
      };
      mbar_wait(afull, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int acc = t & 1;
        mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + (uint32_t)(acc * TC_N);
        uint32_t accumulate = 0;
        for (int b = 0; b < a.nbox; ++b) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int j = b * 4 + jj;  // chunk of the Q row held in this box
            if (j < nchunk) {
              const uint64_t bd = sw128_desc(sB_addr + (uint32_t)(stage * TC_B_BOX + jj * 32));
              if (j < a.nk) {
                tc_mma_f16(dtm, adesc(j), bd, idesc, accumulate);          // h_p . h_q
                accumulate = 1;
                tc_mma_f16(dtm, adesc(a.nk + j), bd, idesc, 1);            // l_p . h_q
              } else {
                tc_mma_f16(dtm, adesc(j - a.nk), bd, idesc, 1);            // h_p . l_q
              }
            }
          }
          tc_commit(&empty[stage]);
          if (++stage == TC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const int64_t p = p0 + row;
    double acc64 = 0.0;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      const int64_t q0 = qlo + (int64_t)t * TC_N;
      const int cnt = (int)lmin(TC_N, qhi - q0);
      const uint32_t tbase = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * TC_N);
      float accf = 0.f;
      uint32_t r[32];
      tmem_ld32(tbase, r);
      tmem_wait_ld();
      for (int c = 0; c < TC_N / 32; ++c) {
        if (c * 32 >= cnt) break;
        float e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) e[j] = __uint_as_float(r[j]);
        if ((c + 1) * 32 < cnt) tmem_ld32(tbase + (uint32_t)((c + 1) * 32), r);
        const float4 *zp = reinterpret_cast<const float4 *>(a.z + q0 + c * 32);
        const int lim = cnt - c * 32;
#pragma unroll
        for (int g4 = 0; g4 < 8; ++g4) {
          const float4 zz = __ldg(zp + g4);
          const float zv[4] = {zz.x, zz.y, zz.z, zz.w};
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int j = g4 * 4 + e4;
            const float zj = j < lim ? zv[e4] : 0.f;
            accf = fmaf(ex2_approx(fminf(e[j], 0.f)), zj, accf);
          }
        }
        tmem_wait_ld();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc64 += (double)accf;
    }
    if (p < a.np) {
      if (a.out64) a.out64[(int64_t)blockIdx.y * a.np + p] = acc64;
      if (a.out32) a.out32[p] = (float)acc64;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
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
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_t)p;
    else
      cudaGetLastError();
  }
  return fn;
}

static int make_map(CUtensorMap *map, const __half *base, int64_t rows, int k_elems, int box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return fail(FALKON_EUNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)k_elems, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)k_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void *)base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FALKON_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return FALKON_OK;
}

static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");

int tc_prepare(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C, int64_t m,
               double sigma, const double *mu, Prepared *pp) {
  const int d16 = tc_d16(d);
  const int kp = 2 * d16;
  const double g = std::sqrt(TC_LOG2E) / sigma;
  const int64_t n_pad = round_up<int64_t>(std::max<int64_t>(n, 1), TC_N);
  const int64_t m_pad = round_up<int64_t>(m, TC_N);
  void *xp, *cp;
  FK_TRY(ws_get(ctx, WS_XP, sizeof(__half) * n_pad * kp, &xp));
  FK_TRY(ws_get(ctx, WS_CP, sizeof(__half) * m_pad * kp, &cp));
  const int threads = 256;
  {
    LaunchScope ls(ctx, FALKON_T_PREP);
    const int64_t blocks = std::min<int64_t>(cdiv<int64_t>(m, threads / 32), 65535);
    tc_pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(C, m, d, mu, g, d16, (__half *)cp);
  }
  FK_LAUNCH_CHECK();
  if (n > 0) {
    LaunchScope ls(ctx, FALKON_T_PREP);
    const int64_t blocks = std::min<int64_t>(cdiv<int64_t>(n, threads / 32), (int64_t)ctx->sm_count * 64);
    tc_pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(X, n, d, mu, g, d16, (__half *)xp);
    FK_LAUNCH_CHECK();
  }
  pp->dq = d16;
  pp->Xp = xp;
  pp->Cp = cp;
  pp->xa = nullptr;
  pp->cb = nullptr;
  CUtensorMap *maps = reinterpret_cast<CUtensorMap *>(pp->tmaps);
  FK_TRY(make_map(&maps[0], (const __half *)xp, n, kp, TC_M));  // X as P (pass A)
  FK_TRY(make_map(&maps[1], (const __half *)cp, m, kp, TC_N));  // C as Q (pass A)
  FK_TRY(make_map(&maps[2], (const __half *)cp, m, kp, TC_M));  // C as P (pass B)
  FK_TRY(make_map(&maps[3], (const __half *)xp, n, kp, TC_N));  // X as Q (pass B)
  return FALKON_OK;
}

static size_t tc_smem_bytes(int nbox) {
  return 1024 + (size_t)nbox * TC_A_BOX + (size_t)TC_STAGES * TC_B_BOX + 256;
}

int tc_pass(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z, double *out64,
            float *out32) {
  const CUtensorMap *maps = reinterpret_cast<const CUtensorMap *>(pp.tmaps);
  const int d16 = pp.dq;
  const int nbox = (int)cdiv<int64_t>(2 * d16, TC_BK);
  const int64_t np = passA ? pp.n : pp.m, nq = passA ? pp.m : pp.n;
  if (np <= 0) return FALKON_OK;
  const size_t smem = tc_smem_bytes(nbox);
  static bool attr = false;
  if (!attr) {
    FK_CUDA(cudaFuncSetAttribute(tc_kvp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tc_smem_bytes(cdiv(2 * TC_MAX_D16, TC_BK))));
    attr = true;
  }
  // grid: P tiles x Q splits, sized to whole waves of one CTA per SM
  const int64_t gx = cdiv<int64_t>(np, TC_M);
  const int64_t qt = cdiv<int64_t>(std::max<int64_t>(nq, 1), TC_N);
  int64_t best_s = 1;
  double best_eff = -1.0;
  for (int64_t s = 1; s <= 32; ++s) {
    if (s > 1 && qt / s < 4) break;
    const int64_t ctas = gx * s;
    const int64_t waves = cdiv<int64_t>(ctas, ctx->sm_count);
    const double eff = (double)ctas / (double)(waves * ctx->sm_count);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best_s = s;
    }
    if (ctas >= 8 * ctx->sm_count && eff > 0.9) break;
  }
  int64_t qps = round_up<int64_t>(cdiv<int64_t>(nq, best_s), TC_N);
  const int64_t splits = std::max<int64_t>(1, cdiv<int64_t>(nq, qps));
  double *part = out64;
  if (splits > 1 || !out64) {
    void *pw;
    FK_TRY(ws_get(ctx, WS_PART, sizeof(double) * splits * np, &pw));
    part = (double *)pw;
  }
  TcArgs args;
  args.z = z;
  args.np = np;
  args.nq = nq;
  args.q_per_split = qps;
  args.nk = d16 / 16;
  args.nbox = nbox;
  args.out64 = part;
  args.out32 = splits == 1 ? out32 : nullptr;
  {
    LaunchScope ls(ctx, passA ? FALKON_T_PASS_A : FALKON_T_PASS_B);
    tc_kvp_kernel<<<dim3((unsigned)gx, (unsigned)splits), TC_THREADS, smem, ctx->stream>>>(
        passA ? maps[0] : maps[2], passA ? maps[1] : maps[3], args);
  }
  FK_LAUNCH_CHECK();
  if (splits > 1 || (!out64 && !out32)) FK_TRY(reduce_partials(ctx, part, splits, np, out64, out32));
  return FALKON_OK;
}

}  // namespace falkon
