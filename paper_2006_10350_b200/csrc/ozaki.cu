// ozaki.cu — the preconditioner's big fp64 GEMMs on the int8 tensor cores (FALKON_OPT_OZAKI).
//
// The blocked Cholesky factorisations of Kmm and of T T^T/m + lambda I (Alg. 1 lines 13-17,
// PAPER.md:127-133; the paper's out-of-core POTRF, App. C Alg. 4) spend
// almost all of their m^3/3 flops each in the trailing updates  S_ij -= L_ik L_jk^T.  On B200
// the fp64 DMMA pipe (~37 TF/s measured) binds them; the int8 tensor pipe is ~120x faster per
// operation.  Ozaki scheme I turns one fp64 GEMM into exact integer GEMMs:
//
//   every row i of A (and of B) is scaled by a power of two, a_ik = 2^e_i x_ik, |x_ik| < 1,
//   and split without error into OZ_S signed 7-bit slices  x_ik = sum_p q^(p)_ik 2^(-7(p+1))
//   (+ a residual below 2^(-7 OZ_S) = 2^-56, below the fp64 significand of the row maximum);
//   then  (A B^T)_ij = 2^(e_i + f_j) sum_{p,q} 2^(-7(p+q+2)) (Q^(p) Q'^(q)T)_ij,
//
// where each slice product is an int8 x int8 -> int32 MMA (tcgen05.mma kind::i8), exact while
// K * 127^2 * (products per level) < 2^31 (K <= OZ_KMAX = 4096 per call; LAUUM in k chunks of
// 4096 at absolute boundaries).  Products with p + q >= OZ_S are dropped (each below
// 2^-70 K 127^2 of the scaled rows' product: the order of the fp64 GEMM's own rounding),
// leaving 36 slice products in 8 levels L = p + q; the levels are summed in int32 inside TMEM
// (8 accumulators of 128 x 64 per CTA) and combined once per tile in fp64, smallest level first.
// The result is deterministic (integer sums; fixed combination order) and independent of the
// call's row range (the distributed schedule reproduces the single-GPU factors bitwise), but
// not bitwise equal to the DMMA GEMM: factors agree to ~1e-13 relative (tests/test_gpu_ozaki.py).
//
// Kernel (default): persistent 2-CTA clusters, one 256 x 64 C tile per pair as
// tcgen05.mma.cta_group::2 (M = 256, N = 64, K = 32); each CTA stages its 128 A rows and a
// 32-row half of the B slices (one 3-D TMA box per operand: k, rows, 8 slices; 32-byte rows,
// SWIZZLE_32B) through a 5-stage ring of 40 KB; warp 0 TMA producer, warp 1 of the leader the
// MMA issuer (36 MMAs per stage), warp 2 TMEM allocator, warps 4-11 the epilogue (thread = TMEM
// lane = C row, 32 of the tile's columns), which releases TMEM before its fp64 read-modify-write
// of C.  FALKON_OZ_PAIR=0 selects the single-CTA kernel (128 x 64 tiles, 4 x 48 KB stages).
#include <math.h>

#include <algorithm>

#include <cuda.h>

#include "common.cuh"
#include "precond.cuh"
#include "tcgen05.cuh"

namespace falkon {

#ifndef OZ_S_OVR
#define OZ_S_OVR 8
#endif
#ifndef OZ_BN_OVR
#define OZ_BN_OVR 64
#endif
constexpr int OZ_S = OZ_S_OVR;     // slices per operand (7 bits each: 56-bit significands)
constexpr int OZ_BM = 128;         // C tile rows (TMEM lanes)
constexpr int OZ_BN = OZ_BN_OVR;         // C tile columns; 8 level accumulators x 64 = 512 TMEM columns
constexpr int OZ_BK = 32;          // int8 per K box = one MMA's K (32 B rows, SWIZZLE_32B)
#ifndef OZ_KMAX_OVR
#define OZ_KMAX_OVR 4096
#endif
constexpr int OZ_KMAX = OZ_KMAX_OVR;  // 8 * K * 127^2 < 2^31 (K < 16,640): level sums exact in int32
static_assert((int64_t)8 * OZ_KMAX * 127 * 127 < ((int64_t)1 << 31), "int32 level sums");
static_assert(OZ_S == 8, "the pack's one-conversion split assumes 8 slices of 7 bits (56 bits)");
constexpr int OZ_STAGES = 4;
constexpr int64_t OZ_MIN_LD = 512;  // preconditioners of m < 512 stay on DMMA (launch-bound)
constexpr int OZ_ASL = OZ_BM * OZ_BK;                   // 4 KB per A slice box
constexpr int OZ_BSL = OZ_BN * OZ_BK;                   // 2 KB per B slice box
constexpr int OZ_STAGE = OZ_S * (OZ_ASL + OZ_BSL);      // 48 KB
constexpr int OZ_EPIW = 8;                              // epilogue warps (2 per TMEM lane quarter)
constexpr int OZ_THREADS = 128 + 32 * OZ_EPIW;
constexpr int OZ_SMEM = 1024 + OZ_STAGES * OZ_STAGE + 256;

// ------------------------------------------------------------------ error-free splitting
// Rows [r0, r0 + rows) x k [k0, k0 + K) of view V (times kscale[k] if given) -> slices out[(p * rpad + i) * kpad + k]
// (int8) and row exponents expo[i] (max_k |a_ik| = f 2^e, f in [0.5, 1)).  Rows past `rows`
// and k past K are zero.  One block per 32 rows; 32 x 32 tiles pass through shared memory so
// the view is read along its contiguous dimension whatever its orientation.
__global__ void __launch_bounds__(256) oz_pack_kernel(View V, int64_t r0, int64_t rows, int64_t k0,
                                                      int64_t K, int64_t kpad, int64_t rpad,
                                                      int8_t *__restrict__ out,
                                                      int *__restrict__ expo,
                                                      const double *__restrict__ kscale) {
  __shared__ double t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t rb = (int64_t)blockIdx.x * 32;
  auto load = [&](int64_t kc) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int a = ty + 8 * i;
      const int rr = V.trans ? tx : a, kk = V.trans ? a : tx;  // lanes walk the storage
      const int64_t r = rb + rr, k = kc + kk;
      double v = (r < rows && k < K) ? vget(V, r0 + r, k0 + k) : 0.0;
      if (kscale && k < K) v *= kscale[k0 + k];  // weighted LAUUM (Alg. 2): B(j, k) D(k)
      t[rr][kk] = v;
    }
  };
  double mx[4] = {0.0, 0.0, 0.0, 0.0};  // rows ty + 8 i
  for (int64_t kc = 0; kc < K; kc += 32) {
    __syncthreads();
    load(kc);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) mx[i] = fmax(mx[i], fabs(t[ty + 8 * i][tx]));
  }
  int e[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double v = mx[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    e[i] = 0;
    if (v > 0.0) frexp(v, &e[i]);
    if (tx == 0) expo[rb + ty + 8 * i] = e[i];
  }
  // phase 2: thread -> (row tid / 8, 4 consecutive k): one 32-bit store of 4 slice bytes per slice
  __shared__ int es[32];
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) es[ty + 8 * i] = e[i];
  }
  const int pr = threadIdx.x >> 3, pk = (threadIdx.x & 7) * 4;
  for (int64_t kc = 0; kc < kpad; kc += 32) {
    __syncthreads();
    load(kc);
    __syncthreads();
    const double sc = __longlong_as_double((long long)(1023 - es[pr]) << 52);  // 2^-e, exact
    uint32_t w[OZ_S];
#pragma unroll
    for (int p = 0; p < OZ_S; ++p) w[p] = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // the 56-bit truncation toward zero of y in one conversion; slice p = base-128 digit p of
      // |Y| with the sign of y (the same digits as repeated y *= 128, q = trunc(y), y -= q)
      const double y = t[pr][pk + u] * sc;                             // |y| < 1, exact
      const long long Y = __double2ll_rz(y * 72057594037927936.0);     // 2^56 y, exact scale
      const unsigned long long A = Y < 0 ? (unsigned long long)(-Y) : (unsigned long long)Y;
#pragma unroll
      for (int p = 0; p < OZ_S; ++p) {
        int q = (int)((A >> (7 * (OZ_S - 1 - p))) & 127u);
        if (Y < 0) q = -q;
        w[p] |= (uint32_t)(uint8_t)(int8_t)q << (8 * u);
      }
    }
    const int64_t row = rb + pr;
#pragma unroll
    for (int p = 0; p < OZ_S; ++p)
      *reinterpret_cast<uint32_t *>(out + ((int64_t)p * rpad + row) * kpad + kc + pk) = w[p];
  }
}

// ------------------------------------------------------------------ int8 tcgen05 GEMM
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

struct OzArgs {
  GemmArgs g;
  const int *ea, *eb;     // row exponents of the packed A / B rows
  int64_t brow0;          // packed row of B row rb (rb - ra when B shares A's slab, else 0)
  int rpa, rpb;           // rows per slice of the A / B slabs
  int nkb;                // K boxes
  int64_t ntiles;         // C tiles (tri_tiles: the lower ones, or all when tri_rect)
  int diag;               // FALKON_OZ_DIAG (timing only, wrong results): 1 no C read-modify-
                          // write, 2 no MMAs, 3 no TMA loads
  int tri_rect;           // tri_tiles on a tall region (N < M): rectangular order, upper tiles skipped
};

// K-major SWIZZLE_32B descriptor (8-row groups of 32 B, SBO 256 B)
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}
// tile t -> (ti, tj) for row tiles of BM rows; false: a tile above the diagonal of a tall
// tri_tiles region (skipped by every role alike, so the roles' tile sequences stay in step)
template <int BM>
__device__ __forceinline__ bool oz_tile(const OzArgs &a, int64_t t, int64_t &ti, int64_t &tj) {
  constexpr int R = BM / OZ_BN;
  if (a.g.tri_tiles && !a.tri_rect) {  // row tile ti holds R (ti + 1) column tiles of the lower region
    ti = (int64_t)((sqrt(8.0 * (double)t / R + 1.0) - 1.0) * 0.5);
    while (R * (ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (R * ti * (ti + 1) / 2 > t) --ti;
    tj = t - R * ti * (ti + 1) / 2;
    return true;
  }
  const int64_t ntj = cdiv<int64_t>(a.g.N, OZ_BN);
  ti = t / ntj;
  tj = t % ntj;
  return !(a.g.tri_tiles && tj >= R * (ti + 1));
}
__device__ __forceinline__ void tma_load_3d_pair(void *dst, const CUtensorMap *map, int c0, int c1,
                                                 int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar) & TC_PEER_MASK)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ double pow2(int e) {  // exact 2^e for normal e
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// Persistent: CTA c takes tiles c, c + grid, ...; the TMA ring runs on across tiles (the next
// tile's boxes land while the epilogue drains), the epilogue releases TMEM right after its
// tcgen05.ld's and then does the fp64 read-modify-write of C beside the next tile's MMAs.
// PAIR: clusters of two CTAs run one tcgen05.mma.cta_group::2 of M = 256 (each CTA's 128 A rows)
// x N = 64 (each CTA stages ITS 32-row half of the B slices): per CTA 40 KB per stage instead of
// 48 KB and 5 KB of shared-memory operand reads per 128 x 64 x 32 product instead of 6 KB (the
// two bounds of the single-CTA kernel).  The leader waits on its full barrier for both CTAs'
// boxes, issues the MMAs and commits to both CTAs' empty / tfull barriers; both epilogues
// release the accumulators on the leader's tempty.
template <bool PAIR>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   OzArgs a) {
  constexpr int BMP = PAIR ? 2 * OZ_BM : OZ_BM;       // C rows per tile (pair)
  constexpr int BROWS = PAIR ? OZ_BN / 2 : OZ_BN;     // B rows staged by this CTA
  constexpr int BSL = BROWS * OZ_BK;
  constexpr int STAGE = OZ_S * (OZ_ASL + BSL);
  constexpr int NST = PAIR ? 5 : OZ_STAGES;
  extern __shared__ uint8_t oz_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) &
                                            ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + NST * STAGE);
  uint64_t *empty = full + NST, *tfull = empty + NST, *tempty = tfull + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 1);
  const GemmArgs &g = a.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cid = PAIR ? blockIdx.x >> 1 : blockIdx.x;  // cluster (pair) id
  const int64_t ncl = PAIR ? gridDim.x >> 1 : gridDim.x;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, PAIR ? 2 * OZ_EPIW : OZ_EPIW);  // one arrival per epilogue warp
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tslot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tslot)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the partner's barriers initialised before any remote arrival
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t crank = PAIR ? cluster_rank() : 0;

  if (warp == 0) {  // TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = cid; t < a.ntiles; t += ncl) {
      int64_t ti, tj;
      if (!oz_tile<BMP>(a, t, ti, tj)) continue;
      const int ra = (int)(ti * BMP + OZ_BM * crank);
      const int rb = (int)(a.brow0 + tj * OZ_BN + BROWS * crank);
      for (int kb = 0; kb < a.nkb; ++kb) {
        mbar_wait_safe(&empty[stage], phase ^ 1);
        if (elect_one()) {
          uint8_t *st = sm + stage * STAGE;
          if (!PAIR && a.diag == 3) {
            mbar_arrive(&full[stage]);
          } else if (PAIR) {  // both CTAs' boxes complete on the leader's full barrier
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * STAGE);
            tma_load_3d_pair(st, &ta, kb * OZ_BK, ra, 0, &full[stage]);
            tma_load_3d_pair(st + OZ_S * OZ_ASL, &tb, kb * OZ_BK, rb, 0, &full[stage]);
          } else {
            mbar_expect_tx(&full[stage], STAGE);
            // one 3-D box (k, rows, slice) per operand: all OZ_S slices of the tile's rows
            tma_load_3d(st, &ta, kb * OZ_BK, ra, 0, &full[stage]);
            tma_load_3d(st + OZ_S * OZ_ASL, &tb, kb * OZ_BK, rb, 0, &full[stage]);
          }
        }
        __syncwarp();
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && crank == 0) {  // MMA issuer (the pair's leader): level L = p + q
    // accumulates in TMEM columns [64 L, 64 L + 64).  kind::i8 instruction descriptor: D s32
    // (bits 4-5 = 2), A and B signed (bits 7-9, 10-12 = 1), K-major, N >> 3 at 17, M >> 4 at 24
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) |
                           ((uint32_t)(BMP >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0, it = 0;
    for (int64_t t = cid; t < a.ntiles; t += ncl) {
      int64_t ti, tj;
      if (!oz_tile<BMP>(a, t, ti, tj)) continue;
      mbar_wait_safe(tempty, (it & 1) ^ 1);  // the epilogue has read the previous tile
      tc_fence_after();
      for (int kb = 0; kb < a.nkb; ++kb) {
        mbar_wait_safe(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t base = sw32_desc(smem_u32(sm + stage * STAGE));
          for (int p = 0; p < ((!PAIR && a.diag == 2) ? 0 : OZ_S); ++p) {
            const uint64_t ad = base + (uint64_t)((p * OZ_ASL) >> 4);
            for (int q = 0; q < OZ_S - p; ++q) {  // the p = 0 pass opens every level
              const uint64_t bd = base + (uint64_t)((OZ_S * OZ_ASL + q * BSL) >> 4);
              if (PAIR) tc_mma_i8_pair(tmem + (uint32_t)((p + q) * OZ_BN), ad, bd, idesc, (kb | p) ? 1u : 0u);
              else tc_mma_i8(tmem + (uint32_t)((p + q) * OZ_BN), ad, bd, idesc, (kb | p) ? 1u : 0u);
            }
          }
          if (PAIR) tc_commit_pair(&empty[stage]);
          else tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == NST) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) {
        if (PAIR) tc_commit_pair(tfull);
        else tc_commit(tfull);
      }
      __syncwarp();
      ++it;
    }
  } else if (warp >= 4) {  // epilogue: thread = C row of the tile, 32 of its 64 columns
    const int lg = warp & 3, ch = (warp - 4) >> 2;
    const uint32_t tl = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(32 * ch);
    uint32_t it = 0;
    for (int64_t t = cid; t < a.ntiles; t += ncl) {
      int64_t ti, tj;
      if (!oz_tile<BMP>(a, t, ti, tj)) continue;
      const int64_t gi = ti * BMP + OZ_BM * crank + lg * 32 + lane, j0 = tj * OZ_BN + 32 * ch;
      mbar_wait_safe(tfull, it & 1);
      tc_fence_after();
      double sum[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) sum[c] = 0.0;
#pragma unroll
      for (int L = OZ_S - 1; L >= 0; --L) {  // smallest level first
        uint32_t r[32];
        tmem_ld32(tl + (uint32_t)(L * OZ_BN), r);
        tmem_wait_ld_regs(r);
        const double sc = pow2(-7 * (L + 2));
#pragma unroll
        for (int c = 0; c < 32; ++c) sum[c] = fma((double)(int)r[c], sc, sum[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // TMEM free for the next tile's MMAs (PAIR: on the leader's barrier)
        if (PAIR && crank != 0) mbar_arrive_cluster(tempty, 0);
        else mbar_arrive(tempty);
      }
      if (gi < g.M && a.diag != 1) {
        const int64_t r = g.rc + gi;
        const int er = a.ea[gi];
        auto put = [&](int c) {  // one element through the view (masks, diagonal vector)
          const int64_t gj = j0 + c;
          const int64_t cc = g.cc + gj;
          const bool ok = gj < g.N && !(g.C.tri == 1 && r < cc) && !(g.C.tri == 2 && cc < r);
          if (ok) {
            const int e = er + a.eb[a.brow0 + gj];
            const double ab = (e > -1000 && e < 1000) ? sum[c] * pow2(e) : ldexp(sum[c], e);
            const double cv = g.beta != 0.0 ? g.beta * vget(g.C, r, cc) : 0.0;
            vset(g.C, r, cc, g.alpha * ab + cv);
          }
        };
        // row-major C (trans = 0: the A factor, the LAUUM): a thread's 32 columns are
        // contiguous, so pairs strictly inside the stored part go as one 16-byte access
        // (half the L2 transactions of the lane-strided pattern); the rest element-wise
        const bool vec = !g.C.trans && g.C.tri != 2 && ((r * g.C.ld + g.cc + j0) & 1) == 0;
        if (vec) {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const int64_t gj = j0 + c, cc = g.cc + gj;
            if (gj + 1 < g.N && (g.C.tri != 1 || r > cc + 1)) {
              const int e0 = er + a.eb[a.brow0 + gj], e1 = er + a.eb[a.brow0 + gj + 1];
              const double ab0 = (e0 > -1000 && e0 < 1000) ? sum[c] * pow2(e0) : ldexp(sum[c], e0);
              const double ab1 =
                  (e1 > -1000 && e1 < 1000) ? sum[c + 1] * pow2(e1) : ldexp(sum[c + 1], e1);
              double2 *p = reinterpret_cast<double2 *>(g.C.base + r * g.C.ld + cc);
              double2 o;
              if (g.beta != 0.0) {
                const double2 cv = *p;
                o.x = g.alpha * ab0 + g.beta * cv.x;
                o.y = g.alpha * ab1 + g.beta * cv.y;
              } else {
                o.x = g.alpha * ab0;
                o.y = g.alpha * ab1;
              }
              *p = o;
            } else {
              put(c);
              put(c + 1);
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) put(c);  // unrolled: sum[] stays in registers
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the partner's last commits / arrivals into this CTA are done
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*PFN_encodeTiled_oz)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                       const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                       const cuuint32_t *, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);
static PFN_encodeTiled_oz oz_encode() {
  static const PFN_encodeTiled_oz fn = []() -> PFN_encodeTiled_oz {  // thread-safe, once
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_encodeTiled_oz)p;
    cudaGetLastError();
    return nullptr;
  }();
  return fn;
}
// 3-D map of a slab [slice][rows][kpad] (int8): boxes of OZ_BK x box_rows x all slices
static int oz_map(CUtensorMap *map, const int8_t *slab, int64_t rows, int64_t kpad, int box_rows) {
  PFN_encodeTiled_oz enc = oz_encode();
  if (!enc) return OZ_DECLINED;
  cuuint64_t dims[3] = {(cuuint64_t)kpad, (cuuint64_t)rows, (cuuint64_t)OZ_S};
  cuuint64_t strides[2] = {(cuuint64_t)kpad, (cuuint64_t)(rows * kpad)};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows, (cuuint32_t)OZ_S};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)slab, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FALKON_ECUDA, "cuTensorMapEncodeTiled (ozaki) failed");
  return FALKON_OK;
}

static int oz_pack(falkon_ctx *ctx, const View &v, int64_t r0, int64_t rows, int64_t k0, int64_t K,
                   int64_t kpad, int64_t rpad, int8_t *slab, int *expo, const double *kscale) {
  LaunchScope ls(ctx, FALKON_T_PRECOND);
  oz_pack_kernel<<<(unsigned)(rpad / 32), 256, 0, ctx->stream>>>(v, r0, rows, k0, K, kpad, rpad,
                                                                 slab, expo, kscale);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// C(rc + i, cc + j) *= beta (0: cleared) for j <= i... through the view (the LAUUM's chunks then
// accumulate with beta = 1)
__global__ void oz_scale_lower_kernel(View C, int64_t rc, int64_t cc, int64_t M, int64_t N,
                                      double beta) {
  for (int64_t i = blockIdx.x; i < M; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
      const int64_t r = rc + i, c = cc + j;
      if ((C.tri == 1 && r < c) || (C.tri == 2 && c < r)) continue;
      vset(C, r, c, beta != 0.0 ? beta * vget(C, r, c) : 0.0);
    }
}

// One product with k1 - k0 <= OZ_KMAX (no k_from_row): pack, tensor maps, persistent kernel.
static int oz_gemm_core(falkon_ctx *ctx, const GemmArgs &a) {
  const int64_t K = a.k1 - a.k0;
  const int64_t kpad = round_up<int64_t>(K, OZ_BK);
  const int64_t rpa = round_up<int64_t>(a.M, OZ_BM);
  const bool share = !a.kscale && a.A.base == a.B.base && a.A.ld == a.B.ld &&
                     a.A.trans == a.B.trans && a.A.tri == a.B.tri && a.A.dvec == a.B.dvec &&
                     a.rb >= a.ra && a.rb + a.N <= a.ra + a.M;
  const int64_t rpb = share ? rpa : round_up<int64_t>(a.N, OZ_BM);
  if (OZ_S * std::max(rpa, rpb) > INT32_MAX - 2 * OZ_BM) return OZ_DECLINED;  // TMA coordinates
  const size_t abytes = (size_t)OZ_S * rpa * kpad, bbytes = share ? 0 : (size_t)OZ_S * rpb * kpad;
  const size_t ebytes = sizeof(int) * (size_t)(rpa + (share ? 0 : rpb));
  // one slab per stream: the Cholesky lookahead runs two updates of the same panel at once
  void *ws;
  FK_TRY(ws_get(ctx, ctx->stream == ctx->lo_stream ? WS_OZ1 : WS_OZ0, abytes + bbytes + ebytes, &ws));
  int8_t *sa = (int8_t *)ws, *sb = share ? sa : sa + abytes;
  int *ea = (int *)((int8_t *)ws + abytes + bbytes), *eb = share ? ea : ea + rpa;
  FK_TRY(oz_pack(ctx, a.A, a.ra, a.M, a.k0, K, kpad, rpa, sa, ea, nullptr));
  if (!share) FK_TRY(oz_pack(ctx, a.B, a.rb, a.N, a.k0, K, kpad, rpb, sb, eb, a.kscale));
  CUtensorMap ta, tb;
  FK_TRY(oz_map(&ta, sa, rpa, kpad, OZ_BM));
  FK_TRY(oz_map(&tb, sb, rpb, kpad, OZ_BN));
  OzArgs oa;
  oa.g = a;
  oa.ea = ea;
  oa.eb = eb;
  oa.brow0 = share ? a.rb - a.ra : 0;
  oa.rpa = (int)rpa;
  oa.rpb = (int)rpb;
  oa.nkb = (int)(kpad / OZ_BK);
  {
    const char *e = getenv("FALKON_OZ_DIAG");
    oa.diag = e ? atoi(e) : 0;
  }
  // CTA pairs (default; FALKON_OZ_PAIR=0 selects the single-CTA kernel, A/B): the B map then
  // delivers 32-row halves
  const char *pe = getenv("FALKON_OZ_PAIR");
  const bool pair = !(pe && atoi(pe) == 0) && oa.diag <= 1;
  if (pair) FK_TRY(oz_map(&tb, sb, rpb, kpad, OZ_BN / 2));
  const int bmp = pair ? 2 * OZ_BM : OZ_BM;
  const int64_t nti = cdiv<int64_t>(a.M, bmp), ntj = cdiv<int64_t>(a.N, OZ_BN);
  oa.tri_rect = a.tri_tiles && a.N < a.M;
  oa.ntiles = (a.tri_tiles && !oa.tri_rect) ? (bmp / OZ_BN) * nti * (nti + 1) / 2 : nti * ntj;
  if (pair) {
    const int smem = 1024 + 5 * OZ_S * (OZ_ASL + OZ_BN / 2 * OZ_BK) + 256;
    FK_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t clusters = std::min<int64_t>(oa.ntiles, ctx->sm_count / 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.blockDim = dim3(OZ_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    FK_CUDA(cudaLaunchKernelEx(&cfg, oz_gemm_kernel<true>, ta, tb, oa));
  } else {
    FK_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM));
    const unsigned grid = (unsigned)std::min<int64_t>(oa.ntiles, ctx->sm_count);
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    oz_gemm_kernel<false><<<grid, OZ_THREADS, OZ_SMEM, ctx->stream>>>(ta, tb, oa);
  }
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

int oz_gemm(falkon_ctx *ctx, const GemmArgs &a) {
  if (!ctx->opt.ozaki || !oz_encode()) return OZ_DECLINED;
  if (a.k_from_row) {
    // the LAUUM  C(i, j) = alpha sum_{k >= i} T(i, k) [D(k)] T(j, k) + beta C  (T upper, C lower,
    // i >= j): C scaled by beta once, then k chunks of OZ_KMAX accumulate (beta = 1), chunk
    // [kc, kc + OZ_KMAX) only over the rows i < kc + OZ_KMAX it reaches (T(i, k) = 0 for k < i)
    // the decision depends on the buffer (ld = m), never on a call's M / N: the distributed
    // schedule's per-panel calls then take the same path as the single-GPU build's one call
    if (!(a.tri_tiles && a.ra == a.rb && a.rc == a.ra && a.cc == a.rb && a.N <= a.M &&
          a.C.tri == 1 && a.C.ld >= OZ_MIN_LD))
      return OZ_DECLINED;
    {
      LaunchScope ls(ctx, FALKON_T_PRECOND);
      oz_scale_lower_kernel<<<(unsigned)std::min<int64_t>(a.M, 65535), 256, 0, ctx->stream>>>(
          a.C, a.rc, a.cc, a.M, a.N, a.beta);
    }
    FK_LAUNCH_CHECK();
    // chunk boundaries at absolute multiples of OZ_KMAX: every element sees the same k chunks
    // (hence the same slices, exponents and integer sums) whatever the row range of the call,
    // so the distributed schedule's per-panel calls reproduce the single-GPU build bitwise
    for (int64_t kc = std::max(a.k0, a.ra), ke; kc < a.k1; kc = ke) {
      ke = std::min<int64_t>(a.k1, (kc / OZ_KMAX + 1) * OZ_KMAX);
      GemmArgs s = a;
      s.k_from_row = 0;
      s.k0 = kc;
      s.k1 = ke;
      s.beta = 1.0;
      s.M = std::min<int64_t>(a.M, ke - a.ra);
      s.N = std::min<int64_t>(a.N, ke - a.rb);
      if (s.M <= 0 || s.N <= 0) continue;
      FK_TRY(oz_gemm_core(ctx, s));
    }
    return FALKON_OK;
  }
  const int64_t K = a.k1 - a.k0;
  // the panel solves and the intra-panel updates (k = 128) stay on DMMA: the trailing updates
  // (k = potrf_outer x 128 = 1024 by default) carry almost all of the flops.  As above the
  // decision uses the k range and the buffer size only (schedule-independent results).
  if (a.kscale || K < 256 || K > OZ_KMAX || a.C.ld < OZ_MIN_LD) return OZ_DECLINED;
  return oz_gemm_core(ctx, a);
}

}  // namespace falkon
