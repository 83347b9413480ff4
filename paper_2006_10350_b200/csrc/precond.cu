// precond.cu — the Falkon preconditioner in ONE m x m fp64 buffer, hand-written for sm_100a.
//
// Alg. 1 lines 13-17, Eq. (7), in-place layout of
// PAPER.md:257-265 / Fig. 3:
//   (b) Kmm (+ delta I) computed block-wise in fp64 into the UPPER triangle
//   (c) in-place Cholesky of the upper triangle -> T, with Kmm + delta I = T^T T
//   (d) T T^T / m + lambda I computed block-wise into the LOWER triangle
//   (e) in-place Cholesky of the lower triangle -> A^T, with T T^T/m + lambda I = A^T A
// The two diagonals are kept in the vectors diagT / diagA ("additional care ... matrix
// diagonal"; reading c6).
//
// Both factorizations are the SAME lower Cholesky  S = L L^T  run through a "view":
//   factor T:  L = T^T, logical L(i,j) (i >= j) stored at P[j*ld + i]   (trans = 1)
//   factor A:  L = A^T, logical L(i,j)          stored at P[i*ld + j]   (trans = 0)
// Right-looking blocked algorithm with NB = 128 (PAPER.md:462-466 describes the tile
// version): per block column k
//   1. diag kernel: Cholesky of the 128 x 128 diagonal block in shared memory and its
//      triangular inverse W = L_kk^-1 (both in place, one CTA);
//   2. panel:   L_ik = S_ik W^T                     (fp64 GEMM)
//   3. trailing S_ij -= L_ik L_jk^T, lower tiles    (fp64 GEMM)
// All GEMM-like work runs in one register-tiled fp64 FMA kernel (128 x 128 CTA tile,
// 8 x 8 outputs per thread).  The triangular solves of each CG step (Alg. 1 lines 5, 7,
// 9, 11) are a single-kernel "sync-free" blocked TRSV: CTAs take row blocks in ticket
// order and wait on per-block ready flags, so the solve streams the triangle at HBM rate
// while the dependency chain advances block by block.
#include <math.h>

#include <algorithm>

#include <cuda.h>

#include <vector>

#include "common.cuh"
#include "precond.cuh"

namespace falkon {

constexpr int NB = 128;        // factorization block
constexpr int GT = 128;        // GEMM CTA tile
constexpr int GK = 16;         // GEMM k-chunk (32 with 3 stages measured 7% slower)
constexpr int GSTAGES = 4;     // cp.async pipeline depth of the fp64 GEMM
constexpr int GPAD = 4;        // smem row padding (doubles): row stride = 8 banks (mod 32), so the
                               // 4 k-rows x 4 doubles of a half-warp DMMA fragment load hit 32
                               // distinct banks (GPAD = 8 measured 2-way conflicts in ncu)
constexpr int TB = 64;         // TRSV block

int64_t precond_work_elems(int64_t m);

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// views: precond.cuh

// ------------------------------------------------------------------ Kmm (step b)
// Logical lower triangle of S = Kmm + delta I written through view `S` (+ its diagonal).
// fp64 direct differences on the fp32 inputs (exact upcast), 64 x 64 tiles.
__global__ void __launch_bounds__(256) kmm_kernel(const float *__restrict__ C, int64_t m, int64_t d,
                                                  int kernel, double inv2s2, double invs,
                                                  double jitter, View S) {
  // triangular tile decode: blockIdx.x -> (ti >= tj)
  const int64_t t = blockIdx.x;
  int64_t ti = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int64_t tj = t - ti * (ti + 1) / 2;
  const int64_t r0 = ti * 64, c0 = tj * 64;
  __shared__ double sa[32][65];
  __shared__ double sb[32][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < d; k0 += 32) {
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int rr = e / 32, kk = e % 32;
      const int64_t k = k0 + kk;
      sa[kk][rr] = (r0 + rr < m && k < d) ? (double)C[(r0 + rr) * d + k] : 0.0;
      sb[kk][rr] = (c0 + rr < m && k < d) ? (double)C[(c0 + rr) * d + k] : 0.0;
    }
    __syncthreads();
    const int kn = (int)lmin(32, d - k0);
    for (int kk = 0; kk < kn; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double df = a[i] - b[j];
          acc[i][j] = fma(df, df, acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = r0 + ty * 4 + i, c = c0 + tx * 4 + j;
      if (r < m && c < m && r >= c) {
        const double D = acc[i][j];
        double kv = kernel == FALKON_GAUSSIAN ? exp(-D * inv2s2) : exp(-sqrt(D) * invs);
        if (r == c) kv += jitter;
        vset(S, r, c, kv);
      }
    }
}

// ------------------------------------------------------------------ diagonal block (step 1)
// Cholesky of the nb x nb diagonal block at [k0, k0+nb) of view S, in shared memory, then
// the in-place triangular inverse W = L^-1 written (dense, row-major, zeros above the
// diagonal) to `W`.  Pivot failures record the first global column in *fail.
__global__ void __launch_bounds__(512) potrf_diag_kernel(View S, int64_t k0, int nb,
                                                         double *__restrict__ W,
                                                         double *__restrict__ Dinv,
                                                         unsigned long long *fail) {
  extern __shared__ double sL[];  // nb x (nb+1)
  const int ld = nb + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  // element order follows the view's storage (coalesced for both orientations)
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = S.trans ? e % nb : e / nb, c = S.trans ? e / nb : e % nb;
    sL[r * ld + c] = (r >= c) ? vget(S, k0 + r, k0 + c) : 0.0;
  }
  __syncthreads();
  // unblocked right-looking Cholesky; the rank-1 update runs on a 16 x 32 thread grid
  const int ty = tid >> 5, tx = tid & 31;
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double p = sL[j * ld + j];
      if (!(p > 0.0) || !isfinite(p)) {
        atomicMin(fail, (unsigned long long)(k0 + j));
        sL[j * ld + j] = nan("");
      } else {
        sL[j * ld + j] = sqrt(p);
      }
    }
    __syncthreads();
    const double rjj = 1.0 / sL[j * ld + j];
    for (int i = j + 1 + tid; i < nb; i += nt) sL[i * ld + j] *= rjj;
    __syncthreads();
    for (int i = j + 1 + ty; i < nb; i += nt / 32) {
      const double lij = sL[i * ld + j];
      for (int k = j + 1 + tx; k <= i; k += 32) sL[i * ld + k] = fma(-lij, sL[k * ld + j], sL[i * ld + k]);
    }
    __syncthreads();
  }
  // write L back (lower + diag)
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = S.trans ? e % nb : e / nb, c = S.trans ? e / nb : e % nb;
    if (r >= c) vset(S, k0 + r, k0 + c, sL[r * ld + c]);
  }
  __syncthreads();
  // W = L^-1 by column-parallel forward substitution, 4 lanes per column (nb <= 128, 512
  // threads): W(c,c) = 1/L(c,c);  W(i,c) = -(sum_{c<=k<i} L(i,k) W(k,c)) / L(i,i).
  // W(i,c), i > c, is kept transposed in the free upper triangle (sL[c][i]), its diagonal in
  // wd[], and moved over L once complete.
  __shared__ double wd[NB];
  {
    const int c = tid >> 2, sub = tid & 3;
    const bool act = c < nb;
    for (int i = 0; i < nb; ++i) {
      double acc = 0.0;
      if (act && i > c) {
        int k = c + sub;
        if (sub == 0) {
          acc = sL[i * ld + c] * wd[c];
          k += 4;
        }
        for (; k < i; k += 4) acc = fma(sL[i * ld + k], sL[c * ld + k], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (act && sub == 0 && i >= c) {
        const double rii = 1.0 / sL[i * ld + i];
        if (i == c) wd[c] = rii;
        else sL[c * ld + i] = -acc * rii;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = e / nb, c = e % nb;
    if (r > c) sL[r * ld + c] = sL[c * ld + r];
    else if (r == c) sL[r * ld + r] = wd[r];
  }
  __syncthreads();
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = e / nb, c = e % nb;
    W[(int64_t)r * NB + c] = (r >= c) ? sL[r * ld + c] : 0.0;
  }
  // the 64 x 64 diagonal sub-blocks of W are the inverses of the 64 x 64 diagonal blocks of
  // L (block-triangular inverse): kept for the triangular solves of the CG loop
  if (Dinv) {
    for (int e = tid; e < NB * TB; e += nt) {
      const int r = e / TB, c = e % TB;  // r in [0, 128), c in [0, 64)
      const int h = r / TB, rr = r % TB;
      const int gc = h * TB + c;
      double v = 0.0;
      if (r < nb && gc < nb && rr >= c) v = sL[r * ld + gc];
      if (h * TB < nb) Dinv[(k0 / TB + h) * (int64_t)(TB * TB) + rr * TB + c] = v;
    }
  }
}

// ------------------------------------------------------------------ fp64 GEMM through views
// GemmArgs (precond.cuh): C = alpha A B^T + beta C through views.

// Asynchronous (cp.async, LDGSTS) staging of a GT x GK chunk of a view into shared memory:
// masked elements are zero-filled (src-size 0), diagonal elements read from the view's dvec.
__device__ __forceinline__ void cp_async8z(void *smem, const void *gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ const double *vsrc(const View &v, int64_t r, int64_t c, bool &valid) {
  if (v.tri == 1) {
    if (r < c) { valid = false; return v.base; }
    if (r == c) { valid = true; return v.dvec + r; }
  } else if (v.tri == 2) {
    if (c < r) { valid = false; return v.base; }
    if (r == c) { valid = true; return v.dvec + r; }
  }
  valid = true;
  return v.base + vidx(v, r, c);
}
// true iff every element (r, c), r in [r0, r0+nr), c in [c0, c0+nc) lies in the stored
// (strict) triangle of the view, i.e. needs neither masking nor the diagonal vector
__device__ __forceinline__ bool view_dense(const View &v, int64_t r0, int64_t nr, int64_t c0,
                                           int64_t nc) {
  if (v.tri == 1) return r0 > c0 + nc - 1;
  if (v.tri == 2) return c0 > r0 + nr - 1;
  return true;
}
// masked / diagonal-touching chunks (rare): kept out of line to keep the hot loop small
template <int NTHR, int ROWS>
__device__ __noinline__ void gemm_async_chunk_masked(const View v, double (*s)[ROWS + GPAD],
                                                     int64_t row0, int64_t rmax, int64_t k,
                                                     int64_t kmax) {
  const int tid = threadIdx.x;
  constexpr int RP = NTHR / GK;  // rows per pass (storage contiguous along k)
  constexpr int KP = NTHR / ROWS;  // k-rows per pass (storage contiguous along rows)
  if (!v.trans) {
    const int kk = tid % GK, rr = tid / GK;
    for (int p = 0; p < ROWS / RP; ++p) {
      const int64_t r = row0 + rr + RP * p, kg = k + kk;
      bool ok = r < rmax && kg < kmax;
      const double *src = ok ? vsrc(v, r, kg, ok) : v.base;
      cp_async8z(&s[kk][rr + RP * p], src, ok);
    }
  } else {
    const int rr = tid % ROWS, kk = tid / ROWS;
    for (int p = 0; p < GK / KP; ++p) {
      const int64_t r = row0 + rr, kg = k + kk + KP * p;
      bool ok = r < rmax && kg < kmax;
      const double *src = ok ? vsrc(v, r, kg, ok) : v.base;
      cp_async8z(&s[kk + KP * p][rr], src, ok);
    }
  }
}

template <int NTHR, int ROWS>
__device__ __forceinline__ void gemm_async_chunk(const View &v, double (*s)[ROWS + GPAD],
                                                 int64_t row0, int64_t rmax, int64_t k,
                                                 int64_t kmax) {
  const int tid = threadIdx.x;
  if (view_dense(v, row0, ROWS, k, GK)) {
    // branch-free: out-of-range rows/columns are zero-filled from a clamped address
    constexpr int RP = NTHR / GK;
    constexpr int KP = NTHR / ROWS;
    if (!v.trans) {
      const int kk = tid % GK, rr = tid / GK;
      const int64_t kg = k + kk;
      const bool kok = kg < kmax;
      const int64_t kc = kok ? kg : k;
#pragma unroll
      for (int p = 0; p < ROWS / RP; ++p) {
        const int64_t r = row0 + rr + RP * p;
        const bool ok = kok && r < rmax;
        cp_async8z(&s[kk][rr + RP * p], v.base + (ok ? r : row0) * v.ld + kc, ok);
      }
    } else {
      const int rr = tid % ROWS, kk = tid / ROWS;
      const int64_t r = row0 + rr;
      const bool rok = r < rmax;
      const int64_t rc = rok ? r : row0;
#pragma unroll
      for (int p = 0; p < GK / KP; ++p) {
        const int64_t kg = k + kk + KP * p;
        const bool ok = rok && kg < kmax;
        cp_async8z(&s[kk + KP * p][rr], v.base + (ok ? kg : k) * v.ld + rc, ok);
      }
    }
    return;
  }
  gemm_async_chunk_masked<NTHR, ROWS>(v, s, row0, rmax, k, kmax);
}

template <int TN>
__device__ __noinline__ void gemm_epilogue(const GemmArgs a, const double *sC, int64_t i0,
                                           int64_t j0, int tid, int nthr) {
  constexpr int CLD = TN + 1;
  constexpr int BATCH = 8;  // independent reads in flight per thread
  for (int e0 = tid; e0 < GT * TN; e0 += BATCH * nthr) {
    double cv[BATCH];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int e = e0 + u * nthr;
      const int li_t = a.C.trans ? (e % GT) : (e / TN);
      const int lj_t = a.C.trans ? (e / GT) : (e % TN);
      const int64_t li = i0 + li_t, lj = j0 + lj_t;
      cv[u] = 0.0;
      if (e < GT * TN && li < a.M && lj < a.N && a.beta != 0.0)
        cv[u] = vget(a.C, a.rc + li, a.cc + lj);
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      // storage order: consecutive threads walk the contiguous dimension of C's storage
      const int e = e0 + u * nthr;
      const int li_t = a.C.trans ? (e % GT) : (e / TN);
      const int lj_t = a.C.trans ? (e / GT) : (e % TN);
      const int64_t li = i0 + li_t, lj = j0 + lj_t;
      if (e >= GT * TN || li >= a.M || lj >= a.N) continue;
      const int64_t r = a.rc + li, c = a.cc + lj;
      if (a.C.tri == 1 && r < c) continue;
      if (a.C.tri == 2 && c < r) continue;
      vset(a.C, r, c, a.alpha * sC[li_t * CLD + lj_t] + a.beta * cv[u]);
    }
  }
}

// D(8x8) += A(8x4) B(4x8) on the FP64 tensor path (DMMA).  Fragments (lane t):
//   a = A[t/4][t%4], b = B[t%4][t/4], d = {D[t/4][2(t%4)], D[t/4][2(t%4)+1]}
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// CTA tile 128 x TN (TN = 8 NT WN), 4 x WN warps, warp tile 32 x (8 NT) = 4 x NT DMMA tiles:
//   <2, 8>: 8 warps, 128 x 128, 32 x 64 warp tiles (12 fragments per 32 MMAs), 1 CTA / SM;
//   <4, 4>: 16 warps, 128 x 128, 32 x 32 warp tiles, 1 CTA / SM;
//   <2, 4>: 8 warps, 128 x 64, 32 x 32 warp tiles, 2 CTAs / SM (<= 128 registers): the two
//           CTAs' barriers, prologues and epilogues interleave, so the DMMA pipe (one DMMA per
//           16 cycles per warp, SASS stall count 15) keeps >= 2 issuing warps per SMSP.
// k-chunks of GK are staged global -> shared with cp.async (GSTAGES deep) through the views.
template <int WN, int NT>
__global__ void __launch_bounds__(128 * WN, (WN == 2 && NT == 4) ? 2 : 1)
    gemm_f64_kernel(GemmArgs a) {
  constexpr int NTHR = 128 * WN;
  constexpr int TN = 8 * NT * WN;
  constexpr int R = GT / TN;  // column tiles per 128-row tile width
  int64_t ti, tj;
  if (a.tri_tiles) {
    // row tile ti holds R (ti + 1) column tiles of the lower region
    const int64_t t = blockIdx.x;
    ti = (int64_t)((sqrt(8.0 * (double)t / R + 1.0) - 1.0) * 0.5);
    while (R * (ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (R * ti * (ti + 1) / 2 > t) --ti;
    tj = t - R * ti * (ti + 1) / 2;
  } else {
    ti = blockIdx.y;
    tj = blockIdx.x;
  }
  const int64_t i0 = ti * GT, j0 = tj * TN;
  if (i0 >= a.M || j0 >= a.N) return;
  const int64_t kb = a.k_from_row ? lmax(a.k0, a.ra + i0) : a.k0;
  const int64_t ke = a.k1;

  extern __shared__ __align__(16) double gsm[];
  double(*As)[GK][GT + GPAD] = reinterpret_cast<double(*)[GK][GT + GPAD]>(gsm);
  double(*Bs)[GK][TN + GPAD] =
      reinterpret_cast<double(*)[GK][TN + GPAD]>(gsm + GSTAGES * GK * (GT + GPAD));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp / WN, wc = warp % WN;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][NT][2];
  // Tiles strictly inside C's triangle (the vast majority) accumulate on top of C itself:
  // acc starts at (beta/alpha) C, loaded here so the loads overlap the pipeline fill, and the
  // epilogue is a plain store of alpha * acc (no read-modify-write round trips).
  const bool cdense = view_dense(a.C, a.rc + i0, GT, a.cc + j0, TN) && i0 + GT <= a.M &&
                      j0 + TN <= a.N;
  const int64_t csr = a.C.trans ? 1 : a.C.ld, csc = a.C.trans ? a.C.ld : 1;
  double *cfrag =
      a.C.base + (a.rc + i0 + wr * 32 + g) * csr + (a.cc + j0 + wc * (8 * NT) + 2 * q) * csc;
  if (cdense && a.beta != 0.0) {
    const double sb = a.beta / a.alpha;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[mt][nt][h] = sb * cfrag[(mt * 8) * csr + (nt * 8 + h) * csc];
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }

  const int64_t ra = a.ra + i0, rb = a.rb + j0;
  const int64_t ramax = a.ra + a.M, rbmax = a.rb + a.N;
  const int nch = ke > kb ? (int)cdiv<int64_t>(ke - kb, GK) : 0;
  // GSTAGES-deep cp.async pipeline: chunk c+GSTAGES-1 loads while chunk c is multiplied
#pragma unroll
  for (int c = 0; c < GSTAGES - 1; ++c) {
    if (c < nch) {
      gemm_async_chunk<NTHR, GT>(a.A, As[c], ra, ramax, kb + (int64_t)c * GK, ke);
      gemm_async_chunk<NTHR, TN>(a.B, Bs[c], rb, rbmax, kb + (int64_t)c * GK, ke);
    }
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    if (a.kscale) {  // T D T^T of Alg. 2: scale the staged B chunk by D(k)
      const int st = c % GSTAGES;
      const int64_t kc = kb + (int64_t)c * GK;
      for (int e = tid; e < GK * TN; e += NTHR) {
        const int kk = e / TN, j = e % TN;
        if (kc + kk < ke) Bs[st][kk][j] *= a.kscale[kc + kk];
      }
      __syncthreads();
    }
    {
      const int cn = c + GSTAGES - 1;
      if (cn < nch) {
        gemm_async_chunk<NTHR, GT>(a.A, As[cn % GSTAGES], ra, ramax, kb + (int64_t)cn * GK, ke);
        gemm_async_chunk<NTHR, TN>(a.B, Bs[cn % GSTAGES], rb, rbmax, kb + (int64_t)cn * GK, ke);
      }
      cp_async_commit();
    }
    const int st = c % GSTAGES;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      double af[4], bf[NT];
      const double *arow = &As[st][ks * 4 + q][wr * 32 + g];
      const double *brow = &Bs[st][ks * 4 + q][wc * (8 * NT) + g];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = arow[mt * 8];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = brow[nt * 8];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt], bf[nt]);
    }
  }
  cp_async_wait<0>();
  // epilogue: the accumulator tile is staged in shared memory (the pipeline buffers are
  // free now), then written through the C view in storage order (coalesced), with the
  // view's triangle mask and diagonal vector applied element-wise.
  if (cdense) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          cfrag[(mt * 8) * csr + (nt * 8 + h) * csc] = a.alpha * acc[mt][nt][h];
    return;
  }
  __syncthreads();
  double *sC = gsm;  // [GT][TN + 1]
  constexpr int CLD = TN + 1;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        sC[(wr * 32 + mt * 8 + g) * CLD + wc * (8 * NT) + nt * 8 + 2 * q + h] = acc[mt][nt][h];
  __syncthreads();
  gemm_epilogue<TN>(a, sC, i0, j0, threadIdx.x, blockDim.x);
}

// ------------------------------------------------------------------ TMA-fed variant
// For the big GEMMs (trailing updates, LAUUM: A and B are the same view of the m x m buffer):
// 128 x 64 CTA tile, 8 compute warps of 32 x 32 and one producer warp, 1 CTA per SM, an
// 8-stage ring of 24 KB k-chunks.  The producer loads each dense chunk operand with ONE 2-D
// tensor-map TMA: a non-transposed view (k contiguous) as [rows][16 k] with SWIZZLE_128B
// (conflict-free fragment loads), a transposed view (rows contiguous) as [16 k][rows]; chunks
// touching the diagonal, masked parts or the k tail fall back to per-element cp.async in the
// same layout.  Compute warps only wait on mbarriers, load fragments and issue DMMAs.  Same k
// order per accumulator as gemm_f64_kernel: bitwise-identical results.
constexpr int TM_TN = 64;
constexpr int TM_STAGES = 8;
// doubles per chunk operand: [rows][16 k] swizzled, or [16 k][rows + 4] for a transposed view
// (the TMA box is 4 elements wider than the tile, so the rows land padded — the same
// conflict-free fragment layout as gemm_f64_kernel; the 4 extra values are never read)
template <int TRANS, int ROWS>
constexpr int tm_elems() { return TRANS ? GK * (ROWS + GPAD) : ROWS * GK; }
struct TmaMaps {
  CUtensorMap a, b;
};
__device__ __forceinline__ void tma2d_g2s(void *dst, const CUtensorMap *map, int c0, int c1,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// byte offset of chunk element (r, k) in the stage layout
template <int TRANS, int ROWS>
__device__ __forceinline__ uint32_t tm_off(int r, int k) {
  if (TRANS) return (uint32_t)(k * (ROWS + GPAD) + r) * 8u;
  return (uint32_t)(r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3));
}
template <int TRANS, int ROWS>
__device__ __forceinline__ void tm_slow(const View &v, uint8_t *s, int64_t row0, int64_t rmax,
                                        int64_t k, int64_t kmax, int lane) {
  for (int e = lane; e < ROWS * GK; e += 32) {
    const int rr = TRANS ? e % ROWS : e / GK, kk = TRANS ? e / ROWS : e % GK;
    const int64_t r = row0 + rr, kg = k + kk;
    bool ok = r < rmax && kg < kmax;
    const double *src = ok ? vsrc(v, r, kg, ok) : v.base;
    cp_async8z(s + tm_off<TRANS, ROWS>(rr, kk), src, ok);
  }
}

template <int TRANS>
__global__ void __launch_bounds__(288, 1)
    gemm_f64_tma_kernel(const __grid_constant__ TmaMaps maps, GemmArgs a) {
  constexpr int TN = TM_TN, NT = 4, WN = 2;
  constexpr int R = GT / TN;
  int64_t ti, tj;
  if (a.tri_tiles) {
    const int64_t t = blockIdx.x;
    ti = (int64_t)((sqrt(8.0 * (double)t / R + 1.0) - 1.0) * 0.5);
    while (R * (ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (R * ti * (ti + 1) / 2 > t) --ti;
    tj = t - R * ti * (ti + 1) / 2;
  } else {
    ti = blockIdx.y;
    tj = blockIdx.x;
  }
  const int64_t i0 = ti * GT, j0 = tj * TN;
  if (i0 >= a.M || j0 >= a.N) return;
  const int64_t kb = a.k_from_row ? lmax(a.k0, a.ra + i0) : a.k0;
  const int64_t ke = a.k1;
  const int nch = ke > kb ? (int)cdiv<int64_t>(ke - kb, GK) : 0;

  extern __shared__ __align__(1024) uint8_t tsm_raw[];
  uint8_t *tsm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  constexpr int TM_A = tm_elems<TRANS, GT>(), TM_B = tm_elems<TRANS, TM_TN>();
  constexpr int STAGE_B = (TM_A + TM_B) * 8;
  uint64_t *full = reinterpret_cast<uint64_t *>(tsm + TM_STAGES * STAGE_B);
  uint64_t *empty = full + TM_STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int st = 0; st < TM_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ra = a.ra + i0, rb = a.rb + j0;
  const int64_t ramax = a.ra + a.M, rbmax = a.rb + a.N;

  if (warp == 8) {  // producer
    for (int c = 0; c < nch; ++c) {
      const int st = c % TM_STAGES;
      mbar_wait(&empty[st], ((c / TM_STAGES) & 1) ^ 1);
      const int64_t kc = kb + (int64_t)c * GK;
      uint8_t *sa = tsm + st * STAGE_B, *sb = sa + TM_A * 8;
      const bool kfull = kc + GK <= ke;
      const bool fa = kfull && view_dense(a.A, ra, GT, kc, GK);
      const bool fb = kfull && view_dense(a.B, rb, TN, kc, GK);
      if (!fa) tm_slow<TRANS, GT>(a.A, sa, ra, ramax, kc, ke, lane);
      if (!fb) tm_slow<TRANS, TN>(a.B, sb, rb, rbmax, kc, ke, lane);
      if (!(fa && fb)) asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(&full[st], (fa ? TM_A * 8 : 0) + (fb ? TM_B * 8 : 0));
        // TRANS: coords {row (inner), k}; else {k (inner), row}
        if (fa) tma2d_g2s(sa, &maps.a, TRANS ? (int)ra : (int)kc, TRANS ? (int)kc : (int)ra, &full[st]);
        if (fb) tma2d_g2s(sb, &maps.b, TRANS ? (int)rb : (int)kc, TRANS ? (int)kc : (int)rb, &full[st]);
      }
      __syncwarp();
    }
    return;
  }

  const int wr = warp / WN, wc = warp % WN;
  const int g = lane >> 2, q = lane & 3;
  double acc[4][NT][2];
  const bool cdense = view_dense(a.C, a.rc + i0, GT, a.cc + j0, TN) && i0 + GT <= a.M &&
                      j0 + TN <= a.N;
  const int64_t csr = a.C.trans ? 1 : a.C.ld, csc = a.C.trans ? a.C.ld : 1;
  double *cfrag =
      a.C.base + (a.rc + i0 + wr * 32 + g) * csr + (a.cc + j0 + wc * (8 * NT) + 2 * q) * csc;
  if (cdense && a.beta != 0.0) {
    const double sb = a.beta / a.alpha;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[mt][nt][h] = sb * cfrag[(mt * 8) * csr + (nt * 8 + h) * csc];
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  for (int c = 0; c < nch; ++c) {
    const int st = c % TM_STAGES;
    mbar_wait(&full[st], (c / TM_STAGES) & 1);
    const uint8_t *sa = tsm + st * STAGE_B, *sb = sa + TM_A * 8;
    const int64_t kc = kb + (int64_t)c * GK;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      const int kq = ks * 4 + q;
      double af[4], bf[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
        af[mt] = *reinterpret_cast<const double *>(sa + tm_off<TRANS, GT>(wr * 32 + mt * 8 + g, kq));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        bf[nt] = *reinterpret_cast<const double *>(sb + tm_off<TRANS, TN>(wc * (8 * NT) + nt * 8 + g, kq));
      if (a.kscale) {  // T D T^T of Alg. 2: B(j, k) D(k) on the fragment
        const int64_t kk = kc + kq;
        const double sc = kk < ke ? __ldg(a.kscale + kk) : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bf[nt] *= sc;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (cdense) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          cfrag[(mt * 8) * csr + (nt * 8 + h) * csc] = a.alpha * acc[mt][nt][h];
    return;
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");  // all compute warps are past the ring
  double *sC = reinterpret_cast<double *>(tsm);  // [GT][TN + 1]
  constexpr int CLD = TN + 1;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        sC[(wr * 32 + mt * 8 + g) * CLD + wc * (8 * NT) + nt * 8 + 2 * q + h] = acc[mt][nt][h];
  asm volatile("bar.sync 1, 256;" ::: "memory");
  gemm_epilogue<TN>(a, sC, i0, j0, tid, 256);
}

typedef CUresult (*PFN_encodeTiled_p)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);
static PFN_encodeTiled_p encode_fn() {
  static const PFN_encodeTiled_p fn = []() -> PFN_encodeTiled_p {  // thread-safe one-time lookup
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (PFN_encodeTiled_p)p;
    cudaGetLastError();
    return nullptr;
  }();
  return fn;
}
// map of view v's storage (an ld x ld square of doubles) for chunks of `rows` x GK
static bool tm_map(CUtensorMap *map, const View &v, int64_t extent, int rows) {
  PFN_encodeTiled_p enc = encode_fn();
  if (!enc || (v.ld & 1) || (reinterpret_cast<uintptr_t>(v.base) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)v.ld, (cuuint64_t)extent};
  cuuint64_t strides[1] = {(cuuint64_t)v.ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)(v.trans ? rows + GPAD : GK), (cuuint32_t)(v.trans ? GK : rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)v.base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE,
             v.trans ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// true if launched (A and B the same square view with even ld), false: use the generic kernel
static bool gemm_launch_tma(falkon_ctx *ctx, const GemmArgs &a, int *rc) {
  *rc = FALKON_OK;
  if (a.A.base != a.B.base || a.A.trans != a.B.trans || a.A.ld != a.B.ld) return false;
  TmaMaps maps;
  if (!tm_map(&maps.a, a.A, a.A.ld, GT) || !tm_map(&maps.b, a.B, a.B.ld, TM_TN)) return false;
  constexpr int TN = TM_TN, R = GT / TN;
  const size_t smem = 1024 + (size_t)TM_STAGES * 8 *
                                 (a.A.trans ? tm_elems<1, GT>() + tm_elems<1, TM_TN>()
                                            : tm_elems<0, GT>() + tm_elems<0, TM_TN>()) +
                      16 * TM_STAGES;
  auto fn = a.A.trans ? gemm_f64_tma_kernel<1> : gemm_f64_tma_kernel<0>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    *rc = fail(FALKON_ECUDA, "gemm_f64_tma_kernel smem attribute");
    return true;
  }
  const int64_t tm = cdiv<int64_t>(a.M, GT), tn = cdiv<int64_t>(a.N, TN);
  LaunchScope ls(ctx, FALKON_T_PRECOND);
  if (a.tri_tiles)
    fn<<<(unsigned)(R * tm * (tm + 1) / 2), 288, smem, ctx->stream>>>(maps, a);
  else
    fn<<<dim3((unsigned)tn, (unsigned)tm), 288, smem, ctx->stream>>>(maps, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) *rc = fail(FALKON_ECUDA, std::string("gemm_f64_tma_kernel: ") + cudaGetErrorString(e));
  return true;
}

template <int WN, int NT>
static int gemm_launch(falkon_ctx *ctx, const GemmArgs &a) {
  constexpr int TN = 8 * NT * WN, R = GT / TN;
  const size_t smem = sizeof(double) * GSTAGES * GK * (GT + TN + 2 * GPAD);
  FK_CUDA(cudaFuncSetAttribute(gemm_f64_kernel<WN, NT>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t tm = cdiv<int64_t>(a.M, GT), tn = cdiv<int64_t>(a.N, TN);
  LaunchScope ls(ctx, FALKON_T_PRECOND);
  if (a.tri_tiles) {
    gemm_f64_kernel<WN, NT><<<(unsigned)(R * tm * (tm + 1) / 2), 128 * WN, smem, ctx->stream>>>(a);
  } else {
    gemm_f64_kernel<WN, NT><<<dim3((unsigned)tn, (unsigned)tm), 128 * WN, smem, ctx->stream>>>(a);
  }
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

static int gemm(falkon_ctx *ctx, const GemmArgs &a) {
  if (a.M <= 0 || a.N <= 0) return FALKON_OK;
  {  // FALKON_OPT_OZAKI: int8 tensor-core emulation (ozaki.cu) where it applies
    const int rc = oz_gemm(ctx, a);
    if (rc != OZ_DECLINED) return rc;
  }
  if (ctx->opt.gemm_warps == 5) {  // TMA-fed warp-specialised kernel where it applies
    int rc;
    if (gemm_launch_tma(ctx, a, &rc)) return rc;
  }
  switch (ctx->opt.gemm_warps) {
    case 16: return gemm_launch<4, 4>(ctx, a);
    case 2: return gemm_launch<2, 4>(ctx, a);  // 2 CTAs of 8 warps per SM
    default: return gemm_launch<2, 8>(ctx, a);
  }
}

// ------------------------------------------------------------------ blocked Cholesky
// Inner steps of one outer panel [K0, K1): per 128-column block, the diagonal factor + inverse,
// the panel solve (GEMM with W = L_kk^-1) and the update of the rest of the outer panel.
static int potrf_panel(falkon_ctx *ctx, View S, int64_t m, int64_t K0, int64_t K1, double *Wbuf,
                       double *Dinv, unsigned long long *fail, size_t dsm) {
  View W{Wbuf, NB, 0, 0, nullptr};
  for (int64_t k0 = K0; k0 < K1; k0 += NB) {
    const int nb = (int)std::min<int64_t>(NB, m - k0);
    {
      LaunchScope ls(ctx, FALKON_T_PRECOND);
      potrf_diag_kernel<<<1, 512, dsm, ctx->stream>>>(S, k0, nb, Wbuf, Dinv, fail);
    }
    FK_LAUNCH_CHECK();
    const int64_t k1 = k0 + nb, rem = m - k1;
    if (rem <= 0) break;
    GemmArgs p{};
    p.A = S;
    p.B = W;
    p.C = S;
    p.M = rem;
    p.N = nb;
    p.ra = k1;
    p.rb = 0;
    p.rc = k1;
    p.cc = k0;
    p.k0 = k0;
    p.k1 = k1;
    p.B.base = Wbuf - k0;
    p.alpha = 1.0;
    p.beta = 0.0;
    FK_TRY(gemm(ctx, p));
    if (k1 < K1) {
      GemmArgs u{};
      u.A = S;
      u.B = S;
      u.C = S;
      u.M = rem;
      u.N = K1 - k1;
      u.ra = k1;
      u.rb = k1;
      u.rc = k1;
      u.cc = k1;
      u.k0 = k0;
      u.k1 = k1;
      u.alpha = -1.0;
      u.beta = 1.0;
      FK_TRY(gemm(ctx, u));
    }
  }
  return FALKON_OK;
}

// S(c0:, c0:c1) -= L(c0:, K0:K1) L(c0:c1, K0:K1)^T restricted to the lower triangle: columns
// [c0, c1) of the trailing matrix (c1 = m with tri tiles for the whole rest).
static int potrf_update(falkon_ctx *ctx, View S, int64_t m, int64_t K0, int64_t K1, int64_t c0,
                        int64_t c1) {
  if (c0 >= c1) return FALKON_OK;
  GemmArgs t{};
  t.A = S;
  t.B = S;
  t.C = S;
  t.M = m - c0;
  t.N = c1 - c0;
  t.ra = c0;
  t.rb = c0;
  t.rc = c0;
  t.cc = c0;
  t.k0 = K0;
  t.k1 = K1;
  t.tri_tiles = c1 == m ? 1 : 0;
  t.alpha = -1.0;
  t.beta = 1.0;
  return gemm(ctx, t);
}

// Lookahead (the classic right-looking schedule with depth 1): after outer panel j, the update
// of the NEXT panel's columns (a_j) runs on the high-priority stream right away and panel j+1
// is factored there, while the bulk of the trailing update (b_j, columns beyond panel j+1) runs
// on the low-priority stream.  Ordering: b_j waits for panel j (event P_j); a_j waits for
// b_{j-1} (both write panel j+1's columns); panel j+1 follows a_j on the same stream and
// b_{j-1} covered its columns' older updates.  The diagonal-block factorisations and small
// panel GEMMs (latency-bound, a few SMs) thus hide under the big GEMM.
static int potrf_lookahead(falkon_ctx *ctx, View S, int64_t m, double *Wbuf, double *Dinv,
                           unsigned long long *failw) {
  const size_t dsm = sizeof(double) * NB * (NB + 1);
  FK_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dsm));
  if (!ctx->hi_stream) {
    int least = 0, greatest = 0;
    FK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    FK_CUDA(cudaStreamCreateWithPriority(&ctx->hi_stream, cudaStreamNonBlocking, greatest));
    FK_CUDA(cudaStreamCreateWithPriority(&ctx->lo_stream, cudaStreamNonBlocking, least));
  }
  const int NBO = NB * potrf_outer(ctx);
  const int64_t nob = cdiv<int64_t>(m, NBO);
  std::vector<cudaEvent_t> ev((size_t)(2 * nob + 2));
  for (auto &e : ev) FK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t *evP = ev.data(), *evB = ev.data() + nob, *evFork = ev.data() + 2 * nob,
              *evEnd = evFork + 1;
  cudaStream_t base = ctx->stream, hi = ctx->hi_stream, lo = ctx->lo_stream;
  int rc = FALKON_OK;
  auto on = [&](cudaStream_t s) { ctx->stream = s; };
  do {
    if (cudaEventRecord(*evFork, base) != cudaSuccess) {
      rc = fail(FALKON_ECUDA, "cudaEventRecord (potrf fork)");
      break;
    }
    cudaStreamWaitEvent(hi, *evFork, 0);
    cudaStreamWaitEvent(lo, *evFork, 0);
    for (int64_t j = 0; j < nob; ++j) {
      const int64_t K0 = j * NBO, K1 = std::min<int64_t>(K0 + NBO, m);
      const int64_t K2 = std::min<int64_t>(K1 + NBO, m);
      on(hi);
      if ((rc = potrf_panel(ctx, S, m, K0, K1, Wbuf, Dinv, failw, dsm))) break;
      if (K1 >= m) break;
      cudaEventRecord(evP[j], hi);
      if (j > 0) cudaStreamWaitEvent(hi, evB[j - 1], 0);
      if ((rc = potrf_update(ctx, S, m, K0, K1, K1, K2))) break;  // a_j: next panel's columns
      if (K2 < m) {
        on(lo);
        cudaStreamWaitEvent(lo, evP[j], 0);
        if ((rc = potrf_update(ctx, S, m, K0, K1, K2, m))) break;  // b_j: the rest
      }
      cudaEventRecord(evB[j], lo);
    }
    // join both streams back into the caller's stream
    cudaEventRecord(*evEnd, hi);
    cudaStreamWaitEvent(base, *evEnd, 0);
    cudaEventRecord(*evEnd, lo);
    cudaStreamWaitEvent(base, *evEnd, 0);
  } while (0);
  ctx->stream = base;
  for (auto &e : ev) cudaEventDestroy(e);
  if (rc == FALKON_OK) FK_LAUNCH_CHECK();
  return rc;
}

static int potrf(falkon_ctx *ctx, View S, int64_t m, double *Wbuf, double *Dinv,
                 unsigned long long *fail) {
  const size_t dsm = sizeof(double) * NB * (NB + 1);
  FK_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dsm));
  View W{Wbuf, NB, 0, 0, nullptr};
  // Two-level right-looking blocking: inner NB = 128 steps (diagonal factor + inverse, panel
  // solve as a GEMM with W = L_kk^-1, update of the rest of the NBO-wide outer panel only),
  // then one trailing update of the remaining matrix with K = NBO (FALKON_OPT_POTRF_OUTER x 128;
  // fewer passes
  // over the trailing matrix and doubles the GEMM depth per tile).
  const int NBO = NB * potrf_outer(ctx);
  if (ctx->opt.lookahead && m > 2 * (int64_t)NBO) return potrf_lookahead(ctx, S, m, Wbuf, Dinv, fail);
  for (int64_t K0 = 0; K0 < m; K0 += NBO) {
    const int64_t K1 = std::min<int64_t>(K0 + NBO, m);
    for (int64_t k0 = K0; k0 < K1; k0 += NB) {
      const int nb = (int)std::min<int64_t>(NB, m - k0);
      {
        LaunchScope ls(ctx, FALKON_T_PRECOND);
        potrf_diag_kernel<<<1, 512, dsm, ctx->stream>>>(S, k0, nb, Wbuf, Dinv, fail);
      }
      FK_LAUNCH_CHECK();
      const int64_t k1 = k0 + nb, rem = m - k1;
      if (rem <= 0) break;
      // panel: L(k1:, k0:k1) = S(k1:, k0:k1) W^T, W(j, k) at Wbuf[j*NB + (k - k0)]
      GemmArgs p{};
      p.A = S;
      p.B = W;
      p.C = S;
      p.M = rem;
      p.N = nb;
      p.ra = k1;
      p.rb = 0;
      p.rc = k1;
      p.cc = k0;
      p.k0 = k0;
      p.k1 = k1;
      p.B.base = Wbuf - k0;
      p.alpha = 1.0;
      p.beta = 0.0;
      FK_TRY(gemm(ctx, p));
      if (k1 < K1) {
        // update the rest of the outer panel: S(k1:, k1:K1) -= L(k1:, k0:k1) L(k1:K1, k0:k1)^T
        GemmArgs u{};
        u.A = S;
        u.B = S;
        u.C = S;
        u.M = rem;
        u.N = K1 - k1;
        u.ra = k1;
        u.rb = k1;
        u.rc = k1;
        u.cc = k1;
        u.k0 = k0;
        u.k1 = k1;
        u.alpha = -1.0;
        u.beta = 1.0;
        FK_TRY(gemm(ctx, u));
      }
    }
    const int64_t rem = m - K1;
    if (rem <= 0) break;
    // trailing: S(K1:, K1:) -= L(K1:, K0:K1) L(K1:, K0:K1)^T   (lower tiles)
    GemmArgs t{};
    t.A = S;
    t.B = S;
    t.C = S;
    t.M = rem;
    t.N = rem;
    t.ra = K1;
    t.rb = K1;
    t.rc = K1;
    t.cc = K1;
    t.k0 = K0;
    t.k1 = K1;
    t.tri_tiles = 1;
    t.alpha = -1.0;
    t.beta = 1.0;
    FK_TRY(gemm(ctx, t));
  }
  return FALKON_OK;
}

__global__ void add_diag_kernel(double *dvec, int64_t m, double scale, double add);

// ------------------------------------------------------------------ NEXT-1: distributed build
// 1D block-cyclic blocked Cholesky over G ranks (the multi-GPU layout of PAPER.md:460-469,
// App. C Alg. 4): outer panel j (NBO = potrf_outer x 128 columns of the
// logical lower factor L) is owned by rank j mod G.  Per panel:
//   1. the owner factors it (potrf_panel: diagonal blocks + TRSV inverse blocks, panel solve,
//      intra-panel updates) on its copy of the buffer;
//   2. the factored panel (columns [K0, K1) of L, rows >= K0), its diagonal entries, its TRSV
//      inverse blocks and the owner's pivot-failure word are broadcast;
//   3. every rank applies the panel's trailing update to the column panels IT owns.
// The LAUUM (T D T^T / m) is split the same way: each rank computes its own column panels of
// M.  Storage stays replicated (80 GB at m = 1e5 fits one B200) so the CG's triangular solves
// run locally; the O(m^3) work is split G ways.  Every element sees the same GEMM calls (k
// range, kernel, k order) as the single-GPU schedule, so the factors are bitwise identical.
// me < 0 simulates all G ranks in this process on one device (separate buffers, device copies
// for the broadcasts: the decomposition is testable without a second GPU).
struct DistBuild {
  int G = 1;
  int me = -1;
  double *const *P = nullptr;   // [G] (simulation) or [1] (this rank)
  double *const *diagT = nullptr, *const *diagA = nullptr;
  double *const *work = nullptr;  // per rank: precond_work_elems(m) doubles (TRSV inverses)
  unsigned long long *const *fail = nullptr;  // per rank: 2 pivot-failure words
  double *stage = nullptr;      // (real, G > 1) staging buffer of one A panel: m x NBO doubles
  int nranks_local() const { return me < 0 ? G : 1; }
  int rank_of(int i) const { return me < 0 ? i : me; }  // global rank of local slot i
};

__global__ void fail_min_kernel(unsigned long long *dst, const unsigned long long *src) {
  if (threadIdx.x == 0 && *src < *dst) *dst = *src;
}

// Step 2: panel [K0, K1) of factor `which` (0 = T: view trans 1, L columns = rows of P;
// 1 = A: view trans 0, L columns = column strips of P) from its owner to every rank.
static int dist_exchange(falkon_ctx *ctx, const DistBuild &D, int which, int64_t m, int64_t K0,
                         int64_t K1, int owner) {
  const int64_t nb = K1 - K0;
  const int64_t dv0 = (which == 0 ? 0 : precond_work_elems(m) / 2) + (K0 / TB) * TB * TB;
  const int64_t dvn = (cdiv<int64_t>(K1, TB) - K0 / TB) * TB * TB;
  auto dvec = [&](int i) { return (which == 0 ? D.diagT[i] : D.diagA[i]) + K0; };
  if (D.me < 0) {  // simulation: device copies from the owner's buffers
    for (int r = 0; r < D.G; ++r) {
      if (r == owner) continue;
      if (which == 0)
        FK_CUDA(cudaMemcpyAsync(D.P[r] + K0 * m, D.P[owner] + K0 * m, sizeof(double) * nb * m,
                                cudaMemcpyDeviceToDevice, ctx->stream));
      else
        FK_CUDA(cudaMemcpy2DAsync(D.P[r] + K0 * m + K0, sizeof(double) * m,
                                  D.P[owner] + K0 * m + K0, sizeof(double) * m,
                                  sizeof(double) * nb, m - K0, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
      FK_CUDA(cudaMemcpyAsync(dvec(r), dvec(owner), sizeof(double) * nb, cudaMemcpyDeviceToDevice,
                              ctx->stream));
      FK_CUDA(cudaMemcpyAsync(D.work[r] + dv0, D.work[owner] + dv0, sizeof(double) * dvn,
                              cudaMemcpyDeviceToDevice, ctx->stream));
      fail_min_kernel<<<1, 32, 0, ctx->stream>>>(D.fail[r] + which, D.fail[owner] + which);
    }
    FK_LAUNCH_CHECK();
    return FALKON_OK;
  }
  // real ranks: NCCL broadcasts on the context's communicator (ctx->stream)
  const bool own = D.me == owner;
  if (which == 0) {  // T panels are whole rows of P: broadcast in place
    FK_TRY(nccl_broadcast_bytes(ctx, D.P[0] + K0 * m, sizeof(double) * nb * m, owner));
  } else {  // A panels are column strips: pack, broadcast, unpack
    if (own)
      FK_CUDA(cudaMemcpy2DAsync(D.stage, sizeof(double) * nb, D.P[0] + K0 * m + K0,
                                sizeof(double) * m, sizeof(double) * nb, m - K0,
                                cudaMemcpyDeviceToDevice, ctx->stream));
    FK_TRY(nccl_broadcast_bytes(ctx, D.stage, sizeof(double) * nb * (m - K0), owner));
    if (!own)
      FK_CUDA(cudaMemcpy2DAsync(D.P[0] + K0 * m + K0, sizeof(double) * m, D.stage,
                                sizeof(double) * nb, sizeof(double) * nb, m - K0,
                                cudaMemcpyDeviceToDevice, ctx->stream));
  }
  FK_TRY(nccl_broadcast_bytes(ctx, dvec(0), sizeof(double) * nb, owner));
  FK_TRY(nccl_broadcast_bytes(ctx, D.work[0] + dv0, sizeof(double) * dvn, owner));
  return FALKON_OK;
}

// Steps 1-3 for factor `which` over every outer panel.
static int potrf_dist(falkon_ctx *ctx, const DistBuild &D, int which, int64_t m, double *Wbuf) {
  const size_t dsm = sizeof(double) * NB * (NB + 1);
  FK_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dsm));
  const int64_t NBO = (int64_t)NB * potrf_outer(ctx);
  const int64_t nob = cdiv<int64_t>(m, NBO);
  auto view = [&](int i) {
    return which == 0 ? View{D.P[i], m, 1, 1, D.diagT[i]} : View{D.P[i], m, 0, 1, D.diagA[i]};
  };
  auto dinv = [&](int i) { return D.work[i] + (which == 0 ? 0 : precond_work_elems(m) / 2); };
  for (int64_t j = 0; j < nob; ++j) {
    const int64_t K0 = j * NBO, K1 = std::min<int64_t>(K0 + NBO, m);
    const int owner = (int)(j % D.G);
    for (int i = 0; i < D.nranks_local(); ++i)
      if (D.rank_of(i) == owner)
        FK_TRY(potrf_panel(ctx, view(i), m, K0, K1, Wbuf, dinv(i), D.fail[i] + which, dsm));
    if (D.G > 1) FK_TRY(dist_exchange(ctx, D, which, m, K0, K1, owner));
    for (int i = 0; i < D.nranks_local(); ++i)
      for (int64_t c = j + 1; c < nob; ++c)
        if ((int)(c % D.G) == D.rank_of(i))
          FK_TRY(potrf_update(ctx, view(i), m, K0, K1, c * NBO, std::min<int64_t>(m, (c + 1) * NBO)));
  }
  return FALKON_OK;
}

// LAUUM split by owned column panels: M(i, j) = sum_{k >= i} T(i,k) D(k) T(j,k) / m for the
// columns j of this rank's panels (rows i >= the panel start), the same tiles and k order as the
// single-GPU call (panel starts are multiples of the 128-row GEMM tile).
static int lauum_dist(falkon_ctx *ctx, const DistBuild &D, int64_t m, double lambda,
                      const double *dscale) {
  const int64_t NBO = (int64_t)NB * potrf_outer(ctx);
  const int64_t nob = cdiv<int64_t>(m, NBO);
  for (int i = 0; i < D.nranks_local(); ++i) {
    View L2{D.P[i], m, 0, 1, D.diagA[i]};
    View Tv{D.P[i], m, 0, 2, D.diagT[i]};
    for (int64_t c = 0; c < nob; ++c) {
      if ((int)(c % D.G) != D.rank_of(i)) continue;
      const int64_t c0 = c * NBO, c1 = std::min<int64_t>(m, c0 + NBO);
      GemmArgs g{};
      g.A = Tv;
      g.B = Tv;
      g.C = L2;
      g.M = m - c0;
      g.N = c1 - c0;
      g.ra = g.rb = g.rc = g.cc = c0;
      g.k0 = 0;
      g.k1 = m;
      g.k_from_row = 1;
      g.tri_tiles = 1;
      g.alpha = 1.0 / (double)m;
      g.beta = 0.0;
      g.kscale = dscale;
      FK_TRY(gemm(ctx, g));
    }
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    add_diag_kernel<<<(unsigned)cdiv<int64_t>(m, 256), 256, 0, ctx->stream>>>(D.diagA[i], m, 1.0,
                                                                                lambda);
  }
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

__global__ void add_diag_kernel(double *dvec, int64_t m, double scale, double add) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) dvec[i] = dvec[i] * scale + add;
}

// Reads the two pivot-failure words written by potrf (first failing column or ~0) and
// turns a failure into ENOTPD naming the factor and column.
static int check_pivots(falkon_ctx *ctx, const unsigned long long *failf, int f0, int f1,
                        double jitter, falkon_fit_info *info) {
  unsigned long long hf[2];
  FK_CUDA(cudaMemcpyAsync(hf, failf, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info) {
    info->failed_factor = -1;
    info->failed_column = -1;
    info->jitter_used = jitter;
  }
  for (int f = f0; f <= f1; ++f) {
    if (hf[f] != ~0ULL) {
      if (info) {
        info->failed_factor = f;
        info->failed_column = (int64_t)hf[f];
      }
      return fail(FALKON_ENOTPD, std::string("Cholesky of ") + (f ? "A" : "T") +
                                     " failed at column " + std::to_string(hf[f]));
    }
  }
  return FALKON_OK;
}

// Steps (b)-(c): Kmm + delta I into the upper triangle, factored in place into T.
// `check`: synchronise and report a pivot failure (else the caller checks later).
static int build_T(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                   double sigma, double jitter, double *P, double *diagT, double *dinvT,
                   unsigned long long *failf) {
  void *wb;
  FK_TRY(ws_get(ctx, WS_PW, sizeof(double) * NB * NB, &wb));
  View L1{P, m, 1, 1, diagT};  // L1 = T^T, stored in the upper triangle
  {
    const int64_t tt = cdiv<int64_t>(m, 64);
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    kmm_kernel<<<(unsigned)(tt * (tt + 1) / 2), 256, 0, ctx->stream>>>(
        C, m, d, kernel, 1.0 / (2.0 * sigma * sigma), 1.0 / sigma, jitter, L1);
  }
  FK_LAUNCH_CHECK();
  return potrf(ctx, L1, m, (double *)wb, dinvT, failf);
}

// Steps (d)-(e): M = T D T^T / m + lambda I into the lower triangle (+ diagA), factored in
// place into A^T.  D = diag(dscale) (Alg. 2 line 5) or I (dscale == NULL,
// Alg. 1 line 16).  M(i,j) = sum_{k>=i} T(i,k) D(k) T(j,k).
static int build_A(falkon_ctx *ctx, int64_t m, double lambda, const double *dscale, double *P,
                   double *diagT, double *diagA, double *dinvA, unsigned long long *failf) {
  void *wb;
  FK_TRY(ws_get(ctx, WS_PW, sizeof(double) * NB * NB, &wb));
  View L2{P, m, 0, 1, diagA};  // L2 = A^T, stored in the lower triangle
  View Tv{P, m, 0, 2, diagT};  // T itself (upper view of the same storage)
  {
    GemmArgs g{};
    g.A = Tv;
    g.B = Tv;
    g.C = L2;
    g.M = m;
    g.N = m;
    g.k0 = 0;
    g.k1 = m;
    g.k_from_row = 1;
    g.tri_tiles = 1;
    g.alpha = 1.0 / (double)m;
    g.beta = 0.0;
    g.kscale = dscale;
    FK_TRY(gemm(ctx, g));
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    add_diag_kernel<<<(unsigned)cdiv<int64_t>(m, 256), 256, 0, ctx->stream>>>(diagA, m, 1.0,
                                                                                lambda);
  }
  FK_LAUNCH_CHECK();
  return potrf(ctx, L2, m, (double *)wb, dinvA, failf);
}

// ---- distributed steps (b)-(e) (NEXT-1): Kmm is computed on every rank (O(m^2 d), replicated)
static int build_T_dist(falkon_ctx *ctx, const DistBuild &D, const float *C, int64_t m, int64_t d,
                        int kernel, double sigma, double jitter) {
  void *wb;
  FK_TRY(ws_get(ctx, WS_PW, sizeof(double) * NB * NB, &wb));
  for (int i = 0; i < D.nranks_local(); ++i) {
    View L1{D.P[i], m, 1, 1, D.diagT[i]};
    const int64_t tt = cdiv<int64_t>(m, 64);
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    kmm_kernel<<<(unsigned)(tt * (tt + 1) / 2), 256, 0, ctx->stream>>>(
        C, m, d, kernel, 1.0 / (2.0 * sigma * sigma), 1.0 / sigma, jitter, L1);
  }
  FK_LAUNCH_CHECK();
  return potrf_dist(ctx, D, 0, m, (double *)wb);
}
static int build_A_dist(falkon_ctx *ctx, const DistBuild &D, int64_t m, double lambda,
                        const double *dscale) {
  void *wb;
  FK_TRY(ws_get(ctx, WS_PW, sizeof(double) * NB * NB, &wb));
  FK_TRY(lauum_dist(ctx, D, m, lambda, dscale));
  return potrf_dist(ctx, D, 1, m, (double *)wb);
}

// The build is distributed when the context has a multi-rank NCCL communicator, or when
// FALKON_OPT_DIST_PRECOND forces the distributed schedule (a 1-rank communicator: the
// broadcasts become self-copies; tests the code path on one GPU).
static bool dist_active(const falkon_ctx *ctx) {
  return ctx->nccl_comm && (ctx->world > 1 || ctx->opt.dist_precond);
}
static int dist_for_ctx(falkon_ctx *ctx, int64_t m, double **P, double **dT, double **dA,
                        double **work, unsigned long long **fl, DistBuild *D) {
  D->G = ctx->world;
  D->me = ctx->rank;
  D->P = P;
  D->diagT = dT;
  D->diagA = dA;
  D->work = work;
  D->fail = fl;
  if (ctx->world > 1) {
    void *st;
    FK_TRY(ws_get(ctx, WS_DIST_STAGE,
                  sizeof(double) * (size_t)m * NB * (size_t)potrf_outer(ctx), &st));
    D->stage = (double *)st;
  }
  return FALKON_OK;
}
// failure words: the panel owners' (replicated by a min over ranks) before the host check
static int dist_merge_fail(falkon_ctx *ctx, unsigned long long *failf) {
  return nccl_allreduce_min_u64(ctx, failf, 2);
}

int precond_build(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel, double sigma,
                  double lambda, double jitter, double *P, double *diagT, double *diagA,
                  double *work, falkon_fit_info *info) {
  double *dinvT = work, *dinvA = work ? work + precond_work_elems(m) / 2 : nullptr;
  void *flags;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64, &flags));
  unsigned long long *failf = (unsigned long long *)flags;
  FK_CUDA(cudaMemsetAsync(failf, 0xff, 16, ctx->stream));
  if (dist_active(ctx)) {
    DistBuild D;
    FK_TRY(dist_for_ctx(ctx, m, &P, &diagT, &diagA, &work, &failf, &D));
    FK_TRY(build_T_dist(ctx, D, C, m, d, kernel, sigma, jitter));
    FK_TRY(build_A_dist(ctx, D, m, lambda, nullptr));
    FK_TRY(dist_merge_fail(ctx, failf));
    return check_pivots(ctx, failf, 0, 1, jitter, info);
  }
  FK_TRY(build_T(ctx, C, m, d, kernel, sigma, jitter, P, diagT, dinvT, failf));
  FK_TRY(build_A(ctx, m, lambda, nullptr, P, diagT, diagA, dinvA, failf + 1));
  return check_pivots(ctx, failf, 0, 1, jitter, info);
}

int precond_build_T(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                    double sigma, double jitter, double *P, double *diagT, double *work,
                    falkon_fit_info *info) {
  void *flags;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64, &flags));
  unsigned long long *failf = (unsigned long long *)flags;
  FK_CUDA(cudaMemsetAsync(failf, 0xff, 16, ctx->stream));
  if (dist_active(ctx)) {
    DistBuild D;
    double *dA = nullptr;
    FK_TRY(dist_for_ctx(ctx, m, &P, &diagT, &dA, &work, &failf, &D));
    FK_TRY(build_T_dist(ctx, D, C, m, d, kernel, sigma, jitter));
    FK_TRY(dist_merge_fail(ctx, failf));
    return check_pivots(ctx, failf, 0, 0, jitter, info);
  }
  FK_TRY(build_T(ctx, C, m, d, kernel, sigma, jitter, P, diagT, work, failf));
  return check_pivots(ctx, failf, 0, 0, jitter, info);
}

int precond_build_A(falkon_ctx *ctx, int64_t m, double lambda, const double *dscale, double *P,
                    double *diagT, double *diagA, double *work, double jitter,
                    falkon_fit_info *info) {
  void *flags;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64, &flags));
  unsigned long long *failf = (unsigned long long *)flags;
  FK_CUDA(cudaMemsetAsync(failf, 0xff, 16, ctx->stream));
  if (dist_active(ctx)) {
    DistBuild D;
    FK_TRY(dist_for_ctx(ctx, m, &P, &diagT, &diagA, &work, &failf, &D));
    FK_TRY(build_A_dist(ctx, D, m, lambda, dscale));
    FK_TRY(dist_merge_fail(ctx, failf));
    return check_pivots(ctx, failf, 1, 1, jitter, info);
  }
  FK_TRY(build_A(ctx, m, lambda, dscale, P, diagT, diagA, work + precond_work_elems(m) / 2,
                 failf + 1));
  return check_pivots(ctx, failf, 1, 1, jitter, info);
}

// G ranks simulated in this process (tests): rank r's buffers P[r], diagT[r], diagA[r], work[r].
int precond_build_sim(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel,
                      double sigma, double lambda, double jitter, int G, double *const *P,
                      double *const *diagT, double *const *diagA, double *const *work,
                      falkon_fit_info *info) {
  void *flags;
  FK_TRY(ws_get(ctx, WS_SIM_FLAGS, sizeof(unsigned long long) * 2 * (size_t)G, &flags));
  unsigned long long *f0 = (unsigned long long *)flags;
  FK_CUDA(cudaMemsetAsync(f0, 0xff, sizeof(unsigned long long) * 2 * (size_t)G, ctx->stream));
  std::vector<unsigned long long *> fl((size_t)G);
  for (int r = 0; r < G; ++r) fl[(size_t)r] = f0 + 2 * r;
  DistBuild D;
  D.G = G;
  D.me = -1;
  D.P = P;
  D.diagT = diagT;
  D.diagA = diagA;
  D.work = work;
  D.fail = fl.data();
  FK_TRY(build_T_dist(ctx, D, C, m, d, kernel, sigma, jitter));
  FK_TRY(build_A_dist(ctx, D, m, lambda, nullptr));
  for (int r = 0; r < G; ++r) {  // every rank must report the same failures as rank 0
    FK_TRY(check_pivots(ctx, fl[(size_t)r], 0, 1, jitter, info));
  }
  return FALKON_OK;
}

// ------------------------------------------------------------------ triangular mat-vecs
// y = T x and z = T^T y for the upper factor T (strict upper triangle row-major in P, diagonal
// in diagT): the fp64 predictions on the Nystrom points of Alg. 2 are
// (Kmm + delta I) alpha = T^T (T alpha) once Kmm has been factored in place.  HBM-bound
// streams of the triangle; fixed-order reductions (bitwise-reproducible on every rank).
constexpr int TRMV_SEG = 32;  // row segments of the transposed product

// y_r = diagT_r x_r + sum_{c > r} P[r m + c] x_c : one warp per row, coalesced, shuffle tree
__global__ void __launch_bounds__(256) trmv_upper_kernel(const double *__restrict__ P,
                                                         const double *__restrict__ diagT,
                                                         int64_t m, const double *__restrict__ x,
                                                         double *__restrict__ y) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= m) return;
  const double *row = P + r * m;
  double a0 = 0.0, a1 = 0.0;
  int64_t c = r + 1 + lane;
  for (; c + 32 < m; c += 64) {
    a0 = fma(row[c], x[c], a0);
    a1 = fma(row[c + 32], x[c + 32], a1);
  }
  if (c < m) a0 = fma(row[c], x[c], a0);
  double a = a0 + a1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) y[r] = fma(diagT[r], x[r], a);
}

// part[s][c] = sum_{r in segment s, r < c} P[r m + c] y_r : thread per column, coalesced rows
__global__ void __launch_bounds__(256) trmv_upper_t_part_kernel(const double *__restrict__ P,
                                                                int64_t m,
                                                                const double *__restrict__ y,
                                                                double *__restrict__ part) {
  const int64_t c = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int s = blockIdx.y;
  if (c >= m) return;
  const int64_t seg = cdiv<int64_t>(m, TRMV_SEG);
  const int64_t r0 = s * seg, r1 = lmin(lmin((int64_t)(s + 1) * seg, c), m);
  double a0 = 0.0, a1 = 0.0;
  int64_t r = r0;
  for (; r + 1 < r1; r += 2) {
    a0 = fma(P[r * m + c], y[r], a0);
    a1 = fma(P[(r + 1) * m + c], y[r + 1], a1);
  }
  if (r < r1) a0 = fma(P[r * m + c], y[r], a0);
  part[(int64_t)s * m + c] = a0 + a1;
}
__global__ void trmv_upper_t_final_kernel(const double *__restrict__ diagT, int64_t m,
                                          const double *__restrict__ y,
                                          const double *__restrict__ part, double *__restrict__ z) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double a = diagT[c] * y[c];
  for (int s = 0; s < TRMV_SEG; ++s) a += part[(int64_t)s * m + c];
  z[c] = a;
}

int trmv_TtT(falkon_ctx *ctx, const double *P, const double *diagT, int64_t m, const double *x,
             double *tmp, double *z) {
  void *pp;
  FK_TRY(ws_get(ctx, WS_TRMV, sizeof(double) * TRMV_SEG * m, &pp));
  LaunchScope ls(ctx, FALKON_T_PRECOND);
  trmv_upper_kernel<<<(unsigned)cdiv<int64_t>(m, 8), 256, 0, ctx->stream>>>(P, diagT, m, x, tmp);
  trmv_upper_t_part_kernel<<<dim3((unsigned)cdiv<int64_t>(m, 256), TRMV_SEG), 256, 0,
                             ctx->stream>>>(P, m, tmp, (double *)pp);
  trmv_upper_t_final_kernel<<<(unsigned)cdiv<int64_t>(m, 256), 256, 0, ctx->stream>>>(
      diagT, m, tmp, (const double *)pp, z);
  ctx->launches += 2;
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// ------------------------------------------------------------------ sync-free blocked TRSV
// Solves L z = r (forward) or L^T z = r (backward) for the lower-triangular view L, with
// Dinv = the inverses of L's 64 x 64 diagonal blocks (written by the factorization).
// CTA with ticket b owns row block I (forward: I = b, backward: I = nb-1-b): it streams its
// off-diagonal 64 x 64 tiles from HBM into shared memory with cp.async ahead of the
// dependency front, multiplies each by z_J as soon as z_J is final (sentinel-tagged output,
// see trsv_kernel), then finishes its block with the 64 x 64 inverse (a parallel mat-vec, no
// sequential substitution), so the serial chain per block is ~one L2 round trip plus a few
// shared-memory mat-vecs, and the solve streams the triangle at HBM rate behind it.
constexpr int TS_LD = TB + 2;  // smem row stride (doubles), 16 B aligned rows


__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
// copy a 64 x 64 stored block (rows of 64 contiguous doubles, leading dimension ld) to smem;
// 16-byte copies when every row start is 16-byte aligned (even ld), else 8-byte copies
__device__ __forceinline__ void tile_async(double *dst, const double *src, int64_t ld, int rows,
                                           int cols) {
  if ((ld & 1) == 0) {
    for (int e = threadIdx.x; e < TB * (TB / 2); e += blockDim.x) {
      const int r = e / (TB / 2), c2 = (e % (TB / 2)) * 2;
      if (r < rows && c2 < cols) cp_async16(dst + r * TS_LD + c2, src + (int64_t)r * ld + c2);
    }
  } else {
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
      const int r = e / TB, c = e % TB;
      if (r < rows && c < cols) cp_async8(dst + r * TS_LD + c, src + (int64_t)r * ld + c);
    }
  }
}

constexpr int TRSV_ZR = 16;  // z blocks fetched per L2 round trip

// Readiness of the solution travels with the data: the output vector zo is pre-filled with a
// NaN sentinel (all bits set) and every element is written exactly once, so a consumer that
// reads a non-sentinel value holds the final value -- one L2 round trip from the producer's
// store to the consumer, no fence / counter / second fetch on the dependency chain.
constexpr unsigned long long TRSV_SENT = ~0ULL;
__device__ __forceinline__ bool is_sent(double v) {
  return (unsigned long long)__double_as_longlong(v) == TRSV_SENT;
}

__global__ void __launch_bounds__(256) trsv_kernel(View L, int64_t m, int forward,
                                                   const double *__restrict__ rhs,
                                                   double *zo, const double *__restrict__ Dinv,
                                                   unsigned int *__restrict__ counter) {
  // CTAs take row blocks in solve order (ticket); tiles of L do not depend on z, so they are
  // prefetched (cp.async, 2 deep) regardless of the front; final z_J are fetched in batches of
  // up to TRSV_ZR blocks per L2 round trip; at the front the CTA spins on the sentinel.
  extern __shared__ __align__(16) double tsm[];
  double *sT0 = tsm, *sT1 = tsm + TB * TS_LD;
  double *sD = tsm + 2 * TB * TS_LD;
  double *zr = sD + TB * TS_LD;   // [TRSV_ZR * TB]
  double *sx = zr + TRSV_ZR * TB;  // [TB]
  __shared__ unsigned int s_ticket;
  __shared__ int s_ready;
  const int tid = threadIdx.x;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  if (tid == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t b = s_ticket;  // this block's rank in solve order
  const int64_t I = forward ? b : nblk - 1 - b;
  const int64_t i0 = I * TB;
  const int nI = (int)lmin(TB, m - i0);
  const bool rowmaj = (forward != 0) == (L.trans == 0);
  const int64_t nJ = b;  // steps: the b blocks before this one in solve order
  auto j0of = [&](int64_t s) { return (forward ? s : nblk - 1 - s) * TB; };
  auto issue = [&](int64_t s) {
    const int64_t j0 = j0of(s);
    const int nJc = (int)lmin(TB, m - j0);
    tile_async((s & 1) ? sT1 : sT0, rowmaj ? L.base + i0 * L.ld + j0 : L.base + j0 * L.ld + i0,
               L.ld, rowmaj ? nI : nJc, rowmaj ? nJc : nI);
    cp_async_commit();
  };
  {
    const double *dsrc = Dinv + I * (int64_t)(TB * TB);
    for (int e = tid; e < TB * (TB / 2); e += blockDim.x) {
      const int r = e / (TB / 2), c2 = (e % (TB / 2)) * 2;
      cp_async16(sD + r * TS_LD + c2, dsrc + r * TB + c2);
    }
    cp_async_commit();
  }
  if (nJ > 0) issue(0);
  const int ri = rowmaj ? (tid >> 2) : (tid & 63);
  const int qq = rowmaj ? (tid & 3) : (tid >> 6);
  double acc = 0.0;
  int64_t zlo = 0, zhi = 0;
  for (int64_t s = 0; s < nJ; ++s) {
    if (s + 1 < nJ) issue(s + 1);
    if (s >= zhi) {
      // batch-fetch blocks [s, s + TRSV_ZR); the ready prefix ends at the first sentinel
      const int64_t want = lmin(nJ, s + TRSV_ZR);
      if (tid == 0) s_ready = (int)(want - s);
      __syncthreads();
      for (int e = tid; e < (want - s) * TB; e += blockDim.x) {
        const int64_t st = s + e / TB;
        const int64_t jg = j0of(st) + e % TB;
        const double v = jg < m ? __ldcg(zo + jg) : 0.0;
        zr[e] = v;
        if (is_sent(v)) atomicMin(&s_ready, (int)(e / TB));
      }
      __syncthreads();
      zlo = s;
      zhi = s + s_ready;
      if (zhi == s) {  // at the dependency front: spin on block s itself
        if (tid < TB) {
          const int64_t jg = j0of(s) + tid;
          double v = 0.0;
          if (jg < m) {
            const volatile double *pz = zo + jg;
            do {
              v = *pz;
            } while (is_sent(v));
          }
          zr[tid] = v;
        }
        zhi = s + 1;
      }
      __syncthreads();
    }
    if (s + 1 < nJ) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double *T = (s & 1) ? sT1 : sT0;
    const double *zz = zr + (s - zlo) * TB;
    const int nJc = (int)lmin(TB, m - j0of(s));
    if (ri < nI) {
      if (rowmaj) {
#pragma unroll
        for (int k = 0; k < TB / 4; ++k) {
          const int jj = qq + 4 * k;
          if (jj < nJc) acc = fma(T[ri * TS_LD + jj], zz[jj], acc);
        }
      } else {
#pragma unroll
        for (int k = 0; k < TB / 4; ++k) {
          const int jj = qq * (TB / 4) + k;
          if (jj < nJc) acc = fma(T[jj * TS_LD + ri], zz[jj], acc);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
  // reduce the 4 partial sums of each row, form x = r_I - acc
  double *part = sT0;  // reuse: [4][TB]
  part[qq * TB + ri] = acc;
  __syncthreads();
  if (tid < TB)
    sx[tid] = (tid < nI) ? rhs[i0 + tid] - (part[tid] + part[TB + tid] + part[2 * TB + tid] +
                                           part[3 * TB + tid])
                         : 0.0;
  __syncthreads();
  // z_I = D x (forward, D = Dinv_I) or D^T x (backward): parallel, no substitution
  {
    const int r = tid & 63, q4 = tid >> 6;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < TB / 4; ++k) {
      const int c = q4 * (TB / 4) + k;
      v = fma(forward ? sD[r * TS_LD + c] : sD[c * TS_LD + r], sx[c], v);
    }
    __syncthreads();
    part[q4 * TB + r] = v;
  }
  __syncthreads();
  if (tid < nI) {
    double v = part[tid] + part[TB + tid] + part[2 * TB + tid] + part[3 * TB + tid];
    if (is_sent(v)) v = __longlong_as_double(0x7ff8000000000000LL);  // keep the sentinel unique
    __stcg(zo + i0 + tid, v);
  }
}

// Multi-column variant (multi-output fits): solves KC right-hand sides
// (columns at stride ldx) in one pass over the triangle.  Same schedule and sentinel protocol as
// trsv_kernel; each tile is multiplied into KC accumulators per thread.
constexpr int TRSV_KC = 16;
constexpr int TRSV_ZRM = 4;  // z blocks per batch fetch (x KC columns)

template <int KC>
__global__ void __launch_bounds__(256) trsv_multi_kernel(View L, int64_t m, int forward,
                                                         const double *__restrict__ rhs,
                                                         int64_t ldx, int kc, double *zo,
                                                         const double *__restrict__ Dinv,
                                                         unsigned int *__restrict__ counter) {
  extern __shared__ __align__(16) double tsm[];
  double *sT0 = tsm, *sT1 = tsm + TB * TS_LD;
  double *sD = tsm + 2 * TB * TS_LD;
  double *zr = sD + TB * TS_LD;          // [TRSV_ZRM][KC][TB]
  double *sx = zr + TRSV_ZRM * KC * TB;  // [KC][TB]
  __shared__ unsigned int s_ticket;
  __shared__ int s_ready;
  const int tid = threadIdx.x;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  if (tid == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t b = s_ticket;
  const int64_t I = forward ? b : nblk - 1 - b;
  const int64_t i0 = I * TB;
  const int nI = (int)lmin(TB, m - i0);
  const bool rowmaj = (forward != 0) == (L.trans == 0);
  const int64_t nJ = b;
  auto j0of = [&](int64_t s) { return (forward ? s : nblk - 1 - s) * TB; };
  auto issue = [&](int64_t s) {
    const int64_t j0 = j0of(s);
    const int nJc = (int)lmin(TB, m - j0);
    tile_async((s & 1) ? sT1 : sT0, rowmaj ? L.base + i0 * L.ld + j0 : L.base + j0 * L.ld + i0,
               L.ld, rowmaj ? nI : nJc, rowmaj ? nJc : nI);
    cp_async_commit();
  };
  {
    const double *dsrc = Dinv + I * (int64_t)(TB * TB);
    for (int e = tid; e < TB * (TB / 2); e += blockDim.x) {
      const int r = e / (TB / 2), c2 = (e % (TB / 2)) * 2;
      cp_async16(sD + r * TS_LD + c2, dsrc + r * TB + c2);
    }
    cp_async_commit();
  }
  if (nJ > 0) issue(0);
  const int ri = rowmaj ? (tid >> 2) : (tid & 63);
  const int qq = rowmaj ? (tid & 3) : (tid >> 6);
  double acc[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) acc[c] = 0.0;
  int64_t zlo = 0, zhi = 0;
  for (int64_t s = 0; s < nJ; ++s) {
    if (s + 1 < nJ) issue(s + 1);
    if (s >= zhi) {
      const int64_t want = lmin(nJ, s + TRSV_ZRM);
      if (tid == 0) s_ready = (int)(want - s);
      __syncthreads();
      for (int e = tid; e < (want - s) * KC * TB; e += blockDim.x) {
        const int blk = e / (KC * TB), c = (e / TB) % KC, jj = e % TB;
        const int64_t jg = j0of(s + blk) + jj;
        double v = 0.0;
        if (jg < m && c < kc) {
          v = __ldcg(zo + c * m + jg);
          if (is_sent(v)) atomicMin(&s_ready, blk);
        }
        zr[e] = v;
      }
      __syncthreads();
      zlo = s;
      zhi = s + s_ready;
      if (zhi == s) {  // dependency front: spin on block s (all columns)
        for (int e = tid; e < KC * TB; e += blockDim.x) {
          const int c = e / TB, jj = e % TB;
          const int64_t jg = j0of(s) + jj;
          double v = 0.0;
          if (jg < m && c < kc) {
            const volatile double *pz = zo + c * m + jg;
            do {
              v = *pz;
            } while (is_sent(v));
          }
          zr[e] = v;
        }
        zhi = s + 1;
      }
      __syncthreads();
    }
    if (s + 1 < nJ) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double *T = (s & 1) ? sT1 : sT0;
    const double *zz = zr + (s - zlo) * KC * TB;
    const int nJc = (int)lmin(TB, m - j0of(s));
    if (ri < nI) {
#pragma unroll 4
      for (int k = 0; k < TB / 4; ++k) {
        const int jj = rowmaj ? qq + 4 * k : qq * (TB / 4) + k;
        if (jj < nJc) {
          const double t = rowmaj ? T[ri * TS_LD + jj] : T[jj * TS_LD + ri];
#pragma unroll
          for (int c = 0; c < KC; ++c) acc[c] = fma(t, zz[c * TB + jj], acc[c]);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
  // x = r_I - acc per column (4 partial sums per row, fixed order), then z_I = D x
  double *part = sT0;  // [4][KC][TB] fits in two tile buffers for KC <= 16 ... use sT0..sD
#pragma unroll
  for (int c = 0; c < KC; ++c) part[(qq * KC + c) * TB + ri] = acc[c];
  __syncthreads();
  for (int e = tid; e < KC * TB; e += blockDim.x) {
    const int c = e / TB, r = e % TB;
    double v = 0.0;
    if (r < nI && c < kc)
      v = rhs[c * ldx + i0 + r] - (part[(0 * KC + c) * TB + r] + part[(1 * KC + c) * TB + r] +
                                   part[(2 * KC + c) * TB + r] + part[(3 * KC + c) * TB + r]);
    sx[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < KC * TB; e += blockDim.x) {
    const int c = e / TB, r = e % TB;
    if (r >= nI || c >= kc) continue;
    double v = 0.0;
    for (int k = 0; k < TB; ++k) v = fma(forward ? sD[r * TS_LD + k] : sD[k * TS_LD + r], sx[c * TB + k], v);
    if (is_sent(v)) v = __longlong_as_double(0x7ff8000000000000LL);
    __stcg(zo + c * m + i0 + r, v);
  }
}

// x[:, c] <- op(F)^-1 x[:, c] for the kcols columns of x (column c at x + c ldx)
int trsv_multi(falkon_ctx *ctx, const double *P, const double *diag, const double *work, int64_t m,
               int which, int trans, double *x, int64_t ldx, int64_t kcols) {
  if (kcols == 1) return trsv(ctx, P, diag, work, m, which, trans, x);
  View L{const_cast<double *>(P), m, which == 0 ? 1 : 0, 1, const_cast<double *>(diag)};
  const double *dinv = work + (which == 0 ? 0 : precond_work_elems(m) / 2);
  const int forward = trans ? 1 : 0;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  void *fl, *zb;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64 + sizeof(unsigned int) * (nblk + 64), &fl));
  FK_TRY(ws_get(ctx, WS_TRSV, sizeof(double) * m * TRSV_KC, &zb));
  unsigned int *counter = (unsigned int *)((char *)fl + 32);
  const size_t smem =
      sizeof(double) * (3 * TB * TS_LD + (size_t)(TRSV_ZRM + 1) * TRSV_KC * TB);
  static_assert(4 * TRSV_KC * TB <= 3 * TB * TS_LD + TRSV_ZRM * TRSV_KC * TB,
                "partials fit in the tile + ring buffers");
  FK_CUDA(cudaFuncSetAttribute(trsv_multi_kernel<TRSV_KC>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t c0 = 0; c0 < kcols; c0 += TRSV_KC) {
    const int kc = (int)std::min<int64_t>(TRSV_KC, kcols - c0);
    FK_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), ctx->stream));
    FK_CUDA(cudaMemsetAsync(zb, 0xff, sizeof(double) * m * kc, ctx->stream));
    {
      LaunchScope ls(ctx, FALKON_T_TRSV);
      trsv_multi_kernel<TRSV_KC><<<(unsigned)nblk, 256, smem, ctx->stream>>>(
          L, m, forward, x + c0 * ldx, ldx, kc, (double *)zb, dinv, counter);
    }
    FK_LAUNCH_CHECK();
    FK_CUDA(cudaMemcpy2DAsync(x + c0 * ldx, sizeof(double) * ldx, zb, sizeof(double) * m,
                              sizeof(double) * m, kc, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return FALKON_OK;
}

int64_t precond_work_elems(int64_t m) { return 2 * cdiv<int64_t>(m, TB) * (int64_t)(TB * TB); }

int trsv(falkon_ctx *ctx, const double *P, const double *diag, const double *work, int64_t m,
         int which, int trans, double *x) {
  // which 0: T = L1^T (L1 = view trans=1 of the upper triangle); which 1: A = L2^T.
  // T x = r  <=> L1^T x = r (backward);  T^T x = r <=> L1 x = r (forward); same for A.
  View L{const_cast<double *>(P), m, which == 0 ? 1 : 0, 1, const_cast<double *>(diag)};
  const double *dinv = work + (which == 0 ? 0 : precond_work_elems(m) / 2);
  const int forward = trans ? 1 : 0;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  void *fl, *zb;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64 + sizeof(unsigned int) * (nblk + 64), &fl));
  FK_TRY(ws_get(ctx, WS_TRSV, sizeof(double) * m, &zb));
  unsigned int *counter = (unsigned int *)((char *)fl + 32);
  const size_t smem = sizeof(double) * (3 * TB * TS_LD + (TRSV_ZR + 1) * TB);
  FK_CUDA(cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  FK_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), ctx->stream));
  FK_CUDA(cudaMemsetAsync(zb, 0xff, sizeof(double) * m, ctx->stream));  // sentinel
  {
    LaunchScope ls(ctx, FALKON_T_TRSV);
    trsv_kernel<<<(unsigned)nblk, 256, smem, ctx->stream>>>(L, m, forward, x, (double *)zb, dinv,
                                                            counter);
  }
  FK_LAUNCH_CHECK();
  FK_CUDA(cudaMemcpyAsync(x, zb, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  return FALKON_OK;
}

}  // namespace falkon
