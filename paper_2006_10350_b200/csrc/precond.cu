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

#include "common.cuh"

namespace falkon {

constexpr int NB = 128;        // factorization block
constexpr int GT = 128;        // GEMM CTA tile
constexpr int GK = 16;         // GEMM k-chunk
constexpr int GPAD = 2;        // smem row padding (doubles)
constexpr int TB = 64;         // TRSV block

// ------------------------------------------------------------------ views
// Logical matrix element (r, c) of a view.  tri: 0 = dense; 1 = lower (r > c from
// storage, r == c from dvec, r < c is zero); 2 = upper (c > r from storage, diag from
// dvec, c < r is zero).
struct View {
  double *base;
  int64_t ld;
  int trans;
  int tri;
  double *dvec;
};

__device__ __forceinline__ int64_t vidx(const View &v, int64_t r, int64_t c) {
  return v.trans ? c * v.ld + r : r * v.ld + c;
}
__device__ __forceinline__ double vget(const View &v, int64_t r, int64_t c) {
  if (v.tri == 1) {
    if (r < c) return 0.0;
    if (r == c) return v.dvec[r];
  } else if (v.tri == 2) {
    if (c < r) return 0.0;
    if (r == c) return v.dvec[r];
  }
  return v.base[vidx(v, r, c)];
}
__device__ __forceinline__ void vset(const View &v, int64_t r, int64_t c, double x) {
  if (v.tri == 1) {
    if (r < c) return;
    if (r == c) {
      v.dvec[r] = x;
      return;
    }
  } else if (v.tri == 2) {
    if (c < r) return;
    if (r == c) {
      v.dvec[r] = x;
      return;
    }
  }
  v.base[vidx(v, r, c)] = x;
}

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
                                                         unsigned long long *fail) {
  extern __shared__ double sL[];  // nb x (nb+1)
  const int ld = nb + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = e / nb, c = e % nb;
    sL[r * ld + c] = (r >= c) ? vget(S, k0 + r, k0 + c) : 0.0;
  }
  __syncthreads();
  // unblocked right-looking Cholesky
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
    const double ljj = sL[j * ld + j];
    for (int i = j + 1 + tid; i < nb; i += nt) sL[i * ld + j] /= ljj;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      const int i = j + 1 + e / rem, k = j + 1 + e % rem;
      if (k <= i) sL[i * ld + k] -= sL[i * ld + j] * sL[k * ld + j];
    }
    __syncthreads();
  }
  // write L back (lower + diag)
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = e / nb, c = e % nb;
    if (r >= c) vset(S, k0 + r, k0 + c, sL[r * ld + c]);
  }
  __syncthreads();
  // in-place inverse of lower-triangular L (LAPACK trti2 order: columns right to left)
  __shared__ double xcol[NB];
  for (int j = nb - 1; j >= 0; --j) {
    if (tid == 0) sL[j * ld + j] = 1.0 / sL[j * ld + j];
    for (int i = j + 1 + tid; i < nb; i += nt) xcol[i] = sL[i * ld + j];
    __syncthreads();
    const double ajj = -sL[j * ld + j];
    // x <- Winv[j+1:, j+1:] * x  (Winv lower, already inverted), then scale by ajj
    for (int i = j + 1 + tid; i < nb; i += nt) {
      double s = 0.0;
      for (int k = j + 1; k <= i; ++k) s = fma(sL[i * ld + k], xcol[k], s);
      sL[i * ld + j] = s * ajj;
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += nt) {
    const int r = e / nb, c = e % nb;
    W[(int64_t)r * NB + c] = (r >= c) ? sL[r * ld + c] : 0.0;
  }
}

// ------------------------------------------------------------------ fp64 GEMM through views
// C(i, j) = alpha * sum_{k in [kb, k1)} A(ra + i, k) * B(rb + j, k) + beta * C(rc + i, cc + j)
// for 0 <= i < M, 0 <= j < N.  tri_tiles: only tiles with ti >= tj (square lower region).
// k_from_row: kb = max(k0, ra + ti*GT) (LAUUM: sum over k >= row block).
struct GemmArgs {
  View A, B, C;
  int64_t M, N;
  int64_t ra, rb, rc, cc;
  int64_t k0, k1;
  int k_from_row;
  int tri_tiles;
  double alpha, beta;
};

__device__ __forceinline__ void gemm_load_chunk(const View &v, int64_t row0, int64_t rmax,
                                                int64_t k, int64_t kmax, double (&reg)[8]) {
  const int tid = threadIdx.x;
  if (!v.trans) {
    // storage contiguous along k: 16 threads per row, 16 rows per pass, 8 passes
    const int kk = tid & 15, rr = tid >> 4;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int64_t r = row0 + rr + 16 * p, kg = k + kk;
      reg[p] = (r < rmax && kg < kmax) ? vget(v, r, kg) : 0.0;
    }
  } else {
    // storage contiguous along rows: 128 threads per k, 2 k per pass, 8 passes
    const int rr = tid & 127, kk = tid >> 7;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int64_t r = row0 + rr, kg = k + kk + 2 * p;
      reg[p] = (r < rmax && kg < kmax) ? vget(v, r, kg) : 0.0;
    }
  }
}
__device__ __forceinline__ void gemm_store_chunk(const View &v, double (*s)[GT + GPAD],
                                                 const double (&reg)[8]) {
  const int tid = threadIdx.x;
  if (!v.trans) {
    const int kk = tid & 15, rr = tid >> 4;
#pragma unroll
    for (int p = 0; p < 8; ++p) s[kk][rr + 16 * p] = reg[p];
  } else {
    const int rr = tid & 127, kk = tid >> 7;
#pragma unroll
    for (int p = 0; p < 8; ++p) s[kk + 2 * p][rr] = reg[p];
  }
}

__global__ void __launch_bounds__(256) gemm_f64_kernel(GemmArgs a) {
  int64_t ti, tj;
  if (a.tri_tiles) {
    const int64_t t = blockIdx.x;
    ti = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
  } else {
    ti = blockIdx.y;
    tj = blockIdx.x;
  }
  const int64_t i0 = ti * GT, j0 = tj * GT;
  if (i0 >= a.M || j0 >= a.N) return;
  const int64_t kb = a.k_from_row ? max(a.k0, a.ra + i0) : a.k0;
  const int64_t ke = a.k1;

  extern __shared__ __align__(16) double gsm[];
  double(*As)[GK][GT + GPAD] = reinterpret_cast<double(*)[GK][GT + GPAD]>(gsm);
  double(*Bs)[GK][GT + GPAD] = reinterpret_cast<double(*)[GK][GT + GPAD]>(gsm + 2 * GK * (GT + GPAD));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rbase = (warp >> 1) * 32 + (lane >> 3) * 8;
  const int cbase = (warp & 1) * 64 + (lane & 7) * 8;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  const int64_t ra = a.ra + i0, rb = a.rb + j0;
  const int64_t ramax = a.ra + a.M, rbmax = a.rb + a.N;
  double ra_reg[8], rb_reg[8];
  int st = 0;
  if (kb < ke) {
    gemm_load_chunk(a.A, ra, ramax, kb, ke, ra_reg);
    gemm_load_chunk(a.B, rb, rbmax, kb, ke, rb_reg);
    gemm_store_chunk(a.A, As[0], ra_reg);
    gemm_store_chunk(a.B, Bs[0], rb_reg);
  }
  __syncthreads();
  for (int64_t k = kb; k < ke; k += GK) {
    const bool more = k + GK < ke;
    if (more) {
      gemm_load_chunk(a.A, ra, ramax, k + GK, ke, ra_reg);
      gemm_load_chunk(a.B, rb, rbmax, k + GK, ke, rb_reg);
    }
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      double av[8], bv[8];
      const double2 *pa = reinterpret_cast<const double2 *>(&As[st][kk][rbase]);
      const double2 *pb = reinterpret_cast<const double2 *>(&Bs[st][kk][cbase]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 x = pa[q], y = pb[q];
        av[2 * q] = x.x;
        av[2 * q + 1] = x.y;
        bv[2 * q] = y.x;
        bv[2 * q + 1] = y.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      gemm_store_chunk(a.A, As[st ^ 1], ra_reg);
      gemm_store_chunk(a.B, Bs[st ^ 1], rb_reg);
    }
    __syncthreads();
    st ^= 1;
  }
  // epilogue through the C view (masked by its triangle)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t li = i0 + rbase + i;
    if (li >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t lj = j0 + cbase + j;
      if (lj >= a.N) continue;
      const int64_t r = a.rc + li, c = a.cc + lj;
      if (a.C.tri == 1 && r < c) continue;
      if (a.C.tri == 2 && c < r) continue;
      double x = a.alpha * acc[i][j];
      if (a.beta != 0.0) x += a.beta * vget(a.C, r, c);
      vset(a.C, r, c, x);
    }
  }
}

static int gemm(falkon_ctx *ctx, const GemmArgs &a) {
  if (a.M <= 0 || a.N <= 0) return FALKON_OK;
  const size_t smem = sizeof(double) * 4 * GK * (GT + GPAD);
  static bool attr_set = false;
  if (!attr_set) {
    FK_CUDA(cudaFuncSetAttribute(gemm_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr_set = true;
  }
  const int64_t tm = cdiv<int64_t>(a.M, GT), tn = cdiv<int64_t>(a.N, GT);
  LaunchScope ls(ctx, FALKON_T_PRECOND);
  if (a.tri_tiles) {
    gemm_f64_kernel<<<(unsigned)(tm * (tm + 1) / 2), 256, smem, ctx->stream>>>(a);
  } else {
    gemm_f64_kernel<<<dim3((unsigned)tn, (unsigned)tm), 256, smem, ctx->stream>>>(a);
  }
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

// ------------------------------------------------------------------ blocked Cholesky
static int potrf(falkon_ctx *ctx, View S, int64_t m, double *Wbuf, unsigned long long *fail) {
  const size_t dsm = sizeof(double) * NB * (NB + 1);
  static bool attr_set = false;
  if (!attr_set) {
    FK_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dsm));
    attr_set = true;
  }
  View W{Wbuf, NB, 0, 0, nullptr};
  for (int64_t k0 = 0; k0 < m; k0 += NB) {
    const int nb = (int)std::min<int64_t>(NB, m - k0);
    {
      LaunchScope ls(ctx, FALKON_T_PRECOND);
      potrf_diag_kernel<<<1, 512, dsm, ctx->stream>>>(S, k0, nb, Wbuf, fail);
    }
    FK_LAUNCH_CHECK();
    const int64_t k1 = k0 + nb, rem = m - k1;
    if (rem <= 0) break;
    // panel: L(k1:, k0:k1) = S(k1:, k0:k1) * W^T
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
    // A(r, k) = S(r, k0 + k'): express k in S coordinates; B(j, k) = W(j, k - k0)
    // -> use a shifted W view: W is addressed with column k - k0 via base offset trick
    p.k0 = k0;
    p.k1 = k1;
    p.B.base = Wbuf - k0;  // W(j, k) at Wbuf[j*NB + (k - k0)]
    p.alpha = 1.0;
    p.beta = 0.0;
    FK_TRY(gemm(ctx, p));
    // trailing: S(k1:, k1:) -= L(k1:, k0:k1) L(k1:, k0:k1)^T   (lower tiles)
    GemmArgs t{};
    t.A = S;
    t.B = S;
    t.C = S;
    t.M = rem;
    t.N = rem;
    t.ra = k1;
    t.rb = k1;
    t.rc = k1;
    t.cc = k1;
    t.k0 = k0;
    t.k1 = k1;
    t.tri_tiles = 1;
    t.alpha = -1.0;
    t.beta = 1.0;
    FK_TRY(gemm(ctx, t));
  }
  return FALKON_OK;
}

__global__ void add_diag_kernel(double *dvec, int64_t m, double scale, double add) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) dvec[i] = dvec[i] * scale + add;
}

int precond_build(falkon_ctx *ctx, const float *C, int64_t m, int64_t d, int kernel, double sigma,
                  double lambda, double jitter, double *P, double *diagT, double *diagA,
                  falkon_fit_info *info) {
  void *flags, *wb;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64, &flags));
  FK_TRY(ws_get(ctx, WS_PW, sizeof(double) * NB * NB, &wb));
  unsigned long long *failf = (unsigned long long *)flags;
  FK_CUDA(cudaMemsetAsync(failf, 0xff, 16, ctx->stream));
  View L1{P, m, 1, 1, diagT};  // L1 = T^T, stored in the upper triangle
  View L2{P, m, 0, 1, diagA};  // L2 = A^T, stored in the lower triangle
  View Tv{P, m, 0, 2, diagT};  // T itself (upper view of the same storage)
  // (b) Kmm + delta I
  {
    const int64_t tt = cdiv<int64_t>(m, 64);
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    kmm_kernel<<<(unsigned)(tt * (tt + 1) / 2), 256, 0, ctx->stream>>>(
        C, m, d, kernel, 1.0 / (2.0 * sigma * sigma), 1.0 / sigma, jitter, L1);
  }
  FK_LAUNCH_CHECK();
  // (c) T
  FK_TRY(potrf(ctx, L1, m, (double *)wb, failf));
  // (d) M = T T^T / m + lambda I  -> lower triangle + diagA:  M(i,j) = sum_{k>=i} T(i,k) T(j,k)
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
    FK_TRY(gemm(ctx, g));
    LaunchScope ls(ctx, FALKON_T_PRECOND);
    add_diag_kernel<<<(unsigned)cdiv<int64_t>(m, 256), 256, 0, ctx->stream>>>(diagA, m, 1.0,
                                                                                lambda);
  }
  FK_LAUNCH_CHECK();
  // (e) A^T
  FK_TRY(potrf(ctx, L2, m, (double *)wb, failf + 1));
  unsigned long long hf[2];
  FK_CUDA(cudaMemcpyAsync(hf, failf, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info) {
    info->failed_factor = -1;
    info->failed_column = -1;
    info->jitter_used = jitter;
  }
  for (int f = 0; f < 2; ++f) {
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

// ------------------------------------------------------------------ sync-free blocked TRSV
// Solves L z = r (forward) or L^T z = r (backward) in place for the lower-triangular view L.
// CTA with ticket b owns row block I (forward: I = b, backward: I = nb-1-b).  Off-diagonal
// tiles are streamed from HBM as soon as the needed z_J is flagged ready; the 64 x 64
// diagonal block is then solved by one warp.  flags[J] == gen marks z_J final.
__global__ void __launch_bounds__(256) trsv_kernel(View L, int64_t m, int forward,
                                                   double *__restrict__ z,
                                                   unsigned int *__restrict__ counter,
                                                   unsigned int *__restrict__ flags,
                                                   unsigned int gen) {
  __shared__ unsigned int s_ticket;
  __shared__ double szj[TB];
  __shared__ double part[4][TB];
  __shared__ double sdiag[TB][TB + 1];
  const int tid = threadIdx.x;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  if (tid == 0) s_ticket = atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t b = s_ticket;
  const int64_t I = forward ? b : nblk - 1 - b;
  const int64_t i0 = I * TB;
  const int nI = (int)lmin(TB, m - i0);
  // preload the diagonal tile: sdiag[i][j] = L(i0+i, i0+j) for i >= j
  for (int e = tid; e < TB * TB; e += 256) {
    const int i = e / TB, j = e % TB;
    sdiag[i][j] = (i < nI && j < nI && i >= j) ? vget(L, i0 + i, i0 + j) : 0.0;
  }
  // thread -> (row i, quarter q) of the off-diagonal tile mat-vec
  const int ri = tid & 63, q = tid >> 6;
  double acc = 0.0;
  const int64_t nJ = forward ? I : nblk - 1 - I;
  for (int64_t s = 0; s < nJ; ++s) {
    const int64_t J = forward ? s : nblk - 1 - s;
    const int64_t j0 = J * TB;
    const int nJc = (int)lmin(TB, m - j0);
    if (tid == 0) {
      volatile unsigned int *f = flags + J;
      while (*f != gen) {
      }
      __threadfence();
    }
    __syncthreads();
    if (tid < TB) szj[tid] = (tid < nJc) ? ((volatile double *)z)[j0 + tid] : 0.0;
    __syncthreads();
    if (ri < nI) {
      // forward: acc_i += L(i0+ri, j0+j) z_j ; backward: acc_i += L(j0+j, i0+ri) z_j
      for (int jj = 0; jj < 16; ++jj) {
        const int j = q * 16 + jj;
        if (j < nJc) {
          const double lv = forward ? L.base[vidx(L, i0 + ri, j0 + j)]
                                    : L.base[vidx(L, j0 + j, i0 + ri)];
          acc = fma(lv, szj[j], acc);
        }
      }
    }
    __syncthreads();
  }
  part[q][ri] = acc;
  __syncthreads();
  // one warp solves the diagonal block: rows 2*lane, 2*lane+1
  if (tid < 32) {
    const int lane = tid;
    double x[2];
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * lane + h;
      x[h] = (i < nI) ? z[i0 + i] - (part[0][i] + part[1][i] + part[2][i] + part[3][i]) : 0.0;
    }
    if (forward) {
      for (int j = 0; j < nI; ++j) {
        const int owner = j >> 1;
        double xj = __shfl_sync(0xffffffffu, (j & 1) ? x[1] : x[0], owner);
        xj /= sdiag[j][j];
        if (lane == owner) x[j & 1] = xj;
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * lane + h;
          if (i > j && i < nI) x[h] -= sdiag[i][j] * xj;
        }
      }
    } else {
      for (int j = nI - 1; j >= 0; --j) {
        const int owner = j >> 1;
        double xj = __shfl_sync(0xffffffffu, (j & 1) ? x[1] : x[0], owner);
        xj /= sdiag[j][j];
        if (lane == owner) x[j & 1] = xj;
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * lane + h;
          if (i < j) x[h] -= sdiag[j][i] * xj;  // (L^T)(i, j) = L(j, i)
        }
      }
    }
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * lane + h;
      if (i < nI) z[i0 + i] = x[h];
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(flags + I, gen);
  }
}

int trsv(falkon_ctx *ctx, const double *P, const double *diag, int64_t m, int which, int trans,
         double *x) {
  // which 0: T = L1^T (L1 = view trans=1 of the upper triangle); which 1: A = L2^T.
  // T x = r  <=> L1^T x = r (backward);  T^T x = r <=> L1 x = r (forward); same for A.
  View L{const_cast<double *>(P), m, which == 0 ? 1 : 0, 1, const_cast<double *>(diag)};
  const int forward = trans ? 1 : 0;
  const int64_t nblk = cdiv<int64_t>(m, TB);
  void *fl;
  FK_TRY(ws_get(ctx, WS_FLAGS, 64 + sizeof(unsigned int) * (nblk + 64), &fl));
  unsigned int *counter = (unsigned int *)((char *)fl + 32);
  unsigned int *flags = counter + 8;
  static unsigned int gen_counter = 0;  // monotone generation id (flags never need clearing)
  unsigned int gen = ++gen_counter;
  if (gen == 0) gen = ++gen_counter;
  FK_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), ctx->stream));
  LaunchScope ls(ctx, FALKON_T_TRSV);
  trsv_kernel<<<(unsigned)nblk, 256, 0, ctx->stream>>>(L, m, forward, x, counter, flags, gen);
  FK_LAUNCH_CHECK();
  return FALKON_OK;
}

}  // namespace falkon
