// precond.cuh — matrix views of the preconditioner's m x m buffer and the fp64 GEMM argument
// block, shared by precond.cu (blocked Cholesky, DMMA GEMMs, TRSV) and ozaki.cu (the int8
// tensor-core emulation of the trailing-update GEMMs).
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace falkon {

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
  const double *kscale;  // optional: B(j, k) is multiplied by kscale[k] (weighted LAUUM, Alg. 2)
};

// Ozaki-scheme GEMM (ozaki.cu): the same contract as the DMMA GEMM for the cases it accepts
// (plain k range of at most OZ_KMAX, no kscale); returns FALKON_OK when it ran, OZ_DECLINED when
// the caller must use the DMMA kernels, an error code otherwise.
constexpr int OZ_DECLINED = 1000;
int oz_gemm(falkon_ctx *ctx, const GemmArgs &a);

}  // namespace falkon
