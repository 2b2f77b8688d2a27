// Unit-lower triangular solve  B := trilu(L)^-1 B  on one column strip (reference kernels.py:264-293
// trsm_llu/_trsm_cols: forward substitution per column, diagonal never read).
//
// GPU form, per strip of up to TRSM_CW columns owned by one CTA (the reference splits columns over
// team members the same way, kernels.py:289):  left-looking over 32-row blocks
//     X[kb] = B[kb] - L[kb, 0:kb*32] @ X[0:kb*32]        (DMMA tile, accumulators -> shared memory)
//     X[kb] = trilu(L[kb,kb])^-1 X[kb]                    (32-step substitution, one thread per column)
// so w^2*c/2 of the w^2*c flops run on the FP64 tensor pipe and each column's arithmetic is
// independent of how columns are distributed (same determinism argument as the reference).
#pragma once
#include "mla_common.cuh"
#include "mla_gemm.cuh"

namespace mla {

constexpr int TRSM_CW = 128;   // strip width (== GemmUpdateCfg::BN, so an update tile depends on one strip)
constexpr int TRSM_RB = 32;    // row block
constexpr int TRSM_LDX = 34;   // leading dimension of the X block in shared memory (even: 16-B rows)
constexpr int TRSM_LDL = 33;
constexpr int TRSM_SMEM_DOUBLES = GemmTrsmCfg::SMEM_BYTES / 8 + TRSM_CW * TRSM_LDX + TRSM_RB * TRSM_LDL;

// One row-block step of the left-looking solve: rows [r0, r0+rb) of the strip, rb <= TRSM_RB,
//   X = B[r0:r0+rb, :] - L[r0:r0+rb, 0:r0] @ B[0:r0, :];   X = trilu(L[r0:r0+rb, r0:r0+rb])^-1 X.
// Collective over the CTA.  This is also the panel's "U row-block" step (Crout order): the rows of U
// that a just-factored diagonal block determines, for all the panel's later columns at once.
__device__ inline void trsm_rowblock(const double* __restrict__ L, int r0, int rb, int64_t ldl, double* B,
                                     int cw, int64_t ldb, double* smem) {
  double* ring = smem;
  double* Xs = smem + GemmTrsmCfg::SMEM_BYTES / 8;   // [cw][TRSM_LDX]
  double* Ls = Xs + TRSM_CW * TRSM_LDX;              // [32][TRSM_LDL]  (row i, col l) at Ls[i*LDL+l]
  const int tid = threadIdx.x;
  __syncthreads();
  if (r0 > 0) {
    gemm_tile<GemmTrsmCfg>(L + r0, ldl, B, ldb, r0, B + r0, ldb, Xs, TRSM_LDX, rb, cw, 1.0, -1.0, ring);
  } else {
    for (int x = tid; x < rb * cw; x += kThreads) {
      int c = x / rb, i = x - c * rb;
      Xs[c * TRSM_LDX + i] = B[(int64_t)c * ldb + i];
    }
  }
  for (int x = tid; x < rb * rb; x += kThreads) {
    int l = x / rb, i = x - l * rb;  // column l of the diagonal block, rows contiguous in memory
    Ls[i * TRSM_LDL + l] = L[(int64_t)(r0 + l) * ldl + r0 + i];
  }
  __syncthreads();
  if (tid < cw) {
    double x[TRSM_RB];
    double* xs = Xs + tid * TRSM_LDX;
#pragma unroll
    for (int i = 0; i < TRSM_RB; ++i) x[i] = (i < rb) ? xs[i] : 0.0;
#pragma unroll
    for (int l = 0; l < TRSM_RB - 1; ++l) {
      if (l < rb - 1) {
#pragma unroll
        for (int i = l + 1; i < TRSM_RB; ++i)
          if (i < rb) x[i] = fma(-Ls[i * TRSM_LDL + l], x[l], x[i]);
      }
    }
    double* bo = B + (int64_t)tid * ldb + r0;
#pragma unroll
    for (int i = 0; i < TRSM_RB; ++i)
      if (i < rb) bo[i] = x[i];
  }
}

// Collective over the CTA.  L: w x w (ldl), B: w x cw strip (ldb), cw <= TRSM_CW.
__device__ inline void trsm_strip(const double* __restrict__ L, int w, int64_t ldl, double* B, int cw,
                                  int64_t ldb, double* smem) {
  for (int r0 = 0; r0 < w; r0 += TRSM_RB) trsm_rowblock(L, r0, imin(TRSM_RB, w - r0), ldl, B, cw, ldb, smem);
  __syncthreads();
}

}  // namespace mla
