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

// ---- the solve in 128-row steps with explicitly inverted diagonal blocks --------------------------------------
// For the update's PREP items (w = the panel width, up to 1024) the 32-row form above is latency-bound: 16
// dependent steps of a 32 x 128 x r0 gemm + a 32-step substitution cost ~24 us each whatever their size.
// Here a step is 128 rows and both of its parts are full tiles of the update's tile engine:
//     T     = B[r0:r0+128] - L[r0:r0+128, 0:r0] @ X[0:r0]          (128 x 128 x r0)
//     X[kb] = inv(trilu(L[kb,kb])) @ T                              (128 x 128 x 128)
// 4 steps instead of 16 at w = 512.  The inverses D[kb] are computed once per panel (diag_block_inverse: the
// substitution-based solve above applied to the identity) by whoever produced the panel.  trilu(L) of a
// partial-pivoting panel has |l_ij| <= 1, its 128 x 128 blocks are well conditioned in practice; the
// result differs from substitution in the last bits only (parity: tests/parity.py bound).
constexpr int TRSM_IB = 128;
constexpr int kMaxInvBlocks = 8;                 // panels of up to 1024 columns (kMaxPiv)
// Below this many rows the 32-row substitution form is used: inverting the diagonal blocks costs ~60 us on the
// path from a panel to the solves that use it, which narrow (ET-cut) panels do not earn back.
constexpr int kInvMinRows = 192;
__host__ __device__ constexpr bool trsm_use_inverse(int w) { return w >= kInvMinRows && w <= kMaxInvBlocks * TRSM_IB; }
struct DiagInv { double d[kMaxInvBlocks][TRSM_IB * TRSM_IB]; };   // column-major blocks, leading dimension TRSM_IB

// Collective over the CTA: out (ld TRSM_IB) = trilu(L[r0:r0+rb, r0:r0+rb])^-1, zero outside rb x rb.
__device__ inline void diag_block_inverse(const double* __restrict__ L, int r0, int rb, int64_t ldl, double* out,
                                          double* smem) {
  __syncthreads();
  for (int x = threadIdx.x; x < TRSM_IB * TRSM_IB; x += kThreads) {
    const int c = x / TRSM_IB, i = x - c * TRSM_IB;
    out[x] = (i == c && i < rb) ? 1.0 : 0.0;
  }
  __threadfence();
  __syncthreads();
  trsm_strip(L + (int64_t)r0 * ldl + r0, rb, ldl, out, rb, TRSM_IB, smem);
  __threadfence();
  __syncthreads();
}

// The substitution form as an out-of-line function, for the update's PREP items (a handful of call sites in
// the persistent kernel: inlined, they change the register allocation of the tile loops around them).
static __device__ __noinline__ void trsm_strip_ool(const double* __restrict__ L, int w, int64_t ldl, double* B, int cw,
                                                   int64_t ldb, double* smem) {
  trsm_strip(L, w, ldl, B, cw, ldb, smem);
}

// Collective over the CTA; smem needs GemmUpdateCfg::SMEM_BYTES.  Out of line on purpose (one copy of the
// tile engine per kernel instead of one per call site); hence the tiles without the bulk reduction.
static __device__ __noinline__ void trsm_strip_inv(const double* __restrict__ L, int w, int64_t ldl, double* B, int cw,
                                            int64_t ldb, const DiagInv* inv, double* smem) {
  int kb = 0;
  for (int r0 = 0; r0 < w; r0 += TRSM_IB, ++kb) {
    const int rb = imin(TRSM_IB, w - r0);
    double* Bk = B + r0;
    if (r0 > 0) {
      gemm_tile<GemmUpdateCfg, false>(L + r0, ldl, B, ldb, r0, Bk, ldb, Bk, ldb, rb, cw, 1.0, -1.0, smem);
      __threadfence();     // T (plain stores) must be in L2 before the next tile's cp.async reads it
      __syncthreads();
    }
    // in place: every slice of T is staged (and consumed) before the epilogue's first store
    gemm_tile<GemmUpdateCfg, false>(inv->d[kb], TRSM_IB, Bk, ldb, rb, Bk, ldb, Bk, ldb, rb, cw, 0.0, 1.0, smem);
    __threadfence();
    __syncthreads();
  }
}

}  // namespace mla
