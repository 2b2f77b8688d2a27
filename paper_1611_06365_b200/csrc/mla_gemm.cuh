// FP64 tensor-core (DMMA.8x8x4) tile multiply:  Cout = alpha*Cin + beta*(A @ B)  on one BM x BN
// tile, all operands column-major.  This is the GPU replacement of the reference's packed
// five-loop GEMM (kernels.py:42-160: _pack_a_slabs/_pack_b_slabs/_tile_product/_macro_block):
//   * packing into slab buffers  -> cp.async (LDGSTS, 16 B, zero-fill at the fringes) into a
//     STAGES-deep shared-memory ring; padding of 4 doubles per row makes every DMMA fragment
//     load (LDS.64) bank-conflict free,
//   * the m_r x n_r register micro-tile -> per-warp (WTI x WTJ) accumulator block of DMMA tiles,
//   * ascending-k accumulation from zero, one owner per C element (kernels.py:3-9): kept, so the
//     result does not depend on which CTA picked the tile or when.
//
// Orientation.  mma.m8n8k4 computes D(8x8) = A'(8x4,row) * B'(4x8,col).  We feed A' = U12^T-free:
//   A'[r][k] = B[k][j0+r]   (the k x n operand, k contiguous in memory)
//   B'[k][c] = A[i0+c][k]   (the m x k operand, i contiguous in memory)
// so D[r][c] = sum_k A[i0+c][k] * B[k][j0+r] = (A@B)[i0+c][j0+r]: lane T ends up owning two
// vertically adjacent C entries (rows i0+2*(T%4)+{0,1} of column j0+T/4), i.e. one aligned 16-byte
// word of the column-major C.
#pragma once
#include "mla_common.cuh"

namespace mla {

template <int BM_, int BN_, int WI_, int WJ_, int STAGES_, int BK_ = 16, int THREADS_ = kThreads>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, WI = WI_, WJ = WJ_, STAGES = STAGES_;
  static constexpr int BK = BK_;
  static constexpr int THREADS = THREADS_;   // threads of the CTA (or thread group) running the tile
  static constexpr int LDA_S = BM + 4;  // (BM+4) % 16 == 4 -> conflict-free fragment loads
  static constexpr int LDB_S = BK + 4;
  static constexpr int A_STAGE = BK * LDA_S;
  static constexpr int B_STAGE = BN * LDB_S;
  static constexpr int STAGE = A_STAGE + B_STAGE;  // doubles per stage
  static constexpr int SMEM_BYTES = STAGES * STAGE * 8;
  static constexpr int WTI = BM / WI, WTJ = BN / WJ;
  static constexpr int NI = WTI / 8, NJ = WTJ / 8;
  // can the slice be issued as BK/4 equal unpredicated parts (one per k4 step)?
  static constexpr int PARTS = BK / 4;
  static constexpr bool FAST_OK = (THREADS % (BM / 2) == 0) && (BK % (THREADS / (BM / 2)) == 0) &&
                                  ((BK / (THREADS / (BM / 2))) % PARTS == 0) && (THREADS % (BK / 2) == 0) &&
                                  (BN % (THREADS / (BK / 2)) == 0) && ((BN / (THREADS / (BK / 2))) % PARTS == 0);
  static_assert(WI * WJ * 32 == THREADS, "one warp per (WI, WJ) cell");
  static_assert(BM % 16 == 0 && BN % 8 == 0 && WTI % 8 == 0 && WTJ % 8 == 0, "tile shape");
};

using GemmUpdateCfg = GemmCfg<128, 128, 2, 4, 3, 32>;  // trailing update tiles
// Panel-internal update (N = the panel's device block: 32 columns, or 16 / 8 after slab fitting).  32-deep slices in a
// 2-stage ring: the same shared memory as four 16-deep stages, half as many barriers per tile -- these narrow
// tiles are bound by the latency around each slice, not by the DMMA pipe (panel gemm -5 %, round 2).
using GemmPanelCfg = GemmCfg<128, 32, 8, 1, 2, 32>;
using GemmPanel16Cfg = GemmCfg<128, 16, 8, 1, 2, 32>;
using GemmPanel8Cfg = GemmCfg<128, 8, 8, 1, 2, 32>;
using GemmTrsmCfg = GemmCfg<32, 128, 1, 8, 4>;     // row-block update inside trsm strips

// Issue the cp.async loads of k-tile `kt` into ring slot `slot`.
template <class Cfg, bool AL16>
__device__ __forceinline__ void gemm_load_stage(double* smem, int slot, const double* __restrict__ A,
                                                int64_t lda, const double* __restrict__ B, int64_t ldb,
                                                int K, int kt, int mrem, int nrem) {
  double* sA = smem + slot * Cfg::STAGE;
  double* sB = sA + Cfg::A_STAGE;
  const int k0 = kt * Cfg::BK;
  const int tid = grp_tid<Cfg::THREADS>();
  if (AL16) {
    constexpr int ACH = Cfg::BM / 2;
    for (int c = tid; c < Cfg::BK * ACH; c += Cfg::THREADS) {
      int kk = c / ACH, i = 2 * (c % ACH);
      int valid = (k0 + kk < K) ? imin(imax(mrem - i, 0), 2) * 8 : 0;
      const double* src = valid ? (A + (int64_t)(k0 + kk) * lda + i) : A;
      cp_async16(sA + kk * Cfg::LDA_S + i, src, valid);
    }
    constexpr int BCH = Cfg::BK / 2;
    for (int c = tid; c < Cfg::BN * BCH; c += Cfg::THREADS) {
      int j = c / BCH, kk = 2 * (c % BCH);
      int valid = (j < nrem) ? imin(imax(K - (k0 + kk), 0), 2) * 8 : 0;
      const double* src = valid ? (B + (int64_t)j * ldb + k0 + kk) : B;
      cp_async16(sB + j * Cfg::LDB_S + kk, src, valid);
    }
  } else {
    for (int c = tid; c < Cfg::BK * Cfg::BM; c += Cfg::THREADS) {
      int kk = c / Cfg::BM, i = c % Cfg::BM;
      int valid = (k0 + kk < K && i < mrem) ? 8 : 0;
      const double* src = valid ? (A + (int64_t)(k0 + kk) * lda + i) : A;
      cp_async8(sA + kk * Cfg::LDA_S + i, src, valid);
    }
    for (int c = tid; c < Cfg::BN * Cfg::BK; c += Cfg::THREADS) {
      int j = c / Cfg::BK, kk = c % Cfg::BK;
      int valid = (j < nrem && k0 + kk < K) ? 8 : 0;
      const double* src = valid ? (B + (int64_t)j * ldb + k0 + kk) : B;
      cp_async8(sB + j * Cfg::LDB_S + kk, src, valid);
    }
  }
}

// Fast path of the staging: interior tile (mrem == BM, nrem == BN), whole BK slice inside K, 16-byte
// aligned operands.  All address arithmetic is a per-thread base plus compile-time strides, hoisted out
// of the k loop.  The slice is cut into PARTS = BK/4 parts so the main loop can issue one part per k4
// step: a burst of LDGSTS at the top of a k-tile would sit in the MIO queue in front of the fragment
// LDS.64 and starve the DMMA pipe.
// Per-thread, per-tile constants of the fast path (hoisted out of the k loop).
template <class Cfg>
struct FastSrc {
  const double* ap;     // A + ar*lda + ac            (+ kt*BK*lda per k-tile, + p*AROWS*lda per pass)
  const double* bp;     // B + bc*ldb + bk            (+ kt*BK per k-tile,     + p*BCOLS*ldb per pass)
  int kfull;            // number of whole BK slices (fast slices are kt < kfull); 0: tile not fast
};

template <class Cfg, class Desc>
__device__ __forceinline__ FastSrc<Cfg> make_fast_src(const Desc& d) {
  FastSrc<Cfg> f;
  constexpr int ACH = Cfg::BM / 2, BCH = Cfg::BK / 2;
  const int tid = grp_tid<Cfg::THREADS>();
  const bool fast = Cfg::FAST_OK && d.valid && ((((uintptr_t)d.A | (uintptr_t)d.B) & 15) == 0) &&
                    ((d.lda & 1) == 0) && ((d.ldb & 1) == 0) && d.mrem >= Cfg::BM && d.nrem >= Cfg::BN;
  f.kfull = fast ? d.K / Cfg::BK : 0;
  f.ap = d.A + (int64_t)(tid / ACH) * d.lda + 2 * (tid % ACH);
  f.bp = d.B + (int64_t)(tid / BCH) * d.ldb + 2 * (tid % BCH);
  return f;
}

// Part `part` (of BK/4) of interior slice kt, all addresses from the hoisted constants.
template <class Cfg>
__device__ __forceinline__ void gemm_load_part_hoisted(double* sdstA, double* sdstB, int64_t a_pass, int64_t b_pass,
                                                       const double* ap_kt, const double* bp_kt, int part) {
  constexpr int PARTS = Cfg::BK / 4;
  constexpr int ACH = Cfg::BM / 2, AROWS = Cfg::THREADS / ACH, APASS = Cfg::BK / AROWS;
  constexpr int BCH = Cfg::BK / 2, BCOLS = Cfg::THREADS / BCH, BPASS = Cfg::BN / BCOLS;
#pragma unroll
  for (int pp = 0; pp < APASS / PARTS; ++pp) {
    const int p = part * (APASS / PARTS) + pp;
    cp_async16(sdstA + p * AROWS * Cfg::LDA_S, ap_kt + p * a_pass, 16);
  }
#pragma unroll
  for (int pp = 0; pp < BPASS / PARTS; ++pp) {
    const int p = part * (BPASS / PARTS) + pp;
    cp_async16(sdstB + p * BCOLS * Cfg::LDB_S, bp_kt + p * b_pass, 16);
  }
}

// ---- bulk asynchronous reduction (TMA engine): global[dst] += shared[src] in L2 ----------------------
// Used by the LU update's epilogue: C -= A@B becomes "stage -acc in shared memory, let the TMA engine
// add it into C", so the SM neither reads C nor waits for it and moves straight on to the next tile.
__device__ __forceinline__ void bulk_red_add_f64(double* gdst, const double* ssrc, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// all bulk reductions issued by this thread have been performed (their results are in L2 / global)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
constexpr int RED_LDS = 136;   // doubles per staged column (1088 B: conflict-free STS.128, 16-B aligned)

// Description of one C tile for the pipelined tile engine.
struct TileDesc {
  const double* A; int64_t lda;       // mrem x K
  const double* B; int64_t ldb;       // K x nrem
  const double* Cin; int64_t ldcin;
  double* Cout; int64_t ldcout;       // may be shared memory (generic pointer)
  int K, mrem, nrem;
  double alpha, beta;
  bool valid;
};

template <class Cfg>
__device__ __forceinline__ int tile_kt(const TileDesc& d) { return (d.K + Cfg::BK - 1) / Cfg::BK; }

// Issue (and commit as one group) the loads of k-tile `kt` of tile d into ring slot `slot`; an
// out-of-range kt or an invalid tile commits an empty group so that group accounting stays uniform.
template <class Cfg>
__device__ __forceinline__ void tile_issue(const TileDesc& d, int kt, int slot, double* smem) {
  if (d.valid && kt < tile_kt<Cfg>(d)) {
    const bool al16 = ((((uintptr_t)d.A | (uintptr_t)d.B) & 15) == 0) && ((d.lda & 1) == 0) && ((d.ldb & 1) == 0);
    const int mrem = imin(d.mrem, Cfg::BM), nrem = imin(d.nrem, Cfg::BN);
    if (al16)
      gemm_load_stage<Cfg, true>(smem, slot, d.A, d.lda, d.B, d.ldb, d.K, kt, mrem, nrem);
    else
      gemm_load_stage<Cfg, false>(smem, slot, d.A, d.lda, d.B, d.ldb, d.K, kt, mrem, nrem);
  }
  cp_async_commit();
}

// Prime the ring for tile d: positions 0..STAGES-2 of its k-stream go to slots base.. .
template <class Cfg>
__device__ __forceinline__ void tile_prologue(const TileDesc& d, int base, double* smem) {
  grp_sync<Cfg::THREADS>();  // previous user of the ring is done
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) tile_issue<Cfg>(d, s, (base + s) % Cfg::STAGES, smem);
}

// Main loop + epilogue of tile d whose first STAGES-1 k-tiles are already in flight (tile_prologue or
// the previous tile's main loop).  While d's last k-tiles are consumed the first k-tiles of `next`
// are prefetched into the ring, so the next tile starts without a pipeline bubble and d's epilogue
// (C read-modify-write) overlaps next's loads.  Returns the ring base of `next`.
#ifdef MLA_TILE_PROF
// Instrumented build only (tools/README.md): clock accounting of CTA 0 / thread 0 per tile --
// [0] tiles [1] total clk [2] clk in cp.async wait + barrier [3] epilogue clk [4] staging of the
// first half [5] bulk issue + wait for the engine to have read the first half [6] start-of-tile wait for the
// previous tile's read + issue of the second half's operations [7] proxy fence of the second half
__device__ unsigned long long g_tprof[8];
#endif
#ifndef MLA_TILE_ATTR
#define MLA_TILE_ATTR
#endif
// RED = false compiles the tile without the bulk-reduction epilogue (plain read-modify-write instead): for
// callers that live in out-of-line functions, where ptxas mis-encodes UBLKRED (see the note below).
template <class Cfg, bool RED = true>
__device__ MLA_TILE_ATTR int tile_run(const TileDesc& d, const TileDesc& next, int base, double* smem) {
#ifdef MLA_TILE_PROF
  const bool tp = blockIdx.x == 0 && threadIdx.x == 0;
  long long tp0 = clock64(), tpw = 0;
#endif
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES, NI = Cfg::NI, NJ = Cfg::NJ;
  const int tid = grp_tid<Cfg::THREADS>(), lane = tid & 31, warp = tid >> 5;
  const int wi = warp % Cfg::WI, wj = warp / Cfg::WI;
  const int g = lane >> 2, q = lane & 3;
  const int mrem = imin(d.mrem, Cfg::BM), nrem = imin(d.nrem, Cfg::BN);
  const int KT = tile_kt<Cfg>(d);

  double acc[NJ][NI][2];
#pragma unroll
  for (int a = 0; a < NJ; ++a)
#pragma unroll
    for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // Pull the C tile into L2 now: the epilogue's read-modify-write then pays L2 instead of HBM latency
  // for each of its batches (the DMMA pipe idles during the epilogue).
  if (KT >= 2 && __isGlobal(d.Cin)) {
    constexpr int LPC = (Cfg::BM * 8 + 127) / 128;      // 128-byte lines per tile column
    for (int x = tid; x < nrem * LPC; x += Cfg::THREADS) {
      int col = x / LPC, seg = x - col * LPC;
      if (seg * 16 < mrem)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(d.Cin + (int64_t)col * d.ldcin + seg * 16));
    }
  }

  // the previous tile's epilogue may still be reading its staged accumulators out of the ring slot this
  // tile's first load will overwrite
#ifdef MLA_TILE_PROF
  long long tr0 = clock64();
#endif
  if constexpr (RED && Cfg::FAST_OK) bulk_wait_read0();
#ifdef MLA_TILE_PROF
  if (tp) g_tprof[6] += clock64() - tr0;
#endif

  // fast-path constants of this tile and of the prefetched successor, hoisted out of the k loop
  const FastSrc<Cfg> fd = make_fast_src<Cfg>(d);
  FastSrc<Cfg> fn = make_fast_src<Cfg>(next);
  if (next.valid && (next.lda != d.lda || next.ldb != d.ldb)) fn.kfull = 0;   // strides are shared below
  constexpr int ACH_ = Cfg::BM / 2, BCH_ = Cfg::BK / 2;
  const int64_t a_kt = (int64_t)Cfg::BK * d.lda;
  const int64_t a_pass = (int64_t)(Cfg::THREADS / ACH_) * d.lda, b_pass = (int64_t)(Cfg::THREADS / BCH_) * d.ldb;
  double* const sdA0 = smem + (tid / ACH_) * Cfg::LDA_S + 2 * (tid % ACH_);
  double* const sdB0 = smem + Cfg::A_STAGE + (tid / BCH_) * Cfg::LDB_S + 2 * (tid % BCH_);

  for (int kt = 0; kt < KT; ++kt) {
#ifdef MLA_TILE_PROF
    long long tw0 = clock64();
#endif
    cp_async_wait<STAGES - 2>();
    grp_sync<Cfg::THREADS>();
#ifdef MLA_TILE_PROF
    tpw += clock64() - tw0;
#endif
    const int pos = kt + STAGES - 1;
    const int lslot = (base + pos) % STAGES;
    const bool cur_tile = pos < KT;
    const int lkt = cur_tile ? pos : pos - KT;
    const bool lfast = cur_tile ? (lkt < fd.kfull) : (lkt < fn.kfull);
    const double* ap_kt = (cur_tile ? fd.ap : fn.ap) + lkt * a_kt;
    const double* bp_kt = (cur_tile ? fd.bp : fn.bp) + lkt * Cfg::BK;
    double* const sdA = sdA0 + lslot * Cfg::STAGE;
    double* const sdB = sdB0 + lslot * Cfg::STAGE;
    if (!lfast) tile_issue<Cfg>(cur_tile ? d : next, lkt, lslot, smem);   // fringe / unaligned: whole slice at once
    MLA_STRESS((warp & 1) == (kt & 1) && (kt % 5 == 4 || kt == KT - 1));   // skew the warps inside the k loop
    const double* sA = smem + ((base + kt) % STAGES) * Cfg::STAGE;
    const double* sB = sA + Cfg::A_STAGE;
    const double* pa = sA + q * Cfg::LDA_S + wi * Cfg::WTI + g;       // + k4*4*LDA_S + ni*8
    const double* pb = sB + (wj * Cfg::WTJ + g) * Cfg::LDB_S + q;     // + nj*8*LDB_S + k4*4
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double fi[NI], fj[NJ];
#pragma unroll
      for (int b = 0; b < NI; ++b) fi[b] = pa[k4 * 4 * Cfg::LDA_S + b * 8];
#pragma unroll
      for (int a = 0; a < NJ; ++a) fj[a] = pb[a * 8 * Cfg::LDB_S + k4 * 4];
      if constexpr (Cfg::FAST_OK) {
        if (lfast) gemm_load_part_hoisted<Cfg>(sdA, sdB, a_pass, b_pass, ap_kt, bp_kt, k4);
      }
#pragma unroll
      for (int a = 0; a < NJ; ++a)
#pragma unroll
        for (int b = 0; b < NI; ++b) dmma884(acc[a][b][0], acc[a][b][1], fj[a], fi[b]);
    }
    if (lfast) cp_async_commit();
  }
  if (!next.valid) cp_async_wait<0>();
#ifdef MLA_TILE_PROF
  long long tpe = clock64();
#endif

  // epilogue: lane owns rows i..i+1 of column j for every (nj, ni) block.  Loads are batched per
  // j-block (NI independent 16-byte loads in flight) so the tile's C traffic is not a chain of
  // serialized round trips.
  const double alpha = d.alpha, beta = d.beta;
  const double* Cin = d.Cin;
  double* Cout = d.Cout;
  const int64_t ldcin = d.ldcin, ldcout = d.ldcout;
  const bool vec = ((((uintptr_t)Cin | (uintptr_t)Cout) & 15) == 0) && ((ldcin & 1) == 0) && ((ldcout & 1) == 0);
  const bool full = vec && mrem == Cfg::BM && nrem == Cfg::BN;
  bool red_done = false;
  if constexpr (RED && Cfg::FAST_OK && Cfg::BM == 128 && Cfg::BN == 128 && Cfg::WJ == 4) {
    if (full && alpha == 1.0 && beta == -1.0 && Cin == Cout && KT > 0 && __isGlobal(Cout)) {
      // C -= acc through the TMA engine: -acc is staged, half a tile (64 columns) at a time, in the ring
      // slot this tile consumed last, and added into C by one 1-KiB bulk reduction per column.
      double* stg = smem + ((base + KT - 1) % STAGES) * Cfg::STAGE;
      static_assert(64 * RED_LDS <= Cfg::STAGE, "staging fits one ring slot");
      // that slot is the one the k loop's LAST iteration read its fragments from: every warp must be
      // through with them before the first staging store lands there
#ifndef MLA_NO_EPILOGUE_BARRIER
      grp_sync<Cfg::THREADS>();
#endif
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if ((wj >> 1) == half) {
#pragma unroll
          for (int a = 0; a < NJ; ++a) {
            double* sp = stg + ((wj & 1) * Cfg::WTJ + a * 8 + g) * RED_LDS + wi * Cfg::WTI + 2 * q;
#pragma unroll
            for (int b = 0; b < NI; ++b)
              *reinterpret_cast<double2*>(sp + b * 8) = make_double2(-acc[a][b][0], -acc[a][b][1]);
          }
        }
#ifdef MLA_TILE_PROF
        long long tf0 = clock64();
#endif
        fence_proxy_async_smem();
#ifdef MLA_TILE_PROF
        long long tf1 = clock64();
#endif
        grp_sync<Cfg::THREADS>();
#ifdef MLA_TILE_PROF
        long long tq0 = clock64();
        if (tp && half == 0) g_tprof[4] += tq0 - tpe;
        if (tp && half == 1) { g_tprof[7] += tf1 - tf0; }
#endif
        if (tid < 64) {
          bulk_red_add_f64(Cout + (int64_t)(half * 64 + tid) * ldcout, stg + tid * RED_LDS, Cfg::BM * 8);
          bulk_commit();
#ifdef MLA_TILE_PROF
          if (tp && half == 1) g_tprof[6] += clock64() - tq0;   // (reuses slot 6) issue time of the second half
#endif
          if (half == 0) bulk_wait_read0();   // the second half reuses the staging area
        }
        if (half == 0) grp_sync<Cfg::THREADS>();
#ifdef MLA_TILE_PROF
        if (tp && half == 0) g_tprof[5] += clock64() - tq0;
#endif
      }
      if (!next.valid) {            // somebody else will use this shared memory next
        if (tid < 64) bulk_wait_read0();
        grp_sync<Cfg::THREADS>();
      }
      red_done = true;
    }
  }
  if (red_done) {
  } else if (full) {
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      int j = wj * Cfg::WTJ + a * 8 + g;
      const double* ci = Cin + (int64_t)j * ldcin + wi * Cfg::WTI + 2 * q;
      double* co = Cout + (int64_t)j * ldcout + wi * Cfg::WTI + 2 * q;
      double2 c[NI];
#pragma unroll
      for (int b = 0; b < NI; ++b) c[b] = *reinterpret_cast<const double2*>(ci + b * 8);
#pragma unroll
      for (int b = 0; b < NI; ++b) {
        if (alpha == 1.0) { c[b].x = fma(beta, acc[a][b][0], c[b].x); c[b].y = fma(beta, acc[a][b][1], c[b].y); }
        else { c[b].x = alpha * c[b].x + beta * acc[a][b][0]; c[b].y = alpha * c[b].y + beta * acc[a][b][1]; }
      }
#pragma unroll
      for (int b = 0; b < NI; ++b) *reinterpret_cast<double2*>(co + b * 8) = c[b];
    }
  } else {
#pragma unroll
    for (int a = 0; a < NJ; ++a) {
      int j = wj * Cfg::WTJ + a * 8 + g;
      if (j >= nrem) continue;
#pragma unroll
      for (int b = 0; b < NI; ++b) {
        int i = wi * Cfg::WTI + b * 8 + 2 * q;
        if (i >= mrem) continue;
        const double* ci = Cin + (int64_t)j * ldcin + i;
        double* co = Cout + (int64_t)j * ldcout + i;
        if (vec && i + 1 < mrem) {
          double2 c = *reinterpret_cast<const double2*>(ci);
          if (alpha == 1.0) { c.x = fma(beta, acc[a][b][0], c.x); c.y = fma(beta, acc[a][b][1], c.y); }
          else { c.x = alpha * c.x + beta * acc[a][b][0]; c.y = alpha * c.y + beta * acc[a][b][1]; }
          *reinterpret_cast<double2*>(co) = c;
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (i + e < mrem) {
              double c = ci[e];
              c = (alpha == 1.0) ? fma(beta, acc[a][b][e], c) : alpha * c + beta * acc[a][b][e];
              co[e] = c;
            }
          }
        }
      }
    }
  }
#ifdef MLA_TILE_PROF
  if (tp) { long long e = clock64(); g_tprof[0] += 1; g_tprof[1] += e - tp0; g_tprof[2] += tpw; g_tprof[3] += e - tpe; }
#endif
  return (base + KT) % STAGES;
}

// NOTE: the update's tile engine (tile_run<GemmUpdateCfg>) must stay INLINE in its kernels: compiled as an
// out-of-line function, ptxas (12.9) allocates the bulk reduction's address operands in uniform registers
// >= UR32 and UBLKRED then comes out as ADD.U64 instead of ADD.F64.RN (integer adds into C: garbage).
// build.py scans the SASS of every build for exactly that.

// One stand-alone C tile (no cross-tile prefetch).  A: mrem x K (lda), B: K x nrem (ldb),
// Cin/Cout: mrem x nrem.  Collective over the CTA (256 threads); smem needs Cfg::SMEM_BYTES.
template <class Cfg, bool RED = true>
__device__ void gemm_tile(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                          int64_t ldb, int K, const double* Cin, int64_t ldcin, double* Cout,
                          int64_t ldcout, int mrem, int nrem, double alpha, double beta,
                          double* smem) {
  TileDesc d{A, lda, B, ldb, Cin, ldcin, Cout, ldcout, K, mrem, nrem, alpha, beta, true};
  TileDesc none{};
  none.valid = false;
  tile_prologue<Cfg>(d, 0, smem);
  tile_run<Cfg, RED>(d, none, 0, smem);
}

constexpr int kRowBlockTiles = 64;   // row tiles per L2 row block of the tile order

// A whole C := alpha*C + beta*A@B problem as a list of BM x BN tiles, column-strip major
// (consecutive tile ids walk down the rows of one BN-wide column strip, so the k x BN strip of B
// and the strip's prepare step are shared by neighbours in the queue).
struct GemmProblem {
  double* C; int64_t ldc;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  int m, n, k;
  double alpha, beta;
};

template <class Cfg>
__device__ __forceinline__ int gemm_num_tiles(const GemmProblem& p) {
  return ((p.m + Cfg::BM - 1) / Cfg::BM) * ((p.n + Cfg::BN - 1) / Cfg::BN);
}

template <class Cfg>
__device__ __forceinline__ TileDesc gemm_tile_desc(const GemmProblem& p, int t) {
  // Row-block-major order: the row tiles are cut into blocks of kRowBlockTiles; inside a block the
  // tiles go strip by strip.  The A rows of one block (kRowBlockTiles x BM x k doubles, 16 MiB at
  // k = 256) then stay in L2 while every column strip passes over them, instead of the whole m x k
  // operand being re-read from HBM for every strip.
  // Deep multiplies (k > 512: the catch-up updates of the phased host entry point) shrink the block so that
  // its A rows still fit L2: rbt * BM * k * 8 bytes <= 32 MiB, at least 4 row tiles.
  const int rbt = imax(4, imin(kRowBlockTiles, (kRowBlockTiles * 512) / imax(p.k, 1)));
  const int tm_count = (p.m + Cfg::BM - 1) / Cfg::BM;
  const int tn_count = (p.n + Cfg::BN - 1) / Cfg::BN;
  const int per_block = rbt * tn_count;
  const int rb = t / per_block;
  const int rows_here = imin(rbt, tm_count - rb * rbt);
  const int r = t - rb * per_block;
  const int tn = r / rows_here, tm = rb * rbt + (r - tn * rows_here);
  const int i0 = tm * Cfg::BM, j0 = tn * Cfg::BN;
  double* c = p.C + (int64_t)j0 * p.ldc + i0;
  return TileDesc{p.A + i0, p.lda, p.B + (int64_t)j0 * p.ldb, p.ldb, c, p.ldc, c, p.ldc,
                  p.k, p.m - i0, p.n - j0, p.alpha, p.beta, true};
}

}  // namespace mla
