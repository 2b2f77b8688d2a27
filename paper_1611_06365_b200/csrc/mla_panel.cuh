// Panel factorization: left-looking blocked LU with partial pivoting, collective over a Team of
// CTAs (reference lu.py:140-180 lu_blk_ll + lu.py:44-72 _unb_pivoted).
//
// Per device block [j, j+wb) of the m x w panel (wb = b_inner, halved down to 8 until a CTA's share of
// the block fits its shared-memory slab; ET polls stay at multiples of b_inner):
//   1. U block:  P[0:j, j:j+wb] = trilu(P[0:j,0:j])^-1 P[0:j, j:j+wb]  (lu.py:166) -- in the reference's
//      left-looking order this is a trsm per block (stand-alone lu_blk_ll: columns dealt to the first
//      CTAs); inside the persistent kernel (eager_u) it is already there, see 4b.
//   2. rows [j, m) are dealt to the team in contiguous slabs (one per CTA, like the reference's
//      _share, kernels.py:28-32); each CTA updates its slab with one DMMA gemm
//         S = P[slab, j:j+wb] - P[slab, 0:j] @ U                               (lu.py:167-168)
//      writing the result straight into a shared-memory resident slab when it fits.
//   3. wb pivot steps on the slab (lu.py:48-71).  Each step costs ONE team-wide exchange through
//      global memory: every CTA publishes its local arg-max candidate (value, row -- lowest row
//      wins ties, lu.py:53 -- and that row's wb values), the CTA owning the diagonal row publishes
//      that row (16-byte self-validating words, no fences); after polling all slots every CTA knows
//      the pivot row p, swaps its side of (j+c <-> p), forms the multipliers (lu.py:65-67) and applies
//      the rank-1 update while already searching the next column's maximum.  With the slab in shared
//      memory the update is split: column c+1 at once (it yields the next candidates), the remaining
//      columns on warps 1-7 WHILE warp 0 already runs the next step's exchange.  An exactly-zero column records piv = j+c,
//      raises the singular flag and is skipped (lu.py:56-59).
//   4. the block's wb interchanges are applied to the other panel columns as one parallel
//      permutation plan (equivalent data movement to lu.py:165,173-174,178; applying them eagerly
//      to the right-hand columns as well means an ET cut needs no extra pass).
//   4b. eager_u (Crout order): the rows of U this block determines are computed for ALL later panel
//      columns (one DMMA row-block step per 32 rows), which removes the per-block trsm chain and lets
//      an ET cut hand over leftover columns that already hold their A12 rows.
//   5. ET poll: once per completed block while columns remain (lu.py:177).
//
// Row indices / pivots are panel-local (lu.py:175).
#pragma once
#include "mla_common.cuh"
#include "mla_gemm.cuh"
#include "mla_laswp.cuh"
#include "mla_trsm.cuh"

namespace mla {

constexpr int kMinInner = 8;     // narrowest block the slab-fitting rule goes down to
constexpr int kMaxInner = 128;   // widest block handled by the pivot-step kernel
constexpr int kMaxTeam = 160;    // >= SM count

// Exchange words are 16 bytes {payload, tag} written and read with single 128-bit STRONG.GPU
// transactions (st/ld.relaxed.gpu.b128), so each word validates itself through its tag and the
// per-step exchange needs no memory fence at all.
struct alignas(16) XUnit { unsigned long long lo, hi; };

struct XSlot {                   // one CTA's published candidate for one step parity
  XUnit head;                    // lo = |a| of the candidate (-1: no active row); hi = row<<32 | seq
  XUnit rv[kMaxInner];           // the candidate row's values in the block's columns; hi = seq
  XUnit dg[kMaxInner];           // the diagonal row's values (only its owner writes them); hi = seq
};

__device__ __forceinline__ void st_b128(void* p, unsigned long long lo, unsigned long long hi) {
  asm volatile("{\n .reg .b128 t;\n mov.b128 t, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], t;\n}"
               ::"l"(p), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void ld_b128(const void* p, unsigned long long& lo, unsigned long long& hi) {
  asm volatile("{\n .reg .b128 t;\n ld.relaxed.gpu.global.b128 t, [%2];\n mov.b128 {%0, %1}, t;\n}"
               : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}
// Spin until the word's tag (low 32 bits of hi) equals seq.  Returns false on abort/timeout.
__device__ __forceinline__ bool poll_unit(const XUnit* u, unsigned seq, unsigned* abort_word,
                                          unsigned long long& lo, unsigned long long& hi) {
  ld_b128(u, lo, hi);
  if ((unsigned)hi == seq) return true;
  unsigned long long t0 = globaltimer_ns();
  unsigned it = 0;
  while (true) {
    ld_b128(u, lo, hi);
    if ((unsigned)hi == seq) return true;
    if ((++it & 255u) == 0u) {
      if (ld_relaxed(abort_word) != 0u) return false;
      if (globaltimer_ns() - t0 > kSpinTimeoutNs) { atomicExch(abort_word, 0xDEAD2u); return false; }
    }
  }
}

struct PanelWs {
  XSlot slots[2][kMaxTeam];
  unsigned seq;                  // last sequence number used (monotonic across panels)
  int decision;                  // ET decision broadcast by rank 0
  int pad[2];
  unsigned long long prof[16];   // rank 0's phase times in ns: 0 trsm, 1 gemm/load, 2 pivot steps,
                                 // 3 write-back+plan+swaps, 4 block barrier, 5 exchange part of 2
};

#define MLA_PROF(idx)                                                   \
  do {                                                                  \
    if (rank == 0 && tid == 0) {                                        \
      unsigned long long now_ = globaltimer_ns();                       \
      ws->prof[idx] += now_ - prof_t;                                   \
      prof_t = now_;                                                    \
    }                                                                   \
  } while (0)

struct PanelResult {
  int cols_factored;
  int singular;
};

struct PanelShared {
  double u2[2][kMaxInner];       // pivot row (winner's values) of the current / the previous step
  double red_val[8];
  int red_row[8];
  int piv[kMaxInner];            // block pivots, panel-local rows
  int piv_rel[kMaxInner];        // same, relative to the block's first row (plan input)
  int plan_count;
  int plan_dst[2 * kMaxInner];
  int plan_src[2 * kMaxInner];
  int plan_top[kMaxInner], plan_pv[kMaxInner], plan_keys[2 * kMaxInner], plan_vals[2 * kMaxInner];
  int win_rank, win_row;
  double win_val;
  int flag;
};

// (value desc, row asc) ordering of candidates
__device__ __forceinline__ bool cand_better(double v1, int r1, double v2, int r2) {
  return (v1 > v2) || (v1 == v2 && r1 < r2);
}

// Warp-wide best candidate in every lane: three REDUX (max of the high word, max of the low word
// among the leaders, min row among the ties) instead of a 5-round shuffle butterfly.  |v| >= 0 maps
// order-preservingly onto an unsigned 64-bit key (+1 so that 0.0 beats the "no candidate"
// sentinels, which map to 0).
__device__ __forceinline__ void cand_warp_reduce(double& v, int& r) {
  const unsigned long long k = (v >= 0.0) ? ((unsigned long long)__double_as_longlong(v) + 1ull) : 0ull;
  const unsigned hi = (unsigned)(k >> 32), lo = (unsigned)k;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, (hi == mh) ? lo : 0u);
  const bool lead = (hi == mh) && (lo == ml);
  const unsigned mr = __reduce_min_sync(0xffffffffu, lead ? (unsigned)r : 0xffffffffu);
  const unsigned long long kk = ((unsigned long long)mh << 32) | ml;
  v = kk ? __longlong_as_double((long long)(kk - 1ull)) : -1.0;
  r = (int)mr;
}

// a / pivot for the multipliers (lu.py:65-67 divides; it does not multiply by a reciprocal).  A full
// IEEE division is a ~40-instruction dependent chain per row and step; here the quotient comes from
// the shared reciprocal plus one residual correction, which is the correctly rounded quotient except
// in rare double-rounding cases (<= 1 ulp), far inside the 1e-10 parity bound.
__device__ __forceinline__ double div_by_pivot(double a, double pivot, double rinv) {
  double q = a * rinv;
  double r = fma(-q, pivot, a);
  return fma(r, rinv, q);
}

// Collective over `team`; every thread of every member returns the same PanelResult.
// smem: dynamic shared memory of smem_doubles doubles (>= TRSM_SMEM_DOUBLES).
__device__ inline PanelResult panel_ll(Team& team, double* P, int m, int w, int64_t ld, int* ipiv_out,
                                       int b_inner, const unsigned* stop_flag, unsigned stop_eq,
                                       int stop_after_polls, PanelWs* ws, double* smem, int smem_doubles,
                                       bool eager_u = false) {
  __shared__ PanelShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = team.size, rank = team.rank;
  PanelResult res{0, 0};
  constexpr int RING = GemmPanelCfg::SMEM_BYTES / 8;
  double* ring = smem;
  double* slab_mem = smem + RING;
  const int slab_cap = smem_doubles - RING;

  unsigned seq = *((volatile unsigned*)&ws->seq);
  team.barrier();  // everybody has read seq before anybody can publish / update it
  int polls = 0;
  unsigned long long prof_t = globaltimer_ns();

  int j = 0;
  while (j < w) {
    // device block width: b_inner, clamped to what the step kernel holds (ET polls stay at
    // multiples of b_inner)
    int wb = imin(imin(b_inner, kMaxInner), w - j);
    {
      int to_poll = b_inner - (j % b_inner);  // never straddle a poll position
      wb = imin(wb, to_poll);
    }
    // ... and halved until every CTA's share of the block (rows x wb) fits its shared-memory slab:
    // pivot steps on a resident slab cost a third of steps that stream the block through L2.
    {
      int rpc_max = (((m - j) + T - 1) / T + 31) & ~31;
      int lds_max = ((rpc_max + 1) & ~1) + 2;
      while (wb > kMinInner && lds_max * wb > slab_cap) wb = imax(kMinInner, ((wb >> 1) + 7) & ~7);
    }
    // ---- 1. U block -------------------------------------------------------------------------
    if (j > 0 && !eager_u) {
      {
        // columns of the U block are dealt in shares of >= 8 (one DMMA tile) to the first CTAs
        int nsh = imin(T, (wb + 7) / 8);
        int per = (((wb + nsh - 1) / nsh) + 7) & ~7;
        int c_lo = rank * per, c_hi = imin(wb, c_lo + per);
        if (rank < nsh && c_lo < c_hi)
          trsm_strip(P, j, ld, P + (int64_t)(j + c_lo) * ld, c_hi - c_lo, ld, smem);
      }
      team.barrier();
    }
    MLA_PROF(0);
    // ---- 2. slab + gemm -----------------------------------------------------------------------
    const int R = m - j;
    int rpc = (R + T - 1) / T;
    rpc = (rpc + 31) & ~31;
    const int r0 = j + rank * rpc;
    const int r1 = imin(m, r0 + rpc);
    const int nrows = imax(0, r1 - r0);
    const int lds_res = ((nrows + 1) & ~1) + 2;
    const bool resident = nrows > 0 && lds_res * wb <= slab_cap;
    double* Sb;          // Sb[c*lds + (i - r0)] is entry (i, j+c)
    int64_t lds;
    if (resident) { Sb = slab_mem; lds = lds_res; }
    else { Sb = P + (int64_t)j * ld + r0; lds = ld; }
    if (nrows > 0) {
      if (j > 0) {
        for (int rt = r0; rt < r1; rt += GemmPanelCfg::BM)
          for (int ct = 0; ct < wb; ct += GemmPanelCfg::BN) {
            if (wb - ct <= GemmPanel8Cfg::BN)
              gemm_tile<GemmPanel8Cfg>(P + rt, ld, P + (int64_t)(j + ct) * ld, ld, j,
                                       P + (int64_t)(j + ct) * ld + rt, ld,
                                       Sb + (int64_t)ct * lds + (rt - r0), lds, r1 - rt, wb - ct, 1.0, -1.0,
                                       ring);
            else if (wb - ct <= GemmPanel16Cfg::BN)
              gemm_tile<GemmPanel16Cfg>(P + rt, ld, P + (int64_t)(j + ct) * ld, ld, j,
                                        P + (int64_t)(j + ct) * ld + rt, ld,
                                        Sb + (int64_t)ct * lds + (rt - r0), lds, r1 - rt, wb - ct, 1.0, -1.0,
                                        ring);
            else
              gemm_tile<GemmPanelCfg>(P + rt, ld, P + (int64_t)(j + ct) * ld, ld, j,
                                      P + (int64_t)(j + ct) * ld + rt, ld,
                                      Sb + (int64_t)ct * lds + (rt - r0), lds, r1 - rt, wb - ct, 1.0, -1.0,
                                      ring);
          }
      } else if (resident) {
        for (int x = tid; x < nrows * wb; x += kThreads) {
          int c = x / nrows, i = x - c * nrows;
          Sb[(int64_t)c * lds + i] = P[(int64_t)(j + c) * ld + r0 + i];
        }
      }
    }
    __syncthreads();
    MLA_PROF(1);

    // ---- 3. pivot steps -------------------------------------------------------------------------
    unsigned long long xchg_acc = 0ull;
    // candidate for column 0 of the block
    double cv = -1.0;
    int cr = 0x7fffffff;
    for (int i = r0 + tid; i < r1; i += kThreads) {
      double v = fabs(Sb[i - r0]);
      if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
    }
    // Look-ahead of the exchange over the update (slab in shared memory): a step's rank-1 update is
    // split into F1 = scale + column c+1 (which yields the next candidates) and F2 = columns c+2.. ;
    // F2 of step c-1 runs on warps 1-7 WHILE warp 0 runs the exchange of step c.  The two rows that
    // exchange publishes / interchanges (the local candidate row and the diagonal row) are brought up
    // to date by warp 0 itself and skipped by F2, so the two never touch the same entries.
    const bool la_steps = resident;
    int f2_c = -1;                     // step whose columns f2_c+2.. still await their update
    for (int c = 0; c < wb; ++c) {
      const int jc = j + c;            // diagonal row / global column of this step
      ++seq;
      double* const ucur = sh.u2[c & 1];
      const double* const uprev = sh.u2[(c & 1) ^ 1];
      // A: per-warp candidates -> shared memory; every warp then knows the CTA's candidate row
      cand_warp_reduce(cv, cr);
      if (lane == 0) { sh.red_val[warp] = cv; sh.red_row[warp] = cr; }
      __syncthreads();
      double bv = (lane < 8) ? sh.red_val[lane] : -2.0;
      int br = (lane < 8) ? sh.red_row[lane] : 0x7fffffff;
      cand_warp_reduce(bv, br);
      const bool have = bv >= 0.0;
      const bool own_diag = (jc >= r0 && jc < r1);
      MLA_STRESS((warp & 3) == (c & 3));            // skew the warps between the exchange and the deferred update
      if (warp != 0 && f2_c >= 0) {
        // F2 of the previous step on every row except warp 0's two
        const int64_t lcol = (int64_t)f2_c * lds;
        for (int i = imax(r0, jc) + (tid - 32); i < r1; i += kThreads - 32) {
          if (i == jc || (have && i == br)) continue;
          double* __restrict__ row = Sb + (i - r0);
          const double l = row[lcol];
          for (int cb = f2_c + 2; cb < wb; cb += 8) {
            double x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (cb + e < wb) ? row[(int64_t)(cb + e) * lds] : 0.0;
#pragma unroll
            for (int e = 0; e < 8; ++e) if (cb + e < wb) x[e] = fma(-l, uprev[cb + e], x[e]);
#pragma unroll
            for (int e = 0; e < 8; ++e) if (cb + e < wb) row[(int64_t)(cb + e) * lds] = x[e];
          }
        }
      }
      // B-E: warp 0 runs the whole exchange
      if (warp == 0) {
        unsigned long long xt0 = (rank == 0 && lane == 0) ? globaltimer_ns() : 0ull;
        if (f2_c >= 0) {
          const int64_t lcol = (int64_t)f2_c * lds;
          const bool two = own_diag && !(have && br == jc);
          for (int cc = f2_c + 2 + lane; cc < wb; cc += 32) {
            const double uc = uprev[cc];
            if (have) {
              double* e = Sb + (int64_t)cc * lds + (br - r0);
              *e = fma(-Sb[lcol + (br - r0)], uc, *e);
            }
            if (two) {
              double* e = Sb + (int64_t)cc * lds + (jc - r0);
              *e = fma(-Sb[lcol + (jc - r0)], uc, *e);
            }
          }
          __syncwarp();
        }
        bool good = true;
        double wv;
        int p;
        if (T == 1) {
          // single-CTA team: everything is local, no trip through L2
          wv = bv;
          p = (wv > 0.0) ? br : jc;
          if (wv > 0.0) {
            for (int cc = lane; cc < wb; cc += 32) {
              double uu = Sb[(int64_t)cc * lds + (p - r0)];
              ucur[cc] = uu;
              if (p != jc) {
                double dd = Sb[(int64_t)cc * lds + (jc - r0)];
                Sb[(int64_t)cc * lds + (jc - r0)] = uu;
                Sb[(int64_t)cc * lds + (p - r0)] = dd;
              }
            }
          }
        } else {
          XSlot* slots = ws->slots[seq & 1];
          XSlot* myslot = &slots[rank];
          const int drank = (jc - j) / rpc;
          for (int cc = lane; cc < wb; cc += 32) {
            if (have) st_b128(&myslot->rv[cc], (unsigned long long)__double_as_longlong(Sb[(int64_t)cc * lds + (br - r0)]), seq);
            if (own_diag) st_b128(&myslot->dg[cc], (unsigned long long)__double_as_longlong(Sb[(int64_t)cc * lds + (jc - r0)]), seq);
          }
          if (lane == 0)
            st_b128(&myslot->head, (unsigned long long)__double_as_longlong(have ? bv : -1.0),
                    ((unsigned long long)(unsigned)(have ? br : 0x7fffffff) << 32) | (unsigned long long)seq);
          // ONE hop for small teams: together with the headers, the diagonal row (its owner is known
          // a priori) and every member's candidate row are requested speculatively; the tags say
          // afterwards what was already valid.
          constexpr int SPEC_T = 8;
          const bool spec = (T <= SPEC_T) && (wb <= 32);
          unsigned long long slo[SPEC_T], shi[SPEC_T], dlo = 0, dhi = 0;
#pragma unroll
          for (int t = 0; t < SPEC_T; ++t) { slo[t] = 0; shi[t] = 0; }
          if (lane < wb) {
            ld_b128(&slots[drank].dg[lane], dlo, dhi);
            if (spec) {
#pragma unroll
              for (int t = 0; t < SPEC_T; ++t)
                if (t < T) ld_b128(&slots[t].rv[lane], slo[t], shi[t]);
            }
          }
          // poll every member's header
          double pv = -2.0;
          int prow = 0x7fffffff, prank = -1;
          for (int t = lane; t < T; t += 32) {
            unsigned long long lo, hi;
            if (!poll_unit(&slots[t].head, seq, team.abort_word, lo, hi)) { good = false; break; }
            double v = __longlong_as_double((long long)lo);
            int r = (int)(hi >> 32);
            if (cand_better(v, r, pv, prow)) { pv = v; prow = r; prank = t; }
          }
          wv = pv;
          int wr = prow;
          cand_warp_reduce(wv, wr);
          unsigned who = __ballot_sync(0xffffffffu, pv == wv && prow == wr && prank >= 0);
          int wrank = __shfl_sync(0xffffffffu, prank, who ? (__ffs(who) - 1) : 0);
          good = __all_sync(0xffffffffu, good);
          p = (wv > 0.0) ? wr : jc;
          if (good && wv > 0.0) {
            for (int cc = lane; cc < wb; cc += 32) {
              unsigned long long lo = 0, hi = 0;
              if (spec) {
#pragma unroll
                for (int t = 0; t < SPEC_T; ++t)
                  if (t == wrank) { lo = slo[t]; hi = shi[t]; }
              } else {
                ld_b128(&slots[wrank].rv[cc], lo, hi);
              }
              // the diagonal row was requested before the headers were polled and may have come back stale: ask
              // again NOW, next to the winner's row, so that the two answers travel together instead of one
              // round trip after the other
              // (only the CTA that holds the pivot row needs the diagonal row's values at all)
              const bool need_dg = (p != jc) && (p >= r0 && p < r1);
              unsigned long long lo2 = dlo, hi2 = dhi;
              if (need_dg && (cc >= 32 || (unsigned)hi2 != seq)) ld_b128(&slots[drank].dg[cc], lo2, hi2);
              if ((unsigned)hi != seq && !poll_unit(&slots[wrank].rv[cc], seq, team.abort_word, lo, hi)) { good = false; break; }
              double uu = __longlong_as_double((long long)lo);
              ucur[cc] = uu;
              if (p != jc) {
                // interchange rows jc <-> p inside the block (lu.py:60-64)
                if (own_diag) Sb[(int64_t)cc * lds + (jc - r0)] = uu;
                if (need_dg) {
                  if ((unsigned)hi2 != seq && !poll_unit(&slots[drank].dg[cc], seq, team.abort_word, lo2, hi2)) { good = false; break; }
                  Sb[(int64_t)cc * lds + (p - r0)] = __longlong_as_double((long long)lo2);
                }
              }
            }
            good = __all_sync(0xffffffffu, good);
          }
        }
        if (lane == 0) {
          sh.piv[c] = p;
          sh.win_val = wv;
          sh.flag = good ? 0 : 1;
          if (rank == 0) xchg_acc += globaltimer_ns() - xt0;
        }
      }
      __syncthreads();
      if (sh.flag) { team.ok = false; res.cols_factored = j; return res; }
      f2_c = -1;
      const double wval = sh.win_val;
      if (!(wval > 0.0)) {
        // zero pivot column: record, flag, skip (lu.py:56-59); candidate of the next column fresh
        res.singular = 1;
        cv = -1.0; cr = 0x7fffffff;
        if (c + 1 < wb)
          for (int i = imax(r0, jc + 1) + tid; i < r1; i += kThreads) {
            double v = fabs(Sb[(int64_t)(c + 1) * lds + (i - r0)]);
            if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
          }
        continue;
      }
      // F: scale + rank-1 update of rows below the diagonal, search next column's maximum.
      // Columns are processed in register chunks of 8 so the shared-memory loads of a row are in
      // flight together instead of forming a load->fma->store chain per column.
      const double pivot = ucur[c];
      const double rinv = 1.0 / pivot;
      cv = -1.0; cr = 0x7fffffff;
      if (la_steps) {
        // F1 only; the other columns follow during the next exchange (F2 above)
        const double un = (c + 1 < wb) ? ucur[c + 1] : 0.0;
        for (int i = imax(r0, jc + 1) + tid; i < r1; i += kThreads) {
          double* __restrict__ row = Sb + (i - r0);
          const double l = div_by_pivot(row[(int64_t)c * lds], pivot, rinv);
          row[(int64_t)c * lds] = l;
          if (c + 1 < wb) {
            const double x = fma(-l, un, row[(int64_t)(c + 1) * lds]);
            row[(int64_t)(c + 1) * lds] = x;
            const double v = fabs(x);
            if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
          }
        }
        if (c + 2 < wb) f2_c = c;
      } else if (resident) {
        for (int i = imax(r0, jc + 1) + tid; i < r1; i += kThreads) {
          double* __restrict__ row = Sb + (i - r0);
          const double l = div_by_pivot(row[(int64_t)c * lds], pivot, rinv);
          row[(int64_t)c * lds] = l;
          for (int cb = c + 1; cb < wb; cb += 8) {
            double x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (cb + e < wb) ? row[(int64_t)(cb + e) * lds] : 0.0;
#pragma unroll
            for (int e = 0; e < 8; ++e) if (cb + e < wb) x[e] = fma(-l, ucur[cb + e], x[e]);
#pragma unroll
            for (int e = 0; e < 8; ++e) if (cb + e < wb) row[(int64_t)(cb + e) * lds] = x[e];
            if (cb == c + 1) {
              double v = fabs(x[0]);
              if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
            }
          }
        }
      } else {
        // slab in global memory (too tall for shared memory): the pass is a stream through L2, so
        // four rows per thread are kept in flight (32 independent 8-byte loads) to cover its latency
        constexpr int RU = 4;
        for (int ib = imax(r0, jc + 1) + tid; ib < r1; ib += kThreads * RU) {
          double l[RU];
          double* row[RU];
#pragma unroll
          for (int r = 0; r < RU; ++r) {
            const int i = ib + r * kThreads;
            row[r] = Sb + (imin(i, r1 - 1) - r0);
            l[r] = row[r][(int64_t)c * lds];
          }
#pragma unroll
          for (int r = 0; r < RU; ++r) {
            l[r] = div_by_pivot(l[r], pivot, rinv);
            if (ib + r * kThreads < r1) row[r][(int64_t)c * lds] = l[r];
          }
          for (int cb = c + 1; cb < wb; cb += 8) {
            double x[RU][8];
#pragma unroll
            for (int r = 0; r < RU; ++r)
#pragma unroll
              for (int e = 0; e < 8; ++e) x[r][e] = (cb + e < wb) ? row[r][(int64_t)(cb + e) * lds] : 0.0;
#pragma unroll
            for (int r = 0; r < RU; ++r) {
              const int i = ib + r * kThreads;
              if (i < r1) {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (cb + e < wb) row[r][(int64_t)(cb + e) * lds] = fma(-l[r], ucur[cb + e], x[r][e]);
                if (cb == c + 1) {
                  double v = fabs(fma(-l[r], ucur[cb], x[r][0]));
                  if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
                }
              }
            }
          }
        }
      }
    }
    __syncthreads();
    MLA_PROF(2);
    if (rank == 0 && tid == 0) ws->prof[5] += xchg_acc;
    // ---- write the slab back, record pivots ------------------------------------------------------
    if (tid < wb) {
      sh.piv_rel[tid] = sh.piv[tid] - j;
      if (rank == 0) ipiv_out[j + tid] = sh.piv[tid];
    }
    __syncthreads();
    // warp 0 resolves the block's interchanges into a plan (a serial chain over the wb pivots) WHILE warps 1-7
    // write the slab back; both are needed before step 4
    const bool want_plan = (w - wb > 0);
    if (warp == 0 && want_plan) {
      PlanRef pr{&sh.plan_count, sh.plan_dst, sh.plan_src};
      build_pivot_plan(sh.piv_rel, wb, (int64_t)(m - j), false, pr, sh.plan_top, sh.plan_keys, sh.plan_vals,
                       2 * kMaxInner, sh.plan_pv);
    } else if (resident) {
      const int t0 = want_plan ? tid - 32 : tid, nt = want_plan ? kThreads - 32 : kThreads;
      for (int x = t0; x < nrows * wb; x += nt) {
        int c = x / nrows, i = x - c * nrows;
        P[(int64_t)(j + c) * ld + r0 + i] = Sb[(int64_t)c * lds + i];
      }
    }
    __syncthreads();
    // ---- 4. the block's interchanges reach the other panel columns ------------------------------
    if (w - wb > 0) {
      PlanRef pr{&sh.plan_count, sh.plan_dst, sh.plan_src};
      const int oc = w - wb;  // other columns: [0,j) then [j+wb, w)
      int share = (oc + T - 1) / T;
      int lo = imin(oc, rank * share), hi = imin(oc, lo + share);
      // map [lo,hi) of the concatenated index space onto the two column ranges
      int l0 = imin(lo, j), h0 = imin(hi, j);
      if (h0 > l0) laswp_apply_cols(P + (int64_t)l0 * ld + j, ld, h0 - l0, pr, ring, RING);
      int l1 = imax(lo, j) - j, h1 = imax(hi, j) - j;
      if (h1 > l1) laswp_apply_cols(P + (int64_t)(j + wb + l1) * ld + j, ld, h1 - l1, pr, ring, RING);
    }
    // ---- 4b. Crout order (eager_u): the rows of U this block determines, for all later columns ---
    // U[j:j+wb, j+wb:w] = trilu(L_jj)^-1 (A[j:j+wb, j+wb:w] - L[j:j+wb, 0:j] U[0:j, j+wb:w]).
    // Done here, the next block's update finds its U block complete (no trsm chain per block) and,
    // after an ET cut, the leftover columns already hold their A12 rows (the next iteration's PREP
    // skips them, see mla_getrf.cuh).  Needs this block's interchanges on those columns: barrier.
    if (eager_u && j + wb < w) {
      team.barrier();
      const int nc = w - j - wb;
      int nsh = imin(T, (nc + 7) / 8);
      int per = (((nc + nsh - 1) / nsh) + 7) & ~7;
      if (per > TRSM_CW) { per = TRSM_CW; nsh = (nc + per - 1) / per; }
      for (int sh_i = rank; sh_i < nsh; sh_i += T) {
        int c_lo = sh_i * per, c_hi = imin(nc, c_lo + per);
        for (int rr = 0; rr < wb; rr += TRSM_RB)
          trsm_rowblock(P, j + rr, imin(TRSM_RB, wb - rr), ld, P + (int64_t)(j + wb + c_lo) * ld, c_hi - c_lo, ld, smem);
      }
    }
    j += wb;
    MLA_PROF(3);
    // ---- 5. ET poll (rank 0 decides, everybody follows) ----------------------------------------
    bool poll_here = (j < w) && (j % b_inner == 0) && (stop_flag != nullptr || stop_after_polls > 0);
    if (poll_here && rank == 0 && tid == 0) {
      int dec = 0;
      if (stop_after_polls > 0) dec = (polls + 1 >= stop_after_polls);
      if (stop_flag != nullptr) {
        unsigned f = ld_acquire(stop_flag);   // stop_eq == 0: "set" means non-zero; else == stop_eq
        if (stop_eq ? (f == stop_eq) : (f != 0u)) dec = 1;
      }
      *((volatile int*)&ws->decision) = dec;
    }
    if (poll_here) ++polls;
    team.barrier();
    MLA_PROF(4);
    if (!team.ok) { res.cols_factored = j; return res; }
    if (poll_here) {
      int dec = *((volatile int*)&ws->decision);
      if (dec) break;
    }
  }
  res.cols_factored = j;
  // hand the sequence number on to the next panel
  team.barrier();
  if (rank == 0 && tid == 0) *((volatile unsigned*)&ws->seq) = seq;
  return res;
}

}  // namespace mla
