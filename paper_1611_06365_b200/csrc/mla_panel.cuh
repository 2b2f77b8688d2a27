// Panel factorization: left-looking blocked LU with partial pivoting, collective over a Team of
// CTAs (reference lu.py:140-180 lu_blk_ll + lu.py:44-72 _unb_pivoted).
//
// Per inner block [j, j+wb) of the m x w panel (wb = b_inner):
//   1. U block:  P[0:j, j:j+wb] = trilu(P[0:j,0:j])^-1 P[0:j, j:j+wb]        (trsm_strip, rank 0)
//   2. rows [j, m) are dealt to the team in contiguous slabs (one per CTA, like the reference's
//      _share, kernels.py:28-32); each CTA updates its slab with one DMMA gemm
//         S = P[slab, j:j+wb] - P[slab, 0:j] @ U                               (lu.py:167-168)
//      writing the result straight into a shared-memory resident slab when it fits.
//   3. wb pivot steps on the slab (lu.py:48-71).  Each step costs ONE team-wide exchange through
//      global memory: every CTA publishes its local arg-max candidate (value, row -- lowest row
//      wins ties, lu.py:53 -- and that row's wb values), the CTA owning the diagonal row publishes
//      that row; after an acquire-poll of all slots every CTA knows the pivot row p, swaps its side
//      of (j+c <-> p), divides by the pivot (division, lu.py:65-67) and applies the rank-1 update
//      while already searching the next column's maximum.  An exactly-zero column records piv = j+c,
//      raises the singular flag and is skipped (lu.py:56-59).
//   4. the block's wb interchanges are applied to the other panel columns as one parallel
//      permutation plan (equivalent data movement to lu.py:165,173-174,178; applying them eagerly
//      to the right-hand columns as well means an ET cut needs no extra pass).
//   5. ET poll: once per completed block while columns remain (lu.py:177).
//
// Row indices / pivots are panel-local (lu.py:175).
#pragma once
#include "mla_common.cuh"
#include "mla_gemm.cuh"
#include "mla_laswp.cuh"
#include "mla_trsm.cuh"

namespace mla {

constexpr int kMaxInner = 128;   // widest block handled by the pivot-step kernel
constexpr int kMaxTeam = 160;    // >= SM count

struct XSlot {                   // one CTA's published candidate for one step parity
  double val;                    // |a| of the candidate, -1 when the CTA has no active row
  int row;                       // panel-local row of the candidate
  unsigned tag;                  // step sequence number, written last (release)
  double rowvals[kMaxInner];     // the candidate row's values in the block's columns
  double diag[kMaxInner];        // the diagonal row's values (only its owner writes them)
};

struct PanelWs {
  XSlot slots[2][kMaxTeam];
  unsigned seq;                  // last sequence number used (monotonic across panels)
  int decision;                  // ET decision broadcast by rank 0
  int pad[2];
};

struct PanelResult {
  int cols_factored;
  int singular;
};

struct PanelShared {
  double u[kMaxInner];           // pivot row (winner's values)
  double d[kMaxInner];           // old diagonal row
  double red_val[8];
  int red_row[8];
  int piv[kMaxInner];            // block pivots, panel-local rows
  int piv_rel[kMaxInner];        // same, relative to the block's first row (plan input)
  int plan_count;
  int plan_dst[2 * kMaxInner];
  int plan_src[2 * kMaxInner];
  int plan_top[kMaxInner], plan_lrow[kMaxInner], plan_lcur[kMaxInner];
  int win_rank, win_row;
  double win_val;
  int flag;
};

// (value desc, row asc) ordering of candidates
__device__ __forceinline__ bool cand_better(double v1, int r1, double v2, int r2) {
  return (v1 > v2) || (v1 == v2 && r1 < r2);
}

__device__ __forceinline__ void cand_warp_reduce(double& v, int& r) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, off);
    int orow = __shfl_xor_sync(0xffffffffu, r, off);
    if (cand_better(ov, orow, v, r)) { v = ov; r = orow; }
  }
}

// Collective over `team`; every thread of every member returns the same PanelResult.
// smem: dynamic shared memory of smem_doubles doubles (>= TRSM_SMEM_DOUBLES).
__device__ inline PanelResult panel_ll(Team& team, double* P, int m, int w, int64_t ld, int* ipiv_out,
                                       int b_inner, const unsigned* stop_flag, unsigned stop_eq,
                                       int stop_after_polls, PanelWs* ws, double* smem, int smem_doubles) {
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

  int j = 0;
  while (j < w) {
    // device block width: b_inner, clamped to what the step kernel holds (ET polls stay at
    // multiples of b_inner)
    int wb = imin(imin(b_inner, kMaxInner), w - j);
    {
      int to_poll = b_inner - (j % b_inner);  // never straddle a poll position
      wb = imin(wb, to_poll);
    }
    // ---- 1. U block -------------------------------------------------------------------------
    if (j > 0) {
      if (rank == 0) trsm_strip(P, j, ld, P + (int64_t)j * ld, wb, ld, smem);
      team.barrier();
    }
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
          for (int ct = 0; ct < wb; ct += GemmPanelCfg::BN)
            gemm_tile<GemmPanelCfg>(P + rt, ld, P + (int64_t)(j + ct) * ld, ld, j,
                                    P + (int64_t)(j + ct) * ld + rt, ld,
                                    Sb + (int64_t)ct * lds + (rt - r0), lds, r1 - rt, wb - ct, 1.0, -1.0,
                                    ring);
      } else if (resident) {
        for (int x = tid; x < nrows * wb; x += kThreads) {
          int c = x / nrows, i = x - c * nrows;
          Sb[(int64_t)c * lds + i] = P[(int64_t)(j + c) * ld + r0 + i];
        }
      }
    }
    __syncthreads();

    // ---- 3. pivot steps -------------------------------------------------------------------------
    // candidate for column 0 of the block
    double cv = -1.0;
    int cr = 0x7fffffff;
    for (int i = r0 + tid; i < r1; i += kThreads) {
      double v = fabs(Sb[i - r0]);
      if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
    }
    for (int c = 0; c < wb; ++c) {
      const int jc = j + c;            // diagonal row / global column of this step
      ++seq;
      XSlot* myslot = &ws->slots[seq & 1][rank];
      // A: CTA-level reduce of the candidate
      cand_warp_reduce(cv, cr);
      if (lane == 0) { sh.red_val[warp] = cv; sh.red_row[warp] = cr; }
      __syncthreads();
      double bv = sh.red_val[0];
      int br = sh.red_row[0];
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (cand_better(sh.red_val[k], sh.red_row[k], bv, br)) { bv = sh.red_val[k]; br = sh.red_row[k]; }
      // B: publish candidate row (+ diagonal row from its owner)
      const bool have = bv >= 0.0;
      if (tid < wb) {
        if (have) myslot->rowvals[tid] = Sb[(int64_t)tid * lds + (br - r0)];
        if (jc >= r0 && jc < r1) myslot->diag[tid] = Sb[(int64_t)tid * lds + (jc - r0)];
      }
      __syncthreads();
      if (tid == 0) {
        myslot->val = have ? bv : -1.0;
        myslot->row = have ? br : 0x7fffffff;
        __threadfence();
        st_release(&myslot->tag, seq);
      }
      // C: poll all slots, pick the winner
      double pv = -2.0;
      int prow = 0x7fffffff, prank = -1;
      if (tid < T) {
        XSlot* s = &ws->slots[seq & 1][tid];
        bool good = true;
        if (ld_acquire(&s->tag) != seq) {
          unsigned long long t0 = globaltimer_ns();
          unsigned it = 0;
          while (ld_acquire(&s->tag) != seq) {
            if ((++it & 63u) == 0u) {
              if (ld_relaxed(team.abort_word) != 0u) { good = false; break; }
              if (globaltimer_ns() - t0 > kSpinTimeoutNs) { atomicExch(team.abort_word, 0xDEAD2u); good = false; break; }
            }
          }
        }
        if (good) { pv = *((volatile double*)&s->val); prow = *((volatile int*)&s->row); prank = tid; }
      }
      {
        // reduce (pv, prow, prank) over the CTA
        double v = pv; int r = prow;
        cand_warp_reduce(v, r);
        if (lane == 0) { sh.red_val[warp] = v; sh.red_row[warp] = r; }
        __syncthreads();
        if (tid == 0) {
          double wv = sh.red_val[0]; int wr = sh.red_row[0];
          for (int k = 1; k < 8; ++k)
            if (cand_better(sh.red_val[k], sh.red_row[k], wv, wr)) { wv = sh.red_val[k]; wr = sh.red_row[k]; }
          sh.win_val = wv; sh.win_row = wr;
          sh.flag = (ld_relaxed(team.abort_word) != 0u) ? 1 : 0;
        }
        __syncthreads();
        if (tid < T && pv == sh.win_val && prow == sh.win_row) sh.win_rank = prank;  // unique: rows are distinct
        __syncthreads();
      }
      if (sh.flag) { team.ok = false; res.cols_factored = j; return res; }
      const double wval = sh.win_val;
      const int p = (wval > 0.0) ? sh.win_row : jc;
      if (tid == 0) sh.piv[c] = p;
      if (!(wval > 0.0)) {
        // zero pivot column: record, flag, skip (lu.py:56-59); candidate of the next column fresh
        res.singular = 1;
        cv = -1.0; cr = 0x7fffffff;
        if (c + 1 < wb)
          for (int i = imax(r0, jc + 1) + tid; i < r1; i += kThreads) {
            double v = fabs(Sb[(int64_t)(c + 1) * lds + (i - r0)]);
            if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
          }
        __syncthreads();
        continue;
      }
      // D: fetch the pivot row and the old diagonal row
      const int drank = (jc - j) / rpc;
      if (tid < wb) {
        sh.u[tid] = *((volatile double*)&ws->slots[seq & 1][sh.win_rank].rowvals[tid]);
        sh.d[tid] = *((volatile double*)&ws->slots[seq & 1][drank].diag[tid]);
      }
      __syncthreads();
      // E: interchange rows jc <-> p inside the block (lu.py:60-64)
      if (p != jc && tid < wb) {
        if (jc >= r0 && jc < r1) Sb[(int64_t)tid * lds + (jc - r0)] = sh.u[tid];
        if (p >= r0 && p < r1) Sb[(int64_t)tid * lds + (p - r0)] = sh.d[tid];
      }
      __syncthreads();
      // F: scale + rank-1 update of rows below the diagonal, search next column's maximum
      const double pivot = sh.u[c];
      cv = -1.0; cr = 0x7fffffff;
      for (int i = imax(r0, jc + 1) + tid; i < r1; i += kThreads) {
        double* row = Sb + (i - r0);
        double l = row[(int64_t)c * lds] / pivot;
        row[(int64_t)c * lds] = l;
        if (c + 1 < wb) {
          double x = row[(int64_t)(c + 1) * lds] - l * sh.u[c + 1];
          row[(int64_t)(c + 1) * lds] = x;
          double v = fabs(x);
          if (cand_better(v, i, cv, cr)) { cv = v; cr = i; }
          for (int cc = c + 2; cc < wb; ++cc) row[(int64_t)cc * lds] -= l * sh.u[cc];
        }
      }
      __syncthreads();
    }
    // ---- write the slab back, record pivots ------------------------------------------------------
    if (resident) {
      for (int x = tid; x < nrows * wb; x += kThreads) {
        int c = x / nrows, i = x - c * nrows;
        P[(int64_t)(j + c) * ld + r0 + i] = Sb[(int64_t)c * lds + i];
      }
    }
    if (tid < wb) {
      sh.piv_rel[tid] = sh.piv[tid] - j;
      if (rank == 0) ipiv_out[j + tid] = sh.piv[tid];
    }
    __syncthreads();
    // ---- 4. the block's interchanges reach the other panel columns ------------------------------
    if (w - wb > 0) {
      if (warp == 0) {
        PlanRef pr{&sh.plan_count, sh.plan_dst, sh.plan_src};
        build_pivot_plan(sh.piv_rel, wb, (int64_t)(m - j), false, pr, sh.plan_top, sh.plan_lrow, sh.plan_lcur);
      }
      __syncthreads();
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
    j += wb;
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
