// lu_la on the GPU: ONE persistent cooperative kernel for the whole factorization
// (reference lu.py:197-334).  The reference's two thread teams become an SM partition:
//
//   CTAs [0, sm_pf)   = team PF: after the next panel's columns are updated they factor panel k+1
//                       (panel_ll, collective over the team),
//   CTAs [sm_pf, G)   = team RU: pull work items of the trailing update from atomic queues.
//
// Per outer iteration the work is cut into items (PREP of a 128-column strip = row interchanges of
// the previous panel + trsm with A11, lu.py:251-253,280,289; GEMM = one 128x128 tile of A22 -= A21@A12,
// lu.py:281,306-308; LEFT = interchanges of 256 columns of the L part, lu.py:252) in two atomic queues:
//   PQ: [PREP of the next panel's strips][PREP of the first ~G remainder strips -- fillers that keep
//        every CTA busy while the panel PREP runs][GEMM tiles of the next panel's columns];
//   RQ: first row block (64 row tiles): per remainder strip s a group [PREP of strip s+lookahead]
//        [LEFT strip s][the strip's GEMM tiles of that row block]; then the later row blocks as pure
//        GEMM groups (row-block-major order keeps a block's A21 rows in L2 across all strips); then
//        leftover LEFT strips.  The HBM-bound interchanges thus run between tensor-bound tiles.
// Every CTA first helps to drain PQ (it is the critical path to the next panel); PF CTAs then wait
// for PQ to complete and run the panel while RU CTAs drain RQ.  Pops run one item ahead (two on long
// queues, with an atomic whose round trip overlaps the running tile) so that consecutive GEMM tiles
// chain through the tile engine; completion is counted once per CTA.
//
//   WS  (lu_mb / lu_et, pool.py:377-414): a PF CTA that returns from the panel -- i.e. after the
//        panel team's final barrier, so the donor team has fully quiesced -- simply starts pulling
//        RQ items; the queue's item boundary is the entry point.  Teams only grow, and the split is
//        restored at the next iteration.  lu_ws_static joins only at a q-chunk boundary of the
//        GEMM item range (lu.py:290-304).
//   ET  (lu_et, lu.py:177-179,309-310): the CTA that completes the last RQ item publishes
//        ru_done = iteration; the panel polls it once per finished inner block and cuts there; the
//        leftover columns are folded into the next iteration through `pend` (lu.py:318-326).
//
// A GEMM tile depends only on the PREP of its own column strip (per-strip release/acquire flag), so
// no barrier separates the row interchanges, the triangular solve and the update.  Results do not
// depend on which CTA ran an item: one owner per C tile, fixed k order (kernels.py:3-9).
#pragma once
#include "../../include/mla_b200.h"
#include "mla_common.cuh"
#include "mla_gemm.cuh"
#include "mla_laswp.cuh"
#include "mla_panel.cuh"
#include "mla_trsm.cuh"

namespace mla {

constexpr int kWidthsCap = 8192;
constexpr int kMaxStrips = 1024;   // n <= 128 * 1024 columns
constexpr int LEFT_CW = 256;       // columns per LEFT item
constexpr int PREP_LOOKAHEAD = 12; // a strip is prepared this many strips ahead of its GEMM tiles

struct LuState {
  // iteration descriptor: written by CTA 0 between two grid barriers, read by everybody after
  int q0, q1, pend, w, b_target, npiv_prev, it, done;
  // queues (reset by CTA 0 in the same window)
  unsigned pq_next, pq_done, rq_next, rq_done;
  // flags, tagged with the iteration number (never reset)
  unsigned pf_done, ru_done;
  unsigned pprep_done[kMaxStrips];
  unsigned rprep_done[kMaxStrips];
  // outcome
  int singular, et_events, n_panels, ws_joins, panel_cols;
  // malleable split: panel-team size of the current iteration and the stamps that drive it
  int sm_pf_cur, sm_pf_peak;
  unsigned long long t_panel_end, t_rq_done;
  // device trace (globaltimer ns), one row per outer iteration (first kTraceCap): [0] iteration
  // start, [1] PQ complete (panel may start), [2] panel end, [3] RQ complete, [4] width<<32|k_new
  unsigned long long trace[1024][5];
  // accumulators of the LAST CTA of the grid (an RU CTA), globaltimer ns: [0] in GEMM tiles, [1] tile
  // count, [2] in PREP items, [3] PREP count, [4] in LEFT items, [5] waiting at the iteration
  // barriers + bookkeeping, [6] whole kernel
  unsigned long long dbg[8];
};
constexpr int kTraceCap = 1024;

// Per-CTA event record of the device trace (reference trace.py:16-23 TraceEvent, one private buffer per
// worker, no locking on the hot path): every CTA's thread 0 appends one record per phase it ran.
struct TraceEv {
  unsigned long long t0, t1;     // globaltimer ns
  int iter;                      // outer iteration (0 = prologue panel)
  int kind;                      // TK_*
  int items;                     // queue items executed (panel: columns factored)
  int team;                      // CTAs in the panel team of that iteration
};
enum TraceKind { TK_PQ = 1, TK_PANEL = 2, TK_RQ = 3, TK_RQ_MERGED = 4, TK_PANEL_ALL = 5 };
constexpr int kTraceEvPerCta = 4 * kTraceCap;
constexpr int kGetrfSmemBytes = 218 * 1024;   // dynamic shared memory of the persistent kernels
__host__ __device__ constexpr int mla_traced_smem_doubles() { return kGetrfSmemBytes / 8; }

struct GetrfArgs {
  double* A; int m, n; int64_t ld;
  int* ipiv;                 // global pivots out (device int32[n])
  int b_outer, b_inner, variant, sm_pf, q_chunks;
  int sm_pf_max;             // 0: fixed split; > sm_pf: the panel team may grow up to this many CTAs
  int* progress;             // nullable, host-mapped: receives q0 = number of leading rows that are final
  LuState* st;
  PivPlan* plan;             // plan of the previously factored panel (view rows start at q0)
  PanelWs* pws;
  int* piv_local;            // panel-local pivots of the panel being factored
  unsigned* ctrl;            // CW_* words
  mla_lu_info* info;
  int* widths; int widths_cap;
  TraceEv* tr;               // per-CTA event rings (kTraceEvPerCta records each) of the TRACED kernel, else unused
  DiagInv* dinv;             // two sets of inverted diagonal blocks: iteration `it` solves with set it & 1
  // Windowed run (the phased host entry point): columns [0, k0) are already factored and applied to columns
  // [k0, n); this launch factors columns [k0, n) of the m-row matrix, its interchanges reach back over the
  // columns left of k0 (LEFT items), and the outcome counters / iteration numbering in LuState carry on from
  // the previous launch (the host does not reset LuState).  k0 == 0: a fresh factorization.
  int k0;
  // A later window's first panel: by the panel team (0; the factors then do not depend on where the windows are
  // cut) or by the whole grid like the very first panel (1; faster -- nothing else can run beside it anyway --
  // and used when the caller has given up bit-identity with the unwindowed run, i.e. with deep catch-up).
  int window_first_by_all;
};

// item counts of one iteration, derived identically by every CTA from the descriptor
struct IterShape {
  int q0, q1, pend, w, it, kk;      // kk = q1 - q0 (depth of the update)
  int rows;                          // m - q1
  int nps, tmc;                      // panel strips, row tiles
  int pq_prep, pq_total;
  int rcols, nrs, rq_prep, rq_gemm, nleft, rq_total;
  int la_strips, gs;                 // PREP lookahead (strips) and RQ group size of the first row block
  int rb0;                           // row tiles of the first row block (<= kRowBlockTiles)
};

__device__ __forceinline__ IterShape iter_shape(const LuState* st, int m, int n, int grid) {
  IterShape s;
  s.q0 = *((volatile const int*)&st->q0);
  s.q1 = *((volatile const int*)&st->q1);
  s.pend = *((volatile const int*)&st->pend);
  s.w = *((volatile const int*)&st->w);
  s.it = *((volatile const int*)&st->it);
  s.kk = s.q1 - s.q0;
  s.rows = m - s.q1;
  s.tmc = (s.rows + GemmUpdateCfg::BM - 1) / GemmUpdateCfg::BM;
  s.nps = (s.w + TRSM_CW - 1) / TRSM_CW;
  s.rcols = n - s.q1 - s.w;
  s.nrs = (s.rcols + TRSM_CW - 1) / TRSM_CW;
  // PQ: [panel PREP][first PREP_LOOKAHEAD remainder PREPs][panel GEMM] -- those PREP strips depend
  // on nothing and fill the time the panel GEMM tiles would otherwise wait for the panel PREP.
  // enough fillers that every CTA of the grid has a PREP to do while the panel PREP runs
  s.la_strips = imin(imax(PREP_LOOKAHEAD, grid - s.nps), s.nrs);
  s.pq_prep = s.nps + s.la_strips;
  s.pq_total = s.pq_prep + s.nps * s.tmc;
  // RQ: nrs groups of gs = tmc + 2 items: [PREP of strip s+lookahead][LEFT strip s][GEMM tiles of
  // strip s]; then the LEFT strips that did not fit a group.  PREP and LEFT are HBM-bound row
  // interchanges (+ a small trsm): spread between the tensor-bound GEMM tiles they overlap with them
  // instead of saturating the memory system all at once at the start of the iteration.
  // Row-block-major tile order (see gemm_tile_desc): the first block of kRowBlockTiles row tiles
  // carries the PREP/LEFT items of the groups; the later blocks are pure GEMM groups.
  s.rq_prep = 0;
  s.rb0 = imin(kRowBlockTiles, s.tmc);
  s.gs = s.rb0 + 2;
  s.rq_gemm = s.nrs * s.tmc;
  s.nleft = (s.q0 + LEFT_CW - 1) / LEFT_CW;
  s.rq_total = s.nrs * (s.tmc + 2) + imax(0, s.nleft - s.nrs);
  return s;
}

// PREP of the column strip [c0, c0+cw): previous panel's interchanges (only columns >= pend still
// owe them, lu.py:247-255) then the triangular solve with A11.
__device__ inline void item_prep(const GetrfArgs& a, const IterShape& s, int c0, int cw, unsigned* flag,
                                 double* smem) {
  // columns in [q1, pend) are the leftover of an ET-cut panel: the panel (Crout order) has already
  // given them the interchanges AND their A12 rows
  int lo = imax(c0, s.pend);
  if (lo < c0 + cw) {
    laswp_apply_cols(a.A + (int64_t)lo * a.ld + s.q0, a.ld, c0 + cw - lo, (a.plan + (s.it & 1))->ref(), smem, kLaswpBufDoubles);
    if (trsm_use_inverse(s.kk))
      trsm_strip_inv(a.A + (int64_t)s.q0 * a.ld + s.q0, s.kk, a.ld, a.A + (int64_t)lo * a.ld + s.q0, c0 + cw - lo, a.ld,
                     a.dinv + (s.it & 1), smem);
    else
      trsm_strip_ool(a.A + (int64_t)s.q0 * a.ld + s.q0, s.kk, a.ld, a.A + (int64_t)lo * a.ld + s.q0, c0 + cw - lo, a.ld, smem);
  }
  __syncthreads();
  MLA_STRESS((blockIdx.x + s.it) % 3 == 1);        // ... and some publish their strip late
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, (unsigned)s.it);
  }
}

__device__ inline bool wait_flag_eq(const unsigned* flag, unsigned v, unsigned* abort_word) {
  __shared__ int s_good;
  if (threadIdx.x == 0) {
    bool good = true;
    if (ld_acquire(flag) != v) {
      unsigned long long t0 = globaltimer_ns();
      unsigned it = 0;
      while (ld_acquire(flag) != v) {
        if ((++it & 63u) == 0u) {
          if (ld_relaxed(abort_word) != 0u) { good = false; break; }
          if (globaltimer_ns() - t0 > kSpinTimeoutNs) { atomicExch(abort_word, 0xDEAD3u); good = false; break; }
        }
      }
    }
    s_good = good ? 1 : 0;
  }
  __syncthreads();
  bool g = s_good != 0;
  __syncthreads();
  return g;
}

// GEMM tile (tm, strip) of A22 -= A21 @ A12 for the strip starting at column c0.
__device__ __forceinline__ TileDesc item_gemm_desc(const GetrfArgs& a, const IterShape& s, int tm, int c0, int cw) {
  const int i0 = s.q1 + tm * GemmUpdateCfg::BM;
  double* c = a.A + (int64_t)c0 * a.ld + i0;
  return TileDesc{a.A + (int64_t)s.q0 * a.ld + i0, a.ld, a.A + (int64_t)c0 * a.ld + s.q0, a.ld,
                  c, a.ld, c, a.ld, s.kk, a.m - i0, cw, 1.0, -1.0, true};
}

__device__ inline int pop_item(unsigned* next) {
  __shared__ int s_item;
  if (threadIdx.x == 0) s_item = (int)atomicAdd(next, 1u);
  __syncthreads();
  int t = s_item;
  __syncthreads();
  return t;
}

// CTA-uniform non-blocking test of a strip flag
__device__ inline bool flag_ready(const unsigned* flag, unsigned v) {
  __shared__ int s_rdy;
  if (threadIdx.x == 0) s_rdy = (ld_acquire(flag) == v) ? 1 : 0;
  __syncthreads();
  bool r = s_rdy != 0;
  __syncthreads();
  return r;
}

// Per-CTA memory of the strip flags already seen set during the current queue drain.  A strip's flag is
// written once per drain, so after the first acquire-load that finds it set, this CTA need not go back to L2
// for it: with the row-block-major tile order consecutive tiles of a CTA lie in DIFFERENT strips, and the
// L2 round trip of a flag test (~0.7 us) sat between every two chained tiles while the DMMA pipe idled.
struct StripCache {
  unsigned bits[kMaxStrips / 32];
  __device__ __forceinline__ void clear() {      // collective over the CTA
    __syncthreads();
    for (int i = threadIdx.x; i < kMaxStrips / 32; i += blockDim.x) bits[i] = 0u;
    __syncthreads();
  }
  __device__ __forceinline__ bool has(int strip) const { return (bits[strip >> 5] >> (strip & 31)) & 1u; }
};

// flag_ready with the cache in front: the fast path touches shared memory only.  All threads take the same
// path (the bit is only ever written behind a barrier that every thread which read it as 0 takes part in).
__device__ __forceinline__ bool flag_ready_cached(StripCache& sc, const unsigned* flags, int strip, unsigned v) {
  if (sc.has(strip)) return true;
  __shared__ int s_rdy2;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int r = (ld_acquire(&flags[strip]) == v) ? 1 : 0;
    s_rdy2 = r;
    if (r) sc.bits[strip >> 5] |= 1u << (strip & 31);
  }
  __syncthreads();
  const bool r = s_rdy2 != 0;
  __syncthreads();
  return r;
}

// Drain one of the two queues of the iteration.  which == 0: PQ (next panel's columns), 1: RQ
// (remainder + LEFT strips).  GEMM tiles run through the pipelined tile engine with a one-item
// lookahead: while a tile finishes, the first k-slices of the next GEMM item (if its strip is already
// prepared) are prefetched.  Returns the number of items executed, or -1 on abort.
// Debug accumulators of one CTA live in shared memory during the run (a global read-modify-write per
// tile would itself stall the tile pipeline) and are flushed to LuState::dbg at kernel end.
__shared__ unsigned long long g_dbg[8];

// One decoded queue item.
struct QItem {
  int kind;      // 0 no-op, 1 PREP of a panel strip, 2 PREP of a remainder strip, 3 GEMM tile, 4 LEFT strip
  int strip;     // strip index (PREP/GEMM) or LEFT index
  int tm;        // row tile (GEMM)
};

__device__ __forceinline__ QItem decode_item(const IterShape& s, int which, int t) {
  QItem q{0, 0, 0};
  if (which == 0) {
    if (t < s.nps) { q.kind = 1; q.strip = t; }
    else if (t < s.pq_prep) { q.kind = 2; q.strip = t - s.nps; }
    else { int g = t - s.pq_prep; q.kind = 3; q.strip = g / s.tmc; q.tm = g - q.strip * s.tmc; }
    return q;
  }
  const int ngrp0 = s.nrs * s.gs;          // first row block: [PREP][LEFT][rb0 tiles] per strip
  if (t < ngrp0) {
    const int grp = t / s.gs, slot = t - grp * s.gs;
    if (slot == 0) {
      int ps = grp + s.la_strips;
      if (ps < s.nrs) { q.kind = 2; q.strip = ps; }
    } else if (slot == 1) {
      if (grp < s.nleft) { q.kind = 4; q.strip = grp; }
    } else { q.kind = 3; q.strip = grp; q.tm = slot - 2; }
    return q;
  }
  int r = t - ngrp0;
  const int later = s.nrs * (s.tmc - s.rb0);   // GEMM tiles of the later row blocks
  if (r < later) {
    const int per_block = s.nrs * kRowBlockTiles;
    const int rb = r / per_block;              // 0 = second row block
    const int row0 = s.rb0 + rb * kRowBlockTiles;
    const int rows_here = imin(kRowBlockTiles, s.tmc - row0);
    r -= rb * per_block;
    q.kind = 3;
    q.strip = r / rows_here;
    q.tm = row0 + (r - q.strip * rows_here);
    return q;
  }
  q.kind = 4;
  q.strip = s.nrs + (r - later);
  return q;
}

// Drain one of the two queues of the iteration.  which == 0: PQ (next panel's columns), 1: RQ
// (remainder + LEFT strips).  GEMM tiles run through the pipelined tile engine with a one-item
// lookahead: while a tile finishes, the first k-slices of the next GEMM item (if its strip is already
// prepared) are prefetched.  Returns the number of items executed, or -1 on abort.
#ifndef MLA_RQ_ATTR
#define MLA_RQ_ATTR __forceinline__
#endif
__device__ MLA_RQ_ATTR int run_queue(const GetrfArgs& a, const IterShape& s, double* smem, int which,
                                     bool signal_ru_done) {
  LuState* st = a.st;
  unsigned* next = which ? &st->rq_next : &st->pq_next;
  unsigned* done = which ? &st->rq_done : &st->pq_done;
  unsigned* flags = which ? st->rprep_done : st->pprep_done;   // flags the GEMM tiles of this queue wait on
  const int total = which ? s.rq_total : s.pq_total;
  const int ngemm = which ? s.rq_gemm : s.nps * s.tmc;
  const int col_base = which ? (s.q1 + s.w) : s.q1;
  const int col_end = which ? a.n : (s.q1 + s.w);
  int executed = 0, base = 0;
  bool primed = false;
  __shared__ StripCache s_cache;
  s_cache.clear();
  MLA_STRESS((blockIdx.x + s.it) % 5 == 0);        // some CTAs arrive late at the queue
  // Long queues (>= 16 tiles per CTA) pop one item further ahead with an atomic whose round trip
  // overlaps the running tile's main loop; short queues keep the shallow lookahead so the last
  // tiles of the iteration are not hoarded by one CTA.
  const bool deep = ngemm >= 16 * (int)gridDim.x;
  int ready_strip = -1;          // last strip whose PREP flag this CTA has seen set
  unsigned long long dbg_last_end = 0ull;
  __shared__ int s_fut;
  int t = pop_item(next);
  int tn = 0;
  bool have_tn = false;
  while (t < total) {
    const QItem it = decode_item(s, which, t);
    if (it.kind == 3) {
      const int strip = it.strip;
      const int c0 = col_base + strip * TRSM_CW;
      TileDesc cur = item_gemm_desc(a, s, it.tm, c0, imin(TRSM_CW, col_end - c0));
      if (!primed) {
        if (strip != ready_strip && !s_cache.has(strip)) {
          if (!wait_flag_eq(&flags[strip], (unsigned)s.it, a.ctrl)) return -1;
          if (threadIdx.x == 0) s_cache.bits[strip >> 5] |= 1u << (strip & 31);   // readers are behind the next barrier
        }
        ready_strip = strip;
        base = 0;
        tile_prologue<GemmUpdateCfg>(cur, base, smem);
      }
      // no lookahead over the last G items of the queue: hoarding them would leave other CTAs idle
      const bool look = t + (int)gridDim.x < total;
      if (!have_tn && look) { tn = pop_item(next); have_tn = true; }
      TileDesc nxt{};
      nxt.valid = false;
      // chaining needs the current tile to span the whole prefetch window (KT >= STAGES-1): its
      // prologue was issued without knowing the successor
      if (have_tn && tn < total && tile_kt<GemmUpdateCfg>(cur) >= GemmUpdateCfg::STAGES - 1) {
        const QItem itn = decode_item(s, which, tn);
        if (itn.kind == 3 && (itn.strip == ready_strip || flag_ready_cached(s_cache, flags, itn.strip, (unsigned)s.it))) {
          ready_strip = itn.strip;
          const int c2 = col_base + itn.strip * TRSM_CW;
          nxt = item_gemm_desc(a, s, itn.tm, c2, imin(TRSM_CW, col_end - c2));
        }
      }
      unsigned fut = 0;
      const bool fut_issued = deep && have_tn && tn + 2 * (int)gridDim.x < total;
      if (fut_issued && threadIdx.x == 0)
        asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(fut) : "l"(next) : "memory");
#ifdef MLA_NO_DBG
      const bool dbgc = false;
#else
      const bool dbgc = (blockIdx.x == gridDim.x - 1) && threadIdx.x == 0;
#endif
      unsigned long long dt0 = dbgc ? globaltimer_ns() : 0ull;
      if (dbgc && primed && dbg_last_end) g_dbg[7] += dt0 - dbg_last_end;   // gap between chained tiles
      base = tile_run<GemmUpdateCfg>(cur, nxt, base, smem);
      if (dbgc) { unsigned long long now = globaltimer_ns(); g_dbg[0] += now - dt0; g_dbg[1] += 1; dbg_last_end = now; }
      primed = nxt.valid;
      ++executed;
      if (have_tn) {
        t = tn;
        have_tn = false;
        if (fut_issued) {
          if (threadIdx.x == 0) s_fut = (int)fut;
          __syncthreads();
          tn = s_fut;
          have_tn = true;
          __syncthreads();
        }
      } else {
        t = pop_item(next);
      }
      continue;
    }
#ifdef MLA_NO_DBG
    const bool dbgc2 = false;
#else
    const bool dbgc2 = (blockIdx.x == gridDim.x - 1) && threadIdx.x == 0;
#endif
    unsigned long long dt1 = dbgc2 ? globaltimer_ns() : 0ull;
    if (it.kind == 1) {
      const int c0 = s.q1 + it.strip * TRSM_CW;
      item_prep(a, s, c0, imin(TRSM_CW, s.q1 + s.w - c0), &st->pprep_done[it.strip], smem);
    } else if (it.kind == 2) {
      const int c0 = s.q1 + s.w + it.strip * TRSM_CW;
      item_prep(a, s, c0, imin(TRSM_CW, a.n - c0), &st->rprep_done[it.strip], smem);
    } else if (it.kind == 4) {
      const int c0 = it.strip * LEFT_CW;
      laswp_apply_cols(a.A + (int64_t)c0 * a.ld + s.q0, a.ld, imin(LEFT_CW, s.q0 - c0), (a.plan + (s.it & 1))->ref(), smem,
                       kLaswpBufDoubles);
    }
    if (dbgc2 && it.kind != 0) {
      if (it.kind <= 2) { g_dbg[2] += globaltimer_ns() - dt1; g_dbg[3] += 1; }
      else g_dbg[4] += globaltimer_ns() - dt1;
    }
    primed = false;
    ++executed;
    if (have_tn) { t = tn; have_tn = false; }
    else t = pop_item(next);
  }
  // Completion is reported once per CTA, when it finds the queue empty: a per-item fence + atomic
  // would stall the tile pipeline for two L2 round trips per tile.  The CTA whose report completes
  // the count announces RU done (lu.py:309-310).  The tiles' bulk reductions into C must have been
  // performed before the report.
  bulk_wait_all();
  __syncthreads();
  if (threadIdx.x == 0 && executed > 0) {
    __threadfence();
    unsigned old = atom_add_release(done, (unsigned)executed);
    if (which && old + (unsigned)executed == (unsigned)total) {
      if (signal_ru_done) st_release(&st->ru_done, (unsigned)s.it);
      st->t_rq_done = globaltimer_ns();
      if (s.it <= kTraceCap) st->trace[s.it - 1][3] = globaltimer_ns();
    }
  }
  return executed;
}

__device__ __forceinline__ bool run_pq(const GetrfArgs& a, const IterShape& s, double* smem) {
  return run_queue(a, s, smem, 0, false) >= 0;
}
__device__ __forceinline__ int run_rq(const GetrfArgs& a, const IterShape& s, double* smem, bool signal_ru_done) {
  return run_queue(a, s, smem, 1, signal_ru_done);
}

// The persistent kernel body.  Cooperative launch, one CTA per SM.
// Global pivots (lu.py:236,317: panel-local -> global) and the interchange plan of a factored panel
// that starts at row/column q.  Collective over the CTA; kept out of line so that the persistent
// kernel's tile loops do not depend on it.
static __device__ __noinline__ void publish_pivots(int* ipiv, const int* piv_local, int q, int k_new, int rows,
                                            PivPlan* plan, double* smem) {
  const int tid = threadIdx.x;
  for (int t = tid; t < k_new; t += kThreads) ipiv[q + t] = q + piv_local[t];
  if (tid < 32) {
    int* scratch = reinterpret_cast<int*>(smem);
    build_pivot_plan(piv_local, k_new, (int64_t)rows, false, plan->ref(), scratch, scratch + kMaxPiv,
                     scratch + 3 * kMaxPiv, 2 * kMaxPiv, scratch + 5 * kMaxPiv);
  }
}

// Per-CTA control state of the persistent kernel.  It lives in SHARED memory, written by thread 0 only
// (each write is separated from its readers by a __syncthreads): nothing of the outer loop's bookkeeping
// is then live in registers across the tile loops of the queue drains, whose 128 accumulators + staging
// addresses need the whole register file (with ~50 scalars of bookkeeping live across them ptxas either
// spilled inside the k loop or re-derived the staging addresses there: 1830-2200 instead of ~1570
// instructions per 32-deep k slice, 3-7 % of the whole factorization; round 2).
struct KState {
  unsigned all_target, pf_target;  // arrivals expected so far at the two team barriers
  int ok;                          // 0 once an abort was observed
  int sm_pf;                       // panel-team size of the current iteration
  // bookkeeping carried from iteration to iteration (lu.py:314-326); only CTA 0's copy is used
  int k_new, w_sched, q1_of_panel, b_target, singular, et_events, n_panels, ws_joins, q0, q1, it_next, prebuilt;
  unsigned long long t_iter0, k_t0, b_t0;
  // device trace (TRACE kernels): records written so far, start stamp of the running phase
  int tr_n;
  unsigned long long tr_t0;
};

// TRACE selects the instrumented twin (k_getrf_traced, its own translation unit): the production kernel
// contains no tracing code at all.
template <bool TRACE>
__device__ __forceinline__ void getrf_persistent(const GetrfArgs& a, double* smem, int smem_doubles) {
  __shared__ KState ks;
  __shared__ IterShape sh;         // this iteration's item counts, derived once per CTA (thread 0)
  LuState* st = a.st;
  const int G = gridDim.x, bid = blockIdx.x, tid = threadIdx.x;
  unsigned* const abort_word = a.ctrl;  // CW_ABORT == 0
  const bool la = a.variant != MLA_VARIANT_LU && G >= 2;
  // Panel-team size.  Fixed at sm_pf (the reference's t_pf, restored every iteration, lu.py:270-273),
  // or -- with sm_pf_max > sm_pf -- malleable between iterations: doubled after an iteration in which
  // the panel finished after the remainder update (the panel was the critical path), halved again
  // after one in which it took less than a third of the iteration.  The pivots do not depend on the
  // team size; the factors only through the panel's device block width (slab fitting).
  const int sm_pf_lo = la ? imax(1, imin(a.sm_pf, G - 1)) : G;
  const int sm_pf_hi = la ? imax(sm_pf_lo, imin(a.sm_pf_max, G - 1)) : G;
  const bool ws = la && (a.variant == MLA_VARIANT_LU_MB || a.variant == MLA_VARIANT_LU_ET ||
                         a.variant == MLA_VARIANT_LU_WS_STATIC);
  const bool et = la && a.variant == MLA_VARIANT_LU_ET;
  const int m = a.m, n = a.n;
  const bool dbgk = (bid == G - 1) && tid == 0;

  const int k0 = a.k0;
  if (tid == 0) {
    ks.all_target = 0u; ks.pf_target = 0u; ks.ok = 1; ks.sm_pf = sm_pf_lo;
    ks.k_new = 0; ks.w_sched = 0; ks.q1_of_panel = k0; ks.b_target = a.b_outer; ks.singular = 0; ks.et_events = 0;
    ks.n_panels = 0; ks.ws_joins = 0; ks.q0 = k0; ks.q1 = k0; ks.it_next = 1; ks.prebuilt = 0;
    ks.t_iter0 = 0ull; ks.tr_n = 0; ks.tr_t0 = 0ull;
    if (k0 > 0) {
      // resume: nobody writes LuState before the prologue panel's collective has been entered by every CTA
      ks.singular = *((volatile const int*)&st->singular); ks.et_events = *((volatile const int*)&st->et_events);
      ks.n_panels = *((volatile const int*)&st->n_panels); ks.ws_joins = *((volatile const int*)&st->ws_joins);
      ks.it_next = *((volatile const int*)&st->it) + 1;
      if constexpr (TRACE) {
        // the CTA's event ring carries on behind the records of the earlier windows
        int used = 0;
        while (used < kTraceEvPerCta && a.tr[(size_t)bid * kTraceEvPerCta + used].kind != 0) ++used;
        ks.tr_n = used;
      }
    }
  }
  if (tid < 8) g_dbg[tid] = 0ull;
  __syncthreads();

  // A team exists in registers only for the duration of one collective (a barrier or a panel): it is
  // rebuilt from the shared state and its counter written back, so no Team is live across a queue drain.
  auto team_all = [&]() { Team t; t.init(bid, G, a.ctrl + 2 /*CW_BAR_ALL*/, abort_word, ks.all_target); t.ok = ks.ok != 0; return t; };
  auto team_pf = [&]() { Team t; t.init(bid, ks.sm_pf, a.ctrl + 3 /*CW_BAR_PF*/, abort_word, ks.pf_target); t.ok = ks.ok != 0; return t; };
  auto put_all = [&](const Team& t) { if (tid == 0) { ks.all_target = t.target; if (!t.ok) ks.ok = 0; } __syncthreads(); };
  auto put_pf = [&](const Team& t) { if (tid == 0) { ks.pf_target = t.target; if (!t.ok) ks.ok = 0; } __syncthreads(); };
  auto grid_barrier = [&]() -> bool { Team t = team_all(); t.barrier(); put_all(t); return ks.ok != 0; };
  // device trace (TRACE only): thread 0 of every CTA appends (phase, t0, t1, iteration) records to its ring
  auto tr_begin = [&]() {
    if constexpr (TRACE) { if (tid == 0) ks.tr_t0 = globaltimer_ns(); }
  };
  auto tr_end = [&](int kind, int iter, int items, int team) {
    if constexpr (TRACE) {
      if (tid == 0 && ks.tr_n < kTraceEvPerCta) {
        a.tr[(size_t)bid * kTraceEvPerCta + ks.tr_n] = TraceEv{ks.tr_t0, globaltimer_ns(), iter, kind, items, team};
        ks.tr_n = ks.tr_n + 1;
      }
    }
  };
  // result of a panel this CTA took part in -> shared state (before anything long-running follows)
  auto keep_panel_result = [&](const PanelResult& pr) {
    if (tid == 0) { ks.k_new = pr.cols_factored; ks.singular |= pr.singular; }
  };
  // the first members of the team that factored a panel invert its 128 x 128 diagonal blocks for the solves
  // of the iteration that applies it (set (it_use) & 1); the panel's last team barrier made it visible
  auto invert_diag_blocks = [&](const double* Lpanel, int k_new, int team_rank, int team_size, int it_use) {
    if (!trsm_use_inverse(k_new)) return;
    for (int blk = team_rank; blk * TRSM_IB < k_new; blk += team_size)
      diag_block_inverse(Lpanel, blk * TRSM_IB, imin(TRSM_IB, k_new - blk * TRSM_IB), a.ld, (a.dinv + (it_use & 1))->d[blk], smem);
  };

  // ---- prologue: first panel, the whole grid as one team (lu.py:224-241) --------------------------
  // (a later window's first panel is factored by the panel team instead, like the look-ahead panel it would
  // have been in an unwindowed run: the factors then do not depend on where the windows are cut)
  {
    const int w0 = imin(a.b_outer, n - k0);
    double* const P0 = a.A + (int64_t)k0 * a.ld + k0;
    const int it_first = ks.it_next;
    if (k0 > 0 && la && !a.window_first_by_all) {
      if (bid < ks.sm_pf) {
        tr_begin();
        Team t = team_pf();
        PanelResult pr = panel_ll(t, P0, m - k0, w0, a.ld, a.piv_local, a.b_inner, nullptr, 0u, 0, a.pws, smem, smem_doubles, true);
        keep_panel_result(pr);
        const bool pf_ok = t.ok;
        put_pf(t);
        if (pf_ok) invert_diag_blocks(P0, pr.cols_factored, bid, ks.sm_pf, it_first);
        tr_end(TK_PANEL, it_first - 1, pr.cols_factored, ks.sm_pf);
      }
      if (tid == 0) ks.w_sched = w0;
      __syncthreads();
    } else {
      tr_begin();
      Team t = team_all();
      PanelResult pr = panel_ll(t, P0, m - k0, w0, a.ld, a.piv_local, a.b_inner, nullptr, 0u, 0, a.pws, smem, smem_doubles, true);
      keep_panel_result(pr);
      if (tid == 0) ks.w_sched = w0;
      put_all(t);
      invert_diag_blocks(P0, pr.cols_factored, bid, G, it_first);
      tr_end(TK_PANEL_ALL, it_first - 1, pr.cols_factored, G);
    }
  }
  if (dbgk) ks.k_t0 = globaltimer_ns();

  // The interchange plan is double-buffered by iteration parity: iteration `it` applies plan[it & 1]
  // while the panel lead may already be writing plan[(it + 1) & 1]  (ks.it_next counts the iterations).
  while (true) {
    if (!ks.ok) break;
    // ---- bookkeeping (lu.py:314-326) by CTA 0, between two grid barriers ----------------------------
    if (dbgk) ks.b_t0 = globaltimer_ns();
    if (!grid_barrier()) break;
    if (bid == 0) {
      // global pivots + interchange plan of the just-factored panel, unless the panel team's lead
      // already produced them right after its panel (look-ahead variants)
      if (!ks.prebuilt) {
        publish_pivots(a.ipiv, a.piv_local, ks.q1_of_panel, ks.k_new, m - ks.q1_of_panel, a.plan + (ks.it_next & 1), smem);
      }
      __syncthreads();
      if (tid == 0) {
        const int k_new = ks.k_new, q1_of_panel = ks.q1_of_panel, w_sched = ks.w_sched;
        int b_target = ks.b_target, n_panels = ks.n_panels, et_events = ks.et_events;
        if (a.widths && n_panels < a.widths_cap) a.widths[n_panels] = k_new;
        ++n_panels;
        if (k_new < w_sched) { ++et_events; b_target = imax(a.b_inner, k_new); }
        else if (q1_of_panel > k0) b_target = imin(a.b_outer, 2 * b_target);
        const int pend = q1_of_panel + w_sched;
        const int q0 = q1_of_panel, q1 = q1_of_panel + k_new;
        ks.q0 = q0; ks.q1 = q1; ks.b_target = b_target; ks.n_panels = n_panels; ks.et_events = et_events;
        st->q0 = q0; st->q1 = q1; st->pend = pend;
        if (a.progress) {
          // every write to rows < q0 precedes the grid barrier above; later work touches rows >= q0 only
          __threadfence_system();
          *((volatile int*)a.progress) = q0;
        }
        st->w = imin(b_target, n - q1);
        st->b_target = b_target;
        st->npiv_prev = k_new;
        st->it = st->it + 1;
        st->done = (q1 >= n) ? 1 : 0;
        st->pq_next = 0; st->pq_done = 0; st->rq_next = 0; st->rq_done = 0;
        if (la) {
          int T = ks.sm_pf;
          if (sm_pf_hi > sm_pf_lo && q1_of_panel > k0) {
            const unsigned long long pe = *((volatile unsigned long long*)&st->t_panel_end);
            const unsigned long long rd = *((volatile unsigned long long*)&st->t_rq_done);
            if (rd == 0ull || pe > rd) T = imin(sm_pf_hi, 2 * T);
            else if (3 * (pe - ks.t_iter0) < (rd - ks.t_iter0)) T = imax(sm_pf_lo, T / 2);
          }
          st->sm_pf_cur = T;
          if (T > st->sm_pf_peak) st->sm_pf_peak = T;
          st->t_rq_done = 0ull;
          a.ctrl[3 /*CW_BAR_PF*/] = 0u;   // nobody is inside a panel-team barrier here
        }
        st->singular = ks.singular; st->et_events = et_events; st->n_panels = n_panels; st->ws_joins = ks.ws_joins;
      }
    }
    if (!grid_barrier()) { if (dbgk) g_dbg[5] += globaltimer_ns() - ks.b_t0; break; }
    if (dbgk) g_dbg[5] += globaltimer_ns() - ks.b_t0;
    // ---- this iteration's descriptor -> shared memory (thread 0), then everybody reads it there ------
    if (tid == 0) {
      ks.prebuilt = 0;
      ks.it_next = ks.it_next + 1;
      if (la) {
        ks.sm_pf = *((volatile const int*)&st->sm_pf_cur);
        ks.pf_target = 0u;                                   // the panel team is re-formed every iteration
        if (bid == 0) ks.t_iter0 = globaltimer_ns();
      }
      sh = iter_shape(st, m, n, G);
      ks.q1_of_panel = sh.q1;
      ks.w_sched = sh.w;
      ks.b_target = *((volatile const int*)&st->b_target);
    }
    __syncthreads();
    const bool is_pf = la && bid < ks.sm_pf;
    if (*((volatile const int*)&st->done)) {
      // ---- final_sync (lu.py:328-332): last panel's interchanges for the columns to its left ------
      for (int l = bid; l < sh.nleft; l += G) {
        int c0 = l * LEFT_CW;
        laswp_apply_cols(a.A + (int64_t)c0 * a.ld + sh.q0, a.ld, imin(LEFT_CW, sh.q0 - c0), (a.plan + (sh.it & 1))->ref(), smem,
                         kLaswpBufDoubles);
      }
      break;
    }
    const bool tr = sh.it <= kTraceCap;
    if (tr && bid == 0 && tid == 0) st->trace[sh.it - 1][0] = globaltimer_ns();

    if (!la) {
      // ---- variant lu: update, then panel, one team (lu.py:259-269) --------------------------------
      tr_begin();
      const int e0 = run_queue(a, sh, smem, 0, false);
      if (e0 < 0) break;
      tr_end(TK_PQ, sh.it, e0, G);
      tr_begin();
      const int e1 = run_queue(a, sh, smem, 1, false);
      if (e1 < 0) break;
      tr_end(TK_RQ, sh.it, e1, G);
      if (!grid_barrier()) break;
      tr_begin();
      Team t = team_all();
      PanelResult pr = panel_ll(t, a.A + (int64_t)sh.q1 * a.ld + sh.q1, m - sh.q1, sh.w, a.ld, a.piv_local, a.b_inner, nullptr,
                                0u, 0, a.pws, smem, smem_doubles, true);
      keep_panel_result(pr);
      put_all(t);
      invert_diag_blocks(a.A + (int64_t)sh.q1 * a.ld + sh.q1, pr.cols_factored, bid, G, sh.it + 1);
      tr_end(TK_PANEL_ALL, sh.it, pr.cols_factored, G);
    } else {
      // ---- look-ahead: everybody drains PQ, then PF factors while RU updates (lu.py:270-312) --------
      tr_begin();
      const int e0 = run_queue(a, sh, smem, 0, false);
      if (e0 < 0) break;
      tr_end(TK_PQ, sh.it, e0, ks.sm_pf);
      if (is_pf) {
        if (tid == 0) {
          if (!spin_until_ge(&st->pq_done, (unsigned)sh.pq_total, abort_word)) ks.ok = 0;
        }
        __syncthreads();
        if (tr && bid == 0 && tid == 0) st->trace[sh.it - 1][1] = globaltimer_ns();
        MLA_STRESS((bid + sh.it) % 4 == 2);
        tr_begin();
        Team t = team_pf();
        PanelResult pr = panel_ll(t, a.A + (int64_t)sh.q1 * a.ld + sh.q1, m - sh.q1, sh.w, a.ld, a.piv_local, a.b_inner,
                                  et ? &st->ru_done : nullptr, (unsigned)sh.it, 0, a.pws, smem, smem_doubles, true);
        keep_panel_result(pr);
        const bool pf_ok = t.ok;
        put_pf(t);
        if (pf_ok) invert_diag_blocks(a.A + (int64_t)sh.q1 * a.ld + sh.q1, pr.cols_factored, bid, ks.sm_pf, sh.it + 1);
        tr_end(TK_PANEL, sh.it, pr.cols_factored, ks.sm_pf);
        if (bid == 0 && tid == 0) {
          st_release(&st->pf_done, (unsigned)sh.it);
          st->t_panel_end = globaltimer_ns();
          if (tr) {
            st->trace[sh.it - 1][2] = globaltimer_ns();
            st->trace[sh.it - 1][4] = ((unsigned long long)sh.w << 32) | (unsigned)pr.cols_factored;
          }
        }
        if (bid == 0 && pf_ok) {
          // off the critical path of the update: the next iteration's pivots and plan
          __syncthreads();
          publish_pivots(a.ipiv, a.piv_local, sh.q1, pr.cols_factored, m - sh.q1, a.plan + ((sh.it + 1) & 1), smem);
          __syncthreads();
          if (tid == 0) ks.prebuilt = 1;
        }
        if (!pf_ok) { if (tid == 0) atomicExch(abort_word, 0xDEAD4u); break; }
        if (ws) {
          // worker sharing: the quiesced panel team joins the update queue (pool.py:377-414)
          if (a.variant == MLA_VARIANT_LU_WS_STATIC && sh.rq_total > 0) {
            // join only at the next q-chunk boundary of the GEMM item range (lu.py:290-304)
            if (tid == 0) {
              int q = imax(1, a.q_chunks);
              unsigned head = ld_acquire(&st->rq_next);
              int per = (sh.rq_total + q - 1) / q;
              int gpos = imax(0, (int)head);
              int next_chunk = ((gpos + per - 1) / per) * per;
              unsigned wait_for = (unsigned)imin(next_chunk, sh.rq_total);
              spin_until_ge(&st->rq_next, wait_for, abort_word);
            }
            __syncthreads();
          }
          tr_begin();                                   // the actual join: after the team's last barrier
          const int ex = run_queue(a, sh, smem, 1, et);
          if (ex < 0) break;
          if (ex > 0) tr_end(TK_RQ_MERGED, sh.it, ex, ks.sm_pf);
          if (bid == 0 && tid == 0 && ex > 0) ks.ws_joins = ks.ws_joins + 1;
        }
      } else {
        tr_begin();
        const int ex = run_queue(a, sh, smem, 1, et);
        if (ex < 0) break;
        tr_end(TK_RQ, sh.it, ex, ks.sm_pf);
      }
    }
  }
  if (dbgk) {
    g_dbg[6] += globaltimer_ns() - ks.k_t0;
    for (int i = 0; i < 8; ++i) st->dbg[i] = (k0 > 0 ? st->dbg[i] : 0ull) + g_dbg[i];
  }
  if (bid == 0 && tid == 0 && a.info) {
    a.info->cols_factored = n;
    a.info->singular = st->singular;
    a.info->et_events = st->et_events;
    a.info->n_panels = st->n_panels;
    a.info->ws_joins = st->ws_joins;
    a.info->sm_pf_peak = st->sm_pf_peak;
  }
}

}  // namespace mla
