// Filler queue: a deep multiply  C (m x n) -= A (m x k) @ B (k x n)  cut into work units that ANY CTA may pick
// up whenever it has nothing better to do.
//
// Why.  The windowed (two-level) factorization applies a factored window of W columns to the columns right of
// the next window as ONE multiply of depth W (the tile engine runs those at 34-35 TFLOP/s: C is read and
// written once per window, not once per 512-column panel).  That multiply is off the critical path -- the next
// window does not need it -- so it is not run as a kernel of its own but handed to the persistent kernel that
// factors the next window: update-team CTAs that have drained their queue and would only wait for the panel
// (the reference's "RU team idles until PF is done", lu.py:305-312, which WS/ET attack from the other side)
// execute units of it instead.  What is left when the window is done is drained by k_filler.
//
// Units.  unit u = (chunk c = u / ntiles, tile t = u % ntiles): tile t of C (128 x 128, row-block-major order
// like gemm_tile_desc) receives the contribution of the k range [c * kc, (c + 1) * kc).  Chunks of one tile are
// applied in ascending order -- prog[t] counts the chunks already added, unit (t, c) waits for prog[t] == c --
// so every entry of C sees the same additions in the same order whoever runs them and whenever: the result is
// deterministic.  kc bounds how long a CTA that has started a unit stays away from the critical path
// (1024: ~140 us).
#pragma once
#include "mla_common.cuh"
#include "mla_gemm.cuh"

namespace mla {

struct FillerQ {
  double* C; int64_t ldc;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  int m, n, k, kc;
  int tm_count, tn_count, ntiles, nchunks, total, rbt;
  unsigned next;          // units handed out
  unsigned done;          // units completed (statistics)
  unsigned* prog;         // [ntiles] chunks already added to tile t
};

struct FillerUnit { int tile, chunk; };

__device__ __forceinline__ FillerUnit filler_decode(const FillerQ& q, int u) {
  FillerUnit x;
  x.chunk = u / q.ntiles;
  x.tile = u - x.chunk * q.ntiles;
  return x;
}

__device__ __forceinline__ TileDesc filler_desc(const FillerQ& q, FillerUnit x) {
  const int per_block = q.rbt * q.tn_count;
  const int rb = x.tile / per_block;
  const int rows_here = imin(q.rbt, q.tm_count - rb * q.rbt);
  const int r = x.tile - rb * per_block;
  const int tn = r / rows_here, tm = rb * q.rbt + (r - tn * rows_here);
  const int i0 = tm * GemmUpdateCfg::BM, j0 = tn * GemmUpdateCfg::BN;
  const int k0 = x.chunk * q.kc;
  double* c = q.C + (int64_t)j0 * q.ldc + i0;
  return TileDesc{q.A + (int64_t)k0 * q.lda + i0, q.lda, q.B + (int64_t)j0 * q.ldb + k0, q.ldb, c, q.ldc, c, q.ldc,
                  imin(q.kc, q.k - k0), q.m - i0, q.n - j0, 1.0, -1.0, true};
}

// all bulk reductions of this thread except those of the most recent `N` groups have been performed
template <int N>
__device__ __forceinline__ void bulk_wait_but() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

// Execute units until the queue is empty or -- stop_flag != nullptr -- *stop_flag == stop_val (checked before
// every pop; a started unit is always finished).  Collective over the CTA.  Returns the units executed, -1 on
// abort.  Must be inlined into its kernel (the tile engine's bulk reductions, see mla_gemm.cuh).
__device__ __forceinline__ int filler_run(FillerQ* qg, const unsigned* stop_flag, unsigned stop_val,
                                          unsigned* abort_word, double* smem) {
  __shared__ FillerQ q;
  __shared__ int s_u, s_rdy;
  __syncthreads();
  if (threadIdx.x == 0) {
    q = *qg;
    int u = q.total;
    if (!(stop_flag && ld_acquire(stop_flag) == stop_val)) u = (int)atomicAdd(&qg->next, 1u);
    s_u = u;
  }
  __syncthreads();
  const int total = q.total;
  int u = s_u;
  int executed = 0, base = 0;
  bool primed = false;
  int prev_tile = -1, prev_chunk = 0;       // unit whose completion has not been published yet
  // publish unit (t, c): its additions into C are performed -> the tile's next chunk may go
  auto publish = [&](int t, int c) {
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(&qg->prog[t], (unsigned)(c + 1));
      atomicAdd(&qg->done, 1u);
    }
  };
  while (u < total) {
    const FillerUnit x = filler_decode(q, u);
    const TileDesc cur = filler_desc(q, x);
    if (!primed) {
      // a chunk of the same tile may still be in flight on another CTA (or unpublished on this one)
      if (prev_tile == x.tile) { bulk_wait_all(); __syncthreads(); publish(prev_tile, prev_chunk); prev_tile = -1; }
      if (threadIdx.x == 0) {
        int ok = 1;
        if (ld_acquire(&qg->prog[x.tile]) != (unsigned)x.chunk) {
          const unsigned long long t0 = globaltimer_ns();
          unsigned it = 0;
          while (ld_acquire(&qg->prog[x.tile]) != (unsigned)x.chunk) {
            if ((++it & 63u) == 0u) {
              if (ld_relaxed(abort_word) != 0u) { ok = 0; break; }
              if (globaltimer_ns() - t0 > kSpinTimeoutNs) { atomicExch(abort_word, 0xDEAD5u); ok = 0; break; }
            }
          }
        }
        s_rdy = ok;
      }
      __syncthreads();
      const bool ok = s_rdy != 0;
      __syncthreads();
      if (!ok) return -1;
      base = 0;
      tile_prologue<GemmUpdateCfg>(cur, base, smem);
    }
    // the unit after this one: popped now so that its first slices are prefetched under this unit's tail
    if (threadIdx.x == 0) {
      int un = total, rdy = 0;
      if (!(stop_flag && ld_acquire(stop_flag) == stop_val)) un = (int)atomicAdd(&qg->next, 1u);
      if (un < total) {
        const FillerUnit y = filler_decode(q, un);
        rdy = (y.tile != x.tile && y.tile != prev_tile && ld_acquire(&qg->prog[y.tile]) == (unsigned)y.chunk) ? 1 : 0;
      }
      s_u = un;
      s_rdy = rdy;
    }
    __syncthreads();
    const int un = s_u;
    const bool chain = s_rdy != 0 && tile_kt<GemmUpdateCfg>(cur) >= GemmUpdateCfg::STAGES - 1;
    __syncthreads();
    TileDesc nxt{};
    nxt.valid = false;
    if (chain) nxt = filler_desc(q, filler_decode(q, un));
    base = tile_run<GemmUpdateCfg>(cur, nxt, base, smem);
    primed = nxt.valid;
    ++executed;
    // the unit BEFORE this one is complete once all but this unit's two reduction groups are: its publication
    // costs no wait.  (A unit that took the read-modify-write epilogue -- fringe tile, odd leading dimension --
    // committed no groups: then everything must be waited for.)
    if (prev_tile >= 0) {
      const bool two_groups = cur.mrem >= GemmUpdateCfg::BM && cur.nrem >= GemmUpdateCfg::BN && cur.K > 0 &&
                              (((uintptr_t)cur.Cout & 15) == 0) && ((cur.ldcout & 1) == 0);
      if (two_groups) bulk_wait_but<2>(); else bulk_wait_all();
      __syncthreads();
      publish(prev_tile, prev_chunk);
    }
    prev_tile = x.tile;
    prev_chunk = x.chunk;
    u = un;
  }
  if (prev_tile >= 0) { bulk_wait_all(); __syncthreads(); publish(prev_tile, prev_chunk); }
  bulk_wait_all();
  __syncthreads();
  return executed;
}

}  // namespace mla
