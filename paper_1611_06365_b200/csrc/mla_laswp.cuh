// Row interchanges (reference kernels.py:296-332 laswp/_swap_cols) as a two-step GPU operation.
//
// The reference applies npiv interchanges t <-> ipiv[t] one after the other to each column (a
// dependent chain of npiv swaps per column).  On the GPU the chain is resolved ONCE per pivot block
// into a permutation plan -- the list of touched rows with, for each, the row whose old content
// ends up there -- and every column then performs the same gather/scatter fully in parallel:
//     new[dst[e]] = old[src[e]]      for e in [0, count)
// The result is bit-identical to the sequential swaps (pure data movement).
//
// Traffic: algorithmic 32 B per (pivot, column).  Top rows [0,npiv) of a column are
// contiguous (coalesced); the lower partner rows are 8-byte accesses ld apart (one 32-byte sector
// each) -- inherent to row swaps on a column-major matrix.
#pragma once
#include "mla_common.cuh"

namespace mla {

constexpr int kMaxPiv = 1024;            // widest pivot block a plan can hold
constexpr int kPlanCap = 2 * kMaxPiv;    // touched rows <= 2 * npiv

struct PlanRef {           // a plan stored anywhere (global workspace or shared memory)
  int* count;              // number of (dst, src) moves; 0 when validation failed
  int* dst;
  int* src;
};

struct PivPlan {           // global-memory storage of one full-size plan
  int count;
  int npiv;
  int pad[2];
  int dst[kPlanCap];
  int src[kPlanCap];
  __device__ __forceinline__ PlanRef ref() { return PlanRef{&count, dst, src}; }
};

// Build the plan for ipiv[0..npiv) (view-local indices, view has `rows` rows).  Executed by ONE
// warp (all 32 lanes call it).  Shared scratch: top[npiv], pv[npiv], and an open-addressing hash
// table keys[tsize]/vals[tsize] (tsize a power of two >= 2*npiv) that tracks the lower rows touched
// so far.  The chain of npiv dependent swaps is simulated by lane 0 with O(1) shared-memory work per
// step; validation and the final compaction are warp-parallel.
// Returns false (and count = 0) if an index is out of range -- nothing may then be touched
// (kernels.py:326-327).
// t0 > 0: the block is chunk [t0, t0+npiv) of a longer pivot vector of the same view: interchange s of
// the chunk swaps view rows t0+s and ipiv[s], and ipiv[s] may lie anywhere in [0, rows) -- above the
// chunk as well (the reference's laswp accepts any in-range index, kernels.py:316-327).  Row ids in
// the plan are view rows; "top" rows are [t0, t0+npiv), every other touched row goes through the hash.
__device__ inline bool build_pivot_plan(const int* ipiv, int npiv, int64_t rows, bool reverse,
                                        PlanRef plan, int* top, int* keys, int* vals, int tsize, int* pv,
                                        int t0 = 0) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  for (int t = lane; t < npiv && t < kMaxPiv; t += 32) {
    int p = ipiv[t];
    if (p < 0 || (int64_t)p >= rows) bad = true;
    top[t] = t0 + t;
    pv[t] = p;
  }
  if ((int64_t)t0 + npiv > rows) bad = true;
  for (int x = lane; x < tsize; x += 32) keys[x] = -1;
  bad = __any_sync(0xffffffffu, bad);
  if (bad || npiv > kMaxPiv || tsize < 2 * npiv) {
    if (lane == 0) *plan.count = 0;
    __syncwarp();
    return false;
  }
  __syncwarp();
  if (lane == 0) {
    const unsigned mask = (unsigned)tsize - 1u;
    for (int s = 0; s < npiv; ++s) {
      const int t = reverse ? (npiv - 1 - s) : s;
      const int p = pv[t];
      const int pl = p - t0;
      if (pl == t) continue;
      if (pl >= 0 && pl < npiv) {
        int a = top[t]; top[t] = top[pl]; top[pl] = a;
      } else {
        unsigned h = ((unsigned)p * 2654435761u) & mask;
        while (true) {
          int k = keys[h];
          if (k == p) break;
          if (k < 0) { keys[h] = p; vals[h] = p; break; }
          h = (h + 1u) & mask;
        }
        int a = top[t]; top[t] = vals[h]; vals[h] = a;
      }
    }
  }
  __syncwarp();
  // Compact the moves (identity moves dropped), ordered so that one side of every move walks
  // consecutive rows of the top block (coalesced): (1) the top rows as destinations, in row order;
  // (2) the lower rows that receive a top row, in order of that SOURCE row; (3) lower <- lower.
  for (int t = lane; t < npiv; t += 32) pv[t] = -1;
  __syncwarp();
  for (int x = lane; x < tsize; x += 32)
    if (keys[x] >= 0 && vals[x] >= t0 && vals[x] < t0 + npiv) pv[vals[x] - t0] = keys[x];   // each source row occurs once
  __syncwarp();
  int cnt = 0;
  for (int base = 0; base < 2 * npiv + tsize; base += 32) {
    int e = base + lane;
    int d = -1, sidx = -1;
    if (e < npiv) { d = t0 + e; sidx = top[e]; }
    else if (e < 2 * npiv) { d = pv[e - npiv]; sidx = t0 + (e - npiv); }
    else if (e < 2 * npiv + tsize && keys[e - 2 * npiv] >= 0 &&
             (vals[e - 2 * npiv] < t0 || vals[e - 2 * npiv] >= t0 + npiv)) {
      d = keys[e - 2 * npiv]; sidx = vals[e - 2 * npiv];
    }
    bool keep = (d >= 0) && (d != sidx);
    unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      int pos = cnt + __popc(m & ((1u << lane) - 1u));
      plan.dst[pos] = d;
      plan.src[pos] = sidx;
    }
    cnt += __popc(m);
  }
  if (lane == 0) *plan.count = cnt;
  __syncwarp();
  return true;
}

// Apply a plan to columns [0, ncols) of the view A (rows start at the plan's row 0).  Collective
// over the CTA.  `buf` is shared memory of buf_doubles doubles; its tail holds a copy of the plan's
// index lists, the rest stages CG columns per pass.  Each thread owns plan entries e = tid, tid+T, ..
// and keeps LASWP_CG independent column loads in flight per entry (the moves are pure latency:
// 8-byte accesses one sector each).
constexpr int LASWP_CG = 16;
constexpr int kLaswpBufDoubles = 20 * 1024;   // staging buffer the callers provide (160 KiB)

__device__ inline void laswp_apply_cols(double* __restrict__ A, int64_t ld, int ncols, PlanRef plan,
                                        double* buf, int buf_doubles) {
  const int cnt = *plan.count;
  if (cnt <= 0 || ncols <= 0) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  // index lists at the end of the buffer (2*cnt ints = cnt doubles)
  int* s_src = reinterpret_cast<int*>(buf + buf_doubles - cnt);
  int* s_dst = s_src + cnt;
  const int stage_cap = buf_doubles - cnt;
  int cg = stage_cap / cnt;
  if (cg > LASWP_CG) cg = LASWP_CG;
  if (cg < 1) return;  // cannot happen: callers size buf for kPlanCap
  __syncthreads();
  for (int e = tid; e < cnt; e += nt) { s_src[e] = plan.src[e]; s_dst[e] = plan.dst[e]; }
  __syncthreads();
  for (int c0 = 0; c0 < ncols; c0 += cg) {
    const int nc = imin(cg, ncols - c0);
    double* __restrict__ base = A + (int64_t)c0 * ld;
    if (nc == LASWP_CG) {
      for (int e = tid; e < cnt; e += nt) {
        const double* p = base + s_src[e];
        double v[LASWP_CG];
#pragma unroll
        for (int c = 0; c < LASWP_CG; ++c) v[c] = p[(int64_t)c * ld];
#pragma unroll
        for (int c = 0; c < LASWP_CG; ++c) buf[c * cnt + e] = v[c];
      }
      __syncthreads();
      for (int e = tid; e < cnt; e += nt) {
        double* p = base + s_dst[e];
#pragma unroll
        for (int c = 0; c < LASWP_CG; ++c) p[(int64_t)c * ld] = buf[c * cnt + e];
      }
    } else {
      for (int e = tid; e < cnt; e += nt) {
        const double* p = base + s_src[e];
        for (int c = 0; c < nc; ++c) buf[c * cnt + e] = p[(int64_t)c * ld];
      }
      __syncthreads();
      for (int e = tid; e < cnt; e += nt) {
        double* p = base + s_dst[e];
        for (int c = 0; c < nc; ++c) p[(int64_t)c * ld] = buf[c * cnt + e];
      }
    }
    __syncthreads();
  }
}

}  // namespace mla
