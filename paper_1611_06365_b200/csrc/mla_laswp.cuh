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
// warp (all 32 lanes call it); scratch: 4 arrays of npiv ints of shared memory (top/lrow/lcur/pv).
// Returns false (and count = 0) if an index is out of range -- nothing may then be touched
// (kernels.py:326-327).
__device__ inline bool build_pivot_plan(const int* ipiv, int npiv, int64_t rows, bool reverse,
                                        PlanRef plan, int* top, int* lrow, int* lcur, int* pv) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  // the pivots are copied to shared scratch first: the simulation below is a chain of npiv
  // dependent steps and must not pay a global-memory round trip per step
  for (int t = lane; t < npiv && t < kMaxPiv; t += 32) {
    int p = ipiv[t];
    if (p < 0 || (int64_t)p >= rows) bad = true;
    top[t] = t;
    pv[t] = p;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad || npiv > kMaxPiv) {
    if (lane == 0) *plan.count = 0;
    __syncwarp();
    return false;
  }
  __syncwarp();
  int nlow = 0;  // entries in the lower list (uniform across lanes)
  for (int s = 0; s < npiv; ++s) {
    const int t = reverse ? (npiv - 1 - s) : s;
    const int p = pv[t];
    if (p == t) continue;
    if (p < npiv) {
      if (lane == 0) { int a = top[t]; top[t] = top[p]; top[p] = a; }
      __syncwarp();
    } else {
      int found = -1;
      for (int base = 0; base < nlow; base += 32) {
        int e = base + lane;
        unsigned m = __ballot_sync(0xffffffffu, e < nlow && lrow[e] == p);
        if (m) { found = base + __ffs(m) - 1; break; }
      }
      if (found < 0) {
        found = nlow;
        if (lane == 0) { lrow[nlow] = p; lcur[nlow] = p; }
        ++nlow;
        __syncwarp();
      }
      if (lane == 0) { int a = top[t]; top[t] = lcur[found]; lcur[found] = a; }
      __syncwarp();
    }
  }
  // compact the moves (identity moves dropped)
  int cnt = 0;
  for (int base = 0; base < npiv + nlow; base += 32) {
    int e = base + lane;
    int d = -1, sidx = -1;
    if (e < npiv) { d = e; sidx = top[e]; }
    else if (e < npiv + nlow) { d = lrow[e - npiv]; sidx = lcur[e - npiv]; }
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
// over the CTA.  `buf` is shared memory holding at least cg*count doubles, cg >= 1 columns per
// pass (buf_doubles gives its capacity).
__device__ inline void laswp_apply_cols(double* __restrict__ A, int64_t ld, int ncols, PlanRef plan,
                                        double* buf, int buf_doubles) {
  const int cnt = *plan.count;
  if (cnt <= 0 || ncols <= 0) return;
  int cg = buf_doubles / cnt;
  if (cg > 16) cg = 16;
  if (cg < 1) return;  // cannot happen: callers size buf for kPlanCap
  for (int c0 = 0; c0 < ncols; c0 += cg) {
    const int nc = imin(cg, ncols - c0);
    __syncthreads();
    for (int x = threadIdx.x; x < nc * cnt; x += blockDim.x) {
      int c = x / cnt, e = x - c * cnt;
      buf[x] = A[(int64_t)(c0 + c) * ld + plan.src[e]];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nc * cnt; x += blockDim.x) {
      int c = x / cnt, e = x - c * cnt;
      A[(int64_t)(c0 + c) * ld + plan.dst[e]] = buf[x];
    }
  }
  __syncthreads();
}

}  // namespace mla
