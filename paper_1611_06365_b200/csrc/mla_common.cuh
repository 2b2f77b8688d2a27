// Device-side building blocks shared by every kernel of the LU hot path (sm_100a only).
//
//  * Team: the GPU analogue of the reference's thread team (pool.py:52-72, 129-179).  A team is a
//    set of co-resident CTAs (one per SM) that execute a routine collectively and meet at
//    barriers; `rank`/`size` have the meaning of TeamContext.rank/size.  Barriers are monotonic
//    counters in global memory (one atomic + one acquire-poll per CTA).
//  * acquire/release flag helpers: the reference's CompletionFlag (pool.py:28-49) becomes a
//    single-writer word in global memory, written with st.release.gpu and polled with
//    ld.acquire.gpu at entry points only.
//  * cp.async (LDGSTS) staging helpers with zero-fill, DMMA m8n8k4 wrapper.
//  * A watchdog: every spin loop gives up after MLA_SPIN_TIMEOUT_NS and raises the abort word, so a
//    protocol bug ends the kernel with an error code instead of hanging the GPU.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mla {

constexpr int kThreads = 256;                      // threads per CTA everywhere
constexpr unsigned long long kSpinTimeoutNs = 4000000000ull;  // 4 s

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *p >= target (acquire) or the abort word is raised / the watchdog fires.
// Returns false on abort.  Called by ONE thread per CTA.
__device__ __forceinline__ bool spin_until_ge(const unsigned* p, unsigned target, unsigned* abort_word) {
  if (ld_acquire(p) >= target) return true;
  unsigned long long t0 = globaltimer_ns();
  unsigned it = 0;
  while (true) {
    if (ld_acquire(p) >= target) return true;
    if ((++it & 63u) == 0u) {
      if (ld_relaxed(abort_word) != 0u) return false;
      if (globaltimer_ns() - t0 > kSpinTimeoutNs) {
        atomicExch(abort_word, 0xDEADu);
        return false;
      }
    }
  }
}

struct Team {
  int rank;            // this CTA's rank in the team
  int size;            // CTAs in the team
  unsigned* bar;       // monotonic arrival counter (global memory, zero at kernel start)
  unsigned target;     // arrivals expected at the next barrier (local bookkeeping)
  unsigned* abort_word;
  bool ok;             // false after an abort was observed

  __device__ __forceinline__ void init(int r, int s, unsigned* b, unsigned* ab, unsigned start = 0) {
    rank = r; size = s; bar = b; target = start; abort_word = ab; ok = true;
  }
  // Collective over the team's CTAs: all global writes before it are visible to all after it.
  // `ok` stays uniform across the CTA's threads (thread 0's verdict is broadcast).
  __device__ __forceinline__ void barrier() {
    __shared__ int s_ok;
    target += (unsigned)size;
    __syncthreads();
    if (threadIdx.x == 0) {
      bool good = true;
      if (size > 1) {
        __threadfence();
        atom_add_release(bar, 1u);
        good = spin_until_ge(bar, target, abort_word);
      }
      if (ld_relaxed(abort_word) != 0u) good = false;
      s_ok = good ? 1 : 0;
    }
    __syncthreads();
    if (!s_ok) ok = false;
  }
};

// ---- cp.async (LDGSTS) -----------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// 16-byte copy, src_bytes in {0,8,16}: the rest of the 16 bytes is zero-filled.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes) : "memory");
}
// 8-byte copy, src_bytes in {0,8}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- FP64 tensor core: DMMA.8x8x4 ------------------------------------------------------------
// D(8x8) += A(8x4, row) * B(4x8, col).  Lane T holds A[T/4][T%4], B[T%4][T/4], D[T/4][2*(T%4)+{0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ---- thread groups ---------------------------------------------------------------------------------
// A routine templated on its thread count NT runs either on the whole CTA (NT == kThreads) or on one of
// the CTA's independent groups of NT threads (group g = threadIdx.x / NT).  Groups synchronise on
// their own named barrier (id 1 + g), never on barrier 0, so two groups of a CTA progress
// independently -- one group's epilogue overlaps the other's DMMA stream.
template <int NT>
__device__ __forceinline__ int grp_tid() { return NT == kThreads ? (int)threadIdx.x : (int)(threadIdx.x % NT); }
template <int NT>
__device__ __forceinline__ int grp_id() { return NT == kThreads ? 0 : (int)(threadIdx.x / NT); }
template <int NT>
__device__ __forceinline__ void grp_sync() {
  if (NT == kThreads) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / NT)), "n"(NT) : "memory");
}

// ---- race stress (tools/race_stress.sh) ---------------------------------------------------------------------
// compute-sanitizer is closed on the GPU pool, so shared-memory races are hunted the crude way: a build with
// -DMLA_RACE_STRESS delays SOME warps by a few microseconds at the points where a missing barrier would let a
// fast warp overwrite what a slow one still reads; every deterministic result must stay bit-identical to the
// normal build's.  (With the round-1 epilogue -- no barrier between the k loop and the staging stores -- this
// build produces wrong factors at once: -DMLA_RACE_STRESS -DMLA_NO_EPILOGUE_BARRIER.)
#ifdef MLA_RACE_STRESS
#define MLA_STRESS(cond) do { if (cond) __nanosleep(4000); } while (0)
#else
#define MLA_STRESS(cond) do { } while (0)
#endif

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

}  // namespace mla
