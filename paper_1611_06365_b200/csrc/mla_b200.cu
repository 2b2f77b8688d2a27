// libmla_b200.so -- C ABI (include/mla_b200.h) over the hand-written sm_100a kernels of the
// blocked LU hot path.  Build: see paper_1611_06365_b200/build.py
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <thread>
#include <new>

#include "../../include/mla_b200.h"
#include "mla_common.cuh"
#include "mla_gemm.cuh"
#include "mla_laswp.cuh"
#include "mla_trsm.cuh"
#include "mla_panel.cuh"
#include "mla_getrf.cuh"

using namespace mla;

// ---- control block layout (device words) --------------------------------------------------------
enum CtrlWord {
  CW_ABORT = 0,
  CW_QUEUE_NEXT = 1,
  CW_BAR_ALL = 2,
  CW_BAR_PF = 3,
  CW_ERR_INDEX = 4,
  CW_QUEUE_DONE = 5,   // items of the current apply step completed (all launches of the step)
  CW_STEP_DONE = 6,    // = the step's tag once its queue has been drained: the distributed driver's ru_done
  CW_COUNT = 64
};

constexpr int kDynSmemBytes = 218 * 1024;   // dynamic shared memory of the team kernels
constexpr int kDynSmemDoubles = kDynSmemBytes / 8;
constexpr int kMaxHostPhases = 16;

struct mla_handle_s {
  int device;
  int num_sms;
  int last_cuda;
  unsigned* ctrl;        // CW_COUNT words (device)
  unsigned* ctrl_host;   // pinned mirror
  int sm_pf_max = 0;     // malleable panel team: upper size (0 = fixed split)
  int update_sms = 0;    // grid of mla_apply_panel (0 = every SM)
  PivPlan* plan;         // device: permutation plan of the last pivot block
  PanelWs* panel_ws;     // device: exchange slots of the panel team
  LuState* lu_state;     // device: persistent-kernel state
  int* piv_local;        // device: panel-local pivots of the current panel (kMaxPiv)
  mla_lu_info* info_dev; // device
  mla_lu_info* info_host;  // pinned
  int32_t* widths_dev;   // device, kWidthsCap
  cudaStream_t s_main, s_copy;   // non-blocking streams of the _host entry point (factor / stream results out)
  cudaEvent_t ev_done;
  int* progress_host;    // pinned + mapped: number of leading rows that are final (written by the kernel)
  int* progress_dev;     // device alias of progress_host
  int* next_progress;    // consumed by the next mla_getrf_la launch (nullptr: no progress reports)
  double* a_dev;         // cached device matrix for the _host entry point
  size_t a_dev_bytes;
  int32_t* ipiv_dev;
  size_t ipiv_dev_n;
  double* resid_dev;
  unsigned apply_tag;    // per-call tag of the strip flags used by mla_apply_panel (never reused)
  TraceEv* trace_dev;    // per-CTA event rings of the persistent kernel (nullptr: tracing off)
  DiagInv* dinv;         // device: inverted 128 x 128 diagonal blocks of the current panel(s), two sets
  // phased host entry point: upload stream, one event per uploaded column chunk, window boundaries
  cudaStream_t s_up;
  cudaEvent_t ev_up[kMaxHostPhases];
  int phase_count;       // -1: default policy, 0: one phase (upload, then factor), > 0: explicit boundaries
  int64_t phase_bounds[kMaxHostPhases];
  int phase_deep;        // > 0: catch-up in super-blocks of this many columns, one deep multiply each (0: per panel)
};

#define CK(h, call)                                   \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) {                          \
      (h)->last_cuda = (int)e_;                       \
      return MLA_E_CUDA;                              \
    }                                                 \
  } while (0)

extern "C" const char* mla_version(void) { return "paper_1611_06365_b200 0.1 (sm_100a)"; }

extern "C" int mla_destroy(mla_handle h);

extern "C" int mla_create(int device, mla_handle* out) {
  if (!out) return MLA_E_INVALID;
  mla_handle h = new (std::nothrow) mla_handle_s();
  if (!h) return MLA_E_NOMEM;
  memset(h, 0, sizeof(*h));
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete h; return MLA_E_CUDA; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { delete h; return MLA_E_CUDA; }
  h->num_sms = prop.multiProcessorCount;
  if (cudaMalloc(&h->ctrl, CW_COUNT * sizeof(unsigned)) != cudaSuccess) { delete h; return MLA_E_CUDA; }
  if (cudaMallocHost(&h->ctrl_host, CW_COUNT * sizeof(unsigned)) != cudaSuccess) { cudaFree(h->ctrl); delete h; return MLA_E_CUDA; }
  cudaMemset(h->ctrl, 0, CW_COUNT * sizeof(unsigned));
  bool ok = cudaMalloc(&h->plan, 2 * sizeof(PivPlan)) == cudaSuccess &&
            cudaMalloc(&h->panel_ws, sizeof(PanelWs)) == cudaSuccess &&
            cudaMalloc(&h->lu_state, sizeof(LuState)) == cudaSuccess &&
            cudaMalloc(&h->piv_local, kMaxPiv * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&h->info_dev, sizeof(mla_lu_info)) == cudaSuccess &&
            cudaMallocHost(&h->info_host, sizeof(mla_lu_info)) == cudaSuccess &&
            cudaMalloc(&h->widths_dev, kWidthsCap * sizeof(int32_t)) == cudaSuccess &&
            cudaMalloc(&h->resid_dev, 4 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&h->dinv, 2 * sizeof(DiagInv)) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&h->s_main, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&h->s_copy, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&h->s_up, cudaStreamNonBlocking) == cudaSuccess &&
       cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming) == cudaSuccess &&
       cudaHostAlloc(&h->progress_host, 64, cudaHostAllocMapped) == cudaSuccess &&
       cudaHostGetDevicePointer(&h->progress_dev, h->progress_host, 0) == cudaSuccess;
  for (int i = 0; ok && i < kMaxHostPhases; ++i)
    ok = cudaEventCreateWithFlags(&h->ev_up[i], cudaEventDisableTiming) == cudaSuccess;
  h->phase_count = -1;
  h->phase_deep = 4096;
  if (!ok) { mla_destroy(h); return MLA_E_NOMEM; }
  cudaMemset(h->plan, 0, 2 * sizeof(PivPlan));
  cudaMemset(h->panel_ws, 0, sizeof(PanelWs));
  cudaMemset(h->lu_state, 0, sizeof(LuState));
  h->apply_tag = 0x40000000u;   // far above any iteration number the persistent kernel tags flags with
  *out = h;
  return MLA_OK;
}

extern "C" int mla_destroy(mla_handle h) {
  if (!h) return MLA_E_INVALID;
  cudaFree(h->ctrl);
  cudaFreeHost(h->ctrl_host);
  cudaFree(h->plan);
  cudaFree(h->panel_ws);
  cudaFree(h->lu_state);
  cudaFree(h->piv_local);
  cudaFree(h->info_dev);
  cudaFreeHost(h->info_host);
  cudaFree(h->widths_dev);
  cudaFree(h->resid_dev);
  cudaFree(h->a_dev);
  cudaFree(h->ipiv_dev);
  cudaFree(h->trace_dev);
  cudaFree(h->dinv);
  if (h->s_main) cudaStreamDestroy(h->s_main);
  if (h->s_copy) cudaStreamDestroy(h->s_copy);
  if (h->s_up) cudaStreamDestroy(h->s_up);
  for (int i = 0; i < kMaxHostPhases; ++i) if (h->ev_up[i]) cudaEventDestroy(h->ev_up[i]);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  if (h->progress_host) cudaFreeHost(h->progress_host);
  delete h;
  return MLA_OK;
}

extern "C" int mla_num_sms(mla_handle h) { return h ? h->num_sms : MLA_E_INVALID; }
extern "C" int mla_last_cuda_error(mla_handle h) { return h ? h->last_cuda : MLA_E_INVALID; }

// ---- gemm ------------------------------------------------------------------------------------------
// Persistent tile-queue kernel: every CTA pulls tile ids from one atomic counter (the GPU form of
// the reference's round-robin loop 4, kernels.py:138, made dynamic).  Donor CTAs (the last
// `donors` of the grid) model the reference's worker sharing: they stay parked until *join_flag is
// set, re-checking at tile granularity, then join the same queue (checkpoint_merge, pool.py:377-414).
__global__ void __launch_bounds__(kThreads, 1)
k_gemm(GemmProblem p, unsigned* ctrl, const unsigned* join_flag, int donors) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_tile;
  const int ntiles = gemm_num_tiles<GemmUpdateCfg>(p);
  const bool donor = join_flag != nullptr && (int)blockIdx.x >= (int)gridDim.x - donors;
  if (donor) {
    // parked: wait for the flag or for the queue to drain
    if (threadIdx.x == 0) {
      unsigned long long t0 = globaltimer_ns();
      int go = 0;
      while (true) {
        if (ld_acquire(join_flag) != 0u) { go = 1; break; }
        if (ld_relaxed(ctrl + CW_QUEUE_NEXT) >= (unsigned)ntiles) break;
        if (globaltimer_ns() - t0 > kSpinTimeoutNs) break;
        __nanosleep(200);
      }
      s_tile = go;
    }
    __syncthreads();
    if (!s_tile) return;
    __syncthreads();
  }
  // one-tile lookahead: the next tile's first k-slices are prefetched while the current tile finishes
  auto pop = [&]() {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ctrl + CW_QUEUE_NEXT, 1u);
    __syncthreads();
    int t = s_tile;
    __syncthreads();
    return t;
  };
  int t = pop();
  if (t >= ntiles) return;
  TileDesc cur = gemm_tile_desc<GemmUpdateCfg>(p, t);
  int base = 0;
  tile_prologue<GemmUpdateCfg>(cur, base, smem);
  while (true) {
    int tn = pop();
    TileDesc nxt{};
    nxt.valid = false;
    if (tn < ntiles) nxt = gemm_tile_desc<GemmUpdateCfg>(p, tn);
    const bool chain = nxt.valid && tile_kt<GemmUpdateCfg>(cur) >= GemmUpdateCfg::STAGES - 1;
    if (nxt.valid && !chain) {
      // short-k tiles cannot be chained: run cur alone, then prime nxt from scratch
      TileDesc none{};
      none.valid = false;
      tile_run<GemmUpdateCfg>(cur, none, base, smem);
      cur = nxt;
      base = 0;
      tile_prologue<GemmUpdateCfg>(cur, base, smem);
      continue;
    }
    base = tile_run<GemmUpdateCfg>(cur, nxt, base, smem);
    if (!nxt.valid) break;
    cur = nxt;
  }
  bulk_wait_all();   // this CTA's reductions into C are performed before the kernel retires
}

__global__ void k_scale(double* C, int64_t m, int64_t n, int64_t ldc, double alpha) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      C[i + j * ldc] = alpha * C[i + j * ldc];
}

extern "C" int mla_gemm(mla_handle h, double* C, int64_t m, int64_t n, int64_t ldc, const double* A,
                        int64_t lda, const double* B, int64_t ldb, int64_t k, double alpha, double beta,
                        const uint32_t* join_flag, int donor_ctas, void* stream) {
  if (!h || m < 0 || n < 0 || k < 0) return MLA_E_INVALID;
  if (m == 0 || n == 0) return MLA_OK;
  if (ldc < m || (k > 0 && (lda < m || ldb < k))) return MLA_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (k == 0) {  // kernels.py:226-232
    if (alpha != 1.0) {
      dim3 grid((unsigned)((m + 255) / 256 > 64 ? 64 : (m + 255) / 256), (unsigned)(n > 1024 ? 1024 : n));
      k_scale<<<grid, 256, 0, s>>>(C, m, n, ldc, alpha);
      CK(h, cudaGetLastError());
    }
    return MLA_OK;
  }
  GemmProblem p{C, ldc, A, lda, B, ldb, (int)m, (int)n, (int)k, alpha, beta};
  CK(h, cudaMemsetAsync(h->ctrl + CW_QUEUE_NEXT, 0, sizeof(unsigned), s));
  CK(h, cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmUpdateCfg::SMEM_BYTES));
  int64_t ntiles = ((m + 127) / 128) * ((n + 127) / 128);
  int grid = (int)(ntiles < h->num_sms ? ntiles : h->num_sms);
  if (join_flag) grid = h->num_sms;  // donors need their CTAs to exist
  if (donor_ctas < 0) donor_ctas = 0;
  if (donor_ctas >= grid) donor_ctas = grid - 1;
  k_gemm<<<grid, kThreads, GemmUpdateCfg::SMEM_BYTES, s>>>(p, h->ctrl, join_flag, donor_ctas);
  CK(h, cudaGetLastError());
  return MLA_OK;
}


// ---- trsm ------------------------------------------------------------------------------------------
// Inverses of the 128 x 128 diagonal blocks of trilu(L) (one CTA per block) for the 128-row form of the solve.
__global__ void __launch_bounds__(kThreads, 1)
k_diag_inv(const double* L, int w, int64_t ldl, DiagInv* out) {
  extern __shared__ __align__(16) double smem[];
  for (int blk = blockIdx.x; blk * TRSM_IB < w; blk += gridDim.x)
    diag_block_inverse(L, blk * TRSM_IB, imin(TRSM_IB, w - blk * TRSM_IB), ldl, out->d[blk], smem);
}

static int launch_diag_inv(mla_handle h, const double* L, int64_t w, int64_t ldl, DiagInv* out, cudaStream_t s) {
  const int smem_bytes = TRSM_SMEM_DOUBLES * 8;
  CK(h, cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  k_diag_inv<<<(unsigned)((w + TRSM_IB - 1) / TRSM_IB), kThreads, smem_bytes, s>>>(L, (int)w, ldl, out);
  CK(h, cudaGetLastError());
  return MLA_OK;
}

__global__ void __launch_bounds__(kThreads, 1)
k_trsm(const double* L, int w, int64_t ldl, double* B, int64_t c, int64_t ldb, const DiagInv* inv) {
  extern __shared__ __align__(16) double smem[];
  const int64_t strips = (c + TRSM_CW - 1) / TRSM_CW;
  for (int64_t s = blockIdx.x; s < strips; s += gridDim.x) {
    int64_t c0 = s * TRSM_CW;
    const int cw = (int)(c - c0 < TRSM_CW ? c - c0 : TRSM_CW);
    if (inv) trsm_strip_inv(L, w, ldl, B + c0 * ldb, cw, ldb, inv, smem);
    else trsm_strip(L, w, ldl, B + c0 * ldb, cw, ldb, smem);
  }
}

extern "C" int mla_trsm_llu(mla_handle h, const double* L, int64_t w, int64_t ldl, double* B, int64_t c,
                            int64_t ldb, void* stream) {
  if (!h || w < 0 || c < 0) return MLA_E_INVALID;
  if (w <= 1 || c == 0) return MLA_OK;  // kernels.py:290: nothing to do
  if (ldl < w || ldb < w) return MLA_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  // 192 ... 1024 rows (full LU panels): 128-row steps with inverted diagonal blocks; else 32-row substitution
  const bool blocked = w <= 1024 && trsm_use_inverse((int)w);
  if (blocked) {
    int rc = launch_diag_inv(h, L, w, ldl, h->dinv, s);
    if (rc != MLA_OK) return rc;
  }
  const int smem_bytes = blocked ? GemmUpdateCfg::SMEM_BYTES : TRSM_SMEM_DOUBLES * 8;
  CK(h, cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemBytes));
  int64_t strips = (c + TRSM_CW - 1) / TRSM_CW;
  int grid = (int)(strips < h->num_sms ? strips : h->num_sms);
  k_trsm<<<grid, kThreads, smem_bytes, s>>>(L, (int)w, ldl, B, c, ldb, blocked ? h->dinv : nullptr);
  CK(h, cudaGetLastError());
  return MLA_OK;
}

// ---- laswp -----------------------------------------------------------------------------------------
// Range check of a whole pivot vector (used when it is applied in chunks: NOTHING may be touched if
// ANY index is bad, kernels.py:326-327, so the verdict must exist before the first chunk's plan).
__global__ void k_laswp_validate(const int* ipiv, int64_t npiv, int64_t rows, unsigned* ctrl) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  bool bad = npiv > rows;
  for (int64_t t = threadIdx.x; t < npiv; t += blockDim.x) {
    int p = ipiv[t];
    if (p < 0 || (int64_t)p >= rows) bad = true;
  }
  if (bad) s_bad = 1;
  __syncthreads();
  if (threadIdx.x == 0) ctrl[CW_ERR_INDEX] = s_bad ? 1u : 0u;
}

// Plan of chunk [t0, t0+npiv) of a pivot vector.  prevalidated: a k_laswp_validate verdict is already in
// ctrl[CW_ERR_INDEX] and, if bad, every chunk's plan must come out empty.
__global__ void k_laswp_plan(const int* ipiv, int npiv, int64_t rows, int reverse, int t0, int prevalidated,
                             PivPlan* plan, unsigned* ctrl) {
  __shared__ int top[kMaxPiv], pv[kMaxPiv], keys[2 * kMaxPiv], vals[2 * kMaxPiv];
  if (prevalidated && ctrl[CW_ERR_INDEX] != 0u) {
    if (threadIdx.x == 0) plan->count = 0;
    return;
  }
  bool ok = build_pivot_plan(ipiv, npiv, rows, reverse != 0, plan->ref(), top, keys, vals, 2 * kMaxPiv, pv, t0);
  if (threadIdx.x == 0 && !prevalidated) ctrl[CW_ERR_INDEX] = ok ? 0u : 1u;
}

__global__ void __launch_bounds__(kThreads, 1)
k_laswp_apply(double* A, int64_t cols, int64_t ld, PivPlan* plan) {
  extern __shared__ __align__(16) double smem[];
  // contiguous balanced column shares, like the reference's _share (kernels.py:28-32)
  int64_t per = (cols + gridDim.x - 1) / gridDim.x;
  per = (per + 15) & ~(int64_t)15;
  int64_t lo = blockIdx.x * per, hi = lo + per < cols ? lo + per : cols;
  if (lo >= hi) return;
  laswp_apply_cols(A + lo * ld, ld, (int)(hi - lo), plan->ref(), smem, kLaswpBufDoubles);
}

static int laswp_impl(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
                      int64_t npiv, int reverse, void* stream, bool readback);

extern "C" int mla_laswp(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
                         int64_t npiv, int reverse, void* stream) {
  return laswp_impl(h, A, rows, cols, ld, ipiv, npiv, reverse, stream, true);
}

extern "C" int mla_laswp_async(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
                               int64_t npiv, int reverse, void* stream) {
  return laswp_impl(h, A, rows, cols, ld, ipiv, npiv, reverse, stream, false);
}

static int laswp_impl(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, const int32_t* ipiv,
                      int64_t npiv, int reverse, void* stream, bool readback) {
  if (!h || rows < 0 || cols < 0 || npiv < 0 || (rows > 0 && ld < rows)) return MLA_E_INVALID;
  if (npiv == 0) return MLA_OK;
  if (!ipiv || rows >= (1ll << 31)) return MLA_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  const int smem_bytes = kLaswpBufDoubles * 8;
  CK(h, cudaFuncSetAttribute(k_laswp_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  // Pivot vectors longer than one plan (kMaxPiv) are applied as consecutive chunks of the SAME view
  // (ascending for forward, descending for reverse); the whole vector is range-checked on the device
  // first, and a bad index anywhere empties every chunk's plan, so nothing is touched.
  const int64_t nchunks = (npiv + kMaxPiv - 1) / kMaxPiv;
  const int preval = nchunks > 1 ? 1 : 0;
  if (preval) {
    k_laswp_validate<<<1, 256, 0, s>>>(ipiv, npiv, rows, h->ctrl);
    CK(h, cudaGetLastError());
  }
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int64_t c = reverse ? (nchunks - 1 - ci) : ci;
    const int64_t t0 = c * kMaxPiv;
    const int np = (int)(npiv - t0 < kMaxPiv ? npiv - t0 : kMaxPiv);
    k_laswp_plan<<<1, 32, 0, s>>>(ipiv + t0, np, rows, reverse, (int)t0, preval, h->plan, h->ctrl);
    CK(h, cudaGetLastError());
    if (cols > 0 && rows > 0) {
      int64_t want = (cols + 15) / 16;
      int grid = (int)(want < 2 * h->num_sms ? want : 2 * h->num_sms);
      if (grid < 1) grid = 1;
      k_laswp_apply<<<grid, kThreads, smem_bytes, s>>>(A, cols, ld, h->plan);
      CK(h, cudaGetLastError());
    }
  }
  if (!readback) return MLA_OK;
  CK(h, cudaMemcpyAsync(h->ctrl_host + CW_ERR_INDEX, h->ctrl + CW_ERR_INDEX, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  CK(h, cudaStreamSynchronize(s));
  return h->ctrl_host[CW_ERR_INDEX] != 0u ? MLA_E_INDEX : MLA_OK;
}

// ---- panel (standalone lu_blk_ll) --------------------------------------------------------------------
struct PanelKArgs {
  double* P; int m, w; int64_t ld; int* ipiv; int b_inner;
  const unsigned* stop_flag; int stop_after_polls;
  PanelWs* ws; unsigned* ctrl; mla_lu_info* info;
  int* sing_accum;   // nullable: OR-ed with the panel's singular flag (asynchronous callers)
  unsigned stop_eq;  // 0: the stop flag is "set" when non-zero; else when it equals this tag
  int crout;         // 1: Crout order even when stoppable (stream-ordered drivers: after a cut the leftover
                     //    columns carry the interchanges AND their U rows, like the persistent kernel's panels)
};

__global__ void __launch_bounds__(kThreads, 1) k_panel(PanelKArgs a) {
  extern __shared__ __align__(16) double smem[];
  Team team;
  team.init(blockIdx.x, gridDim.x, a.ctrl + CW_BAR_ALL, a.ctrl + CW_ABORT);
  // Without a stop request nothing can observe the panel half-way, so the U rows are produced in Crout
  // order (no chain of dependent solves per block); a stoppable panel keeps the reference's
  // left-looking order: after a cut the untouched columns carry the interchanges and nothing else
  // (lu.py:177-179, test_lu.py:132-145).
  const bool stoppable = a.stop_flag != nullptr || a.stop_after_polls > 0;
  PanelResult r = panel_ll(team, a.P, a.m, a.w, a.ld, a.ipiv, a.b_inner, a.stop_flag, a.stop_eq, a.stop_after_polls,
                           a.ws, smem, kDynSmemDoubles, !stoppable || a.crout != 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.info->cols_factored = r.cols_factored;
    a.info->singular = r.singular;
    a.info->et_events = (r.cols_factored < a.w) ? 1 : 0;
    a.info->n_panels = 1;
    a.info->ws_joins = 0;
    if (a.sing_accum && r.singular) atomicOr(a.sing_accum, 1);
  }
}

static int check_abort(mla_handle h, cudaStream_t s) {
  if (cudaMemcpyAsync(h->ctrl_host + CW_ABORT, h->ctrl + CW_ABORT, sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return MLA_E_CUDA;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { h->last_cuda = (int)e; return MLA_E_CUDA; }
  if (h->ctrl_host[CW_ABORT] == 0u) return MLA_OK;
  // an aborted panel team leaves its exchange slots / sequence number half-way: start the next one clean
  cudaMemsetAsync(h->panel_ws, 0, sizeof(PanelWs), s);
  return MLA_E_ABORT;
}

extern "C" int mla_panel_ll(mla_handle h, double* P, int64_t m, int64_t w, int64_t ld, int32_t* ipiv, int b_inner,
                            const uint32_t* stop_flag, int stop_after_polls, int team_ctas, mla_lu_info* info,
                            void* stream) {
  if (!h || m < w || w < 0 || b_inner < 1 || (m > 0 && ld < m)) return MLA_E_INVALID;
  if (info) memset(info, 0, sizeof(*info));
  if (w == 0) return MLA_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemBytes));
  int grid = team_ctas;
  if (grid <= 0) {
    int64_t want = (m + 255) / 256;
    grid = (int)(want < 1 ? 1 : want);
  }
  if (grid > h->num_sms) grid = h->num_sms;
  if (grid > kMaxTeam) grid = kMaxTeam;
  CK(h, cudaMemsetAsync(h->ctrl, 0, CW_COUNT * sizeof(unsigned), s));
  PanelKArgs a{P, (int)m, (int)w, ld, ipiv, b_inner, stop_flag, stop_after_polls, h->panel_ws, h->ctrl, h->info_dev,
               nullptr, 0u, 0};
  void* args[] = {&a};
  CK(h, cudaLaunchCooperativeKernel((void*)k_panel, dim3(grid), dim3(kThreads), args, kDynSmemBytes, s));
  CK(h, cudaMemcpyAsync(h->info_host, h->info_dev, sizeof(mla_lu_info), cudaMemcpyDeviceToHost, s));
  int rc = check_abort(h, s);
  if (info) *info = *h->info_host;
  return rc;
}

extern "C" int mla_panel_ll_async(mla_handle h, double* P, int64_t m, int64_t w, int64_t ld, int32_t* ipiv,
                                  int b_inner, int team_ctas, int32_t* singular_accum, const uint32_t* stop_flag,
                                  uint32_t stop_tag, void* stream) {
  if (!h || m < w || w < 0 || b_inner < 1 || (m > 0 && ld < m)) return MLA_E_INVALID;
  if (w == 0) return MLA_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemBytes));
  int grid = team_ctas;
  if (grid <= 0) {
    int64_t want = (m + 255) / 256;
    grid = (int)(want < 1 ? 1 : want);
  }
  if (grid > h->num_sms) grid = h->num_sms;
  if (grid > kMaxTeam) grid = kMaxTeam;
  CK(h, cudaMemsetAsync(h->ctrl, 0, CW_COUNT * sizeof(unsigned), s));
  PanelKArgs a{P, (int)m, (int)w, ld, ipiv, b_inner, stop_flag, 0, h->panel_ws, h->ctrl, h->info_dev, singular_accum,
               stop_tag, 1};
  void* args[] = {&a};
  CK(h, cudaLaunchCooperativeKernel((void*)k_panel, dim3(grid), dim3(kThreads), args, kDynSmemBytes, s));
  return MLA_OK;
}

extern "C" int mla_abort_word(mla_handle h) {
  if (!h) return MLA_E_INVALID;
  unsigned v = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return MLA_E_CUDA;
  if (cudaMemcpy(&v, h->ctrl + CW_ABORT, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return MLA_E_CUDA;
  return (int)(v & 0x7fffffffu);
}

extern "C" int mla_set_update_sms(mla_handle h, int ctas) {
  if (!h || ctas < 0) return MLA_E_INVALID;
  h->update_sms = ctas;
  return MLA_OK;
}

// ---- getrf (persistent kernel) ----------------------------------------------------------------------
static_assert(kDynSmemBytes == kGetrfSmemBytes, "both persistent kernels use the same shared-memory carve-up");
int mla_launch_getrf(const GetrfArgs& a, int grid, int smem_bytes, cudaStream_t s);          // mla_getrf_prod.cu
int mla_launch_getrf_traced(const GetrfArgs& a, int grid, int smem_bytes, cudaStream_t s);   // mla_getrf_traced.cu

// One launch of the persistent kernel: columns [k0, n) of the m-row matrix (k0 > 0: a later window of the phased
// host entry point -- columns [0, k0) are factored and applied, LuState carries on, a raised abort word stays).
static int getrf_launch(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv, int b_outer,
                        int b_inner, int variant, int sm_pf, int q_chunks, mla_lu_info* info_dev,
                        int32_t* widths, int widths_cap, int64_t k0, void* stream, int first_by_all = 0);

extern "C" int mla_getrf_la(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv, int b_outer,
                            int b_inner, int variant, int sm_pf, int q_chunks, mla_lu_info* info_dev,
                            int32_t* widths, int widths_cap, void* stream) {
  return getrf_launch(h, A, m, n, ld, ipiv, b_outer, b_inner, variant, sm_pf, q_chunks, info_dev, widths, widths_cap, 0, stream);
}

static int getrf_launch(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv, int b_outer,
                        int b_inner, int variant, int sm_pf, int q_chunks, mla_lu_info* info_dev,
                        int32_t* widths, int widths_cap, int64_t k0, void* stream, int first_by_all) {
  if (!h || m < n || n < 0 || (m > 0 && ld < m) || k0 < 0 || (k0 > 0 && k0 >= n)) return MLA_E_INVALID;
  if (b_inner < 1 || b_outer < b_inner || b_outer > kMaxPiv) return MLA_E_INVALID;
  if (variant < MLA_VARIANT_LU || variant > MLA_VARIANT_LU_ET) return MLA_E_INVALID;
  if (n > (int64_t)kMaxStrips * TRSM_CW || m >= (1ll << 31)) return MLA_E_INVALID;
  if (variant != MLA_VARIANT_LU && (sm_pf < 1 || sm_pf >= h->num_sms)) return MLA_E_INVALID;  // lu.py:210-214
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (info_dev) CK(h, cudaMemsetAsync(info_dev, 0, sizeof(mla_lu_info), s));
    return MLA_OK;
  }
  int grid = h->num_sms < kMaxTeam ? h->num_sms : kMaxTeam;
  if (k0 == 0) {
    CK(h, cudaMemsetAsync(h->ctrl, 0, CW_COUNT * sizeof(unsigned), s));
    CK(h, cudaMemsetAsync(h->lu_state, 0, sizeof(LuState), s));
    if (h->trace_dev) CK(h, cudaMemsetAsync(h->trace_dev, 0, (size_t)grid * kTraceEvPerCta * sizeof(TraceEv), s));
  } else {
    CK(h, cudaMemsetAsync(h->ctrl + 1, 0, (CW_COUNT - 1) * sizeof(unsigned), s));   // CW_ABORT (word 0) stays
  }
  GetrfArgs a{A, (int)m, (int)n, ld, ipiv, b_outer, b_inner, variant, sm_pf, q_chunks < 1 ? 1 : q_chunks,
              h->sm_pf_max, h->next_progress, h->lu_state, h->plan, h->panel_ws, h->piv_local, h->ctrl, info_dev, widths, widths_cap,
              h->trace_dev, h->dinv, (int)k0, first_by_all};
  h->next_progress = nullptr;
  int e = h->trace_dev ? mla_launch_getrf_traced(a, grid, kDynSmemBytes, s) : mla_launch_getrf(a, grid, kDynSmemBytes, s);
  if (e != 0) { h->last_cuda = e; return MLA_E_CUDA; }
  return MLA_OK;
}

// ---- per-CTA device trace of the persistent kernel (reference trace.py:26-66 Tracer) ---------------------
extern "C" int mla_set_trace(mla_handle h, int enable) {
  if (!h) return MLA_E_INVALID;
  if (!enable) { cudaFree(h->trace_dev); h->trace_dev = nullptr; return MLA_OK; }
  if (h->trace_dev) return MLA_OK;
  int grid = h->num_sms < kMaxTeam ? h->num_sms : kMaxTeam;
  CK(h, cudaMalloc(&h->trace_dev, (size_t)grid * kTraceEvPerCta * sizeof(TraceEv)));
  CK(h, cudaMemset(h->trace_dev, 0, (size_t)grid * kTraceEvPerCta * sizeof(TraceEv)));
  return MLA_OK;
}

extern "C" int mla_getrf_events(mla_handle h, mla_trace_event* out, int max_per_cta) {
  static_assert(sizeof(mla_trace_event) == sizeof(TraceEv), "trace record layout");
  if (!h || !out || max_per_cta < 1) return MLA_E_INVALID;
  if (!h->trace_dev) return 0;
  CK(h, cudaDeviceSynchronize());
  int grid = h->num_sms < kMaxTeam ? h->num_sms : kMaxTeam;
  int per = max_per_cta < kTraceEvPerCta ? max_per_cta : kTraceEvPerCta;
  CK(h, cudaMemcpy2D(out, (size_t)max_per_cta * sizeof(TraceEv), h->trace_dev, (size_t)kTraceEvPerCta * sizeof(TraceEv),
                     (size_t)per * sizeof(TraceEv), grid, cudaMemcpyDeviceToHost));
  return grid;
}

extern "C" int mla_set_panel_sms_max(mla_handle h, int sm_pf_max) {
  if (!h || sm_pf_max < 0) return MLA_E_INVALID;
  h->sm_pf_max = sm_pf_max;
  return MLA_OK;
}

extern "C" int mla_getrf_la_sync(mla_handle h, double* A, int64_t m, int64_t n, int64_t ld, int32_t* ipiv,
                                 int b_outer, int b_inner, int variant, int sm_pf, int q_chunks,
                                 mla_lu_info* info_host, int32_t* widths_host, int widths_cap, void* stream) {
  if (!h) return MLA_E_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  int cap = widths_cap < kWidthsCap ? widths_cap : kWidthsCap;
  if (!widths_host) cap = 0;
  int rc = mla_getrf_la(h, A, m, n, ld, ipiv, b_outer, b_inner, variant, sm_pf, q_chunks, h->info_dev,
                        cap > 0 ? h->widths_dev : nullptr, cap, s);
  if (rc != MLA_OK) return rc;
  if (n == 0) { if (info_host) memset(info_host, 0, sizeof(*info_host)); return MLA_OK; }
  CK(h, cudaMemcpyAsync(h->info_host, h->info_dev, sizeof(mla_lu_info), cudaMemcpyDeviceToHost, s));
  rc = check_abort(h, s);
  if (info_host) *info_host = *h->info_host;
  if (rc == MLA_OK && cap > 0) {
    int np = h->info_host->n_panels < cap ? h->info_host->n_panels : cap;
    CK(h, cudaMemcpy(widths_host, h->widths_dev, np * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  return rc;
}

extern "C" int mla_release_host_cache(mla_handle h) {
  if (!h) return MLA_E_INVALID;
  cudaFree(h->a_dev); h->a_dev = nullptr; h->a_dev_bytes = 0;
  cudaFree(h->ipiv_dev); h->ipiv_dev = nullptr; h->ipiv_dev_n = 0;
  return MLA_OK;
}

static int catch_up(mla_handle h, double* A, int64_t m, int64_t ld, const int32_t* ipiv, int64_t k, int64_t c0,
                    int64_t c1, int b_outer, int64_t deep_block, cudaStream_t s);

extern "C" int mla_set_host_phases(mla_handle h, const int64_t* bounds, int count, int deep) {
  if (!h || count > kMaxHostPhases - 1 || (count > 0 && !bounds)) return MLA_E_INVALID;
  for (int i = 0; i < count; ++i)
    if (bounds[i] <= (i ? bounds[i - 1] : 0)) return MLA_E_INVALID;
  h->phase_count = count < 0 ? -1 : count;
  for (int i = 0; i < count; ++i) h->phase_bounds[i] = bounds[i];
  h->phase_deep = deep < 0 ? 0 : deep;
  return MLA_OK;
}

// Window boundaries of the phased entry point: out[0] < out[1] < ... < out[np-1] == n.  Default policy: windows
// end at n/32, n/8 and 3n/8 (whole multiples of b_outer), so the first one waits for 3 % of the upload only and
// every later one finds its columns uploaded when the window before it is done (measured at n = 32768, 52 GB/s:
// the third window ends 226 ms after the start, the upload 163 ms; more or later cuts only add panel-bound
// tall-and-skinny windows, tools/dev_host_phases.py).
static int host_phase_bounds(mla_handle h, int64_t n, int b_outer, int64_t* out) {
  int np = 0;
  if (h->phase_count > 0) {
    for (int i = 0; i < h->phase_count; ++i) {
      int64_t c = h->phase_bounds[i] / b_outer * b_outer;
      if (c > (np ? out[np - 1] : 0) && c < n) out[np++] = c;
    }
  } else if (h->phase_count < 0 && n >= 8192) {
    const int64_t num[3] = {1, 4, 12};
    for (int i = 0; i < 3; ++i) {
      int64_t c = (n * num[i] / 32) / b_outer * b_outer;
      if (c > (np ? out[np - 1] : 0) && c < n) out[np++] = c;
    }
  }
  out[np++] = n;
  return np;
}

static int getrf_la_host_impl(mla_handle h, double* A_host, int64_t m, int64_t n, int64_t ld_host,
                              int32_t* ipiv_host, int b_outer, int b_inner, int variant, int sm_pf,
                              int q_chunks, mla_lu_info* info_host);

extern "C" int mla_getrf_la_host(mla_handle h, double* A_host, int64_t m, int64_t n, int64_t ld_host,
                                 int32_t* ipiv_host, int b_outer, int b_inner, int variant, int sm_pf,
                                 int q_chunks, mla_lu_info* info_host) {
  int rc = getrf_la_host_impl(h, A_host, m, n, ld_host, ipiv_host, b_outer, b_inner, variant, sm_pf, q_chunks, info_host);
  if (rc != MLA_OK && h) {
    // whatever failed: no copy engine or kernel may still touch the caller's buffers after the return
    cudaStreamSynchronize(h->s_up);
    cudaStreamSynchronize(h->s_main);
    cudaStreamSynchronize(h->s_copy);
    h->next_progress = nullptr;
  }
  return rc;
}

static int getrf_la_host_impl(mla_handle h, double* A_host, int64_t m, int64_t n, int64_t ld_host,
                              int32_t* ipiv_host, int b_outer, int b_inner, int variant, int sm_pf,
                              int q_chunks, mla_lu_info* info_host) {
  if (!h || m < n || n < 0 || (m > 0 && ld_host < m)) return MLA_E_INVALID;
  if (b_inner < 1 || b_outer < b_inner || b_outer > kMaxPiv) return MLA_E_INVALID;
  if (n == 0) { if (info_host) memset(info_host, 0, sizeof(*info_host)); return MLA_OK; }
  const int64_t ld = (m + 1) & ~(int64_t)1;   // even leading dimension: 16-byte aligned columns
  size_t bytes = (size_t)ld * (size_t)n * sizeof(double);
  if (h->a_dev_bytes < bytes) {
    cudaFree(h->a_dev); h->a_dev = nullptr; h->a_dev_bytes = 0;
    CK(h, cudaMalloc(&h->a_dev, bytes));
    h->a_dev_bytes = bytes;
  }
  if (h->ipiv_dev_n < (size_t)n) {
    cudaFree(h->ipiv_dev); h->ipiv_dev = nullptr; h->ipiv_dev_n = 0;
    CK(h, cudaMalloc(&h->ipiv_dev, (size_t)n * sizeof(int32_t)));
    h->ipiv_dev_n = (size_t)n;
  }
  // Upload, factor and download at the same time.
  //  * Upload || factor: the columns travel in chunks on their own stream, and the factorization runs window by
  //    window behind them (left-looking between windows): window [c0, c1) waits for its chunk only, is brought
  //    up to date with the columns [0, c0) factored so far (catch_up: every interchange, then per 512-column
  //    block a solve and a rank-512 update -- with deep == 0 exactly the operations an unwindowed run applies to
  //    these columns, in the same order per entry, so the factors are the same bit for bit; by default most of
  //    the update runs as multiplies of depth 4096) and is then factored by the persistent kernel restricted to
  //    it (look-ahead, WS and ET inside the window).  The last window takes everything left.
  //  * Factor || download: once an outer iteration of the LAST window has started with its panel at row q0,
  //    rows [0, q0) of the whole matrix are final (later interchanges, solves and updates only touch rows
  //    >= q0), so they are copied to the host as row blocks on a second stream.  The kernel reports q0 through
  //    a mapped host word.
  cudaStream_t s = h->s_main;
  *((volatile int*)h->progress_host) = 0;
  int64_t bounds[kMaxHostPhases];
  const int np = host_phase_bounds(h, n, b_outer, bounds);
  // Pinned host memory: all chunk copies are queued at once (they run back to back on the copy engine whatever
  // the calling thread does afterwards).  Pageable host memory: a copy blocks the calling thread while it is
  // staged, so each chunk's copy is issued right in front of its window's work -- the windows before it are then
  // already running on the device.
  bool pinned = false;
  {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, A_host) == cudaSuccess) pinned = (pa.type == cudaMemoryTypeHost);
    else cudaGetLastError();
    if (getenv("MLA_UPLOAD_INTERLEAVED")) pinned = false;   // development: force the pageable order
  }
  auto upload_chunk = [&](int g) -> int {
    const int64_t c0 = g ? bounds[g - 1] : 0, c1 = bounds[g];
    CK(h, cudaMemcpy2DAsync(h->a_dev + c0 * ld, ld * sizeof(double), A_host + c0 * ld_host, ld_host * sizeof(double),
                            m * sizeof(double), c1 - c0, cudaMemcpyHostToDevice, h->s_up));
    CK(h, cudaEventRecord(h->ev_up[g], h->s_up));
    return MLA_OK;
  };
  // MLA_HOST_TIMELINE=1 (development): device stamps at every window's catch-up start / kernel start / kernel
  // end, printed to stderr after the call
  const bool timeline = getenv("MLA_HOST_TIMELINE") != nullptr;
  cudaEvent_t tl[3 * kMaxHostPhases + 1];
  if (timeline) {
    for (int i = 0; i < 3 * np + 1; ++i) cudaEventCreate(&tl[i]);
    cudaEventRecord(tl[3 * np], s);
  }
  for (int g = 0; g < np; ++g) {
    const int64_t c0 = g ? bounds[g - 1] : 0, c1 = bounds[g];
    int rc = MLA_OK;
    if (!pinned) rc = upload_chunk(g);
    else if (g == 0) for (int u = 0; u < np && rc == MLA_OK; ++u) rc = upload_chunk(u);
    if (rc != MLA_OK) return rc;
    CK(h, cudaStreamWaitEvent(s, h->ev_up[g], 0));
    if (timeline) cudaEventRecord(tl[3 * g], s);
    if (c0 > 0) rc = catch_up(h, h->a_dev, m, ld, h->ipiv_dev, c0, c0, c1, b_outer, h->phase_deep, s);
    if (rc != MLA_OK) return rc;
    if (timeline) cudaEventRecord(tl[3 * g + 1], s);
    h->next_progress = (g == np - 1) ? h->progress_dev : nullptr;
    rc = getrf_launch(h, h->a_dev, m, c1, ld, h->ipiv_dev, b_outer, b_inner, variant, sm_pf, q_chunks, h->info_dev,
                      nullptr, 0, c0, s, h->phase_deep > 0 ? 1 : 0);
    h->next_progress = nullptr;
    if (rc != MLA_OK) return rc;
    if (timeline) cudaEventRecord(tl[3 * g + 2], s);
  }
  CK(h, cudaEventRecord(h->ev_done, s));
  const int64_t min_rows = 512;   // row blocks of 128 ... 2048 rows were measured: no difference beyond noise
  int64_t done_rows = 0;
  while (true) {
    cudaError_t q = cudaEventQuery(h->ev_done);
    if (q != cudaSuccess && q != cudaErrorNotReady) { h->last_cuda = (int)q; return MLA_E_CUDA; }
    const bool finished = (q == cudaSuccess);
    int64_t ready = finished ? m : (int64_t)*((volatile int*)h->progress_host);
    if (ready > m) ready = m;
    if (ready - done_rows >= min_rows || (finished && ready > done_rows)) {
      CK(h, cudaMemcpy2DAsync(A_host + done_rows, ld_host * sizeof(double), h->a_dev + done_rows, ld * sizeof(double),
                              (size_t)(ready - done_rows) * sizeof(double), n, cudaMemcpyDeviceToHost, h->s_copy));
      done_rows = ready;
    } else if (!finished) {
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    if (finished && done_rows >= m) break;
  }
  CK(h, cudaMemcpyAsync(ipiv_host, h->ipiv_dev, n * sizeof(int32_t), cudaMemcpyDeviceToHost, h->s_copy));
  CK(h, cudaMemcpyAsync(h->info_host, h->info_dev, sizeof(mla_lu_info), cudaMemcpyDeviceToHost, h->s_copy));
  CK(h, cudaStreamSynchronize(h->s_copy));
  int rc = check_abort(h, s);
  if (info_host) *info_host = *h->info_host;
  if (timeline) {
    for (int g = 0; g < np; ++g) {
      float t0 = 0, t1 = 0, t2 = 0;
      cudaEventElapsedTime(&t0, tl[3 * np], tl[3 * g]);
      cudaEventElapsedTime(&t1, tl[3 * np], tl[3 * g + 1]);
      cudaEventElapsedTime(&t2, tl[3 * np], tl[3 * g + 2]);
      fprintf(stderr, "[mla host timeline] window %d [%lld, %lld): chunk ready %.1f ms, catch-up done %.1f (%.1f), kernel done %.1f (%.1f)\n",
              g, (long long)(g ? bounds[g - 1] : 0), (long long)bounds[g], t0, t1, t1 - t0, t2, t2 - t1);
    }
    for (int i = 0; i < 3 * np + 1; ++i) cudaEventDestroy(tl[i]);
  }
  return rc;
}

// ---- apply one factored panel to a block of columns (multi-GPU update step) ------------------------
// The per-iteration update of the 1-D block-cyclic driver (distributed.py) as ONE persistent launch:
//   T (rows x cols, the owned columns right of the panel, view starting at the panel's first row)
//   P (rows x w, the broadcast panel: unit-lower L11 on top of L21), ipiv (w panel-local pivots)
//   T := interchanges(T);  T[0:w] := trilu(L11)^-1 T[0:w];  T[w:] -= L21 @ T[0:w]
// i.e. laswp -> trsm_llu -> gemm_malleable of lu.py:251-253, 280-281 / 289, 306-308, with the same
// work-queue structure as the single-GPU kernel: PREP strips first, GEMM tiles (row-block-major,
// chained) wait on their strip's release/acquire flag.  The plan comes from k_laswp_plan.
struct ApplyArgs {
  const double* P; int64_t ldp; int rows, w;
  double* T; int64_t ldt; int cols;
  int skip_cols;            // leading columns of T that already carry the interchanges and their U rows
  double* L; int64_t ldl; int left_cols;   // columns LEFT of the panel (interchanges only; nullable)
  PivPlan* plan; unsigned* ctrl; unsigned* flags; unsigned tag;
  const DiagInv* inv;       // inverted diagonal blocks of the panel's unit-lower top block (mla_apply_panel_prepare)
  // catch-up steps of the phased host entry point (left-looking: every interchange was applied up front):
  int no_swaps;             // 1: the strips skip the interchanges (no plan is read)
  int gemm_rows;            // the rank-w update stops at this row of the view (== rows: the whole height)
};

__global__ void __launch_bounds__(kThreads, 1) k_apply_panel(ApplyArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int nstrips = (a.cols + TRSM_CW - 1) / TRSM_CW;
  const int nleft = (a.left_cols + LEFT_CW - 1) / LEFT_CW;
  const int rows_below = a.gemm_rows - a.w;
  const int tmc = (rows_below + GemmUpdateCfg::BM - 1) / GemmUpdateCfg::BM;
  const int first_gemm = nstrips + nleft;
  const int total = first_gemm + nstrips * tmc;
  unsigned* next = a.ctrl + CW_QUEUE_NEXT;
  auto decode = [&](int t, int& strip, int& tm) {   // GEMM items, row-block-major (see gemm_tile_desc)
    const int g = t - first_gemm;
    const int per_block = kRowBlockTiles * nstrips;
    const int rb = g / per_block;
    const int rows_here = imin(kRowBlockTiles, tmc - rb * kRowBlockTiles);
    const int r = g - rb * per_block;
    strip = r / rows_here;
    tm = rb * kRowBlockTiles + (r - strip * rows_here);
  };
  auto desc = [&](int strip, int tm) {
    const int c0 = strip * TRSM_CW, i0 = a.w + tm * GemmUpdateCfg::BM;
    double* c = a.T + (int64_t)c0 * a.ldt + i0;
    return TileDesc{a.P + i0, a.ldp, a.T + (int64_t)c0 * a.ldt, a.ldt, c, a.ldt, c, a.ldt,
                    a.w, a.gemm_rows - i0, imin(TRSM_CW, a.cols - c0), 1.0, -1.0, true};
  };
  // a pivot index out of range (k_laswp_plan's verdict): nothing may be touched, and the caller must
  // hear about it -- the abort word is what the asynchronous entry points report (mla_abort_word)
  if (!a.no_swaps && *((volatile unsigned*)(a.ctrl + CW_ERR_INDEX)) != 0u) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(a.ctrl + CW_ABORT, 0xBAD1u);
    return;
  }
  int base = 0, ready_strip = -1, executed = 0;
  bool primed = false;
  __shared__ StripCache s_cache;     // strip flags this CTA has already seen set (one L2 trip per strip, not per tile)
  s_cache.clear();
  int t = pop_item(next);
  int tn = -1;                       // item popped ahead (-1: none)
  auto advance = [&]() { if (tn >= 0) { t = tn; tn = -1; } else t = pop_item(next); };
  while (t < total) {
    ++executed;
    if (t < nstrips) {
      // PREP of strip t: interchanges + solve with the panel's unit-lower top block (lu.py:251-253, 280);
      // columns below skip_cols are the leftover of an ET-cut panel and already hold both
      const int c0 = t * TRSM_CW, c1 = imin(a.cols, c0 + TRSM_CW), lo = imax(c0, a.skip_cols);
      if (lo < c1) {
        if (!a.no_swaps) laswp_apply_cols(a.T + (int64_t)lo * a.ldt, a.ldt, c1 - lo, a.plan->ref(), smem, kLaswpBufDoubles);
        if (trsm_use_inverse(a.w)) trsm_strip_inv(a.P, a.w, a.ldp, a.T + (int64_t)lo * a.ldt, c1 - lo, a.ldt, a.inv, smem);
        else trsm_strip_ool(a.P, a.w, a.ldp, a.T + (int64_t)lo * a.ldt, c1 - lo, a.ldt, smem);
      }
      __syncthreads();
      if (threadIdx.x == 0) { __threadfence(); st_release(&a.flags[t], a.tag); }
      primed = false;
      advance();
      continue;
    }
    if (t < first_gemm) {
      // LEFT: the panel's interchanges for the owned columns to its left (lu.py:252, 329-332)
      const int c0 = (t - nstrips) * LEFT_CW;
      laswp_apply_cols(a.L + (int64_t)c0 * a.ldl, a.ldl, imin(LEFT_CW, a.left_cols - c0), a.plan->ref(), smem,
                       kLaswpBufDoubles);
      primed = false;
      advance();
      continue;
    }
    int strip, tm;
    decode(t, strip, tm);
    TileDesc cur = desc(strip, tm);
    if (!primed) {
      if (strip != ready_strip && !s_cache.has(strip)) {
        if (!wait_flag_eq(&a.flags[strip], a.tag, a.ctrl + CW_ABORT)) return;
        if (threadIdx.x == 0) s_cache.bits[strip >> 5] |= 1u << (strip & 31);   // read again only behind the next barrier
      }
      ready_strip = strip;
      base = 0;
      tile_prologue<GemmUpdateCfg>(cur, base, smem);
    }
    if (tn < 0) tn = pop_item(next);
    TileDesc nxt{};
    nxt.valid = false;
    if (tn < total && tn >= first_gemm && tile_kt<GemmUpdateCfg>(cur) >= GemmUpdateCfg::STAGES - 1) {
      int s2, m2;
      decode(tn, s2, m2);
      if (s2 == ready_strip || flag_ready_cached(s_cache, a.flags, s2, a.tag)) { ready_strip = s2; nxt = desc(s2, m2); }
    }
    base = tile_run<GemmUpdateCfg>(cur, nxt, base, smem);
    primed = nxt.valid;
    t = tn;
    tn = -1;
  }
  // Completion, once per CTA (all launches of the step count into the same word): the CTA whose report
  // completes the queue publishes the step's tag -- the distributed driver's ru_done (lu.py:309-310),
  // polled by the look-ahead panel running beside this kernel.
  bulk_wait_all();
  __syncthreads();
  if (threadIdx.x == 0 && executed > 0) {
    __threadfence();
    unsigned old = atom_add_release(a.ctrl + CW_QUEUE_DONE, (unsigned)executed);
    if (old + (unsigned)executed == (unsigned)total) st_release(a.ctrl + CW_STEP_DONE, a.tag);
  }
}

// prepare: interchange plan, empty queue, fresh flag tag.  launch: `ctas` CTAs (0 = update_sms / all) that
// drain the prepared queue; a second launch of the same step (other stream) joins the same queue -- the
// distributed driver's worker sharing: the SMs that factored the next panel join the update when done.
extern "C" int mla_apply_panel_prepare(mla_handle h, const double* P, int64_t ldp, const int32_t* ipiv, int64_t w,
                                       int64_t rows, void* stream) {
  if (!h || !P || rows < w || w < 0 || w > kMaxPiv || ldp < rows) return MLA_E_INVALID;
  if (w == 0) return MLA_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (trsm_use_inverse((int)w)) { int rc = launch_diag_inv(h, P, w, ldp, h->dinv, s); if (rc != MLA_OK) return rc; }
  k_laswp_plan<<<1, 32, 0, s>>>(ipiv, (int)w, rows, 0, 0, 0, h->plan, h->ctrl);
  CK(h, cudaGetLastError());
  CK(h, cudaMemsetAsync(h->ctrl + CW_QUEUE_NEXT, 0, sizeof(unsigned), s));
  CK(h, cudaMemsetAsync(h->ctrl + CW_QUEUE_DONE, 0, sizeof(unsigned), s));
  ++h->apply_tag;
  return MLA_OK;
}

extern "C" int mla_apply_panel_launch(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ldp, double* T,
                                      int64_t cols, int64_t ldt, int64_t skip_cols, double* L, int64_t left_cols,
                                      int64_t ldl, int ctas, void* stream) {
  if (!h || rows < w || w < 0 || cols < 0 || ctas < 0 || skip_cols < 0 || left_cols < 0) return MLA_E_INVALID;
  if (rows > 0 && (ldp < rows || (cols > 0 && ldt < rows) || (left_cols > 0 && (ldl < rows || !L)))) return MLA_E_INVALID;
  if (w > kMaxPiv || cols > (int64_t)kMaxStrips * TRSM_CW || left_cols >= (1ll << 31)) return MLA_E_INVALID;
  if (w == 0 || (cols == 0 && left_cols == 0)) return MLA_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CK(h, cudaFuncSetAttribute(k_apply_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemBytes));
  ApplyArgs a{P, ldp, (int)rows, (int)w, T, ldt, (int)cols, (int)(skip_cols < cols ? skip_cols : cols), L, ldl,
              (int)left_cols, h->plan, h->ctrl, h->lu_state->rprep_done, h->apply_tag, h->dinv, 0, (int)rows};
  void* args[] = {&a};
  int grid = h->num_sms < kMaxTeam ? h->num_sms : kMaxTeam;
  if (h->update_sms > 0 && h->update_sms < grid) grid = h->update_sms;
  if (ctas > 0 && ctas < grid) grid = ctas;
  CK(h, cudaLaunchCooperativeKernel((void*)k_apply_panel, dim3(grid), dim3(kThreads), args, kDynSmemBytes, s));
  return MLA_OK;
}

extern "C" int mla_apply_panel(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ldp, double* T,
                               int64_t cols, int64_t ldt, const int32_t* ipiv, void* stream) {
  if (!h || rows < w || w < 0 || cols < 0 || (rows > 0 && (ldp < rows || ldt < rows))) return MLA_E_INVALID;
  if (w > kMaxPiv || cols > (int64_t)kMaxStrips * TRSM_CW) return MLA_E_INVALID;
  if (w == 0 || cols == 0) return MLA_OK;
  int rc = mla_apply_panel_prepare(h, P, ldp, ipiv, w, rows, stream);
  if (rc != MLA_OK) return rc;
  return mla_apply_panel_launch(h, P, rows, w, ldp, T, cols, ldt, 0, nullptr, 0, 0, 0, stream);
}

// Left-looking catch-up of the phased host entry point: columns [c0, c1) of the m-row matrix A have seen nothing
// of the factorization so far; columns [0, k), k <= c0, are factored (unit-lower L below / U above the diagonal,
// global pivots in ipiv).  All k interchanges first (the L rows are already in their final order, so the new
// columns must be brought into it before any row of L meets them), then per b_outer-column block [p0, p0 + w)
// the solve with its unit-lower diagonal block and the rank-w update of the rows below -- one k_apply_panel
// launch each, without interchanges.
// deep_block > 0: the factored columns are taken in super-blocks of deep_block columns; inside a super-block the
// rank-w updates stop at the super-block's last row, and the rows below it get ONE multiply of depth deep_block
// per super-block (C is then read and written once per super-block instead of once per b_outer block, and most
// of the work runs as a few long multiplies at 34-35 TFLOP/s instead of many short launches that each start with
// a latency-bound solve).  Same result up to rounding; no longer bit-identical to an unwindowed run.
static int catch_up(mla_handle h, double* A, int64_t m, int64_t ld, const int32_t* ipiv, int64_t k, int64_t c0,
                    int64_t c1, int b_outer, int64_t deep_block, cudaStream_t s) {
  if (k <= 0 || c1 <= c0) return MLA_OK;
  int rc = laswp_impl(h, A + c0 * ld, m, c1 - c0, ld, ipiv, k, 0, (void*)s, false);
  if (rc != MLA_OK) return rc;
  CK(h, cudaFuncSetAttribute(k_apply_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemBytes));
  const int grid = h->num_sms < kMaxTeam ? h->num_sms : kMaxTeam;
  const int64_t sb = deep_block > 0 ? (deep_block + b_outer - 1) / b_outer * b_outer : k;
  for (int64_t s0 = 0; s0 < k; s0 += sb) {
    const int64_t s1 = s0 + sb < k ? s0 + sb : k;            // super-block [s0, s1)
    const bool deep = deep_block > 0 && m > s1;
    for (int64_t p0 = s0; p0 < s1; p0 += b_outer) {
      const int64_t w = s1 - p0 < b_outer ? s1 - p0 : b_outer;
      const double* P = A + p0 * ld + p0;
      const int64_t rows = m - p0;
      if (trsm_use_inverse((int)w)) { rc = launch_diag_inv(h, P, w, ld, h->dinv, s); if (rc != MLA_OK) return rc; }
      CK(h, cudaMemsetAsync(h->ctrl + CW_QUEUE_NEXT, 0, sizeof(unsigned), s));
      CK(h, cudaMemsetAsync(h->ctrl + CW_QUEUE_DONE, 0, sizeof(unsigned), s));
      ++h->apply_tag;
      ApplyArgs a{P, ld, (int)rows, (int)w, A + c0 * ld + p0, ld, (int)(c1 - c0), 0, nullptr, 0, 0, h->plan, h->ctrl,
                  h->lu_state->rprep_done, h->apply_tag, h->dinv, 1, (int)(deep ? s1 - p0 : rows)};
      void* args[] = {&a};
      CK(h, cudaLaunchCooperativeKernel((void*)k_apply_panel, dim3(grid), dim3(kThreads), args, kDynSmemBytes, s));
    }
    if (deep) {
      rc = mla_gemm(h, A + c0 * ld + s1, m - s1, c1 - c0, ld, A + s0 * ld + s1, ld, A + c0 * ld + s0, ld, s1 - s0, 1.0, -1.0,
                    nullptr, 0, (void*)s);
      if (rc != MLA_OK) return rc;
    }
  }
  return MLA_OK;
}

extern "C" int mla_step_flag(mla_handle h, uint32_t** flag_dev, uint32_t* tag) {
  if (!h) return MLA_E_INVALID;
  if (flag_dev) *flag_dev = h->ctrl + CW_STEP_DONE;
  if (tag) *tag = h->apply_tag;
  return MLA_OK;
}

// ---- pack one factored panel for the broadcast (multi-GPU driver) ---------------------------------------
// out: [4 x int32 header: factored width, singular, scheduled width, rows][w x int32 panel-local pivots, padded
// to a multiple of 4][rows x w doubles, column-major, leading dimension rows].  The factored width and the
// singular flag come from the info record the panel kernel of THIS handle left on the device, so the
// whole chain panel -> pack -> broadcast is stream-ordered.
__global__ void k_pack_panel(const double* __restrict__ P, int64_t ld, int64_t rows, int w, const int* __restrict__ ipiv,
                             const mla_lu_info* info, int* out_i32, double* out_panel) {
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      out_i32[0] = info ? info->cols_factored : w;
      out_i32[1] = info ? info->singular : 0;
      out_i32[2] = w;
      out_i32[3] = (int)rows;
    }
    for (int t = threadIdx.x; t < w; t += blockDim.x) out_i32[4 + t] = ipiv[t];
  }
  const int64_t half = rows >> 1;        // 16-byte moves when both sides are aligned
  const bool vec = ((ld & 1) == 0) && ((rows & 1) == 0) && ((((uintptr_t)P | (uintptr_t)out_panel) & 15) == 0);
  for (int c = blockIdx.y; c < w; c += gridDim.y) {
    const double* src = P + (int64_t)c * ld;
    double* dst = out_panel + (int64_t)c * rows;
    if (vec) {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < half; i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<double2*>(dst)[i] = reinterpret_cast<const double2*>(src)[i];
    } else {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    }
  }
}

extern "C" int64_t mla_packed_panel_doubles(int64_t rows, int64_t w) {
  if (rows < 0 || w < 0) return MLA_E_INVALID;
  const int64_t ints = 4 + ((w + 3) & ~(int64_t)3);
  return ints / 2 + rows * w;
}

extern "C" int mla_pack_panel(mla_handle h, const double* P, int64_t rows, int64_t w, int64_t ld, const int32_t* ipiv,
                              int use_panel_info, double* out, void* stream) {
  if (!h || !P || !ipiv || !out || rows < w || w < 1 || w > kMaxPiv || ld < rows) return MLA_E_INVALID;
  const int64_t ints = 4 + ((w + 3) & ~(int64_t)3);
  dim3 grid((unsigned)((rows / 2 + 255) / 256 > 16 ? 16 : ((rows / 2 + 255) / 256 < 1 ? 1 : (rows / 2 + 255) / 256)),
            (unsigned)(w > 512 ? 512 : w));
  k_pack_panel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, ld, rows, (int)w, ipiv, use_panel_info ? h->info_dev : nullptr,
                                                       reinterpret_cast<int*>(out), out + ints / 2);
  CK(h, cudaGetLastError());
  return MLA_OK;
}

// ---- fill_random -----------------------------------------------------------------------------------
// matrix.py:47-59: draw k = i + j*total_rows (0-based) of the stream uses state seed + (k+1)*gamma.
__global__ void k_fill_random(double* A, int64_t rows, int64_t cols, int64_t ld, unsigned long long seed,
                              int64_t col0, int64_t total_rows, double scale, double shift,
                              const double* row_scale) {
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
      unsigned long long k = (unsigned long long)(i + (j + col0) * total_rows);
      unsigned long long z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z = z ^ (z >> 31);
      double u = __ddiv_rn((double)(z >> 11) + 1.0, 9007199254740994.0);
      double v = __dadd_rn(__dmul_rn(scale, u), shift);   // no FMA: matches the host's two roundings
      if (row_scale) v = __dmul_rn(v, row_scale[i]);
      A[i + j * ld] = v;
    }
}

extern "C" int mla_fill_random(mla_handle h, double* A, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                               int64_t col0, int64_t total_rows, double scale, double shift,
                               const double* row_scale, void* stream) {
  if (!h || rows < 0 || cols < 0 || (rows > 0 && ld < rows)) return MLA_E_INVALID;
  if (rows == 0 || cols == 0) return MLA_OK;
  if (total_rows <= 0) total_rows = rows;
  dim3 grid((unsigned)((rows + 255) / 256 > 256 ? 256 : (rows + 255) / 256), (unsigned)(cols > 4096 ? 4096 : cols));
  k_fill_random<<<grid, 256, 0, (cudaStream_t)stream>>>(A, rows, cols, ld, (unsigned long long)seed, col0, total_rows,
                                                        scale, shift, row_scale);
  CK(h, cudaGetLastError());
  return MLA_OK;
}

// ---- profiling counters of the panel team (ns, rank 0): see PanelWs::prof ---------------------------
extern "C" int mla_panel_profile(mla_handle h, uint64_t* out16, int reset) {
  if (!h || !out16) return MLA_E_INVALID;
  CK(h, cudaDeviceSynchronize());
  CK(h, cudaMemcpy(out16, h->panel_ws->prof, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (reset) CK(h, cudaMemset(h->panel_ws->prof, 0, 16 * sizeof(uint64_t)));
  return MLA_OK;
}

// ---- device trace of the last mla_getrf_la call: rows of 5 uint64 (see LuState::trace) ---------------
extern "C" int mla_getrf_trace(mla_handle h, uint64_t* out, int max_rows) {
  if (!h || !out || max_rows < 0) return MLA_E_INVALID;
  CK(h, cudaDeviceSynchronize());
  int rows = max_rows < kTraceCap ? max_rows : kTraceCap;
  CK(h, cudaMemcpy(out, h->lu_state->trace, (size_t)rows * 5 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return rows;
}

extern "C" int mla_getrf_debug(mla_handle h, uint64_t* out8) {
  if (!h || !out8) return MLA_E_INVALID;
  CK(h, cudaDeviceSynchronize());
#ifdef MLA_TILE_PROF
  // instrumented build (tools/README.md): per-tile clock accounting of CTA 0 instead
  CK(h, cudaMemcpyFromSymbol(out8, g_tprof, 8 * sizeof(uint64_t)));
  unsigned long long zero[8] = {0};
  CK(h, cudaMemcpyToSymbol(g_tprof, zero, sizeof(zero)));
  return MLA_OK;
#endif
  CK(h, cudaMemcpy(out8, h->lu_state->dbg, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return MLA_OK;
}
