// libmla_b200.so -- C ABI (include/mla_b200.h) over the hand-written sm_100a kernels of the
// blocked LU hot path.  Build: see paper_1611_06365_b200/build.py
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/mla_b200.h"
#include "mla_common.cuh"
#include "mla_gemm.cuh"

using namespace mla;

// ---- control block layout (device words) --------------------------------------------------------
enum CtrlWord {
  CW_ABORT = 0,
  CW_QUEUE_NEXT = 1,
  CW_BAR_ALL = 2,
  CW_BAR_PF = 3,
  CW_ERR_INDEX = 4,
  CW_COUNT = 64
};

struct mla_handle_s {
  int device;
  int num_sms;
  int last_cuda;
  unsigned* ctrl;        // CW_COUNT words (device)
  unsigned* ctrl_host;   // pinned mirror
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
  *out = h;
  return MLA_OK;
}

extern "C" int mla_destroy(mla_handle h) {
  if (!h) return MLA_E_INVALID;
  cudaFree(h->ctrl);
  cudaFreeHost(h->ctrl_host);
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
  while (true) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ctrl + CW_QUEUE_NEXT, 1u);
    __syncthreads();
    const int t = s_tile;
    __syncthreads();
    if (t >= ntiles) break;
    gemm_run_tile<GemmUpdateCfg>(p, t, smem);
  }
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

// ---- TEMPORARY STUBS (replaced as kernels land) ----
extern "C" int mla_trsm_llu(mla_handle, const double*, int64_t, int64_t, double*, int64_t, int64_t, void*) { return MLA_E_INVALID; }
extern "C" int mla_laswp(mla_handle, double*, int64_t, int64_t, int64_t, const int32_t*, int64_t, int, void*) { return MLA_E_INVALID; }
extern "C" int mla_panel_ll(mla_handle, double*, int64_t, int64_t, int64_t, int32_t*, int, const uint32_t*, int, int, mla_lu_info*, void*) { return MLA_E_INVALID; }
extern "C" int mla_getrf_la(mla_handle, double*, int64_t, int64_t, int64_t, int32_t*, int, int, int, int, int, mla_lu_info*, int32_t*, int, void*) { return MLA_E_INVALID; }
extern "C" int mla_getrf_la_sync(mla_handle, double*, int64_t, int64_t, int64_t, int32_t*, int, int, int, int, int, mla_lu_info*, int32_t*, int, void*) { return MLA_E_INVALID; }
extern "C" int mla_getrf_la_host(mla_handle, double*, int64_t, int64_t, int64_t, int32_t*, int, int, int, int, int, mla_lu_info*) { return MLA_E_INVALID; }
extern "C" int mla_fill_random(mla_handle, double*, int64_t, int64_t, int64_t, uint64_t, int64_t, int64_t, double, double, const double*, void*) { return MLA_E_INVALID; }
extern "C" int mla_residual_lu(mla_handle, double*, const double*, int64_t, int64_t, int64_t, int64_t, const int32_t*, double*, void*) { return MLA_E_INVALID; }
