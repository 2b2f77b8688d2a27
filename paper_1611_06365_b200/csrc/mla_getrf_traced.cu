// The instrumented twin of the persistent LU kernel: the same getrf_persistent body with per-CTA event
// records (mla_set_trace / mla_getrf_events, include/mla_b200.h).  It lives in its own translation unit so
// that the production kernel's code generation cannot depend on it and both compile in parallel.
#include "mla_getrf.cuh"

using namespace mla;

__global__ void __launch_bounds__(kThreads, 1) k_getrf_traced(GetrfArgs a) {
  extern __shared__ __align__(16) double smem[];
  getrf_persistent<true>(a, smem, mla_traced_smem_doubles());
}

int mla_launch_getrf_traced(const GetrfArgs& a, int grid, int smem_bytes, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_getrf_traced, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return (int)e;
  GetrfArgs copy = a;
  void* args[] = {&copy};
  return (int)cudaLaunchCooperativeKernel((void*)k_getrf_traced, dim3(grid), dim3(kThreads), args, smem_bytes, s);
}
