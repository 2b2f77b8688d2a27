// The production persistent LU kernel, alone in its translation unit: NVVM's inlining of the tile loops
// depends on module-wide call counts, so kernels that share the tile engine (k_gemm, k_apply_panel) must not be
// able to change this kernel's code generation (round 2: an unrelated edit of k_apply_panel cost it 3 %).
#include "mla_getrf.cuh"

using namespace mla;

__global__ void __launch_bounds__(kThreads, 1) k_getrf(GetrfArgs a) {
  extern __shared__ __align__(16) double smem[];
  getrf_persistent<false>(a, smem, mla_traced_smem_doubles());
}

int mla_launch_getrf(const GetrfArgs& a, int grid, int smem_bytes, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(k_getrf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return (int)e;
  GetrfArgs copy = a;
  void* args[] = {&copy};
  return (int)cudaLaunchCooperativeKernel((void*)k_getrf, dim3(grid), dim3(kThreads), args, smem_bytes, s);
}
