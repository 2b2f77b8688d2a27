// Ceiling of the gemm main loop's inner structure: 8 warps, per k4 step 12 conflict-free LDS.64
// fragment loads + 32 DMMA.8x8x4 on 32 independent accumulators, operands resident in shared memory
// (no global traffic, optional __syncthreads every KT k4-steps).  Compare with fp64_peak.cu (37.0).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
constexpr int BM = 128, BN = 128, BK = 32, LDA = BM + 4, LDB = BK + 4;
template <int SYNC_EVERY>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters) {
  extern __shared__ double smem[];
  double* sA = smem;                 // [BK][LDA]
  double* sB = smem + BK * LDA;      // [BN][LDB]
  for (int i = threadIdx.x; i < BK * LDA + BN * LDB; i += 256) smem[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wi = warp % 2, wj = warp / 2, g = lane >> 2, q = lane & 3;
  double acc[4][8][2];
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* pa = sA + q * LDA + wi * 64 + g;
  const double* pb = sB + (wj * 32 + g) * LDB + q;
  for (int it = 0; it < iters; ++it) {
    if (SYNC_EVERY && (it % SYNC_EVERY) == 0) __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double fi[8], fj[4];
#pragma unroll
      for (int b = 0; b < 8; ++b) fi[b] = pa[k4 * 4 * LDA + b * 8];
#pragma unroll
      for (int a = 0; a < 4; ++a) fj[a] = pb[a * 8 * LDB + k4 * 4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) dmma884(acc[a][b][0], acc[a][b][1], fj[a], fi[b]);
    }
  }
  double s = 0;
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 8; ++b) s += acc[a][b][0] + acc[a][b][1];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
template <int S> void run(const char* name, double* out) {
  int smemb = (BK * LDA + BN * LDB) * 8, iters = 2000;
  cudaFuncSetAttribute(k<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemb);
  k<S><<<148, 256, smemb>>>(out, iters); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<S><<<148, 256, smemb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0 * 8 * iters * 8 * 32 * 512.0;
  printf("%s: %.3f ms  %.2f TFLOP/s  %s\n", name, ms, fl / ms * 1e-9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double* out; cudaMalloc(&out, 148 * 256 * 8);
  run<0>("LDS+DMMA loop, no barrier      ", out);
  run<1>("LDS+DMMA loop, barrier / k-tile", out);
  return 0;
}
