// Ceiling experiment 2: the LDS+DMMA loop of dmma_loop_ceiling.cu PLUS the operand staging traffic of
// the real kernel (64 KiB per k-tile into a 3-stage ring), in three flavours:
//   mode 0: no staging            mode 1: LDGSTS 16 B, 16 per thread per k-tile, interleaved per k4
//   mode 2: cp.async.bulk, 160 requests per k-tile (32 x 1 KiB + 128 x 256 B)
//   mode 3: cp.async.bulk, 32 x 1 KiB (A) + 32 x 1 KiB (B as contiguous rows: layout-agnostic traffic test)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
constexpr int BM = 128, BN = 128, BK = 32, LDA = BM + 4, LDB = BK + 4, STAGE = BK * LDA + BN * LDB, STAGES = 3;
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(double* out, const double* gA, const double* gB, int iters) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long bar[STAGES];
  const int tid = threadIdx.x;
  for (int i = tid; i < STAGES * STAGE; i += 256) smem[i] = 1e-3 * (i % 97);
  if (tid == 0) { for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5, wi = warp % 2, wj = warp / 2, g = lane >> 2, q = lane & 3;
  double acc[4][8][2];
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const double* A = gA + (size_t)blockIdx.x * 1024 * 128;   // per-CTA source region (L2 resident)
  const double* B = gB + (size_t)blockIdx.x * 1024 * 128;
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
    const int cs = it % STAGES, ls = (it + 2) % STAGES;
    if (MODE == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    if ((MODE == 2 || MODE == 3) && it >= 2) {
      unsigned ok = 0; for (int sp = 0; sp < (1 << 22) && !ok; ++sp)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(s32(&bar[cs])), "r"((phase >> cs) & 1u) : "memory");
      phase ^= 1u << cs;
    }
    __syncthreads();
    double* lA = smem + ls * STAGE; double* lB = lA + BK * LDA;
    const int koff = (it % 32) * BK;
    if (MODE == 2 || MODE == 3) {
      if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[ls])), "r"(65536u) : "memory");
      if (tid < 32) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(s32(lA + tid * LDA)), "l"(A + (size_t)(koff + tid) * 128), "r"(s32(&bar[ls])) : "memory");
      if (MODE == 2) { if (tid >= 32 && tid < 160) { int j = tid - 32; asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(s32(lB + j * LDB)), "l"(B + (size_t)j * 1024 + koff), "r"(s32(&bar[ls])) : "memory"); } }
      else { if (tid >= 32 && tid < 64) { int j = tid - 32; asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(s32(lB + j * 132)), "l"(B + (size_t)(koff + j) * 128), "r"(s32(&bar[ls])) : "memory"); } }
    }
    const double* sA = smem + cs * STAGE; const double* sB = sA + BK * LDA;
    const double* pa = sA + q * LDA + wi * 64 + g; const double* pb = sB + (wj * 32 + g) * LDB + q;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double fi[8], fj[4];
#pragma unroll
      for (int b = 0; b < 8; ++b) fi[b] = pa[k4 * 4 * LDA + b * 8];
#pragma unroll
      for (int a = 0; a < 4; ++a) fj[a] = pb[a * 8 * LDB + k4 * 4];
      if (MODE == 1) {
        const int ar = tid / 64, ac = 2 * (tid % 64);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(lA + (ar + 4 * k4) * LDA + ac)), "l"(A + (size_t)(koff + ar + 4 * k4) * 128 + ac) : "memory");
        const int bc = tid / 16, bk = 2 * (tid % 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(lB + (bc + 16 * k4) * LDB + bk)), "l"(B + (size_t)(bc + 16 * k4) * 1024 + koff + bk) : "memory");
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) dmma884(acc[a][b][0], acc[a][b][1], fj[a], fi[b]);
    }
    if (MODE == 1) asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (MODE == 1) asm volatile("cp.async.wait_group 0;" ::: "memory");
  double s = 0;
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 8; ++b) s += acc[a][b][0] + acc[a][b][1];
  out[blockIdx.x * 256 + tid] = s;
}
template <int M> void run(const char* name, double* out, double* gA, double* gB) {
  int smemb = STAGES * STAGE * 8, iters = 2000;
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemb);
  k<M><<<148, 256, smemb>>>(out, gA, gB, iters); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<M><<<148, 256, smemb>>>(out, gA, gB, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 148.0 * 8 * iters * 8 * 32 * 512.0;
  printf("%s: %.3f ms  %.2f TFLOP/s  %s\n", name, ms, fl / ms * 1e-9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  double *out, *gA, *gB; cudaMalloc(&out, 148 * 256 * 8);
  size_t n = (size_t)148 * 1024 * 128; cudaMalloc(&gA, n * 8); cudaMalloc(&gB, n * 8); cudaMemset(gA, 0, n * 8); cudaMemset(gB, 0, n * 8);
  run<0>("no staging                         ", out, gA, gB);
  run<1>("LDGSTS 16B x16/thread, interleaved ", out, gA, gB);
  run<2>("bulk 32x1KiB + 128x256B            ", out, gA, gB);
  run<3>("bulk 64x1KiB                       ", out, gA, gB);
  return 0;
}
