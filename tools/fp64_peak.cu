// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 / m16n8k8 f64) issue-bound
// rate and plain DFMA rate.  These are the roofline denominators MEASURED_PEAKS.json lacks.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1688(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int NACC>
__global__ void k_dmma884(double* out, int iters) {
  double acc[NACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = i; acc[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma884(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma1688(double* out, int iters) {
  double acc[NACC][4];
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0 + threadIdx.x * 1e-6; b[1] = 0.5;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = i; acc[i][1] = -i; acc[i][2] = 1; acc[i][3] = 2; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma1688(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double acc[NACC];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
static float timeit(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock %d kHz\n", p.name, sms, p.clockRate);
  double* out; cudaMalloc(&out, sizeof(double) * 1024 * 1024 * 4);
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int threads = warps * 32;
    for (int bps = 1; bps <= 2; ++bps) {
      int grid = sms * bps;
      double nw = double(grid) * warps;
      { float ms = timeit([&] { k_dmma884<16><<<grid, threads>>>(out, iters); });
        double fl = nw * iters * 16.0 * 512.0;
        printf("dmma884  warps/cta %2d cta/sm %d : %8.3f ms  %7.2f TFLOP/s\n", warps, bps, ms, fl / ms * 1e-9); }
      { float ms = timeit([&] { k_dmma1688<8><<<grid, threads>>>(out, iters); });
        double fl = nw * iters * 8.0 * 2048.0;
        printf("dmma1688 warps/cta %2d cta/sm %d : %8.3f ms  %7.2f TFLOP/s\n", warps, bps, ms, fl / ms * 1e-9); }
      { float ms = timeit([&] { k_dfma<16><<<grid, threads>>>(out, iters); });
        double fl = nw * 32.0 * iters * 16.0 * 2.0;
        printf("dfma     warps/cta %2d cta/sm %d : %8.3f ms  %7.2f TFLOP/s\n", warps, bps, ms, fl / ms * 1e-9); }
    }
  }
  // sustained: 3 s of dmma884 at 8 warps/cta, 2 cta/sm
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int grid = sms * 2, threads = 256, reps = 60;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_dmma884<16><<<grid, threads>>>(out, iters * 8);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = double(grid) * 8 * double(iters) * 8 * 16.0 * 512.0 * reps;
    printf("dmma884 sustained %.1f ms : %7.2f TFLOP/s\n", ms, fl / ms * 1e-9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
