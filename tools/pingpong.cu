// one-way latency of a tagged 128-bit word between two CTAs through L2 (STRONG.GPU st/ld)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st_b128(void* p, unsigned long long lo, unsigned long long hi) {
  asm volatile("{\n .reg .b128 t;\n mov.b128 t, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], t;\n}" ::"l"(p), "l"(lo), "l"(hi) : "memory");
}
__device__ __forceinline__ void ld_b128(const void* p, unsigned long long& lo, unsigned long long& hi) {
  asm volatile("{\n .reg .b128 t;\n ld.relaxed.gpu.global.b128 t, [%2];\n mov.b128 {%0, %1}, t;\n}" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
}
__global__ void pingpong(unsigned long long* buf, int iters, int peer_stride, long long* cycles) {
  // CTA 0 and CTA (gridDim.x-1) play; the others idle
  int me = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x - 1 ? 1 : -1);
  if (me < 0 || threadIdx.x != 0) return;
  unsigned long long* mine = buf + me * 32;
  unsigned long long* theirs = buf + (1 - me) * 32;
  long long t0 = clock64();
  for (int s = 1; s <= iters; ++s) {
    unsigned long long lo, hi;
    if (me == 0) {
      st_b128(mine, s, s);
      do { ld_b128(theirs, lo, hi); } while (hi != (unsigned long long)s);
    } else {
      do { ld_b128(theirs, lo, hi); } while (hi != (unsigned long long)s);
      st_b128(mine, s, s);
    }
  }
  cycles[me] = clock64() - t0;
}
// all-to-all: T CTAs each publish a header, every CTA's warp 0 polls all T headers
__global__ void alltoall(unsigned long long* buf, int iters, long long* cycles) {
  int T = gridDim.x, rank = blockIdx.x, lane = threadIdx.x;
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  for (int s = 1; s <= iters; ++s) {
    unsigned long long* slots = buf + (s & 1) * 4096;
    if (lane == 0) st_b128(slots + rank * 2, s, s);
    for (int t = lane; t < T; t += 32) {
      unsigned long long lo, hi;
      do { ld_b128(slots + t * 2, lo, hi); } while (hi != (unsigned long long)s);
    }
    __syncwarp();
  }
  if (lane == 0) cycles[rank] = clock64() - t0;
}
int main() {
  unsigned long long* buf; long long* cyc;
  cudaMalloc(&buf, 1 << 20); cudaMemset(buf, 0, 1 << 20);
  cudaMallocManaged(&cyc, 1024 * sizeof(long long));
  int iters = 2000;
  for (int grid : {2, 16, 148}) {
    cudaMemset(buf, 0, 1 << 20);
    void* args[] = {&buf, &iters, &grid, &cyc};
    cudaLaunchCooperativeKernel((void*)pingpong, dim3(grid), dim3(32), args, 0, 0);
    cudaDeviceSynchronize();
    printf("pingpong grid %3d: %.0f cycles per round trip (%.2f us at 1.965 GHz)  %s\n", grid, (double)cyc[0] / iters, (double)cyc[0] / iters / 1965.0, cudaGetErrorString(cudaGetLastError()));
  }
  for (int T : {2, 4, 8, 16, 32, 64, 148}) {
    cudaMemset(buf, 0, 1 << 20);
    void* args[] = {&buf, &iters, &cyc};
    cudaLaunchCooperativeKernel((void*)alltoall, dim3(T), dim3(32), args, 0, 0);
    cudaDeviceSynchronize();
    printf("alltoall T=%3d: %.0f cycles per exchange (%.2f us)  %s\n", T, (double)cyc[0] / iters, (double)cyc[0] / iters / 1965.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
