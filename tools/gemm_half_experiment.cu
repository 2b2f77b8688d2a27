// EXPERIMENT kept for the record, NOT part of libmla_b200.so: the update's tile engine run
// (mode 0) as 128-thread CTAs on 128x64 tiles, two CTAs per SM, so that one CTA's epilogue overlaps the
// other's DMMA stream, and (mode 1) as two independent 128-thread groups inside one 256-thread CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -o tools/gemm_half_experiment \
//        tools/gemm_half_experiment.cu && tools/gemm_half_experiment [m n k mode]
#include <cstdio>
#include <cstdlib>
#include "../paper_1611_06365_b200/csrc/mla_common.cuh"
#include "../paper_1611_06365_b200/csrc/mla_gemm.cuh"
using namespace mla;
enum { CW_QUEUE_NEXT = 1 };
namespace mla { using GemmHalfCfg = GemmCfg<128, 64, 2, 2, 2, 32, 128>; }

// EXPERIMENT (tools/dev_gemm_half.py): the same tile engine as 128-thread CTAs on 128x64 tiles, two CTAs
// per SM, so that one CTA's epilogue / barrier bubbles overlap the other's DMMA stream.
__global__ void __launch_bounds__(128, 2)
k_gemm_half(GemmProblem p, unsigned* ctrl) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_tile;
  using Cfg = GemmHalfCfg;
  const int ntiles = gemm_num_tiles<Cfg>(p);
  auto pop = [&]() {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ctrl + CW_QUEUE_NEXT, 1u);
    __syncthreads();
    int t = s_tile;
    __syncthreads();
    return t;
  };
  int t = pop();
  if (t >= ntiles) return;
  TileDesc cur = gemm_tile_desc<Cfg>(p, t);
  int base = 0;
  tile_prologue<Cfg>(cur, base, smem);
  while (true) {
    int tn = pop();
    TileDesc nxt{};
    nxt.valid = false;
    if (tn < ntiles && tile_kt<Cfg>(cur) >= Cfg::STAGES - 1) nxt = gemm_tile_desc<Cfg>(p, tn);
    base = tile_run<Cfg>(cur, nxt, base, smem);
    if (nxt.valid) { cur = nxt; continue; }
    if (tn >= ntiles) break;
    cur = gemm_tile_desc<Cfg>(p, tn);
    base = 0;
    tile_prologue<Cfg>(cur, base, smem);
  }
  bulk_wait_all();
}

// Same idea inside ONE 256-thread CTA: two independent 128-thread groups, each with its own ring and its
// own named barrier, each pulling 128x64 half-tiles from the queue.
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_dual(GemmProblem p, unsigned* ctrl) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_tile[2];
  using Cfg = GemmHalfCfg;
  const int g = grp_id<Cfg::THREADS>(), gtid = grp_tid<Cfg::THREADS>();
  double* gsmem = smem + g * (Cfg::SMEM_BYTES / 8);
  const int ntiles = gemm_num_tiles<Cfg>(p);
  auto pop = [&]() {
    if (gtid == 0) s_tile[g] = (int)atomicAdd(ctrl + CW_QUEUE_NEXT, 1u);
    grp_sync<Cfg::THREADS>();
    int t = s_tile[g];
    grp_sync<Cfg::THREADS>();
    return t;
  };
  int t = pop();
  if (t >= ntiles) return;
  TileDesc cur = gemm_tile_desc<Cfg>(p, t);
  int base = 0;
  tile_prologue<Cfg>(cur, base, gsmem);
  while (true) {
    int tn = pop();
    TileDesc nxt{};
    nxt.valid = false;
    if (tn < ntiles && tile_kt<Cfg>(cur) >= Cfg::STAGES - 1) nxt = gemm_tile_desc<Cfg>(p, tn);
    base = tile_run<Cfg>(cur, nxt, base, gsmem);
    if (nxt.valid) { cur = nxt; continue; }
    if (tn >= ntiles) break;
    cur = gemm_tile_desc<Cfg>(p, tn);
    base = 0;
    tile_prologue<Cfg>(cur, base, gsmem);
  }
  bulk_wait_all();
}


int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 16384, n = argc > 2 ? atoi(argv[2]) : 16384, k = argc > 3 ? atoi(argv[3]) : 256;
  int mode = argc > 4 ? atoi(argv[4]) : 0;
  double *A, *B, *C; unsigned* ctrl;
  cudaMalloc(&A, (size_t)m * k * 8); cudaMalloc(&B, (size_t)k * n * 8); cudaMalloc(&C, (size_t)m * n * 8);
  cudaMalloc(&ctrl, 64 * 4);
  cudaMemset(A, 0, (size_t)m * k * 8); cudaMemset(B, 0, (size_t)k * n * 8); cudaMemset(C, 0, (size_t)m * n * 8);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  GemmProblem p{C, m, A, m, B, k, m, n, k, 1.0, -1.0};
  cudaFuncSetAttribute(k_gemm_half, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmHalfCfg::SMEM_BYTES);
  cudaFuncSetAttribute(k_gemm_dual, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * GemmHalfCfg::SMEM_BYTES);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(ctrl, 0, 64 * 4);
    cudaEventRecord(e0);
    if (mode == 0) k_gemm_half<<<2 * prop.multiProcessorCount, 128, GemmHalfCfg::SMEM_BYTES>>>(p, ctrl);
    else k_gemm_dual<<<prop.multiProcessorCount, kThreads, 2 * GemmHalfCfg::SMEM_BYTES>>>(p, ctrl);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d  %d x %d x %d: %.3f ms  %.2f TFLOP/s\n", mode, m, n, k, ms, 2.0 * m * n * k / ms / 1e9);
  }
  return 0;
}
