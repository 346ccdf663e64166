// tmem_bench.cu — microbenchmarks of the sm_100a primitives the fused MLP
// kernel is built from (dev tool; results summarised in DESIGN.md §6):
//   1. tcgen05.ld 32x32b throughput vs number of warps
//   2. tcgen05.st 32x32b throughput
//   3. tcgen05.mma kind::f16 M=128, N in {16,32,64,128,256}, K=16, A from TMEM (ts)
//      and from SMEM (ss): cycles per instruction
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_bench tmem_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2310_06822_b200/csrc/nb_device.cuh"

using namespace nb;

__global__ void k_ld(int iters, int nwarps_active, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < nwarps_active) {
    for (int i = 0; i < iters; ++i) {
      uint32_t v[32];
      tmem_ld32(t, v);
      tmem_ld32(t + 32, v);  // two x32 loads = 64 columns
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= v[j];
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

__global__ void k_st(int iters, int nwarps_active, unsigned long long* out) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < nwarps_active) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = j * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
      tmem_st16(t, r);
      tmem_st16(t + 16, r);
      tmem_wait_st();
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

// MMA issue throughput: one thread issues `iters` MMAs of shape 128xNx16 back to back,
// then commits and waits.
template <int N, bool TS, int NACC = 1>
__global__ void k_mma(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 256 * 16 + 128 * 16; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N);
    const uint32_t sb = smem_u32(smem);
    const uint64_t bdesc = make_sdesc(sb, 128, 256);
    const uint64_t adesc = make_sdesc(sb + 256 * 16 * 2, 128, 256);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t dcol = (uint32_t)((i % NACC) * (NACC > 1 ? (256 / NACC) : 0));
      if (TS)
        mma_ts(tm + dcol, tm + 256 + (uint32_t)(i % 2) * 128, bdesc, idesc, 1);
      else
        mma_ss(tm + dcol, adesc, bdesc, idesc, 1);
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}

static double median_cycles(unsigned long long* d, int n) {
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  unsigned long long s = 0;
  for (int i = 0; i < n; ++i) s += h[i];
  return (double)s / n;
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  cudaMalloc(&sink, 64);
  const int iters = 2000, grid = 148;
  for (int nw : {1, 2, 4, 8, 16}) {
    k_ld<<<grid, 512>>>(iters, nw, d, sink);
    cudaDeviceSynchronize();
    double c = median_cycles(d, grid);
    double bytes = (double)iters * nw * 32 * 64 * 4;
    printf("tcgen05.ld  warps=%2d: %.1f cycles/iter, %.1f B/cycle/SM\n", nw, c / iters, bytes / c);
  }
  for (int nw : {1, 4, 8, 16}) {
    k_st<<<grid, 512>>>(iters, nw, d);
    cudaDeviceSynchronize();
    double c = median_cycles(d, grid);
    double bytes = (double)iters * nw * 32 * 32 * 4;
    printf("tcgen05.st  warps=%2d: %.1f cycles/iter, %.1f B/cycle/SM\n", nw, c / iters, bytes / c);
  }
#define RUN_MMA(NN, TS, NA)                                                                         \
  {                                                                                             \
    cudaFuncSetAttribute(k_mma<NN, TS, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    k_mma<NN, TS, NA><<<grid, 128, 64 * 1024>>>(iters, d);                                          \
    cudaError_t e = cudaDeviceSynchronize();                                                    \
    double c = median_cycles(d, grid);                                                          \
    printf("mma %s M=128 N=%3d K=16 nacc=%d: %.1f cycles/instr (%.0f MAC/cycle/SM) %s\n",               \
           TS ? "ts" : "ss", NN, NA, c / iters, 128.0 * NN * 16 * iters / c, cudaGetErrorString(e)); \
  }
  RUN_MMA(16, true, 1) RUN_MMA(32, true, 1) RUN_MMA(64, true, 1) RUN_MMA(128, true, 1) RUN_MMA(256, true, 1)
  RUN_MMA(64, false, 1) RUN_MMA(128, false, 1) RUN_MMA(256, false, 1)
  RUN_MMA(32, true, 2) RUN_MMA(32, true, 4) RUN_MMA(64, true, 2) RUN_MMA(64, true, 4) RUN_MMA(128, true, 2)
  RUN_MMA(64, false, 2) RUN_MMA(64, false, 4) RUN_MMA(32, false, 4)
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
