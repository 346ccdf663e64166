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


// MMA throughput while other warps stream tcgen05.ld / tcgen05.st traffic
template <int N, int LDW, bool ST>
__global__ void k_mma_contended(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
    stop = 0;
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N);
    const uint32_t sb = smem_u32(smem);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t kk = i & 3;
      mma_ts(tm, tm + 128 + kk * 8, make_sdesc(sb + kk * 256, 128, 1024), idesc, kk > 0);
    }
    mma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (warp >= 1 && warp <= LDW) {
    const uint32_t t = tm + ((uint32_t)((warp & 3) * 32) << 16) + 192 + (uint32_t)(((warp - 1) >> 2) * 64);
    uint32_t acc = 0;
    while (!stop) {
      uint32_t v[32];
      tmem_ld32(t, v);
      tmem_wait_ld();
      if (ST) {
        uint32_t r[16];
        for (int j = 0; j < 16; ++j) r[j] = v[j] ^ v[j + 16];
        tmem_st16(t + 32, r);
        tmem_wait_st();
      }
      acc ^= v[3];
    }
    if (acc == 0x1234567) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}


// latency: issue NK MMAs (one layer) + commit, wait on the mbarrier; repeat
template <int N, int NK>
__global__ void k_mma_latency(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N);
    const uint32_t sb = smem_u32(smem);
    unsigned long long t0 = clock64(), tissue = 0;
    for (int r = 0; r < reps; ++r) {
      unsigned long long a = clock64();
#pragma unroll
      for (int kk = 0; kk < NK; ++kk)
        mma_ts(tm, tm + 256 + kk * 8, make_sdesc(sb + kk * 256, 128, NK * 256), idesc, kk > 0);
      mma_commit(smem_u32(&bar));
      tissue += clock64() - a;
      mbar_wait(smem_u32(&bar), r & 1);
      tc_fence_after();
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    out[200 + blockIdx.x] = tissue;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tslot);
}


__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
// same as k_mma_latency but the whole warp runs the loop; one elected lane issues
template <int N, int NK>
__global__ void k_mma_latency_warp(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N);
    const uint32_t sb = smem_u32(smem);
    const uint64_t d0 = make_sdesc(sb, 128, NK * 256);
    unsigned long long t0 = clock64(), tissue = 0;
    for (int r = 0; r < reps; ++r) {
      unsigned long long a = clock64();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk)
          mma_ts(tm, tm + 256 + kk * 8, d0 + (uint64_t)(kk * 16), idesc, kk > 0);
        mma_commit(smem_u32(&bar));
      }
      __syncwarp();
      tissue += clock64() - a;
      mbar_wait(smem_u32(&bar), r & 1);
      tc_fence_after();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x] = t1 - t0;
      out[200 + blockIdx.x] = tissue;
    }
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
#define RUN_C(NN, LW, ST)                                                                      \
  {                                                                                           \
    cudaFuncSetAttribute(k_mma_contended<NN, LW, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    k_mma_contended<NN, LW, ST><<<grid, 544, 64 * 1024>>>(iters, d);                          \
    cudaError_t e = cudaDeviceSynchronize();                                                  \
    double c = median_cycles(d, grid);                                                        \
    printf("mma ts N=%3d K=16 SBO=1024 with %2d ld warps st=%d: %.1f cycles/instr %s\n", NN, LW, (int)ST, c / iters, cudaGetErrorString(e)); \
  }
  RUN_C(64, 0, false) RUN_C(64, 4, false) RUN_C(64, 16, false) RUN_C(64, 16, true) RUN_C(128, 0, false) RUN_C(128, 16, true)
#define RUN_L(NN, NK)                                                                      \
  {                                                                                           \
    cudaFuncSetAttribute(k_mma_latency<NN, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    k_mma_latency<NN, NK><<<grid, 128, 64 * 1024>>>(500, d);                          \
    cudaError_t e = cudaDeviceSynchronize();                                                  \
    double c = median_cycles(d, grid);                                                        \
    unsigned long long hi[148]; cudaMemcpy(hi, d + 200, sizeof(hi), cudaMemcpyDeviceToHost); \
    double is = 0; for (int i = 0; i < 148; ++i) is += hi[i]; is /= 148;                      \
    printf("layer latency N=%3d K=%3d: %.1f cycles per (issue+commit+wait), issue part %.1f %s\n", NN, NK * 16, c / 500, is / 500, cudaGetErrorString(e)); \
  }
  RUN_L(64, 1) RUN_L(64, 4) RUN_L(128, 1) RUN_L(128, 8)
#define RUN_LW(NN, NK)                                                                      \
  {                                                                                           \
    cudaFuncSetAttribute(k_mma_latency_warp<NN, NK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    k_mma_latency_warp<NN, NK><<<grid, 128, 64 * 1024>>>(500, d);                          \
    cudaError_t e = cudaDeviceSynchronize();                                                  \
    double c = median_cycles(d, grid);                                                        \
    unsigned long long hi[148]; cudaMemcpy(hi, d + 200, sizeof(hi), cudaMemcpyDeviceToHost); \
    double is = 0; for (int i = 0; i < 148; ++i) is += hi[i]; is /= 148;                      \
    printf("warp-elect layer latency N=%3d K=%3d: %.1f cycles, issue part %.1f %s\n", NN, NK * 16, c / 500, is / 500, cudaGetErrorString(e)); \
  }
  RUN_LW(64, 1) RUN_LW(64, 4) RUN_LW(128, 8)
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
