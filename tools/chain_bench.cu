// chain_bench.cu — ceiling of the fused kernel's MMA issue structure (dev tool):
// NSLOT independent slot chains of WPS warps; per "layer" the slot's warps meet
// at a named barrier, the lead warp's elected lane issues G tcgen05.mma
// (M=128, N=64, K=16, A from TMEM) + commit, and all warps wait on the slot's
// mbarrier.  No epilogue.  Reports cycles per MMA instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o chain_bench chain_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2310_06822_b200/csrc/nb_device.cuh"

using namespace nb;

__device__ __forceinline__ bool try_wait_nohint(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
static __device__ int g_wait_mode;  // 0: try_wait + hint, 1: try_wait, 2: test_wait spin

template <int NSLOT, int WPS, int G, bool DUMMY_ST, bool CPM = false>
__global__ void k_chain(int iters, unsigned long long* out, int spin) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(smem_u32(&tslot));
  if (threadIdx.x == 32) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(smem_u32(&bars[s]), CPM ? G : 1);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const int s = warp / WPS;
  const bool leadw = (warp % WPS) == 0;
  const uint32_t idesc = make_idesc_bf16(128, 64);
  const uint64_t bdesc = make_sdesc(smem_u32(smem), 128, 1024);
  const uint32_t d = tm + s * 64, a = tm + NSLOT * 64 + s * 32;
  const uint32_t trow = tm + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t ph = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (spin > 0) {  // synthetic epilogue latency (ALU-free)
      const long long t = clock64();
      while (clock64() - t < spin) {
      }
    }
    if (DUMMY_ST) {  // the A-operand stores an epilogue would do (32 columns per row)
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) r[j] = j + it;
      tmem_st16(trow + NSLOT * 64 + s * 32 + (uint32_t)((warp % WPS) / 4) * 16, r);
      if (WPS == 4) tmem_st16(trow + NSLOT * 64 + s * 32 + 16, r);
      tmem_wait_st();
    }
    tc_fence_before();
    asm volatile("bar.sync %0, %1;" ::"r"(s + 1), "n"(WPS * 32) : "memory");
    if (leadw) {
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          mma_ts(d, a + (g % 4) * 8, bdesc + (uint64_t)((g % 4) * 16), idesc, g > 0);
          if (CPM) mma_commit(smem_u32(&bars[s]));
        }
        if (!CPM) mma_commit(smem_u32(&bars[s]));
      }
      __syncwarp();
    }
    {
      const int wm = g_wait_mode;
      if (wm == 0) mbar_wait(smem_u32(&bars[s]), ph);
      else if (wm == 1) while (!try_wait_nohint(smem_u32(&bars[s]), ph)) {}
      else while (!mbar_test_wait(smem_u32(&bars[s]), ph)) {}
    }
    ph ^= 1u;
    tc_fence_after();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

static double avg(unsigned long long* d, int n) {
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  unsigned long long s = 0;
  for (int i = 0; i < n; ++i) s += h[i];
  return (double)s / n;
}

static int g_spin = 0;

int main() {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  const int iters = 2000, grid = 148;
#define RUN(NS, WP, G, ST, ...)                                                                  \
  {                                                                                               \
    auto k = k_chain<NS, WP, G, ST, ##__VA_ARGS__>;                                                              \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);             \
    k<<<grid, NS * WP * 32, 120 * 1024>>>(iters, d, g_spin);                                      \
    cudaError_t e = cudaDeviceSynchronize();                                                      \
    double c = avg(d, grid);                                                                      \
    printf("slots=%d wps=%d G=%d st=%d spin=%d: %.1f cycles per MMA, %.0f per group-round %s\n", NS, WP, G, \
           (int)ST, g_spin, c / ((double)iters * NS * G), c / iters, cudaGetErrorString(e));     \
  }
  RUN(1, 4, 5, false) RUN(2, 4, 5, false) RUN(3, 4, 5, false) RUN(4, 4, 5, false) RUN(5, 4, 5, false)
  RUN(5, 4, 4, false) RUN(5, 4, 1, false) RUN(5, 1, 5, false)
  RUN(5, 4, 5, true) RUN(4, 8, 5, true) RUN(5, 4, 4, true)
  for (int wm : {0, 1, 2}) {
    cudaMemcpyToSymbol(g_wait_mode, &wm, sizeof(int));
    printf("-- wait mode %d\n", wm);
    for (int sp : {0, 400, 800}) {
      g_spin = sp;
      RUN(5, 4, 5, true) RUN(5, 4, 1, true)
    }
  }
  { int wm = 0; cudaMemcpyToSymbol(g_wait_mode, &wm, sizeof(int)); }
  g_spin = 0;
  printf("-- commit after every MMA:\n");
  RUN(5, 4, 5, false, true) RUN(3, 4, 5, false, true) RUN(5, 1, 5, false, true)
  return 0;
}
