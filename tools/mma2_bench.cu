// mma2_bench.cu — tcgen05.mma cta_group::2 (M = 256 over a CTA pair) issue
// throughput vs N, A from TMEM (dev tool; compare tmem_bench's cta_group::1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma2_bench mma2_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2310_06822_b200/csrc/nb_device.cuh"

using namespace nb;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N, int NACC>
__global__ void __cluster_dims__(2, 1, 1) k_mma2(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 32) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3F80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(256, N);
    const uint64_t bdesc = make_sdesc(smem_u32(smem), 128, 256);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t dcol = (uint32_t)((i % NACC) * (256 / NACC > N ? N : 0));
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + dcol),
          "r"(tm + 384), "l"(bdesc), "r"(idesc), "r"(1u) : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)),
        "h"((uint16_t)3) : "memory");
    mbar_wait(smem_u32(&bar), 0);
    out[blockIdx.x / 2] = clock64() - t0;
  }
  if (rank == 1 && threadIdx.x == 0) mbar_wait(smem_u32(&bar), 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

static double median(unsigned long long* d, int n) {
  unsigned long long h[1024];
  cudaMemcpy(h, d, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  unsigned long long s = 0;
  for (int i = 0; i < n; ++i) s += h[i];
  return (double)s / n;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 1024);
  const int iters = 2000, grid = 148;
#define RUN(NN, NA)                                                                               \
  {                                                                                               \
    cudaFuncSetAttribute(k_mma2<NN, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
    k_mma2<NN, NA><<<grid, 128, 64 * 1024>>>(iters, d);                                           \
    cudaError_t e = cudaDeviceSynchronize();                                                      \
    double c = median(d, grid / 2);                                                               \
    printf("mma2 ts M=256 N=%3d K=16 nacc=%d: %.1f cycles/instr (%.0f MAC/cycle/SM) %s\n", NN, NA, \
           c / iters, 128.0 * NN * 16 * iters / c, cudaGetErrorString(e));                        \
  }
  RUN(32, 1) RUN(64, 1) RUN(64, 2) RUN(128, 1) RUN(256, 1)
  return 0;
}
