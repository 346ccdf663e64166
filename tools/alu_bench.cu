// alu_bench.cu — per-SM throughput of the epilogue's instruction mix (dev tool):
// F2FP.RELU.BF16.F32.PACK_AB, FADD2, FFMA2, FMNMX, IADD3, PRMT, LDS.128 broadcast.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_bench alu_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define ITERS 4096

template <int OP>
__global__ void k(float* out, unsigned long long* cyc, float a0, float a1) {
  __shared__ float4 sb[64];
  if (threadIdx.x < 64) sb[threadIdx.x] = make_float4(a0, a1, a0, a1);
  __syncthreads();
  float x[16];
  uint32_t u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    x[i] = a0 * (threadIdx.x + i);
    u[i] = __float_as_uint(x[i]);
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (OP == 0) {  // F2FP relu pack
        uint32_t r;
        asm volatile("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[i + 1]));
        x[i] = __uint_as_float(r ^ 0x3f800000u);
      } else if (OP == 1) {  // FADD2
        asm volatile(
            "{.reg .b64 ra, rb; mov.b64 ra, {%0, %1}; mov.b64 rb, {%2, %3}; add.rn.f32x2 ra, ra, rb; "
            "mov.b64 {%0, %1}, ra;}"
            : "+f"(x[i]), "+f"(x[i + 1])
            : "f"(a0), "f"(a1));
      } else if (OP == 2) {  // FFMA2
        asm volatile(
            "{.reg .b64 ra, rb; mov.b64 ra, {%0, %1}; mov.b64 rb, {%2, %3}; fma.rn.f32x2 ra, ra, rb, ra; "
            "mov.b64 {%0, %1}, ra;}"
            : "+f"(x[i]), "+f"(x[i + 1])
            : "f"(a0), "f"(a1));
      } else if (OP == 3) {  // FMNMX
        asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a0));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i + 1]) : "f"(a1));
      } else if (OP == 4) {  // IADD3 (x2 to match 2 elements)
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(u[i + 1]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i + 1]) : "r"(u[i]));
      } else if (OP == 5) {  // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(u[i]) : "r"(u[i + 1]));
      } else if (OP == 6) {  // LDS.128 broadcast
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"((uint32_t)__cvta_generic_to_shared(&sb[(it + i) & 63])));
        x[i] += v.x;
      } else if (OP == 7) {  // FADD scalar x2
        asm volatile("add.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(a0));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(x[i + 1]) : "f"(a1));
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i] + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  k<OP><<<148, warps * 32>>>(out, cyc, 1.0001f, 0.9999f);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  double instr = (double)ITERS * 8 * warps;  // warp-instructions of the measured op (per 2 elements)
  printf("%-8s warps=%2d: %.2f cycles per warp-instr per SM  (%.1f elem-pairs/clk/SM)\n", name, warps,
         c / instr, 32.0 * instr / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 16}) {
    run<0>("F2FP", w);
    run<1>("FADD2", w);
    run<2>("FFMA2", w);
    run<3>("FMNMXx2", w);
    run<4>("IADDx2", w);
    run<5>("PRMT", w);
    run<6>("LDS128", w);
    run<7>("FADDx2", w);
  }
  return 0;
}
