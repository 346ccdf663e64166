// nb_simt.cu — CUDA-core kernels of libnb:
//   * a1 encoder (bf16 hi/lo split) and the bf16 parameter pack,
//   * the fp32 fused forward/calibrate/score kernel (BASELINE.json configs[0]),
//   * the fp32 training step (forward + Eq. (1) gradient + back-propagation,
//     deterministic fixed-order gradient reduction), and Adam.
// Paper: PAPER.md (arXiv 2310.06822) §3.1 Eq. (1), Alg. 1 P:207-222,
// §3.3 early-out P:231-279, §3.4 P:285-297.
#include <cuda_bf16.h>

#include "nb_adam.cuh"
#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

// ---------------------------------------------------------------------------
// a1 encoder: each fp32 coordinate x -> bf16 pair (hi, lo) = (RNE(x), RNE(x - hi)),
// so the layer-1 product (hi + lo) W keeps ~16 mantissa bits of the input
// (R20; record parameterisations P:777).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void encode_pairs(const float* x, int d0, uint32_t (&col)[8]) {
  uint16_t e[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) e[j] = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j < d0) {
      __nv_bfloat16 hi = __float2bfloat16_rn(x[j]);
      __nv_bfloat16 lo = __float2bfloat16_rn(x[j] - __bfloat162float(hi));
      e[j] = __bfloat16_as_ushort(hi);
      e[d0 + j] = __bfloat16_as_ushort(lo);
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) col[c] = (uint32_t)e[2 * c] | ((uint32_t)e[2 * c + 1] << 16);
}

__global__ void k_encode_bf16(const float* __restrict__ q, int64_t n, int d0, uint4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = j < d0 ? q[i * d0 + j] : 0.f;
    uint32_t c[8];
    encode_pairs(x, d0, c);
    out[2 * i] = make_uint4(c[0], c[1], c[2], c[3]);
    out[2 * i + 1] = make_uint4(c[4], c[5], c[6], c[7]);
  }
}

cudaError_t launch_encode(const nb_model* m, const float* q, int64_t n, void* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (m->d.precision == NB_FP32)
    return cudaMemcpyAsync(out, q, sizeof(float) * n * m->d0, cudaMemcpyDeviceToDevice, s);
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_encode_bf16<<<blocks, 256, 0, s>>>(q, n, m->d0, (uint4*)out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// bf16 pack: fp32 canonical blob -> the shared-memory image of nb_internal.cuh
// (UMMA K-major core matrices for W_l; fp32 biases / output / heads).
// Layer 1's K = 16 image holds W_1 twice: columns [0, d0) multiply the hi
// halves, [d0, 2 d0) the lo halves of the encoded input.
// ---------------------------------------------------------------------------
__global__ void k_pack_bf16(PackArgs a) {
  const int W = a.W;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // CTA-pair widths: image v holds output rows [v W/2, (v+1) W/2) of each layer
  const int rows = W / (int)a.pl.pairs;
  for (int l = 0; l < a.L; ++l) {
    const int K = (int)a.pl.k_of[l];
    for (int64_t e = tid; e < (int64_t)W * K; e += stride) {
      int n = (int)(e / K), k = (int)(e % K);
      float v;
      if (l == 0 && a.pl.pe_lo) {  // PE layout: [hi | ones | .. | lo at pe_lo]
        const int lo = (int)a.pl.pe_lo;
        int src = k < a.d0 ? k : ((k >= lo && k < lo + a.d0) ? k - lo : -1);
        v = src >= 0 ? a.theta[a.po.W[0] + (int64_t)n * a.d0 + src] : 0.f;
        const int j = k - a.d0;
        if (a.pl.bias_l0 && j >= 0 && j < 3) v = bias_piece(a.theta[a.po.b[0] + n], j);
      } else if (l == 0) {
        int src = k < a.d0 ? k : (k < 2 * a.d0 ? k - a.d0 : -1);
        v = src >= 0 ? a.theta[a.po.W[0] + (int64_t)n * a.d0 + src] : 0.f;
        const int j = k - 2 * a.d0;  // bias split columns (the encoder's ones)
        if (a.pl.bias_l0 && j >= 0 && j < 3) v = bias_piece(a.theta[a.po.b[0] + n], j);
      } else {
        v = a.theta[a.po.W[l] + (int64_t)n * W + k];
      }
      const int img_i = n / rows, nl = n % rows;
      __nv_bfloat16* img =
          (__nv_bfloat16*)(a.out + (size_t)img_i * a.pl.bytes + a.pl.off_w[l]);
      int64_t off = (int64_t)(nl / 8) * (K / 8) * 64 + (k / 8) * 64 + (nl % 8) * 8 + (k % 8);
      img[off] = __float2bfloat16_rn(v);
    }
  }
  // CTA-pair images: one shared bias block per image, layer l >= 1 in columns 3 (l - 1) + j
  if (a.pl.bb_shared) {
    for (int64_t e = tid; e < (int64_t)(a.L - 1) * W * 3; e += stride) {
      const int l = 1 + (int)(e / (W * 3)), n = (int)((e / 3) % W), jj = (int)(e % 3);
      __nv_bfloat16* img = (__nv_bfloat16*)(a.out + (size_t)(n / rows) * a.pl.bytes + a.pl.off_bb[0]);
      const int nl = n % rows, k = 3 * (l - 1) + jj;
      img[(int64_t)(nl / 8) * (kEncK / 8) * 64 + (k / 8) * 64 + (nl % 8) * 8 + (k % 8)] =
          __float2bfloat16_rn(bias_piece(a.theta[a.po.b[l] + n], jj));
    }
  }
  // bias-as-MMA blocks of layers l >= 1: [W][16] K-major, k = 0..2 = split of b_l
  for (int l = 1; l < a.L && !a.pl.bb_shared; ++l) {
    if (!a.pl.off_bb[l]) continue;
    __nv_bfloat16* img = (__nv_bfloat16*)(a.out + a.pl.off_bb[l]);
    for (int64_t e = tid; e < (int64_t)W * kEncK; e += stride) {
      const int n = (int)(e / kEncK), k = (int)(e % kEncK);
      const float v = k < 3 ? bias_piece(a.theta[a.po.b[l] + n], k) : 0.f;
      img[(int64_t)(n / 8) * (kEncK / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 + (k % 8)] =
          __float2bfloat16_rn(v);
    }
  }
  // transposed pair images: W_l[o][i] -> image i / 128, row i % 128, column o (K = W)
  if (a.out_bwd) {
    for (int l = 1; l < a.L; ++l) {
      for (int64_t e = tid; e < (int64_t)W * W; e += stride) {
        const int o = (int)(e / W), i = (int)(e % W);
        __nv_bfloat16* img = (__nv_bfloat16*)(a.out_bwd + (size_t)(i / rows) * a.bl.bytes + a.bl.off_wt[l]);
        const int r = i % rows;
        img[(int64_t)(r / 8) * (W / 8) * 64 + (o / 8) * 64 + (r % 8) * 8 + (o % 8)] =
            __float2bfloat16_rn(a.theta[a.po.W[l] + e]);
      }
    }
    for (int64_t e = tid; e < (int64_t)W; e += stride) {
      for (int im = 0; im < 2; ++im) {
        uint8_t* b = a.out_bwd + (size_t)im * a.bl.bytes;
        ((float*)(b + a.bl.off_wout))[e] = a.theta[a.po.wout + e];
        for (int k = 0; k < a.nh; ++k) ((float*)(b + a.bl.off_u[k]))[e] = a.theta[a.po.u[k] + e];
      }
    }
  }
  float* bias = (float*)(a.out + a.pl.off_bias);
  for (int64_t e = tid; e < (int64_t)a.L * W; e += stride)
    bias[e] = a.theta[a.po.b[e / W] + e % W];
  float* wo = (float*)(a.out + a.pl.off_wout);
  for (int64_t e = tid; e < W; e += stride) wo[e] = a.theta[a.po.wout + e];
  if (tid == 0) {
    float* bo = (float*)(a.out + a.pl.off_bout);
    bo[0] = a.theta[a.po.bout];
    bo[1] = bo[2] = bo[3] = 0.f;
    float* c = (float*)(a.out + a.pl.off_c);
    c[0] = a.nh > 0 ? a.theta[a.po.c[0]] : 0.f;
    c[1] = a.nh > 1 ? a.theta[a.po.c[1]] : 0.f;
    c[2] = c[3] = 0.f;
  }
  for (int k = 0; k < a.nh; ++k) {
    float* u = (float*)(a.out + a.pl.off_u[k]);
    for (int64_t e = tid; e < W; e += stride) u[e] = a.theta[a.po.u[k] + e];
  }
}

cudaError_t launch_pack_bf16(const nb_model* m, cudaStream_t s) {
  PackArgs a;
  a.theta = m->theta;
  a.out = m->packed;
  a.out_bwd = m->packed_bwd;
  a.bl = m->bl;
  a.pl = m->pl;
  a.po = m->po;
  a.W = m->d.width;
  a.L = m->d.hidden_layers;
  a.d0 = m->din;  // layer-1 input features (hi columns [0, din), lo [din, 2 din))
  a.nh = m->d.n_heads;
  k_pack_bf16<<<148, 256, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  // CTA-pair images: replicate the fp32 tail (biases, output, heads) of image 0
  for (uint32_t i = 1; i < m->pl.pairs && e == cudaSuccess; ++i)
    e = cudaMemcpyAsync(m->packed + (size_t)i * m->pl.bytes + m->pl.off_bias,
                        m->packed + m->pl.off_bias, m->pl.core_bytes - m->pl.off_bias,
                        cudaMemcpyDeviceToDevice, s);  // (bias blocks differ per image)
  return e;
}

// ---------------------------------------------------------------------------
// fp32 fused forward (+ calibrate / score), one query per thread, all weights
// in shared memory.  h_0 = x; z_l = W_l h_{l-1} + b_l; h_l = ReLU(z_l);
// z = w_out . h_L + b_out; e_k = u_k . h_{l_k} + c_k.
// Summation order per output: bias first, then inputs in index order.
// ---------------------------------------------------------------------------
struct SimtArgs {
  ParamOffsets po;
  int P, d0, L, nh, ha0, ha1;
  int din, act, pe;  // layer-1 inputs, nb_activation, positional-encoding depth
};

// Layer-1 input of one record (R42): the record itself, then for
// each frequency 2^k pi (k < pe / 2) sin and cos of every coordinate.
// sincospif reduces 2^k x exactly (the scaling by a power of two is exact).
__device__ __forceinline__ void simt_features(const float* x, int d0, int pe, float* f) {
  for (int j = 0; j < d0; ++j) f[j] = x[j];
  for (int k = 0; k < pe / 2; ++k)
    for (int j = 0; j < d0; ++j) {
      float sv, cv;
      sincospif(ldexpf(x[j], k), &sv, &cv);
      f[d0 + 2 * k * d0 + j] = sv;
      f[d0 + (2 * k + 1) * d0 + j] = cv;
    }
}
// hidden activation (R1 ReLU, R41 sine) and its derivative at z
__device__ __forceinline__ float simt_act(float z, int act) { return act == NB_SINE ? sinf(z) : fmaxf(z, 0.f); }
__device__ __forceinline__ float simt_dact(float z, int act) {
  return act == NB_SINE ? cosf(z) : (z > 0.f ? 1.f : 0.f);  // ReLU'(0) = 0 (R25)
}

template <int W, int MODE>
__global__ void __launch_bounds__(256) k_fwd_simt(const float* __restrict__ theta, SimtArgs s,
                                                  FwdArgs a) {
  extern __shared__ float sp[];
  for (int i = threadIdx.x; i < s.P; i += blockDim.x) sp[i] = theta[i];
  __syncthreads();
  WarpAcc acc;
  acc.init();
  const int nl = 1 + s.nh;
  const int64_t warp_stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = (MODE == kForward && a.n_dev) ? (int64_t)*a.n_dev : a.n;  // hierarchies
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += warp_stride) {
    const int64_t i = base + (threadIdx.x & 31);
    const bool valid = i < n;
    float h[W];
    float e[2] = {0.f, 0.f};
    bool bad = false;
    {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (valid && j < s.d0) ? a.q[i * s.d0 + j] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) bad = bad || (j < s.d0 && !isfinite(x[j]));
      const float* W0 = sp + s.po.W[0];
      const float* b0 = sp + s.po.b[0];
      if (s.pe == 0) {
#pragma unroll
        for (int o = 0; o < W; ++o) {
          float acc_o = b0[o];
          for (int k = 0; k < s.d0; ++k) acc_o = fmaf(W0[o * s.d0 + k], x[k], acc_o);
          h[o] = simt_act(acc_o, s.act);
        }
      } else {
        float f[kSimtMaxIn];
        simt_features(x, s.d0, s.pe, f);
#pragma unroll
        for (int o = 0; o < W; ++o) {
          float acc_o = b0[o];
          for (int k = 0; k < s.din; ++k) acc_o = fmaf(W0[o * s.din + k], f[k], acc_o);
          h[o] = simt_act(acc_o, s.act);
        }
      }
    }
    for (int l = 1; l <= s.L; ++l) {
      if (l > 1) {
        const float* Wl = sp + s.po.W[l - 1];
        const float* bl = sp + s.po.b[l - 1];
        float hn[W];
#pragma unroll
        for (int o = 0; o < W; ++o) {
          float acc_o = bl[o];
#pragma unroll
          for (int k = 0; k < W; ++k) acc_o = fmaf(Wl[o * W + k], h[k], acc_o);
          hn[o] = simt_act(acc_o, s.act);
        }
#pragma unroll
        for (int o = 0; o < W; ++o) h[o] = hn[o];
      }
      int hk = (s.nh > 0 && s.ha0 == l) ? 0 : ((s.nh > 1 && s.ha1 == l) ? 1 : -1);
      if (hk >= 0) {
        const float* u = sp + s.po.u[hk];
        float t = sp[s.po.c[hk]];
#pragma unroll
        for (int j = 0; j < W; ++j) t = fmaf(u[j], h[j], t);
        e[hk] = t;
      }
    }
    float z = sp[s.po.bout];
    {
      const float* wo = sp + s.po.wout;
#pragma unroll
      for (int j = 0; j < W; ++j) z = fmaf(wo[j], h[j], z);
    }
    if (bad) z = __int_as_float(0x7FC00000);  // non-finite record -> NaN logit (R26)
    if (MODE == kCalibrate && valid && !isfinite(z)) atomicOr(a.flags, kFlagNonFinite);
    if (MODE == kForward) {
      if (valid) {
        a.logits[i * nl] = z;
        if (s.nh > 0) a.logits[i * nl + 1] = e[0];
        if (s.nh > 1) a.logits[i * nl + 2] = e[1];
        if (a.prob) a.prob[i] = 1.f / (1.f + expf(-z));
        if (!isfinite(z)) atomicOr(a.flags, kFlagNonFinite);
      }
    } else {
      int y = valid ? a.y[i] : 0;
      classify_row<MODE>(acc, valid, y, z, e, s.nh, a.tau, a.flags, a.invert);
    }
  }
  if (MODE != kForward) flush_warp<MODE>(acc, s.nh, a.counts, a.keys);
  if (MODE == kScore && a.ticket) {
    __syncthreads();
    if (threadIdx.x < 32) finalize_counts(a);
  }
}

bool simt_supported(const nb_desc& d) {
  const int r = d.kind == NB_POINT ? d.space_dim : 2 * d.space_dim;
  return (d.width == 16 || d.width == 32 || d.width == 64) && d.hidden_layers >= 1 &&
         d.hidden_layers <= kMaxLayers && r * (1 + d.pe_depth) <= kSimtMaxIn;
}

template <int W>
static cudaError_t launch_simt_w(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  SimtArgs s;
  s.po = m->po;
  s.P = (int)m->P;
  s.d0 = m->d0;
  s.din = m->din;
  s.act = m->d.activation;
  s.pe = m->d.pe_depth;
  s.L = m->d.hidden_layers;
  s.nh = m->d.n_heads;
  s.ha0 = m->d.head_after[0];
  s.ha1 = m->d.head_after[1];
  size_t smem = sizeof(float) * m->P;
  int64_t blocks = (a.n + 255) / 256;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)m->num_sms * 8));
  switch (mode) {
    case kForward:
      cudaFuncSetAttribute(k_fwd_simt<W, kForward>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_fwd_simt<W, kForward><<<grid, 256, smem, st>>>(m->theta, s, a);
      break;
    case kCalibrate:
      cudaFuncSetAttribute(k_fwd_simt<W, kCalibrate>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_fwd_simt<W, kCalibrate><<<grid, 256, smem, st>>>(m->theta, s, a);
      break;
    default:
      cudaFuncSetAttribute(k_fwd_simt<W, kScore>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_fwd_simt<W, kScore><<<grid, 256, smem, st>>>(m->theta, s, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_fwd_simt(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t s) {
  switch (m->d.width) {
    case 16: return launch_simt_w<16>(m, mode, a, s);
    case 32: return launch_simt_w<32>(m, mode, a, s);
    case 64: return launch_simt_w<64>(m, mode, a, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// fp32 training step (CUDA cores).
//   K1 (one sample per thread): forward keeping h_0..h_L, loss of Eq. (1)
//      with FN weight alpha and FP weight beta, dL/dz = w (sigma(z) - y) / B,
//      head losses added, back-propagation dL/dz_l (ReLU'(0) = 0);
//      writes h_l and delta_l rows to scratch.
//   K2 (one parameter per thread, 16 fixed row chunks): partial sums over rows
//      in row order; K3 sums the 16 chunks in order -> deterministic gradient.
// ---------------------------------------------------------------------------
constexpr int kGradChunks = 16;

struct TrainScratch {
  float* h;      // [L+1][n][Wmax]
  float* dlt;    // [L][n][W]
  float* gout;   // [n][1 + nh]  dL/dz, dL/de_k
  float* part;   // [kGradChunks][P]
};

static TrainScratch carve_simt(nb_model* m, int64_t n) {
  const int W = m->d.width, L = m->d.hidden_layers, nh = m->d.n_heads;
  const int Wm = std::max(W, m->din);
  uint8_t* p = (uint8_t*)m->train_scratch;
  TrainScratch t;
  t.h = (float*)p; p += sizeof(float) * (size_t)(L + 1) * n * Wm;
  t.dlt = (float*)p; p += sizeof(float) * (size_t)L * n * W;
  t.gout = (float*)p; p += sizeof(float) * (size_t)n * (1 + nh);
  t.part = (float*)p;
  return t;
}

size_t train_simt_scratch_bytes(const nb_model* m, int64_t n) {
  const int W = m->d.width, L = m->d.hidden_layers, nh = m->d.n_heads;
  const int Wm = std::max(W, m->din);
  return sizeof(float) * ((size_t)(L + 1) * n * Wm + (size_t)L * n * W + (size_t)n * (1 + nh) +
                          (size_t)kGradChunks * m->P) + 256;
}

__device__ __forceinline__ float softplusf(float u) {
  return fmaxf(u, 0.f) + log1pf(expf(-fabsf(u)));
}

template <int W>
__global__ void __launch_bounds__(128) k_train_fwd_bwd_simt(const float* __restrict__ theta,
                                                            SimtArgs s, const float* __restrict__ q,
                                                            const uint8_t* __restrict__ y,
                                                            int64_t n, float invB, float alpha,
                                                            float beta, TrainScratch t,
                                                            double* loss_out,
                                                            unsigned long long* stats) {
  extern __shared__ float sp[];
  for (int i = threadIdx.x; i < s.P; i += blockDim.x) sp[i] = theta[i];
  __syncthreads();
  const int Wm = W > s.din ? W : s.din;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = i < n;
  float loss = 0.f;
  unsigned st[4] = {0, 0, 0, 0};
  if (valid) {
    float hs[kMaxLayers + 1][W];  // h_0 (layer-1 input, din <= W) .. h_L
    float ds[kMaxLayers][W];      // activation derivative at z_l (ReLU mask, or cos z_l)
    {
      float x[8], f[kSimtMaxIn];
      for (int j = 0; j < 8; ++j) x[j] = j < s.d0 ? q[i * s.d0 + j] : 0.f;
      simt_features(x, s.d0, s.pe, f);
#pragma unroll
      for (int j = 0; j < W; ++j) hs[0][j] = j < s.din ? f[j] : 0.f;
    }
    float e[2] = {0.f, 0.f};
    for (int l = 1; l <= s.L; ++l) {
      const int in = l == 1 ? s.din : W;
      const float* Wl = sp + s.po.W[l - 1];
      const float* bl = sp + s.po.b[l - 1];
#pragma unroll
      for (int o = 0; o < W; ++o) {
        float a = bl[o];
        for (int k = 0; k < in; ++k) a = fmaf(Wl[o * in + k], hs[l - 1][k], a);
        hs[l][o] = simt_act(a, s.act);
        ds[l - 1][o] = simt_dact(a, s.act);
      }
      for (int k = 0; k < s.nh; ++k)
        if ((k == 0 ? s.ha0 : s.ha1) == l) {
          float a = sp[s.po.c[k]];
#pragma unroll
          for (int j = 0; j < W; ++j) a = fmaf(sp[s.po.u[k] + j], hs[l][j], a);
          e[k] = a;
        }
    }
    float z = sp[s.po.bout];
#pragma unroll
    for (int j = 0; j < W; ++j) z = fmaf(sp[s.po.wout + j], hs[s.L][j], z);
    const int yi = y[i] ? 1 : 0;
    const float w = yi ? alpha : beta;
    // Eq. (1): alpha y softplus(-z) + beta (1-y) softplus(z); gradient w (sigma - y) / B
    loss += w * softplusf(yi ? -z : z);
    const float gz = w * (1.f / (1.f + expf(-z)) - (float)yi) * invB;
    const int nl = 1 + s.nh;
    t.gout[i * nl] = gz;
    float ge[2] = {0.f, 0.f};
    for (int k = 0; k < s.nh; ++k) {
      loss += w * softplusf(yi ? -e[k] : e[k]);
      ge[k] = w * (1.f / (1.f + expf(-e[k])) - (float)yi) * invB;
      t.gout[i * nl + 1 + k] = ge[k];
    }
    const bool pred = z >= 0.f;
    st[0] = pred && yi; st[1] = pred && !yi; st[2] = !pred && yi; st[3] = !pred && !yi;
    // back-propagation: dh = dL/dh_l, delta_l = dh * [h_l > 0]
    float dh[W];
#pragma unroll
    for (int j = 0; j < W; ++j) dh[j] = gz * sp[s.po.wout + j];
    for (int l = s.L; l >= 1; --l) {
      for (int k = 0; k < s.nh; ++k)
        if ((k == 0 ? s.ha0 : s.ha1) == l) {
#pragma unroll
          for (int j = 0; j < W; ++j) dh[j] = fmaf(ge[k], sp[s.po.u[k] + j], dh[j]);
        }
      float* drow = t.dlt + ((int64_t)(l - 1) * n + i) * W;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        dh[j] *= ds[l - 1][j];
        drow[j] = dh[j];
      }
      float* hrow = t.h + ((int64_t)(l - 1) * n + i) * Wm;
      const int in = l == 1 ? s.din : W;
      for (int k = 0; k < in; ++k) hrow[k] = hs[l - 1][k];
      if (l > 1) {
        const float* Wl = sp + s.po.W[l - 1];
        float nd[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
          float a = 0.f;
#pragma unroll
          for (int o = 0; o < W; ++o) a = fmaf(dh[o], Wl[o * W + k], a);
          nd[k] = a;
        }
#pragma unroll
        for (int k = 0; k < W; ++k) dh[k] = nd[k];
      }
    }
    float* hrow = t.h + ((int64_t)s.L * n + i) * Wm;
#pragma unroll
    for (int j = 0; j < W; ++j) hrow[j] = hs[s.L][j];
  }
  // loss and batch statistics (logging only)
  for (int o = 16; o > 0; o >>= 1) loss += __shfl_xor_sync(0xFFFFFFFFu, loss, o);
  unsigned c[4];
  for (int k = 0; k < 4; ++k) c[k] = __popc(__ballot_sync(0xFFFFFFFFu, st[k] != 0));
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(loss_out, (double)loss * (double)invB);
    for (int k = 0; k < 4; ++k)
      if (c[k]) atomicAdd(stats + k, (unsigned long long)c[k]);
  }
}

// Gradient of parameter p: sum over rows r of f(r) * g(r) (fixed row order).
struct GradArgs {
  ParamOffsets po;
  int P, d0, W, L, nh, ha0, ha1, Wm;
  int64_t n;
};

__device__ __forceinline__ void param_terms(const GradArgs& g, const TrainScratch& t, int p,
                                            const float** A, int64_t* sa, const float** Bv,
                                            int64_t* sb) {
  // returns two row-strided streams whose products are summed; *Bv == nullptr -> sum of A
  const int W = g.W;
  const int nl = 1 + g.nh;
  for (int l = 0; l < g.L; ++l) {
    const int in = l == 0 ? g.d0 : W;
    if (p >= g.po.W[l] && p < g.po.W[l] + (int64_t)W * in) {
      int o = (int)((p - g.po.W[l]) / in), k = (int)((p - g.po.W[l]) % in);
      *A = t.dlt + (int64_t)l * g.n * W + o; *sa = W;
      *Bv = t.h + (int64_t)l * g.n * g.Wm + k; *sb = g.Wm;
      return;
    }
    if (p >= g.po.b[l] && p < g.po.b[l] + W) {
      *A = t.dlt + (int64_t)l * g.n * W + (p - g.po.b[l]); *sa = W;
      *Bv = nullptr;
      return;
    }
  }
  if (p >= g.po.wout && p < g.po.wout + W) {
    *A = t.gout; *sa = nl;
    *Bv = t.h + (int64_t)g.L * g.n * g.Wm + (p - g.po.wout); *sb = g.Wm;
    return;
  }
  if (p == g.po.bout) { *A = t.gout; *sa = nl; *Bv = nullptr; return; }
  for (int k = 0; k < g.nh; ++k) {
    int lk = k == 0 ? g.ha0 : g.ha1;
    if (p >= g.po.u[k] && p < g.po.u[k] + W) {
      *A = t.gout + 1 + k; *sa = nl;
      *Bv = t.h + (int64_t)lk * g.n * g.Wm + (p - g.po.u[k]); *sb = g.Wm;
      return;
    }
    if (p == g.po.c[k]) { *A = t.gout + 1 + k; *sa = nl; *Bv = nullptr; return; }
  }
  *A = nullptr;
}

__global__ void k_grad_partial(GradArgs g, TrainScratch t) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (p >= g.P) return;
  const float* A; const float* B; int64_t sa, sb;
  param_terms(g, t, p, &A, &sa, &B, &sb);
  const int64_t rows = (g.n + kGradChunks - 1) / kGradChunks;
  const int64_t r0 = chunk * rows, r1 = min(g.n, r0 + rows);
  float acc = 0.f;
  if (A) {
    if (B) {
      for (int64_t r = r0; r < r1; ++r) acc = fmaf(A[r * sa], B[r * sb], acc);
    } else {
      for (int64_t r = r0; r < r1; ++r) acc += A[r * sa];
    }
  }
  t.part[(int64_t)chunk * g.P + p] = acc;
}

__global__ void k_grad_sum(const float* __restrict__ part, int P, float* __restrict__ grad) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  float a = 0.f;
  for (int c = 0; c < kGradChunks; ++c) a += part[(int64_t)c * P + p];
  grad[p] = a;
}

cudaError_t launch_train_simt(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                              int64_t n_global, float alpha, float beta, cudaStream_t st) {
  SimtArgs s;
  s.po = m->po;
  s.P = (int)m->P;
  s.d0 = m->d0;
  s.L = m->d.hidden_layers;
  s.nh = m->d.n_heads;
  s.ha0 = m->d.head_after[0];
  s.ha1 = m->d.head_after[1];
  s.din = m->din;
  s.act = m->d.activation;
  s.pe = m->d.pe_depth;
  TrainScratch t = carve_simt(m, n);
  const float invB = 1.0f / (float)n_global;
  const size_t smem = sizeof(float) * m->P;
  const int blocks = (int)((n + 127) / 128);
  if (n > 0) {
    switch (m->d.width) {
#define NB_TRAIN_CASE(WW)                                                                    \
  case WW:                                                                                   \
    cudaFuncSetAttribute(k_train_fwd_bwd_simt<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                         \
    k_train_fwd_bwd_simt<WW><<<blocks, 128, smem, st>>>(m->theta, s, q, y, n, invB, alpha,   \
                                                        beta, t, m->d_loss, m->d_stats);     \
    break;
      NB_TRAIN_CASE(16)
      NB_TRAIN_CASE(32)
      default:
        return cudaErrorInvalidValue;
#undef NB_TRAIN_CASE
    }
  }
  GradArgs g;
  g.po = m->po;
  g.P = (int)m->P;
  g.d0 = m->din;  // layer-1 input features
  g.W = m->d.width;
  g.L = m->d.hidden_layers;
  g.nh = m->d.n_heads;
  g.ha0 = m->d.head_after[0];
  g.ha1 = m->d.head_after[1];
  g.Wm = std::max(g.W, g.d0);
  g.n = n;
  dim3 grid((g.P + 127) / 128, kGradChunks);
  k_grad_partial<<<grid, 128, 0, st>>>(g, t);
  k_grad_sum<<<(g.P + 255) / 256, 256, 0, st>>>(t.part, g.P, m->grad);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Adam (PyTorch semantics, R8) on the fp32 master weights.
__global__ void k_adam(float* __restrict__ th, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, int64_t P, float lr_over_bc1,
                       float inv_sqrt_bc2, float b1, float b2, float eps, float l1, float l2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    float gi = g[i] + reg_grad(th[i], l1, l2);
    float mi = b1 * m[i] + (1.f - b1) * gi;
    float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    th[i] -= lr_over_bc1 * mi / (sqrtf(vi) * inv_sqrt_bc2 + eps);
  }
}

// Adam fused with the bf16 re-pack (nb_adam.cuh adam_pack_one): the thread
// that updates parameter i also writes every packed copy of it.
__global__ void k_adam_pack(float* __restrict__ th, float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ g, int64_t P, AdamArgs h, PackArgs a) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x)
    adam_pack_one(i, g[i], th, m, v, h, a);
}

void adam_setup(nb_model* m, float lr, AdamArgs* h, PackArgs* a) {
  m->step += 1;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double bc1 = 1.0 - pow(b1, (double)m->step), bc2 = 1.0 - pow(b2, (double)m->step);
  a->theta = m->theta;
  a->out = m->packed;
  a->out_bwd = m->packed_bwd;
  a->bl = m->bl;
  a->pl = m->pl;
  a->po = m->po;
  a->W = m->d.width;
  a->L = m->d.hidden_layers;
  a->d0 = m->din;
  a->nh = m->d.n_heads;
  *h = AdamArgs{(float)(lr / bc1), (float)(1.0 / sqrt(bc2)), (float)b1, (float)b2, (float)eps, m->l1, m->l2};
}

cudaError_t launch_adam_pack(nb_model* m, float lr, cudaStream_t s) {
  AdamArgs h;
  PackArgs a;
  adam_setup(m, lr, &h, &a);
  int blocks = (int)std::min<int64_t>((m->P + 255) / 256, 1024);
  return launch_pdl(k_adam_pack, dim3(blocks), dim3(256), 0, s, true, m->theta, m->adam_m, m->adam_v,
                    (const float*)m->grad, m->P, h, a);
}

cudaError_t launch_adam(nb_model* m, float lr, cudaStream_t s) {
  m->step += 1;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double bc1 = 1.0 - pow(b1, (double)m->step), bc2 = 1.0 - pow(b2, (double)m->step);
  int blocks = (int)std::min<int64_t>((m->P + 255) / 256, 1024);
  k_adam<<<blocks, 256, 0, s>>>(m->theta, m->adam_m, m->adam_v, m->grad, m->P,
                                (float)(lr / bc1), (float)(1.0 / sqrt(bc2)), (float)b1, (float)b2,
                                (float)eps, m->l1, m->l2);
  return cudaGetLastError();
}

}  // namespace nb
