// nb_adam.cuh — Adam (PyTorch semantics, "Adam ... 1e-3", R8)
// fused with the bf16 re-pack of one parameter, shared by k_adam_pack
// (nb_simt.cu, after a gradient allreduce) and the gradient reduce k_dw_reduce
// (nb_train_tc.cu, no communicator).  Product code only (no relation to oracle/).
#pragma once
#include <cuda_bf16.h>

#include "nb_internal.cuh"

namespace nb {

struct PackArgs {
  const float* theta;
  uint8_t* out;
  uint8_t* out_bwd;  // transposed pair images (w = 256) or NULL
  BwdLayout bl;
  PackLayout pl;
  ParamOffsets po;
  int W, L, d0, nh;
};

// Piece j of the exact three-way bf16 split b = hi + mid + lo (each piece is
// exactly representable in bf16; their fp32 sum is b for normal-range b).
__device__ __forceinline__ float bias_piece(float b, int j) {
  const float hi = __bfloat162float(__float2bfloat16_rn(b));
  const float r = b - hi;
  const float mid = __bfloat162float(__float2bfloat16_rn(r));
  const float lo = __bfloat162float(__float2bfloat16_rn(r - mid));
  return j == 0 ? hi : (j == 1 ? mid : lo);
}

// L1 + L2 regularisation (Suppl. §2.2; R38): the
// gradient of l1 * sum |theta| + l2 * sum theta^2 over all parameters.
__device__ __forceinline__ float reg_grad(float t, float l1, float l2) {
  return l1 * (t > 0.f ? 1.f : (t < 0.f ? -1.f : 0.f)) + 2.f * l2 * t;
}

struct AdamArgs {
  float lr_over_bc1, inv_sqrt_bc2, b1, b2, eps, l1, l2;
};

// Host: advance the model's Adam step counter and fill the step's arguments
// (bias corrections of step t, the model's pack layout) — nb_simt.cu.
void adam_setup(nb_model* m, float lr, AdamArgs* h, PackArgs* a);

__device__ __forceinline__ void store_bf16(uint8_t* img, int K, int n, int k, float v) {
  reinterpret_cast<__nv_bfloat16*>(img)[(int64_t)(n / 8) * (K / 8) * 64 + (k / 8) * 64 + (n % 8) * 8 +
                                        (k % 8)] = __float2bfloat16_rn(v);
}

// The Adam step of parameter i (gradient g_raw of Eq. (1), regularisation
// added here, R38) and every packed copy of it (weight image element(s),
// fp32 tail entries, bias split pieces) — the values k_pack_bf16 writes;
// padding positions of the image never change after the first full pack.
__device__ __forceinline__ void adam_pack_one(int64_t i, float g_raw, float* __restrict__ th,
                                              float* __restrict__ m, float* __restrict__ v,
                                              const AdamArgs& h, const PackArgs& a) {
  const int W = a.W, rows = W / (int)a.pl.pairs;
  const float gi = g_raw + reg_grad(th[i], h.l1, h.l2);
  const float mi = h.b1 * m[i] + (1.f - h.b1) * gi;
  const float vi = h.b2 * v[i] + (1.f - h.b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  const float t = th[i] - h.lr_over_bc1 * mi / (sqrtf(vi) * h.inv_sqrt_bc2 + h.eps);
  th[i] = t;
  // ---- re-pack parameter i
  auto fp32_tail = [&](uint32_t off_bytes) {  // replicated in every pair image
    for (uint32_t im = 0; im < a.pl.pairs; ++im)
      *reinterpret_cast<float*>(a.out + (size_t)im * a.pl.bytes + off_bytes) = t;
  };
  bool done = false;
  for (int l = 0; l < a.L && !done; ++l) {
    const int in = l == 0 ? a.d0 : W;
    const int64_t ow = a.po.W[l], ob = a.po.b[l];
    if (i >= ow && i < ow + (int64_t)W * in) {
      const int n = (int)((i - ow) / in), k = (int)((i - ow) % in);
      uint8_t* img = a.out + (size_t)(n / rows) * a.pl.bytes + a.pl.off_w[l];
      store_bf16(img, (int)a.pl.k_of[l], n % rows, k, t);
      if (l == 0)  // lo copy (after hi, or at pe_lo for PE nets)
        store_bf16(img, (int)a.pl.k_of[0], n % rows, (a.pl.pe_lo ? (int)a.pl.pe_lo : a.d0) + k, t);
      if (l > 0 && a.out_bwd)  // transposed pair image: row = input feature k, column = n
        store_bf16(a.out_bwd + (size_t)(k / rows) * a.bl.bytes + a.bl.off_wt[l], W, k % rows, n, t);
      done = true;
    } else if (i >= ob && i < ob + W) {
      const int n = (int)(i - ob);
      fp32_tail(a.pl.off_bias + 4u * (uint32_t)(l * W + n));
      uint8_t* imgb = a.out + (size_t)(n / rows) * a.pl.bytes;  // the image holding row n
      if (l == 0 && a.pl.bias_l0) {
        for (int j = 0; j < 3; ++j)
          store_bf16(imgb + a.pl.off_w[0], (int)a.pl.k_of[0], n % rows,
                     (a.pl.pe_lo ? 1 : 2) * a.d0 + j, bias_piece(t, j));
      } else if (l > 0 && a.pl.bb_shared) {
        for (int j = 0; j < 3; ++j)
          store_bf16(imgb + a.pl.off_bb[0], kEncK, n % rows, 3 * (l - 1) + j, bias_piece(t, j));
      } else if (l > 0 && a.pl.off_bb[l]) {
        for (int j = 0; j < 3; ++j) store_bf16(a.out + a.pl.off_bb[l], kEncK, n, j, bias_piece(t, j));
      }
      done = true;
    }
  }
  if (done) return;
  auto bwd_tail = [&](uint32_t off_bytes) {
    if (a.out_bwd)
      for (int im = 0; im < 2; ++im) *reinterpret_cast<float*>(a.out_bwd + (size_t)im * a.bl.bytes + off_bytes) = t;
  };
  if (i >= a.po.wout && i < a.po.wout + W) {
    fp32_tail(a.pl.off_wout + 4u * (uint32_t)(i - a.po.wout));
    bwd_tail(a.bl.off_wout + 4u * (uint32_t)(i - a.po.wout));
  } else if (i == a.po.bout) {
    fp32_tail(a.pl.off_bout);
  }
  for (int k = 0; k < a.nh; ++k) {
    if (i >= a.po.u[k] && i < a.po.u[k] + W) {
      fp32_tail(a.pl.off_u[k] + 4u * (uint32_t)(i - a.po.u[k]));
      bwd_tail(a.bl.off_u[k] + 4u * (uint32_t)(i - a.po.u[k]));
    } else if (i == a.po.c[k]) {
      fp32_tail(a.pl.off_c + 4u * (uint32_t)k);
    }
  }
}

}  // namespace nb
