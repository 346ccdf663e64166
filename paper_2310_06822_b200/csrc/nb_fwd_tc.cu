// nb_fwd_tc.cu — fused MLP forward + classify/count/calibrate on tcgen05
// tensor cores (sm_100a).  Hot-path rows a1-a6:
//   a1 encode (fp32 record -> bf16 hi/lo pair, in the epilogue warps),
//   a2/a3 layers z_l = W_l h_{l-1} + b_l on tcgen05.mma (M=128 rows per tile,
//         N = w, K = 16 or w; A = activations in TMEM, B = weights in SMEM),
//         epilogue bias + ReLU + RNE bf16 pack back into TMEM as the next A,
//   a4 output / exit-head dot products in fp32 on the epilogue threads,
//   a5/a6 classify with the calibrated thresholds and count (warp ballots),
//         or fold the positives' logits into the calibration minimum.
// Paper: MLP P:285-290 §3.4, early-out heads P:258-277 §3.3, cost cases
// P:157-176 §3.1.  Activations never leave the SM (TMEM is the tensor core's
// register file), weights are bulk-copied into shared memory once per CTA.
//
// CTA = 9 warps, persistent over 128-row tiles.  Warps 0-3 (slot 0) and 4-7
// (slot 1) each own one tile in flight and run its epilogues; warp 8 issues
// the MMAs, alternating slot 0 / slot 1 layer by layer so that one slot's
// epilogue overlaps the other slot's MMAs.  Synchronisation: mbarriers
// a_full[s] (epilogue -> MMA: next A operand is in TMEM) and acc_full[s]
// (tcgen05.commit -> epilogue: accumulator ready).
#include <cuda_bf16.h>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

struct TcParams {
  FwdArgs a;
  const uint8_t* packed;
  PackLayout pl;
  int d0, L, nh, ha0, ha1;
  int64_t num_tiles;
};

__device__ __forceinline__ void encode_cols(const float* x, int d0, uint32_t (&col)[8]) {
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

template <int W>
struct TcShape {
  static constexpr int kCols = (3 * W <= 256) ? 256 : 512;  // TMEM allocation
  __device__ static constexpr uint32_t acc_col(int s) { return (uint32_t)(s * W); }
  __device__ static constexpr uint32_t a_col(int s) { return (uint32_t)(2 * W + s * (W / 2)); }
};

template <int W, int MODE>
__global__ void __launch_bounds__(288, 1) k_fwd_tc(const TcParams p) {
  static_assert(W % 32 == 0 && W >= 32 && W <= 128, "tile plan covers w = 32..128");
  using S = TcShape<W>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_off = (p.pl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  const uint32_t w_bar = smem_u32(bars + 0);
  const uint32_t a_full[2] = {smem_u32(bars + 1), smem_u32(bars + 2)};
  const uint32_t acc_full[2] = {smem_u32(bars + 3), smem_u32(bars + 4)};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 8) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(a_full[0], 128);
      mbar_init(a_full[1], 128);
      mbar_init(acc_full[0], 1);
      mbar_init(acc_full[1], 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u) {
        uint32_t len = min(32768u, p.pl.bytes - off);
        bulk_g2s(sbase + off, p.packed + off, len, w_bar);
      }
    }
    __syncwarp();
    tmem_alloc<S::kCols>(smem_u32(tmem_slot));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  mbar_wait(w_bar, 0);

  const int64_t n = p.a.n;
  const int64_t G = gridDim.x;

  if (warp == 8) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(128, W);
      uint32_t ph[2] = {0u, 0u};
      for (int64_t jp = 0;; jp += 2) {
        const int64_t t0 = blockIdx.x + jp * G;
        if (t0 >= p.num_tiles) break;
        const bool has1 = t0 + G < p.num_tiles;
        for (int l = 0; l < p.L; ++l) {
          const uint32_t K = p.pl.k_of[l];
          const uint32_t sbo = (K / 8u) * 128u;
          const uint32_t bimg = sbase + p.pl.off_w[l];
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (s == 1 && !has1) continue;
            mbar_wait(a_full[s], ph[s]);
            ph[s] ^= 1u;
            tc_fence_after();
            const uint32_t d = tmem + S::acc_col(s);
            const uint32_t a = tmem + S::a_col(s);
            for (uint32_t kk = 0; kk < K / 16u; ++kk)
              mma_ts(d, a + kk * 8u, make_sdesc(bimg + kk * 256u, 128u, sbo), idesc, kk > 0u);
            mma_commit(acc_full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps ----------------
    const int s = warp >> 2;           // tile slot
    const int qw = warp & 3;           // TMEM lane quarter
    const int rit = qw * 32 + lane;    // row within the tile
    const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
    const float* bias_all = reinterpret_cast<const float*>(smem + p.pl.off_bias);
    const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout);
    const float bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
    const float* cst = reinterpret_cast<const float*>(smem + p.pl.off_c);
    const float* u0 = reinterpret_cast<const float*>(smem + p.pl.off_u[0]);
    const float* u1 = reinterpret_cast<const float*>(smem + p.pl.off_u[1]);
    WarpAcc acc;
    acc.init();
    uint32_t ph = 0;
    const int nl = 1 + p.nh;

    int64_t tile = blockIdx.x + (int64_t)s * G;
    float x[8];
    int ycur = 0;
    auto load_row = [&](int64_t t, float (&xx)[8], int& yy) {
      const int64_t r = t * kTile + rit;
      const bool v = t < p.num_tiles && r < n;
#pragma unroll
      for (int j = 0; j < 8; ++j) xx[j] = (v && j < p.d0) ? __ldg(p.a.q + r * p.d0 + j) : 0.f;
      yy = (MODE != kForward && v) ? (int)__ldg(p.a.y + r) : 0;
    };
    auto put_input = [&](const float (&xx)[8]) {
      uint32_t c[8];
      encode_cols(xx, p.d0, c);
      tmem_st8(trow + S::a_col(s), c);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(a_full[s]);
    };
    if (tile < p.num_tiles) {
      load_row(tile, x, ycur);
      put_input(x);
    }
    while (tile < p.num_tiles) {
      const int64_t next = tile + 2 * G;
      float xn[8];
      int yn = 0;
      load_row(next, xn, yn);
      float z = bout, e[2] = {cst[0], cst[1]};
      for (int l = 0; l < p.L; ++l) {
        mbar_wait(acc_full[s], ph);
        ph ^= 1u;
        tc_fence_after();
        const bool last = (l == p.L - 1);
        const int hk = (p.nh > 0 && p.ha0 == l + 1) ? 0 : ((p.nh > 1 && p.ha1 == l + 1) ? 1 : -1);
        const float* bias = bias_all + l * W;
        const float* uu = hk == 0 ? u0 : u1;
#pragma unroll
        for (int c = 0; c < W / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(trow + S::acc_col(s) + 32u * c, v);
          tmem_wait_ld();
          float t[32];
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + 32 * c + i);
            t[i + 0] = __uint_as_float(v[i + 0]) + b4.x;
            t[i + 1] = __uint_as_float(v[i + 1]) + b4.y;
            t[i + 2] = __uint_as_float(v[i + 2]) + b4.z;
            t[i + 3] = __uint_as_float(v[i + 3]) + b4.w;
          }
          if (hk >= 0) {
            float ek = e[hk];
#pragma unroll
            for (int i = 0; i < 32; ++i) ek = fmaf(fmaxf(t[i], 0.f), uu[32 * c + i], ek);
            e[hk] = ek;
          }
          if (!last) {
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack_relu_bf16x2(t[2 * j], t[2 * j + 1]);
            tmem_st16(trow + S::a_col(s) + 16u * c, pk);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) z = fmaf(fmaxf(t[i], 0.f), wout[32 * c + i], z);
          }
        }
        if (!last) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(a_full[s]);
        }
      }
      // this slot's A region is free again: stage the next tile's input
      if (next < p.num_tiles) put_input(xn);
      const int64_t r = tile * kTile + rit;
      const bool valid = r < n;
      if (MODE == kForward) {
        if (valid) {
          p.a.logits[r * nl] = z;
          if (p.nh > 0) p.a.logits[r * nl + 1] = e[0];
          if (p.nh > 1) p.a.logits[r * nl + 2] = e[1];
          if (p.a.prob) p.a.prob[r] = 1.f / (1.f + __expf(-z));
          if (!isfinite(z)) atomicOr(p.a.flags, kFlagNonFinite);
        }
      } else {
        classify_row<MODE>(acc, valid, ycur, z, e, p.nh, p.a.tau, p.a.flags);
      }
      tile = next;
      ycur = yn;
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = xn[j];
    }
    if (MODE != kForward) flush_warp<MODE>(acc, p.nh, p.a.counts, p.a.keys);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc<S::kCols>(tmem);
  }
}

bool tc_supported(const nb_desc& d) {
  if (d.precision != NB_BF16) return false;
  if (!(d.width == 32 || d.width == 64 || d.width == 128)) return false;
  if (d.hidden_layers < 1 || d.hidden_layers > kMaxLayers) return false;
  return true;
}

template <int W, int MODE>
static cudaError_t launch_tc_wm(const nb_model* m, const FwdArgs& a, cudaStream_t st) {
  TcParams p;
  p.a = a;
  p.packed = m->packed;
  p.pl = m->pl;
  p.d0 = m->d0;
  p.L = m->d.hidden_layers;
  p.nh = m->d.n_heads;
  p.ha0 = m->d.head_after[0];
  p.ha1 = m->d.head_after[1];
  p.num_tiles = (a.n + kTile - 1) / kTile;
  if (p.num_tiles == 0) return cudaSuccess;
  // one CTA per SM: the request also reserves > half of the SM's shared memory
  size_t smem = ((m->pl.bytes + 15) & ~15u) + 64;
  smem = std::max<size_t>(smem, 116 * 1024);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_tc<W, MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(p.num_tiles, m->num_sms);
  k_fwd_tc<W, MODE><<<grid, 288, smem, st>>>(p);
  return cudaGetLastError();
}

template <int W>
static cudaError_t launch_tc_w(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc_wm<W, kForward>(m, a, st);
  if (mode == kCalibrate) return launch_tc_wm<W, kCalibrate>(m, a, st);
  return launch_tc_wm<W, kScore>(m, a, st);
}

cudaError_t launch_fwd_tc(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  switch (m->d.width) {
    case 32: return launch_tc_w<32>(m, mode, a, st);
    case 64: return launch_tc_w<64>(m, mode, a, st);
    case 128: return launch_tc_w<128>(m, mode, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace nb
