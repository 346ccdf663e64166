// nb_fwd_tc2.cu — fused forward + classify/count/calibrate for widths that do
// not fit one SM (w = 256, BASELINE.json configs[4]): CTA pairs on tcgen05
// cta_group::2 (M = 256 rows per MMA: 128 per CTA).  Same rows a1-a6 and the
// same arithmetic as nb_fwd_tc.cu.
//
// Each CTA of a 2-CTA cluster holds half of every layer's weight rows in shared
// memory (its "pair image", 196 KB for 6->256x4->1) and its own 128 rows of the
// tile-pair in TMEM: accumulator D (256 fp32 columns) + bf16 A (128 columns).
// The leader CTA's elected thread issues the pair's MMAs once both CTAs have
// staged A (a_full: one cluster-scope arrive per CTA after a CTA-wide named
// barrier) and commits them to both CTAs' acc_full barriers (multicast).
// 16 warps per CTA: warp w reads TMEM lane quarter w % 4 and column group
// w / 4 (64 columns); group 0 stages inputs and classifies.
// mbarrier waits spin without a suspend-time hint in this translation unit:
// the pair kernel's issuer and epilogue warps wake faster (measured: c5
// score 4.47 -> 4.39 ms per 2^24 boxes; no effect on the other kernels)
#define NB_MBAR_NOHINT 1
#include <cuda_bf16.h>

#include <cstdlib>

#include "nb_device.cuh"
#include "nb_fwd_tc.cuh"  // encode_cols_pe, sin_act (sine / PE pair kernels)
#include "nb_internal.cuh"

namespace nb {

struct TcParams2 {
  FwdArgs a;
  const uint8_t* packed;  // pl.pairs images
  PackLayout pl;
  int d0, L, nh, ha0, ha1;
  int act, pe;            // k_fwd_tc2p<EXT>: nb_activation and PE depth (R41, R42)
  int64_t num_pairs;      // 256-row tile pairs
  unsigned long long* trace;  // NB_TRACE builds: timeline of CTA 0 (k_fwd_tc2p)
};

#ifdef NB_TRACE
extern unsigned long long* g_trace_buffer;
#define NB_TR2(region, code)                                                       \
  do {                                                                             \
    if (blockIdx.x == 0 && p.trace && lane == 0 && tr_i < 2000) {                  \
      p.trace[((region) * 2000 + tr_i) * 2] = clock64();                          \
      p.trace[((region) * 2000 + tr_i) * 2 + 1] = (unsigned long long)(code);     \
      ++tr_i;                                                                      \
    }                                                                              \
  } while (0)
#else
#define NB_TR2(region, code) \
  do {                       \
  } while (0)
#endif

template <bool ONES>
__device__ __forceinline__ void encode_cols2(const float* x, int d0, uint32_t (&col)[8]) {
  uint32_t h[8], l[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    __nv_bfloat16 hi = __float2bfloat16_rn(x[j]);
    __nv_bfloat16 lo = __float2bfloat16_rn(x[j] - __bfloat162float(hi));
    h[j] = __bfloat16_as_ushort(hi);
    l[j] = __bfloat16_as_ushort(lo);
  }
  uint32_t e[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v = (k == j && j < d0) ? h[j] : v;
      v = (k == d0 + j && j < d0) ? l[j] : v;
    }
    if (ONES && k >= 2 * d0 && k < 2 * d0 + 3) v = 0x3F80u;  // layer 1's bias columns (R35)
    e[k] = v;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) col[c] = e[2 * c] | (e[2 * c + 1] << 16);
}

__device__ __forceinline__ void add2p(float& d0, float& d1, float a0, float a1, float b0,
                                      float b1) {
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fma2p(float& c0, float& c1, float a0, float a1, float b0,
                                      float b1) {
  asm("{.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%0, %1};\n\t"
      "fma.rn.f32x2 rc, ra, rb, rc;\n\tmov.b64 {%0, %1}, rc;}"
      : "+f"(c0), "+f"(c1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

template <int MODE>
__device__ __forceinline__ void classify2(uint32_t* cnt, uint32_t (&key)[3], bool valid, int y,
                                          float z, const float* e, int nh, const float* tau,
                                          unsigned int* flags, int invert = 0) {
  if (MODE == kCalibrate) {
    if (valid && (invert ? y == 0 : y == 1)) {
      key[0] = min(key[0], dkey(invert ? -z : z));
      if (nh > 0) key[1] = min(key[1], dkey(e[0]));
      if (nh > 1) key[2] = min(key[2], dkey(e[1]));
    }
  }
  if (MODE == kScore) {
    int bin;
    bool pred;
    if (nh > 0 && !(e[0] >= tau[1])) { pred = false; bin = 0; }
    else if (nh > 1 && !(e[1] >= tau[2])) { pred = false; bin = 1; }
    else { pred = z >= tau[0]; bin = pred ? 3 : 2; }
    const bool yy = y != 0;
    const bool nonfin = !isfinite(z) || (nh > 0 && !isfinite(e[0])) || (nh > 1 && !isfinite(e[1]));
    const unsigned full = 0xFFFFFFFFu;
    const uint32_t c0 = __popc(__ballot_sync(full, valid && pred && yy));
    const uint32_t c1 = __popc(__ballot_sync(full, valid && pred && !yy));
    const uint32_t c2 = __popc(__ballot_sync(full, valid && !pred && yy));
    const uint32_t c3 = __popc(__ballot_sync(full, valid && !pred && !yy));
    const uint32_t b0 = __popc(__ballot_sync(full, valid && bin == 0));
    const uint32_t b1 = __popc(__ballot_sync(full, valid && bin == 1));
    const uint32_t b2 = __popc(__ballot_sync(full, valid && bin == 2));
    const uint32_t b3 = __popc(__ballot_sync(full, valid && bin == 3));
    const uint32_t nf = __popc(__ballot_sync(full, valid && nonfin));
    if ((threadIdx.x & 31) == 0) {
      cnt[0] += c0; cnt[1] += c1; cnt[2] += c2; cnt[3] += c3;
      cnt[4] += b0; cnt[5] += b1; cnt[6] += b2; cnt[7] += b3; cnt[8] += nf;
    }
  }
  if (valid && y > 1) atomicOr(flags, kFlagLabel);
}

// BF: bias folding (R35) — layer 1's bias through the encoder's ones columns,
// layer l >= 1's through one K = 16 MMA of a per-layer ones block in TMEM
// (columns ONES0 + 8 (l - 1)) against the pair image's shared bias block.
template <int LC, int MODE, bool BF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_fwd_tc2(const TcParams2 p) {
  constexpr int W = 256, NWARP = 16, CPT = 64;
  const int L = LC ? LC : p.L;
  const int NH = p.nh;
  const int h0 = p.nh > 0 ? p.ha0 - 1 : -1, h1 = p.nh > 1 ? p.ha1 - 1 : -1;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t rank = cluster_rank();
  const uint32_t bar_off = (p.pl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  // [0] weights  [1] acc_full  [2] a_full (leader)  [3,4] stage  [5] pad
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  float* xch = reinterpret_cast<float*>(tmem_slot + 4);                   // [2][3 groups][128][3]
  uint32_t* ctr = reinterpret_cast<uint32_t*>(xch + 2 * 3 * 128 * 3);      // [16][12]
  float* qst = reinterpret_cast<float*>(ctr + NWARP * 12);                 // [2][128*8]
  uint8_t* yst = reinterpret_cast<uint8_t*>(qst + 2 * kTile * 8);          // [2][128]
  const uint32_t w_bar = smem_u32(bars), acc_full = smem_u32(bars + 1), a_full = smem_u32(bars + 2);
  auto stage_bar = [&](int b) { return smem_u32(bars + 3 + b); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(acc_full, 1);
      mbar_init(a_full, 2);
      mbar_init(stage_bar(0), 1);
      mbar_init(stage_bar(1), 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      const uint8_t* img = p.packed + (size_t)rank * p.pl.bytes;
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u)
        bulk_g2s(sbase + off, img + off, min(32768u, p.pl.bytes - off), w_bar);
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < NWARP * 12; i += blockDim.x) ctr[i] = 0u;
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  if (BF) {  // ones block of hidden layer l: bf16 1.0 at k = 3 (l - 1) .. 3 (l - 1) + 2
    if (warp < 4) {
      for (int l = 1; l < (LC ? LC : p.L); ++l) {
        uint32_t ones[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int k0 = 2 * c, k1 = 2 * c + 1, lo = 3 * (l - 1), hi = lo + 3;
          ones[c] = ((k0 >= lo && k0 < hi) ? 0x3F80u : 0u) | ((k1 >= lo && k1 < hi) ? 0x3F800000u : 0u);
        }
        tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 384u + 8u * (uint32_t)(l - 1), ones);
      }
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  mbar_wait(w_bar, 0);

  const int64_t n = p.a.n;
  const int64_t npairs = gridDim.x / 2;
  const int64_t pid = blockIdx.x / 2;
  const int qw = warp & 3, grp = warp >> 2, col0 = grp * CPT;
  const bool lead = grp == 0;
  const bool issuer = warp == 0 && lane == 0;      // stages records, signals the leader
  const bool leader = rank == 0;
  const int rit = qw * 32 + lane;                  // row within this CTA's half tile
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const uint32_t ACOL = 256;                       // bf16 A operand columns [256, 384)
  const uint32_t ONES0 = 384;                      // BF: ones blocks [384, 384 + 8 (L - 1))
  const float* bias_all = reinterpret_cast<const float*>(smem + p.pl.off_bias);
  const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout) + col0;
  const float bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
  const float* cst = reinterpret_cast<const float*>(smem + p.pl.off_c);
  const float* u0 = reinterpret_cast<const float*>(smem + p.pl.off_u[0]) + col0;
  const float* u1 = reinterpret_cast<const float*>(smem + p.pl.off_u[1]) + col0;
  uint32_t* cnt = ctr + warp * 12;
  uint32_t key[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
  const int nl = 1 + NH, d0 = p.d0;
  const uint32_t idesc = make_idesc_bf16(256, W);
  const uint32_t a_full_leader = mapa_shared(a_full, 0);
  uint32_t ph = 0, aph = 0;

  // Both CTAs staged the next A: CTA-wide named barrier, then one cluster
  // arrive per CTA on the leader's a_full; the leader issues layer l's MMAs.
  auto sync_and_issue = [&](int l) {
    tc_fence_before();
    asm volatile("bar.sync 1, 512;" ::: "memory");
    if (warp == 0) {
      if (lane == 0) mbar_arrive_remote_cta(a_full_leader);
      if (leader) {
        mbar_wait(a_full, aph);
        aph ^= 1u;
        tc_fence_after();
        if (elect_one()) {
          if (l == 0) {
            mma_ts2(tmem, tmem + ACOL, make_sdesc(sbase + p.pl.off_w[0], 128u, (kEncK / 8u) * 128u),
                    idesc, 0u);
          } else {
            if (BF)  // bias first: D = ones_l * [splits]^T, then D += A W^T
              mma_ts2(tmem, tmem + ONES0 + 8u * (uint32_t)(l - 1),
                      make_sdesc(sbase + p.pl.off_bb[0], 128u, (kEncK / 8u) * 128u), idesc, 0u);
            const uint64_t bd = make_sdesc(sbase + p.pl.off_w[l], 128u, (W / 8u) * 128u);
#pragma unroll
            for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
              mma_ts2(tmem, tmem + ACOL + kk * 8u, bd + (uint64_t)(kk * 16u), idesc,
                      (BF || kk > 0u) ? 1u : 0u);
          }
          mma_commit2(acc_full);
        }
      }
      __syncwarp();
    }
  };

  auto half_base = [&](int64_t t) { return t * 2 * kTile + (int64_t)rank * kTile; };
  auto full_half = [&](int64_t t) { return half_base(t) + kTile <= n; };
  auto stage_issue = [&](int64_t t, int b) {
    if (!issuer || t >= p.num_pairs || !full_half(t)) return;
    const uint32_t qb = (uint32_t)(kTile * d0 * 4);
    mbar_arrive_expect_tx(stage_bar(b), qb + (MODE != kForward ? (uint32_t)kTile : 0u));
    bulk_g2s(smem_u32(qst + b * kTile * 8), p.a.q + half_base(t) * d0, qb, stage_bar(b));
    if (MODE != kForward) bulk_g2s(smem_u32(yst + b * kTile), p.a.y + half_base(t), kTile, stage_bar(b));
  };
  uint32_t sph[2] = {0u, 0u};
  int ycur = 0;
  auto put_input = [&](int64_t t, int i) {
    if (lead) {
      float x[8];
      const int b = i & 1;
      if (full_half(t)) {
        mbar_wait(stage_bar(b), sph[b]);
        sph[b] ^= 1u;
        const float* qs = qst + b * kTile * 8 + rit * d0;
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = j < d0 ? qs[j] : 0.f;
        ycur = MODE != kForward ? (int)yst[b * kTile + rit] : 0;
      } else {
        const int64_t r = half_base(t) + rit;
        const bool v = r < n;
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = (v && j < d0) ? __ldg(p.a.q + r * d0 + j) : 0.f;
        ycur = (MODE != kForward && v) ? (int)__ldg(p.a.y + r) : 0;
      }
      uint32_t c[8];
      encode_cols2<BF>(x, d0, c);
      tmem_st8(trow + ACOL, c);
      if (MODE == kTrain && 2 * t + rank < p.a.tr.num_tiles) {  // layer-1 input image (dW GEMM)
        uint8_t* base = p.a.tr.x_img + (2 * t + rank) * img_tile_bytes(16);
#pragma unroll
        for (int fg = 0; fg < 2; ++fg)
          *reinterpret_cast<uint4*>(base + (fg * 16 + rit / 8) * 128 + (rit % 8) * 16) =
              make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
      }
      tmem_wait_st();
    }
    sync_and_issue(0);
  };

  int64_t tile = pid;
  stage_issue(tile, 0);
  stage_issue(tile + npairs, 1);
  int i_tile = 0;
  if (tile < p.num_pairs) put_input(tile, 0);
  uint32_t par = 0;
  while (tile < p.num_pairs) {
    const int64_t next = tile + npairs;
    int ythis = 0;
    float z0 = lead ? bout : 0.f, z1 = 0.f;
    float e0a = (lead && NH > 0) ? cst[0] : 0.f, e0b = 0.f;
    float e1a = (lead && NH > 1) ? cst[1] : 0.f, e1b = 0.f;
#pragma unroll
    for (int l = 0; l < (LC ? LC : kMaxLayers); ++l) {
      if (!LC && l >= L) break;
      mbar_wait(acc_full, ph);
      ph ^= 1u;
      tc_fence_after();
      if (l == 0) stage_issue(next + npairs, i_tile & 1);
      const bool last = (l == L - 1);
      const float* bias = bias_all + l * W + col0;
      uint32_t v[CPT];
      tmem_ld32(trow + (uint32_t)col0, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(trow + (uint32_t)col0 + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      if (last) {
        // the accumulator is in registers: stage the next tile-pair right away
        ythis = ycur;
        ++i_tile;
        if (next < p.num_pairs) put_input(next, i_tile);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float* t = reinterpret_cast<float*>(v + 32 * c);
        if (!BF) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + 32 * c + i);
            add2p(t[i], t[i + 1], t[i], t[i + 1], b4.x, b4.y);
            add2p(t[i + 2], t[i + 3], t[i + 2], t[i + 3], b4.z, b4.w);
          }
        }
        if (!last || MODE == kTrain) {
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = pack_relu_bf16x2(t[2 * j], t[2 * j + 1]);
          if (!last) tmem_st16(trow + ACOL + (uint32_t)((col0 + 32 * c) / 2), pk);
          if (MODE == kTrain && 2 * tile + rank < p.a.tr.num_tiles) {  // h_{l+1} image
            uint8_t* base = p.a.tr.h_img[l] + (2 * tile + rank) * img_tile_bytes(W);
            const int fg0 = (col0 + 32 * c) / 8;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<uint4*>(base + ((fg0 + i) * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                  make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
        if (l == h0 || l == h1 || last) {
#pragma unroll
          for (int i = 0; i < 32; ++i) t[i] = relu_nan(t[i]);
          const int o = 32 * c;
          if (l == h0) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) fma2p(e0a, e0b, t[i], t[i + 1], u0[o + i], u0[o + i + 1]);
          }
          if (l == h1) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) fma2p(e1a, e1b, t[i], t[i + 1], u1[o + i], u1[o + i + 1]);
          }
          if (last) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) fma2p(z0, z1, t[i], t[i + 1], wout[o + i], wout[o + i + 1]);
          }
        }
      }
      if (!last) {
        tmem_wait_st();
        sync_and_issue(l + 1);
      }
    }
    // combine the four column groups of each row (fixed order g0 + g1 + g2 + g3)
    float z = z0 + z1;
    float e[2] = {e0a + e0b, e1a + e1b};
    float* xb = xch + (size_t)par * 3 * 128 * 3;
    if (!lead) {
      float* o = xb + ((size_t)(grp - 1) * 128 + rit) * 3;
      o[0] = z;
      o[1] = e[0];
      o[2] = e[1];
    }
    asm volatile("bar.sync %0, 128;" ::"r"(2 + qw) : "memory");  // the 4 warps of quarter qw
    if (lead) {
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        const float* o = xb + ((size_t)g * 128 + rit) * 3;
        z += o[0];
        e[0] += o[1];
        e[1] += o[2];
      }
      const int64_t r = half_base(tile) + rit;
      const bool valid = r < n;
      if (MODE == kCalibrate && valid && !isfinite(z)) atomicOr(p.a.flags, kFlagNonFinite);
      if (MODE == kForward) {
        if (valid) {
          p.a.logits[r * nl] = z;
          if (NH > 0) p.a.logits[r * nl + 1] = e[0];
          if (NH > 1) p.a.logits[r * nl + 2] = e[1];
          if (p.a.prob) p.a.prob[r] = 1.f / (1.f + __expf(-z));
          if (!isfinite(z)) atomicOr(p.a.flags, kFlagNonFinite);
        }
      } else if (MODE == kTrain) {
        // Eq. (1): w = alpha if y else beta; term w softplus(-+z);
        // dL/dz = w (sigmoid(z) - y) / B; exit heads add the same term
        const float yf = (float)ythis;
        const float w = valid ? (ythis ? p.a.tr.alpha : p.a.tr.beta) : 0.f;
        auto sp = [](float u) { return fmaxf(u, 0.f) + log1pf(__expf(-fabsf(u))); };
        float lsum = w * sp(ythis ? -z : z);
        const float gz = w * (1.f / (1.f + __expf(-z)) - yf) * p.a.tr.inv_b;
        float ge[2] = {0.f, 0.f};
        for (int k = 0; k < NH; ++k) {
          lsum += w * sp(ythis ? -e[k] : e[k]);
          ge[k] = w * (1.f / (1.f + __expf(-e[k])) - yf) * p.a.tr.inv_b;
        }
        if (valid) {
          p.a.tr.g32[r * 3] = gz;
          p.a.tr.g32[r * 3 + 1] = ge[0];
          p.a.tr.g32[r * 3 + 2] = ge[1];
        }
        if (2 * tile + rank < p.a.tr.num_tiles) {
          uint8_t* hb = p.a.tr.hd_img + (2 * tile + rank) * img_tile_bytes(8) + (rit / 8) * 128 +
                        (rit % 8) * 16;
          *reinterpret_cast<uint4*>(hb) =
              make_uint4(pack_bf16x2(gz, ge[0]), pack_bf16x2(ge[1], 0.f), 0u, 0u);
        }
        for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xFFFFFFFFu, lsum, o);
        const bool pred = z >= 0.f, yy = ythis != 0;
        const uint32_t c0 = __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && yy));
        const uint32_t c1 = __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && !yy));
        const uint32_t c2 = __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && yy));
        const uint32_t c3 = __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && !yy));
        if (lane == 0) {
          atomicAdd(p.a.tr.loss, (double)lsum * (double)p.a.tr.inv_b);
          cnt[0] += c0; cnt[1] += c1; cnt[2] += c2; cnt[3] += c3;
        }
      } else {
        classify2<MODE>(cnt, key, valid, ythis, z, e, NH, p.a.tau, p.a.flags, p.a.invert);
      }
    }
    par ^= 1u;
    tile = next;
  }
  if (MODE == kTrain && lead && lane == 0) {
    for (int i = 0; i < 4; ++i)
      if (cnt[i]) atomicAdd(p.a.tr.stats + i, (unsigned long long)cnt[i]);
  }
  if (lead && MODE != kForward && MODE != kTrain) {
    if (MODE == kCalibrate) {
      for (int k = 0; k <= NH; ++k) {
        const uint32_t mk = __reduce_min_sync(0xFFFFFFFFu, key[k]);
        if (lane == 0 && mk != 0xFFFFFFFFu) atomicMin(p.a.keys + k, mk);
      }
    }

  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs (issued by the leader) and reads are done
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (MODE == kScore && warp == 1) flush_cta_counts(ctr, NWARP, NH, p.a.counts);
  if (MODE == kScore && warp == 1 && p.a.ticket) finalize_counts(p.a);
}


// ---------------------------------------------------------------------------
// Pipelined CTA-pair kernel (w = 256; forward / calibrate / score, no exit
// heads): the tensor pipe is kept busy through the epilogues.  One tile pair
// lives in TMEM at a time, but every layer is split into two N = 128 halves
// with their own accumulators and the activations are double-buffered:
//   TMEM  D_a [0, 128)   output features {0..63, 128..191} (image rows 0..63 of each CTA)
//         D_b [128, 256)  output features {64..127, 192..255} (image rows 64..127)
//         A0, A1 [256, 384), [384, 512)  bf16 activations (A_in of stage s = A[s & 1])
// A stage is one layer of one tile pair (stages run across tiles without a
// gap).  The 16 epilogue warps drain D_a, signal, then drain D_b and signal
// (warp w: TMEM lane quarter w % 4, 32 columns of each half); each signal is
// one arrive per CTA on the leader's mbarrier.  A 17th warp issues the pair's
// MMAs (leader CTA): for stage s + 1,
//   after "a done"(s): D_a's K-steps over the features half a produced
//                      (k in {0..3, 8..11}); layer 0: D_a's K = 16 step
//   after "b done"(s): D_a's remaining K-steps, commit acc_a; D_b's 16 K-steps
//                      (D_b is free only now), commit acc_b
// so D_a's epilogue overlaps D_b's MMAs and D_b's epilogue overlaps the next
// stage's first D_a K-steps.  Hidden-layer biases enter through one K = 16
// pair MMA per half and layer (R35: a constant ones A operand in shared
// memory, 8 rows repeated by SBO = 0, against the pair image's shared split
// bias block); layer 1's bias rides in the encoder's ones columns.
// An 18th warp combines each row's output-head partials in a fixed order
// (g0 + g1 + g2 + g3, each group's a-half then b-half) and classifies /
// calibrates / writes the logits, off the epilogue's critical path
// (partials double-buffered by tile parity, xfull / xfree mbarriers).
// D0: compile-time record width for the encoder (0: run time).  EXT: the
// paper's sine activation and NeRF positional encoding (
// R41, R42; run-time p.act / p.pe, D0 > 0 for PE): sin(z) epilogues and a
// K = 64 layer-1 operand in the PE layout (4 K-steps).
template <int LC, int MODE, int D0, bool EXT = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(576, 1) k_fwd_tc2p(const TcParams2 p) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  constexpr int W = 256, NEPI = 16, CPT = 32;
  const int L = LC ? LC : p.L;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t rank = cluster_rank();
  const uint32_t bar_off = (p.pl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  // [0] weights  [1] acc_a  [2] acc_b  [3] a_done (leader)  [4] b_done (leader)  [5,6] stage
  // [11] b_done1 (leader): the second half of every warp's D_b columns (split signal)
  // [7,8] xfull  [9,10] xfree
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  float* xch = reinterpret_cast<float*>(tmem_slot + 4);                   // [2][4 groups][128]
  uint32_t* ctr = reinterpret_cast<uint32_t*>(xch + 2 * 4 * 128);          // [12] classifier counters
  float* qst = reinterpret_cast<float*>(ctr + 16);                         // [2][128*8]
  uint8_t* yst = reinterpret_cast<uint8_t*>(qst + 2 * kTile * 8);          // [2][128] staged labels
  uint8_t* ylab = yst + 2 * kTile;                                          // [2][128] labels by tile parity
  // bias MMA A operands: per hidden layer l >= 1 one 8-row K = 16 core-matrix
  // pair with bf16 1.0 at k = 3 (l - 1) .. 3 (l - 1) + 2 (the columns of layer
  // l's bias split in the pair image's shared block); SBO = 0 repeats the 8
  // rows for all 128 rows of the tile
  uint8_t* ones = smem + (((uint32_t)(ylab + 2 * kTile - smem) + 127u) & ~127u);  // [L - 1][256 B]
  const uint32_t w_bar = smem_u32(bars), acc_a = smem_u32(bars + 1), acc_b = smem_u32(bars + 2);
  const uint32_t a_done = smem_u32(bars + 3), b_done = smem_u32(bars + 4), b_done1 = smem_u32(bars + 11);
  auto stage_bar = [&](int b) { return smem_u32(bars + 5 + b); };
  auto xfull = [&](int b) { return smem_u32(bars + 7 + b); };
  auto xfree = [&](int b) { return smem_u32(bars + 9 + b); };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(acc_a, 1);
      mbar_init(acc_b, 1);
      mbar_init(a_done, 2 * NEPI);  // one arrive per epilogue warp of both CTAs
      mbar_init(b_done, 2 * NEPI);
      mbar_init(b_done1, 2 * NEPI);
      mbar_init(stage_bar(0), 1);
      mbar_init(stage_bar(1), 1);
      for (int b = 0; b < 2; ++b) {
        mbar_init(xfull(b), NEPI);
        mbar_init(xfree(b), 1);
      }
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      const uint8_t* img = p.packed + (size_t)rank * p.pl.bytes;
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u)
        bulk_g2s(sbase + off, img + off, min(32768u, p.pl.bytes - off), w_bar);
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 16; i += blockDim.x) ctr[i] = 0u;
  const bool bias_mma = p.pl.bb_shared != 0;
  if (bias_mma) {
    for (int i = threadIdx.x; i < (L - 1) * 8 * 16; i += blockDim.x) {
      const int l = 1 + i / 128, r = (i / 16) % 8, kk = i % 16;
      const bool one = kk >= 3 * (l - 1) && kk < 3 * (l - 1) + 3;
      *reinterpret_cast<uint16_t*>(ones + (l - 1) * 256 + (kk / 8) * 128 + r * 16 + (kk % 8) * 2) =
          one ? (uint16_t)0x3F80u : (uint16_t)0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  mbar_wait(w_bar, 0);

  const int64_t n = p.a.n;
  const int64_t npairs = gridDim.x / 2;
  const int64_t pid = blockIdx.x / 2;
  const bool leader = rank == 0;
  const bool epi = warp < NEPI;
  const bool classifier = warp == NEPI + 1;
  const int qw = warp & 3, g = (warp >> 2) & 3;
  // my 32 columns of D_a / D_b and the output features they hold
  const int fa = g < 2 ? 32 * g : 128 + 32 * (g - 2);
  const int fb = g < 2 ? 64 + 32 * g : 192 + 32 * (g - 2);
  const uint32_t ca = (uint32_t)(32 * g), cb = 128u + (uint32_t)(32 * g);
  const int rit = qw * 32 + lane;                  // row within this CTA's half tile
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  auto acol = [](uint32_t b) { return 256u + 128u * b; };
  const float* bias_all = reinterpret_cast<const float*>(smem + p.pl.off_bias);
  const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout);
  const float bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
  uint32_t key = 0xFFFFFFFFu;
  const int d0 = D0 ? D0 : p.d0;
  const bool bias0 = p.pl.bias_l0 != 0;
  const uint32_t idesc = make_idesc_bf16(256, 128);
  const uint32_t a_done_leader = mapa_shared(a_done, 0), b_done_leader = mapa_shared(b_done, 0);
  const uint32_t b_done1_leader = mapa_shared(b_done1, 0);
  // B descriptors of layer l, image rows [64 h, 64 h + 64) of this CTA
  const bool sine = EXT && p.act == NB_SINE;
  const uint32_t k0steps = p.pl.k_of[0] / 16u;  // layer-1 K-steps (1; 4 with PE)
  auto bdesc = [&](int l, int h) {
    const uint32_t K = l == 0 ? p.pl.k_of[0] : (uint32_t)W;
    const uint32_t sbo = K / 8u * 128u;
    return make_sdesc(sbase + p.pl.off_w[l] + (uint32_t)h * 8u * sbo, 128u, sbo);
  };

  auto half_base = [&](int64_t t) { return t * 2 * kTile + (int64_t)rank * kTile; };
  auto full_half = [&](int64_t t) { return half_base(t) + kTile <= n; };
  const bool tma_thread = warp == 0 && lane == 0;
  auto stage_issue = [&](int64_t t, int b) {  // records (+ labels) of tile t -> staging buffer b
    if (!tma_thread || t >= p.num_pairs || !full_half(t)) return;
    const uint32_t qb = (uint32_t)(kTile * d0 * 4);
    mbar_arrive_expect_tx(stage_bar(b), qb + (MODE != kForward ? (uint32_t)kTile : 0u));
    bulk_g2s(smem_u32(qst + b * kTile * 8), p.a.q + half_base(t) * d0, qb, stage_bar(b));
    if (MODE != kForward) bulk_g2s(smem_u32(yst + b * kTile), p.a.y + half_base(t), kTile, stage_bar(b));
  };
  // column group 0: encode tile t (local index i) into A[abuf] columns 0..7, its labels into ylab[i & 1]
  auto encode = [&](int64_t t, int i, uint32_t abuf) {
    float x[8];
    const int b = i & 1;
    int yv = 0;
    if (full_half(t)) {
      mbar_wait(stage_bar(b), (uint32_t)(i >> 1) & 1u);
      const float* qs = qst + b * kTile * 8 + rit * d0;
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = j < d0 ? qs[j] : 0.f;
      yv = MODE != kForward ? (int)yst[b * kTile + rit] : 0;
    } else {
      const int64_t r = half_base(t) + rit;
      const bool v = r < n;
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (v && j < d0) ? __ldg(p.a.q + r * d0 + j) : 0.f;
      yv = (MODE != kForward && v) ? (int)__ldg(p.a.y + r) : 0;
    }
    // the classifier has finished tile i - 2 (same label / partial buffers)
    if (i >= 2) mbar_wait(xfree(b), (uint32_t)((i >> 1) - 1) & 1u);
    ylab[b * kTile + rit] = (uint8_t)yv;
    uint32_t c[8];
    if (EXT && D0 > 0 && p.pe > 0) {  // positional encoding: K = 64 PE operand layout (R42)
      uint32_t cp[32];
      encode_cols_pe<(D0 > 0 ? D0 : 1)>(x, p.pe, cp);
#pragma unroll
      for (int g4 = 0; g4 < 4; ++g4)
        tmem_st8(trow + acol(abuf) + 8u * (uint32_t)g4, *reinterpret_cast<const uint32_t(*)[8]>(cp + 8 * g4));
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = cp[j];
    } else {
      if (bias0) encode_cols2<true>(x, d0, c);
      else encode_cols2<false>(x, d0, c);
      tmem_st8(trow + acol(abuf), c);
    }
    if (MODE == kTrain && 2 * t + rank < p.a.tr.num_tiles) {  // layer-1 input image (dW GEMM)
      uint8_t* base = p.a.tr.x_img + (2 * t + rank) * img_tile_bytes(16);
#pragma unroll
      for (int fg = 0; fg < 2; ++fg)
        *reinterpret_cast<uint4*>(base + (fg * 16 + rit / 8) * 128 + (rit % 8) * 16) =
            make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
    }
  };
  // end of this warp's part of one half's epilogue (its D columns read, its A
  // columns written): one arrive per warp on the leader's barrier, no CTA-wide
  // barrier (the issuer waits for all 32 warps of the pair)
  // h: 0 = D_a, 1 = the first 16 of the warp's D_b columns, 2 = the other 16
  // (D_b is signalled in two parts so the issuer starts the next D_a's
  // K-steps over the first part's features while the second part is stored)
  auto signal = [&](int h) {
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_remote_cta(h == 0 ? a_done_leader : (h == 1 ? b_done_leader : b_done1_leader));
  };
  // the 4 column-group-0 warps finished reading a staging buffer
  auto g0_sync = [&]() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
  int tr_i = 0;
  (void)tr_i;
  const int tr_reg = warp == 16 ? 0 : (warp == 0 ? 1 : (warp == 8 ? 2 : (warp == 15 ? 3 : -1)));
  (void)tr_reg;

  if (warp == NEPI) {
    // ---------------- MMA issuer (leader CTA, one elected thread) ----------------
    if (leader) {
      uint32_t adph = 0, bdph = 0;
      auto bias_desc = [&](int h) {  // the pair image's shared bias block, rows [64 h, 64 h + 64)
        return make_sdesc(sbase + p.pl.off_bb[0] + (uint32_t)h * 8u * 256u, 128u, 256u);
      };
      auto ones_desc = [&](int l) { return make_sdesc(smem_u32(ones + (l - 1) * 256), 128u, 0u); };
      auto issue = [&](int ln, uint32_t ab) {
        mbar_wait(a_done, adph);
        adph ^= 1u;
        NB_TR2(0, 0 | (ln << 8));
        tc_fence_after();
        const uint32_t A = tmem + acol(ab);
        if (elect_one()) {
          if (ln == 0) {
            for (uint32_t kk = 0; kk < k0steps; ++kk)
              mma_ts2(tmem, A + kk * 8u, bdesc(0, 0) + (uint64_t)(kk * 16u), idesc, kk > 0 ? 1u : 0u);
            mma_commit2(acc_a);
          } else {
            const uint64_t bd = bdesc(ln, 0);
            if (bias_mma) mma_ss2(tmem, ones_desc(ln), bias_desc(0), idesc, 0u);  // D_a = b (split)
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
              const uint32_t kk = j < 4 ? j : j + 4;  // features 0..63, 128..191
              mma_ts2(tmem, A + kk * 8u, bd + (uint64_t)(kk * 16u), idesc, (bias_mma || j > 0) ? 1u : 0u);
            }
          }
        }
        __syncwarp();
        NB_TR2(0, 1 | (ln << 8));
        mbar_wait(b_done, bdph);
        tc_fence_after();
        if (ln > 0 && elect_one()) {  // K-steps over the features of D_b's first parts
          const uint64_t bd = bdesc(ln, 0);
#pragma unroll
          for (uint32_t j = 0; j < 4; ++j) {
            const uint32_t kk = (j < 2 ? 4u : 12u) + 2u * (j & 1u);  // features 64.., 96.., 192.., 224.. (+0..15)
            mma_ts2(tmem, A + kk * 8u, bd + (uint64_t)(kk * 16u), idesc, 1u);
          }
        }
        __syncwarp();
        mbar_wait(b_done1, bdph);
        bdph ^= 1u;
        NB_TR2(0, 2 | (ln << 8));
        tc_fence_after();
        if (elect_one()) {
          if (ln == 0) {
            for (uint32_t kk = 0; kk < k0steps; ++kk)
              mma_ts2(tmem + 128u, A + kk * 8u, bdesc(0, 1) + (uint64_t)(kk * 16u), idesc, kk > 0 ? 1u : 0u);
            mma_commit2(acc_b);
          } else {
            const uint64_t bd = bdesc(ln, 0), bd1 = bdesc(ln, 1);
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
              const uint32_t kk = (j < 2 ? 5u : 13u) + 2u * (j & 1u);  // the second parts (+16..31)
              mma_ts2(tmem, A + kk * 8u, bd + (uint64_t)(kk * 16u), idesc, 1u);
            }
            mma_commit2(acc_a);
            if (bias_mma) mma_ss2(tmem + 128u, ones_desc(ln), bias_desc(1), idesc, 0u);
#pragma unroll
            for (uint32_t kk = 0; kk < 16; ++kk)
              mma_ts2(tmem + 128u, A + kk * 8u, bd1 + (uint64_t)(kk * 16u), idesc,
                      (bias_mma || kk > 0) ? 1u : 0u);
            mma_commit2(acc_b);
          }
        }
        __syncwarp();
        NB_TR2(0, 3 | (ln << 8));
      };
      uint32_t s = 0;
      for (int64_t tile = pid; tile < p.num_pairs; tile += npairs)
        for (int l = 0; l < L; ++l, ++s) issue(l, s & 1u);
    }
  } else if (epi) {
    // ---------------- epilogue warps ----------------
    int64_t tile = pid;
    stage_issue(tile, 0);
    stage_issue(tile + npairs, 1);
    if (tile < p.num_pairs) {  // stage 0's input, then "stage -1 done" for both halves
      if (g == 0) {
        encode(tile, 0, 0u);
        g0_sync();
        stage_issue(tile + 2 * npairs, 0);  // buffer 0 consumed
      }
      signal(0);
      signal(1);
      signal(2);
    }
    uint32_t s = 0;  // stage counter (acc barrier parity, A buffer)
    int i_tile = 0;  // local tile index
    while (tile < p.num_pairs) {
      const int64_t next = tile + npairs;
      const bool has_next = next < p.num_pairs;
      float zp = 0.f, zq = 0.f;
      for (int l = 0; l < L; ++l, ++s) {
        const bool last = l == L - 1;
        const bool add_bias = l > 0 ? !bias_mma : !bias0;
        const uint32_t ao = acol((s + 1) & 1u);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(h ? acc_b : acc_a, s & 1u);
          if (tr_reg > 0) NB_TR2(tr_reg, (4 + h * 4) | (l << 8));
          tc_fence_after();
          uint32_t v[CPT];
          tmem_ld32(trow + (h ? cb : ca), v);
          tmem_wait_ld();
          float* t = reinterpret_cast<float*>(v);
          const int f0 = h ? fb : fa;
          if (add_bias) {
            const float* bias = bias_all + l * W + f0;
#pragma unroll
            for (int i = 0; i < CPT; i += 4) {
              const float4 b4 = *reinterpret_cast<const float4*>(bias + i);
              add2p(t[i], t[i + 1], t[i], t[i + 1], b4.x, b4.y);
              add2p(t[i + 2], t[i + 3], t[i + 2], t[i + 3], b4.z, b4.w);
            }
          }
          uint32_t pk[16];
          if (!last || MODE == kTrain) {
            if (sine) {
#pragma unroll
              for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(sin_act(t[2 * j]), sin_act(t[2 * j + 1]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) pk[j] = pack_relu_bf16x2(t[2 * j], t[2 * j + 1]);
            }
          }
          if (tr_reg > 0) NB_TR2(tr_reg, (5 + h * 4) | (l << 8));
          // 1) the accumulator columns are read: hand the issuer the next
          //    MMAs' operands first (D_b in two 16-feature parts, so the next
          //    D_a's K-steps over the first part start while the second is stored)
          if (!last) {
            if (h == 1) {
              tmem_st8(trow + ao + (uint32_t)(f0 / 2), *reinterpret_cast<const uint32_t(*)[8]>(pk));
              signal(1);
              tmem_st8(trow + ao + (uint32_t)(f0 / 2) + 8u, *reinterpret_cast<const uint32_t(*)[8]>(pk + 8));
              signal(2);
            } else {
              tmem_st16(trow + ao + (uint32_t)(f0 / 2), pk);
              signal(0);
            }
          } else if (h == 0) {
            if (g == 0 && has_next) encode(next, i_tile + 1, (s + 1) & 1u);  // the next tile's layer-1 operand
            signal(0);
          } else {
            signal(1);
            signal(2);
          }
          if (tr_reg > 0) NB_TR2(tr_reg, (6 + h * 4) | (l << 8));
          // 2) off the MMA critical path: the training images, the output head
          NB_CHECK(f0 % 32 == 0 && f0 + CPT <= W);
          if (MODE == kTrain && 2 * tile + rank < p.a.tr.num_tiles) {  // h_{l+1} image (R34 masks, dW)
            // core-matrix offset ((f0 / 8 + q4) * 16 + rit / 8) * 128 + (rit % 8) * 16 written as
            // f0 * 256 + (row part) + q4 * 2048 (f0 % 32 == 0): one base register, immediate
            // offsets per store (the per-(half, q4) offsets the compiler hoisted were spilled)
            uint8_t* base = p.a.tr.h_img[l] + (2 * tile + rank) * img_tile_bytes(W) +
                            ((uint32_t)f0 * 256u + (uint32_t)(rit / 8) * 128u + (uint32_t)(rit % 8) * 16u);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              *reinterpret_cast<uint4*>(base + q4 * 2048) =
                  make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
            if (p.a.tr.c_img[l]) {  // ReLU'(h) bit mask of my 32 features for the backward (R25, R34)
              uint32_t mw = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j)
                mw |= ((pk[j] & 0x7FFFu) ? 1u : 0u) << (2 * j) | ((pk[j] & 0x7FFF0000u) ? 1u : 0u) << (2 * j + 1);
              reinterpret_cast<uint32_t*>(p.a.tr.c_img[l] + (2 * tile + rank) * 4096)[(f0 / 32) * 128 + rit] = mw;
            }
          }
          if (last) {
            const float* wo = wout + f0;
            if (sine) {
#pragma unroll
              for (int i = 0; i < CPT; i += 2) fma2p(zp, zq, sin_act(t[i]), sin_act(t[i + 1]), wo[i], wo[i + 1]);
            } else {
#pragma unroll
              for (int i = 0; i < CPT; i += 2)
                fma2p(zp, zq, relu_nan(t[i]), relu_nan(t[i + 1]), wo[i], wo[i + 1]);
            }
            if (h == 1) {  // this group's partial of the output logit -> the classifier
              xch[((i_tile & 1) * 4 + g) * 128 + rit] = zp + zq;
              __syncwarp();
              if (lane == 0) mbar_arrive(xfull(i_tile & 1));
            }
          }
          if (h == 0 && last && has_next && g == 0) {  // staging buffer (i_tile + 1) & 1 consumed
            g0_sync();
            stage_issue(next + 2 * npairs, (i_tile + 1) & 1);
          }
        }
      }
      ++i_tile;
      tile = next;
    }
  } else if (classifier) {
    // ---------------- row combine + classify / calibrate / logits ----------------
    int i = 0;
    for (int64_t tile = pid; tile < p.num_pairs; tile += npairs, ++i) {
      const int b = i & 1;
      mbar_wait(xfull(b), (uint32_t)(i >> 1) & 1u);
      const float* xb = xch + b * 4 * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = 32 * j + lane;
        const float z = bout + (((xb[row] + xb[128 + row]) + xb[256 + row]) + xb[384 + row]);
        const int yv = ylab[b * kTile + row];
        const int64_t r = half_base(tile) + row;
        const bool valid = r < n;
        NB_CHECK(!valid || (r >= 0 && r < n));
        if (MODE == kForward) {
          if (valid) {
            p.a.logits[r] = z;
            if (p.a.prob) p.a.prob[r] = 1.f / (1.f + __expf(-z));
            if (!isfinite(z)) atomicOr(p.a.flags, kFlagNonFinite);
          }
        } else if (MODE == kTrain) {
          // Eq. (1): w = alpha if y else beta, term w softplus(-+z),
          // dL/dz = w (sigmoid(z) - y) / B (R4, R5); batch counts at z >= 0 (R31)
          const float w = valid ? (yv ? p.a.tr.alpha : p.a.tr.beta) : 0.f;
          const float sp = fmaxf(yv ? -z : z, 0.f) + log1pf(__expf(-fabsf(z)));
          float lsum = w * sp;
          const float gz = w * (1.f / (1.f + __expf(-z)) - (float)yv) * p.a.tr.inv_b;
          if (valid) {
            p.a.tr.g32[r * 3] = gz;
            p.a.tr.g32[r * 3 + 1] = 0.f;
            p.a.tr.g32[r * 3 + 2] = 0.f;
          }
          const int64_t rt = 2 * tile + rank;
          if (rt < p.a.tr.num_tiles)
            *reinterpret_cast<uint4*>(p.a.tr.hd_img + rt * img_tile_bytes(8) + (row / 8) * 128 + (row % 8) * 16) =
                make_uint4(pack_bf16x2(gz, 0.f), 0u, 0u, 0u);
          for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xFFFFFFFFu, lsum, o);
          const bool pred = z >= 0.f, yy = yv != 0;
          const uint32_t c0 = __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && yy));
          const uint32_t c1 = __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && !yy));
          const uint32_t c2 = __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && yy));
          const uint32_t c3 = __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && !yy));
          if (lane == 0) {
            if (lsum != 0.f) atomicAdd(p.a.tr.loss, (double)lsum * (double)p.a.tr.inv_b);
            ctr[0] += c0; ctr[1] += c1; ctr[2] += c2; ctr[3] += c3;
          }
          if (valid && yv > 1) atomicOr(p.a.flags, kFlagLabel);
        } else if (MODE == kCalibrate) {
          if (valid && !isfinite(z)) atomicOr(p.a.flags, kFlagNonFinite);
          if (valid && (p.a.invert ? yv == 0 : yv == 1)) key = min(key, dkey(p.a.invert ? -z : z));
          if (valid && yv > 1) atomicOr(p.a.flags, kFlagLabel);
        } else {
          uint32_t k3[3] = {0u, 0u, 0u};
          classify2<MODE>(ctr, k3, valid, yv, z, nullptr, 0, p.a.tau, p.a.flags);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(xfree(b));
    }
    if (MODE == kCalibrate) {
      const uint32_t mk = __reduce_min_sync(0xFFFFFFFFu, key);
      if (lane == 0 && mk != 0xFFFFFFFFu) atomicMin(p.a.keys, mk);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs (issued by the leader) and reads are done
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  if (MODE == kTrain && warp == 1 && lane < 4 && ctr[lane]) atomicAdd(p.a.tr.stats + lane, (unsigned long long)ctr[lane]);
  if (MODE == kScore && warp == 1) flush_cta_counts(ctr, 1, 0, p.a.counts);
  if (MODE == kScore && warp == 1 && p.a.ticket) finalize_counts(p.a);
}

template <int LC, int MODE, int D0, bool EXT = false>
static cudaError_t launch_tc2p_m(const nb_model* m, const FwdArgs& a, cudaStream_t st) {
  TcParams2 p;
  p.a = a;
  p.packed = m->packed;
  p.pl = m->pl;
  p.d0 = m->d0;
  p.L = m->d.hidden_layers;
  p.nh = 0;
  p.ha0 = p.ha1 = 0;
  p.act = m->d.activation;
  p.pe = m->d.pe_depth;
#ifdef NB_TRACE
  p.trace = g_trace_buffer;
#else
  p.trace = nullptr;
#endif
  p.num_pairs = (a.n + 2 * kTile - 1) / (2 * kTile);
  if (p.num_pairs == 0) return cudaSuccess;
  const size_t smem = ((m->pl.bytes + 15) & ~15u) + 8 * 12 + 16 + sizeof(float) * 2 * 4 * 128 + 4 * 16 +
                      sizeof(float) * 2 * kTile * 8 + 4 * kTile + 128 + 256 * kMaxLayers;
  cudaError_t e = cudaFuncSetAttribute(k_fwd_tc2p<LC, MODE, D0, EXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int pairs = (int)std::min<int64_t>(p.num_pairs, m->num_sms / 2);
  return launch_pdl(k_fwd_tc2p<LC, MODE, D0, EXT>, dim3(2 * pairs), dim3(576), smem, st, MODE == kTrain, p);
}

// sine / PE pair kernels (forward, calibrate, score; generic layer count)
template <int D0>
static cudaError_t launch_tc2p_ext(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc2p_m<0, kForward, D0, true>(m, a, st);
  if (mode == kCalibrate) return launch_tc2p_m<0, kCalibrate, D0, true>(m, a, st);
  if (mode == kScore) return launch_tc2p_m<0, kScore, D0, true>(m, a, st);
  return cudaErrorInvalidValue;  // training of sine / PE pair nets: not built (nb_train_step refuses)
}

template <int LC, int D0>
static cudaError_t launch_tc2p_l(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc2p_m<LC, kForward, D0>(m, a, st);
  if (mode == kTrain) return launch_tc2p_m<LC, kTrain, D0>(m, a, st);
  if (mode == kCalibrate) return launch_tc2p_m<LC, kCalibrate, D0>(m, a, st);
  return launch_tc2p_m<LC, kScore, D0>(m, a, st);
}

bool tc2_supported(const nb_desc& d) {
  // layer 1 is one K = 16 step on CTA pairs: records of up to 6 floats
  const int r = d.kind == NB_POINT ? d.space_dim : 2 * d.space_dim;
  if (d.precision != NB_BF16 || d.width != 256 || d.hidden_layers < 1 || d.hidden_layers > kMaxLayers)
    return false;
  if (d.activation != NB_RELU || d.pe_depth > 0)  // sine / PE pairs: no exit heads; PE of 2D / 3D points
    return d.n_heads == 0 && (d.pe_depth == 0 ? enc_k(r) <= kEncK
                                              : (r == 2 || r == 3) && r * (1 + d.pe_depth) + 3 <= 32);
  return enc_k(r) <= kEncK;
}

template <int LC, int MODE, bool BF>
static cudaError_t launch_tc2_m(const nb_model* m, const FwdArgs& a, cudaStream_t st) {
  TcParams2 p;
  p.a = a;
  p.packed = m->packed;
  p.pl = m->pl;
  p.d0 = m->d0;
  p.L = m->d.hidden_layers;
  p.nh = m->d.n_heads;
  p.ha0 = m->d.head_after[0];
  p.ha1 = m->d.head_after[1];
  p.trace = nullptr;
  p.num_pairs = (a.n + 2 * kTile - 1) / (2 * kTile);
  if (p.num_pairs == 0) return cudaSuccess;
  const size_t smem = ((m->pl.bytes + 15) & ~15u) + 8 * 6 + 16 + sizeof(float) * 2 * 3 * 128 * 3 +
                      4 * 16 * 12 + sizeof(float) * 2 * kTile * 8 + 2 * kTile;
  cudaError_t e = cudaFuncSetAttribute(k_fwd_tc2<LC, MODE, BF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int pairs = (int)std::min<int64_t>(p.num_pairs, m->num_sms / 2);
  k_fwd_tc2<LC, MODE, BF><<<2 * pairs, 512, smem, st>>>(p);
  return cudaGetLastError();
}

template <int LC, bool BF>
static cudaError_t launch_tc2_l(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc2_m<LC, kForward, BF>(m, a, st);
  if (mode == kTrain) return launch_tc2_m<LC, kTrain, BF>(m, a, st);
  if (mode == kCalibrate) return launch_tc2_m<LC, kCalibrate, BF>(m, a, st);
  return launch_tc2_m<LC, kScore, BF>(m, a, st);
}

// Measurement switch: the single-slot kernel for every mode (NB_TC2_SINGLE=1).
static bool tc2_single() {
  static const bool v = getenv("NB_TC2_SINGLE") != nullptr;
  return v;
}

cudaError_t launch_fwd_tc2(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (m->d.activation != NB_RELU || m->d.pe_depth > 0) {  // sine / PE (R41, R42)
    if (m->d.pe_depth == 0) return launch_tc2p_ext<0>(m, mode, a, st);
    if (m->d0 == 2) return launch_tc2p_ext<2>(m, mode, a, st);
    if (m->d0 == 3) return launch_tc2p_ext<3>(m, mode, a, st);
    return cudaErrorInvalidValue;
  }
  if (m->d.n_heads == 0 && !tc2_single()) {  // pipelined halves
    if (m->d.hidden_layers == 4 && m->d0 == 6) return launch_tc2p_l<4, 6>(m, mode, a, st);  // BJ configs[4]
    return launch_tc2p_l<0, 0>(m, mode, a, st);
  }
  const bool bf = m->pl.bias_l0 && m->pl.bb_shared;
  if (m->d.hidden_layers == 4)
    return bf ? launch_tc2_l<4, true>(m, mode, a, st) : launch_tc2_l<4, false>(m, mode, a, st);
  return bf ? launch_tc2_l<0, true>(m, mode, a, st) : launch_tc2_l<0, false>(m, mode, a, st);
}

}  // namespace nb
