// nb_train_tc2.cu — backward chain of the w = 256 bf16 training step (rows
// a7-a8 for BASELINE.json configs[4]) on CTA pairs (tcgen05 cta_group::2).
//
// Per 256-row tile pair, CTA v owns rows [128 v, 128 v + 128) (row-tile 2 t + v):
//   delta_L = (dL/dz w_out + sum_k dL/de_k u_k [l_k = L]) * [h_L > 0]
//   delta_{l-1} = (delta_l W_l + heads) * [h_{l-1} > 0]     (ReLU'(0) = 0, R25)
// The MMA is D[m][i] = sum_o delta[m][o] W_l[o][i]: M = 256 (both CTAs' rows,
// A = delta in each CTA's TMEM), N = 256 input features, K = 256 output
// features.  cta_group::2 splits B along N, so each CTA holds the transposed
// image of its 128 input features (BwdLayout, packed beside the forward
// images).  Same arithmetic as the single-CTA k_bwd_tc (nb_train_tc.cu):
// deltas rounded to bf16, masks from the bf16 activations (R34).
#include <cuda_bf16.h>

#include <cstdlib>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

struct BwdParams2 {
  const uint8_t* packed_bwd;  // 2 images
  BwdLayout bl;
  int L, nh, ha0, ha1;
  int64_t n, num_pairs, num_tiles;
  const uint8_t* h_img[kMaxLayers];  // h_1..h_L images (F = 256)
  uint8_t* d_img[kMaxLayers];        // delta_1..delta_L images (F = 256)
  const float* g32;                  // [n][3]
  const uint32_t* m_img[kMaxLayers]; // pipelined kernel: h_l > 0 bit masks (1024 words per row tile) or NULL
};

__device__ __forceinline__ uint32_t img_off2(int r, int fg) {
  return (uint32_t)((fg * 16 + r / 8) * 128 + (r % 8) * 16);
}

// 16 warps per CTA: warp w reads TMEM lane quarter w % 4 and column group
// w / 4 (64 of the 256 features of its 32 rows).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_bwd_tc2(const BwdParams2 p) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  constexpr int W = 256, CPT = 64;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t rank = cluster_rank();
  const uint32_t bar_off = (p.bl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);  // [0] image [1] acc_full [2] a_full
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const uint32_t w_bar = smem_u32(bars), acc_full = smem_u32(bars + 1), a_full = smem_u32(bars + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(acc_full, 1);
      mbar_init(a_full, 2);
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.bl.bytes);
      const uint8_t* img = p.packed_bwd + (size_t)rank * p.bl.bytes;
      for (uint32_t off = 0; off < p.bl.bytes; off += 32768u)
        bulk_g2s(sbase + off, img + off, min(32768u, p.bl.bytes - off), w_bar);
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  mbar_wait(w_bar, 0);

  const int qw = warp & 3, grp = warp >> 2, col0 = grp * CPT;
  const int rit = qw * 32 + lane;
  const bool leader = rank == 0;
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const uint32_t ACOL = 256;  // bf16 delta (A) columns [256, 384)
  const float* wout = reinterpret_cast<const float*>(smem + p.bl.off_wout);
  const float* u0 = reinterpret_cast<const float*>(smem + p.bl.off_u[0]);
  const float* u1 = reinterpret_cast<const float*>(smem + p.bl.off_u[1]);
  const int h0 = p.nh > 0 ? p.ha0 : -1, h1 = p.nh > 1 ? p.ha1 : -1;  // 1-based layers
  const uint32_t idesc = make_idesc_bf16(256, W);
  const uint32_t a_full_leader = mapa_shared(a_full, 0);
  uint32_t ph = 0, aph = 0;
  const int64_t npairs = gridDim.x / 2;

  for (int64_t t = blockIdx.x / 2; t < p.num_pairs; t += npairs) {
    const int64_t tile = 2 * t + rank;
    const bool have = tile < p.num_tiles;
    const int64_t r = tile * kTile + rit;
    const bool valid = have && r < p.n;
    const float gz = valid ? p.g32[r * 3] : 0.f;
    const float ge0 = valid ? p.g32[r * 3 + 1] : 0.f, ge1 = valid ? p.g32[r * 3 + 2] : 0.f;
    // h row of this warp's 64 features, loaded one layer ahead
    uint4 hcur[CPT / 8], hnext[CPT / 8];
    auto load_h = [&](uint4 (&h)[CPT / 8], int l1) {
      const uint8_t* hrow = p.h_img[l1 - 1] + tile * img_tile_bytes(W);
#pragma unroll
      for (int q = 0; q < CPT / 8; ++q)
        h[q] = have ? *reinterpret_cast<const uint4*>(hrow + img_off2(rit, col0 / 8 + q))
                    : make_uint4(0u, 0u, 0u, 0u);
    };
    load_h(hcur, p.L);
    for (int l = p.L; l >= 1; --l) {
      if (l > 1) load_h(hnext, l - 1);
      if (l < p.L) {
        mbar_wait(acc_full, ph);
        ph ^= 1u;
        tc_fence_after();
      }
      uint8_t* drow = p.d_img[l - 1] + tile * img_tile_bytes(W);
#pragma unroll
      for (int c = 0; c < CPT / 32; ++c) {
        uint32_t v[32];
        if (l < p.L) {
          tmem_ld32(trow + (uint32_t)(col0 + 32 * c), v);
          tmem_wait_ld();
        }
        float g[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = col0 + 32 * c + i;
          float d = (l < p.L) ? __uint_as_float(v[i]) : gz * wout[j];
          if (l == h0) d = fmaf(ge0, u0[j], d);
          if (l == h1) d = fmaf(ge1, u1[j], d);
          g[i] = d;
        }
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 hv = hcur[4 * c + q];
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 8 * q + 2 * e;
            const float m0 = (hw[e] & 0x7FFFu) ? g[i] : 0.f;  // h > 0 (h >= 0 by ReLU)
            const float m1 = (hw[e] & 0x7FFF0000u) ? g[i + 1] : 0.f;
            pk[4 * q + e] = pack_bf16x2(m0, m1);
          }
        }
        if (have) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(drow + img_off2(rit, (col0 + 32 * c) / 8 + q)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
        if (l >= 2) tmem_st16(trow + ACOL + (uint32_t)((col0 + 32 * c) / 2), pk);
      }
      if (l > 1) {
#pragma unroll
        for (int q = 0; q < CPT / 8; ++q) hcur[q] = hnext[q];
      }
      if (l >= 2) {
        // delta_l of both CTAs is in TMEM: the leader issues dL/dh_{l-1} = delta_l W_l
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync 1, 512;" ::: "memory");
        if (warp == 0) {
          if (lane == 0) mbar_arrive_remote_cta(a_full_leader);
          if (leader) {
            mbar_wait(a_full, aph);
            aph ^= 1u;
            tc_fence_after();
            if (elect_one()) {
              const uint64_t bd = make_sdesc(sbase + p.bl.off_wt[l - 1], 128u, (W / 8u) * 128u);
#pragma unroll
              for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
                mma_ts2(tmem, tmem + ACOL + kk * 8u, bd + (uint64_t)(kk * 16u), idesc, kk > 0u);
              mma_commit2(acc_full);
            }
          }
          __syncwarp();
        }
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
}


// ---------------------------------------------------------------------------
// Pipelined backward chain on CTA pairs (no exit heads): the k_fwd_tc2p plan
// applied to delta_{l-1} = (delta_l W_l) * [h_{l-1} > 0].  A stage is one
// layer l = L..1 of one tile pair; the MMA g_{l-1} = delta_l W_l (l >= 2) is
// split into two N = 128 halves of input features (D_a: rows 0..63 of each
// CTA's transposed image = features {0..63, 128..191}; D_b the rest) with
// double-buffered bf16 deltas as A.  16 epilogue warps handle 32 features of
// each half per row (mask from the h image prefetched one stage ahead, bf16
// round, delta image store, TMEM A store) and arrive per warp on the leader's
// a_done / b_done; a 17th warp issues the K-steps of D_a over half a's
// features after a_done, the rest and D_b after b_done.  Arithmetic equals
// k_bwd_tc2's (R34): same bf16 roundings, fp32 accumulation in the MMA.
template <bool BITS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(544, 1) k_bwd_tc2p(const BwdParams2 p) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  constexpr int W = 256, NEPI = 16, CPT = 32;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t rank = cluster_rank();
  const uint32_t bar_off = (p.bl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  // [0] image  [1] acc_a  [2] acc_b  [3] a_done (leader)  [4] b_done (leader)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  const uint32_t w_bar = smem_u32(bars), acc_a = smem_u32(bars + 1), acc_b = smem_u32(bars + 2);
  const uint32_t a_done = smem_u32(bars + 3), b_done = smem_u32(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(acc_a, 1);
      mbar_init(acc_b, 1);
      mbar_init(a_done, 2 * NEPI);
      mbar_init(b_done, 2 * NEPI);
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.bl.bytes);
      const uint8_t* img = p.packed_bwd + (size_t)rank * p.bl.bytes;
      for (uint32_t off = 0; off < p.bl.bytes; off += 32768u)
        bulk_g2s(sbase + off, img + off, min(32768u, p.bl.bytes - off), w_bar);
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);
  mbar_wait(w_bar, 0);

  const int L = p.L;
  const int64_t npairs = gridDim.x / 2;
  const bool leader = rank == 0;
  const int qw = warp & 3, g = (warp >> 2) & 3;
  const int fa = g < 2 ? 32 * g : 128 + 32 * (g - 2);
  const int fb = g < 2 ? 64 + 32 * g : 192 + 32 * (g - 2);
  const uint32_t ca = (uint32_t)(32 * g), cb = 128u + (uint32_t)(32 * g);
  const int rit = qw * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  auto acol = [](uint32_t b) { return 256u + 128u * b; };
  const float* wout = reinterpret_cast<const float*>(smem + p.bl.off_wout);
  const uint32_t idesc = make_idesc_bf16(256, 128);
  const uint32_t a_done_leader = mapa_shared(a_done, 0), b_done_leader = mapa_shared(b_done, 0);

  if (warp == NEPI) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader) {
      uint32_t adph = 0, bdph = 0, s = 0;
      for (int64_t t = blockIdx.x / 2; t < p.num_pairs; t += npairs) {
        for (int l = L; l >= 1; --l, ++s) {
          mbar_wait(a_done, adph);
          adph ^= 1u;
          tc_fence_after();
          const uint32_t A = tmem + acol(s & 1u);
          // B: transposed image of W_l, rows = this CTA's input features, K = 256 outputs
          const uint32_t sbo = (uint32_t)W / 8u * 128u;
          const uint64_t bd0 = make_sdesc(sbase + p.bl.off_wt[l - 1], 128u, sbo);
          const uint64_t bd1 = make_sdesc(sbase + p.bl.off_wt[l - 1] + 8u * sbo, 128u, sbo);
          if (l >= 2 && elect_one()) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
              const uint32_t kk = j < 4 ? j : j + 4;  // output features 0..63, 128..191
              mma_ts2(tmem, A + kk * 8u, bd0 + (uint64_t)(kk * 16u), idesc, j > 0 ? 1u : 0u);
            }
          }
          __syncwarp();
          mbar_wait(b_done, bdph);
          bdph ^= 1u;
          tc_fence_after();
          if (l >= 2 && elect_one()) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
              const uint32_t kk = j < 4 ? j + 4 : j + 8;
              mma_ts2(tmem, A + kk * 8u, bd0 + (uint64_t)(kk * 16u), idesc, 1u);
            }
            mma_commit2(acc_a);
#pragma unroll
            for (uint32_t kk = 0; kk < 16; ++kk)
              mma_ts2(tmem + 128u, A + kk * 8u, bd1 + (uint64_t)(kk * 16u), idesc, kk > 0 ? 1u : 0u);
            mma_commit2(acc_b);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < NEPI) {
    // ---------------- epilogue warps ----------------
    uint32_t s = 0, mph = 0;
    auto load_mask = [&](uint4 (&hm)[4], int64_t rt, int l1, int f0) {  // h_{l1} of features f0..f0+31
      const uint8_t* hrow = p.h_img[l1 - 1] + rt * img_tile_bytes(W);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        hm[q] = rt < p.num_tiles ? *reinterpret_cast<const uint4*>(hrow + ((f0 / 8 + q) * 16 + rit / 8) * 128 + (rit % 8) * 16)
                                 : make_uint4(0u, 0u, 0u, 0u);
    };
    // with bit masks (written by the forward) one word per half replaces the h loads
    constexpr bool bits = BITS;
    auto load_bits = [&](int64_t rt, int l1, int f0) -> uint32_t {
      return rt < p.num_tiles ? __ldg(p.m_img[l1 - 1] + rt * 1024 + (f0 / 32) * 128 + rit) : 0u;
    };
    uint4 hma[4], hmb[4];
    uint32_t mwa = 0, mwb = 0;
    int64_t t = blockIdx.x / 2;
    if (t < p.num_pairs) {
      if constexpr (bits) {
        mwa = load_bits(2 * t + rank, L, fa);
        mwb = load_bits(2 * t + rank, L, fb);
      } else {
        load_mask(hma, 2 * t + rank, L, fa);
        load_mask(hmb, 2 * t + rank, L, fb);
      }
    }
    for (; t < p.num_pairs; t += npairs) {
      const int64_t rt = 2 * t + rank;
      const bool have = rt < p.num_tiles;
      const int64_t r = rt * kTile + rit;
      const bool valid = have && r < p.n;
      const float gz = valid ? p.g32[r * 3] : 0.f;
      const int64_t tn = t + npairs;
      for (int l = L; l >= 1; --l, ++s) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f0 = h ? fb : fa;
          uint32_t v[CPT];  // g_l of my 32 features (fp32 bits)
          if (l < L) {
            mbar_wait(h ? acc_b : acc_a, mph);
            tc_fence_after();
            tmem_ld32(trow + (h ? cb : ca), v);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int i = 0; i < CPT; ++i) v[i] = __float_as_uint(gz * wout[f0 + i]);
          }
          const float* gv = reinterpret_cast<const float*>(v);
          uint4 (&hm)[4] = h ? hmb : hma;
          uint32_t& mw = h ? mwb : mwa;
          uint32_t pk[16];
          if constexpr (bits) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              pk[j] = pack_bf16x2(((mw >> (2 * j)) & 1u) ? gv[2 * j] : 0.f, ((mw >> (2 * j + 1)) & 1u) ? gv[2 * j + 1] : 0.f);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t hw[4] = {hm[q].x, hm[q].y, hm[q].z, hm[q].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int i = 8 * q + 2 * e;
                const float m0 = (hw[e] & 0x7FFFu) ? gv[i] : 0.f;  // h > 0 (h >= 0 by ReLU)
                const float m1 = (hw[e] & 0x7FFF0000u) ? gv[i + 1] : 0.f;
                pk[4 * q + e] = pack_bf16x2(m0, m1);
              }
            }
          }
          if (have) {
            uint8_t* drow = p.d_img[l - 1] + rt * img_tile_bytes(W);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<uint4*>(drow + ((f0 / 8 + q) * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                  make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
          if (l >= 2) tmem_st16(trow + acol(s & 1u) + (uint32_t)(f0 / 2), pk);
          // the next stage's mask (layer l - 1 of this tile, or layer L of the next)
          if constexpr (bits) {
            if (l > 1) mw = load_bits(rt, l - 1, f0);
            else if (tn < p.num_pairs) mw = load_bits(2 * tn + rank, L, f0);
          } else {
            if (l > 1) load_mask(hm, rt, l - 1, f0);
            else if (tn < p.num_pairs) load_mask(hm, 2 * tn + rank, L, f0);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote_cta(h ? b_done_leader : a_done_leader);
        }
        if (l < L) mph ^= 1u;
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
}

cudaError_t launch_bwd_tc2(const nb_model* m, const uint8_t* const* h_img, uint8_t* const* d_img,
                           const float* g32, int64_t n, cudaStream_t st, const uint8_t* const* m_img) {
  BwdParams2 p;
  p.packed_bwd = m->packed_bwd;
  p.bl = m->bl;
  p.L = m->d.hidden_layers;
  p.nh = m->d.n_heads;
  p.ha0 = m->d.head_after[0];
  p.ha1 = m->d.head_after[1];
  p.n = n;
  p.num_tiles = (n + kTile - 1) / kTile;
  p.num_pairs = (n + 2 * kTile - 1) / (2 * kTile);
  for (int l = 0; l < kMaxLayers; ++l) {
    p.h_img[l] = l < p.L ? h_img[l] : nullptr;
    p.d_img[l] = l < p.L ? d_img[l] : nullptr;
  }
  p.g32 = g32;
  for (int l = 0; l < kMaxLayers; ++l)
    p.m_img[l] = (m_img && l < p.L) ? reinterpret_cast<const uint32_t*>(m_img[l]) : nullptr;
  if (p.num_pairs == 0) return cudaSuccess;
  const size_t smem = ((m->bl.bytes + 15) & ~15u) + 64;
  const int pairs = (int)std::min<int64_t>(p.num_pairs, m->num_sms / 2);
  static const bool single = getenv("NB_TC2_SINGLE") != nullptr;  // measurement switch
  if (p.nh == 0 && p.L >= 2 && !single) {  // pipelined halves
    auto kern = p.m_img[0] ? k_bwd_tc2p<true> : k_bwd_tc2p<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(2 * pairs), dim3(544), smem, st, true, p);
  }
  cudaError_t e = cudaFuncSetAttribute(k_bwd_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_bwd_tc2, dim3(2 * pairs), dim3(512), smem, st, true, p);
}

}  // namespace nb
