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
};

__device__ __forceinline__ uint32_t img_off2(int r, int fg) {
  return (uint32_t)((fg * 16 + r / 8) * 128 + (r % 8) * 16);
}

// 16 warps per CTA: warp w reads TMEM lane quarter w % 4 and column group
// w / 4 (64 of the 256 features of its 32 rows).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_bwd_tc2(const BwdParams2 p) {
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

cudaError_t launch_bwd_tc2(const nb_model* m, const uint8_t* const* h_img, uint8_t* const* d_img,
                           const float* g32, int64_t n, cudaStream_t st) {
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
  if (p.num_pairs == 0) return cudaSuccess;
  const size_t smem = ((m->bl.bytes + 15) & ~15u) + 64;
  cudaError_t e = cudaFuncSetAttribute(k_bwd_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int pairs = (int)std::min<int64_t>(p.num_pairs, m->num_sms / 2);
  k_bwd_tc2<<<2 * pairs, 512, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace nb
