// nb_train_fused.cu — the fused bf16 training step of BASELINE.json
// configs[1]'s architecture (w = 64, up to 4 hidden layers, no exit heads):
// forward, the asymmetric loss of Eq. (1) (Alg. 1),
// back-propagation and the dW / db GEMMs in ONE persistent kernel (rows a7,
// a8).  Per 128-row tile, everything stays on chip:
//   forward   layers on tcgen05 (A in TMEM, bias folded, R35); each h_l is also
//             written to shared memory as an MN-major row-tile image
//   loss      dL/dz = w (sigmoid(z) - y) / B, w = alpha | beta (Eq. 1, R4, R5)
//   backward  delta_l = g_l * [h_l > 0] (R25, R34); g_{l-1} = delta_l W_l on
//             tcgen05 (B = W_l read MN-major from the forward's image)
//   dW        D_l += delta_l^T [h_{l-1} | 1] (A = the delta image, B = the h
//             image followed by a constant ones block -> db), accumulated in
//             TMEM over all of the CTA's tiles; the head's dz^T [h_L | 1] rides
//             in row 64 of the last layer's delta image.
// At the end each CTA writes its dW accumulators as partials in the layout of
// nb_train_tc.cu's k_dw_tc; k_dw_reduce (fixed order), the NCCL allreduce
// (with a communicator) and k_adam_pack follow.  (Finishing the step inside
// this launch — grid barrier, reduce, Adam + re-pack — was measured slower
// than the two short launches: 53 vs 45 us per c2 step.)
// The backward issues g_{l-1} = delta_l W_l first and commits it on its own
// barrier, so the next layer's delta epilogue starts while the dW MMAs of
// layer l still run (they commit to dw_bar, waited before the delta image is
// rewritten).
// The arithmetic equals the unfused path (forward kTrain + k_bwd_tc + k_dw_tc):
// same bf16 roundings, same fp32 accumulations per tile.
#include <cuda_bf16.h>

#include <cmath>
#include <cstring>

#include "nb_fwd_tc.cuh"

namespace nb {

struct FusedParams {
  const uint8_t* packed;
  PackLayout pl;
  const float* q;
  const uint8_t* y;
  int64_t n, num_tiles;
  int L, d0;
  float alpha, beta, inv_b;
  double* loss;
  unsigned long long* stats;
  unsigned int* flags;
  float* partial;  // [job][cta][kDwColsF][128]
};
constexpr int kFusedW = 64;
constexpr int kDwColsF = 272;  // = nb_train_tc.cu kDwCols

// MN-major row-tile image element offset (bytes) of row r, feature group fg
__device__ __forceinline__ uint32_t fimg(int r, int fg) {
  return (uint32_t)((fg * 16 + r / 8) * 128 + (r % 8) * 16);
}

// TMEM columns: working D [0, 64), A [64, 96), forward ones block [96, 104),
// dW accumulators: job 0 [128, 160) (N = 16 + 16), hidden job l >= 1 at
// 160 + 80 (l - 1) (N = 64 + 16), head [400, 480).
__device__ __forceinline__ uint32_t dw_col(int job, int L) {
  return job == 0 ? 128u : (job <= L - 1 ? 160u + 80u * (uint32_t)(job - 1) : 400u);
}

// 8 warps: warp w owns TMEM lane quarter w % 4 (rows) and column half w / 4.
template <int LC>
__global__ void __launch_bounds__(256, 1) k_train_fused(const FusedParams p) {
  constexpr int W = kFusedW;
  const int L = LC ? LC : p.L;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  // layout: weights image | x image (16 + 16 ones features) | h_0..h_{L-1} images
  // (64 + 16 ones features each) | delta image (128 features) | barriers
  const uint32_t off_x = (p.pl.bytes + 1023u) & ~1023u;
  const uint32_t x_bytes = 32u * 256u;
  const uint32_t off_h = off_x + x_bytes;
  const uint32_t h_bytes = 80u * 256u;
  const uint32_t off_d = off_h + 4u * h_bytes;
  const uint32_t d_bytes = 128u * 256u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_d + d_bytes);  // [0] w [1] acc [2] dw
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  float* xz = reinterpret_cast<float*>(tmem_slot + 4);  // [128] head partial of half 1, then dz
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qw = warp & 3, hf = warp >> 2, col0 = 32 * hf;
  const int rit = qw * 32 + lane;  // row of the tile (lane quarter qw)
  const uint32_t w_bar = smem_u32(bars), acc_bar = smem_u32(bars + 1), dw_bar = smem_u32(bars + 2);
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      mbar_init(acc_bar, 1);
      mbar_init(dw_bar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u)
        bulk_g2s(sbase + off, p.packed + off, min(32768u, p.pl.bytes - off), w_bar);
    }
    __syncwarp();
    tmem_alloc<512>(smem_u32(tmem_slot));
  }
  // constant parts of the images: ones blocks (feature 0 = 1.0) after x and
  // each h; the delta image's features 64..127 start at zero
  for (int i = threadIdx.x; i < 128 * 2; i += blockDim.x) {
    const int r = i & 127, g = i >> 7;  // feature groups 0, 1 of a ones block
    const uint4 v = make_uint4(g == 0 ? 0x3F80u : 0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(smem + off_x + 16u * 256u + fimg(r, g)) = v;
    for (int l = 0; l < 4; ++l) *reinterpret_cast<uint4*>(smem + off_h + l * h_bytes + 64u * 256u + fimg(r, g)) = v;
  }
  for (int i = threadIdx.x; i < (int)(d_bytes / 16); i += blockDim.x)
    reinterpret_cast<uint4*>(smem + off_d)[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  if (warp < 4) {  // forward bias-folding ones block (k = 0, 1, 2 of every row)
    const uint32_t ones[8] = {0x3F803F80u, 0x00003F80u, 0u, 0u, 0u, 0u, 0u, 0u};
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 96u, ones);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(w_bar, 0);

  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const uint32_t DCOL = 0, ACOL = 64, ONES = 96;
  const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout) + col0;
  const float bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
  const uint32_t idesc_f = make_idesc_bf16(128, W);          // forward: A TMEM (K-major), B K-major
  const uint32_t idesc_b = make_idesc_bf16(128, W, 0, 1);    // backward: B = W_l read MN-major
  const uint32_t idesc_80 = make_idesc_bf16(128, 80, 1, 1);  // dW: A, B MN-major images
  const uint32_t idesc_32 = make_idesc_bf16(128, 32, 1, 1);
  const int d0 = p.d0;
  uint32_t ph = 0, dph = 0;
  bool first = true;  // no dW accumulation yet in this CTA
  uint32_t lcnt[4] = {0u, 0u, 0u, 0u};
  double lsum_all = 0.0;

  auto sync = [&]() {  // all warps: TMEM stores and smem image writes done
    tc_fence_before();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    tc_fence_after();
  };
  auto issue = [&](auto&& body) {
    if (warp == 0) {
      if (elect_one()) body();
      __syncwarp();
    }
  };
  auto wait_acc = [&]() {
    mbar_wait(acc_bar, ph);
    ph ^= 1u;
    tc_fence_after();
  };
  // K-major / MN-major descriptors
  auto wdesc = [&](int l) {  // forward B of layer l (K-major)
    return make_sdesc(sbase + p.pl.off_w[l], 128u, (l == 0 ? kEncK / 8u : W / 8u) * 128u);
  };
  auto mn_desc = [&](uint32_t off) { return make_sdesc(sbase + off, 128u, 2048u); };

  for (int64_t tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
    const int64_t r = tile * kTile + rit;
    const bool valid = r < p.n;
    int yv = 0;
    // the previous tile's dW job 0 reads the x image: wait for it
    if (!first) {
      mbar_wait(dw_bar, dph);
      dph ^= 1u;
    }
    if (hf == 0) {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (valid && j < d0) ? __ldg(p.q + r * d0 + j) : 0.f;
      yv = valid ? (int)__ldg(p.y + r) : 0;
      uint32_t c[8];
      encode_cols<0, true>(x, d0, c);
      tmem_st8(trow + ACOL, c);
      // x image features 0..15 (the encoded operand incl. the bias ones; the dW
      // reduce reads only the hi/lo columns and the ones block at 16)
#pragma unroll
      for (int fg = 0; fg < 2; ++fg)
        *reinterpret_cast<uint4*>(smem + off_x + fimg(rit, fg)) =
            make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
      tmem_wait_st();
    }
    sync();
    issue([&] {
      mma_ts(tmem + DCOL, tmem + ACOL, wdesc(0), idesc_f, 0u);
      mma_commit(acc_bar);
    });
    // ---------------- forward ----------------
    float zpart = 0.f;
    for (int l = 0; l < L; ++l) {
      wait_acc();
      uint32_t v[32];
      tmem_ld32(trow + DCOL + (uint32_t)col0, v);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack_relu_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
      // h_l image (MN-major) for the backward masks and the dW GEMMs
#pragma unroll
      for (int g = 0; g < 4; ++g)
        *reinterpret_cast<uint4*>(smem + off_h + l * h_bytes + fimg(rit, col0 / 8 + g)) =
            make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
      if (l < L - 1) {
        tmem_st16(trow + ACOL + (uint32_t)(col0 / 2), pk);
        tmem_wait_st();
        sync();
        issue([&] {
          mma_ts(tmem + DCOL, tmem + ONES, make_sdesc(sbase + p.pl.off_bb[l + 1], 128u, (kEncK / 8u) * 128u),
                 idesc_f, 0u);
          const uint64_t bd = wdesc(l + 1);
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk) mma_ts(tmem + DCOL, tmem + ACOL + kk * 8u, bd + kk * 16u, idesc_f, 1u);
          mma_commit(acc_bar);
        });
      } else {
        // output head in fp32 (R33): z = w_out . relu(z_L) + b_out, two column halves
        float za = 0.f, zb = 0.f;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          za = fmaf(fmaxf(__uint_as_float(v[j]), 0.f), wout[j], za);
          zb = fmaf(fmaxf(__uint_as_float(v[j + 1]), 0.f), wout[j + 1], zb);
        }
        zpart = za + zb;
      }
    }
    // ---------------- loss (Eq. 1) ----------------
    if (hf == 1) xz[rit] = zpart;
    __syncthreads();
    float dz = 0.f;
    if (hf == 0) {
      const float z = bout + (zpart + xz[rit]);
      const float yf = (float)yv;
      const float wgt = valid ? (yv ? p.alpha : p.beta) : 0.f;
      const float sp = fmaxf(yv ? -z : z, 0.f) + log1pf(__expf(-fabsf(z)));
      lsum_all += (double)(wgt * sp);
      dz = wgt * (1.f / (1.f + __expf(-z)) - yf) * p.inv_b;
      const bool pred = z >= 0.f, yy = yv != 0;
      lcnt[0] += __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && yy));
      lcnt[1] += __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && !yy));
      lcnt[2] += __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && yy));
      lcnt[3] += __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && !yy));
      if (valid && yv > 1) atomicOr(p.flags, kFlagLabel);
    }
    __syncthreads();
    if (hf == 0) xz[rit] = dz;
    __syncthreads();
    if (hf == 1) dz = xz[rit];
    // ---------------- backward + dW ----------------
    for (int l = L - 1; l >= 0; --l) {
      uint32_t v[32];
      if (l < L - 1) {
        wait_acc();  // g_l = delta_{l+1} W_{l+1} (and job l+1's dW MMAs before it)
        tmem_ld32(trow + DCOL + (uint32_t)col0, v);
        tmem_wait_ld();
      }
      // delta_l = g_l * [h_l > 0], rounded to bf16; written to the delta image
      // (features 0..63; feature 64 = dz for the head job on the last layer)
      uint32_t pk[16];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint4 hv = *reinterpret_cast<const uint4*>(smem + off_h + l * h_bytes + fimg(rit, col0 / 8 + g));
        const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = 8 * g + 2 * e;
          const float g0 = (l < L - 1) ? __uint_as_float(v[j]) : dz * wout[j];
          const float g1 = (l < L - 1) ? __uint_as_float(v[j + 1]) : dz * wout[j + 1];
          pk[4 * g + e] = pack_bf16x2((hw[e] & 0x7FFFu) ? g0 : 0.f, (hw[e] & 0x7FFF0000u) ? g1 : 0.f);
        }
      }
      if (l < L - 1) {  // the dW MMAs of layer l + 1 still read the delta image
        mbar_wait(dw_bar, dph);
        dph ^= 1u;
      }
#pragma unroll
      for (int g = 0; g < 4; ++g)
        *reinterpret_cast<uint4*>(smem + off_d + fimg(rit, col0 / 8 + g)) =
            make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
      if (hf == 0 && l == L - 1)  // dz in feature 64 (feature group 8, element 0)
        *reinterpret_cast<uint4*>(smem + off_d + fimg(rit, 8)) = make_uint4(pack_bf16x2(dz, 0.f), 0u, 0u, 0u);
      else if (hf == 0 && l == L - 2)  // cleared again (rows >= 64 of the other jobs are ignored)
        *reinterpret_cast<uint4*>(smem + off_d + fimg(rit, 8)) = make_uint4(0u, 0u, 0u, 0u);
      if (l >= 1) {
        tmem_st16(trow + ACOL + (uint32_t)(col0 / 2), pk);
        tmem_wait_st();
      }
      sync();
      const uint32_t acc0 = first ? 0u : 1u;
      issue([&] {
        const uint64_t ad = mn_desc(off_d);
        if (l == 0) {  // job 0: delta_0^T [x | 1] (N = 32)
          const uint64_t bd = mn_desc(off_x);
#pragma unroll
          for (uint32_t kk = 0; kk < 8; ++kk)
            mma_ss(tmem + dw_col(0, L), ad + kk * 16u, bd + kk * 16u, idesc_32, (acc0 || kk > 0u) ? 1u : 0u);
          mma_commit(dw_bar);
        } else {
          // g_{l-1} = delta_l W_l (B MN-major: K = out of layer l), committed
          // alone so the next delta epilogue need not wait for the dW MMAs
          const uint64_t bdesc = make_sdesc(sbase + p.pl.off_w[l], (W / 8u) * 128u, 128u);
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk)
            mma_ts(tmem + DCOL, tmem + ACOL + kk * 8u, bdesc + (uint64_t)((kk * 32u * W) >> 4), idesc_b, kk > 0u);
          mma_commit(acc_bar);
          // job l: delta_l^T [h_{l-1} | 1] (N = 80)
          const uint64_t bd = mn_desc(off_h + (l - 1) * h_bytes);
#pragma unroll
          for (uint32_t kk = 0; kk < 8; ++kk)
            mma_ss(tmem + dw_col(l, L), ad + kk * 16u, bd + kk * 16u, idesc_80, (acc0 || kk > 0u) ? 1u : 0u);
          if (l == L - 1) {  // head: row 64 of delta_{L-1}^T [h_{L-1} | 1]
            const uint64_t hd = mn_desc(off_h + (L - 1) * h_bytes);
#pragma unroll
            for (uint32_t kk = 0; kk < 8; ++kk)
              mma_ss(tmem + dw_col(L, L), ad + kk * 16u, hd + kk * 16u, idesc_80, (acc0 || kk > 0u) ? 1u : 0u);
          }
          mma_commit(dw_bar);
        }
      });
    }
    first = false;
  }
  // ---------------- flush ----------------
  if (!first) {  // the last tile's job 0
    mbar_wait(dw_bar, dph);
    tc_fence_after();
  }
  if (hf == 0 && lane == 0) {
    for (int i = 0; i < 4; ++i)
      if (lcnt[i]) atomicAdd(p.stats + i, (unsigned long long)lcnt[i]);
  }
  double ls = lsum_all;
  for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xFFFFFFFFu, ls, o);
  if (lane == 0 && ls != 0.0) atomicAdd(p.loss, ls * (double)p.inv_b);
  // dW accumulators -> partials (D row = thread row, column-major, coalesced)
  const int njobs = L + 1;
  for (int job = 0; job < njobs && hf == 0; ++job) {
    const int N = job == 0 ? 32 : 80;
    float* out = p.partial + ((int64_t)(job * gridDim.x + blockIdx.x) * kDwColsF) * 128 + rit;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t w[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
            "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]),
            "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
          : "r"(trow + dw_col(job, L) + (uint32_t)c0));
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) out[(int64_t)(c0 + i) * 128] = first ? 0.f : __uint_as_float(w[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

bool train_fused_supported(const nb_model* m) {
  const nb_desc& d = m->d;
  return d.precision == NB_BF16 && d.width == kFusedW && d.n_heads == 0 && d.hidden_layers >= 2 &&
         d.activation == NB_RELU && d.pe_depth == 0 &&
         d.hidden_layers <= 4 && m->pl.pairs == 1 && m->pl.bias_l0 && 2 * m->d0 + 3 <= kEncK;
}

size_t train_fused_smem(const nb_model* m) {
  const size_t off_x = (m->pl.bytes + 1023u) & ~(size_t)1023u;
  return off_x + 32 * 256 + 4 * 80 * 256 + 128 * 256 + 64 + 128 * 4;
}

cudaError_t launch_train_fused(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                               int64_t n_global, float alpha, float beta, float* partial,
                               int* cpj, cudaStream_t st) {
  FusedParams p;
  memset(&p, 0, sizeof(p));
  p.packed = m->packed;
  p.pl = m->pl;
  p.q = q;
  p.y = y;
  p.n = n;
  p.num_tiles = (n + kTile - 1) / kTile;
  p.L = m->d.hidden_layers;
  p.d0 = m->d0;
  p.alpha = alpha;
  p.beta = beta;
  p.inv_b = 1.0f / (float)n_global;
  p.loss = m->d_loss;
  p.stats = m->d_stats;
  p.flags = m->d_flags;
  p.partial = partial;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.num_tiles, m->num_sms));
  *cpj = grid;
  const size_t smem = train_fused_smem(m);
  auto kern = p.L == 4 ? k_train_fused<4> : k_train_fused<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace nb
