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
#include <cstdlib>
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
  unsigned long long* trace;  // NB_TRACE builds (tools/trace_fused.py)
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

// ---------------------------------------------------------------------------
// k_train_fused2: the same step with TWO row tiles in flight per CTA.
// Warps 0-3 run slot 0's epilogues, warps 4-7 slot 1's (warp w owns TMEM lane
// quarter w % 4 and all 64 columns), warp 8 is the MMA issuer: one thread
// walks a fixed program — step k of slot 0, step k of slot 1, step k + 1 of
// slot 0, ... — waiting on each slot's `ready` barrier, so one slot's
// epilogue overlaps the other's MMAs and the dW accumulation order is fixed
// (deterministic sums).  The dW GEMMs run transposed, D^T_l += [h_{l-1} | 1]^T
// delta_l (M = input features + the ones feature, N = 64), so the four
// accumulators plus the head's ([h_L | 1]^T dz, N = 16) take 272 TMEM columns
// and both slots' working sets fit beside them:
//   D_0 [0, 64)  D_1 [64, 128)  A_0 [128, 160)  A_1 [160, 192)  ones [192, 200)
//   dW job l at 224 + 64 l (l < 4), head at 480 (N = 16).
// Each slot's shared memory: x image (16 features + ones group), h_0..h_3
// images (64 features + ones group; h_{L-1} is also the delta image once the
// head MMA has read it), dz image (16 features, dz in feature 0); the
// backward takes ReLU' from the h images (read before h_{L-1}'s reuse).  An A
// operand spans 128 features = 32 KB from its image start: features beyond
// the image read the next buffer and land in TMEM lanes nobody reads.
// ---------------------------------------------------------------------------
constexpr uint32_t kF2X = 24u * 256u;         // x image: 16 features + ones group
constexpr uint32_t kF2H = 72u * 256u;         // h image: 64 features + ones group
constexpr uint32_t kF2DZ = 16u * 256u;        // dz image (head B operand, N = 16)
constexpr uint32_t kF2Slot = kF2X + 4u * kF2H + kF2DZ;
constexpr uint32_t kF2Pad = 32768u - (kF2H + kF2DZ);  // the last A span (h_3 of slot 1) stays in bounds
__host__ __device__ constexpr uint32_t f2_off_slot(uint32_t pl_bytes, int s) {
  return ((pl_bytes + 1023u) & ~1023u) + (uint32_t)s * kF2Slot;
}
__host__ __device__ constexpr uint32_t f2_bars(uint32_t pl_bytes) { return f2_off_slot(pl_bytes, 2) + kF2Pad; }

#ifdef NB_TRACE
extern unsigned long long* g_trace_buffer;
// tools/trace_fused.py: per CTA 64 (globaltimer, code) events; thread 0 uses
// [0, 16), slot s's warp 4 s lane 0 uses [16 + 24 s, 40 + 24 s)
#define NB_TRF(idx, code)                                                           \
  do {                                                                              \
    if (p.trace && (idx) < 64) {                                                    \
      uint64_t t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
      p.trace[((int64_t)blockIdx.x * 64 + (idx)) * 2] = t_;                         \
      p.trace[((int64_t)blockIdx.x * 64 + (idx)) * 2 + 1] = (unsigned long long)(code); \
    }                                                                               \
  } while (0)
// fine events of CTA 0 (clock64): region r (0 issuer, 1 + s slot s lead lane), 512 each
#define NB_TRC(region, code)                                                        \
  do {                                                                              \
    if (p.trace && blockIdx.x == 0 && trc < 512) {                                  \
      const int64_t b_ = 148 * 64 * 2 + ((int64_t)(region) * 512 + trc) * 2;        \
      p.trace[b_] = clock64();                                                      \
      p.trace[b_ + 1] = (unsigned long long)(code);                                 \
      ++trc;                                                                        \
    }                                                                               \
  } while (0)
#else
#define NB_TRF(idx, code) \
  do {                    \
  } while (0)
#define NB_TRC(region, code) \
  do {                       \
  } while (0)
#endif

template <int L>
__global__ void __launch_bounds__(288, 1) k_train_fused2(const FusedParams p) {
  constexpr int W = kFusedW;
  static_assert(L >= 2 && L <= 4, "fused2 plan");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + f2_bars(p.pl.bytes));
  // [0] weights, [1 + s] ready (TMEM operands), [3 + s] acc, [5 + s] head,
  // [7 + s] dw, [9 + s] ready (images).  Two ready barriers: consecutive
  // arrives on one of them are always separated by a wait on an MMA the
  // issuer launched for the earlier one, so no phase is overrun.
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t w_bar = smem_u32(bars);
  if (threadIdx.x == 0) NB_TRF(0, 0);
  if (warp == 8) {
    if (lane == 0) {
      mbar_init(w_bar, 1);
      for (int s = 0; s < 2; ++s) {
        mbar_init(smem_u32(bars + 1 + s), 4);
        mbar_init(smem_u32(bars + 3 + s), 1);
        mbar_init(smem_u32(bars + 5 + s), 1);
        mbar_init(smem_u32(bars + 7 + s), 1);
        mbar_init(smem_u32(bars + 9 + s), 4);
      }
      fence_barrier_init();
      // programmatic dependent of the previous step's gradient reduce (Adam +
      // re-pack): everything above overlaps its tail; the weights it wrote
      // are read only after the wait
      griddep_wait();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u)
        bulk_g2s(sbase + off, p.packed + off, min(32768u, p.pl.bytes - off), w_bar);
    }
    __syncwarp();
    tmem_alloc<512>(smem_u32(tmem_slot));
  }
  // constant image parts: the ones groups (feature 0 of the group = 1.0), the
  // dz images (only feature 0 is rewritten per tile) and the pad
  for (int i = threadIdx.x; i < 2 * 128; i += blockDim.x) {
    const int s = i >> 7, r = i & 127;
    const uint32_t so = f2_off_slot(p.pl.bytes, s);
    const uint4 one = make_uint4(0x3F80u, 0u, 0u, 0u), zero = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(smem + so + fimg(r, 2)) = one;
    for (int l = 0; l < 4; ++l) *reinterpret_cast<uint4*>(smem + so + kF2X + l * kF2H + fimg(r, 8)) = one;
    for (int g = 0; g < 2; ++g) *reinterpret_cast<uint4*>(smem + so + kF2X + 4 * kF2H + fimg(r, g)) = zero;
  }
  for (uint32_t i = threadIdx.x; i < kF2Pad / 16u; i += blockDim.x)
    reinterpret_cast<uint4*>(smem + f2_off_slot(p.pl.bytes, 2))[i] = make_uint4(0u, 0u, 0u, 0u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);
  constexpr uint32_t ONES = 192u, DW0 = 224u, HEAD = 480u;
  if (warp < 4) {  // forward bias-folding ones block (k = 0, 1, 2 of every row)
    const uint32_t ones[8] = {0x3F803F80u, 0x00003F80u, 0u, 0u, 0u, 0u, 0u, 0u};
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + ONES, ones);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // before any global access (batch, statistics, partials)
  mbar_wait(w_bar, 0);
  if (threadIdx.x == 0) NB_TRF(1, 1);
  const int64_t G = gridDim.x;
  const bool any = (int64_t)blockIdx.x < p.num_tiles;
  int tri = 16 + 24 * (warp >> 2);  // trace slot of this slot's lead lane

  // Per tile and slot, the epilogue signals `ready` ACTIONS = 3L times; action a
  // lets the issuer launch:
  //   0            layer 0 (A = encoded x)              -> acc
  //   1 .. L-1     layer l (A = h_{l-1} in TMEM)        -> acc
  //   L            g_{L-2} = delta_{L-1} W_{L-1}        -> acc
  //   L+1          head: [h_{L-1} | 1]^T dz             -> head
  //   then per l = L-2 .. 0: dW job l + 1 (delta_{l+1} image written, -> dw)
  //                and for l >= 1 g_{l-1} = delta_l W_l (-> acc);
  //   last         dW job 0                              -> dw
  // The chain (acc) never waits for an image write: TMEM operands are
  // signalled first; a delta image is written one chain step later, once the
  // MMA that read the buffer before (head, previous dW job) has finished.
  constexpr int ACTIONS = 3 * L;
  if (warp == 8) {
    // ---------------- MMA issuer (the warp waits, one elected lane issues) ----------------
    const uint32_t idesc_f = make_idesc_bf16(128, W);          // A TMEM, B K-major
    const uint32_t idesc_b = make_idesc_bf16(128, W, 0, 1);    // B = W_l read MN-major
    const uint32_t idesc_dw = make_idesc_bf16(128, 64, 1, 1);  // A, B MN-major images
    const uint32_t idesc_hd = make_idesc_bf16(128, 16, 1, 1);
    auto mn_desc = [&](uint32_t off) { return make_sdesc(sbase + off, 128u, 2048u); };
    uint32_t rph[2] = {0u, 0u}, sph[2] = {0u, 0u};
    int trc = 0;
    (void)trc;
    for (int64_t k = 0;; ++k) {
      const bool act[2] = {(int64_t)blockIdx.x + 2 * k * G < p.num_tiles,
                           (int64_t)blockIdx.x + (2 * k + 1) * G < p.num_tiles};
      if (!act[0]) break;
#pragma unroll
      for (int a = 0; a < ACTIONS; ++a) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (!act[s]) continue;
          const uint32_t so = f2_off_slot(p.pl.bytes, s);
          const uint32_t D = 64u * s, A = 128u + 32u * s;
          const uint32_t acc_bar = smem_u32(bars + 3 + s), dw_bar = smem_u32(bars + 7 + s);
          const bool first = k == 0 && s == 0;  // the CTA's first dW contribution
          // image actions: head, dW jobs; the rest wait on TMEM operands
          const bool img = a == L + 1 || a == ACTIONS - 1 || (a >= L + 2 && ((a - (L + 2)) & 1) == 0);
          if (img) {
            mbar_wait(smem_u32(bars + 9 + s), sph[s]);
            sph[s] ^= 1u;
          } else {
            mbar_wait(smem_u32(bars + 1 + s), rph[s]);
            rph[s] ^= 1u;
          }
          tc_fence_after();
          if (lane == 0) NB_TRC(0, 100 * s + a);
          auto g_mma = [&](int l) {  // g_{l-1} = delta_l W_l (B MN-major: K = out of layer l)
            const uint64_t bdesc = make_sdesc(sbase + p.pl.off_w[l], (W / 8u) * 128u, 128u);
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk)
              mma_ts(tmem + D, tmem + A + kk * 8u, bdesc + (uint64_t)((kk * 32u * W) >> 4), idesc_b, kk > 0u);
            mma_commit(acc_bar);
          };
          auto dw_mma = [&](int l) {  // [h_{l-1} | 1]^T delta_l (x image for l = 0); delta image = h_{L-1}'s buffer
            const uint64_t ad = mn_desc(so + (l == 0 ? 0u : kF2X + (l - 1) * kF2H));
            const uint64_t bd = mn_desc(so + kF2X + (L - 1) * kF2H);
#pragma unroll
            for (uint32_t kk = 0; kk < 8; ++kk)
              mma_ss(tmem + DW0 + 64u * l, ad + kk * 16u, bd + kk * 16u, idesc_dw, (!first || kk > 0u) ? 1u : 0u);
            mma_commit(dw_bar);
          };
          if (elect_one()) {
            if (a == 0) {
              mma_ts(tmem + D, tmem + A, make_sdesc(sbase + p.pl.off_w[0], 128u, (kEncK / 8u) * 128u), idesc_f, 0u);
              mma_commit(acc_bar);
            } else if (a < L) {
              mma_ts(tmem + D, tmem + ONES, make_sdesc(sbase + p.pl.off_bb[a], 128u, (kEncK / 8u) * 128u),
                     idesc_f, 0u);
              const uint64_t bd = make_sdesc(sbase + p.pl.off_w[a], 128u, (W / 8u) * 128u);
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk) mma_ts(tmem + D, tmem + A + kk * 8u, bd + kk * 16u, idesc_f, 1u);
              mma_commit(acc_bar);
            } else if (a == L) {
              g_mma(L - 1);
            } else if (a == L + 1) {
              const uint64_t ad = mn_desc(so + kF2X + (L - 1) * kF2H), bd = mn_desc(so + kF2X + 4 * kF2H);
#pragma unroll
              for (uint32_t kk = 0; kk < 8; ++kk)
                mma_ss(tmem + HEAD, ad + kk * 16u, bd + kk * 16u, idesc_hd, (!first || kk > 0u) ? 1u : 0u);
              mma_commit(smem_u32(bars + 5 + s));
            } else if (a < ACTIONS - 1) {
              const int j = a - (L + 2);  // dW job L-1-j/2 (even j), g_mma(L-2-(j-1)/2) (odd j)
              if ((j & 1) == 0) dw_mma(L - 1 - j / 2);
              else g_mma(L - 2 - (j - 1) / 2);
            } else {
              dw_mma(0);
            }
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---------------- epilogue warps of slot s ----------------
    const int s = warp >> 2, qw = warp & 3, rit = qw * 32 + lane;
    const uint32_t so = f2_off_slot(p.pl.bytes, s);
    const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
    const uint32_t D = 64u * s, A = 128u + 32u * s;
    const uint32_t ready = smem_u32(bars + 1 + s), ready_img = smem_u32(bars + 9 + s);
    const uint32_t acc_bar = smem_u32(bars + 3 + s);
    const uint32_t head_bar = smem_u32(bars + 5 + s), dw_bar = smem_u32(bars + 7 + s);
    const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout);
    const float bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
    uint8_t* ximg = smem + so;
    uint8_t* dimg = smem + so + kF2X + (L - 1) * kF2H;
    uint8_t* dzimg = smem + so + kF2X + 4 * kF2H;
    uint32_t aph = 0, hph = 0, dph = 0;
    int trc = 0;
    (void)trc;
    const bool lead = qw == 0 && lane == 0;
    uint32_t lcnt[4] = {0u, 0u, 0u, 0u};
    double lsum = 0.0;
    const int d0 = p.d0;
    // TMEM operand ready (tcgen05.st done): no shared-memory publication needed
    auto arrive_tm = [&]() {
      if (lead) NB_TRC(1 + s, 3);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ready);
    };
    // images written: publish the generic-proxy stores to the MMA (async proxy)
    auto arrive_sm = [&]() {
      if (lead) NB_TRC(1 + s, 5);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ready_img);
    };
    auto wait_acc = [&]() {
      if (lead) NB_TRC(1 + s, 1);
      mbar_wait(acc_bar, aph);
      aph ^= 1u;
      tc_fence_after();
      if (lead) NB_TRC(1 + s, 2);
    };
    auto wait_dw = [&]() {  // the last dW job issued has read its images
      mbar_wait(dw_bar, dph);
      dph ^= 1u;
    };
    auto ld64 = [&](uint32_t (&v)[64]) {
      tmem_ld32(trow + D, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(trow + D + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
    };
    auto put_img = [&](uint8_t* img, const uint32_t (&pk)[32]) {
#pragma unroll
      for (int g = 0; g < 8; ++g)
        *reinterpret_cast<uint4*>(img + fimg(rit, g)) = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
    };
    auto put_a = [&](const uint32_t (&pk)[32]) {
      tmem_st16(trow + A, *reinterpret_cast<const uint32_t(*)[16]>(pk));
      tmem_st16(trow + A + 16u, *reinterpret_cast<const uint32_t(*)[16]>(pk + 16));
      tmem_wait_st();
    };
    // ReLU' (R25): a bf16 half h >= 0 is nonzero iff (h & 0x7FFF) + 0x7FFF
    // carries into bit 15; the pair mask selects the packed gradient (a masked
    // half is +0, the same bits as rounding a masked 0)
    auto pair_mask = [](uint32_t hw) {
      const uint32_t t = ((hw & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x80008000u;
      return (t >> 15) * 0xFFFFu;
    };
    // the next tile's record and label are loaded one tile ahead
    float xn[8];
    int yn = 0;
    auto load_x = [&](int64_t t) {
      const int64_t r = t * kTile + rit;
      const bool ok = t < p.num_tiles && r < p.n;
#pragma unroll
      for (int j = 0; j < 8; ++j) xn[j] = (ok && j < d0) ? __ldg(p.q + r * d0 + j) : 0.f;
      yn = ok ? (int)__ldg(p.y + r) : 0;
    };
    int64_t tile = blockIdx.x + (int64_t)s * G;
    load_x(tile);
    bool first_tile = true;
    for (; tile < p.num_tiles; tile += 2 * G) {
      const bool valid = tile * kTile + rit < p.n;
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = xn[j];
      const int yv = yn;
      if (lead) NB_TRF(tri++, 10 + s);
      load_x(tile + 2 * G);
      if (!first_tile) wait_dw();  // the previous tile's dW job 0: x, h and delta images free
      {
        uint32_t c[8];
        encode_cols<0, true>(x, d0, c);
        tmem_st8(trow + A, c);
#pragma unroll
        for (int fg = 0; fg < 2; ++fg)
          *reinterpret_cast<uint4*>(ximg + fimg(rit, fg)) = make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
        tmem_wait_st();
      }
      arrive_tm();  // action 0 (the x image is published by the head action's arrive)
      // ---------------- forward ----------------
      float z = 0.f;
      uint32_t hL[32];  // h_{L-1}, packed
#pragma unroll
      for (int l = 0; l < L; ++l) {
        wait_acc();
        uint32_t v[64];
        ld64(v);
        if (lead) NB_TRC(1 + s, 4);
        if (l == L - 1) {
          // output head in fp32 (R33), summed as k_train_fused's two column halves
          float zh[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float za = 0.f, zb = 0.f;
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              za = fmaf(fmaxf(__uint_as_float(v[32 * h + j]), 0.f), wout[32 * h + j], za);
              zb = fmaf(fmaxf(__uint_as_float(v[32 * h + j + 1]), 0.f), wout[32 * h + j + 1], zb);
            }
            zh[h] = za + zb;
          }
          z = bout + (zh[0] + zh[1]);
#pragma unroll
          for (int j = 0; j < 32; ++j) hL[j] = pack_relu_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        } else {
          uint32_t pk[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) pk[j] = pack_relu_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
          put_a(pk);
          arrive_tm();                               // action l + 1
          put_img(smem + so + kF2X + l * kF2H, pk);  // h_l image (dW, ReLU'), published by a later arrive
        }
      }
      // ---------------- loss gradient and delta_{L-1} ----------------
      const float yf = (float)yv;
      const float wgt = valid ? (yv ? p.alpha : p.beta) : 0.f;
      const float dz = wgt * (__frcp_rn(1.f + __expf(-z)) - yf) * p.inv_b;  // rcp_rn(x) == 1.f / x
      // pd: the delta whose image (dW operand) is written one chain step later
      uint32_t pd[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) pd[j] = pack_bf16x2(dz * wout[2 * j], dz * wout[2 * j + 1]) & pair_mask(hL[j]);
      put_a(pd);
      arrive_tm();  // action L: g_{L-2}
      put_img(dimg, hL);  // h_{L-1} image (the head MMA's A)
      *reinterpret_cast<uint4*>(dzimg + fimg(rit, 0)) = make_uint4(pack_bf16x2(dz, 0.f), 0u, 0u, 0u);
      arrive_sm();  // action L + 1: head
      if (lead) NB_TRF(tri++, 20 + s);
      // ---------------- backward + dW ----------------
#pragma unroll
      for (int l = L - 2; l >= 0; --l) {
        uint4 hv[8];  // h_l image row (ReLU' of layer l)
#pragma unroll
        for (int g = 0; g < 8; ++g) hv[g] = *reinterpret_cast<const uint4*>(smem + so + kF2X + l * kF2H + fimg(rit, g));
        wait_acc();  // g_l = delta_{l+1} W_{l+1}
        uint32_t v[64];
        ld64(v);
        if (lead) NB_TRC(1 + s, 4);
        // delta_{l+1}'s image once its buffer is free (the head MMA read h_{L-1},
        // dW job l + 2 read delta_{l+2})
        if (l == L - 2) {
          mbar_wait(head_bar, hph);
          hph ^= 1u;
        } else {
          wait_dw();
        }
        put_img(dimg, pd);
        arrive_sm();  // dW job l + 1
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint4 q4 = hv[j >> 2];
          const uint32_t hw = (j & 3) == 0 ? q4.x : ((j & 3) == 1 ? q4.y : ((j & 3) == 2 ? q4.z : q4.w));
          pd[j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])) & pair_mask(hw);
        }
        if (l >= 1) {
          put_a(pd);
          arrive_tm();  // g_{l-1}
        }
      }
      wait_dw();  // dW job 1 has read delta_1
      put_img(dimg, pd);
      arrive_sm();  // dW job 0
      {  // loss value and batch counts at z >= 0 (off the chain)
        const float sp = fmaxf(yv ? -z : z, 0.f) + log1pf(__expf(-fabsf(z)));
        lsum += (double)(wgt * sp);
        const bool pred = z >= 0.f, yy = yv != 0;
        lcnt[0] += __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && yy));
        lcnt[1] += __popc(__ballot_sync(0xFFFFFFFFu, valid && pred && !yy));
        lcnt[2] += __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && yy));
        lcnt[3] += __popc(__ballot_sync(0xFFFFFFFFu, valid && !pred && !yy));
        if (valid && yv > 1) atomicOr(p.flags, kFlagLabel);
      }
      first_tile = false;
      if (lead) NB_TRF(tri++, 30 + s);
    }
    if (!first_tile) {  // the last tile's dW job 0
      wait_dw();
      tc_fence_after();
    }
    if (lane == 0) {
      for (int i = 0; i < 4; ++i)
        if (lcnt[i]) atomicAdd(p.stats + i, (unsigned long long)lcnt[i]);
    }
    double ls = lsum;
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xFFFFFFFFu, ls, o);
    if (lane == 0 && ls != 0.0) atomicAdd(p.loss, ls * (double)p.inv_b);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) NB_TRF(2, 2);
  // dW accumulators -> partials in k_dw_tc's layout ([col][128 D rows] per job
  // and CTA): TMEM lane f = input feature = partial column, column m = output
  // row; job 0's meaningful lanes are f <= 16, the others' f <= 64 (ones).
  if (warp < 8) {
    const int qw = warp & 3, f = qw * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
    for (int job = warp >> 2; job <= L; job += 2) {
      const int fmax = job == 0 ? 16 : 64;
      if (qw * 32 > fmax) continue;
      float* out = p.partial + ((int64_t)(job * gridDim.x + blockIdx.x) * kDwColsF + f) * 128;
      if (job == L) {  // head: feature f -> row f of partial column 0 (contiguous, reduce kind 4)
        uint32_t w[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
              "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]),
              "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
            : "r"(trow + HEAD));
        tmem_wait_ld();
        if (f <= fmax) p.partial[((int64_t)(job * gridDim.x + blockIdx.x) * kDwColsF) * 128 + f] = any ? __uint_as_float(w[0]) : 0.f;
        continue;
      }
      uint32_t v[64];
      tmem_ld32(trow + DW0 + 64u * job, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32(trow + DW0 + 64u * job + 32u, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      if (f <= fmax) {
#pragma unroll
        for (int m = 0; m < 64; m += 4)
          *reinterpret_cast<float4*>(out + m) =
              any ? make_float4(__uint_as_float(v[m]), __uint_as_float(v[m + 1]), __uint_as_float(v[m + 2]),
                                __uint_as_float(v[m + 3]))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) NB_TRF(3, 3);
  if (warp == 8) {
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

static size_t train_fused2_smem(const nb_model* m) { return f2_bars(m->pl.bytes) + 128; }

// Measurement switch: the one-tile-per-CTA kernel (NB_FUSED1=1).
static bool fused1_forced() {
  static const bool v = getenv("NB_FUSED1") != nullptr;
  return v;
}

cudaError_t launch_train_fused(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                               int64_t n_global, float alpha, float beta, float* partial,
                               int* cpj, int* head_row, cudaStream_t st) {
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
#ifdef NB_TRACE
  p.trace = g_trace_buffer;
#endif
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.num_tiles, m->num_sms));
  *cpj = grid;
  const size_t smem2 = train_fused2_smem(m);
  if (!fused1_forced() && smem2 <= 227 * 1024) {
    // two tiles in flight; the dW accumulators are transposed: the head
    // gradient lands in column 0, rows 0..64 of its partial (reduce kind 4)
    *head_row = -1;
    auto kern = p.L == 4 ? k_train_fused2<4> : (p.L == 3 ? k_train_fused2<3> : k_train_fused2<2>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    if (e != cudaSuccess) return e;
    // programmatic dependent launch: the prologue (barriers, TMEM, constant
    // image parts) overlaps the previous kernel in the stream
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(288);
    cfg.dynamicSmemBytes = smem2;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool no_pdl = getenv("NB_NO_PDL_FUSED") != nullptr;  // measurement switch
    cfg.attrs = at;
    cfg.numAttrs = no_pdl ? 0 : 1;  // (measured: 31.4 -> 30.5 us per c2 step)
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  *head_row = 64;  // the head gradient rides in row 64 of the last layer's delta image
  const size_t smem = train_fused_smem(m);
  auto kern = p.L == 4 ? k_train_fused<4> : k_train_fused<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace nb
