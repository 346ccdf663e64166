// nb_train_tc.cu — bf16 training step on tcgen05 tensor cores (rows a7-a9).
//
//  1. forward in kTrain mode (nb_fwd_tc.cu): same arithmetic as inference;
//     writes the row-tile images of the encoded input X and of h_1..h_L, and
//     dL/dz, dL/de_k of Eq. (1) (head terms P:261) per row.
//  2. k_bwd_tc: per 128-row tile, back-propagation through the hidden layers
//     delta_L = (dL/dz w_out + sum_k dL/de_k u_k [l_k = L]) * [h_L > 0],
//     delta_{l-1} = (delta_l W_l + heads) * [h_{l-1} > 0]   (ReLU'(0) = 0, R25)
//     as tcgen05.mma with A = delta_l (TMEM) and B = W_l read MN-major from the
//     same shared-memory weight image the forward uses; writes delta images.
//  3. k_dw_tc: dW_l = delta_l^T [h_{l-1} | 1] summed over row tiles with
//     tcgen05.mma (A, B both MN-major from row-tile images; the constant "ones"
//     block gives db_l = sum delta_l), per-CTA partials in fp32.  ONE launch
//     covers every layer's job (blockIdx.y = job, blockIdx.x = CTA of the job).
//  4. k_dw_reduce: fixed-order sum of the CTA partials into the canonical
//     gradient blob (deterministic, all jobs, coalesced); then NCCL allreduce,
//     Adam, bf16 re-pack (nb_api.cu).
#include <cuda_bf16.h>

#include <cstdlib>

#include "nb_adam.cuh"
#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

constexpr int kDwMaxN = 256;  // features per dW MMA (plus the 16-wide ones block)

// ---------------------------------------------------------------------------
// backward chain
// ---------------------------------------------------------------------------
struct BwdParams {
  const uint8_t* packed;
  PackLayout pl;
  int L, nh, ha0, ha1;
  int64_t n, num_tiles;
  const uint8_t* h_img[kMaxLayers];  // h_1..h_L images (F = W)
  uint8_t* d_img[kMaxLayers];        // delta_1..delta_L images (F = W)
  const float* g32;                  // [n][3]
  const uint8_t* c_img[kMaxLayers];  // sine nets: cos(z_l) images; delta = g * cos (R41)
  const uint32_t* m_img[kMaxLayers]; // ReLU nets: h_l > 0 bit masks (W * 4 words per row tile) or NULL
  int sine;
};

__device__ __forceinline__ uint32_t img_off(int r, int fg) {
  return (uint32_t)((fg * 16 + r / 8) * 128 + (r % 8) * 16);
}

// NSLOT tiles in flight, 4 warps (one per TMEM lane quarter) per slot, each
// thread owns one row and walks its W columns in 32-column chunks.
template <int W, bool BITS>
__global__ void __launch_bounds__(2 * 4 * 32, 1) k_bwd_tc(const BwdParams p) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  constexpr int NSLOT = 2, WPS = 4;
  constexpr int COLS = (NSLOT * (W + W / 2) <= 256) ? 256 : 512;
  static_assert(NSLOT * (W + W / 2) <= 512, "TMEM plan");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_off = (p.pl.core_bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);  // [0] weights, [1+s] acc_full
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      mbar_init(smem_u32(bars), 1);
      for (int s = 0; s < NSLOT; ++s) mbar_init(smem_u32(bars + 1 + s), 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(smem_u32(bars), p.pl.core_bytes);
      for (uint32_t off = 0; off < p.pl.core_bytes; off += 32768u)
        bulk_g2s(sbase + off, p.packed + off, min(32768u, p.pl.core_bytes - off), smem_u32(bars));
    }
    __syncwarp();
    tmem_alloc<COLS>(smem_u32(tmem_slot));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  mbar_wait(smem_u32(bars), 0);

  const int s = warp / WPS, qw = warp & 3, rit = qw * 32 + lane;
  const bool mma_warp = (warp % WPS) == 0;
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const uint32_t acc = (uint32_t)(s * W), acol = (uint32_t)(NSLOT * W + s * (W / 2));
  const uint32_t acc_full = smem_u32(bars + 1 + s);
  const uint32_t slot_bar = 1u + (uint32_t)s;
  const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout);
  const float* u0 = reinterpret_cast<const float*>(smem + p.pl.off_u[0]);
  const float* u1 = reinterpret_cast<const float*>(smem + p.pl.off_u[1]);
  const int h0 = p.nh > 0 ? p.ha0 : -1, h1 = p.nh > 1 ? p.ha1 : -1;  // 1-based layers
  // B = W_l^T: the K-major [out][in] image read MN-major (MN = in, K = out)
  const uint32_t idesc = make_idesc_bf16(128, W, 0, 1);
  uint32_t ph = 0;
  const int64_t G = gridDim.x;

  // Global-memory latency is kept off the per-layer chain: each thread's h row
  // of the next layer (ReLU masks) and the next tile's dL/dz are loaded one
  // step ahead into registers.
  // BITS: the forward's bit masks (word c of a row = [h_l > 0] of features
  // 32c .. 32c + 31) replace the h rows: 16 B instead of 2W B per row and layer.
  constexpr int HW = BITS ? 1 : W / 8;  // uint4 per h row
  constexpr int MW = W / 32;            // mask words per row
  auto load_h = [&](uint4 (&h)[HW], int l1, int64_t t) {  // h_{l1} row of tile t (l1 1-based)
    const uint8_t* hrow = (p.sine ? p.c_img[l1 - 1] : p.h_img[l1 - 1]) + t * img_tile_bytes(W);
#pragma unroll
    for (int q = 0; q < HW; ++q) h[q] = *reinterpret_cast<const uint4*>(hrow + img_off(rit, q));
  };
  auto load_m = [&](uint32_t (&mk)[MW], int l1, int64_t t) {
    const uint32_t* mrow = p.m_img[l1 - 1] + t * (W * 4) + rit;
#pragma unroll
    for (int c = 0; c < MW; ++c) mk[c] = __ldg(mrow + c * 128);
  };
  auto load_g = [&](float (&gg)[3], int64_t t) {
    const int64_t r = t * kTile + rit;
    const bool valid = t < p.num_tiles && r < p.n;
#pragma unroll
    for (int k = 0; k < 3; ++k) gg[k] = valid ? p.g32[r * 3 + k] : 0.f;
  };
  uint4 hcur[HW], hnext[HW];
  uint32_t mcur[MW], mnext[MW];
  float gcur[3], gnext[3];
  int64_t tile = blockIdx.x + (int64_t)s * G;
  if (tile < p.num_tiles) {
    if (BITS) load_m(mcur, p.L, tile);
    else load_h(hcur, p.L, tile);
    load_g(gcur, tile);
  }
  for (; tile < p.num_tiles; tile += NSLOT * G) {
    const int64_t next = tile + NSLOT * G;
    load_g(gnext, next);
    const float gz = gcur[0], ge0 = gcur[1], ge1 = gcur[2];
    // l (1-based) runs L .. 1; the value in flight is dL/dh_l
    for (int l = p.L; l >= 1; --l) {
      uint32_t v[32];
      uint8_t* drow = p.d_img[l - 1] + tile * img_tile_bytes(W);
      if (BITS) {
        if (l > 1) load_m(mnext, l - 1, tile);
        else if (next < p.num_tiles) load_m(mnext, p.L, next);
      } else {
        if (l > 1) load_h(hnext, l - 1, tile);
        else if (next < p.num_tiles) load_h(hnext, p.L, next);
      }
      if (l < p.L) {
        mbar_wait(acc_full, ph);
        ph ^= 1u;
        tc_fence_after();
      }
#pragma unroll
      for (int c = 0; c < W / 32; ++c) {
        if (l < p.L) {
          tmem_ld32(trow + acc + 32u * c, v);
          tmem_wait_ld();
        }
        float g[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = 32 * c + i;
          float d = (l < p.L) ? __uint_as_float(v[i]) : gz * wout[j];
          if (l == h0) d = fmaf(ge0, u0[j], d);
          if (l == h1) d = fmaf(ge1, u1[j], d);
          g[i] = d;
        }
        uint32_t pk[16];
        if (BITS) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pk[j] = pack_bf16x2(((mcur[c] >> (2 * j)) & 1u) ? g[2 * j] : 0.f,
                                ((mcur[c] >> (2 * j + 1)) & 1u) ? g[2 * j + 1] : 0.f);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 hv = hcur[4 * c + q];
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = 8 * q + 2 * e;
              float m0, m1;
              if (p.sine) {  // g * cos(z_l)
                m0 = g[i] * __uint_as_float(hw[e] << 16);
                m1 = g[i + 1] * __uint_as_float(hw[e] & 0xFFFF0000u);
              } else {
                m0 = (hw[e] & 0x7FFFu) ? g[i] : 0.f;           // h > 0 (h >= 0 by ReLU)
                m1 = (hw[e] & 0x7FFF0000u) ? g[i + 1] : 0.f;
              }
              pk[4 * q + e] = pack_bf16x2(m0, m1);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(drow + img_off(rit, 4 * c + q)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        if (l >= 2) tmem_st16(trow + acol + 16u * c, pk);
      }
      if (BITS) {
#pragma unroll
        for (int q = 0; q < MW; ++q) mcur[q] = mnext[q];
      } else {
#pragma unroll
        for (int q = 0; q < HW; ++q) hcur[q] = hnext[q];
      }
      if (l >= 2) {
        // delta_l is in TMEM: MMA dL/dh_{l-1} = delta_l W_l (K = out of layer l)
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(slot_bar), "n"(WPS * 32) : "memory");
        if (mma_warp) {
          tc_fence_after();
          if (elect_one()) {
            // MN-major: SBO = MN (in-group) stride 128 B, LBO = K (out-group) stride
            const uint64_t bdesc =
                make_sdesc(sbase + p.pl.off_w[l - 1], (W / 8u) * 128u, 128u);
#pragma unroll
            for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
              mma_ts(tmem + acc, tmem + acol + kk * 8u, bdesc + (uint64_t)((kk * 32u * W) >> 4),
                     idesc, kk > 0u);
            mma_commit(acc_full);
          }
          __syncwarp();
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) gcur[k] = gnext[k];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<COLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// dW GEMM: D[m][f] = sum over rows of A[m][row] B[f][row] for one job
//   A = row-tile images with FA features (delta_l or the head-gradient image),
//   B = row-tile images with FB features (h_{l-1}, X, ...) followed by the
//       constant ones block (feature FB = 1) -> D[m][FB] = sum_rows A[m][row].
// One CTA accumulates a contiguous range of tiles in TMEM (M = 128 rows of D;
// rows >= FA are don't-care), then writes its fp32 partial.
// ---------------------------------------------------------------------------
struct DwJob {
  const uint8_t* a_img;
  int fa;        // features of the A image (rows of D that are meaningful)
  int m_off;     // first A feature of this job (M half for w = 256)
  const uint8_t* b_img;
  int fb;        // features of the B image (<= 256)
  // reduction of this job's partials into the gradient blob (k_dw_reduce)
  int kind;      // 0: W[m][k] <- D[m][k], b[m] <- D[m][fb]
                 // 1: layer 1: W[m][j] <- D[m][j] + D[m][d0 + j], b[m] <- D[m][16]
                 // 2: head row `row`: v[j] <- D[row][j], c <- D[row][fb]
                 // 3: layer 1 of a PE net (PackLayout::pe_lo): W[m][j] <- D[m][j] + D[m][32 + j], b[m] <- D[m][fb]
                 // 4: head, transposed partial (k_train_fused2): v[j] <- D[0][row j], c <- D[0][row in]
                 //    (contiguous per CTA, so the reduce's loads coalesce)
  int rows, row, d0, in;
  float* w_out;
  float* b_out;
};
constexpr int kMaxDwJobs = 2 * kMaxLayers + 3;
constexpr int kDwCols = kDwMaxN + 16;  // partial columns per CTA (features + ones block)
// partial of CTA c of job j, column col, D row m: [(j * cpj + c) * kDwCols + col] * 128 + m
// Adam + bf16 re-pack fused into k_dw_reduce (no communicator: the reduced
// gradient is final, so the thread that writes g_i also steps parameter i).
struct AdamFuse {
  int on;
  float* th;
  float* m;
  float* v;
  const float* grad;  // gradient blob base (w_out / b_out point into it)
  AdamArgs h;
  PackArgs a;
};
struct DwJobs {
  DwJob job[kMaxDwJobs];
  AdamFuse adam;
  int njobs, cpj;
  int nst;        // TMA pipeline stages (<= kDwMaxStages)
  int accumulate; // add into the partials (micro-batches after the first)
  uint32_t stage; // bytes per stage (A 32 KB + B of the widest job + ones block)
  float* partial;
  unsigned long long* zero_next;  // k_dw_reduce: the next step's statistics buffer (8 words) to zero
};
constexpr int kDwMaxStages = 6;

__global__ void __launch_bounds__(128, 1) k_dw_tc(const __grid_constant__ DwJobs js, int64_t num_tiles) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  const DwJob& j = js.job[blockIdx.y];
  extern __shared__ __align__(1024) uint8_t smem[];
  // stage: A tile 128 features (16 groups) x 128 rows = 32 KB, then B + ones: (fb + 16) x 256 B
  const uint32_t a_bytes = 128u * 256u;
  const uint32_t stage = js.stage;
  const int NST = js.nst;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * stage);  // [st] full, [NST + st] empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kDwMaxStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = smem_u32(smem);
  const int N = j.fb + 16;
  for (int st = 0; st < NST; ++st) {
    // ones block after each stage's B image: feature fb = 1.0 for every row
    uint8_t* ones = smem + st * stage + a_bytes + j.fb * 256;
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
      const int r = i / 16, f = i % 16;
      *reinterpret_cast<uint16_t*>(ones + img_off(r, f / 8) + (f % 8) * 2) = f == 0 ? 0x3F80 : 0;
    }
    // rows of A beyond fa are read but never used: keep them finite
    const int z0 = (j.m_off > 0 ? 0 : j.fa * 256) / 16;
    for (int i = z0 + threadIdx.x; i < (int)a_bytes / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(smem + st * stage)[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < 2 * NST; ++i) mbar_init(smem_u32(bars + i), 1);
      fence_barrier_init();
    }
    __syncwarp();
    tmem_alloc<512>(smem_u32(tmem_slot));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  const int64_t per = (num_tiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = min(num_tiles, blockIdx.x * per), t1 = min(num_tiles, t0 + per);
  const int fa_job = min(128, j.fa - j.m_off);
  const uint32_t a_copy = (uint32_t)fa_job * 256u;  // bytes of this job's A features per tile
  const uint32_t idesc = make_idesc_bf16(128, j.fb, 1, 1);
  const uint32_t idesc1 = make_idesc_bf16(128, 16, 1, 1);
  const int64_t ntl = t1 - t0;
  if (warp == 0) {
    // producer (lane 0) runs up to NST tiles ahead of the MMAs; a stage is
    // refilled once the commit of the tile that last used it has arrived
    auto issue_copy = [&](int i, int st, uint32_t eph) {
      if (i >= NST) mbar_wait(smem_u32(bars + NST + st), eph);
      const uint32_t bar = smem_u32(bars + st);
      const int64_t t = t0 + i;
      mbar_arrive_expect_tx(bar, a_copy + (uint32_t)j.fb * 256u);
      bulk_g2s(sbase + st * stage, j.a_img + t * img_tile_bytes(j.fa) + (int64_t)j.m_off * 256,
               a_copy, bar);
      bulk_g2s(sbase + st * stage + a_bytes, j.b_img + t * img_tile_bytes(j.fb),
               (uint32_t)j.fb * 256u, bar);
    };
    // producer state (lane 0): next tile to copy, its stage and that stage's
    // empty-barrier parity; consumer state: stage and full-barrier parity
    int issued = 0, ist = 0, cst = 0;
    uint32_t pround = 0, fph = 0;  // tile k = pround * NST + ist waits for commit (pround - 1)
    for (int i = 0; i < (int)ntl; ++i) {
      // NST - 1 tiles in flight: refilling the stage of tile i - 1 (whose MMAs
      // may still run) is left to the next iteration
      const int ahead = NST >= 3 ? NST - 1 : NST;
      if (lane == 0) {
        for (; issued < (int)ntl && issued < i + ahead; ++issued) {
          issue_copy(issued, ist, (pround & 1u) ^ 1u);
          if (++ist == NST) {
            ist = 0;
            ++pround;
          }
        }
      }
      __syncwarp();
      const int st = cst;
      mbar_wait(smem_u32(bars + st), fph);
      if (++cst == NST) {
        cst = 0;
        fph ^= 1u;
      }
      tc_fence_after();
      if (elect_one()) {
        const uint32_t as = sbase + st * stage, bs = as + a_bytes;
        // MN-major row-tile images: SBO (feature-group stride) 2048 B, LBO (row-group) 128 B
        const uint64_t ad = make_sdesc(as, 128u, 2048u);
        const uint64_t bd = make_sdesc(bs, 128u, 2048u);
        const uint64_t od = make_sdesc(bs + (uint32_t)j.fb * 256u, 128u, 2048u);
#pragma unroll
        for (uint32_t kk = 0; kk < 8; ++kk) {
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          mma_ss(tmem, ad + kk * 16u, bd + kk * 16u, idesc, acc);
          mma_ss(tmem + (uint32_t)j.fb, ad + kk * 16u, od + kk * 16u, idesc1, acc);
        }
        mma_commit(smem_u32(bars + NST + st));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // wait for all MMAs: the last tile's commit
  if (ntl > 0) {
    const int i = (int)ntl - 1;
    mbar_wait(smem_u32(bars + NST + i % NST), (uint32_t)((i / NST) & 1));
  }
  tc_fence_after();
  // epilogue: thread = row m of D (lane quarter = warp), N fp32 columns; the
  // partial is column-major ([col][128 rows]) so a warp's stores are coalesced
  const int m = warp * 32 + lane;
  float* out = js.partial + ((int64_t)(blockIdx.y * js.cpj + blockIdx.x) * kDwCols) * 128 + m;
  for (int c = 0; c < N; c += 16) {
    uint32_t v[32];
    if (c + 32 <= N) {
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = t1 > t0 ? __uint_as_float(v[i]) : 0.f;
        out[(int64_t)(c + i) * 128] = js.accumulate ? out[(int64_t)(c + i) * 128] + x : x;
      }
      c += 16;
    } else {
      uint32_t w[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
            "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]),
            "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float x = t1 > t0 ? __uint_as_float(w[i]) : 0.f;
        out[(int64_t)(c + i) * 128] = js.accumulate ? out[(int64_t)(c + i) * 128] + x : x;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Fixed-order reduction of the CTA partials into the gradient blob, every job
// at once (deterministic: CTA order 0..cpj-1).  One thread per output element,
// D row m fastest, so a warp's partial loads are coalesced.
//   kind 0: hidden layer l >= 2: W[m][k] <- D[m][k], b[m] <- D[m][fb]
//   kind 1: layer 1: W[m][j] <- D[m][j] + D[m][d0 + j], b[m] <- D[m][16]
//   kind 2: head row `row` of the head-gradient image: v[j] <- D[row][j], c <- D[row][fb]
// Block = 32 consecutive output elements x S slices of the CTA range (S fixed
// by the CTA count: <= 8 partials per slice): thread (e, s) sums CTAs
// [s * per, (s + 1) * per) in order (its loads in flight at once), then slice
// 0 adds the S slice sums in order — a fixed tree, so the result is
// deterministic.  With js.adam.on, that
// thread also takes parameter i's Adam step and re-pack (nb_adam.cuh).
constexpr int kRedSlices = 16;
__global__ void __launch_bounds__(32 * kRedSlices) k_dw_reduce(const __grid_constant__ DwJobs js) {
  __shared__ float part[kRedSlices][32];
  // the next step's fused kernel is a programmatic dependent of this one: it
  // may be scheduled now (it waits for this grid before touching memory)
  griddep_launch_dependents();
  if (blockIdx.x == 0 && threadIdx.x < 8 && js.zero_next) js.zero_next[threadIdx.x] = 0ull;
  const int e_in = threadIdx.x & 31, sl = threadIdx.x >> 5, S = blockDim.x >> 5;
  int e = blockIdx.x * 32 + e_in;  // global element index over all jobs (< 2^31)
  int jj = 0;
  for (; jj < js.njobs; ++jj) {
    const DwJob& r = js.job[jj];
    const int total = (r.kind >= 2 && r.kind != 3 ? 1 : r.rows) * (r.in + 1);
    if (e < total) break;
    e -= total;
  }
  const bool active = jj < js.njobs;
  float acc = 0.f;
  int k = 0, m = 0;
  if (active) {
    const DwJob& r = js.job[jj];
    const bool head = r.kind == 2 || r.kind == 4;
    const unsigned rows = head ? 1u : (unsigned)r.rows;
    k = (int)((unsigned)e / rows);                        // output column (k == in: bias)
    m = r.kind == 2 ? r.row : (r.kind == 4 ? k : (int)((unsigned)e % rows));  // row of D
    const int c0 = r.kind == 4 ? 0 : (k == r.in ? r.fb : k);
    const int c1 = (k != r.in && r.kind == 1) ? r.d0 + k : ((k != r.in && r.kind == 3) ? 32 + k : -1);
    const float* P = js.partial + ((int64_t)(jj * js.cpj) * kDwCols) * 128 + m;
    const int64_t cs = (int64_t)kDwCols * 128;  // CTA stride
    const int per = (js.cpj + S - 1) / S;
    const int cb = sl * per, ce = min(js.cpj, cb + per);
    for (int c = cb; c < ce; c += 16) {
      float x0[16], x1[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const bool ok = c + u < ce;
        x0[u] = ok ? __ldg(P + (c + u) * cs + (int64_t)c0 * 128) : 0.f;
        x1[u] = (ok && c1 >= 0) ? __ldg(P + (c + u) * cs + (int64_t)c1 * 128) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (c + u < ce) {
          acc += x0[u];
          if (c1 >= 0) acc += x1[u];
        }
      }
    }
  }
  part[sl][e_in] = acc;
  __syncthreads();
  if (sl == 0 && active) {
    float t = 0.f;
    for (int q = 0; q < S; ++q) t += part[q][e_in];
    const DwJob& r = js.job[jj];
    float* out;
    if (r.kind == 2 || r.kind == 4) {
      out = k == r.in ? r.b_out : r.w_out + k;
    } else {
      const int mo = m + r.m_off;
      out = k == r.in ? r.b_out + mo : r.w_out + (int64_t)mo * r.in + k;
    }
    *out = t;
    if (js.adam.on)
      adam_pack_one(out - js.adam.grad, t, js.adam.th, js.adam.m, js.adam.v, js.adam.h, js.adam.a);
  }
}

static cudaError_t launch_dw_reduce(const DwJobs& js, cudaStream_t st) {
  int64_t total = 0;
  for (int jj = 0; jj < js.njobs; ++jj) {
    const DwJob& r = js.job[jj];
    total += (int64_t)(r.kind == 2 || r.kind == 4 ? 1 : r.rows) * (r.in + 1);
  }
  // slices of <= 8 CTA partials each (one round of loads), at most kRedSlices
  // slices of the CTA range per output group (measured, NB_RED_SLICES sweep:
  // 148 partials (fused c2) 4 slices 28.9 us per step vs 16: 29.2, 2: 33.9;
  // 16 partials (c3) 2 slices 76.0 us vs 8: 81.9, 16: 88.0)
  int S = js.cpj >= 64 ? 4 : std::max(1, std::min(kRedSlices, (js.cpj + 7) / 8));
  if (const char* ev = getenv("NB_RED_SLICES")) S = std::max(1, std::min(kRedSlices, atoi(ev)));  // measurement
  // a plain launch: as a programmatic dependent of the fused step kernel its
  // 400 CTAs, scheduled early, slowed that kernel's tail (c2 step 30.5 ->
  // 35.9 us, measured); the next step's kernel is the programmatic one
  k_dw_reduce<<<(unsigned)((total + 31) / 32), 32 * S, 0, st>>>(js);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool train_tc_supported(const nb_desc& d) {
  // sine / positional-encoding nets: w = 64, 128 (the EXT forward kernels, R41, R42)
  const bool plain = d.activation == NB_RELU && d.pe_depth == 0;
  return d.precision == NB_BF16 && (d.width == 64 || d.width == 128 || (d.width == 256 && plain)) &&
         d.hidden_layers >= 2;
}

struct TrainLayout {
  size_t x_img, h_img[kMaxLayers], c_img[kMaxLayers], d_img[kMaxLayers], hd_img, g32, partial, total;
};

static TrainLayout train_layout(const nb_model* m, int64_t n, int grid) {
  const int W = m->d.width, L = m->d.hidden_layers;
  const int64_t T = (n + kTile - 1) / kTile;
  TrainLayout t;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  t.x_img = take(T * img_tile_bytes((int)m->pl.k_of[0]));
  for (int l = 0; l < L; ++l) t.h_img[l] = take(T * img_tile_bytes(W));
  const bool sine = m->d.activation == NB_SINE;
  // sine nets: cos(z_l) images; ReLU nets: the backward's h_l > 0 bit masks
  // (W / 32 words per row, W * 16 B per row tile; the CTA-pair path without heads)
  const bool masks = !sine && !(m->pl.pairs == 2 && m->d.n_heads > 0) && !getenv("NB_NO_MASKS");
  for (int l = 0; l < L; ++l) t.c_img[l] = sine ? take(T * img_tile_bytes(W)) : (masks ? take(T * W * 16) : 0);
  for (int l = 0; l < L; ++l) t.d_img[l] = take(T * img_tile_bytes(W));
  // the dW GEMM reads 128 features of A per tile: pad the last tile's images
  take(img_tile_bytes(128));
  t.hd_img = take(T * img_tile_bytes(8) + img_tile_bytes(128));
  t.g32 = take((size_t)T * kTile * 3 * sizeof(float));
  // njobs * cpj <= grid for the unfused path; the fused kernel (w = 64) keeps
  // one partial per CTA per job: (L + 1) * grid
  t.partial = take((size_t)(L + 1) * grid * 128 * kDwCols * sizeof(float));
  t.total = off;
  return t;
}

static int64_t train_chunk_rows(const nb_model* m, int64_t n);

size_t train_tc_scratch_bytes(const nb_model* m, int64_t n) {
  return train_layout(m, train_chunk_rows(m, n), m->num_sms).total;
}

template <int W>
static cudaError_t launch_bwd(nb_model* m, const BwdParams& p, cudaStream_t st) {
  size_t smem = ((m->pl.core_bytes + 15) & ~15u) + 64;
  smem = std::max<size_t>(smem, 116 * 1024);
  auto kern = p.m_img[0] ? k_bwd_tc<W, true> : k_bwd_tc<W, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(p.num_tiles, m->num_sms);
  return launch_pdl(kern, dim3(grid), dim3(2 * 4 * 32), smem, st, true, p);
}

static cudaError_t run_dw(DwJobs& js, int64_t T, cudaStream_t st) {
  int fbmax = 0;
  for (int i = 0; i < js.njobs; ++i) fbmax = std::max(fbmax, js.job[i].fb);
  js.stage = (uint32_t)(128 * 256 + (fbmax + 16) * 256);
  const size_t fixed = 8 * 2 * kDwMaxStages + 16;
  js.nst = (int)std::min<size_t>(kDwMaxStages, (227 * 1024 - fixed) / js.stage);
  if (const char* ev = getenv("NB_DW_STAGES"))  // measurement override
    js.nst = std::max(2, std::min(js.nst, atoi(ev)));
  const size_t smem = (size_t)js.nst * js.stage + fixed;
  cudaError_t e = cudaFuncSetAttribute(k_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_dw_tc, dim3(js.cpj, js.njobs), dim3(128), smem, st, true, js, T);
}

// Rows per training micro-batch: bounds the scratch (activation / delta
// images, ~2 GB) for very large local batches; dW partials accumulate across
// micro-batches in a fixed order (deterministic), and one reduce follows the
// last.  (L2-sized micro-batches of ~64 MB were measured slower: the kernels
// are latency-bound below ~2^16 rows, e.g. c5 2^18 rows 0.74 -> 2.9 ms.)
static int64_t train_chunk_rows(const nb_model* m, int64_t n) {
  const int64_t per_row = 2 * ((int64_t)m->pl.k_of[0] + 3 * (int64_t)m->d.hidden_layers * m->d.width + 8) + 12;
  int64_t c = ((int64_t)2 << 30) / per_row;
  if (const char* ev = getenv("NB_TRAIN_CHUNK")) c = atoll(ev);  // test / measurement override
  c = std::max<int64_t>(256, c / 256 * 256);
  return std::max<int64_t>(1, std::min(n, c));
}

cudaError_t launch_fwd_tc(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st);
cudaError_t launch_fwd_tc2(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st);
bool train_fused_supported(const nb_model* m);
cudaError_t launch_train_fused(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                               int64_t n_global, float alpha, float beta, float* partial,
                               int* cpj, int* head_row, cudaStream_t st);

// One micro-batch: forward (kTrain) + backward chain + dW GEMMs (partials
// written when `first`, accumulated otherwise).
static cudaError_t train_chunk(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                               int64_t n_global, float alpha, float beta, bool first,
                               DwJobs& js, const TrainLayout& tl, cudaStream_t st) {
  const int W = m->d.width, L = m->d.hidden_layers;
  const int64_t T = (n + kTile - 1) / kTile;
  uint8_t* base = (uint8_t*)m->train_scratch;
  // 1. forward with activation images and dL/dz
  FwdArgs a;
  memset(&a, 0, sizeof(a));
  a.q = q;
  a.y = y;
  a.n = n;
  a.counts = m->d_counts;
  a.keys = m->d_keys;
  a.flags = m->d_flags;
  a.tr.x_img = base + tl.x_img;
  const bool sine = m->d.activation == NB_SINE;
  for (int l = 0; l < L; ++l) a.tr.h_img[l] = base + tl.h_img[l];
  for (int l = 0; l < L; ++l) a.tr.c_img[l] = tl.c_img[l] ? base + tl.c_img[l] : nullptr;
  a.tr.hd_img = base + tl.hd_img;
  a.tr.g32 = (float*)(base + tl.g32);
  a.tr.alpha = alpha;
  a.tr.beta = beta;
  a.tr.inv_b = 1.0f / (float)n_global;
  a.tr.loss = m->d_loss;
  a.tr.stats = m->d_stats;
  a.tr.num_tiles = T;
  const bool pairs = m->pl.pairs == 2;  // w = 256: CTA-pair forward and backward
  cudaError_t e = pairs ? launch_fwd_tc2(m, kTrain, a, st) : launch_fwd_tc(m, kTrain, a, st);
  if (e != cudaSuccess) return set_error("training forward: %s", cudaGetErrorString(e)), e;
  // 2. backward chain
  BwdParams bp;
  bp.packed = m->packed;
  bp.pl = m->pl;
  bp.L = L;
  bp.nh = m->d.n_heads;
  bp.ha0 = m->d.head_after[0];
  bp.ha1 = m->d.head_after[1];
  bp.n = n;
  bp.num_tiles = T;
  for (int l = 0; l < L; ++l) {
    bp.h_img[l] = base + tl.h_img[l];
    bp.d_img[l] = base + tl.d_img[l];
    bp.c_img[l] = sine ? base + tl.c_img[l] : nullptr;
  }
  for (int l = 0; l < kMaxLayers; ++l)
    bp.m_img[l] = (!sine && l < L && tl.c_img[l]) ? reinterpret_cast<const uint32_t*>(base + tl.c_img[l]) : nullptr;
  bp.sine = sine ? 1 : 0;
  bp.g32 = (float*)(base + tl.g32);
  if (pairs)
  {
    const uint8_t* mk[kMaxLayers];
    for (int l = 0; l < kMaxLayers; ++l) mk[l] = (l < L && tl.c_img[l]) ? base + tl.c_img[l] : nullptr;
    e = launch_bwd_tc2(m, bp.h_img, bp.d_img, bp.g32, n, st, tl.c_img[0] ? mk : nullptr);
  }
  else
    e = W == 64 ? launch_bwd<64>(m, bp, st) : launch_bwd<128>(m, bp, st);
  if (e != cudaSuccess) return set_error("backward chain: %s", cudaGetErrorString(e)), e;
  // 3. dW GEMMs of every job (one launch)
  js.accumulate = first ? 0 : 1;
  return run_dw(js, T, st);
}

cudaError_t launch_train_tc(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                            int64_t n_global, float alpha, float beta, float fuse_lr, cudaStream_t st) {
  const int W = m->d.width, L = m->d.hidden_layers, d0 = m->d0;
  AdamFuse af{};
  if (fuse_lr > 0.f) {
    af.on = 1;
    af.th = m->theta;
    af.m = m->adam_m;
    af.v = m->adam_v;
    af.grad = m->grad;
    adam_setup(m, fuse_lr, &af.h, &af.a);
  }
  const int64_t chunk = train_chunk_rows(m, n);
  TrainLayout tl = train_layout(m, chunk, m->num_sms);
  uint8_t* base = (uint8_t*)m->train_scratch;
  if (n > 0 && n <= chunk && train_fused_supported(m) && !getenv("NB_NO_FUSED")) {
    // w = 64: forward + loss + backward + dW in one kernel (nb_train_fused.cu)
    DwJobs fj{};
    fj.adam = af;
    fj.zero_next = reinterpret_cast<unsigned long long*>(m->d_loss_base + 8 * m->lbuf);
    fj.partial = (float*)(base + tl.partial);
    float* g = m->grad;
    fj.job[fj.njobs++] = DwJob{nullptr, W, 0, nullptr, 16, 1, W, 0, d0, d0, g + m->po.W[0], g + m->po.b[0]};
    for (int l = 1; l < L; ++l)
      fj.job[fj.njobs++] = DwJob{nullptr, W, 0, nullptr, W, 0, W, 0, d0, W, g + m->po.W[l], g + m->po.b[l]};
    // the head gradient: D row head_row (set by the kernel choice)
    DwJob& hj = fj.job[fj.njobs++];
    hj = DwJob{nullptr, W, 0, nullptr, W, 2, 1, 64, d0, W, g + m->po.wout, g + m->po.bout};
    cudaError_t e = launch_train_fused(m, q, y, n, n_global, alpha, beta, fj.partial, &fj.cpj, &hj.row, st);
    if (e != cudaSuccess) return e;
    if (hj.row < 0) {  // k_train_fused2: the head's partial is stored transposed (one contiguous column)
      hj.kind = 4;
      hj.row = 0;
    }
    return launch_dw_reduce(fj, st);
  }
  // dW jobs (image pointers are the same for every micro-batch)
  DwJobs js{};
  js.partial = (float*)(base + tl.partial);
  float* g = m->grad;
  auto add = [&](const uint8_t* a_img, int fa, const uint8_t* b_img, int fb, int kind, int rows,
                 int row, int in, float* w_out, float* b_out) {
    // A with more than 128 features (w = 256): one job per 128-feature M half
    for (int mo = 0; mo < fa; mo += 128) {
      DwJob& j = js.job[js.njobs++];
      j = DwJob{a_img, fa, mo, b_img, fb, kind, std::min(rows, 128), row, d0, in, w_out, b_out};
    }
  };
  for (int l = 0; l < L; ++l) {
    if (l == 0 && m->pl.pe_lo)  // PE operand: hi [0, d_in), lo [32, 32 + d_in), K = 64
      add(base + tl.d_img[0], W, base + tl.x_img, 64, 3, W, 0, m->din, g + m->po.W[0], g + m->po.b[0]);
    else if (l == 0)
      add(base + tl.d_img[0], W, base + tl.x_img, 16, 1, W, 0, d0, g + m->po.W[0], g + m->po.b[0]);
    else
      add(base + tl.d_img[l], W, base + tl.h_img[l - 1], W, 0, W, 0, W, g + m->po.W[l], g + m->po.b[l]);
  }
  // output head: row 0 of the head-gradient image against h_L; exit heads: rows 1, 2
  add(base + tl.hd_img, 8, base + tl.h_img[L - 1], W, 2, 1, 0, W, g + m->po.wout, g + m->po.bout);
  for (int k = 0; k < m->d.n_heads; ++k)
    add(base + tl.hd_img, 8, base + tl.h_img[m->d.head_after[k] - 1], W, 2, 1, 1 + k, W,
        g + m->po.u[k], g + m->po.c[k]);
  // a fixed CTA grid per job, the same for every micro-batch (deterministic sums)
  js.cpj = std::max(1, m->num_sms / js.njobs);
  cudaError_t e = cudaSuccess;
  if (n == 0) {  // empty batch: zero gradient
    e = cudaMemsetAsync(js.partial, 0, sizeof(float) * 128 * kDwCols * js.cpj * js.njobs, st);
  }
  for (int64_t c0 = 0; c0 < n && e == cudaSuccess; c0 += chunk) {
    const int64_t rows = std::min(chunk, n - c0);
    e = train_chunk(m, q + c0 * d0, y + c0, rows, n_global, alpha, beta, c0 == 0, js, tl, st);
  }
  if (e != cudaSuccess) return e;
  // 4. fixed-order reduction of all partials into the gradient blob (+ Adam)
  js.adam = af;
  js.zero_next = reinterpret_cast<unsigned long long*>(m->d_loss_base + 8 * m->lbuf);
  return launch_dw_reduce(js, st);
}

}  // namespace nb
