// nb_fwd_exit.cu — early-exit compaction for the fused score (SURVEY §8 K9,
// row a4/a5 for models with exit heads, BASELINE.json configs[3]).
//
// Paper: "if its output is negative, the query is classified as negative and
// the computation stops" (early-out, §3.3); the predictor is the
// conjunction of the exit heads and the final output (R22).  The
// dense kernel (nb_fwd_tc.cuh) evaluates every head on every row, so exits
// save nothing: an MMA tile is 128 rows and a row cannot leave it.  Here the
// network is cut at its heads into SEGMENTS ([0, h1], (h1, h2], (h2, L]) and
// each segment is one persistent launch over full 128-row tiles:
//
//   segment 0: records -> encode -> layers -> head 1 -> exits counted,
//              survivors' bf16 activations appended to an image region
//   segment k: image tiles (bulk copy, A operand from shared memory) ->
//              layers -> head k+1 (or the output) -> exits / classify
//
// Every slot stream (CTA b, slot s; r = s * G + b) owns one output REGION and
// appends its survivors in its own tile order, so the compacted order — and
// hence every count — is deterministic.  The next segment's tiles are the
// regions' tiles concatenated (a prefix sum over the region counts, computed
// by every CTA at start); only each region's last tile is ragged.
//
// The activations handed from one segment to the next are exactly the bf16
// values the dense kernel feeds its next MMA, and the per-row arithmetic is
// the same, so counts equal the dense kernel's (tests/test_gpu_parity.py);
// only the non-finite counter differs when a row exits before a non-finite
// later logit would have been computed (R40).
//
// Image layout (per 128-row tile, 32 KB): element (row r, feature f) at
//   ((f / 8) * 16 + r / 8) * 128 + (r % 8) * 16 + (f % 8) * 2
// — UMMA K-major no-swizzle core matrices with LBO = 2048 (K), SBO = 128 (M).
#include "nb_fwd_tc.cuh"

namespace nb {

namespace {

constexpr int kXW = 128;         // width of the compaction kernels
constexpr int kXSlots = 2;       // tile slots per CTA
constexpr int kXWps = 8;         // warps per slot (row quarter x column half)
constexpr int kXWarps = kXSlots * kXWps;
constexpr uint32_t kImgTile = (uint32_t)kXW * kTile * 2;  // 32 KB
constexpr int kMaxRegions = 2 * 160;

struct ExitParams {
  FwdArgs a;                 // q, y, n (segment 0), counts, flags, finalisation
  const uint8_t* packed;
  int d0;
  int lb;                    // first layer of the segment
  float tau_end;             // threshold of the head ending the segment / output
  uint32_t hc_off;           // packed offset of that head's fp32 constant (c_k / b_out)
  // weights: up to 2 * SEG + 1 bulk copies packed -> shared memory
  uint32_t cp_src[16], cp_dst[16], cp_len[16];
  int ncp;
  uint32_t wbytes;           // bytes of the shared weight area
  uint32_t s_w[8], s_bb[8];  // shared offsets of the segment's layer images / bias blocks
  uint32_t s_head;           // head vector (W floats: u_k / w_out)
  // regions (R = kXSlots * gridDim.x)
  const uint8_t* in_img;
  const float* in_rec;       // IN = 2: survivors' records of the previous segment (regions)
  float* out_rec;            // REC: survivors' records appended to this slot's region
  const uint8_t* in_lab;
  const uint32_t* in_cnt;
  uint8_t* out_img;
  uint8_t* out_lab;
  uint32_t* out_cnt;
  int64_t cap;               // tiles per region (both directions)
  int64_t num_tiles;         // segment 0: ceil(n / 128)
};

// shared-memory carve (identical on host and device)
struct ExitSmem {
  uint32_t bars, tslot, xch, xpos, qcnt, ctr, pref, rcnt, stage, lab, total;
  __host__ __device__ ExitSmem(uint32_t wbytes, bool in_img) {
    uint32_t o = (wbytes + 127u) & ~127u;
    bars = o;  o += 8 * (1 + kXSlots + 2 * kXSlots);       // weights, acc_full[s], stage[s][2]
    tslot = o; o += 16;
    xch = o;   o += 4 * kXSlots * 2 * 4 * 32;               // head partial of the other half
    xpos = o;  o += 4 * kXSlots * 2 * 4 * 32;               // compacted position (or -1)
    qcnt = o;  o += 4 * kXSlots * 2 * 4;                    // survivors per row quarter
    ctr = o;   o += 4 * kXWarps * 12;
    pref = o;  o += 4 * (kMaxRegions + 4);
    rcnt = o;  o += 4 * kMaxRegions;                        // input region row counts
    o = (o + 127u) & ~127u;
    stage = o;  // per slot, 2 buffers: image tile (32 KB) or records (128 x 8 fp32)
    o += (uint32_t)kXSlots * 2u * (in_img ? kImgTile : (uint32_t)kTile * 8u * 4u);
    lab = o;   o += kXSlots * 2 * kTile;
    total = o;
  }
};

__device__ __forceinline__ void st_img_row(uint8_t* tile, int row, int fg0, const uint32_t (&w)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    *reinterpret_cast<uint4*>(tile + ((fg0 + i) * 16 + row / 8) * 128 + (row % 8) * 16) =
        make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

// SEG hidden layers [lb, lb + SEG); IN = 0: the caller's fp32 records,
// 1: the previous segment's image regions, 2: the previous segment's record
// regions (the segment then starts at layer 0 and recomputes the layers
// before it); HEAD = exit head ending the segment (0, 1), or -1: the segment
// ends with the output layer and classifies.  REC: survivors hand their
// fp32 record (d0 floats, 16 B for c4) to the next segment instead of their
// bf16 activations (256 B).
template <int SEG, int IN, int HEAD, int D0C, bool REC = false>
__global__ void __launch_bounds__(kXWarps * 32, 1) k_score_exit(const ExitParams p) {
  constexpr bool IN_IMG = IN == 1, IN_REG = IN != 0;  // input from regions (prefix-summed tiles)
  constexpr int W = kXW, NSLOT = kXSlots, WPS = kXWps, NEPI = kXWarps;
  constexpr int CPT = W * 4 / WPS, NCH = CPT / 32;  // 64 columns per thread
  constexpr bool FINAL = HEAD < 0;
  constexpr uint32_t COLS = 512, kOnesCol = COLS - 8;
  extern __shared__ __align__(1024) uint8_t smem[];
  const ExitSmem L(p.wbytes, IN_IMG);
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  float* xch = reinterpret_cast<float*>(smem + L.xch);
  int* xpos = reinterpret_cast<int*>(smem + L.xpos);
  uint32_t* qcnt = reinterpret_cast<uint32_t*>(smem + L.qcnt);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(smem + L.ctr);
  uint32_t* pref = reinterpret_cast<uint32_t*>(smem + L.pref);
  uint32_t* rcnt = reinterpret_cast<uint32_t*>(smem + L.rcnt);
  auto acc_full = [&](int s) { return smem_u32(bars + 1 + s); };
  auto stage_bar = [&](int s, int b) { return smem_u32(bars + 1 + NSLOT + 2 * s + b); };
  constexpr uint32_t kStageBytes = IN_IMG ? kImgTile : (uint32_t)kTile * 8u * 4u;
  auto stage_ptr = [&](int s, int b) { return smem + L.stage + (uint32_t)(2 * s + b) * kStageBytes; };
  auto lab_ptr = [&](int s, int b) { return smem + L.lab + (uint32_t)(2 * s + b) * kTile; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, R = NSLOT * G;

  if (warp == 0) {
    if (lane == 0) {
      mbar_init(smem_u32(bars), 1);
      for (int s = 0; s < NSLOT; ++s) {
        mbar_init(acc_full(s), 1);
        mbar_init(stage_bar(s, 0), 1);
        mbar_init(stage_bar(s, 1), 1);
      }
      fence_barrier_init();
      uint32_t tot = 0;
      for (int i = 0; i < p.ncp; ++i) tot += p.cp_len[i];
      mbar_arrive_expect_tx(smem_u32(bars), tot);
      for (int i = 0; i < p.ncp; ++i)
        bulk_g2s(sbase + p.cp_dst[i], p.packed + p.cp_src[i], p.cp_len[i], smem_u32(bars));
    }
    __syncwarp();
    tmem_alloc<COLS>(smem_u32(tmem_slot));
  }
  for (int i = threadIdx.x; i < NEPI * 12; i += blockDim.x) ctr[i] = 0u;
  // tiles of this segment: regions' tile counts, exclusive prefix in pref[0..R]
  int64_t num_tiles = p.num_tiles;
  if (IN_REG) {
    uint32_t c = 0;
    if ((int)threadIdx.x < R) {
      const uint32_t rc = __ldg(p.in_cnt + threadIdx.x);
      rcnt[threadIdx.x] = rc;
      c = (rc + kTile - 1) / kTile;
    }
    uint32_t x = c;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t* wt = reinterpret_cast<uint32_t*>(xpos);
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += wt[w];
    if ((int)threadIdx.x < R) pref[threadIdx.x + 1] = base + x;
    if (threadIdx.x == 0) pref[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (IN_REG) num_tiles = pref[R];
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  {  // ones block (bias folding): k = 0, 1, 2 of every row are 1.0
    if (warp < 4) {
      const uint32_t ones[8] = {0x3F803F80u, 0x00003F80u, 0u, 0u, 0u, 0u, 0u, 0u};
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kOnesCol, ones);
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  mbar_wait(smem_u32(bars), 0);

  const int s = warp / WPS;
  const int qw = warp & 3;
  const int half = (warp % WPS) >> 2;
  const int col0 = half * CPT;
  const bool lead = half == 0;
  const bool mma_warp = (warp % WPS) == 0;
  const bool issuer = mma_warp && lane == 0;
  const int rit = qw * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const float* hvec = reinterpret_cast<const float*>(smem + p.s_head) + col0;
  const float hconst = __ldg(reinterpret_cast<const float*>(p.packed + p.hc_off));
  uint32_t* cnt = ctr + warp * 12;
  const uint32_t slot_bar = 1u + (uint32_t)s;
  const uint32_t lead_bar = 3u + (uint32_t)s;                  // the slot's 4 lead warps
  const uint32_t half_bar = 8u + (uint32_t)(s * 4 + qw);       // the 2 warps of a row quarter
  const int d0 = D0C ? D0C : p.d0;
  const uint32_t idesc = make_idesc_bf16(128, W);
  const uint32_t acc_c = (uint32_t)(s * W);
  const uint32_t a_c = (uint32_t)(NSLOT * W + s * (W / 2));   // next A / held activations
  const uint32_t enc_c = (uint32_t)(NSLOT * W + NSLOT * (W / 2) + s * 8);  // segment 0 input
  const int region = s * G + blockIdx.x;                       // output region of this slot

  // input tile t -> (region, tile in region, valid rows)
  auto locate = [&](int64_t t, int& r, int& j, int& rows) {
    if (!IN_REG) {
      r = 0; j = 0;
      rows = (int)min((int64_t)kTile, p.a.n - t * kTile);
      return;
    }
    int lo = 0, hi = R;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pref[mid] <= (uint32_t)t) lo = mid; else hi = mid - 1;
    }
    r = lo;
    j = (int)(t - pref[lo]);
    rows = min(kTile, (int)(rcnt[lo] - (uint32_t)j * kTile));
  };

  auto sync_and_issue = [&](int li, int b) {
    tc_fence_before();
    asm volatile("bar.sync %0, %1;" ::"r"(slot_bar), "n"(WPS * 32) : "memory");
    if (mma_warp) {
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem + acc_c;
        if (li == 0 && !IN_IMG) {  // layer 0: encoded records (bias via the ones columns)
          mma_ts(d, tmem + enc_c, make_sdesc(sbase + p.s_w[0], 128u, (kEncK / 8u) * 128u), idesc, 0u);
        } else {
          mma_ts(d, tmem + kOnesCol, make_sdesc(sbase + p.s_bb[li], 128u, (kEncK / 8u) * 128u), idesc, 0u);
          const uint64_t bdesc = make_sdesc(sbase + p.s_w[li], 128u, (W / 8u) * 128u);
          if (li == 0) {  // A = the staged image tile (shared memory, K-major)
            const uint64_t adesc = make_sdesc(smem_u32(stage_ptr(s, b)), 2048u, 128u);
#pragma unroll
            for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
              mma_ss(d, adesc + (uint64_t)(kk * 256u), bdesc + (uint64_t)(kk * 16u), idesc, 1u);
          } else {
#pragma unroll
            for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
              mma_ts(d, tmem + a_c + kk * 8u, bdesc + (uint64_t)(kk * 16u), idesc, 1u);
          }
        }
        mma_commit(acc_full(s));
      }
      __syncwarp();
    }
  };

  auto stage_issue = [&](int64_t t, int b) {
    if (!issuer || t >= num_tiles) return;
    const uint32_t bar = stage_bar(s, b);
    if (IN_IMG) {
      int r, j, rows;
      locate(t, r, j, rows);
      const int64_t ti = (int64_t)r * p.cap + j;
      mbar_arrive_expect_tx(bar, kImgTile + (uint32_t)kTile);
      bulk_g2s(smem_u32(stage_ptr(s, b)), p.in_img + ti * kImgTile, kImgTile, bar);
      bulk_g2s(smem_u32(lab_ptr(s, b)), p.in_lab + ti * kTile, kTile, bar);
    } else if (IN == 2) {  // a whole region tile (rows past the region count are masked)
      int r, j, rows;
      locate(t, r, j, rows);
      const int64_t ti = (int64_t)r * p.cap + j;
      const uint32_t qb = (uint32_t)(kTile * d0 * 4);
      mbar_arrive_expect_tx(bar, qb + (uint32_t)kTile);
      bulk_g2s(smem_u32(stage_ptr(s, b)), p.in_rec + ti * kTile * d0, qb, bar);
      bulk_g2s(smem_u32(lab_ptr(s, b)), p.in_lab + ti * kTile, kTile, bar);
    } else {
      if ((t + 1) * kTile > p.a.n) return;  // ragged last tile: read directly
      const uint32_t qb = (uint32_t)(kTile * d0 * 4);
      mbar_arrive_expect_tx(bar, qb + (uint32_t)kTile);
      bulk_g2s(smem_u32(stage_ptr(s, b)), p.a.q + t * kTile * d0, qb, bar);
      bulk_g2s(smem_u32(lab_ptr(s, b)), p.a.y + t * kTile, kTile, bar);
    }
  };

  uint32_t sph[2] = {0u, 0u};
  int ycur = 0;      // lead threads: label byte of the staged row (bit 0 y, bit 1 counted non-finite)
  bool vcur = false;
  const float* srccur = nullptr;  // REC: the staged row's record in global memory (lead threads)
  auto put_input = [&](int64_t t, int i) {
    const int b = i & 1;
    int r, j, rows;
    locate(t, r, j, rows);
    if (IN_IMG) {
      if (lead || mma_warp) {
        mbar_wait(stage_bar(s, b), sph[b]);
        sph[b] ^= 1u;
      }
      vcur = rit < rows;
      ycur = lead ? (int)lab_ptr(s, b)[rit] : 0;
      sync_and_issue(0, b);
      return;
    }
    if (lead) {
      float x[8];
      const bool full = IN == 2 || (t + 1) * kTile <= p.a.n;
      vcur = rit < rows;
      int yv;
      if (IN == 2) srccur = p.in_rec + (((int64_t)r * p.cap + j) * kTile + rit) * d0;
      else srccur = p.a.q + (t * kTile + rit) * d0;
      if (full) {
        mbar_wait(stage_bar(s, b), sph[b]);
        sph[b] ^= 1u;
        const float* qs = reinterpret_cast<const float*>(stage_ptr(s, b)) + rit * d0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) x[jj] = jj < d0 ? qs[jj] : 0.f;
        yv = (int)lab_ptr(s, b)[rit];
      } else {
        const int64_t rr = t * kTile + rit;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) x[jj] = (vcur && jj < d0) ? __ldg(p.a.q + rr * d0 + jj) : 0.f;
        yv = vcur ? (int)__ldg(p.a.y + rr) : 0;
      }
      if (IN == 2) {
        ycur = yv;  // bit 0 y, bit 1 non-finite already counted (set by an earlier segment)
      } else {
        if (vcur && yv > 1) atomicOr(p.a.flags, kFlagLabel);
        ycur = yv != 0 ? 1 : 0;
      }
      uint32_t c[8];
      encode_cols<D0C, true>(x, d0, c);
      tmem_st8(trow + enc_c, c);
      tmem_wait_st();
    }
    sync_and_issue(0, b);
  };

  int64_t tile = blockIdx.x + (int64_t)s * G;
  stage_issue(tile, 0);
  stage_issue(tile + NSLOT * G, 1);
  int i_tile = 0;
  if (tile < num_tiles) put_input(tile, 0);
  uint32_t ph = 0, par = 0;
  uint32_t out_base = 0;  // survivors appended to this slot's region so far (lead warps)
  uint8_t* out_img = p.out_img;
  while (tile < num_tiles) {
    const int64_t next = tile + NSLOT * G;
    int ythis = 0;
    bool vthis = false;
    const float* srcthis = nullptr;
    float za = lead ? hconst : 0.f, zb = 0.f;
#pragma unroll
    for (int li = 0; li < SEG; ++li) {
      mbar_wait(acc_full(s), ph);
      ph ^= 1u;
      tc_fence_after();
      if (li == 0) stage_issue(next + NSLOT * G, i_tile & 1);
      const bool last = li == SEG - 1;
      uint32_t v[CPT];
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        tmem_ld32(trow + acc_c + (uint32_t)(col0 + 32 * c), *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
      tmem_wait_ld();
      if (last) {  // accumulator in registers: start the slot's next tile
        ythis = ycur;
        vthis = vcur;
        srcthis = srccur;
        ++i_tile;
        if (next < num_tiles) put_input(next, i_tile);
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        float* t = reinterpret_cast<float*>(v + 32 * c);
        if (!(last && FINAL)) {  // next A operand, or the activations handed to the next segment
          uint32_t pk[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) pk[jj] = pack_relu_bf16x2(t[2 * jj], t[2 * jj + 1]);
          tmem_st16(trow + a_c + (uint32_t)((col0 + 32 * c) / 2), pk);
        }
        if (last) {
#pragma unroll
          for (int i = 0; i < 32; ++i) t[i] = relu_nan(t[i]);
          const int o = 32 * c;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 w4 = *reinterpret_cast<const float4*>(hvec + o + i);
            fma2(za, zb, t[i], t[i + 1], w4.x, w4.y);
            fma2(za, zb, t[i + 2], t[i + 3], w4.z, w4.w);
          }
        }
      }
      if (!last) {
        tmem_wait_st();
        sync_and_issue(li + 1, 0);
      }
    }
    // combine the two column halves of each row
    float z = za + zb;
    {
      float* xb = xch + ((s * 2 + par) * 4 + qw) * 32 + lane;
      if (!lead) xb[0] = z;
      asm volatile("bar.sync %0, 64;" ::"r"(half_bar) : "memory");
      if (lead) z += xb[0];
    }
    const bool yy = (ythis & 1) != 0;
    const bool nf_done = (ythis & 2) != 0;
    if (FINAL) {
      if (lead) {
        const unsigned full = 0xFFFFFFFFu;
        const bool pred = vthis && z >= p.tau_end;
        const uint32_t bp = __ballot_sync(full, pred);
        const uint32_t bv = __ballot_sync(full, vthis);
        const uint32_t by = __ballot_sync(full, vthis && yy);
        const uint32_t bn = __ballot_sync(full, vthis && !nf_done && !isfinite(z));
        if (lane == 0) {
          cnt[0] += __popc(bp & by);
          cnt[1] += __popc(bp & ~by);
          cnt[2] += __popc(bv & ~bp & by);
          cnt[3] += __popc(bv & ~bp & ~by);
          cnt[6] += __popc(bv & ~bp);
          cnt[8] += __popc(bn);
        }
      }
    } else {
      tmem_wait_st();
      int pos = -1;
      if (lead) {
        const unsigned full = 0xFFFFFFFFu;
        const bool surv = vthis && z >= p.tau_end;  // NaN exits
        const bool nf = vthis && !nf_done && !isfinite(z);
        const uint32_t bs = __ballot_sync(full, surv);
        const uint32_t bv = __ballot_sync(full, vthis);
        const uint32_t by = __ballot_sync(full, vthis && yy);
        const uint32_t bn = __ballot_sync(full, nf);
        if (lane == 0) {
          cnt[2] += __popc(bv & ~bs & by);
          cnt[3] += __popc(bv & ~bs & ~by);
          cnt[4 + HEAD] += __popc(bv & ~bs);
          cnt[8] += __popc(bn);
          qcnt[(s * 2 + par) * 4 + qw] = __popc(bs);
        }
        asm volatile("bar.sync %0, 128;" ::"r"(lead_bar) : "memory");
        const uint32_t* qc = qcnt + (s * 2 + par) * 4;
        uint32_t below = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t cq = qc[q];
          below += q < qw ? cq : 0u;
          tot += cq;
        }
        if (surv) {
          pos = (int)(out_base + below + __popc(bs & ((1u << lane) - 1u)));
          p.out_lab[(int64_t)region * p.cap * kTile + pos] = (uint8_t)((yy ? 1 : 0) | ((nf || nf_done) ? 2 : 0));
          if (REC) {  // the row's record (16 B for c4): the next segment recomputes from it
            float* o = p.out_rec + ((int64_t)region * p.cap * kTile + pos) * d0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
              if (jj < d0) o[jj] = __ldg(srcthis + jj);
          }
        }
        out_base += tot;
        xpos[((s * 2 + par) * 4 + qw) * 32 + lane] = pos;
      }
      if (!REC) {
      asm volatile("bar.sync %0, 64;" ::"r"(half_bar) : "memory");
      if (!lead) pos = xpos[((s * 2 + par) * 4 + qw) * 32 + lane];
#ifndef NB_EXIT_NOSTORE
      uint32_t w[32];
      tmem_ld32(trow + a_c + (uint32_t)(col0 / 2), w);
      tmem_wait_ld();
      if (pos >= 0) {
        uint8_t* ot = out_img + ((int64_t)region * p.cap + (pos >> 7)) * kImgTile;
        st_img_row(ot, pos & (kTile - 1), col0 / 8, w);
      }
#endif
      }
    }
    par ^= 1u;
    tile = next;
  }
  if (!FINAL && lead && qw == 0 && lane == 0) p.out_cnt[region] = out_base;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<COLS>(tmem);
  }
  if (warp == 1) flush_cta_counts(ctr, NEPI, 2, p.a.counts);
  if (warp == 1 && p.a.ticket) finalize_counts(p.a, false);
}

template <int SEG, int IN, int HEAD, int D0C, bool REC = false>
cudaError_t launch_seg(const nb_model* m, ExitParams p, cudaStream_t st) {
  const ExitSmem L(p.wbytes, IN == 1);
  const size_t smem = std::max<size_t>(L.total, 116 * 1024);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = k_score_exit<SEG, IN, HEAD, D0C, REC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<m->num_sms, kXWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

// Shared weight area of segment [lb, lb + seg): layer images, bias blocks, head.
void plan_weights(const nb_model* m, ExitParams& p, int lb, int seg, int head) {
  const PackLayout& pl = m->pl;
  uint32_t o = 0;
  p.ncp = 0;
  auto add = [&](uint32_t src, uint32_t len) {
    p.cp_src[p.ncp] = src;
    p.cp_dst[p.ncp] = o;
    p.cp_len[p.ncp] = len;
    ++p.ncp;
    const uint32_t d = o;
    o += (len + 127u) & ~127u;
    return d;
  };
  for (int i = 0; i < seg; ++i) {
    const int l = lb + i;
    p.s_w[i] = add(pl.off_w[l], (uint32_t)kXW * pl.k_of[l] * 2u);
    p.s_bb[i] = l >= 1 ? add(pl.off_bb[l], (uint32_t)kXW * kEncK * 2u) : 0u;
  }
  // head vector u_k (or w_out); its constant c_k (or b_out) is read from global
  p.s_head = add(head >= 0 ? pl.off_u[head] : pl.off_wout, (uint32_t)kXW * 4u);
  p.hc_off = head >= 0 ? pl.off_c + 4u * (uint32_t)head : pl.off_bout;
  p.wbytes = o;
}

}  // namespace

bool exit_compaction_supported(const nb_model* m) {
  const nb_desc& d = m->d;
  return d.precision == NB_BF16 && d.width == kXW && m->pl.pairs == 1 && m->pl.bias_l0 != 0 &&
         m->pl.k_of[0] == (uint32_t)kEncK &&
         d.activation == NB_RELU && d.pe_depth == 0 &&
         d.n_heads == 2 && d.head_after[0] == 2 && d.head_after[1] == 4 && d.hidden_layers == 6 &&
         m->num_sms * kXSlots <= kMaxRegions;
}

// Score with early exits: per chunk of rows, segment 0 (records -> head 1),
// segment 1 (image -> head 2), segment 2 (image -> output, classify).  All
// launches add to a.counts; the last one finalises into a.fin_out.
static int64_t g_exit_chunk = 0;  // rows per chunk override (tests), 0 = default
extern "C" void nb_debug_set_exit_chunk(int64_t rows) { g_exit_chunk = rows; }
static int g_exit_records = 0;    // record hand-off instead of activation images
extern "C" void nb_debug_set_exit_records(int on) { g_exit_records = on ? 1 : 0; }

cudaError_t launch_score_exit(nb_model* m, const FwdArgs& a, cudaStream_t st, int* kernels) {
  *kernels = 0;
  // hand-off between segments: the survivors' bf16 activation images (256 B
  // per c4 row; default, the faster one) or their fp32 records (16 B; the
  // later segments recompute the earlier layers: 8x less DRAM traffic, ~7 %
  // slower on a trained c4 model) — nb_debug_set_exit_records
  // or NB_EXIT_RECORDS=1
  static const bool env_records = getenv("NB_EXIT_RECORDS") != nullptr;
  const bool images = !(env_records || g_exit_records);
  static const int64_t env_chunk = [] {
    const char* e = getenv("NB_EXIT_CHUNK");
    return e ? atoll(e) : (int64_t)1 << 24;
  }();
  const int64_t want = std::max<int64_t>(kTile, (g_exit_chunk > 0 ? g_exit_chunk : env_chunk) / kTile * kTile);
  const int64_t chunk = std::min<int64_t>(want, (a.n + kTile - 1) / kTile * kTile);
  const int R = m->num_sms * kXSlots;
  const int d0 = m->d0;
  const int64_t t0 = (chunk + kTile - 1) / kTile;
  const int64_t cap = (t0 + R + R - 1) / R;
  const size_t row_bytes = images ? (size_t)kImgTile : (size_t)kTile * d0 * 4;  // per region tile
  const size_t img_bytes = (size_t)R * cap * row_bytes, lab_bytes = (size_t)R * cap * kTile;
  const size_t need = 2 * (img_bytes + lab_bytes) + 2 * 4 * (size_t)R;
  if (m->exit_scratch_bytes < need) {
    cudaFree(m->exit_scratch);
    m->exit_scratch = nullptr;
    m->exit_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&m->exit_scratch, need);
    if (e != cudaSuccess) return e;
    m->exit_scratch_bytes = need;
  }
  uint8_t* base = (uint8_t*)m->exit_scratch;
  uint8_t* img[2] = {base, base + img_bytes};
  uint8_t* lab[2] = {base + 2 * img_bytes, base + 2 * img_bytes + lab_bytes};
  uint32_t* cnt[2] = {(uint32_t*)(base + 2 * (img_bytes + lab_bytes)),
                      (uint32_t*)(base + 2 * (img_bytes + lab_bytes)) + R};
  const int h0 = m->d.head_after[0], h1 = m->d.head_after[1], L = m->d.hidden_layers;
  for (int64_t r0 = 0; r0 < a.n; r0 += chunk) {
    const int64_t rows = std::min(chunk, a.n - r0);
    const bool last_chunk = r0 + rows >= a.n;
    ExitParams p{};
    p.a = a;
    p.a.ticket = nullptr;
    p.packed = m->packed;
    p.d0 = d0;
    p.cap = cap;
    // segment 0: records -> layers [0, h0) -> head 1
    p.a.q = a.q + r0 * d0;
    p.a.y = a.y + r0;
    p.a.n = rows;
    p.num_tiles = (rows + kTile - 1) / kTile;
    p.lb = 0;
    p.tau_end = a.tau[1];
    plan_weights(m, p, 0, h0, 0);
    p.out_lab = lab[0]; p.out_cnt = cnt[0];
    cudaError_t e;
    if (images) {
      p.out_img = img[0];
      e = d0 == 4 ? launch_seg<2, 0, 0, 4>(m, p, st) : launch_seg<2, 0, 0, 0>(m, p, st);
    } else {
      p.out_rec = (float*)img[0];
      e = d0 == 4 ? launch_seg<2, 0, 0, 4, true>(m, p, st) : launch_seg<2, 0, 0, 0, true>(m, p, st);
    }
    if (e != cudaSuccess) return e;
    *kernels += 3;
    // segment 1: image -> layers [h0, h1) -> head 2, or records -> layers [0, h1) -> head 2
    p.tau_end = a.tau[2];
    p.in_lab = lab[0]; p.in_cnt = cnt[0];
    p.out_lab = lab[1]; p.out_cnt = cnt[1];
    if (images) {
      p.lb = h0;
      plan_weights(m, p, h0, h1 - h0, 1);
      p.in_img = img[0]; p.out_img = img[1];
      e = launch_seg<2, 1, 1, 0>(m, p, st);
    } else {
      p.lb = 0;
      plan_weights(m, p, 0, h1, 1);
      p.in_rec = (const float*)img[0]; p.out_rec = (float*)img[1];
      e = d0 == 4 ? launch_seg<4, 2, 1, 4, true>(m, p, st) : launch_seg<4, 2, 1, 0, true>(m, p, st);
    }
    if (e != cudaSuccess) return e;
    // segment 2: image -> layers [h1, L) -> output, or records -> layers [0, L) -> output; classify
    p.tau_end = a.tau[0];
    p.in_lab = lab[1]; p.in_cnt = cnt[1];
    p.out_img = nullptr; p.out_rec = nullptr; p.out_lab = nullptr; p.out_cnt = nullptr;
    if (last_chunk) p.a.ticket = a.ticket;
    if (images) {
      p.lb = h1;
      plan_weights(m, p, h1, L - h1, -1);
      p.in_img = img[1];
      e = launch_seg<2, 1, -1, 0>(m, p, st);
    } else {
      p.lb = 0;
      plan_weights(m, p, 0, L, -1);
      p.in_rec = (const float*)img[1];
      e = d0 == 4 ? launch_seg<6, 2, -1, 4>(m, p, st) : launch_seg<6, 2, -1, 0>(m, p, st);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace nb
