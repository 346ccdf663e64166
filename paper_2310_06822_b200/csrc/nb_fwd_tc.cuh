// nb_fwd_tc.cuh — fused MLP forward + classify/count/calibrate on tcgen05
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
// register file); weights are bulk-copied into shared memory once per CTA.
//
// CTA (persistent, one per SM) = NSLOT x WPS epilogue warps + 1 MMA warp.
// Each slot owns one 128-row tile in flight; its WPS warps split the tile's
// columns (warp w reads TMEM lane quarter w % 4, column half (w % WPS) / 4).
// The MMA thread walks the slots round-robin layer by layer, so one slot's
// epilogue overlaps the other slots' MMAs.  Synchronisation: mbarriers
// a_full[s] (epilogue -> MMA: next A operand is in TMEM) and acc_full[s]
// (tcgen05.commit -> epilogue: accumulator ready).
// Measured primitive costs that shape this plan (tools/tmem_bench.cu): an
// M=128 K=16 MMA costs >= 46 cycles for N <= 64 and N/2 cycles for N >= 128;
// one warp's tcgen05.ld of 64 columns + wait costs ~93 cycles, so the
// epilogue needs many warps and all loads of a layer issued before one wait.
#pragma once
#include <cuda_bf16.h>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

struct TcParams {
  FwdArgs a;
  const uint8_t* packed;
  PackLayout pl;
  int d0, L, nh, ha0, ha1;
  int act, pe, din, k0;  // generic kernels: nb_activation, PE depth, layer-1 inputs and K (R41, R42)
  int64_t num_tiles;
  unsigned long long* trace;  // NB_TRACE builds only: timeline of CTA 0
};

#ifdef NB_TRACE
// Debug timeline (tools/trace_fwd.py): each tracing thread of CTA 0 owns a
// region of 2000 (clock64, code) pairs; stores only, no atomics on the path.
#define NB_TR(region, code)                                                          \
  do {                                                                               \
    if (blockIdx.x == 0 && p.trace && tr_i < 2000) {                                 \
      p.trace[((region) * 2000 + tr_i) * 2] = clock64();                            \
      p.trace[((region) * 2000 + tr_i) * 2 + 1] = (unsigned long long)(code);       \
      ++tr_i;                                                                        \
    }                                                                                \
  } while (0)
#else
#define NB_TR(region, code) \
  do {                      \
  } while (0)
#endif
#define NB_EV(type, s, l) ((type) | ((s) << 4) | ((l) << 8))

// a1 encode: fp32 record -> the K = 16 bf16 layer-1 operand of one row,
// [x_hi(0..d0-1), x_lo(0..d0-1), 0 ...] (R20), two bf16 per 32-bit
// column (even k in the low half).  ONES puts 1.0 at k = 2 d0 .. 2 d0 + 2: the
// A side of layer 1's bias columns (bias folding).  D0C is the
// compile-time d0 of the specialised kernels (0 = use the run-time d0).
template <int D0C, bool ONES>
__device__ __forceinline__ void encode_cols(const float* x, int d0_rt, uint32_t (&col)[8]) {
  const int d0 = D0C ? D0C : d0_rt;
  uint32_t h[8], l[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    __nv_bfloat16 hi = __float2bfloat16_rn(x[j]);
    __nv_bfloat16 lo = __float2bfloat16_rn(x[j] - __bfloat162float(hi));
    h[j] = __bfloat16_as_ushort(hi);
    l[j] = __bfloat16_as_ushort(lo);
  }
  // element e of the 16-wide row: e < d0 -> hi[e]; d0 <= e < 2 d0 -> lo[e - d0]; else 0
  uint32_t e[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    uint32_t v = 0;
    if (D0C) {
      if (k < D0C) v = h[k];
      else if (k < 2 * D0C) v = l[k - D0C];
      else if (ONES && k < 2 * D0C + 3) v = 0x3F80u;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v = (k == j && j < d0) ? h[j] : v;
        v = (k == d0 + j && j < d0) ? l[j] : v;
      }
      if (ONES && k >= 2 * d0 && k < 2 * d0 + 3) v = 0x3F80u;
    }
    e[k] = v;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) col[c] = e[2 * c] | (e[2 * c + 1] << 16);
}

// a1 encode with positional encoding (EXT kernels, R42): the
// d_in = D0 (1 + pe) features [x, sin(2^k pi x), cos(2^k pi x) per frequency]
// of one record, each split into a bf16 (hi, lo) pair, in the PE operand
// layout (PackLayout::pe_lo): hi at [0, d_in), the bias ones at
// [d_in, d_in + 3), lo at [32, 32 + d_in); K = 64, 32 packed columns.  D0 is
// compile-time so every feature index is a register.
template <int D0>
__device__ __forceinline__ void encode_cols_pe(const float* x, int pe, uint32_t (&col)[32]) {
  constexpr int kMaxF = 29;  // d_in + 3 <= 32
  const int din = D0 * (1 + pe);
  float f[kMaxF];
#pragma unroll
  for (int j = 0; j < kMaxF; ++j) f[j] = j < D0 ? x[j] : 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (2 * k < pe) {
#pragma unroll
      for (int j = 0; j < D0; ++j) {
        float sv, cv;
        sincospif(ldexpf(x[j], k), &sv, &cv);
        if (D0 + 2 * k * D0 + j < kMaxF) f[D0 + 2 * k * D0 + j] = sv;
        if (D0 + (2 * k + 1) * D0 + j < kMaxF) f[D0 + (2 * k + 1) * D0 + j] = cv;
      }
    }
  }
  uint32_t e[64];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const uint32_t hi = k < kMaxF ? __bfloat16_as_ushort(__float2bfloat16_rn(f[k < kMaxF ? k : 0])) : 0u;
    e[k] = k < din ? hi : (k < din + 3 ? 0x3F80u : 0u);
    uint32_t lo = 0u;
    if (k < kMaxF) {
      const float v = f[k];
      lo = __bfloat16_as_ushort(__float2bfloat16_rn(v - __bfloat162float(__float2bfloat16_rn(v))));
    }
    e[32 + k] = k < din ? lo : 0u;
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) col[c] = e[2 * c] | (e[2 * c + 1] << 16);
}

// sine hidden activation (R41): the SFU sine (sin.approx:
// x / 2 pi, then MUFU.SIN); |error| <= ~2^-21 + |x| 2^-22, i.e. < 3e-5 for
// |x| < 100 — far below the bf16 rounding (2^-9 relative) of the result
__device__ __forceinline__ float sin_act(float x) { return __sinf(x); }

__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fma2(float& c0, float& c1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%0, %1};\n\t"
      "fma.rn.f32x2 rc, ra, rb, rc;\n\tmov.b64 {%0, %1}, rc;}"
      : "+f"(c0), "+f"(c1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Classification with per-warp counters kept in shared memory (lane 0 adds
// the warp's ballot counts) to save registers in the epilogue warps.  Counts
// come from three or four ballots per warp: pred, y, valid (and the exit bins
// when the model has heads); with no heads the bins are derived at flush.
template <int MODE, int NHC>
__device__ __forceinline__ void classify_row_smem(uint32_t* cnt, uint32_t (&key)[3], bool valid,
                                                  int y, float z, const float* e, int nh_rt,
                                                  const float* tau, unsigned int* flags,
                                                  int invert = 0) {
  const int nh = NHC >= 0 ? NHC : nh_rt;
  if (MODE == kCalibrate) {
    if (valid && (invert ? y == 0 : y == 1)) {
      key[0] = min(key[0], dkey(invert ? -z : z));
      if (nh > 0) key[1] = min(key[1], dkey(e[0]));
      if (nh > 1) key[2] = min(key[2], dkey(e[1]));
    }
  }
  if (MODE == kScore && NHC == 0) {
    // no exit heads: count the raw masks tp = pred & y, pred, pos = y (and
    // non-finite); finalize_counts derives fp, fn, tn and the bins from them
    const unsigned full = 0xFFFFFFFFu;
    const uint32_t bp = __ballot_sync(full, valid && z >= tau[0]);
    const uint32_t by = __ballot_sync(full, valid && y != 0);
    const uint32_t bn = __ballot_sync(full, valid && !isfinite(z));
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(cnt + 0, (uint32_t)__popc(bp & by));
      atomicAdd(cnt + 1, (uint32_t)__popc(bp));
      atomicAdd(cnt + 2, (uint32_t)__popc(by));
      if (bn) atomicAdd(cnt + 8, (uint32_t)__popc(bn));
    }
  } else if (MODE == kScore) {
    const unsigned full = 0xFFFFFFFFu;
    bool pass0 = true, pass1 = true;
    if (nh > 0) pass0 = e[0] >= tau[1];
    if (nh > 1) pass1 = e[1] >= tau[2];
    const bool pred = pass0 && pass1 && z >= tau[0];
    const bool nonfin = !isfinite(z) || (nh > 0 && !isfinite(e[0])) || (nh > 1 && !isfinite(e[1]));
    const uint32_t bv = __ballot_sync(full, valid);
    const uint32_t bp = __ballot_sync(full, valid && pred);
    const uint32_t by = __ballot_sync(full, valid && y != 0);
    const uint32_t bn = __ballot_sync(full, valid && nonfin);
    uint32_t b0 = 0, b1 = 0;
    if (nh > 0) {
      b0 = __ballot_sync(full, valid && !pass0);
      b1 = __ballot_sync(full, valid && pass0 && !pass1);
    }
    if ((threadIdx.x & 31) == 0) {
      cnt[0] += __popc(bp & by);
      cnt[1] += __popc(bp & ~by);
      cnt[2] += __popc(bv & ~bp & by);
      cnt[3] += __popc(bv & ~bp & ~by);
      if (nh > 0) {  // exit bins: exit@1, exit@2, final-negative (final-positive = tp + fp)
        cnt[4] += __popc(b0);
        cnt[5] += __popc(b1);
        cnt[6] += __popc(bv & ~bp & ~b0 & ~b1);
      }
      cnt[8] += __popc(bn);
    }
  }
  if (valid && y > 1) atomicOr(flags, kFlagLabel);
}

template <int MODE>
__device__ __forceinline__ void flush_smem(uint32_t* cnt, uint32_t (&key)[3], int nh,
                                           unsigned long long* counts, unsigned int* keys) {
  const int lane = threadIdx.x & 31;
  if (MODE == kCalibrate) {
    for (int k = 0; k <= nh; ++k) {
      const uint32_t m = __reduce_min_sync(0xFFFFFFFFu, key[k]);
      if (lane == 0 && m != 0xFFFFFFFFu) atomicMin(keys + k, m);
    }
  }
  if (MODE == kScore && lane == 0) {
    cnt[7] = cnt[0] + cnt[1];                        // final-positive
    if (nh == 0) cnt[6] = cnt[2] + cnt[3];           // final-negative
    for (int i = 0; i < kNumCounters; ++i)
      if (cnt[i]) atomicAdd(counts + i, (unsigned long long)cnt[i]);
  }
}

#ifndef NB_W64_NSLOT  // measurement variants: build.py -DNB_W64_NSLOT=4 -DNB_W64_WPS=8
#define NB_W64_NSLOT 5
#define NB_W64_WPS 4
#endif
template <int W>
struct TcPlan;
template <>
struct TcPlan<32> { static constexpr int NSLOT = 4, WPS = 4, COLS = 256; };
template <>
struct TcPlan<64> { static constexpr int NSLOT = NB_W64_NSLOT, WPS = NB_W64_WPS, COLS = 512; };
template <>
struct TcPlan<128> { static constexpr int NSLOT = 2, WPS = 8, COLS = 512; };

// LC / H0C / H1C: compile-time layer count and exit-head layers (1-based, 0 =
// none) of the specialised instantiations; LC == 0 selects the generic kernel
// that reads them from TcParams at run time.
//
// There is no dedicated MMA warp: each slot's lead warp (lane quarter 0,
// column half 0) issues its own slot's MMAs right after the slot's warps
// meet at a named barrier, so every slot is an independent chain
//   [stage A in TMEM] -> bar.sync -> MMA layer l -> commit -> acc_full ->
//   [epilogue l: ld, bias, ReLU, bf16 pack, st] -> bar.sync -> MMA layer l+1
// and the tensor pipe interleaves the slots' MMAs (no head-of-line blocking).
//
// BF (bias folding): every layer's bias enters the accumulator through the
// tensor core instead of an epilogue FADD per element — layer 1 through the
// encoder's ones columns, layer l >= 1 through one extra K = 16 MMA whose A is
// a constant ones block in TMEM and whose B holds the exact bf16 split of b_l
// (PackLayout::off_bb).  The epilogue of a hidden layer is then just
// tcgen05.ld -> cvt.rn.relu.bf16x2 -> tcgen05.st.  D0C: compile-time d0.
// EXT: generic kernels of sine / positional-encoding nets (run-time p.act,
// p.pe; R41, R42) — kept apart so the ReLU kernels' register
// allocation is unaffected.
template <int W, int LC, int H0C, int H1C, int MODE, int D0C, bool BF, bool EXT = false>
__global__ void __launch_bounds__(TcPlan<W>::NSLOT * TcPlan<W>::WPS * 32, 1)
    k_fwd_tc(const TcParams p) {
  griddep_wait();  // programmatic dependent in the training chain (no-op otherwise)
  const int L = LC ? LC : p.L;
  const int NH = LC ? ((H0C ? 1 : 0) + (H1C ? 1 : 0)) : p.nh;
  const int h0 = LC ? H0C - 1 : (p.nh > 0 ? p.ha0 - 1 : -1);
  const int h1 = LC ? H1C - 1 : (p.nh > 1 ? p.ha1 - 1 : -1);
  constexpr int NSLOT = TcPlan<W>::NSLOT, WPS = TcPlan<W>::WPS, COLS = TcPlan<W>::COLS;
  constexpr int NEPI = NSLOT * WPS;        // warps
  constexpr int CPT = W * 4 / WPS;         // accumulator columns per thread
  constexpr int NCH = CPT / 32;            // 32-column chunks per thread
  // With enough registers all of a layer's loads are issued before one wait,
  // and the next tile is staged as soon as the last layer's accumulator is in
  // registers (its layer-0 MMA then overlaps this tile's output epilogue).
  constexpr bool kAllLoads = NEPI <= 16 || (BF && W == 64);
  constexpr int NHC = LC ? ((H0C ? 1 : 0) + (H1C ? 1 : 0)) : -1;
  constexpr uint32_t kOnesCol = COLS - 8;  // bias-folding A operand (8 columns)
  static_assert(CPT % 32 == 0, "chunking");
  static_assert(NSLOT * W + NSLOT * (W / 2) + (BF ? 8 : 0) <= COLS, "TMEM plan");
  static_assert(NSLOT <= 7, "named barriers 1..NSLOT and 8..");
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_off = (p.pl.bytes + 15u) & ~15u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_off);
  // bars[0] weights, bars[1 + s] acc_full of slot s
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 + 2 * NSLOT);  // 16-B aligned
  float* xch = reinterpret_cast<float*>(tmem_slot + 4);  // [NSLOT][2][4][32][3] head partials
  uint32_t* ctr = reinterpret_cast<uint32_t*>(xch + NSLOT * 2 * 4 * 32 * 3);  // [NEPI][12]
  uint64_t* sbars = reinterpret_cast<uint64_t*>(ctr + NEPI * 12);            // [NSLOT][2]
  float* qst = reinterpret_cast<float*>(sbars + 2 * NSLOT);                  // [NSLOT][2][128*8]
  uint8_t* yst = reinterpret_cast<uint8_t*>(qst + NSLOT * 2 * kTile * 8);   // [NSLOT][2][128]
  // UMMA B descriptors of every layer's weight image ([0, 8)) and bias block
  // ([8, 16)), computed once so the issuing lane only loads them
  uint64_t* dtab = reinterpret_cast<uint64_t*>(yst + NSLOT * 2 * kTile);
  auto stage_bar = [&](int s, int b) { return smem_u32(sbars + 2 * s + b); };
  auto q_stage = [&](int s, int b) { return qst + (size_t)(2 * s + b) * kTile * 8; };
  auto y_stage = [&](int s, int b) { return yst + (size_t)(2 * s + b) * kTile; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef NB_TRACE
  unsigned long long tr_i = 0;
#endif
  auto acc_full = [&](int s) { return smem_u32(bars + 1 + s); };
  auto acc_col = [](int s) { return (uint32_t)(s * W); };
  auto a_col = [](int s) { return (uint32_t)(NSLOT * W + s * (W / 2)); };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t w_bar = smem_u32(bars);
      mbar_init(w_bar, 1);
      for (int s = 0; s < NSLOT; ++s) {
        mbar_init(acc_full(s), 1);
        mbar_init(stage_bar(s, 0), 1);
        mbar_init(stage_bar(s, 1), 1);
      }
      fence_barrier_init();
      mbar_arrive_expect_tx(w_bar, p.pl.bytes);
      for (uint32_t off = 0; off < p.pl.bytes; off += 32768u) {
        const uint32_t len = min(32768u, p.pl.bytes - off);
        bulk_g2s(sbase + off, p.packed + off, len, w_bar);
      }
    }
    __syncwarp();
    tmem_alloc<COLS>(smem_u32(tmem_slot));
  }
  for (int i = threadIdx.x; i < NEPI * 12; i += blockDim.x) ctr[i] = 0u;
  if (threadIdx.x < kMaxLayers) {
    const int l = threadIdx.x;
    dtab[l] = make_sdesc(sbase + p.pl.off_w[l], 128u, (l == 0 ? p.pl.k_of[0] / 8u : W / 8u) * 128u);
    dtab[kMaxLayers + l] = make_sdesc(sbase + p.pl.off_bb[l], 128u, (kEncK / 8u) * 128u);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  NB_CHECK((tmem & 0xFFFFu) == 0u);  // the whole allocation starts at column 0
  if (BF) {  // ones block: k = 0, 1, 2 of every row are 1.0 (bf16), the rest 0
    if (warp < 4) {
      const uint32_t ones[8] = {0x3F803F80u, 0x00003F80u, 0u, 0u, 0u, 0u, 0u, 0u};
      tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kOnesCol, ones);
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const bool dyn_n = MODE == kForward && p.a.n_dev;  // device-side row count (hierarchies)
  const int64_t n = dyn_n ? (int64_t)*p.a.n_dev : p.a.n;
  const int64_t num_tiles = dyn_n ? (n + kTile - 1) / kTile : p.num_tiles;
  const int64_t G = gridDim.x;

  const int s = warp / WPS;              // tile slot
  const int qw = warp & 3;               // TMEM lane quarter
  const int half = (warp % WPS) >> 2;    // column half (WPS == 8)
  const int col0 = half * CPT;
  const bool lead = half == 0;           // owns input staging and classification
  const bool mma_warp = (warp % WPS) == 0;             // issues the slot's MMAs
  const bool issuer = mma_warp && lane == 0;           // stages the slot's records
  const int rit = qw * 32 + lane;        // row within the tile
  const uint32_t trow = tmem + ((uint32_t)(qw * 32) << 16);
  const float* bias_all = reinterpret_cast<const float*>(smem + p.pl.off_bias);
  const float* wout = reinterpret_cast<const float*>(smem + p.pl.off_wout) + col0;
  float bout = 0.f;  // read once the weights are resident (below)
  const float* cst = reinterpret_cast<const float*>(smem + p.pl.off_c);
  const float* u0 = reinterpret_cast<const float*>(smem + p.pl.off_u[0]) + col0;
  const float* u1 = reinterpret_cast<const float*>(smem + p.pl.off_u[1]) + col0;
  uint32_t* cnt = ctr + warp * 12;       // per-warp counters in shared memory
  uint32_t key[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
  uint32_t ph = 0;
  const int nl = 1 + NH;
  const uint32_t slot_bar = 1u + (uint32_t)s;              // all WPS warps of the slot
  // the 2 warps of a row quarter combine their column halves; with too many
  // slots for private named barriers the whole slot meets instead
  constexpr bool kPairBars = 8 + NSLOT * 4 <= 16;
  const uint32_t half_bar = kPairBars ? 8u + (uint32_t)(s * 4 + qw) : slot_bar;
  const int d0 = D0C ? D0C : p.d0;
  const uint32_t idesc = make_idesc_bf16(128, W);

  // all warps of the slot have stored the next A operand: the lead warp issues
  // layer l's MMAs (one elected lane) and commits them to acc_full[s]
  auto sync_and_issue = [&](int l) {
    tc_fence_before();
    asm volatile("bar.sync %0, %1;" ::"r"(slot_bar), "n"(WPS * 32) : "memory");
    if (mma_warp) {
      if (lane == 0) NB_TR(1 + s, NB_EV(0, s, l));
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = tmem + acc_col(s);
        const uint32_t a = tmem + a_col(s);
        if (l == 0) {
          mma_ts(d, a, dtab[0], idesc, 0u);
          // positional encoding (K0 = 32 .. 64) or 8-float records (K0 = 32)
          for (uint32_t kk = 1; kk < (uint32_t)p.k0 / 16u; ++kk)
            mma_ts(d, a + kk * 8u, dtab[0] + (uint64_t)(kk * 16u), idesc, 1u);
        } else {
          if (BF)  // bias first: D = ones * [hi mid lo]^T, then D += A W^T
            mma_ts(d, tmem + kOnesCol, dtab[kMaxLayers + l], idesc, 0u);
          const uint64_t bdesc = dtab[l];
#pragma unroll
          for (uint32_t kk = 0; kk < (uint32_t)W / 16u; ++kk)
            mma_ts(d, a + kk * 8u, bdesc + (uint64_t)(kk * 16u), idesc, (BF || kk > 0u) ? 1u : 0u);
        }
        mma_commit(acc_full(s));
      }
      __syncwarp();
      if (lane == 0) NB_TR(1 + s, NB_EV(1, s, l));
    }
  };

  // Records of a full tile are staged into shared memory by the TMA bulk-copy
  // engine one tile ahead (double-buffered per slot); a ragged last tile is
  // read directly.
  auto full_tile = [&](int64_t t) { return (t + 1) * kTile <= n; };
  auto stage_issue = [&](int64_t t, int b) {
    if (!issuer || t >= num_tiles || !full_tile(t)) return;
    const uint32_t qb = (uint32_t)(kTile * d0 * 4);
    const uint32_t bar = stage_bar(s, b);
    constexpr bool kY = MODE != kForward;
    mbar_arrive_expect_tx(bar, qb + (kY ? (uint32_t)kTile : 0u));
    bulk_g2s(smem_u32(q_stage(s, b)), p.a.q + t * kTile * d0, qb, bar);
    if (kY) bulk_g2s(smem_u32(y_stage(s, b)), p.a.y + t * kTile, kTile, bar);
  };
  uint32_t sph[2] = {0u, 0u};
  int ycur = 0;
  // encode the slot's i-th tile t into the slot's TMEM A region, then issue layer 0
  auto put_input = [&](int64_t t, int i) {
    if (lead) {
      float x[8];
      const int b = i & 1;
      if (full_tile(t)) {
        mbar_wait(stage_bar(s, b), sph[b]);
        sph[b] ^= 1u;
        const float* qs = q_stage(s, b) + rit * d0;
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = j < d0 ? qs[j] : 0.f;
        ycur = MODE != kForward ? (int)y_stage(s, b)[rit] : 0;
      } else {
        const int64_t r = t * kTile + rit;
        const bool v = r < n;
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = (v && j < d0) ? __ldg(p.a.q + r * d0 + j) : 0.f;
        ycur = (MODE != kForward && v) ? (int)__ldg(p.a.y + r) : 0;
      }
      if (EXT && D0C > 0) {  // positional encoding (D0C = record floats)
        uint32_t c[32];
        encode_cols_pe<D0C>(x, p.pe, c);
#pragma unroll
        for (int g = 0; g < 4; ++g)
          tmem_st8(trow + a_col(s) + (uint32_t)(8 * g), *reinterpret_cast<const uint32_t(*)[8]>(c + 8 * g));
        if (MODE == kTrain) {  // layer-1 input image (F = 64) for the dW GEMM
          uint8_t* base = p.a.tr.x_img + t * img_tile_bytes(64);
#pragma unroll
          for (int fg = 0; fg < 8; ++fg)
            *reinterpret_cast<uint4*>(base + (fg * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
        }
      } else {
        uint32_t c[8];
        encode_cols<D0C, BF>(x, d0, c);
        tmem_st8(trow + a_col(s), c);
        if (!D0C && p.k0 > kEncK) {  // 8-float records (4D rays / planes / boxes, R48): K = 32,
          uint32_t c2[8];            // the bias ones at k = 2 d0 .. 2 d0 + 2 land in the second block
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            uint32_t v = 0;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int k = kEncK + 2 * cc + h2;
              if (BF && k >= 2 * d0 && k < 2 * d0 + 3) v |= 0x3F80u << (16 * h2);
            }
            c2[cc] = v;
          }
          tmem_st8(trow + a_col(s) + 8u, c2);
        }
        if (MODE == kTrain) {  // layer-1 input image for the dW GEMM (ReLU, no PE)
          uint8_t* base = p.a.tr.x_img + t * img_tile_bytes(16);
#pragma unroll
          for (int fg = 0; fg < 2; ++fg)
            *reinterpret_cast<uint4*>(base + (fg * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                make_uint4(c[4 * fg], c[4 * fg + 1], c[4 * fg + 2], c[4 * fg + 3]);
        }
      }
      tmem_wait_st();
    }
    if (mma_warp && lane == 0) NB_TR(1 + s, NB_EV(5, s, 0));
    sync_and_issue(0);
  };

  int64_t tile = blockIdx.x + (int64_t)s * G;
  // the slot's first two record tiles are requested before waiting for the
  // weights, so the two HBM latencies overlap instead of adding up
  stage_issue(tile, 0);
  stage_issue(tile + NSLOT * G, 1);
  mbar_wait(smem_u32(bars), 0);
  bout = *reinterpret_cast<const float*>(smem + p.pl.off_bout);
  int i_tile = 0;
  if (tile < num_tiles) put_input(tile, 0);
  uint32_t par = 0;
  while (tile < num_tiles) {
    const int64_t next = tile + NSLOT * G;
    int ythis = 0;
    float z0 = lead ? bout : 0.f, z1 = 0.f;
    float e0a = (lead && NH > 0) ? cst[0] : 0.f, e0b = 0.f;
    float e1a = (lead && NH > 1) ? cst[1] : 0.f, e1b = 0.f;
#pragma unroll
    for (int l = 0; l < (LC ? LC : kMaxLayers); ++l) {
      if (!LC && l >= L) break;
      mbar_wait(acc_full(s), ph);
      if (mma_warp && lane == 0) NB_TR(1 + s, NB_EV(2, s, l));
      ph ^= 1u;
      tc_fence_after();
      // layer 0 of this tile has consumed its staged input: refill that buffer
      if (l == 0) stage_issue(next + NSLOT * G, i_tile & 1);
      const bool last = (l == L - 1);
      const float* bias = bias_all + l * W + col0;
      uint32_t v[kAllLoads ? CPT : 32];
      if (kAllLoads) {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          tmem_ld32(trow + acc_col(s) + (uint32_t)(col0 + 32 * c),
                    *reinterpret_cast<uint32_t(*)[32]>(v + (kAllLoads ? 32 * c : 0)));
        tmem_wait_ld();
      }
      if (mma_warp && lane == 0) NB_TR(1 + s, NB_EV(3, s, l));
      if (kAllLoads && last) {
        // the accumulator is in registers and the last MMA has completed: stage
        // the slot's next tile now so its layer-0 MMA overlaps this epilogue
        ythis = ycur;
        ++i_tile;
        if (next < num_tiles) put_input(next, i_tile);
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (!kAllLoads) {
          tmem_ld32(trow + acc_col(s) + (uint32_t)(col0 + 32 * c),
                    *reinterpret_cast<uint32_t(*)[32]>(v));
          tmem_wait_ld();
        }
        float* t = reinterpret_cast<float*>(v + (kAllLoads ? 32 * c : 0));
        if (!BF) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias + 32 * c + i);
            add2(t[i], t[i + 1], t[i], t[i + 1], b4.x, b4.y);
            add2(t[i + 2], t[i + 3], t[i + 2], t[i + 3], b4.z, b4.w);
          }
        }
        if (!last || MODE == kTrain) {
          uint32_t pk[16];
          if (EXT && p.act == NB_SINE) {
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack_bf16x2(sin_act(t[2 * j]), sin_act(t[2 * j + 1]));
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) pk[j] = pack_relu_bf16x2(t[2 * j], t[2 * j + 1]);
          }
          if (!last) tmem_st16(trow + a_col(s) + (uint32_t)((col0 + 32 * c) / 2), pk);
          if (MODE == kTrain) {  // h_{l+1} image (activations kept for back-propagation)
            uint8_t* base = p.a.tr.h_img[l] + tile * img_tile_bytes(W);
            const int fg0 = (col0 + 32 * c) / 8;
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<uint4*>(base + ((fg0 + i) * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                  make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            if (!(EXT && p.act == NB_SINE) && p.a.tr.c_img[l]) {  // [h > 0] bits for the backward
              uint32_t mw = 0;
#pragma unroll
              for (int j = 0; j < 16; ++j)
                mw |= ((pk[j] & 0x7FFFu) ? 1u : 0u) << (2 * j) | ((pk[j] & 0x7FFF0000u) ? 1u : 0u) << (2 * j + 1);
              reinterpret_cast<uint32_t*>(p.a.tr.c_img[l] + tile * (W * 16))[(col0 + 32 * c) / 32 * 128 + rit] = mw;
            }
            if (EXT && p.act == NB_SINE) {  // sigma'(z) = cos z for the backward chain (R41)
              uint32_t ck[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) ck[j] = pack_bf16x2(__cosf(t[2 * j]), __cosf(t[2 * j + 1]));
              uint8_t* cb = p.a.tr.c_img[l] + tile * img_tile_bytes(W);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                *reinterpret_cast<uint4*>(cb + ((fg0 + i) * 16 + rit / 8) * 128 + (rit % 8) * 16) =
                    make_uint4(ck[4 * i], ck[4 * i + 1], ck[4 * i + 2], ck[4 * i + 3]);
            }
          }
        }
        if (l == h0 || l == h1 || last) {
          if (EXT && p.act == NB_SINE) {
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] = sin_act(t[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] = relu_nan(t[i]);
          }
          const int o = 32 * c;
          // head vectors: 16-B aligned (pack layout, col0 % 32 == 0) -> LDS.128
          auto dot = [&](float& sa, float& sb, const float* w) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(w + o + i);
              fma2(sa, sb, t[i], t[i + 1], w4.x, w4.y);
              fma2(sa, sb, t[i + 2], t[i + 3], w4.z, w4.w);
            }
          };
          if (l == h0) dot(e0a, e0b, u0);
          if (l == h1) dot(e1a, e1b, u1);
          if (last) dot(z0, z1, wout);
        }
      }
      if (!last) {
        tmem_wait_st();
        if (mma_warp && lane == 0) NB_TR(1 + s, NB_EV(4, s, l));
        sync_and_issue(l + 1);
      }
    }
    if (!kAllLoads) {
      ythis = ycur;
      ++i_tile;
      if (next < num_tiles) put_input(next, i_tile);
    }
    float z = z0 + z1;
    float e[2] = {e0a + e0b, e1a + e1b};
    if (WPS == 8) {  // combine the two column halves of each row
      float* xb = xch + ((((size_t)s * 2 + par) * 4 + qw) * 32 + lane) * 3;
      if (!lead) {
        xb[0] = z;
        xb[1] = e[0];
        xb[2] = e[1];
      }
      asm volatile("bar.sync %0, %1;" ::"r"(half_bar), "n"(kPairBars ? 64 : WPS * 32) : "memory");
      if (lead) {
        z += xb[0];
        e[0] += xb[1];
        e[1] += xb[2];
      }
      par ^= 1u;
    }
    if (lead) {
      const int64_t r = tile * kTile + rit;
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
        const int64_t r3 = r * 3;
        if (valid) {
          p.a.tr.g32[r3] = gz;
          p.a.tr.g32[r3 + 1] = ge[0];
          p.a.tr.g32[r3 + 2] = ge[1];
        }
        uint8_t* hb = p.a.tr.hd_img + tile * img_tile_bytes(8) + (rit / 8) * 128 + (rit % 8) * 16;
        *reinterpret_cast<uint4*>(hb) = make_uint4(pack_bf16x2(gz, ge[0]), pack_bf16x2(ge[1], 0.f), 0u, 0u);
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
        classify_row_smem<MODE, NHC>(cnt, key, valid, ythis, z, e, NH, p.a.tau, p.a.flags, p.a.invert);
      }
    }
    tile = next;
  }
  if (MODE == kCalibrate && lead) flush_smem<MODE>(cnt, key, NH, p.a.counts, p.a.keys);
  if (MODE == kTrain && lead && lane == 0) {
    for (int i = 0; i < 4; ++i)
      if (cnt[i]) atomicAdd(p.a.tr.stats + i, (unsigned long long)cnt[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<COLS>(tmem);
  }
  if (MODE == kScore && warp == 1) flush_cta_counts(ctr, NEPI, NHC == 0 ? -1 : NH, p.a.counts);
  if (MODE == kScore && warp == 1 && p.a.ticket) finalize_counts(p.a, NHC == 0);
}

// Trace buffer of NB_TRACE builds (defined in nb_fwd_tc.cu).
extern unsigned long long* g_trace_buffer;

template <int W, int LC, int H0C, int H1C, int MODE, int D0C, bool BF, bool EXT = false>
inline cudaError_t launch_tc_wm(const nb_model* m, const FwdArgs& a, cudaStream_t st) {
  constexpr int NSLOT = TcPlan<W>::NSLOT, WPS = TcPlan<W>::WPS;
  TcParams p;
  p.a = a;
  p.packed = m->packed;
  p.pl = m->pl;
  p.d0 = m->d0;
  p.L = m->d.hidden_layers;
  p.nh = m->d.n_heads;
  p.ha0 = m->d.head_after[0];
  p.ha1 = m->d.head_after[1];
  p.act = m->d.activation;
  p.pe = m->d.pe_depth;
  p.din = m->din;
  p.k0 = (int)m->pl.k_of[0];
  p.num_tiles = (a.n + kTile - 1) / kTile;
  p.trace = g_trace_buffer;
  if (p.num_tiles == 0) return cudaSuccess;
  // weights | barriers + tmem slot | head-partial exchange | counters | staging;
  // requesting >= 116 KB also forces one CTA per SM (TMEM is allocated whole)
  const uint32_t img = BF ? m->pl.bytes : m->pl.core_bytes;
  p.pl.bytes = img;
  size_t smem = ((img + 15) & ~15u) + 8 * (2 + 2 * NSLOT) + 16 +
                sizeof(float) * NSLOT * 2 * 4 * 32 * 3 + 4 * NSLOT * WPS * 12 + 8 * 2 * NSLOT +
                sizeof(float) * NSLOT * 2 * kTile * 8 + NSLOT * 2 * kTile + 16 * 8;
  smem = std::max<size_t>(smem, 116 * 1024);
  auto kern = k_fwd_tc<W, LC, H0C, H1C, MODE, D0C, BF, EXT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(p.num_tiles, m->num_sms);
  return launch_pdl(kern, dim3(grid), dim3(NSLOT * WPS * 32), smem, st, MODE == kTrain, p);
}

// Generic sine / PE kernels (bias folded; forward, calibrate, score).  D0 > 0:
// positional encoding of D0-float records; D0 = 0: no encoding (sine only).
template <int W, int D0>
inline cudaError_t launch_tc_ext_d(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc_wm<W, 0, 0, 0, kForward, D0, true, true>(m, a, st);
  if (mode == kCalibrate) return launch_tc_wm<W, 0, 0, 0, kCalibrate, D0, true, true>(m, a, st);
  if (mode == kScore) return launch_tc_wm<W, 0, 0, 0, kScore, D0, true, true>(m, a, st);
  if (mode == kTrain && W >= 64) return launch_tc_wm<W, 0, 0, 0, kTrain, D0, true, true>(m, a, st);
  return cudaErrorInvalidValue;
}
cudaError_t launch_tc_ext32(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st);
cudaError_t launch_tc_ext64(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st);
cudaError_t launch_tc_ext128(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st);

template <int W, int LC, int H0C, int H1C, int D0C, bool BF>
inline cudaError_t launch_tc_modes(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  if (mode == kForward) return launch_tc_wm<W, LC, H0C, H1C, kForward, D0C, BF>(m, a, st);
  if (mode == kCalibrate) return launch_tc_wm<W, LC, H0C, H1C, kCalibrate, D0C, BF>(m, a, st);
  if (mode == kTrain) return launch_tc_wm<W, LC, H0C, H1C, kTrain, D0C, BF>(m, a, st);
  return launch_tc_wm<W, LC, H0C, H1C, kScore, D0C, BF>(m, a, st);
}

// One translation unit per BASELINE.json architecture (parallel builds):
// fold selects the bias-folded (BF) or epilogue-bias instantiation.
cudaError_t launch_tc_w64l4_d3(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);
cudaError_t launch_tc_w128l4_d6(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);
cudaError_t launch_tc_w128l6h24_d4(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);
cudaError_t launch_tc_gen32(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);
cudaError_t launch_tc_gen64(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);
cudaError_t launch_tc_gen128(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st, bool fold);

}  // namespace nb
