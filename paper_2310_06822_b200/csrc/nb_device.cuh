// nb_device.cuh — device helpers shared by the libnb kernels: the fused
// classify/count/calibrate reduction (rows a5, a6 of the hot path) and small
// PTX wrappers.  Product code only (no relation to oracle/).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "nb_internal.cuh"

namespace nb {

__device__ __forceinline__ uint32_t dkey(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Per-warp reduction state of one kernel: counts (uniform across the warp,
// from ballots) and per-thread min keys for calibration.
struct WarpAcc {
  uint32_t c[kNumCounters];
  uint32_t key[3];
  __device__ void init() {
#pragma unroll
    for (int i = 0; i < kNumCounters; ++i) c[i] = 0;
    key[0] = key[1] = key[2] = 0xFFFFFFFFu;
  }
};

// One row per lane: classify (a5) or fold into the calibration minimum (a6).
// yhat = [e_1 >= tau_1] and [e_2 >= tau_2] and [z >= tau]  (R21/R22).
template <int MODE>
__device__ __forceinline__ void classify_row(WarpAcc& acc, bool valid, int y, float z,
                                             const float* e, int nh, const float* tau,
                                             unsigned int* flags, int invert = 0) {
  if (MODE == kCalibrate) {
    if (valid && (invert ? y == 0 : y == 1)) {
      acc.key[0] = min(acc.key[0], dkey(invert ? -z : z));
      if (nh > 0) acc.key[1] = min(acc.key[1], dkey(e[0]));
      if (nh > 1) acc.key[2] = min(acc.key[2], dkey(e[1]));
    }
  }
  if (MODE == kScore) {
    int bin = 3;
    bool pred = true;
    if (nh > 0 && !(e[0] >= tau[1])) { pred = false; bin = 0; }
    else if (nh > 1 && !(e[1] >= tau[2])) { pred = false; bin = 1; }
    else { pred = z >= tau[0]; bin = pred ? 3 : 2; }
    bool yy = y != 0;
    bool nonfin = !isfinite(z) || (nh > 0 && !isfinite(e[0])) || (nh > 1 && !isfinite(e[1]));
    const unsigned full = 0xFFFFFFFFu;
    acc.c[0] += __popc(__ballot_sync(full, valid && pred && yy));
    acc.c[1] += __popc(__ballot_sync(full, valid && pred && !yy));
    acc.c[2] += __popc(__ballot_sync(full, valid && !pred && yy));
    acc.c[3] += __popc(__ballot_sync(full, valid && !pred && !yy));
    if (nh > 0) {
      acc.c[4] += __popc(__ballot_sync(full, valid && bin == 0));
      acc.c[5] += __popc(__ballot_sync(full, valid && bin == 1));
      acc.c[6] += __popc(__ballot_sync(full, valid && bin == 2));
      acc.c[7] += __popc(__ballot_sync(full, valid && bin == 3));
    }
    acc.c[8] += __popc(__ballot_sync(full, valid && nonfin));
  }
  if (valid && y > 1) atomicOr(flags, kFlagLabel);
}

// Flush a warp's accumulators to global memory (one atomic per counter).
template <int MODE>
__device__ __forceinline__ void flush_warp(WarpAcc& acc, int nh, unsigned long long* counts,
                                           unsigned int* keys) {
  const int lane = threadIdx.x & 31;
  if (MODE == kCalibrate) {
    for (int k = 0; k <= nh; ++k) {
      uint32_t m = __reduce_min_sync(0xFFFFFFFFu, acc.key[k]);
      if (lane == 0 && m != 0xFFFFFFFFu) atomicMin(keys + k, m);
    }
  }
  if (MODE == kScore && lane == 0) {
    if (nh == 0) acc.c[7] = acc.c[0] + acc.c[1], acc.c[6] = acc.c[2] + acc.c[3];
#pragma unroll
    for (int i = 0; i < kNumCounters; ++i)
      if (acc.c[i]) atomicAdd(counts + i * kCtrStride, (unsigned long long)acc.c[i]);
  }
}

// CTA-level count flush (score mode): one warp sums the per-warp shared-memory
// counters ctr[w * 12 + i] of all nwarps warps and adds each total with ONE
// atomic per CTA (exit bin 3 = tp + fp, and bin 2 = fn + tn without heads).
// nh < 0: the counters are raw (tp, pred, pos, ..., nonfinite); passed as is.
__device__ __forceinline__ void flush_cta_counts(const uint32_t* ctr, int nwarps, int nh,
                                                 unsigned long long* counts) {
  const int lane = threadIdx.x & 31;
  uint32_t v = 0;
  if (lane < kNumCounters)
    for (int w = 0; w < nwarps; ++w) v += ctr[w * 12 + lane];
  const uint32_t c0 = __shfl_sync(0xFFFFFFFFu, v, 0), c1 = __shfl_sync(0xFFFFFFFFu, v, 1);
  const uint32_t c2 = __shfl_sync(0xFFFFFFFFu, v, 2), c3 = __shfl_sync(0xFFFFFFFFu, v, 3);
  if (lane == 7 && nh >= 0) v = c0 + c1;
  if (lane == 6 && nh == 0) v = c2 + c3;
  if (lane < kNumCounters && v) atomicAdd(counts + lane * kCtrStride, (unsigned long long)v);
}

// Last-CTA finalisation of the fused score counters (row a5).  Called by all
// 32 lanes of one warp per CTA after a __syncthreads that follows all of the
// CTA's counter atomics.  Lane 0's fence is cumulative over the writes the
// barrier made visible to it, so the ticket orders the whole CTA's counts.
// The CTA drawing the last ticket moves the totals to a.fin_out (one lane per
// counter) and re-arms counters and ticket for the next launch (stream order
// makes that safe).
// raw: the counters hold (tp, pred, pos, -, -, -, -, -, nonfinite) of a model
// without exit heads; the totals are derived here with n = a.n valid rows.
__device__ __forceinline__ void finalize_counts(const FwdArgs& a, bool raw = false) {
  const int lane = threadIdx.x & 31;
  unsigned int t = 0;
  if (lane == 0) {
    __threadfence();
    t = atomicAdd(a.ticket, 1u);
  }
  t = __shfl_sync(0xFFFFFFFFu, t, 0);
  if (t == gridDim.x * gridDim.y * gridDim.z - 1) {
    __threadfence();
    unsigned long long v = 0;
    if (lane < kNumCounters) v = __ldcg(a.counts + lane * kCtrStride);
    if (raw) {
      const unsigned long long tp = __shfl_sync(0xFFFFFFFFu, v, 0), pred = __shfl_sync(0xFFFFFFFFu, v, 1);
      const unsigned long long pos = __shfl_sync(0xFFFFFFFFu, v, 2), n = (unsigned long long)a.n;
      const unsigned long long tt[kNumCounters] = {tp, pred - tp, pos - tp, n - pred - pos + tp,
                                                   0ull, 0ull, n - pred, pred, 0ull};
#pragma unroll
      for (int i = 0; i < kNumCounters - 1; ++i)
        if (lane == i) v = tt[i];
    }
    if (lane < kNumCounters) {
      if (a.fin_add) atomicAdd(a.fin_out + lane, v);
      else a.fin_out[lane] = v;
      // re-arm the idle set for the next launch (this set is re-armed by it);
      // host-mapped fin_out is visible at kernel completion
      a.counts_next[lane * kCtrStride] = 0ull;
    }
    if (lane == 0) *a.ticket_next = 0u;
  }
}

// ---------------------------------------------------------------------------
// PTX wrappers: mbarrier, bulk copy, tcgen05 (sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
#if defined(NB_MBAR_NOHINT) || defined(NB_CHECKS)
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
#else
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, 10000000;\n\t"
#endif
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Programmatic dependent launch (PDL): wait until the grids this one depends
// on have completed and their writes are visible (returns at once for a
// launch without the programmatic-serialization attribute), and allow the
// dependent grid to be scheduled (it still waits on its own griddep_wait).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Non-blocking probe of an mbarrier phase.
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// NB_CHECKS builds (libnb_checked.so, tests/test_gpu_checked.py): the
// stand-in for compute-sanitizer's synccheck/memcheck on the hand-rolled
// pipelines.  A wait that has not completed after 2^24 polls (seconds; the
// checked build polls without a suspend-time hint) is
// a lost arrive or a phase error: report the barrier and trap instead of
// hanging; NB_CHECK() traps on a violated invariant (bounds, alignment).
#ifdef NB_CHECKS
#define NB_CHECK(cond, ...)                                                          \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("NB_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x, #cond);                              \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define NB_CHECK(cond, ...) \
  do {                      \
  } while (0)
#endif

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#ifdef NB_CHECKS
  uint64_t polls = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++polls == (1ull << 24)) {
      printf("NB_CHECK mbarrier timeout: bar 0x%x parity %u block %d thread %d\n", bar, parity,
             (int)blockIdx.x, (int)threadIdx.x);
      __trap();
    }
  }
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier (TMA engine).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  NB_CHECK(((uintptr_t)src & 15u) == 0 && (dst & 15u) == 0 && (bytes & 15u) == 0 && bytes > 0);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// One lane of the (converged) warp returns true (elect.sync).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]^T, kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc]^T
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 consecutive 32-bit columns <- 16 registers per thread
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}

// ---- CTA pairs (cta_group::2): cluster helpers, pair MMA and commit --------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// Remote arrive with the default semantics (release at CTA scope): the cheap
// signal the pair's MMA issuer waits on (tcgen05 ordering comes from the
// wait::st + fence::before_thread_sync pair before it).
__device__ __forceinline__ void mbar_arrive_remote_cta(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
#if defined(NB_MBAR_NOHINT) || defined(NB_CHECKS)
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
#else
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, 10000000;\n\t"
#endif
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mma_ts2(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// pair MMA with A from shared memory (each CTA's own rows at the same address)
__device__ __forceinline__ void mma_ss2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}


// ReLU that keeps NaN (max.NaN): a non-finite record's NaN survives the last
// hidden layer into the logit (R26) at the cost of a plain FMNMX.
__device__ __forceinline__ float relu_nan(float x) {
  float r;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
  return r;
}

// relu + round-to-nearest-even pack of two fp32 into bf16x2 (lo = a, hi = b)
__device__ __forceinline__ uint32_t pack_relu_bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// UMMA shared-memory descriptor, K-major (or MN-major), no swizzle.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// Instruction descriptor kind::f16: bf16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, int a_mn_major = 0,
                                                       int b_mn_major = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) |
         ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace nb
