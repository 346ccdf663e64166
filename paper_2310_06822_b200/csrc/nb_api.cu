// nb_api.cu — the C ABI of include/nb.h: validation, model state, dispatch of
// the hot-path kernels, sticky-flag reporting and the collectives.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

static nb_status cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return NB_E_CUDA;
}

#define NB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e__ = (call);                           \
    if (e__ != cudaSuccess) return cuda_fail(e__, #call); \
  } while (0)

static bool desc_valid(const nb_desc* d, int* d0_out) {
  if (!d) return false;
  if (d->kind < NB_POINT || d->kind > NB_BOX) return false;
  if (d->space_dim < 2 || d->space_dim > 4) return false;
  if (d->width < 1 || d->width > 256) return false;
  if (d->hidden_layers < 1 || d->hidden_layers > kMaxLayers) return false;
  if (d->n_heads < 0 || d->n_heads > 2) return false;
  for (int k = 0; k < d->n_heads; ++k)
    if (d->head_after[k] < 1 || d->head_after[k] > d->hidden_layers) return false;
  if (d->n_heads == 2 && d->head_after[0] >= d->head_after[1]) return false;
  if (d->precision != NB_FP32 && d->precision != NB_BF16) return false;
  if (d->activation != NB_RELU && d->activation != NB_SINE) return false;
  if (d->pe_depth < 0 || d->pe_depth > 16 || (d->pe_depth & 1)) return false;
  int d0 = d->kind == NB_POINT ? d->space_dim : 2 * d->space_dim;
  if (d0 > 8) return false;
  if (d0_out) *d0_out = d0;
  return true;
}

// Layer-1 input features: the record, or its positional encoding (R42).
static int input_features(const nb_desc& d) {
  const int r = d.kind == NB_POINT ? d.space_dim : 2 * d.space_dim;
  return r * (1 + d.pe_depth);
}

static void param_offsets(const nb_desc& d, int din, ParamOffsets* o) {
  int64_t p = 0, in = din;
  for (int l = 0; l < d.hidden_layers; ++l) {
    o->W[l] = p; p += in * d.width;
    o->b[l] = p; p += d.width;
    in = d.width;
  }
  o->wout = p; p += d.width;
  o->bout = p; p += 1;
  for (int k = 0; k < 2; ++k) {
    if (k < d.n_heads) {
      o->u[k] = p; p += d.width;
      o->c[k] = p; p += 1;
    } else {
      o->u[k] = o->c[k] = 0;
    }
  }
}

static uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Widths above 128 run on CTA pairs (tcgen05 cta_group::2): each CTA's image
// holds half of every layer's output rows (pl.pairs = 2 images back to back).
static void pack_layout(const nb_desc& d, PackLayout* pl) {
  uint32_t off = 0;
  const uint32_t W = (uint32_t)d.width;
  pl->pairs = (d.precision == NB_BF16 && W > 128) ? 2u : 1u;
  const uint32_t rows = W / pl->pairs;
  const int din = input_features(d);
  const bool pe_split = d.pe_depth > 0 && d.precision == NB_BF16;
  const uint32_t K0 = pe_split ? 64u : (uint32_t)enc_k(din);
  pl->pe_lo = pe_split ? 32u : 0u;
  for (int l = 0; l < d.hidden_layers; ++l) {
    const uint32_t K = l == 0 ? K0 : W;
    pl->off_w[l] = off;
    pl->k_of[l] = K;
    off = align_up(off + rows * K * 2u, 128u);
  }
  pl->off_bias = off; off = align_up(off + 4u * W * d.hidden_layers, 16u);
  pl->off_wout = off; off = align_up(off + 4u * W, 16u);
  pl->off_bout = off; off += 16u;
  for (int k = 0; k < 2; ++k) {
    pl->off_u[k] = off;
    if (k < d.n_heads) off = align_up(off + 4u * W, 16u);
  }
  pl->off_c = off; off += 16u;
  off = align_up(off, 128u);
  pl->core_bytes = off;
  const bool shared = pl->pairs == 2 && d.precision == NB_BF16 && 3 * (d.hidden_layers - 1) <= kEncK;
  const bool fold = (pl->pairs == 1 && d.precision == NB_BF16) || shared;
  pl->bias_l0 = (fold && (pe_split ? din + 3 <= 32 : 2 * din + 3 <= (int)K0)) ? 1u : 0u;
  pl->bb_shared = shared ? 1u : 0u;
  for (int l = 0; l < kMaxLayers; ++l) pl->off_bb[l] = 0;
  if (shared) {
    pl->off_bb[0] = off;
    off = align_up(off + rows * (uint32_t)kEncK * 2u, 128u);
  } else {
    for (int l = 1; fold && l < d.hidden_layers; ++l) {
      pl->off_bb[l] = off;
      off = align_up(off + W * (uint32_t)kEncK * 2u, 128u);
    }
  }
  pl->bytes = align_up(off, 16u);
}

static void bwd_layout(const nb_desc& d, BwdLayout* bl) {
  uint32_t off = 0;
  const uint32_t W = (uint32_t)d.width;
  for (int l = 0; l < kMaxLayers; ++l) {
    bl->off_wt[l] = 0;
    if (l >= 1 && l < d.hidden_layers) {
      bl->off_wt[l] = off;
      off = align_up(off + (W / 2) * W * 2u, 128u);
    }
  }
  bl->off_wout = off; off = align_up(off + 4u * W, 16u);
  for (int k = 0; k < 2; ++k) {
    bl->off_u[k] = off;
    off = align_up(off + 4u * W, 16u);
  }
  bl->bytes = align_up(off, 128u);
}

// Report sticky in-kernel flags (and clear them).  Host mirror is pinned.
static nb_status take_flags(nb_model* m, cudaStream_t s, nb_status ok) {
  unsigned int f = 0;
  NB_CUDA(cudaMemcpyAsync(&f, m->d_flags, sizeof(f), cudaMemcpyDeviceToHost, s));
  NB_CUDA(cudaStreamSynchronize(s));
  if (f) NB_CUDA(cudaMemsetAsync(m->d_flags, 0, sizeof(unsigned int), s));
  if (f & kFlagLabel) {
    set_error("label outside {0,1}");
    return NB_E_LABEL;
  }
  if (f & kFlagNonFinite) {
    set_error("non-finite logit");
    return NB_E_NONFINITE;
  }
  return ok;
}

// Kernel-time instrumentation (nb_model_set_timing): CUDA events bracket the
// hot-path kernel launches on the caller's stream; the elapsed time of all
// bracketed launches since the last nb_model_kernel_ms() call is accumulated.
static bool timing_on(const nb_model* m) { return m->timing && m->ev_used < nb_model::kEvPool; }
static void timing_begin(const nb_model* m, cudaStream_t s) {
  if (timing_on(m)) cudaEventRecord(m->ev_pool[2 * m->ev_used], s);
}
static void timing_end(const nb_model* m, cudaStream_t s) {
  if (!timing_on(m)) return;
  nb_model* mm = const_cast<nb_model*>(m);
  cudaEventRecord(mm->ev_pool[2 * mm->ev_used + 1], s);
  mm->ev_used += 1;
  mm->kernel_launches += 1;
}

// NB_CHECKS self-test (tests/test_gpu_checked.py): a kernel waits on an
// mbarrier phase that never completes; the checked build must trap with a
// diagnostic instead of hanging.  Release builds return NB_E_UNSUPPORTED.
__global__ void k_selftest_lost_arrive() {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
    mbar_wait(smem_u32(&bar), 0u);  // nobody arrives
  }
}
extern "C" int nb_debug_selftest_lost_arrive(void) {
#ifdef NB_CHECKS
  k_selftest_lost_arrive<<<1, 32>>>();
  return (int)cudaDeviceSynchronize();
#else
  return NB_E_UNSUPPORTED;
#endif
}

// Measurement / test switch: score models with exit heads densely (every head
// on every row, nb_fwd_tc.cuh) instead of with early-exit compaction.
static bool g_dense_exits = false;
extern "C" void nb_debug_set_dense_exits(int v) { g_dense_exits = v != 0; }

static cudaError_t launch_forward_any(const nb_model* m, int mode, const FwdArgs& a,
                                      cudaStream_t s) {
  timing_begin(m, s);
  if (mode == kScore && !g_dense_exits && exit_compaction_supported(m)) {
    int k = 0;
    cudaError_t e = launch_score_exit(const_cast<nb_model*>(m), a, s, &k);
    if (timing_on(m)) const_cast<nb_model*>(m)->kernel_launches += k - 1;  // + timing_end's one
    timing_end(m, s);
    return e;
  }
  cudaError_t e = m->d.precision != NB_BF16 ? launch_fwd_simt(m, mode, a, s)
                  : m->pl.pairs == 2        ? launch_fwd_tc2(m, mode, a, s)
                                            : launch_fwd_tc(m, mode, a, s);
  timing_end(m, s);
  return e;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// The fused kernels stage full 128-row tiles of q and y into shared memory
// with cp.async.bulk, which needs 16-byte aligned global addresses (tile
// offsets are multiples of 16 B, so the base pointers decide): misaligned
// views are rejected before any launch (nb.h "Alignment").
static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static nb_status misaligned(const char* where) {
  set_error("%s: q and y must be 16-byte aligned device pointers", where);
  return NB_E_ARG;
}

}  // namespace nb

using namespace nb;

extern "C" {

int64_t nb_record_floats(int32_t kind, int32_t space_dim) {
  if (kind < NB_POINT || kind > NB_BOX || space_dim < 2 || space_dim > 4) return -1;
  return kind == NB_POINT ? space_dim : 2 * space_dim;
}

int64_t nb_num_params(const nb_desc* d) {
  if (!desc_valid(d, nullptr)) return -1;
  int64_t n = 0, in = input_features(*d);
  for (int l = 0; l < d->hidden_layers; ++l) {
    n += (in + 1) * (int64_t)d->width;
    in = d->width;
  }
  return n + (int64_t)(d->width + 1) * (1 + d->n_heads);
}

const char* nb_status_string(nb_status s) {
  switch (s) {
    case NB_OK: return "ok";
    case NB_E_ARG: return "invalid argument";
    case NB_E_SHAPE: return "shape mismatch";
    case NB_E_NONFINITE: return "non-finite value";
    case NB_E_LABEL: return "label outside {0,1}";
    case NB_E_NO_POSITIVES: return "no positive labels (tau = +inf)";
    case NB_E_CUDA: return "CUDA error";
    case NB_E_NCCL: return "NCCL error";
    case NB_E_UNSUPPORTED: return "unsupported configuration";
    case NB_E_OOM: return "out of memory";
  }
  return "unknown status";
}

const char* nb_last_error(void) { return g_err.c_str(); }

nb_status nb_device_check(int32_t device, int32_t* cc_out) {
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (cc_out) *cc_out = major * 10 + minor;
  if (major != 10 || minor != 0) {
    set_error("libnb is built for sm_100a only (device cc %d.%d)", major, minor);
    return NB_E_UNSUPPORTED;
  }
  return NB_OK;
}

nb_status nb_model_create(const nb_desc* desc, int32_t device, nb_model** out) {
  int d0;
  if (!out || !desc_valid(desc, &d0)) {
    set_error("invalid nb_desc");
    return NB_E_ARG;
  }
  const bool ok_arch = desc->precision == NB_BF16 ? (tc_supported(*desc) || tc2_supported(*desc))
                                                  : simt_supported(*desc);
  if (!ok_arch) {
    set_error("no kernel for precision %d width %d", desc->precision, desc->width);
    return NB_E_UNSUPPORTED;
  }
  nb_status st = nb_device_check(device, nullptr);
  if (st != NB_OK) return st;
  DeviceGuard g(device);
  nb_model* m = new nb_model();
  m->d = *desc;
  for (int k = desc->n_heads; k < 2; ++k) m->d.head_after[k] = 0;
  m->device = device;
  m->d0 = d0;
  m->din = input_features(*desc);
  m->P = nb_num_params(desc);
  param_offsets(m->d, m->din, &m->po);
  pack_layout(m->d, &m->pl);
  // CTA-pair kernels keep one pair image (+ ~16 KB of staging, barriers and
  // ones operands) in shared memory: deeper / PE pair nets do not fit
  if (m->pl.pairs == 2 && m->pl.bytes + 16u * 1024u > 227u * 1024u) {
    set_error("w = 256 image of %u bytes exceeds the shared memory of a CTA pair", m->pl.bytes);
    delete m;
    return NB_E_UNSUPPORTED;
  }
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes);
  };
  A((void**)&m->theta, sizeof(float) * m->P);
  A((void**)&m->adam_m, sizeof(float) * m->P);
  A((void**)&m->adam_v, sizeof(float) * m->P);
  A((void**)&m->grad, sizeof(float) * m->P);
  A((void**)&m->packed, (size_t)m->pl.bytes * m->pl.pairs);
  if (m->pl.pairs == 2) {
    bwd_layout(m->d, &m->bl);
    A((void**)&m->packed_bwd, (size_t)m->bl.bytes * 2);
  }
  A((void**)&m->d_tau, sizeof(float) * 4);
  // kernel counters i * kCtrStride (kept zero between launches by the
  // finalising CTA), finalised totals at kFinOff, a zero block at kZeroOff
  A((void**)&m->d_counts, sizeof(unsigned long long) * 256);
  A((void**)&m->d_keys, sizeof(unsigned int) * 4);
  A((void**)&m->d_flags, sizeof(unsigned int) * 4);
  // two 64-B step-statistics buffers: [0, 16) loss (double), [16, 48) batch stats (4 x u64)
  A((void**)&m->d_loss_base, 128);
  if (e == cudaSuccess) {
    m->d_loss = m->d_loss_base;
    m->d_stats = reinterpret_cast<unsigned long long*>(m->d_loss + 2);
  }
  if (e == cudaSuccess) e = cudaMallocHost((void**)&m->h_pinned, 256);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&m->ev_copy[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_done[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    nb_model_destroy(m);
    set_error("nb_model_create: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? NB_E_OOM : NB_E_CUDA;
  }
  if (m->d.precision == NB_BF16) {
    e = launch_pack_bf16(m, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      nb_model_destroy(m);
      return cuda_fail(e, "pack");
    }
  }
  *out = m;
  return NB_OK;
}

void nb_model_destroy(nb_model* m) {
  if (!m) return;
  DeviceGuard g(m->device);
  comm_destroy(m);
  cudaFree(m->theta);
  cudaFree(m->adam_m);
  cudaFree(m->adam_v);
  cudaFree(m->grad);
  cudaFree(m->packed);
  cudaFree(m->packed_bwd);
  cudaFree(m->d_tau);
  cudaFree(m->d_counts);
  cudaFree(m->d_keys);
  cudaFree(m->d_flags);
  cudaFree(m->d_loss_base);
  cudaFree(m->train_scratch);
  cudaFree(m->exit_scratch);
  cudaFree(m->hier_scratch);
  for (int i = 0; i < 2; ++i) {
    cudaFree(m->stage_q[i]);
    cudaFree(m->stage_y[i]);
    if (m->ev_copy[i]) cudaEventDestroy(m->ev_copy[i]);
    if (m->ev_done[i]) cudaEventDestroy(m->ev_done[i]);
  }
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  if (m->graph_stream) cudaStreamSynchronize(m->graph_stream);
  for (int i = 0; i < 2; ++i) {
    if (m->graph_exec2[i]) cudaGraphExecDestroy((cudaGraphExec_t)m->graph_exec2[i]);
    if (m->ev_graph[i]) cudaEventDestroy(m->ev_graph[i]);
    if (m->ev_graph_done[i]) cudaEventDestroy(m->ev_graph_done[i]);
  }
  if (m->graph_stream) cudaStreamDestroy(m->graph_stream);
  if (m->ev_pool) {
    for (int i = 0; i < 2 * nb_model::kEvPool; ++i) cudaEventDestroy(m->ev_pool[i]);
    delete[] m->ev_pool;
  }
  if (m->h_pinned) cudaFreeHost(m->h_pinned);
  delete m;
}

nb_status nb_model_set_params(nb_model* m, const float* host, int64_t n) {
  if (!m || !host) return set_error("null argument"), NB_E_ARG;
  if (n != m->P) return set_error("expected %lld params, got %lld", (long long)m->P, (long long)n), NB_E_SHAPE;
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(host[i])) return set_error("non-finite parameter %lld", (long long)i), NB_E_NONFINITE;
  DeviceGuard g(m->device);
  NB_CUDA(cudaMemcpy(m->theta, host, sizeof(float) * n, cudaMemcpyHostToDevice));
  NB_CUDA(cudaMemset(m->adam_m, 0, sizeof(float) * n));
  NB_CUDA(cudaMemset(m->adam_v, 0, sizeof(float) * n));
  m->step = 0;
  if (m->d.precision == NB_BF16) {
    NB_CUDA(launch_pack_bf16(m, 0));
    NB_CUDA(cudaDeviceSynchronize());
  }
  return NB_OK;
}

nb_status nb_model_get_params(const nb_model* m, float* host, int64_t n) {
  if (!m || !host) return set_error("null argument"), NB_E_ARG;
  if (n != m->P) return set_error("expected %lld params", (long long)m->P), NB_E_SHAPE;
  DeviceGuard g(m->device);
  NB_CUDA(cudaDeviceSynchronize());
  NB_CUDA(cudaMemcpy(host, m->theta, sizeof(float) * n, cudaMemcpyDeviceToHost));
  return NB_OK;
}

nb_status nb_model_get_grad(const nb_model* m, float* host, int64_t n) {
  if (!m || !host) return set_error("null argument"), NB_E_ARG;
  if (n != m->P) return set_error("expected %lld params", (long long)m->P), NB_E_SHAPE;
  DeviceGuard g(m->device);
  NB_CUDA(cudaDeviceSynchronize());
  NB_CUDA(cudaMemcpy(host, m->grad, sizeof(float) * n, cudaMemcpyDeviceToHost));
  return NB_OK;
}

nb_status nb_model_set_timing(nb_model* m, int32_t enable) {
  if (!m) return set_error("null model"), NB_E_ARG;
  DeviceGuard g(m->device);
  if (enable && !m->ev_pool) {
    m->ev_pool = new cudaEvent_t[2 * nb_model::kEvPool];
    for (int i = 0; i < 2 * nb_model::kEvPool; ++i) NB_CUDA(cudaEventCreate(&m->ev_pool[i]));
  }
  m->timing = enable ? 1 : 0;
  m->ev_used = 0;
  m->kernel_launches = 0;
  return NB_OK;
}

nb_status nb_model_kernel_time(nb_model* m, double* ms, int64_t* launches) {
  if (!m || !ms || !launches) return set_error("null argument"), NB_E_ARG;
  DeviceGuard g(m->device);
  double tot = 0.0;
  for (int i = 0; i < m->ev_used; ++i) {
    NB_CUDA(cudaEventSynchronize(m->ev_pool[2 * i + 1]));
    float t = 0.f;
    NB_CUDA(cudaEventElapsedTime(&t, m->ev_pool[2 * i], m->ev_pool[2 * i + 1]));
    tot += t;
  }
  *ms = tot;
  *launches = m->kernel_launches;  // kernels (an early-exit score is 3 per chunk)
  m->ev_used = 0;
  m->kernel_launches = 0;
  return NB_OK;
}

nb_status nb_model_get_adam(const nb_model* m, float* mh, float* vh, int64_t* step) {
  if (!m || !mh || !vh || !step) return set_error("null argument"), NB_E_ARG;
  DeviceGuard g(m->device);
  NB_CUDA(cudaDeviceSynchronize());
  NB_CUDA(cudaMemcpy(mh, m->adam_m, sizeof(float) * m->P, cudaMemcpyDeviceToHost));
  NB_CUDA(cudaMemcpy(vh, m->adam_v, sizeof(float) * m->P, cudaMemcpyDeviceToHost));
  *step = m->step;
  return NB_OK;
}

nb_status nb_model_set_adam(nb_model* m, const float* mh, const float* vh, int64_t step) {
  if (!m || !mh || !vh || step < 0) return set_error("bad argument"), NB_E_ARG;
  DeviceGuard g(m->device);
  NB_CUDA(cudaMemcpy(m->adam_m, mh, sizeof(float) * m->P, cudaMemcpyHostToDevice));
  NB_CUDA(cudaMemcpy(m->adam_v, vh, sizeof(float) * m->P, cudaMemcpyHostToDevice));
  m->step = step;
  return NB_OK;
}

nb_status nb_model_set_thresholds(nb_model* m, const float* tau, int32_t n) {
  if (!m || !tau) return set_error("null argument"), NB_E_ARG;
  if (n != 1 + m->d.n_heads) return set_error("expected %d thresholds", 1 + m->d.n_heads), NB_E_SHAPE;
  for (int k = 0; k < n; ++k) m->tau[k] = tau[k];
  DeviceGuard g(m->device);
  NB_CUDA(cudaMemcpy(m->d_tau, m->tau, sizeof(float) * 3, cudaMemcpyHostToDevice));
  return NB_OK;
}

nb_status nb_model_get_thresholds(const nb_model* m, float* tau, int32_t n) {
  if (!m || !tau) return set_error("null argument"), NB_E_ARG;
  if (n != 1 + m->d.n_heads) return set_error("expected %d thresholds", 1 + m->d.n_heads), NB_E_SHAPE;
  for (int k = 0; k < n; ++k) tau[k] = m->tau[k];
  return NB_OK;
}

nb_status nb_encode(const nb_model* m, const float* q, int64_t n, void* x_out, void* stream) {
  if (!m || n < 0 || (n > 0 && (!q || !x_out))) return set_error("bad argument"), NB_E_ARG;
  if (m->d.pe_depth > 0 && m->d.precision != NB_BF16)
    return set_error("nb_encode: fp32 positional-encoding nets encode inside the kernels only"),
           NB_E_UNSUPPORTED;
  DeviceGuard g(m->device);
  if (m->d.pe_depth > 0)
    NB_CUDA(launch_encode_pe(m, q, n, x_out, (cudaStream_t)stream));
  else
    NB_CUDA(launch_encode(m, q, n, x_out, (cudaStream_t)stream));
  return NB_OK;
}

static FwdArgs base_args(const nb_model* m, const float* q, const uint8_t* y, int64_t n) {
  FwdArgs a;
  memset(&a, 0, sizeof(a));
  a.q = q;
  a.y = y;
  a.n = n;
  for (int k = 0; k < 3; ++k) a.tau[k] = m->tau[k];
  a.counts = m->d_counts;
  a.fin_out = m->d_counts + kFinOff;  // finalised totals (score mode)
  a.ticket = m->d_flags + 2;          // last-CTA ticket
  a.counts_next = m->d_counts + 8;
  a.ticket_next = m->d_flags + 3;
  a.fin_add = 0;
  a.keys = m->d_keys;
  a.flags = m->d_flags;
  return a;
}

nb_status nb_forward(const nb_model* m, const float* q, int64_t n, float* logits, float* prob,
                     void* stream) {
  if (!m || n < 0 || (n > 0 && (!q || !logits))) return set_error("bad argument"), NB_E_ARG;
  if (n == 0) return NB_OK;
  if (!aligned16(q)) return misaligned("nb_forward");
  DeviceGuard g(m->device);
  FwdArgs a = base_args(m, q, nullptr, n);
  a.logits = logits;
  a.prob = prob;
  NB_CUDA(launch_forward_any(m, kForward, a, (cudaStream_t)stream));
  return NB_OK;
}

static nb_status calibrate_impl(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                                float* tau_out, void* stream, int invert) {
  if (!m || !tau_out || n < 0 || (n > 0 && (!q || !y))) return set_error("bad argument"), NB_E_ARG;
  if (invert && m->d.n_heads > 0)
    return set_error("inverted calibration: models without exit heads"), NB_E_UNSUPPORTED;
  if (n > 0 && (!aligned16(q) || !aligned16(y))) return misaligned("nb_calibrate");
  DeviceGuard g(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int nl = 1 + m->d.n_heads;
  NB_CUDA(cudaMemsetAsync(m->d_keys, 0xFF, sizeof(unsigned int) * 4, s));
  FwdArgs a = base_args(m, q, y, n);
  a.invert = invert;
  if (n > 0) NB_CUDA(launch_forward_any(m, kCalibrate, a, s));
  if (m->comm && comm_allreduce_u32_min(m, m->d_keys, nl, s))
    return NB_E_NCCL;
  unsigned int* hk = (unsigned int*)m->h_pinned;
  NB_CUDA(cudaMemcpyAsync(hk, m->d_keys, sizeof(unsigned int) * 4, cudaMemcpyDeviceToHost, s));
  NB_CUDA(cudaStreamSynchronize(s));
  bool none = false;
  for (int k = 0; k < nl; ++k) {
    if (hk[k] == 0xFFFFFFFFu) {
      m->tau[k] = INFINITY;
      none = true;
    } else if (invert) {  // the key holds min(-z) over negatives: tau = next float above max z
      m->tau[k] = nextafterf(-key2f(hk[k]), INFINITY);
    } else {
      m->tau[k] = key2f(hk[k]);
    }
    tau_out[k] = m->tau[k];
  }
  NB_CUDA(cudaMemcpyAsync(m->d_tau, m->tau, sizeof(float) * 3, cudaMemcpyHostToDevice, s));
  nb_status st = take_flags(m, s, NB_OK);
  if (st != NB_OK) return st;
  if (none) {
    set_error(invert ? "calibration set has no negatives" : "calibration set has no positives");
    return NB_E_NO_POSITIVES;
  }
  return NB_OK;
}

nb_status nb_calibrate(nb_model* m, const float* q, const uint8_t* y, int64_t n, float* tau_out,
                       void* stream) {
  return calibrate_impl(m, q, y, n, tau_out, stream, 0);
}

nb_status nb_calibrate_inverted(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                                float* tau_out, void* stream) {
  return calibrate_impl(m, q, y, n, tau_out, stream, 1);
}

// Score launches alternate between two counter sets / tickets: each launch's
// finalising CTA zeroes the other set, which the next launch uses.
static void use_score_set(nb_model* m, FwdArgs& a) {
  const int p = m->score_parity;
  m->score_parity ^= 1;
  a.counts = m->d_counts + 8 * p;
  a.counts_next = m->d_counts + 8 * (1 - p);
  a.ticket = m->d_flags + 2 + p;
  a.ticket_next = m->d_flags + 3 - p;
}

static void counts_out(const unsigned long long* c, nb_counts* out) {
  out->tp = c[0]; out->fp = c[1]; out->fn = c[2]; out->tn = c[3];
  for (int k = 0; k < 4; ++k) out->exit_hist[k] = c[4 + k];
  out->nonfinite = c[8];
}

nb_status nb_score(const nb_model* m_, const float* q, const uint8_t* y, int64_t n, nb_counts* out,
                   void* stream) {
  nb_model* m = const_cast<nb_model*>(m_);
  if (!m || !out || n < 0 || (n > 0 && (!q || !y))) return set_error("bad argument"), NB_E_ARG;
  if (n > 0 && (!aligned16(q) || !aligned16(y))) return misaligned("nb_score");
  DeviceGuard g(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* fin = m->d_counts + kFinOff;
  if (n > 0) {
    FwdArgs a = base_args(m, q, y, n);
    use_score_set(m, a);
    NB_CUDA(launch_forward_any(m, kScore, a, s));
  } else {
    NB_CUDA(cudaMemsetAsync(fin, 0, sizeof(unsigned long long) * kNumCounters, s));
  }
  if (m->comm && comm_allreduce_u64_sum(m, fin, kNumCounters, s)) return NB_E_NCCL;
  unsigned long long* hc = m->h_pinned;
  NB_CUDA(cudaMemcpyAsync(hc, fin, sizeof(unsigned long long) * kNumCounters,
                          cudaMemcpyDeviceToHost, s));
  NB_CUDA(cudaStreamSynchronize(s));
  counts_out(hc, out);
  nb_status st = take_flags(m, s, NB_OK);
  if (st == NB_OK && out->nonfinite) {  // warning-class: the counts are written
    set_error("%llu records produced a non-finite logit", (unsigned long long)out->nonfinite);
    st = NB_E_NONFINITE;
  }
  return st;
}

// Device-visible address of `out` (device memory, or pinned host memory mapped
// into the device's address space); NULL if the device cannot write it.
static void* device_view(void* out) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, out) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return out;
  if (at.type == cudaMemoryTypeHost) return at.devicePointer;
  return nullptr;
}

nb_status nb_score_async(const nb_model* m_, const float* q, const uint8_t* y, int64_t n,
                         nb_counts* out, void* stream) {
  static_assert(sizeof(nb_counts) == sizeof(unsigned long long) * kNumCounters, "nb_counts layout");
  nb_model* m = const_cast<nb_model*>(m_);
  if (!m || !out || n < 0 || (n > 0 && (!q || !y))) return set_error("bad argument"), NB_E_ARG;
  if (n > 0 && (!aligned16(q) || !aligned16(y))) return misaligned("nb_score_async");
  DeviceGuard g(m->device);
  void* dout = device_view(out);
  if (!dout) return set_error("nb_score_async: out must be device or pinned host memory"), NB_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // the device counter order is the nb_counts field order (tp fp fn tn exit[4] nonfinite)
  if (n == 0) {
    NB_CUDA(cudaMemcpyAsync(out, m->d_counts + kZeroOff, sizeof(nb_counts), cudaMemcpyDefault, s));
    return NB_OK;
  }
  FwdArgs a = base_args(m, q, y, n);
  use_score_set(m, a);
  if (!m->comm) {  // one launch: the last CTA writes the totals straight into `out`
    a.fin_out = (unsigned long long*)dout;
    NB_CUDA(launch_forward_any(m, kScore, a, s));
    return NB_OK;
  }
  NB_CUDA(launch_forward_any(m, kScore, a, s));
  if (comm_allreduce_u64_sum(m, a.fin_out, kNumCounters, s)) return NB_E_NCCL;
  NB_CUDA(cudaMemcpyAsync(out, a.fin_out, sizeof(nb_counts), cudaMemcpyDefault, s));
  return NB_OK;
}

nb_status nb_score_host(const nb_model* m_, const float* qh, const uint8_t* yh, int64_t n,
                        nb_counts* out, void* stream) {
  nb_model* m = const_cast<nb_model*>(m_);
  if (!m || !out || n < 0 || (n > 0 && (!qh || !yh))) return set_error("bad argument"), NB_E_ARG;
  DeviceGuard g(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t chunk = (int64_t)1 << 20;  // rows per staged chunk (multiple of 128)
  if (m->stage_rows < chunk) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(m->stage_q[i]);
      cudaFree(m->stage_y[i]);
      m->stage_q[i] = nullptr;
      m->stage_y[i] = nullptr;
      NB_CUDA(cudaMalloc((void**)&m->stage_q[i], sizeof(float) * chunk * m->d0));
      NB_CUDA(cudaMalloc((void**)&m->stage_y[i], chunk));
    }
    m->stage_rows = chunk;
  }
  unsigned long long* fin = m->d_counts + kFinOff;
  NB_CUDA(cudaMemsetAsync(fin, 0, sizeof(unsigned long long) * kNumCounters, s));
  // the copy stream may only start once the counters are reset / prior work done
  NB_CUDA(cudaEventRecord(m->ev_done[0], s));
  NB_CUDA(cudaEventRecord(m->ev_done[1], s));
  int64_t i = 0;
  for (int64_t r0 = 0; r0 < n; r0 += chunk, ++i) {
    const int b = (int)(i & 1);
    const int64_t rows = std::min(chunk, n - r0);
    NB_CUDA(cudaStreamWaitEvent(m->copy_stream, m->ev_done[b], 0));
    NB_CUDA(cudaMemcpyAsync(m->stage_q[b], qh + r0 * m->d0, sizeof(float) * rows * m->d0,
                            cudaMemcpyHostToDevice, m->copy_stream));
    NB_CUDA(cudaMemcpyAsync(m->stage_y[b], yh + r0, rows, cudaMemcpyHostToDevice, m->copy_stream));
    NB_CUDA(cudaEventRecord(m->ev_copy[b], m->copy_stream));
    NB_CUDA(cudaStreamWaitEvent(s, m->ev_copy[b], 0));
    FwdArgs a = base_args(m, m->stage_q[b], m->stage_y[b], rows);
    use_score_set(m, a);
    a.fin_add = 1;  // every chunk's last CTA adds its totals into fin
    NB_CUDA(launch_forward_any(m, kScore, a, s));
    NB_CUDA(cudaEventRecord(m->ev_done[b], s));
  }
  if (m->comm && comm_allreduce_u64_sum(m, fin, kNumCounters, s)) return NB_E_NCCL;
  unsigned long long* hc = m->h_pinned;
  NB_CUDA(cudaMemcpyAsync(hc, fin, sizeof(unsigned long long) * kNumCounters,
                          cudaMemcpyDeviceToHost, s));
  NB_CUDA(cudaStreamSynchronize(s));
  counts_out(hc, out);
  nb_status st = take_flags(m, s, NB_OK);
  if (st == NB_OK && out->nonfinite) {  // warning-class: the counts are written
    set_error("%llu records produced a non-finite logit", (unsigned long long)out->nonfinite);
    st = NB_E_NONFINITE;
  }
  return st;
}

// Validation and scratch sizing of a training step of n_local rows.
static nb_status train_prepare(nb_model* m, const float* q, const uint8_t* y, int64_t n_local,
                               int64_t n_global, float alpha, float beta, float lr, cudaStream_t s) {
  if (!m || n_local < 0 || n_global < n_local || n_global <= 0 ||
      (n_local > 0 && (!q || !y)))
    return set_error("bad argument"), NB_E_ARG;
  if (!(alpha > 0.f) || !(beta >= 0.f) || !(lr > 0.f)) return set_error("bad alpha/beta/lr"), NB_E_ARG;
  if (n_local > 0 && (!aligned16(q) || !aligned16(y))) return misaligned("nb_train_step");
  const bool tc = m->d.precision == NB_BF16;
  if (tc && !train_tc_supported(m->d)) {
    set_error("bf16 training not built for width %d / sine / positional encoding", m->d.width);
    return NB_E_UNSUPPORTED;
  }
  if (!tc && (m->d.width > 32 || m->din > m->d.width)) {
    set_error("fp32 training supports width <= 32 and input features <= width");
    return NB_E_UNSUPPORTED;
  }
  size_t need = tc ? train_tc_scratch_bytes(m, n_local) : train_simt_scratch_bytes(m, n_local);
  if (need > m->train_scratch_bytes) {
    NB_CUDA(cudaStreamSynchronize(s));
    cudaFree(m->train_scratch);
    m->train_scratch = nullptr;
    m->train_scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&m->train_scratch, need);
    if (e != cudaSuccess) return set_error("train scratch: %s", cudaGetErrorString(e)), NB_E_OOM;
    m->train_scratch_bytes = need;
  }
  return NB_OK;
}

// The launches of one training step on stream s (no synchronisation).
static nb_status train_enqueue(nb_model* m, const float* q, const uint8_t* y, int64_t n_local,
                               int64_t n_global, float alpha, float beta, float lr, cudaStream_t s) {
  const bool tc = m->d.precision == NB_BF16;
  // this step's statistics buffer; tensor-core steps find it zeroed by the
  // previous step's gradient reduce (or by model creation)
  m->d_loss = m->d_loss_base + 8 * m->lbuf;
  m->d_stats = reinterpret_cast<unsigned long long*>(m->d_loss + 2);
  m->lbuf ^= 1;
  if (!tc) NB_CUDA(cudaMemsetAsync(m->d_loss, 0, 64, s));
  if (tc) {
    g_err.clear();
    // without a communicator the reduced gradient is final: Adam rides in the reduce
    // Adam inside the gradient reduce saves a launch while the reduce is
    // latency-bound; above ~2^17 parameters the reduce's element order
    // (D row fastest) makes the Adam loads strided and the separate
    // coalesced k_adam_pack wins (measured: c2/c3 -2/-4 us, c5 +9 us)
    static const bool no_fuse = getenv("NB_ADAM_SEPARATE") != nullptr;  // measurement switch
    const bool fuse = !m->comm && !no_fuse && m->P <= (1 << 17);
    const cudaError_t e = launch_train_tc(m, q, y, n_local, n_global, alpha, beta, fuse ? lr : 0.f, s);
    if (e != cudaSuccess) {  // keep the failing stage's detail
      const std::string stage = g_err;
      cuda_fail(e, "nb_train_step");
      if (!stage.empty()) g_err += " [" + stage + "]";
      return NB_E_CUDA;
    }
  } else {
    NB_CUDA(launch_train_simt(m, q, y, n_local, n_global, alpha, beta, s));
  }
  if (m->comm) {
    if (comm_allreduce_f32_sum(m, m->grad, m->P, s)) return NB_E_NCCL;
  }
  if (tc && (m->comm || m->P > (1 << 17) || getenv("NB_ADAM_SEPARATE"))) NB_CUDA(launch_adam_pack(m, lr, s));
  else if (!tc) NB_CUDA(launch_adam(m, lr, s));
  return NB_OK;
}

nb_status nb_train_step(nb_model* m, const float* q, const uint8_t* y, int64_t n_local,
                        int64_t n_global, float alpha, float beta, float lr, nb_step_stats* stats,
                        void* stream) {
  if (!m) return set_error("null model"), NB_E_ARG;
  DeviceGuard g(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  nb_status st = train_prepare(m, q, y, n_local, n_global, alpha, beta, lr, s);
  if (st != NB_OK) return st;
  st = train_enqueue(m, q, y, n_local, n_global, alpha, beta, lr, s);
  if (st != NB_OK) return st;
  if (stats) {
    if (m->comm) {
      if (comm_allreduce_f64_sum(m, m->d_loss, 1, s)) return NB_E_NCCL;
      if (comm_allreduce_u64_sum(m, m->d_stats, 4, s)) return NB_E_NCCL;
    }
    unsigned long long* hs = m->h_pinned;
    NB_CUDA(cudaMemcpyAsync(hs, m->d_stats, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaMemcpyAsync(hs + 4, m->d_loss, sizeof(double), cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    stats->tp = hs[0]; stats->fp = hs[1]; stats->fn = hs[2]; stats->tn = hs[3];
    double l;
    memcpy(&l, hs + 4, sizeof(double));
    stats->loss = l;
    return take_flags(m, s, NB_OK);
  }
  return NB_OK;
}

nb_status nb_train_steps(nb_model* m, const float* q, const uint8_t* y, int64_t n_local, int64_t n_global,
                         int32_t steps, float alpha0, float alpha1, float beta, float lr, void* stream) {
  if (!m || steps < 1 || !(alpha1 > 0.f)) return set_error("bad argument"), NB_E_ARG;
  // every step's batch view must stay 16-byte aligned (nb.h "Alignment")
  if (steps > 1 && (n_local % 16 != 0)) return set_error("nb_train_steps: n_local must be a multiple of 16"), NB_E_ARG;
  DeviceGuard g(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  nb_status st = train_prepare(m, q, y, n_local, n_global, alpha0, beta, lr, s);
  if (st != NB_OK) return st;
  auto alpha_t = [&](int32_t t) {
    return steps == 1 ? alpha0 : (float)((double)alpha0 + ((double)alpha1 - alpha0) * t / (double)(steps - 1));
  };
  const int64_t d0 = m->d0;
  if (m->comm || steps == 1) {  // plain stream order (collectives stay outside graphs)
    for (int32_t t = 0; t < steps; ++t) {
      st = train_enqueue(m, q + (size_t)t * n_local * d0, y + (size_t)t * n_local, n_local, n_global,
                         alpha_t(t), beta, lr, s);
      if (st != NB_OK) return st;
    }
    return NB_OK;
  }
  // capture the step sequence on the model's graph stream, replay it once
  if (!m->graph_stream) NB_CUDA(cudaStreamCreateWithFlags(&m->graph_stream, cudaStreamNonBlocking));
  if (!m->ev_graph[0]) {
    NB_CUDA(cudaEventCreateWithFlags(&m->ev_graph[0], cudaEventDisableTiming));
    NB_CUDA(cudaEventCreateWithFlags(&m->ev_graph[1], cudaEventDisableTiming));
    NB_CUDA(cudaEventCreateWithFlags(&m->ev_graph_done[0], cudaEventDisableTiming));
    NB_CUDA(cudaEventCreateWithFlags(&m->ev_graph_done[1], cudaEventDisableTiming));
  }
  // two executable graphs alternate: the one from two calls ago has finished
  // (its completion event) before it is released, so this call's capture on
  // the host overlaps the previous call's execution on the device
  const int slot = m->graph_slot;
  m->graph_slot ^= 1;
  if (m->graph_exec2[slot]) {
    NB_CUDA(cudaEventSynchronize(m->ev_graph_done[slot]));
    cudaGraphExecDestroy((cudaGraphExec_t)m->graph_exec2[slot]);
    m->graph_exec2[slot] = nullptr;
  }
  cudaStream_t cs = m->graph_stream;
  NB_CUDA(cudaEventRecord(m->ev_graph[0], s));
  NB_CUDA(cudaStreamWaitEvent(cs, m->ev_graph[0], 0));
  NB_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int32_t t = 0; t < steps && st == NB_OK; ++t)
    st = train_enqueue(m, q + (size_t)t * n_local * d0, y + (size_t)t * n_local, n_local, n_global, alpha_t(t),
                       beta, lr, cs);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  if (st != NB_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ec != cudaSuccess) return cuda_fail(ec, "nb_train_steps: capture");
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return cuda_fail(ei, "nb_train_steps: instantiate");
  m->graph_exec2[slot] = exec;
  NB_CUDA(cudaGraphLaunch(exec, cs));
  NB_CUDA(cudaEventRecord(m->ev_graph_done[slot], cs));
  NB_CUDA(cudaStreamWaitEvent(s, m->ev_graph_done[slot], 0));
  return NB_OK;
}

nb_status nb_model_set_regularization(nb_model* m, float l1, float l2) {
  if (!m || !(l1 >= 0.f) || !(l2 >= 0.f)) return set_error("bad argument"), NB_E_ARG;
  m->l1 = l1;
  m->l2 = l2;
  return NB_OK;
}

nb_status nb_schedule_init(nb_schedule* s, int32_t space_dim, int64_t step_every, int64_t max_steps) {
  if (!s || space_dim < 2 || space_dim > 4 || step_every < 1 || max_steps < 1)
    return set_error("bad argument"), NB_E_ARG;
  memset(s, 0, sizeof(*s));
  s->space_dim = space_dim;
  s->patience = 6;
  s->step_every = step_every;
  s->max_steps = max_steps;
  s->alpha = 1.0;
  s->beta = 1.0;
  s->lambda = 0.0;
  return NB_OK;
}

nb_status nb_schedule_after_step(nb_schedule* s, uint64_t batch_fn) {
  if (!s) return set_error("null argument"), NB_E_ARG;
  s->window_fn += batch_fn;
  s->step += 1;
  if (s->step % s->step_every == 0) {  // end of a scheduling window
    if (s->window_fn > 0) {
      s->triggers += 1;
      const double base = s->space_dim == 2 ? 1.0 / 20 : (s->space_dim == 3 ? 1.0 / 100 : 1.0 / 200);
      s->beta = std::max(1e-3, s->beta - base / (double)s->triggers);
      s->alpha = 1.0 + 0.2 * (double)s->triggers;
      s->stable = 0;
    } else {
      s->stable += 1;
    }
    s->window_fn = 0;
  }
  s->lambda = 5e-7 * std::min(1.0, (double)s->step / (double)s->max_steps);
  if (s->stable >= s->patience || s->step >= s->max_steps) s->stop = 1;
  return NB_OK;
}

double nb_alpha(int64_t t, int64_t T) {
  if (T <= 1) return 1000.0;
  return 1.0 + 999.0 * (double)t / (double)(T - 1);
}

nb_status nb_comm_unique_id(uint8_t id[128]) {
  if (!id) return set_error("null id"), NB_E_ARG;
  return comm_unique_id(id) ? NB_E_NCCL : NB_OK;
}

nb_status nb_comm_init(nb_model* m, const uint8_t id[128], int32_t rank, int32_t world) {
  if (!m || !id || world < 1 || rank < 0 || rank >= world) return set_error("bad argument"), NB_E_ARG;
  DeviceGuard g(m->device);
  return comm_init(m, id, rank, world) ? NB_E_NCCL : NB_OK;
}

nb_status nb_comm_version(int32_t* v) {
  if (!v) return NB_E_ARG;
  int vv = 0;
  if (comm_version(&vv)) return NB_E_NCCL;
  *v = vv;
  return NB_OK;
}

// Node forward for the hierarchy: the model's fused kernel in forward mode,
// its row count read on the device (n_dev) below the launch's upper bound n.
static cudaError_t hier_forward(const nb_model* m, const float* q, int64_t n, const unsigned long long* n_dev,
                                float* logits, cudaStream_t s) {
  FwdArgs a = base_args(m, q, nullptr, n);
  a.logits = logits;
  a.n_dev = n_dev;
  return launch_forward_any(m, kForward, a, s);
}

nb_status nb_hier_score(nb_model* const* nodes, int32_t n_nodes, const int32_t* parent, const float* q,
                        const uint8_t* y, int64_t n, nb_counts* out, void* stream) {
  if (!nodes || n_nodes < 1 || !parent || !out || n < 0 || n > INT32_MAX || (n > 0 && (!q || !y)))
    return set_error("bad argument"), NB_E_ARG;
  if (parent[0] != -1) return set_error("parent[0] must be -1 (root)"), NB_E_ARG;
  for (int i = 0; i < n_nodes; ++i) {
    if (!nodes[i]) return set_error("null node"), NB_E_ARG;
    if (i > 0 && (parent[i] < 0 || parent[i] >= i)) return set_error("parent[i] must precede i"), NB_E_ARG;
    if (nodes[i]->device != nodes[0]->device || nodes[i]->d0 != nodes[0]->d0)
      return set_error("nodes must share the device and the record layout"), NB_E_ARG;
    if (nodes[i]->comm) return set_error("hierarchies run on one GPU"), NB_E_UNSUPPORTED;
    // node kernels read their row count on the device (k_fwd_tc, k_fwd_simt)
    if (nodes[i]->pl.pairs != 1)
      return set_error("hierarchy nodes: widths <= 128 (no CTA-pair models)"), NB_E_UNSUPPORTED;
  }
  if (!aligned16(q)) return misaligned("nb_hier_score");
  DeviceGuard g(nodes[0]->device);
  unsigned long long c[5] = {0, 0, 0, 0, 0};
  NB_CUDA(hier_score(nodes, n_nodes, parent, q, y, n, c, (cudaStream_t)stream, hier_forward));
  memset(out, 0, sizeof(*out));
  out->tp = c[0]; out->fp = c[1]; out->fn = c[2]; out->tn = c[3];
  out->nonfinite = c[4];
  if (out->nonfinite) {  // warning-class, as nb_score: the counts are written
    set_error("%llu records produced a non-finite logit", (unsigned long long)out->nonfinite);
    return NB_E_NONFINITE;
  }
  return NB_OK;
}

nb_status nb_grid_create(int32_t space_dim, int32_t R, int32_t frames, const uint8_t* host,
                         int32_t device, nb_grid** out) {
  if (!host || !out || space_dim < 2 || space_dim > 4 || R < 1 || R > 4096 ||
      (space_dim == 4 && frames < 1))
    return set_error("bad grid"), NB_E_ARG;
  DeviceGuard g(device);
  nb_grid* gr = new nb_grid();
  gr->space_dim = space_dim;
  gr->R = R;
  gr->frames = space_dim == 4 ? frames : 1;
  gr->device = device;
  size_t cells = (size_t)gr->frames;
  for (int j = 0; j < (space_dim == 4 ? 3 : space_dim); ++j) cells *= (size_t)R;
  cudaError_t e = cudaMalloc((void**)&gr->occ, cells);
  if (e == cudaSuccess) e = cudaMemcpy(gr->occ, host, cells, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && space_dim == 3) {
    e = cudaMalloc((void**)&gr->sat, sizeof(int32_t) * (size_t)(R + 1) * (R + 1) * (R + 1));
    if (e == cudaSuccess) e = launch_sat_build(gr, 0);
    if (e == cudaSuccess) e = launch_blk_build(gr, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e == cudaSuccess && space_dim == 2) {
    e = launch_sat2_build(gr, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e == cudaSuccess && space_dim == 4) {  // 4D boxes / hyperplanes (R48)
    e = launch_grid4_build(gr, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    nb_grid_destroy(gr);
    return cuda_fail(e, "nb_grid_create");
  }
  *out = gr;
  return NB_OK;
}

void nb_grid_destroy(nb_grid* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  cudaFree(g->occ);
  cudaFree(g->sat);
  cudaFree(g->blk);
  delete g;
}

nb_status nb_label(const nb_grid* g, int32_t kind, const float* q, int64_t n, uint8_t* y,
                   void* stream) {
  if (!g || n < 0 || (n > 0 && (!q || !y))) return set_error("bad argument"), NB_E_ARG;
  if (kind != NB_POINT && kind != NB_RAY && kind != NB_BOX && kind != NB_PLANE) {
    set_error("GPU labeller: unknown query kind");
    return NB_E_ARG;
  }
  if (n == 0) return NB_OK;
  DeviceGuard dg(g->device);
  NB_CUDA(launch_label(g, kind, q, n, y, (cudaStream_t)stream));
  return NB_OK;
}

}  // extern "C"
