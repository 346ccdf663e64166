// nb_internal.cuh — internal declarations of libnb.so (not part of the ABI).
//
// Product code only: nothing here is shared with oracle/ (which must stay an
// independent implementation of the paper).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/nb.h"

#include <utility>

namespace nb {

constexpr int kMaxLayers = 8;
constexpr int kTile = 128;          // rows per MMA tile (M = 128)
constexpr int kEncK = 16;           // layer-1 K after the bf16 (hi, lo) split (no encoding)
// layer-1 K for d_in input features: hi and lo halves plus three bias ones
// columns, rounded up to the MMA K step (16 for every record without PE)
__host__ __device__ constexpr int enc_k(int din) { return (2 * din + 3 + 15) / 16 * 16; }
constexpr int kSimtMaxIn = 64;      // fp32 path: layer-1 input features (with PE)
constexpr int kTcMaxEncK = 64;      // bf16 path: layer-1 K (2 d_in + 3 <= 64)
constexpr int kNumCounters = 9;     // tp fp fn tn exit[4] nonfinite
constexpr int kCtrStride = 16;      // device counters 128 B apart (one L2 line each); set 1 at +8
constexpr int kFinOff = kNumCounters * kCtrStride;  // nb_model::d_counts: finalised totals
constexpr int kZeroOff = kFinOff + 16;              // ... and a block that stays zero
constexpr uint32_t kFlagNonFinite = 1u, kFlagLabel = 2u;

void set_error(const char* fmt, ...);

// Byte layout of the packed bf16 parameter image that a CTA copies into shared
// memory once (cp.async.bulk).  B operands are K-major, no-swizzle UMMA core
// matrices: element (n, k) of an [N][K] matrix sits at
//   (n / 8) * SBO + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2,  SBO = K / 8 * 128.
struct PackLayout {
  uint32_t off_w[kMaxLayers];  // layer l B image (layer 0: [W][16], others [W][W])
  uint32_t k_of[kMaxLayers];   // K of each layer image (16 or W)
  uint32_t off_bias;           // fp32 [L][W]
  uint32_t off_wout;           // fp32 [W]
  uint32_t off_bout;           // fp32 (padded to 16 B)
  uint32_t off_u[2];           // fp32 [W] per head
  uint32_t off_c;              // fp32 [2] head biases (padded)
  uint32_t core_bytes;         // the image up to here (what the training kernels copy)
  // Bias-as-MMA blocks (pairs == 1 only, DESIGN.md §6 "bias folding"): layer
  // l >= 1 has an [W][16] K-major B image whose k = 0, 1, 2 columns hold the
  // exact bf16 split hi + mid + lo of b_l (a ones block in TMEM is its A);
  // layer 0's image holds the same split in columns 2 d0 .. 2 d0 + 2 when
  // bias_l0 != 0 (the in-kernel encoder puts ones there).
  uint32_t off_bb[kMaxLayers];
  uint32_t bias_l0;
  uint32_t pe_lo;
  // positional-encoding nets (bf16): layer 1 is K = 64 with hi halves in
  // columns [0, d_in), the bias ones at [d_in, d_in + 3) and lo halves at
  // [pe_lo, pe_lo + d_in), pe_lo = 32 (compile-time operand indices in the
  // encoder); 0 = the default [hi | lo | ones] order
  // CTA-pair images (pairs == 2): ONE shared [rows][16] bias block at
  // off_bb[0] holds the split of every hidden layer l >= 1 in columns
  // 3 (l - 1) .. 3 (l - 1) + 2 (a per-layer ones block in TMEM selects them)
  uint32_t bb_shared;
  uint32_t bytes;              // one image, multiple of 16
  uint32_t pairs;              // 1, or 2 for CTA-pair widths (2 images, each with W/2 rows)
};

// Transposed pair images for the w = 256 backward chain (CTA pairs): image v
// holds, for each hidden layer l >= 1, W_l^T rows = input features
// [128 v, 128 v + 128) x K = 256 output features (K-major core matrices, the
// N half of cta_group::2's B), then fp32 w_out and the head vectors.
struct BwdLayout {
  uint32_t off_wt[kMaxLayers];  // layer l >= 1
  uint32_t off_wout, off_u[2];
  uint32_t bytes;               // one image
};

struct ParamOffsets {  // canonical fp32 blob offsets (nb.h nb_num_params)
  int64_t W[kMaxLayers], b[kMaxLayers], wout, bout, u[2], c[2];
};

}  // namespace nb

struct nb_model {
  nb_desc d;
  int device = 0;
  int d0 = 0;                 // record floats (query stride)
  int din = 0;                // layer-1 input features: d0, or d0 (1 + pe_depth) (R42)
  int64_t P = 0;
  int num_sms = 0;
  nb::ParamOffsets po;
  nb::PackLayout pl;
  float* theta = nullptr;     // fp32 master, canonical layout [P]
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  float* grad = nullptr;      // [P] gradient of the current step
  int64_t step = 0;
  float l1 = 0.f, l2 = 0.f;   // L1 / L2 regularisation added to the gradient by Adam (R38)
  uint8_t* packed = nullptr;  // bf16 packed image (pl.bytes)
  nb::BwdLayout bl;
  uint8_t* packed_bwd = nullptr;  // w = 256 training: 2 transposed pair images (bl.bytes)
  float tau[3] = {0, 0, 0};
  float* d_tau = nullptr;     // [3]
  unsigned long long* d_counts = nullptr;  // counters (strided), totals, zeros: 256 words
  unsigned int* d_keys = nullptr;          // [3] order-preserving min keys
  unsigned int* d_flags = nullptr;         // sticky flags, [2], [3] score tickets
  int score_parity = 0;                    // counter set of the next score launch
  double* d_loss = nullptr;                // [1] loss of the current step's buffer
  unsigned long long* d_stats = nullptr;   // [4] batch tp fp fn tn (current buffer)
  // the step statistics are double-buffered (2 x 64 B at d_loss_base): a
  // tensor-core step accumulates into buffer `lbuf` and its gradient reduce
  // zeroes the other one for the next step, so no memset sits between the
  // steps' kernels (programmatic dependent launch, nb_train_tc.cu)
  double* d_loss_base = nullptr;
  int lbuf = 0;
  unsigned long long* h_pinned = nullptr;  // pinned host mirror for small readbacks
  // training scratch (grown on demand outside the timed hot path)
  void* train_scratch = nullptr;
  size_t train_scratch_bytes = 0;
  // early-exit compaction scratch (nb_fwd_exit.cu): 2 image/label region sets
  void* exit_scratch = nullptr;
  size_t exit_scratch_bytes = 0;
  // hierarchy scratch (nb_hier_score, held by the root node; grown on demand)
  void* hier_scratch = nullptr;
  size_t hier_scratch_bytes = 0;
  // nb_train_steps: the captured step sequence (CUDA graph) and its stream
  cudaStream_t graph_stream = nullptr;
  void* graph_exec2[2] = {nullptr, nullptr};  // cudaGraphExec_t of the last two calls
  int graph_slot = 0;
  cudaEvent_t ev_graph[2] = {nullptr, nullptr};
  cudaEvent_t ev_graph_done[2] = {nullptr, nullptr};
  // host-buffer serving path
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  float* stage_q[2] = {nullptr, nullptr};
  uint8_t* stage_y[2] = {nullptr, nullptr};
  int64_t stage_rows = 0;
  // communicator
  void* comm = nullptr;
  int rank = 0, world = 1;
  // kernel-time instrumentation (off by default)
  int timing = 0;
  static constexpr int kEvPool = 4096;     // event pairs recorded without host syncs
  cudaEvent_t* ev_pool = nullptr;          // [2 * kEvPool]
  int ev_used = 0;
  int64_t kernel_launches = 0;
};

struct nb_grid {
  int space_dim = 0, R = 0, frames = 1, device = 0;
  uint8_t* occ = nullptr;   // device copy of the grid
  int32_t* sat = nullptr;   // (R+1)^3 summed-area table (3D only)
  uint8_t* blk = nullptr;   // 3D: any-occupied flag per 8^3-voxel block (plane labeller)
};

namespace nb {

// ---- launchers (each returns cudaGetLastError of its launch) ---------------
enum Mode { kForward = 0, kCalibrate = 1, kScore = 2, kTrain = 3 };

// Training-mode outputs of the forward kernel (bf16 training).
// "Row-tile images": per 128-row tile, a [F features][128 rows] bf16 matrix in
// UMMA MN-major no-swizzle core-matrix order,
//   byte(r, f) = ((f / 8) * 16 + r / 8) * 128 + (r % 8) * 16 + (f % 8) * 2,
// tile t at t * F * 256 bytes; consumed directly by the dW GEMM (bulk copy).
struct TrainArgs {
  uint8_t* x_img;                // encoded layer-1 input, F = 16
  uint8_t* h_img[kMaxLayers];    // h_l (post-activation, bf16), F = w, l = 1..L
  uint8_t* c_img[kMaxLayers];    // sine nets: cos(z_l) (bf16), F = w — the activation derivative;
                                 // ReLU: h_l > 0 bit masks (W * 16 B per row tile, word (f / 32) * 128 + row)
                                 // for the backward (k_bwd_tc / k_bwd_tc2p), NULL for CTA pairs with heads
  uint8_t* hd_img;               // [dL/dz, dL/de_1, dL/de_2, 0..] bf16, F = 8
  float* g32;                    // fp32 [n][3]: dL/dz, dL/de_1, dL/de_2
  float alpha, beta, inv_b;      // Eq. (1) weights, 1 / n_global
  double* loss;
  unsigned long long* stats;     // batch tp fp fn tn at z >= 0
  int64_t num_tiles;             // 128-row tiles with images (CTA-pair kernel bound)
};

struct FwdArgs {
  const float* q;
  const uint8_t* y;
  int64_t n;
  float* logits;
  float* prob;
  float tau[3];
  unsigned long long* counts;
  // a5 finalisation (kScore): when ticket != NULL the last CTA to finish moves
  // the totals to fin_out (plain store, or atomicAdd when fin_add) and
  // re-zeroes `counts` and the ticket, so a launch needs no memset or copy
  unsigned long long* fin_out;
  unsigned int* ticket;
  int fin_add;
  // the other (idle) counter set and ticket: the finalising CTA zeroes them for
  // the next launch, which uses them (launches alternate between two sets)
  unsigned long long* counts_next;
  unsigned int* ticket_next;
  unsigned int* keys;
  unsigned int* flags;
  int invert;  // kCalibrate: certainly-hit threshold (min of -z over negatives, nb_calibrate_inverted)
  // kForward of k_fwd_tc: when set, the row count is read from device memory
  // (written by an earlier kernel; n is then only the launch's upper bound)
  const unsigned long long* n_dev;
  TrainArgs tr;
};

__host__ __device__ constexpr int64_t img_tile_bytes(int features) { return (int64_t)features * 256; }

cudaError_t launch_pack_bf16(const nb_model* m, cudaStream_t s);
cudaError_t launch_encode(const nb_model* m, const float* q, int64_t n, void* out, cudaStream_t s);
cudaError_t launch_encode_pe(const nb_model* m, const float* q, int64_t n, void* out, cudaStream_t s);
cudaError_t launch_fwd_simt(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t s);
cudaError_t launch_fwd_tc(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t s);
cudaError_t launch_fwd_tc2(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t s);
bool exit_compaction_supported(const nb_model* m);
cudaError_t launch_score_exit(nb_model* m, const FwdArgs& a, cudaStream_t s, int* kernels);
bool tc_supported(const nb_desc& d);
bool tc2_supported(const nb_desc& d);
bool simt_supported(const nb_desc& d);

cudaError_t launch_train_simt(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                              int64_t n_global, float alpha, float beta, cudaStream_t s);
// fuse_lr > 0: the gradient reduce also takes the Adam step + re-pack (no
// communicator); 0: the caller launches Adam after the allreduce
cudaError_t launch_train_tc(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                            int64_t n_global, float alpha, float beta, float fuse_lr, cudaStream_t s);
bool train_tc_supported(const nb_desc& d);
cudaError_t launch_bwd_tc2(const nb_model* m, const uint8_t* const* h_img, uint8_t* const* d_img,
                           const float* g32, int64_t n, cudaStream_t st,
                           const uint8_t* const* m_img = nullptr);  // h_l > 0 bit masks (pipelined)
size_t train_tc_scratch_bytes(const nb_model* m, int64_t n);
size_t train_simt_scratch_bytes(const nb_model* m, int64_t n);
cudaError_t launch_adam(nb_model* m, float lr, cudaStream_t s);
cudaError_t launch_adam_pack(nb_model* m, float lr, cudaStream_t s);  // Adam + bf16 re-pack
cudaError_t launch_label(const nb_grid* g, int kind, const float* q, int64_t n, uint8_t* y,
                         cudaStream_t s);
cudaError_t launch_sat_build(nb_grid* g, cudaStream_t s);
cudaError_t launch_blk_build(nb_grid* g, cudaStream_t s);
cudaError_t launch_sat2_build(nb_grid* g, cudaStream_t s);
cudaError_t launch_grid4_build(nb_grid* g, cudaStream_t s);  // 4D SAT + block flags (R48)
cudaError_t hier_score(nb_model* const* nodes, int n_nodes, const int32_t* parent, const float* q,
                       const uint8_t* y, int64_t n, unsigned long long* h_counts /*[5]*/, cudaStream_t st,
                       cudaError_t (*forward)(const nb_model*, const float*, int64_t,
                                              const unsigned long long*, float*, cudaStream_t));

// NCCL (dlopen'ed); all return 0 on success
int comm_unique_id(uint8_t id[128]);
int comm_init(nb_model* m, const uint8_t id[128], int rank, int world);
void comm_destroy(nb_model* m);
int comm_allreduce_u64_sum(nb_model* m, unsigned long long* buf, size_t count, cudaStream_t s);
int comm_allreduce_u32_min(nb_model* m, unsigned int* buf, size_t count, cudaStream_t s);
int comm_allreduce_f32_sum(nb_model* m, float* buf, size_t count, cudaStream_t s);
int comm_allreduce_f64_sum(nb_model* m, double* buf, size_t count, cudaStream_t s);
int comm_version(int* v);

// order-preserving fp32 <-> u32 key (min of keys == key of min)
__host__ __device__ inline uint32_t f2key(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ inline float key2f(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  float f;
  memcpy(&f, &b, 4);
  return f;
}


// Launch a training-chain kernel as a programmatic dependent of the previous
// kernel in the stream (pdl): its launch and CTA rasterisation overlap the
// predecessor's tail; the kernel itself calls griddep_wait() before touching
// memory.  (The fused w = 64 step kernel overlaps its prologue too.)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace nb
