/* nb.h — C ABI of the B200-native Neural Bounding hot path (libnb.so).
 *
 * The library implements the data-parallel hot path of "Neural Bounding"
 * (Liu, Fischer, Yoo, Ritschel; arXiv 2310.06822; /root/reference/PAPER.md,
 * cited as P:<line>):  a small MLP h_theta that classifies encoded
 * point / ray / plane / box queries as "maybe object" (1) or "certainly not
 * object" (0) with strictly zero false negatives on its labelled set
 * (problem statement P:133-145 §3.1, "the FN rate ... must be zero" P:75,
 * "FP is the only figure of merit" P:372), trained with the asymmetric loss
 * of Eq. (1) and Alg. 1.
 *
 * Conventions for every call (DESIGN.md §4 restates them):
 *  - Pointers named q, y, x_out, logits, prob, tau_dev are DEVICE pointers on
 *    the model's device, owned by the caller; the library never frees them.
 *    Calls whose name ends in _host take HOST pointers instead.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Query records are fp32, row-major [n][nb_record_floats(kind, dim)]:
 *      point: x (n floats; 4D is (x, y, z, t));  ray: (origin, unit direction);
 *      plane: (p0, unit normal);  box: (min corner, max corner);
 *      4D records carry 4 + 4 floats (Suppl. Tab. 4/5 "4D Ray, Plane, Box").
 *  - Labels y are uint8 in {0, 1}, one per record.
 *  - Alignment: device q and y passed to nb_forward, nb_calibrate*,
 *    nb_score, nb_score_async, nb_train_step and nb_hier_score must be
 *    16-byte aligned (the kernels stage whole 128-row tiles with
 *    cp.async.bulk).  A misaligned pointer (e.g. a view starting at row 1)
 *    returns NB_E_ARG before any launch.  Allocations are aligned; a row
 *    offset r keeps both aligned when r is a multiple of 16.
 *  - The model owns its weights (fp32 master + packed bf16 copy), Adam state,
 *    thresholds, scratch and communicator; nothing is allocated on the hot path.
 *  - Calls filling host structs (nb_counts, tau_out, nb_step_stats) synchronise
 *    `stream`; nb_encode / nb_forward / nb_label are asynchronous.
 *  - Errors: argument/shape validation happens before any launch (NB_E_ARG,
 *    NB_E_SHAPE) and leaves outputs untouched.  In-kernel sticky flags report
 *    non-finite logits (NB_E_NONFINITE) and labels outside {0,1} (NB_E_LABEL)
 *    on the next synchronising call, whose outputs are still written.
 *    NB_E_NO_POSITIVES is warning-class: tau = +inf is written.
 *    CUDA/NCCL failures return NB_E_CUDA / NB_E_NCCL; nb_last_error() gives
 *    the thread-local detail string.
 *  - With a communicator (nb_comm_init), n is the LOCAL shard; counts and tau
 *    returned are GLOBAL (one NCCL allreduce each); nb_train_step allreduces
 *    the gradient.  All ranks must issue collective calls in the same order.
 *  - Threading: one writer per model (train_step, calibrate, set_*);
 *    concurrent nb_forward / nb_encode calls on distinct streams are allowed.
 *    nb_score / nb_score_async / nb_score_host / nb_calibrate use the model's
 *    counter scratch (two alternating sets) and must be issued in order on one
 *    stream per model (they may interleave with nb_forward on it).
 */
#ifndef NB_H
#define NB_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NB_OK = 0,
  NB_E_ARG = 1,          /* null pointer / bad enum / negative size          */
  NB_E_SHAPE = 2,        /* dimension mismatch (record width, param count)    */
  NB_E_NONFINITE = 3,    /* some record produced a non-finite logit           */
  NB_E_LABEL = 4,        /* some label was not 0 or 1                         */
  NB_E_NO_POSITIVES = 5, /* calibration set without positives: tau = +inf     */
  NB_E_CUDA = 6,
  NB_E_NCCL = 7,
  NB_E_UNSUPPORTED = 8,  /* architecture outside the compiled kernel set      */
  NB_E_OOM = 9
} nb_status;

/* Query parameterisations, Suppl. §3.2. */
typedef enum { NB_POINT = 0, NB_RAY = 1, NB_PLANE = 2, NB_BOX = 3 } nb_query_kind;

/* Arithmetic of the forward/backward contractions.
 * NB_FP32: fp32 FMA chains on CUDA cores (BASELINE.json configs[0]).
 * NB_BF16: bf16 weights/activations, fp32 accumulation on tcgen05 tensor cores
 *          (configs[1..4]); inputs enter as a bf16 (hi, lo) pair (R20). */
typedef enum { NB_FP32 = 0, NB_BF16 = 1 } nb_precision;

/* Hidden activation: ReLU (BASELINE.json, R1) or the paper's sine
 * ("Sinusoidal activations are used in the hidden layers"; h = sin(z),
 * frequency 1, R41). */
typedef enum { NB_RELU = 0, NB_SINE = 1 } nb_activation;

/* MLP architecture (§3.4; Suppl. Tab. 4): d_in -> width x hidden_layers -> 1,
 * optional early-exit heads reading hidden layers head_after[k] (1-based;
 * P:231-279 §3.3, R22).  d_in = r (1 + pe_depth) for r record floats:
 * pe_depth = 0 feeds the record itself; an even pe_depth = L > 0 applies the
 * NeRF positional encoding of Suppl. §3 (R42)
 *   gamma(x) = (x, sin(2^0 pi x), cos(2^0 pi x), ..., sin(2^(L/2-1) pi x), cos(...))
 * ordered as [x_1..x_r, then per frequency k: sin(2^k pi x_1..r), cos(2^k pi x_1..r)]
 * (2D points with L = 8 give the paper's 18 inputs).  Zero-initialised
 * activation / pe_depth mean ReLU without encoding. */
typedef struct {
  int32_t kind;          /* nb_query_kind                                    */
  int32_t space_dim;     /* 2, 3 or 4 (4 = 3D + time; 4D rays / planes /
                            boxes are 8-float records over (x, y, z, t), R48;
                            bf16: widths 32..128, layer 1 K = 32)             */
  int32_t width;         /* hidden width w                                   */
  int32_t hidden_layers; /* L >= 1                                           */
  int32_t n_heads;       /* 0..2 early-exit heads                            */
  int32_t head_after[2]; /* 1-based hidden layer read by each head           */
  int32_t precision;     /* nb_precision                                     */
  int32_t activation;    /* nb_activation (0 = ReLU)                         */
  int32_t pe_depth;      /* 0, or even L in 2..16 (positional encoding)      */
} nb_desc;

/* Confusion counts of the calibrated predictor (P:157-176 cost cases);
 * exit_hist: [0] left at head 1, [1] left at head 2, [2] final negative,
 * [3] final positive.  tp + fp + fn + tn = n (global under a communicator). */
typedef struct {
  uint64_t tp, fp, fn, tn;
  uint64_t exit_hist[4];
  uint64_t nonfinite;
} nb_counts;

/* Batch statistics of one training step: loss value of Eq. (1) (plus head
 * terms) and the batch confusion counts at the rounding rule z >= 0
 * — the paper's convergence curves.                    */
typedef struct {
  double loss;
  uint64_t tp, fp, fn, tn;
} nb_step_stats;

typedef struct nb_model nb_model; /* opaque */
typedef struct nb_grid nb_grid;   /* opaque: occupancy grid for the GPU labeller */

/* ---- sizes ---------------------------------------------------------------- */
/* Floats per query record: n for points, 2n for ray/plane/box; -1 if invalid. */
int64_t nb_record_floats(int32_t kind, int32_t space_dim);
/* Parameters of the canonical fp32 blob: sum over layers of (d_in + 1) d_out
 * plus (w + 1) for the output and each head (the 3->50->50->1 net has the
 * paper's 2,801).  Layout: per hidden layer W_l[out][in] row-major then
 * b_l; then w_out[w], b_out; then per head u_k[w], c_k.  -1 if invalid.      */
int64_t nb_num_params(const nb_desc* desc);

const char* nb_status_string(nb_status s);
/* Detail of the last error on the calling thread ("" if none). */
const char* nb_last_error(void);
/* Compute capability major*10+minor of `device`, and whether this build has
 * kernels for it (sm_100a only).  Returns NB_E_UNSUPPORTED otherwise.      */
nb_status nb_device_check(int32_t device, int32_t* cc_out);

/* ---- model lifecycle ------------------------------------------------------ */
/* Allocates all device state on `device`.  Parameters start at zero. */
nb_status nb_model_create(const nb_desc* desc, int32_t device, nb_model** out);
void      nb_model_destroy(nb_model* m);
/* Host fp32 canonical blob of nb_num_params values; resets Adam state/step. */
nb_status nb_model_set_params(nb_model* m, const float* host, int64_t n);
nb_status nb_model_get_params(const nb_model* m, float* host, int64_t n);
/* Thresholds tau[0] (output), tau[1+k] (head k), logit space (R21). */
nb_status nb_model_set_thresholds(nb_model* m, const float* tau_host, int32_t n);
nb_status nb_model_get_thresholds(const nb_model* m, float* tau_host, int32_t n);
/* Gradient dL/dtheta of the last nb_train_step (after the allreduce), fp32 [P],
 * canonical layout: the parity hook for rows a7/a8 (DESIGN.md §5 P3).       */
nb_status nb_model_get_grad(const nb_model* m, float* host, int64_t n);
/* Adam state (checkpoint/resume): m, v as fp32 [P] host arrays, step count. */
nb_status nb_model_get_adam(const nb_model* m, float* m_host, float* v_host, int64_t* step);
nb_status nb_model_set_adam(nb_model* m, const float* m_host, const float* v_host, int64_t step);

/* Kernel-time instrumentation: when enabled, CUDA events bracket every
 * hot-path kernel launch of this model on the caller's stream (adding one
 * event synchronisation per launch).  nb_model_kernel_time returns the summed
 * device time (ms) and launch count since the previous call, then resets.  */
nb_status nb_model_set_timing(nb_model* m, int32_t enable);
nb_status nb_model_kernel_time(nb_model* m, double* ms, int64_t* launches);

/* ---- communicator (NCCL over NVLink/NVSwitch) ----------------------------- */
/* 128-byte NCCL unique id, produced on rank 0 and broadcast by the caller. */
nb_status nb_comm_unique_id(uint8_t id[128]);
nb_status nb_comm_init(nb_model* m, const uint8_t id[128], int32_t rank, int32_t world);
/* Query the NCCL library actually loaded: version code (e.g. 22809). */
nb_status nb_comm_version(int32_t* version);

/* ---- hot path ------------------------------------------------------------- */
/* a1 encoder (R20).  NB_BF16: x_out is uint16 [n][16] bf16 bit
 * patterns (hi(0..d0-1), lo(0..d0-1), zeros); NB_FP32: x_out is fp32 [n][d0]
 * (identity).  The compute calls below encode in-kernel; this exposes the exact
 * layer-1 operand for parity.  NB_BF16 models with pe_depth = L > 0 (R42):
 * x_out is uint16 [n][64], the K = 64 positional-encoding operand the kernels
 * build (features gamma(x) in fp32, each split into a bf16 (hi, lo) pair:
 * hi at [0, d_in), lo at [32, 32 + d_in), zeros elsewhere; d_in = r (1 + L)).
 * NB_FP32 models with pe_depth > 0 return NB_E_UNSUPPORTED.                */
nb_status nb_encode(const nb_model* m, const float* q, int64_t n, void* x_out, void* stream);

/* a1-a4: logits[n][1 + n_heads] (output logit z, then head logits e_k), fp32;
 * prob (may be NULL): sigmoid(z) [n].                                */
nb_status nb_forward(const nb_model* m, const float* q, int64_t n, float* logits, float* prob,
                     void* stream);

/* a6: tau = min over labelled positives of the logit (and of each head logit),
 * stored in the model and copied to tau_out (host, 1 + n_heads floats).  With
 * these thresholds the predictor has FN = 0 on this set (BASELINE.json north
 * star; replaces the fixed eps = 1e-5 of P:772).  No positives: +inf, and
 * NB_E_NO_POSITIVES.  Under a communicator tau is the global minimum.       */
nb_status nb_calibrate(nb_model* m, const float* q, const uint8_t* y, int64_t n, float* tau_out,
                       void* stream);

/* Inverted ("certainly hit") bounding ("conservatively bounds
 * which spatial locations certainly are hit ... by flipping the asymmetry
 * weights"; train with the FP weight ramped instead of the FN weight):
 * tau = the next float above the maximum logit over labelled NEGATIVES, so
 * the predictor z >= tau has FP = 0 on this set (R43).  Models
 * without exit heads (NB_E_UNSUPPORTED otherwise); no negatives -> tau = +inf
 * and the warning-class NB_E_NO_POSITIVES.  nb_score then counts with it.   */
nb_status nb_calibrate_inverted(nb_model* m, const float* q, const uint8_t* y, int64_t n,
                                float* tau_out, void* stream);

/* a1-a5: fused forward + classify + count with the model's thresholds:
 * yhat = [e_1 >= tau_1] and [e_2 >= tau_2] and [z >= tau]; counts to *out (host).
 * Records with a non-finite logit are counted in out->nonfinite (a NaN never
 * passes z >= tau) and make the call return the warning-class NB_E_NONFINITE
 * with the counts written.                                                  */
nb_status nb_score(const nb_model* m, const float* q, const uint8_t* y, int64_t n,
                   nb_counts* out, void* stream);
/* Asynchronous nb_score: the same kernel, allreduce and counts, but the counts
 * are copied (cudaMemcpyAsync, cudaMemcpyDefault) to `out`, which must be
 * pinned host or device memory, when `stream` gets there; nothing synchronises.
 * Sticky in-kernel flags are reported by the next synchronising call.  The
 * model's counter scratch is reused, so calls on one model must be issued on
 * one stream (they serialise there).                                       */
nb_status nb_score_async(const nb_model* m, const float* q, const uint8_t* y, int64_t n,
                         nb_counts* out, void* stream);
/* Same as nb_score with HOST q/y (pinned or pageable): the library streams the
 * records to the device in chunks, overlapping copies with the fused kernel
 * (end-to-end serving path).                                              */
nb_status nb_score_host(const nb_model* m, const float* q_host, const uint8_t* y_host,
                        int64_t n, nb_counts* out, void* stream);

/* a1-a9: one Adam step on the loss of Eq. (1) over the local batch, normalised
 * by n_global (R4); alpha, beta are the FN / FP weights of the
 * current step (a10 schedule, nb_alpha); Adam (0.9, 0.999, 1e-8) with
 * learning rate lr.  stats may be NULL (no synchronisation).        */
nb_status nb_train_step(nb_model* m, const float* q, const uint8_t* y, int64_t n_local,
                        int64_t n_global, float alpha, float beta, float lr, nb_step_stats* stats,
                        void* stream);

/* a1-a9 over `steps` consecutive training steps in one call: step t uses rows
 * [t n_local, (t + 1) n_local) of q [steps n_local][d0] and y, the FN weight
 * alpha_t = alpha0 + (alpha1 - alpha0) t / (steps - 1) (a10's ramp over this
 * range), and beta, lr as nb_train_step.  Without a communicator the step
 * sequence is captured into a CUDA graph on a model-owned stream and
 * launched once (no per-launch gaps; the results equal `steps` nb_train_step
 * calls); with one, the steps are issued in stream order.  n_local must be a
 * multiple of 16 when steps > 1 (aligned batch views).  Asynchronous.      */
nb_status nb_train_steps(nb_model* m, const float* q, const uint8_t* y, int64_t n_local, int64_t n_global,
                         int32_t steps, float alpha0, float alpha1, float beta, float lr, void* stream);

/* a10: FN weight of step t of T: alpha_t = 1 + 999 t / (T - 1) (R6);
 * beta_t = 1.                                                               */
double nb_alpha(int64_t t, int64_t T);

/* ---- the paper's training control (Suppl.
 * §2.1-2.2; readings DESIGN.md R37-R39) --------------------------- */
/* L1 / L2 regularisation: every later nb_train_step's Adam adds
 * l1 sign(theta) + 2 l2 theta to the gradient (all parameters). >= 0.        */
nb_status nb_model_set_regularization(nb_model* m, float l1, float l2);

/* FN-gated step schedule.  Every step_every training steps ("every 10,000
 * iterations") the window's summed batch FN (nb_step_stats.fn) is
 * inspected: if it is not 0, the k-th such trigger lowers the FP weight beta
 * by base / k (base 1/20, 1/100, 1/200 for 2D, 3D, 4D, Suppl. §2.1's harmonic
 * decrements, floored at 1e-3) and raises the FN weight alpha by 0.2 (R37);
 * lambda (used for both l1 and l2) grows linearly from 0 to 5e-7 over
 * max_steps (Suppl. §2.2, R38); stop is set once 6 consecutive windows had
 * FN = 0 (R39) or max_steps steps were taken.  Host-only, no GPU.   */
typedef struct {
  int32_t space_dim;
  int32_t patience;        /* stable windows before stopping (6)             */
  int64_t step_every;      /* window length in steps (10,000 in the paper)   */
  int64_t max_steps;       /* iteration cap (lambda ramp length)             */
  double alpha, beta;      /* weights for the next nb_train_step             */
  double lambda;           /* regularisation weight for the next step        */
  int64_t step;            /* steps reported so far                          */
  int64_t triggers;        /* windows with FN > 0 so far                     */
  uint64_t window_fn;      /* FN summed over the current window              */
  int32_t stable;          /* consecutive windows with FN = 0                */
  int32_t stop;            /* early-stop / cap reached                       */
} nb_schedule;
nb_status nb_schedule_init(nb_schedule* s, int32_t space_dim, int64_t step_every, int64_t max_steps);
/* Report one finished step's batch FN; updates alpha, beta, lambda, stop.   */
nb_status nb_schedule_after_step(nb_schedule* s, uint64_t batch_fn);

/* ---- neural bounding hierarchies (§3.2) ------ */
/* Node i bounds the union of the indicators below it; parent[0] = -1 (root),
 * 0 <= parent[i] < i.  A record is predicted positive iff some root-to-leaf
 * path has every node predicting positive (each node's calibrated
 * predictor, exit heads included; R45).  Evaluated with pruning:
 * a node runs only on the rows its parent passed (gather -> the node's fused
 * forward -> compaction).  Writes tp/fp/fn/tn of that predictor against y
 * (exit_hist = 0) and in nonfinite the records with a non-finite logit at
 * some evaluated node (they fail that node; warning-class NB_E_NONFINITE
 * with the counts written).  All nodes on one device with the same record
 * layout, no communicator; n < 2^31.  The whole tree is enqueued without
 * host round trips and `stream` is synchronised once, at the end; scratch
 * is held by nodes[0] and reused (it grows only when a call needs more).  */
nb_status nb_hier_score(nb_model* const* nodes, int32_t n_nodes, const int32_t* parent, const float* q,
                        const uint8_t* y, int64_t n, nb_counts* out, void* stream);

/* ---- ground-truth labeller (harness support, not a hot-path row) ----------- */
/* Occupancy grid uint8 host array, row-major, axis 0 slowest; 4D grids are
 * [frames][R][R][R].  Builds a summed-area table on the device for boxes.   */
nb_status nb_grid_create(int32_t space_dim, int32_t R, int32_t frames, const uint8_t* host,
                         int32_t device, nb_grid** out);
void      nb_grid_destroy(nb_grid* g);
/* y[i] = g(record i) exactly: point lookup, fp64 DDA for rays, SAT for boxes,
 * fp64 voxel-corner cut test for planes (R15-R17, R19; g = any f
 * over the region).  Rays, planes (lines) and boxes: 2D, 3D and 4D
 * grids (4D: the space-time cells of [frames][R][R][R], R48).              */
nb_status nb_label(const nb_grid* g, int32_t kind, const float* q, int64_t n, uint8_t* y,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NB_H */
