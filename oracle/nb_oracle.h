/* nb_oracle.h — plain, slow CPU oracle for the Neural Bounding hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2310_06822_b200/csrc, include/nb.h) and never includes them.
 *
 * Every function follows PAPER.md (arXiv 2310.06822) step by step, in fp64
 * unless stated; citations are PAPER.md line numbers (P:n) with the section.
 * Readings of silent/ambiguous points are DESIGN.md §2 (R1..R36).
 *
 * Parity status of each function is listed in DESIGN.md §5; the only
 * "parity unpinned" item is a whole multi-step training trajectory.
 */
#ifndef NB_ORACLE_H
#define NB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Query kinds: parameterisations of Suppl. §3.2. */
enum { ORA_POINT = 0, ORA_RAY = 1, ORA_PLANE = 2, ORA_BOX = 3 };

/* Forward modes. */
enum { ORA_FP64 = 0,       /* the plain definition, fp64 throughout */
       ORA_BF16_EMU = 1 }; /* kernel-precision emulation for decisions (DESIGN.md §5 P4) */

typedef struct {
  int32_t d0;            /* input width = record floats (n, or 2n)        */
  int32_t width;         /* hidden width w                                */
  int32_t layers;        /* hidden layers L                               */
  int32_t n_heads;       /* early-exit heads (0..2), §3.3       */
  int32_t head_after[2]; /* 1-based hidden layer each head reads          */
  int32_t act;           /* 0 ReLU (BJ, R1); 1 sine h = sin(z) (R41) */
  int32_t pe;            /* positional-encoding depth L (Suppl. §3, R42) */
} ora_arch;

typedef struct { uint64_t tp, fp, fn, tn, exit_hist[4], nonfinite; } ora_counts;
typedef struct { double loss; uint64_t tp, fp, fn, tn; } ora_stats;

/* ---- indicator f and query function g (§3.1) ---------------- */
/* grid: uint8 occupancy, row-major, axis 0 slowest; for space_dim 4 the
 * layout is [frames][R][R][R] and t selects the frame (R15).              */
int  ora_indicator(const uint8_t* grid, int32_t space_dim, int32_t R, int32_t frames,
                   const double* x);
/* Exact labels y = g(r) for n records (R16-R19; 4D rays, hyperplanes and
 * boxes over the [frames][R][R][R] space-time cells, R48).  Returns 0 or -1. */
int  ora_label(const uint8_t* grid, int32_t space_dim, int32_t R, int32_t frames,
               int32_t kind, const float* q, int64_t n, uint8_t* y);
/* Independent brute-force labellers used only to pin ora_label. */
int  ora_label_brute(const uint8_t* grid, int32_t space_dim, int32_t R, int32_t frames,
                     int32_t kind, const float* q, int64_t n, uint8_t* y);
/* Summed-area table S[(R+1)^3], S[i][j][k] = sum of occ over i'<i,j'<j,k'<k. */
void ora_sat_build(const uint8_t* grid, int32_t R, int32_t* S);

/* ---- encoder a1 (R20) -------------------------------------------- */
/* bf16 hi/lo split: out[i][0..d0) = RNE_bf16(x), out[i][d0..2d0) = RNE_bf16(x - hi),
 * zero padded to 16 (bf16 bit patterns).                                   */
void ora_encode_bf16(const float* q, int64_t n, int32_t d0, uint16_t* out);
/* Positional-encoding operand (R42): fp64 gamma(x) -> fp32 -> bf16 (hi, lo),
 * hi at [0, d_in), lo at [32, 32 + d_in) of 64 columns per record.         */
void ora_encode_pe(const float* q, int64_t n, int32_t d0, int32_t pe, uint16_t* out);
uint16_t ora_bf16_rne(float x);

/* ---- MLP h_theta (§3.4; Suppl. Tab. 4) -------------------------- */
int64_t ora_num_params(const ora_arch* a);
/* logits[i][0] = output logit z, logits[i][1+k] = exit-head logit e_k. */
void ora_forward(const ora_arch* a, const double* theta, const float* q, int64_t n,
                 int32_t mode, double* logits);

/* ---- asymmetric loss, Eq. (1) P:189-204 / Alg. 1 P:207-222 --------------- */
/* Returns L-hat over the batch (normalised by n_global, R4) and accumulates
 * dL/dtheta into grad (zeroed by the callee).  stats: batch counts at z >= 0. */
double ora_loss_grad(const ora_arch* a, const double* theta, const float* q,
                     const uint8_t* y, int64_t n, int64_t n_global, double alpha,
                     double beta, double* grad, ora_stats* stats);
/* Same for the network evaluated in `mode` (ORA_BF16_EMU: gradient of the
 * bf16-precision forward of R33, the kernel's arithmetic). */
double ora_loss_grad_mode(const ora_arch* a, const double* theta, const float* q,
                          const uint8_t* y, int64_t n, int64_t n_global, double alpha,
                          double beta, double* grad, ora_stats* stats, int32_t mode);
/* Per-sample loss term only (for KATs): w * softplus(+-z). */
double ora_weighted_bce(double z, int32_t y, double alpha, double beta);

/* ---- Adam (§3.4; PyTorch semantics, R8) ----------------------------- */
void ora_adam(int64_t P, double* theta, double* m, double* v, int64_t t, double lr,
              double b1, double b2, double eps, const double* g);

/* ---- schedule alpha(t) (R6) ----------------------------------------------- */
double ora_alpha(int64_t t, int64_t T);

/* ---- calibrate / score (a5, a6) --------------------- */
/* tau[0] = min_{y=1} z, tau[1+k] = min_{y=1} e_k; +inf if no positives (ret 1). */
int  ora_calibrate(int32_t n_heads, const double* logits, const uint8_t* y, int64_t n,
                   double* tau);
void ora_score(int32_t n_heads, const double* logits, const uint8_t* y, int64_t n,
               const double* tau, ora_counts* out);

int  ora_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
