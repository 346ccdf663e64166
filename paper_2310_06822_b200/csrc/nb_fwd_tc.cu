// nb_fwd_tc.cu — dispatcher of the fused tcgen05 forward kernels
// (nb_fwd_tc.cuh) and the generic instantiations (run-time d0, L, heads).
#include "nb_fwd_tc.cuh"

namespace nb {

bool tc_supported(const nb_desc& d) {
  if (d.precision != NB_BF16) return false;
  if (!(d.width == 32 || d.width == 64 || d.width == 128)) return false;
  if (d.hidden_layers < 1 || d.hidden_layers > kMaxLayers) return false;
  // layer-1 operand (hi, lo and bias columns) fits the slot's A region
  const int r = d.kind == NB_POINT ? d.space_dim : 2 * d.space_dim;
  if (d.pe_depth > 0)  // PE operand layout: d_in + 3 <= 32, K = 64 (PackLayout::pe_lo)
    return d.width >= 64 && r * (1 + d.pe_depth) + 3 <= 32;
  return enc_k(r) <= d.width;
}

// nb_encode of a positional-encoding net (R42): the K = 64 layer-1 operand of
// each record as the kernels build it (encode_cols_pe: fp32 sincospif
// features, bf16 hi / lo split; hi at [0, d_in), lo at [32, 32 + d_in)),
// with the three bias ones columns [d_in, d_in + 3) cleared — 64 bf16 per row.
template <int D0>
__global__ void k_encode_pe(const float* __restrict__ q, int64_t n, int pe, uint4* __restrict__ out) {
  const int din = D0 * (1 + pe);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = j < D0 ? q[i * D0 + j] : 0.f;
    uint32_t c[32];
    encode_cols_pe<D0>(x, pe, c);
#pragma unroll
    for (int k = 0; k < 32; ++k) {  // clear the bias ones (elements din .. din + 2)
      const bool lo_one = 2 * k >= din && 2 * k < din + 3, hi_one = 2 * k + 1 >= din && 2 * k + 1 < din + 3;
      c[k] &= (lo_one ? 0xFFFF0000u : 0xFFFFFFFFu) & (hi_one ? 0x0000FFFFu : 0xFFFFFFFFu);
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) out[8 * i + g] = make_uint4(c[4 * g], c[4 * g + 1], c[4 * g + 2], c[4 * g + 3]);
  }
}

cudaError_t launch_encode_pe(const nb_model* m, const float* q, int64_t n, void* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  switch (m->d0) {
    case 2: k_encode_pe<2><<<blocks, 256, 0, st>>>(q, n, m->d.pe_depth, (uint4*)out); break;
    case 3: k_encode_pe<3><<<blocks, 256, 0, st>>>(q, n, m->d.pe_depth, (uint4*)out); break;
    case 4: k_encode_pe<4><<<blocks, 256, 0, st>>>(q, n, m->d.pe_depth, (uint4*)out); break;
    case 6: k_encode_pe<6><<<blocks, 256, 0, st>>>(q, n, m->d.pe_depth, (uint4*)out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// NB_TRACE builds: device buffer set by nb_debug_set_trace (tools/trace_fwd.py).
unsigned long long* g_trace_buffer = nullptr;
static bool g_no_fold = false;
#ifdef NB_TRACE
extern "C" void nb_debug_set_trace(void* dev_buf) { g_trace_buffer = (unsigned long long*)dev_buf; }
#endif

// Specialised (fully unrolled, compile-time d0) kernels for the BASELINE.json
// architectures; every other architecture runs the generic instantiation
// (LC = 0, run-time d0, L and heads).  Both fold the biases into the MMAs
// whenever layer 1's K = 16 operand has room for them (2 d0 + 3 <= 16).
cudaError_t launch_fwd_tc(const nb_model* m, int mode, const FwdArgs& a, cudaStream_t st) {
  const nb_desc& d = m->d;
  const int h0 = d.n_heads > 0 ? d.head_after[0] : 0, h1 = d.n_heads > 1 ? d.head_after[1] : 0;
  const bool bf = m->pl.bias_l0 != 0;
  const bool plain = d.activation == NB_RELU && d.pe_depth == 0;  // specialised kernels: ReLU, no PE
  if (bf && plain && d.width == 64 && d.hidden_layers == 4 && d.n_heads == 0 && m->d0 == 3)
    return launch_tc_w64l4_d3(m, mode, a, st, !g_no_fold);
  if (bf && plain && d.width == 128 && d.hidden_layers == 4 && d.n_heads == 0 && m->d0 == 6)
    return launch_tc_w128l4_d6(m, mode, a, st, !g_no_fold);
  if (bf && plain && d.width == 128 && d.hidden_layers == 6 && h0 == 2 && h1 == 4 && m->d0 == 4)
    return launch_tc_w128l6h24_d4(m, mode, a, st, !g_no_fold);
  const bool fold = bf && !g_no_fold;
  switch (d.width) {
    case 32: return launch_tc_gen32(m, mode, a, st, fold);
    case 64: return launch_tc_gen64(m, mode, a, st, fold);
    case 128: return launch_tc_gen128(m, mode, a, st, fold);
  }
  return cudaErrorInvalidValue;
}

// Measurement switch (tools/quickbench.py NB_NO_FOLD=1): epilogue-bias kernels.
extern "C" void nb_debug_set_no_fold(int v) { g_no_fold = v != 0; }

}  // namespace nb
