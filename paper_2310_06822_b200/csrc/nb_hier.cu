// nb_hier.cu — neural bounding hierarchies (P:224-229
// §3.2: "stack our neural bounding volumes into hierarchies ... the tree's
// structure needs to be supplied by the user").
//
// Every node is an nb_model bounding the union of the indicators below it;
// a query is predicted positive iff some root-to-leaf path has every node
// predicting positive (each node's own calibrated predictor, exit heads
// included).  Evaluation prunes like a BVH: a node runs only on the rows its
// parent passed — the rows are gathered into a dense array, scored by the
// node's fused forward kernel, and the passing rows compacted into the
// node's survivor list; leaves mark their survivors.  Per-node row order is
// not fixed (warp-aggregated compaction), but each row's logits are computed
// independently, so the predicted set and the counts are exact.
#include <algorithm>
#include <vector>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

namespace {

__global__ void k_gather(const float* __restrict__ q, const int32_t* __restrict__ idx,
                         const unsigned long long* __restrict__ c_dev, int d0, float* __restrict__ out) {
  const int64_t c = (int64_t)*c_dev;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < c * d0;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d0;
    out[e] = q[(int64_t)idx[r] * d0 + e % d0];
  }
}

// rows of this node whose predictor passes: yhat = [e_1 >= tau_1][e_2 >= tau_2][z >= tau]
// (c_dev: row count written by the previous node's compaction; NULL -> c).
// A row with a non-finite evaluated logit fails (NaN never passes >=) and is
// flagged in nf[row] (R26), so the call can report it.
__global__ void k_compact(const float* __restrict__ logits, int nl, float t0, float t1, float t2,
                          const int32_t* __restrict__ idx_in, int64_t c, const unsigned long long* __restrict__ c_dev,
                          int32_t* __restrict__ idx_out, unsigned long long* __restrict__ count,
                          uint8_t* __restrict__ nf) {
  if (c_dev) c = (int64_t)*c_dev;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < c;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = base + lane;
    bool pass = false;
    int32_t row = 0;
    if (r < c) {
      const float* z = logits + r * nl;
      row = idx_in ? idx_in[r] : (int32_t)r;
      bool fin = isfinite(z[0]);
      for (int k = 1; k < nl; ++k) fin = fin && isfinite(z[k]);
      if (!fin) nf[row] = 1;
      pass = z[0] >= t0 && (nl < 2 || z[1] >= t1) && (nl < 3 || z[2] >= t2);
    }
    const uint32_t b = __ballot_sync(0xFFFFFFFFu, pass);
    unsigned long long off = 0;
    if (lane == 0 && b) off = atomicAdd(count, (unsigned long long)__popc(b));
    off = __shfl_sync(0xFFFFFFFFu, off, 0);
    if (pass) idx_out[off + __popc(b & ((1u << lane) - 1u))] = row;
  }
}

__global__ void k_mark(const int32_t* __restrict__ idx, const unsigned long long* __restrict__ c_dev,
                       uint8_t* __restrict__ flag) {
  const int64_t c = (int64_t)*c_dev;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < c; r += (int64_t)gridDim.x * blockDim.x)
    flag[idx[r]] = 1;
}

__global__ void k_hier_count(const uint8_t* __restrict__ flag, const uint8_t* __restrict__ nf,
                             const uint8_t* __restrict__ y, int64_t n, unsigned long long* __restrict__ counts) {
  uint32_t c[5] = {0, 0, 0, 0, 0};
  const int lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = base + lane;
    const bool v = r < n, p = v && flag[r], yy = v && y[r];
    c[0] += __popc(__ballot_sync(0xFFFFFFFFu, p && yy));
    c[1] += __popc(__ballot_sync(0xFFFFFFFFu, p && !yy));
    c[2] += __popc(__ballot_sync(0xFFFFFFFFu, v && !p && yy));
    c[3] += __popc(__ballot_sync(0xFFFFFFFFu, v && !p && !yy));
    c[4] += __popc(__ballot_sync(0xFFFFFFFFu, v && nf[r]));
  }
  if (lane == 0)
    for (int k = 0; k < 5; ++k)
      if (c[k]) atomicAdd(counts + k, (unsigned long long)c[k]);
}

unsigned grid_for(int64_t work) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8)); }

}  // namespace

// Every launch is sized for the upper bound n (survivor counts never leave
// the device: the node kernels read their row count from the previous
// node's compaction counter), so the whole tree is enqueued without a host
// round trip; forward(m, q, n_upper, n_dev, logits, st) is the node's fused
// forward reading its row count from n_dev (NULL: n_upper rows).
cudaError_t hier_score(nb_model* const* nodes, int n_nodes, const int32_t* parent, const float* q,
                       const uint8_t* y, int64_t n, unsigned long long* h_counts, cudaStream_t st,
                       cudaError_t (*forward)(const nb_model*, const float*, int64_t,
                                              const unsigned long long*, float*, cudaStream_t)) {
  const int d0 = nodes[0]->d0;
  int nlmax = 1;
  for (int i = 0; i < n_nodes; ++i) nlmax = std::max(nlmax, 1 + nodes[i]->d.n_heads);
  // scratch (every sub-buffer 256-B aligned: the node kernels bulk-copy records with TMA)
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t idx_bytes = up(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1));
  const size_t q_bytes = up(sizeof(float) * (size_t)n * d0), l_bytes = up(sizeof(float) * (size_t)n * nlmax);
  const size_t f_bytes = up((size_t)n + 1);
  const size_t bytes = idx_bytes * n_nodes + q_bytes + l_bytes + 2 * f_bytes + up(8 * (5 + (size_t)n_nodes));
  // the scratch lives on the root model and is reused by later calls; it only
  // grows (outside any steady state) when a call needs more
  nb_model* root = nodes[0];
  cudaError_t e = cudaSuccess;
  if (bytes > root->hier_scratch_bytes) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    cudaFree(root->hier_scratch);
    root->hier_scratch = nullptr;
    root->hier_scratch_bytes = 0;
    e = cudaMalloc(&root->hier_scratch, bytes);
    if (e != cudaSuccess) return e;
    root->hier_scratch_bytes = bytes;
  }
  uint8_t* base = (uint8_t*)root->hier_scratch;
  int32_t* idx = (int32_t*)base;
  float* qg = (float*)(base + idx_bytes * n_nodes);
  float* lg = (float*)((uint8_t*)qg + q_bytes);
  uint8_t* flag = (uint8_t*)lg + l_bytes;
  uint8_t* nf = flag + f_bytes;
  unsigned long long* cnt = (unsigned long long*)(nf + f_bytes);
  unsigned long long* node_cnt = cnt + 5;  // survivors per node
  e = cudaMemsetAsync(flag, 0, 2 * f_bytes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (5 + n_nodes), st);
  std::vector<char> is_leaf(n_nodes, 1);
  for (int i = 1; i < n_nodes; ++i) is_leaf[parent[i]] = 0;
  for (int i = 0; i < n_nodes && e == cudaSuccess && n > 0; ++i) {
    const nb_model* m = nodes[i];
    const int nl = 1 + m->d.n_heads;
    int32_t* out = idx + (size_t)i * (idx_bytes / 4);
    if (i == 0) {
      e = forward(m, q, n, nullptr, lg, st);
      if (e != cudaSuccess) break;
      k_compact<<<grid_for(n), 256, 0, st>>>(lg, nl, m->tau[0], m->tau[1], m->tau[2], nullptr, n, nullptr, out,
                                            node_cnt, nf);
    } else {
      const int32_t* in = idx + (size_t)parent[i] * (idx_bytes / 4);
      const unsigned long long* c_in = node_cnt + parent[i];
      k_gather<<<grid_for(n * d0), 256, 0, st>>>(q, in, c_in, d0, qg);
      e = forward(m, qg, n, c_in, lg, st);
      if (e != cudaSuccess) break;
      k_compact<<<grid_for(n), 256, 0, st>>>(lg, nl, m->tau[0], m->tau[1], m->tau[2], in, 0, c_in, out,
                                            node_cnt + i, nf);
    }
    if (is_leaf[i]) k_mark<<<grid_for(n), 256, 0, st>>>(out, node_cnt + i, flag);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && n > 0) k_hier_count<<<grid_for(n), 256, 0, st>>>(flag, nf, y, n, cnt);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h_counts, cnt, sizeof(unsigned long long) * 5, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace nb
