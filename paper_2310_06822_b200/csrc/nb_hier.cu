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
// node's survivor list; leaves mark their survivors (consecutive siblings
// share their parent's gather).  The compaction is
// order-preserving (two passes over fixed row chunks: survivor counts, then
// each chunk writes at the prefix of the counts before it), so every
// survivor list is ascending and the next node's gather reads the records in
// order; each row's logits are computed independently, so the predicted set
// and the counts are exact.  (A warp-aggregated atomic compaction cost 92 us
// per 2^22 rows: 131 K returning atomics on one counter.)
#include <algorithm>
#include <vector>

#include "nb_device.cuh"
#include "nb_internal.cuh"

namespace nb {

namespace {

// one thread per survivor row: its record is copied whole (the survivor list
// is ascending, so a warp reads records close together)
__global__ void k_gather(const float* __restrict__ q, const int32_t* __restrict__ idx,
                         const unsigned long long* __restrict__ c_dev, int d0, float* __restrict__ out) {
  const int64_t c = (int64_t)*c_dev;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < c; r += (int64_t)gridDim.x * blockDim.x) {
    const float* src = q + (int64_t)__ldg(idx + r) * d0;
    float* dst = out + r * d0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < d0) dst[j] = __ldg(src + j);
  }
}

// Order-preserving compaction, pass 1: survivors per chunk of kCmpRows rows
// (one block per chunk, 256 threads x 16 rows), non-finite rows flagged.
constexpr int kCmpThreads = 256, kCmpPer = 16, kCmpRows = kCmpThreads * kCmpPer;

__device__ __forceinline__ bool node_pass(const float* __restrict__ logits, int nl, float t0, float t1, float t2,
                                          int64_t r, bool* nonfin) {
  const float* z = logits + r * nl;
  bool fin = isfinite(z[0]);
  for (int k = 1; k < nl; ++k) fin = fin && isfinite(z[k]);
  *nonfin = !fin;
  return z[0] >= t0 && (nl < 2 || z[1] >= t1) && (nl < 3 || z[2] >= t2);
}

__global__ void __launch_bounds__(kCmpThreads) k_compact_count(
    const float* __restrict__ logits, int nl, float t0, float t1, float t2, const int32_t* __restrict__ idx_in,
    int64_t c, const unsigned long long* __restrict__ c_dev, uint32_t* __restrict__ chunk_cnt,
    uint8_t* __restrict__ nf) {
  if (c_dev) c = (int64_t)*c_dev;
  const int64_t chunk = blockIdx.x;
  if (chunk * kCmpRows >= c) return;
  __shared__ uint32_t wsum[kCmpThreads / 32];
  uint32_t cnt = 0;
#pragma unroll 4
  for (int i = 0; i < kCmpPer; ++i) {
    const int64_t r = chunk * kCmpRows + i * kCmpThreads + threadIdx.x;
    if (r < c) {
      bool nonfin;
      cnt += node_pass(logits, nl, t0, t1, t2, r, &nonfin) ? 1u : 0u;
      if (nonfin) nf[idx_in ? idx_in[r] : (int32_t)r] = 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCmpThreads / 32; ++w) t += wsum[w];
    chunk_cnt[chunk] = t;
  }
}

// pass 2: chunk `chunk` writes its survivors (ascending) from the sum of the
// counts of the chunks before it; the last chunk also writes the total.
__global__ void __launch_bounds__(kCmpThreads) k_compact_write(
    const float* __restrict__ logits, int nl, float t0, float t1, float t2, const int32_t* __restrict__ idx_in,
    int64_t c, const unsigned long long* __restrict__ c_dev, const uint32_t* __restrict__ chunk_cnt,
    int32_t* __restrict__ idx_out, unsigned long long* __restrict__ count) {
  if (c_dev) c = (int64_t)*c_dev;
  const int64_t chunk = blockIdx.x;
  const int64_t nchunks = (c + kCmpRows - 1) / kCmpRows;
  if (chunk >= nchunks) return;
  __shared__ uint32_t wsum[kCmpThreads / 32];
  __shared__ unsigned long long base_s;
  // exclusive prefix of the chunk counts (fixed order: deterministic)
  unsigned long long pre = 0;
  for (int64_t j = threadIdx.x; j < chunk; j += kCmpThreads) pre += chunk_cnt[j];
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
  __shared__ unsigned long long psum[kCmpThreads / 32];
  if ((threadIdx.x & 31) == 0) psum[threadIdx.x >> 5] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kCmpThreads / 32; ++w) t += psum[w];
    base_s = t;
    if (chunk == nchunks - 1) *count = t + chunk_cnt[chunk];
  }
  __syncthreads();
  unsigned long long run = base_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < kCmpPer; ++i) {
    const int64_t r = chunk * kCmpRows + i * kCmpThreads + threadIdx.x;
    bool pass = false;
    if (r < c) {
      bool nonfin;
      pass = node_pass(logits, nl, t0, t1, t2, r, &nonfin);
    }
    const uint32_t b = __ballot_sync(0xFFFFFFFFu, pass);
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    uint32_t below = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kCmpThreads / 32; ++w) {
      const uint32_t x = wsum[w];
      below += w < warp ? x : 0u;
      tot += x;
    }
    if (pass) idx_out[run + below + __popc(b & ((1u << lane) - 1u))] = idx_in ? idx_in[r] : (int32_t)r;
    run += tot;
    __syncthreads();  // wsum reused by the next row group
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
  const int64_t nchunks = std::max<int64_t>(1, (n + kCmpRows - 1) / kCmpRows);
  const size_t ch_bytes = up(sizeof(uint32_t) * (size_t)nchunks);
  const size_t bytes = idx_bytes * n_nodes + q_bytes + l_bytes + 2 * f_bytes + up(8 * (5 + (size_t)n_nodes)) + ch_bytes;
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
  uint32_t* chunk_cnt = (uint32_t*)((uint8_t*)cnt + up(8 * (5 + (size_t)n_nodes)));
  // order-preserving compaction of a node's logits into its survivor list
  auto compact = [&](const nb_model* m, const int32_t* in, int64_t c, const unsigned long long* c_dev,
                     int32_t* out, unsigned long long* count) {
    const int nl = 1 + m->d.n_heads;
    k_compact_count<<<(unsigned)nchunks, kCmpThreads, 0, st>>>(lg, nl, m->tau[0], m->tau[1], m->tau[2], in, c,
                                                                c_dev, chunk_cnt, nf);
    k_compact_write<<<(unsigned)nchunks, kCmpThreads, 0, st>>>(lg, nl, m->tau[0], m->tau[1], m->tau[2], in, c,
                                                                c_dev, chunk_cnt, out, count);
  };
  e = cudaMemsetAsync(flag, 0, 2 * f_bytes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (5 + n_nodes), st);
  std::vector<char> is_leaf(n_nodes, 1);
  for (int i = 1; i < n_nodes; ++i) is_leaf[parent[i]] = 0;
  int gathered = -1;  // the node whose survivors qg holds (siblings share one gather)
  for (int i = 0; i < n_nodes && e == cudaSuccess && n > 0; ++i) {
    const nb_model* m = nodes[i];
    const int nl = 1 + m->d.n_heads;
    int32_t* out = idx + (size_t)i * (idx_bytes / 4);
    if (i == 0) {
      e = forward(m, q, n, nullptr, lg, st);
      if (e != cudaSuccess) break;
      compact(m, nullptr, n, nullptr, out, node_cnt);
    } else {
      const int32_t* in = idx + (size_t)parent[i] * (idx_bytes / 4);
      const unsigned long long* c_in = node_cnt + parent[i];
      if (gathered != parent[i]) k_gather<<<grid_for(n), 256, 0, st>>>(q, in, c_in, d0, qg);
      gathered = parent[i];
      e = forward(m, qg, n, c_in, lg, st);
      if (e != cudaSuccess) break;
      compact(m, in, 0, c_in, out, node_cnt + i);
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
