// nb_label.cu — ground-truth labeller on the GPU (harness support, not a
// hot-path row): y = g(record) = any f over the region,
// the exact readings of DESIGN.md R15-R17:
//   point: f(x) = grid[min(R-1, floor(x R))...], 0 outside [0,1]^n;
//   ray:   positive-length traversal of an occupied half-open voxel cell
//          (Amanatides-Woo in fp64);
//   box:   any occupied cell in [cell(lo), cell(hi)] via a summed-area table;
//   plane: any occupied voxel whose closed cube has corners on both closed
//          sides of n.(x - p0) = 0 (R19), corner values in fp64 exactly as the
//          oracle writes them; 8^3 blocks whose corners are all clearly on
//          one side (margin 1e-12) are skipped (a voxel cube lies inside its
//          block's cube, so only blocks without a cut voxel are pruned).
// This file is compiled with -fmad=false so every fp64 operation is rounded
// exactly as written (no FMA contraction).
#include <stdint.h>

#include <algorithm>

#include "nb_internal.cuh"

namespace nb {

__device__ __forceinline__ int cell_of(double x, int R) {
  long long i = (long long)floor(x * (double)R);
  return (int)(i > R - 1 ? R - 1 : i);
}

__device__ int label_point(const nb_grid g, const float* r) {
  const int sd = g.space_dim;
  for (int j = 0; j < sd; ++j) {
    double v = (double)r[j];
    if (!(v >= 0.0 && v <= 1.0)) return 0;
  }
  const int R = g.R;
  if (sd == 2) return g.occ[(size_t)cell_of(r[0], R) * R + cell_of(r[1], R)] != 0;
  size_t idx = ((size_t)cell_of(r[0], R) * R + cell_of(r[1], R)) * R + cell_of(r[2], R);
  if (sd == 4) idx += (size_t)cell_of(r[3], g.frames) * R * R * R;
  return g.occ[idx] != 0;
}

__device__ int label_ray(const nb_grid g, const float* r) {
  const int R = g.R;
  double o[3] = {r[0], r[1], r[2]}, d[3] = {r[3], r[4], r[5]};
  // clip the half-line s >= 0 to the closed unit cube (slab test)
  double s0 = 0.0, s1 = INFINITY;
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0) {
      if (o[a] < 0.0 || o[a] > 1.0) return 0;
    } else {
      double ta = (0.0 - o[a]) / d[a], tb = (1.0 - o[a]) / d[a];
      double lo = ta < tb ? ta : tb, hi = ta < tb ? tb : ta;
      s0 = lo > s0 ? lo : s0;
      s1 = hi < s1 ? hi : s1;
    }
  }
  if (!(s1 > s0)) return 0;
  int cell[3], dir[3];
  double next[3];
  for (int a = 0; a < 3; ++a) {
    const double xr = (o[a] + s0 * d[a]) * (double)R;
    long long c = (long long)floor(xr);
    if (d[a] < 0.0 && (double)c == xr) c -= 1;  // entering downward through a face
    c = c < 0 ? 0 : (c > R - 1 ? R - 1 : c);
    cell[a] = (int)c;
    dir[a] = d[a] > 0.0 ? 1 : (d[a] < 0.0 ? -1 : 0);
    if (dir[a] > 0) next[a] = ((double)(cell[a] + 1) / (double)R - o[a]) / d[a];
    else if (dir[a] < 0) next[a] = ((double)cell[a] / (double)R - o[a]) / d[a];
    else next[a] = INFINITY;
  }
  double s = s0;
  while (true) {
    const int a = (next[0] <= next[1]) ? ((next[0] <= next[2]) ? 0 : 2)
                                       : ((next[1] <= next[2]) ? 1 : 2);
    const double e = next[a] < s1 ? next[a] : s1;
    if (e > s && g.occ[((size_t)cell[0] * R + cell[1]) * R + cell[2]]) return 1;
    if (!(next[a] < s1)) return 0;
    s = e;
    cell[a] += dir[a];
    if (cell[a] < 0 || cell[a] >= R) return 0;
    next[a] = (dir[a] > 0 ? ((double)(cell[a] + 1) / (double)R - o[a])
                          : ((double)cell[a] / (double)R - o[a])) / d[a];
  }
}

__device__ int label_box(const nb_grid g, const float* r) {
  const int R = g.R;
  int a[3], b[3];
  for (int j = 0; j < 3; ++j) {
    double lo = r[j], hi = r[3 + j];
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > 1.0 ? 1.0 : hi;
    if (!(hi >= lo)) return 0;
    a[j] = cell_of(lo, R);
    b[j] = cell_of(hi, R) + 1;
  }
  const size_t R1 = (size_t)R + 1;
  auto S = [&](int i, int j, int k) -> long long { return g.sat[((size_t)i * R1 + j) * R1 + k]; };
  long long c = S(b[0], b[1], b[2]) - S(a[0], b[1], b[2]) - S(b[0], a[1], b[2]) -
                S(b[0], b[1], a[2]) + S(a[0], a[1], b[2]) + S(a[0], b[1], a[2]) +
                S(b[0], a[1], a[2]) - S(a[0], a[1], a[2]);
  return c > 0;
}

__device__ int label_plane(const nb_grid g, const float* r) {
  const int R = g.R, NB = (R + 7) / 8;
  const double p0[3] = {r[0], r[1], r[2]}, nrm[3] = {r[3], r[4], r[5]};
  auto sval = [&](int i, int j, int k) {
    const double x = (double)i / R - p0[0];
    const double y = (double)j / R - p0[1];
    const double z = (double)k / R - p0[2];
    return nrm[0] * x + nrm[1] * y + nrm[2] * z;
  };
  for (int bi = 0; bi < NB; ++bi)
    for (int bj = 0; bj < NB; ++bj)
      for (int bk = 0; bk < NB; ++bk) {
        if (!g.blk[((size_t)bi * NB + bj) * NB + bk]) continue;
        const int i0 = 8 * bi, j0 = 8 * bj, k0 = 8 * bk;
        const int i1 = min(R, i0 + 8), j1 = min(R, j0 + 8), k1 = min(R, k0 + 8);
        double mn = INFINITY, mx = -INFINITY;
        for (int c = 0; c < 8; ++c) {
          const double v = sval((c & 4) ? i1 : i0, (c & 2) ? j1 : j0, (c & 1) ? k1 : k0);
          mn = v < mn ? v : mn;
          mx = v > mx ? v : mx;
        }
        if (mn > 1e-12 || mx < -1e-12) continue;
        for (int i = i0; i < i1; ++i)
          for (int j = j0; j < j1; ++j)
            for (int k = k0; k < k1; ++k) {
              if (!g.occ[((size_t)i * R + j) * R + k]) continue;
              int neg = 0, pos = 0;
              for (int c = 0; c < 8; ++c) {
                const double s = sval(i + ((c >> 2) & 1), j + ((c >> 1) & 1), k + (c & 1));
                if (s <= 0.0) neg = 1;
                if (s >= 0.0) pos = 1;
              }
              if (neg && pos) return 1;
            }
      }
  return 0;
}

// ---- 2D rays, boxes and lines (pixel readings; the same fp64 expressions as
// the oracle's ray2_dda / box2_sat / line2_scan_res)
__device__ int label_ray2(const nb_grid g, const float* r) {
  const int R = g.R;
  const double o[2] = {r[0], r[1]}, d[2] = {r[2], r[3]};
  double s0 = 0.0, s1 = INFINITY;
  for (int a = 0; a < 2; ++a) {
    if (d[a] == 0.0) {
      if (o[a] < 0.0 || o[a] > 1.0) return 0;
    } else {
      double ta = (0.0 - o[a]) / d[a], tb = (1.0 - o[a]) / d[a];
      double lo = ta < tb ? ta : tb, hi = ta < tb ? tb : ta;
      s0 = lo > s0 ? lo : s0;
      s1 = hi < s1 ? hi : s1;
    }
  }
  if (!(s1 > s0)) return 0;
  int cell[2], dir[2];
  double next[2];
  for (int a = 0; a < 2; ++a) {
    const double xr = (o[a] + s0 * d[a]) * (double)R;
    long long c = (long long)floor(xr);
    if (d[a] < 0.0 && (double)c == xr) c -= 1;
    c = c < 0 ? 0 : (c > R - 1 ? R - 1 : c);
    cell[a] = (int)c;
    dir[a] = d[a] > 0.0 ? 1 : (d[a] < 0.0 ? -1 : 0);
    if (dir[a] > 0) next[a] = ((double)(cell[a] + 1) / (double)R - o[a]) / d[a];
    else if (dir[a] < 0) next[a] = ((double)cell[a] / (double)R - o[a]) / d[a];
    else next[a] = INFINITY;
  }
  double s = s0;
  while (true) {
    const int a = next[1] < next[0] ? 1 : 0;
    const double e = next[a] < s1 ? next[a] : s1;
    if (e > s && g.occ[(size_t)cell[0] * R + cell[1]]) return 1;
    if (!(next[a] < s1)) return 0;
    s = e;
    cell[a] += dir[a];
    if (cell[a] < 0 || cell[a] >= R) return 0;
    next[a] = (dir[a] > 0 ? ((double)(cell[a] + 1) / (double)R - o[a])
                          : ((double)cell[a] / (double)R - o[a])) / d[a];
  }
}

__device__ int label_box2(const nb_grid g, const float* r) {
  const int R = g.R;
  int a[2], b[2];
  for (int j = 0; j < 2; ++j) {
    double lo = r[j], hi = r[2 + j];
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > 1.0 ? 1.0 : hi;
    if (!(hi >= lo)) return 0;
    a[j] = cell_of(lo, R);
    b[j] = cell_of(hi, R) + 1;
  }
  const size_t R1 = (size_t)R + 1;
  auto S = [&](int i, int j) -> long long { return g.sat[(size_t)i * R1 + j]; };
  return (S(b[0], b[1]) - S(a[0], b[1]) - S(b[0], a[1]) + S(a[0], a[1])) > 0;
}

__device__ int label_line2(const nb_grid g, const float* r) {
  const int R = g.R;
  const double p0[2] = {r[0], r[1]}, nrm[2] = {r[2], r[3]};
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      if (!g.occ[(size_t)i * R + j]) continue;
      int neg = 0, pos = 0;
      for (int c = 0; c < 4; ++c) {
        const double x = (double)(i + ((c >> 1) & 1)) / ((double)1 * R) - p0[0];
        const double y = (double)(j + (c & 1)) / ((double)1 * R) - p0[1];
        const double sv = nrm[0] * x + nrm[1] * y;
        if (sv <= 0.0) neg = 1;
        if (sv >= 0.0) pos = 1;
      }
      if (neg && pos) return 1;
    }
  return 0;
}


// ---- 4D (space x time) rays, hyperplanes and boxes (R48; the oracle's
// ray4_dda / box4_sat / plane4_scan_res expressions): cells of the
// [F][R][R][R] grid over (x, y, z, t), axis resolution R, R, R, F.
__device__ __forceinline__ int res4(const nb_grid& g, int ax) { return ax < 3 ? g.R : g.frames; }
__device__ __forceinline__ size_t cell4(const nb_grid& g, const int* c) {
  return (((size_t)c[3] * g.R + c[0]) * g.R + c[1]) * g.R + c[2];
}

__device__ int label_ray4(const nb_grid g, const float* r) {
  double o[4], d[4];
  for (int j = 0; j < 4; ++j) {
    o[j] = r[j];
    d[j] = r[4 + j];
  }
  double a0 = 0.0, b0 = INFINITY;
  for (int j = 0; j < 4; ++j) {
    if (d[j] == 0.0) {
      if (o[j] < 0.0 || o[j] > 1.0) return 0;
      continue;
    }
    double t0 = (0.0 - o[j]) / d[j], t1 = (1.0 - o[j]) / d[j];
    if (t0 > t1) { const double t = t0; t0 = t1; t1 = t; }
    if (t0 > a0) a0 = t0;
    if (t1 < b0) b0 = t1;
  }
  if (!(b0 > a0)) return 0;
  const double s_in = a0, s_out = b0;
  int idx[4], step[4];
  double tmax[4];
  for (int j = 0; j < 4; ++j) {
    const int Rj = res4(g, j);
    const double p = o[j] + s_in * d[j];
    const double pr = p * (double)Rj;
    long long i = (long long)floor(pr);
    if ((double)i == pr && d[j] < 0.0) i -= 1;
    if (i < 0) i = 0;
    if (i > Rj - 1) i = Rj - 1;
    idx[j] = (int)i;
    if (d[j] > 0.0) {
      step[j] = 1;
      tmax[j] = ((double)(idx[j] + 1) / (double)Rj - o[j]) / d[j];
    } else if (d[j] < 0.0) {
      step[j] = -1;
      tmax[j] = ((double)idx[j] / (double)Rj - o[j]) / d[j];
    } else {
      step[j] = 0;
      tmax[j] = INFINITY;
    }
  }
  double s = s_in;
  for (;;) {
    int a = 0;
    for (int j = 1; j < 4; ++j)
      if (tmax[j] < tmax[a]) a = j;
    const double s_next = tmax[a] < s_out ? tmax[a] : s_out;
    if (s_next > s && g.occ[cell4(g, idx)]) return 1;
    if (tmax[a] >= s_out) return 0;
    s = s_next;
    idx[a] += step[a];
    const int Ra = res4(g, a);
    if (idx[a] < 0 || idx[a] >= Ra) return 0;
    tmax[a] = (step[a] > 0 ? ((double)(idx[a] + 1) / (double)Ra - o[a]) : ((double)idx[a] / (double)Ra - o[a])) / d[a];
  }
}

__device__ int label_box4(const nb_grid g, const float* r) {
  int a[4], b[4];
  for (int j = 0; j < 4; ++j) {
    double lo = r[j], hi = r[4 + j];
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > 1.0 ? 1.0 : hi;
    if (!(hi >= lo)) return 0;
    a[j] = cell_of(lo, res4(g, j));
    b[j] = cell_of(hi, res4(g, j)) + 1;
  }
  const size_t R1 = (size_t)g.R + 1;
  long long cnt = 0;
  for (int c = 0; c < 16; ++c) {
    int id[4], sign = 1;
    for (int ax = 0; ax < 4; ++ax) {
      if ((c >> ax) & 1) id[ax] = b[ax];
      else { id[ax] = a[ax]; sign = -sign; }
    }
    cnt += sign * (long long)g.sat[(((size_t)id[3] * R1 + id[0]) * R1 + id[1]) * R1 + id[2]];
  }
  return cnt > 0;
}

// hyperplane cut test over occupied cells; 8^3 x 8-frame blocks whose corners
// are all clearly on one side (margin 1e-12) are skipped (g.blk flags)
__device__ int label_plane4(const nb_grid g, const float* r) {
  const int R = g.R, F = g.frames, NB = (R + 7) / 8, NT = (F + 7) / 8;
  double p0[4], nrm[4];
  for (int j = 0; j < 4; ++j) {
    p0[j] = r[j];
    nrm[j] = r[4 + j];
  }
  auto sval = [&](const int* c) {
    double s = 0.0;
    for (int ax = 0; ax < 4; ++ax) {
      const double x = (double)c[ax] / (double)res4(g, ax) - p0[ax];
      s += nrm[ax] * x;
    }
    return s;
  };
  for (int bt = 0; bt < NT; ++bt)
    for (int bi = 0; bi < NB; ++bi)
      for (int bj = 0; bj < NB; ++bj)
        for (int bk = 0; bk < NB; ++bk) {
          if (!g.blk[(((size_t)bt * NB + bi) * NB + bj) * NB + bk]) continue;
          const int lo[4] = {8 * bi, 8 * bj, 8 * bk, 8 * bt};
          const int hi[4] = {min(R, lo[0] + 8), min(R, lo[1] + 8), min(R, lo[2] + 8), min(F, lo[3] + 8)};
          double mn = INFINITY, mx = -INFINITY;
          for (int c = 0; c < 16; ++c) {
            int cc[4];
            for (int ax = 0; ax < 4; ++ax) cc[ax] = ((c >> ax) & 1) ? hi[ax] : lo[ax];
            const double v = sval(cc);
            mn = v < mn ? v : mn;
            mx = v > mx ? v : mx;
          }
          if (mn > 1e-12 || mx < -1e-12) continue;
          int c4[4];
          for (c4[3] = lo[3]; c4[3] < hi[3]; ++c4[3])
            for (c4[0] = lo[0]; c4[0] < hi[0]; ++c4[0])
              for (c4[1] = lo[1]; c4[1] < hi[1]; ++c4[1])
                for (c4[2] = lo[2]; c4[2] < hi[2]; ++c4[2]) {
                  if (!g.occ[cell4(g, c4)]) continue;
                  int neg = 0, pos = 0;
                  for (int k = 0; k < 16; ++k) {
                    int cc[4];
                    for (int ax = 0; ax < 4; ++ax) cc[ax] = c4[ax] + ((k >> ax) & 1);
                    const double sv = sval(cc);
                    if (sv <= 0.0) neg = 1;
                    if (sv >= 0.0) pos = 1;
                  }
                  if (neg && pos) return 1;
                }
        }
  return 0;
}

__global__ void k_label(const nb_grid g, int kind, const float* __restrict__ q, int64_t n,
                        uint8_t* __restrict__ y) {
  const int nf = kind == NB_POINT ? g.space_dim : 2 * g.space_dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float r[8];
    for (int j = 0; j < nf; ++j) r[j] = q[i * nf + j];
    int v = 0;
    if (kind == NB_POINT) v = label_point(g, r);
    else if (g.space_dim == 4) v = kind == NB_RAY ? label_ray4(g, r) : (kind == NB_BOX ? label_box4(g, r) : label_plane4(g, r));
    else if (g.space_dim == 2) v = kind == NB_RAY ? label_ray2(g, r) : (kind == NB_BOX ? label_box2(g, r) : label_line2(g, r));
    else if (kind == NB_RAY) v = label_ray(g, r);
    else if (kind == NB_PLANE) v = label_plane(g, r);
    else v = label_box(g, r);
    y[i] = (uint8_t)v;
  }
}

__global__ void k_blk_build(const uint8_t* __restrict__ occ, int R, uint8_t* __restrict__ blk) {
  const int NB = (R + 7) / 8;
  const size_t nb3 = (size_t)NB * NB * NB;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nb3;
       b += (size_t)gridDim.x * blockDim.x) {
    const int bi = (int)(b / ((size_t)NB * NB)), bj = (int)((b / NB) % NB), bk = (int)(b % NB);
    uint8_t any = 0;
    for (int i = 8 * bi; i < min(R, 8 * bi + 8); ++i)
      for (int j = 8 * bj; j < min(R, 8 * bj + 8); ++j)
        for (int k = 8 * bk; k < min(R, 8 * bk + 8); ++k) any |= occ[((size_t)i * R + j) * R + k];
    blk[b] = any ? 1 : 0;
  }
}

cudaError_t launch_blk_build(nb_grid* g, cudaStream_t s) {
  const int NB = (g->R + 7) / 8;
  const size_t nb3 = (size_t)NB * NB * NB;
  cudaError_t e = cudaMalloc((void**)&g->blk, nb3);
  if (e != cudaSuccess) return e;
  k_blk_build<<<(unsigned)std::min<size_t>((nb3 + 255) / 256, 4096), 256, 0, s>>>(g->occ, g->R, g->blk);
  return cudaGetLastError();
}

__global__ void k_sat2(const uint8_t* __restrict__ occ, int R, int32_t* __restrict__ S) {
  // one thread per row prefix, then per column: (R+1)^2 table with a zero border
  const size_t R1 = (size_t)R + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= R; i += gridDim.x * blockDim.x) {
    int32_t acc = 0;
    S[(size_t)i * R1] = 0;
    for (int j = 1; j <= R; ++j) {
      if (i > 0) acc += occ[(size_t)(i - 1) * R + (j - 1)];
      S[(size_t)i * R1 + j] = acc;
    }
  }
}
__global__ void k_sat2_cols(int R, int32_t* __restrict__ S) {
  const size_t R1 = (size_t)R + 1;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= R; j += gridDim.x * blockDim.x)
    for (int i = 1; i <= R; ++i) S[(size_t)i * R1 + j] += S[(size_t)(i - 1) * R1 + j];
}

cudaError_t launch_sat2_build(nb_grid* g, cudaStream_t s) {
  const int R = g->R;
  cudaError_t e = cudaMalloc((void**)&g->sat, sizeof(int32_t) * (size_t)(R + 1) * (R + 1));
  if (e != cudaSuccess) return e;
  k_sat2<<<(R + 256) / 256, 256, 0, s>>>(g->occ, R, g->sat);
  k_sat2_cols<<<(R + 256) / 256, 256, 0, s>>>(R, g->sat);
  return cudaGetLastError();
}

cudaError_t launch_label(const nb_grid* g, int kind, const float* q, int64_t n, uint8_t* y,
                         cudaStream_t s) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_label<<<blocks, 256, 0, s>>>(*g, kind, q, n, y);
  return cudaGetLastError();
}

// Summed-area table: three prefix-sum passes, one per axis, over (R+1)^3 with a
// zero border.  S[i][j][k] = number of occupied cells (i' < i, j' < j, k' < k).
__global__ void k_sat_init(const uint8_t* __restrict__ occ, int R, int32_t* __restrict__ S) {
  const size_t R1 = (size_t)R + 1, tot = R1 * R1 * R1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < tot;
       t += (size_t)gridDim.x * blockDim.x) {
    int k = (int)(t % R1), j = (int)((t / R1) % R1), i = (int)(t / (R1 * R1));
    S[t] = (i && j && k) ? occ[((size_t)(i - 1) * R + (j - 1)) * R + (k - 1)] : 0;
  }
}

__global__ void k_sat_scan(int R, int axis, int32_t* __restrict__ S) {
  const size_t R1 = (size_t)R + 1;
  const size_t lines = R1 * R1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < lines;
       t += (size_t)gridDim.x * blockDim.x) {
    size_t u = t / R1, v = t % R1, base, stride;
    if (axis == 0) { base = u * R1 + v; stride = R1 * R1; }
    else if (axis == 1) { base = u * R1 * R1 + v; stride = R1; }
    else { base = (u * R1 + v) * R1; stride = 1; }
    int32_t acc = 0;
    for (size_t i = 0; i < R1; ++i) {
      acc += S[base + i * stride];
      S[base + i * stride] = acc;
    }
  }
}

// 4D summed-area table over (t, x, y, z): (F+1) (R+1)^3 with a zero border,
// built by one prefix pass per axis (the oracle's sat4_build order of sums is
// irrelevant: integer sums are exact).
__global__ void k_sat4_init(const uint8_t* __restrict__ occ, int R, int F, int32_t* __restrict__ S) {
  const size_t R1 = (size_t)R + 1, tot = (size_t)(F + 1) * R1 * R1 * R1;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < tot; t += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(t % R1), j = (int)((t / R1) % R1), i = (int)((t / (R1 * R1)) % R1);
    const int f = (int)(t / (R1 * R1 * R1));
    S[t] = (f && i && j && k) ? occ[(((size_t)(f - 1) * R + (i - 1)) * R + (j - 1)) * R + (k - 1)] : 0;
  }
}
__global__ void k_sat4_scan(int R, int F, int axis, int32_t* __restrict__ S) {
  const size_t R1 = (size_t)R + 1, F1 = (size_t)F + 1;
  const size_t len = axis == 0 ? F1 : R1;
  const size_t stride = axis == 0 ? R1 * R1 * R1 : (axis == 1 ? R1 * R1 : (axis == 2 ? R1 : 1));
  const size_t lines = F1 * R1 * R1 * R1 / len;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < lines; t += (size_t)gridDim.x * blockDim.x) {
    // decompose t over the other three axes (outer index, inner index by stride)
    const size_t inner = t % stride, outer = t / stride;
    const size_t base = outer * stride * len + inner;
    int32_t acc = 0;
    for (size_t i = 0; i < len; ++i) {
      acc += S[base + i * stride];
      S[base + i * stride] = acc;
    }
  }
}
__global__ void k_blk4_build(const uint8_t* __restrict__ occ, int R, int F, uint8_t* __restrict__ blk) {
  const int NB = (R + 7) / 8, NT = (F + 7) / 8;
  const size_t nb = (size_t)NT * NB * NB * NB;
  for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nb; b += (size_t)gridDim.x * blockDim.x) {
    const int bk = (int)(b % NB), bj = (int)((b / NB) % NB), bi = (int)((b / ((size_t)NB * NB)) % NB);
    const int bt = (int)(b / ((size_t)NB * NB * NB));
    uint8_t any = 0;
    for (int f = 8 * bt; f < min(F, 8 * bt + 8); ++f)
      for (int i = 8 * bi; i < min(R, 8 * bi + 8); ++i)
        for (int j = 8 * bj; j < min(R, 8 * bj + 8); ++j)
          for (int k = 8 * bk; k < min(R, 8 * bk + 8); ++k) any |= occ[(((size_t)f * R + i) * R + j) * R + k];
    blk[b] = any ? 1 : 0;
  }
}
cudaError_t launch_grid4_build(nb_grid* g, cudaStream_t s) {
  const int R = g->R, F = g->frames;
  const size_t R1 = (size_t)R + 1;
  cudaError_t e = cudaMalloc((void**)&g->sat, sizeof(int32_t) * (size_t)(F + 1) * R1 * R1 * R1);
  if (e != cudaSuccess) return e;
  k_sat4_init<<<2048, 256, 0, s>>>(g->occ, R, F, g->sat);
  for (int ax = 0; ax < 4; ++ax) k_sat4_scan<<<512, 128, 0, s>>>(R, F, ax, g->sat);
  const int NB = (R + 7) / 8, NT = (F + 7) / 8;
  const size_t nb = (size_t)NT * NB * NB * NB;
  e = cudaMalloc((void**)&g->blk, nb);
  if (e != cudaSuccess) return e;
  k_blk4_build<<<(unsigned)std::min<size_t>((nb + 255) / 256, 4096), 256, 0, s>>>(g->occ, R, F, g->blk);
  return cudaGetLastError();
}

cudaError_t launch_sat_build(nb_grid* g, cudaStream_t s) {
  k_sat_init<<<1024, 256, 0, s>>>(g->occ, g->R, g->sat);
  for (int ax = 0; ax < 3; ++ax) k_sat_scan<<<256, 128, 0, s>>>(g->R, ax, g->sat);
  return cudaGetLastError();
}

}  // namespace nb
