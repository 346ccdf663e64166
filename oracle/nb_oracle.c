/* nb_oracle.c — plain, slow CPU oracle (TEST INFRASTRUCTURE, see nb_oracle.h).
 *
 * Built with: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 * No blocking, fusion or reordering beyond the paper's definitions: every
 * loop below is the definition written out, one query at a time.
 */
#include "nb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int ora_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Indicator f (§3.1): 1 inside/on the object, 0 elsewhere.
 * Grid voxels are half-open cells [i/R,(i+1)/R); the closed upper face x=1
 * belongs to the last cell; outside [0,1]^n f = 0 (reading R15).           */
static int cell_index(double x, int32_t R) {
  int64_t i = (int64_t)floor(x * (double)R);
  if (i > R - 1) i = R - 1;
  return (int)i;
}

int ora_indicator(const uint8_t* grid, int32_t space_dim, int32_t R, int32_t frames,
                  const double* x) {
  for (int j = 0; j < space_dim; ++j)
    if (!(x[j] >= 0.0 && x[j] <= 1.0)) return 0;
  if (space_dim == 2) {
    int i0 = cell_index(x[0], R), i1 = cell_index(x[1], R);
    return grid[(int64_t)i0 * R + i1] != 0;
  }
  if (space_dim == 3) {
    int i0 = cell_index(x[0], R), i1 = cell_index(x[1], R), i2 = cell_index(x[2], R);
    return grid[((int64_t)i0 * R + i1) * R + i2] != 0;
  }
  /* 4D: (x, y, z, t), frame = min(F-1, floor(t F)) */
  int fr = cell_index(x[3], frames);
  int i0 = cell_index(x[0], R), i1 = cell_index(x[1], R), i2 = cell_index(x[2], R);
  return grid[(((int64_t)fr * R + i0) * R + i1) * R + i2] != 0;
}

static int occ3(const uint8_t* g, int32_t R, int i, int j, int k) {
  return g[((int64_t)i * R + j) * R + k] != 0;
}

/* ------------------------------------------------------------------------ */
/* Ray query (reading R16): g = 1 iff the half-line o + s d, s >= 0, has a
 * positive-length piece inside some occupied (half-open, R15) voxel cell of
 * [0,1]^3, i.e. g = max of f over the ray up to measure-zero touches.     */
static int ray_clip(const double* o, const double* d, double* s_in, double* s_out) {
  double a = 0.0, b = INFINITY;
  for (int j = 0; j < 3; ++j) {
    if (d[j] == 0.0) {
      if (o[j] < 0.0 || o[j] > 1.0) return 0;
      continue;
    }
    double t0 = (0.0 - o[j]) / d[j], t1 = (1.0 - o[j]) / d[j];
    if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
    if (t0 > a) a = t0;
    if (t1 < b) b = t1;
  }
  *s_in = a; *s_out = b;
  return b > a;
}

/* Amanatides-Woo voxel traversal in fp64 between s_in and s_out. */
static int ray_dda(const uint8_t* g, int32_t R, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray_clip(o, d, &s_in, &s_out)) return 0;
  int idx[3], step[3];
  double tmax[3];
  for (int j = 0; j < 3; ++j) {
    double p = o[j] + s_in * d[j];
    double pr = p * (double)R;
    int64_t i = (int64_t)floor(pr);
    if ((double)i == pr && d[j] < 0.0) i -= 1; /* on a face, moving down */
    if (i < 0) i = 0;
    if (i > R - 1) i = R - 1;
    idx[j] = (int)i;
    if (d[j] > 0.0) {
      step[j] = 1;
      tmax[j] = ((double)(idx[j] + 1) / (double)R - o[j]) / d[j];
    } else if (d[j] < 0.0) {
      step[j] = -1;
      tmax[j] = ((double)idx[j] / (double)R - o[j]) / d[j];
    } else {
      step[j] = 0;
      tmax[j] = INFINITY;
    }
  }
  double s = s_in;
  for (;;) {
    int a = 0;
    if (tmax[1] < tmax[a]) a = 1;
    if (tmax[2] < tmax[a]) a = 2;
    double s_next = tmax[a] < s_out ? tmax[a] : s_out;
    if (s_next > s && occ3(g, R, idx[0], idx[1], idx[2])) return 1;
    if (tmax[a] >= s_out) return 0;
    s = s_next;
    idx[a] += step[a];
    if (idx[a] < 0 || idx[a] >= R) return 0;
    tmax[a] = (step[a] > 0 ? ((double)(idx[a] + 1) / (double)R - o[a])
                           : ((double)idx[a] / (double)R - o[a])) / d[a];
  }
}

/* Brute force: test every occupied voxel against the ray; along an axis with
 * d = 0 the ray lies in the half-open cell of its constant coordinate.   */
static int ray_brute(const uint8_t* g, int32_t R, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray_clip(o, d, &s_in, &s_out)) return 0;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j)
      for (int k = 0; k < R; ++k) {
        if (!occ3(g, R, i, j, k)) continue;
        int c[3] = {i, j, k};
        double a = s_in, b = s_out;
        int ok = 1;
        for (int ax = 0; ax < 3 && ok; ++ax) {
          double lo = (double)c[ax] / (double)R, hi = (double)(c[ax] + 1) / (double)R;
          if (d[ax] == 0.0) { /* constant coordinate: its half-open cell (R15) */
            if (cell_index(o[ax], R) != c[ax]) ok = 0;
            continue;
          }
          double t0 = (lo - o[ax]) / d[ax], t1 = (hi - o[ax]) / d[ax];
          if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
          if (t0 > a) a = t0;
          if (t1 < b) b = t1;
        }
        if (ok && b > a) return 1;
      }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Box query (reading R17): g = max f over the closed box [lo, hi]; with the
 * floor-cell indicator the touched cells are [cell(lo), cell(hi)] per axis. */
void ora_sat_build(const uint8_t* grid, int32_t R, int32_t* S) {
  int64_t R1 = R + 1;
  memset(S, 0, sizeof(int32_t) * R1 * R1 * R1);
  for (int i = 1; i <= R; ++i)
    for (int j = 1; j <= R; ++j)
      for (int k = 1; k <= R; ++k) {
        int32_t v = occ3(grid, R, i - 1, j - 1, k - 1);
        S[(i * R1 + j) * R1 + k] = v + S[((i - 1) * R1 + j) * R1 + k] +
                                   S[(i * R1 + (j - 1)) * R1 + k] + S[(i * R1 + j) * R1 + (k - 1)] -
                                   S[((i - 1) * R1 + (j - 1)) * R1 + k] -
                                   S[((i - 1) * R1 + j) * R1 + (k - 1)] -
                                   S[(i * R1 + (j - 1)) * R1 + (k - 1)] +
                                   S[((i - 1) * R1 + (j - 1)) * R1 + (k - 1)];
      }
}

static int box_cells(const double* lo, const double* hi, int32_t R, int* a, int* b) {
  for (int j = 0; j < 3; ++j) {
    double l = lo[j] < 0.0 ? 0.0 : lo[j];
    double h = hi[j] > 1.0 ? 1.0 : hi[j];
    if (!(h >= l)) return 0; /* empty (or outside) */
    a[j] = cell_index(l, R);
    b[j] = cell_index(h, R);
  }
  return 1;
}

static int box_sat(const int32_t* S, int32_t R, const double* lo, const double* hi) {
  int a[3], b[3];
  if (!box_cells(lo, hi, R, a, b)) return 0;
  int64_t R1 = R + 1;
#define SAT(i, j, k) ((int64_t)S[((int64_t)(i) * R1 + (j)) * R1 + (k)])
  int64_t i0 = a[0], i1 = b[0] + 1, j0 = a[1], j1 = b[1] + 1, k0 = a[2], k1 = b[2] + 1;
  int64_t cnt = SAT(i1, j1, k1) - SAT(i0, j1, k1) - SAT(i1, j0, k1) - SAT(i1, j1, k0) +
                SAT(i0, j0, k1) + SAT(i0, j1, k0) + SAT(i1, j0, k0) - SAT(i0, j0, k0);
#undef SAT
  return cnt > 0;
}

static int box_scan(const uint8_t* g, int32_t R, const double* lo, const double* hi) {
  int a[3], b[3];
  if (!box_cells(lo, hi, R, a, b)) return 0;
  for (int i = a[0]; i <= b[0]; ++i)
    for (int j = a[1]; j <= b[1]; ++j)
      for (int k = a[2]; k <= b[2]; ++k)
        if (occ3(g, R, i, j, k)) return 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Plane query (reading R19): g = 1 iff the plane n.(x - p0) = 0 meets the
 * closed cube of some occupied voxel (corners on both closed sides).      */
static int plane_scan(const uint8_t* g, int32_t R, const double* p0, const double* nrm) {
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j)
      for (int k = 0; k < R; ++k) {
        if (!occ3(g, R, i, j, k)) continue;
        int neg = 0, pos = 0;
        for (int c = 0; c < 8; ++c) {
          double x = (double)(i + ((c >> 2) & 1)) / R - p0[0];
          double y = (double)(j + ((c >> 1) & 1)) / R - p0[1];
          double z = (double)(k + (c & 1)) / R - p0[2];
          double s = nrm[0] * x + nrm[1] * y + nrm[2] * z;
          if (s <= 0.0) neg = 1;
          if (s >= 0.0) pos = 1;
        }
        if (neg && pos) return 1;
      }
  return 0;
}

/* Brute-force plane: the same cut test on every voxel of a finer
 * (2x) subdivision restricted to occupied parents: a parent cube is cut iff
 * one of its 8 children is cut (convexity), an independent evaluation.   */
static int plane_brute(const uint8_t* g, int32_t R, const double* p0, const double* nrm) {
  for (int i = 0; i < 2 * R; ++i)
    for (int j = 0; j < 2 * R; ++j)
      for (int k = 0; k < 2 * R; ++k) {
        if (!occ3(g, R, i / 2, j / 2, k / 2)) continue;
        int neg = 0, pos = 0;
        for (int c = 0; c < 8; ++c) {
          double x = (double)(i + ((c >> 2) & 1)) / (2.0 * R) - p0[0];
          double y = (double)(j + ((c >> 1) & 1)) / (2.0 * R) - p0[1];
          double z = (double)(k + (c & 1)) / (2.0 * R) - p0[2];
          double s = nrm[0] * x + nrm[1] * y + nrm[2] * z;
          if (s <= 0.0) neg = 1;
          if (s >= 0.0) pos = 1;
        }
        if (neg && pos) return 1;
      }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* 2D rays, boxes and lines: the readings R15-R19 with
 * pixels instead of voxels; grid [R][R], axis 0 slowest.                  */
static int occ2(const uint8_t* g, int32_t R, int i, int j) { return g[(int64_t)i * R + j] != 0; }

static int ray2_clip(const double* o, const double* d, double* s_in, double* s_out) {
  double a = 0.0, b = INFINITY;
  for (int j = 0; j < 2; ++j) {
    if (d[j] == 0.0) {
      if (o[j] < 0.0 || o[j] > 1.0) return 0;
      continue;
    }
    double t0 = (0.0 - o[j]) / d[j], t1 = (1.0 - o[j]) / d[j];
    if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
    if (t0 > a) a = t0;
    if (t1 < b) b = t1;
  }
  *s_in = a; *s_out = b;
  return b > a;
}

static int ray2_dda(const uint8_t* g, int32_t R, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray2_clip(o, d, &s_in, &s_out)) return 0;
  int idx[2], step[2];
  double tmax[2];
  for (int j = 0; j < 2; ++j) {
    double pr = (o[j] + s_in * d[j]) * (double)R;
    int64_t i = (int64_t)floor(pr);
    if ((double)i == pr && d[j] < 0.0) i -= 1;
    if (i < 0) i = 0;
    if (i > R - 1) i = R - 1;
    idx[j] = (int)i;
    if (d[j] > 0.0) { step[j] = 1; tmax[j] = ((double)(idx[j] + 1) / (double)R - o[j]) / d[j]; }
    else if (d[j] < 0.0) { step[j] = -1; tmax[j] = ((double)idx[j] / (double)R - o[j]) / d[j]; }
    else { step[j] = 0; tmax[j] = INFINITY; }
  }
  double s = s_in;
  for (;;) {
    int a = tmax[1] < tmax[0] ? 1 : 0;
    double s_next = tmax[a] < s_out ? tmax[a] : s_out;
    if (s_next > s && occ2(g, R, idx[0], idx[1])) return 1;
    if (tmax[a] >= s_out) return 0;
    s = s_next;
    idx[a] += step[a];
    if (idx[a] < 0 || idx[a] >= R) return 0;
    tmax[a] = (step[a] > 0 ? ((double)(idx[a] + 1) / (double)R - o[a])
                           : ((double)idx[a] / (double)R - o[a])) / d[a];
  }
}

static int ray2_brute(const uint8_t* g, int32_t R, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray2_clip(o, d, &s_in, &s_out)) return 0;
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      if (!occ2(g, R, i, j)) continue;
      int c[2] = {i, j};
      double a = s_in, b = s_out;
      int ok = 1;
      for (int ax = 0; ax < 2 && ok; ++ax) {
        double lo = (double)c[ax] / (double)R, hi = (double)(c[ax] + 1) / (double)R;
        if (d[ax] == 0.0) {
          if (cell_index(o[ax], R) != c[ax]) ok = 0;
          continue;
        }
        double t0 = (lo - o[ax]) / d[ax], t1 = (hi - o[ax]) / d[ax];
        if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
        if (t0 > a) a = t0;
        if (t1 < b) b = t1;
      }
      if (ok && b > a) return 1;
    }
  return 0;
}

static int box2_cells(const double* lo, const double* hi, int32_t R, int* a, int* b) {
  for (int j = 0; j < 2; ++j) {
    double l = lo[j] < 0.0 ? 0.0 : lo[j];
    double h = hi[j] > 1.0 ? 1.0 : hi[j];
    if (!(h >= l)) return 0;
    a[j] = cell_index(l, R);
    b[j] = cell_index(h, R);
  }
  return 1;
}

/* 2D summed-area table S[i][j] = occupied pixels (i' < i, j' < j). */
static void sat2_build(const uint8_t* g, int32_t R, int32_t* S) {
  const int64_t R1 = R + 1;
  memset(S, 0, sizeof(int32_t) * R1 * R1);
  for (int i = 1; i <= R; ++i)
    for (int j = 1; j <= R; ++j)
      S[i * R1 + j] = occ2(g, R, i - 1, j - 1) + S[(i - 1) * R1 + j] + S[i * R1 + j - 1] -
                      S[(i - 1) * R1 + j - 1];
}

static int box2_sat(const int32_t* S, int32_t R, const double* lo, const double* hi) {
  int a[2], b[2];
  if (!box2_cells(lo, hi, R, a, b)) return 0;
  const int64_t R1 = R + 1, i0 = a[0], i1 = b[0] + 1, j0 = a[1], j1 = b[1] + 1;
  return (S[i1 * R1 + j1] - S[i0 * R1 + j1] - S[i1 * R1 + j0] + S[i0 * R1 + j0]) > 0;
}

static int box2_scan(const uint8_t* g, int32_t R, const double* lo, const double* hi) {
  int a[2], b[2];
  if (!box2_cells(lo, hi, R, a, b)) return 0;
  for (int i = a[0]; i <= b[0]; ++i)
    for (int j = a[1]; j <= b[1]; ++j)
      if (occ2(g, R, i, j)) return 1;
  return 0;
}

/* line n.(x - p0) = 0 meets the closed square of an occupied pixel: its
 * corners lie on both closed sides (R19 in 2D).                           */
static int line2_scan_res(const uint8_t* g, int32_t R, int sub, const double* p0, const double* nrm) {
  for (int i = 0; i < sub * R; ++i)
    for (int j = 0; j < sub * R; ++j) {
      if (!occ2(g, R, i / sub, j / sub)) continue;
      int neg = 0, pos = 0;
      for (int c = 0; c < 4; ++c) {
        double x = (double)(i + ((c >> 1) & 1)) / ((double)sub * R) - p0[0];
        double y = (double)(j + (c & 1)) / ((double)sub * R) - p0[1];
        double sv = nrm[0] * x + nrm[1] * y;
        if (sv <= 0.0) neg = 1;
        if (sv >= 0.0) pos = 1;
      }
      if (neg && pos) return 1;
    }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* 4D (space x time) rays, hyperplanes and boxes (
 * Suppl. Tab. 4/5 "4D Ray, Plane, Box"; "pairs of Cartesian
 * nD start- and direction-vectors ... corners ... p0 and normal").
 * Reading R48: coordinates (x, y, z, t) in [0,1]^4, cells are the half-open
 * space-time cells [i/R,(i+1)/R) x ... x [f/F,(f+1)/F) of the [F][R][R][R]
 * grid (the 4D point indicator's cells, R15 per axis); R16, R17 and R19
 * carry over with 4 axes.                                                 */
static int res4(int32_t R, int32_t F, int ax) { return ax < 3 ? R : F; }

static int occ4(const uint8_t* g, int32_t R, const int* c) { /* c = (x, y, z, t) cell */
  return g[(((int64_t)c[3] * R + c[0]) * R + c[1]) * R + c[2]] != 0;
}

static int ray4_clip(const double* o, const double* d, double* s_in, double* s_out) {
  double a = 0.0, b = INFINITY;
  for (int j = 0; j < 4; ++j) {
    if (d[j] == 0.0) {
      if (o[j] < 0.0 || o[j] > 1.0) return 0;
      continue;
    }
    double t0 = (0.0 - o[j]) / d[j], t1 = (1.0 - o[j]) / d[j];
    if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
    if (t0 > a) a = t0;
    if (t1 < b) b = t1;
  }
  *s_in = a; *s_out = b;
  return b > a;
}

/* Amanatides-Woo traversal over 4 axes (axis resolution R, R, R, F). */
static int ray4_dda(const uint8_t* g, int32_t R, int32_t F, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray4_clip(o, d, &s_in, &s_out)) return 0;
  int idx[4], step[4];
  double tmax[4];
  for (int j = 0; j < 4; ++j) {
    const int Rj = res4(R, F, j);
    double p = o[j] + s_in * d[j];
    double pr = p * (double)Rj;
    int64_t i = (int64_t)floor(pr);
    if ((double)i == pr && d[j] < 0.0) i -= 1; /* on a face, moving down */
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
    double s_next = tmax[a] < s_out ? tmax[a] : s_out;
    if (s_next > s && occ4(g, R, idx)) return 1;
    if (tmax[a] >= s_out) return 0;
    s = s_next;
    idx[a] += step[a];
    const int Ra = res4(R, F, a);
    if (idx[a] < 0 || idx[a] >= Ra) return 0;
    tmax[a] = (step[a] > 0 ? ((double)(idx[a] + 1) / (double)Ra - o[a])
                           : ((double)idx[a] / (double)Ra - o[a])) / d[a];
  }
}

/* Brute force: slab test of the ray against every occupied cell. */
static int ray4_brute(const uint8_t* g, int32_t R, int32_t F, const double* o, const double* d) {
  double s_in, s_out;
  if (!ray4_clip(o, d, &s_in, &s_out)) return 0;
  int c[4];
  for (c[3] = 0; c[3] < F; ++c[3])
    for (c[0] = 0; c[0] < R; ++c[0])
      for (c[1] = 0; c[1] < R; ++c[1])
        for (c[2] = 0; c[2] < R; ++c[2]) {
          if (!occ4(g, R, c)) continue;
          double a = s_in, b = s_out;
          int ok = 1;
          for (int ax = 0; ax < 4 && ok; ++ax) {
            const int Ra = res4(R, F, ax);
            double lo = (double)c[ax] / (double)Ra, hi = (double)(c[ax] + 1) / (double)Ra;
            if (d[ax] == 0.0) { /* constant coordinate: its half-open cell (R15) */
              if (cell_index(o[ax], Ra) != c[ax]) ok = 0;
              continue;
            }
            double t0 = (lo - o[ax]) / d[ax], t1 = (hi - o[ax]) / d[ax];
            if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
            if (t0 > a) a = t0;
            if (t1 < b) b = t1;
          }
          if (ok && b > a) return 1;
        }
  return 0;
}

static int box4_cells(const double* lo, const double* hi, int32_t R, int32_t F, int* a, int* b) {
  for (int j = 0; j < 4; ++j) {
    double l = lo[j] < 0.0 ? 0.0 : lo[j];
    double h = hi[j] > 1.0 ? 1.0 : hi[j];
    if (!(h >= l)) return 0;
    a[j] = cell_index(l, res4(R, F, j));
    b[j] = cell_index(h, res4(R, F, j));
  }
  return 1;
}

/* 4D summed-area table S[(F+1)][(R+1)^3] over (t, x, y, z): S[f][i][j][k] =
 * number of occupied cells with t-cell < f, x-cell < i, y-cell < j, z-cell < k,
 * built one axis at a time (prefix sums along x, y, z, then t).          */
static int32_t* sat4_build(const uint8_t* g, int32_t R, int32_t F) {
  const int64_t R1 = R + 1, F1 = F + 1;
  int32_t* S = (int32_t*)calloc((size_t)(F1 * R1 * R1 * R1), sizeof(int32_t));
#define S4(f, i, j, k) S[(((int64_t)(f) * R1 + (i)) * R1 + (j)) * R1 + (k)]
  for (int f = 1; f <= F; ++f)
    for (int i = 1; i <= R; ++i)
      for (int j = 1; j <= R; ++j)
        for (int k = 1; k <= R; ++k) {
          const int c[4] = {i - 1, j - 1, k - 1, f - 1};
          S4(f, i, j, k) = occ4(g, R, c);
        }
  for (int f = 1; f <= F; ++f) /* prefix along z, y, x within each frame */
    for (int i = 1; i <= R; ++i)
      for (int j = 1; j <= R; ++j)
        for (int k = 1; k <= R; ++k) S4(f, i, j, k) += S4(f, i, j, k - 1);
  for (int f = 1; f <= F; ++f)
    for (int i = 1; i <= R; ++i)
      for (int j = 1; j <= R; ++j)
        for (int k = 1; k <= R; ++k) S4(f, i, j, k) += S4(f, i, j - 1, k);
  for (int f = 1; f <= F; ++f)
    for (int i = 1; i <= R; ++i)
      for (int j = 1; j <= R; ++j)
        for (int k = 1; k <= R; ++k) S4(f, i, j, k) += S4(f, i - 1, j, k);
  for (int f = 1; f <= F; ++f) /* then along t */
    for (int i = 1; i <= R; ++i)
      for (int j = 1; j <= R; ++j)
        for (int k = 1; k <= R; ++k) S4(f, i, j, k) += S4(f - 1, i, j, k);
#undef S4
  return S;
}

/* Inclusion-exclusion over the 16 corners of [a, b] (cells inclusive). */
static int box4_sat(const int32_t* S, int32_t R, int32_t F, const double* lo, const double* hi) {
  int a[4], b[4];
  if (!box4_cells(lo, hi, R, F, a, b)) return 0;
  const int64_t R1 = R + 1;
  int64_t cnt = 0;
  for (int c = 0; c < 16; ++c) {
    int idx[4], sign = 1;
    for (int ax = 0; ax < 4; ++ax) {
      if ((c >> ax) & 1) idx[ax] = b[ax] + 1;
      else { idx[ax] = a[ax]; sign = -sign; }
    }
    cnt += sign * (int64_t)S[(((int64_t)idx[3] * R1 + idx[0]) * R1 + idx[1]) * R1 + idx[2]];
  }
  return cnt > 0;
}

static int box4_scan(const uint8_t* g, int32_t R, int32_t F, const double* lo, const double* hi) {
  int a[4], b[4], c[4];
  if (!box4_cells(lo, hi, R, F, a, b)) return 0;
  for (c[3] = a[3]; c[3] <= b[3]; ++c[3])
    for (c[0] = a[0]; c[0] <= b[0]; ++c[0])
      for (c[1] = a[1]; c[1] <= b[1]; ++c[1])
        for (c[2] = a[2]; c[2] <= b[2]; ++c[2])
          if (occ4(g, R, c)) return 1;
  return 0;
}

/* Hyperplane n.(x - p0) = 0 against the closed 4D cell boxes at subdivision
 * `sub` (1: the cells themselves; 2: each cell split in 2^4 children, an
 * independent evaluation of the same predicate by convexity).            */
static int plane4_scan_res(const uint8_t* g, int32_t R, int32_t F, int sub, const double* p0,
                           const double* nrm) {
  int c[4];
  for (c[3] = 0; c[3] < F * sub; ++c[3])
    for (c[0] = 0; c[0] < R * sub; ++c[0])
      for (c[1] = 0; c[1] < R * sub; ++c[1])
        for (c[2] = 0; c[2] < R * sub; ++c[2]) {
          const int pc[4] = {c[0] / sub, c[1] / sub, c[2] / sub, c[3] / sub};
          if (!occ4(g, R, pc)) continue;
          int neg = 0, pos = 0;
          for (int k = 0; k < 16; ++k) {
            double s = 0.0;
            for (int ax = 0; ax < 4; ++ax) {
              const double x = (double)(c[ax] + ((k >> ax) & 1)) / ((double)res4(R, F, ax) * sub) - p0[ax];
              s += nrm[ax] * x;
            }
            if (s <= 0.0) neg = 1;
            if (s >= 0.0) pos = 1;
          }
          if (neg && pos) return 1;
        }
  return 0;
}

static int label_one(const uint8_t* grid, int32_t sd, int32_t R, int32_t frames, int32_t kind,
                     const float* r, const int32_t* S, int brute) {
  double v[8];
  int nf = (kind == ORA_POINT) ? sd : 2 * sd;
  for (int j = 0; j < nf; ++j) v[j] = (double)r[j];
  if (sd == 4 && kind != ORA_POINT) {
    switch (kind) {
      case ORA_RAY: return brute ? ray4_brute(grid, R, frames, v, v + 4) : ray4_dda(grid, R, frames, v, v + 4);
      case ORA_BOX: return brute ? box4_scan(grid, R, frames, v, v + 4) : box4_sat(S, R, frames, v, v + 4);
      case ORA_PLANE: return plane4_scan_res(grid, R, frames, brute ? 2 : 1, v, v + 4);
    }
    return 0;
  }
  if (sd == 2 && kind != ORA_POINT) {
    switch (kind) {
      case ORA_RAY: return brute ? ray2_brute(grid, R, v, v + 2) : ray2_dda(grid, R, v, v + 2);
      case ORA_BOX: return brute ? box2_scan(grid, R, v, v + 2) : box2_sat(S, R, v, v + 2);
      case ORA_PLANE: return line2_scan_res(grid, R, brute ? 2 : 1, v, v + 2);
    }
    return 0;
  }
  switch (kind) {
    case ORA_POINT: return ora_indicator(grid, sd, R, frames, v);
    case ORA_RAY: return brute ? ray_brute(grid, R, v, v + 3) : ray_dda(grid, R, v, v + 3);
    case ORA_BOX: return brute ? box_scan(grid, R, v, v + 3) : box_sat(S, R, v, v + 3);
    case ORA_PLANE: return brute ? plane_brute(grid, R, v, v + 3) : plane_scan(grid, R, v, v + 3);
  }
  return 0;
}

static int label_impl(const uint8_t* grid, int32_t sd, int32_t R, int32_t frames, int32_t kind,
                      const float* q, int64_t n, uint8_t* y, int brute) {
  if (kind == ORA_POINT && !(sd >= 2 && sd <= 4)) return -1;
  if (kind != ORA_POINT && !(sd >= 2 && sd <= 4)) return -1;
  int nf = (kind == ORA_POINT) ? sd : 2 * sd;
  int32_t* S = NULL;
  if (kind == ORA_BOX && !brute && sd == 4) {
    S = sat4_build(grid, R, frames);
  } else if (kind == ORA_BOX && !brute && sd == 3) {
    S = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R + 1) * (R + 1) * (R + 1));
    ora_sat_build(grid, R, S);
  } else if (kind == ORA_BOX && !brute) {
    S = (int32_t*)malloc(sizeof(int32_t) * (size_t)(R + 1) * (R + 1));
    sat2_build(grid, R, S);
  }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i)
    y[i] = (uint8_t)label_one(grid, sd, R, frames, kind, q + i * nf, S, brute);
  free(S);
  return 0;
}

int ora_label(const uint8_t* grid, int32_t sd, int32_t R, int32_t frames, int32_t kind,
              const float* q, int64_t n, uint8_t* y) {
  return label_impl(grid, sd, R, frames, kind, q, n, y, 0);
}

int ora_label_brute(const uint8_t* grid, int32_t sd, int32_t R, int32_t frames, int32_t kind,
                    const float* q, int64_t n, uint8_t* y) {
  return label_impl(grid, sd, R, frames, kind, q, n, y, 1);
}

/* ------------------------------------------------------------------------ */
/* bf16 round-to-nearest-even of an fp32 value (bit manipulation).         */
uint16_t ora_bf16_rne(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static float bf16_to_f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static float bf16_round(float x) { return bf16_to_f(ora_bf16_rne(x)); }

/* Encoder a1 (R20): each fp32 coordinate becomes the pair (hi, lo) of bf16
 * values with hi = RNE(x), lo = RNE(x - hi); x - hi is exact in fp32.     */
void ora_encode_bf16(const float* q, int64_t n, int32_t d0, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint16_t* o = out + i * 16;
    for (int j = 0; j < 16; ++j) o[j] = 0;
    for (int j = 0; j < d0; ++j) {
      float x = q[i * d0 + j];
      uint16_t hi = ora_bf16_rne(x);
      float r = x - bf16_to_f(hi);
      o[j] = hi;
      o[d0 + j] = ora_bf16_rne(r);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Input of layer 1 (Suppl. §3, NeRF positional encoding; R42):
 * gamma(x) = (x_1..x_r, then for k = 0 .. L/2-1: sin(2^k pi x_1..r),
 * cos(2^k pi x_1..r)), L = pe; "2D point * 8 encodings, plus the 2D input"
 * = 18 values for r = 2, L = 8.  pe = 0: the record itself.              */
static int input_dim(const ora_arch* a) { return a->d0 * (1 + a->pe); }

static void positional_encoding(const ora_arch* a, const float* r, double* f) {
  const int d = a->d0;
  for (int j = 0; j < d; ++j) f[j] = (double)r[j];
  for (int k = 0; k < a->pe / 2; ++k)
    for (int j = 0; j < d; ++j) {
      const double u = ldexp(3.14159265358979323846, k) * (double)r[j];
      f[d + 2 * k * d + j] = sin(u);
      f[d + (2 * k + 1) * d + j] = cos(u);
    }
}

/* Hidden activation sigma and its derivative: ReLU (R1, R25: ReLU'(0) = 0) or
 * sine with frequency 1 ("Sinusoidal activations"; R41).            */
/* The K = 64 bf16 operand of a PE net (R42, R20): each fp64 feature of
 * gamma(x) rounded to fp32, then split into the bf16 pair hi = RNE(f),
 * lo = RNE(f - hi); hi at [0, d_in), lo at [32, 32 + d_in), zeros elsewhere. */
void ora_encode_pe(const float* q, int64_t n, int32_t d0, int32_t pe, uint16_t* out) {
  ora_arch a;
  memset(&a, 0, sizeof(a));
  a.d0 = d0;
  a.pe = pe;
  const int din = input_dim(&a);
  double f[64];
  for (int64_t i = 0; i < n; ++i) {
    uint16_t* o = out + i * 64;
    for (int j = 0; j < 64; ++j) o[j] = 0;
    positional_encoding(&a, q + i * d0, f);
    for (int j = 0; j < din && j < 32; ++j) {
      const float x = (float)f[j];
      const uint16_t hi = ora_bf16_rne(x);
      o[j] = hi;
      o[32 + j] = ora_bf16_rne(x - bf16_to_f(hi));
    }
  }
}

static double act_fn(const ora_arch* a, double z) { return a->act ? sin(z) : (z > 0.0 ? z : 0.0); }
static double act_grad(const ora_arch* a, double z) { return a->act ? cos(z) : (z > 0.0 ? 1.0 : 0.0); }

/* MLP h_theta (§3.4): h_0 = gamma(x); z_l = W_l h_{l-1} + b_l;
 * h_l = sigma(z_l); z = w_out . h_L + b_out; yhat = sigmoid(z).
 * Exit heads (§3.3, R22): e_k = u_k . h_{l_k} + c_k.
 * Canonical parameter blob (R32): per hidden layer W_l[out][in] then b_l;
 * then w_out[w], b_out; then per head u_k[w], c_k.                       */
int64_t ora_num_params(const ora_arch* a) {
  int64_t n = 0, in = input_dim(a);
  for (int l = 0; l < a->layers; ++l) {
    n += (in + 1) * (int64_t)a->width;
    in = a->width;
  }
  n += a->width + 1;
  n += (int64_t)a->n_heads * (a->width + 1);
  return n;
}

typedef struct { int64_t W[16], b[16], wout, bout, u[2], c[2]; } offsets;

static void param_offsets(const ora_arch* a, offsets* o) {
  int64_t p = 0, in = input_dim(a);
  for (int l = 0; l < a->layers; ++l) {
    o->W[l] = p; p += in * a->width;
    o->b[l] = p; p += a->width;
    in = a->width;
  }
  o->wout = p; p += a->width;
  o->bout = p; p += 1;
  for (int k = 0; k < a->n_heads; ++k) {
    o->u[k] = p; p += a->width;
    o->c[k] = p; p += 1;
  }
}

static int head_at(const ora_arch* a, int l1) { /* head index reading hidden layer l1 (1-based) */
  for (int k = 0; k < a->n_heads; ++k)
    if (a->head_after[k] == l1) return k;
  return -1;
}

/* One query forward.  acts (optional, fp64 mode): h_0..h_L stored as
 * [L+1][max(d_in,w)] and pre-activations z_1..z_L as [L][w].             */
static void forward_one(const ora_arch* a, const offsets* of, const double* th, const float* r,
                        int mode, double* out, double* acts, double* pre) {
  const int w = a->width, L = a->layers, d0 = input_dim(a);
  const int stride = (d0 > w ? d0 : w);
  double hbuf[2][512];
  double* h = hbuf[0];
  double* hn = hbuf[1];
  positional_encoding(a, r, h);
  if (mode == ORA_BF16_EMU) {  /* fp32 feature -> bf16 (hi, lo) pair (R20) */
    for (int j = 0; j < d0; ++j) {
      float x = (float)h[j];
      float hi = bf16_round(x);
      float lo = bf16_round(x - hi);
      h[j] = (double)hi + (double)lo;
    }
  }
  if (acts) for (int j = 0; j < d0; ++j) acts[j] = h[j];
  int in = d0;
  for (int l = 0; l < L; ++l) {
    const double* W = th + of->W[l];
    const double* b = th + of->b[l];
    double rl[512]; /* post-ReLU values before any bf16 rounding */
    for (int o = 0; o < w; ++o) {
      double s = 0.0;
      for (int k = 0; k < in; ++k) {
        double wk = W[(int64_t)o * in + k];
        if (mode == ORA_BF16_EMU) wk = (double)bf16_round((float)wk);
        s += wk * h[k];
      }
      if (mode == ORA_BF16_EMU) {
        float z = (float)s + (float)b[o];
        float rr = (float)act_fn(a, (double)z);
        if (pre) pre[(int64_t)l * w + o] = (double)z;
        rl[o] = rr;
        hn[o] = (l < L - 1) ? (double)bf16_round(rr) : (double)rr;
      } else {
        double z = s + b[o];
        if (pre) pre[(int64_t)l * w + o] = z;
        rl[o] = act_fn(a, z);
        hn[o] = rl[o];
      }
    }
    int k = head_at(a, l + 1);
    if (k >= 0) {
      const double* u = th + of->u[k];
      double s = 0.0;
      for (int j = 0; j < w; ++j) s += u[j] * rl[j];
      s += th[of->c[k]];
      out[1 + k] = (mode == ORA_BF16_EMU) ? (double)(float)s : s;
    }
    if (acts) for (int j = 0; j < w; ++j) acts[(int64_t)(l + 1) * stride + j] = hn[j];
    double* t = h; h = hn; hn = t;
    in = w;
  }
  const double* wo = th + of->wout;
  double s = 0.0;
  for (int j = 0; j < w; ++j) s += wo[j] * h[j];
  s += th[of->bout];
  out[0] = (mode == ORA_BF16_EMU) ? (double)(float)s : s;
}

void ora_forward(const ora_arch* a, const double* theta, const float* q, int64_t n, int32_t mode,
                 double* logits) {
  offsets of;
  param_offsets(a, &of);
  const int nl = 1 + a->n_heads;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    forward_one(a, &of, theta, q + i * a->d0, mode, logits + i * nl, NULL, NULL); /* d0 = record */
}

/* ------------------------------------------------------------------------ */
/* Eq. (1): per sample -[alpha y log(s(z)) + beta (1-y) log(1-s(z))]
 * = alpha y softplus(-z) + beta (1-y) softplus(z) exactly (R5).          */
static double softplus(double u) { return (u > 0.0 ? u : 0.0) + log1p(exp(-fabs(u))); }
static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

double ora_weighted_bce(double z, int32_t y, double alpha, double beta) {
  return y ? alpha * softplus(-z) : beta * softplus(z);
}

/* Gradient of the loss of the network evaluated in `mode`: ORA_FP64 is the
 * plain definition; ORA_BF16_EMU differentiates the bf16-precision forward of
 * R33 (its rounded activations and fp32 pre-activations give the ReLU masks,
 * bf16 weights propagate the deltas), the rest in fp64.                    */
static double loss_grad_impl(const ora_arch* a, const double* th, const float* q,
                             const uint8_t* y, int64_t n, int64_t n_global, double alpha,
                             double beta, double* grad, ora_stats* st, int mode) {
  offsets of;
  param_offsets(a, &of);
  const int w = a->width, L = a->layers, d0 = input_dim(a);
  const int stride = (d0 > w ? d0 : w);
  const int64_t P = ora_num_params(a);
  memset(grad, 0, sizeof(double) * P);
  double* acts = (double*)malloc(sizeof(double) * (L + 1) * stride);
  double* pre = (double*)malloc(sizeof(double) * L * w);
  double* dh = (double*)malloc(sizeof(double) * w);   /* dL/dh_l */
  double* dz = (double*)malloc(sizeof(double) * w);   /* dL/dz_l */
  double loss = 0.0;
  uint64_t tp = 0, fp = 0, fn = 0, tn = 0;
  const double B = (double)n_global;
  for (int64_t i = 0; i < n; ++i) {
    double out[3];
    forward_one(a, &of, th, q + (int64_t)i * a->d0, mode, out, acts, pre);
    const int yi = y[i] ? 1 : 0;
    const double wi = yi ? alpha : beta;
    /* output logit and its gradient dL/dz = w (sigmoid(z) - y) / B (a7) */
    loss += ora_weighted_bce(out[0], yi, alpha, beta) / B;
    int pred = out[0] >= 0.0; /* batch stats, rounding rule P:287 (R31) */
    tp += pred && yi; fp += pred && !yi; fn += !pred && yi; tn += !pred && !yi;
    double gz = wi * (sigmoid(out[0]) - yi) / B;
    const double* hL = acts + (int64_t)L * stride;
    for (int j = 0; j < w; ++j) {
      grad[of.wout + j] += gz * hL[j];
      dh[j] = gz * th[of.wout + j];
    }
    grad[of.bout] += gz;
    double ge[2] = {0, 0};
    for (int k = 0; k < a->n_heads; ++k) {
      loss += ora_weighted_bce(out[1 + k], yi, alpha, beta) / B; /* L_Early sum */
      ge[k] = wi * (sigmoid(out[1 + k]) - yi) / B;
    }
    /* back-propagate through hidden layers l = L..1 */
    for (int l = L - 1; l >= 0; --l) {
      int k = head_at(a, l + 1);
      if (k >= 0) {
        const double* hl = acts + (int64_t)(l + 1) * stride;
        for (int j = 0; j < w; ++j) {
          grad[of.u[k] + j] += ge[k] * hl[j];
          dh[j] += ge[k] * th[of.u[k] + j];
        }
        grad[of.c[k]] += ge[k];
      }
      for (int o = 0; o < w; ++o) dz[o] = dh[o] * act_grad(a, pre[(int64_t)l * w + o]); /* R25, R41 */
      const int in = (l == 0) ? d0 : w;
      const double* hin = acts + (int64_t)l * stride;
      const double* W = th + of.W[l];
      for (int o = 0; o < w; ++o) {
        grad[of.b[l] + o] += dz[o];
        for (int kk = 0; kk < in; ++kk) grad[of.W[l] + (int64_t)o * in + kk] += dz[o] * hin[kk];
      }
      if (l > 0) {
        for (int kk = 0; kk < in; ++kk) {
          double s = 0.0;
          for (int o = 0; o < w; ++o) {
            double wv = W[(int64_t)o * in + kk];
            if (mode == ORA_BF16_EMU) wv = (double)bf16_round((float)wv);
            s += dz[o] * wv;
          }
          dh[kk] = s;
        }
      }
    }
  }
  free(acts); free(pre); free(dh); free(dz);
  if (st) { st->loss = loss; st->tp = tp; st->fp = fp; st->fn = fn; st->tn = tn; }
  return loss;
}

double ora_loss_grad(const ora_arch* a, const double* th, const float* q, const uint8_t* y,
                     int64_t n, int64_t n_global, double alpha, double beta, double* grad,
                     ora_stats* st) {
  return loss_grad_impl(a, th, q, y, n, n_global, alpha, beta, grad, st, ORA_FP64);
}

double ora_loss_grad_mode(const ora_arch* a, const double* th, const float* q, const uint8_t* y,
                          int64_t n, int64_t n_global, double alpha, double beta, double* grad,
                          ora_stats* st, int32_t mode) {
  return loss_grad_impl(a, th, q, y, n, n_global, alpha, beta, grad, st, mode);
}

/* ------------------------------------------------------------------------ */
/* Adam (Kingma & Ba; PyTorch semantics): m <- b1 m + (1-b1) g;
 * v <- b2 v + (1-b2) g^2; theta <- theta - lr mhat / (sqrt(vhat) + eps).  */
void ora_adam(int64_t P, double* th, double* m, double* v, int64_t t, double lr, double b1,
              double b2, double eps, const double* g) {
  double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  for (int64_t i = 0; i < P; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    double mh = m[i] / bc1, vh = v[i] / bc2;
    th[i] -= lr * mh / (sqrt(vh) + eps);
  }
}

/* alpha_t = 1 + 999 t / (T - 1), the BASELINE.json c1 ramp (R6). */
double ora_alpha(int64_t t, int64_t T) {
  if (T <= 1) return 1000.0;
  return 1.0 + 999.0 * (double)t / (double)(T - 1);
}

/* ------------------------------------------------------------------------ */
/* Calibration (a6, R21): tau = min over labelled positives of the logit, so
 * yhat = [z >= tau] has FN = 0 on the set.  Heads likewise.               */
int ora_calibrate(int32_t n_heads, const double* logits, const uint8_t* y, int64_t n,
                  double* tau) {
  const int nl = 1 + n_heads;
  for (int k = 0; k < nl; ++k) tau[k] = INFINITY;
  int any = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!y[i]) continue;
    any = 1;
    for (int k = 0; k < nl; ++k) {
      double z = logits[i * nl + k];
      if (z < tau[k]) tau[k] = z;
    }
  }
  return any ? 0 : 1;
}

/* Confusion counts (P:157-176 cost cases) of the calibrated predictor
 * yhat = [e_1 >= tau_1] and [e_2 >= tau_2] and [z >= tau] (R22); exit bins:
 * 0 = left at head 1, 1 = left at head 2, 2 = final negative, 3 = final positive. */
void ora_score(int32_t n_heads, const double* logits, const uint8_t* y, int64_t n,
               const double* tau, ora_counts* c) {
  memset(c, 0, sizeof(*c));
  const int nl = 1 + n_heads;
  for (int64_t i = 0; i < n; ++i) {
    const double* z = logits + i * nl;
    int pred = 1, bin = -1;
    for (int k = 0; k < n_heads; ++k) {
      if (!(z[1 + k] >= tau[1 + k])) { pred = 0; bin = k; break; }
    }
    if (pred) {
      pred = z[0] >= tau[0];
      bin = pred ? 3 : 2;
    }
    for (int k = 0; k < nl; ++k)
      if (!isfinite(z[k])) { c->nonfinite++; break; }
    c->exit_hist[bin]++;
    int yi = y[i] != 0;
    c->tp += pred && yi; c->fp += pred && !yi; c->fn += !pred && yi; c->tn += !pred && !yi;
  }
}
