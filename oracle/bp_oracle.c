/*
 * bp_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference back-projection kernels, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg as the checker and CPU baseline.  It is never linked into, called by or
 * shipped with the product library (paper_2104_13248_b200/libconebp_b200.so).
 *
 * Every function follows the reference's float32 operation order exactly
 * (build with -ffp-contract=off: no FMA contraction; x86-64 SSE float math is
 * IEEE binary32 with round-to-nearest), so its output is bitwise identical to
 * the numba kernels; tests/test_oracle_golden.py pins that against golden
 * vectors produced by the live reference (tests/golden/make_golden.py).
 *
 *   oracle_baseline          /root/reference/pkg/src/conebp/_kernels.py:29-61
 *   oracle_transpose         _kernels.py:64-106
 *   oracle_share             _kernels.py:109-159
 *   oracle_symmetry          _kernels.py:162-222
 *   oracle_subline           _kernels.py:225-288
 *   oracle_subline_prefetch  _kernels.py:291-369
 *   oracle_voxels            _kernels.py:38-61 evaluated on a voxel list (global
 *                            indices) -- the subset oracle of SURVEY.md 8(c)
 *
 * Parallelism: pthreads over z-slices (baseline, as prange over k at :42) or
 * over (i, j) columns (rungs, as prange over the ij list at :76...); every voxel
 * has one writer and a fixed ascending-s chain, so results do not depend on the
 * thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

enum { V_BASELINE = 0, V_TRANSPOSE = 1, V_SHARE = 2, V_SYMMETRY = 3, V_SUBLINE = 4, V_PREFETCH = 5 };

/* (((a*fi + b*fj) + c*fk) + d) with separately rounded operations (_kernels.py:48) */
static inline float dot4(const float* r, float fi, float fj, float fk) {
  float p0 = r[0] * fi;
  float p1 = r[1] * fj;
  float s = p0 + p1;
  float p2 = r[2] * fk;
  s = s + p2;
  return s + r[3];
}

/* ------------------------------------------------------------------ baseline */
typedef struct {
  const float* img; /* [np][rows][nw]: detector rows [v0, v0+rows) (NATURAL) */
  const float* mats;
  float* vol;       /* [nz_slab][ny][nx], slab slices [k_lo, k_hi) of a global grid */
  i64 np, nh, nw, v0, rows, nx, ny, k_lo, k_hi;
  i64 k_begin, k_end; /* this worker's slice range (global) */
  i64 s;
  i64 band_viol;
} base_job;

static void baseline_slices(base_job* jb) {
  const float one = 1.0f, zero = 0.0f;
  const float umax = (float)(jb->nw - 1), vmax = (float)(jb->nh - 1);
  const i64 s = jb->s, nw = jb->nw, nx = jb->nx, ny = jb->ny;
  const float* r0 = jb->mats + 12 * s;
  const float* r1 = r0 + 4;
  const float* r2 = r0 + 8;
  const float* plane = jb->img + s * jb->rows * nw;
  for (i64 k = jb->k_begin; k < jb->k_end; ++k) {
    const float fk = (float)k;
    float* vk = jb->vol + (k - jb->k_lo) * nx * ny;
    for (i64 j = 0; j < ny; ++j) {
      const float fj = (float)j;
      for (i64 i = 0; i < nx; ++i) {
        const float fi = (float)i;
        const float z = dot4(r2, fi, fj, fk);
        const float f = one / z;
        const float x = dot4(r0, fi, fj, fk) * f;
        const float y = dot4(r1, fi, fj, fk) * f;
        if (x >= zero && x < umax && y >= zero && y < vmax) {
          const int ix = (int)x;
          const int iy = (int)y;
          const float ax = x - (float)ix;
          const float ay = y - (float)iy;
          const i64 row = (i64)iy - jb->v0;
          if (row < 0 || row + 1 >= jb->rows) {
            jb->band_viol++;
            continue;
          }
          const float* p0 = plane + row * nw + ix;
          const float* p1 = p0 + nw;
          const float s0 = p0[0] * (one - ax) + p0[1] * ax;
          const float s1 = p1[0] * (one - ax) + p1[1] * ax;
          const float val = s0 * (one - ay) + s1 * ay;
          const float w = f * f;
          vk[j * nx + i] += val * w;
        }
      }
    }
  }
}

typedef struct {
  base_job* jobs;
  int n;
  int idx;
} base_worker;

static void* base_thread(void* arg) {
  base_worker* w = (base_worker*)arg;
  base_job* jb = &w->jobs[w->idx];
  /* the angle loop is outside the parallel region in the reference (:38 vs :42);
     slices are independent, so each worker walks all angles over its own slices */
  for (i64 s = 0; s < jb->np; ++s) {
    jb->s = s;
    baseline_slices(jb);
  }
  return NULL;
}

/* Baseline on NATURAL layouts, slab [k_lo, k_hi) of the global grid, detector band
 * [v0, v0+rows).  Returns the number of samples that needed rows outside the band. */
i64 oracle_baseline(const float* img, i64 np, i64 nh, i64 nw, i64 v0, i64 rows, const float* mats, float* vol,
                    i64 nx, i64 ny, i64 k_lo, i64 k_hi, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  i64 nzs = k_hi - k_lo;
  if (nzs <= 0) return 0;
  if (nthreads > nzs) nthreads = (int)nzs;
  base_job* jobs = (base_job*)calloc((size_t)nthreads, sizeof(base_job));
  base_worker* ws = (base_worker*)calloc((size_t)nthreads, sizeof(base_worker));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    base_job* jb = &jobs[t];
    jb->img = img; jb->mats = mats; jb->vol = vol;
    jb->np = np; jb->nh = nh; jb->nw = nw; jb->v0 = v0; jb->rows = rows;
    jb->nx = nx; jb->ny = ny; jb->k_lo = k_lo; jb->k_hi = k_hi;
    jb->k_begin = k_lo + nzs * t / nthreads;
    jb->k_end = k_lo + nzs * (t + 1) / nthreads;
    ws[t].jobs = jobs; ws[t].n = nthreads; ws[t].idx = t;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, base_thread, &ws[t]);
  base_thread(&ws[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  i64 viol = 0;
  for (int t = 0; t < nthreads; ++t) viol += jobs[t].band_viol;
  free(jobs); free(ws); free(th);
  return viol;
}

/* ------------------------------------------------------------- voxel list */
/* vals[q] += sum over s of the baseline update of voxel idx[3q..3q+2] (global i,j,k) */
typedef struct {
  const float* img; const float* mats; const i64* idx; float* vals;
  i64 np, nh, nw, q0, q1;
} vox_job;

static void* vox_thread(void* arg) {
  vox_job* jb = (vox_job*)arg;
  const float one = 1.0f, zero = 0.0f;
  const float umax = (float)(jb->nw - 1), vmax = (float)(jb->nh - 1);
  for (i64 q = jb->q0; q < jb->q1; ++q) {
    const float fi = (float)jb->idx[3 * q], fj = (float)jb->idx[3 * q + 1], fk = (float)jb->idx[3 * q + 2];
    float acc = jb->vals[q];
    for (i64 s = 0; s < jb->np; ++s) {
      const float* r0 = jb->mats + 12 * s;
      const float z = dot4(r0 + 8, fi, fj, fk);
      const float f = one / z;
      const float x = dot4(r0, fi, fj, fk) * f;
      const float y = dot4(r0 + 4, fi, fj, fk) * f;
      if (x >= zero && x < umax && y >= zero && y < vmax) {
        const int ix = (int)x, iy = (int)y;
        const float ax = x - (float)ix, ay = y - (float)iy;
        const float* p0 = jb->img + (s * jb->nh + iy) * jb->nw + ix;
        const float* p1 = p0 + jb->nw;
        const float s0 = p0[0] * (one - ax) + p0[1] * ax;
        const float s1 = p1[0] * (one - ax) + p1[1] * ax;
        const float val = s0 * (one - ay) + s1 * ay;
        const float w = f * f;
        acc += val * w;
      }
    }
    jb->vals[q] = acc;
  }
  return NULL;
}

void oracle_voxels(const float* img, i64 np, i64 nh, i64 nw, const float* mats, const i64* idx, i64 n, float* vals,
                   int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  vox_job* jobs = (vox_job*)calloc((size_t)nthreads, sizeof(vox_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    vox_job* jb = &jobs[t];
    jb->img = img; jb->mats = mats; jb->idx = idx; jb->vals = vals;
    jb->np = np; jb->nh = nh; jb->nw = nw;
    jb->q0 = n * t / nthreads; jb->q1 = n * (t + 1) / nthreads;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, vox_thread, &jobs[t]);
  vox_thread(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th);
}

/* ------------------------------------------------------------------ rungs */
/* transposed layouts: img_t [np][nw][nh], vol_t [nx][ny][nz]; columns c = j*nx + i
 * (make_ij_list order, tensors.py:162-175) */
typedef struct {
  const float* img; const float* mats; float* vol;
  i64 np, nh, nw, nx, ny, nz, nb;
  i64 c0, c1;
  int variant;
} rung_job;

#define IMG(s, u, v) img[((s) * nw + (u)) * nh + (v)]

static void rung_column(const rung_job* jb, i64 i, i64 j, float* F, float* W, float* X, unsigned char* ok,
                        float* line, float* sums, float* sums2) {
  const float* img = jb->img;
  const float* mats = jb->mats;
  const i64 nh = jb->nh, nw = jb->nw, nz = jb->nz, nb = jb->nb;
  const float one = 1.0f, zero = 0.0f;
  const float umax = (float)(nw - 1), vmax = (float)(nh - 1), vtop = (float)(nh - 1);
  const float fi = (float)i, fj = (float)j, fk0 = 0.0f;
  float* col = jb->vol + (i * jb->ny + j) * nz;
  const i64 n_batches = jb->np / nb, nzh = nz / 2;
  for (i64 b = 0; b < n_batches; ++b) {
    const i64 s_base = b * nb;
    if (jb->variant == V_TRANSPOSE) { /* _kernels.py:81-106 */
      for (i64 k = 0; k < nz; ++k) {
        const float fk = (float)k;
        float acc = col[k];
        for (i64 t = 0; t < nb; ++t) {
          const i64 s = s_base + t;
          const float* r0 = mats + 12 * s;
          const float z = dot4(r0 + 8, fi, fj, fk);
          const float f = one / z;
          const float x = dot4(r0, fi, fj, fk) * f;
          const float y = dot4(r0 + 4, fi, fj, fk) * f;
          if (x >= zero && x < umax && y >= zero && y < vmax) {
            const int iu = (int)x, iv = (int)y;
            const float au = x - (float)iu, av = y - (float)iv;
            const float s0 = IMG(s, iu, iv) * (one - av) + IMG(s, iu, iv + 1) * av;
            const float s1 = IMG(s, iu + 1, iv) * (one - av) + IMG(s, iu + 1, iv + 1) * av;
            const float val = s0 * (one - au) + s1 * au;
            acc += val * (f * f);
          }
        }
        col[k] = acc;
      }
      continue;
    }
    /* hoisted terms at fk0 = 0 (_kernels.py:133-140) */
    for (i64 t = 0; t < nb; ++t) {
      const float* r0 = mats + 12 * (s_base + t);
      F[t] = one / dot4(r0 + 8, fi, fj, fk0);
      W[t] = F[t] * F[t];
      X[t] = dot4(r0, fi, fj, fk0) * F[t];
      ok[t] = (X[t] >= zero && X[t] < umax) ? 1 : 0;
    }
    if (jb->variant == V_SHARE) { /* :141-159 */
      for (i64 k = 0; k < nz; ++k) {
        const float fk = (float)k;
        float acc = col[k];
        for (i64 t = 0; t < nb; ++t) {
          if (!ok[t]) continue;
          const i64 s = s_base + t;
          const float y = dot4(mats + 12 * s + 4, fi, fj, fk) * F[t];
          if (y >= zero && y < vmax) {
            const float x = X[t];
            const int iu = (int)x, iv = (int)y;
            const float au = x - (float)iu, av = y - (float)iv;
            const float s0 = IMG(s, iu, iv) * (one - av) + IMG(s, iu, iv + 1) * av;
            const float s1 = IMG(s, iu + 1, iv) * (one - av) + IMG(s, iu + 1, iv + 1) * av;
            const float val = s0 * (one - au) + s1 * au;
            acc += val * W[t];
          }
        }
        col[k] = acc;
      }
    } else if (jb->variant == V_SYMMETRY) { /* :196-222 */
      for (i64 k = 0; k < nzh; ++k) {
        const float fk = (float)k;
        float acc = col[k], acc2 = col[nz - 1 - k];
        for (i64 t = 0; t < nb; ++t) {
          if (!ok[t]) continue;
          const i64 s = s_base + t;
          const float x = X[t];
          const int iu = (int)x;
          const float au = x - (float)iu;
          const float y = dot4(mats + 12 * s + 4, fi, fj, fk) * F[t];
          if (y >= zero && y < vmax) {
            const int iv = (int)y;
            const float av = y - (float)iv;
            const float s0 = IMG(s, iu, iv) * (one - av) + IMG(s, iu, iv + 1) * av;
            const float s1 = IMG(s, iu + 1, iv) * (one - av) + IMG(s, iu + 1, iv + 1) * av;
            acc += (s0 * (one - au) + s1 * au) * W[t];
          }
          const float y2 = vtop - y;
          if (y2 >= zero && y2 < vmax) {
            const int iv = (int)y2;
            const float av = y2 - (float)iv;
            const float s0 = IMG(s, iu, iv) * (one - av) + IMG(s, iu, iv + 1) * av;
            const float s1 = IMG(s, iu + 1, iv) * (one - av) + IMG(s, iu + 1, iv + 1) * av;
            acc2 += (s0 * (one - au) + s1 * au) * W[t];
          }
        }
        col[k] = acc;
        col[nz - 1 - k] = acc2;
      }
    } else if (jb->variant == V_SUBLINE) { /* :261-288, one sub-line per ok angle */
      for (i64 t = 0; t < nb; ++t) {
        if (!ok[t]) continue;
        const i64 s = s_base + t;
        const int iu = (int)X[t];
        const float dx = X[t] - (float)iu;
        const float a0 = one - dx;
        for (i64 m = 0; m < nh; ++m) line[t * nh + m] = IMG(s, iu, m) * a0 + IMG(s, iu + 1, m) * dx;
      }
      for (i64 k = 0; k < nzh; ++k) {
        const float fk = (float)k;
        float acc = col[k], acc2 = col[nz - 1 - k];
        for (i64 t = 0; t < nb; ++t) {
          if (!ok[t]) continue;
          const i64 s = s_base + t;
          const float* ln = line + t * nh;
          const float y = dot4(mats + 12 * s + 4, fi, fj, fk) * F[t];
          if (y >= zero && y < vmax) {
            const int iv = (int)y;
            const float av = y - (float)iv;
            acc += (ln[iv] * (one - av) + ln[iv + 1] * av) * W[t];
          }
          const float y2 = vtop - y;
          if (y2 >= zero && y2 < vmax) {
            const int iv = (int)y2;
            const float av = y2 - (float)iv;
            acc2 += (ln[iv] * (one - av) + ln[iv + 1] * av) * W[t];
          }
        }
        col[k] = acc;
        col[nz - 1 - k] = acc2;
      }
    } else { /* V_PREFETCH, :329-369: dual buffers, angle-outer order per batch */
      for (i64 k = 0; k < nzh; ++k) {
        sums[k] = col[k];
        sums2[k] = col[nz - 1 - k];
      }
      float* buf[2] = {line, line + nh};
      if (ok[0]) {
        const int iu = (int)X[0];
        const float dx = X[0] - (float)iu, a0 = one - dx;
        for (i64 m = 0; m < nh; ++m) buf[0][m] = IMG(s_base, iu, m) * a0 + IMG(s_base, iu + 1, m) * dx;
      }
      for (i64 t = 0; t < nb; ++t) {
        if (t + 1 < nb && ok[t + 1]) {
          const i64 s = s_base + t + 1;
          const int iu = (int)X[t + 1];
          const float dx = X[t + 1] - (float)iu, a0 = one - dx;
          float* cur = buf[(t + 1) % 2];
          for (i64 m = 0; m < nh; ++m) cur[m] = IMG(s, iu, m) * a0 + IMG(s, iu + 1, m) * dx;
        }
        if (ok[t]) {
          const i64 s = s_base + t;
          const float* r1 = mats + 12 * s + 4;
          const float Ft = F[t], Wt = W[t];
          const float* cur = buf[t % 2];
          for (i64 k = 0; k < nzh; ++k) {
            const float fk = (float)k;
            const float y = dot4(r1, fi, fj, fk) * Ft;
            if (y >= zero && y < vmax) {
              const int iv = (int)y;
              const float av = y - (float)iv;
              sums[k] += (cur[iv] * (one - av) + cur[iv + 1] * av) * Wt;
            }
            const float y2 = vtop - y;
            if (y2 >= zero && y2 < vmax) {
              const int iv = (int)y2;
              const float av = y2 - (float)iv;
              sums2[k] += (cur[iv] * (one - av) + cur[iv + 1] * av) * Wt;
            }
          }
        }
      }
      for (i64 k = 0; k < nzh; ++k) {
        col[k] = sums[k];
        col[nz - 1 - k] = sums2[k];
      }
    }
  }
}

static void* rung_thread(void* arg) {
  rung_job* jb = (rung_job*)arg;
  const i64 nb = jb->nb, nh = jb->nh, nz = jb->nz;
  float* F = (float*)malloc(sizeof(float) * (size_t)nb);
  float* W = (float*)malloc(sizeof(float) * (size_t)nb);
  float* X = (float*)malloc(sizeof(float) * (size_t)nb);
  unsigned char* ok = (unsigned char*)malloc((size_t)nb);
  float* line = (float*)malloc(sizeof(float) * (size_t)(nb > 2 ? nb : 2) * (size_t)nh);
  float* sums = (float*)malloc(sizeof(float) * (size_t)(nz / 2 + 1));
  float* sums2 = (float*)malloc(sizeof(float) * (size_t)(nz / 2 + 1));
  for (i64 c = jb->c0; c < jb->c1; ++c) rung_column(jb, c % jb->nx, c / jb->nx, F, W, X, ok, line, sums, sums2);
  free(F); free(W); free(X); free(ok); free(line); free(sums); free(sums2);
  return NULL;
}

/* Optimized rungs on TRANSPOSED layouts (variant 1..5), batch size nb | np. */
int oracle_rung(int variant, const float* img_t, i64 np, i64 nh, i64 nw, const float* mats, float* vol_t, i64 nx,
                i64 ny, i64 nz, i64 nb, int nthreads) {
  if (variant < V_TRANSPOSE || variant > V_PREFETCH || nb < 1 || np % nb) return -1;
  if (variant >= V_SYMMETRY && (nz & 1)) return -1;
  if (nthreads < 1) nthreads = 1;
  const i64 ncol = nx * ny;
  if (nthreads > ncol) nthreads = (int)ncol;
  rung_job* jobs = (rung_job*)calloc((size_t)nthreads, sizeof(rung_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    rung_job* jb = &jobs[t];
    jb->img = img_t; jb->mats = mats; jb->vol = vol_t;
    jb->np = np; jb->nh = nh; jb->nw = nw; jb->nx = nx; jb->ny = ny; jb->nz = nz; jb->nb = nb;
    jb->c0 = ncol * t / nthreads; jb->c1 = ncol * (t + 1) / nthreads;
    jb->variant = variant;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, rung_thread, &jobs[t]);
  rung_thread(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th);
  return 0;
}
