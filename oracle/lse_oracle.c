/*
 * lse_oracle.c -- CPU restatement of the reference LSE loop in C (OpenMP).
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ as a second checker
 * and by bench.py as the timed CPU baseline ("port").  It restates, in the
 * reference's exact float64 operation order:
 *   engine.py:148-174  _advance_once      (update, finiteness, reinit, smoothing)
 *   multi-band region term (C3; oracle/lse_oracle.py region_velocity_bands):
 *                      D = sum_k (c+_k - c-_k)(2 I_k - c+_k - c-_k), bands
 *                      accumulated left to right, then models.py:109-119
 *   engine.py:222-254  EvolutionRun._step_once / advance (checkpoint convergence)
 *   models.py:84-119   edge_velocity / region_velocity
 *   models.py:144-162  zhang_velocity (mean separation)
 *   models.py:71-81    edge_function
 *   grid.py:102-118    region_means  (numpy pairwise summation of the masked,
 *                                     row-major-compacted array, then / n)
 *   kernels.py:67-95   convolve_same (scipy correlate1d symmetric order),
 *                      gradient_central (np.gradient), hypot (libm, as np.hypot)
 * Compile with -ffp-contract=off so no FMA changes the rounding.
 * Parity is pinned by tests/test_oracle_c.py against tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int model; /* 0 edge, 1 region, 2 zhang */
  double dt;
  int ts_reg;
  int reinit_period;
  int reg_period;
  long long max_iters;
  long long conv_check_every;
  long long conv_window;
  double edge_gain;
  int ts_pre;
  const double* reg_w; /* axis weights, ts_reg */
  const double* pre_w; /* axis weights, ts_pre */
  double nu;           /* zhang speed constant */
  int nbands;          /* model 3 (multi-band region): bands of the image */
} oracle_params;

/* scipy correlate1d, symmetric branch, zero padding. axis 0 = along rows. */
static void correlate1d(const double* in, double* out, int H, int W, const double* w, int ts,
                        int axis) {
  const int r = ts / 2;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < H; ++i) {
    for (int x = 0; x < W; ++x) {
      double acc;
      if (axis == 0) {
        acc = in[(size_t)i * W + x] * w[r];
        for (int d = r; d >= 1; --d) {
          double a = i - d >= 0 ? in[(size_t)(i - d) * W + x] : 0.0;
          double b = i + d < H ? in[(size_t)(i + d) * W + x] : 0.0;
          acc = acc + (a + b) * w[r - d];
        }
      } else {
        const double* row = in + (size_t)i * W;
        acc = row[x] * w[r];
        for (int d = r; d >= 1; --d) {
          double a = x - d >= 0 ? row[x - d] : 0.0;
          double b = x + d < W ? row[x + d] : 0.0;
          acc = acc + (a + b) * w[r - d];
        }
      }
      out[(size_t)i * W + x] = acc;
    }
  }
}

static void convolve_same(const double* in, double* tmp, double* out, int H, int W,
                          const double* w, int ts) {
  correlate1d(in, tmp, H, W, w, ts, 0);
  correlate1d(tmp, out, H, W, w, ts, 1);
}

static inline void np_gradient(const double* f, int H, int W, int i, int x, double* fx,
                               double* fy) {
  const double c = f[(size_t)i * W + x];
  if (x == 0) *fx = f[(size_t)i * W + 1] - c;
  else if (x == W - 1) *fx = c - f[(size_t)i * W + W - 2];
  else *fx = (f[(size_t)i * W + x + 1] - f[(size_t)i * W + x - 1]) / 2.0;
  if (i == 0) *fy = f[(size_t)W + x] - c;
  else if (i == H - 1) *fy = c - f[(size_t)(H - 2) * W + x];
  else *fy = (f[(size_t)(i + 1) * W + x] - f[(size_t)(i - 1) * W + x]) / 2.0;
}

/* numpy pairwise summation (the algorithm of ndarray.mean for float64) */
static double pairwise(const double* a, long long n) {
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    long long i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  double lo, hi;
  if (n > (1LL << 20)) {
#pragma omp task shared(lo)
    lo = pairwise(a, n2);
#pragma omp task shared(hi)
    hi = pairwise(a + n2, n - n2);
#pragma omp taskwait
  } else {
    lo = pairwise(a, n2);
    hi = pairwise(a + n2, n - n2);
  }
  return lo + hi;
}

static double pairwise_par(const double* a, long long n) {
  double res = 0.0;
#pragma omp parallel
#pragma omp single
  res = pairwise(a, n);
  return res;
}

/* grid.py:102-118: the row-major prefix counts of {phi >= 0}; returns the
 * count, or -1 when a side is empty */
static long long partition_rows(const double* phi, int H, int W, long long* row_pos) {
  const long long n = (long long)H * W;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < H; ++i) {
    long long c = 0;
    for (int x = 0; x < W; ++x) c += phi[(size_t)i * W + x] >= 0.0;
    row_pos[i] = c;
  }
  long long total = 0;
  for (int i = 0; i < H; ++i) {
    long long c = row_pos[i];
    row_pos[i] = total;
    total += c;
  }
  return (total == 0 || total == n) ? -1 : total;
}

/* means of img over {phi >= 0} / {phi < 0} (numpy pairwise sums of the
 * row-major compacted sides; buf holds the positive side then the negative) */
static void side_means(const double* img, const double* phi, int H, int W, double* buf,
                       const long long* row_pos, long long total, double* cp, double* cm) {
  const long long n = (long long)H * W;
  double* buf_pos = buf;
  double* buf_neg = buf + total;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < H; ++i) {
    long long kp = row_pos[i], kn = (long long)i * W - row_pos[i];
    for (int x = 0; x < W; ++x) {
      const size_t o = (size_t)i * W + x;
      if (phi[o] >= 0.0) buf_pos[kp++] = img[o];
      else buf_neg[kn++] = img[o];
    }
  }
  *cp = pairwise_par(buf_pos, total) / (double)total;
  *cm = pairwise_par(buf_neg, n - total) / (double)(n - total);
}

/* grid.py:102-118; returns 0 when a side is empty */
static int region_means(const double* img, const double* phi, int H, int W, double* buf,
                        long long* row_pos, double* cp, double* cm) {
  const long long total = partition_rows(phi, H, W, row_pos);
  if (total < 0) return 0;
  side_means(img, phi, H, W, buf, row_pos, total, cp, cm);
  return 1;
}

/* models.py:71-81 */
void oracle_edge_function(const double* img, int H, int W, const double* w, int ts, double gain,
                          double* g) {
  const size_t n = (size_t)H * W;
  double* t = (double*)malloc(n * sizeof(double));
  double* s = (double*)malloc(n * sizeof(double));
  convolve_same(img, t, s, H, W, w, ts);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < H; ++i)
    for (int x = 0; x < W; ++x) {
      double fx, fy;
      np_gradient(s, H, W, i, x, &fx, &fy);
      double a = gain * fx, b = gain * fy;
      g[(size_t)i * W + x] = 1.0 / (1.0 + a * a + b * b);
    }
  free(t);
  free(s);
}

/* EvolutionRun (engine.py:193-269) restated: a context owns the work
 * buffers and the checkpoint history, so repeated oracle_advance() calls walk
 * the same trajectory one run would (engine.py:242-254). */
typedef struct {
  int H, W;
  oracle_params p;
  const double* img;  /* (H, W), or nbands planes for model 3 */
  double* phi; /* caller-owned, in/out */
  double *u, *t, *g, *buf, *D;
  long long* rows;
  unsigned char* ck;  /* checkpoint masks, allocated at the first checkpoint */
  long long n_ck;
  long long iteration;
  int converged, degenerate;
} oracle_ctx;

oracle_ctx* oracle_create(const double* img, int H, int W, const oracle_params* p, double* phi) {
  const size_t n = (size_t)H * W;
  oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof(oracle_ctx));
  c->H = H;
  c->W = W;
  c->p = *p;
  c->img = img;
  c->phi = phi;
  c->u = (double*)malloc(n * sizeof(double));
  c->t = (double*)malloc(n * sizeof(double));
  c->rows = (long long*)malloc((size_t)H * sizeof(long long));
  if (p->model == 0) {
    c->g = (double*)malloc(n * sizeof(double));
    oracle_edge_function(img, H, W, p->pre_w, p->ts_pre, p->edge_gain, c->g);
  } else {
    c->buf = (double*)malloc(n * sizeof(double));
    if (p->model == 3) c->D = (double*)malloc(n * sizeof(double));
  }
  return c;
}

void oracle_destroy(oracle_ctx* c) {
  if (!c) return;
  free(c->u);
  free(c->t);
  free(c->g);
  free(c->buf);
  free(c->D);
  free(c->rows);
  free(c->ck);
  free(c);
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());   /* 0: every host thread */
#else
  (void)n;
#endif
}

void oracle_state(const oracle_ctx* c, long long* iteration, int* converged, int* degenerate) {
  *iteration = c->iteration;
  *converged = c->converged;
  *degenerate = c->degenerate;
}

/* Up to n_iters iterations.  Returns 0, or the iteration at which
 * NumericalInstabilityError is raised (phi then holds the last good state). */
long long oracle_advance(oracle_ctx* c, long long n_iters) {
  const int H = c->H, W = c->W;
  const oracle_params* p = &c->p;
  const double* img = c->img;
  double* phi = c->phi;
  double *u = c->u, *t = c->t, *g = c->g;
  const size_t n = (size_t)H * W;
  long long err = 0;
  for (long long s = 0; s < n_iters; ++s) {
    if (c->converged || c->iteration >= p->max_iters) break;
    const long long it = c->iteration + 1;
    double cp = 0, cm = 0, dc = 0, peak = 0, mid = 0;
    int zero = 0;
    const int two_mean = p->model == 1 || p->model == 2 || p->model == 3;
    if (p->model == 3) {
      /* multi-band region term: per-band means, D accumulated over the bands */
      const long long total = partition_rows(phi, H, W, c->rows);
      if (total < 0) {
        zero = 1;
      } else {
        double* D = c->D;
        for (int k = 0; k < p->nbands; ++k) {
          const double* band = img + (size_t)k * n;
          double bcp, bcm;
          side_means(band, phi, H, W, c->buf, c->rows, total, &bcp, &bcm);
          const double bdc = bcp - bcm;
#pragma omp parallel for schedule(static)
          for (long long q = 0; q < (long long)n; ++q) {
            const double term = bdc * (2.0 * band[q] - bcp - bcm);
            D[q] = k == 0 ? term : D[q] + term;
          }
        }
        double pk = 0.0;
#pragma omp parallel for reduction(max : pk) schedule(static)
        for (long long q = 0; q < (long long)n; ++q) {
          const double d = fabs(D[q]);
          if (d > pk) pk = d;
        }
        peak = pk;
        if (peak == 0.0) zero = 1;
      }
    } else if (two_mean) {
      if (!region_means(img, phi, H, W, c->buf, c->rows, &cp, &cm)) {
        zero = 1;
      } else {
        dc = cp - cm;
        mid = 0.5 * (cp + cm);                       /* models.py:153 */
        double pk = 0.0;
        if (p->model == 1) {
#pragma omp parallel for reduction(max : pk) schedule(static)
          for (long long k = 0; k < (long long)n; ++k) {
            double d = fabs(dc * (2.0 * img[k] - cp - cm));
            if (d > pk) pk = d;
          }
        } else {
#pragma omp parallel for reduction(max : pk) schedule(static)
          for (long long k = 0; k < (long long)n; ++k) {
            double d = fabs(img[k] - mid);             /* models.py:154 */
            if (d > pk) pk = d;
          }
        }
        peak = pk;
        if (peak == 0.0) zero = 1;
      }
    }
    int bad = 0;
#pragma omp parallel for reduction(| : bad) schedule(static)
    for (int i = 0; i < H; ++i)
      for (int x = 0; x < W; ++x) {
        const size_t q = (size_t)i * W + x;
        double v;
        if (two_mean && zero) {
          v = 0.0;
        } else {
          double fx, fy;
          np_gradient(phi, H, W, i, x, &fx, &fy);
          double h = hypot(fx, fy);
          if (p->model == 3) v = (c->D[q] / peak) * h;
          else if (p->model == 1) v = (dc * (2.0 * img[q] - cp - cm) / peak) * h;
          else if (p->model == 2) v = (p->nu * ((img[q] - mid) / peak)) * h;   /* models.py:162 */
          else v = g[q] * h;
        }
        double out = phi[q] + p->dt * v;
        u[q] = out;
        bad |= !isfinite(out);
      }
    double* res = u;
    if (!bad) {
      if (p->reinit_period > 0 && it % p->reinit_period == 0) {
#pragma omp parallel for schedule(static)
        for (long long k = 0; k < (long long)n; ++k) u[k] = u[k] > 0.0 ? 1.0 : -1.0;
      }
      if (it % p->reg_period == 0) convolve_same(u, t, u, H, W, p->reg_w, p->ts_reg);
#pragma omp parallel for reduction(| : bad) schedule(static)
      for (long long k = 0; k < (long long)n; ++k) bad |= !isfinite(res[k]);
    }
    if (bad) {
      err = it;
      break;
    }
    memcpy(phi, res, n * sizeof(double));
    c->iteration = it;
    if (two_mean && zero) c->degenerate = 1;
    if (it % p->conv_check_every == 0) {
      const long long cw = p->conv_window;
      if (!c->ck) c->ck = (unsigned char*)malloc(n * (size_t)(cw + 1));
      unsigned char* slot = c->ck + (size_t)(c->n_ck % (cw + 1)) * n;
#pragma omp parallel for schedule(static)
      for (long long k = 0; k < (long long)n; ++k) slot[k] = phi[k] > 0.0;
      c->n_ck++;
      if (c->n_ck >= cw) {
        int eq = 1;
        for (long long j = 1; j < cw && eq; ++j) {
          const unsigned char* prev = c->ck + (size_t)((c->n_ck - 1 - j) % (cw + 1)) * n;
          eq = memcmp(prev, slot, n) == 0;
        }
        if (eq) c->converged = 1;
      }
    }
  }
  return err;
}

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
