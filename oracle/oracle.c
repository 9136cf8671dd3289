/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the cubic-spline
 * hot path of Hornbeck, "Fast Cubic Spline Interpolation" (arXiv 2001.09253).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2001_09253_b200/) never imports, links or calls it,
 * and shares no code, header, table or constant with it.
 *
 * Citations: "P:<line>" is a line of the paper text.
 *
 * Everything is computed in IEEE binary64 (fp32 inputs are widened exactly by
 * the caller).  Built with -O2 -ffp-contract=off and no -ffast-math, so every
 * expression below is evaluated exactly as written, one rounding per operation.
 *
 * Functions:
 *   oracle_build  -- the paper's new_second_derivative() sweep,
 *                    its sentinel test generalised to per-end bc bits.
 *   oracle_locate -- textbook bisection: the largest j in [0, n-2] with
 *                    x_j <= q (reading c1 of DESIGN.md); -1 outside [x_0, x_{n-1}]
 *                    or NaN (Eq. nr_formula requires x_j <= x <= x_{j+1}).
 *   oracle_interp -- Eq. nr_formula, the A/B/C/D form.
 *   *_batch       -- loops of the above over independent curves (optionally
 *                    over POSIX threads; each curve stays sequential).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_BC_CLAMP_START 1
#define ORACLE_BC_CLAMP_END 2

/* Returns 0 on success, -1 for an invalid argument (n < 3), and 1 for
 * bad data (knots not strictly increasing or not finite; non-finite
 * values or clamped slopes), in which case y2 is filled with NaN. */
int oracle_build(const double *knots, const double *values, int64_t n, int bc,
                 double start_deriv, double end_deriv, double *ypp) {
  if (n < 3) return -1;
  /* assert len(knots) > 2 and strictly increasing knots. */
  int bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(knots[i]) || !isfinite(values[i])) bad = 1;
    if (i > 0 && !(knots[i] > knots[i - 1])) bad = 1;
  }
  if ((bc & ORACLE_BC_CLAMP_START) && !isfinite(start_deriv)) bad = 1;
  if ((bc & ORACLE_BC_CLAMP_END) && !isfinite(end_deriv)) bad = 1;
  if (bad) {
    for (int64_t i = 0; i < n; ++i) ypp[i] = NAN;
    return 1;
  }

  /* c_p = [0]*n (the one scratch list of P:723-728); d' lives in ypp. */
  double *c_p = (double *)malloc((size_t)n * sizeof(double));
  if (!c_p) return -1;

  /* recycle these values in later routines. */
  double new_x = knots[1];
  double new_y = values[1];
  double cj = knots[1] - knots[0];
  double new_dj = (values[1] - values[0]) / cj;

  /* initialise the forward substitution. */
  if (!(bc & ORACLE_BC_CLAMP_START)) { /* natural: start_deriv > .99e30 */
    c_p[0] = 0;
    ypp[0] = 0;
  } else { /* clamped start row */
    c_p[0] = 0.5;
    ypp[0] = 3 * (new_dj - start_deriv) / cj;
  }

  /* forward substitution portion. */
  int64_t j = 1;
  while (j < (n - 1)) {
    double old_x = new_x;
    double old_y = new_y;
    double aj = cj;
    double old_dj = new_dj;

    new_x = knots[j + 1];
    new_y = values[j + 1];

    cj = new_x - old_x;
    new_dj = (new_y - old_y) / cj;
    double bj = 2 * (cj + aj);
    double inv_denom = 1. / (bj - aj * c_p[j - 1]);
    double dj = 6 * (new_dj - old_dj);

    ypp[j] = (dj - aj * ypp[j - 1]) * inv_denom;
    c_p[j] = cj * inv_denom;
    j += 1;
  }

  /* handle the end derivative. */
  if (!(bc & ORACLE_BC_CLAMP_END)) { /* natural */
    c_p[j] = 0;
    ypp[j] = 0;
  } else { /* clamped end row, P:1017-1018 (a_n = h, b_n = 2h; reading c4) */
    double aj = cj;
    double old_dj = new_dj;
    cj = 0; /* "this has the same effect as skipping c_n" */
    new_dj = end_deriv;
    double bj = 2 * (cj + aj);
    double inv_denom = 1. / (bj - aj * c_p[j - 1]);
    double dj = 6 * (new_dj - old_dj);
    ypp[j] = (dj - aj * ypp[j - 1]) * inv_denom;
    c_p[j] = cj * inv_denom;
  }

  /* backward substitution portion (y''_n = d'_n is a no-op). */
  while (j > 0) {
    j -= 1;
    ypp[j] = ypp[j] - c_p[j] * ypp[j + 1];
  }
  free(c_p);
  return 0;
}

/* Textbook bisection (not shared with any GPU search).  Reading c1: the
 * interval of q is the largest j in [0, n-2] with x_j <= q; q = x_{n-1} maps
 * to n-2.  Outside [x_0, x_{n-1}] or NaN: -1 (P:276 requires x_j <= x <= x_{j+1}). */
int64_t oracle_locate(const double *x, int64_t n, double q) {
  if (!(q >= x[0]) || !(q <= x[n - 1])) return -1; /* also catches NaN */
  int64_t lo = 0, hi = n - 1;                       /* x[lo] <= q, and hi == n-1 or x[hi] > q */
  while (hi - lo > 1) {
    int64_t mid = lo + (hi - lo) / 2;
    if (x[mid] <= q) lo = mid;
    else hi = mid;
  }
  return lo;
}

/* Eq. nr_formula: y = A y_j + B y_{j+1} + C y''_j + D y''_{j+1}. */
double oracle_interp(double q, const double *x, const double *y, const double *ypp, int64_t j) {
  double h = x[j + 1] - x[j];
  double A = (x[j + 1] - q) / h;
  double B = (q - x[j]) / h;
  double C = (A * A * A - A) * (h * h) / 6;
  double D = (B * B * B - B) * (h * h) / 6;
  return A * y[j] + B * y[j + 1] + C * ypp[j] + D * ypp[j + 1];
}

/* ------------------------------------------------------------------ batches */

typedef struct {
  const double *x, *y, *yp1, *ypn, *y2c, *q;
  double *y2, *out;
  int64_t *idx;
  int64_t n, m, c0, c1;
  int bc;
  int nbad;
} job_t;

static void *build_worker(void *arg) {
  job_t *J = (job_t *)arg;
  J->nbad = 0;
  for (int64_t c = J->c0; c < J->c1; ++c) {
    double s = (J->bc & ORACLE_BC_CLAMP_START) ? J->yp1[c] : 0.0;
    double e = (J->bc & ORACLE_BC_CLAMP_END) ? J->ypn[c] : 0.0;
    int r = oracle_build(J->x + c * J->n, J->y + c * J->n, J->n, J->bc, s, e, J->y2 + c * J->n);
    if (r != 0) J->nbad++;
  }
  return NULL;
}

static void *eval_worker(void *arg) {
  /* [c0, c1) is a range of flattened (curve, query) positions here. */
  job_t *J = (job_t *)arg;
  J->nbad = 0;
  for (int64_t f = J->c0; f < J->c1; ++f) {
    int64_t c = f / J->m;
    const double *xc = J->x + c * J->n, *yc = J->y + c * J->n, *zc = J->y2c + c * J->n;
    double q = J->q[f];
    int64_t j = oracle_locate(xc, J->n, q);
    J->idx[f] = j;
    if (j < 0) {
      J->out[f] = NAN;
      J->nbad++;
    } else {
      J->out[f] = oracle_interp(q, xc, yc, zc, j);
    }
  }
  return NULL;
}

static int run_jobs(job_t *proto, int64_t batch, int nthreads, void *(*fn)(void *)) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > batch) nthreads = (int)(batch > 0 ? batch : 1);
  job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  int total = 0;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *proto;
    jobs[t].c0 = batch * t / nthreads;
    jobs[t].c1 = batch * (t + 1) / nthreads;
  }
  if (nthreads == 1) {
    fn(&jobs[0]);
  } else {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < nthreads; ++t) total += jobs[t].nbad;
  free(jobs);
  free(th);
  return total;
}

/* Returns the number of curves with bad data (y2 NaN-filled), or -1 for n < 3. */
int oracle_build_batch(const double *x, const double *y, int64_t n, int64_t batch, int bc,
                       const double *yp1, const double *ypn, double *y2, int nthreads) {
  if (n < 3) return -1;
  job_t J = {0};
  J.x = x; J.y = y; J.n = n; J.bc = bc; J.yp1 = yp1; J.ypn = ypn; J.y2 = y2;
  return run_jobs(&J, batch, nthreads, build_worker);
}

/* Returns the number of out-of-range / NaN queries (idx -1, out NaN). */
int oracle_eval_batch(const double *x, const double *y, const double *y2, int64_t n, int64_t batch,
                      const double *q, int64_t m, double *out, int64_t *idx, int nthreads) {
  job_t J = {0};
  if (m <= 0 || batch <= 0) return 0;
  J.x = x; J.y = y; J.y2c = y2; J.n = n; J.q = q; J.m = m; J.out = out; J.idx = idx;
  return run_jobs(&J, batch * m, nthreads, eval_worker);
}
