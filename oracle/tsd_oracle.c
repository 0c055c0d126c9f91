/*
 * tsd_oracle.c -- CPU ORACLE (test infrastructure only; see tsd_oracle.h).
 *
 * Plain-C restatement of the reference hot path. Operation order follows the
 * reference line by line so that, compiled without FMA contraction
 * (oracle/Makefile: -ffp-contract=off, no -march), results are bit-identical
 * to the reference headers; tests/test_cpu.py
 * (test_oracle_restatement_is_bit_identical_to_reference) checks exactly that
 * against tests/golden/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.
 */
#include "tsd_oracle.h"

#include <float.h>
#include <pthread.h>
#include <stddef.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* 1 + tsdict::errc ordinal (reference include/tsdict/errors.hpp:13-35) */
enum {
  ST_OK = 0,
  ST_WINDOW_TOO_SMALL = 1,
  ST_WINDOW_TOO_LARGE = 2,
  ST_NON_FINITE_INPUT = 3,
  ST_LENGTH_MISMATCH = 4,
  ST_SERIES_TOO_SHORT = 5,
  ST_WINDOW_MISMATCH = 8,
  ST_EMPTY_DICTIONARY = 9,
  ST_INVALID_ARGUMENT = 16,
};

/* series.hpp:50-60 detail::kahan_sum */
typedef struct {
  double sum, comp;
} kahan;
static inline void kahan_add(kahan* k, double x) {
  double y = x - k->comp;
  double t = k->sum + y;
  k->comp = (t - k->sum) - y;
  k->sum = t;
}

/* series.hpp:75-77 */
static inline double constancy_threshold(double max_abs_sample) {
  return 1e-8 * (max_abs_sample > 1.0 ? max_abs_sample : 1.0);
}

/* series.hpp:83-150 compute_stats */
int tsdo_compute_stats(const double* x, size_t n, size_t m, double* means, double* stds, double* invn,
                       unsigned char* flat) {
  if (m < 2) return ST_WINDOW_TOO_SMALL;                     /* :85 */
  if (m > n) return ST_WINDOW_TOO_LARGE;                     /* :86 */
  for (size_t i = 0; i < n; ++i)                             /* :87, :62-68 */
    if (!isfinite(x[i])) return ST_NON_FINITE_INPUT;

  kahan total = {0.0, 0.0};                                  /* :89-94 */
  double max_abs = 0.0;
  for (size_t i = 0; i < n; ++i) {
    kahan_add(&total, x[i]);
    double ax = fabs(x[i]);
    max_abs = max_abs > ax ? max_abs : ax;
  }
  const double grand_mean = total.sum / (double)n;           /* :95 */

  double* ps1 = (double*)calloc(n + 1, sizeof(double));      /* :98-106 */
  double* ps2 = (double*)calloc(n + 1, sizeof(double));
  kahan s1 = {0.0, 0.0}, s2 = {0.0, 0.0};
  for (size_t i = 0; i < n; ++i) {
    const double c = x[i] - grand_mean;
    kahan_add(&s1, c);
    kahan_add(&s2, c * c);
    ps1[i + 1] = s1.sum;
    ps2[i + 1] = s2.sum;
  }

  const size_t cnt = n - m + 1;                              /* :108-110 */
  const double md = (double)m;
  const double eps = constancy_threshold(max_abs);
  for (size_t i = 0; i < cnt; ++i) {                         /* :118-148 */
    const double w1 = ps1[i + m] - ps1[i];
    const double w2 = ps2[i + m] - ps2[i];
    const double mean_c = w1 / md;
    double var = (w2 - w1 * mean_c) / md;
    if (var < 0.0) var = 0.0;
    double sd = sqrt(var);
    double mean = grand_mean + mean_c;
    const double cancel_err = 4.4e-16 * (ps2[i + m] + fabs(w1 * mean_c)) / md;
    if (sd * 1e-9 < cancel_err) {                            /* :130-142 two-pass fallback */
      kahan wsum = {0.0, 0.0};
      for (size_t t = 0; t < m; ++t) kahan_add(&wsum, x[i + t]);
      mean = wsum.sum / md;
      kahan wss = {0.0, 0.0};
      for (size_t t = 0; t < m; ++t) {
        const double d = x[i + t] - mean;
        kahan_add(&wss, d * d);
      }
      var = wss.sum / md;
      if (var < 0.0) var = 0.0;
      sd = sqrt(var);
    }
    means[i] = mean;
    stds[i] = sd;
    const int fl = sd < eps;
    flat[i] = fl ? 1 : 0;
    invn[i] = fl ? 0.0 : 1.0 / (sd * sqrt(md));
  }
  free(ps1);
  free(ps2);
  return ST_OK;
}

/* series.hpp:153-161 corr_to_dist */
double tsdo_corr_to_dist(double rho, size_t m) {
  if (rho > 1.0) rho = 1.0;
  if (rho < -1.0) rho = -1.0;
  double d = sqrt(2.0 * (double)m * (1.0 - rho));
  const double dmax = 2.0 * sqrt((double)m);
  if (d < 0.0) d = 0.0;
  if (d > dmax) d = dmax;
  return d;
}

/* profiles.hpp:70-77 acc_update: higher correlation wins, ties -> lower index */
static inline void acc_update(double* corr, int64_t* nn, size_t cell, double c, int64_t neighbor) {
  if (c > corr[cell] || (c == corr[cell] && neighbor < nn[cell])) {
    corr[cell] = c;
    nn[cell] = neighbor;
  }
}

/* profiles.hpp:89-99 make_diffs */
static void make_diffs(const double* v, size_t cnt, size_t m, const double* means, double* df, double* dg) {
  df[0] = 0.0;
  dg[0] = 0.0;
  for (size_t t = 1; t < cnt; ++t) {
    df[t] = 0.5 * (v[t + m - 1] - v[t - 1]);
    dg[t] = (v[t + m - 1] - means[t]) + (v[t - 1] - means[t - 1]);
  }
}

/* profiles.hpp:101-108 window_dot */
static inline double window_dot(const double* a, size_t ia, double mu_a, const double* b, size_t ib, double mu_b,
                                size_t m) {
  double acc = 0.0;
  for (size_t s = 0; s < m; ++s) acc += (a[ia + s] - mu_a) * (b[ib + s] - mu_b);
  return acc;
}

/* profiles.hpp:110-114 */
static inline double clamp_corr(double c) {
  if (c > 1.0) return 1.0;
  if (c < -1.0) return -1.0;
  return c;
}

/* profiles.hpp:142-158 finish_profile */
static void finish_profile(const double* corr, const int64_t* nn, size_t cells, size_t m, double* val, int64_t* idx) {
  for (size_t i = 0; i < cells; ++i) {
    if (nn[i] == -1) {
      val[i] = INFINITY;
      idx[i] = -1;
    } else {
      val[i] = tsdo_corr_to_dist(corr[i], m);
      idx[i] = nn[i];
    }
  }
}

typedef struct {
  double *means, *stds, *invn, *df, *dg;
  unsigned char* flat;
  size_t cnt;
} prepared;

static void prep_free(prepared* p) {
  free(p->means);
  free(p->stds);
  free(p->invn);
  free(p->df);
  free(p->dg);
  free(p->flat);
}

static int prep(const double* x, size_t n, size_t m, prepared* p) {
  memset(p, 0, sizeof *p);
  if (m < 2) return ST_WINDOW_TOO_SMALL;
  if (m > n) return ST_WINDOW_TOO_LARGE;
  p->cnt = n - m + 1;
  p->means = (double*)malloc(p->cnt * sizeof(double));
  p->stds = (double*)malloc(p->cnt * sizeof(double));
  p->invn = (double*)malloc(p->cnt * sizeof(double));
  p->df = (double*)malloc(p->cnt * sizeof(double));
  p->dg = (double*)malloc(p->cnt * sizeof(double));
  p->flat = (unsigned char*)malloc(p->cnt);
  int st = tsdo_compute_stats(x, n, m, p->means, p->stds, p->invn, p->flat);
  if (st != ST_OK) {
    prep_free(p);
    return st;
  }
  make_diffs(x, p->cnt, m, p->means, p->df, p->dg);
  return ST_OK;
}

/* profiles.hpp:306-342 ab_join, sequential diagonal order (threads = 1) */
int tsdo_ab_join(const double* a, size_t na, const double* b, size_t nb, size_t m, double* val, int64_t* idx) {
  if (m >= 2 && (na < m || nb < m)) return ST_SERIES_TOO_SHORT; /* :307-309 */
  prepared sa, sb;
  int st = prep(a, na, m, &sa);                                 /* :310 */
  if (st) return st;
  st = prep(b, nb, m, &sb);                                     /* :311 */
  if (st) {
    prep_free(&sa);
    return st;
  }
  const size_t ca = sa.cnt, cb = sb.cnt;
  double* corr = (double*)malloc(ca * sizeof(double));          /* :63-68 corr_acc */
  int64_t* nn = (int64_t*)malloc(ca * sizeof(int64_t));
  for (size_t i = 0; i < ca; ++i) {
    corr[i] = -2.0;
    nn[i] = -1;
  }
  const size_t ndiag = ca + cb - 1;                             /* :320 */
  for (size_t di = 0; di < ndiag; ++di) {                       /* :321-339 */
    const ptrdiff_t delta = (ptrdiff_t)di - (ptrdiff_t)(cb - 1);
    const size_t i0 = delta > 0 ? (size_t)delta : 0;
    const size_t j0 = delta > 0 ? 0 : (size_t)(-delta);
    const size_t la = ca - i0, lb = cb - j0;
    const size_t len = la < lb ? la : lb;
    double cov = window_dot(a, i0, sa.means[i0], b, j0, sb.means[j0], m);
    for (size_t s = 0; s < len; ++s) {
      const size_t i = i0 + s, j = j0 + s;
      if (s != 0) cov += sa.df[i] * sb.dg[j] + sa.dg[i] * sb.df[j];
      double c = cov * sa.invn[i] * sb.invn[j];
      if (sa.flat[i] && sb.flat[j]) {
        c = 1.0;
      } else {
        c = clamp_corr(c);
      }
      acc_update(corr, nn, i, c, (int64_t)j);
    }
  }
  finish_profile(corr, nn, ca, m, val, idx);                    /* :341 */
  free(corr);
  free(nn);
  prep_free(&sa);
  prep_free(&sb);
  return ST_OK;
}

/* profiles.hpp:266-301 self_join, excl parameterised (reference: m/2, :273) */
int tsdo_self_join(const double* t, size_t n, size_t m, size_t excl, double* val, int64_t* idx) {
  if (m >= 2 && n < 2 * m) return ST_SERIES_TOO_SHORT;          /* :268-270 */
  prepared s;
  int st = prep(t, n, m, &s);                                   /* :271 */
  if (st) return st;
  const size_t cnt = s.cnt;
  double* corr = (double*)malloc(cnt * sizeof(double));
  int64_t* nn = (int64_t*)malloc(cnt * sizeof(int64_t));
  for (size_t i = 0; i < cnt; ++i) {
    corr[i] = -2.0;
    nn[i] = -1;
  }
  const size_t ndiag = cnt > excl + 1 ? cnt - excl - 1 : 0;     /* :282 */
  for (size_t di = 0; di < ndiag; ++di) {                       /* :283-298 */
    const size_t d = excl + 1 + di;
    double cov = window_dot(t, 0, s.means[0], t, d, s.means[d], m);
    const size_t len = cnt - d;
    for (size_t q = 0; q < len; ++q) {
      if (q != 0) cov += s.df[q] * s.dg[q + d] + s.df[q + d] * s.dg[q];
      double c = cov * s.invn[q] * s.invn[q + d];
      if (s.flat[q] && s.flat[q + d]) {
        c = 1.0;
      } else {
        c = clamp_corr(c);
      }
      acc_update(corr, nn, q, c, (int64_t)(q + d));
      acc_update(corr, nn, q + d, c, (int64_t)q);
    }
  }
  finish_profile(corr, nn, cnt, m, val, idx);
  free(corr);
  free(nn);
  prep_free(&s);
  return ST_OK;
}

/* profiles.hpp:118-140 run_diagonals + :266-301 self_join with `threads`
 * host threads: thread w walks diagonals di = w, w + T, ... into its own
 * accumulator; the accumulators are merged in thread order with acc_merge's
 * rule (profiles.hpp:79-85), so the result is bit-identical to threads = 1
 * (profiles.hpp:12-17). Exclusion zone as a parameter, as tsdo_self_join. */
typedef struct {
  const double* t;
  const prepared* s;
  size_t m, excl, ndiag, w, nthreads;
  double* corr;
  int64_t* nn;
} sj_task;

static void* sj_worker(void* arg) {
  sj_task* k = (sj_task*)arg;
  const prepared* s = k->s;
  const size_t cnt = s->cnt;
  for (size_t i = 0; i < cnt; ++i) {
    k->corr[i] = -2.0;
    k->nn[i] = -1;
  }
  for (size_t di = k->w; di < k->ndiag; di += k->nthreads) {
    const size_t d = k->excl + 1 + di;
    double cov = window_dot(k->t, 0, s->means[0], k->t, d, s->means[d], k->m);
    const size_t len = cnt - d;
    for (size_t q = 0; q < len; ++q) {
      if (q != 0) cov += s->df[q] * s->dg[q + d] + s->df[q + d] * s->dg[q];
      double c = cov * s->invn[q] * s->invn[q + d];
      if (s->flat[q] && s->flat[q + d]) {
        c = 1.0;
      } else {
        c = clamp_corr(c);
      }
      acc_update(k->corr, k->nn, q, c, (int64_t)(q + d));
      acc_update(k->corr, k->nn, q + d, c, (int64_t)q);
    }
  }
  return NULL;
}

int tsdo_self_join_mt(const double* t, size_t n, size_t m, size_t excl, unsigned threads, double* val,
                      int64_t* idx) {
  if (m >= 2 && n < 2 * m) return ST_SERIES_TOO_SHORT;
  prepared s;
  int st = prep(t, n, m, &s);
  if (st) return st;
  const size_t cnt = s.cnt;
  const size_t ndiag = cnt > excl + 1 ? cnt - excl - 1 : 0;
  size_t T = threads ? threads : 1;
  if (T > ndiag) T = ndiag ? ndiag : 1;
  sj_task* tasks = (sj_task*)calloc(T, sizeof(sj_task));
  pthread_t* th = (pthread_t*)calloc(T, sizeof(pthread_t));
  for (size_t w = 0; w < T; ++w) {
    tasks[w] = (sj_task){t, &s, m, excl, ndiag, w, T, (double*)malloc(cnt * sizeof(double)),
                         (int64_t*)malloc(cnt * sizeof(int64_t))};
    pthread_create(&th[w], NULL, sj_worker, &tasks[w]);
  }
  for (size_t w = 0; w < T; ++w) pthread_join(th[w], NULL);
  for (size_t w = 1; w < T; ++w) /* acc_merge in thread order */
    for (size_t i = 0; i < cnt; ++i)
      acc_update(tasks[0].corr, tasks[0].nn, i, tasks[w].corr[i], tasks[w].nn[i]);
  finish_profile(tasks[0].corr, tasks[0].nn, cnt, m, val, idx);
  for (size_t w = 0; w < T; ++w) {
    free(tasks[w].corr);
    free(tasks[w].nn);
  }
  free(tasks);
  free(th);
  prep_free(&s);
  return ST_OK;
}

/* Rows r0 .. r0+nr-1 of the self-join profile (profiles.hpp:266-301 with the
 * exclusion zone as a parameter), for checking large self-joins on sampled
 * row blocks: every diagonal delta = j - i with |delta| > excl that crosses
 * the block starts at the block's first row on it with window_dot
 * (profiles.hpp:101-108) and follows the reference's recurrence (:288, lower
 * window index first) down the block; correlation, flat rule, clamp and
 * acc_update as :289-296. The values differ from a whole-series run only by
 * the recurrence's rounding (its diagonals start at row 0 in the reference). */
int tsdo_self_join_rows(const double* t, size_t n, size_t m, size_t excl, size_t r0, size_t nr, double* val,
                        int64_t* idx) {
  if (m >= 2 && n < 2 * m) return ST_SERIES_TOO_SHORT;
  prepared s;
  int st = prep(t, n, m, &s);
  if (st) return st;
  const size_t cnt = s.cnt;
  if (r0 >= cnt || nr == 0) {
    prep_free(&s);
    return ST_INVALID_ARGUMENT;
  }
  if (r0 + nr > cnt) nr = cnt - r0;
  double* corr = (double*)malloc(nr * sizeof(double));
  int64_t* nn = (int64_t*)malloc(nr * sizeof(int64_t));
  for (size_t i = 0; i < nr; ++i) {
    corr[i] = -2.0;
    nn[i] = -1;
  }
  /* delta from -(r0 + nr - 1) to cnt - 1 - r0 */
  const ptrdiff_t dlo = -(ptrdiff_t)(r0 + nr - 1), dhi = (ptrdiff_t)(cnt - 1 - r0);
  for (ptrdiff_t delta = dlo; delta <= dhi; ++delta) {
    const size_t ad = (size_t)(delta < 0 ? -delta : delta);
    if (ad <= excl) continue;
    size_t i = r0;
    if (delta < 0 && (size_t)(-delta) > i) i = (size_t)(-delta);
    size_t iend = r0 + nr;
    if (delta > 0 && cnt - (size_t)delta < iend) iend = cnt - (size_t)delta;
    if (i >= iend) continue;
    const size_t q0 = delta > 0 ? i : i - ad; /* lower window of the pair */
    double cov = window_dot(t, q0, s.means[q0], t, q0 + ad, s.means[q0 + ad], m);
    for (size_t q = q0; i < iend; ++i, ++q) {
      if (q != q0) cov += s.df[q] * s.dg[q + ad] + s.df[q + ad] * s.dg[q];
      double c = cov * s.invn[q] * s.invn[q + ad];
      if (s.flat[q] && s.flat[q + ad]) {
        c = 1.0;
      } else {
        c = clamp_corr(c);
      }
      acc_update(corr, nn, i - r0, c, (int64_t)(delta > 0 ? q + ad : q));
    }
  }
  finish_profile(corr, nn, nr, m, val, idx);
  free(corr);
  free(nn);
  prep_free(&s);
  return ST_OK;
}

/* dictionary.hpp:149-193 dict_min_profile (join_dictionary's m == D.m check,
 * dict_join.hpp:44-46, is the caller's job) */
int tsdo_dict_join(const double* q, size_t nq, const double* seg_vals, const size_t* seg_len,
                   const size_t* seg_start, size_t nseg, size_t m, double* val, int64_t* idx) {
  if (nseg == 0) return ST_EMPTY_DICTIONARY;                    /* :151 */
  for (size_t s = 0; s < nseg; ++s)                             /* :152-156 */
    if (seg_len[s] < m) return ST_WINDOW_MISMATCH;
  if (m < 2) return ST_WINDOW_TOO_SMALL;                        /* :157 */
  if (m > nq) return ST_WINDOW_TOO_LARGE;                       /* :158 */

  size_t* seg_off = (size_t*)malloc(nseg * sizeof(size_t));
  size_t off = 0;
  size_t maxc = 0;
  for (size_t s = 0; s < nseg; ++s) {
    seg_off[s] = off;
    off += seg_len[s];
    if (seg_len[s] - m + 1 > maxc) maxc = seg_len[s] - m + 1;
  }
  const size_t cnt = nq - m + 1;                                /* :164-169 */
  for (size_t i = 0; i < cnt; ++i) {
    val[i] = INFINITY;
    idx[i] = -1;
  }
  const size_t block = 16384;                                   /* :175 */
  double* pv = (double*)malloc((block < cnt ? block : cnt) * sizeof(double));
  int64_t* pi = (int64_t*)malloc((block < cnt ? block : cnt) * sizeof(int64_t));
  int st = ST_OK;
  for (size_t c0 = 0; c0 < cnt && st == ST_OK; c0 += block) {   /* :176-191 */
    const size_t c1 = cnt < c0 + block ? cnt : c0 + block;
    const double* chunk = q + c0;
    const size_t chunk_n = c1 - 1 + m - c0;
    for (size_t s = 0; s < nseg; ++s) {
      st = tsdo_ab_join(chunk, chunk_n, seg_vals + seg_off[s], seg_len[s], m, pv, pi); /* :182 */
      if (st) break;
      const int64_t offset = (int64_t)seg_start[s];
      for (size_t i = 0; i < c1 - c0; ++i) {                    /* :184-189 strict < */
        if (pv[i] < val[c0 + i]) {
          val[c0 + i] = pv[i];
          idx[c0 + i] = pi[i] + offset;
        }
      }
    }
  }
  free(pv);
  free(pi);
  free(seg_off);
  return st;
}

/* ---------------------------------------------------------------------------
 * long-double brute force, tests/oracles.hpp
 * ------------------------------------------------------------------------- */

typedef struct {
  long double *mean, *sd;
  unsigned char* flat;
} lstats;

/* oracles.hpp:28-51 stats_of */
static void stats_of(const double* v, size_t n, size_t m, lstats* ws) {
  const size_t cnt = n - m + 1;
  double max_abs = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double ax = fabs(v[i]);
    max_abs = max_abs > ax ? max_abs : ax;
  }
  const long double eps = constancy_threshold(max_abs);
  ws->mean = (long double*)malloc(cnt * sizeof(long double));
  ws->sd = (long double*)malloc(cnt * sizeof(long double));
  ws->flat = (unsigned char*)malloc(cnt);
  for (size_t i = 0; i < cnt; ++i) {
    long double s = 0.0L;
    for (size_t t = 0; t < m; ++t) s += v[i + t];
    const long double mu = s / (long double)m;
    long double qq = 0.0L;
    for (size_t t = 0; t < m; ++t) {
      const long double d = v[i + t] - mu;
      qq += d * d;
    }
    ws->mean[i] = mu;
    ws->sd[i] = sqrtl(qq / (long double)m);
    ws->flat[i] = ws->sd[i] < eps;
  }
}

static void lstats_free(lstats* w) {
  free(w->mean);
  free(w->sd);
  free(w->flat);
}

/* oracles.hpp:55-70 pair_dist */
static double pair_dist_ws(const double* a, size_t i, const lstats* wa, const double* b, size_t j, const lstats* wb,
                           size_t m) {
  const long double cap = 2.0L * sqrtl((long double)m);
  if (wa->flat[i] && wb->flat[j]) return 0.0;
  if (wa->flat[i] || wb->flat[j]) return sqrt(2.0 * (double)m);
  long double acc = 0.0L;
  for (size_t t = 0; t < m; ++t) {
    const long double za = (a[i + t] - wa->mean[i]) / wa->sd[i];
    const long double zb = (b[j + t] - wb->mean[j]) / wb->sd[j];
    const long double d = za - zb;
    acc += d * d;
  }
  long double d = sqrtl(acc);
  if (d > cap) d = cap;
  return (double)d;
}

/* single pair: same arithmetic as oracles.hpp:55-70 with stats_of's
 * series-wide flat threshold (oracles.hpp:30-32), only the two windows' moments */
double tsdo_pair_dist(const double* a, size_t na, size_t i, const double* b, size_t nb, size_t j, size_t m) {
  lstats wa, wb;
  /* restrict stats_of to the single window while keeping the series-wide threshold */
  double max_a = 0.0, max_b = 0.0;
  for (size_t t = 0; t < na; ++t) max_a = fabs(a[t]) > max_a ? fabs(a[t]) : max_a;
  for (size_t t = 0; t < nb; ++t) max_b = fabs(b[t]) > max_b ? fabs(b[t]) : max_b;
  stats_of(a + i, m, m, &wa);
  stats_of(b + j, m, m, &wb);
  wa.flat[0] = wa.sd[0] < (long double)constancy_threshold(max_a);
  wb.flat[0] = wb.sd[0] < (long double)constancy_threshold(max_b);
  double d = pair_dist_ws(a + i, 0, &wa, b + j, 0, &wb, m);
  lstats_free(&wa);
  lstats_free(&wb);
  return d;
}

/* oracles.hpp:115-136 ab_join_brute */
int tsdo_ab_join_brute(const double* a, size_t na, const double* b, size_t nb, size_t m, double* val,
                       int64_t* idx) {
  if (m < 2) return ST_WINDOW_TOO_SMALL;
  if (na < m || nb < m) return ST_SERIES_TOO_SHORT;
  lstats wa, wb;
  stats_of(a, na, m, &wa);
  stats_of(b, nb, m, &wb);
  const size_t ca = na - m + 1, cb = nb - m + 1;
  for (size_t i = 0; i < ca; ++i) {
    val[i] = INFINITY;
    idx[i] = -1;
    for (size_t j = 0; j < cb; ++j) {
      const double d = pair_dist_ws(a, i, &wa, b, j, &wb, m);
      if (d < val[i]) {
        val[i] = d;
        idx[i] = (int64_t)j;
      }
    }
  }
  lstats_free(&wa);
  lstats_free(&wb);
  return ST_OK;
}

/* oracles.hpp:92-113 self_join_brute, exclusion parameterised */
int tsdo_self_join_brute(const double* t, size_t n, size_t m, size_t excl, double* val, int64_t* idx) {
  if (m < 2) return ST_WINDOW_TOO_SMALL;
  if (n < m) return ST_SERIES_TOO_SHORT;
  lstats ws;
  stats_of(t, n, m, &ws);
  const size_t cnt = n - m + 1;
  for (size_t i = 0; i < cnt; ++i) {
    val[i] = INFINITY;
    idx[i] = -1;
    for (size_t j = 0; j < cnt; ++j) {
      const size_t gap = i > j ? i - j : j - i;
      if (gap <= excl) continue;
      const double d = pair_dist_ws(t, i, &ws, t, j, &ws, m);
      if (d < val[i]) {
        val[i] = d;
        idx[i] = (int64_t)j;
      }
    }
  }
  lstats_free(&ws);
  return ST_OK;
}
