/* agk_oracle.c — CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 * See agk_oracle.h for scope and the reference file:line each part follows. Every floating
 * point expression keeps the reference's evaluation order so that, built with -O3 -DNDEBUG
 * (no FMA contraction on baseline x86-64), results are bitwise equal to oracle/_ref. */
#include "agk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- FFT (fft.cpp:15-137) */

static size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

typedef struct {
  size_t n;
  size_t* bitrev;
  double* tw; /* interleaved (cos, sin)(-2 pi k / n), k < n/2 (fft.cpp:80-84) */
} fft_plan;

static int plan_init(fft_plan* p, size_t n) {
  p->n = n;
  p->bitrev = (size_t*)malloc(n * sizeof(size_t));
  p->tw = (double*)malloc((n / 2 + 1) * 2 * sizeof(double));
  if (!p->bitrev || !p->tw) return -1;
  size_t log2n = 0;
  while (((size_t)1 << log2n) < n) ++log2n;
  for (size_t i = 0; i < n; ++i) {
    size_t rev = 0;
    for (size_t b = 0; b < log2n; ++b)
      if (i & ((size_t)1 << b)) rev |= (size_t)1 << (log2n - 1 - b);
    p->bitrev[i] = rev;
  }
  for (size_t k = 0; k < n / 2; ++k) {
    const double phi = -2.0 * M_PI * (double)k / (double)n;
    p->tw[2 * k] = cos(phi);
    p->tw[2 * k + 1] = sin(phi);
  }
  return 0;
}

static void plan_free(fft_plan* p) {
  free(p->bitrev);
  free(p->tw);
}

/* Iterative radix-2 DIT on interleaved re/im (fft.cpp:86-132). */
static void plan_transform(const fft_plan* p, double* a, int invert) {
  const size_t n = p->n;
  for (size_t i = 0; i < n; ++i) {
    const size_t j = p->bitrev[i];
    if (i < j) {
      double t = a[2 * i]; a[2 * i] = a[2 * j]; a[2 * j] = t;
      t = a[2 * i + 1]; a[2 * i + 1] = a[2 * j + 1]; a[2 * j + 1] = t;
    }
  }
  for (size_t i = 0; i + 1 < n; i += 2) {
    const double ur = a[2 * i], ui = a[2 * i + 1];
    const double vr = a[2 * i + 2], vi = a[2 * i + 3];
    a[2 * i] = ur + vr;
    a[2 * i + 1] = ui + vi;
    a[2 * i + 2] = ur - vr;
    a[2 * i + 3] = ui - vi;
  }
  const double sign = invert ? -1.0 : 1.0;
  for (size_t len = 4; len <= n; len <<= 1) {
    const size_t half = len / 2, step = n / len;
    for (size_t base = 0; base < n; base += len) {
      double* lo = a + 2 * base;
      double* hi = a + 2 * (base + half);
      for (size_t j = 0; j < half; ++j) {
        const double wr = p->tw[2 * j * step];
        const double wi = sign * p->tw[2 * j * step + 1];
        const double xr = hi[2 * j], xi = hi[2 * j + 1];
        const double vr = xr * wr - xi * wi;
        const double vi = xr * wi + xi * wr;
        const double ur = lo[2 * j], ui = lo[2 * j + 1];
        lo[2 * j] = ur + vr;
        lo[2 * j + 1] = ui + vi;
        hi[2 * j] = ur - vr;
        hi[2 * j + 1] = ui - vi;
      }
    }
  }
  if (invert) {
    const double scale = 1.0 / (double)n;
    for (size_t i = 0; i < 2 * n; ++i) a[i] *= scale;
  }
}

/* ---------------------------------------------------------------- RHS (rhs.cpp) */

static int model_ok(const ora_model* md) {
  return md && md->m >= 2 && (md->k || (md->r >= 1 && md->u && md->v));
}

/* K(i,j) of a DenseKernel (kernels.hpp:42), 1-based */
static double dense_at(const ora_model* md, size_t i, size_t j) { return md->k[(i - 1) * md->m + (j - 1)]; }

/* kernel_row_sums (rhs.cpp:24-46): low-rank branch 27-36, dense branch 37-45 */
static void row_sums(const ora_model* md, const double* n, double* rowsum) {
  const size_t m = md->m, r = md->r;
  if (md->k) {
    for (size_t s = 0; s < m; ++s) {
      const double* row = md->k + s * m;
      double acc = 0.0;
      for (size_t j = 0; j < m; ++j) acc += row[j] * n[j];
      rowsum[s] = acc;
    }
    return;
  }
  for (size_t s = 0; s < m; ++s) rowsum[s] = 0.0;
  for (size_t a = 0; a < r; ++a) {
    double w = 0.0;
    const double* vrow = md->v + a * m;
    for (size_t j = 0; j < m; ++j) w += vrow[j] * n[j];
    const double* ucol = md->u + a;
    for (size_t s = 0; s < m; ++s) rowsum[s] += ucol[s * r] * w;
  }
}

/* U column a equals `other` (stride) bitwise-as-double (rhs.cpp:103-108) */
static int ucol_equals(const ora_model* md, size_t a, const double* other, size_t stride) {
  for (size_t i = 0; i < md->m; ++i)
    if (md->u[i * md->r + a] != other[i * stride]) return 0;
  return 1;
}

/* Rank dedupe of birth_term (rhs.cpp:96-124): skip[a] set when rank a repeats an earlier
 * unskipped rank b directly or swapped; weight[b] counts the folded copies. */
static void dedupe(const ora_model* md, double* weight, unsigned char* skip) {
  const size_t m = md->m, r = md->r;
  for (size_t a = 0; a < r; ++a) { weight[a] = 1.0; skip[a] = 0; }
  for (size_t a = 1; a < r; ++a) {
    for (size_t b = 0; b < a; ++b) {
      if (skip[b]) continue;
      const int swapped = ucol_equals(md, a, md->v + b * m, 1) && ucol_equals(md, b, md->v + a * m, 1);
      int same = ucol_equals(md, a, md->u + b, r);
      if (same) {
        for (size_t j = 0; j < m; ++j)
          if (md->v[a * m + j] != md->v[b * m + j]) { same = 0; break; }
      }
      if (swapped || same) {
        weight[b] += 1.0;
        skip[a] = 1;
        break;
      }
    }
  }
}

#ifndef ORA_PAD_FACTOR
#define ORA_PAD_FACTOR 1 /* 2: an equally valid variant with a twice longer FFT (noise-floor build) */
#endif

int ora_birth_term(const ora_model* md, const double* n, double* out) {
  if (!model_ok(md)) return -1;
  const size_t m = md->m, r = md->r;
  if (md->k) { /* dense branch (rhs.cpp:153-159) */
    out[0] = 0.0;
    for (size_t s = 2; s <= m; ++s) {
      double acc = 0.0;
      for (size_t i = 1; i < s; ++i) acc += dense_at(md, i, s - i) * n[i - 1] * n[s - i - 1];
      out[s - 1] = 0.5 * acc;
    }
    return 0;
  }
  const size_t padded = next_pow2(2 * m) * ORA_PAD_FACTOR;
  fft_plan plan;
  if (plan_init(&plan, padded)) return -1;
  double* packed = (double*)malloc(2 * padded * sizeof(double));
  double* acc = (double*)calloc(2 * padded, sizeof(double));
  double* weight = (double*)malloc(r * sizeof(double));
  unsigned char* skip = (unsigned char*)malloc(r);
  dedupe(md, weight, skip);
  for (size_t a = 0; a < r; ++a) {
    if (skip[a]) continue;
    for (size_t i = 0; i < m; ++i) { /* rhs.cpp:131-133 */
      packed[2 * i] = md->u[i * r + a] * n[i];
      packed[2 * i + 1] = md->v[a * m + i] * n[i];
    }
    for (size_t i = m; i < padded; ++i) packed[2 * i] = packed[2 * i + 1] = 0.0;
    plan_transform(&plan, packed, 0);
    const double w = weight[a];
    for (size_t k = 0; k < padded; ++k) { /* rhs.cpp:138-144, std::complex arithmetic */
      const size_t mk = (padded - k) & (padded - 1);
      const double zr = packed[2 * k], zi = packed[2 * k + 1];
      const double mr = packed[2 * mk], mi = -packed[2 * mk + 1]; /* conj */
      const double ar = 0.5 * (zr + mr), ai = 0.5 * (zi + mi);
      const double dr = zr - mr, di = zi - mi;
      const double br = 0.0 * dr - (-0.5) * di, bi = 0.0 * di + (-0.5) * dr; /* (0,-0.5)*d */
      const double pr = ar * br - ai * bi, pi = ar * bi + ai * br;
      acc[2 * k] += w * pr;
      acc[2 * k + 1] += w * pi;
    }
  }
  plan_transform(&plan, acc, 1);
  out[0] = 0.0;
  for (size_t s = 2; s <= m; ++s) out[s - 1] = 0.5 * acc[2 * (s - 2)];
  free(packed); free(acc); free(weight); free(skip);
  plan_free(&plan);
  return 0;
}

int ora_death_term(const ora_model* md, const double* n, double* out) {
  if (!model_ok(md)) return -1;
  double* rowsum = (double*)malloc(md->m * sizeof(double));
  row_sums(md, n, rowsum);
  for (size_t s = 0; s < md->m; ++s) out[s] = n[s] * rowsum[s];
  free(rowsum);
  return 0;
}

int ora_shattering_terms(const ora_model* md, const double* n, double lambda, double* out) {
  if (!model_ok(md)) return -1;
  if (!isfinite(lambda) || lambda < 0.0) return -1;
  const size_t m = md->m, r = md->r;
  double* rowsum = (double*)malloc(m * sizeof(double));
  row_sums(md, n, rowsum);
  double pair_gain = 0.0, mono_gain = 0.0;
  if (md->k) { /* dense branch (rhs.cpp:197-205) */
    for (size_t i = 2; i <= m; ++i)
      for (size_t j = 2; j <= m; ++j) pair_gain += (double)(i + j) * dense_at(md, i, j) * n[i - 1] * n[j - 1];
    for (size_t j = 2; j <= m; ++j) mono_gain += (double)j * dense_at(md, 1, j) * n[j - 1];
  }
  for (size_t a = 0; a < (md->k ? 0 : r); ++a) { /* rhs.cpp:185-196 */
    double su0 = 0.0, su1 = 0.0, sv0 = 0.0, sv1 = 0.0;
    for (size_t i = 2; i <= m; ++i) {
      const double size = (double)i;
      const double u = md->u[(i - 1) * r + a], v = md->v[a * m + (i - 1)];
      su0 += u * n[i - 1];
      su1 += size * u * n[i - 1];
      sv0 += v * n[i - 1];
      sv1 += size * v * n[i - 1];
    }
    pair_gain += su1 * sv0 + su0 * sv1;
    mono_gain += md->u[a] * sv1;
  }
  out[0] = 0.5 * lambda * pair_gain + lambda * n[0] * mono_gain;
  for (size_t s = 2; s <= m; ++s) out[s - 1] = -lambda * n[s - 1] * rowsum[s - 1];
  free(rowsum);
  return 0;
}

static int sources_ok(const ora_model* md) {
  for (size_t q = 0; q < md->num_sources; ++q) {
    if (md->source_k[q] < 1 || md->source_k[q] > md->m) return 0;
    if (!isfinite(md->source_rate[q]) || md->source_rate[q] < 0.0) return 0;
  }
  return 1;
}

int ora_eval_rhs(const ora_model* md, const double* n, double* out) {
  if (!model_ok(md)) return -1;
  const size_t m = md->m;
  if (md->variant == ORA_AGGREGATION_SOURCES && !sources_ok(md)) return -1;
  double* birth = (double*)malloc(m * sizeof(double));
  double* death = (double*)malloc(m * sizeof(double));
  int rc = ora_birth_term(md, n, birth);
  if (!rc) rc = ora_death_term(md, n, death);
  if (!rc) {
    for (size_t s = 0; s < m; ++s) out[s] = birth[s] - death[s];
    if (md->variant == ORA_AGGREGATION_SOURCES) {
      for (size_t q = 0; q < md->num_sources; ++q) out[md->source_k[q] - 1] += md->source_rate[q];
    } else if (md->variant == ORA_AGGREGATION_SHATTERING) {
      rc = ora_shattering_terms(md, n, md->shatter_rate, birth);
      if (!rc) for (size_t s = 0; s < m; ++s) out[s] += birth[s];
    }
  }
  free(birth); free(death);
  return rc;
}

static double entry(const ora_model* md, size_t i, size_t j) {
  if (md->k) return dense_at(md, i, j);
  double acc = 0.0;
  for (size_t a = 0; a < md->r; ++a) acc += md->u[(i - 1) * md->r + a] * md->v[a * md->m + (j - 1)];
  return acc;
}

int ora_eval_rhs_dense(const ora_model* md, const double* n, double* out) {
  if (!model_ok(md) || md->m > 4096) return -1;
  const size_t m = md->m;
  for (size_t s = 1; s <= m; ++s) { /* rhs.cpp:249-260 */
    double birth = 0.0;
    for (size_t i = 1; i + 1 <= s; ++i) birth += entry(md, i, s - i) * n[i - 1] * n[s - i - 1];
    birth *= 0.5;
    double death = 0.0;
    for (size_t i = 1; i <= m; ++i) death += entry(md, s, i) * n[i - 1];
    death *= n[s - 1];
    out[s - 1] = birth - death;
  }
  if (md->variant == ORA_AGGREGATION_SOURCES) {
    for (size_t q = 0; q < md->num_sources; ++q) out[md->source_k[q] - 1] += md->source_rate[q];
  } else if (md->variant == ORA_AGGREGATION_SHATTERING) {
    const double lambda = md->shatter_rate;
    double pair_gain = 0.0, mono_gain = 0.0;
    for (size_t i = 2; i <= m; ++i)
      for (size_t j = 2; j <= m; ++j) pair_gain += (double)(i + j) * entry(md, i, j) * n[i - 1] * n[j - 1];
    for (size_t j = 2; j <= m; ++j) mono_gain += (double)j * entry(md, 1, j) * n[j - 1];
    out[0] += 0.5 * lambda * pair_gain + lambda * n[0] * mono_gain;
    for (size_t s = 2; s <= m; ++s) {
      double rowsum = 0.0;
      for (size_t i = 1; i <= m; ++i) rowsum += entry(md, s, i) * n[i - 1];
      out[s - 1] -= lambda * n[s - 1] * rowsum;
    }
  }
  return 0;
}

int ora_euler_stability_bound(const ora_model* md, const double* n, double a, double* bound) {
  if (!(a > 0.0) || !model_ok(md)) return -1;
  double* rowsum = (double*)malloc(md->m * sizeof(double));
  row_sums(md, n, rowsum);
  double peak = 0.0;
  for (size_t s = 0; s < md->m; ++s) peak = (peak < rowsum[s]) ? rowsum[s] : peak; /* std::max */
  free(rowsum);
  *bound = (!(peak > 0.0)) ? INFINITY : a / peak;
  return 0;
}

/* ---------------------------------------------------------------- steppers (steppers.cpp) */

#define ERR_FLOOR 1e-300          /* steppers.cpp:11 */
#define NEG_REJECT_FRACTION 1e-3  /* steppers.cpp:14 */

static const double a21 = 1.0 / 4.0;
static const double a31 = 3.0 / 32.0, a32 = 9.0 / 32.0;
static const double a41 = 1932.0 / 2197.0, a42 = -7200.0 / 2197.0, a43 = 7296.0 / 2197.0;
static const double a51 = 439.0 / 216.0, a52 = -8.0, a53 = 3680.0 / 513.0, a54 = -845.0 / 4104.0;
static const double a61 = -8.0 / 27.0, a62 = 2.0, a63 = -3544.0 / 2565.0, a64 = 1859.0 / 4104.0,
                    a65 = -11.0 / 40.0;
static const double b5[6] = {16.0 / 135.0, 0.0, 6656.0 / 12825.0, 28561.0 / 56430.0, -9.0 / 50.0, 2.0 / 55.0};
static const double b4[6] = {25.0 / 216.0, 0.0, 1408.0 / 2565.0, 2197.0 / 4104.0, -1.0 / 5.0, 0.0};

void ora_control_defaults(ora_control* c) {
  c->stepper = ORA_RKF45;
  c->mode = ORA_ADAPTIVE;
  c->tau = 0.0;
  c->tol = 1e-6;
  c->safety = 0.0;
  c->growth_max = 2.0;
  c->shrink_min = 0.5;
  c->tau_min = 1e-12;
  c->max_rejects = 40;
  c->relative_error = 0;
}

static void call_rhs(ora_rhs* f, size_t m, const double* in, double* out) {
  f->evals += 1;
  switch (f->kind) {
    case ORA_RHS_MODEL: ora_eval_rhs(f->model, in, out); break;
    case ORA_RHS_DECAY: for (size_t i = 0; i < m; ++i) out[i] = -in[i]; break;
    case ORA_RHS_STILL: for (size_t i = 0; i < m; ++i) out[i] = 0.0; break;
    case ORA_RHS_DRAIN: out[0] = -f->param; for (size_t i = 1; i < m; ++i) out[i] = 0.0; break;
    case ORA_RHS_BURST_INF: for (size_t i = 0; i < m; ++i) out[i] = INFINITY; break;
    default: for (size_t i = 0; i < m; ++i) out[i] = NAN; break;
  }
}

static int all_finite(const double* v, size_t m) {
  for (size_t i = 0; i < m; ++i) if (!isfinite(v[i])) return 0;
  return 1;
}
static double l2_diff(const double* a, const double* b, size_t m) {
  double acc = 0.0;
  for (size_t i = 0; i < m; ++i) { const double d = a[i] - b[i]; acc += d * d; }
  return sqrt(acc);
}
static double l2_norm(const double* a, size_t m) {
  double acc = 0.0;
  for (size_t i = 0; i < m; ++i) acc += a[i] * a[i];
  return sqrt(acc);
}
static double linf_norm(const double* a, size_t m) {
  double acc = 0.0;
  for (size_t i = 0; i < m; ++i) { const double x = fabs(a[i]); acc = (acc < x) ? x : acc; }
  return acc;
}
static int has_rejectable_negative(const double* v, size_t m) {
  const double floor_ = -NEG_REJECT_FRACTION * linf_norm(v, m);
  for (size_t i = 0; i < m; ++i) if (v[i] < floor_) return 1;
  return 0;
}
static int evals_per_step(int kind) { return kind == ORA_RK2 ? 2 : kind == ORA_RK4 ? 4 : 6; }
static double effective_safety(const ora_control* c) {
  if (c->safety > 0.0) return c->safety;
  return c->stepper == ORA_RKF45 ? 0.9 : 0.25;
}
static double dmax(double a, double b) { return (a < b) ? b : a; }       /* std::max */
static double dclamp(double v, double lo, double hi) {                    /* std::clamp */
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

typedef struct { double *k1, *k2, *k3, *k4, *k5, *k6, *stage, *full, *mid, *half; } step_ws;

static int ws_alloc(step_ws* w, size_t m) {
  double* blk = (double*)calloc(10 * m, sizeof(double));
  if (!blk) return -1;
  w->k1 = blk; w->k2 = blk + m; w->k3 = blk + 2 * m; w->k4 = blk + 3 * m; w->k5 = blk + 4 * m;
  w->k6 = blk + 5 * m; w->stage = blk + 6 * m; w->full = blk + 7 * m; w->mid = blk + 8 * m;
  w->half = blk + 9 * m;
  return 0;
}
static void ws_free(step_ws* w) { free(w->k1); }

static void rk2(ora_rhs* f, size_t m, const double* n, double tau, double* out, step_ws* w) {
  call_rhs(f, m, n, w->k1);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + tau * w->k1[i];
  call_rhs(f, m, w->stage, w->k2);
  for (size_t i = 0; i < m; ++i) out[i] = n[i] + 0.5 * tau * (w->k1[i] + w->k2[i]);
}

static void rk4(ora_rhs* f, size_t m, const double* n, double tau, double* out, step_ws* w) {
  call_rhs(f, m, n, w->k1);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + 0.5 * tau * w->k1[i];
  call_rhs(f, m, w->stage, w->k2);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + 0.5 * tau * w->k2[i];
  call_rhs(f, m, w->stage, w->k3);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + tau * w->k3[i];
  call_rhs(f, m, w->stage, w->k4);
  for (size_t i = 0; i < m; ++i)
    out[i] = n[i] + tau * (w->k1[i] + 2.0 * w->k2[i] + 2.0 * w->k3[i] + w->k4[i]) / 6.0;
}

static double rkf45(ora_rhs* f, size_t m, const double* n, double tau, double* out4, double* out5,
                    step_ws* w) {
  call_rhs(f, m, n, w->k1);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + tau * a21 * w->k1[i];
  call_rhs(f, m, w->stage, w->k2);
  for (size_t i = 0; i < m; ++i) w->stage[i] = n[i] + tau * (a31 * w->k1[i] + a32 * w->k2[i]);
  call_rhs(f, m, w->stage, w->k3);
  for (size_t i = 0; i < m; ++i)
    w->stage[i] = n[i] + tau * (a41 * w->k1[i] + a42 * w->k2[i] + a43 * w->k3[i]);
  call_rhs(f, m, w->stage, w->k4);
  for (size_t i = 0; i < m; ++i)
    w->stage[i] = n[i] + tau * (a51 * w->k1[i] + a52 * w->k2[i] + a53 * w->k3[i] + a54 * w->k4[i]);
  call_rhs(f, m, w->stage, w->k5);
  for (size_t i = 0; i < m; ++i)
    w->stage[i] = n[i] + tau * (a61 * w->k1[i] + a62 * w->k2[i] + a63 * w->k3[i] +
                                a64 * w->k4[i] + a65 * w->k5[i]);
  call_rhs(f, m, w->stage, w->k6);
  double err2 = 0.0;
  for (size_t i = 0; i < m; ++i) {
    out5[i] = n[i] + tau * (b5[0] * w->k1[i] + b5[2] * w->k3[i] + b5[3] * w->k4[i] +
                            b5[4] * w->k5[i] + b5[5] * w->k6[i]);
    out4[i] = n[i] + tau * (b4[0] * w->k1[i] + b4[2] * w->k3[i] + b4[3] * w->k4[i] +
                            b4[4] * w->k5[i]);
    const double d = out5[i] - out4[i];
    err2 += d * d;
  }
  return sqrt(err2);
}

int ora_rk_step(ora_rhs* f, int stepper, size_t m, const double* n, double tau, double* out,
                double* out5, double* err) {
  step_ws w;
  if (ws_alloc(&w, m)) return -1;
  if (stepper == ORA_RK2) rk2(f, m, n, tau, out, &w);
  else if (stepper == ORA_RK4) rk4(f, m, n, tau, out, &w);
  else {
    const double e = rkf45(f, m, n, tau, out, out5 ? out5 : w.half, &w);
    if (err) *err = e;
  }
  ws_free(&w);
  return 0;
}

/* fixed_step (steppers.cpp:161-186) */
static void fixed_step(ora_rhs* f, size_t m, const double* n, double tau, int kind, ora_outcome* o,
                       double* state, step_ws* w) {
  o->tau_used = tau;
  o->tau_next = tau;
  o->rhs_evals = evals_per_step(kind);
  if (kind == ORA_RK2) rk2(f, m, n, tau, state, w);
  else if (kind == ORA_RK4) rk4(f, m, n, tau, state, w);
  else o->error_estimate = rkf45(f, m, n, tau, state, w->half, w);
  if (!all_finite(state, m)) o->status = ORA_STEP_NONFINITE;
}

/* step_doubling_adaptive (steppers.cpp:188-244) */
static void doubling(ora_rhs* f, size_t m, const double* n, double tau, const ora_control* c,
                     ora_outcome* o, double* state, step_ws* w) {
  const int is_rk2 = c->stepper == ORA_RK2;
  const double p = is_rk2 ? 2.0 : 4.0;
  const double safety = effective_safety(c);
  const int per_step = evals_per_step(c->stepper);
  for (;;) {
    if (tau < c->tau_min) { o->status = ORA_STEP_TAU_UNDERFLOW; o->tau_used = tau; return; }
    if (is_rk2) {
      rk2(f, m, n, tau, w->full, w); rk2(f, m, n, 0.5 * tau, w->mid, w); rk2(f, m, w->mid, 0.5 * tau, w->half, w);
    } else {
      rk4(f, m, n, tau, w->full, w); rk4(f, m, n, 0.5 * tau, w->mid, w); rk4(f, m, w->mid, 0.5 * tau, w->half, w);
    }
    o->rhs_evals += 3 * per_step;
    const int finite = all_finite(w->full, m) && all_finite(w->half, m);
    double err;
    if (!finite) {
      err = INFINITY;
    } else {
      err = l2_diff(w->half, w->full, m);
      if (c->relative_error) err /= dmax(1.0, l2_norm(w->half, m));
      if (has_rejectable_negative(w->half, m)) err = INFINITY;
    }
    if (err > c->tol) {
      tau *= 0.5;
      if (++o->rejects > c->max_rejects) {
        o->status = finite ? ORA_STEP_TOO_MANY_REJECTS : ORA_STEP_NONFINITE;
        o->tau_used = tau;
        return;
      }
      continue;
    }
    memcpy(state, w->half, m * sizeof(double));
    o->tau_used = tau;
    o->error_estimate = err;
    const double raw = safety * tau * pow(c->tol / dmax(err, ERR_FLOOR), 1.0 / p);
    o->tau_next = dclamp(raw, c->shrink_min * tau, c->growth_max * tau);
    return;
  }
}

/* fehlberg_adaptive (steppers.cpp:246-291) */
static void fehlberg(ora_rhs* f, size_t m, const double* n, double tau, const ora_control* c,
                     ora_outcome* o, double* state, step_ws* w) {
  const double safety = effective_safety(c);
  for (;;) {
    if (tau < c->tau_min) { o->status = ORA_STEP_TAU_UNDERFLOW; o->tau_used = tau; return; }
    double err = rkf45(f, m, n, tau, w->full, w->half, w);
    o->rhs_evals += 6;
    const int finite = all_finite(w->full, m) && all_finite(w->half, m) && isfinite(err);
    if (!finite) {
      err = INFINITY;
    } else {
      if (c->relative_error) err /= dmax(1.0, l2_norm(w->full, m));
      if (has_rejectable_negative(w->full, m)) err = INFINITY;
    }
    const double factor = dclamp(safety * pow(c->tol / dmax(err, ERR_FLOOR), 0.2), c->shrink_min, c->growth_max);
    if (err > c->tol) {
      tau *= factor;
      if (++o->rejects > c->max_rejects) {
        o->status = finite ? ORA_STEP_TOO_MANY_REJECTS : ORA_STEP_NONFINITE;
        o->tau_used = tau;
        return;
      }
      continue;
    }
    memcpy(state, w->full, m * sizeof(double));
    o->tau_used = tau;
    o->error_estimate = err;
    o->tau_next = factor * tau;
    return;
  }
}

static void outcome_init(ora_outcome* o) {
  o->tau_used = 0.0; o->tau_next = 0.0; o->error_estimate = NAN;
  o->rejects = 0; o->rhs_evals = 0; o->status = ORA_STEP_OK;
}

static int control_ok(const ora_control* c) { /* StepControl::validate (steppers.cpp:70-85) */
  if (c->mode == ORA_FIXED && !(c->tau > 0.0)) return 0;
  if (c->mode == ORA_ADAPTIVE && !(c->tol > 0.0)) return 0;
  if (c->safety < 0.0 || c->safety >= 1.0) return 0;
  if (!(c->tau_min > 0.0)) return 0;
  if (!(c->shrink_min < 1.0 && 1.0 < c->growth_max)) return 0;
  if (c->max_rejects < 1) return 0;
  return 1;
}

static int advance_ws(ora_rhs* f, size_t m, const double* n, double tau, const ora_control* c,
                      ora_outcome* o, double* state, step_ws* w) {
  outcome_init(o);
  if (!(tau > 0.0)) return -1;
  if (c->mode == ORA_FIXED) fixed_step(f, m, n, tau, c->stepper, o, state, w);
  else if (c->stepper == ORA_RKF45) fehlberg(f, m, n, tau, c, o, state, w);
  else doubling(f, m, n, tau, c, o, state, w);
  return 0;
}

int ora_advance(ora_rhs* f, size_t m, const double* n, double tau, const ora_control* c,
                ora_outcome* o, double* state_out) {
  step_ws w;
  if (ws_alloc(&w, m)) return -1;
  double* state = (double*)calloc(m, sizeof(double));
  const int rc = advance_ws(f, m, n, tau, c, o, state, &w);
  /* StepOutcome::state is empty unless the step was accepted; report zeros then. */
  memcpy(state_out, state, m * sizeof(double));
  free(state);
  ws_free(&w);
  return rc;
}

/* ---------------------------------------------------------------- run loop (simulator.cpp) */

static void push_record(ora_run_report* rep, double t, double tau, const double* n, size_t m,
                        double err, uint64_t evals) {
  if (rep->records && rep->num_records < rep->records_capacity) {
    ora_record* rec = &rep->records[rep->num_records];
    rec->t = t; rec->tau = tau; rec->density = 0.0; rec->mass = 0.0; rec->m2 = 0.0;
    for (size_t k = 1; k <= m; ++k) {
      const double x = n[k - 1], kk = (double)k;
      rec->density += x;
      rec->mass += kk * x;
      rec->m2 += kk * kk * x;
    }
    rec->error_estimate = err;
    rec->rhs_evals = evals;
    rec->rejects = rep->total_rejects;
  }
  rep->num_records += 1;
}

int ora_run(ora_rhs* f, size_t m, const ora_run_desc* d, ora_run_report* rep) {
  if (!control_ok(&d->control) || !(d->t_end >= 0.0) || !isfinite(d->t_end)) return -1;
  if (d->record == 1 && !(d->record_interval > 0.0)) return -1;
  for (size_t q = 0; q < d->num_snapshots; ++q) {
    const double s = d->snapshot_times[q];
    if (!(s >= 0.0) || s > d->t_end) return -1;
    if (q > 0 && s <= d->snapshot_times[q - 1]) return -1;
  }
  if (d->initial_tau < 0.0 || !isfinite(d->initial_tau)) return -1;
  if (f->kind == ORA_RHS_MODEL && (!model_ok(f->model) || f->model->m != m)) return -1;

  f->evals = 0;
  rep->termination = 0; rep->abort_status = 0; rep->abort_t = 0.0; rep->abort_tau = 0.0;
  rep->total_rhs_evals = 0; rep->total_accepted = 0; rep->total_rejects = 0;
  rep->num_snapshots_taken = 0; rep->num_records = 0;

  step_ws w;
  if (ws_alloc(&w, m)) return -1;
  double* state = (double*)malloc(m * sizeof(double));
  double* next = (double*)malloc(m * sizeof(double));
  memcpy(state, d->initial, m * sizeof(double));
  double t = 0.0;
  const int recording = d->record != 2;
  double next_record_t = d->record_interval;
  if (recording) push_record(rep, t, 0.0, state, m, NAN, f->evals);

  size_t snap = 0;
#define TAKE_SNAPSHOTS()                                                                   \
  while (snap < d->num_snapshots && d->snapshot_times[snap] == t) {                        \
    if (rep->snapshots) memcpy(rep->snapshots + snap * m, state, m * sizeof(double));      \
    ++snap;                                                                                \
    rep->num_snapshots_taken = snap;                                                       \
  }
  TAKE_SNAPSHOTS();

  double proposal;
  if (d->control.mode == ORA_FIXED) {
    proposal = d->control.tau;
  } else if (d->initial_tau > 0.0) {
    proposal = d->initial_tau;
  } else {
    proposal = 0.01;
    if (f->kind == ORA_RHS_MODEL) ora_euler_stability_bound(f->model, state, 0.25, &proposal);
    else proposal = INFINITY;
    if (!isfinite(proposal) || proposal <= 0.0) proposal = 0.01;
    if (d->t_end > 0.0) proposal = (d->t_end < proposal) ? d->t_end : proposal; /* std::min */
  }

  while (t < d->t_end) {
    double t_target = d->t_end;
    if (snap < d->num_snapshots && d->snapshot_times[snap] < d->t_end) t_target = d->snapshot_times[snap];
    const double remaining = t_target - t;
    const double slack = 1e-12 * dmax(1.0, fabs(t_target));
    const int shortened = remaining - proposal <= slack;
    const double tau_try = shortened ? remaining : proposal;

    ora_outcome o;
    advance_ws(f, m, state, tau_try, &d->control, &o, next, &w);
    rep->total_rhs_evals = f->evals;
    if (o.status != ORA_STEP_OK) {
      rep->termination = 1;
      rep->abort_status = o.status;
      rep->abort_t = t;
      rep->abort_tau = o.tau_used > 0.0 ? o.tau_used : tau_try;
      rep->total_rejects += (uint64_t)o.rejects;
      break;
    }
    double* tmp = state; state = next; next = tmp;
    rep->total_rejects += (uint64_t)o.rejects;
    rep->total_accepted += 1;
    const int landed = o.tau_used == tau_try;
    t = (landed && tau_try == remaining) ? t_target : t + o.tau_used;
    if (d->control.mode == ORA_ADAPTIVE && (!shortened || o.rejects > 0)) proposal = o.tau_next;
    if (d->record == 0) {
      push_record(rep, t, o.tau_used, state, m, o.error_estimate, f->evals);
    } else if (d->record == 1 && t >= next_record_t) {
      push_record(rep, t, o.tau_used, state, m, o.error_estimate, f->evals);
      next_record_t = d->record_interval * (floor(t / d->record_interval) + 1.0);
    }
    TAKE_SNAPSHOTS();
  }
#undef TAKE_SNAPSHOTS
  if (recording && rep->termination == 0) {
    const int have = rep->num_records > 0 && rep->num_records <= rep->records_capacity && rep->records;
    const double last_t = have ? rep->records[rep->num_records - 1].t : -INFINITY;
    if (rep->num_records == 0 || last_t < t) push_record(rep, t, 0.0, state, m, NAN, f->evals);
  }
  rep->final_t = t;
  rep->total_rhs_evals = f->evals;
  if (rep->final_state) memcpy(rep->final_state, state, m * sizeof(double));
  free(state); free(next);
  ws_free(&w);
  return 0;
}
