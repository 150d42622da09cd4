/* agk_truth.c — TEST INFRASTRUCTURE ONLY. The low-rank RHS of agk_oracle.c evaluated entirely in
 * x87 long double (64-bit mantissa): same algorithm as the reference (rhs.cpp:87-235, packed
 * two-real FFT, radix-2), 11 more bits everywhere. Used as the accuracy yardstick where the
 * reference's own fp64 rounding is visible at the 1e-11 level (kernels whose U and V spread over
 * many decades make the packed FFT lose ~log10(max|U n| / max|V n|) digits). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "agk_oracle.h"

typedef long double ld;

static size_t np2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

static void fft_ld(ld* a, size_t n, int inv) {
  for (size_t i = 1, j = 0; i < n; ++i) { /* bit reversal */
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      ld t = a[2 * i]; a[2 * i] = a[2 * j]; a[2 * j] = t;
      t = a[2 * i + 1]; a[2 * i + 1] = a[2 * j + 1]; a[2 * j + 1] = t;
    }
  }
  const ld pi = 3.141592653589793238462643383279502884L;
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t j = 0; j < len / 2; ++j) {
      const ld ang = (inv ? 2.0L : -2.0L) * pi * (ld)j / (ld)len;
      const ld wr = cosl(ang), wi = sinl(ang);
      for (size_t base = 0; base < n; base += len) {
        ld* lo = a + 2 * (base + j);
        ld* hi = a + 2 * (base + j + len / 2);
        const ld xr = hi[0] * wr - hi[1] * wi, xi = hi[0] * wi + hi[1] * wr;
        hi[0] = lo[0] - xr;
        hi[1] = lo[1] - xi;
        lo[0] += xr;
        lo[1] += xi;
      }
    }
  }
  if (inv)
    for (size_t i = 0; i < 2 * n; ++i) a[i] /= (ld)n;
}

/* eval_rhs with every intermediate in long double; rounding to double only at the end */
int ora_eval_rhs_truth(const ora_model* md, const double* n, double* out) {
  if (!md || md->m < 2 || md->r < 1 || md->k) return -1; /* low-rank kernels only */
  const size_t m = md->m, r = md->r, P = np2(2 * m);
  ld* z = (ld*)malloc(2 * P * sizeof(ld));
  ld* acc = (ld*)calloc(2 * P, sizeof(ld));
  ld* w = (ld*)calloc(r, sizeof(ld));
  ld* res = (ld*)calloc(m, sizeof(ld));
  for (size_t a = 0; a < r; ++a) {
    for (size_t i = 0; i < P; ++i) {
      z[2 * i] = i < m ? (ld)md->u[i * r + a] * (ld)n[i] : 0.0L;
      z[2 * i + 1] = i < m ? (ld)md->v[a * m + i] * (ld)n[i] : 0.0L;
    }
    for (size_t j = 0; j < m; ++j) w[a] += (ld)md->v[a * m + j] * (ld)n[j];
    fft_ld(z, P, 0);
    for (size_t k = 0; k < P; ++k) {
      const size_t mk = (P - k) & (P - 1);
      const ld zr = z[2 * k], zi = z[2 * k + 1], mr = z[2 * mk], mi = -z[2 * mk + 1];
      const ld ar = 0.5L * (zr + mr), ai = 0.5L * (zi + mi);
      const ld br = 0.5L * (zi - mi), bi = -0.5L * (zr - mr);
      acc[2 * k] += ar * br - ai * bi;
      acc[2 * k + 1] += ar * bi + ai * br;
    }
  }
  fft_ld(acc, P, 1);
  for (size_t s = 0; s < m; ++s) {
    ld rowsum = 0.0L;
    for (size_t a = 0; a < r; ++a) rowsum += (ld)md->u[s * r + a] * w[a];
    const ld birth = s >= 1 ? 0.5L * acc[2 * (s - 1)] : 0.0L;
    res[s] = birth - (ld)n[s] * rowsum;
    if (md->variant == ORA_AGGREGATION_SHATTERING && s >= 1) res[s] -= (ld)md->shatter_rate * (ld)n[s] * rowsum;
  }
  if (md->variant == ORA_AGGREGATION_SOURCES)
    for (size_t q = 0; q < md->num_sources; ++q) res[md->source_k[q] - 1] += (ld)md->source_rate[q];
  if (md->variant == ORA_AGGREGATION_SHATTERING) {
    ld pair = 0.0L, mono = 0.0L;
    for (size_t a = 0; a < r; ++a) {
      ld su0 = 0, su1 = 0, sv0 = 0, sv1 = 0;
      for (size_t i = 2; i <= m; ++i) {
        const ld x = (ld)md->u[(i - 1) * r + a] * (ld)n[i - 1], y = (ld)md->v[a * m + i - 1] * (ld)n[i - 1];
        su0 += x; su1 += (ld)i * x; sv0 += y; sv1 += (ld)i * y;
      }
      pair += su1 * sv0 + su0 * sv1;
      mono += (ld)md->u[a] * sv1;
    }
    res[0] += 0.5L * (ld)md->shatter_rate * pair + (ld)md->shatter_rate * (ld)n[0] * mono;
  }
  for (size_t s = 0; s < m; ++s) out[s] = (double)res[s];
  free(z); free(acc); free(w); free(res);
  return 0;
}
