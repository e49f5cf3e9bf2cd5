/* Long-double CPU restatement of the reference likelihood path, plus the
 * analytic gradient the reference lacks.
 *
 * TEST INFRASTRUCTURE ONLY (the parity oracle). The product never links it.
 *
 * Restated from the reference, not copied:
 *   pair rates       proj/include/sthawkes/kernels.hpp:26-50, 76-101
 *                    (background over ALL sources incl. the self term;
 *                     trigger only for strictly earlier source times)
 *   compensator      kernels.hpp:54-65   mu0(Phi((T-t)/tauT)-Phi(-t/tauT))
 *                                        - theta expm1(-omega (T-t))
 *   total/validity   likelihood.cpp:10-55 (lambda<=0 or non-finite -> -inf)
 * Differences by design: every sum is carried in long double (x87 80-bit),
 * and the per-row sums factor the constant norms out of the pair loop. For
 * time-sorted input the pair loop visits only sources within a time window
 * outside which every term is below e^-100 of the row's background self term
 * (mu0 cB: the background exponent dt^2/2tauT^2 > 100, the trigger exponent
 * omega dt > 100 + ln(theta cT / (mu0 cB))); the skipped terms total less
 * than N e^-100 < 4e-38 of every lambda_i and of every gradient sum's scale,
 * far below long-double rounding. Unsorted input takes the full loop.
 *
 * Gradient: with E^B = exp(-r^2/2tauX^2 - dt^2/2tauT^2)
 * over all j and E^T = [t_j<t_i] exp(-omega dt - r^2/2h^2),
 *   S_B=sum E^B, S_Br=sum E^B r^2, S_Bt=sum E^B dt^2,
 *   S_T=sum E^T, S_Tt=sum E^T dt,  S_Tr=sum E^T r^2,
 *   lambda = mu0 cB S_B + theta cT S_T, cB=(2pi)^-3/2/(tauX^2 tauT), cT=omega/(2pi h^2)
 * and d loglik/dp = sum_i (d lambda_i/dp)/lambda_i - d Lambda_i/dp.
 */
#include "hawkes_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>

static const long double kPiL = 3.14159265358979323846264338327950288L;

static int params_valid(const double* p) {
  for (int k = 0; k < 6; ++k) {
    if (!isfinite(p[k])) return 0;
  }
  /* types.hpp:59-63: all positive except theta >= 0 */
  return p[0] > 0 && p[1] > 0 && p[2] > 0 && p[4] > 0 && p[5] > 0 && p[3] >= 0;
}

static long double cdfl(long double z) { return 0.5L * erfcl(-z / sqrtl(2.0L)); }
static long double pdfl(long double z) { return expl(-0.5L * z * z) / sqrtl(2.0L * kPiL); }

double oracle_normal_cdf(double z) { return (double)cdfl((long double)z); }

int oracle_loglik_grad(const double* x, const double* y, const double* t,
                       int64_t n, double window_end, const double* p,
                       int threads, double* loglik, int* valid, double* grad,
                       double* per_event, double* sums, double* grad_abs) {
  if (!params_valid(p) || n < 1) return 1;
  const long double mu0 = p[0], tx = p[1], tt = p[2], th = p[3], om = p[4], h = p[5];
  const long double cB = powl(2.0L * kPiL, -1.5L) / (tx * tx * tt);
  const long double cT = om / (2.0L * kPiL * h * h);
  const long double T = window_end;

  long double* row = (long double*)malloc(sizeof(long double) * 8 * (size_t)n);
  int bad = 0;
  /* source window (sorted times): |dt| <= wB for the background, dt <= wT
   * for the trigger, both with the e^-100 margin above */
  int sorted = 1;
  for (int64_t i = 1; i < n && sorted; ++i) sorted = t[i] >= t[i - 1];
  const long double kCut = 100.0L;
  const long double boost = logl(th * cT / (mu0 * cB));
  const long double wB = tt * sqrtl(2.0L * kCut) * 1.000001L;
  const long double wT = (kCut + (boost > 0 ? boost : 0)) / om * 1.000001L;
  const long double wLo = wB > wT ? wB : wT;
  if (threads > 0) omp_set_num_threads(threads);

#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    long double sB = 0, sBr = 0, sBt = 0, sT = 0, sTt = 0, sTr = 0;
    const long double xi = x[i], yi = y[i], ti = t[i];
    int64_t j0 = 0, j1 = n;
    if (sorted) {  /* first source at or after ti - wLo, first after ti + wB */
      int64_t a = 0, b = i;
      while (a < b) {
        const int64_t m = (a + b) / 2;
        if ((long double)t[m] < ti - wLo) a = m + 1; else b = m;
      }
      j0 = a;
      a = i, b = n;
      while (a < b) {
        const int64_t m = (a + b) / 2;
        if ((long double)t[m] <= ti + wB) a = m + 1; else b = m;
      }
      j1 = a;
    }
    for (int64_t j = j0; j < j1; ++j) {
      const long double dx = xi - x[j], dy = yi - y[j], dt = ti - t[j];
      const long double r2 = dx * dx + dy * dy;
      const long double eb = expl(-r2 / (2 * tx * tx) - dt * dt / (2 * tt * tt));
      sB += eb;
      sBr += eb * r2;
      sBt += eb * dt * dt;
      if (t[j] < t[i]) {
        const long double et = expl(-om * dt - r2 / (2 * h * h));
        sT += et;
        sTt += et * dt;
        sTr += et * r2;
      }
    }
    if (sums) {
      double* s = sums + 6 * i;
      s[0] = (double)sB; s[1] = (double)sBr; s[2] = (double)sBt;
      s[3] = (double)sT; s[4] = (double)sTt; s[5] = (double)sTr;
    }
    const long double lam = mu0 * cB * sB + th * cT * sT;
    const long double D = T - ti;
    const long double Phi1 = cdfl(D / tt), Phi0 = cdfl(-ti / tt);
    const long double em1 = expm1l(-om * D);
    const long double Lam = mu0 * (Phi1 - Phi0) - th * em1;
    long double* o = row + 8 * i;
    /* validity is decided on the double-rounded rate, as the reference's
     * double arithmetic would (likelihood.cpp:35-39) */
    const double lamd = (double)lam;
    if (!(lamd > 0) || !isfinite(lamd)) {
      bad |= 1;
      for (int k = 0; k < 8; ++k) o[k] = 0;
      continue;
    }
    o[0] = logl(lam) - Lam;
    /* d lambda / d p */
    const long double dl[6] = {
        cB * sB,
        mu0 * cB * (-2 * sB / tx + sBr / (tx * tx * tx)),
        mu0 * cB * (-sB / tt + sBt / (tt * tt * tt)),
        cT * sT,
        th * cT * (sT / om - sTt),
        th * cT * (-2 * sT / h + sTr / (h * h * h))};
    /* d Lambda / d p */
    const long double dL[6] = {
        Phi1 - Phi0,
        0,
        -mu0 * (pdfl(D / tt) * D + pdfl(ti / tt) * ti) / (tt * tt),
        -em1,
        th * D * expl(-om * D),
        0};
    for (int k = 0; k < 6; ++k) o[1 + k] = dl[k] / lam - dL[k];
  }

  long double tot[7] = {0, 0, 0, 0, 0, 0, 0};
  long double absum[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 7; ++k) tot[k] += row[8 * i + k];
    for (int k = 0; k < 6; ++k) absum[k] += fabsl(row[8 * i + 1 + k]);
    if (per_event) per_event[i] = (double)row[8 * i];
  }
  if (grad_abs) {
    for (int k = 0; k < 6; ++k) grad_abs[k] = (double)absum[k];
  }
  free(row);
  const int ok = !bad && isfinite((double)tot[0]);
  *valid = ok;
  *loglik = ok ? (double)tot[0] : -INFINITY;
  if (grad) {
    for (int k = 0; k < 6; ++k) grad[k] = ok ? (double)tot[1 + k] : NAN;
  }
  return 0;
}
