/* Long-double CPU restatement of the reference hot path -- the parity ORACLE.
 * TEST INFRASTRUCTURE ONLY: linked/loaded by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the checker; never by the product path.
 */
#ifndef HAWKES_ORACLE_H
#define HAWKES_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Params order follows hawkes::Params (types.hpp:51-57):
 * p[0]=mu0 p[1]=tauX p[2]=tauT p[3]=theta p[4]=omega p[5]=h.
 *
 * Dense O(N^2) log-likelihood and its 6-parameter gradient.
 *   loglik, valid   : as hawkes::logLikelihood (likelihood.cpp:10-55);
 *                     valid=0 -> loglik=-inf and grad = NaN.
 *   grad[6]         : d loglik / d p[k] (may be NULL).
 *   per_event[n]    : log(lambda_i) - Lambda_i, 0 for degenerate rows (NULL ok).
 *   sums[6*n]       : per-row raw sums (S_B,S_Br,S_Bt,S_T,S_Tt,S_Tr), row-major
 *                     by row (NULL ok) -- for kernel-level diagnostics.
 *   grad_abs[6]     : sum_i |d l_i / d p[k]|, the scale of each gradient
 *                     component's summands (NULL ok); the parity tolerance
 *                     near stationary points is relative to it.
 * threads <= 0 uses all OpenMP threads. Returns 0, or 1 on invalid params. */
int oracle_loglik_grad(const double* x, const double* y, const double* t,
                       int64_t n, double window_end, const double* p,
                       int threads, double* loglik, int* valid, double* grad,
                       double* per_event, double* sums, double* grad_abs);

/* Long-double Phi / phi (erfc-based), for known-answer checks. */
double oracle_normal_cdf(double z);

#ifdef __cplusplus
}
#endif
#endif
