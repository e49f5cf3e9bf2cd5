/* sthk_sim.h -- synthetic event generators for benchmarks and tests.
 *
 * Restates the reference's seeded generators so that benchmark inputs are
 * bit-identical to the ones the reference's own tests and SURVEY recipes
 * build:
 *   hawkes::Rng                     proj/include/sthawkes/rng.hpp:27-96
 *   hawkes::generateBenchmarkCloud  proj/src/simulate.cpp:83-95
 *   hawkes::simulateClusterProcess  proj/src/simulate.cpp:10-81
 * Bit-identity with the reference build is checked in
 * tests/test_sim_cpu.py against the reference compiled in oracle/_ref.
 * Not part of the likelihood hot path.
 */
#ifndef STHK_SIM_H
#define STHK_SIM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* window = {xmin, xmax, ymin, ymax, tEnd}. n uniform events, stably sorted
 * by time; *window_end = tEnd. Returns 0, or 1 on invalid arguments. */
int sthk_sim_cloud(int64_t n, const double* window, uint64_t seed, double* x,
                   double* y, double* t, double* window_end);

/* Branching (cluster) simulation with parameters p[6] (Params order; theta,
 * omega, h drive the offspring), homogeneous immigrant rate per unit area.
 * Writes min(total, capacity) time-sorted events; parent[i] = 0 for
 * immigrants, else the 1-based sorted index of the parent; *count = total.
 * Returns 0, 1 on invalid arguments, 2 when no event was generated. */
int sthk_sim_cluster(const double* p, const double* window, double rate,
                     uint64_t seed, int64_t capacity, double* x, double* y,
                     double* t, int* parent, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif
