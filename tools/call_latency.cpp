// Per-call wall latency of the C ABI for MH-style moves on C2 data (first N
// events, argv[1], default 85k):
// mu0 move (trigger cache hit: finalize only), h move (plan cached, trigger
// sweep), omega move (plan + trigger sweep), full eval (caches off).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../include/sthk.h"
#include "../include/sthk_sim.h"
int main(int argc, char** argv) {
  const int64_t cap = 90000;
  std::vector<double> x(cap), y(cap), t(cap);
  std::vector<int> par(cap);
  int64_t cnt = 0;
  const double truth[6] = {1, 1.6, 14, 0.344, 1440, 0.0695};
  const double win[5] = {0, 15, 0, 15, 4750};
  sthk_sim_cluster(truth, win, 0.053217, 2005, cap, x.data(), y.data(), t.data(), par.data(), &cnt);
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 85000;
  printf("N = %lld\n", static_cast<long long>(n));
  sthk_engine* e = nullptr;
  int dev = 0;
  sthk_create(&dev, 1, &e);
  if (argc > 2 && std::atoi(argv[2]) == 0) {
    sthk_set_graphs(e, 0);
    printf("(graphs off)\n");
  }
  sthk_load_events(e, x.data(), y.data(), t.data(), n, t[n - 1]);
  double p[6] = {0.66, 1.6, 14, 0.344, 1440, 0.0695};
  double ll; int valid;
  sthk_set_params(e, p);
  sthk_loglik(e, &ll, &valid, nullptr);
  auto run = [&](const char* name, int k, double f) {
    const int reps = 400;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) {
      p[k] *= (i & 1) ? 1.0 / f : f;
      sthk_set_params(e, p);
      sthk_loglik(e, &ll, &valid, nullptr);
    }
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
    sthk_stats st; sthk_get_stats(e, &st);
    // device time of the same move (timing level 2: kernel stamps, no events)
    sthk_set_timing(e, 2);
    double dev_ms = 0;
    for (int i = 0; i < 40; ++i) {
      p[k] *= (i & 1) ? 1.0 / f : f;
      sthk_set_params(e, p);
      sthk_loglik(e, &ll, &valid, nullptr);
      sthk_stats s2; sthk_get_stats(e, &s2);
      dev_ms += s2.eval_ms;
    }
    sthk_set_timing(e, 0);
    printf("%-28s %8.1f us/call  device %6.1f us  launches %lld  (cache_hit %d, trigger_cache_hit %d)\n",
           name, us, dev_ms / 40 * 1e3, static_cast<long long>(st.kernel_launches), st.cache_hit,
           st.trigger_cache_hit);
  };
  run("mu0 move", 0, 1.01);
  run("theta move", 3, 1.01);
  run("h move", 5, 1.01);
  run("omega move", 4, 1.01);
  sthk_set_background_cache(e, 0);
  run("mu0 move, caches off", 0, 1.01);
  sthk_set_background_cache(e, 1);
  // empty-ish: the same params (all caches hit)
  run("no change", 0, 1.0);
  // end-to-end pieces (caches off): load_events from pinned buffers, eval
  {
    double *hx, *hy, *ht;
    cudaMallocHost(&hx, 8 * n); cudaMallocHost(&hy, 8 * n); cudaMallocHost(&ht, 8 * n);
    for (int64_t i = 0; i < n; ++i) { hx[i] = x[i]; hy[i] = y[i]; ht[i] = t[i]; }
    sthk_set_background_cache(e, 0);
    double g[6];
    const int reps = 50;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) sthk_load_events(e, hx, hy, ht, n, t[n - 1]);
    auto t1 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) sthk_loglik_grad(e, &ll, &valid, g, nullptr);
    auto t2 = std::chrono::steady_clock::now();
    {
      double* d; cudaMalloc(&d, 24 * n);
      cudaStream_t st; cudaStreamCreate(&st);
      auto a0 = std::chrono::steady_clock::now();
      for (int i = 0; i < reps; ++i) {
        cudaMemcpyAsync(d, hx, 8 * n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d + n, hy, 8 * n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d + 2 * n, ht, 8 * n, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
      }
      auto a1 = std::chrono::steady_clock::now();
      printf("raw 3 x H2D pinned + sync     %8.1f us/call\n", std::chrono::duration<double, std::micro>(a1 - a0).count() / reps);
      cudaFree(d);
    }
    {  // host time of the enqueue alone (full evaluation, caches off), then the wait
      double enq = 0, tot = 0;
      for (int i = 0; i < reps; ++i) {
        p[0] *= (i & 1) ? 1.0 / 1.01 : 1.01;
        sthk_set_params(e, p);
        auto b0 = std::chrono::steady_clock::now();
        sthk_enqueue(e, 1, 0);
        auto b1 = std::chrono::steady_clock::now();
        sthk_result(e, &ll, &valid, g, nullptr);
        auto b2 = std::chrono::steady_clock::now();
        enq += std::chrono::duration<double, std::micro>(b1 - b0).count();
        tot += std::chrono::duration<double, std::micro>(b2 - b0).count();
      }
      printf("enqueue host time (full eval) %8.1f us/call of %8.1f us\n", enq / reps, tot / reps);
    }
    {  // the same split for a mu0 move over the cached sums (finalize only)
      sthk_set_background_cache(e, 1);
      sthk_loglik(e, &ll, &valid, nullptr);
      double enq = 0, tot = 0, sp = 0;
      for (int i = 0; i < 4 * reps; ++i) {
        p[0] *= (i & 1) ? 1.0 / 1.01 : 1.01;
        auto a0 = std::chrono::steady_clock::now();
        sthk_set_params(e, p);
        auto b0 = std::chrono::steady_clock::now();
        sthk_enqueue(e, 0, 0);
        auto b1 = std::chrono::steady_clock::now();
        sthk_result(e, &ll, &valid, nullptr, nullptr);
        auto b2 = std::chrono::steady_clock::now();
        sp += std::chrono::duration<double, std::micro>(b0 - a0).count();
        enq += std::chrono::duration<double, std::micro>(b1 - b0).count();
        tot += std::chrono::duration<double, std::micro>(b2 - a0).count();
      }
      printf("mu0 move: set_params %.1f + enqueue %.1f us of %.1f us/call\n", sp / (4 * reps),
             enq / (4 * reps), tot / (4 * reps));
      sthk_set_background_cache(e, 0);
    }
    printf("load_events (pinned)         %8.1f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
    printf("loglik_grad (caches off)     %8.1f us/call\n", std::chrono::duration<double, std::micro>(t2 - t1).count() / reps);
  }
  sthk_destroy(e);
  return 0;
}
