#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
int main() {
  const size_t n = 85000, b = 8 * n;
  double *h[3], *d[3];
  for (int i = 0; i < 3; ++i) { cudaMallocHost(&h[i], b); cudaMalloc(&d[i], b); for (size_t k = 0; k < n; ++k) h[i][k] = k; }
  double* hb; cudaMallocHost(&hb, 3 * b); double* db; cudaMalloc(&db, 3 * b);
  cudaStream_t s[3]; for (int i = 0; i < 3; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  cudaEvent_t ev[3]; for (int i = 0; i < 3; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  auto run = [&](const char* name, auto f) {
    for (int w = 0; w < 20; ++w) f();
    const int R = 200;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < R; ++r) f();
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
    printf("%-40s %7.1f us  (%.1f GB/s)\n", name, us, 3 * b / us / 1e3);
  };
  run("3 copies, 1 stream + sync", [&] { for (int i = 0; i < 3; ++i) cudaMemcpyAsync(d[i], h[i], b, cudaMemcpyHostToDevice, s[0]); cudaStreamSynchronize(s[0]); });
  run("3 copies, 3 streams + join + sync", [&] {
    cudaEventRecord(ev[0], s[0]); cudaStreamWaitEvent(s[1], ev[0]); cudaStreamWaitEvent(s[2], ev[0]);
    for (int i = 0; i < 3; ++i) cudaMemcpyAsync(d[i], h[i], b, cudaMemcpyHostToDevice, s[i]);
    cudaEventRecord(ev[1], s[1]); cudaEventRecord(ev[2], s[2]); cudaStreamWaitEvent(s[0], ev[1]); cudaStreamWaitEvent(s[0], ev[2]);
    cudaStreamSynchronize(s[0]); });
  run("1 contiguous copy (3x size) + sync", [&] { cudaMemcpyAsync(db, hb, 3 * b, cudaMemcpyHostToDevice, s[0]); cudaStreamSynchronize(s[0]); });
  run("empty sync", [&] { cudaStreamSynchronize(s[0]); });
  return 0;
}
