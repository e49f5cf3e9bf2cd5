// H2D patterns for the event load (development probe): three cudaMemcpyAsync
// on one or three streams, one contiguous copy, and a zero-copy kernel that
// reads the three pinned host arrays over PCIe and writes the device copies.
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void gather3(const double2* __restrict__ a, const double2* __restrict__ b,
                        const double2* __restrict__ c, double2* da, double2* db, double2* dc, size_t n2) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 va = a[i], vb = b[i], vc = c[i];
    da[i] = va; db[i] = vb; dc[i] = vc;
  }
}
int main() {
  const size_t n = 85000, b = 8 * n;
  double *h[3], *d[3];
  for (int i = 0; i < 3; ++i) { cudaMallocHost(&h[i], b); cudaMalloc(&d[i], b); for (size_t k = 0; k < n; ++k) h[i][k] = k; }
  double* hb; cudaMallocHost(&hb, 3 * b); double* db; cudaMalloc(&db, 3 * b);
  cudaStream_t s[3]; for (int i = 0; i < 3; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  cudaEvent_t ev[3]; for (int i = 0; i < 3; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  double* hd[3]; for (int i = 0; i < 3; ++i) cudaHostGetDevicePointer(&hd[i], h[i], 0);
  auto run = [&](const char* name, auto f) {
    for (int w = 0; w < 20; ++w) f();
    const int R = 200;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < R; ++r) f();
    double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / R;
    printf("%-44s %7.1f us  (%.1f GB/s)\n", name, us, 3 * b / us / 1e3);
  };
  run("3 copies, 1 stream + sync", [&] { for (int i = 0; i < 3; ++i) cudaMemcpyAsync(d[i], h[i], b, cudaMemcpyHostToDevice, s[0]); cudaStreamSynchronize(s[0]); });
  run("3 copies, 3 streams + join + sync", [&] {
    cudaEventRecord(ev[0], s[0]); cudaStreamWaitEvent(s[1], ev[0]); cudaStreamWaitEvent(s[2], ev[0]);
    for (int i = 0; i < 3; ++i) cudaMemcpyAsync(d[i], h[i], b, cudaMemcpyHostToDevice, s[i]);
    cudaEventRecord(ev[1], s[1]); cudaEventRecord(ev[2], s[2]); cudaStreamWaitEvent(s[0], ev[1]); cudaStreamWaitEvent(s[0], ev[2]);
    cudaStreamSynchronize(s[0]); });
  run("1 contiguous copy (3x size) + sync", [&] { cudaMemcpyAsync(db, hb, 3 * b, cudaMemcpyHostToDevice, s[0]); cudaStreamSynchronize(s[0]); });
  for (int blocks : {148, 296, 592, 1184}) {
    char name[64]; snprintf(name, sizeof name, "zero-copy gather kernel, %d x 256 + sync", blocks);
    run(name, [&] { gather3<<<blocks, 256, 0, s[0]>>>((const double2*)hd[0], (const double2*)hd[1], (const double2*)hd[2],
                                                     (double2*)d[0], (double2*)d[1], (double2*)d[2], n / 2);
                    cudaStreamSynchronize(s[0]); });
  }
  run("empty sync", [&] { cudaStreamSynchronize(s[0]); });
  return 0;
}
