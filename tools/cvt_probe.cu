// Microbenchmark: do FP64<->int conversions (F2I.F64 / I2F.F64) share the
// FP64 (DFMA) pipe on sm_100a? Times a pure-DFMA loop, a pure-conversion loop
// and both interleaved (independent chains); if the mix costs ~max(parts)
// the conversions run on another pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(double* out, int iters, double a, double b) {
  double x[8], y[8];
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 1e-3 + i;
    y[i] = threadIdx.x + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) {
        x[i] = fma(x[i], a, b);
        x[i] = fma(x[i], a, b);
      }
      if (MODE == 1 || MODE == 2) y[i] = __int2double_rn(__double2int_rn(y[i]) + 1);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* d;
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaMalloc(&d, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto k, const char* name) {
    k<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %.3f ms per launch\n", name, ms / 5);
  };
  run(probe<0>, "2 DFMA x 8 chains");
  run(probe<1>, "F2I.F64 + IADD + I2F.F64 x 8 chains");
  run(probe<2>, "both (independent chains)");
  return 0;
}
