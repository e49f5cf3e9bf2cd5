// Measures the sustained FP64 DFMA throughput of the device (the roofline
// denominator for the pair kernels; MEASURED_PEAKS.json carries no FP64 entry).
// 8 independent FMA chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) out[0] = s;
}
int main(int argc, char** argv) {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const int iters = 4096, threads = 256;
  for (int blocksPerSm : {4, 8}) {
    const int blocks = sms * blocksPerSm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    float best = 1e30f, total = 0.f; int reps = 20;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0);
      dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; total += ms;
    }
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    printf("{\"sms\": %d, \"blocks_per_sm\": %d, \"fp64_tflops_burst\": %.3f, \"fp64_tflops_mean\": %.3f}\n",
           sms, blocksPerSm, flops / (best * 1e-3) / 1e12, flops / (total / reps * 1e-3) / 1e12);
  }
  return 0;
}
