// Device diagnostics used by the benchmark: a DFMA throughput probe giving
// the roofline denominator for the FP64-bound pair kernels (MEASURED_PEAKS.json
// carries HBM and bf16 peaks only). 8 independent FMA chains per thread,
// 8 CTAs x 256 threads per SM.
#include <cuda_runtime.h>

#include "../../include/sthk.h"

namespace {
__global__ void dfma_probe(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) out[0] = s;
}
}  // namespace

extern "C" int sthk_measure_fp64_peak(int device, int reps, double* tflops_best,
                                      double* tflops_mean) {
  if (!tflops_best || reps < 1) return STHK_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return STHK_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return STHK_ECUDA;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048, threads = 256, blocks = sms * 8;
  for (int w = 0; w < 3; ++w) dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
  float best = 1e30f, total = 0.f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, st);
    dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
    total += ms;
  }
  const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
  *tflops_best = flops / (best * 1e-3) / 1e12;
  if (tflops_mean) *tflops_mean = flops / (total / reps * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? STHK_OK : STHK_ECUDA;
}
