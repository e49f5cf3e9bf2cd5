// FP64 microbenchmarks on B200 (design probes, not product code):
//   1. DFMA dependent-chain latency (cycles)
//   2. DFMA throughput vs ILP per thread and warps per SM
//   3. DMMA (mma.sync f64) throughput, shapes m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16
//   4. DFMA and DMMA issued together: do they share a pipe?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (x == 1.2345) out[0] = x;
}

template <int ILP>
__global__ void dfma_ilp(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32 / ILP; ++u) {
#pragma unroll
      for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C/D 2 regs per thread
__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
// m16n8k4: A 2, B 1, C 4
__device__ __forceinline__ void mma1684(double (&d)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}
// m16n8k16: A 8, B 4, C 4
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
        "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int CH>
__global__ void dmma884_loop(double* out, int iters, double a) {
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x + c;
  const double b = a * 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) mma884(d[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 1.2345) out[0] = s;
}

template <int CH>
__global__ void dmma1684_loop(double* out, int iters, double a) {
  double d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = threadIdx.x + c;
  const double b = a * 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) mma1684(d[c], a, a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1.2345) out[0] = s;
}

template <int CH>
__global__ void dmma16816_loop(double* out, int iters, double a) {
  double d[CH][4];
  double av[8], bv[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) av[k] = a + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) bv[k] = a - k;
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) mma16816(d[c], av, bv);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1.2345) out[0] = s;
}

// mixed: per iteration R DFMAs (8 chains) and one m8n8k4 DMMA chain set
template <int R>
__global__ void mixed_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  double d[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < 4; ++c) mma884(d[c], a, b);
#pragma unroll
      for (int r = 0; r < R; ++r) x[r & 7] = fma(x[r & 7], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
  if (s == 1.2345) out[0] = s;
}

template <typename F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) launch();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  // 1. latency
  {
    const int iters = 1000;
    lat_kernel<<<1, 32>>>(out, cyc, iters, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dfma_latency_cycles %.2f\n", double(c) / (iters * 32.0));
  }
  // 2. DFMA throughput vs ILP and warps/SM (threads per CTA = 128, CTAs/SM varied)
  const int iters = 1024;
  for (int cps : {1, 2, 3, 4, 8}) {
    const int blocks = sms * cps, threads = 128;
    const double fl = 2.0 * 32 * double(iters) * blocks * threads;
    float t1 = time_it([&] { dfma_ilp<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
    float t2 = time_it([&] { dfma_ilp<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
    float t4 = time_it([&] { dfma_ilp<4><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
    float t8 = time_it([&] { dfma_ilp<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
    printf("dfma warps/SM=%2d TF: ilp1 %.2f ilp2 %.2f ilp4 %.2f ilp8 %.2f\n", cps * 4,
           fl / t1 / 1e9, fl / t2 / 1e9, fl / t4 / 1e9, fl / t8 / 1e9);
  }
  // 3. DMMA throughput
  for (int cps : {1, 2, 4, 8}) {
    const int blocks = sms * cps, threads = 128;
    const double warps = blocks * threads / 32.0;
    const double f884 = 2.0 * 8 * 8 * 4 * 8 * double(iters) * warps;
    float a1 = time_it([&] { dmma884_loop<1><<<blocks, threads>>>(out, iters, 0.999); });
    float a4 = time_it([&] { dmma884_loop<4><<<blocks, threads>>>(out, iters, 0.999); });
    const double f1684 = 2.0 * 16 * 8 * 4 * 8 * double(iters) * warps;
    float b4 = time_it([&] { dmma1684_loop<4><<<blocks, threads>>>(out, iters, 0.999); });
    const double f16816 = 2.0 * 16 * 8 * 16 * 8 * double(iters) * warps;
    float c2 = time_it([&] { dmma16816_loop<2><<<blocks, threads>>>(out, iters, 0.999); });
    printf("dmma warps/SM=%2d TF: m8n8k4 ch1 %.2f ch4 %.2f | m16n8k4 ch4 %.2f | m16n8k16 ch2 %.2f\n",
           cps * 4, f884 / a1 / 1e9, f884 * 4 / a4 / 1e9, f1684 * 4 / b4 / 1e9,
           f16816 * 2 / c2 / 1e9);
  }
  // 4. mixed: 4 DMMA m8n8k4 + R DFMA per inner step
  {
    const int blocks = sms * 4, threads = 128;
    const double warps = blocks * threads / 32.0;
    const double fm = 2.0 * 256 * 4 * 8 * double(iters) * warps;
    float t0 = time_it([&] { mixed_loop<0><<<blocks, threads>>>(out, iters, 0.999, 1e-7); });
    float t16 = time_it([&] { mixed_loop<16><<<blocks, threads>>>(out, iters, 0.999, 1e-7); });
    float t32 = time_it([&] { mixed_loop<32><<<blocks, threads>>>(out, iters, 0.999, 1e-7); });
    float t64 = time_it([&] { mixed_loop<64><<<blocks, threads>>>(out, iters, 0.999, 1e-7); });
    // pure DFMA equivalents
    const double fd = 2.0 * 8 * double(iters) * blocks * threads;
    printf("mixed (4 dmma884 + R dfma per step) ms: R0 %.3f R16 %.3f R32 %.3f R64 %.3f ; dmma-only TF %.2f\n",
           t0, t16, t32, t64, fm / t0 / 1e9);
    float p16 = time_it([&] { dfma_ilp<8><<<blocks, threads>>>(out, iters * 4, 0.999, 1e-7); });
    float p32 = time_it([&] { dfma_ilp<8><<<blocks, threads>>>(out, iters * 8, 0.999, 1e-7); });
    printf("  dfma-only for R16 work ms %.3f, for R32 work ms %.3f (TF %.2f)\n", p16, p32,
           fd * 16 / p16 / 1e9);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
