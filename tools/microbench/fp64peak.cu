// fp64peak.cu — sustained fp64 FMA throughput of this B200 (the denominator of
// bench.py's roofline_fp64; MEASURED_PEAKS.json has no fp64 figure).
//
// Every SM runs resident warps of independent DFMA chains (8 per thread, no
// memory traffic); the rate is timed with CUDA events over `ms` milliseconds
// of back-to-back launches, i.e. under the same power cap as a long step.
// Measurement infrastructure only (not part of libpic).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) dfma_kernel(double *out, double a, double b) {
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;   // never true: keeps the chains alive
}

}  // namespace

extern "C" {

// Runs DFMA launches for about `ms` milliseconds; returns fp64 TFLOP/s
// (2 flops per FMA) or a negative value on a CUDA error.
__attribute__((visibility("default"))) double fp64_fma_tflops(double ms) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1.0;
  double *out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1.0;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int blocks = sms * 8, threads = 256;   // 64 warps per SM
  const double flops_per_launch = 2.0 * CHAINS * (double)ITERS * blocks * threads;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // calibrate: one launch
  dfma_kernel<<<blocks, threads, 0, st>>>(out, 0.999999, 1e-9);
  cudaEventRecord(a, st);
  dfma_kernel<<<blocks, threads, 0, st>>>(out, 0.999999, 1e-9);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float one = 0.f;
  cudaEventElapsedTime(&one, a, b);
  int n = (int)(ms / (one > 0.f ? one : 1.f));
  if (n < 3) n = 3;
  cudaEventRecord(a, st);
  for (int i = 0; i < n; ++i) dfma_kernel<<<blocks, threads, 0, st>>>(out, 0.999999, 1e-9);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(st);
  cudaFree(out);
  if (e != cudaSuccess || t <= 0.f) return -1.0;
  return flops_per_launch * n / (t * 1e-3) / 1e12;
}

}  // extern "C"
