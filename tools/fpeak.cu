// FP64 / FP32 FMA peak microbenchmark (roofline denominator for the MPdist
// distance kernels; MEASURED_PEAKS.json only carries HBM and bf16).
// Independent FMA chains per thread, grid = SMs * 8 CTAs, CUDA-event timed.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == (T)12345.678) out[threadIdx.x] = s;
}
// FP64 FMA interleaved with int ALU work (does the ALU pipe co-issue?)
__global__ void mixed_loop(double* out, int iters, double a, double b) {
  double acc[8]; unsigned u[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c] = threadIdx.x + c; u[c] = threadIdx.x * 7 + c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) { acc[c] = fma(acc[c], a, b); u[c] = __vimax3_u32(u[c] ^ 0x55u, u[(c+1)&7], u[(c+3)&7]); }
  }
  double s = 0; unsigned t = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) { s += acc[c]; t += u[c]; }
  if (s == 12345.678 || t == 7u) out[threadIdx.x] = s + t;
}
int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 5;  // long runs: clocks sampled under load by tools/fpeak_run.py
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* d; cudaMalloc(&d, 1 << 20);
  float* f; cudaMalloc(&f, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256, iters = 20000;
  double best64 = 0, best32 = 0, bestmix = 0;
  for (int rep = 0; rep < reps; ++rep) {
    float ms;
    cudaEventRecord(e0); fma_loop<double, 8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double tf = 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12; if (tf > best64) best64 = tf;
    cudaEventRecord(e0); fma_loop<float, 8><<<blocks, threads>>>(f, iters * 2, 0.999999f, 1e-7f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    tf = 2.0 * 8 * iters * 2 * (double)blocks * threads / (ms * 1e-3) / 1e12; if (tf > best32) best32 = tf;
    cudaEventRecord(e0); mixed_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    tf = 2.0 * 8 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12; if (tf > bestmix) bestmix = tf;
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"fp64_fma_tflops\": %.2f, \"fp32_fma_tflops\": %.2f, \"fp64_fma_with_int_alu_tflops\": %.2f, \"clock_khz\": %d, \"err\": \"%s\"}\n",
         sms, best64, best32, bestmix, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
