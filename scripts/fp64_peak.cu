// FP64 FMA-pipe peak probe (B200): every thread runs 8 independent DFMA
// chains; flops = 2 * fma count; best of 5 timed launches (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fma_chains(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __fma_rn(x[j], a, b);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_chains<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_chains<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * iters * double(blocks) * threads;
  printf("{\"fp64_fma_tflops\": %.2f, \"how\": \"%d blocks x %d threads x 8 independent DFMA chains x %d iters, best of 5, CUDA events\", \"sms\": %d}\n",
         flops / (best * 1e-3) / 1e12, blocks, threads, iters, sms);
  return 0;
}
