// FP32 FFMA throughput microbenchmark (burst and sustained) -- the measured denominator for the
// SIMT contraction's "alu" roofline (SURVEY.md §7 "Roofline denominators").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma_peak tools/ffma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 16;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) ffma_kernel(float *out, float a, float b, int reps) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 64
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1234.5f) out[0] = s;  // keep the chains alive
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  float *d;
  cudaMalloc(&d, 4);
  const int blocks = p.multiProcessorCount * 4, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_kernel<<<blocks, threads>>>(d, 0.999f, 1e-3f, 1);
  cudaDeviceSynchronize();
  float best = 0.f;
  for (int rep = 0; rep < 5; ++rep) {  // burst: ~5 ms launches
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(d, 0.999f, 1e-3f, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * CHAINS * ITERS * 2.0 * double(blocks) * threads;
    best = fmaxf(best, float(flops / (ms * 1e-3) / 1e12));
  }
  // sustained: ~2 s of back-to-back launches
  int n = 0;
  cudaEventRecord(e0);
  float ms = 0.f;
  for (;;) {
    ffma_kernel<<<blocks, threads>>>(d, 0.999f, 1e-3f, 2);
    ++n;
    if (n % 50 == 0) {
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms > 2000.f) break;
    }
  }
  const double flops = 2.0 * CHAINS * ITERS * 2.0 * double(blocks) * threads * n;
  printf("{\"sms\": %d, \"fp32_tflops_burst\": %.2f, \"fp32_tflops_sustained\": %.2f, \"err\": \"%s\"}\n",
         p.multiProcessorCount, best, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
