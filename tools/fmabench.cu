// FP32 FMA-pipe throughput probe (B200): the attention kernel's exact fp32 fma chains run on CUDA cores, so
// its roofline peak is this measured rate.  Each thread runs 8 independent chains of 3-register FFMA (the
// operands are per-thread, so ptxas emits the register form the attention kernel uses, not the immediate or
// uniform-register form).  Measured on B200 (profiles/fp32_peak.json): 124 FFMA / clock / SM, 72.3 TFLOP/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fmabench.bin tools/fmabench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fma_kernel(float* out, float a, float b, int iters) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 0.001f + k;
  const float c = b * 0.5f + threadIdx.x * 1e-9f;
  const float av = a + threadIdx.x * 1e-9f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = __fmaf_rn(x[k], av, c);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 1.2345f) out[threadIdx.x] = s;                  // keeps the chains live
}

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    fma_kernel<<<blocks, threads>>>(out, 0.9999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = (double)blocks * threads * iters * 8, rate = fmas / (best * 1e-3);
  printf("{\"ms\": %.3f, \"ffma_per_s\": %.4g, \"fp32_tflops\": %.2f, \"ffma_per_clk_per_sm\": %.1f, \"sms\": %d}\n",
         best, rate, 2 * rate / 1e12, rate / sms / (khz * 1e3), sms);
  return 0;
}
