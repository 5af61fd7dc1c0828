// scatter_bench.cu — the access-pattern ceiling of the classify scan (not product code): random 64-B / 128-B
// segments gathered from a 15 GiB span by 16-B lane loads (4 / 8 lanes per segment, 8 loads in flight per
// thread), next to a contiguous 16-B-per-lane stream; and, for the bulk writer, contiguous read+write streams
// at R bytes read per byte written (R = 1: a copy; R = 3, 4 bracket the bulk writer's 3.2 : 1 DRAM mix).
// Prints achieved GB/s (bytes requested / kernel time).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scatter_bench tools/scatter_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}
template <int SEG>
__global__ void gather(const uint4* __restrict__ buf, uint64_t nseg_span, int iters, uint64_t* sink) {
  constexpr int LPS = SEG / 16;                           // lanes per segment
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t g = t / LPS;                               // segment group of this thread
  const int part = (int)(t % LPS);
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint64_t seg = mix(g * 1315423911ull + (uint64_t)(it * 8 + j)) % nseg_span;
      v[j] = __ldg(buf + seg * LPS + part);
    }
#pragma unroll
    for (int j = 0; j < 8; j++) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}
__global__ void stream(const uint4* __restrict__ buf, uint64_t n16, uint64_t* sink) {
  uint32_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(buf + i);
    acc += v.x ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}
template <int R>
__global__ void rw_stream(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n_out) {
  for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n_out; o += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v[R];
#pragma unroll
    for (int j = 0; j < R; j++) v[j] = __ldcs(in + (uint64_t)j * n_out + o);   // R contiguous streams
    uint4 w = v[0];
#pragma unroll
    for (int j = 1; j < R; j++) { w.x ^= v[j].x; w.y ^= v[j].y; w.z ^= v[j].z; w.w ^= v[j].w; }
    __stcs(out + o, w);
  }
}
int main() {
  const uint64_t span = 15ull << 30;
  uint4* buf;
  uint64_t* sink;
  if (cudaMalloc(&buf, span) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, span);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int threads = 256, blocks = 148 * 8, iters = 64;
  float ms;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    gather<64><<<blocks, threads>>>(buf, span / 64, iters, sink);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)blocks * threads / 4 * iters * 8 * 64;
    printf("random 64-B segments : %8.1f GB/s (%.0f MB)\n", bytes / ms / 1e6, bytes / 1e6);
    cudaEventRecord(a);
    gather<128><<<blocks, threads>>>(buf, span / 128, iters, sink);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    bytes = (double)blocks * threads / 8 * iters * 8 * 128;
    printf("random 128-B segments: %8.1f GB/s (%.0f MB)\n", bytes / ms / 1e6, bytes / 1e6);
    const uint64_t n16 = (4ull << 30) / 16;
    cudaEventRecord(a);
    stream<<<148 * 8, 256>>>(buf, n16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("contiguous read      : %8.1f GB/s (4096 MB)\n", (double)(4ull << 30) / ms / 1e6);
    // read R x 2 GiB + write 2 GiB (output in the upper part of the span)
    const uint64_t n_out = (2ull << 30) / 16;
    uint4* outp = buf + (12ull << 30) / 16;
    for (int R = 1; R <= 4; R++) {
      cudaEventRecord(a);
      if (R == 1) rw_stream<1><<<148 * 8, 256>>>(buf, outp, n_out);
      if (R == 2) rw_stream<2><<<148 * 8, 256>>>(buf, outp, n_out);
      if (R == 3) rw_stream<3><<<148 * 8, 256>>>(buf, outp, n_out);
      if (R == 4) rw_stream<4><<<148 * 8, 256>>>(buf, outp, n_out);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("read:write %d:1 stream: %8.1f GB/s (%d MB)\n", R, (double)(R + 1) * (2ull << 30) / ms / 1e6,
             (int)((R + 1) * 2048));
    }
  }
  return 0;
}
