// membench.cu — memory-system probes behind the decode-step kernel design (not product code).
//   1. random 64-B reads (4 lanes x 16 B) scattered over the first `span` bytes of a 15 GiB buffer:
//      achieved GB/s vs span (TLB reach / DRAM random-access efficiency);
//   2. pointer chase by one warp over `span`: dependent-load latency vs span (TLB miss cost);
//   3. strided 256-B row read+write (the decode window push pattern): GB/s vs stride.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull; return x ^ (x >> 31);
}

__global__ void rand_read64(const uint8_t* buf, uint64_t span, int nreq, int iters, uint32_t* out) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 2, q = threadIdx.x & 3;
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
    const int r = g + it * (gridDim.x * blockDim.x >> 2);
    if (r >= nreq) break;
    const uint64_t off = (mix((uint64_t)r * 7919u) % (span / 64)) * 64;
    const uint4 v = *reinterpret_cast<const uint4*>(buf + off + 16 * q);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void chase(const uint8_t* buf, uint64_t span, int steps, uint64_t* out) {
  uint64_t x = 1;
  for (int i = 0; i < steps; i++) {
    const uint64_t off = (mix(x + i) % (span / 64)) * 64;
    x += *reinterpret_cast<const uint32_t*>(buf + off);   // dependent on the previous load
  }
  out[0] = x;
}

__global__ void strided_rows(uint8_t* buf, uint64_t stride, int rows) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  uint2* row = reinterpret_cast<uint2*>(buf + (uint64_t)w * stride);
  const uint2 v = row[lane];                                     // 256 B read
  row[lane] = make_uint2(v.x + 1, v.y);                          // 256 B write
}

int main() {
  const uint64_t total = 15ull << 30;
  uint8_t* buf;
  uint32_t* o32;
  uint64_t* o64;
  CK(cudaMalloc(&buf, total));
  CK(cudaMalloc(&o32, 64));
  CK(cudaMalloc(&o64, 64));
  CK(cudaMemset(buf, 1, total));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int nreq = 1 << 21;                                      // 2M x 64 B = 128 MiB per launch
  printf("random 64-B reads, %d requests (128 MiB):\n", nreq);
  for (uint64_t span : {256ull << 20, 1ull << 30, 2ull << 30, 4ull << 30, 8ull << 30, 15ull << 30}) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a);
      rand_read64<<<148 * 8, 256>>>(buf, span, nreq, (nreq * 4 + 148 * 8 * 256 - 1) / (148 * 8 * 256), o32);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("  span %6.2f GiB: %8.1f us  %7.1f GB/s\n", span / double(1 << 30), best * 1e3, nreq * 64.0 / (best * 1e-3) / 1e9);
  }
  printf("pointer chase (1 thread, 4096 dependent 4-B loads):\n");
  for (uint64_t span : {16ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 8ull << 30, 15ull << 30}) {
    float best = 1e9f;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a);
      chase<<<1, 1>>>(buf, span, 4096, o64);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("  span %6.2f GiB: %7.1f ns per load\n", span / double(1 << 30), best * 1e6 / 4096);
  }
  printf("strided 256-B rows read+write, 16384 rows:\n");
  for (uint64_t stride : {256ull, 512ull, 4096ull, 16384ull, 16384ull + 256, 65536ull, 524288ull}) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a);
      strided_rows<<<16384 / 8, 256>>>(buf, stride, 16384);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("  stride %7llu B: %7.2f us  %7.1f GB/s\n", (unsigned long long)stride, best * 1e3, 16384 * 512.0 / (best * 1e-3) / 1e9);
  }
  return 0;
}
