// membench2.cu — decode window-push access pattern probes (not product code): per unit, read t_c's
// K row and V row (256 B each) and overwrite them, 16384 units, warp per unit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void win(uint8_t* kb, uint8_t* vb, uint64_t ustride, int U, int slot_mode, uint64_t* sink) {
  const int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (u >= U) return;
  const int ws = slot_mode == 0 ? 17 : (u * 7) % 64;
  uint2* k = reinterpret_cast<uint2*>(kb + (uint64_t)u * ustride + ws * 256) + lane;
  uint2* v = reinterpret_cast<uint2*>(vb + (uint64_t)u * ustride + ws * 256) + lane;
  const uint2 a = *k, b = *v;
  *k = make_uint2(a.x + 1, a.y);
  *v = make_uint2(b.x + 1, b.y);
}
int main() {
  uint8_t* buf;
  uint64_t* sink;
  cudaMalloc(&buf, 2ull << 30);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 0, 2ull << 30);
  uint8_t* flush;
  cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  struct V { const char* name; uint64_t voff, ustride; int mode; } vs[] = {
    {"separate K/V (+256MiB), stride 16K, same slot", 256ull << 20, 16384, 0},
    {"separate K/V (+256MiB+4K), stride 16K, same slot", (256ull << 20) + 4096, 16384, 0},
    {"separate K/V (+256MiB), stride 16K+256, same slot", 256ull << 20, 16384 + 256, 0},
    {"separate K/V (+256MiB), stride 16K, slot varies", 256ull << 20, 16384, 1},
    {"interleaved K|V (+256B), stride 32K, same slot", 256, 32768, 0},
    {"interleaved K|V (+256B), stride 32K+512, same slot", 256, 32768 + 512, 0},
    {"K only-ish: V at +8K, stride 16K, same slot", 8192, 16384, 0},
  };
  for (auto& x : vs) {
    float best = 1e9f, sum = 0;
    for (int rep = 0; rep < 8; rep++) {
      cudaMemset(flush, rep, 512ull << 20);
      cudaEventRecord(a);
      win<<<16384 / 8, 256>>>(buf, buf + x.voff, x.ustride, 16384, x.mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
      sum += ms;
    }
    printf("%-55s best %7.2f us  mean %7.2f us\n", x.name, best * 1e3, sum / 8 * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
