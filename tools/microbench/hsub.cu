// f16x2 add / fma throughput with normal vs subnormal operands (is there a
// data-dependent slowdown on B200?). Each thread runs 8 independent chains.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

__global__ void k_add(uint32_t seed_bits, uint32_t inc_bits, int iters, uint32_t* out) {
  uint32_t v[8];
  for (int c = 0; c < 8; ++c) v[c] = seed_bits;
  const uint32_t inc = inc_bits;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(v[c]) : "r"(inc));
#pragma unroll
    for (int c = 0; c < 8; ++c) asm volatile("sub.rn.f16x2 %0, %0, %1;" : "+r"(v[c]) : "r"(inc));
  }
  uint32_t s = 0;
  for (int c = 0; c < 8; ++c) s ^= v[c];
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Case { const char* name; uint32_t seed, inc; } cases[] = {
      {"normal (1.0 +- 0.5)", 0x3c003c00u, 0x38003800u},
      {"subnormal (2^-20 +- 2^-22)", 0x00100010u, 0x00040004u},
      {"zeros (0 +- 0)", 0x00000000u, 0x00000000u},
      {"mixed (1.0 +- 2^-22)", 0x3c003c00u, 0x00040004u},
  };
  const int iters = 20000, blocks = 148 * 8, threads = 256;
  for (auto& c : cases) {
    k_add<<<blocks, threads>>>(c.seed, c.inc, 100, d);
    cudaEventRecord(a);
    k_add<<<blocks, threads>>>(c.seed, c.inc, iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = double(blocks) * threads * iters * 16 * 2;  // half-adds
    printf("%-30s %.3f ms  %.2f T half-adds/s\n", c.name, ms, ops / ms / 1e9);
  }
  return 0;
}
