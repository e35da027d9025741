// Pipe-mix microbenchmark: can FP32 FMUL (fmalite) and F2FP.F16.F32 packs
// run beside f16x2 HMUL2/HADD2 (fmaheavy) without slowing them? Decides
// whether part of the reference-exact fp16 products can be offloaded.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ unsigned hmul2(unsigned a, unsigned b) {
  unsigned r; asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ unsigned hadd2(unsigned a, unsigned b) {
  unsigned r; asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ float fmul(float a, float b) {
  float r; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ unsigned f2h2(float a, float b) {
  unsigned r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }

__device__ __forceinline__ unsigned hfma2(unsigned a, unsigned b, unsigned c) {
  unsigned r; asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }

// all f16x2 work as fma.rn.f16x2 (mul = fma(a, b, -0), add = fma(a, 1, b))
__global__ void fma_only_k(unsigned* out, int iters) {
  constexpr int ILP = 8;
  unsigned h[ILP];
  for (int i = 0; i < ILP; ++i) h[i] = 0x3c003c00u + threadIdx.x + i;
  const unsigned m = 0x3c003c01u, one = 0x3c003c00u, nz = 0x80008000u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
#pragma unroll
      for (int q = 0; q < 8; ++q) h[i] = (q & 1) ? hfma2(h[i], one, m) : hfma2(h[i], m, nz);
    }
  }
  unsigned s = 0;
  for (int i = 0; i < ILP; ++i) s ^= h[i];
  if (s == 0x12345678u) out[0] = s;
}

// H: f16x2 ops per iteration per ILP slot, F: fmul, C: cvt packs
template <int H, int F, int CV>
__global__ void mix_k(unsigned* out, int iters) {
  constexpr int ILP = 8;
  unsigned h[ILP];
  float f[ILP];
  unsigned c[ILP];
  for (int i = 0; i < ILP; ++i) {
    h[i] = 0x3c003c00u + threadIdx.x + i;
    f[i] = 1.0f + threadIdx.x * 1e-7f + i;
    c[i] = 0;
  }
  const unsigned m = 0x3c003c01u;
  const float g = 0.99999f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
#pragma unroll
      for (int q = 0; q < H; ++q) h[i] = (q & 1) ? hadd2(h[i], m) : hmul2(h[i], m);
#pragma unroll
      for (int q = 0; q < F; ++q) f[i] = fmul(f[i], g);
#pragma unroll
      for (int q = 0; q < CV; ++q) c[i] ^= f2h2(f[i], f[(i + 1) % ILP]);
    }
  }
  unsigned s = 0;
  for (int i = 0; i < ILP; ++i) s ^= h[i] ^ __float_as_uint(f[i]) ^ c[i];
  if (s == 0x12345678u) out[0] = s;
}

template <int H, int F, int CV>
int run(const char* name) {
  unsigned* d; CK(cudaMalloc(&d, 4));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int iters = 4096, blocks = sms * 8, threads = 256;
  mix_k<H, F, CV><<<blocks, threads>>>(d, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  mix_k<H, F, CV><<<blocks, threads>>>(d, iters);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_iters = double(blocks) * threads / 32 * iters * 8;  // x ILP
  const double cycles = ms * 1e-3 * clk * 1e3 * sms;  // SM-cycles at the nominal clock
  printf("%-28s %8.3f ms  per SM-cycle: f16x2 %.2f  fmul %.2f  cvt %.2f warp-instr\n", name, ms,
         warp_iters * H / cycles, warp_iters * F / cycles, warp_iters * CV / cycles);
  return 0;
}

int run_fma() {
  unsigned* d; CK(cudaMalloc(&d, 4));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  const int iters = 4096, blocks = sms * 8, threads = 256;
  fma_only_k<<<blocks, threads>>>(d, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  fma_only_k<<<blocks, threads>>>(d, iters);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_iters = double(blocks) * threads / 32 * iters * 8;
  const double cycles = ms * 1e-3 * clk * 1e3 * sms;
  printf("%-28s %8.3f ms  per SM-cycle: f16x2 %.2f warp-instr (%.1f T half-ops/s)\n", "fma.rn.f16x2 only", ms,
         warp_iters * 8 / cycles, warp_iters * 8 * 64 / (ms * 1e-3) / 1e12);
  return 0;
}

int main() {
  run_fma();
  run<8, 0, 0>("f16x2 only");
  run<0, 8, 0>("fmul only");
  run<0, 1, 4>("cvt.f16x2.f32 (+1 fmul)");
  run<8, 4, 0>("f16x2 8 + fmul 4");
  run<8, 8, 0>("f16x2 8 + fmul 8");
  run<8, 1, 2>("f16x2 8 + cvt 2");
  run<8, 4, 2>("f16x2 8 + fmul 4 + cvt 2");
  run<6, 4, 2>("f16x2 6 + fmul 4 + cvt 2");
  return 0;
}
