// On-device test problems (make_test_problem,
// deblur.cpp:201-229, for a whole batch of images): x_true (the BASELINE
// blob image), b_true = A x_true (the device operator) and the noise of
// Rng::normal (deblur.cpp:24-42) scaled to noise_level * ||b_true||.
//
// The random stream is the reference's: std::mt19937_64 restated on the
// device, one CTA per image — state in shared memory, each twist of the 312
// words in three dependency phases (words i < 156 read only old words; words
// 156..310 read the new words i - 156; word 311 reads the new words 0 and
// 155), outputs tempered in order — so the 64-bit outputs and the uniforms
// double(u >> 11) * 2^-53 are bit-identical to the host Rng
// (tests/test_gpu_problem_dev.py). Box-Muller (u1 = 1 - uniform, mag =
// sqrt(-2 log u1), cos / sin of 2 pi u2, spare = sin branch) uses the CUDA
// double-precision log / sin / cos (<= 1-2 ulp from glibc), so the normals
// — and through them noise and b — agree with the host generator to the
// last bits only; the blob image's exp likewise. The blob parameters (80
// uniform draws per image) come from the host Rng, exactly.
#include <cstdint>

#include "common.cuh"
#include "problem_dev.h"

namespace kp {
namespace {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ull, MT_UM = 0xFFFFFFFF80000000ull, MT_LM = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t hi_word, uint64_t far) {
  const uint64_t y = (lo_word & MT_UM) | (hi_word & MT_LM);
  return far ^ (y >> 1) ^ ((y & 1ull) ? MT_A : 0ull);
}

// Twist the state in place (std::mersenne_twister_engine::_M_gen_rand).
// Threads 0..MT_N-1 (blockDim >= 312).
__device__ void twist(uint64_t* mt) {
  const int i = threadIdx.x;
  uint64_t v = 0;
  if (i < MT_N - MT_M) v = mix(mt[i], mt[i + 1], mt[i + MT_M]);
  __syncthreads();
  if (i < MT_N - MT_M) mt[i] = v;
  __syncthreads();
  if (i >= MT_N - MT_M && i < MT_N - 1) v = mix(mt[i], mt[i + 1], mt[i + MT_M - MT_N]);
  __syncthreads();
  if (i >= MT_N - MT_M && i < MT_N - 1) mt[i] = v;
  __syncthreads();
  if (i == MT_N - 1) mt[i] = mix(mt[MT_N - 1], mt[0], mt[MT_M - 1]);
  __syncthreads();
}

__device__ void seed_state(uint64_t* mt, uint64_t seed) {
  if (threadIdx.x == 0) {  // sequential recurrence (312 steps)
    mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
  }
  __syncthreads();
}

__device__ __forceinline__ double uniform01(uint64_t u) { return double(u >> 11) * 0x1.0p-53; }

// Raw 64-bit outputs (test hook) for image blockIdx.x.
__global__ void mt_raw_kernel(const uint64_t* seeds, long count, uint64_t* out) {
  __shared__ uint64_t mt[MT_N];
  seed_state(mt, seeds[blockIdx.x]);
  out += size_t(blockIdx.x) * count;
  for (long base = 0; base < count; base += MT_N) {
    twist(mt);
    const long k = base + threadIdx.x;
    if (threadIdx.x < MT_N && k < count) out[k] = temper(mt[threadIdx.x]);
    __syncthreads();
  }
}

// Rng::normal() draws for image blockIdx.x: pair j (normals 2j, 2j+1) from
// uniforms 2j, 2j+1 of the stream; 312 outputs per twist = 156 pairs.
__global__ void rng_normals_kernel(const uint64_t* seeds, long count, double* out) {
  __shared__ uint64_t mt[MT_N];
  seed_state(mt, seeds[blockIdx.x]);
  out += size_t(blockIdx.x) * count;
  for (long base = 0; base < count; base += MT_N) {
    twist(mt);
    const int t = threadIdx.x;
    if (t < MT_N / 2) {
      const long k = base + 2 * t;
      if (k < count) {
        const double u1 = 1.0 - uniform01(temper(mt[2 * t]));
        const double u2 = uniform01(temper(mt[2 * t + 1]));
        const double mag = sqrt(-2.0 * log(u1));
        const double ang = 2.0 * 3.14159265358979323846 * u2;
        out[k] = mag * cos(ang);
        if (k + 1 < count) out[k + 1] = mag * sin(ang);
      }
    }
    __syncthreads();
  }
}

// x(i, j) = clip(sum_b amp_b exp(-((i - ci_b)^2 + (j - cj_b)^2) / (2 w_b^2)), 0, 1),
// blobs summed in order (kpg_blob_image); params[img][b] = {ci, cj, w, amp}.
__global__ void blob_image_kernel(int n, int blobs, const double* params, double* out) {
  const int img = blockIdx.y;
  params += size_t(img) * blobs * 4;
  out += size_t(img) * n * n;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < size_t(n) * n;
       q += size_t(gridDim.x) * blockDim.x) {
    const int j = int(q / n), i = int(q - size_t(j) * n);
    double v = 0.0;
    for (int b = 0; b < blobs; ++b) {
      const double ci = params[4 * b], cj = params[4 * b + 1], w = params[4 * b + 2], amp = params[4 * b + 3];
      const double inv = 1.0 / (2.0 * w * w);
      const double dj2 = (j - cj) * (j - cj), di2 = (i - ci) * (i - ci);
      v += amp * exp(-(di2 + dj2) * inv);
    }
    out[q] = fmin(1.0, fmax(0.0, v));
  }
}

// per image: [0] sum b_true^2, [1] sum g^2 over a fixed grid (deterministic)
constexpr int NORM_THREADS = 256, NORM_CTAS = 148;
__global__ void norms_kernel(const double* bt, const double* g, size_t nn, double* part) {
  const int img = blockIdx.y;
  bt += img * nn, g += img * nn;
  double s0 = 0.0, s1 = 0.0;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < nn; q += size_t(gridDim.x) * blockDim.x)
    s0 += bt[q] * bt[q], s1 += g[q] * g[q];
  __shared__ double red[NORM_THREADS / 32][2];
  for (int off = 16; off > 0; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = s0, red[threadIdx.x >> 5][1] = s1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < NORM_THREADS / 32; ++w) a += red[w][0], b += red[w][1];
    part[(size_t(img) * gridDim.x + blockIdx.x) * 2] = a;
    part[(size_t(img) * gridDim.x + blockIdx.x) * 2 + 1] = b;
  }
}

// noise = scale_i * g (in place), b = b_true + noise; scale_i = level_i *
// sqrt(sum b_true^2) / sqrt(sum g^2) from the partials (fixed order)
__global__ void noise_finish_kernel(const double* part, int ctas, const double* levels, size_t nn,
                                    const double* bt, double* noise, double* b, double* noise_norms) {
  const int img = blockIdx.y;
  __shared__ double scale;
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k < ctas; ++k) a += part[(size_t(img) * ctas + k) * 2], c += part[(size_t(img) * ctas + k) * 2 + 1];
    const double lv = levels[img];
    scale = lv == 0.0 ? 0.0 : lv * sqrt(a) / sqrt(c);
    if (blockIdx.x == 0 && noise_norms) noise_norms[img] = scale * sqrt(c);
  }
  __syncthreads();
  bt += img * nn, noise += img * nn, b += img * nn;
  for (size_t q = blockIdx.x * size_t(blockDim.x) + threadIdx.x; q < nn; q += size_t(gridDim.x) * blockDim.x) {
    const double e = scale * noise[q];
    noise[q] = e;
    b[q] = bt[q] + e;
  }
}

}  // namespace

void mt19937_64_raw(const uint64_t* seeds_dev, int batch, long count, uint64_t* out_dev) {
  LaunchScope scope(KC_VECTOR);
  mt_raw_kernel<<<batch, 320, 0, ctx().stream>>>(seeds_dev, count, out_dev);
  check_launch("mt19937_64 raw");
}

void rng_normals_dev(const uint64_t* seeds_dev, int batch, long count, double* out_dev) {
  LaunchScope scope(KC_VECTOR);
  rng_normals_kernel<<<batch, 320, 0, ctx().stream>>>(seeds_dev, count, out_dev);
  check_launch("rng normals");
}

void blob_images_dev(int n, int batch, int blobs, const double* params_dev, double* out_dev) {
  LaunchScope scope(KC_VECTOR);
  blob_image_kernel<<<dim3(592, batch), 256, 0, ctx().stream>>>(n, blobs, params_dev, out_dev);
  check_launch("blob images");
}

void add_noise_dev(int batch, size_t nn, const double* levels_dev, const double* b_true, double* g_noise,
                   double* b, double* noise_norms_dev) {
  DBuf<double> part(size_t(batch) * NORM_CTAS * 2);
  {
    LaunchScope scope(KC_VECTOR);
    norms_kernel<<<dim3(NORM_CTAS, batch), NORM_THREADS, 0, ctx().stream>>>(b_true, g_noise, nn, part.p);
    check_launch("noise norms");
  }
  LaunchScope scope(KC_VECTOR);
  noise_finish_kernel<<<dim3(592, batch), 256, 0, ctx().stream>>>(part.p, NORM_CTAS, levels_dev, nn, b_true,
                                                                  g_noise, b, noise_norms_dev);
  check_launch("noise finish");
}

}  // namespace kp
