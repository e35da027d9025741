// On-device test-problem generation (see problem_dev.cu).
#pragma once

#include <cstddef>
#include <cstdint>

namespace kp {
// raw std::mt19937_64 outputs: count per seed (image), out[img * count + k]
void mt19937_64_raw(const uint64_t* seeds_dev, int batch, long count, uint64_t* out_dev);
// Rng::normal() streams (deblur.cpp:30-41), count per seed
void rng_normals_dev(const uint64_t* seeds_dev, int batch, long count, double* out_dev);
// blob images from per-image blob parameters {ci, cj, w, amp} x blobs
void blob_images_dev(int n, int batch, int blobs, const double* params_dev, double* out_dev);
// noise = level * ||b_true|| / ||g|| * g (g given in `g_noise`, overwritten), b = b_true + noise
void add_noise_dev(int batch, size_t nn, const double* levels_dev, const double* b_true, double* g_noise,
                   double* b, double* noise_norms_dev);
}  // namespace kp
