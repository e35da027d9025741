// Host-side problem generation and operator setup (not on the hot path).
//
// Restates the reference's test-problem generator (deblur.cpp) and the
// setup helpers the hot path consumes (nearest_kron, factor.cpp:25-58), plus
// the generators the BASELINE configs need but the reference API cannot
// express (blob image, anisotropic Gaussian PSF, Gaussian*motion PSF, rank
// cap). Both arms — the CUDA path and the CPU oracle — consume
// exactly these arrays, so the inputs are pinned identically.
//
// SVDs and FP64 GEMMs use numpy's bundled OpenBLAS (LAPACK dgesdd / dgemm).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_la.h"

namespace kpg {

// Rng (deblur.cpp:24-42): mt19937_64 with hand-rolled uniform / Box-Muller.
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double uniform() { return double(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double mag = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * M_PI * u2;
    spare_ = mag * std::sin(ang);
    have_spare_ = true;
    return mag * std::cos(ang);
  }

 private:
  std::mt19937_64 eng_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// banded_toeplitz (deblur.cpp:157-165)
void banded_toeplitz(const double* w, int len, int c, int n, double* t) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int k = i - j + c;
      t[size_t(j) * n + i] = (k >= 0 && k < len) ? w[k] : 0.0;
    }
}

}  // namespace kpg

using namespace kpg;

static thread_local std::string g_gen_err;

#define KPG_TRY(...)                       \
  try {                                    \
    __VA_ARGS__;                           \
    return 0;                              \
  } catch (const std::invalid_argument& e) { \
    g_gen_err = e.what();                  \
    return 1;                              \
  } catch (const std::exception& e) {      \
    g_gen_err = e.what();                  \
    return 2;                              \
  }

extern "C" {

const char* kpg_last_error(void) { return g_gen_err.c_str(); }

void kpg_rng_normals(uint64_t seed, long count, double* out) {
  Rng rng(seed);
  for (long i = 0; i < count; ++i) out[i] = rng.normal();
}
void kpg_rng_uniforms(uint64_t seed, long count, double lo, double hi,
                      double* out) {
  Rng rng(seed);
  for (long i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}
// The blob parameters kpg_blob_image draws, {ci, cj, w, amp} per blob
// (for the on-device generator, problem_dev.cu).
void kpg_blob_params(int n, uint64_t seed, int blobs, double* out) {
  Rng rng(seed);
  for (int b = 0; b < blobs; ++b) {
    out[4 * b] = rng.uniform(0.0, double(n));
    out[4 * b + 1] = rng.uniform(0.0, double(n));
    out[4 * b + 2] = rng.uniform(5.0, 30.0);
    out[4 * b + 3] = rng.uniform();
  }
}

// make_psf (deblur.cpp:130-155). kind: 0 gaussian, 1 defocus, 2 motion
// (45-degree diagonal), 3 shake, 4 speckle. out: np*np column-major.
int kpg_make_psf(int kind, int np, double sigma, double radius, int length,
                 int steps, int blob_count, double blob_sigma, uint64_t seed,
                 double* out) {
  KPG_TRY({
    if (np < 1 || np % 2 == 0)
      throw std::invalid_argument("make_psf: psf size must be odd and positive");
    const int c = np / 2;
    auto at = [&](int i, int j) -> double& { return out[size_t(j) * np + i]; };
    std::memset(out, 0, sizeof(double) * size_t(np) * np);
    Rng rng(seed);
    if (kind == 0) {  // fill_gaussian (deblur.cpp:66-73)
      if (sigma <= 0.0) throw std::invalid_argument("make_psf: sigma must be > 0");
      std::vector<double> g(np);
      for (int i = 0; i < np; ++i)
        g[i] = std::exp(-0.5 * double(i - c) * double(i - c) / (sigma * sigma));
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i) at(i, j) = g[i] * g[j];
    } else if (kind == 1) {  // fill_defocus (:75-84)
      if (radius < 0.0) throw std::invalid_argument("make_psf: radius must be >= 0");
      for (int i = 0; i < np; ++i)
        for (int j = 0; j < np; ++j) {
          const double d2 = double(i - c) * (i - c) + double(j - c) * (j - c);
          at(i, j) = d2 <= radius * radius ? 1.0 : 0.0;
        }
    } else if (kind == 2) {  // fill_motion (:86-94)
      if (length < 1) throw std::invalid_argument("make_psf: length must be >= 1");
      const int start = -((length - 1) / 2);
      if (c + start < 0 || c + start + length - 1 >= np)
        throw std::invalid_argument("make_psf: motion segment exceeds psf array");
      for (int k = 0; k < length; ++k) at(c + start + k, c + start + k) = 1.0;
    } else if (kind == 3) {  // fill_shake (:96-107)
      if (steps < 1) throw std::invalid_argument("make_psf: steps must be >= 1");
      double pr = c, pc = c;
      for (int s = 0; s < steps; ++s) {
        const int i = int(std::lround(pr));
        const int j = int(std::lround(pc));
        at(i, j) += 1.0;
        pr = std::min(std::max(pr + rng.uniform(-1.0, 1.0), 0.0), double(np - 1));
        pc = std::min(std::max(pc + rng.uniform(-1.0, 1.0), 0.0), double(np - 1));
      }
    } else if (kind == 4) {  // fill_speckle (:109-126)
      if (blob_count < 1) throw std::invalid_argument("make_psf: blob_count must be >= 1");
      if (blob_sigma <= 0.0) throw std::invalid_argument("make_psf: blob_sigma must be > 0");
      for (int b = 0; b < blob_count; ++b) {
        const double bi = rng.uniform(0.0, double(np - 1));
        const double bj = rng.uniform(0.0, double(np - 1));
        const double amp = rng.uniform(0.5, 1.5);
        for (int i = 0; i < np; ++i)
          for (int j = 0; j < np; ++j) {
            const double d2 = (i - bi) * (i - bi) + (j - bj) * (j - bj);
            at(i, j) += amp * std::exp(-0.5 * d2 / (blob_sigma * blob_sigma));
          }
      }
    } else {
      throw std::invalid_argument("make_psf: unknown blur kind");
    }
    double sum = 0.0;  // psf.values /= psf.values.sum()
    for (size_t q = 0; q < size_t(np) * np; ++q) sum += out[q];
    for (size_t q = 0; q < size_t(np) * np; ++q) out[q] /= sum;
  })
}

// NEW (config 2/3, not expressible in the reference): anisotropic Gaussian
// p(i,j) ~ exp(-1/2 d^T Cov^{-1} d), d = (i - c, j - c), normalised.
int kpg_psf_aniso_gaussian(int np, double c00, double c01, double c11,
                           double* out) {
  KPG_TRY({
    if (np < 1 || np % 2 == 0) throw std::invalid_argument("psf size must be odd");
    const double det = c00 * c11 - c01 * c01;
    if (!(det > 0.0)) throw std::invalid_argument("covariance must be SPD");
    const double i00 = c11 / det, i01 = -c01 / det, i11 = c00 / det;
    const int c = np / 2;
    double sum = 0.0;
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i) {
        const double di = i - c, dj = j - c;
        const double q = i00 * di * di + 2.0 * i01 * di * dj + i11 * dj * dj;
        const double v = std::exp(-0.5 * q);
        out[size_t(j) * np + i] = v;
        sum += v;
      }
    for (size_t q = 0; q < size_t(np) * np; ++q) out[q] /= sum;
  })
}

// NEW (config 5): isotropic Gaussian (sigma) convolved with a `length`-sample
// linear motion segment at `angle_deg` (counter-clockwise from the column
// axis, rows pointing down), evaluated exactly: sum over samples t in
// [-(L-1)/2, (L-1)/2] of a Gaussian centred at (c - t sin a, c + t cos a).
int kpg_psf_gauss_motion(int np, double sigma, int length, double angle_deg,
                         double* out) {
  KPG_TRY({
    if (np < 1 || np % 2 == 0) throw std::invalid_argument("psf size must be odd");
    if (length < 1 || sigma <= 0.0) throw std::invalid_argument("bad motion psf");
    const int c = np / 2;
    const double a = angle_deg * M_PI / 180.0;
    const double half = 0.5 * (length - 1);
    std::memset(out, 0, sizeof(double) * size_t(np) * np);
    for (int s = 0; s < length; ++s) {
      const double t = -half + s;
      const double ri = c - t * std::sin(a), cj = c + t * std::cos(a);
      for (int j = 0; j < np; ++j)
        for (int i = 0; i < np; ++i) {
          const double d2 = (i - ri) * (i - ri) + (j - cj) * (j - cj);
          out[size_t(j) * np + i] += std::exp(-0.5 * d2 / (sigma * sigma));
        }
    }
    double sum = 0.0;
    for (size_t q = 0; q < size_t(np) * np; ++q) sum += out[q];
    for (size_t q = 0; q < size_t(np) * np; ++q) out[q] /= sum;
  })
}

// default_test_image (deblur.cpp:231-246)
int kpg_default_test_image(int n, double* out) {
  KPG_TRY({
    if (n < 1) throw std::invalid_argument("default_test_image: n must be >= 1");
    for (size_t q = 0; q < size_t(n) * n; ++q) out[q] = 0.1;
    const int r0 = int(0.20 * n), r1 = int(0.55 * n);
    const int c0 = int(0.15 * n), c1 = int(0.45 * n);
    for (int i = r0; i < r1; ++i)
      for (int j = c0; j < c1; ++j) out[size_t(j) * n + i] = 0.7;
    const double dr = 0.62 * n, dc = 0.68 * n, rad = 0.18 * n;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if ((i - dr) * (i - dr) + (j - dc) * (j - dc) <= rad * rad)
          out[size_t(j) * n + i] = 1.0;
  })
}

// NEW (all BASELINE configs): seeded sum of Gaussian blobs, clipped to
// [0, 1]. Draw order per blob: centre row U[0,n), centre col U[0,n), width
// U[5,30], amplitude U[0,1].
int kpg_blob_image(int n, uint64_t seed, int blobs, double* out) {
  KPG_TRY({
    if (n < 1 || blobs < 0) throw std::invalid_argument("blob_image: bad size");
    Rng rng(seed);
    std::vector<double> ci(blobs), cj(blobs), w(blobs), amp(blobs);
    for (int b = 0; b < blobs; ++b) {
      ci[b] = rng.uniform(0.0, double(n));
      cj[b] = rng.uniform(0.0, double(n));
      w[b] = rng.uniform(5.0, 30.0);
      amp[b] = rng.uniform();
    }
    for (size_t q = 0; q < size_t(n) * n; ++q) out[q] = 0.0;
    for (int b = 0; b < blobs; ++b) {
      const double inv = 1.0 / (2.0 * w[b] * w[b]);
      for (int j = 0; j < n; ++j) {
        const double dj2 = (j - cj[b]) * (j - cj[b]);
        for (int i = 0; i < n; ++i) {
          const double di2 = (i - ci[b]) * (i - ci[b]);
          out[size_t(j) * n + i] += amp[b] * std::exp(-(di2 + dj2) * inv);
        }
      }
    }
    for (size_t q = 0; q < size_t(n) * n; ++q)
      out[q] = std::min(1.0, std::max(0.0, out[q]));
  })
}

// psf_to_kronsum (deblur.cpp:167-199) with an optional rank cap (NEW,
// configs 2/3/5; max_rank <= 0 = no cap). Writes up to `capacity` terms:
// row_factors / col_factors hold r consecutive n*n col-major matrices.
// truncated_psf (optional, np*np) receives sum_{k<r} s_k u_k v_k^T — the
// capped PSF array that configs 2/3/5 also hand to nearest_kron.
int kpg_psf_to_kronsum(const double* psf, int np, int crow, int ccol, int n,
                       double tol, int max_rank, int capacity,
                       double* row_factors, double* col_factors, int* r_out,
                       double* truncated_psf) {
  KPG_TRY({
    if (n < np) throw std::invalid_argument("psf_to_kronsum: image smaller than psf");
    if (tol < 0.0) throw std::invalid_argument("psf_to_kronsum: negative truncation_tol");
    kpla::Svd s = kpla::svd(psf, np, np);
    int r = 0;
    if (truncated_psf) std::memset(truncated_psf, 0, sizeof(double) * size_t(np) * np);
    std::vector<double> u(np), v(np), wr(np), wc(np);
    for (int k = 0; k < np; ++k) {
      if (s.s[k] <= 0.0) break;
      if (k > 0 && s.s[k] <= tol * s.s[0]) break;
      if (max_rank > 0 && r >= max_rank) break;
      if (r >= capacity) throw std::invalid_argument("psf_to_kronsum: capacity too small");
      for (int i = 0; i < np; ++i) u[i] = s.u[size_t(k) * np + i];
      for (int i = 0; i < np; ++i) v[i] = s.v[size_t(k) * np + i];
      int imax = 0;  // sign fix: largest |u| entry positive
      for (int i = 1; i < np; ++i)
        if (std::fabs(u[i]) > std::fabs(u[imax])) imax = i;
      if (u[imax] < 0.0)
        for (int i = 0; i < np; ++i) u[i] = -u[i], v[i] = -v[i];
      const double root = std::sqrt(s.s[k]);
      for (int i = 0; i < np; ++i) wr[i] = root * v[i], wc[i] = root * u[i];
      banded_toeplitz(wr.data(), np, ccol, n, row_factors + size_t(r) * n * n);
      banded_toeplitz(wc.data(), np, crow, n, col_factors + size_t(r) * n * n);
      if (truncated_psf)
        for (int j = 0; j < np; ++j)
          for (int i = 0; i < np; ++i)
            truncated_psf[size_t(j) * np + i] += s.s[k] * u[i] * v[j];
      ++r;
    }
    if (r == 0) throw std::invalid_argument("psf_to_kronsum: psf has no nonzero terms");
    *r_out = r;
  })
}

// nearest_kron, Toeplitz weighting (factor.cpp:25-58). weighting 1 =
// Toeplitz (default), 0 = uniform (dominant term of psf_to_kronsum).
int kpg_nearest_kron(const double* psf, int np, int crow, int ccol, int n,
                     int weighting, double* row_factor, double* col_factor) {
  KPG_TRY({
    if (n < np) throw std::invalid_argument("nearest_kron: image smaller than psf");
    if (weighting == 0) {
      int r = 0;
      if (kpg_psf_to_kronsum(psf, np, crow, ccol, n, 1.0, 1, 1, row_factor,
                             col_factor, &r, nullptr) != 0)
        throw std::runtime_error(g_gen_err);
      return 0;
    }
    std::vector<double> dr(np), dc(np), wtd(size_t(np) * np);
    for (int i = 0; i < np; ++i) dr[i] = std::sqrt(double(n - std::abs(i - crow)));
    for (int j = 0; j < np; ++j) dc[j] = std::sqrt(double(n - std::abs(j - ccol)));
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < np; ++i)
        wtd[size_t(j) * np + i] = dr[i] * psf[size_t(j) * np + i] * dc[j];
    kpla::Svd s = kpla::svd(wtd.data(), np, np);
    std::vector<double> u(s.u.begin(), s.u.begin() + np), v(s.v.begin(), s.v.begin() + np);
    int imax = 0;
    for (int i = 1; i < np; ++i)
      if (std::fabs(u[i]) > std::fabs(u[imax])) imax = i;
    if (u[imax] < 0.0)
      for (int i = 0; i < np; ++i) u[i] = -u[i], v[i] = -v[i];
    const double root = std::sqrt(s.s[0]);
    std::vector<double> acol(np), arow(np);
    for (int i = 0; i < np; ++i) acol[i] = root * (u[i] / dr[i]);
    for (int i = 0; i < np; ++i) arow[i] = root * (v[i] / dc[i]);
    banded_toeplitz(arow.data(), np, ccol, n, row_factor);
    banded_toeplitz(acol.data(), np, crow, n, col_factor);
  })
}

// Host FP64 kronsum_apply (kron.cpp:73-79) for b_true = A x_true; setup only.
int kpg_kronsum_apply_host(int n, int r, const double* rowf, const double* colf,
                           const double* y, double* out) {
  KPG_TRY({
    const size_t nn = size_t(n) * n;
    std::vector<double> t(nn), u(nn);
    std::fill(out, out + nn, 0.0);
    for (int k = 0; k < r; ++k) {
      kpla::dgemm('N', 'N', n, n, n, 1.0, colf + k * nn, n, y, n, 0.0, t.data(), n);
      kpla::dgemm('N', 'T', n, n, n, 1.0, t.data(), n, rowf + k * nn, n, 0.0, u.data(), n);
      for (size_t i = 0; i < nn; ++i) out[i] += u[i];
    }
  })
}

// make_test_problem noise step (deblur.cpp:214-227): noise =
// noise_level * ||b_true|| / ||g|| * g with g ~ Rng(seed).normal().
int kpg_add_noise(long count, const double* b_true, double noise_level,
                  uint64_t seed, double* noise, double* b) {
  KPG_TRY({
    if (noise_level < 0.0) throw std::invalid_argument("make_test_problem: negative noise level");
    if (noise_level == 0.0) {
      for (long i = 0; i < count; ++i) noise[i] = 0.0, b[i] = b_true[i];
      return 0;
    }
    Rng rng(seed);
    double gn = 0.0, bn = 0.0;
    for (long i = 0; i < count; ++i) {
      noise[i] = rng.normal();
      gn += noise[i] * noise[i];
      bn += b_true[i] * b_true[i];
    }
    const double scale = noise_level * std::sqrt(bn) / std::sqrt(gn);
    for (long i = 0; i < count; ++i) {
      noise[i] = scale * noise[i];
      b[i] = b_true[i] + noise[i];
    }
  })
}

// LAPACK SVD exposed for host callers (dgesdd; u, v n-by-n col-major).
int kpg_svd(const double* a, int m, int n, double* u, double* s, double* v) {
  KPG_TRY({
    kpla::Svd r = kpla::svd(a, m, n);
    std::memcpy(u, r.u.data(), r.u.size() * sizeof(double));
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    std::memcpy(v, r.v.data(), r.v.size() * sizeof(double));
  })
}

void kpg_set_blas_threads(int t) { kpla::set_threads(t); }

}  // extern "C"
