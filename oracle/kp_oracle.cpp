// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into, or called by, the
// product library (paper_2311_15393_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it.
//
// CPU restatement of the reference `kronprec` hot path (/root/reference/proj),
// which cannot be compiled here: it needs Eigen 3.4 (absent).
// Every function cites the reference lines it follows. Parity pin: the
// reference's own known-answer tests (test_precision.cpp, test_lpblas.cpp,
// test_factor.cpp, test_krylov.cpp, test_regparam.cpp, acceptance.cpp) are
// re-expressed in tests/test_oracle_kat.py and must pass against this file.
//
// Deviations that are unavoidable without Eigen, all tolerance-level:
//  * FP64 GEMMs go through OpenBLAS dgemm (numpy's bundled libscipy_openblas64_)
//    instead of Eigen's GEMM: different summation order.
//  * SVDs use LAPACK dgesdd instead of Eigen::JacobiSVD: singular vectors may
//    differ by sign (and rounding); the preconditioner is sign-invariant.
//  * dot/norm reductions are plain left-to-right loops, not Eigen packets.
// The low-precision arithmetic (precision.cpp, lpblas.cpp) is restated
// bit-exactly; lp_matmul is STREAMED per output element (same pairwise tree,
// same roundings) instead of materialising the m x (K n) product matrix
// (lpblas.cpp:65-67), which needs 69 GB at n=2048.

#include "kp_oracle.h"

#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

// ---- OpenBLAS / LAPACK (ILP64, numpy-bundled) -------------------------------
extern "C" {
void scipy_dgemm_64_(const char* ta, const char* tb, const long* m,
                     const long* n, const long* k, const double* alpha,
                     const double* a, const long* lda, const double* b,
                     const long* ldb, const double* beta, double* c,
                     const long* ldc, size_t, size_t);
void scipy_dgesdd_64_(const char* jobz, const long* m, const long* n,
                      double* a, const long* lda, double* s, double* u,
                      const long* ldu, double* vt, const long* ldvt,
                      double* work, const long* lwork, long* iwork, long* info,
                      size_t);
void scipy_openblas_set_num_threads64_(int);
}

namespace kpo {

struct NoRootError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

static thread_local std::string g_err;
static thread_local uint64_t g_round_calls = 0;  // precision.cpp:11
static int g_threads = 1;

// ---- precision.cpp -----------------------------------------------------------
struct Fmt {
  int t = 53, emax = 1023;
  bool sub = true;
  int emin() const { return 1 - emax; }  // precision.cpp:76
  double max_finite() const {            // precision.cpp:68-70
    return std::ldexp(2.0 - std::ldexp(1.0, 1 - t), emax);
  }
  double overflow_threshold() const {  // precision.cpp:72-74
    return std::ldexp(2.0 - std::ldexp(1.0, -t), emax);
  }
  bool covers_double() const {  // precision.cpp:78-80
    return t >= 53 && emax >= 1023 && sub;
  }
  bool is_fp16() const { return t == 11 && emax == 15 && sub; }
};
static Fmt fmt_of(kp_format f) {
  Fmt r;
  r.t = f.significand_bits;
  r.emax = f.max_exponent;
  r.sub = f.subnormals_enabled != 0;
  return r;
}

// precision.cpp:15-21
static double nearest_even_int(double z) {
  const double f = std::floor(z);
  const double d = z - f;
  if (d > 0.5) return f + 1.0;
  if (d < 0.5) return f;
  return std::fmod(f, 2.0) == 0.0 ? f : f + 1.0;
}

// precision.cpp:23-41
static double round_finite_nonzero(double x, const Fmt& fmt) {
  const int t = fmt.t;
  const int emin = fmt.emin();
  const double mag = std::fabs(x);
  if (mag >= fmt.overflow_threshold()) return std::copysign(HUGE_VAL, x);
  int shift;
  const int e = std::ilogb(mag);
  if (e < emin)
    shift = fmt.sub ? emin - t + 1 : emin;
  else
    shift = e - t + 1;
  const double r = std::ldexp(nearest_even_int(std::ldexp(x, -shift)), shift);
  return r == 0.0 ? std::copysign(0.0, x) : r;
}

// precision.cpp:82-86
static inline double round_value(double x, const Fmt& fmt) {
  if (fmt.covers_double()) return x;
  if (!std::isfinite(x) || x == 0.0) return x;
  return round_finite_nonzero(x, fmt);
}

// precision.cpp:88-95 (one tally per call, regardless of size)
static void round_inplace(double* a, size_t n, const Fmt& fmt) {
  ++g_round_calls;
  if (fmt.covers_double()) return;
  for (size_t i = 0; i < n; ++i) a[i] = round_value(a[i], fmt);
}

// ---- lpblas.cpp --------------------------------------------------------------
static int stages_of(long k) {  // while-loop trips of pairwise_block_reduce
  int s = 0;
  while (k > 1) {
    k = k / 2 + k % 2;
    ++s;
  }
  return s;
}

// Literal transcription of lpblas.cpp:13-30 + :59-70 (materialises the
// m x (K n) product matrix). Small sizes only; used to validate the streamed
// forms below bit for bit.
static void lp_matmul_literal(const double* a, long m, long K, const double* b,
                              long n, const Fmt& fmt, double* out) {
  const bool live = !fmt.covers_double();
  std::vector<double> c(size_t(m) * K * n);
  for (long i = 0; i < K; ++i)  // c.middleCols(i*n, n) = a.col(i) * b.row(i)
    for (long j = 0; j < n; ++j)
      for (long r = 0; r < m; ++r)
        c[size_t(i * n + j) * m + r] = a[size_t(i) * m + r] * b[size_t(j) * K + i];
  if (live) round_inplace(c.data(), c.size(), fmt);
  long k = K;
  const long w = n;
  while (k > 1) {
    const long pairs = k / 2, carry = k % 2;
    std::vector<double> next(size_t(m) * (pairs + carry) * w);
    for (long i = 0; i < pairs; ++i)
      for (long col = 0; col < w; ++col)
        for (long r = 0; r < m; ++r)
          next[size_t(i * w + col) * m + r] =
              c[size_t(2 * i * w + col) * m + r] +
              c[size_t((2 * i + 1) * w + col) * m + r];
    if (live) round_inplace(next.data(), size_t(m) * pairs * w, fmt);
    if (carry)
      for (long col = 0; col < w; ++col)
        for (long r = 0; r < m; ++r)
          next[size_t(pairs * w + col) * m + r] =
              c[size_t((k - 1) * w + col) * m + r];
    c.swap(next);
    k = pairs + carry;
  }
  std::memcpy(out, c.data(), sizeof(double) * size_t(m) * n);
}

// Streamed pairwise tree for one output element, generic format. The stage
// tree of pairwise_block_reduce (adjacent pairs, odd tail carried unrounded)
// equals a binary counter over the addends whose leftover levels are merged
// bottom-up at the end; each freshly formed sum is rounded exactly once, as in
// the stage-wise round_inplace(next.leftCols(pairs * w)).
struct TreeAcc {
  double lvl[64];
  uint64_t occ = 0;
  void push(double v, const Fmt& f, bool live) {
    int L = 0;
    while (occ & (uint64_t(1) << L)) {
      double s = lvl[L] + v;
      v = live ? round_value(s, f) : s;
      occ &= ~(uint64_t(1) << L);
      ++L;
    }
    lvl[L] = v;
    occ |= uint64_t(1) << L;
  }
  double finish(const Fmt& f, bool live) {
    bool have = false;
    double acc = 0.0;
    for (int L = 0; L < 64; ++L) {
      if (!(occ & (uint64_t(1) << L))) continue;
      if (!have) {
        acc = lvl[L];
        have = true;
      } else {
        double s = lvl[L] + acc;
        acc = live ? round_value(s, f) : s;
      }
    }
    return acc;
  }
};

static void lp_matmul_streamed_generic(const double* a, long m, long K,
                                       const double* b, long n, const Fmt& fmt,
                                       double* out) {
  const bool live = !fmt.covers_double();
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (long j = 0; j < n; ++j)
    for (long r = 0; r < m; ++r) {
      TreeAcc acc;
      for (long i = 0; i < K; ++i) {
        double p = a[size_t(i) * m + r] * b[size_t(j) * K + i];
        acc.push(live ? round_value(p, fmt) : p, fmt, live);
      }
      out[size_t(j) * m + r] = acc.finish(fmt, live);
    }
}

// fp16 fast path: every input is a binary16 value (or +-inf / NaN). Products
// of two binary16 values are exact in binary32, and binary32 arithmetic
// followed by one RNE conversion to binary16 equals correctly rounded
// binary16 arithmetic (24 >= 2*11+2, the double-rounding-innocuous bound), so
// the F16C pipeline below is bit-identical to round_value(double) on the same
// tree. tests/test_oracle_kat.py checks it against the generic path.
static inline __m256 r16(__m256 v) {
  return _mm256_cvtph_ps(
      _mm256_cvtps_ph(v, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC));
}

static bool all_fp16(const double* p, size_t n) {
  const Fmt h{11, 15, true};
  for (size_t i = 0; i < n; ++i) {
    const double v = p[i];
    if (std::isnan(v)) continue;
    if (round_value(v, h) != v) return false;
  }
  return true;
}

static void lp_matmul_fp16_fast(const double* a, long m, long K,
                                const double* b, long n, double* out) {
  // a is m x K column-major: repack as float, rows padded to a multiple of 8.
  const long mp = (m + 7) / 8 * 8;
  std::vector<float> af(size_t(mp) * K, 0.0f), bf(size_t(K) * n);
  for (long i = 0; i < K; ++i)
    for (long r = 0; r < m; ++r) af[size_t(i) * mp + r] = float(a[size_t(i) * m + r]);
  for (size_t q = 0; q < bf.size(); ++q) bf[q] = float(b[q]);
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (long j = 0; j < n; ++j) {
    const float* bj = bf.data() + size_t(j) * K;
    for (long r0 = 0; r0 < mp; r0 += 8) {
      __m256 lvl[64];
      uint64_t occ = 0;
      auto push = [&](__m256 v, int L) {
        while (occ & (uint64_t(1) << L)) {
          v = r16(_mm256_add_ps(lvl[L], v));
          occ &= ~(uint64_t(1) << L);
          ++L;
        }
        lvl[L] = v;
        occ |= uint64_t(1) << L;
      };
      long i = 0;
      for (; i + 8 <= K; i += 8) {  // aligned 8-leaf subtree, then level 3
        __m256 p[8];
        for (int q = 0; q < 8; ++q)
          p[q] = r16(_mm256_mul_ps(_mm256_loadu_ps(af.data() + size_t(i + q) * mp + r0),
                                   _mm256_set1_ps(bj[i + q])));
        __m256 s0 = r16(_mm256_add_ps(p[0], p[1]));
        __m256 s1 = r16(_mm256_add_ps(p[2], p[3]));
        __m256 s2 = r16(_mm256_add_ps(p[4], p[5]));
        __m256 s3 = r16(_mm256_add_ps(p[6], p[7]));
        __m256 t0 = r16(_mm256_add_ps(s0, s1));
        __m256 t1 = r16(_mm256_add_ps(s2, s3));
        push(r16(_mm256_add_ps(t0, t1)), 3);
      }
      for (; i < K; ++i)
        push(r16(_mm256_mul_ps(_mm256_loadu_ps(af.data() + size_t(i) * mp + r0),
                               _mm256_set1_ps(bj[i]))),
             0);
      bool have = false;
      __m256 acc = _mm256_setzero_ps();
      for (int L = 0; L < 64; ++L) {
        if (!(occ & (uint64_t(1) << L))) continue;
        if (!have) {
          acc = lvl[L];
          have = true;
        } else {
          acc = r16(_mm256_add_ps(lvl[L], acc));
        }
      }
      float tmp[8];
      _mm256_storeu_ps(tmp, acc);
      for (int q = 0; q < 8 && r0 + q < m; ++q)
        out[size_t(j) * m + r0 + q] = double(tmp[q]);
    }
  }
}

// Double-covering formats (fp64): the same stage tree with no rounding,
// eight consecutive output rows at a time. All eight share the counter state
// (it depends only on the leaf index), so every sum is the one TreeAcc forms;
// A is read through a row-major copy so each row streams contiguously.
static void lp_matmul_tree_f64(const double* a, long m, long K, const double* b, long n,
                               double* out) {
  std::vector<double> at(size_t(m) * K);
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (long r = 0; r < m; ++r)
    for (long i = 0; i < K; ++i) at[size_t(r) * K + i] = a[size_t(i) * m + r];
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (long j = 0; j < n; ++j) {
    const double* bj = b + size_t(j) * K;
    for (long r0 = 0; r0 < m; r0 += 8) {
      const int R = int(std::min<long>(8, m - r0));
      const double* ar[8];
      for (int q = 0; q < 8; ++q) ar[q] = at.data() + size_t(r0 + (q < R ? q : 0)) * K;
      double lvl[64][8];
      uint64_t occ = 0;
      // aligned 8-leaf blocks: their subtree is fixed ((01)(23))((45)(67)) and
      // the block value enters the counter at level 3 (bits 0-2 are clear)
      const long K8 = K & ~7L;
      for (long i0 = 0; i0 < K8; i0 += 8) {
        double v[8];
        for (int q = 0; q < 8; ++q) {
          const double* x = ar[q] + i0;
          const double* y = bj + i0;
          const double s01 = x[0] * y[0] + x[1] * y[1], s23 = x[2] * y[2] + x[3] * y[3];
          const double s45 = x[4] * y[4] + x[5] * y[5], s67 = x[6] * y[6] + x[7] * y[7];
          v[q] = (s01 + s23) + (s45 + s67);
        }
        int L = 3;
        while (occ & (uint64_t(1) << L)) {
          for (int q = 0; q < 8; ++q) v[q] = lvl[L][q] + v[q];
          occ &= ~(uint64_t(1) << L);
          ++L;
        }
        for (int q = 0; q < 8; ++q) lvl[L][q] = v[q];
        occ |= uint64_t(1) << L;
      }
      for (long i = K8; i < K; ++i) {
        double v[8];
        for (int q = 0; q < 8; ++q) v[q] = ar[q][i] * bj[i];
        int L = 0;
        while (occ & (uint64_t(1) << L)) {
          for (int q = 0; q < 8; ++q) v[q] = lvl[L][q] + v[q];
          occ &= ~(uint64_t(1) << L);
          ++L;
        }
        for (int q = 0; q < 8; ++q) lvl[L][q] = v[q];
        occ |= uint64_t(1) << L;
      }
      double acc[8];
      bool have = false;
      for (int L = 0; L < 64; ++L) {
        if (!(occ & (uint64_t(1) << L))) continue;
        for (int q = 0; q < 8; ++q) acc[q] = have ? lvl[L][q] + acc[q] : lvl[L][q];
        have = true;
      }
      for (int q = 0; q < R; ++q) out[size_t(j) * m + r0 + q] = acc[q];
    }
  }
}

// lp_matmul (lpblas.cpp:59-70). mode: 0 auto (fast fp16 / fp64 tree when
// applicable), 1 literal, 2 streamed generic.
static void lp_matmul(const double* a, long m, long K, const double* b, long n,
                      const Fmt& fmt, double* out, int mode = 0) {
  if (K == 0) throw std::invalid_argument("lp_matmul: empty input");
  if (mode == 1) {
    lp_matmul_literal(a, m, K, b, n, fmt, out);
    return;
  }
  if (!fmt.covers_double()) g_round_calls += 1 + stages_of(K);
  if (mode == 0 && fmt.is_fp16() && all_fp16(a, size_t(m) * K) &&
      all_fp16(b, size_t(K) * n))
    lp_matmul_fp16_fast(a, m, K, b, n, out);
  else if (mode == 0 && fmt.covers_double())
    lp_matmul_tree_f64(a, m, K, b, n, out);
  else
    lp_matmul_streamed_generic(a, m, K, b, n, fmt, out);
}

// ---- dense FP64 helpers ------------------------------------------------------
static void dgemm(char ta, char tb, long m, long n, long k, double alpha,
                  const double* a, long lda, const double* b, long ldb,
                  double beta, double* c, long ldc) {
  scipy_dgemm_64_(&ta, &tb, &m, &n, &k, &alpha, a, &lda, b, &ldb, &beta, c,
                  &ldc, 1, 1);
}
static double dot(const double* x, const double* y, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
static double nrm(const double* x, size_t n) { return std::sqrt(dot(x, x, n)); }
static bool all_finite(const double* x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

// ---- kron.cpp ----------------------------------------------------------------
struct KronSum {
  int n = 0, r = 0;
  const double* rowf = nullptr;  // r consecutive n*n col-major
  const double* colf = nullptr;
};

// kron_apply (kron.cpp:62-71): vec(D * X * C^T), D = col_factor, C = row_factor.
// transposed: kron_apply(C^T, D^T, y) = vec(D^T X C)  (kron.cpp:81-88).
static void kronsum_apply(const KronSum& a, const double* y, double* out,
                          bool transpose) {
  if (a.r < 1) throw std::invalid_argument("KroneckerSum: no terms");
  const long n = a.n;
  const size_t nn = size_t(n) * n;
  std::vector<double> t(nn), u(nn);
  std::fill(out, out + nn, 0.0);
  for (int k = 0; k < a.r; ++k) {
    const double* C = a.rowf + k * nn;
    const double* D = a.colf + k * nn;
    if (!transpose) {
      dgemm('N', 'N', n, n, n, 1.0, D, n, y, n, 0.0, t.data(), n);
      dgemm('N', 'T', n, n, n, 1.0, t.data(), n, C, n, 0.0, u.data(), n);
    } else {
      dgemm('T', 'N', n, n, n, 1.0, D, n, y, n, 0.0, t.data(), n);
      dgemm('N', 'N', n, n, n, 1.0, t.data(), n, C, n, 0.0, u.data(), n);
    }
    for (size_t i = 0; i < nn; ++i) out[i] += u[i];
  }
}

// normal_matvec (krylov.cpp:146-152)
static void normal_matvec(const KronSum& a, double lambda, const double* p,
                          double* out) {
  const size_t nn = size_t(a.n) * a.n;
  std::vector<double> ap(nn);
  kronsum_apply(a, p, ap.data(), false);
  kronsum_apply(a, ap.data(), out, true);
  const double l2 = lambda * lambda;
  for (size_t i = 0; i < nn; ++i) out[i] = out[i] + l2 * p[i];
}

// ---- factor.cpp --------------------------------------------------------------
struct Svd {
  std::vector<double> u, s, v;  // n x n col-major, n, n x n
};

// svd_dense (factor.cpp:14-23) on LAPACK dgesdd.
static Svd svd_dense(const double* a, long m, long n) {
  if (m * n == 0) throw std::invalid_argument("svd_dense: empty matrix");
  if (!all_finite(a, size_t(m) * n))
    throw std::invalid_argument("svd_dense: non-finite entries");
  std::vector<double> w(a, a + size_t(m) * n);
  Svd out;
  const long mn = std::min(m, n);
  out.s.resize(mn);
  out.u.resize(size_t(m) * m);
  std::vector<double> vt(size_t(n) * n);
  long lwork = -1, info = 0;
  std::vector<long> iwork(8 * mn);
  double wq = 0.0;
  const char jobz = 'A';
  scipy_dgesdd_64_(&jobz, &m, &n, w.data(), &m, out.s.data(), out.u.data(), &m,
                   vt.data(), &n, &wq, &lwork, iwork.data(), &info, 1);
  lwork = long(wq) + 1;
  std::vector<double> work(lwork);
  scipy_dgesdd_64_(&jobz, &m, &n, w.data(), &m, out.s.data(), out.u.data(), &m,
                   vt.data(), &n, work.data(), &lwork, iwork.data(), &info, 1);
  if (info != 0) throw std::runtime_error("svd_dense: backend did not converge");
  out.v.resize(size_t(n) * n);
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < n; ++j) out.v[size_t(j) * n + i] = vt[size_t(i) * n + j];
  return out;
}

// banded_toeplitz (deblur.cpp:157-165)
static void banded_toeplitz(const double* w, int len, int c, int n, double* t) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int k = i - j + c;
      t[size_t(j) * n + i] = (k >= 0 && k < len) ? w[k] : 0.0;
    }
}

// nearest_kron, Toeplitz weighting (factor.cpp:25-58)
static void nearest_kron(const double* psf, int np, int crow, int ccol, int n,
                         double* row_factor, double* col_factor) {
  if (n < np) throw std::invalid_argument("nearest_kron: image smaller than psf");
  std::vector<double> dr(np), dc(np), wtd(size_t(np) * np);
  for (int i = 0; i < np; ++i) dr[i] = std::sqrt(double(n - std::abs(i - crow)));
  for (int j = 0; j < np; ++j) dc[j] = std::sqrt(double(n - std::abs(j - ccol)));
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < np; ++i)
      wtd[size_t(j) * np + i] = dr[i] * psf[size_t(j) * np + i] * dc[j];
  const Svd s = svd_dense(wtd.data(), np, np);
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
}

struct Precond {
  int n = 0;
  Svd svd_r, svd_c;
  double lambda = 0.0;
  Fmt fmt;
  std::vector<double> s_weights, vr_lp, vc_lp, s_lp;
};

// weight_matrix (factor.cpp:62-76)
static std::vector<double> weight_matrix(const Svd& r, const Svd& c, int n,
                                         double lambda) {
  std::vector<double> s(size_t(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double prod = r.s[j] * c.s[i];
      const double denom = prod * prod + lambda * lambda;
      if (denom == 0.0)
        throw std::invalid_argument(
            "build_preconditioner: singular factors need lambda > 0");
      s[size_t(j) * n + i] = 1.0 / denom;
    }
  return s;
}

static std::vector<double> rounded(const std::vector<double>& a, const Fmt& f) {
  std::vector<double> r = a;
  round_inplace(r.data(), r.size(), f);
  return r;
}

// build_preconditioner (factor.cpp:80-104), SVDs supplied.
static Precond* precond_from_svd(int n, Svd sr, Svd sc, double lambda,
                                 const Fmt& fmt) {
  if (lambda < 0.0) throw std::invalid_argument("build_preconditioner: negative lambda");
  auto* p = new Precond;
  p->n = n;
  p->svd_r = std::move(sr);
  p->svd_c = std::move(sc);
  p->lambda = lambda;
  p->fmt = fmt;
  try {
    p->s_weights = weight_matrix(p->svd_r, p->svd_c, n, lambda);
  } catch (...) {
    delete p;
    throw;
  }
  p->vr_lp = rounded(p->svd_r.v, fmt);
  p->vc_lp = rounded(p->svd_c.v, fmt);
  p->s_lp = rounded(p->s_weights, fmt);
  return p;
}

// with_lambda (factor.cpp:106-115)
static Precond* with_lambda(const Precond& p, double lambda) {
  if (lambda < 0.0) throw std::invalid_argument("with_lambda: negative lambda");
  auto* q = new Precond(p);
  q->lambda = lambda;
  q->s_weights = weight_matrix(q->svd_r, q->svd_c, q->n, lambda);
  q->s_lp = rounded(q->s_weights, q->fmt);
  return q;
}

static std::vector<double> transposed(const std::vector<double>& a, int n) {
  std::vector<double> t(a.size());
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) t[size_t(i) * n + j] = a[size_t(j) * n + i];
  return t;
}

// precond_solve (factor.cpp:117-132)
static void precond_solve(const Precond& p, const double* r, double* z,
                          int mode = 0) {
  const int n = p.n;
  const size_t nn = size_t(n) * n;
  const bool live = !p.fmt.covers_double();
  std::vector<double> rm(r, r + nn);
  if (live) round_inplace(rm.data(), nn, p.fmt);
  const std::vector<double> vcT = transposed(p.vc_lp, n);
  const std::vector<double> vrT = transposed(p.vr_lp, n);
  std::vector<double> t1(nn), t2(nn), w(nn), t3(nn);
  lp_matmul(vcT.data(), n, n, rm.data(), n, p.fmt, t1.data(), mode);
  lp_matmul(t1.data(), n, n, p.vr_lp.data(), n, p.fmt, t2.data(), mode);
  for (size_t i = 0; i < nn; ++i) w[i] = p.s_lp[i] * t2[i];
  if (live) round_inplace(w.data(), nn, p.fmt);
  lp_matmul(p.vc_lp.data(), n, n, w.data(), n, p.fmt, t3.data(), mode);
  lp_matmul(t3.data(), n, n, vrT.data(), n, p.fmt, z, mode);
}

// approx_spectrum (factor.cpp:134-153)
static void approx_spectrum(const Precond& p, std::vector<double>& sigma,
                            std::vector<long>& perm) {
  const long n = p.n;
  std::vector<double> products(size_t(n) * n);
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < n; ++i) products[j * n + i] = p.svd_r.s[j] * p.svd_c.s[i];
  perm.resize(products.size());
  std::iota(perm.begin(), perm.end(), 0L);
  std::stable_sort(perm.begin(), perm.end(), [&](long a, long b) {
    return products[a] > products[b];
  });
  sigma.resize(products.size());
  for (size_t k = 0; k < products.size(); ++k) sigma[k] = products[perm[k]];
}

// project / project_b / project_x (factor.cpp:157-177)
static void project(const Precond& p, const std::vector<double>& left,
                    const std::vector<double>& right, const double* x,
                    double* out) {
  const long n = p.n;
  const size_t nn = size_t(n) * n;
  std::vector<double> t(nn), full(nn);
  dgemm('T', 'N', n, n, n, 1.0, left.data(), n, x, n, 0.0, t.data(), n);
  dgemm('N', 'N', n, n, n, 1.0, t.data(), n, right.data(), n, 0.0, full.data(), n);
  std::vector<double> sigma;
  std::vector<long> perm;
  approx_spectrum(p, sigma, perm);
  for (size_t k = 0; k < nn; ++k) out[k] = full[perm[k]];
}

// ---- krylov.cpp --------------------------------------------------------------
struct Recorder {  // krylov.cpp:29-56
  const kp_solver_options& opts;
  kp_history& h;
  double per_iter_work;
  size_t nn;
  double xnorm = 0.0;
  std::vector<double> diff;
  Recorder(const kp_solver_options& o, kp_history& hh, double work, size_t n)
      : opts(o), h(hh), per_iter_work(work), nn(n) {
    if (opts.x_true) xnorm = nrm(opts.x_true, nn);
    diff.resize(nn);
    h.rows = 0;
    h.n_cosines = 0;
    h.iterations_used = 0;
    h.converged = 0;
    h.msolve_count = 0;
    h.abort_reason[0] = 0;
  }
  void row(int k, const double* x, double resid) {
    if (h.rows >= h.capacity) throw std::invalid_argument("history capacity exceeded");
    if (opts.x_true) {
      for (size_t i = 0; i < nn; ++i) diff[i] = x[i] - opts.x_true[i];
      if (h.relative_error) h.relative_error[h.rows] = nrm(diff.data(), nn) / xnorm;
    }
    h.residual_norm[h.rows] = resid;
    h.work_units[h.rows] = per_iter_work * k;
    if (opts.record_iterates && h.iterates)
      std::memcpy(h.iterates + size_t(h.rows) * nn, x, nn * sizeof(double));
    h.rows++;
    h.iterations_used = k;
  }
  void cosine(const double* cur, const double* prev) {
    if (!opts.track_search_direction_orthogonality) return;
    const double denom = nrm(cur, nn) * nrm(prev, nn);
    const double v = denom > 0.0 ? std::fabs(dot(cur, prev, nn)) / denom : 0.0;
    if (h.residual_cosines && h.n_cosines < h.capacity)
      h.residual_cosines[h.n_cosines] = v;
    h.n_cosines++;
  }
  void abort(const std::string& s) {
    std::snprintf(h.abort_reason, sizeof(h.abort_reason), "%s", s.c_str());
  }
};

// check_common (krylov.cpp:12-27)
static void check_common(const KronSum& a, const kp_solver_options& o) {
  if (o.max_iterations < 1)
    throw std::invalid_argument("solver: max_iterations must be at least 1");
  if (!(o.rel_residual_tol > 0.0))
    throw std::invalid_argument("solver: tolerance must be positive");
  if (o.x_true && nrm(o.x_true, size_t(a.n) * a.n) == 0.0)
    throw std::invalid_argument("solver: x_true must be nonzero");
}

// pcg_core (krylov.cpp:58-142)
static void pcg_core(const KronSum& a, const double* b, const Precond& m,
                     const kp_solver_options& opts, bool flexible, double* xo,
                     kp_history& hist) {
  check_common(a, opts);
  if (m.n != a.n) throw std::invalid_argument("solver: preconditioner size mismatch");
  const size_t nn = size_t(a.n) * a.n;
  std::vector<double> x(nn, 0.0), r(nn), z(nn), p(nn), q(nn), r_prev;
  kronsum_apply(a, b, r.data(), true);
  const double r0 = nrm(r.data(), nn);
  Recorder rec(opts, hist, 2.25, nn);
  rec.row(0, x.data(), r0);
  auto done = [&] { std::memcpy(xo, x.data(), nn * sizeof(double)); };
  if (r0 == 0.0) {
    hist.converged = 1;
    return done();
  }
  precond_solve(m, r.data(), z.data());
  hist.msolve_count = 1;
  if (!all_finite(z.data(), nn)) {
    rec.abort("non-finite preconditioner output before iteration 1");
    return done();
  }
  p = z;
  double rho = dot(r.data(), z.data(), nn);
  if (!std::isfinite(rho) || rho <= 0.0) {
    rec.abort("preconditioner lost positivity before iteration 1");
    return done();
  }
  const bool keep_prev = flexible;
  for (int k = 1; k <= opts.max_iterations; ++k) {
    normal_matvec(a, opts.lambda, p.data(), q.data());
    const double pq = dot(p.data(), q.data(), nn);
    if (!std::isfinite(pq)) {
      rec.abort("non-finite curvature at iteration " + std::to_string(k));
      break;
    }
    if (pq <= 0.0) {
      rec.abort("curvature breakdown at iteration " + std::to_string(k));
      break;
    }
    const double alpha = rho / pq;
    if (keep_prev) r_prev = r;
    for (size_t i = 0; i < nn; ++i) x[i] += alpha * p[i];
    for (size_t i = 0; i < nn; ++i) r[i] -= alpha * q[i];
    const double rnorm = nrm(r.data(), nn);
    if (!std::isfinite(rnorm)) {
      rec.abort("non-finite residual at iteration " + std::to_string(k));
      break;
    }
    if (opts.track_search_direction_orthogonality) rec.cosine(r.data(), z.data());
    rec.row(k, x.data(), rnorm);
    if (rnorm <= opts.rel_residual_tol * r0) {
      hist.converged = 1;
      break;
    }
    if (k == opts.max_iterations) break;
    precond_solve(m, r.data(), z.data());
    ++hist.msolve_count;
    if (!all_finite(z.data(), nn)) {
      rec.abort("non-finite preconditioner output at iteration " +
                std::to_string(k) + " (overflow in the storage format)");
      break;
    }
    const double rz = dot(r.data(), z.data(), nn);
    double beta;
    if (flexible) {
      double s = 0.0;
      for (size_t i = 0; i < nn; ++i) s += z[i] * (r[i] - r_prev[i]);
      beta = s / rho;
    } else {
      beta = rz / rho;
    }
    if (!std::isfinite(beta) || !std::isfinite(rz)) {
      rec.abort("non-finite inner product at iteration " + std::to_string(k));
      break;
    }
    for (size_t i = 0; i < nn; ++i) p[i] = z[i] + beta * p[i];
    rho = rz;
    if (rho <= 0.0) {
      rec.abort("preconditioner lost positivity at iteration " + std::to_string(k));
      break;
    }
  }
  done();
}

// cgls (krylov.cpp:154-208)
static void cgls(const KronSum& a, const double* b, const kp_solver_options& opts,
                 double* xo, kp_history& hist) {
  check_common(a, opts);
  const size_t nn = size_t(a.n) * a.n;
  const double l2 = opts.lambda * opts.lambda;
  std::vector<double> x(nn, 0.0), rt(b, b + nn), s(nn), p, q(nn), snew(nn);
  kronsum_apply(a, rt.data(), s.data(), true);
  const double s0 = nrm(s.data(), nn);
  Recorder rec(opts, hist, 2.0, nn);
  rec.row(0, x.data(), s0);
  auto done = [&] { std::memcpy(xo, x.data(), nn * sizeof(double)); };
  if (s0 == 0.0) {
    hist.converged = 1;
    return done();
  }
  p = s;
  double gamma = dot(s.data(), s.data(), nn);
  std::vector<double> s_prev = s;
  for (int k = 1; k <= opts.max_iterations; ++k) {
    kronsum_apply(a, p.data(), q.data(), false);
    const double delta = dot(q.data(), q.data(), nn) + l2 * dot(p.data(), p.data(), nn);
    if (!std::isfinite(delta)) {
      rec.abort("non-finite curvature at iteration " + std::to_string(k));
      break;
    }
    if (delta == 0.0) {
      rec.abort("curvature breakdown at iteration " + std::to_string(k));
      break;
    }
    const double alpha = gamma / delta;
    for (size_t i = 0; i < nn; ++i) x[i] += alpha * p[i];
    for (size_t i = 0; i < nn; ++i) rt[i] -= alpha * q[i];
    kronsum_apply(a, rt.data(), snew.data(), true);
    for (size_t i = 0; i < nn; ++i) snew[i] = snew[i] - l2 * x[i];
    const double snorm = nrm(snew.data(), nn);
    if (!std::isfinite(snorm)) {
      rec.abort("non-finite residual at iteration " + std::to_string(k));
      break;
    }
    rec.cosine(snew.data(), s_prev.data());
    rec.row(k, x.data(), snorm);
    if (snorm <= opts.rel_residual_tol * s0) {
      hist.converged = 1;
      break;
    }
    const double gnew = dot(snew.data(), snew.data(), nn);
    const double beta = gnew / gamma;
    for (size_t i = 0; i < nn; ++i) p[i] = snew[i] + beta * p[i];
    gamma = gnew;
    if (opts.track_search_direction_orthogonality) s_prev = snew;
  }
  done();
}

// ---- regparam.cpp ------------------------------------------------------------
struct Spectral {
  std::vector<double> sigma, bhat, xhat;
  bool has_x = false;
  long n = 0;
};

static double probe(const std::function<double(double)>& f, double x,
                    const char* who) {  // regparam.cpp:36-42
  const double v = f(x);
  if (std::isnan(v)) throw std::runtime_error(std::string(who) + ": objective is NaN");
  return v;
}

static void check_spectral(const Spectral& sd, bool need_x) {  // :16-28
  if (sd.sigma.empty()) throw std::invalid_argument("spectral data: empty spectrum");
  if (sd.bhat.size() != sd.sigma.size())
    throw std::invalid_argument("spectral data: sigma and b lengths differ");
  if (need_x && !sd.has_x) throw std::invalid_argument("selector requires x coordinates");
  for (double s : sd.sigma)
    if (s < 0.0) throw std::invalid_argument("spectral data: negative singular value");
  if (!(*std::max_element(sd.sigma.begin(), sd.sigma.end()) > 0.0))
    throw std::invalid_argument("spectral data: all singular values zero");
}

static std::pair<double, double> selector_bracket(const Spectral& sd) {  // :30-34
  const double smax = *std::max_element(sd.sigma.begin(), sd.sigma.end());
  const double smin = *std::min_element(sd.sigma.begin(), sd.sigma.end());
  return {std::max(smin, 1e-10 * smax), smax};
}

// minimize_1d (regparam.cpp:149-181)
static std::pair<double, double> minimize_1d(const std::function<double(double)>& f,
                                             double lo, double hi, double tol) {
  if (!(lo < hi)) throw std::invalid_argument("minimize_1d: requires lo < hi");
  if (!(tol > 0.0)) throw std::invalid_argument("minimize_1d: tol must be positive");
  constexpr double invphi = 0.6180339887498949;
  double a = lo, b = hi;
  double c = b - invphi * (b - a);
  double d = a + invphi * (b - a);
  double fc = probe(f, c, "minimize_1d");
  double fd = probe(f, d, "minimize_1d");
  for (int it = 0; it < 300 && b - a > tol * (1.0 + std::min(std::abs(a), std::abs(b)));
       ++it) {
    if (fc < fd) {
      b = d;
      d = c;
      fd = fc;
      c = b - invphi * (b - a);
      if (c <= a || c >= d) break;
      fc = probe(f, c, "minimize_1d");
    } else {
      a = c;
      c = d;
      fc = fd;
      d = a + invphi * (b - a);
      if (d <= c || d >= b) break;
      fd = probe(f, d, "minimize_1d");
    }
  }
  return fc < fd ? std::make_pair(c, fc) : std::make_pair(d, fd);
}

// find_root (regparam.cpp:184-214)
static double find_root(const std::function<double(double)>& f, double lo,
                        double hi, double tol) {
  if (!(lo < hi)) throw std::invalid_argument("find_root: requires lo < hi");
  if (!(tol > 0.0)) throw std::invalid_argument("find_root: tol must be positive");
  double flo = probe(f, lo, "find_root");
  double fhi = probe(f, hi, "find_root");
  if (!std::isfinite(flo) || !std::isfinite(fhi))
    throw std::runtime_error("find_root: endpoint value not finite");
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  if ((flo > 0.0) == (fhi > 0.0))
    throw std::invalid_argument("find_root: no sign change over [lo, hi]");
  double a = lo, b = hi;
  while (b - a > tol * (1.0 + 0.5 * (std::abs(a) + std::abs(b)))) {
    const double m = a + 0.5 * (b - a);
    if (m <= a || m >= b) break;
    const double fm = probe(f, m, "find_root");
    if (!std::isfinite(fm)) throw std::runtime_error("find_root: function value not finite");
    if (fm == 0.0) return m;
    if ((fm > 0.0) == (flo > 0.0)) {
      a = m;
      flo = fm;
    } else {
      b = m;
    }
  }
  return a + 0.5 * (b - a);
}

struct LogSearch {
  double lambda = 0.0, value = 0.0;
  bool flat = false;
};

// minimize_log (regparam.cpp:54-88)
static LogSearch minimize_log(const std::function<double(double)>& g, double lo,
                              double hi) {
  constexpr double kInf = std::numeric_limits<double>::infinity();
  if (hi <= lo * (1.0 + 1e-12)) return {lo, probe(g, lo, "minimize_log"), true};
  const double ulo = std::log(lo), uhi = std::log(hi);
  const int grid = 1024;
  int best_k = -1;
  double best_v = kInf, vmin = kInf, vmax = -kInf;
  for (int k = 0; k < grid; ++k) {
    const double u = ulo + (uhi - ulo) * k / (grid - 1);
    const double v = probe(g, std::exp(u), "minimize_log");
    if (!std::isfinite(v)) continue;
    vmin = std::min(vmin, v);
    vmax = std::max(vmax, v);
    if (v < best_v) {
      best_v = v;
      best_k = k;
    }
  }
  if (best_k < 0) throw std::runtime_error("minimize_log: objective infinite everywhere");
  const double scale = std::max({std::abs(vmin), std::abs(vmax), 1e-300});
  if (vmax - vmin <= 1e-14 * scale) {
    const double mid = std::exp(0.5 * (ulo + uhi));
    return {mid, probe(g, mid, "minimize_log"), true};
  }
  const double step = (uhi - ulo) / (grid - 1);
  const double a = std::max(ulo, ulo + (best_k - 1) * step);
  const double b = std::min(uhi, ulo + (best_k + 1) * step);
  const auto r = minimize_1d([&](double u) { return g(std::exp(u)); }, a, b, 1e-12);
  return {std::exp(r.first), r.second, false};
}

// objectives (regparam.cpp:216-246)
static double opt_objective(const Spectral& sd, double lambda) {
  if (!sd.has_x) throw std::invalid_argument("opt_objective: x coordinates missing");
  double acc = 0.0;
  for (size_t i = 0; i < sd.sigma.size(); ++i) {
    const double s = sd.sigma[i];
    const double d = s * s + lambda * lambda;
    const double t = s * sd.bhat[i] / d - sd.xhat[i];
    acc += t * t;
  }
  return acc;
}
static double gcv_objective(const Spectral& sd, double lambda) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < sd.sigma.size(); ++i) {
    const double d = sd.sigma[i] * sd.sigma[i] + lambda * lambda;
    const double t = sd.bhat[i] / d;
    num += t * t;
    den += 1.0 / d;
  }
  return double(sd.n) * num / (den * den);
}
static double wgcv_trace(const Spectral& sd, double omega, double lambda) {
  double acc = 0.0;
  for (double s : sd.sigma) {
    const double s2 = s * s;
    acc += ((1.0 - omega) * s2 + lambda * lambda) / (s2 + lambda * lambda);
  }
  return acc;
}
static double wgcv_objective(const Spectral& sd, double omega, double lambda) {
  const double l2 = lambda * lambda;
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < sd.sigma.size(); ++i) {
    const double s2 = sd.sigma[i] * sd.sigma[i];
    const double d = s2 + l2;
    const double t = l2 * sd.bhat[i] / d;
    num += t * t;
    den += ((1.0 - omega) * s2 + l2) / d;
  }
  num *= double(sd.n);
  if (den == 0.0) return std::numeric_limits<double>::infinity();
  return num / (den * den);
}
static double discrepancy_gap(const Spectral& sd, double epsilon, double lambda) {
  const double l2 = lambda * lambda;
  double acc = 0.0;
  for (size_t i = 0; i < sd.sigma.size(); ++i) {
    const double d = sd.sigma[i] * sd.sigma[i] + l2;
    const double t = l2 * sd.bhat[i] / d;
    acc += t * t;
  }
  return acc - epsilon * epsilon;
}

static kp_param_choice run_selector_on(double lo, double hi, int method,
                                       const std::function<double(double)>& g) {
  const LogSearch r = minimize_log(g, lo, hi);
  kp_param_choice c{};
  c.lambda = r.lambda;
  c.method = method;
  c.objective_value = r.value;
  c.bracket_lo = lo;
  c.bracket_hi = hi;
  c.flat_objective = r.flat;
  c.grid_index = -1;
  return c;
}

// discrepancy (regparam.cpp:288-327)
static kp_param_choice discrepancy(const Spectral& sd, double noise_norm, double eta) {
  check_spectral(sd, false);
  if (!(noise_norm > 0.0)) throw std::invalid_argument("discrepancy: noise_norm must be positive");
  if (!(eta > 0.0)) throw std::invalid_argument("discrepancy: eta must be positive");
  const double eps = eta * noise_norm;
  const double smax = *std::max_element(sd.sigma.begin(), sd.sigma.end());
  const double lo = 1e-10 * smax, hi = smax;
  const double glo = discrepancy_gap(sd, eps, lo);
  const double ghi = discrepancy_gap(sd, eps, hi);
  if (ghi < 0.0)
    throw NoRootError(
        "no root; eta * noise_norm too large: the residual cannot reach it "
        "inside the bracket");
  if (glo > 0.0)
    throw NoRootError(
        "no root; eta * noise_norm too small: the residual exceeds it "
        "everywhere in the bracket");
  double lambda;
  if (glo == 0.0)
    lambda = lo;
  else if (ghi == 0.0)
    lambda = hi;
  else
    lambda = std::exp(find_root(
        [&](double u) { return discrepancy_gap(sd, eps, std::exp(u)); },
        std::log(lo), std::log(hi), 1e-12));
  kp_param_choice c{};
  c.lambda = lambda;
  c.method = 3;
  c.eta = eta;
  c.noise_norm = noise_norm;
  c.objective_value = discrepancy_gap(sd, eps, lambda);
  c.bracket_lo = lo;
  c.bracket_hi = hi;
  c.grid_index = -1;
  return c;
}

}  // namespace kpo

// =============================================================================
// extern "C" surface for tests (ctypes)
// =============================================================================
using namespace kpo;

#define KPO_TRY(...)                                 \
  try {                                              \
    __VA_ARGS__;                                            \
    return KP_OK;                                    \
  } catch (const NoRootError& e) {                   \
    g_err = e.what();                                \
    return KP_ERR_NO_ROOT;                           \
  } catch (const std::invalid_argument& e) {         \
    g_err = e.what();                                \
    return KP_ERR_INVALID_ARGUMENT;                  \
  } catch (const std::exception& e) {                \
    g_err = e.what();                                \
    return KP_ERR_RUNTIME;                           \
  }

static Spectral make_spectral(const double* sigma, const double* bhat,
                              const double* xhat, long n) {
  Spectral s;
  s.sigma.assign(sigma, sigma + n);
  s.bhat.assign(bhat, bhat + n);
  if (xhat) {
    s.xhat.assign(xhat, xhat + n);
    s.has_x = true;
  }
  s.n = n;
  return s;
}

extern "C" {

const char* kpo_last_error(void) { return g_err.c_str(); }
void kpo_set_threads(int t) {
  g_threads = t < 1 ? 1 : t;
  scipy_openblas_set_num_threads64_(g_threads);
}
int kpo_get_threads(void) { return g_threads; }
unsigned long long kpo_round_calls(void) { return g_round_calls; }

double kpo_round_value(double x, kp_format f) { return round_value(x, fmt_of(f)); }
void kpo_round_array(double* a, long n, kp_format f) {
  round_inplace(a, size_t(n), fmt_of(f));
}

// pairwise_sum (lpblas.cpp:34-37)
int kpo_pairwise_sum(const double* z, long n, kp_format f, double* out) {
  KPO_TRY({
    if (n == 0) throw std::invalid_argument("pairwise_sum: empty input");
    const Fmt fmt = fmt_of(f);
    const bool live = !fmt.covers_double();
    if (live) g_round_calls += stages_of(n);
    TreeAcc acc;
    for (long i = 0; i < n; ++i) acc.push(z[i], fmt, live);
    *out = acc.finish(fmt, live);
  })
}
// lp_dot (lpblas.cpp:39-47)
int kpo_lp_dot(const double* x, const double* y, long n, kp_format f, double* out) {
  KPO_TRY({
    if (n == 0) throw std::invalid_argument("lp_dot: empty input");
    const Fmt fmt = fmt_of(f);
    const bool live = !fmt.covers_double();
    if (live) g_round_calls += 1 + stages_of(n);
    TreeAcc acc;
    for (long i = 0; i < n; ++i) {
      const double p = x[i] * y[i];
      acc.push(live ? round_value(p, fmt) : p, fmt, live);
    }
    *out = acc.finish(fmt, live);
  })
}
// lp_matvec (lpblas.cpp:49-57) == lp_matmul with one column
int kpo_lp_matvec(const double* a, long m, long k, const double* v, kp_format f,
                  double* out) {
  KPO_TRY({
    if (k == 0) throw std::invalid_argument("lp_matvec: empty input");
    lp_matmul(a, m, k, v, 1, fmt_of(f), out, 2);
  })
}
int kpo_lp_matmul(const double* a, long m, long k, const double* b, long n,
                  kp_format f, double* out, int mode) {
  KPO_TRY(lp_matmul(a, m, k, b, n, fmt_of(f), out, mode))
}

int kpo_kronsum_apply(int n, int r, const double* rowf, const double* colf,
                      const double* y, double* out, int transpose) {
  KPO_TRY({
    KronSum a{n, r, rowf, colf};
    kronsum_apply(a, y, out, transpose != 0);
  })
}
int kpo_normal_matvec(int n, int r, const double* rowf, const double* colf,
                      double lambda, const double* p, double* out) {
  KPO_TRY({
    KronSum a{n, r, rowf, colf};
    normal_matvec(a, lambda, p, out);
  })
}

int kpo_svd(const double* a, int m, int n, double* u, double* s, double* v) {
  KPO_TRY({
    Svd r = svd_dense(a, m, n);
    std::memcpy(u, r.u.data(), r.u.size() * sizeof(double));
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    std::memcpy(v, r.v.data(), r.v.size() * sizeof(double));
  })
}
int kpo_nearest_kron(const double* psf, int np, int crow, int ccol, int n,
                     double* row_factor, double* col_factor) {
  KPO_TRY(nearest_kron(psf, np, crow, ccol, n, row_factor, col_factor))
}

int kpo_precond_build(const double* a_r, const double* a_c, int n, double lambda,
                      kp_format f, void** out) {
  KPO_TRY({
    if (lambda < 0.0) throw std::invalid_argument("build_preconditioner: negative lambda");
    Svd r = svd_dense(a_r, n, n);
    Svd c = svd_dense(a_c, n, n);
    *out = precond_from_svd(n, std::move(r), std::move(c), lambda, fmt_of(f));
  })
}
int kpo_precond_from_svd(int n, const double* u_r, const double* s_r,
                         const double* v_r, const double* u_c, const double* s_c,
                         const double* v_c, double lambda, kp_format f, void** out) {
  KPO_TRY({
    const size_t nn = size_t(n) * n;
    Svd r, c;
    r.u.assign(u_r, u_r + nn);
    r.s.assign(s_r, s_r + n);
    r.v.assign(v_r, v_r + nn);
    c.u.assign(u_c, u_c + nn);
    c.s.assign(s_c, s_c + n);
    c.v.assign(v_c, v_c + nn);
    *out = precond_from_svd(n, std::move(r), std::move(c), lambda, fmt_of(f));
  })
}
int kpo_precond_with_lambda(const void* p, double lambda, void** out) {
  KPO_TRY(*out = with_lambda(*static_cast<const Precond*>(p), lambda))
}
void kpo_precond_destroy(void* p) { delete static_cast<Precond*>(p); }
int kpo_precond_export(const void* pv, int field, double* out) {
  KPO_TRY({
    const Precond& p = *static_cast<const Precond*>(pv);
    const std::vector<double>* v = nullptr;
    switch (field) {
      case 0: v = &p.s_weights; break;
      case 1: v = &p.s_lp; break;
      case 2: v = &p.vr_lp; break;
      case 3: v = &p.vc_lp; break;
      case 4: v = &p.svd_r.s; break;
      case 5: v = &p.svd_c.s; break;
      case 6: v = &p.svd_r.u; break;
      case 7: v = &p.svd_r.v; break;
      case 8: v = &p.svd_c.u; break;
      case 9: v = &p.svd_c.v; break;
      default: throw std::invalid_argument("precond_export: bad field");
    }
    std::memcpy(out, v->data(), v->size() * sizeof(double));
  })
}
int kpo_precond_solve(const void* p, const double* r, double* z, int mode) {
  KPO_TRY(precond_solve(*static_cast<const Precond*>(p), r, z, mode))
}
int kpo_spectral(const void* pv, const double* b, const double* x_true,
                 double* sigma, double* bhat, double* xhat) {
  KPO_TRY({
    const Precond& p = *static_cast<const Precond*>(pv);
    std::vector<double> s;
    std::vector<long> perm;
    approx_spectrum(p, s, perm);
    std::memcpy(sigma, s.data(), s.size() * sizeof(double));
    project(p, p.svd_c.u, p.svd_r.u, b, bhat);
    if (x_true && xhat) project(p, p.svd_c.v, p.svd_r.v, x_true, xhat);
  })
}

int kpo_cgls(int n, int r, const double* rowf, const double* colf,
             const double* b, const kp_solver_options* o, double* x,
             kp_history* h) {
  KPO_TRY({
    KronSum a{n, r, rowf, colf};
    cgls(a, b, *o, x, *h);
  })
}
int kpo_pcg(int n, int r, const double* rowf, const double* colf,
            const double* b, const void* m, const kp_solver_options* o,
            int flexible, double* x, kp_history* h) {
  KPO_TRY({
    KronSum a{n, r, rowf, colf};
    pcg_core(a, b, *static_cast<const Precond*>(m), *o, flexible != 0, x, *h);
  })
}

int kpo_gcv_objective(const double* s, const double* b, long n, double lambda,
                      double* out) {
  KPO_TRY(*out = gcv_objective(make_spectral(s, b, nullptr, n), lambda))
}
int kpo_opt_objective(const double* s, const double* b, const double* x, long n,
                      double lambda, double* out) {
  KPO_TRY(*out = opt_objective(make_spectral(s, b, x, n), lambda))
}
int kpo_wgcv_objective(const double* s, const double* b, long n, double omega,
                       double lambda, double* out) {
  KPO_TRY(*out = wgcv_objective(make_spectral(s, b, nullptr, n), omega, lambda))
}
int kpo_discrepancy_gap(const double* s, const double* b, long n, double eps,
                        double lambda, double* out) {
  KPO_TRY(*out = discrepancy_gap(make_spectral(s, b, nullptr, n), eps, lambda))
}
int kpo_minimize_1d(double (*f)(double), double lo, double hi, double tol,
                    double* x, double* fx) {
  KPO_TRY({
    auto r = minimize_1d([&](double v) { return f(v); }, lo, hi, tol);
    *x = r.first;
    *fx = r.second;
  })
}
int kpo_find_root(double (*f)(double), double lo, double hi, double tol,
                  double* x) {
  KPO_TRY(*x = find_root([&](double v) { return f(v); }, lo, hi, tol))
}
// lambda_opt / gcv / wgcv (regparam.cpp:248-286)
int kpo_select(int method, const double* s, const double* b, const double* x,
               long n, double omega, kp_param_choice* out) {
  KPO_TRY({
    Spectral sd = make_spectral(s, b, x, n);
    if (method == 0) {
      check_spectral(sd, true);
      const auto [lo, hi] = selector_bracket(sd);
      *out = run_selector_on(lo, hi, 0, [&](double l) { return opt_objective(sd, l); });
    } else if (method == 1) {
      check_spectral(sd, false);
      const auto [lo, hi] = selector_bracket(sd);
      *out = run_selector_on(lo, hi, 1, [&](double l) { return gcv_objective(sd, l); });
    } else if (method == 2) {
      check_spectral(sd, false);
      if (!(omega > 0.0)) throw std::invalid_argument("wgcv: omega must be positive");
      auto [lo, hi] = selector_bracket(sd);
      if (omega > 1.0 && wgcv_trace(sd, omega, lo) < 0.0 &&
          wgcv_trace(sd, omega, hi) > 0.0) {
        double a = std::log(lo), bb = std::log(hi);
        while (bb - a > 1e-13 * (1.0 + std::abs(bb))) {
          const double m = 0.5 * (a + bb);
          (wgcv_trace(sd, omega, std::exp(m)) > 0.0 ? bb : a) = m;
        }
        lo = std::exp(bb);
      }
      *out = run_selector_on(lo, hi, 2,
                             [&](double l) { return wgcv_objective(sd, omega, l); });
      out->omega = omega;
    } else {
      throw std::invalid_argument("select: bad method");
    }
  })
}
int kpo_discrepancy(const double* s, const double* b, long n, double noise_norm,
                    double eta, kp_param_choice* out) {
  KPO_TRY(*out = discrepancy(make_spectral(s, b, nullptr, n), noise_norm, eta))
}
// North-star GCV on an explicit grid: first argmin of gcv_objective.
int kpo_gcv_grid(const double* s, const double* b, long n, const double* lambdas,
                 int m, double* values, kp_param_choice* out) {
  KPO_TRY({
    Spectral sd = make_spectral(s, b, nullptr, n);
    check_spectral(sd, false);
    int best = -1;
    double bv = std::numeric_limits<double>::infinity();
    for (int k = 0; k < m; ++k) {
      const double v = probe([&](double l) { return gcv_objective(sd, l); },
                             lambdas[k], "gcv_grid");
      if (values) values[k] = v;
      if (v < bv) {
        bv = v;
        best = k;
      }
    }
    if (best < 0) throw std::runtime_error("gcv_grid: objective infinite everywhere");
    *out = kp_param_choice{};
    out->lambda = lambdas[best];
    out->method = 4;
    out->objective_value = bv;
    out->bracket_lo = lambdas[0];
    out->bracket_hi = lambdas[m - 1];
    out->grid_index = best;
  })
}
// filtered_solution (regparam.cpp:329-349)
int kpo_filtered_solution(const void* pv, const double* b, double lambda,
                          double* x) {
  KPO_TRY({
    const Precond& p = *static_cast<const Precond*>(pv);
    if (lambda < 0.0) throw std::invalid_argument("filtered_solution: negative lambda");
    const long n = p.n;
    const size_t nn = size_t(n) * n;
    std::vector<double> t(nn), bh(nn), coef(nn);
    dgemm('T', 'N', n, n, n, 1.0, p.svd_c.u.data(), n, b, n, 0.0, t.data(), n);
    dgemm('N', 'N', n, n, n, 1.0, t.data(), n, p.svd_r.u.data(), n, 0.0, bh.data(), n);
    const double l2 = lambda * lambda;
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < n; ++i) {
        const double s = p.svd_r.s[j] * p.svd_c.s[i];
        const double den = s * s + l2;
        if (den == 0.0)
          throw std::invalid_argument("filtered_solution: zero singular value with lambda = 0");
        coef[j * n + i] = s / den * bh[j * n + i];
      }
    dgemm('N', 'N', n, n, n, 1.0, p.svd_c.v.data(), n, coef.data(), n, 0.0, t.data(), n);
    dgemm('N', 'T', n, n, n, 1.0, t.data(), n, p.svd_r.v.data(), n, 0.0, x, n);
  })
}

}  // extern "C"
