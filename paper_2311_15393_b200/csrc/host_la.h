// Host dense linear algebra for setup paths (SVDs of the Kronecker factors,
// b_true generation): numpy's bundled OpenBLAS (ILP64, `scipy_` prefix),
// linked directly. Never used on the solve path.
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

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

namespace kpla {

struct Svd {
  std::vector<double> u, s, v;  // m x m, min(m,n), n x n (column-major)
};

inline void set_threads(int t) { scipy_openblas_set_num_threads64_(t < 1 ? 1 : t); }

inline void dgemm(char ta, char tb, long m, long n, long k, double alpha,
                  const double* a, long lda, const double* b, long ldb,
                  double beta, double* c, long ldc) {
  scipy_dgemm_64_(&ta, &tb, &m, &n, &k, &alpha, a, &lda, b, &ldb, &beta, c,
                  &ldc, 1, 1);
}

// Full SVD with nonincreasing singular values (svd_dense contract,
// factor.cpp:14-23): invalid_argument on empty / non-finite input,
// runtime_error when LAPACK does not converge.
inline Svd svd(const double* a, long m, long n) {
  if (m * n == 0) throw std::invalid_argument("svd_dense: empty matrix");
  for (long q = 0; q < m * n; ++q)
    if (!std::isfinite(a[q]))
      throw std::invalid_argument("svd_dense: non-finite entries");
  std::vector<double> w(a, a + m * n);
  Svd out;
  const long mn = m < n ? m : n;
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

}  // namespace kpla
