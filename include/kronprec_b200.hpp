// kronprec_b200.hpp — header-only C++ mirror of the reference `kronprec`
// solver API (/root/reference/proj/include/kronprec/*.hpp) over the C ABI in
// kronprec_b200.h. Same names, argument meaning and exception types; dense
// matrices are column-major std::vector<double> (Eigen's storage order), so
// an Eigen caller passes .data() pointers.
#pragma once

#include <algorithm>
#include <memory>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronprec_b200.h"

namespace kronprec_b200 {

using Vec = std::vector<double>;

// kronprec::NoRootError (regparam.hpp:51-53)
struct NoRootError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == KP_OK) return;
  const std::string msg = kp_last_error();
  switch (status) {
    case KP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case KP_ERR_NO_ROOT: throw NoRootError(msg);
    case KP_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// PrecisionFormat presets (precision.cpp:45-48)
inline kp_format fp16() { return {11, 15, 1}; }
inline kp_format bfloat16() { return {8, 127, 1}; }
inline kp_format fp32() { return {24, 127, 1}; }
inline kp_format fp64() { return {53, 1023, 1}; }

// round_array (precision.cpp:82-95)
inline Vec round_array(const Vec& a, kp_format fmt) {
  Vec out(a.size());
  check(kp_round_array(a.data(), long(a.size()), fmt, out.data()));
  return out;
}
// round_value (precision.cpp:82-86)
inline double round_value(double x, kp_format fmt) {
  double out = 0.0;
  check(kp_round_value(x, fmt, &out));
  return out;
}
// RoundCallSession / round_call_count (precision.hpp:55-66)
class RoundCallSession {
 public:
  RoundCallSession() : start_(now()) {}
  std::uint64_t count() const { return now() - start_; }

 private:
  static std::uint64_t now() {
    unsigned long long n = 0;
    check(kp_round_call_count(&n));
    return n;
  }
  std::uint64_t start_;
};
inline std::uint64_t round_call_count(const RoundCallSession& s) { return s.count(); }
// lp_matmul (lpblas.cpp:59-70): a m x k, b k x n, column-major
inline Vec lp_matmul(const Vec& a, const Vec& b, int m, int k, int n, kp_format fmt) {
  if (a.size() != size_t(m) * k || b.size() != size_t(k) * n)
    throw std::invalid_argument("lp_matmul: shape mismatch");
  Vec c(size_t(m) * n);
  check(kp_lp_matmul(m, k, n, a.data(), b.data(), fmt, c.data()));
  return c;
}
// lp_matvec (lpblas.cpp:48-57): a m x k column-major
inline Vec lp_matvec(const Vec& a, const Vec& v, int m, int k, kp_format fmt) {
  if (a.size() != size_t(m) * k || v.size() != size_t(k)) throw std::invalid_argument("lp_matvec: shape mismatch");
  return lp_matmul(a, v, m, k, 1, fmt);
}
// lp_dot (lpblas.cpp:39-46)
inline double lp_dot(const Vec& x, const Vec& y, kp_format fmt) {
  if (x.size() != y.size()) throw std::invalid_argument("lp_dot: length mismatch");
  if (x.empty()) throw std::invalid_argument("lp_dot: empty input");
  return lp_matmul(x, y, 1, int(x.size()), 1, fmt)[0];
}
// pairwise_sum (lpblas.cpp:34-37): the addends are taken as already rounded
inline double pairwise_sum(const Vec& z, kp_format fmt) {
  if (z.empty()) throw std::invalid_argument("pairwise_sum: empty input");
  const Vec ones(z.size(), 1.0);
  double out = 0.0;
  check(kp_lp_matmul_ex(1, int(z.size()), 1, z.data(), ones.data(), fmt, 0, &out));
  return out;
}

// KronTerm / KroneckerSum (kron.hpp:12-22): factors are n*n column-major.
struct KronTerm {
  Vec row_factor, col_factor;
};

// SvdTriple (factor.hpp:14-18): column-major n x n u, v; s nonincreasing.
struct SvdTriple {
  Vec u, s, v;
};

// Psf (deblur.hpp:47-54): n_p x n_p column-major values and the center.
struct Psf {
  Vec values;
  int np = 0;
  int center_row = 0, center_col = 0;
};

class KroneckerSum {
 public:
  KroneckerSum(std::vector<KronTerm> terms, int n) : terms_(std::move(terms)), n_(n) {
    if (terms_.empty()) throw std::invalid_argument("KroneckerSum: no terms");
    const size_t nn = size_t(n) * n;
    Vec rows, cols;
    for (const auto& t : terms_) {
      if (t.row_factor.size() != nn || t.col_factor.size() != nn)
        throw std::invalid_argument("KroneckerSum: factor shape mismatch");
      rows.insert(rows.end(), t.row_factor.begin(), t.row_factor.end());
      cols.insert(cols.end(), t.col_factor.begin(), t.col_factor.end());
    }
    kp_operator* op = nullptr;
    check(kp_operator_create(n, int(terms_.size()), rows.data(), cols.data(), &op));
    op_.reset(op, [](kp_operator* p) { kp_operator_destroy(p); });
  }
  int n() const { return n_; }
  const kp_operator* handle() const { return op_.get(); }

 private:
  std::vector<KronTerm> terms_;
  int n_;
  std::shared_ptr<kp_operator> op_;
};

// psf_to_kronsum (deblur.hpp:69-70); max_rank > 0 caps the number of terms.
inline KroneckerSum psf_to_kronsum(const Psf& psf, int n, double truncation_tol = 1e-12,
                                   int max_rank = 0) {
  if (psf.np < 1 || psf.values.size() != size_t(psf.np) * psf.np)
    throw std::invalid_argument("psf_to_kronsum: psf values must be np x np");
  const int cap = max_rank > 0 ? std::min(max_rank, psf.np) : psf.np;
  const size_t nn = size_t(n) * n;
  Vec rows(size_t(cap) * nn), cols(size_t(cap) * nn);
  int r = 0;
  check(kp_psf_to_kronsum(psf.values.data(), psf.np, psf.center_row, psf.center_col, n, truncation_tol,
                          max_rank, cap, rows.data(), cols.data(), &r));
  std::vector<KronTerm> terms(r);
  for (int k = 0; k < r; ++k) {
    terms[k].row_factor.assign(rows.begin() + k * nn, rows.begin() + (k + 1) * nn);
    terms[k].col_factor.assign(cols.begin() + k * nn, cols.begin() + (k + 1) * nn);
  }
  return KroneckerSum(std::move(terms), n);
}
// nearest_kron (factor.hpp:34-35)
inline KronTerm nearest_kron(const Psf& psf, int n, int weighting = KP_KRON_TOEPLITZ) {
  if (psf.np < 1 || psf.values.size() != size_t(psf.np) * psf.np)
    throw std::invalid_argument("nearest_kron: psf values must be np x np");
  KronTerm t;
  t.row_factor.resize(size_t(n) * n);
  t.col_factor.resize(size_t(n) * n);
  check(kp_nearest_kron(psf.values.data(), psf.np, psf.center_row, psf.center_col, n, weighting,
                        t.row_factor.data(), t.col_factor.data()));
  return t;
}

inline Vec kronsum_apply(const KroneckerSum& k, const Vec& y) {  // kron.cpp:73-79
  Vec out(y.size());
  if (y.size() != size_t(k.n()) * k.n()) throw std::invalid_argument("kron_apply: vector length is not n^2");
  check(kp_kronsum_apply(k.handle(), y.data(), out.data()));
  return out;
}
inline Vec kronsum_apply_transpose(const KroneckerSum& k, const Vec& y) {  // kron.cpp:81-88
  Vec out(y.size());
  if (y.size() != size_t(k.n()) * k.n()) throw std::invalid_argument("kron_apply: vector length is not n^2");
  check(kp_kronsum_apply_transpose(k.handle(), y.data(), out.data()));
  return out;
}
// kron_apply (kron.cpp:62-71): (C (x) D) y = vec(D unvec(y) C^T)
inline Vec kron_apply(const Vec& c, const Vec& d, int n, const Vec& y) {
  if (n < 1 || c.size() != size_t(n) * n || d.size() != size_t(n) * n)
    throw std::invalid_argument("kron_apply: factors must be square and equally sized");
  if (y.size() != size_t(n) * n) throw std::invalid_argument("kron_apply: vector length is not n^2");
  return kronsum_apply(KroneckerSum({KronTerm{c, d}}, n), y);
}
// svd_dense (factor.cpp:14-23): backend KP_SVD_HOST (LAPACK) or KP_SVD_DEVICE (cuSOLVER)
inline SvdTriple svd_dense(const Vec& a, int n, int backend = 0) {
  if (n < 1 || a.size() != size_t(n) * n) throw std::invalid_argument("svd_dense: square, non-empty matrix expected");
  SvdTriple t{Vec(size_t(n) * n), Vec(size_t(n)), Vec(size_t(n) * n)};
  check(kp_svd(a.data(), n, backend, t.u.data(), t.s.data(), t.v.data()));
  return t;
}
inline Vec normal_matvec(const KroneckerSum& a, double lambda, const Vec& p) {  // krylov.cpp:146-152
  if (p.size() != size_t(a.n()) * a.n()) throw std::invalid_argument("normal_matvec: length mismatch");
  Vec out(p.size());
  check(kp_normal_matvec(a.handle(), lambda, p.data(), out.data()));
  return out;
}

// KronSvdPreconditioner (factor.hpp:42-54)
class KronSvdPreconditioner {
 public:
  explicit KronSvdPreconditioner(kp_precond* p) : p_(p, [](kp_precond* q) { kp_precond_destroy(q); }) {}
  const kp_precond* handle() const { return p_.get(); }
  int n() const {
    int n;
    double l;
    kp_format f;
    int a;
    check(kp_precond_info(p_.get(), &n, &l, &f, &a));
    return n;
  }

 private:
  std::shared_ptr<kp_precond> p_;
};

inline KronSvdPreconditioner build_preconditioner(const Vec& a_r, const Vec& a_c, int n,
                                                  double lambda, kp_format fmt,
                                                  int accum = KP_ACCUM_REFERENCE) {
  if (n < 1 || a_r.size() != size_t(n) * n || a_c.size() != size_t(n) * n)  // factor.cpp:84-87
    throw std::invalid_argument("build_preconditioner: factors must be square and equally sized");
  kp_precond* p = nullptr;  // factor.cpp:80-104
  check(kp_precond_build(a_r.data(), a_c.data(), n, lambda, fmt, accum, &p));
  return KronSvdPreconditioner(p);
}
// The same preconditioner from SVDs the caller already holds (the
// reference's KronSvdPreconditioner::svd_r / svd_c): no SVD is recomputed.
inline KronSvdPreconditioner build_preconditioner_from_svd(const SvdTriple& r, const SvdTriple& c, int n,
                                                           double lambda, kp_format fmt,
                                                           int accum = KP_ACCUM_REFERENCE) {
  const size_t nn = size_t(n) * n;
  if (n < 1 || r.u.size() != nn || r.v.size() != nn || c.u.size() != nn || c.v.size() != nn ||
      r.s.size() != size_t(n) || c.s.size() != size_t(n))
    throw std::invalid_argument("build_preconditioner: factors must be square and equally sized");
  kp_precond* p = nullptr;
  check(kp_precond_build_from_svd(n, r.u.data(), r.s.data(), r.v.data(), c.u.data(), c.s.data(),
                                  c.v.data(), lambda, fmt, accum, &p));
  return KronSvdPreconditioner(p);
}
inline KronSvdPreconditioner with_lambda(const KronSvdPreconditioner& p, double lambda) {
  kp_precond* q = nullptr;  // factor.cpp:106-115
  check(kp_precond_with_lambda(p.handle(), lambda, &q));
  return KronSvdPreconditioner(q);
}
inline Vec precond_solve(const KronSvdPreconditioner& p, const Vec& r) {  // factor.cpp:117-132
  const int n = p.n();
  if (r.size() != size_t(n) * n) throw std::invalid_argument("precond_solve: vector length is not n^2");
  Vec z(r.size());
  check(kp_precond_solve(p.handle(), r.data(), z.data()));
  return z;
}

// SolverOptions / ConvergenceHistory / SolveResult (krylov.hpp:14-47)
struct SolverOptions {
  double lambda = 0.0;
  int max_iterations = 100;
  double rel_residual_tol = 1e-8;
  const Vec* x_true = nullptr;
  bool track_search_direction_orthogonality = false;
};
struct ConvergenceHistory {
  std::vector<double> relative_error, residual_norm, work_units, residual_cosines;
  int iterations_used = 0;
  bool converged = false;
  std::string abort_reason;
  int msolve_count = 0;
};
struct SolveResult {
  Vec x;
  ConvergenceHistory history;
};

namespace detail {
template <typename F>
SolveResult solve(const KroneckerSum& a, const Vec& b, const SolverOptions& o, F&& call) {
  const size_t nn = size_t(a.n()) * a.n();  // check_common, krylov.cpp:12-27
  if (b.size() != nn) throw std::invalid_argument("solver: right-hand side length mismatch");
  if (o.max_iterations < 1) throw std::invalid_argument("solver: max_iterations must be at least 1");
  if (!(o.rel_residual_tol > 0.0)) throw std::invalid_argument("solver: tolerance must be positive");
  if (o.x_true) {
    if (o.x_true->size() != nn) throw std::invalid_argument("solver: x_true length mismatch");
    bool nonzero = false;
    for (double v : *o.x_true) nonzero = nonzero || v != 0.0;
    if (!nonzero) throw std::invalid_argument("solver: x_true must be nonzero");
  }
  const int cap = o.max_iterations + 1;
  SolveResult r;
  r.x.resize(nn);
  ConvergenceHistory& h = r.history;
  h.relative_error.resize(cap);
  h.residual_norm.resize(cap);
  h.work_units.resize(cap);
  h.residual_cosines.resize(cap);
  kp_history kh{};
  kh.capacity = cap;
  kh.relative_error = h.relative_error.data();
  kh.residual_norm = h.residual_norm.data();
  kh.work_units = h.work_units.data();
  kh.residual_cosines = h.residual_cosines.data();
  kp_solver_options ko{};
  ko.lambda = o.lambda;
  ko.max_iterations = o.max_iterations;
  ko.rel_residual_tol = o.rel_residual_tol;
  ko.x_true = o.x_true ? o.x_true->data() : nullptr;
  ko.track_search_direction_orthogonality = o.track_search_direction_orthogonality;
  check(call(ko, kh, r.x.data()));
  h.relative_error.resize(o.x_true ? kh.rows : 0);
  h.residual_norm.resize(kh.rows);
  h.work_units.resize(kh.rows);
  h.residual_cosines.resize(kh.n_cosines);
  h.iterations_used = kh.iterations_used;
  h.converged = kh.converged != 0;
  h.abort_reason = kh.abort_reason;
  h.msolve_count = kh.msolve_count;
  return r;
}
}  // namespace detail

inline SolveResult cgls(const KroneckerSum& a, const Vec& b, const SolverOptions& o) {
  return detail::solve(a, b, o, [&](kp_solver_options& ko, kp_history& kh, double* x) {
    return kp_cgls(a.handle(), b.data(), &ko, x, &kh);
  });
}
inline SolveResult pcg(const KroneckerSum& a, const Vec& b, const KronSvdPreconditioner& m,
                       const SolverOptions& o) {
  return detail::solve(a, b, o, [&](kp_solver_options& ko, kp_history& kh, double* x) {
    return kp_pcg(a.handle(), b.data(), m.handle(), &ko, x, &kh);
  });
}
inline SolveResult fpcg(const KroneckerSum& a, const Vec& b, const KronSvdPreconditioner& m,
                        const SolverOptions& o) {
  return detail::solve(a, b, o, [&](kp_solver_options& ko, kp_history& kh, double* x) {
    return kp_fpcg(a.handle(), b.data(), m.handle(), &ko, x, &kh);
  });
}

// SpectralData + selectors (regparam.hpp:19-90)
class SpectralData {
 public:
  SpectralData(const KronSvdPreconditioner& p, const Vec& b, const Vec* x_true = nullptr) {
    kp_spectral* s = nullptr;
    check(kp_spectral_create_x(p.handle(), b.data(), x_true ? x_true->data() : nullptr, &s));
    s_.reset(s, [](kp_spectral* q) { kp_spectral_destroy(q); });
  }
  const kp_spectral* handle() const { return s_.get(); }

 private:
  std::shared_ptr<kp_spectral> s_;
};
inline SpectralData make_spectral_data(const KronSvdPreconditioner& p, const Vec& b) {
  return SpectralData(p, b);
}
inline SpectralData make_spectral_data(const KronSvdPreconditioner& p, const Vec& b,
                                       const Vec& x_true) {
  return SpectralData(p, b, &x_true);
}
// approx_spectrum / project_b / project_x (factor.hpp:76-88, factor.cpp:134-187)
struct ApproxSpectrum {
  Vec sigma;
  std::vector<long> perm;
};
inline ApproxSpectrum approx_spectrum(const KronSvdPreconditioner& p) {
  const int n = p.n();
  Vec sr(static_cast<size_t>(n), 0.0), sc(static_cast<size_t>(n), 0.0);
  check(kp_precond_export(p.handle(), 4, sr.data()));
  check(kp_precond_export(p.handle(), 5, sc.data()));
  const size_t nn = size_t(n) * n;
  Vec products(nn);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) products[size_t(j) * n + i] = sr[j] * sc[i];
  ApproxSpectrum out{Vec(nn), std::vector<long>(nn)};
  for (size_t k = 0; k < nn; ++k) out.perm[k] = long(k);
  std::stable_sort(out.perm.begin(), out.perm.end(), [&](long a, long b) { return products[a] > products[b]; });
  for (size_t k = 0; k < nn; ++k) out.sigma[k] = products[size_t(out.perm[k])];
  return out;
}
inline Vec project_b(const KronSvdPreconditioner& p, const Vec& b) {
  const size_t nn = size_t(p.n()) * p.n();
  if (b.size() != nn) throw std::invalid_argument("project: vector length is not n^2");
  SpectralData sd(p, b);
  Vec sigma(nn), bh(nn);
  check(kp_spectral_export(sd.handle(), sigma.data(), bh.data()));
  return bh;
}
inline Vec project_x(const KronSvdPreconditioner& p, const Vec& x) {
  const size_t nn = size_t(p.n()) * p.n();
  if (x.size() != nn) throw std::invalid_argument("project: vector length is not n^2");
  SpectralData sd(p, x, &x);
  Vec xh(nn);
  check(kp_spectral_export_xhat(sd.handle(), xh.data()));
  return xh;
}
inline double opt_objective(const SpectralData& sd, double lambda) {
  double v;
  check(kp_opt_objective(sd.handle(), lambda, &v));
  return v;
}
inline double wgcv_objective(const SpectralData& sd, double omega, double lambda) {
  double v;
  check(kp_wgcv_objective(sd.handle(), omega, lambda, &v));
  return v;
}
inline kp_param_choice lambda_opt(const SpectralData& sd) {
  kp_param_choice c;
  check(kp_lambda_opt(sd.handle(), &c));
  return c;
}
inline kp_param_choice wgcv(const SpectralData& sd, double omega) {
  kp_param_choice c;
  check(kp_wgcv(sd.handle(), omega, &c));
  return c;
}
inline Vec filtered_solution(const KronSvdPreconditioner& p, const Vec& b, double lambda) {
  Vec x(b.size());
  check(kp_filtered_solution(p.handle(), b.data(), lambda, x.data()));
  return x;
}
inline double gcv_objective(const SpectralData& sd, double lambda) {
  double v;
  check(kp_gcv_objective(sd.handle(), lambda, &v));
  return v;
}
inline double discrepancy_gap(const SpectralData& sd, double eps, double lambda) {
  double v;
  check(kp_discrepancy_gap(sd.handle(), eps, lambda, &v));
  return v;
}
inline kp_param_choice gcv(const SpectralData& sd) {
  kp_param_choice c;
  check(kp_gcv(sd.handle(), &c));
  return c;
}
inline kp_param_choice discrepancy(const SpectralData& sd, double noise_norm, double eta) {
  kp_param_choice c;
  check(kp_discrepancy(sd.handle(), noise_norm, eta, &c));
  return c;
}

}  // namespace kronprec_b200
