// kronprec_b200.hpp — header-only C++ mirror of the reference `kronprec`
// solver API (/root/reference/proj/include/kronprec/*.hpp) over the C ABI in
// kronprec_b200.h. Same names, argument meaning and exception types; dense
// matrices are column-major std::vector<double> (Eigen's storage order), so
// an Eigen caller passes .data() pointers.
#pragma once

#include <memory>
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
// lp_matmul (lpblas.cpp:59-70): a m x k, b k x n, column-major
inline Vec lp_matmul(const Vec& a, const Vec& b, int m, int k, int n, kp_format fmt) {
  if (a.size() != size_t(m) * k || b.size() != size_t(k) * n)
    throw std::invalid_argument("lp_matmul: shape mismatch");
  Vec c(size_t(m) * n);
  check(kp_lp_matmul(m, k, n, a.data(), b.data(), fmt, c.data()));
  return c;
}

// KronTerm / KroneckerSum (kron.hpp:12-22): factors are n*n column-major.
struct KronTerm {
  Vec row_factor, col_factor;
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
  kp_precond* p = nullptr;  // factor.cpp:80-104
  check(kp_precond_build(a_r.data(), a_c.data(), n, lambda, fmt, accum, &p));
  return KronSvdPreconditioner(p);
}
inline KronSvdPreconditioner with_lambda(const KronSvdPreconditioner& p, double lambda) {
  kp_precond* q = nullptr;  // factor.cpp:106-115
  check(kp_precond_with_lambda(p.handle(), lambda, &q));
  return KronSvdPreconditioner(q);
}
inline Vec precond_solve(const KronSvdPreconditioner& p, const Vec& r) {  // factor.cpp:117-132
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
  const size_t nn = size_t(a.n()) * a.n();
  if (b.size() != nn) throw std::invalid_argument("solver: right-hand side length mismatch");
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
