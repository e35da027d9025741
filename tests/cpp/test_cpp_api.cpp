// C++ consumer of include/kronprec_b200.hpp — reads like the reference's
// doctest cases (test_krylov.cpp "exact inverse converges in one iteration",
// test_factor.cpp "identity factors halve the rounded residual").
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "kronprec_b200.hpp"

using namespace kronprec_b200;

static int fails = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

static Vec eye(int n) {
  Vec m(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) m[size_t(i) * n + i] = 1.0;
  return m;
}

int main() {
  // identity operator: CGLS converges in one step
  const int n = 4;
  KroneckerSum I({KronTerm{eye(n), eye(n)}}, n);
  Vec b(16);
  for (int i = 0; i < 16; ++i) b[i] = std::sin(1.0 + i);
  SolverOptions o;
  o.lambda = 0.0;
  o.x_true = &b;
  SolveResult r = cgls(I, b, o);
  CHECK(r.history.converged && r.history.iterations_used == 1);
  CHECK(std::fabs(r.history.relative_error.back()) <= 1e-14);

  // identity preconditioner at lambda 1 halves the fp16-rounded residual
  KronSvdPreconditioner m = build_preconditioner(eye(n), eye(n), n, 1.0, fp16());
  Vec z = precond_solve(m, Vec(16, 0.1));
  CHECK(z[0] == 0.5 * 0.0999755859375);

  // exact-inverse preconditioner: PCG converges in one iteration
  Vec t(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) t[size_t(j) * n + i] = (i == j) ? 0.5 : (std::abs(i - j) == 1 ? 0.25 : 0.0);
  KroneckerSum A({KronTerm{t, t}}, n);
  KronSvdPreconditioner mx = build_preconditioner(t, t, n, 0.05, fp64());
  SolverOptions po;
  po.lambda = 0.05;
  SolveResult rp = pcg(A, b, mx, po);
  CHECK(rp.history.converged && rp.history.iterations_used == 1);

  // rounding-call budget (test_factor.cpp:302-317, test_krylov.cpp:259-287)
  {
    const int n8 = 8;
    Vec t8(size_t(n8) * n8, 0.0);
    for (int i = 0; i < n8; ++i)
      for (int j = 0; j < n8; ++j) t8[size_t(j) * n8 + i] = (i == j) ? 0.5 : (std::abs(i - j) == 1 ? 0.25 : 0.0);
    KronSvdPreconditioner p16 = build_preconditioner(t8, t8, n8, 0.05, fp16());
    RoundCallSession s;
    (void)precond_solve(p16, Vec(64, 1.0));
    CHECK(s.count() == 2 + 4 * (1 + 3));
    KronSvdPreconditioner p64 = build_preconditioner(t8, t8, n8, 0.05, fp64());
    RoundCallSession s2;
    (void)precond_solve(p64, Vec(64, 1.0));
    CHECK(s2.count() == 0);
    KroneckerSum A8({KronTerm{t8, t8}}, n8);
    Vec b8(64);
    for (int i = 0; i < 64; ++i) b8[i] = std::sin(0.3 + i);
    SolverOptions o8;
    o8.lambda = 0.05, o8.max_iterations = 10, o8.rel_residual_tol = 1e-12;
    RoundCallSession base;
    (void)cgls(A8, b8, o8);
    CHECK(round_call_count(base) == 0);
    RoundCallSession prec;
    SolveResult r8 = pcg(A8, b8, p16, o8);
    CHECK(round_call_count(prec) == std::uint64_t(18) * std::uint64_t(r8.history.msolve_count));
    CHECK(r8.history.msolve_count >= r8.history.iterations_used);
    RoundCallSession dbl;
    (void)pcg(A8, b8, p64, o8);
    CHECK(round_call_count(dbl) == 0);
    CHECK(round_value(0.1, fp16()) == 0.0999755859375);
  }

  // kron_apply / svd_dense / approx_spectrum / project_b / project_x (kron.hpp:29-31, factor.hpp:19, 76-88)
  {
    const int n3 = 3;
    Vec c3 = {1, 2, 3, 0, 1, 4, 5, 6, 0}, d3 = {2, 0, 1, 1, 3, 0, 0, 1, 1}, y3(9);
    for (int i = 0; i < 9; ++i) y3[i] = 1.0 + i;
    Vec k3 = kron_apply(c3, d3, n3, y3);
    // (C (x) D) y entry (j n + i) = sum_{l,m} C(j,l) D(i,m) y(l n + m)
    for (int j = 0; j < n3; ++j)
      for (int i = 0; i < n3; ++i) {
        double ref = 0.0;
        for (int l = 0; l < n3; ++l)
          for (int m2 = 0; m2 < n3; ++m2) ref += c3[l * n3 + j] * d3[m2 * n3 + i] * y3[l * n3 + m2];
        CHECK(std::fabs(k3[j * n3 + i] - ref) <= 1e-12);
      }
    SvdTriple sv = svd_dense(c3, n3);
    CHECK(sv.s[0] >= sv.s[1] && sv.s[1] >= sv.s[2] && sv.s[2] >= 0.0);
    KronSvdPreconditioner p3 = build_preconditioner(c3, d3, n3, 0.1, fp16());
    ApproxSpectrum as = approx_spectrum(p3);
    for (size_t k = 1; k < as.sigma.size(); ++k) CHECK(as.sigma[k - 1] >= as.sigma[k]);
    Vec pb = project_b(p3, y3), px = project_x(p3, y3);
    double nb = 0, nx = 0, ny = 0;
    for (int i = 0; i < 9; ++i) nb += pb[i] * pb[i], nx += px[i] * px[i], ny += y3[i] * y3[i];
    CHECK(std::fabs(nb - ny) <= 1e-10 * ny && std::fabs(nx - ny) <= 1e-10 * ny);  // orthogonal bases
    CHECK(lp_dot(Vec{2048, 1, 1, 1}, Vec{1, 1, 1, 1}, fp16()) == 2050.0);        // test_lpblas.cpp pin
    CHECK(pairwise_sum(Vec{2048, 1, 1, 1}, fp16()) == 2050.0);
    CHECK(lp_matvec(Vec{2048, 1, 1, 1}, Vec{1, 1, 1, 1}, 1, 4, fp16())[0] == 2050.0);
  }

  // emulated low-precision BLAS (test_lpblas.cpp pins)
  CHECK(round_array(Vec{1.0 + 1.0 / 4096}, fp16())[0] == 1.0);
  const Vec c = lp_matmul(Vec{1, 3, 2, 4}, Vec{5, 7, 6, 8}, 2, 2, 2, fp16());  // [[1,2],[3,4]] x [[5,6],[7,8]]
  CHECK(c[0] == 19 && c[1] == 43 && c[2] == 22 && c[3] == 50);
  CHECK(lp_matmul(Vec{2048, 1, 1, 1}, Vec{1, 1, 1, 1}, 1, 4, 1, fp16())[0] == 2050.0);

  // optimal lambda and the filtered solution (regparam.cpp:248-252, 329-349)
  SpectralData sdx = make_spectral_data(mx, b, b);
  const kp_param_choice opt = lambda_opt(sdx);
  CHECK(opt.lambda > 0.0 && std::isfinite(opt.objective_value));
  const Vec xf = filtered_solution(mx, b, 0.05);
  CHECK(xf.size() == b.size() && std::isfinite(xf[0]));

  // operator setup from a PSF (deblur.hpp:69-70, factor.hpp:34-35): a
  // separable 5 x 5 PSF is one Kronecker term, and nearest_kron returns it
  Psf psf;
  psf.np = 5;
  psf.center_row = psf.center_col = 2;
  const double g[5] = {0.1, 0.2, 0.4, 0.2, 0.1};
  for (int j = 0; j < 5; ++j)
    for (int i = 0; i < 5; ++i) psf.values.push_back(g[i] * g[j]);
  KroneckerSum ap = psf_to_kronsum(psf, 16);
  const Vec ones(256, 1.0);
  const Vec ay = kronsum_apply(ap, ones);
  CHECK(std::fabs(ay[8 * 16 + 8] - 1.0) <= 1e-12);  // interior pixel: the PSF sums to 1
  const KronTerm nk = nearest_kron(psf, 16);
  CHECK(nk.row_factor.size() == 256 && std::fabs(nk.row_factor[8 * 16 + 8] * nk.col_factor[8 * 16 + 8] - 0.16) <= 1e-12);
  KroneckerSum ap2 = psf_to_kronsum(psf, 16, 1e-12, 1);  // rank cap
  CHECK(std::fabs(kronsum_apply(ap2, ones)[8 * 16 + 8] - 1.0) <= 1e-12);

  // the preconditioner from caller-held SVDs (KronSvdPreconditioner::svd_r /
  // svd_c) equals the one the library builds: diagonal factors, u = v = I
  Vec d(size_t(n) * n, 0.0);
  const double dv[4] = {2.0, 1.5, 1.0, 0.5};
  for (int i = 0; i < n; ++i) d[size_t(i) * n + i] = dv[i];
  SvdTriple sv{eye(n), Vec(dv, dv + 4), eye(n)};
  KronSvdPreconditioner ms = build_preconditioner_from_svd(sv, sv, n, 0.1, fp16());
  KronSvdPreconditioner mb = build_preconditioner(d, d, n, 0.1, fp16());
  const Vec zs = precond_solve(ms, b), zb = precond_solve(mb, b);
  bool same = true;
  for (int i = 0; i < 16; ++i) same = same && zs[i] == zb[i];
  CHECK(same);

  // the reference's argument checks (krylov.cpp:12-27, factor.cpp:84-87, :119-120)
  bool threw_len = false;
  try { precond_solve(ms, Vec(15, 1.0)); } catch (const std::invalid_argument&) { threw_len = true; }
  CHECK(threw_len);
  bool threw_fac = false;
  try { build_preconditioner(eye(n), Vec(15, 1.0), n, 0.1, fp16()); } catch (const std::invalid_argument&) { threw_fac = true; }
  CHECK(threw_fac);
  const Vec zero(16, 0.0);
  SolverOptions oz;
  oz.x_true = &zero;
  bool threw_x = false;
  try { cgls(I, b, oz); } catch (const std::invalid_argument&) { threw_x = true; }
  CHECK(threw_x);
  SolverOptions o0;
  o0.max_iterations = 0;
  bool threw_it = false;
  try { cgls(I, b, o0); } catch (const std::invalid_argument&) { threw_it = true; }
  CHECK(threw_it);

  // errors surface as the reference's exception types
  bool threw = false;
  try { build_preconditioner(eye(2), eye(2), 2, -1.0, fp64()); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  SpectralData sd = make_spectral_data(mx, b);
  threw = false;
  try { discrepancy(sd, 1e6, 1.0); } catch (const NoRootError&) { threw = true; }
  CHECK(threw);
  std::printf(fails ? "cpp api: %d failures\n" : "cpp api: ok\n", fails);
  return fails ? 1 : 0;
}
