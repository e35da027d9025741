// Fused FP64 CG vector kernels, the device-resident solver state machine and
// the spectral (lambda-selection) reductions.
#pragma once

#include "common.cuh"

namespace kp {

// Solver status values (DevState::status).
// ST_INVALID: x_true is all zero (krylov.cpp:21-25 throws invalid_argument)
enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_ABORTED = 2, ST_MAXIT = 3, ST_INVALID = 4 };
// Abort codes -> reference messages (krylov.cpp:75-139, 175-194).
enum {
  AB_NONE = 0,
  AB_M_NONFINITE_INIT = 1,   // "non-finite preconditioner output before iteration 1"
  AB_POSITIVITY_INIT = 2,    // "preconditioner lost positivity before iteration 1"
  AB_CURV_NONFINITE = 3,     // "non-finite curvature at iteration k"
  AB_CURV_BREAKDOWN = 4,     // "curvature breakdown at iteration k"
  AB_RESID_NONFINITE = 5,    // "non-finite residual at iteration k"
  AB_M_NONFINITE = 6,        // "non-finite preconditioner output at iteration k (overflow ...)"
  AB_INNER_NONFINITE = 7,    // "non-finite inner product at iteration k"
  AB_POSITIVITY = 8,         // "preconditioner lost positivity at iteration k"
};

struct DevState {
  int status;
  int k;  // iteration being executed (1-based)
  int abort_code;
  int abort_iter;
  int msolve_count;
  int iterations_used;
  int rows;
  int ncos;
  int maxit;
  int flexible;
  int track_cos;
  int has_xt;
  int record;
  unsigned ticket;  // CTAs done in the running fused kernel (last-CTA tails); 0 between kernels
  double tol, l2, work_per_iter;
  double r0, xnorm, rho, alpha, beta, gamma, pnorm2, rz, snorm_prev;
};

// History arrays on device (capacity rows).
struct DevHistory {
  double* resid;
  double* relerr;
  double* cosines;
  double* iterates;  // capacity * nn, optional
  int capacity;
};

// Partial-sum buffers are [ctas][4] doubles.
constexpr int VEC_CTAS = 1184;  // fixed grid of the vector kernels (8 x 148 SMs)
constexpr int VEC_THREADS = 256;

// ---- generic helpers -------------------------------------------------------
void vec_copy(double* dst, const double* src, size_t n, const int* status);
void vec_zero(double* dst, size_t n);
// partials[cta*4+0] = sum x*y over the fixed VEC_CTAS grid
void vec_dot_partials(const double* x, const double* y, size_t n, double* partials);
// dst16[l*ldh + i] = round16(src[l*n + i]) (RNE binary16, overflow -> inf)
void cast_f64_to_f16_padded(const double* src, __half* dst, int rows, int cols, long ld_src,
                            long ld_dst, const int* status);

// S weights of the Kronecker-SVD preconditioner (factor.cpp:62-76) into s64
// (FP64) and/or s16 (binary16), column-major n x n.
void precond_weights(const double* s_r, const double* s_c, int n, double l2, double* s64,
                     __half* s16);

// Last step of the tensor-mode M-solve: z[l*n + i] = double(z16[l*ldh + i])
// (exact) with the M-solve dot partials over the fixed VEC_CTAS grid:
// [0] z.d0, [1] z.(d1a - d1b) (d1b optional), [2] #non-finite z.
// batch > 1: image i's z16 at i * n * ldh, vectors at i * n^2, partials at
// i * VEC_CTAS slots.
void msolve_finish_f16(const __half* z16, long ldh, int n, double* z, const double* d0,
                       const double* d1a, const double* d1b, double* partials,
                       const int* status, int batch = 1);

// ---- PCG -------------------------------------------------------------------
// Every PCG kernel takes `batch` (default 1): a batch of independent solves
// (kp_pcg_batch) runs image i with DevState st[i], history rows from
// i * h.capacity, vectors at i * n^2 (binary16 r at i * n * ldh) and its own
// partial slots (i * slots per image). batch = 1 is the single solve.
// init after r = A^T b (partials_r: [ctas] of ||r||^2) and xnorm partials.
void pcg_init_scalar(DevState* st, DevHistory h, const double* part_r, int nr,
                     const double* part_xt, int nxt, int batch = 1);
// after first M-solve (partials: [0]=r.z, [2]=#nonfinite)
void pcg_init_msolve_scalar(DevState* st, const double* part_z, int nz, int batch = 1);
void pcg_alpha_scalar(DevState* st, const double* part_pq, int n, int batch = 1);
// CTAs (= partials) pcg_update uses at size n (fixed for a given n)
int pcg_update_ctas(int n);
// Scalar steps folded into the neighbouring vector kernel (small n, where
// each launch is a fixed ~2 us on the iteration's critical path): possible
// when the slot sum fits one vector CTA (a function of the slot count only,
// so batched and single solves fold identically; the sums are the same
// fixed-order reductions, so the results are bit-identical either way).
bool pcg_fold_ok(int slots);
// x += a p; r -= a q; [r_prev = r]; R16 = round16(r); partials:
// [0] ||r||^2, [1] ||x - xt||^2, [2] r.z, [3] ||z||^2.
// part_pq != nullptr: alpha (pcg_alpha_scalar over part_pq / n_pq slots) is
// formed in every CTA first; fold_resid: the last CTA to finish runs
// pcg_resid_scalar over the kernel's own partials.
void pcg_update(DevState* st, DevHistory h, double* x, double* r, double* r_prev,
                const double* p, const double* q, const double* z, const double* xt, __half* r16,
                int n, long ldh, double* partials, int batch = 1, const double* part_pq = nullptr,
                int n_pq = 0, bool fold_resid = false);
void pcg_resid_scalar(DevState* st, DevHistory h, const double* part, int n, int batch = 1);
void pcg_beta_scalar(DevState* st, const double* part_z, int n, int batch = 1);
// p = z + beta p; part_z != nullptr: beta (pcg_beta_scalar over part_z / nz
// slots) formed in every CTA first, the rho / positivity / k step by the
// last CTA to finish
void pcg_p_update(DevState* st, double* p, const double* z, size_t nn, int batch = 1,
                  const double* part_z = nullptr, int nz = 0);
// out->status = ST_RUNNING while any of st[0..count) runs, else ST_CONVERGED
void batch_status(const DevState* st, int count, DevState* out);

// ---- CGLS ------------------------------------------------------------------
void cgls_init_scalar(DevState* st, DevHistory h, const double* part_s, int ns,
                      const double* part_xt, int nxt);
void cgls_alpha_scalar(DevState* st, const double* part_q, int nq, const double* part_p, int np);
// x += a p; rt -= a q; partials [1] ||x - xt||^2
void cgls_update(DevState* st, DevHistory h, double* x, double* rt, const double* p,
                 const double* q, const double* xt, size_t nn, double* partials);
void cgls_resid_scalar(DevState* st, DevHistory h, const double* part_s, int ns,
                       const double* part_x, int nx);
// p = s + beta p; [s_prev = s]; partials [0] ||p||^2
void cgls_p_update(DevState* st, double* p, const double* s, double* s_prev, size_t nn,
                   double* partials);

// ---- spectral ----------------------------------------------------------------
// Per-lambda sums over sigma(i,j) = s_r[j] s_c[i], d = sigma^2 + lambda^2
// (regparam.cpp:216-246), written to out[q*2 + {0,1}] (device):
enum SpectralKind {
  SK_GCV = 0,     // sum (bhat/d)^2,          sum 1/d
  SK_RESID = 1,   // sum (lambda^2 bhat/d)^2, 0
  SK_OPT = 2,     // sum (sigma bhat/d - xhat)^2, 0
  SK_WGCV = 3,    // sum (lambda^2 bhat/d)^2, sum ((1-omega) sigma^2 + lambda^2)/d
  SK_WTRACE = 4,  // sum ((1-omega) sigma^2 + lambda^2)/d, 0
};
// c(i,j) *= sigma / (sigma^2 + l2) (filtered_solution coefficients), device
void spectral_filter(const double* s_r, const double* s_c, int n, double l2, double* c);
// batch > 1: `batch` rows (lambdas at row * m, out rows row * m + q) over
// the coefficients of image img_index[row] (device; nullptr: image = row) at
// image * n^2, each summed exactly as a single call would.
void spectral_sums(int kind, const double* s_r, const double* s_c, const double* bhat,
                   const double* xhat, int n, const double* lambdas, int m, double omega,
                   double* out, int batch = 1, const int* img_index = nullptr);

}  // namespace kp
