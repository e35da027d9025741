/*
 * kronprec_b200.h — C ABI of the B200-native PCG / FPCG / CGLS hot path.
 *
 * Drop-in boundary for the reference `kronprec` solver path (namespace
 * kronprec, the headers under /root/reference/proj/include/kronprec). Every entry point
 * names the reference interface it replaces. Plain pointers and sizes only:
 * matrices are dense column-major float64 (n-by-n, leading dimension n),
 * vectors are vec() = column stacking (kron.cpp:52-60), exactly like the
 * reference's Eigen::MatrixXd / VectorXd arguments.
 *
 * Error model (mirrors the reference's exception types):
 *   KP_OK                    0  success
 *   KP_ERR_INVALID_ARGUMENT  1  std::invalid_argument (shape / argument errors)
 *   KP_ERR_RUNTIME           2  std::runtime_error (SVD failure, NaN objective)
 *   KP_ERR_NO_ROOT           3  kronprec::NoRootError (discrepancy principle)
 *   KP_ERR_CUDA              4  CUDA runtime / launch failure (no CPU fallback)
 *   KP_ERR_UNSUPPORTED       5  option combination not implemented on device
 * The message of the last failure on the calling thread is kp_last_error().
 * Solver numerical breakdowns are NOT errors: as in the reference
 * (krylov.cpp:75-139) they are reported in kp_history.abort_reason with
 * converged = 0 and status KP_OK.
 *
 * Threading: one library context per process, one CUDA stream per context;
 * handles are not thread-safe. Host buffers are owned by the caller; handles
 * own device memory.
 */
#ifndef KRONPREC_B200_H
#define KRONPREC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_OK 0
#define KP_ERR_INVALID_ARGUMENT 1
#define KP_ERR_RUNTIME 2
#define KP_ERR_NO_ROOT 3
#define KP_ERR_CUDA 4
#define KP_ERR_UNSUPPORTED 5

/* PrecisionFormat (precision.hpp:14-37). significand_bits counts the implicit
 * bit (fp16: t=11, emax=15). A format with t>=53, emax>=1023 and subnormals
 * "covers double" and makes every rounding the identity. */
typedef struct kp_format {
  int significand_bits;
  int max_exponent;
  int subnormals_enabled;
} kp_format;

/* Accumulation semantics of the low-precision preconditioner solve.
 * KP_ACCUM_REFERENCE: every product rounded to fmt, sums over the fixed
 *   pairwise tree with one rounding per stage — bit-identical to
 *   lp_matmul (lpblas.cpp:13-70). Default.
 * KP_ACCUM_TENSOR: fp16 operands on the tcgen05 tensor pipe, fp32
 *   accumulation, one rounding of each GEMM result to fp16 (north-star mode;
 *   iteration counts may differ from the reference by a few). fp16 only. */
#define KP_ACCUM_REFERENCE 0
#define KP_ACCUM_TENSOR 1

/* Engine of the reference-exact binary16 products (KP_ACCUM_REFERENCE).
 * Both give bit-identical results (lp_matmul, lpblas.cpp:59-70):
 *   KP_FP16_PRODUCTS_CUDA_CORES  rounded products and tree adds on the f16x2
 *                                pipe (gemm_f16ref)
 *   KP_FP16_PRODUCTS_TENSOR      rounded products from tcgen05 MMAs with an
 *                                f16 accumulator and a diagonal-expanded B
 *                                operand, tree adds on the f16x2 pipe
 *                                (gemm_f16x)
 *   KP_FP16_PRODUCTS_AUTO        tensor from n >= 512 (default; environment
 *                                KP_FP16_PRODUCTS=cuda|tensor|auto) */
#define KP_FP16_PRODUCTS_AUTO 0
#define KP_FP16_PRODUCTS_CUDA_CORES 1
#define KP_FP16_PRODUCTS_TENSOR 2

/* SolverOptions (krylov.hpp:14-22). When device_pointers != 0, b, x and
 * x_true passed to the solvers are device pointers (kp_device_alloc). */
typedef struct kp_solver_options {
  double lambda;
  int max_iterations;
  double rel_residual_tol;
  const double* x_true; /* NULL = no relative-error track */
  int track_search_direction_orthogonality;
  int record_iterates; /* requires kp_history.iterates != NULL */
  int device_pointers;
} kp_solver_options;

/* ConvergenceHistory (krylov.hpp:29-42). The caller provides arrays with
 * `capacity` rows (max_iterations + 1 is always enough); row k is the state
 * after k iterations. iterates (optional) holds capacity * n^2 doubles. */
typedef struct kp_history {
  int capacity;
  double* relative_error;   /* may be NULL; filled only when x_true given */
  double* residual_norm;
  double* work_units;
  double* residual_cosines; /* may be NULL; capacity entries */
  double* iterates;         /* may be NULL */
  int rows;                 /* rows written (= iterations_used + 1) */
  int n_cosines;
  int iterations_used;
  int converged;
  int msolve_count;
  char abort_reason[192];   /* empty on a clean run */
} kp_history;

/* ParamChoice (regparam.hpp:36-46). method: 0 opt, 1 gcv, 2 wgcv,
 * 3 discrepancy, 4 gcv on an explicit grid. */
typedef struct kp_param_choice {
  double lambda;
  int method;
  double omega;
  double eta;
  double noise_norm;
  double objective_value;
  double bracket_lo;
  double bracket_hi;
  int flat_objective;
  int grid_index; /* grid selectors only; -1 otherwise */
} kp_param_choice;

typedef struct kp_operator kp_operator; /* KroneckerSum (kron.hpp:19-22)   */
typedef struct kp_precond kp_precond;   /* KronSvdPreconditioner (factor.hpp:42-54) */
typedef struct kp_spectral kp_spectral; /* SpectralData (regparam.hpp:19-24) */

/* ---- context ---------------------------------------------------------- */
const char* kp_last_error(void);
/* Every host thread has its own context: kp_init selects the device and
 * creates the calling thread's stream (a thread that never calls it gets the
 * device current for it). Handles are used by one thread at a time. */
int kp_init(int device);
int kp_synchronize(void);
int kp_device_alloc(size_t bytes, void** dptr);
int kp_device_free(void* dptr);
int kp_memcpy_h2d(void* dst, const void* src, size_t bytes);
int kp_memcpy_d2h(void* dst, const void* src, size_t bytes);
/* Per-kernel-class device timing (CUDA events on the library stream).
 * class ids: 0 fp64 operator GEMM, 1 preconditioner GEMM, 2 vector kernels,
 * 3 spectral / lambda kernels, 4 preconditioner auxiliaries (row sign
 * hashes and zero-sign fix-ups of the tensor fp16 product engine). */
int kp_profile_enable(int on);
int kp_profile_read(int kernel_class, double* total_ms, long long* launches);
int kp_profile_reset(void);
long long kp_launch_count(void);   /* kernels launched by this library (all threads) */
/* How solves ran their iterations: as one device-side loop (a CUDA graph
 * with a WHILE conditional node; the default) or as host-polled graph
 * replays (profiled solves, KP_GRAPH_LOOP=0, or a loop graph that could not
 * be built). Counts since load, all threads. */
int kp_drive_stats(long long* loop_solves, long long* polled_solves);
/* Process-wide engine for reference-exact binary16 products (see above);
 * kp_get_fp16_products reports whether size n would use the tensor engine. */
int kp_set_fp16_products(int mode);
int kp_get_fp16_products(int n, int* uses_tensor);
/* Device timestamps on the library stream (slots 0..15), for callers that
 * time whole solves on the device. */
int kp_event_record(int slot);
int kp_event_elapsed(int slot_start, int slot_end, float* ms);
/* Page-locked host buffers (fast H2D / D2H for host-pointer calls). */
int kp_host_alloc(size_t bytes, void** hptr);
int kp_host_free(void* hptr);

/* ---- operator setup from a PSF: deblur.hpp / factor.hpp --------------- */
/* psf_to_kronsum (deblur.hpp:69-70, deblur.cpp:167-199): SVD of the n_p x n_p
 * PSF array (column-major, center (center_row, center_col)); every term with
 * s_k > truncation_tol * s_0 becomes a pair of n x n banded Toeplitz factors
 * (sign-fixed so the largest |u| entry is positive). max_rank > 0 keeps only
 * the first max_rank terms (the BASELINE configs' rank cap; 0 = none).
 * row_factors / col_factors receive `capacity` n*n blocks; *rank the number of
 * terms written. Pass them to kp_operator_create. */
int kp_psf_to_kronsum(const double* psf, int np, int center_row, int center_col, int n,
                      double truncation_tol, int max_rank, int capacity, double* row_factors,
                      double* col_factors, int* rank);
/* nearest_kron (factor.hpp:34-35, factor.cpp:25-58): one Kronecker pair
 * (A_r, A_c) for the preconditioner; weighting KronWeighting::Uniform or
 * ::Toeplitz (the reference default). */
#define KP_KRON_UNIFORM 0
#define KP_KRON_TOEPLITZ 1
int kp_nearest_kron(const double* psf, int np, int center_row, int center_col, int n, int weighting,
                    double* row_factor, double* col_factor);

/* ---- operator: kron.hpp / kron.cpp ------------------------------------ */
/* row_factors / col_factors: r consecutive n-by-n column-major matrices,
 * term k = (row_factor_k, col_factor_k) as in KronTerm (kron.hpp:12-15). */
int kp_operator_create(int n, int r, const double* row_factors,
                       const double* col_factors, kp_operator** out);
int kp_operator_destroy(kp_operator* op);
int kp_operator_info(const kp_operator* op, int* n, int* r);
/* Operator algorithm. KP_OP_AUTO (default) uses the banded-Toeplitz kernels
 * when every factor is a banded Toeplitz matrix (the psf_to_kronsum
 * structure, deblur.cpp:157-199) with at most 64 diagonals and r <= 8, and
 * the dense DMMA GEMMs otherwise; KP_OP_DENSE forces the dense product the
 * reference computes (kron.cpp:69-70); KP_OP_BANDED fails with
 * KP_ERR_INVALID_ARGUMENT if the structure is absent. The environment
 * variable KP_OPERATOR=dense|banded sets the default at creation. */
#define KP_OP_AUTO 0
#define KP_OP_DENSE 1
#define KP_OP_BANDED 2
/* banded with both correlation passes in ONE kernel (shared-memory halo
 * tiles, no r n^2 intermediate in HBM); short bands only (17 or 19
 * diagonals in both directions), KP_ERR_INVALID_ARGUMENT otherwise. Opt-in:
 * measured no faster than the two passes on B200. */
#define KP_OP_BANDED_FUSED 3
int kp_operator_set_mode(kp_operator* op, int mode);
/* mode in use (KP_OP_DENSE / KP_OP_BANDED / KP_OP_BANDED_FUSED) and the
 * number of diagonals of the column and row factors when banded (0
 * otherwise). */
int kp_operator_get_mode(const kp_operator* op, int* mode, int* col_taps, int* row_taps);
/* kronsum_apply (kron.cpp:73-79) / kronsum_apply_transpose (kron.cpp:81-88) */
int kp_kronsum_apply(const kp_operator* op, const double* y, double* out);
int kp_kronsum_apply_transpose(const kp_operator* op, const double* y,
                               double* out);
/* normal_matvec (krylov.cpp:146-152): A^T(A p) + lambda^2 p */
int kp_normal_matvec(const kp_operator* op, double lambda, const double* p,
                     double* out);

/* ---- preconditioner: factor.hpp / factor.cpp -------------------------- */
/* svd_dense (factor.cpp:14-23): a = u diag(s) v^T, s nonincreasing; a, u, v
 * n x n column-major host arrays, s length n. Backend KP_SVD_HOST: LAPACK
 * dgesdd on the host (the oracle's routine); KP_SVD_DEVICE: cuSOLVER FP64
 * on the GPU (gesvd, or one-sided Jacobi gesvdj with KP_SVD_ALGO=gesvdj).
 * Vectors agree up to sign; everything the path computes from them (M, the
 * GCV sums, the discrepancy lambda) is invariant to that. */
#define KP_SVD_HOST 0
#define KP_SVD_DEVICE 1
int kp_svd(const double* a, int n, int backend, double* u, double* s, double* v);
/* backend kp_precond_build uses (process-wide; env KP_SVD=device|host) */
int kp_set_svd_backend(int backend);
int kp_get_svd_backend(int* backend);
/* build_preconditioner (factor.cpp:80-104): SVDs of a_r, a_c (backend above),
 * weights S(i,j)=1/((s_r(j) s_c(i))^2+lambda^2), rounded V_r, V_c, S.
 * Any format: binary16 runs on the f16x2 GEMMs (or tcgen05 with
 * KP_ACCUM_TENSOR), double-covering formats on DMMA GEMMs, every other
 * (t, emax, subnormals) on the exact generic emulation. */
int kp_precond_build(const double* a_r, const double* a_c, int n,
                     double lambda, kp_format fmt, int accum,
                     kp_precond** out);
/* Same, from a caller-supplied SVD (u, s, v per factor; s nonincreasing). */
int kp_precond_build_from_svd(int n, const double* u_r, const double* s_r,
                              const double* v_r, const double* u_c,
                              const double* s_c, const double* v_c,
                              double lambda, kp_format fmt, int accum,
                              kp_precond** out);
/* with_lambda (factor.cpp:106-115) */
int kp_precond_with_lambda(const kp_precond* p, double lambda,
                           kp_precond** out);
int kp_precond_destroy(kp_precond* p);
/* precond_solve (factor.cpp:117-132) */
int kp_precond_solve(const kp_precond* p, const double* r, double* z);
/* Export a field (n*n doubles, or n for singular values):
 * 0 s_weights, 1 s_lp, 2 vr_lp, 3 vc_lp, 4 svd_r.s, 5 svd_c.s,
 * 6 svd_r.u, 7 svd_r.v, 8 svd_c.u, 9 svd_c.v */
int kp_precond_export(const kp_precond* p, int field, double* out);
int kp_precond_info(const kp_precond* p, int* n, double* lambda,
                    kp_format* fmt, int* accum);

/* ---- emulated low-precision BLAS: precision.hpp / lpblas.hpp ----------- */
/* round_array (precision.cpp:82-95) for any format; host arrays. */
int kp_round_array(const double* x, long count, kp_format fmt, double* out);
/* round_value (precision.cpp:82-86): scalar rounding, not tallied. */
int kp_round_value(double x, kp_format fmt, double* out);
/* RoundCallSession / round_call_count (precision.hpp:55-66, precision.cpp:11,
 * 90, 111-119): the calling thread's tally of vectorised rounding calls. The
 * device path fuses the roundings into its kernels, so the tally is kept
 * analytically: every API call adds the number of round_inplace calls the
 * reference makes for it (round_array 1; lp_matmul 1 + ceil(log2 k) for a
 * live format; build_preconditioner 3; with_lambda 1; precond_solve and every
 * M-solve of pcg / fpcg 2 + 4 (1 + ceil(log2 n)) for a live format, 0 for a
 * double-covering one). A session is the difference of two reads. */
int kp_round_call_count(unsigned long long* count);
/* lp_matmul (lpblas.cpp:59-70): c = tree_k round(a(:,k) b(k,:)), one
 * rounding per pairwise stage; a m x k, b k x n, c m x n, column-major host
 * arrays. Bit-identical to the reference for every format. */
int kp_lp_matmul(int m, int k, int n, const double* a, const double* b,
                 kp_format fmt, double* c);
/* round_leaves = 0: the products are taken as pre-rounded addends, which
 * with b = ones gives pairwise_sum (lpblas.cpp:34-37). */
int kp_lp_matmul_ex(int m, int k, int n, const double* a, const double* b,
                    kp_format fmt, int round_leaves, double* c);

/* ---- solvers: krylov.hpp / krylov.cpp --------------------------------- */
int kp_cgls(const kp_operator* op, const double* b,
            const kp_solver_options* opts, double* x, kp_history* hist);
int kp_pcg(const kp_operator* op, const double* b, const kp_precond* m,
           const kp_solver_options* opts, double* x, kp_history* hist);
int kp_fpcg(const kp_operator* op, const double* b, const kp_precond* m,
            const kp_solver_options* opts, double* x, kp_history* hist);
/* Batched pcg / fpcg over `batch` independent right-hand sides that share
 * the operator and the preconditioner factors, image i with its own
 * lambda (lambdas[i], host array; opts->lambda is ignored) — the
 * reference's per-image pipeline (cli.cpp:469-486 run_single: with_lambda
 * + pcg) for a whole batch in one device state machine (BASELINE C4).
 * b, x (and opts->x_true, if set) hold batch * n^2 doubles, image i at
 * i * n^2 (host or device per opts->device_pointers); hist points at
 * `batch` kp_history structs. Each image's iterates, history and abort
 * reason equal what kp_pcg / kp_fpcg with with_lambda(m, lambdas[i]) gives.
 * Requires the fp16 format (KP_ACCUM_REFERENCE or KP_ACCUM_TENSOR);
 * record_iterates is not supported (KP_ERR_INVALID_ARGUMENT). */
int kp_pcg_batch(const kp_operator* op, const kp_precond* m, int batch,
                 const double* b, const double* lambdas,
                 const kp_solver_options* opts, double* x, kp_history* hist);
int kp_fpcg_batch(const kp_operator* op, const kp_precond* m, int batch,
                  const double* b, const double* lambdas,
                  const kp_solver_options* opts, double* x, kp_history* hist);

/* ---- lambda selection: regparam.hpp / regparam.cpp -------------------- */
/* make_spectral_data (regparam.cpp:119-126): device-resident sigma_hat =
 * s_r(j) s_c(i) and b_hat = vec(U_c^T B U_r) from the FP64 SVD factors. */
int kp_spectral_create(const kp_precond* p, const double* b,
                       kp_spectral** out);
/* make_spectral_data(p, b, x_true) (regparam.cpp:127-134): also x_hat =
 * vec(V_c^T X_true V_r), required by kp_lambda_opt / kp_opt_objective. */
int kp_spectral_create_x(const kp_precond* p, const double* b,
                         const double* x_true, kp_spectral** out);
int kp_spectral_destroy(kp_spectral* sd);
/* Sorted nonincreasing like approx_spectrum/project_b (factor.cpp:134-177). */
int kp_spectral_export(const kp_spectral* sd, double* sigma_hat,
                       double* b_hat);
/* x_hat in the same (sorted) order as kp_spectral_export. */
int kp_spectral_export_xhat(const kp_spectral* sd, double* x_hat);
/* Pointwise criteria (regparam.cpp:216-246). */
int kp_gcv_objective(const kp_spectral* sd, double lambda, double* value);
int kp_opt_objective(const kp_spectral* sd, double lambda, double* value);
int kp_wgcv_objective(const kp_spectral* sd, double omega, double lambda,
                      double* value);
int kp_discrepancy_gap(const kp_spectral* sd, double epsilon, double lambda,
                       double* value);
/* GCV over an explicit lambda grid (one batched reduction); argmin is the
 * first minimum, as a left-to-right scan would pick it. */
int kp_gcv_grid(const kp_spectral* sd, const double* lambdas, int m,
                double* values, kp_param_choice* choice);
/* gcv (regparam.cpp:254-258): 1024-point log grid + golden refinement. */
int kp_gcv(const kp_spectral* sd, kp_param_choice* choice);
/* lambda_opt (regparam.cpp:248-252): needs kp_spectral_create_x. */
int kp_lambda_opt(const kp_spectral* sd, kp_param_choice* choice);
/* wgcv (regparam.cpp:260-286), omega > 0. */
int kp_wgcv(const kp_spectral* sd, double omega, kp_param_choice* choice);
/* filtered_solution (regparam.cpp:329-349): direct Tikhonov solution for
 * the Kronecker approximation, FP64 on the device; x is n*n (host). */
int kp_filtered_solution(const kp_precond* p, const double* b, double lambda,
                         double* x);
/* discrepancy (regparam.cpp:288-327); KP_ERR_NO_ROOT when no root. The
 * bisection (find_root, regparam.cpp:184-214) evaluates two levels of
 * candidate midpoints per device launch; lambda is bit-identical to the
 * one-point-at-a-time bisection. */
int kp_discrepancy(const kp_spectral* sd, double noise_norm, double eta,
                   kp_param_choice* choice);
/* make_test_problem (deblur.cpp:201-229) for `batch` images on the device:
 * x_true = the BASELINE blob image of image_seeds[i] (`blobs` Gaussian blobs,
 * clipped to [0, 1]), b_true = A x_true with this operator, noise =
 * Rng(noise_seeds[i]).normal() draws scaled to noise_levels[i] *
 * ||b_true||, b = b_true + noise. The mt19937_64 stream is the reference's
 * bit for bit (kp_rng_raw); the normals use the device log / sin / cos, so
 * noise and b match the host generator to the last bits. x_true, b, noise
 * (optional): batch * n^2 doubles (host or device per device_pointers);
 * noise_norms (optional, host): ||noise_i||. */
int kp_generate_test_problems(const kp_operator* op, int batch,
                              const unsigned long long* image_seeds, int blobs,
                              const unsigned long long* noise_seeds,
                              const double* noise_levels, double* x_true, double* b,
                              double* noise, double* noise_norms, int device_pointers);
/* std::mt19937_64 on the device (test hook): `count` raw outputs per seed,
 * out[i * count + k]. */
int kp_rng_raw(const unsigned long long* seeds, int batch, long count, unsigned long long* out);
/* The discrepancy lambda of `batch` right-hand sides b (batch * n^2 host
 * doubles, image i at i * n^2) sharing the preconditioner factors of p:
 * make_spectral_data(p, b_i) + discrepancy(sd_i, noise_norms[i], eta) for
 * every image, with all images' bisections advancing together (one batched
 * reduction launch per round). lambdas[i] is bit-identical to
 * kp_discrepancy's; status[i] = 0, KP_ERR_NO_ROOT or KP_ERR_RUNTIME (then
 * lambdas[i] = NaN). */
int kp_discrepancy_batch(const kp_precond* p, int batch, const double* b,
                         const double* noise_norms, double eta, double* lambdas,
                         int* status);
/* The same with b in device memory when device_pointers != 0 (a batch
 * generated by kp_generate_test_problems or left by an earlier call stays
 * resident: lambda selection + kp_pcg_batch without host round trips). */
int kp_discrepancy_batch_ex(const kp_precond* p, int batch, const double* b,
                            const double* noise_norms, double eta,
                            double* lambdas, int* status, int device_pointers);

#ifdef __cplusplus
}
#endif

#endif /* KRONPREC_B200_H */
