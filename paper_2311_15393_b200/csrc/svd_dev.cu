// Device SVD of the Kronecker factors (the setup path,
// factor.cpp:14-23 svd_dense / :80-104 build_preconditioner). The reference
// runs Eigen's JacobiSVD on the host; at n = 4096 the host LAPACK call the
// library used so far (dgesdd, the oracle's routine) takes ~15 s per
// factor pair, ~20x the whole C5 solve. Here the factor is uploaded once
// and decomposed by cuSOLVER in FP64 on the B200:
//   gesvdj  one-sided Jacobi (the reference's algorithm family), U and V
//           returned directly, singular values sorted nonincreasing
//   gesvd   Householder bidiagonalisation + QR (returns V^T; transposed on
//           the device)
// KP_SVD_ALGO=gesvd|gesvdj picks one (default gesvd, measured faster at
// n = 4096). The result has the svd_dense contract: A = U diag(s) V^T with
// s nonincreasing, invalid_argument on empty / non-finite input,
// runtime_error when the backend does not converge. Singular vectors agree
// with LAPACK's up to sign (and rotation within repeated singular values);
// M, the GCV sums and the discrepancy lambda are invariant to both
// (tests/test_gpu_configs.py::test_setup_svd_backend_invariance).
#include <cusolverDn.h>

#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "svd_dev.h"

namespace kp {
namespace {

void cs_check(cusolverStatus_t st, const char* what) {
  if (st != CUSOLVER_STATUS_SUCCESS)
    throw CudaError(std::string("cuSOLVER ") + what + " failed: " + std::to_string(int(st)));
}

struct SolverHandle {
  cusolverDnHandle_t h = nullptr;
  int device = -1;
  ~SolverHandle() {
    if (h) cusolverDnDestroy(h);
  }
};

cusolverDnHandle_t handle() {
  static thread_local SolverHandle sh;
  Ctx& c = ctx();
  if (!sh.h || sh.device != c.device) {
    if (sh.h) cusolverDnDestroy(sh.h);
    cs_check(cusolverDnCreate(&sh.h), "create");
    sh.device = c.device;
  }
  cs_check(cusolverDnSetStream(sh.h, c.stream), "set stream");
  return sh.h;
}

__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst, int n) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = bx + threadIdx.x, c = by + j;
    if (r < n && c < n) t[j][threadIdx.x] = src[size_t(c) * n + r];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = by + threadIdx.x, c = bx + j;
    if (r < n && c < n) dst[size_t(c) * n + r] = t[threadIdx.x][j];
  }
}

int algo() {
  static const int a = [] {
    const char* e = getenv("KP_SVD_ALGO");
    return e && std::string(e) == "gesvdj" ? 1 : 0;
  }();
  return a;
}

}  // namespace

void device_svd(const double* a_host, int n, double* u, double* s, double* v) {
  if (n < 1) throw InvalidArgument("svd_dense: empty matrix");
  const size_t nn = size_t(n) * n;
  for (size_t q = 0; q < nn; ++q)
    if (!std::isfinite(a_host[q])) throw InvalidArgument("svd_dense: non-finite entries");
  cusolverDnHandle_t h = handle();
  cudaStream_t st = ctx().stream;
  DBuf<double> A(nn), U(nn), V(nn), S(n);
  DBuf<int> info(1);
  KP_CUDA(cudaMemcpyAsync(A.p, a_host, nn * sizeof(double), cudaMemcpyHostToDevice, st));
  int lwork = 0;
  if (algo() == 1) {
    gesvdjInfo_t params = nullptr;
    cs_check(cusolverDnCreateGesvdjInfo(&params), "gesvdj info");
    try {
      cs_check(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, A.p, n, S.p, U.p, n, V.p, n,
                                            &lwork, params),
               "gesvdj buffer size");
      DBuf<double> work(static_cast<size_t>(lwork));
      cs_check(cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 0, n, n, A.p, n, S.p, U.p, n, V.p, n, work.p,
                                 lwork, info.p, params),
               "gesvdj");
      int hinfo = 0;
      KP_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      KP_CUDA(cudaStreamSynchronize(st));
      if (hinfo != 0) throw std::runtime_error("svd_dense: backend did not converge");
    } catch (...) {
      cusolverDnDestroyGesvdjInfo(params);
      throw;
    }
    cusolverDnDestroyGesvdjInfo(params);
  } else {
    cs_check(cusolverDnDgesvd_bufferSize(h, n, n, &lwork), "gesvd buffer size");
    DBuf<double> work(static_cast<size_t>(lwork));
    DBuf<double> VT(nn);
    cs_check(cusolverDnDgesvd(h, 'A', 'A', n, n, A.p, n, S.p, U.p, n, VT.p, n, work.p, lwork, nullptr, info.p),
             "gesvd");
    int hinfo = 0;
    KP_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    KP_CUDA(cudaStreamSynchronize(st));
    if (hinfo != 0) throw std::runtime_error("svd_dense: backend did not converge");
    LaunchScope scope(KC_SPECTRAL);
    transpose_kernel<<<dim3(cdiv(n, 32), cdiv(n, 32)), dim3(32, 8), 0, st>>>(VT.p, V.p, n);
    check_launch("svd transpose");
  }
  KP_CUDA(cudaMemcpyAsync(u, U.p, nn * sizeof(double), cudaMemcpyDeviceToHost, st));
  KP_CUDA(cudaMemcpyAsync(v, V.p, nn * sizeof(double), cudaMemcpyDeviceToHost, st));
  KP_CUDA(cudaMemcpyAsync(s, S.p, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st));
  KP_CUDA(cudaStreamSynchronize(st));
}

}  // namespace kp
