// Device SVD of an n x n FP64 matrix (cuSOLVER; see svd_dev.cu).
#pragma once

namespace kp {
// a_host column-major n x n; u, v (n x n, column-major) and s (n,
// nonincreasing) on the host: A = U diag(s) V^T (svd_dense contract,
// factor.cpp:14-23).
void device_svd(const double* a_host, int n, double* u, double* s, double* v);
}  // namespace kp
