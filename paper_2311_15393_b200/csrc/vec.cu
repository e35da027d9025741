// Fused FP64 CG vector kernels (krylov.cpp:58-208), the device-resident
// solver state machine, and the lambda-selection reductions
// (regparam.cpp:224-246).
//
// Every kernel first reads DevState::status and returns when the solve has
// stopped, so the host can enqueue iterations without synchronising; the
// scalar kernels reproduce the reference's check order and abort messages.
// All reductions use a grid fixed for a given n (VEC_CTAS, or fewer CTAs
// for pcg_update at small n) and fixed-order combination, so
// results are run-to-run deterministic.
#include "vec.cuh"

namespace kp {
namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Block-wide sum of NV values per thread; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*red)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp][q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w][q];
      v[q] = s;
    }
  }
}

// Sum of component q of a [n][4] partials array in fixed order by the first
// T threads of the block (T a power of two >= 32, <= blockDim.x; every
// thread of the block must call it), returned to all threads: thread t < T
// sums slots t, t + T, ..., warp sums by xor shuffles, then the T / 32 warp
// sums in order from 0.0 — a function of (n, T) only, so a scalar kernel of
// T threads and a wider vector CTA folding the same step agree bit for bit.
// L2 loads: the slots may come from other CTAs of the running kernel.
constexpr int SCALAR_THREADS = 1024;
__device__ double sum_slots(const double* part, int n, int q, int T) {
  __shared__ double red[SCALAR_THREADS / 32];
  __shared__ double out;
  double v = 0.0;
  if (int(threadIdx.x) < T)
    for (int i = threadIdx.x; i < n; i += T) v += __ldcg(part + size_t(i) * 4 + q);
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (T >> 5); ++w) s += red[w];
    out = s;
  }
  __syncthreads();
  return out;
}
__device__ double sum_partials(const double* part, int n, int q) { return sum_slots(part, n, q, blockDim.x); }

// Last-CTA election for the folded scalar tails: every CTA of the (x) grid
// calls it once after writing its partials; true in all threads of the CTA
// that finished last, which then sees every CTA's writes. Resets the ticket.
__device__ bool last_cta(DevState* st) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    if (last) st->ticket = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ bool stopped(const DevState* st) { return st->status != ST_RUNNING; }

// Batched solves (kp_pcg_batch): image `img` owns DevState st[img], history
// rows [img * capacity, ...), its vectors at img * nn and its partial slots
// at img * (slots per image). Single solves use img = 0.
__device__ __forceinline__ DevHistory hist_of(DevHistory h, int img, size_t nn) {
  if (img) {
    const size_t o = size_t(img) * h.capacity;
    h.resid += o;
    if (h.relerr) h.relerr += o;
    if (h.cosines) h.cosines += o;
    if (h.iterates) h.iterates += o * nn;
  }
  return h;
}

// ---------------------------------------------------------------------------
__global__ void copy_kernel(double* dst, const double* src, size_t n, const int* status) {
  pdl_wait();
  if (status && *status) return;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}
__global__ void zero_kernel(double* dst, size_t n) {
  pdl_wait();
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    dst[i] = 0.0;
}
__global__ void dot_partials_kernel(const double* x, const double* y, size_t n, double* part) {
  pdl_wait();
  __shared__ double red[VEC_THREADS / 32][1];
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    v[0] += x[i] * y[i];
  block_sum<1>(v, red);
  if (threadIdx.x == 0) {
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = v[0], o[1] = 0.0, o[2] = 0.0, o[3] = 0.0;
  }
}

__global__ void cast_f16_kernel(const double* src, __half* dst, int rows, int cols, long ld_src,
                                long ld_dst, const int* status) {
  pdl_wait();
  if (status && *status) return;
  const size_t total = size_t(rows) * cols;
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const size_t l = idx / cols, i = idx % cols;
    dst[l * ld_dst + i] = __double2half(src[l * ld_src + i]);  // cvt.rn.f16.f64
  }
}

// Tensor-mode M-solve tail: the last tcgen05 product stores binary16 z
// (one rounding, as its FP64 epilogue did); this pass widens it to FP64 and
// forms the dot partials pcg_beta needs, at HBM speed instead of inside the
// GEMM's epilogue. Pairs of rows (half2 -> double2) when VEC2.
template <bool VEC2>
__global__ void msolve_finish_f16_kernel(const __half* z16, long ldh, int n, double* z,
                                         const double* d0, const double* d1a, const double* d1b,
                                         double* part, const int* status) {
  pdl_wait();
  if (status && *status) return;
  const size_t nn = size_t(n) * n;
  {  // batch image blockIdx.y
    const size_t img = blockIdx.y;
    z16 += img * n * ldh, z += img * nn;
    if (d0) d0 += img * nn;
    if (d1a) d1a += img * nn;
    if (d1b) d1b += img * nn;
    part += img * gridDim.x * 4;
  }
  __shared__ double red[VEC_THREADS / 32][3];
  const unsigned un = unsigned(n);
  const bool same = d0 && d1a == d0;
  double v[3] = {0.0, 0.0, 0.0};
  if (VEC2) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nn / 2;
         k += size_t(gridDim.x) * blockDim.x) {
      const unsigned i = unsigned(2 * k), l = i / un, row = i - l * un;
      const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(z16 + size_t(l) * ldh + row));
      const double2 zi = make_double2(double(hf.x), double(hf.y));
      reinterpret_cast<double2*>(z)[k] = zi;
      double2 a0 = make_double2(0.0, 0.0);
      if (d0) {
        a0 = reinterpret_cast<const double2*>(d0)[k];
        v[0] += zi.x * a0.x;
        v[0] += zi.y * a0.y;
      }
      if (d1a) {
        double2 a1 = same ? a0 : reinterpret_cast<const double2*>(d1a)[k];
        if (d1b) {
          const double2 b1 = reinterpret_cast<const double2*>(d1b)[k];
          a1.x -= b1.x, a1.y -= b1.y;
        }
        v[1] += zi.x * a1.x;
        v[1] += zi.y * a1.y;
      }
      if (!isfinite(zi.x)) v[2] += 1.0;
      if (!isfinite(zi.y)) v[2] += 1.0;
    }
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nn;
         i += size_t(gridDim.x) * blockDim.x) {
      const unsigned l = unsigned(i) / un, row = unsigned(i) - l * un;
      const double zi = double(__half2float(z16[size_t(l) * ldh + row]));
      z[i] = zi;
      if (d0) v[0] += zi * d0[i];
      if (d1a) v[1] += zi * (d1b ? d1a[i] - d1b[i] : d1a[i]);
      if (!isfinite(zi)) v[2] += 1.0;
    }
  }
  block_sum<3>(v, red);
  if (threadIdx.x == 0) {
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = v[0], o[1] = v[1], o[2] = v[2], o[3] = 0.0;
  }
}

// S(i,j) = 1 / ((s_r(j) s_c(i))^2 + lambda^2) at j*n + i (factor.cpp:62-76),
// unfused IEEE operations so it equals the host formula bit for bit; stored
// as FP64 or rounded once to binary16 (round_array of the FP64 weights).
__global__ void weights_kernel(const double* s_r, const double* s_c, int n, double l2,
                               double* s64, __half* s16) {
  pdl_wait();
  const size_t nn = size_t(n) * n;
  const unsigned un = unsigned(n);
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < nn;
       idx += size_t(gridDim.x) * blockDim.x) {
    const unsigned j = unsigned(idx / un), i = unsigned(idx - size_t(j) * un);
    const double prod = __dmul_rn(s_r[j], s_c[i]);
    const double w = __ddiv_rn(1.0, __dadd_rn(__dmul_rn(prod, prod), l2));
    if (s64) s64[idx] = w;
    if (s16) s16[idx] = __double2half(w);
  }
}

// ---------------------------------------------------------------------------
// PCG (pcg_core, krylov.cpp:58-142)
__global__ void pcg_init_scalar_kernel(DevState* st, DevHistory h, const double* part_r, int nr,
                                       const double* part_xt, int nxt) {
  pdl_wait();
  const int img = blockIdx.x;  // one block per image
  st += img, h = hist_of(h, img, 0), part_r += size_t(img) * nr * 4, part_xt += size_t(img) * nxt * 4;
  if (stopped(st)) return;
  const double rr = sum_partials(part_r, nr, 0);
  const double xx = st->has_xt ? sum_partials(part_xt, nxt, 0) : 0.0;
  if (threadIdx.x) return;
  if (st->has_xt && xx == 0.0) {  // solver: x_true must be nonzero
    st->status = ST_INVALID;
    return;
  }
  st->r0 = sqrt(rr);
  st->xnorm = sqrt(xx);
  h.resid[0] = st->r0;  // rec.row(0, x = 0, r0)
  if (st->has_xt) h.relerr[0] = st->xnorm / st->xnorm;
  st->rows = 1;
  st->iterations_used = 0;
  st->k = 1;
  if (st->r0 == 0.0) st->status = ST_CONVERGED;
}

__global__ void pcg_init_msolve_scalar_kernel(DevState* st, const double* part_z, int nz) {
  pdl_wait();
  st += blockIdx.x, part_z += size_t(blockIdx.x) * nz * 4;
  if (stopped(st)) return;
  const double rz = sum_partials(part_z, nz, 0);
  const double bad = sum_partials(part_z, nz, 2);
  if (threadIdx.x) return;
  st->msolve_count = 1;
  if (bad > 0.0) {
    st->status = ST_ABORTED, st->abort_code = AB_M_NONFINITE_INIT, st->abort_iter = 0;
    return;
  }
  st->rho = rz;
  if (!isfinite(rz) || rz <= 0.0)
    st->status = ST_ABORTED, st->abort_code = AB_POSITIVITY_INIT, st->abort_iter = 0;
}

// alpha = rho / p.q with the curvature checks (krylov.cpp:100-109); all
// threads get alpha, `writer` records it / the abort. False: aborted.
__device__ bool pcg_alpha_body(DevState* st, const double* part, int n, int T, bool writer, double& alpha) {
  const double pq = sum_slots(part, n, 0, T);
  if (!isfinite(pq)) {
    if (writer) st->status = ST_ABORTED, st->abort_code = AB_CURV_NONFINITE, st->abort_iter = st->k;
    return false;
  }
  if (pq <= 0.0) {
    if (writer) st->status = ST_ABORTED, st->abort_code = AB_CURV_BREAKDOWN, st->abort_iter = st->k;
    return false;
  }
  alpha = st->rho / pq;
  if (writer) st->alpha = alpha;
  return true;
}

__global__ void pcg_alpha_scalar_kernel(DevState* st, const double* part, int n) {
  pdl_wait();
  st += blockIdx.x, part += size_t(blockIdx.x) * n * 4;
  if (stopped(st)) return;
  double alpha;
  pcg_alpha_body(st, part, n, blockDim.x, threadIdx.x == 0, alpha);
}

// ||r||, history row, convergence / cap (krylov.cpp:113-126) from the
// pcg_update partials; thread 0 writes.
__device__ void pcg_resid_body(DevState* st, DevHistory h, const double* part, int n, int T) {
  const double rr = sum_slots(part, n, 0, T);
  const double ee = st->has_xt ? sum_slots(part, n, 1, T) : 0.0;
  const double rz = st->track_cos ? sum_slots(part, n, 2, T) : 0.0;
  const double zz = st->track_cos ? sum_slots(part, n, 3, T) : 0.0;
  if (threadIdx.x) return;
  const int k = st->k;
  const double rnorm = sqrt(rr);
  if (!isfinite(rnorm)) {
    st->status = ST_ABORTED, st->abort_code = AB_RESID_NONFINITE, st->abort_iter = k;
    return;
  }
  if (st->track_cos) {  // rec.cosine(r, z) (krylov.cpp:40-46)
    const double denom = rnorm * sqrt(zz);
    if (h.cosines) h.cosines[st->ncos] = denom > 0.0 ? fabs(rz) / denom : 0.0;
    st->ncos++;
  }
  const int row = st->rows;
  h.resid[row] = rnorm;
  if (st->has_xt) h.relerr[row] = sqrt(ee) / st->xnorm;
  st->rows = row + 1;
  st->iterations_used = k;
  if (rnorm <= st->tol * st->r0) {
    st->status = ST_CONVERGED;
    return;
  }
  if (k == st->maxit) st->status = ST_MAXIT;
}


// Elements are processed in pairs (16-byte vector accesses) when n is even
// and every pointer is 16-byte aligned (VEC2), else one at a time. Both
// elements of a pair lie in the same column, so the binary16 copy of r is a
// single half2 store into the padded B-operand layout (row l, ldh stride).
template <bool VEC2>
__global__ void __launch_bounds__(VEC_THREADS, 4) pcg_update_kernel(DevState* st, DevHistory h, double* x, double* r,
                                  double* r_prev, const double* p, const double* q,
                                  const double* z, const double* xt, __half* r16, int n,
                                  long ldh, double* part, const double* part_pq, int n_pq,
                                  int t_pq, int t_resid) {
  pdl_wait();
  {  // image blockIdx.y of a batch
    const int img = blockIdx.y;
    const size_t o = size_t(img) * n * n;
    st += img, h = hist_of(h, img, size_t(n) * n);
    x += o, r += o, p += o, q += o;
    if (r_prev) r_prev += o;
    if (z) z += o;
    if (xt) xt += o;
    if (r16) r16 += size_t(img) * n * ldh;
    part += size_t(img) * gridDim.x * 4;
    if (part_pq) part_pq += size_t(img) * n_pq * 4;
  }
  if (stopped(st)) return;
  __shared__ double red[VEC_THREADS / 32][4];
  double alpha;
  if (part_pq) {  // folded pcg_alpha_scalar: every CTA forms the same alpha
    if (!pcg_alpha_body(st, part_pq, n_pq, t_pq, blockIdx.x == 0 && threadIdx.x == 0, alpha)) return;
  } else {
    alpha = st->alpha;
  }
  const bool has_xt = st->has_xt, cos = st->track_cos;
  const unsigned un = unsigned(n);
  double* it = (st->record && h.iterates) ? h.iterates + size_t(st->rows) * n * n : nullptr;
  const size_t nn = size_t(n) * n;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (VEC2) {
    const size_t np = nn / 2;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < np;
         k += size_t(gridDim.x) * blockDim.x) {
      const size_t i = 2 * k;
      const double2 ri = reinterpret_cast<const double2*>(r)[k];
      const double2 pi = reinterpret_cast<const double2*>(p)[k];
      const double2 qi = reinterpret_cast<const double2*>(q)[k];
      double2 xi = reinterpret_cast<const double2*>(x)[k];
      if (r_prev) reinterpret_cast<double2*>(r_prev)[k] = ri;
      xi.x += alpha * pi.x, xi.y += alpha * pi.y;
      const double2 rn = make_double2(ri.x - alpha * qi.x, ri.y - alpha * qi.y);
      reinterpret_cast<double2*>(x)[k] = xi;
      reinterpret_cast<double2*>(r)[k] = rn;
      if (it) reinterpret_cast<double2*>(it)[k] = xi;
      if (r16) {
        const unsigned l = unsigned(i) / un, row = unsigned(i) - l * un;
        __half2 hv;
        hv.x = __double2half(rn.x);
        hv.y = __double2half(rn.y);
        *reinterpret_cast<__half2*>(r16 + size_t(l) * ldh + row) = hv;
      }
      v[0] += rn.x * rn.x;
      v[0] += rn.y * rn.y;
      if (has_xt) {
        const double2 ti = reinterpret_cast<const double2*>(xt)[k];
        const double d0 = xi.x - ti.x, d1 = xi.y - ti.y;
        v[1] += d0 * d0;
        v[1] += d1 * d1;
      }
      if (cos) {
        const double2 zi = reinterpret_cast<const double2*>(z)[k];
        v[2] += rn.x * zi.x;
        v[2] += rn.y * zi.y;
        v[3] += zi.x * zi.x;
        v[3] += zi.y * zi.y;
      }
    }
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nn;
         i += size_t(gridDim.x) * blockDim.x) {
      const double ri = r[i];
      if (r_prev) r_prev[i] = ri;
      const double xi = x[i] + alpha * p[i];
      const double rn = ri - alpha * q[i];
      x[i] = xi;
      r[i] = rn;
      if (it) it[i] = xi;
      if (r16) {
        const unsigned l = unsigned(i) / un, row = unsigned(i) - l * un;
        r16[size_t(l) * ldh + row] = __double2half(rn);
      }
      v[0] += rn * rn;
      if (has_xt) {
        const double d = xi - xt[i];
        v[1] += d * d;
      }
      if (cos) {
        const double zi = z[i];
        v[2] += rn * zi;
        v[3] += zi * zi;
      }
    }
  }
  block_sum<4>(v, red);
  if (threadIdx.x == 0) {
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = v[0], o[1] = v[1], o[2] = v[2], o[3] = v[3];
  }
  // folded pcg_resid_scalar: the last CTA reduces every CTA's partials
  if (t_resid && last_cta(st)) pcg_resid_body(st, h, part, gridDim.x, t_resid);
}

__global__ void pcg_resid_scalar_kernel(DevState* st, DevHistory h, const double* part, int n) {
  pdl_wait();
  st += blockIdx.x, h = hist_of(h, blockIdx.x, 0), part += size_t(blockIdx.x) * n * 4;
  if (stopped(st)) return;
  pcg_resid_body(st, h, part, n, blockDim.x);
}

// beta from the M-solve partials (krylov.cpp:127-132: z.r or z.(r - r_prev)
// over rho) with the non-finite checks; `writer` counts the M-solve and
// records beta / rz / the abort. False: aborted.
__device__ bool pcg_beta_body(DevState* st, const double* part, int n, int T, bool writer, double& beta,
                              double& rz) {
  rz = sum_slots(part, n, 0, T);
  const double zdr = sum_slots(part, n, 1, T);
  const double bad = sum_slots(part, n, 2, T);
  const int k = st->k;
  if (writer) st->msolve_count++;
  if (bad > 0.0) {
    if (writer) st->status = ST_ABORTED, st->abort_code = AB_M_NONFINITE, st->abort_iter = k;
    return false;
  }
  beta = st->flexible ? zdr / st->rho : rz / st->rho;
  if (!isfinite(beta) || !isfinite(rz)) {
    if (writer) st->status = ST_ABORTED, st->abort_code = AB_INNER_NONFINITE, st->abort_iter = k;
    return false;
  }
  if (writer) st->beta = beta, st->rz = rz;
  return true;
}

__global__ void pcg_beta_scalar_kernel(DevState* st, const double* part, int n) {
  pdl_wait();
  st += blockIdx.x, part += size_t(blockIdx.x) * n * 4;
  if (stopped(st)) return;
  double beta, rz;
  pcg_beta_body(st, part, n, blockDim.x, threadIdx.x == 0, beta, rz);
}

// rho = rz and the positivity check, then the next iteration (krylov.cpp:133-138)
__device__ void pcg_next_iteration(DevState* st, double rz) {
  st->rho = rz;
  if (st->rho <= 0.0) {
    st->status = ST_ABORTED, st->abort_code = AB_POSITIVITY, st->abort_iter = st->k;
    return;
  }
  st->k++;
}

// p = z + beta p, then the rho step. part_z: beta folded in (every CTA forms
// it from the M-solve partials; the rho step, which changes the rho those
// CTAs read, waits for the last CTA to finish).
__global__ void pcg_p_update_kernel(DevState* st, double* p, const double* z, size_t nn, bool vec2,
                                    const double* part_z, int nz, int t_z) {
  pdl_wait();
  st += blockIdx.y, p += blockIdx.y * nn, z += blockIdx.y * nn;  // image blockIdx.y of a batch
  if (stopped(st)) return;
  double beta, rz = 0.0;
  if (part_z) {
    if (!pcg_beta_body(st, part_z + size_t(blockIdx.y) * nz * 4, nz, t_z, blockIdx.x == 0 && threadIdx.x == 0,
                       beta, rz))
      return;
  } else {
    beta = st->beta;
  }
  if (vec2) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nn / 2;
         k += size_t(gridDim.x) * blockDim.x) {
      const double2 zi = reinterpret_cast<const double2*>(z)[k];
      double2 pi = reinterpret_cast<const double2*>(p)[k];
      pi.x = zi.x + beta * pi.x, pi.y = zi.y + beta * pi.y;
      reinterpret_cast<double2*>(p)[k] = pi;
    }
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nn;
         i += size_t(gridDim.x) * blockDim.x)
      p[i] = z[i] + beta * p[i];
  }
  if (part_z) {
    if (last_cta(st) && threadIdx.x == 0) pcg_next_iteration(st, rz);
    return;
  }
  // unfolded: by one thread once its share of p is done (no other CTA reads
  // rho or k; a CTA that starts after an abort skips its share of p, which
  // the stopped solve never reads again)
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  pcg_next_iteration(st, st->rz);
}

// ---------------------------------------------------------------------------
// CGLS (krylov.cpp:154-208)
__global__ void cgls_init_scalar_kernel(DevState* st, DevHistory h, const double* part_s, int ns,
                                        const double* part_xt, int nxt) {
  pdl_wait();
  if (stopped(st)) return;
  const double ss = sum_partials(part_s, ns, 0);
  const double xx = st->has_xt ? sum_partials(part_xt, nxt, 0) : 0.0;
  if (threadIdx.x) return;
  if (st->has_xt && xx == 0.0) {  // solver: x_true must be nonzero
    st->status = ST_INVALID;
    return;
  }
  st->r0 = sqrt(ss);
  st->xnorm = sqrt(xx);
  h.resid[0] = st->r0;
  if (st->has_xt) h.relerr[0] = st->xnorm / st->xnorm;
  st->rows = 1;
  st->iterations_used = 0;
  st->k = 1;
  st->gamma = ss;   // gamma = s.squaredNorm()
  st->pnorm2 = ss;  // p = s
  st->snorm_prev = st->r0;
  if (st->r0 == 0.0) st->status = ST_CONVERGED;
}

__global__ void cgls_alpha_scalar_kernel(DevState* st, const double* part_q, int nq,
                                         const double* part_p, int np) {
  pdl_wait();
  if (stopped(st)) return;
  const double qq = sum_partials(part_q, nq, 0);
  const double pp = (st->k > 1) ? sum_partials(part_p, np, 0) : 0.0;
  if (threadIdx.x) return;
  if (st->k > 1) st->pnorm2 = pp;
  const double delta = qq + st->l2 * st->pnorm2;
  if (!isfinite(delta)) {
    st->status = ST_ABORTED, st->abort_code = AB_CURV_NONFINITE, st->abort_iter = st->k;
    return;
  }
  if (delta == 0.0) {
    st->status = ST_ABORTED, st->abort_code = AB_CURV_BREAKDOWN, st->abort_iter = st->k;
    return;
  }
  st->alpha = st->gamma / delta;
}

template <bool VEC2>
__global__ void cgls_update_kernel(const DevState* st, DevHistory h, double* x, double* rt,
                                   const double* p, const double* q, const double* xt, size_t nn,
                                   double* part) {
  pdl_wait();
  if (stopped(st)) return;
  __shared__ double red[VEC_THREADS / 32][1];
  const double alpha = st->alpha;
  const bool has_xt = st->has_xt;
  double* it = (st->record && h.iterates) ? h.iterates + size_t(st->rows) * nn : nullptr;
  double v[1] = {0.0};
  if (VEC2) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nn / 2;
         k += size_t(gridDim.x) * blockDim.x) {
      const double2 pi = reinterpret_cast<const double2*>(p)[k];
      const double2 qi = reinterpret_cast<const double2*>(q)[k];
      double2 xi = reinterpret_cast<const double2*>(x)[k];
      double2 ri = reinterpret_cast<const double2*>(rt)[k];
      xi.x += alpha * pi.x, xi.y += alpha * pi.y;
      ri.x -= alpha * qi.x, ri.y -= alpha * qi.y;
      reinterpret_cast<double2*>(x)[k] = xi;
      reinterpret_cast<double2*>(rt)[k] = ri;
      if (it) reinterpret_cast<double2*>(it)[k] = xi;
      if (has_xt) {
        const double2 ti = reinterpret_cast<const double2*>(xt)[k];
        const double d0 = xi.x - ti.x, d1 = xi.y - ti.y;
        v[0] += d0 * d0;
        v[0] += d1 * d1;
      }
    }
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nn;
         i += size_t(gridDim.x) * blockDim.x) {
      const double xi = x[i] + alpha * p[i];
      x[i] = xi;
      rt[i] = rt[i] - alpha * q[i];
      if (it) it[i] = xi;
      if (has_xt) {
        const double d = xi - xt[i];
        v[0] += d * d;
      }
    }
  }
  block_sum<1>(v, red);
  if (threadIdx.x == 0) {
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = 0.0, o[1] = v[0], o[2] = 0.0, o[3] = 0.0;
  }
}

// part_s from the s = A^T rt - l2 x GEMM epilogue: [0] ||s||^2, [1] s.s_prev
__global__ void cgls_resid_scalar_kernel(DevState* st, DevHistory h, const double* part_s, int ns,
                                         const double* part_x, int nx) {
  pdl_wait();
  if (stopped(st)) return;
  const double ss = sum_partials(part_s, ns, 0);
  const double sp = st->track_cos ? sum_partials(part_s, ns, 1) : 0.0;
  const double ee = st->has_xt ? sum_partials(part_x, nx, 1) : 0.0;
  if (threadIdx.x) return;
  const int k = st->k;
  const double snorm = sqrt(ss);
  if (!isfinite(snorm)) {
    st->status = ST_ABORTED, st->abort_code = AB_RESID_NONFINITE, st->abort_iter = k;
    return;
  }
  if (st->track_cos) {  // rec.cosine(snew, s_prev)
    const double denom = snorm * st->snorm_prev;
    if (h.cosines) h.cosines[st->ncos] = denom > 0.0 ? fabs(sp) / denom : 0.0;
    st->ncos++;
  }
  const int row = st->rows;
  h.resid[row] = snorm;
  if (st->has_xt) h.relerr[row] = sqrt(ee) / st->xnorm;
  st->rows = row + 1;
  st->iterations_used = k;
  if (snorm <= st->tol * st->r0) {
    st->status = ST_CONVERGED;
    return;
  }
  const double beta = ss / st->gamma;
  st->beta = beta;
  st->gamma = ss;
  st->snorm_prev = snorm;
  if (k == st->maxit) {
    st->status = ST_MAXIT;
    return;
  }
}

template <bool VEC2>
__global__ void cgls_p_update_kernel(DevState* st, double* p, const double* s, double* s_prev,
                                     size_t nn, double* part) {
  pdl_wait();
  if (stopped(st)) return;
  __shared__ double red[VEC_THREADS / 32][1];
  const double beta = st->beta;
  double v[1] = {0.0};
  if (VEC2) {
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nn / 2;
         k += size_t(gridDim.x) * blockDim.x) {
      const double2 si = reinterpret_cast<const double2*>(s)[k];
      double2 pi = reinterpret_cast<const double2*>(p)[k];
      pi.x = si.x + beta * pi.x, pi.y = si.y + beta * pi.y;
      reinterpret_cast<double2*>(p)[k] = pi;
      if (s_prev) reinterpret_cast<double2*>(s_prev)[k] = si;
      v[0] += pi.x * pi.x;
      v[0] += pi.y * pi.y;
    }
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nn;
         i += size_t(gridDim.x) * blockDim.x) {
      const double si = s[i];
      const double pi = si + beta * p[i];
      p[i] = pi;
      if (s_prev) s_prev[i] = si;
      v[0] += pi * pi;
    }
  }
  block_sum<1>(v, red);
  if (threadIdx.x == 0) {
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = v[0], o[1] = 0.0, o[2] = 0.0, o[3] = 0.0;
  }
}
__global__ void cgls_next_kernel(DevState* st) {
  pdl_wait();
  if (stopped(st) || threadIdx.x) return;
  st->k++;
}

// ---------------------------------------------------------------------------
// Spectral sums (regparam.cpp:216-246). sigma(i,j) = s_r[j] * s_c[i] at
// linear index j*n + i; two sums per lambda (see SpectralKind in vec.cuh).
// LC lambdas per pass over b_hat (LC = 1 for the single-lambda probes of the
// root finders, 16 for grids).
template <int LC, int KIND>
__global__ void spectral_sums_kernel(const double* s_r, const double* s_c, const double* bhat,
                                     const double* xhat, int n, const double* lambdas, int m,
                                     double omega, double* part, const int* img_index) {
  pdl_wait();
  {  // batch row blockIdx.y: its own lambdas and partials; the coefficients of
     // image img_index[y] (or y)
    const size_t row = blockIdx.y, img = img_index ? size_t(img_index[row]) : row;
    bhat += img * size_t(n) * n;
    if (xhat) xhat += img * size_t(n) * n;
    lambdas += row * m;
    part += row * size_t(m) * gridDim.x * 2;
  }
  __shared__ double red[VEC_THREADS / 32][2 * LC];
  const size_t nn = size_t(n) * n;
  const unsigned un = unsigned(n);
  const double om1 = 1.0 - omega;
  for (int q0 = 0; q0 < m; q0 += LC) {
    double l2[LC];
    double v[2 * LC];
#pragma unroll
    for (int c = 0; c < LC; ++c) {
      const double l = (q0 + c < m) ? lambdas[q0 + c] : 1.0;
      l2[c] = l * l;
      v[2 * c] = 0.0, v[2 * c + 1] = 0.0;
    }
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < nn;
         idx += size_t(gridDim.x) * blockDim.x) {
      const unsigned j = unsigned(idx / un), i = unsigned(idx - size_t(j) * un);
      const double s = s_r[j] * s_c[i];
      const double s2 = s * s, b = bhat[idx];
      const double x = (KIND == SK_OPT) ? xhat[idx] : 0.0;
#pragma unroll
      for (int c = 0; c < LC; ++c) {
        const double d = s2 + l2[c];
        if (KIND == SK_GCV) {  // (b/d)^2, 1/d
          const double t = b / d;
          v[2 * c] += t * t;
          v[2 * c + 1] += 1.0 / d;
        } else if (KIND == SK_RESID) {  // (l^2 b/d)^2
          const double t = l2[c] * b / d;
          v[2 * c] += t * t;
        } else if (KIND == SK_OPT) {  // (s b/d - x)^2
          const double t = s * b / d - x;
          v[2 * c] += t * t;
        } else if (KIND == SK_WGCV) {  // (l^2 b/d)^2, ((1-w) s^2 + l^2)/d
          const double t = l2[c] * b / d;
          v[2 * c] += t * t;
          v[2 * c + 1] += (om1 * s2 + l2[c]) / d;
        } else {  // SK_WTRACE: ((1-w) s^2 + l^2)/d
          v[2 * c] += (om1 * s2 + l2[c]) / d;
        }
      }
    }
    block_sum<2 * LC>(v, red);
    if (threadIdx.x == 0)
      for (int c = 0; c < LC && q0 + c < m; ++c) {
        part[(size_t(q0 + c) * gridDim.x + blockIdx.x) * 2 + 0] = v[2 * c];
        part[(size_t(q0 + c) * gridDim.x + blockIdx.x) * 2 + 1] = v[2 * c + 1];
      }
    __syncthreads();
  }
}

// Tikhonov filter in place: c(i,j) = sigma / (sigma^2 + l2) * c(i,j)
// (regparam.cpp:329-349).
__global__ void spectral_filter_kernel(const double* s_r, const double* s_c, int n, double l2,
                                       double* c) {
  pdl_wait();
  const size_t nn = size_t(n) * n;
  const unsigned un = unsigned(n);
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < nn;
       idx += size_t(gridDim.x) * blockDim.x) {
    const unsigned j = unsigned(idx / un), i = unsigned(idx - size_t(j) * un);
    const double s = __dmul_rn(s_r[j], s_c[i]);
    const double den = __dadd_rn(__dmul_rn(s, s), l2);
    c[idx] = __dmul_rn(__ddiv_rn(s, den), c[idx]);
  }
}

// out[q*width + j] = sum over ctas of part[(q*ctas + cta)*width + j]; one
// block per q, fixed-order strided partial sums + tree (deterministic).
__global__ void finish_sums_kernel(const double* part, int ctas, int width, int m, double* out) {
  pdl_wait();
  __shared__ double red[VEC_THREADS / 32][1];
  const int q = blockIdx.x;
  if (q >= m) return;
  for (int j = 0; j < width; ++j) {
    double v[1] = {0.0};
    for (int c = threadIdx.x; c < ctas; c += blockDim.x) v[0] += part[(size_t(q) * ctas + c) * width + j];
    block_sum<1>(v, red);
    if (threadIdx.x == 0) out[size_t(q) * width + j] = v[0];
    __syncthreads();
  }
}

constexpr int LCHUNK = 16;

unsigned vec_grid(size_t nn) {
  return unsigned(std::min<size_t>(VEC_CTAS, std::max<size_t>(1, (nn + VEC_THREADS - 1) / VEC_THREADS)));
}

}  // namespace

// Host wrappers. The reducing vector kernels use VEC_CTAS CTAs (pcg_update:
// pcg_update_ctas(n), fewer at small n) so the reduction order is fixed for a
// given n; CTAs beyond the data simply contribute zero.
#define KP_LAUNCH(cls, kernel, grid, block, ...)                   \
  do {                                                             \
    LaunchScope scope_(cls);                                       \
    launch_pdl(kernel, dim3(grid), dim3(block), 0, __VA_ARGS__);   \
    check_launch(#kernel);                                         \
  } while (0)

namespace {
// Batch summary: out->status = ST_RUNNING while any image runs, else
// ST_CONVERGED (drives the host polling and gates the shared kernels).
__global__ void batch_status_kernel(const DevState* st, int count, DevState* out) {
  pdl_wait();
  __shared__ int running;
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < count; i += blockDim.x)
    if (st[i].status == ST_RUNNING) running = 1;
  __syncthreads();
  if (threadIdx.x == 0) out->status = running ? ST_RUNNING : ST_CONVERGED;
}

}  // namespace

void batch_status(const DevState* st, int count, DevState* out) {
  LaunchScope scope(KC_VECTOR);
  launch_pdl(batch_status_kernel, dim3(1), dim3(256), 0, st, count, out);
  check_launch("batch_status");
}

// Threads of a single-block scalar kernel summing `parts` partial slots: one
// slot per thread up to 1024 (a 32-slot sum needs one warp, not 32 — these
// kernels sit on every iteration's critical path at small n). A function of
// the slot counts only, so batched and single solves reduce identically.
static unsigned scalar_threads(int parts, int parts2 = 0) {
  const int p = parts > parts2 ? parts : parts2;
  unsigned t = 32;
  while (t < unsigned(p) && t < unsigned(SCALAR_THREADS)) t <<= 1;
  return t;
}

void vec_copy(double* dst, const double* src, size_t n, const int* status) {
  KP_LAUNCH(KC_VECTOR, copy_kernel, vec_grid(n), VEC_THREADS, dst, src, n, status);
}
void precond_weights(const double* s_r, const double* s_c, int n, double l2, double* s64,
                     __half* s16) {
  KP_LAUNCH(KC_PRECOND, weights_kernel, vec_grid(size_t(n) * n), VEC_THREADS, s_r, s_c, n, l2, s64,
            s16);
}
void vec_zero(double* dst, size_t n) {
  KP_LAUNCH(KC_VECTOR, zero_kernel, vec_grid(n), VEC_THREADS, dst, n);
}
void vec_dot_partials(const double* x, const double* y, size_t n, double* partials) {
  KP_LAUNCH(KC_VECTOR, dot_partials_kernel, VEC_CTAS, VEC_THREADS, x, y, n, partials);
}
void cast_f64_to_f16_padded(const double* src, __half* dst, int rows, int cols, long ld_src,
                            long ld_dst, const int* status) {
  KP_LAUNCH(KC_VECTOR, cast_f16_kernel, vec_grid(size_t(rows) * cols), VEC_THREADS, src, dst,
            rows, cols, ld_src, ld_dst, status);
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void msolve_finish_f16(const __half* z16, long ldh, int n, double* z, const double* d0,
                       const double* d1a, const double* d1b, double* partials,
                       const int* status, int batch) {
  const bool vec2 = n % 2 == 0 && ldh % 2 == 0 && al16(z) && al16(d0) && al16(d1a) && al16(d1b);
  const dim3 grid(VEC_CTAS, batch);
  if (vec2)
    KP_LAUNCH(KC_VECTOR, msolve_finish_f16_kernel<true>, grid, VEC_THREADS, z16, ldh, n, z, d0,
              d1a, d1b, partials, status);
  else
    KP_LAUNCH(KC_VECTOR, msolve_finish_f16_kernel<false>, grid, VEC_THREADS, z16, ldh, n, z,
              d0, d1a, d1b, partials, status);
}

void pcg_init_scalar(DevState* st, DevHistory h, const double* part_r, int nr,
                     const double* part_xt, int nxt, int batch) {
  KP_LAUNCH(KC_VECTOR, pcg_init_scalar_kernel, batch, scalar_threads(nr, nxt), st, h, part_r, nr, part_xt, nxt);
}
void pcg_init_msolve_scalar(DevState* st, const double* part_z, int nz, int batch) {
  KP_LAUNCH(KC_VECTOR, pcg_init_msolve_scalar_kernel, batch, scalar_threads(nz), st, part_z, nz);
}
void pcg_alpha_scalar(DevState* st, const double* part_pq, int n, int batch) {
  KP_LAUNCH(KC_VECTOR, pcg_alpha_scalar_kernel, batch, scalar_threads(n), st, part_pq, n);
}

bool pcg_fold_ok(int slots) { return scalar_threads(slots) <= unsigned(VEC_THREADS); }

int pcg_update_ctas(int n) {
  // one pair (or element) per thread at most; the fixed VEC_CTAS from n ~ 1560 up
  const size_t units = (n % 2 == 0) ? size_t(n) * n / 2 : size_t(n) * n;
  return int(vec_grid(units));
}
void pcg_update(DevState* st, DevHistory h, double* x, double* r, double* r_prev, const double* p,
                const double* q, const double* z, const double* xt, __half* r16, int n, long ldh,
                double* partials, int batch, const double* part_pq, int n_pq, bool fold_resid) {
  const bool vec2 = n % 2 == 0 && al16(x) && al16(r) && al16(r_prev) && al16(p) && al16(q) &&
                    al16(z) && al16(xt) && al16(h.iterates) && ldh % 2 == 0;
  const int ctas = pcg_update_ctas(n);
  const dim3 grid(ctas, batch);
  if ((part_pq && !pcg_fold_ok(n_pq)) || (fold_resid && !pcg_fold_ok(ctas)))
    throw std::logic_error("pcg_update: scalar step too wide to fold");
  const int t_pq = part_pq ? int(scalar_threads(n_pq)) : 0, t_resid = fold_resid ? int(scalar_threads(ctas)) : 0;
  if (vec2)
    KP_LAUNCH(KC_VECTOR, pcg_update_kernel<true>, grid, VEC_THREADS, st, h, x, r, r_prev, p, q,
              z, xt, r16, n, ldh, partials, part_pq, n_pq, t_pq, t_resid);
  else
    KP_LAUNCH(KC_VECTOR, pcg_update_kernel<false>, grid, VEC_THREADS, st, h, x, r, r_prev, p,
              q, z, xt, r16, n, ldh, partials, part_pq, n_pq, t_pq, t_resid);
}
void pcg_resid_scalar(DevState* st, DevHistory h, const double* part, int n, int batch) {
  KP_LAUNCH(KC_VECTOR, pcg_resid_scalar_kernel, batch, scalar_threads(n), st, h, part, n);
}
void pcg_beta_scalar(DevState* st, const double* part_z, int n, int batch) {
  KP_LAUNCH(KC_VECTOR, pcg_beta_scalar_kernel, batch, scalar_threads(n), st, part_z, n);
}
void pcg_p_update(DevState* st, double* p, const double* z, size_t nn, int batch, const double* part_z,
                  int nz) {
  const bool vec2 = nn % 2 == 0 && al16(p) && al16(z);
  if (part_z && !pcg_fold_ok(nz)) throw std::logic_error("pcg_p_update: scalar step too wide to fold");
  KP_LAUNCH(KC_VECTOR, pcg_p_update_kernel, dim3(vec_grid(nn), batch), VEC_THREADS, st, p, z, nn, vec2,
            part_z, nz, part_z ? int(scalar_threads(nz)) : 0);
}

void cgls_init_scalar(DevState* st, DevHistory h, const double* part_s, int ns,
                      const double* part_xt, int nxt) {
  KP_LAUNCH(KC_VECTOR, cgls_init_scalar_kernel, 1, scalar_threads(ns, nxt), st, h, part_s, ns, part_xt, nxt);
}
void cgls_alpha_scalar(DevState* st, const double* part_q, int nq, const double* part_p, int np) {
  KP_LAUNCH(KC_VECTOR, cgls_alpha_scalar_kernel, 1, scalar_threads(nq, np), st, part_q, nq, part_p, np);
}
void cgls_update(DevState* st, DevHistory h, double* x, double* rt, const double* p,
                 const double* q, const double* xt, size_t nn, double* partials) {
  if (nn % 2 == 0 && al16(x) && al16(rt) && al16(p) && al16(q) && al16(xt) && al16(h.iterates))
    KP_LAUNCH(KC_VECTOR, cgls_update_kernel<true>, VEC_CTAS, VEC_THREADS, st, h, x, rt, p, q, xt,
              nn, partials);
  else
    KP_LAUNCH(KC_VECTOR, cgls_update_kernel<false>, VEC_CTAS, VEC_THREADS, st, h, x, rt, p, q, xt,
              nn, partials);
}
void cgls_resid_scalar(DevState* st, DevHistory h, const double* part_s, int ns,
                       const double* part_x, int nx) {
  KP_LAUNCH(KC_VECTOR, cgls_resid_scalar_kernel, 1, scalar_threads(ns, nx), st, h, part_s, ns, part_x, nx);
}
void cgls_p_update(DevState* st, double* p, const double* s, double* s_prev, size_t nn,
                   double* partials) {
  if (nn % 2 == 0 && al16(p) && al16(s) && al16(s_prev))
    KP_LAUNCH(KC_VECTOR, cgls_p_update_kernel<true>, VEC_CTAS, VEC_THREADS, st, p, s, s_prev, nn,
              partials);
  else
    KP_LAUNCH(KC_VECTOR, cgls_p_update_kernel<false>, VEC_CTAS, VEC_THREADS, st, p, s, s_prev, nn,
              partials);
  KP_LAUNCH(KC_VECTOR, cgls_next_kernel, 1, 32, st);
}

void spectral_filter(const double* s_r, const double* s_c, int n, double l2, double* c) {
  KP_LAUNCH(KC_SPECTRAL, spectral_filter_kernel, vec_grid(size_t(n) * n), VEC_THREADS, s_r, s_c, n,
            l2, c);
}

template <int KIND>
void launch_sums(const double* s_r, const double* s_c, const double* bhat, const double* xhat,
                 int n, const double* lambdas, int m, double omega, double* part, int batch,
                 const int* img_index) {
  // lambdas per pass: 1, 4 (the discrepancy look-ahead's 3) or LCHUNK; every
  // value is summed in the same element order whatever the width
  const dim3 grid(VEC_CTAS, batch);
  if (m == 1)
    KP_LAUNCH(KC_SPECTRAL, (spectral_sums_kernel<1, KIND>), grid, VEC_THREADS, s_r, s_c, bhat,
              xhat, n, lambdas, m, omega, part, img_index);
  else if (m <= 4)
    KP_LAUNCH(KC_SPECTRAL, (spectral_sums_kernel<4, KIND>), grid, VEC_THREADS, s_r, s_c, bhat,
              xhat, n, lambdas, m, omega, part, img_index);
  else
    KP_LAUNCH(KC_SPECTRAL, (spectral_sums_kernel<LCHUNK, KIND>), grid, VEC_THREADS, s_r, s_c,
              bhat, xhat, n, lambdas, m, omega, part, img_index);
}

void spectral_sums(int kind, const double* s_r, const double* s_c, const double* bhat,
                   const double* xhat, int n, const double* lambdas, int m, double omega,
                   double* out, int batch, const int* img_index) {
  DBuf<double> part(size_t(batch) * m * VEC_CTAS * 2);
  switch (kind) {
    case SK_GCV: launch_sums<SK_GCV>(s_r, s_c, bhat, xhat, n, lambdas, m, omega, part.p, batch, img_index); break;
    case SK_RESID: launch_sums<SK_RESID>(s_r, s_c, bhat, xhat, n, lambdas, m, omega, part.p, batch, img_index); break;
    case SK_OPT: launch_sums<SK_OPT>(s_r, s_c, bhat, xhat, n, lambdas, m, omega, part.p, batch, img_index); break;
    case SK_WGCV: launch_sums<SK_WGCV>(s_r, s_c, bhat, xhat, n, lambdas, m, omega, part.p, batch, img_index); break;
    case SK_WTRACE: launch_sums<SK_WTRACE>(s_r, s_c, bhat, xhat, n, lambdas, m, omega, part.p, batch, img_index); break;
    default: throw InvalidArgument("spectral_sums: bad kind");
  }
  // one finishing block per (image, lambda) row, in the same fixed order
  KP_LAUNCH(KC_SPECTRAL, finish_sums_kernel, batch * m, VEC_THREADS, part.p, VEC_CTAS, 2, batch * m, out);
}

}  // namespace kp
