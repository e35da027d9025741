// Emulated low-precision arithmetic for any PrecisionFormat (see
// lp_generic.cuh). Every operation follows the reference's FP64 order: the
// product or pairwise sum is formed in double (IEEE round-to-nearest), then
// rounded to the format, exactly as round_inplace does on the materialised
// arrays (lpblas.cpp:13-70).
#include "lp_generic.cuh"

#include <math_constants.h>

namespace kp {
namespace {

// round_value (precision.cpp:15-41, 82-86): nearest representable value,
// ties to even; infinities, NaN and zeros pass through.
__device__ __forceinline__ double lp_round(double x, const LpFormat& f) {
  if (f.t >= 53 && f.emax >= 1023 && f.sub) return x;
  if (!isfinite(x) || x == 0.0) return x;
  const int t = f.t, emin = 1 - f.emax;
  const double mag = fabs(x);
  const double threshold = ldexp(2.0 - ldexp(1.0, -t), f.emax);  // overflow_threshold()
  if (mag >= threshold) return copysign(CUDART_INF, x);
  const int e = ilogb(mag);
  const int shift = e < emin ? (f.sub ? emin - t + 1 : emin) : e - t + 1;
  const double r = ldexp(rint(ldexp(x, -shift)), shift);  // rint: ties to even
  return r == 0.0 ? copysign(0.0, x) : r;
}

__global__ void round_kernel(const double* x, size_t count, LpFormat f, double* out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = lp_round(x[i], f);
}

constexpr int TI = 32, TJ = 8, TK = 32, MAXLVL = 40;

// One output per thread; operand tiles staged through shared memory along
// whichever dimension is contiguous. The pairwise tree is a binary counter
// over the leaves (local-memory stack), merged bottom-up at the end — the
// stage tree of pairwise_block_reduce with its carried odd tails.
__global__ void __launch_bounds__(TI * TJ) lp_gemm_kernel(const LpGemmArgs g) {
  if (g.status && *g.status) return;
  __shared__ double as[TK][TI + 1];
  __shared__ double bs[TK][TJ + 1];
  const int tx = threadIdx.x, ty = threadIdx.y, l = ty * TI + tx;
  const int i0 = blockIdx.x * TI, j0 = blockIdx.y * TJ;
  const int i = i0 + tx, j = j0 + ty;
  const bool live = !g.f.covers_double();
  double st[MAXLVL];
  unsigned long long cnt = 0;
  for (int k0 = 0; k0 < g.K; k0 += TK) {
#pragma unroll
    for (int rep = 0; rep < (TI * TK) / (TI * TJ); ++rep) {
      const int q = l + rep * TI * TJ;
      int ii, kk;
      if (g.ai == 1) ii = q % TI, kk = q / TI;
      else kk = q % TK, ii = q / TK;
      const int gi = i0 + ii, gk = k0 + kk;
      as[kk][ii] = (gi < g.M && gk < g.K) ? g.a[long(gi) * g.ai + long(gk) * g.ak] : 0.0;
    }
    {
      int kk, jj;
      if (g.bk == 1) kk = l % TK, jj = l / TK;
      else jj = l % TJ, kk = l / TJ;
      const int gj = j0 + jj, gk = k0 + kk;
      bs[kk][jj] = (gj < g.N && gk < g.K) ? g.b[long(gk) * g.bk + long(gj) * g.bj] : 0.0;
    }
    __syncthreads();
    const int kn = min(TK, g.K - k0);
    for (int kk = 0; kk < kn; ++kk) {
      double v = as[kk][tx] * bs[kk][ty];
      if (live && g.round_leaves) v = lp_round(v, g.f);
      int lvl = 0;
      unsigned long long c = cnt;
      while (c & 1ull) {
        v = st[lvl] + v;
        if (live) v = lp_round(v, g.f);
        ++lvl;
        c >>= 1;
      }
      st[lvl] = v;
      ++cnt;
    }
    __syncthreads();
  }
  if (i >= g.M || j >= g.N) return;
  double acc = 0.0;
  bool have = false;
  for (int L = 0; L < MAXLVL; ++L) {
    if (!((cnt >> L) & 1ull)) continue;
    if (have) {
      acc = st[L] + acc;
      if (live) acc = lp_round(acc, g.f);
    } else {
      acc = st[L];
      have = true;
    }
  }
  if (g.scale) {
    acc = g.scale[long(i) + long(j) * g.ls] * acc;
    if (live) acc = lp_round(acc, g.f);
  }
  g.c[long(i) + long(j) * g.ldc] = acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__global__ void partials_kernel(const double* z, size_t count, const double* d0, const double* d1a,
                                const double* d1b, double* part, const int* status) {
  if (status && *status) return;
  __shared__ double red[8][3];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    const double v = z[i];
    if (d0) s0 += v * d0[i];
    if (d1a) s1 += v * (d1b ? d1a[i] - d1b[i] : d1a[i]);
    if (!isfinite(v)) s2 += 1.0;
  }
  s0 = warp_sum(s0), s1 = warp_sum(s1), s2 = warp_sum(s2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp][0] = s0, red[warp][1] = s1, red[warp][2] = s2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) a0 += red[w][0], a1 += red[w][1], a2 += red[w][2];
    double* o = part + size_t(blockIdx.x) * 4;
    o[0] = a0, o[1] = a1, o[2] = a2, o[3] = 0.0;
  }
}

__global__ void count_not_f16_kernel(const double* x, size_t count, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    const double v = x[i];
    if (!(double(__half2float(__double2half(v))) == v)) ++c;
  }
  if (c) atomicAdd(out, c);
}

__global__ void pack_f16_kernel(const double* src, long rs, long cs, int rows, int cols,
                                __half* dst, long ld, uint16_t pad) {
  const size_t total = size_t(rows) * ld;
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const long r = long(idx / ld), c = long(idx % ld);
    dst[idx] = c < cols ? __double2half(src[r * rs + c * cs]) : __ushort_as_half(pad);
  }
}

unsigned grid_for(size_t count) {
  return unsigned(std::min<size_t>(148 * 8, std::max<size_t>(1, (count + 255) / 256)));
}

}  // namespace

void lp_round_array(const double* x, size_t count, LpFormat f, double* out, int kernel_class) {
  if (!count) return;
  LaunchScope scope(kernel_class);
  round_kernel<<<grid_for(count), 256, 0, ctx().stream>>>(x, count, f, out);
  check_launch("lp_round_array");
}

void lp_gemm_generic(const LpGemmArgs& g, int kernel_class) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.K <= 0) throw InvalidArgument("lp_matmul: empty input");
  LaunchScope scope(kernel_class);
  const dim3 grid(unsigned((g.M + TI - 1) / TI), unsigned((g.N + TJ - 1) / TJ));
  lp_gemm_kernel<<<grid, dim3(TI, TJ), 0, ctx().stream>>>(g);
  check_launch("lp_gemm_generic");
}

void lp_vector_partials(const double* z, size_t count, const double* d0, const double* d1a,
                        const double* d1b, double* part, const int* status, int kernel_class) {
  LaunchScope scope(kernel_class);
  partials_kernel<<<LP_PART_CTAS, 256, 0, ctx().stream>>>(z, count, d0, d1a, d1b, part, status);
  check_launch("lp_vector_partials");
}

long long count_not_f16(const double* x, size_t count) {
  DBuf<unsigned long long> c(1);
  KP_CUDA(cudaMemsetAsync(c.p, 0, sizeof(unsigned long long), ctx().stream));
  {
    LaunchScope scope(KC_PRECOND);
    count_not_f16_kernel<<<grid_for(count), 256, 0, ctx().stream>>>(x, count, c.p);
    check_launch("count_not_f16");
  }
  unsigned long long h = 0;
  c.download(&h, 1);
  KP_CUDA(cudaStreamSynchronize(ctx().stream));
  return (long long)h;
}

void pack_f16(const double* src, long rs, long cs, int rows, int cols, __half* dst, long ld,
              uint16_t pad) {
  LaunchScope scope(KC_PRECOND);
  pack_f16_kernel<<<grid_for(size_t(rows) * ld), 256, 0, ctx().stream>>>(src, rs, cs, rows, cols,
                                                                        dst, ld, pad);
  check_launch("pack_f16");
}

}  // namespace kp
