// Banded-Toeplitz Kronecker-sum operator: A x = vec(sum_k A_c^k X A_r^kT)
// when every factor is a banded Toeplitz matrix (banded_toeplitz,
// deblur.cpp:157-165 — the structure psf_to_kronsum always produces).
//
// The dense product the reference computes (kron.cpp:69-70) multiplies by
// the zeros outside the band; here each term is two 1-D correlations with
// the factor's diagonal values:
//   pass A (band_cols): Y_k(a, l) = sum_u wc_k[u] X(a + sc + u, l)   (all k)
//   pass B (band_rows): out(a, j) = sum_k sum_u wr_k[u] Y_k(a, j + sr + u)
// with zero boundary conditions (rows / columns outside [0, n) are zero), so
// the result equals the dense product up to the FP64 summation order. The
// transpose uses the reversed taps. Work per apply: 2 r (Lc + Lr) n^2 flop
// (C5: 1.4e10 vs 1.4e12 dense) on the FP64 (DFMA) pipe.
//
// Both passes keep the taps in the kernel-parameter constant bank (uniform
// operands of DFMA), stage a halo tile in shared memory, and register-tile 8
// consecutive outputs per thread along the correlation axis, so every new
// shared-memory value feeds 8 DFMAs. Tile strides are odd (in doubles) so
// lanes walking different columns never share a bank.
#include "banded.cuh"

#include <cstdlib>

namespace kp {
namespace {

constexpr int A_TA = 64, A_TL = 32, A_THREADS = 256;    // pass A tile: 64 rows x 32 cols
constexpr int B_TA = 32, B_TJ = 64, B_THREADS = 256;    // pass B tile: 32 rows x 64 cols

__device__ __forceinline__ bool stopped(const int* status) { return status && *status != 0; }

// 8-wide register-tiled correlation: acc[q] += sum_u w[u] * src(q + u), where
// src(i) = base[i * stride]; taps is a multiple of 8.
template <typename Src>
__device__ __forceinline__ void corr8(double (&acc)[8], const double* w, int taps, Src src) {
  double x[16];
#pragma unroll
  for (int v = 0; v < 8; ++v) x[v] = src(v);
  for (int u0 = 0; u0 < taps; u0 += 8) {
#pragma unroll
    for (int v = 0; v < 8; ++v) x[8 + v] = src(u0 + 8 + v);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double wv = w[u0 + v];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(wv, x[q + v], acc[q]);
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = x[8 + v];
  }
}

// corr8 over the actual tap count: full blocks of 8, then the remaining
// taps % 8 one at a time (no DFMAs on the zero padding). Used by pass B,
// where it is faster; pass A keeps the padded loop (fewer registers).
// Reads src up to index taps + 7.
template <typename Src>
__device__ __forceinline__ void corr8_tail(double (&acc)[8], const double* w, int taps, Src src) {
  double x[16];
#pragma unroll
  for (int v = 0; v < 8; ++v) x[v] = src(v);
  const int full = taps & ~7;
  for (int u0 = 0; u0 < full; u0 += 8) {
#pragma unroll
    for (int v = 0; v < 8; ++v) x[8 + v] = src(u0 + 8 + v);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double wv = w[u0 + v];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(wv, x[q + v], acc[q]);
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = x[8 + v];
  }
  for (int v = full; v < taps; ++v) {  // x[0..7] = src(v .. v + 7)
    const double wv = w[v];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(wv, x[q], acc[q]);
#pragma unroll
    for (int q = 0; q < 7; ++q) x[q] = x[q + 1];
    x[7] = src(v + 8);
  }
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
}

// Compile-time tap count: fully unrolled, exact taps (no zero padding), the
// 8-value window kept as a register ring (src(i) in slot i % 8, refilled
// right after its last use), weights as constant-bank DFMA operands.
// Reads src(0 .. TAPS + 6).
template <int TAPS, typename Src>
__device__ __forceinline__ void corr8_fixed(double (&acc)[8], const double* w, Src src) {
  double ring[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) ring[v] = src(v);
#pragma unroll
  for (int u = 0; u < TAPS; ++u) {
    const double wv = w[u];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(wv, ring[(u + q) & 7], acc[q]);
    if (u + 8 <= TAPS + 6) ring[u & 7] = src(u + 8);
  }
}

// Compile-time tap count with the register footprint of corr8 (pass A keeps
// 4 CTAs per SM; the fully unrolled form hoists every load and drops to 2):
// runtime loop over the full 8-tap blocks, then the TAPS % 8 remaining taps
// unrolled with compile-time window indices. Reads src(0 .. TAPS + 6).
template <int TAPS, typename Src>
__device__ __forceinline__ void corr8_blocks(double (&acc)[8], const double* w, Src src) {
  constexpr int FULL = TAPS & ~7, TAIL = TAPS & 7;
  double x[16];
#pragma unroll
  for (int v = 0; v < 8; ++v) x[v] = src(v);
#pragma unroll 1
  for (int u0 = 0; u0 < FULL; u0 += 8) {
#pragma unroll
    for (int v = 0; v < 8; ++v) x[8 + v] = src(u0 + 8 + v);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double wv = w[u0 + v];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(wv, x[q + v], acc[q]);
    }
#pragma unroll
    for (int v = 0; v < 8; ++v) x[v] = x[8 + v];
  }
  if constexpr (TAIL > 0) {
#pragma unroll
    for (int v = 0; v + 1 < TAIL; ++v) x[8 + v] = src(FULL + 8 + v);
#pragma unroll
    for (int v = 0; v < TAIL; ++v) {
      const double wv = w[FULL + v];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(wv, x[q + v], acc[q]);
    }
  }
}

// TAPS > 0: kernels specialised for that exact tap count (the BASELINE PSF
// supports); TAPS == 0: runtime tap count, padded to a multiple of 8.
template <int TAPS>
__host__ __device__ constexpr int cols_stride(int padded_taps) {
  return (A_TA + (TAPS > 0 ? TAPS - 1 : padded_taps)) | 1;  // odd; generic keeps corr8's slack
}
template <int TAPS>
__host__ __device__ constexpr int rows_halo(int padded_taps) {
  return TAPS > 0 ? B_TJ + TAPS - 1 : B_TJ + padded_taps;  // generic: +1 row corr8 slack
}

constexpr int A_SO = A_TA + 2;  // staged output tile stride: 16-byte aligned, conflict-free 128-bit accesses
#ifndef KP_BAND_A_MINB
#define KP_BAND_A_MINB 4
#endif
template <int TAPS>
__global__ void __launch_bounds__(A_THREADS, KP_BAND_A_MINB) band_cols_kernel(const double* __restrict__ X,
                                                              double* __restrict__ Y, int n, int r,
                                                              const __grid_constant__ BandTaps t,
                                                              const int* status) {
  pdl_wait();
  if (stopped(status)) return;
  extern __shared__ double sm[];
  X += size_t(blockIdx.z) * n * n;  // batched images (grid.z)
  Y += size_t(blockIdx.z) * r * n * n;
  const int S = cols_stride<TAPS>(t.taps);  // odd column stride (no bank sharing across lanes)
  double* Xs = sm;                          // [A_TL][S]
  const int a0 = blockIdx.y * A_TA, l0 = blockIdx.x * A_TL;
  {  // halo tile: warp w copies columns w, w + 8, ..; lanes walk the rows (coalesced)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int vmax = A_TA + (TAPS > 0 ? TAPS : t.taps) - 1;  // rows with data, zeros beyond
    const uint32_t xs = static_cast<uint32_t>(__cvta_generic_to_shared(Xs));
    for (int c = warp; c < A_TL; c += A_THREADS / 32) {
      const int l = l0 + c;
      const double* col = X + size_t(l) * n;  // dereferenced only when l < n
      for (int v = lane; v < S; v += 32) {
        const int i = a0 + t.shift + v;
        const bool ok = l < n && v < vmax && i >= 0 && i < n;
        cp_async8(xs + uint32_t(c * S + v) * 8u, ok ? col + i : X, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t nn = size_t(n) * n;
  const bool vec = (n & 1) == 0;
  // Each thread's 8 outputs are 8 rows of one column (lanes = 32 columns), so
  // storing them straight from registers touches 32 lines per instruction.
  // Instead the Y_k tile goes through shared memory ([A_TL][A_SO]) and each
  // warp stores whole 512-byte column runs.
  double* Ys = Xs + A_TL * S;
  for (int k = 0; k < r; ++k) {
#pragma unroll
    for (int h = 0; h < A_TA / 8 / (A_THREADS / 32); ++h) {
      const int b = warp + h * (A_THREADS / 32);  // 8-row block
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const double* base = Xs + lane * S + 8 * b;
      if constexpr (TAPS > 0)
        corr8_blocks<TAPS>(acc, t.w[k], [&](int i) { return base[i]; });
      else
        corr8(acc, t.w[k], t.taps, [&](int i) { return base[i]; });
#pragma unroll
      for (int q = 0; q < 8; q += 2)
        *reinterpret_cast<double2*>(Ys + lane * A_SO + 8 * b + q) = make_double2(acc[q], acc[q + 1]);
    }
    __syncthreads();
    double* Yk = Y + k * nn;
    if (vec) {  // a warp stores one column: 32 lanes x 2 rows
#pragma unroll
      for (int it = 0; it < A_TL * A_TA / 2 / A_THREADS; ++it) {
        const int idx = threadIdx.x + it * A_THREADS;
        const int c = idx / (A_TA / 2), pr = 2 * (idx % (A_TA / 2));
        const int lc = l0 + c, a = a0 + pr;
        if (lc < n && a < n)
          *reinterpret_cast<double2*>(Yk + size_t(lc) * n + a) =
              *reinterpret_cast<const double2*>(Ys + c * A_SO + pr);
      }
    } else {
      for (int idx = threadIdx.x; idx < A_TL * A_TA; idx += A_THREADS) {
        const int c = idx / A_TA, rr = idx % A_TA;
        const int lc = l0 + c, a = a0 + rr;
        if (lc < n && a < n) Yk[size_t(lc) * n + a] = Ys[c * A_SO + rr];
      }
    }
    __syncthreads();  // Ys is rewritten by the next term
  }
}

// Pass B. The Y_k tiles (B_TJ + taps - 1 columns of B_TA rows) are
// double-buffered with cp.async so term k+1 streams in while term k's
// correlation runs.
template <int TAPS, bool BATCH>
// 41 taps (C5): held to 64 registers (4 CTAs / SM; unconstrained, the
// batched epilogue's pointers took it to 82 and 2 CTAs / SM: 0.28 -> 0.38 ms
// per pass); the shorter bands measured best unconstrained (min blocks 0 =
// no occupancy target: 64 / 64 / 55 registers at 31 / 19 / 17 taps, where
// a target of 1 let ptxas take 85).
__global__ void __launch_bounds__(B_THREADS, TAPS == 41 ? 4 : 0) band_rows_kernel(const double* __restrict__ Y, int n,
                                                              int r, const __grid_constant__ BandTaps t,
                                                              const F64Epilogue e,
                                                              const int* status) {
  pdl_wait();
  if (stopped(status)) return;
  extern __shared__ double sm[];
  if (BATCH) Y += size_t(blockIdx.z) * r * n * n;  // batched images (grid.z)
  const int rows = (TAPS > 0 ? TAPS : t.taps) + B_TJ - 1;  // rows loaded
  const int buf_doubles = rows_halo<TAPS>(t.taps) * B_TA;
  const int a0 = blockIdx.y * B_TA, j0 = blockIdx.x * B_TJ;
  const int a = threadIdx.x % B_TA, jq = threadIdx.x / B_TA;  // jq in [0, 8): 8-column block
  const size_t nn = size_t(n) * n;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const bool vec = (n & 1) == 0;  // 16-byte copies (pairs of rows) when n is even
  // Copy plan of the 16-byte path, computed once: thread -> row pair aa,
  // tile columns jw0 + 16 it (it < PLAN); per term only the base moves.
  constexpr int PAIRS = B_TA / 2, STEP = B_THREADS / PAIRS;
  constexpr int PLAN = (B_TJ + (TAPS > 0 ? TAPS - 1 : BAND_MAX_TAPS) + STEP - 1) / STEP;
  static_assert(B_THREADS % PAIRS == 0, "copy plan");
  const int aa = 2 * (threadIdx.x % PAIRS), jw0 = threadIdx.x / PAIRS;
  uint32_t in_tile = 0, in_range = 0;
#pragma unroll
  for (int it = 0; it < PLAN; ++it) {
    const int jw = jw0 + STEP * it, j = j0 + t.shift + jw;
    if (jw < rows) in_tile |= 1u << it;
    if (jw < rows && j >= 0 && j < n && a0 + aa < n) in_range |= 1u << it;
  }
  const long goff0 = (long(j0 + t.shift + jw0) * n + a0 + aa) * long(sizeof(double));
  const long gstep = long(STEP) * n * long(sizeof(double));
  const uint32_t soff0 = uint32_t(jw0 * B_TA + aa) * 8u;
  auto load = [&](int k, int buf) {
    const double* Yk = Y + k * nn;
    const uint32_t dst0 = sbase + uint32_t(buf * buf_doubles) * 8u;
    if (vec) {
      const char* g = reinterpret_cast<const char*>(Yk) + goff0;  // tile column jw0 (may be outside Y)
      const uint32_t d = dst0 + soff0;
#pragma unroll
      for (int it = 0; it < PLAN; ++it) {
        if (in_tile & (1u << it)) {
          const bool v = in_range & (1u << it);
          const char* src = g + it * gstep;
          cp_async16(d + uint32_t(it * STEP * B_TA * 8), v ? src : reinterpret_cast<const char*>(Y), v);
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < rows * B_TA; idx += B_THREADS) {
        const int jw = idx / B_TA, aa = idx % B_TA;
        const int j = j0 + t.shift + jw, ai = a0 + aa;
        const bool v = j >= 0 && j < n && ai < n;
        cp_async8(dst0 + uint32_t(idx) * 8u, v ? Yk + size_t(j) * n + ai : Y, v);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  load(0, 0);
  for (int k = 0; k < r; ++k) {
    if (k + 1 < r) {
      load(k + 1, (k + 1) & 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* Ys = sm + (k & 1) * buf_doubles;
    const double* base = Ys + (8 * jq) * B_TA + a;
    if constexpr (TAPS > 0)
      corr8_fixed<TAPS>(acc, t.w[k], [&](int i) { return base[i * B_TA]; });
    else
      corr8_tail(acc, t.w[k], t.real, [&](int i) { return base[i * B_TA]; });
    __syncthreads();  // buffer (k & 1) is refilled at iteration k + 1
  }
  // epilogue (same contract as the GEMM epilogue; image blockIdx.z)
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const int m = a0 + a;
  if constexpr (!BATCH) {
    // single image: the epilogue reads e.* straight from the parameter bank
    // (copying the pointers into locals costs registers and, at 41 taps,
    // occupancy)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = j0 + 8 * jq + q;
      if (m >= n || j >= n) continue;
      double v = acc[q];
      const long vi = long(m) * e.vm + long(j) * e.vn;
      if (e.mul) v *= e.mul[vi];
      if (e.addv) v = __dadd_rn(v, __dmul_rn(e.addc, e.addv[vi]));  // + lambda^2 p, unfused as Eigen
      e.C[long(m) * e.cm + long(j) * e.cn] = v;
      if (e.partials) {
        if (e.d0) s0 += v * (e.d0_self ? v : e.d0[vi]);
        if (e.d1a) s1 += v * (e.d1b ? (e.d1a[vi] - e.d1b[vi]) : e.d1a[vi]);
        if (e.count_nonfinite && !isfinite(v)) s2 += 1.0;
      }
    }
  } else {
    const long zo = long(blockIdx.z) * e.img;
    double* const C = e.C + zo;
    const double* const mul = e.mul ? e.mul + zo : nullptr;
    const double* const addv = e.addv ? e.addv + zo : nullptr;
    const double addc = e.addc_img ? e.addc_img[blockIdx.z] : e.addc;
    const double* const d0 = e.d0 ? e.d0 + zo : nullptr;
    const double* const d1a = e.d1a ? e.d1a + zo : nullptr;
    const double* const d1b = e.d1b ? e.d1b + zo : nullptr;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = j0 + 8 * jq + q;
      if (m >= n || j >= n) continue;
      double v = acc[q];
      const long vi = long(m) * e.vm + long(j) * e.vn;
      if (mul) v *= mul[vi];
      if (addv) v = __dadd_rn(v, __dmul_rn(addc, addv[vi]));
      C[long(m) * e.cm + long(j) * e.cn] = v;
      if (e.partials) {
        if (e.d0) s0 += v * (e.d0_self ? v : d0[vi]);
        if (d1a) s1 += v * (d1b ? (d1a[vi] - d1b[vi]) : d1a[vi]);
        if (e.count_nonfinite && !isfinite(v)) s2 += 1.0;
      }
    }
  }
  if (e.partials) {
    __shared__ double red[B_THREADS / 32][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, off);
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    if (lane == 0) red[warp][0] = s0, red[warp][1] = s1, red[warp][2] = s2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double x0 = 0, x1 = 0, x2 = 0;
      for (int w = 0; w < B_THREADS / 32; ++w) x0 += red[w][0], x1 += red[w][1], x2 += red[w][2];
      double* o = e.partials + ((BATCH ? long(blockIdx.z) * e.part_img : 0L) + long(blockIdx.y) * gridDim.x +
                                blockIdx.x) * 4;
      o[0] = x0, o[1] = x1, o[2] = x2, o[3] = 0.0;
    }
  }
}

// Fused passes (A + B in one kernel) for short bands, where the two-pass
// form is bound by its r n^2 HBM intermediate rather than by DFMA (C4: 17
// taps, 2 * 17 flop per 16 B moved per pass): each CTA loads the X halo of
// its 64 x 64 output tile (64 + Lc - 1 rows, 64 + Lr - 1 columns) once,
// computes Y_k on those columns in shared memory (pass A's correlation on
// (64 + Lr - 1) / 64 of the columns) and correlates Y_k's rows into the
// output registers (pass B), term by term. HBM traffic is x in + out (+ the
// epilogue's vectors); the result equals the two-pass kernels' up to FP64
// summation order (same taps, same per-element accumulation order: pass A's
// sum over u of the column taps, then pass B's over the row taps, terms in
// order). TC / TR: compile-time tap counts.
constexpr int F_TA = 64, F_TJ = 64, F_THREADS = 256;
template <int TC, int TR>
struct FusedDims {
  static constexpr int XR = F_TA + TC - 1;          // X halo rows
  static constexpr int NC = F_TJ + TR - 1;          // X halo / Y columns
  static constexpr int SX = XR | 1;                 // odd column stride of X (doubles)
  static constexpr int SY = F_TA + 1;               // column stride of Y
  static constexpr size_t SMEM = (size_t(NC) * SX + size_t(NC) * SY) * sizeof(double);
};

template <int TC, int TR>
__global__ void __launch_bounds__(F_THREADS) band_fused_kernel(const double* __restrict__ X, int n, int r,
                                                               const __grid_constant__ BandTaps tc,
                                                               const __grid_constant__ BandTaps tr,
                                                               const F64Epilogue e, const int* status) {
  using D = FusedDims<TC, TR>;
  pdl_wait();
  if (stopped(status)) return;
  extern __shared__ double sm[];
  double* Xs = sm;                 // [NC][SX]: Xs[c * SX + i] = X(a0 + sc + i, j0 + sr + c)
  double* Ys = sm + D::NC * D::SX;  // [NC][SY]: Ys[c * SY + a] = Y_k(a0 + a, j0 + sr + c)
  X += size_t(blockIdx.z) * n * n;
  const int a0 = blockIdx.y * F_TA, j0 = blockIdx.x * F_TJ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {  // X halo: warp per column, lanes down the rows (coalesced), zeros outside [0, n)
    const uint32_t xs = static_cast<uint32_t>(__cvta_generic_to_shared(Xs));
    for (int c = warp; c < D::NC; c += F_THREADS / 32) {
      const int l = j0 + tr.shift + c;
      const double* col = X + size_t(l) * n;
      for (int v = lane; v < D::XR; v += 32) {
        const int i = a0 + tc.shift + v;
        const bool ok = l >= 0 && l < n && i >= 0 && i < n;
        cp_async8(xs + uint32_t(c * D::SX + v) * 8u, ok ? col + i : X, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  __syncthreads();
  // output tasks: (row a, 8-column block jb), two per thread
  constexpr int OUT_TASKS = F_TA * (F_TJ / 8) / F_THREADS;
  double acc[OUT_TASKS][8];
#pragma unroll
  for (int h = 0; h < OUT_TASKS; ++h)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[h][q] = 0.0;
  constexpr int Y_TASKS = D::NC * (F_TA / 8);  // (column c, 8-row block b)
  for (int k = 0; k < r; ++k) {
    // pass A on the halo columns: Y_k(a, c) = sum_u wc_k[u] X(a + sc + u, c)
    for (int id = threadIdx.x; id < Y_TASKS; id += F_THREADS) {
      const int c = id % D::NC, b = id / D::NC;
      double y[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const double* base = Xs + c * D::SX + 8 * b;
      corr8_fixed<TC>(y, tc.w[k], [&](int i) { return base[i]; });
#pragma unroll
      for (int q = 0; q < 8; ++q) Ys[c * D::SY + 8 * b + q] = y[q];
    }
    __syncthreads();
    // pass B: out(a, j) += sum_u wr_k[u] Y_k(a, j + sr + u)
#pragma unroll
    for (int h = 0; h < OUT_TASKS; ++h) {
      const int id = threadIdx.x + h * F_THREADS;
      const int a = id % F_TA, jb = id / F_TA;
      const double* base = Ys + (8 * jb) * D::SY + a;
      corr8_fixed<TR>(acc[h], tr.w[k], [&](int i) { return base[i * D::SY]; });
    }
    __syncthreads();  // Ys is rewritten by the next term
  }
  // epilogue (band_rows' contract; image blockIdx.z)
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  const long zo = long(blockIdx.z) * e.img;
  double* const C = e.C + zo;
  const double* const mul = e.mul ? e.mul + zo : nullptr;
  const double* const addv = e.addv ? e.addv + zo : nullptr;
  const double addc = e.addc_img ? e.addc_img[blockIdx.z] : e.addc;
  const double* const d0 = e.d0 ? e.d0 + zo : nullptr;
  const double* const d1a = e.d1a ? e.d1a + zo : nullptr;
  const double* const d1b = e.d1b ? e.d1b + zo : nullptr;
#pragma unroll
  for (int h = 0; h < OUT_TASKS; ++h) {
    const int id = threadIdx.x + h * F_THREADS;
    const int m = a0 + id % F_TA, jb = id / F_TA;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = j0 + 8 * jb + q;
      if (m >= n || j >= n) continue;
      double v = acc[h][q];
      const long vi = long(m) * e.vm + long(j) * e.vn;
      if (mul) v *= mul[vi];
      if (addv) v = __dadd_rn(v, __dmul_rn(addc, addv[vi]));  // + lambda^2 p, unfused as Eigen
      C[long(m) * e.cm + long(j) * e.cn] = v;
      if (e.partials) {
        if (e.d0) s0 += v * (e.d0_self ? v : d0[vi]);
        if (d1a) s1 += v * (d1b ? (d1a[vi] - d1b[vi]) : d1a[vi]);
        if (e.count_nonfinite && !isfinite(v)) s2 += 1.0;
      }
    }
  }
  if (e.partials) {
    __shared__ double red[F_THREADS / 32][3];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, off);
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    if (lane == 0) red[warp][0] = s0, red[warp][1] = s1, red[warp][2] = s2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double x0 = 0, x1 = 0, x2 = 0;
      for (int w = 0; w < F_THREADS / 32; ++w) x0 += red[w][0], x1 += red[w][1], x2 += red[w][2];
      double* o = e.partials + (long(blockIdx.z) * e.part_img + long(blockIdx.y) * gridDim.x + blockIdx.x) * 4;
      o[0] = x0, o[1] = x1, o[2] = x2, o[3] = 0.0;
    }
  }
}

template <int TC, int TR>
void launch_fused(const double* X, int n, int r, const BandTaps& tc, const BandTaps& tr, const F64Epilogue& e,
                  const int* status, int batch) {
  using D = FusedDims<TC, TR>;
  auto k = band_fused_kernel<TC, TR>;
  set_smem_limit(reinterpret_cast<const void*>(k), D::SMEM);
  dim3 grid(cdiv(n, F_TJ), cdiv(n, F_TA), batch);
  launch_pdl(k, grid, dim3(F_THREADS), D::SMEM, X, n, r, tc, tr, e, status);
}

// Tap counts with specialised kernels (the BASELINE PSFs: 41 (C5), 31
// (C2/C3), 19 (C1), 17 (C4)); any other count runs the generic kernels.
template <template <int> class F, typename... Args>
void by_taps(int real, Args&&... args) {
  switch (real) {
    case 17: F<17>::run(args...); break;
    case 19: F<19>::run(args...); break;
    case 31: F<31>::run(args...); break;
    case 41: F<41>::run(args...); break;
    default: F<0>::run(args...); break;
  }
}

template <int TAPS>
struct ColsLaunch {
  static void run(const double* X, double* Y, int n, int r, const BandTaps& t, const int* status,
                  int batch) {
    const size_t smem = size_t(A_TL) * (cols_stride<TAPS>(t.taps) + A_SO) * sizeof(double);
    auto k = band_cols_kernel<TAPS>;
    set_smem_limit(reinterpret_cast<const void*>(k), smem);
    dim3 grid(cdiv(n, A_TL), cdiv(n, A_TA), batch);
    launch_pdl(k, grid, dim3(A_THREADS), smem, X, Y, n, r, t, status);
  }
};
template <int TAPS>
struct RowsLaunch {
  static void run(const double* Y, int n, int r, const BandTaps& t, const F64Epilogue& e,
                  const int* status, int batch) {
    const size_t smem = 2 * size_t(rows_halo<TAPS>(t.taps)) * B_TA * sizeof(double);  // two buffers
    auto k = batch > 1 ? band_rows_kernel<TAPS, true> : band_rows_kernel<TAPS, false>;
    set_smem_limit(reinterpret_cast<const void*>(k), smem);
    dim3 grid(cdiv(n, B_TJ), cdiv(n, B_TA), batch);
    launch_pdl(k, grid, dim3(B_THREADS), smem, Y, n, r, t, e, status);
  }
};

bool generic_only() {
  static const bool g = [] {
    const char* e = getenv("KP_BAND_GENERIC");
    return e && atoi(e) != 0;
  }();
  return g;
}

}  // namespace

void band_cols(const double* X, double* Y, int n, int r, const BandTaps& t, const int* status,
               int batch) {
  LaunchScope scope(KC_OPERATOR);
  by_taps<ColsLaunch>(generic_only() ? 0 : t.real, X, Y, n, r, t, status, batch);
  check_launch("band_cols");
}

int band_rows_num_ctas(int n) { return int(cdiv(n, B_TJ) * cdiv(n, B_TA)); }

bool band_fused_supported(int col_taps, int row_taps) {
  return col_taps == row_taps && (col_taps == 17 || col_taps == 19);
}
int band_fused_num_ctas(int n) { return int(cdiv(n, F_TJ) * cdiv(n, F_TA)); }

void band_fused(const double* X, int n, int r, const BandTaps& tc, const BandTaps& tr, const F64Epilogue& e,
                const int* status, int batch) {
  LaunchScope scope(KC_OPERATOR);
  if (tc.real == 17 && tr.real == 17)
    launch_fused<17, 17>(X, n, r, tc, tr, e, status, batch);
  else if (tc.real == 19 && tr.real == 19)
    launch_fused<19, 19>(X, n, r, tc, tr, e, status, batch);
  else
    throw InvalidArgument("band_fused: unsupported tap counts");
  check_launch("band_fused");
}

void band_rows(const double* Y, int n, int r, const BandTaps& t, const F64Epilogue& e,
               const int* status, int batch) {
  LaunchScope scope(KC_OPERATOR);
  by_taps<RowsLaunch>(generic_only() ? 0 : t.real, Y, n, r, t, e, status, batch);
  check_launch("band_rows");
}

}  // namespace kp
