// FP64 GEMM C = A * B^T (both operands K-major) on the DMMA pipe.
//
// Replaces the dense Eigen products of kron_apply (kron.cpp:62-71) summed over
// terms (kron.cpp:73-88): the Kronecker-sum is folded into the GEMM K (or M)
// dimension by the caller (api.cu), so one launch covers all r terms.
//
// Design (sm_100a): mma.sync.aligned.m16n8k16 f64 (DMMA; measured 37.0 TF/s
// peak on B200, profiles/r01_microbench_peaks.txt), multistage pipeline into
// XOR-swizzled K-major tiles (16 doubles = one 128-byte row per M/N index;
// 16-byte chunk c of row r lives at c ^ (r & 7) - the TMA SWIZZLE_128B
// pattern), so every fragment load is a conflict-free LDS.128. The 128 x 128
// tiles are staged by TMA (cp.async.bulk.tensor 3-D boxes of 16 doubles x 128
// rows over (k, row, term), zero fill outside the matrix, one elected thread,
// full mbarrier per stage; the per-iteration __syncthreads frees the stage
// being refilled); the 64 x 64 tiles of small problems and operands TMA
// cannot address (odd leading dimension, unaligned base) use cp.async. The K index inside an MMA is permuted
// (logical k = t + 4j <-> physical 4t + j) so each lane fetches its four K
// values as 32 contiguous bytes; A and B use the same permutation, which only
// reorders the exact FP64 sum.
#include "gemm_f64.cuh"

#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

namespace kp {
namespace {

constexpr int BK = 16;  // doubles per K tile (one 128-byte smem row)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void lds128(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

__device__ __forceinline__ void dmma16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// Tile rasterisation: groups of GROUP_M M-tiles sweep all N-tiles so a wave
// of CTAs shares A and B tiles in L2.
constexpr int GROUP_M = 16;

template <int BM, int BN, int WM, int WN, int STAGES, int KSUB, bool VEC16, bool TMA>
__device__ __forceinline__ void gemm_f64_body(const F64GemmArgs& args, const CUtensorMap* map_a,
                                              const CUtensorMap* map_b) {
  pdl_wait();
  constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  constexpr int THREADS = WARPS_M * WARPS_N * 32;
  constexpr int MT = WM / 16, NT = WN / 8;
  constexpr int KT_DEPTH = BK * KSUB;                 // K per pipeline stage
  constexpr int SUB_DOUBLES = (BM + BN) * BK;         // one 16-deep sub-tile
  constexpr int STAGE_DOUBLES = SUB_DOUBLES * KSUB;

  if (args.status && *args.status != 0) return;

  extern __shared__ __align__(1024) double smem_dyn[];
  // SWIZZLE_128B boxes repeat every 1024 bytes: the TMA path needs that alignment
  double* smem = TMA ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023))
                     : smem_dyn;
  __shared__ __align__(8) uint64_t full_bar[STAGES];

  const int M = args.M, N = args.N;
  const int grid_m = (M + BM - 1) / BM, grid_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  const int group = pid / (GROUP_M * grid_n);
  const int first_m = group * GROUP_M;
  const int gsize = min(grid_m - first_m, GROUP_M);
  const int tile_m = first_m + (pid % (GROUP_M * grid_n)) % gsize;
  const int tile_n = (pid % (GROUP_M * grid_n)) / gsize;
  const int m_base = tile_m * BM, n_base = tile_n * BN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int g = lane >> 2, t = lane & 3;

  const int Kb = args.Kb;
  const int kt_per_batch = (Kb + KT_DEPTH - 1) / KT_DEPTH;
  const int total_kt = args.nb * kt_per_batch;

  const uint32_t smem_base = smem_u32(smem);

  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&full_bar[s]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map_b)) : "memory");
    }
    __syncthreads();
  }

  auto load_tile = [&](int kt, int stage) {
    const int b = kt / kt_per_batch;
    const int k0 = (kt % kt_per_batch) * KT_DEPTH;
    if constexpr (TMA) {
      // one thread: KSUB boxes of 16 doubles x BM (BN) rows per operand
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const uint32_t fb = smem_u32(&full_bar[stage]);
        mbar_expect_tx(fb, uint32_t(STAGE_DOUBLES * 8));
#pragma unroll
        for (int sub = 0; sub < KSUB; ++sub) {
          const uint32_t sa = smem_base + uint32_t(stage * STAGE_DOUBLES + sub * SUB_DOUBLES) * 8u;
          tma_load_3d(sa, map_a, fb, k0 + sub * BK, m_base, b);
          tma_load_3d(sa + uint32_t(BM * BK) * 8u, map_b, fb, k0 + sub * BK, n_base, b);
        }
      }
      return;
    }
    constexpr int CHUNKS_A = BM * 8, CHUNKS_B = BN * 8, CHUNKS = (CHUNKS_A + CHUNKS_B) * KSUB;
#pragma unroll
    for (int id = tid; id < CHUNKS; id += THREADS) {
      const int sub = id / (CHUNKS_A + CHUNKS_B);
      const int rid = id % (CHUNKS_A + CHUNKS_B);
      const bool isA = rid < CHUNKS_A;
      const int cid = isA ? rid : rid - CHUNKS_A;
      const int row = cid >> 3, ch = cid & 7;
      const int grow = (isA ? m_base : n_base) + row;
      const int rows = isA ? M : N;
      const F64Operand& op = isA ? args.A : args.B;
      const int kk = k0 + sub * BK + ch * 2;
      const uint32_t sa = smem_base + uint32_t(stage * STAGE_DOUBLES + sub * SUB_DOUBLES) * 8u;
      const uint32_t sb = sa + uint32_t(BM * BK) * 8u;
      const uint32_t dst = (isA ? sa : sb) + uint32_t(row * 128 + ((ch ^ (row & 7)) << 4));
      const double* src = op.p + long(b) * op.bstride + long(grow) * op.ld + kk;
      if (VEC16) {
        const bool v = grow < rows && kk < Kb;
        cp_async16(dst, v ? src : op.p, v);
      } else {
        const bool v0 = grow < rows && kk < Kb;
        const bool v1 = grow < rows && kk + 1 < Kb;
        cp_async8(dst, v0 ? src : op.p, v0);
        cp_async8(dst + 8, v1 ? src + 1 : op.p, v1);
      }
    }
  };

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total_kt) load_tile(s, s);
    if constexpr (!TMA) cp_async_commit();
  }

  for (int kt = 0; kt < total_kt; ++kt) {
    if constexpr (TMA)
      mbar_wait(smem_u32(&full_bar[kt % STAGES]), uint32_t((kt / STAGES) & 1));
    else
      cp_async_wait<STAGES - 2>();
    __syncthreads();  // every warp is done with the stage refilled below
    {
      const int nk = kt + STAGES - 1;
      if (nk < total_kt) load_tile(nk, nk % STAGES);
      if constexpr (!TMA) cp_async_commit();
    }
    const int stage = kt % STAGES;
#pragma unroll
    for (int sub = 0; sub < KSUB; ++sub) {
      const uint32_t sa = smem_base + uint32_t(stage * STAGE_DOUBLES + sub * SUB_DOUBLES) * 8u;
      const uint32_t sb = sa + uint32_t(BM * BK) * 8u;
      double bf[NT][4];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int row = wn * WN + j * 8 + g;
        const uint32_t rb = sb + uint32_t(row * 128);
        lds128(rb + uint32_t(((2 * t) ^ (row & 7)) << 4), bf[j][0], bf[j][1]);
        lds128(rb + uint32_t(((2 * t + 1) ^ (row & 7)) << 4), bf[j][2], bf[j][3]);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        double af[8];
        const int r0 = wm * WM + i * 16 + g, r1 = r0 + 8;
        const uint32_t ra0 = sa + uint32_t(r0 * 128), ra1 = sa + uint32_t(r1 * 128);
        // a[v0 + 2 v1] = A[g + 8 v0][4t + v1]
        lds128(ra0 + uint32_t(((2 * t) ^ (r0 & 7)) << 4), af[0], af[2]);
        lds128(ra0 + uint32_t(((2 * t + 1) ^ (r0 & 7)) << 4), af[4], af[6]);
        lds128(ra1 + uint32_t(((2 * t) ^ (r1 & 7)) << 4), af[1], af[3]);
        lds128(ra1 + uint32_t(((2 * t + 1) ^ (r1 & 7)) << 4), af[5], af[7]);
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma16(acc[i][j], af, bf[j]);
      }
    }
  }
  if constexpr (!TMA) cp_async_wait<0>();

  // ---- epilogue ----
  const F64Epilogue& e = args.epi;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int m = m_base + wm * WM + i * 16 + g + ((q >> 1) << 3);
        const int n = n_base + wn * WN + j * 8 + 2 * t + (q & 1);
        if (m < M && n < N) {
          double v = acc[i][j][q];
          const long vi = long(m) * e.vm + long(n) * e.vn;
          if (e.mul) v *= e.mul[vi];
          if (e.addv) v = __dadd_rn(v, __dmul_rn(e.addc, e.addv[vi]));  // + lambda^2 p, unfused as Eigen
          e.C[long(m) * e.cm + long(n) * e.cn] = v;
          if (e.partials) {
            if (e.d0) s0 += v * (e.d0_self ? v : e.d0[vi]);
            if (e.d1a) s1 += v * (e.d1b ? (e.d1a[vi] - e.d1b[vi]) : e.d1a[vi]);
            if (e.count_nonfinite && !isfinite(v)) s2 += 1.0;
          }
        }
      }
  if (e.partials) {
    __shared__ double red[THREADS / 32][3];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, off);
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    if (lane == 0) red[warp][0] = s0, red[warp][1] = s1, red[warp][2] = s2;
    __syncthreads();
    if (tid == 0) {
      double a0 = 0, a1 = 0, a2 = 0;
      for (int w = 0; w < THREADS / 32; ++w) a0 += red[w][0], a1 += red[w][1], a2 += red[w][2];
      double* o = e.partials + long(pid) * 4;
      o[0] = a0, o[1] = a1, o[2] = a2, o[3] = 0.0;
    }
  }
}

template <int BM, int BN, int WM, int WN, int STAGES, int KSUB, bool VEC16>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    gemm_f64_kernel(const F64GemmArgs args) {
  gemm_f64_body<BM, BN, WM, WN, STAGES, KSUB, VEC16, false>(args, nullptr, nullptr);
}

template <int BM, int BN, int WM, int WN, int STAGES, int KSUB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32)
    gemm_f64_tma_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        const F64GemmArgs args) {
  gemm_f64_body<BM, BN, WM, WN, STAGES, KSUB, true, true>(args, &map_a, &map_b);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    KP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// (k, row, term) view of a K-major operand: Kb x rows x nb doubles, box 16 x box_rows x 1
CUtensorMap make_map_f64(const F64Operand& op, int rows, int Kb, int nb, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {cuuint64_t(Kb), cuuint64_t(rows), cuuint64_t(nb)};
  const cuuint64_t bstride = op.bstride ? cuuint64_t(op.bstride) : cuuint64_t(op.ld) * rows;
  const cuuint64_t strides[2] = {cuuint64_t(op.ld) * 8, bstride * 8};
  const cuuint32_t box[3] = {cuuint32_t(BK), cuuint32_t(box_rows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(op.p), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (f64) failed: " + std::to_string(int(r)));
  return m;
}

// KP_F64_TMA=0 keeps the cp.async staging for the big tiles (A/B measurement).
bool f64_tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("KP_F64_TMA");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

template <int BM, int BN, int WM, int WN, int STAGES, int KSUB>
void launch_cfg(const F64GemmArgs& a, bool allow_tma = false) {
  constexpr int THREADS = (BM / WM) * (BN / WN) * 32;
  constexpr size_t SMEM = size_t(STAGES) * KSUB * (BM + BN) * BK * sizeof(double);
  const unsigned grid = cdiv(a.M, BM) * cdiv(a.N, BN);
  const bool vec16 = (a.Kb % 2 == 0) && (a.A.ld % 2 == 0) && (a.B.ld % 2 == 0) &&
                     (a.A.bstride % 2 == 0) && (a.B.bstride % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(a.A.p) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(a.B.p) % 16 == 0);
  if (vec16 && allow_tma && f64_tma_enabled() && SMEM + 1024 <= 227 * 1024) {
    auto k = gemm_f64_tma_kernel<BM, BN, WM, WN, STAGES, KSUB>;
    set_smem_limit(reinterpret_cast<const void*>(k), SMEM + 1024);
    const CUtensorMap ma = make_map_f64(a.A, a.M, a.Kb, a.nb, BM), mb = make_map_f64(a.B, a.N, a.Kb, a.nb, BN);
    launch_pdl(k, dim3(grid), dim3(THREADS), SMEM + 1024, ma, mb, a);
  } else if (vec16) {
    auto k = gemm_f64_kernel<BM, BN, WM, WN, STAGES, KSUB, true>;
    set_smem_limit(reinterpret_cast<const void*>(k), SMEM);
    launch_pdl(k, dim3(grid), dim3(THREADS), SMEM, a);
  } else {
    auto k = gemm_f64_kernel<BM, BN, WM, WN, STAGES, KSUB, false>;
    set_smem_limit(reinterpret_cast<const void*>(k), SMEM);
    launch_pdl(k, dim3(grid), dim3(THREADS), SMEM, a);
  }
}

// Big-tile variant (experiment switch KP_F64_CFG, default 0).
int big_cfg() {
  static int cfg = [] {
    const char* e = getenv("KP_F64_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

bool use_big_tiles(int M, int N) {
  // 128x128 tiles once they still give at least ~one CTA per SM.
  return long(cdiv(M, 128)) * cdiv(N, 128) >= ctx().num_sms;
}

void launch_big(const F64GemmArgs& a) {
  // Measured at C5 (profiles/r01_sweep_f64.txt): 0: 30.5, 1: 30.6, 2: 32.2,
  // 3: 31.6, 4: 27.7 TF/s; all variants are bitwise identical.
  switch (big_cfg()) {
    case 1: launch_cfg<128, 128, 32, 32, 4, 1>(a); break;   // 16 warps of 32x32
    case 3: launch_cfg<128, 128, 32, 32, 3, 2>(a); break;   // 16 warps, 32-deep stages
    case 4: launch_cfg<128, 64, 32, 32, 4, 1>(a); break;    // 8 warps, 2 CTAs/SM
    case 5: launch_cfg<128, 128, 64, 32, 4, 1>(a); break;   // 8 warps, 16-deep stages
    default: launch_cfg<128, 128, 64, 32, 3, 2>(a, true); break;  // 8 warps, 32-deep stages, TMA
  }
}

int big_tile_n() { return big_cfg() == 4 ? 64 : 128; }

}  // namespace

int gemm_f64_num_ctas(int M, int N) {
  if (use_big_tiles(M, N)) return int(cdiv(M, 128) * cdiv(N, big_tile_n()));
  return int(cdiv(M, 64) * cdiv(N, 64));
}

void gemm_f64(const F64GemmArgs& a, int kernel_class) {
  if (a.M <= 0 || a.N <= 0) return;
  LaunchScope scope(kernel_class);
  if (use_big_tiles(a.M, a.N))
    launch_big(a);
  else
    launch_cfg<64, 64, 32, 32, 4, 1>(a);
  check_launch("gemm_f64");
}

}  // namespace kp
