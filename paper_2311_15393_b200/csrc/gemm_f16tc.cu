// tcgen05 tensor-core binary16 GEMM for the preconditioner solve in
// KP_ACCUM_TENSOR mode (north star: "fp16-storage tcgen05 GEMMs with the
// diagonal scaling fused into the epilogue"). C(m,n) = sum_k A(m,k) B(n,k)
// with fp16 operands and fp32 accumulation in TMEM, one RNE rounding of the
// result to binary16 (or FP64 for the last product of the solve).
//
// Differences from the reference's lp_matmul (lpblas.cpp:59-70): products and
// partial sums are not rounded to binary16 — only the result is. This is the
// tensor-pipe semantics the BASELINE north star accepts (+-2 iterations,
// 1e-3 final error); KP_ACCUM_REFERENCE keeps the bit-exact emulation.
//
// Structure (canonical sm_100 warp-specialised persistent GEMM):
//   warp 0      TMA producer: cp.async.bulk.tensor 2-D loads of 128 x 64
//               K-major SWIZZLE_128B tiles into a STAGES-deep smem ring
//               (full / empty mbarriers)
//   warp 1      MMA issuer: allocates 2 x BN TMEM columns, one elected lane
//               issues tcgen05.mma.kind::f16 (M=128, N=BN, K=16) from smem
//               descriptors, commits stage releases and accumulator-ready
//               signals (tcgen05.commit -> mbarrier)
//   warps 2..9  epilogue: tcgen05.ld the accumulator (warp w owns TMEM lanes
//               32*(w%4)..; the two warps of a quadrant take alternate 32-column
//               chunks, doubling the loads in flight), round to binary16, fuse
//               S.* / FP64 output / dot partials, release the TMEM buffer
// Tiles are distributed persistently over the grid with double-buffered
// accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

#include "gemm_f16ref.cuh"
#include "gemm_f16tc.cuh"

namespace kp {
namespace {

constexpr int BM = 128, BKH = 64, STAGES = 4;
constexpr int EPI_WARPS = 8;       // two warps per TMEM lane quadrant
constexpr int NUM_THREADS = 32 * (2 + EPI_WARPS);
constexpr int TILE_A_BYTES = BM * BKH * 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (tcgen05, version 1):
// rows of 128 B, 8-row groups 1024 B apart (SBO), LBO unused.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
template <int BN>
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  // kind::f16 instruction descriptor: D=F32, A=B=F16, K-major, M=128, N=BN
  constexpr uint32_t IDESC = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_f16tc_kernel(const __grid_constant__ CUtensorMap map_a,
                      const __grid_constant__ CUtensorMap map_b, const F16GemmArgs args) {
  pdl_wait();
  constexpr int TILE_B_BYTES = BN * BKH * 2;
  constexpr int STAGE_BYTES = TILE_A_BYTES + TILE_B_BYTES;
  // double-buffered fp32 accumulators; the allocation is a power of two >= 32 columns
  constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  if (args.status && *args.status != 0) return;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[EPI_WARPS][3];

  const int M = args.M, N = args.N;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int KT = (args.K + BKH - 1) / BKH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = smem_u32(smem);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&full_bar[s]), 1), mbar_init(smem_u32(&empty_bar[s]), 1);
    for (int s = 0; s < 2; ++s) mbar_init(smem_u32(&tfull_bar[s]), 1), mbar_init(smem_u32(&tempty_bar[s]), EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  // Grouped rasterisation over the persistent tile sequence.
  auto tile_coords = [&](int t, int& mb, int& nb) {
    constexpr int GROUP = 8;
    const int group = t / (GROUP * tiles_n);
    const int first = group * GROUP;
    const int gs = min(tiles_m - first, GROUP);
    mb = (first + (t % (GROUP * tiles_n)) % gs) * BM;
    nb = ((t % (GROUP * tiles_n)) / gs) * BN;
  };

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, mb, nb);
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          mbar_expect_tx(fb, STAGE_BYTES);
          const uint32_t sa = sbase + uint32_t(stage * STAGE_BYTES);
          tma_load_2d(sa, &map_a, fb, kt * BKH, mb);
          tma_load_2d(sa + TILE_A_BYTES, &map_b, fb, kt * BKH, nb);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        mbar_wait(smem_u32(&tempty_bar[acc]), uint32_t(((local >> 1) & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t sa = sbase + uint32_t(stage * STAGE_BYTES), sb = sa + TILE_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BKH / 16; ++kk)  // +32 B per K=16 inside the 128-B swizzle atom
            umma_f16<BN>(d, make_desc(sa + kk * 32), make_desc(sb + kk * 32), (kt | kk) != 0);
          umma_commit(smem_u32(&empty_bar[stage]));  // frees the smem stage when done
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        umma_commit(smem_u32(&tfull_bar[acc]));  // accumulator ready
      }
    }
  } else {  // ===== epilogue warps 2..9 =====
    const int quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int ew = warp - 2;            // epilogue warp index 0..7
    const int half = ew >> 2;           // which alternate 32-column chunks
    const F16Epilogue& e = args.epi;
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int acc = local & 1;
      mbar_wait(smem_u32(&tfull_bar[acc]), uint32_t((local >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int m = mb + quad * 32 + lane;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll 1
      for (int c0 = 32 * half; c0 < BN; c0 += 64) {
        uint32_t v[32];
        tmem_ld32(tmem + (uint32_t(quad * 32) << 16) + uint32_t(acc * BN + c0), v);
        if (m >= M) continue;
        if (e.mode == F16OUT_F64) {
          // Batches of 8 columns: all vector loads of a batch are issued
          // before any store, so their latencies overlap.
          double* __restrict__ Cd = e.Cd;
          const double* __restrict__ d0 = e.d0;
          const double* __restrict__ d1a = e.d1a;
          const double* __restrict__ d1b = e.d1b;
          const bool part = e.partials != nullptr;
          const bool same = d0 != nullptr && d1a == d0;
#pragma unroll
          for (int j0 = 0; j0 < 32; j0 += 8) {
            double a0[8], a1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int n = nb + c0 + j0 + j;
              const long vi = long(m) * e.vm + long(n) * e.vn;
              const bool ok = part && n < N;
              a0[j] = (ok && d0) ? d0[vi] : 0.0;
              // FPCG passes d0 == d1a == r: load r once
              const double ra = same ? a0[j] : ((ok && d1a) ? d1a[vi] : 0.0);
              a1[j] = (ok && d1a) ? (d1b ? ra - d1b[vi] : ra) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int n = nb + c0 + j0 + j;
              if (n < N) {
                const double z = double(__half2float(__float2half_rn(__uint_as_float(v[j0 + j]))));
                Cd[long(m) * e.cm + long(n) * e.cn] = z;
                if (part) {
                  if (d0) s0 += z * a0[j];
                  if (d1a) s1 += z * a1[j];
                  if (!isfinite(z)) s2 += 1.0;
                }
              }
            }
          }
          continue;
        }
        // batched products stacked along M: this tile's image and local row
        const int img = e.m_img ? mb / e.m_img : 0;
        const int ml = m - img * e.m_img;
        __half* __restrict__ Ch = e.Ch + img * e.c_img;
        if (e.mode == F16OUT_HALF_SCALED) {  // w = round16(S .* t2), as the reference
          const __half* __restrict__ sc = e.scale + img * e.s_img;
          __half sv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {  // all scale loads first
            const int n = nb + c0 + j;
            sv[j] = n < N ? sc[long(ml) * e.sm + long(n) * e.sn] : __ushort_as_half(0);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = nb + c0 + j;
            if (n < N)
              Ch[long(ml) * e.cm + long(n) * e.cn] = __hmul_rn(sv[j], __float2half_rn(__uint_as_float(v[j])));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = nb + c0 + j;
            if (n < N) Ch[long(ml) * e.cm + long(n) * e.cn] = __float2half_rn(__uint_as_float(v[j]));
          }
        }
      }
      // release the accumulator buffer to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[acc]));
      if (e.mode == F16OUT_F64 && e.partials) {  // fixed-order per-tile partials
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, off);
          s1 += __shfl_xor_sync(0xffffffffu, s1, off);
          s2 += __shfl_xor_sync(0xffffffffu, s2, off);
        }
        if (lane == 0) red[ew][0] = s0, red[ew][1] = s1, red[ew][2] = s2;
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0) {
          double a0 = 0, a1 = 0, a2 = 0;
          for (int w = 0; w < EPI_WARPS; ++w) a0 += red[w][0], a1 += red[w][1], a2 += red[w][2];
          double* o = e.partials + long(t) * 4;
          o[0] = a0, o[1] = a1, o[2] = a2, o[3] = 0.0;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * EPI_WARPS) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    KP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D K-major fp16 operand: dim0 = K (ld elements, contiguous), dim1 = rows;
// box = 64 x box_rows with 128-byte swizzle (matches make_desc).
CUtensorMap make_map(const F16Operand& op, int rows, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(op.ld), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(op.ld) * 2};
  const cuuint32_t box[2] = {cuuint32_t(BKH), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(op.p),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

template <int BN>
void launch_tc(const F16GemmArgs& a) {
  constexpr size_t SMEM = size_t(STAGES) * (TILE_A_BYTES + BN * BKH * 2) + 1024;
  auto k = gemm_f16tc_kernel<BN>;
  set_smem_limit(reinterpret_cast<const void*>(k), SMEM);
  const CUtensorMap ma = make_map(a.A, a.M, BM), mb = make_map(a.B, a.N, BN);
  const int tiles = int(cdiv(a.M, BM) * cdiv(a.N, BN));
  const int grid = std::min(tiles, ctx().num_sms);
  launch_pdl(k, dim3(grid), dim3(NUM_THREADS), SMEM, ma, mb, a);
}

// Tile width: BN = 256 for the binary16-output products (half the A traffic
// per flop: 97.6 vs 131.5 us per n = 4096 product), BN = 128 for FP64 output
// (lp_matmul's FP64 result), whose epilogue is memory bound and needs the
// finer tiles to overlap it with the MMAs. The M-solve's last product stores
// binary16 z and leaves widening + dots to msolve_finish_f16 (vec.cu).
// KP_F16TC_BN = 128 | 192 | 256 forces one width for all products.
int tc_bn(int mode) {
  static int forced = [] {
    const char* e = getenv("KP_F16TC_BN");
    return e ? atoi(e) : 0;
  }();
  if (forced == 128 || forced == 192 || forced == 256) return forced;
  return mode == F16OUT_F64 ? 128 : 256;
}

}  // namespace

// Partials are written per output tile (FP64-output products only).
int gemm_f16tc_num_ctas(int M, int N) { return int(cdiv(M, BM) * cdiv(N, tc_bn(F16OUT_F64))); }

void gemm_f16tc(const F16GemmArgs& a, int kernel_class) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K <= 0) throw InvalidArgument("lp_matmul: empty input");
  if (a.A.ld % BKH || a.B.ld % BKH || a.A.ld < a.K || a.B.ld < a.K)
    throw InvalidArgument("gemm_f16tc: operand leading dimension must be a multiple of 64 >= K");
  LaunchScope scope(kernel_class);
  switch (tc_bn(a.epi.mode)) {
    case 256: launch_tc<256>(a); break;
    case 192: launch_tc<192>(a); break;
    default: launch_tc<128>(a); break;
  }
  check_launch("gemm_f16tc");
}

}  // namespace kp
