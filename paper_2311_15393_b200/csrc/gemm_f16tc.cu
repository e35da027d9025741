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
// Structure: 128x128 output tile per CTA (UMMA M=128, N=128, K=16,
// cta_group::1), 128 threads. All threads stream K-major operand tiles with
// cp.async into the canonical K-major SWIZZLE_128B layout (row r = 128 bytes
// of K, 16-byte chunk c at c ^ (r & 7), 8-row groups 1024 B apart); thread 0
// issues tcgen05.mma from shared-memory descriptors and commits each stage to
// an mbarrier that gates the reuse of that stage's buffers; the epilogue reads
// the accumulator with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31).
#include "gemm_f16ref.cuh"
#include "gemm_f16tc.cuh"

namespace kp {
namespace {

constexpr int BM = 128, BN = 128, BKH = 64, THREADS = 128, STAGES = 3;
constexpr int ROW_BYTES = BKH * 2;                      // 128
constexpr int TILE_A = BM * ROW_BYTES, TILE_B = BN * ROW_BYTES;
constexpr int STAGE_BYTES = TILE_A + TILE_B;            // 32 KB
constexpr int TMEM_COLS = 128;
constexpr int GROUP_M = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
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
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity));
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "version 1").
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;         // SBO: 8-row groups 1024 B apart
  d |= uint64_t(1) << 46;                 // descriptor version (Blackwell)
  d |= uint64_t(2) << 61;                 // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: D=F32, A=B=F16, both K-major, M=128, N=128.
constexpr uint32_t IDESC = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
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

__global__ void __launch_bounds__(THREADS) gemm_f16tc_kernel(const F16GemmArgs args) {
  if (args.status && *args.status != 0) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t mbar[STAGES];
  __shared__ uint32_t tmem_base_sh;

  const int M = args.M, N = args.N;
  const int grid_m = (M + BM - 1) / BM, grid_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  const int group = pid / (GROUP_M * grid_n);
  const int first_m = group * GROUP_M;
  const int gsize = min(grid_m - first_m, GROUP_M);
  const int tile_m = first_m + (pid % (GROUP_M * grid_n)) % gsize;
  const int tile_n = (pid % (GROUP_M * grid_n)) / gsize;
  const int m_base = tile_m * BM, n_base = tile_n * BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const uint32_t sbase = smem_u32(smem);
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&mbar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  const int KT = (args.K + BKH - 1) / BKH;
  auto load_tile = [&](int kt, int stage) {
    const uint32_t sa = sbase + uint32_t(stage * STAGE_BYTES);
    const uint32_t sb = sa + TILE_A;
    constexpr int CA = BM * 8, CB = BN * 8;
#pragma unroll 4
    for (int id = tid; id < CA + CB; id += THREADS) {
      const bool isA = id < CA;
      const int cid = isA ? id : id - CA;
      const int row = cid >> 3, ch = cid & 7;
      const int grow = (isA ? m_base : n_base) + row;
      const bool v = grow < (isA ? M : N);
      const F16Operand& op = isA ? args.A : args.B;
      const __half* src = op.p + long(grow) * op.ld + kt * BKH + ch * 8;
      cp_async16((isA ? sa : sb) + uint32_t(row * ROW_BYTES + ((ch ^ (row & 7)) << 4)),
                 v ? src : op.p, v);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int stage = kt % STAGES;
    cp_async_wait<STAGES - 2>();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic -> async proxy
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t sa = sbase + uint32_t(stage * STAGE_BYTES), sb = sa + TILE_A;
#pragma unroll
      for (int kk = 0; kk < BKH / 16; ++kk)  // K=16 per UMMA: +32 B inside the swizzle atom
        umma_f16(tmem, make_desc(sa + kk * 32), make_desc(sb + kk * 32), (kt | kk) != 0);
      umma_commit(smem_u32(&mbar[stage]));
    }
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      const int ns = nk % STAGES;
      if (kt >= 1) mbar_wait(smem_u32(&mbar[ns]), uint32_t(((kt - 1) / STAGES) & 1));
      load_tile(nk, ns);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  // all MMAs done: the last commit covers every earlier tcgen05.mma
  mbar_wait(smem_u32(&mbar[(KT - 1) % STAGES]), uint32_t(((KT - 1) / STAGES) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // ---- epilogue: thread (warp w, lane l) owns output row m = 32w + l ----
  const F16Epilogue& e = args.epi;
  const int m = m_base + warp * 32 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = n_base + c0 + j;
      if (n >= N) break;
      const float acc = __uint_as_float(v[j]);
      const __half h = __float2half_rn(acc);  // the GEMM result in binary16
      if (e.mode == F16OUT_HALF) {
        e.Ch[long(m) * e.cm + long(n) * e.cn] = h;
      } else if (e.mode == F16OUT_HALF_SCALED) {  // w = round16(S .* t2), as the reference
        const __half sc = e.scale[long(m) * e.sm + long(n) * e.sn];
        e.Ch[long(m) * e.cm + long(n) * e.cn] = __hmul_rn(sc, h);
      } else {
        const double z = double(__half2float(h));
        e.Cd[long(m) * e.cm + long(n) * e.cn] = z;
        if (e.partials) {
          const long vi = long(m) * e.vm + long(n) * e.vn;
          if (e.d0) s0 += z * e.d0[vi];
          if (e.d1a) s1 += z * (e.d1b ? (e.d1a[vi] - e.d1b[vi]) : e.d1a[vi]);
          if (!isfinite(z)) s2 += 1.0;
        }
      }
    }
  }
  if (e.mode == F16OUT_F64 && e.partials) {
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
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

}  // namespace

int gemm_f16tc_num_ctas(int M, int N) { return int(cdiv(M, BM) * cdiv(N, BN)); }

void gemm_f16tc(const F16GemmArgs& a, int kernel_class) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K <= 0) throw InvalidArgument("lp_matmul: empty input");
  if (a.A.ld % BKH || a.B.ld % BKH || a.A.ld < a.K || a.B.ld < a.K)
    throw InvalidArgument("gemm_f16tc: operand leading dimension must be a multiple of 64 >= K");
  constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024;
  static bool attr = false;
  if (!attr) {
    KP_CUDA(cudaFuncSetAttribute(gemm_f16tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(SMEM)));
    attr = true;
  }
  LaunchScope scope(kernel_class);
  gemm_f16tc_kernel<<<gemm_f16tc_num_ctas(a.M, a.N), THREADS, SMEM, ctx().stream>>>(a);
  check_launch("gemm_f16tc");
}

}  // namespace kp
