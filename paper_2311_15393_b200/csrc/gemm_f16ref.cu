// Reference-exact binary16 GEMM: C(m,n) = pairwise-tree over k of
// round16(A(m,k) * B(n,k)), each freshly formed sum rounded once — the value
// lp_matmul (lpblas.cpp:59-70 + pairwise_block_reduce :13-30) produces,
// computed per output element instead of materialising the m x (K n) matrix.
//
// Arithmetic: explicit mul.rn.f16x2 / add.rn.f16x2 (IEEE binary16, RNE,
// subnormals kept, no FMA contraction) on the CUDA-core f16x2 pipe — measured
// 36.9 T half-ops/s on B200 (profiles/r01_microbench_peaks.txt). The tensor
// pipe cannot be used: it accumulates in fp32 without per-add rounding.
//
// Tree bookkeeping: the stage tree of pairwise_block_reduce (adjacent pairs,
// odd tail carried) equals a binary counter over the leaves whose leftover
// levels are merged bottom-up at the end. Leaves are consumed in aligned
// 8-leaf register subtrees, two of which form a 16-leaf value pushed into a
// per-thread counter stack kept in shared memory (levels >= 4). Padded leaves
// (k in [K, ld)) are exact -0 products and leave every sum unchanged.
//
// Packing: one f16x2 register holds outputs (m, n) and (m, n+16) of the same
// k, so A is broadcast (PRMT) and all tree adds are vertical.
//
// Split K inside the CTA (KS = 2 or 4 groups of 128 threads, small
// products): when the padded k-tile count is KS * V with V a power of two,
// the tree over the KS * V units is KS complete subtrees of V units joined
// by a balanced top (a0 + a1 for KS = 2, (a0 + a1) + (a2 + a3) for KS = 4),
// so group g streams units [gV, (g+1)V) and group 0 adds the KS subtree
// values in that order — bit-identical, with KS times the warps per tile
// (a 256 x 256 product has only 64 tiles: latency-bound with one warp per
// SM sub-partition).
#include "gemm_f16ref.cuh"

#include <cstdlib>

namespace kp {
namespace {

constexpr int BKH = 64, THREADS = 128;
constexpr int ROW_BYTES = BKH * 2;  // 128
// Tiles BM x BN: BN = 64 (4 m-rows x 2 n-pairs = 8 packed accumulators per
// thread) or 32 (4 x 1; twice the CTAs and warps for problems too small to
// fill the SMs); BM = 32, or 16 (2 x 1) when even the 32 x 32 grid leaves SMs
// idle (a 256 x 256 product: 128 CTAs instead of 64).
constexpr int stage_bytes(int bm, int bn) { return (bm + bn) * ROW_BYTES; }
constexpr int nacc(int bm, int bn) { return (bm / 8) * (bn / 32); }
constexpr int GROUP_M = 8;

__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t lows(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x5410); }
__device__ __forceinline__ uint32_t highs(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x7632); }
__device__ __forceinline__ uint32_t bcast_lo(uint32_t a) { return __byte_perm(a, 0, 0x1010); }
__device__ __forceinline__ uint32_t bcast_hi(uint32_t a) { return __byte_perm(a, 0, 0x3232); }

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
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t part(const uint4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}

// STAGES: cp.async pipeline depth. UNIT: leaves per value pushed into the
// shared-memory counter stack (16: levels >= 4 in smem; 32: level 4 also in
// registers; 64: levels 4 and 5 in registers — the whole 64-leaf k-tile is
// reduced in registers and pushed once, the smallest stack).
template <int STAGES, int UNIT, int BN, int KS, int BM>
__global__ void __launch_bounds__(THREADS * KS) gemm_f16ref_kernel(const F16GemmArgs args, int levels) {
  pdl_wait();
  constexpr int NP = BN / 32, MI = BM / 8, NACC = nacc(BM, BN), STAGE_BYTES = stage_bytes(BM, BN);
  if (args.status && *args.status != 0) return;
  extern __shared__ __align__(128) unsigned char smem_all[];
  const int kgroup = KS > 1 ? int(threadIdx.x) / THREADS : 0;  // this thread's K range (split K)
  // per group: STAGES tiles, then its counter stack
  unsigned char* smem = smem_all + size_t(kgroup) * (STAGES * STAGE_BYTES + size_t(levels) * NACC * THREADS * 4);
  uint32_t* stack = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES);

  const int M = args.M, N = args.N;
  const int grid_m = (M + BM - 1) / BM, grid_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  const int group = pid / (GROUP_M * grid_n);
  const int first_m = group * GROUP_M;
  const int gsize = min(grid_m - first_m, GROUP_M);
  const int tile_m = first_m + (pid % (GROUP_M * grid_n)) % gsize;
  const int tile_n = (pid % (GROUP_M * grid_n)) / gsize;
  const int m_base = tile_m * BM, n_base = tile_n * BN;

  const int tid = int(threadIdx.x) - kgroup * THREADS, lane = tid & 31, warp = tid >> 5;
  const int tn = lane & 15, tm = warp * 2 + (lane >> 4);

  // K extent actually streamed: whole 64-wide tiles (padding is neutral);
  // with split K this group's KT of them, starting at k-tile kt0.
  const int KT_all = (args.K + BKH - 1) / BKH;
  const int KT = KT_all / KS, kt0 = kgroup * KT;
  const uint32_t sbase = smem_u32(smem);

  // Per-thread copy plan, computed once: chunk i of every k-tile is the 16-byte
  // piece id = tid + i * THREADS (ids < CA are A rows, the rest B rows), so
  // the k-loop only advances 64-bit source pointers (ALU adds, no IMADs on
  // the FMA pipe the f16x2 math needs).
  constexpr int CA = BM * 8, CB = BN * 8, NCH = (CA + CB) / THREADS;
  static_assert((CA + CB) % THREADS == 0 && CA % THREADS == 0, "copy plan");
  const __half* src0[NCH];
  uint32_t dst_off[NCH];
  bool valid[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int id = tid + i * THREADS;
    const bool isA = id < CA;  // compile-time per i (tid < THREADS)
    const int cid = isA ? id : id - CA;
    const int row = cid >> 3, ch = cid & 7;
    const int grow = (isA ? m_base : n_base) + row;
    valid[i] = grow < (isA ? M : N);
    const F16Operand& op = isA ? args.A : args.B;
    src0[i] = valid[i] ? op.p + long(grow) * op.ld + ch * 8 : op.p;
    dst_off[i] = (isA ? 0u : uint32_t(BM * ROW_BYTES)) +
                 uint32_t(row * ROW_BYTES + ((ch ^ (row & 7)) << 4));
  }
  auto load_tile = [&](int kt, int stage) {
    const uint32_t sa = sbase + uint32_t(stage * STAGE_BYTES);
#pragma unroll
    for (int i = 0; i < NCH; ++i)
      cp_async16(sa + dst_off[i], valid[i] ? src0[i] + (kt0 + kt) * BKH : src0[i], valid[i]);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }

  uint32_t l3[NACC], l4[NACC], l5[NACC];
  int c16 = 0;  // UNIT-leaf values pushed so far
  // Per-thread constants: rows tm + 8i (A) all share (row & 7) = tm, rows
  // tn + 16j (B) share tn & 7, so the swizzled chunk offset of sub-chunk s is
  // (s << 4) ^ x for one x per operand; the row offsets are immediates.
  const uint32_t a_off = uint32_t(tm * ROW_BYTES), b_off = uint32_t(BM * ROW_BYTES + tn * ROW_BYTES);
  const uint32_t xa = uint32_t((tm & 7) << 4), xb = uint32_t((tn & 7) << 4);
  uint32_t* const my_stack = stack + tid;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_tile(nk, nk % STAGES);
      cp_async_commit();
    }
    const uint32_t st = sbase + uint32_t((kt % STAGES) * STAGE_BYTES);
    const uint32_t sa = st + a_off, sb = st + b_off;
#pragma unroll
    for (int sub = 0; sub < 8; ++sub) {  // 8-leaf sub-chunk = one 16-byte smem chunk
      const uint32_t ca = uint32_t(sub << 4) ^ xa, cb = uint32_t(sub << 4) ^ xb;
      uint4 af[MI], bfr[2 * NP];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = lds128(sa + ca + uint32_t(i * 8 * ROW_BYTES));
#pragma unroll
      for (int j = 0; j < 2 * NP; ++j) bfr[j] = lds128(sb + cb + uint32_t(j * 16 * ROW_BYTES));
      uint32_t v8[NACC];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        uint32_t blo[4], bhi[4];
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          blo[kp] = lows(part(bfr[2 * p], kp), part(bfr[2 * p + 1], kp));
          bhi[kp] = highs(part(bfr[2 * p], kp), part(bfr[2 * p + 1], kp));
        }
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          uint32_t s4[4];
#pragma unroll
          for (int kp = 0; kp < 4; ++kp) {
            const uint32_t a = part(af[i], kp);
            const uint32_t p0 = hmul2(bcast_lo(a), blo[kp]);  // leaf k = 2kp
            const uint32_t p1 = hmul2(bcast_hi(a), bhi[kp]);  // leaf k = 2kp+1
            s4[kp] = hadd2(p0, p1);
          }
          v8[i * NP + p] = hadd2(hadd2(s4[0], s4[1]), hadd2(s4[2], s4[3]));
        }
      }
      if ((sub & 1) == 0) {
#pragma unroll
        for (int q = 0; q < NACC; ++q) l3[q] = v8[q];
      } else if (UNIT >= 32 && (sub & 3) == 1) {
#pragma unroll
        for (int q = 0; q < NACC; ++q) l4[q] = hadd2(l3[q], v8[q]);
      } else if (UNIT == 64 && sub == 3) {  // 32-leaf value (subs 0-3) stays in registers
#pragma unroll
        for (int q = 0; q < NACC; ++q) l5[q] = hadd2(l4[q], hadd2(l3[q], v8[q]));
      } else {
        uint32_t v[NACC];
#pragma unroll
        for (int q = 0; q < NACC; ++q) v[q] = hadd2(l3[q], v8[q]);
        if (UNIT >= 32) {
#pragma unroll
          for (int q = 0; q < NACC; ++q) v[q] = hadd2(l4[q], v[q]);
        }
        if (UNIT == 64) {  // one 64-leaf value per k-tile
#pragma unroll
          for (int q = 0; q < NACC; ++q) v[q] = hadd2(l5[q], v[q]);
        }
        uint32_t* lvl = my_stack;
        int cnt = c16;
        while (cnt & 1) {  // uniform across the CTA
#pragma unroll
          for (int q = 0; q < NACC; ++q) v[q] = hadd2(lvl[q * THREADS], v[q]);
          cnt >>= 1;
          lvl += NACC * THREADS;
        }
#pragma unroll
        for (int q = 0; q < NACC; ++q) lvl[q * THREADS] = v[q];
        ++c16;
      }
    }
  }
  cp_async_wait<0>();

  // Bottom-up merge of the leftover counter levels (bits of c16).
  uint32_t acc[NACC];
  bool have = false;
  for (int L = 0; L < levels; ++L) {
    if (!((c16 >> L) & 1)) continue;
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      const uint32_t s = stack[(L * NACC + q) * THREADS + tid];
      acc[q] = have ? hadd2(s, acc[q]) : s;
    }
    have = true;
  }
  if (!have) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) acc[q] = 0x80008000u;  // K == 0 cannot occur (checked)
  }
  if constexpr (KS > 1) {  // join the KS subtrees in tree order; group 0 finishes
    uint32_t* xch = reinterpret_cast<uint32_t*>(smem_all);  // the stage buffers are free now
    __syncthreads();
    if (kgroup > 0) {
#pragma unroll
      for (int q = 0; q < NACC; ++q) xch[((kgroup - 1) * NACC + q) * THREADS + tid] = acc[q];
    }
    __syncthreads();
    if (kgroup > 0) return;
    uint32_t a1[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) a1[q] = xch[q * THREADS + tid];
    if constexpr (KS == 2) {
#pragma unroll
      for (int q = 0; q < NACC; ++q) acc[q] = hadd2(acc[q], a1[q]);
    } else {
#pragma unroll
      for (int q = 0; q < NACC; ++q) {
        const uint32_t a2 = xch[(1 * NACC + q) * THREADS + tid], a3 = xch[(2 * NACC + q) * THREADS + tid];
        acc[q] = hadd2(hadd2(acc[q], a1[q]), hadd2(a2, a3));
      }
    }
  }

  // ---- epilogue ----
  const F16Epilogue& e = args.epi;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  // batched products: this tile's image (tiles never straddle images)
  int nl_base;
  const int img = epi_image(e, n_base, nl_base);
  const int NL = e.n_img ? e.n_img : N;
  __half* const Ch = e.Ch ? e.Ch + img * e.c_img : nullptr;
  double* const Cd = e.Cd ? e.Cd + img * e.c_img : nullptr;
  const __half* const scale = e.scale ? e.scale + img * e.s_img : nullptr;
  const double* const d0 = e.d0 ? e.d0 + img * e.v_img : nullptr;
  const double* const d1a = e.d1a ? e.d1a + img * e.v_img : nullptr;
  const double* const d1b = e.d1b ? e.d1b + img * e.v_img : nullptr;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m_base + tm + 8 * i;
        const int n = nl_base + tn + 32 * p + 16 * h;  // image-local column
        if (m >= M || n >= NL) continue;
        const uint32_t word = acc[i * NP + p];
        const unsigned short bits = h ? (unsigned short)(word >> 16) : (unsigned short)(word & 0xffffu);
        if (e.mode == F16OUT_HALF) {
          Ch[long(m) * e.cm + long(n) * e.cn] = __ushort_as_half(bits);
        } else if (e.mode == F16OUT_HALF_SCALED) {
          const __half sc = scale[long(m) * e.sm + long(n) * e.sn];
          unsigned short r;
          asm("mul.rn.f16 %0, %1, %2;" : "=h"(r) : "h"(__half_as_ushort(sc)), "h"(bits));
          Ch[long(m) * e.cm + long(n) * e.cn] = __ushort_as_half(r);
        } else {
          const double v = double(__half2float(__ushort_as_half(bits)));
          Cd[long(m) * e.cm + long(n) * e.cn] = v;
          if (e.partials) {
            const long vi = long(m) * e.vm + long(n) * e.vn;
            if (d0) s0 += v * d0[vi];
            if (d1a) s1 += v * (d1b ? (d1a[vi] - d1b[vi]) : d1a[vi]);
            if (!isfinite(v)) s2 += 1.0;
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
    asm volatile("bar.sync 1, %0;\n" ::"n"(THREADS) : "memory");  // group 0's warps only
    if (tid == 0) {
      double a0 = 0, a1 = 0, a2 = 0;
      for (int w = 0; w < THREADS / 32; ++w) a0 += red[w][0], a1 += red[w][1], a2 += red[w][2];
      // batched: per-image slot = the tile's position in that image's own grid
      const long slot = e.n_img ? long(img) * e.part_img + long(tile_m) * (e.n_img / BN) + nl_base / BN
                                : long(tile_m) * grid_n + tile_n;
      double* o = e.partials + slot * 4;
      o[0] = a0, o[1] = a1, o[2] = a2, o[3] = 0.0;
    }
  }
}

__global__ void fill_u16_kernel(unsigned short* p, size_t n, unsigned short bits) {
  pdl_wait();
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    p[i] = bits;
}

// Tile width for an M x N product: BN = 32 when the 32 x 64 tiles alone would
// give fewer than 8 CTAs per SM (n <= 1024), else 64.
int f16ref_bn(int M, int N) {
  static const int forced = [] {
    const char* e = getenv("KP_F16REF_BN");
    return e ? atoi(e) : 0;
  }();
  if (forced == 32 || forced == 64) return forced;
  return cdiv(M, 32) * cdiv(N, 64) < 8 * ctx().num_sms ? 32 : 64;
}
// Tile height: 16 when the 32 x 32 grid has fewer CTAs than SMs (n < ~390),
// else 32. KP_F16REF_BM=32 forces 32.
int f16ref_bm(int M, int N) {
  static const int forced = [] {
    const char* e = getenv("KP_F16REF_BM");
    return e ? atoi(e) : 0;
  }();
  if (forced == 32) return 32;
  return f16ref_bn(M, N) == 32 && cdiv(M, 32) * cdiv(N, 32) < ctx().num_sms ? 16 : 32;
}

template <int STAGES, int UNIT, int BN, int KS, int BM>
void launch_f16ref_bn(const F16GemmArgs& a, int kernel_class) {
  const int kt = (a.K + BKH - 1) / BKH / KS;
  const int units = kt * (BKH / UNIT);
  int levels = 1;
  while ((1 << levels) <= units) ++levels;
  const size_t smem =
      size_t(KS) * (size_t(STAGES) * stage_bytes(BM, BN) + size_t(levels) * nacc(BM, BN) * THREADS * 4);
  auto kern = gemm_f16ref_kernel<STAGES, UNIT, BN, KS, BM>;
  set_smem_limit(reinterpret_cast<const void*>(kern), smem);
  LaunchScope scope(kernel_class);
  const unsigned grid = cdiv(a.M, BM) * cdiv(a.N, BN);
  launch_pdl(kern, dim3(grid), dim3(THREADS * KS), smem, a, levels);
  check_launch("gemm_f16ref");
}

// Split K inside the CTA (see the header) when the tile grid cannot fill
// the SMs (< 2 CTAs per SM) and the padded k-tile count is KS times a power
// of two. KP_F16REF_KSPLIT=1 disables.
int f16ref_ksplit(int tiles, int K) {
  static const int off = [] {
    const char* e = getenv("KP_F16REF_KSPLIT");
    return e && atoi(e) == 1;
  }();
  if (off || tiles >= 2 * ctx().num_sms) return 1;
  const int kt = (K + BKH - 1) / BKH;
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  if (kt % 4 == 0 && pow2(kt / 4)) return 4;
  if (kt % 2 == 0 && pow2(kt / 2)) return 2;
  return 1;
}

template <int STAGES, int UNIT, int BN, int BM>
void launch_f16ref_ks(const F16GemmArgs& a, int kernel_class) {
  const int tiles = int(cdiv(a.M, BM) * cdiv(a.N, BN));
  switch (f16ref_ksplit(tiles, a.K)) {
    case 4: launch_f16ref_bn<STAGES, UNIT, BN, 4, BM>(a, kernel_class); break;
    case 2: launch_f16ref_bn<STAGES, UNIT, BN, 2, BM>(a, kernel_class); break;
    default: launch_f16ref_bn<STAGES, UNIT, BN, 1, BM>(a, kernel_class); break;
  }
}

template <int STAGES, int UNIT>
void launch_f16ref(const F16GemmArgs& a, int kernel_class) {
  // batched products take the tile shape of one image's product, so every
  // image is tiled (and its partials grouped) exactly as a single product
  const int nimg = a.epi.n_img ? a.epi.n_img : a.N;
  if (f16ref_bn(a.M, nimg) == 64)
    launch_f16ref_ks<STAGES, UNIT, 64, 32>(a, kernel_class);
  else if (f16ref_bm(a.M, nimg) == 32)
    launch_f16ref_ks<STAGES, UNIT, 32, 32>(a, kernel_class);
  else
    launch_f16ref_ks<STAGES, UNIT, 32, 16>(a, kernel_class);
}

int f16ref_cfg() {
  static int cfg = [] {
    const char* e = getenv("KP_F16REF_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

}  // namespace

int gemm_f16ref_num_ctas(int M, int N) { return int(cdiv(M, f16ref_bm(M, N)) * cdiv(N, f16ref_bn(M, N))); }
int gemm_f16ref_partials_per_image(int M, int N, int n_img) {
  return int(cdiv(M, f16ref_bm(M, n_img)) * (n_img / f16ref_bn(M, n_img)));
}

void gemm_f16ref(const F16GemmArgs& a, int kernel_class) {
  if (a.M <= 0 || a.N <= 0) return;
  if (a.K <= 0) throw InvalidArgument("lp_matmul: empty input");
  if (a.A.ld % BKH || a.B.ld % BKH || a.A.ld < a.K || a.B.ld < a.K)
    throw InvalidArgument("gemm_f16ref: operand leading dimension must be a multiple of 64 >= K");
  // n=4096 (profiles/r01_sweep_f16ref.txt): <3,16> 30.45, <2,32> 31.21,
  // <3,32> 31.38, <2,16> 30.51, <2,64> 31.83, <3,64> 31.49 T half-ops/s; all
  // bit-identical. <2,64> keeps the smallest counter stack (4 CTAs / SM).
  switch (f16ref_cfg()) {
    case 1: launch_f16ref<2, 32>(a, kernel_class); break;
    case 2: launch_f16ref<3, 32>(a, kernel_class); break;
    case 3: launch_f16ref<2, 16>(a, kernel_class); break;
    case 4: launch_f16ref<3, 16>(a, kernel_class); break;
    case 6: launch_f16ref<3, 64>(a, kernel_class); break;
    default: launch_f16ref<2, 64>(a, kernel_class); break;
  }
}

void fill_u16(__half* p, size_t count, uint16_t bits) {
  if (!count) return;
  LaunchScope scope(KC_VECTOR);
  const unsigned grid = std::min<unsigned>(cdiv(long(count), 256), 4096u);
  fill_u16_kernel<<<grid, 256, 0, ctx().stream>>>(reinterpret_cast<unsigned short*>(p), count, bits);
  check_launch("fill_u16");
}

}  // namespace kp
