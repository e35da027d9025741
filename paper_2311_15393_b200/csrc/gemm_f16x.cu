// Reference-exact binary16 GEMM with the rounded products made on the tcgen05
// tensor pipe: C(m,n) = pairwise tree over k of round16(A(m,k) * B(n,k)),
// every freshly formed sum rounded once — the value lp_matmul
// (lpblas.cpp:59-70, pairwise_block_reduce :13-30) produces, bit for bit (see
// "signed zeros" below), same operand / epilogue contract as gemm_f16ref.
//
// Products. A kind::f16 MMA whose B operand is "diagonal-expanded" — column
// c = kl*8 + jl of the expanded B has exactly one live k (= kl) — computes
// D(m, c) = A(m, kl) * B(jl, kl) as a single exact product; with an f16
// accumulator that is round16(a*b) (one RNE rounding of an exact product),
// i.e. the reference's rounded leaf (lpblas.cpp:65-67). Measured on B200 over
// 1.45e9 random products (all bit classes incl. subnormal, inf, NaN operands
// in B; tools/microbench/tcx.cu, profiles/r02_microbench_tcx.txt): every
// nonzero and NaN leaf equals mul.rn.f16; only the sign of zero leaves can
// differ. One MMA (M=128, N=128, K=16) makes 16 k-leaves for 8 outputs of
// 128 rows; the f16x2 pipe is left with the tree adds only (HADD2), which
// halves its load against gemm_f16ref (HMUL2 + HADD2 per leaf pair).
//
// Signed zeros. Let a leaf be "zero" if round16(a*b) = +-0. If an output has
// any nonzero leaf, every node of its tree is either an all-zero subtree or
// carries the same bits in both computations (x + +-0 = x; a zero reached by
// cancellation is +0 under RNE and absorbs any zero sibling), so the output
// is bit-identical. An output all of whose leaves are zero is -0 iff every
// leaf is -0, i.e. iff sign(A(m,k)) != sign(B(n,k)) for every k < K (the
// product sign rule holds for underflowed and exact-zero products alike).
// The epilogue lists the outputs whose tree value is +-0; a small fix-up
// kernel recomputes exactly those signs from the operands. Zero
// outputs are rare (all 4096 leaves must vanish), so the fix-up is almost
// always a no-op launch.
//
// Non-finite operands. Expanded-B filler entries are +0 and multiply every A
// value of the slice, so A must be finite (inf * 0 = NaN would leak into
// other columns). The M-solve passes the (finite) singular-vector factors as
// A and the data (residual, intermediates — possibly inf) as B; lp_matmul
// checks A first and otherwise uses gemm_f16ref.
//
// Structure (persistent, one CTA per SM, 640 threads):
//   warp 0      TMA: A tile 128 x 64 (SWIZZLE_128B) + raw B tile 32 x 64
//   warp 1      TMEM alloc (512 columns = 2 leaf buffers of 256), one
//               lane issues the 8 MMAs of a stage (4 k-slices x 2 halves of
//               16 outputs, N = 256), one tcgen05.commit per buffer
//   warps 2-3   expanders: scatter the raw B tile into the double-buffered
//               expanded tiles (4 groups x 128 rows x 64 k, zeros in place)
//   warps 4-19  epilogue: set g (4 warps, one per TMEM lane quadrant) drains
//               columns (g%2)*128.. of buffer g/2 (tcgen05.ld
//               32x32b.x64.pack::16b), forms 16-leaf
//               HADD2 trees, keeps the per-output binary counter (64-leaf
//               units; levels 0-2 in registers, higher levels in smem) and
//               writes the fused epilogue at the end of the tile.
// Tile: 128 rows x 32 outputs; grouped rasterisation over the tile sequence.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include "gemm_f16ref.cuh"
#include "gemm_f16x.cuh"

namespace kp {
namespace {

#ifndef KP_F16X_TRACE
#define KP_F16X_TRACE 0
#endif
#ifndef KP_F16X_NSTAGE
#define KP_F16X_NSTAGE 2
#endif
#ifndef KP_F16X_REGLV
#define KP_F16X_REGLV 2
#endif
constexpr int BM = 128, BN = 32, BK = 64, NSTAGE = KP_F16X_NSTAGE, NGROUP = 4, NCOL = 128;
#ifndef KP_F16X_PAIR
#define KP_F16X_PAIR 1
#endif
// Measured and removed (profiles/r02_f16x_variants.txt, r02_f16x_timeline.txt):
// releasing the buffer before tcgen05.wait::ld (wrong results), two 64-column
// loads per step in the 16-warp kernel with or without overlapped adds, a
// barrier-enforced alternation of the two buffers' warps between loading and
// adding (3.47 ms).
#ifndef KP_F16X_NISS
#define KP_F16X_NISS 1
#endif
// KP_F16X_NISS: MMA-issuing threads. 1: warp 1 issues every buffer, warps 2-3
// expand B. 2: warps 1 and 2 issue the even / odd TMEM buffers (an MMA +
// commit costs the issuing thread ~120 cycles), warp 3 expands alone.
constexpr int NISS = KP_F16X_NISS;
constexpr int GPB = KP_F16X_PAIR ? 2 : 1;             // output groups per TMEM buffer
constexpr int NMMA = GPB * NCOL, NBUF = NGROUP / GPB;
// KP_F16X_W8: 8 epilogue warps with two output groups each (one per TMEM
// buffer) and software-pipelined 64-column loads (140 registers, every load
// under the adds of the previous chunk), instead of 16 warps with one group
// and one 128-column load per step. Bit-identical; measured slower (3.113 vs
// 2.888 ms at n = 4096, profiles/r02_f16x_variants.txt), so off.
#ifndef KP_F16X_W8
#define KP_F16X_W8 0
#endif
static_assert(!KP_F16X_W8 || (KP_F16X_PAIR == 1 && !KP_F16X_TRACE), "W8 needs the paired buffers; the timeline build is the 16-warp kernel");
constexpr int NSET = KP_F16X_W8 ? 2 : 1;  // output groups per epilogue thread
constexpr int EPI_WARPS = 16 / NSET, EPI_THREADS = 32 * EPI_WARPS;
constexpr int NUM_THREADS = 32 * 4 + EPI_THREADS;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int BRAW_BYTES = BN * BK * 2;         // 4 KB
constexpr int STAGE_BYTES = A_BYTES + BRAW_BYTES;
constexpr int BEXP_GROUP_BYTES = NCOL * BK * 2; // 16 KB: 128 expanded rows x 64 k
constexpr int BEXP_BYTES = NGROUP * BEXP_GROUP_BYTES;
constexpr int REG_LEVELS = KP_F16X_REGLV;       // counter levels kept in registers (2 or 3)

#if KP_F16X_TRACE
// Timeline instrumentation (profiling builds only): clock64 stamps of CTA 0's
// second tile. [0, 4096): issuer(s), ((kt*4+kk)*NBUF+h)*4 + {before tempty
// wait, after it, after mma+commit, -}; [4096, 4096 + 2*256*8): epilogue warps
// 4 and 12, (kt*4+kk)*8 + {before tfull wait, after, after wait::ld, after
// arrive, after adds}; [8192 + 256*issuer, +64*4): issuer stage waits.
__device__ long long f16x_trace[16384];
#define TR(cond, idx) do { if (cond) f16x_trace[idx] = clock64(); } while (0)
#else
#define TR(cond, idx) do { } while (0)
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
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
#ifndef KP_F16X_SUSPEND
#define KP_F16X_SUSPEND 0
#endif
// Epilogue waits: with a suspend-time hint the waiting warp sleeps until the
// phase completes instead of re-polling (the polls take issue slots from the
// warps doing the tree adds on the same sub-partition).
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
#if KP_F16X_SUSPEND
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity), "n"(KP_F16X_SUSPEND)
      : "memory");
#else
  mbar_wait(bar, parity);
#endif
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
// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05, version 1).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
// kind::f16, D = F16 (bits 4-5 = 0), A = B = F16, K-major, M = 128, N = 128.
__device__ __forceinline__ void umma_leaves(uint32_t tmem_d, uint64_t da, uint64_t db) {
  constexpr uint32_t IDESC = (uint32_t(NMMA >> 3) << 17) | (uint32_t(BM >> 4) << 24);
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
#define R8(i) "=r"(v[i + 0]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), \
              "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
// 128 TMEM columns of 16-bit leaves -> 64 registers, adjacent columns packed
// (asynchronous: tmem_ld_wait() before the registers are read)
__device__ __forceinline__ void tmem_ld128_pack(uint32_t ta, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56)
      : "r"(ta));
}
#define R8(i) "=r"(v[i + 0]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), \
              "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
// 64 TMEM columns -> 32 registers, adjacent columns packed (asynchronous)
__device__ __forceinline__ void tmem_ld64_pack(uint32_t ta, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : R8(0), R8(8), R8(16), R8(24)
      : "r"(ta));
}
#undef R8
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
#undef R8

// byte offset of element (row, k) in a SWIZZLE_128B K-major tile (64-wide rows)
__device__ __forceinline__ uint32_t swz(int row, int k) {
  return uint32_t((row >> 3) * 1024 + (row & 7) * 128 + (((k >> 3) ^ (row & 7)) << 4) + (k & 7) * 2);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_f16x_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const F16GemmArgs args, int levels, int xflags) {
  pdl_wait();
  if (args.status && *args.status != 0) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* bexp = smem + NSTAGE * STAGE_BYTES;
  uint32_t* stack = reinterpret_cast<uint32_t*>(bexp + 2 * BEXP_BYTES);
  __shared__ __align__(8) uint64_t full_bar[NSTAGE], empty_bar[NSTAGE];
  __shared__ __align__(8) uint64_t bfull_bar[2], bempty_bar[2];
  __shared__ __align__(8) uint64_t tfull_bar[NBUF], tempty_bar[NBUF];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[EPI_WARPS][3];

  const int M = args.M, N = args.N;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int KT = (args.K + BK - 1) / BK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem), bbase = smem_u32(bexp);

  // expanded-B buffers: zeros everywhere; the expander only ever rewrites the
  // live positions (row c = kl*8 + jl, k = 16*kk + kl)
  for (int i = tid; i < 2 * BEXP_BYTES / 16; i += NUM_THREADS)
    reinterpret_cast<uint4*>(bexp)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(smem_u32(&full_bar[s]), 1), mbar_init(smem_u32(&empty_bar[s]), NISS);
    for (int s = 0; s < 2; ++s)
      mbar_init(smem_u32(&bfull_bar[s]), NISS == 1 ? 2 : 1), mbar_init(smem_u32(&bempty_bar[s]), NISS);
    for (int h = 0; h < NBUF; ++h)
      mbar_init(smem_u32(&tfull_bar[h]), 1), mbar_init(smem_u32(&tempty_bar[h]), 4 * GPB);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        smem_u32(&tmem_base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  auto tile_coords = [&](int t, int& mb, int& nb) {
    constexpr int GROUP = 8;
    const int group = t / (GROUP * tiles_n);
    const int first = group * GROUP;
    const int gs = min(tiles_m - first, GROUP);
    mb = (first + (t % (GROUP * tiles_n)) % gs) * BM;
    nb = ((t % (GROUP * tiles_n)) / gs) * BN;
  };

  if (warp == 0) {
    if (lane == 0 && !(xflags & 8)) {  // ===== TMA producer =====
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
          tma_load_2d(sa, &map_a, fb, kt * BK, mb);
          tma_load_2d(sa + A_BYTES, &map_b, fb, kt * BK, nb);
          if (++stage == NSTAGE) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1 || (NISS == 2 && warp == 2)) {
    if (lane == 0) {  // ===== MMA issuer(s) =====
      const int h0 = warp - 1;  // first buffer of this issuer (stride NISS)
      const uint32_t tfull0 = smem_u32(&tfull_bar[0]), tempty0 = smem_u32(&tempty_bar[0]);
      int stage = 0;
      uint32_t phase = 0;
      int bi = 0;  // expanded-B buffer use counter
      uint32_t tphase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        [[maybe_unused]] const bool tr = t == blockIdx.x + gridDim.x && blockIdx.x == 0 && KT == 64;
        for (int kt = 0; kt < KT; ++kt, ++bi) {
          const int b = bi & 1;
          TR(tr, 8192 + (warp - 1) * 256 + kt * 4 + 0);
          if (!(xflags & 8)) mbar_wait(smem_u32(&full_bar[stage]), phase);                    // A landed
          TR(tr, 8192 + (warp - 1) * 256 + kt * 4 + 1);
          if (!(xflags & 2)) mbar_wait(smem_u32(&bfull_bar[b]), uint32_t((bi >> 1) & 1));     // B expanded
          TR(tr, 8192 + (warp - 1) * 256 + kt * 4 + 2);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          // descriptors: the start-address field advances by 2 per 32-byte k-slice
          const uint64_t da = make_desc(sbase + uint32_t(stage * STAGE_BYTES));
          const uint64_t db = make_desc(bbase + uint32_t(b * BEXP_BYTES));
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // one N = 128 MMA per output group g into its own TMEM buffer, so
            // each epilogue set waits only on its own leaves
#pragma unroll
            for (int h = h0; h < NBUF; h += NISS) {
              TR(tr, ((kt * 4 + kk) * NBUF + h) * 4 + 0);
              mbar_wait(tempty0 + 8 * h, tphase ^ 1);
              TR(tr, ((kt * 4 + kk) * NBUF + h) * 4 + 1);
              asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
              umma_leaves(tmem + uint32_t(h * NMMA), da + uint64_t(2 * kk),
                          db + uint64_t(((xflags & 1 ? 0 : h) * GPB * BEXP_GROUP_BYTES) >> 4) + uint64_t(2 * kk));
              umma_commit(tfull0 + 8 * h);
              TR(tr, ((kt * 4 + kk) * NBUF + h) * 4 + 2);
            }
            tphase ^= 1;
          }
          umma_commit(smem_u32(&empty_bar[stage]));  // A / raw B stage reusable
          umma_commit(smem_u32(&bempty_bar[b]));     // expanded-B buffer reusable
          if (++stage == NSTAGE) stage = 0, phase ^= 1;
        }
      }
    }
  } else if ((NISS == 1 && warp == 2) || warp == 3) {  // ===== B expanders =====
    // lane j scatters raw row j (output column nb + j): element k goes to
    // group j/8, expanded row (k%16)*8 + j%8, column k. Warp 2 takes
    // k = 0..31, warp 3 k = 32..63. With k = 8ch + e the swizzled offset is
    // (8(ch&1) + e)*1024 + (j%8)*128 + ((ch ^ j%8) << 4) + 2e.
    int stage = 0;
    uint32_t phase = 0;
    int bi = 0;
    constexpr int NCH = NISS == 1 ? 4 : 8;  // 16-byte k chunks per expander warp
    const int jl = lane & 7, ch0 = NISS == 1 ? (warp - 2) * 4 : 0;
    const uint32_t lane_off = uint32_t((lane >> 3) * BEXP_GROUP_BYTES + jl * 128);
    uint32_t xo[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) xo[c] = uint32_t(((ch0 + c) ^ jl) << 4);
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kt = 0; kt < KT; ++kt, ++bi) {
        const int b = bi & 1;
        if (!(xflags & 8)) mbar_wait(smem_u32(&full_bar[stage]), phase);
        mbar_wait(smem_u32(&bempty_bar[b]), uint32_t(((bi >> 1) & 1) ^ 1));
        const unsigned char* raw = smem + stage * STAGE_BYTES + A_BYTES + lane * (BK * 2) + ch0 * 16;
        unsigned char* dst = bexp + b * BEXP_BYTES + lane_off;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const uint4 q = *reinterpret_cast<const uint4*>(raw + c * 16);
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
          unsigned char* d = dst + xo[c] + ((ch0 + c) & 1) * 8 * 1024;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            *reinterpret_cast<unsigned short*>(d + e * 1024 + 2 * e) =
                (unsigned short)(w[e >> 1] >> ((e & 1) * 16));
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bfull_bar[b]));
        if (++stage == NSTAGE) stage = 0, phase ^= 1;
      }
    }
  } else if (warp >= 4) {  // ===== epilogue sets =====
    const int et = tid - 128;              // 0..EPI_THREADS-1
    const int quad = warp & 3;             // TMEM lane quadrant
    // Output groups of this thread: NSET = 1: group (warp-4)/4; NSET = 2 (8
    // epilogue warps): groups half and half + 2 - one from each TMEM buffer.
    const int g0 = (warp - 4) >> 2;
    const uint32_t tlane = tmem + (uint32_t(quad * 32) << 16);
    const F16Epilogue& e = args.epi;
    const int SL = levels > REG_LEVELS ? levels - REG_LEVELS : 0;  // counter levels kept in shared memory
    uint32_t tphase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, mb, nb);
      uint32_t r0[NSET][4], r1[NSET][4], r2[NSET][4], p01[NSET][4], v64[NSET][4];
      int cnt[NSET];
#pragma unroll
      for (int st = 0; st < NSET; ++st) cnt[st] = 0;
      // push the 64-leaf unit v64[st] into the per-output binary counter
      // (the low REG_LEVELS levels in registers, higher levels in shared memory)
      auto push_unit = [&](const int st) {
        uint32_t* const stk = stack + size_t(st) * SL * 4 * EPI_THREADS;
        const int cn = cnt[st];
        if (!(cn & 1)) {
#pragma unroll
          for (int p = 0; p < 4; ++p) r0[st][p] = v64[st][p];
        } else {
#pragma unroll
          for (int p = 0; p < 4; ++p) v64[st][p] = hadd2(r0[st][p], v64[st][p]);
          if (!(cn & 2)) {
#pragma unroll
            for (int p = 0; p < 4; ++p) r1[st][p] = v64[st][p];
          } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) v64[st][p] = hadd2(r1[st][p], v64[st][p]);
            bool carry = true;
            if constexpr (REG_LEVELS == 3) {
              if (!(cn & 4)) {
#pragma unroll
                for (int p = 0; p < 4; ++p) r2[st][p] = v64[st][p];
                carry = false;
              } else {
#pragma unroll
                for (int p = 0; p < 4; ++p) v64[st][p] = hadd2(r2[st][p], v64[st][p]);
              }
            }
            if (carry) {
              int c = cn >> REG_LEVELS, lvl = 0;
              while (c & 1) {
#pragma unroll
                for (int p = 0; p < 4; ++p) v64[st][p] = hadd2(stk[(lvl * 4 + p) * EPI_THREADS + et], v64[st][p]);
                c >>= 1;
                ++lvl;
              }
#pragma unroll
              for (int p = 0; p < 4; ++p) stk[(lvl * 4 + p) * EPI_THREADS + et] = v64[st][p];
            }
          }
        }
        cnt[st] = cn + 1;
      };
      // merge the 16-leaf sum s16 of k-slice kk into the 64-leaf unit of set st
      auto merge16 = [&](const int st, const int kk, const uint32_t (&s16)[4]) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          if (kk == 0 || kk == 2) v64[st][p] = s16[p];
          else if (kk == 1) p01[st][p] = hadd2(v64[st][p], s16[p]);
          else v64[st][p] = hadd2(p01[st][p], hadd2(v64[st][p], s16[p]));
        }
        if (kk == 3) push_unit(st);
      };
#if KP_F16X_W8
      // 8 epilogue warps, two per sub-partition: every 64-column load runs
      // under the tree adds of the previously loaded 64 columns, and a warp
      // alternates between the two TMEM buffers (X / Y: the two leaf chunks).
      uint32_t X[32], Y[32], h0[4];
      auto tree8 = [&](const uint32_t (&v)[32], uint32_t (&o)[4]) {  // v[kl*4 + p], 8 leaves per output
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t a = hadd2(hadd2(v[0 * 4 + p], v[1 * 4 + p]), hadd2(v[2 * 4 + p], v[3 * 4 + p]));
          const uint32_t b = hadd2(hadd2(v[4 * 4 + p], v[5 * 4 + p]), hadd2(v[6 * 4 + p], v[7 * 4 + p]));
          o[p] = hadd2(a, b);
        }
      };
      auto finish = [&](const int st, const int kk) {  // s16 = h0 + tree8(Y)
        uint32_t hi[4], s16[4];
        tree8(Y, hi);
#pragma unroll
        for (int p = 0; p < 4; ++p) s16[p] = hadd2(h0[p], hi[p]);
        merge16(st, kk, s16);
      };
      const uint32_t tfull0 = smem_u32(&tfull_bar[0]), tempty0 = smem_u32(&tempty_bar[0]);
      for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
          for (int st = 0; st < 2; ++st) {
            const uint32_t tb = tlane + uint32_t(st * NMMA + g0 * NCOL);
            mbar_wait_sleep(tfull0 + 8 * st, tphase);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            tmem_ld64_pack(tb, X);  // leaves kl = 0..7
            // the previous chunk pair (other buffer): its second half is still in Y
            if (st == 1) finish(0, kk);
            else if (kk > 0) finish(1, kk - 1);
            else if (kt > 0) finish(1, 3);
            tmem_ld_wait();
            tmem_ld64_pack(tb + 64, Y);  // leaves kl = 8..15
            tree8(X, h0);
            tmem_ld_wait();
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty0 + 8 * st);
          }
          tphase ^= 1;
        }
      }
      finish(1, 3);
#else
      [[maybe_unused]] const bool tr =
          t == blockIdx.x + gridDim.x && blockIdx.x == 0 && KT == 64 && lane == 0 && (warp == 4 || warp == 12);
      [[maybe_unused]] const int trb = 4096 + (warp == 12 ? 2048 : 0);
      const uint32_t my_tfull = smem_u32(&tfull_bar[g0 / GPB]), my_tempty = smem_u32(&tempty_bar[g0 / GPB]);
      const uint32_t tbuf = tlane + uint32_t(g0 * NCOL);
      for (int kt = 0; kt < KT; ++kt) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          TR(tr, trb + (kt * 4 + kk) * 8 + 0);
          mbar_wait_sleep(my_tfull, tphase);
          TR(tr, trb + (kt * 4 + kk) * 8 + 1);
          tphase ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          // 16-leaf trees of outputs (2p, 2p+1): leaves kl = 0..15 sit in
          // TMEM columns kl*8 + jl; s16 = ((l0+l1)+(l2+l3) + ...) exactly as
          // pairwise_block_reduce pairs them
          uint32_t s16[4];
          {
            uint32_t v[64];  // v[kl*4 + p]
            tmem_ld128_pack(tbuf, v);  // two x32 loads in flight under one wait: 3.16 vs 2.89 ms
            tmem_ld_wait();  // required before the release: an early arrive was measured wrong
            TR(tr, trb + (kt * 4 + kk) * 8 + 2);
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(my_tempty);
            TR(tr, trb + (kt * 4 + kk) * 8 + 3);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              uint32_t s8[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) s8[q] = hadd2(v[(2 * q) * 4 + p], v[(2 * q + 1) * 4 + p]);
              const uint32_t a = hadd2(s8[0], s8[1]), b = hadd2(s8[2], s8[3]);
              const uint32_t c = hadd2(s8[4], s8[5]), d = hadd2(s8[6], s8[7]);
              s16[p] = hadd2(hadd2(a, b), hadd2(c, d));
            }
          }
          merge16(0, kk, s16);
#if KP_F16X_TRACE
          if (tr) { asm volatile("" ::"r"(v64[0][0]), "r"(v64[0][1]), "r"(v64[0][2]), "r"(v64[0][3])); }
          TR(tr, trb + (kt * 4 + kk) * 8 + 4);
#endif
        }
      }
#endif
      const int m = mb + quad * 32 + lane;
      int nlb;
      const int img = epi_image(e, nb, nlb);
      const int NL = e.n_img ? e.n_img : N;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int st = 0; st < NSET; ++st) {
      const int g = g0 + 2 * st;
      // bottom-up merge of the leftover counter levels (bits of cnt)
      uint32_t acc[4];
      bool have = false;
      const uint32_t* const stk = stack + size_t(st) * SL * 4 * EPI_THREADS;
      for (int L = 0; L < levels; ++L) {
        if (!((cnt[st] >> L) & 1)) continue;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t s = L == 0                      ? r0[st][p]
                             : L == 1                      ? r1[st][p]
                             : (REG_LEVELS == 3 && L == 2) ? r2[st][p]
                                                           : stk[((L - REG_LEVELS) * 4 + p) * EPI_THREADS + et];
          acc[p] = have ? hadd2(s, acc[p]) : s;
        }
        have = true;
      }
      // ---- epilogue: row m, outputs n0 .. n0+7 (image-local; see F16Epilogue) ----
      const int n0 = nlb + g * 8;
      const int ng0 = nb + g * 8;  // global column (B operand row, hash index)
      uint32_t zbits = 0;  // outputs whose tree value is +-0
      if (m < M) {
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (((acc[p] >> (16 * h)) & 0x7fffu) == 0 && n0 + 2 * p + h < NL) zbits |= 1u << (2 * p + h);
        if (zbits) {
          // Zero outputs: the reference value is -0 iff sign(A(m,k)) != sign(B(n,k))
          // for all k < K. Necessary condition on the row sign hashes:
          // hash_a[m] + hash_b[n] == hsum. Otherwise the value is +0 (set here);
          // candidates keep their bits and go to the exact fix-up.
          const unsigned long long ha = args.hash_a[m];
          uint32_t cand = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (((zbits >> q) & 1) && ha + args.hash_b[ng0 + q] == args.hsum) cand |= 1u << q;
          const uint32_t plus = zbits & ~cand;
#pragma unroll
          for (int p = 0; p < 4; ++p)
            acc[p] &= ~((((plus >> (2 * p)) & 1) ? 0x8000u : 0u) | (((plus >> (2 * p + 1)) & 1) ? 0x80000000u : 0u));
          zbits = cand;
        }
        const bool full = n0 + 8 <= NL;
        __half* const Ch = e.Ch ? e.Ch + img * e.c_img : nullptr;
        if (e.mode == F16OUT_HALF) {
          if (full && e.cn == 1 && ((e.cm * m + n0) & 7) == 0) {
            *reinterpret_cast<uint4*>(Ch + long(m) * e.cm + n0) = make_uint4(acc[0], acc[1], acc[2], acc[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (n0 + q < NL)
                Ch[long(m) * e.cm + long(n0 + q) * e.cn] =
                    __ushort_as_half((unsigned short)((acc[q >> 1] >> (16 * (q & 1))) & 0xffffu));
          }
        } else if (e.mode == F16OUT_HALF_SCALED) {  // w = round16(S .* t2)
          const __half* const scale = e.scale + img * e.s_img;
          uint32_t sc[4];
          if (full && e.sn == 1 && ((e.sm * m + n0) & 7) == 0) {
            const uint4 s4 = *reinterpret_cast<const uint4*>(scale + long(m) * e.sm + n0);
            sc[0] = s4.x, sc[1] = s4.y, sc[2] = s4.z, sc[3] = s4.w;
          } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const int n = n0 + 2 * p;
              const uint32_t lo = n < NL ? __half_as_ushort(scale[long(m) * e.sm + long(n) * e.sn]) : 0u;
              const uint32_t hi = n + 1 < NL ? __half_as_ushort(scale[long(m) * e.sm + long(n + 1) * e.sn]) : 0u;
              sc[p] = lo | (hi << 16);
            }
          }
          uint32_t w[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(w[p]) : "r"(sc[p]), "r"(acc[p]));
          if (full && e.cn == 1 && ((e.cm * m + n0) & 7) == 0) {
            *reinterpret_cast<uint4*>(Ch + long(m) * e.cm + n0) = make_uint4(w[0], w[1], w[2], w[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (n0 + q < NL)
                Ch[long(m) * e.cm + long(n0 + q) * e.cn] =
                    __ushort_as_half((unsigned short)((w[q >> 1] >> (16 * (q & 1))) & 0xffffu));
          }
        } else {  // FP64 result (+ fused dot partials)
          double* const Cd = e.Cd + img * e.c_img;
          const double* const d0 = e.d0 ? e.d0 + img * e.v_img : nullptr;
          const double* const d1a = e.d1a ? e.d1a + img * e.v_img : nullptr;
          const double* const d1b = e.d1b ? e.d1b + img * e.v_img : nullptr;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int n = n0 + q;
            if (n >= NL) continue;
            const double v =
                double(__half2float(__ushort_as_half((unsigned short)((acc[q >> 1] >> (16 * (q & 1))) & 0xffffu))));
            Cd[long(m) * e.cm + long(n) * e.cn] = v;
            if (e.partials) {
              const long vi = long(m) * e.vm + long(n) * e.vn;
              if (d0) s0 += v * d0[vi];
              if (d1a) s1 += v * (d1b ? (d1a[vi] - d1b[vi]) : d1a[vi]);
              if (!isfinite(v)) s2 += 1.0;
            }
          }
        }
      }
      if (zbits) {  // rare (hash match): record the output for the exact sign fix-up
        const unsigned base = atomicAdd(args.zfix, unsigned(__popc(zbits)));
        unsigned* list = args.zfix + 2;
        int q = 0;
        for (uint32_t zb = zbits; zb; zb &= zb - 1, ++q)
          list[base + q] = unsigned(long(m) * N + ng0 + (__ffs(zb) - 1));
      }
      }  // sets
      if (e.mode == F16OUT_F64 && e.partials) {  // fixed-order per-tile partials
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, off);
          s1 += __shfl_xor_sync(0xffffffffu, s1, off);
          s2 += __shfl_xor_sync(0xffffffffu, s2, off);
        }
        const int ew = warp - 4;
        if (lane == 0) red[ew][0] = s0, red[ew][1] = s1, red[ew][2] = s2;
        asm volatile("bar.sync 1, %0;\n" ::"n"(EPI_THREADS) : "memory");
        if (ew == 0 && lane == 0) {
          double a0 = 0, a1 = 0, a2 = 0;
          for (int w = 0; w < EPI_WARPS; ++w) a0 += red[w][0], a1 += red[w][1], a2 += red[w][2];
          // slot = the tile's row-major position in its image's tile grid (a
          // batched image reduces its partials in the same order as a single
          // product of that image)
          const long slot = e.n_img ? long(img) * e.part_img + long(mb / BM) * (e.n_img / BN) + nlb / BN
                                    : long(mb / BM) * tiles_n + nb / BN;
          double* o = e.partials + slot * 4;
          o[0] = a0, o[1] = a1, o[2] = a2, o[3] = 0.0;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(EPI_THREADS) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// Row sign hashes: out[r] = sum over k < K with sign(X(r,k)) = 1 of R(k)
// (mod 2^64), R(k) = splitmix64(k) from a table. If row a of A and row b of
// B have opposite signs at every k then hash_a + hash_b = sum_k R(k); the
// converse fails only on a 64-bit collision, which the fix-up re-checks.
// SMEM_R: the R table staged in shared memory, permuted so that lane l's value
// for its chunk (l + 32 i) and element e sits at ((i*8 + e)*32 + l) - one
// conflict-free LDS.64 per element instead of a 64-byte-strided global load
// (n = 4096: ~40 -> ~21 us per launch with the 16-warp CTAs and batched loads below).
template <bool SMEM_R>
__global__ void row_sign_hash_kernel(const __half* X, long ld, int rows, int K,
                                     const unsigned long long* R, unsigned long long* out) {
  pdl_wait();
  extern __shared__ unsigned long long Rs[];
  const int lane = threadIdx.x & 31;
  const long warp0 = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (long(gridDim.x) * blockDim.x) >> 5;
  const int KV = K / 8;
  if (SMEM_R) {
    for (int k = threadIdx.x; k < KV * 8; k += blockDim.x) {
      const int c = k >> 3, e = k & 7;
      Rs[((c >> 5) * 8 + e) * 32 + (c & 31)] = R[k];
    }
    __syncthreads();
  }
  for (long r = warp0; r < rows; r += nwarps) {
    const uint4* row = reinterpret_cast<const uint4*>(X + r * ld);
    unsigned long long h = 0;
    // 4 loads in flight per lane (the kernel is bound by load latency, not
    // bandwidth); unguarded when the row is whole batches (K % 1024 == 0)
    auto add_chunk = [&](const uint4& q, int i, int c) {
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if ((w[e >> 1] >> (16 * (e & 1) + 15)) & 1u) h += SMEM_R ? Rs[(i * 8 + e) * 32 + lane] : R[8 * c + e];
    };
    if ((KV & 127) == 0) {
      for (int i0 = 0; 32 * i0 < KV; i0 += 4) {
        const uint4 v0 = __ldg(row + lane + 32 * i0), v1 = __ldg(row + lane + 32 * (i0 + 1));
        const uint4 v2 = __ldg(row + lane + 32 * (i0 + 2)), v3 = __ldg(row + lane + 32 * (i0 + 3));
        add_chunk(v0, i0, lane + 32 * i0), add_chunk(v1, i0 + 1, lane + 32 * (i0 + 1));
        add_chunk(v2, i0 + 2, lane + 32 * (i0 + 2)), add_chunk(v3, i0 + 3, lane + 32 * (i0 + 3));
      }
    } else {
      int i = 0;
      for (int c = lane; c < KV; c += 32, ++i) add_chunk(row[c], i, c);
    }
    const unsigned short* rs = reinterpret_cast<const unsigned short*>(X + r * ld);
    for (int k = KV * 8 + lane; k < K; k += 32)
      if (rs[k] & 0x8000u) h += R[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if (lane == 0) out[r] = h;
  }
}

__global__ void hash_table_kernel(unsigned long long* R, int K) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    unsigned long long z = (unsigned long long)k + 0x9E3779B97F4A7C15ull;  // splitmix64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    R[k] = z ^ (z >> 31);
  }
}

// Sign fix-up of outputs whose tree value was +-0 (see the header): the
// reference value is -0 iff sign(A(m,k)) != sign(B(n,k)) for every k < K.
// One warp per listed output (16-byte operand loads); the last CTA resets the
// list count and its own completion counter.
__global__ void f16x_zero_fix_kernel(const F16GemmArgs args) {
  pdl_wait();
  unsigned* cnt = args.zfix;
  const unsigned count = *cnt;  // written by the GEMM this launch follows (stream order)
  if (count == 0) return;       // every CTA sees the same count
  const unsigned* list = args.zfix + 2;
  const int lane = threadIdx.x & 31;
  const long warp0 = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nwarps = (long(gridDim.x) * blockDim.x) >> 5;
  const F16Epilogue& e = args.epi;
  const int N = args.N, K = args.K;
  const int KV = K / 8;  // whole 8-element chunks; the tail is checked per element
  for (long q = warp0; q < count; q += nwarps) {
    const long idx = list[q];
    const int m = int(idx / N), ng = int(idx % N);
    int n;
    const int img = epi_image(e, ng, n);
    const unsigned short* a = reinterpret_cast<const unsigned short*>(args.A.p) + long(m) * args.A.ld;
    const unsigned short* b = reinterpret_cast<const unsigned short*>(args.B.p) + long(ng) * args.B.ld;
    bool opposite = true;
    for (int c = lane; c < KV; c += 32) {
      const uint4 x = reinterpret_cast<const uint4*>(a)[c], y = reinterpret_cast<const uint4*>(b)[c];
      const uint32_t s = ((x.x ^ y.x) & (x.y ^ y.y) & (x.z ^ y.z) & (x.w ^ y.w)) & 0x80008000u;
      opposite &= s == 0x80008000u;
    }
    for (int k = KV * 8 + lane; k < K; k += 32) opposite &= ((a[k] ^ b[k]) & 0x8000u) != 0;
    opposite = __all_sync(0xffffffffu, opposite);
    if (lane == 0) {
      const unsigned short z = opposite ? 0x8000u : 0x0000u;
      if (e.mode == F16OUT_HALF) {
        e.Ch[img * e.c_img + long(m) * e.cm + long(n) * e.cn] = __ushort_as_half(z);
      } else if (e.mode == F16OUT_HALF_SCALED) {
        unsigned short r;
        asm("mul.rn.f16 %0, %1, %2;" : "=h"(r)
            : "h"(__half_as_ushort(e.scale[img * e.s_img + long(m) * e.sm + long(n) * e.sn])), "h"(z));
        e.Ch[img * e.c_img + long(m) * e.cm + long(n) * e.cn] = __ushort_as_half(r);
      } else {
        e.Cd[img * e.c_img + long(m) * e.cm + long(n) * e.cn] = opposite ? -0.0 : 0.0;
      }
    }
  }
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(cnt + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    cnt[1] = 0;
    *cnt = 0;
  }
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

CUtensorMap make_map(const F16Operand& op, int rows, int box_rows, bool swizzle) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(op.ld), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(op.ld) * 2};
  const cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(op.p), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

int counter_levels(int K) {
  const int units = (K + BK - 1) / BK;
  int levels = 1;
  while ((1 << levels) <= units) ++levels;
  return levels;
}


unsigned long long splitmix64(unsigned long long k) {
  unsigned long long z = k + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// R(k) table for k < K on the calling thread's device (grown on demand; kept
// for the process lifetime, shared by all threads of the device).
const unsigned long long* sign_hash_table(int K) {
  static std::mutex mu;
  static std::map<int, std::pair<unsigned long long*, int>> tables;
  std::lock_guard<std::mutex> lk(mu);
  auto& t = tables[ctx().device];
  if (t.second < K) {
    const int cap = std::max(K, 4096);
    unsigned long long* p = nullptr;
    KP_CUDA(cudaMalloc(&p, size_t(cap) * sizeof(unsigned long long)));
    hash_table_kernel<<<cdiv(cap, 256), 256, 0, ctx().stream>>>(p, cap);
    check_launch("sign hash table");
    KP_CUDA(cudaStreamSynchronize(ctx().stream));  // usable from every stream
    t = {p, cap};  // the previous (smaller) table stays allocated: graphs may reference it
  }
  return t.first;
}

void row_hash_launch(const F16Operand& X, int rows, int K, unsigned long long* out) {
  LaunchScope scope(KC_PRECOND_AUX);
  const unsigned long long* R = sign_hash_table(K);
  const int grid = std::max(1, std::min<int>(2 * ctx().num_sms, int(cdiv(rows, 8))));
  // table slots: whole 32-chunk groups (the permuted layout pads the last group)
  const size_t smem = size_t(cdiv(K / 8, 32)) * 32 * 8 * sizeof(unsigned long long);
  static const bool smem_off = [] {
    const char* e = getenv("KP_HASH_SMEM");
    return e && atoi(e) == 0;
  }();
  if (!smem_off && smem > 0 && smem <= 96 * 1024 && rows >= 16 * ctx().num_sms) {
    // two 16-warp CTAs per SM, each staging the table once
    set_smem_limit(reinterpret_cast<const void*>(row_sign_hash_kernel<true>), smem);
    launch_pdl(row_sign_hash_kernel<true>, dim3(2 * ctx().num_sms), dim3(512), smem, X.p, X.ld, rows, K, R, out);
  } else {
    launch_pdl(row_sign_hash_kernel<false>, dim3(grid), dim3(256), 0, X.p, X.ld, rows, K, R, out);
  }
  check_launch("row sign hash");
}

}  // namespace

#if KP_F16X_TRACE
}  // namespace kp
extern "C" int kp_debug_f16x_trace(long long* out, int n) {
  return int(cudaMemcpyFromSymbol(out, kp::f16x_trace, sizeof(long long) * size_t(n)));
}
namespace kp {
#endif
long f16x_zfix_words(int M, int N) { return long(M) * N; }
int gemm_f16x_num_ctas(int M, int N) { return int(cdiv(M, BM) * cdiv(N, BN)); }
int gemm_f16x_partials_per_image(int M, int n_img) { return int(cdiv(M, BM) * (n_img / BN)); }

unsigned long long f16x_hash_sum(int K) {
  unsigned long long s = 0;
  for (int k = 0; k < K; ++k) s += splitmix64((unsigned long long)k);
  return s;
}

void f16x_row_hash(const F16Operand& X, int rows, int K, unsigned long long* out) {
  row_hash_launch(X, rows, K, out);
}

void gemm_f16x(const F16GemmArgs& a_in, int kernel_class) {
  if (a_in.M <= 0 || a_in.N <= 0) return;
  if (a_in.K <= 0) throw InvalidArgument("lp_matmul: empty input");
  if (a_in.A.ld % BK || a_in.B.ld % BK || a_in.A.ld < a_in.K || a_in.B.ld < a_in.K)
    throw InvalidArgument("gemm_f16x: operand leading dimension must be a multiple of 64 >= K");
  if (!a_in.zfix || !a_in.hash_a || !a_in.hash_b) throw InvalidArgument("gemm_f16x: zero-sign workspace missing");
  F16GemmArgs a = a_in;
  a.hsum = f16x_hash_sum(a.K);
  if (!a.hash_a_ready) row_hash_launch(a.A, a.M, a.K, a.hash_a);
  row_hash_launch(a.B, a.N, a.K, a.hash_b);
  const int levels = counter_levels(a.K);
  const int smem_levels = levels > REG_LEVELS ? levels - REG_LEVELS : 0;
  const size_t smem = 1024 + size_t(NSTAGE) * STAGE_BYTES + 2 * size_t(BEXP_BYTES) +
                      size_t(smem_levels) * 4 * EPI_THREADS * 4 * NSET;
  if (smem > 227 * 1024) throw InvalidArgument("gemm_f16x: K too large for the counter stack");
  set_smem_limit(reinterpret_cast<const void*>(gemm_f16x_kernel), smem);
  const CUtensorMap ma = make_map(a.A, a.M, BM, true), mb = make_map(a.B, a.N, BN, false);
  const int tiles = gemm_f16x_num_ctas(a.M, a.N);
  const int grid = std::min(tiles, ctx().num_sms);
  {
    LaunchScope scope(kernel_class);
    // xflags: ablation switches of the profiling experiments (skip the TMA
    // waits / the expansion / per-group B slices); always 0 here
    launch_pdl(gemm_f16x_kernel, dim3(grid), dim3(NUM_THREADS), smem, ma, mb, a, levels, 0);
    check_launch("gemm_f16x");
  }
  {
    LaunchScope scope(KC_PRECOND_AUX);
    launch_pdl(f16x_zero_fix_kernel, dim3(ctx().num_sms), dim3(256), 0, a);
    check_launch("gemm_f16x zero fix-up");
  }
}

}  // namespace kp
