// C ABI of the B200 hot path (include/kronprec_b200.h): handles, setup, the
// device-driven PCG / FPCG / CGLS loops and lambda selection.
//
// Reference behaviour mirrored here (file:line in /root/reference/proj):
//   KroneckerSum / kronsum_apply(_transpose)   kron.hpp:19-35, kron.cpp:73-88
//   normal_matvec                              krylov.cpp:146-152
//   build_preconditioner / with_lambda          factor.cpp:80-115
//   precond_solve                              factor.cpp:117-132
//   pcg / fpcg (pcg_core), cgls                krylov.cpp:58-142, 154-208
//   make_spectral_data, gcv, discrepancy        regparam.cpp:119-134, 254-327
#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/kronprec_b200.h"
#include "banded.cuh"
#include "common.cuh"
#include "gemm_f16ref.cuh"
#include "gemm_f16tc.cuh"
#include "gemm_f16x.cuh"
#include "svd_dev.h"
#include "problem_dev.h"

extern "C" void kpg_blob_params(int n, uint64_t seed, int blobs, double* out);  // problem.cpp
#include "lp_generic.cuh"
#include "gemm_f64.cuh"
#include "host_la.h"
#include "vec.cuh"

// ============================================================================
// context
// ============================================================================
namespace kp {

static thread_local std::string g_last_error;

// One context (device, stream, profiling state) per host thread: handles
// follow the reference's "one handle per thread" rule, and independent solves
// issued from different threads run concurrently on their own streams.
Ctx& ctx() {
  static thread_local Ctx c;
  return c;
}

std::atomic<long long> g_launches{0};
std::atomic<long long> g_loop_solves{0}, g_polled_solves{0};  // drive() modes (kp_drive_stats)

void ensure_init() {
  Ctx& c = ctx();
  if (c.device >= 0) return;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw CudaError(std::string("no CUDA device available: ") + cudaGetErrorString(e) +
                    " (the B200 path has no CPU fallback)");
  int dev = 0;
  KP_CUDA(cudaGetDevice(&dev));  // the calling thread's current device
  KP_CUDA(cudaSetDevice(dev));
  KP_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
  KP_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, dev));
  init_pool(dev);
  c.device = dev;
}

void init_pool(int device) {
  cudaMemPool_t pool;
  KP_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = ~uint64_t(0);
  KP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
}

void set_smem_limit(const void* kernel, size_t bytes) {
  auto& cur = ctx().smem_attr[kernel];
  if (bytes <= cur) return;
  KP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  cur = bytes;
}

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

LaunchScope::LaunchScope(int c) : cls(c) {
  Ctx& x = ctx();
  x.launches++;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (x.profile) {
    if (!x.pool.empty()) {
      ev = x.pool.back();
      x.pool.pop_back();
    } else {
      KP_CUDA(cudaEventCreate(&ev.first));
      KP_CUDA(cudaEventCreate(&ev.second));
    }
    KP_CUDA(cudaEventRecord(ev.first, x.stream));
  }
}
LaunchScope::~LaunchScope() noexcept(false) {
  if (ev.first) {
    Ctx& x = ctx();
    KP_CUDA(cudaEventRecord(ev.second, x.stream));
    x.pending[cls].push_back(ev);
  }
}

static void profile_collect() {
  Ctx& x = ctx();
  KP_CUDA(cudaStreamSynchronize(x.stream));
  for (int c = 0; c < KC_COUNT; ++c) {
    for (auto& ev : x.pending[c]) {
      float ms = 0.f;
      KP_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
      x.total_ms[c] += ms;
      x.count[c]++;
      x.pool.push_back(ev);
    }
    x.pending[c].clear();
  }
}

static void sync() { KP_CUDA(cudaStreamSynchronize(ctx().stream)); }

// Device-side solve loop (drive()): the condition of the WHILE graph node is
// "status still RUNNING"; `count` counts the bodies run (reset by the head
// node) and bounds the loop at `limit` bodies whatever the status says.
__global__ void loop_cond_kernel(cudaGraphConditionalHandle h, const int* status, int* count, int limit,
                                 int head) {
  pdl_wait();
  const int c = head ? 0 : *count + 1;
  *count = c;
  cudaGraphSetConditional(h, (*status == ST_RUNNING && c < limit) ? 1u : 0u);
}
static void loop_cond(cudaGraphConditionalHandle h, const int* status, int* count, int limit, bool head) {
  LaunchScope scope(KC_VECTOR);
  launch_pdl(loop_cond_kernel, dim3(1), dim3(1), 0, h, status, count, limit, head ? 1 : 0);
  check_launch("solve loop condition");
}

// ============================================================================
// small device helpers
// ============================================================================
__global__ void transpose_blocks_kernel(const double* src, double* dst, int n, int r) {
  __shared__ double tile[32][33];
  const int b = blockIdx.z;
  const size_t off = size_t(b) * n * n;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = y0 + j, rr = x0 + threadIdx.x;
    if (c < n && rr < n) tile[j][threadIdx.x] = src[off + size_t(c) * n + rr];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = x0 + j, rr = y0 + threadIdx.x;
    if (c < n && rr < n) dst[off + size_t(c) * n + rr] = tile[threadIdx.x][j];
  }
}
// dst = transpose of each of the r n-by-n column-major blocks of src
static void transpose_blocks(const double* src, double* dst, int n, int r) {
  LaunchScope s(KC_VECTOR);
  dim3 grid(cdiv(n, 32), cdiv(n, 32), r), block(32, 8);
  transpose_blocks_kernel<<<grid, block, 0, ctx().stream>>>(src, dst, n, r);
  check_launch("transpose_blocks");
}

// Host-pinned scratch for small readbacks.
template <typename T>
struct Pinned {
  T* p = nullptr;
  size_t n = 0;
  explicit Pinned(size_t count) : n(count) { KP_CUDA(cudaMallocHost(&p, count * sizeof(T))); }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

// Buffer that is either caller-owned device memory or a staged copy of host
// memory (kp_solver_options.device_pointers).
struct VecArg {
  const double* d = nullptr;
  DBuf<double> own;
  VecArg(const double* src, size_t nn, bool device) {
    if (!src) return;
    if (device) {
      d = src;
    } else {
      own.alloc(nn);
      own.upload(src, nn);
      d = own.p;
    }
  }
};

}  // namespace kp

using namespace kp;

// ============================================================================
// handle types
// ============================================================================
// Solver workspace cached per operator: device vectors, partial-sum arrays,
// history rows, the DevState and a pinned status word, reused across solves
// (a C5 solve would otherwise spend ~0.1 s in cudaMalloc / cudaFree).
struct SolverWorkspace {
  std::map<std::string, DBuf<double>> bufs;
  DBuf<DevState> state;
  DevState* host_state = nullptr;
  double* get(const std::string& key, size_t count) {
    auto& b = bufs[key];
    if (b.n < count) b.alloc(count);
    return b.p;
  }
  DevState* dev_state() {
    if (!state.p) state.alloc(1);
    return state.p;
  }
  // batched solves (kp_pcg_batch): one DevState per image (+ the summary in
  // dev_state()) and a pinned copy for the readback
  DBuf<DevState> bstates;
  DevState* host_bstates = nullptr;
  int host_bstates_n = 0;
  DevState* dev_states(int count) {
    if (bstates.n < size_t(count)) bstates.alloc(count);
    return bstates.p;
  }
  DevState* pinned_states(int count) {
    if (host_bstates_n < count) {
      if (host_bstates) cudaFreeHost(host_bstates);
      KP_CUDA(cudaMallocHost(&host_bstates, size_t(count) * sizeof(DevState)));
      host_bstates_n = count;
    }
    return host_bstates;
  }
  DevState* pinned_state() {
    if (!host_state) KP_CUDA(cudaMallocHost(&host_state, sizeof(DevState)));
    return host_state;
  }
  // two pinned status slots + events for the pipelined status polls of drive()
  int* poll_slots() {
    if (!poll) {
      KP_CUDA(cudaMallocHost(&poll, 2 * sizeof(int)));
      for (auto& e : poll_ev) KP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return poll;
  }
  int* poll = nullptr;
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  cudaGraphExec_t exec = nullptr;  // last solve's iteration graph (drive())
  cudaGraphExec_t exec_loop = nullptr;  // last solve's device-loop graph (drive())
  DBuf<int> loop_count;                 // bodies run by the device loop
  int* loop_counter() {
    if (!loop_count.p) loop_count.alloc(1);
    return loop_count.p;
  }
  ~SolverWorkspace() {
    if (exec) cudaGraphExecDestroy(exec);
    if (exec_loop) cudaGraphExecDestroy(exec_loop);
    if (host_state) cudaFreeHost(host_state);
    if (host_bstates) cudaFreeHost(host_bstates);
    if (poll) cudaFreeHost(poll);
    for (auto& e : poll_ev)
      if (e) cudaEventDestroy(e);
  }
};

struct kp_operator {
  int n = 0, r = 0;
  SolverWorkspace ws;
  DBuf<double> Cs_rm, Cs_cm, Rr_rm, Rr_cm;  // r stacked n*n blocks (dense path)
  DBuf<double> W;                           // r*n*n workspace
  DBuf<double> Wb;                          // batched banded applies: batch*r*n*n
  DBuf<double> part;                        // epilogue partials
  // banded-Toeplitz path (banded.cu)
  bool is_banded = false;
  int mode = KP_OP_AUTO;
  int col_taps = 0, row_taps = 0;
  BandTaps cols_fw, cols_tr, rows_fw, rows_tr;
  bool use_banded() const { return is_banded && mode != KP_OP_DENSE; }
  // short bands: both passes in one kernel (no r n^2 intermediate in HBM)
  bool use_fused() const { return use_banded() && mode == KP_OP_BANDED_FUSED; }
};

struct PrecondShared {
  int n = 0;
  std::vector<double> u_r, s_r, v_r, u_c, s_c, v_c;  // FP64 SVDs (host)
  DBuf<double> d_u_r, d_u_c, d_s_r, d_s_c;            // for spectral data
  DBuf<double> d_v_r, d_v_c;                          // x_true projection (col-major)
  DBuf<double> d_vc_rm, d_vr_rm;                      // filtered solution (row-major)
  // binary16 operands (padded, K-major), exact / tensor modes
  long ldh = 0;
  DBuf<__half> vc_a, vr_b, vct_a, vrt_b;
  // FP64 operands (fmt covers double)
  DBuf<double> vc, vr, vct, vrt;
  // extremes of s_r(j) s_c(i) over all (i, j), computed once (spectral data)
  bool have_range = false;
  double smin = 0.0, smax = 0.0;
  // gemm_f16x row sign hashes of the four binary16 factor operands (lazy)
  DBuf<unsigned long long> hash_vc_a, hash_vr_b, hash_vct_a, hash_vrt_b;
  std::mutex lazy_mu;  // guards the lazily created members above (shared across handles)
};

struct kp_precond {
  std::shared_ptr<PrecondShared> sh;
  int n = 0;
  double lambda = 0.0;
  kp_format fmt{};
  int accum = KP_ACCUM_REFERENCE;
  DBuf<double> s64;               // fp64 format
  DBuf<__half> s16;               // fp16 format (col-major n*n)
  // workspace
  DBuf<__half> r16, t1h, wh, t3h;
  DBuf<double> t1d, wd, t3d;
  DBuf<double> rlp;  // generic formats: round_array(unvec(r), fmt)
  DBuf<double> part;
  DBuf<unsigned> zfix;  // gemm_f16x zero-sign fix-up workspace (zeroed)
  DBuf<unsigned long long> hash_b;  // gemm_f16x B-operand row sign hashes
  // batched M-solves (kp_pcg_batch, fp16): images stacked along the GEMM N
  // dimension; per-image S (one lambda each) and binary16 intermediates
  int bcap = 0;
  DBuf<__half> b_r16, b_t1h, b_wh, b_t3h, b_s16;
  DBuf<double> b_part;
  DBuf<unsigned> b_zfix;
  DBuf<unsigned long long> b_hash;
};

struct kp_spectral {
  int n = 0;
  std::shared_ptr<PrecondShared> sh;
  DBuf<double> bhat;
  DBuf<double> xhat;  // optional: coordinates of x_true (regparam.hpp:23)
  double smax = 0.0, smin = 0.0;
};

namespace {

bool covers_double(const kp_format& f) {
  return f.significand_bits >= 53 && f.max_exponent >= 1023 && f.subnormals_enabled;
}
bool is_fp16(const kp_format& f) {
  return f.significand_bits == 11 && f.max_exponent == 15 && f.subnormals_enabled;
}
// Neither fp16 (f16x2 GEMMs) nor double-covering (DMMA GEMMs): the generic
// emulation path (lp_generic.cu), exact for any (t, emax, subnormals).
bool is_generic(const kp_format& f) { return !covers_double(f) && !is_fp16(f); }

// RoundCallSession (precision.hpp:55-66, precision.cpp:11,90): the reference
// tallies its vectorised rounding calls per thread. The device path fuses
// those roundings into kernels, so the tally is kept analytically - the
// number of round_inplace calls the reference makes for the same API call.
thread_local unsigned long long g_round_calls = 0;
int tree_stages(long k) {  // pairwise_block_reduce (lpblas.cpp:13-30): stages for k blocks
  int stages = 0;
  while (k > 1) k = k / 2 + k % 2, ++stages;
  return stages;
}
// precond_solve (factor.cpp:117-132): round r, round S .* t2, four lp_matmul
unsigned long long msolve_round_calls(const kp_format& fmt, int n) {
  return covers_double(fmt) ? 0ull : 2ull + 4ull * (1 + tree_stages(n));
}
LpFormat lp_format(const kp_format& f) {
  LpFormat l;
  l.t = f.significand_bits, l.emax = f.max_exponent, l.sub = f.subnormals_enabled != 0;
  return l;
}
void check_format(const kp_format& f) {
  if (f.significand_bits < 2 || f.significand_bits > 53 || f.max_exponent < 1 ||
      f.max_exponent > 1023)
    throw InvalidArgument("precision format: need 2 <= t <= 53 and 1 <= emax <= 1023");
}
long round_up(long v, long m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// operator application (kron.cpp:73-88) as two DMMA GEMMs with the Kronecker
// sum folded into the M (first) and K (second) dimensions.
void op_apply(kp_operator* op, const double* in, double* out, bool transpose,
              const F64Epilogue* extra, const int* status) {
  const int n = op->n, r = op->r;
  if (op->use_fused()) {
    F64Epilogue e;
    if (extra) e = *extra;
    e.C = out, e.cm = 1, e.cn = n, e.vm = 1, e.vn = n;
    band_fused(in, n, r, transpose ? op->cols_tr : op->cols_fw, transpose ? op->rows_tr : op->rows_fw, e, status);
    return;
  }
  if (op->use_banded()) {
    band_cols(in, op->W.p, n, r, transpose ? op->cols_tr : op->cols_fw, status);
    F64Epilogue e;
    if (extra) e = *extra;
    e.C = out, e.cm = 1, e.cn = n, e.vm = 1, e.vn = n;
    band_rows(op->W.p, n, r, transpose ? op->rows_tr : op->rows_fw, e, status);
    return;
  }
  const long nn = long(n) * n;
  F64GemmArgs g1;
  g1.M = r * n, g1.N = n, g1.nb = 1, g1.Kb = n;
  g1.A = {transpose ? op->Cs_cm.p : op->Cs_rm.p, n, 0};
  g1.B = {in, n, 0};
  g1.epi.C = op->W.p, g1.epi.cm = n, g1.epi.cn = 1;
  g1.status = status;
  gemm_f64(g1, KC_OPERATOR);
  F64GemmArgs g2;
  g2.M = n, g2.N = n, g2.nb = r, g2.Kb = n;
  g2.A = {op->W.p, n, nn};
  g2.B = {transpose ? op->Rr_cm.p : op->Rr_rm.p, n, nn};
  if (extra) g2.epi = *extra;
  g2.epi.C = out, g2.epi.cm = 1, g2.epi.cn = n, g2.epi.vm = 1, g2.epi.vn = n;
  g2.status = status;
  gemm_f64(g2, KC_OPERATOR);
}

int op_partials_ctas(const kp_operator* op) {
  if (op->use_fused()) return band_fused_num_ctas(op->n);
  return op->use_banded() ? band_rows_num_ctas(op->n) : gemm_f64_num_ctas(op->n, op->n);
}

// Diagonal values of a Toeplitz matrix F (n-by-n column-major): diag[d+n-1]
// = F(j+d, j). Returns false if some diagonal is not constant.
bool toeplitz_diagonals(const double* F, int n, std::vector<double>& diag) {
  diag.assign(2 * size_t(n) - 1, 0.0);
  for (int d = -(n - 1); d <= n - 1; ++d) {
    const int j0 = d >= 0 ? 0 : -d;
    const double v = F[size_t(j0) * n + (j0 + d)];
    for (int j = j0; j < n && j + d < n; ++j)
      if (F[size_t(j) * n + (j + d)] != v) return false;
    diag[size_t(d + n - 1)] = v;
  }
  return true;
}

// Detect the banded-Toeplitz structure of all factors and derive the four
// correlation tap sets (see banded.cu for the forms).
void detect_banded(kp_operator* op, const double* rows, const double* cols) {
  const int n = op->n, r = op->r;
  if (r > BAND_MAX_TERMS) return;
  std::vector<std::vector<double>> dr(r), dc(r);
  int cmin = n, cmax = -n, rmin = n, rmax = -n;
  for (int k = 0; k < r; ++k) {
    if (!toeplitz_diagonals(rows + size_t(k) * n * n, n, dr[k])) return;
    if (!toeplitz_diagonals(cols + size_t(k) * n * n, n, dc[k])) return;
    for (int d = -(n - 1); d <= n - 1; ++d) {
      if (dc[k][d + n - 1] != 0.0) cmin = std::min(cmin, d), cmax = std::max(cmax, d);
      if (dr[k][d + n - 1] != 0.0) rmin = std::min(rmin, d), rmax = std::max(rmax, d);
    }
  }
  if (cmin > cmax) cmin = cmax = 0;  // all-zero factors: one zero tap
  if (rmin > rmax) rmin = rmax = 0;
  const int lc = cmax - cmin + 1, lr = rmax - rmin + 1;
  const int pc = (lc + 7) / 8 * 8, pr = (lr + 7) / 8 * 8;
  if (pc > BAND_MAX_TAPS || pr > BAND_MAX_TAPS) return;
  auto fill = [&](BandTaps& t, int taps, int real, int shift,
                  const std::vector<std::vector<double>>& dg, auto offset_of) {
    t = BandTaps{};
    t.taps = taps;
    t.real = real;
    t.shift = shift;
    for (int k = 0; k < r; ++k)
      for (int u = 0; u < taps; ++u) {
        const int d = offset_of(u);
        t.w[k][u] = (d >= -(n - 1) && d <= n - 1 && u < taps) ? dg[k][size_t(d + n - 1)] : 0.0;
      }
  };
  // A: Y = A_c X -> Y(a) = sum_u c[cmax-u] X(a - cmax + u); out: sum_u r[rmax-u] Y(j - rmax + u)
  fill(op->cols_fw, pc, lc, -cmax, dc, [&](int u) { return u < lc ? cmax - u : 1 << 30; });
  fill(op->rows_fw, pr, lr, -rmax, dr, [&](int u) { return u < lr ? rmax - u : 1 << 30; });
  // A^T: Y(a) = sum_u c[cmin+u] X(a + cmin + u); out: sum_u r[rmin+u] Y(j + rmin + u)
  fill(op->cols_tr, pc, lc, cmin, dc, [&](int u) { return u < lc ? cmin + u : 1 << 30; });
  fill(op->rows_tr, pr, lr, rmin, dr, [&](int u) { return u < lr ? rmin + u : 1 << 30; });
  op->col_taps = lc;
  op->row_taps = lr;
  op->is_banded = true;
}

// Reference-exact binary16 products: KP_FP16_PRODUCTS_CUDA_CORES runs
// gemm_f16ref (HMUL2 + HADD2 on the f16x2 pipe), KP_FP16_PRODUCTS_TENSOR
// gemm_f16x (rounded leaves from tcgen05 MMAs, HADD2 trees); both are
// bit-identical to lp_matmul. AUTO picks gemm_f16x from n >= 512, where its
// 128 x 32 tiles fill the SMs (env KP_FP16_PRODUCTS=cuda|tensor|auto sets the
// process default).
std::atomic<int> g_fp16_products{-1};
int fp16_products_setting() {
  int v = g_fp16_products.load();
  if (v < 0) {
    v = KP_FP16_PRODUCTS_AUTO;
    if (const char* e = getenv("KP_FP16_PRODUCTS")) {
      const std::string s(e);
      if (s == "cuda") v = KP_FP16_PRODUCTS_CUDA_CORES;
      else if (s == "tensor") v = KP_FP16_PRODUCTS_TENSOR;
    }
    g_fp16_products.store(v);
  }
  return v;
}
bool use_f16x(int n) {
  const int v = fp16_products_setting();
  if (v == KP_FP16_PRODUCTS_CUDA_CORES) return false;
  if (v == KP_FP16_PRODUCTS_TENSOR) return true;
  return n >= 512;
}
bool msolve_f16x(const kp_precond* p) {
  return is_fp16(p->fmt) && p->accum == KP_ACCUM_REFERENCE && use_f16x(p->n);
}

int msolve_partials_ctas(const kp_precond* p) {
  if (is_generic(p->fmt)) return LP_PART_CTAS;
  if (covers_double(p->fmt)) return gemm_f64_num_ctas(p->n, p->n);
  if (p->accum == KP_ACCUM_TENSOR || msolve_f16x(p)) return VEC_CTAS;  // msolve_finish_f16 partials
  return gemm_f16ref_num_ctas(p->n, p->n);  // gemm_f16ref's fused FP64 epilogue, one slot per tile
}

// zero-initialised gemm_f16x fix-up workspace for M x N products
void ensure_zfix(DBuf<unsigned>& z, int M, int N) {
  const size_t words = size_t(f16x_zfix_words(M, N)) + 2;
  if (z.n >= words) return;
  z.alloc(words);
  KP_CUDA(cudaMemsetAsync(z.p, 0, words * sizeof(unsigned), ctx().stream));
}

void ensure_ws(kp_precond* p) {
  const int n = p->n;
  const size_t nn = size_t(n) * n;
  if (is_generic(p->fmt)) {
    if (!p->t1d.p) p->t1d.alloc(nn), p->wd.alloc(nn), p->t3d.alloc(nn), p->rlp.alloc(nn);
    if (!p->part.p) p->part.alloc(size_t(LP_PART_CTAS) * 4);
  } else if (covers_double(p->fmt)) {
    if (!p->t1d.p) p->t1d.alloc(nn), p->wd.alloc(nn), p->t3d.alloc(nn);
    if (!p->part.p) p->part.alloc(size_t(gemm_f64_num_ctas(n, n)) * 4);
  } else {
    const long ldh = p->sh->ldh;
    if (!p->r16.p) {
      p->r16.alloc(size_t(n) * ldh), p->t1h.alloc(size_t(n) * ldh);
      p->wh.alloc(size_t(n) * ldh), p->t3h.alloc(size_t(n) * ldh);
      fill_u16(p->r16.p, p->r16.n, 0x0000);  // B operands: +0 padding
      fill_u16(p->wh.p, p->wh.n, 0x0000);
      fill_u16(p->t1h.p, p->t1h.n, 0x8000);  // A operands: -0 padding
      fill_u16(p->t3h.p, p->t3h.n, 0x8000);
    }
    if (!p->part.p || p->part.n < size_t(msolve_partials_ctas(p)) * 4)
      p->part.alloc(size_t(msolve_partials_ctas(p)) * 4);
    if (msolve_f16x(p)) {
      ensure_zfix(p->zfix, n, n);
      if (!p->hash_b.p) p->hash_b.alloc(size_t(n));
      auto* sh = p->sh.get();
      std::lock_guard<std::mutex> lk(sh->lazy_mu);
      if (!sh->hash_vc_a.p) {  // the factor operands never change: hash them once
        sh->hash_vc_a.alloc(n), sh->hash_vr_b.alloc(n), sh->hash_vct_a.alloc(n), sh->hash_vrt_b.alloc(n);
        f16x_row_hash({sh->vc_a.p, ldh}, n, n, sh->hash_vc_a.p);
        f16x_row_hash({sh->vr_b.p, ldh}, n, n, sh->hash_vr_b.p);
        f16x_row_hash({sh->vct_a.p, ldh}, n, n, sh->hash_vct_a.p);
        f16x_row_hash({sh->vrt_b.p, ldh}, n, n, sh->hash_vrt_b.p);
        sync();  // shared across handles / threads
      }
    }
  }
}

// precond_solve (factor.cpp:117-132). In fp16 mode r16 must already hold
// round16(unvec(r)) (written by the caller's fused update kernel); r is the
// FP64 residual used by the fused dot products.
void msolve(kp_precond* p, const double* r, double* z, const double* d0, const double* d1a,
            const double* d1b, const int* status) {
  const int n = p->n;
  auto* sh = p->sh.get();
  ensure_ws(p);
  if (is_generic(p->fmt)) {  // precond_solve (factor.cpp:117-132), every rounding explicit
    const size_t nn = size_t(n) * n;
    const LpFormat f = lp_format(p->fmt);
    lp_round_array(r, nn, f, p->rlp.p, KC_PRECOND);  // round_inplace(rm)
    LpGemmArgs g;
    g.M = n, g.N = n, g.K = n, g.f = f, g.status = status, g.ldc = n;
    g.a = sh->vc.p, g.ai = n, g.ak = 1;  // t1 = lp(vc_lp^T, rm)
    g.b = p->rlp.p, g.bk = 1, g.bj = n, g.c = p->t1d.p;
    lp_gemm_generic(g, KC_PRECOND);
    g.a = p->t1d.p, g.ai = 1, g.ak = n;  // w = round(s_lp .* lp(t1, vr_lp))
    g.b = sh->vr.p, g.bk = 1, g.bj = n, g.c = p->wd.p, g.scale = p->s64.p, g.ls = n;
    lp_gemm_generic(g, KC_PRECOND);
    g.scale = nullptr;
    g.a = sh->vc.p, g.ai = 1, g.ak = n;  // t3 = lp(vc_lp, w)
    g.b = p->wd.p, g.bk = 1, g.bj = n, g.c = p->t3d.p;
    lp_gemm_generic(g, KC_PRECOND);
    g.a = p->t3d.p, g.ai = 1, g.ak = n;  // z = lp(t3, vr_lp^T)
    g.b = sh->vr.p, g.bk = n, g.bj = 1, g.c = z;
    lp_gemm_generic(g, KC_PRECOND);
    lp_vector_partials(z, nn, d0, d1a, d1b, p->part.p, status, KC_PRECOND);
    return;
  }
  if (covers_double(p->fmt)) {
    F64GemmArgs g;
    g.M = n, g.N = n, g.nb = 1, g.Kb = n, g.status = status;
    g.A = {sh->vc.p, n, 0}, g.B = {r, n, 0};  // t1 = V_c^T R
    g.epi = F64Epilogue{}, g.epi.C = p->t1d.p, g.epi.cm = n, g.epi.cn = 1;
    gemm_f64(g, KC_PRECOND);
    g.A = {p->t1d.p, n, 0}, g.B = {sh->vr.p, n, 0};  // w = S .* (t1 V_r)
    g.epi = F64Epilogue{}, g.epi.C = p->wd.p, g.epi.cm = 1, g.epi.cn = n;
    g.epi.vm = 1, g.epi.vn = n, g.epi.mul = p->s64.p;
    gemm_f64(g, KC_PRECOND);
    g.A = {sh->vct.p, n, 0}, g.B = {p->wd.p, n, 0};  // t3 = V_c w
    g.epi = F64Epilogue{}, g.epi.C = p->t3d.p, g.epi.cm = n, g.epi.cn = 1;
    gemm_f64(g, KC_PRECOND);
    g.A = {p->t3d.p, n, 0}, g.B = {sh->vrt.p, n, 0};  // z = t3 V_r^T
    g.epi = F64Epilogue{}, g.epi.C = z, g.epi.cm = 1, g.epi.cn = n, g.epi.vm = 1, g.epi.vn = n;
    g.epi.d0 = d0, g.epi.d1a = d1a, g.epi.d1b = d1b, g.epi.count_nonfinite = 1;
    g.epi.partials = p->part.p;
    gemm_f64(g, KC_PRECOND);
    return;
  }
  if (!is_fp16(p->fmt)) throw Unsupported("precond_solve: only fp16 and double-covering formats run on the B200 path");
  const long ldh = sh->ldh;
  if (p->accum == KP_ACCUM_REFERENCE) {
    // gemm_f16x needs a finite A operand (the expanded-B filler zeros multiply
    // it): A is always a singular-vector factor, B the data. The second and
    // fourth products are therefore formed transposed (out^T = B'^T A'^T),
    // which also makes every epilogue store row-contiguous. gemm_f16ref runs
    // the same orientation (same values either way; the fused dot partials
    // then group z identically for both engines and for batched solves).
    const bool f16x = msolve_f16x(p);
    auto gemm_x = [f16x](const F16GemmArgs& a, int cls) { f16x ? gemm_f16x(a, cls) : gemm_f16ref(a, cls); };
    F16GemmArgs g;
    g.M = n, g.N = n, g.K = n, g.status = status;
    if (f16x) g.zfix = p->zfix.p, g.hash_a_ready = true, g.hash_b = p->hash_b.p;
    g.hash_a = sh->hash_vc_a.p;
    g.A = {sh->vc_a.p, ldh}, g.B = {p->r16.p, ldh};  // t1(a,j) = lp(V_c^T R)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t1h.p, g.epi.cm = ldh, g.epi.cn = 1;
    gemm_x(g, KC_PRECOND);
    g.hash_a = sh->hash_vr_b.p;
    g.A = {sh->vr_b.p, ldh}, g.B = {p->t1h.p, ldh};  // w(a,b) = round(S .* lp(t1 V_r)), as (b, a)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF_SCALED, g.epi.Ch = p->wh.p, g.epi.cm = ldh,
    g.epi.cn = 1, g.epi.scale = p->s16.p, g.epi.sm = n, g.epi.sn = 1;
    gemm_x(g, KC_PRECOND);
    g.hash_a = sh->hash_vct_a.p;
    g.A = {sh->vct_a.p, ldh}, g.B = {p->wh.p, ldh};  // t3(i,b) = lp(V_c w)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t3h.p, g.epi.cm = ldh, g.epi.cn = 1;
    gemm_x(g, KC_PRECOND);
    g.hash_a = sh->hash_vrt_b.p;
    g.A = {sh->vrt_b.p, ldh}, g.B = {p->t3h.p, ldh};  // z(i,j) = lp(t3 V_r^T), as (j, i)
    // binary16 z into t1h (free once the second product has read it), then
    // one HBM pass widens it (exactly) and forms the dot partials: an FP64
    // epilogue with the dots inside the product cost 16 % more per product
    // (its stores / loads stall the warps that drain TMEM)
    // (gemm_f16ref, small n: the FP64 epilogue with fused dots saves that
    // extra launch, which is what counts at n < 512)
    if (f16x) {
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t1h.p, g.epi.cm = ldh, g.epi.cn = 1;
      gemm_x(g, KC_PRECOND);
      msolve_finish_f16(p->t1h.p, ldh, n, z, d0, d1a, d1b, p->part.p, status);
    } else {
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_F64, g.epi.Cd = z, g.epi.cm = n, g.epi.cn = 1;
      g.epi.vm = n, g.epi.vn = 1, g.epi.d0 = d0, g.epi.d1a = d1a, g.epi.d1b = d1b;
      g.epi.partials = p->part.p;
      gemm_x(g, KC_PRECOND);
    }
    return;
  }
  // KP_ACCUM_TENSOR: tcgen05 kind::f16 products (gemm_f16tc). Its epilogue
  // threads own output rows (TMEM lanes), so t1 and t3 are computed
  // transposed (t1^T = R^T V_c, t3^T = w^T V_c^T) to store M-contiguously.
  F16GemmArgs g;
  g.M = n, g.N = n, g.K = n, g.status = status;
  g.A = {p->r16.p, ldh}, g.B = {sh->vc_a.p, ldh};
  g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t1h.p, g.epi.cm = 1, g.epi.cn = ldh;
  gemm_f16tc(g, KC_PRECOND);
  g.A = {p->t1h.p, ldh}, g.B = {sh->vr_b.p, ldh};  // w = round(S .* (t1 V_r))
  g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF_SCALED, g.epi.Ch = p->wh.p, g.epi.cm = 1,
  g.epi.cn = ldh, g.epi.scale = p->s16.p, g.epi.sm = 1, g.epi.sn = n;
  gemm_f16tc(g, KC_PRECOND);
  g.A = {p->wh.p, ldh}, g.B = {sh->vct_a.p, ldh};
  g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t3h.p, g.epi.cm = 1, g.epi.cn = ldh;
  gemm_f16tc(g, KC_PRECOND);
  // binary16 z into t1h (free once the second product has consumed it), then
  // one HBM pass widens it and forms the dot partials
  g.A = {p->t3h.p, ldh}, g.B = {sh->vrt_b.p, ldh};  // z = t3 V_r^T
  g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->t1h.p, g.epi.cm = 1, g.epi.cn = ldh;
  gemm_f16tc(g, KC_PRECOND);
  msolve_finish_f16(p->t1h.p, ldh, n, z, d0, d1a, d1b, p->part.p, status);
}

void cast_r16(kp_precond* p, const double* r, const int* status) {
  ensure_ws(p);
  cast_f64_to_f16_padded(r, p->r16.p, p->n, p->n, p->n, p->sh->ldh, status);
}

// weight_matrix (factor.cpp:62-76)
std::vector<double> weight_matrix(const PrecondShared& sh, double lambda) {
  const int n = sh.n;
  std::vector<double> s(size_t(n) * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const double prod = sh.s_r[j] * sh.s_c[i];
      const double denom = prod * prod + lambda * lambda;
      if (denom == 0.0)
        throw InvalidArgument("build_preconditioner: singular factors need lambda > 0");
      s[size_t(j) * n + i] = 1.0 / denom;
    }
  return s;
}

void set_weights(kp_precond* p) {
  const int n = p->n;
  const size_t nn = size_t(n) * n;
  const auto& sh = *p->sh;
  // denominators are monotone in s_r(j) s_c(i) >= 0, so the smallest one is
  // zero iff any is (the reference's per-element check, factor.cpp:70-72)
  auto amin = [](const std::vector<double>& v) {
    double m = std::numeric_limits<double>::infinity();
    for (double x : v) m = std::min(m, std::fabs(x));
    return m;
  };
  const double pmin = amin(sh.s_r) * amin(sh.s_c);
  const double l2 = p->lambda * p->lambda;
  if (pmin * pmin + l2 == 0.0)
    throw InvalidArgument("build_preconditioner: singular factors need lambda > 0");
  if (covers_double(p->fmt) || is_generic(p->fmt)) {
    p->s64.alloc(nn);
    precond_weights(sh.d_s_r.p, sh.d_s_c.p, n, l2, p->s64.p, nullptr);
    if (is_generic(p->fmt)) lp_round_array(p->s64.p, nn, lp_format(p->fmt), p->s64.p, KC_PRECOND);
  } else {
    p->s16.alloc(nn);
    precond_weights(sh.d_s_r.p, sh.d_s_c.p, n, l2, nullptr, p->s16.p);  // round_array(S)
  }
}

std::vector<double> host_transpose(const std::vector<double>& a, int n) {
  std::vector<double> t(a.size());
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) t[size_t(i) * n + j] = a[size_t(j) * n + i];
  return t;
}

kp_precond* precond_from_svd(int n, std::vector<double> ur, std::vector<double> sr,
                             std::vector<double> vr, std::vector<double> uc,
                             std::vector<double> sc, std::vector<double> vc, double lambda,
                             kp_format fmt, int accum) {
  if (n < 1) throw InvalidArgument("build_preconditioner: empty factors");
  if (lambda < 0.0) throw InvalidArgument("build_preconditioner: negative lambda");
  check_format(fmt);
  if (accum == KP_ACCUM_TENSOR && !is_fp16(fmt))
    throw InvalidArgument("build_preconditioner: tensor accumulation requires fp16");
  auto sh = std::make_shared<PrecondShared>();
  sh->n = n;
  sh->u_r = std::move(ur), sh->s_r = std::move(sr), sh->v_r = std::move(vr);
  sh->u_c = std::move(uc), sh->s_c = std::move(sc), sh->v_c = std::move(vc);
  const size_t nn = size_t(n) * n;
  sh->d_u_r.alloc(nn), sh->d_u_r.upload(sh->u_r.data(), nn);
  sh->d_u_c.alloc(nn), sh->d_u_c.upload(sh->u_c.data(), nn);
  sh->d_s_r.alloc(n), sh->d_s_r.upload(sh->s_r.data(), n);
  sh->d_s_c.alloc(n), sh->d_s_c.upload(sh->s_c.data(), n);
  const std::vector<double> vct = host_transpose(sh->v_c, n), vrt = host_transpose(sh->v_r, n);
  if (is_generic(fmt)) {  // vr_lp, vc_lp = round_array(V, fmt), FP64 col-major
    sh->vc.alloc(nn), sh->vc.upload(sh->v_c.data(), nn);
    sh->vr.alloc(nn), sh->vr.upload(sh->v_r.data(), nn);
    lp_round_array(sh->vc.p, nn, lp_format(fmt), sh->vc.p, KC_PRECOND);
    lp_round_array(sh->vr.p, nn, lp_format(fmt), sh->vr.p, KC_PRECOND);
  } else if (covers_double(fmt)) {
    sh->vc.alloc(nn), sh->vc.upload(sh->v_c.data(), nn);
    sh->vr.alloc(nn), sh->vr.upload(sh->v_r.data(), nn);
    sh->vct.alloc(nn), sh->vct.upload(vct.data(), nn);
    sh->vrt.alloc(nn), sh->vrt.upload(vrt.data(), nn);
  } else {
    sh->ldh = round_up(n, 64);
    const size_t hn = size_t(n) * sh->ldh;
    DBuf<double> tmp(nn);
    auto put = [&](DBuf<__half>& dst, const std::vector<double>& src, uint16_t pad) {
      dst.alloc(hn);
      fill_u16(dst.p, hn, pad);
      tmp.upload(src.data(), nn);
      cast_f64_to_f16_padded(tmp.p, dst.p, n, n, n, sh->ldh, nullptr);  // round_array(v, fmt)
      sync();
    };
    put(sh->vc_a, sh->v_c, 0x8000);  // A of t1 = V_c^T R   (row a = V_c(:,a))
    put(sh->vr_b, sh->v_r, 0x0000);  // B of t1 V_r          (row j = V_r(:,j))
    put(sh->vct_a, vct, 0x8000);     // A of V_c w           (row b = V_c(b,:))
    put(sh->vrt_b, vrt, 0x0000);     // B of t3 V_r^T        (row c = V_r(c,:))
  }
  auto* p = new kp_precond;
  p->sh = sh;
  p->n = n;
  p->lambda = lambda;
  p->fmt = fmt;
  p->accum = accum;
  try {
    set_weights(p);
  } catch (...) {
    delete p;
    throw;
  }
  sync();
  return p;
}

// ---------------------------------------------------------------------------
// solver driver
struct Solve {
  kp_operator* op;
  size_t nn;
  DevState* st = nullptr;  // device
  double *resid = nullptr, *relerr = nullptr, *cosines = nullptr, *iterates = nullptr;
  DevHistory dh{};
  int capacity = 0;
};

struct Vec {
  double* p;
};

// Device view of a solver input: the caller's device pointer, or a copy of
// the host buffer into the cached workspace slot `key`.
const double* stage_vec(SolverWorkspace& ws, const char* key, const double* src, size_t nn,
                        bool device) {
  if (device) return src;
  double* d = ws.get(key, nn);
  KP_CUDA(cudaMemcpyAsync(d, src, nn * sizeof(double), cudaMemcpyHostToDevice, ctx().stream));
  return d;
}

void check_common(const kp_operator* op, const kp_solver_options* o, kp_history* h) {
  if (!op) throw InvalidArgument("solver: null operator");
  if (!o || !h) throw InvalidArgument("solver: null options or history");
  if (o->max_iterations < 1) throw InvalidArgument("solver: max_iterations must be at least 1");
  if (!(o->rel_residual_tol > 0.0)) throw InvalidArgument("solver: tolerance must be positive");
  if (h->capacity < 1 || !h->residual_norm || !h->work_units)
    throw InvalidArgument("solver: history arrays missing");
  if (o->record_iterates) {  // the iterate buffer is sized for max_iterations + 1 rows up front
    if (!h->iterates) throw InvalidArgument("solver: record_iterates needs kp_history.iterates");
    size_t free_b = 0, total_b = 0;
    KP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double need = double(o->max_iterations + 1) * double(op->n) * op->n * sizeof(double);
    if (need > 0.5 * double(free_b))
      throw InvalidArgument("solver: record_iterates needs (max_iterations + 1) n^2 doubles of device memory");
  }
}

std::string abort_message(int code, int k) {
  const std::string ks = std::to_string(k);
  switch (code) {
    case AB_M_NONFINITE_INIT: return "non-finite preconditioner output before iteration 1";
    case AB_POSITIVITY_INIT: return "preconditioner lost positivity before iteration 1";
    case AB_CURV_NONFINITE: return "non-finite curvature at iteration " + ks;
    case AB_CURV_BREAKDOWN: return "curvature breakdown at iteration " + ks;
    case AB_RESID_NONFINITE: return "non-finite residual at iteration " + ks;
    case AB_M_NONFINITE:
      return "non-finite preconditioner output at iteration " + ks +
             " (overflow in the storage format)";
    case AB_INNER_NONFINITE: return "non-finite inner product at iteration " + ks;
    case AB_POSITIVITY: return "preconditioner lost positivity at iteration " + ks;
    default: return "";
  }
}

void setup_state(Solve& s, const kp_solver_options* o, bool has_xt, bool flexible,
                 double work) {
  DevState h{};
  h.status = ST_RUNNING;
  h.k = 1;
  h.maxit = o->max_iterations;
  h.flexible = flexible;
  h.track_cos = o->track_search_direction_orthogonality != 0;
  h.has_xt = has_xt;
  h.record = o->record_iterates != 0;
  h.tol = o->rel_residual_tol;
  h.l2 = o->lambda * o->lambda;
  h.work_per_iter = work;
  SolverWorkspace& ws = s.op->ws;
  s.st = ws.dev_state();
  KP_CUDA(cudaMemcpyAsync(s.st, &h, sizeof(DevState), cudaMemcpyHostToDevice, ctx().stream));
  s.capacity = o->max_iterations + 1;
  s.resid = ws.get("h_resid", s.capacity);
  s.relerr = ws.get("h_relerr", s.capacity);
  s.cosines = ws.get("h_cos", s.capacity);
  s.iterates = o->record_iterates ? ws.get("h_iterates", size_t(s.capacity) * s.nn) : nullptr;
  if (s.iterates)  // row 0 is the starting guess x0 = 0
    KP_CUDA(cudaMemsetAsync(s.iterates, 0, s.nn * sizeof(double), ctx().stream));
  s.dh.resid = s.resid;
  s.dh.relerr = s.relerr;
  s.dh.cosines = s.cosines;
  s.dh.iterates = s.iterates;
  s.dh.capacity = s.capacity;
}

// Runs `iteration` repeatedly until the device status leaves RUNNING. Without
// profiling the iteration is captured once into a CUDA graph and replayed;
// the host polls the status word in growing chunks (overshoot iterations are
// device no-ops).
// Which PCG scalar steps fold into the neighbouring vector kernels (their
// slot sums fit one vector CTA: small n). KP_FOLD_SCALARS=0 keeps the
// separate scalar kernels (identical results).
struct PcgFold {
  bool alpha, resid, beta;
};
static PcgFold pcg_fold(int n_op_slots, int n_vec_slots, int n_msolve_slots) {
  const char* e = getenv("KP_FOLD_SCALARS");
  if (e && e[0] == '0') return {false, false, false};
  return {pcg_fold_ok(n_op_slots), pcg_fold_ok(n_vec_slots), pcg_fold_ok(n_msolve_slots)};
}

// The whole iteration loop as ONE graph launch: a head kernel sets the
// condition from the status word, a WHILE conditional node replays the
// captured iteration (+ a one-thread kernel that re-evaluates the condition)
// until the status leaves RUNNING — no host polls, no overshoot iterations.
// Returns false (nothing enqueued) when the graph cannot be built, e.g. an
// iteration whose capture holds a node type conditional bodies do not allow;
// drive() then falls back to host-polled replay.
bool drive_loop(Solve& s, int maxit, const std::function<void()>& iteration) {
  Ctx& c = ctx();
  SolverWorkspace& ws = s.op->ws;
  int* count = ws.loop_counter();
  const int* status = &s.st->status;
  const int limit = maxit + 2;  // the state machine stops at maxit; this only guards
  cudaGraph_t g = nullptr;
  KP_CUDA(cudaGraphCreate(&g, 0));
  const long long before = c.launches;
  long long body_launches = 0;
  cudaGraphConditionalHandle h;
  auto fail = [&]() {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    g_launches.fetch_sub(c.launches - before, std::memory_order_relaxed);  // captured, not launched
    c.launches = before;
    return false;
  };
  if (cudaGraphConditionalHandleCreate(&h, g, 0, 0) != cudaSuccess) return fail();
  if (cudaStreamBeginCaptureToGraph(c.stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess)
    return fail();
  cudaGraph_t cap = nullptr;
  try {
    loop_cond(h, status, count, limit, true);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &cap);
    throw;
  }
  if (cudaStreamEndCapture(c.stream, &cap) != cudaSuccess) return fail();
  cudaGraphNode_t head;
  size_t nnodes = 1;
  if (cudaGraphGetNodes(g, &head, &nnodes) != cudaSuccess || nnodes != 1) return fail();
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t loop;
  if (cudaGraphAddNode(&loop, g, &head, 1, &cp) != cudaSuccess) return fail();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
      cudaSuccess)
    return fail();
  const long long body0 = c.launches;
  try {
    iteration();
    loop_cond(h, status, count, limit, false);
  } catch (...) {
    cudaStreamEndCapture(c.stream, &cap);
    fail();
    throw;
  }
  body_launches = c.launches - body0;
  if (cudaStreamEndCapture(c.stream, &cap) != cudaSuccess) return fail();
  if (ws.exec_loop) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ws.exec_loop, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(ws.exec_loop);
      ws.exec_loop = nullptr;
    }
  }
  if (!ws.exec_loop && cudaGraphInstantiate(&ws.exec_loop, g, 0) != cudaSuccess) {
    ws.exec_loop = nullptr;
    return fail();
  }
  cudaGraphDestroy(g);
  g = nullptr;
  // captured launches are counted when they run: head + body x bodies run
  g_launches.fetch_sub(c.launches - before, std::memory_order_relaxed);
  c.launches = before;
  KP_CUDA(cudaGraphLaunch(ws.exec_loop, c.stream));
  int* slot = ws.poll_slots();
  KP_CUDA(cudaMemcpyAsync(slot, count, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync();
  const long long ran = 1 + body_launches * (long long)slot[0];
  c.launches += ran;
  g_launches.fetch_add(ran, std::memory_order_relaxed);
  g_loop_solves.fetch_add(1, std::memory_order_relaxed);
  if (slot[0] >= limit) throw std::runtime_error("solver: device loop guard reached (status never left RUNNING)");
  return true;
}

static bool loop_graphs_enabled() {  // read per solve (tests switch it)
  const char* e = getenv("KP_GRAPH_LOOP");
  return !(e && e[0] == '0');
}

void drive(Solve& s, int maxit, const std::function<void()>& iteration) {
  Ctx& c = ctx();
  if (!c.profile && loop_graphs_enabled() && drive_loop(s, maxit, iteration)) return;
  g_polled_solves.fetch_add(1, std::memory_order_relaxed);
  cudaGraphExec_t exec = nullptr;
  long long per_iter_launches = 0;
  if (!c.profile) {
    const long long before = c.launches;
    KP_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      iteration();
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t graph;
    KP_CUDA(cudaStreamEndCapture(c.stream, &graph));
    // Reuse the workspace's executable graph when the new capture has the
    // same topology (repeated solves on one operator): an in-place parameter
    // update is much cheaper than instantiation.
    SolverWorkspace& ws = s.op->ws;
    if (ws.exec) {
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(ws.exec, graph, &info) != cudaSuccess) {
        cudaGetLastError();  // clear the update failure
        cudaGraphExecDestroy(ws.exec);
        ws.exec = nullptr;
      }
    }
    if (!ws.exec) KP_CUDA(cudaGraphInstantiate(&ws.exec, graph, 0));
    exec = ws.exec;
    KP_CUDA(cudaGraphDestroy(graph));
    per_iter_launches = c.launches - before;
    c.launches = before;
    g_launches.fetch_sub(per_iter_launches, std::memory_order_relaxed);  // captured, not launched
  }
  // Pipelined polling: after enqueueing a chunk of iterations the host reads
  // the status the PREVIOUS chunk left (pinned slot + event), so the device
  // always has the next chunk queued and never idles on the host round trip.
  // Overshoot is at most one chunk of no-op iterations (every kernel returns
  // once the status leaves RUNNING). A chunk is 1 iteration while an
  // iteration is long (> 1 ms, where a no-op iteration still costs launches),
  // else it doubles up to 16.
  int* slot = s.op->ws.poll_slots();
  cudaEvent_t* ev = s.op->ws.poll_ev;
  // (Profiled runs use the same pipelined loop; the no-op launches of an
  // overshoot iteration are excluded by the caller's working-launch counts —
  // history.msolve_count and iterations_used — not by serialising the loop,
  // which would expose host launch latency in the per-launch events.)
  int done = 0, chunk = 1, cur = 0;
  bool pending = false;
  auto t_prev = std::chrono::steady_clock::now();
  int prev_todo = 1;
  while (done < maxit) {
    const int todo = std::min(chunk, maxit - done);
    for (int i = 0; i < todo; ++i) {
      if (exec) {
        KP_CUDA(cudaGraphLaunch(exec, c.stream));
        c.launches += per_iter_launches;
        g_launches.fetch_add(per_iter_launches, std::memory_order_relaxed);
      } else {
        iteration();
      }
    }
    done += todo;
    KP_CUDA(cudaMemcpyAsync(&slot[cur], &s.st->status, sizeof(int), cudaMemcpyDeviceToHost,
                            c.stream));
    KP_CUDA(cudaEventRecord(ev[cur], c.stream));
    if (pending) {  // the chunk before this one
      KP_CUDA(cudaEventSynchronize(ev[cur ^ 1]));
      if (slot[cur ^ 1] != ST_RUNNING) break;
      const auto t = std::chrono::steady_clock::now();
      const double per_iter_ms =
          std::chrono::duration<double, std::milli>(t - t_prev).count() / prev_todo;
      t_prev = t;
      chunk = per_iter_ms > 1.0 ? 1 : std::min(chunk * 2, 16);
    }
    pending = true;
    prev_todo = todo;
    cur ^= 1;
  }
}

void finish(Solve& s, const kp_solver_options* o, kp_history* h, double work) {
  auto d2h = [](void* dst, const void* src, size_t bytes) {
    if (bytes) KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx().stream));
  };
  DevState* pst = s.op->ws.pinned_state();
  d2h(pst, s.st, sizeof(DevState));
  sync();
  const DevState st = *pst;
  if (st.status == ST_INVALID) throw InvalidArgument("solver: x_true must be nonzero");
  const int rows = std::min(st.rows, h->capacity);
  const int ncos = std::min(st.ncos, h->capacity);
  d2h(h->residual_norm, s.resid, rows * sizeof(double));
  if (o->x_true && h->relative_error) d2h(h->relative_error, s.relerr, rows * sizeof(double));
  if (o->track_search_direction_orthogonality && h->residual_cosines && ncos > 0)
    d2h(h->residual_cosines, s.cosines, ncos * sizeof(double));
  if (o->record_iterates && h->iterates)
    d2h(h->iterates, s.iterates, size_t(rows) * s.nn * sizeof(double));
  sync();
  for (int k = 0; k < rows; ++k) h->work_units[k] = work * k;
  h->rows = rows;
  h->n_cosines = ncos;
  h->iterations_used = st.iterations_used;
  h->converged = st.status == ST_CONVERGED;
  h->msolve_count = st.msolve_count;
  const std::string msg = st.status == ST_ABORTED ? abort_message(st.abort_code, st.abort_iter) : "";
  std::snprintf(h->abort_reason, sizeof(h->abort_reason), "%s", msg.c_str());
}

// pcg_core (krylov.cpp:58-142)
void run_pcg(kp_operator* op, const double* b_in, kp_precond* m, const kp_solver_options* o,
             double* x_out, kp_history* hist, bool flexible) {
  check_common(op, o, hist);
  if (!m) throw InvalidArgument("solver: null preconditioner");
  if (m->n != op->n) throw InvalidArgument("solver: preconditioner size mismatch");
  const int n = op->n;
  const size_t nn = size_t(n) * n;
  const bool dev = o->device_pointers != 0;
  SolverWorkspace& ws = op->ws;
  const double* b = stage_vec(ws, "b", b_in, nn, dev);
  const double* xt = o->x_true ? stage_vec(ws, "xt", o->x_true, nn, dev) : nullptr;
  Solve s;
  s.op = op;
  s.nn = nn;
  setup_state(s, o, xt != nullptr, flexible, 2.25);
  int* status = &s.st->status;
  double* x = dev ? x_out : ws.get("x", nn);
  Vec r{ws.get("r", nn)}, p{ws.get("p", nn)}, q{ws.get("q", nn)}, z{ws.get("z", nn)};
  Vec rprev{flexible ? ws.get("rprev", nn) : nullptr}, ap{ws.get("ap", nn)};
  const int nop = op_partials_ctas(op);
  const int nms = msolve_partials_ctas(m);
  Vec part_op{ws.get("part_op", size_t(nop) * 4)}, part_vec{ws.get("part_vec", size_t(VEC_CTAS) * 4)};
  Vec part_xt{ws.get("part_xt", size_t(VEC_CTAS) * 4)};
  const bool fp16 = is_fp16(m->fmt);

  vec_zero(x, nn);
  F64Epilogue e;
  e.d0_self = 1;
  e.d0 = r.p;  // any non-null: self product
  e.partials = part_op.p;
  op_apply(op, b, r.p, true, &e, status);  // r = A^T b, ||r||^2 partials
  if (xt) vec_dot_partials(xt, xt, nn, part_xt.p);
  pcg_init_scalar(s.st, s.dh, part_op.p, nop, part_xt.p, VEC_CTAS);
  if (fp16) cast_r16(m, r.p, status);
  msolve(m, r.p, z.p, r.p, nullptr, nullptr, status);
  pcg_init_msolve_scalar(s.st, m->part.p, nms);
  vec_copy(p.p, z.p, nn, status);

  const PcgFold fold = pcg_fold(nop, pcg_update_ctas(n), nms);
  auto iteration = [&]() {
    // q = A^T (A p) + lambda^2 p, with p.q partials (normal_matvec)
    op_apply(op, p.p, ap.p, false, nullptr, status);
    F64Epilogue ne;
    ne.addv = p.p, ne.addc = o->lambda * o->lambda;
    ne.d0 = p.p, ne.partials = part_op.p;
    op_apply(op, ap.p, q.p, true, &ne, status);
    if (!fold.alpha) pcg_alpha_scalar(s.st, part_op.p, nop);
    pcg_update(s.st, s.dh, x, r.p, flexible ? rprev.p : nullptr, p.p, q.p, z.p, xt,
               fp16 ? m->r16.p : nullptr, n, fp16 ? m->sh->ldh : 0, part_vec.p, 1,
               fold.alpha ? part_op.p : nullptr, nop, fold.resid);
    if (!fold.resid) pcg_resid_scalar(s.st, s.dh, part_vec.p, pcg_update_ctas(n));
    msolve(m, r.p, z.p, r.p, flexible ? r.p : nullptr, flexible ? rprev.p : nullptr, status);
    if (!fold.beta) pcg_beta_scalar(s.st, m->part.p, nms);
    pcg_p_update(s.st, p.p, z.p, nn, 1, fold.beta ? m->part.p : nullptr, nms);
  };
  drive(s, o->max_iterations, iteration);
  finish(s, o, hist, 2.25);
  if (!dev) {
    KP_CUDA(cudaMemcpyAsync(x_out, x, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
    sync();
  }
}

// ---------------------------------------------------------------------------
// Batched PCG / FPCG (kp_pcg_batch): `B` independent right-hand sides share
// the operator and the preconditioner factors, each with its own lambda —
// BASELINE C4, the reference's per-image pipeline (cli.cpp:469-486) run for
// a whole batch at once. Every iteration is one set of launches for all
// images: the banded operator passes take the images in grid.z, the four
// binary16 M-solve products stack the images along the GEMM N dimension
// (per-image S in the epilogue, per-image dot partials), and the vector /
// scalar kernels keep one DevState per image (its own alpha, beta, rho,
// stop test and abort; a stopped image is frozen while the others run). Each
// image's arithmetic is exactly the single solve's (same kernels, same
// per-image reduction grids), so results equal kp_pcg image by image.

bool msolve_batch_stacked(const kp_precond* p, int B) {
  // f16x tiles are 32 wide, f16ref tiles up to 64, tcgen05 (tensor mode)
  // tiles 128 tall: images must start on a tile
  if (p->accum == KP_ACCUM_TENSOR) return p->n % 128 == 0;
  return msolve_f16x(p) ? p->n % 32 == 0 : p->n % 64 == 0;
}
// Partial slots per image of a batched M-solve.
int msolve_batch_slots_all(const kp_precond* p, int B) {
  if (p->accum == KP_ACCUM_TENSOR || msolve_f16x(p)) return VEC_CTAS;  // msolve_finish_f16
  if (!msolve_batch_stacked(p, B)) return msolve_partials_ctas(p);
  return gemm_f16ref_partials_per_image(p->n, B * p->n, p->n);
}

void ensure_batch_ws(kp_precond* p, int B, const std::vector<double>& lambdas) {
  const int n = p->n;
  const size_t nn = size_t(n) * n;
  const long ldh = p->sh->ldh;
  ensure_ws(p);  // factor hashes etc.
  if (p->bcap < B) {
    const size_t rows = size_t(B) * n;
    p->b_r16.alloc(rows * ldh), p->b_t1h.alloc(rows * ldh), p->b_wh.alloc(rows * ldh), p->b_t3h.alloc(rows * ldh);
    fill_u16(p->b_r16.p, p->b_r16.n, 0x0000);  // same padding rule as the single solve
    fill_u16(p->b_wh.p, p->b_wh.n, 0x0000);
    fill_u16(p->b_t1h.p, p->b_t1h.n, 0x8000);
    fill_u16(p->b_t3h.p, p->b_t3h.n, 0x8000);
    p->b_s16.alloc(size_t(B) * nn);
    p->bcap = B;
  }
  // partial slots depend on the engine (process-wide setting): size them per call
  if (p->b_part.n < size_t(B) * msolve_batch_slots_all(p, B) * 4)
    p->b_part.alloc(size_t(B) * msolve_batch_slots_all(p, B) * 4);
  if (msolve_f16x(p) && p->b_zfix.n < size_t(f16x_zfix_words(n, B * n)) + 2) {
    ensure_zfix(p->b_zfix, n, B * n);
    p->b_hash.alloc(size_t(B) * n);
  }
  // per-image S = round16(1 / ((s_r s_c)^2 + lambda_i^2)) (factor.cpp:62-76)
  const auto& sh = *p->sh;
  auto amin = [](const std::vector<double>& v) {
    double m = std::numeric_limits<double>::infinity();
    for (double x : v) m = std::min(m, std::fabs(x));
    return m;
  };
  const double pmin = amin(sh.s_r) * amin(sh.s_c);
  for (int i = 0; i < B; ++i) {
    const double l2 = lambdas[i] * lambdas[i];
    if (pmin * pmin + l2 == 0.0) throw InvalidArgument("build_preconditioner: singular factors need lambda > 0");
    precond_weights(sh.d_s_r.p, sh.d_s_c.p, n, l2, nullptr, p->b_s16.p + size_t(i) * nn);
  }
}

// The four products of precond_solve (factor.cpp:117-132) for B images; the
// binary16 residuals are already in b_r16 (image i at rows i*n).
void msolve_batch(kp_precond* p, int B, double* z, const double* d0, const double* d1a,
                  const double* d1b, const int* status) {
  const int n = p->n;
  const size_t nn = size_t(n) * n;
  auto* sh = p->sh.get();
  const long ldh = sh->ldh;
  const bool f16x = msolve_f16x(p);
  const bool stacked = msolve_batch_stacked(p, B);
  const int slots = msolve_batch_slots_all(p, B);
  const int groups = stacked ? 1 : B, per = stacked ? B : 1;
  if (p->accum == KP_ACCUM_TENSOR) {
    // tcgen05 products (msolve's tensor orientation: the data is the A
    // operand), images stacked along M; binary16 z, then one widening pass
    for (int gi = 0; gi < groups; ++gi) {
      const long ho = long(gi) * n * ldh;
      const size_t vo = size_t(gi) * nn;
      F16GemmArgs g;
      g.M = per * n, g.N = n, g.K = n, g.status = status;
      auto batch_epi = [&](F16Epilogue& e) {
        if (stacked && B > 1) e.m_img = n, e.c_img = long(n) * ldh, e.s_img = long(nn);
      };
      g.A = {p->b_r16.p + ho, ldh}, g.B = {sh->vc_a.p, ldh};  // t1^T = R^T V_c
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t1h.p + ho, g.epi.cm = 1, g.epi.cn = ldh;
      batch_epi(g.epi);
      gemm_f16tc(g, KC_PRECOND);
      g.A = {p->b_t1h.p + ho, ldh}, g.B = {sh->vr_b.p, ldh};  // w = round(S .* (t1 V_r))
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF_SCALED, g.epi.Ch = p->b_wh.p + ho, g.epi.cm = 1,
      g.epi.cn = ldh, g.epi.scale = p->b_s16.p + vo, g.epi.sm = 1, g.epi.sn = n;
      batch_epi(g.epi);
      gemm_f16tc(g, KC_PRECOND);
      g.A = {p->b_wh.p + ho, ldh}, g.B = {sh->vct_a.p, ldh};  // t3^T = w^T V_c^T
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t3h.p + ho, g.epi.cm = 1, g.epi.cn = ldh;
      batch_epi(g.epi);
      gemm_f16tc(g, KC_PRECOND);
      g.A = {p->b_t3h.p + ho, ldh}, g.B = {sh->vrt_b.p, ldh};  // z = t3 V_r^T, binary16 into t1h
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t1h.p + ho, g.epi.cm = 1, g.epi.cn = ldh;
      batch_epi(g.epi);
      gemm_f16tc(g, KC_PRECOND);
      msolve_finish_f16(p->b_t1h.p + ho, ldh, n, z + vo, d0 ? d0 + vo : nullptr, d1a ? d1a + vo : nullptr,
                        d1b ? d1b + vo : nullptr, p->b_part.p + size_t(gi) * slots * 4, status, per);
    }
    return;
  }
  for (int gi = 0; gi < groups; ++gi) {
    const long ho = long(gi) * n * ldh;  // image offset when not stacked
    const size_t vo = size_t(gi) * nn;
    F16GemmArgs g;
    g.M = n, g.N = per * n, g.K = n, g.status = status;
    if (f16x) g.zfix = p->b_zfix.p, g.hash_a_ready = true, g.hash_b = p->b_hash.p;
    auto batch_epi = [&](F16Epilogue& e, long c_img) {
      if (stacked && B > 1) e.n_img = n, e.c_img = c_img, e.s_img = long(nn), e.v_img = long(nn), e.part_img = slots;
    };
    auto run = [&]() { f16x ? gemm_f16x(g, KC_PRECOND) : gemm_f16ref(g, KC_PRECOND); };
    g.hash_a = sh->hash_vc_a.p;
    g.A = {sh->vc_a.p, ldh}, g.B = {p->b_r16.p + ho, ldh};  // t1(a, j) = lp(V_c^T R)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t1h.p + ho, g.epi.cm = ldh, g.epi.cn = 1;
    batch_epi(g.epi, long(n) * ldh);
    run();
    g.hash_a = sh->hash_vr_b.p;
    g.A = {sh->vr_b.p, ldh}, g.B = {p->b_t1h.p + ho, ldh};  // w(a,b) = round(S .* lp(t1 V_r)), as (b, a)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF_SCALED, g.epi.Ch = p->b_wh.p + ho, g.epi.cm = ldh,
    g.epi.cn = 1, g.epi.scale = p->b_s16.p + vo, g.epi.sm = n, g.epi.sn = 1;
    batch_epi(g.epi, long(n) * ldh);
    run();
    g.hash_a = sh->hash_vct_a.p;
    g.A = {sh->vct_a.p, ldh}, g.B = {p->b_wh.p + ho, ldh};  // t3(i,b) = lp(V_c w)
    g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t3h.p + ho, g.epi.cm = ldh, g.epi.cn = 1;
    batch_epi(g.epi, long(n) * ldh);
    run();
    g.hash_a = sh->hash_vrt_b.p;
    g.A = {sh->vrt_b.p, ldh}, g.B = {p->b_t3h.p + ho, ldh};  // z(i,j) = lp(t3 V_r^T), as (j, i)
    if (f16x) {  // binary16 z, widened with the dots in one pass (as msolve)
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_HALF, g.epi.Ch = p->b_t1h.p + ho, g.epi.cm = ldh, g.epi.cn = 1;
      batch_epi(g.epi, long(n) * ldh);
      run();
      msolve_finish_f16(p->b_t1h.p + ho, ldh, n, z + vo, d0 ? d0 + vo : nullptr, d1a ? d1a + vo : nullptr,
                        d1b ? d1b + vo : nullptr, p->b_part.p + size_t(gi) * slots * 4, status, per);
    } else {
      g.epi = F16Epilogue{}, g.epi.mode = F16OUT_F64, g.epi.Cd = z + vo, g.epi.cm = n, g.epi.cn = 1;
      g.epi.vm = n, g.epi.vn = 1;
      g.epi.d0 = d0 ? d0 + vo : nullptr, g.epi.d1a = d1a ? d1a + vo : nullptr;
      g.epi.d1b = d1b ? d1b + vo : nullptr;
      g.epi.partials = p->b_part.p + size_t(gi) * slots * 4;
      batch_epi(g.epi, long(nn));
      run();
    }
  }
}

// A (or A^T) applied to B images; `extra` partials land in per-image slots
// of op_partials_ctas(op) each; addc_dev / addc_host: per-image coefficient
// of extra->addv (lambda_i^2).
void op_apply_batch(kp_operator* op, int B, const double* in, double* out, bool transpose,
                    const F64Epilogue* extra, const double* addc_dev, const std::vector<double>* addc_host,
                    const int* status) {
  const int n = op->n, r = op->r;
  const size_t nn = size_t(n) * n;
  if (op->use_fused()) {
    F64Epilogue e;
    if (extra) e = *extra;
    e.C = out, e.cm = 1, e.cn = n, e.vm = 1, e.vn = n;
    e.img = long(nn), e.part_img = band_fused_num_ctas(n);
    if (e.addv) e.addc_img = addc_dev;
    band_fused(in, n, r, transpose ? op->cols_tr : op->cols_fw, transpose ? op->rows_tr : op->rows_fw, e, status, B);
    return;
  }
  if (op->use_banded()) {
    if (op->Wb.n < size_t(B) * r * nn) op->Wb.alloc(size_t(B) * r * nn);
    band_cols(in, op->Wb.p, n, r, transpose ? op->cols_tr : op->cols_fw, status, B);
    F64Epilogue e;
    if (extra) e = *extra;
    e.C = out, e.cm = 1, e.cn = n, e.vm = 1, e.vn = n;
    e.img = long(nn), e.part_img = band_rows_num_ctas(n);
    if (e.addv) e.addc_img = addc_dev;
    band_rows(op->Wb.p, n, r, transpose ? op->rows_tr : op->rows_fw, e, status, B);
    return;
  }
  const int slots = op_partials_ctas(op);
  for (int i = 0; i < B; ++i) {  // dense operator: one image at a time
    const size_t o = size_t(i) * nn;
    F64Epilogue e;
    if (extra) {
      e = *extra;
      if (e.addv) e.addv += o, e.addc = (*addc_host)[i];
      if (e.d0 && !e.d0_self) e.d0 += o;
      if (e.d1a) e.d1a += o;
      if (e.d1b) e.d1b += o;
      if (e.mul) e.mul += o;
      if (e.partials) e.partials += size_t(i) * slots * 4;
    }
    op_apply(op, in + o, out + o, transpose, extra ? &e : nullptr, status);
  }
}

void run_pcg_batch(kp_operator* op, kp_precond* m, int B, const double* b_in, const double* lambdas,
                   const kp_solver_options* o, double* x_out, kp_history* hist, bool flexible) {
  if (!op) throw InvalidArgument("solver: null operator");
  if (B < 1) throw InvalidArgument("pcg_batch: batch must be at least 1");
  if (!o || !hist || !lambdas || !b_in || !x_out) throw InvalidArgument("pcg_batch: null argument");
  if (!m) throw InvalidArgument("solver: null preconditioner");
  if (m->n != op->n) throw InvalidArgument("solver: preconditioner size mismatch");
  if (o->max_iterations < 1) throw InvalidArgument("solver: max_iterations must be at least 1");
  if (!(o->rel_residual_tol > 0.0)) throw InvalidArgument("solver: tolerance must be positive");
  if (o->record_iterates) throw InvalidArgument("pcg_batch: record_iterates is not supported for batches");
  if (!is_fp16(m->fmt))
    throw InvalidArgument("pcg_batch: batched solves need the fp16 preconditioner (reference-exact or tensor mode)");
  for (int i = 0; i < B; ++i)
    if (hist[i].capacity < 1 || !hist[i].residual_norm || !hist[i].work_units)
      throw InvalidArgument("solver: history arrays missing");
  const int n = op->n;
  const size_t nn = size_t(n) * n, bnn = size_t(B) * nn;
  const bool dev = o->device_pointers != 0;
  SolverWorkspace& ws = op->ws;
  std::vector<double> lam(lambdas, lambdas + B), l2(B);
  for (int i = 0; i < B; ++i) l2[i] = lam[i] * lam[i];
  ensure_batch_ws(m, B, lam);
  const double* b = stage_vec(ws, "b_b", b_in, bnn, dev);
  const double* xt = o->x_true ? stage_vec(ws, "b_xt", o->x_true, bnn, dev) : nullptr;

  // per-image states (setup_state's fields, lambda_i) and the batch summary
  const int cap = o->max_iterations + 1;
  std::vector<DevState> hs(B);
  for (int i = 0; i < B; ++i) {
    DevState& h = hs[i];
    h = DevState{};
    h.status = ST_RUNNING, h.k = 1, h.maxit = o->max_iterations, h.flexible = flexible;
    h.track_cos = o->track_search_direction_orthogonality != 0;
    h.has_xt = xt != nullptr, h.record = 0, h.tol = o->rel_residual_tol, h.l2 = l2[i];
    h.work_per_iter = 2.25;
  }
  DevState* states = ws.dev_states(B);
  KP_CUDA(cudaMemcpyAsync(states, hs.data(), B * sizeof(DevState), cudaMemcpyHostToDevice, ctx().stream));
  Solve s;
  s.op = op;
  s.nn = nn;
  s.st = ws.dev_state();  // summary
  {
    DevState sm{};
    sm.status = ST_RUNNING;
    KP_CUDA(cudaMemcpyAsync(s.st, &sm, sizeof(DevState), cudaMemcpyHostToDevice, ctx().stream));
  }
  s.capacity = cap;
  s.dh.resid = ws.get("b_h_resid", size_t(B) * cap);
  s.dh.relerr = ws.get("b_h_relerr", size_t(B) * cap);
  s.dh.cosines = ws.get("b_h_cos", size_t(B) * cap);
  s.dh.iterates = nullptr;
  s.dh.capacity = cap;
  const int* status = &s.st->status;
  double* l2_dev = ws.get("b_l2", B);
  KP_CUDA(cudaMemcpyAsync(l2_dev, l2.data(), B * sizeof(double), cudaMemcpyHostToDevice, ctx().stream));

  double* x = dev ? x_out : ws.get("b_x", bnn);
  double *r = ws.get("b_r", bnn), *p = ws.get("b_p", bnn), *q = ws.get("b_q", bnn), *z = ws.get("b_z", bnn);
  double* rprev = flexible ? ws.get("b_rprev", bnn) : nullptr;
  double* ap = ws.get("b_ap", bnn);
  const int nop = op_partials_ctas(op);
  const int nms = msolve_batch_slots_all(m, B);
  const int nvec = pcg_update_ctas(n);
  double* part_op = ws.get("b_part_op", size_t(B) * nop * 4);
  double* part_vec = ws.get("b_part_vec", size_t(B) * nvec * 4);
  double* part_xt = ws.get("b_part_xt", size_t(B) * VEC_CTAS * 4);
  const long ldh = m->sh->ldh;

  vec_zero(x, bnn);
  F64Epilogue e;
  e.d0_self = 1;
  e.d0 = r;  // any non-null: self product
  e.partials = part_op;
  op_apply_batch(op, B, b, r, true, &e, nullptr, nullptr, status);  // r = A^T b, ||r||^2
  if (xt)
    for (int i = 0; i < B; ++i) vec_dot_partials(xt + size_t(i) * nn, xt + size_t(i) * nn, nn, part_xt + size_t(i) * VEC_CTAS * 4);
  pcg_init_scalar(states, s.dh, part_op, nop, part_xt, VEC_CTAS, B);
  for (int i = 0; i < B; ++i)
    cast_f64_to_f16_padded(r + size_t(i) * nn, m->b_r16.p + size_t(i) * n * ldh, n, n, n, ldh, status);
  msolve_batch(m, B, z, r, nullptr, nullptr, status);
  pcg_init_msolve_scalar(states, m->b_part.p, nms, B);
  batch_status(states, B, s.st);
  vec_copy(p, z, bnn, status);

  const PcgFold fold = pcg_fold(nop, nvec, nms);
  auto iteration = [&]() {
    op_apply_batch(op, B, p, ap, false, nullptr, nullptr, nullptr, status);
    F64Epilogue ne;
    ne.addv = p, ne.d0 = p, ne.partials = part_op;
    op_apply_batch(op, B, ap, q, true, &ne, l2_dev, &l2, status);  // A^T A p + lambda_i^2 p
    if (!fold.alpha) pcg_alpha_scalar(states, part_op, nop, B);
    pcg_update(states, s.dh, x, r, rprev, p, q, z, xt, m->b_r16.p, n, ldh, part_vec, B,
               fold.alpha ? part_op : nullptr, nop, fold.resid);
    if (!fold.resid) pcg_resid_scalar(states, s.dh, part_vec, nvec, B);
    batch_status(states, B, s.st);
    msolve_batch(m, B, z, r, flexible ? r : nullptr, rprev, status);
    if (!fold.beta) pcg_beta_scalar(states, m->b_part.p, nms, B);
    pcg_p_update(states, p, z, nn, B, fold.beta ? m->b_part.p : nullptr, nms);
    batch_status(states, B, s.st);
  };
  drive(s, o->max_iterations, iteration);

  // per-image histories (finish() for each image)
  auto d2h = [](void* dst, const void* src, size_t bytes) {
    if (bytes) KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx().stream));
  };
  DevState* pst = ws.pinned_states(B);
  d2h(pst, states, B * sizeof(DevState));
  sync();
  for (int i = 0; i < B; ++i)
    if (pst[i].status == ST_INVALID) throw InvalidArgument("solver: x_true must be nonzero");
  for (int i = 0; i < B; ++i) {
    const DevState st = pst[i];
    kp_history* h = hist + i;
    const int rows = std::min(st.rows, h->capacity);
    const int ncos = std::min(st.ncos, h->capacity);
    d2h(h->residual_norm, s.dh.resid + size_t(i) * cap, rows * sizeof(double));
    if (xt && h->relative_error) d2h(h->relative_error, s.dh.relerr + size_t(i) * cap, rows * sizeof(double));
    if (o->track_search_direction_orthogonality && h->residual_cosines && ncos > 0)
      d2h(h->residual_cosines, s.dh.cosines + size_t(i) * cap, ncos * sizeof(double));
    for (int k = 0; k < rows; ++k) h->work_units[k] = 2.25 * k;
    h->rows = rows;
    h->n_cosines = ncos;
    h->iterations_used = st.iterations_used;
    h->converged = st.status == ST_CONVERGED;
    h->msolve_count = st.msolve_count;
    const std::string msg = st.status == ST_ABORTED ? abort_message(st.abort_code, st.abort_iter) : "";
    std::snprintf(h->abort_reason, sizeof(h->abort_reason), "%s", msg.c_str());
  }
  if (!dev) d2h(x_out, x, bnn * sizeof(double));
  sync();
}

// cgls (krylov.cpp:154-208)
void run_cgls(kp_operator* op, const double* b_in, const kp_solver_options* o, double* x_out,
              kp_history* hist) {
  check_common(op, o, hist);
  const int n = op->n;
  const size_t nn = size_t(n) * n;
  const bool dev = o->device_pointers != 0;
  SolverWorkspace& ws = op->ws;
  const double* b = stage_vec(ws, "b", b_in, nn, dev);
  const double* xt = o->x_true ? stage_vec(ws, "xt", o->x_true, nn, dev) : nullptr;
  Solve s;
  s.op = op;
  s.nn = nn;
  setup_state(s, o, xt != nullptr, false, 2.0);
  int* status = &s.st->status;
  double* x = dev ? x_out : ws.get("x", nn);
  const bool track = o->track_search_direction_orthogonality != 0;
  Vec rt{ws.get("r", nn)}, sv{ws.get("z", nn)}, p{ws.get("p", nn)}, q{ws.get("q", nn)};
  Vec sprev{track ? ws.get("rprev", nn) : nullptr};
  const int nop = op_partials_ctas(op);
  Vec part_q{ws.get("part_op", size_t(nop) * 4)}, part_s{ws.get("part_s", size_t(nop) * 4)};
  Vec part_vec{ws.get("part_vec", size_t(VEC_CTAS) * 4)}, part_p{ws.get("part_p", size_t(VEC_CTAS) * 4)};
  Vec part_xt{ws.get("part_xt", size_t(VEC_CTAS) * 4)};

  vec_zero(x, nn);
  vec_copy(rt.p, b, nn, nullptr);
  F64Epilogue e;
  e.d0_self = 1, e.d0 = sv.p, e.partials = part_s.p;
  op_apply(op, rt.p, sv.p, true, &e, status);  // s = A^T rt
  if (xt) vec_dot_partials(xt, xt, nn, part_xt.p);
  cgls_init_scalar(s.st, s.dh, part_s.p, nop, part_xt.p, VEC_CTAS);
  vec_copy(p.p, sv.p, nn, status);
  if (track) vec_copy(sprev.p, sv.p, nn, status);

  auto iteration = [&]() {
    F64Epilogue qe;
    qe.d0_self = 1, qe.d0 = q.p, qe.partials = part_q.p;
    op_apply(op, p.p, q.p, false, &qe, status);  // q = A p, ||q||^2
    cgls_alpha_scalar(s.st, part_q.p, nop, part_p.p, VEC_CTAS);
    cgls_update(s.st, s.dh, x, rt.p, p.p, q.p, xt, nn, part_vec.p);
    F64Epilogue se;  // s = A^T rt - lambda^2 x, ||s||^2 and s.s_prev
    se.addv = x, se.addc = -(o->lambda * o->lambda);
    se.d0_self = 1, se.d0 = sv.p;
    se.d1a = track ? sprev.p : nullptr;
    se.partials = part_s.p;
    op_apply(op, rt.p, sv.p, true, &se, status);
    cgls_resid_scalar(s.st, s.dh, part_s.p, nop, part_vec.p, VEC_CTAS);
    cgls_p_update(s.st, p.p, sv.p, track ? sprev.p : nullptr, nn, part_p.p);
  };
  drive(s, o->max_iterations, iteration);
  finish(s, o, hist, 2.0);
  if (!dev) {
    KP_CUDA(cudaMemcpyAsync(x_out, x, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
    sync();
  }
}

// ---------------------------------------------------------------------------
// lambda selection helpers (regparam.cpp)
double probe(const std::function<double(double)>& f, double x, const char* who) {
  const double v = f(x);
  if (std::isnan(v)) throw std::runtime_error(std::string(who) + ": objective is NaN");
  return v;
}

// Objective values for m lambdas in one batched device reduction
// (regparam.cpp:216-246): kind SK_GCV -> gcv_objective, SK_RESID ->
// discrepancy_gap (+ eps^2), SK_OPT -> opt_objective, SK_WGCV ->
// wgcv_objective, SK_WTRACE -> the wgcv trace term.
void spectral_values(const kp_spectral* sd, int kind, const double* lambdas, int m, double omega,
                     double eps, double* values) {
  if (kind == SK_OPT && !sd->xhat.p) throw InvalidArgument("opt_objective: x coordinates missing");
  DBuf<double> dl(m), out(size_t(m) * 2);
  dl.upload(lambdas, m);
  spectral_sums(kind, sd->sh->d_s_r.p, sd->sh->d_s_c.p, sd->bhat.p, sd->xhat.p, sd->n, dl.p, m,
                omega, out.p);
  std::vector<double> h(size_t(m) * 2);
  out.download(h.data(), h.size());
  sync();
  const double N = double(sd->n) * sd->n;
  for (int q = 0; q < m; ++q) {
    const double a = h[2 * q], b = h[2 * q + 1];
    switch (kind) {
      case SK_GCV: values[q] = N * a / (b * b); break;
      case SK_RESID: values[q] = a - eps * eps; break;
      case SK_WGCV:
        values[q] = b == 0.0 ? std::numeric_limits<double>::infinity() : (a * N) / (b * b);
        break;
      default: values[q] = a; break;  // SK_OPT, SK_WTRACE
    }
  }
}
double spectral_value(const kp_spectral* sd, int kind, double lambda, double omega = 0.0,
                      double eps = 0.0) {
  double v;
  spectral_values(sd, kind, &lambda, 1, omega, eps, &v);
  return v;
}
void gcv_values(const kp_spectral* sd, const double* lambdas, int m, double* values) {
  spectral_values(sd, SK_GCV, lambdas, m, 0.0, 0.0, values);
}
double gcv_value(const kp_spectral* sd, double lambda) { return spectral_value(sd, SK_GCV, lambda); }
double gap_value(const kp_spectral* sd, double eps, double lambda) {
  return spectral_value(sd, SK_RESID, lambda, 0.0, eps);
}

// minimize_1d (regparam.cpp:149-181)
std::pair<double, double> minimize_1d(const std::function<double(double)>& f, double lo, double hi,
                                      double tol) {
  constexpr double invphi = 0.6180339887498949;
  double a = lo, b = hi;
  double c = b - invphi * (b - a), d = a + invphi * (b - a);
  double fc = probe(f, c, "minimize_1d"), fd = probe(f, d, "minimize_1d");
  for (int it = 0; it < 300 && b - a > tol * (1.0 + std::min(std::abs(a), std::abs(b))); ++it) {
    if (fc < fd) {
      b = d, d = c, fd = fc;
      c = b - invphi * (b - a);
      if (c <= a || c >= d) break;
      fc = probe(f, c, "minimize_1d");
    } else {
      a = c, c = d, fc = fd;
      d = a + invphi * (b - a);
      if (d <= c || d >= b) break;
      fd = probe(f, d, "minimize_1d");
    }
  }
  return fc < fd ? std::make_pair(c, fc) : std::make_pair(d, fd);
}

// find_root (regparam.cpp:184-214)
double find_root(const std::function<double(double)>& f, double lo, double hi, double tol) {
  double flo = probe(f, lo, "find_root"), fhi = probe(f, hi, "find_root");
  if (!std::isfinite(flo) || !std::isfinite(fhi))
    throw std::runtime_error("find_root: endpoint value not finite");
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  if ((flo > 0.0) == (fhi > 0.0)) throw InvalidArgument("find_root: no sign change over [lo, hi]");
  double a = lo, b = hi;
  while (b - a > tol * (1.0 + 0.5 * (std::abs(a) + std::abs(b)))) {
    const double m = a + 0.5 * (b - a);
    if (m <= a || m >= b) break;
    const double fm = probe(f, m, "find_root");
    if (!std::isfinite(fm)) throw std::runtime_error("find_root: function value not finite");
    if (fm == 0.0) return m;
    if ((fm > 0.0) == (flo > 0.0)) {
      a = m, flo = fm;
    } else {
      b = m;
    }
  }
  return a + 0.5 * (b - a);
}

// find_root with look-ahead: the same bisection, decision for decision, but
// the midpoints of the next LEVELS levels (every node of the binary tree the
// walk can take from [a, b]) are evaluated in one batched launch, so the ~42
// dependent device round trips of a discrepancy solve become ~21. (Each extra
// lambda costs ~9 us of FP64 divisions over n^2 = 1M coefficients against
// ~28 us of per-launch round trip, so two levels — three values — is the
// measured optimum; six levels were slower than none.) Midpoints use
// find_root's formula on the same operands, and the batched objective equals
// the single-value one bit for bit (per-lambda sums in a fixed order), so the
// walk reproduces find_root exactly; nodes off the walked path are discarded
// unchecked. fbatch(xs, m, values) evaluates f at m points.
double find_root_batched(const std::function<void(const double*, int, double*)>& fbatch,
                         double lo, double hi, double tol) {
  constexpr int LEVELS = 2, NODES = (1 << LEVELS) - 1;
  double ends[2] = {lo, hi}, fe[2];
  fbatch(ends, 2, fe);
  double flo = fe[0], fhi = fe[1];
  if (std::isnan(flo) || std::isnan(fhi)) throw std::runtime_error("find_root: objective is NaN");
  if (!std::isfinite(flo) || !std::isfinite(fhi))
    throw std::runtime_error("find_root: endpoint value not finite");
  if (flo == 0.0) return lo;
  if (fhi == 0.0) return hi;
  if ((flo > 0.0) == (fhi > 0.0)) throw InvalidArgument("find_root: no sign change over [lo, hi]");
  auto open = [&](double a, double b) { return b - a > tol * (1.0 + 0.5 * (std::abs(a) + std::abs(b))); };
  double a = lo, b = hi;
  double na[NODES], nb[NODES], nm[NODES], fv[NODES];
  while (open(a, b)) {
    // node i covers [na, nb]; children 2i+1 = [na, m], 2i+2 = [m, nb]
    na[0] = a, nb[0] = b;
    for (int i = 0; i < NODES; ++i) {
      nm[i] = na[i] + 0.5 * (nb[i] - na[i]);
      if (2 * i + 2 < NODES) {
        na[2 * i + 1] = na[i], nb[2 * i + 1] = nm[i];
        na[2 * i + 2] = nm[i], nb[2 * i + 2] = nb[i];
      }
    }
    fbatch(nm, NODES, fv);
    int node = 0;
    for (int level = 0; level < LEVELS; ++level) {
      if (!open(a, b)) break;
      const double m = a + 0.5 * (b - a);  // == nm[node]
      if (m <= a || m >= b) return a + 0.5 * (b - a);
      const double fm = fv[node];
      if (std::isnan(fm)) throw std::runtime_error("find_root: objective is NaN");
      if (!std::isfinite(fm)) throw std::runtime_error("find_root: function value not finite");
      if (fm == 0.0) return m;
      if ((fm > 0.0) == (flo > 0.0)) {
        a = m, flo = fm;
        node = 2 * node + 2;
      } else {
        b = m;
        node = 2 * node + 1;
      }
    }
  }
  return a + 0.5 * (b - a);
}

// check_spectral (regparam.cpp:16-28): singular values are products of the
// factor SVDs' values, never negative; reject an all-zero spectrum.
void check_spectral(const kp_spectral* sd, bool need_x) {
  if (!sd) throw InvalidArgument("spectral data: null");
  if (need_x && !sd->xhat.p) throw InvalidArgument("selector requires x coordinates");
  if (!(sd->smax > 0.0)) throw InvalidArgument("spectral data: all singular values zero");
}

// minimize_log (regparam.cpp:54-88): 1024-point log grid (one batched
// launch), then golden-section refinement around the best grid point.
kp_param_choice minimize_log(const kp_spectral* sd, int kind, double omega, double lo, double hi,
                             int method) {
  auto g = [&](double l) { return spectral_value(sd, kind, l, omega); };
  kp_param_choice c{};
  c.method = method, c.bracket_lo = lo, c.bracket_hi = hi, c.grid_index = -1;
  if (hi <= lo * (1.0 + 1e-12)) {
    c.lambda = lo, c.objective_value = probe(g, lo, "minimize_log"), c.flat_objective = 1;
    return c;
  }
  const double ulo = std::log(lo), uhi = std::log(hi);
  const int grid = 1024;
  std::vector<double> ls(grid), vs(grid);
  for (int k = 0; k < grid; ++k) ls[k] = std::exp(ulo + (uhi - ulo) * k / (grid - 1));
  spectral_values(sd, kind, ls.data(), grid, omega, 0.0, vs.data());
  int best_k = -1;
  double best_v = std::numeric_limits<double>::infinity();
  double vmin = best_v, vmax = -best_v;
  for (int k = 0; k < grid; ++k) {
    const double v = vs[k];
    if (std::isnan(v)) throw std::runtime_error("minimize_log: objective is NaN");
    if (!std::isfinite(v)) continue;
    vmin = std::min(vmin, v), vmax = std::max(vmax, v);
    if (v < best_v) best_v = v, best_k = k;
  }
  if (best_k < 0) throw std::runtime_error("minimize_log: objective infinite everywhere");
  const double scale = std::max({std::abs(vmin), std::abs(vmax), 1e-300});
  if (vmax - vmin <= 1e-14 * scale) {
    const double mid = std::exp(0.5 * (ulo + uhi));
    c.lambda = mid, c.objective_value = probe(g, mid, "minimize_log"), c.flat_objective = 1;
    return c;
  }
  const double step = (uhi - ulo) / (grid - 1);
  const double a = std::max(ulo, ulo + (best_k - 1) * step);
  const double b = std::min(uhi, ulo + (best_k + 1) * step);
  const auto r = minimize_1d([&](double u) { return g(std::exp(u)); }, a, b, 1e-12);
  c.lambda = std::exp(r.first), c.objective_value = r.second;
  return c;
}

// selector bracket [max(sigma_min, 1e-10 sigma_max), sigma_max] (regparam.cpp:30-34)
std::pair<double, double> selector_bracket(const kp_spectral* sd) {
  return {std::max(sd->smin, 1e-10 * sd->smax), sd->smax};
}

// vec(Ul^T X Ur) for n x n column-major X (device), FP64 DMMA GEMMs
// (project_b, factor.cpp:157-177; the x_true projection uses the V factors).
void project_dev(int n, const double* ul, const double* ur, const double* x, double* out) {
  const size_t nn = size_t(n) * n;
  DBuf<double> t(nn);
  F64GemmArgs g;
  g.M = n, g.N = n, g.nb = 1, g.Kb = n;
  g.A = {ul, n, 0}, g.B = {x, n, 0};
  g.epi.C = t.p, g.epi.cm = n, g.epi.cn = 1;
  gemm_f64(g, KC_SPECTRAL);
  g.A = {t.p, n, 0}, g.B = {ur, n, 0};
  g.epi = F64Epilogue{}, g.epi.C = out, g.epi.cm = 1, g.epi.cn = n;
  gemm_f64(g, KC_SPECTRAL);
}

}  // namespace

// ============================================================================
// extern "C"
// ============================================================================
#define KP_API(...)                                     \
  try {                                                 \
    ensure_init();                                      \
    __VA_ARGS__;                                        \
    return KP_OK;                                       \
  } catch (const kp::NoRoot& e) {                       \
    kp::g_last_error = e.what();                        \
    return KP_ERR_NO_ROOT;                              \
  } catch (const kp::CudaError& e) {                    \
    kp::g_last_error = e.what();                        \
    return KP_ERR_CUDA;                                 \
  } catch (const kp::Unsupported& e) {                  \
    kp::g_last_error = e.what();                        \
    return KP_ERR_UNSUPPORTED;                          \
  } catch (const std::invalid_argument& e) {            \
    kp::g_last_error = e.what();                        \
    return KP_ERR_INVALID_ARGUMENT;                     \
  } catch (const std::exception& e) {                   \
    kp::g_last_error = e.what();                        \
    return KP_ERR_RUNTIME;                              \
  }

extern "C" {
// host setup routines of problem.cpp (same library)
const char* kpg_last_error(void);
int kpg_psf_to_kronsum(const double* psf, int np, int crow, int ccol, int n, double tol, int max_rank,
                       int capacity, double* row_factors, double* col_factors, int* r_out,
                       double* truncated_psf);
int kpg_nearest_kron(const double* psf, int np, int crow, int ccol, int n, int weighting,
                     double* row_factor, double* col_factor);
}

namespace {
void check_gen(int status) {  // problem.cpp status (1 invalid_argument, 2 runtime)
  if (status == 0) return;
  if (status == 1) throw InvalidArgument(kpg_last_error());
  throw std::runtime_error(kpg_last_error());
}
}  // namespace

// Host-only entry points (setup on the CPU, no device needed).
#define KP_API_HOST(...)                                \
  try {                                                 \
    __VA_ARGS__;                                        \
    return KP_OK;                                       \
  } catch (const std::invalid_argument& e) {            \
    kp::g_last_error = e.what();                        \
    return KP_ERR_INVALID_ARGUMENT;                     \
  } catch (const std::exception& e) {                   \
    kp::g_last_error = e.what();                        \
    return KP_ERR_RUNTIME;                              \
  }

extern "C" {

const char* kp_last_error(void) { return kp::g_last_error.c_str(); }

int kp_init(int device) {
  KP_API({
    Ctx& c = ctx();
    if (device != c.device) {
      // Handles created on the previous device keep the stream they were
      // allocated on (DBuf frees on it), so the old stream is not destroyed;
      // the per-kernel smem limits and events belong to the old device.
      KP_CUDA(cudaSetDevice(device));
      KP_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.smem_attr.clear();
      for (auto& e : c.events) e = nullptr;
      KP_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
      init_pool(device);
      c.device = device;
    }
  })
}
int kp_synchronize(void) { KP_API(sync()) }
int kp_device_alloc(size_t bytes, void** dptr) { KP_API(KP_CUDA(cudaMalloc(dptr, bytes))) }
int kp_device_free(void* dptr) { KP_API(KP_CUDA(cudaFree(dptr))) }
int kp_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  KP_API(KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx().stream)); sync())
}
int kp_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  KP_API(KP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx().stream)); sync())
}
int kp_profile_enable(int on) { KP_API(ctx().profile = on != 0) }
int kp_profile_reset(void) {
  KP_API({
    profile_collect();
    for (int c = 0; c < KC_COUNT; ++c) ctx().total_ms[c] = 0.0, ctx().count[c] = 0;
  })
}
int kp_profile_read(int cls, double* total_ms, long long* launches) {
  KP_API({
    if (cls < 0 || cls >= KC_COUNT) throw InvalidArgument("profile_read: bad class");
    profile_collect();
    *total_ms = ctx().total_ms[cls];
    *launches = ctx().count[cls];
  })
}
long long kp_launch_count(void) { return kp::g_launches.load(); }
int kp_drive_stats(long long* loop_solves, long long* polled_solves) {
  KP_API({
    if (loop_solves) *loop_solves = kp::g_loop_solves.load();
    if (polled_solves) *polled_solves = kp::g_polled_solves.load();
  })
}
int kp_set_fp16_products(int mode) {
  KP_API({
    if (mode < KP_FP16_PRODUCTS_AUTO || mode > KP_FP16_PRODUCTS_TENSOR)
      throw InvalidArgument("fp16 products: mode must be KP_FP16_PRODUCTS_AUTO, _CUDA_CORES or _TENSOR");
    fp16_products_setting();
    g_fp16_products.store(mode);
  })
}
int kp_get_fp16_products(int n, int* uses_tensor) {
  KP_API({
    if (!uses_tensor) throw InvalidArgument("fp16 products: null output");
    *uses_tensor = use_f16x(n) ? 1 : 0;
  })
}
int kp_event_record(int slot) {
  KP_API({
    if (slot < 0 || slot >= 16) throw InvalidArgument("event slot out of range");
    Ctx& c = ctx();  // the calling thread's events, created on its device
    if (!c.events[slot]) KP_CUDA(cudaEventCreate(&c.events[slot]));
    KP_CUDA(cudaEventRecord(c.events[slot], c.stream));
  })
}
int kp_event_elapsed(int a, int b, float* ms) {
  KP_API({
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !ctx().events[a] || !ctx().events[b])
      throw InvalidArgument("event slot not recorded");
    KP_CUDA(cudaEventSynchronize(ctx().events[b]));
    KP_CUDA(cudaEventElapsedTime(ms, ctx().events[a], ctx().events[b]));
  })
}
int kp_host_alloc(size_t bytes, void** hptr) { KP_API(KP_CUDA(cudaMallocHost(hptr, bytes))) }
int kp_host_free(void* hptr) { KP_API(KP_CUDA(cudaFreeHost(hptr))) }

// ---- operator ------------------------------------------------------------
int kp_operator_create(int n, int r, const double* row_factors, const double* col_factors,
                       kp_operator** out) {
  KP_API({
    if (r < 1) throw InvalidArgument("KroneckerSum: no terms");
    if (n < 1 || !row_factors || !col_factors || !out)
      throw InvalidArgument("KroneckerSum: factor shape mismatch");
    auto op = std::make_unique<kp_operator>();
    op->n = n, op->r = r;
    const size_t tot = size_t(r) * n * n;
    op->Cs_cm.alloc(tot), op->Cs_cm.upload(col_factors, tot);
    op->Rr_cm.alloc(tot), op->Rr_cm.upload(row_factors, tot);
    op->Cs_rm.alloc(tot), op->Rr_rm.alloc(tot);
    transpose_blocks(op->Cs_cm.p, op->Cs_rm.p, n, r);
    transpose_blocks(op->Rr_cm.p, op->Rr_rm.p, n, r);
    op->W.alloc(tot);
    detect_banded(op.get(), row_factors, col_factors);
    if (const char* env = getenv("KP_OPERATOR")) {
      if (std::string(env) == "dense") op->mode = KP_OP_DENSE;
      if (std::string(env) == "banded") op->mode = KP_OP_BANDED;
    }
    op->part.alloc(size_t(std::max(band_rows_num_ctas(n), gemm_f64_num_ctas(n, n))) * 4);
    sync();
    *out = op.release();
  })
}
int kp_operator_destroy(kp_operator* op) { KP_API(delete op) }
int kp_operator_info(const kp_operator* op, int* n, int* r) {
  KP_API({
    if (!op) throw InvalidArgument("null operator");
    *n = op->n, *r = op->r;
  })
}
int kp_operator_set_mode(kp_operator* op, int mode) {
  KP_API({
    if (!op || mode < KP_OP_AUTO || mode > KP_OP_BANDED_FUSED) throw InvalidArgument("operator mode");
    if (mode == KP_OP_BANDED_FUSED && !(op->is_banded && band_fused_supported(op->col_taps, op->row_taps)))
      throw InvalidArgument("KroneckerSum: the fused banded kernel needs 17 or 19 diagonals per factor");
    if ((mode == KP_OP_BANDED || mode == KP_OP_BANDED_FUSED) && !op->is_banded)
      throw InvalidArgument("KroneckerSum: factors are not banded Toeplitz");
    op->mode = mode;
  })
}
int kp_operator_get_mode(const kp_operator* op, int* mode, int* col_taps, int* row_taps) {
  KP_API({
    if (!op) throw InvalidArgument("null operator");
    *mode = op->use_fused() ? KP_OP_BANDED_FUSED : op->use_banded() ? KP_OP_BANDED : KP_OP_DENSE;
    *col_taps = op->use_banded() ? op->col_taps : 0;
    *row_taps = op->use_banded() ? op->row_taps : 0;
  })
}
int kp_kronsum_apply(const kp_operator* opc, const double* y, double* out) {
  KP_API({
    auto* op = const_cast<kp_operator*>(opc);
    const size_t nn = size_t(op->n) * op->n;
    DBuf<double> dy(nn), dz(nn);
    dy.upload(y, nn);
    op_apply(op, dy.p, dz.p, false, nullptr, nullptr);
    dz.download(out, nn);
    sync();
  })
}
int kp_kronsum_apply_transpose(const kp_operator* opc, const double* y, double* out) {
  KP_API({
    auto* op = const_cast<kp_operator*>(opc);
    const size_t nn = size_t(op->n) * op->n;
    DBuf<double> dy(nn), dz(nn);
    dy.upload(y, nn);
    op_apply(op, dy.p, dz.p, true, nullptr, nullptr);
    dz.download(out, nn);
    sync();
  })
}
int kp_normal_matvec(const kp_operator* opc, double lambda, const double* p, double* out) {
  KP_API({
    auto* op = const_cast<kp_operator*>(opc);
    const size_t nn = size_t(op->n) * op->n;
    DBuf<double> dp(nn), da(nn), dz(nn);
    dp.upload(p, nn);
    op_apply(op, dp.p, da.p, false, nullptr, nullptr);
    F64Epilogue e;
    e.addv = dp.p, e.addc = lambda * lambda;
    op_apply(op, da.p, dz.p, true, &e, nullptr);
    dz.download(out, nn);
    sync();
  })
}

// psf_to_kronsum (deblur.cpp:167-199) and nearest_kron (factor.cpp:25-58):
// host setup, FP64 SVD of the n_p x n_p PSF array.
int kp_psf_to_kronsum(const double* psf, int np, int center_row, int center_col, int n,
                      double truncation_tol, int max_rank, int capacity, double* row_factors,
                      double* col_factors, int* rank) {
  KP_API_HOST({
    if (!psf || np < 1 || !row_factors || !col_factors || !rank || capacity < 1)
      throw InvalidArgument("psf_to_kronsum: bad arguments");
    if (center_row < 0 || center_row >= np || center_col < 0 || center_col >= np)
      throw InvalidArgument("psf_to_kronsum: center outside the psf");
    check_gen(kpg_psf_to_kronsum(psf, np, center_row, center_col, n, truncation_tol, max_rank, capacity,
                                 row_factors, col_factors, rank, nullptr));
  })
}
int kp_nearest_kron(const double* psf, int np, int center_row, int center_col, int n, int weighting,
                    double* row_factor, double* col_factor) {
  KP_API_HOST({
    if (!psf || np < 1 || !row_factor || !col_factor) throw InvalidArgument("nearest_kron: bad arguments");
    if (weighting != KP_KRON_UNIFORM && weighting != KP_KRON_TOEPLITZ)
      throw InvalidArgument("nearest_kron: unknown weighting");
    if (center_row < 0 || center_row >= np || center_col < 0 || center_col >= np)
      throw InvalidArgument("nearest_kron: center outside the psf");
    check_gen(kpg_nearest_kron(psf, np, center_row, center_col, n, weighting, row_factor, col_factor));
  })
}

// ---- preconditioner ---------------------------------------------------------
// Setup SVD backend of kp_precond_build (svd_dense, factor.cpp:14-23):
// host LAPACK dgesdd (the oracle's routine; default) or cuSOLVER on the
// device (svd_dev.cu). Env KP_SVD=device|host sets the process default.
std::atomic<int> g_svd_backend{-1};
int svd_backend() {
  int v = g_svd_backend.load();
  if (v < 0) {
    const char* e = getenv("KP_SVD");
    v = e && std::string(e) == "device" ? KP_SVD_DEVICE : KP_SVD_HOST;
    g_svd_backend.store(v);
  }
  return v;
}
kpla::Svd factor_svd(const double* a, int n, int backend) {
  if (backend == KP_SVD_DEVICE) {
    kpla::Svd o;
    o.u.resize(size_t(n) * n), o.v.resize(size_t(n) * n), o.s.resize(n);
    device_svd(a, n, o.u.data(), o.s.data(), o.v.data());
    return o;
  }
  return kpla::svd(a, n, n);
}

int kp_set_svd_backend(int backend) {
  KP_API({
    if (backend != KP_SVD_HOST && backend != KP_SVD_DEVICE)
      throw InvalidArgument("svd backend: must be KP_SVD_HOST or KP_SVD_DEVICE");
    svd_backend();
    g_svd_backend.store(backend);
  })
}
int kp_get_svd_backend(int* backend) {
  KP_API({
    if (!backend) throw InvalidArgument("svd backend: null output");
    *backend = svd_backend();
  })
}
int kp_svd(const double* a, int n, int backend, double* u, double* s, double* v) {
  KP_API({
    if (n < 1 || !a || !u || !s || !v) throw InvalidArgument("svd_dense: empty matrix");
    if (backend != KP_SVD_HOST && backend != KP_SVD_DEVICE)
      throw InvalidArgument("svd backend: must be KP_SVD_HOST or KP_SVD_DEVICE");
    kpla::Svd o = factor_svd(a, n, backend);
    std::memcpy(u, o.u.data(), o.u.size() * sizeof(double));
    std::memcpy(s, o.s.data(), o.s.size() * sizeof(double));
    std::memcpy(v, o.v.data(), o.v.size() * sizeof(double));
  })
}

int kp_precond_build(const double* a_r, const double* a_c, int n, double lambda, kp_format fmt,
                     int accum, kp_precond** out) {
  KP_API({
    if (n < 1 || !a_r || !a_c) throw InvalidArgument("build_preconditioner: factors must be square and equally sized");
    if (lambda < 0.0) throw InvalidArgument("build_preconditioner: negative lambda");
    const int be = svd_backend();
    kpla::Svd r = factor_svd(a_r, n, be);
    kpla::Svd c = factor_svd(a_c, n, be);
    *out = precond_from_svd(n, std::move(r.u), std::move(r.s), std::move(r.v), std::move(c.u),
                            std::move(c.s), std::move(c.v), lambda, fmt, accum);
    g_round_calls += 3;  // round_array of V_r, V_c, S (factor.cpp:100-102)
  })
}
int kp_precond_build_from_svd(int n, const double* u_r, const double* s_r, const double* v_r,
                              const double* u_c, const double* s_c, const double* v_c,
                              double lambda, kp_format fmt, int accum, kp_precond** out) {
  KP_API({
    const size_t nn = size_t(n) * n;
    auto vec = [&](const double* p, size_t k) { return std::vector<double>(p, p + k); };
    *out = precond_from_svd(n, vec(u_r, nn), vec(s_r, n), vec(v_r, nn), vec(u_c, nn), vec(s_c, n),
                            vec(v_c, nn), lambda, fmt, accum);
    g_round_calls += 3;
  })
}
int kp_precond_with_lambda(const kp_precond* p, double lambda, kp_precond** out) {
  KP_API({
    if (!p) throw InvalidArgument("with_lambda: null preconditioner");
    if (lambda < 0.0) throw InvalidArgument("with_lambda: negative lambda");
    auto q = std::make_unique<kp_precond>();
    q->sh = p->sh, q->n = p->n, q->lambda = lambda, q->fmt = p->fmt, q->accum = p->accum;
    set_weights(q.get());
    *out = q.release();
    g_round_calls += 1;  // round_array of S (factor.cpp:113)
  })
}
int kp_precond_destroy(kp_precond* p) { KP_API(delete p) }
int kp_round_call_count(unsigned long long* count) {
  KP_API({
    if (!count) throw InvalidArgument("round_call_count: null output");
    *count = g_round_calls;
  })
}
int kp_precond_solve(const kp_precond* pc, const double* r, double* z) {
  KP_API({
    auto* p = const_cast<kp_precond*>(pc);
    const size_t nn = size_t(p->n) * p->n;
    DBuf<double> dr(nn), dz(nn);
    dr.upload(r, nn);
    if (is_fp16(p->fmt)) cast_r16(p, dr.p, nullptr);
    msolve(p, dr.p, dz.p, nullptr, nullptr, nullptr, nullptr);
    dz.download(z, nn);
    sync();
    g_round_calls += msolve_round_calls(p->fmt, p->n);
  })
}
int kp_precond_export(const kp_precond* p, int field, double* out) {
  KP_API({
    if (!p) throw InvalidArgument("precond_export: null");
    const int n = p->n;
    const size_t nn = size_t(n) * n;
    auto* sh = p->sh.get();
    auto put = [&](const std::vector<double>& v) { std::memcpy(out, v.data(), v.size() * sizeof(double)); };
    auto put_half = [&](const __half* d, long ld, bool transpose_back) {
      std::vector<__half> h(size_t(n) * ld);
      KP_CUDA(cudaMemcpyAsync(h.data(), d, h.size() * sizeof(__half), cudaMemcpyDeviceToHost, ctx().stream));
      sync();
      for (int a = 0; a < n; ++a)
        for (int i = 0; i < n; ++i) {
          const double v = double(__half2float(h[size_t(a) * ld + i]));
          if (transpose_back) out[size_t(i) * n + a] = v;  // row a holds column a
          else out[size_t(a) * n + i] = v;
        }
    };
    auto put_dev = [&](const double* d) {
      KP_CUDA(cudaMemcpyAsync(out, d, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
      sync();
    };
    if (is_generic(p->fmt) && field >= 1 && field <= 3) {  // rounded copies on the device
      put_dev(field == 1 ? p->s64.p : field == 2 ? sh->vr.p : sh->vc.p);
      return KP_OK;
    }
    switch (field) {
      case 0: put(weight_matrix(*sh, p->lambda)); break;
      case 1:
        if (covers_double(p->fmt)) put(weight_matrix(*sh, p->lambda));
        else put_half(p->s16.p, n, false);
        break;
      case 2:
        if (covers_double(p->fmt)) put(sh->v_r);
        else put_half(sh->vr_b.p, sh->ldh, false);
        break;
      case 3:
        if (covers_double(p->fmt)) put(sh->v_c);
        else put_half(sh->vc_a.p, sh->ldh, false);
        break;
      case 4: put(sh->s_r); break;
      case 5: put(sh->s_c); break;
      case 6: put(sh->u_r); break;
      case 7: put(sh->v_r); break;
      case 8: put(sh->u_c); break;
      case 9: put(sh->v_c); break;
      default: throw InvalidArgument("precond_export: bad field");
    }
  })
}
int kp_precond_info(const kp_precond* p, int* n, double* lambda, kp_format* fmt, int* accum) {
  KP_API({
    if (!p) throw InvalidArgument("null preconditioner");
    *n = p->n, *lambda = p->lambda, *fmt = p->fmt, *accum = p->accum;
  })
}

// ---- emulated low-precision BLAS (precision.cpp, lpblas.cpp) ---------------------
int kp_round_array(const double* x, long count, kp_format fmt, double* out) {
  KP_API({
    check_format(fmt);
    if (count < 0 || (count && (!x || !out))) throw InvalidArgument("round_array: bad arguments");
    g_round_calls += 1;  // round_inplace counts every call (precision.cpp:90)
    if (!count) return KP_OK;
    DBuf<double> d(static_cast<size_t>(count));
    d.upload(x, size_t(count));
    lp_round_array(d.p, size_t(count), lp_format(fmt), d.p, KC_PRECOND);
    d.download(out, size_t(count));
    sync();
  })
}
// round_value (precision.cpp:82-86): one scalar through the same device kernel;
// scalar rounding is not tallied (precision.hpp:40).
int kp_round_value(double x, kp_format fmt, double* out) {
  KP_API({
    check_format(fmt);
    if (!out) throw InvalidArgument("round_value: null output");
    DBuf<double> d(1);
    d.upload(&x, 1);
    lp_round_array(d.p, 1, lp_format(fmt), d.p, KC_PRECOND);
    d.download(out, 1);
    sync();
  })
}
// lp_matmul (lpblas.cpp:59-70): a is m x k, b is k x n, c is m x n, all
// column-major host arrays. fp16 with binary16-representable inputs runs on
// the f16x2 GEMM (gemm_f16ref); everything else on the generic emulation.
// round_leaves = 0 treats the products as pre-rounded addends (pairwise_sum).
int kp_lp_matmul_ex(int m, int k, int n, const double* a, const double* b, kp_format fmt,
                    int round_leaves, double* c) {
  KP_API({
    check_format(fmt);
    if (m < 0 || n < 0 || k < 0) throw InvalidArgument("lp_matmul: negative dimension");
    if (k == 0) throw InvalidArgument("lp_matmul: empty input");
    if (!covers_double(fmt)) g_round_calls += (round_leaves ? 1 : 0) + tree_stages(k);  // lpblas.cpp:24,68
    if (m == 0 || n == 0) return KP_OK;
    const size_t na = size_t(m) * k, nb = size_t(k) * n, nc = size_t(m) * n;
    DBuf<double> da(na), db(nb), dc(nc);
    da.upload(a, na);
    db.upload(b, nb);
    if (is_fp16(fmt) && round_leaves && count_not_f16(da.p, na) + count_not_f16(db.p, nb) == 0) {
      const long ldh = round_up(k, 64);
      DBuf<__half> ha(size_t(m) * ldh), hb(size_t(n) * ldh);
      pack_f16(da.p, 1, m, m, k, ha.p, ldh, 0x8000);  // A(i,kk) = a[i + kk m], -0 padding
      pack_f16(db.p, k, 1, n, k, hb.p, ldh, 0x0000);  // B(j,kk) = b[kk + j k], +0 padding
      F16GemmArgs g;
      g.M = m, g.N = n, g.K = k;
      g.A = {ha.p, ldh}, g.B = {hb.p, ldh};
      g.epi.mode = F16OUT_F64, g.epi.Cd = dc.p, g.epi.cm = 1, g.epi.cn = m;
      bool a_finite = true;  // gemm_f16x: A must be finite (see gemm_f16x.cu)
      for (size_t q = 0; q < na && a_finite; ++q) a_finite = std::isfinite(a[q]);
      if (a_finite && use_f16x(std::min(m, n))) {
        DBuf<unsigned> zf;
        ensure_zfix(zf, m, n);
        DBuf<unsigned long long> hsa(m), hsb(n);
        g.zfix = zf.p, g.hash_a = hsa.p, g.hash_b = hsb.p;
        gemm_f16x(g, KC_PRECOND);
      } else {
        gemm_f16ref(g, KC_PRECOND);
      }
    } else {
      LpGemmArgs g;
      g.M = m, g.N = n, g.K = k, g.f = lp_format(fmt), g.round_leaves = round_leaves != 0;
      g.a = da.p, g.ai = 1, g.ak = m;
      g.b = db.p, g.bk = 1, g.bj = k;
      g.c = dc.p, g.ldc = m;
      lp_gemm_generic(g, KC_PRECOND);
    }
    dc.download(c, nc);
    sync();
  })
}
int kp_lp_matmul(int m, int k, int n, const double* a, const double* b, kp_format fmt,
                 double* c) {
  return kp_lp_matmul_ex(m, k, n, a, b, fmt, 1, c);
}

// ---- solvers --------------------------------------------------------------------
int kp_cgls(const kp_operator* op, const double* b, const kp_solver_options* o, double* x,
            kp_history* h) {
  KP_API(run_cgls(const_cast<kp_operator*>(op), b, o, x, h))
}
int kp_pcg(const kp_operator* op, const double* b, const kp_precond* m, const kp_solver_options* o,
           double* x, kp_history* h) {
  KP_API({
    run_pcg(const_cast<kp_operator*>(op), b, const_cast<kp_precond*>(m), o, x, h, false);
    if (h) g_round_calls += (unsigned long long)h->msolve_count * msolve_round_calls(m->fmt, m->n);
  })
}
int kp_fpcg(const kp_operator* op, const double* b, const kp_precond* m,
            const kp_solver_options* o, double* x, kp_history* h) {
  KP_API({
    run_pcg(const_cast<kp_operator*>(op), b, const_cast<kp_precond*>(m), o, x, h, true);
    if (h) g_round_calls += (unsigned long long)h->msolve_count * msolve_round_calls(m->fmt, m->n);
  })
}
int kp_pcg_batch(const kp_operator* op, const kp_precond* m, int batch, const double* b,
                 const double* lambdas, const kp_solver_options* o, double* x, kp_history* h) {
  KP_API({
    run_pcg_batch(const_cast<kp_operator*>(op), const_cast<kp_precond*>(m), batch, b, lambdas, o, x, h, false);
    for (int i = 0; h && i < batch; ++i)
      g_round_calls += (unsigned long long)h[i].msolve_count * msolve_round_calls(m->fmt, m->n);
  })
}
int kp_fpcg_batch(const kp_operator* op, const kp_precond* m, int batch, const double* b,
                  const double* lambdas, const kp_solver_options* o, double* x, kp_history* h) {
  KP_API({
    run_pcg_batch(const_cast<kp_operator*>(op), const_cast<kp_precond*>(m), batch, b, lambdas, o, x, h, true);
    for (int i = 0; h && i < batch; ++i)
      g_round_calls += (unsigned long long)h[i].msolve_count * msolve_round_calls(m->fmt, m->n);
  })
}

// ---- lambda selection ------------------------------------------------------------
// make_spectral_data (regparam.cpp:119-134): b_hat = vec(U_c^T B U_r) and,
// with x_true, x_hat = vec(V_c^T X V_r) on the device.
int kp_spectral_create_x(const kp_precond* p, const double* b, const double* x_true,
                         kp_spectral** out) {
  KP_API({
    if (!p || !b) throw InvalidArgument("make_spectral_data: null argument");
    const int n = p->n;
    const size_t nn = size_t(n) * n;
    auto sd = std::make_unique<kp_spectral>();
    sd->n = n;
    sd->sh = p->sh;
    auto& sh = *sd->sh;
    sd->bhat.alloc(nn);
    {
      DBuf<double> db(nn);
      db.upload(b, nn);
      project_dev(n, sh.d_u_c.p, sh.d_u_r.p, db.p, sd->bhat.p);
      if (x_true) {
        {
          std::lock_guard<std::mutex> lk(sh.lazy_mu);
          if (!sh.d_v_r.p) {
            sh.d_v_r.alloc(nn), sh.d_v_r.upload(sh.v_r.data(), nn);
            sh.d_v_c.alloc(nn), sh.d_v_c.upload(sh.v_c.data(), nn);
            sync();
          }
        }
        sd->xhat.alloc(nn);
        db.upload(x_true, nn);
        project_dev(n, sh.d_v_c.p, sh.d_v_r.p, db.p, sd->xhat.p);
      }
      sync();
    }
    std::lock_guard<std::mutex> lk(sh.lazy_mu);
    if (!sh.have_range) {
      const auto& sr = sh.s_r;
      const auto& sc = sh.s_c;
      sh.smax = sr[0] * sc[0];
      sh.smin = std::numeric_limits<double>::infinity();
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sh.smin = std::min(sh.smin, sr[j] * sc[i]);
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sh.smax = std::max(sh.smax, sr[j] * sc[i]);
      sh.have_range = true;
    }
    sd->smin = sh.smin, sd->smax = sh.smax;
    *out = sd.release();
  })
}
int kp_spectral_create(const kp_precond* p, const double* b, kp_spectral** out) {
  return kp_spectral_create_x(p, b, nullptr, out);
}
// filtered_solution (regparam.cpp:329-349): X = V_c (F .* (U_c^T B U_r)) V_r^T
// with F(i,j) = sigma / (sigma^2 + lambda^2), sigma = s_r(j) s_c(i); FP64.
int kp_filtered_solution(const kp_precond* p, const double* b, double lambda, double* x) {
  KP_API({
    if (!p || !b || !x) throw InvalidArgument("filtered_solution: null argument");
    if (lambda < 0.0) throw InvalidArgument("filtered_solution: negative lambda");
    const int n = p->n;
    const size_t nn = size_t(n) * n;
    auto& sh = *p->sh;
    if (lambda == 0.0) {
      double mn = std::numeric_limits<double>::infinity();
      for (double v : sh.s_r) mn = std::min(mn, std::fabs(v));
      double mc = std::numeric_limits<double>::infinity();
      for (double v : sh.s_c) mc = std::min(mc, std::fabs(v));
      if ((mn * mc) * (mn * mc) == 0.0)
        throw InvalidArgument("filtered_solution: zero singular value with lambda = 0");
    }
    std::unique_lock<std::mutex> lk(sh.lazy_mu);
    if (!sh.d_vc_rm.p) {  // row-major copies of V_c, V_r (K-major operands below)
      sh.d_vc_rm.alloc(nn), sh.d_vc_rm.upload(host_transpose(sh.v_c, n).data(), nn);
      sh.d_vr_rm.alloc(nn), sh.d_vr_rm.upload(host_transpose(sh.v_r, n).data(), nn);
      sync();
    }
    lk.unlock();
    DBuf<double> db(nn), bh(nn), t(nn);
    db.upload(b, nn);
    project_dev(n, sh.d_u_c.p, sh.d_u_r.p, db.p, bh.p);
    spectral_filter(sh.d_s_r.p, sh.d_s_c.p, n, lambda * lambda, bh.p);  // coef in place
    F64GemmArgs g;  // t = V_c coef ; X = t V_r^T
    g.M = n, g.N = n, g.nb = 1, g.Kb = n;
    g.A = {sh.d_vc_rm.p, n, 0}, g.B = {bh.p, n, 0};
    g.epi.C = t.p, g.epi.cm = n, g.epi.cn = 1;
    gemm_f64(g, KC_SPECTRAL);
    g.A = {t.p, n, 0}, g.B = {sh.d_vr_rm.p, n, 0};
    g.epi = F64Epilogue{}, g.epi.C = db.p, g.epi.cm = 1, g.epi.cn = n;
    gemm_f64(g, KC_SPECTRAL);
    db.download(x, nn);
    sync();
  })
}
int kp_spectral_export_xhat(const kp_spectral* sd, double* x_hat) {
  KP_API({
    if (!sd || !sd->xhat.p) throw InvalidArgument("spectral data: x coordinates missing");
    const int n = sd->n;
    const size_t nn = size_t(n) * n;
    std::vector<double> prod(nn), xh(nn);
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < n; ++i) prod[j * n + i] = sd->sh->s_r[j] * sd->sh->s_c[i];
    sd->xhat.download(xh.data(), nn);
    sync();
    std::vector<long> perm(nn);
    std::iota(perm.begin(), perm.end(), 0L);
    std::stable_sort(perm.begin(), perm.end(), [&](long a, long b) { return prod[a] > prod[b]; });
    for (size_t k = 0; k < nn; ++k) x_hat[k] = xh[perm[k]];
  })
}
int kp_spectral_destroy(kp_spectral* sd) { KP_API(delete sd) }
int kp_spectral_export(const kp_spectral* sd, double* sigma_hat, double* b_hat) {
  KP_API({
    const int n = sd->n;
    const size_t nn = size_t(n) * n;
    std::vector<double> prod(nn), bh(nn);
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < n; ++i) prod[j * n + i] = sd->sh->s_r[j] * sd->sh->s_c[i];
    sd->bhat.download(bh.data(), nn);
    sync();
    std::vector<long> perm(nn);
    std::iota(perm.begin(), perm.end(), 0L);
    std::stable_sort(perm.begin(), perm.end(), [&](long a, long b) { return prod[a] > prod[b]; });
    for (size_t k = 0; k < nn; ++k) {
      if (sigma_hat) sigma_hat[k] = prod[perm[k]];
      if (b_hat) b_hat[k] = bh[perm[k]];
    }
  })
}
int kp_gcv_objective(const kp_spectral* sd, double lambda, double* value) {
  KP_API(*value = gcv_value(sd, lambda))
}
int kp_discrepancy_gap(const kp_spectral* sd, double epsilon, double lambda, double* value) {
  KP_API(*value = gap_value(sd, epsilon, lambda))
}
int kp_gcv_grid(const kp_spectral* sd, const double* lambdas, int m, double* values,
                kp_param_choice* choice) {
  KP_API({
    if (!sd || !lambdas || m < 1) throw InvalidArgument("gcv_grid: bad arguments");
    std::vector<double> v(m);
    gcv_values(sd, lambdas, m, v.data());
    int best = -1;
    double bv = std::numeric_limits<double>::infinity();
    for (int q = 0; q < m; ++q) {
      if (std::isnan(v[q])) throw std::runtime_error("gcv_grid: objective is NaN");
      if (v[q] < bv) bv = v[q], best = q;
    }
    if (best < 0) throw std::runtime_error("gcv_grid: objective infinite everywhere");
    if (values) std::memcpy(values, v.data(), m * sizeof(double));
    if (choice) {
      *choice = kp_param_choice{};
      choice->lambda = lambdas[best];
      choice->method = 4;
      choice->objective_value = bv;
      choice->bracket_lo = lambdas[0];
      choice->bracket_hi = lambdas[m - 1];
      choice->grid_index = best;
    }
  })
}
// gcv (regparam.cpp:254-258) = run_selector(minimize_log)
int kp_gcv(const kp_spectral* sd, kp_param_choice* choice) {
  KP_API({
    check_spectral(sd, false);
    const auto br = selector_bracket(sd);
    *choice = minimize_log(sd, SK_GCV, 0.0, br.first, br.second, 1);
  })
}
// lambda_opt (regparam.cpp:248-252)
int kp_lambda_opt(const kp_spectral* sd, kp_param_choice* choice) {
  KP_API({
    check_spectral(sd, true);
    const auto br = selector_bracket(sd);
    *choice = minimize_log(sd, SK_OPT, 0.0, br.first, br.second, 0);
  })
}
// wgcv (regparam.cpp:260-286): for omega > 1 start where the trace term
// turns positive (log-bisection to 1e-13 relative width)
int kp_wgcv(const kp_spectral* sd, double omega, kp_param_choice* choice) {
  KP_API({
    check_spectral(sd, false);
    if (!(omega > 0.0)) throw InvalidArgument("wgcv: omega must be positive");
    auto [lo, hi] = selector_bracket(sd);
    auto tr = [&](double l) { return spectral_value(sd, SK_WTRACE, l, omega); };
    if (omega > 1.0 && tr(lo) < 0.0 && tr(hi) > 0.0) {
      double a = std::log(lo), b = std::log(hi);
      while (b - a > 1e-13 * (1.0 + std::abs(b))) {
        const double m = 0.5 * (a + b);
        (tr(std::exp(m)) > 0.0 ? b : a) = m;
      }
      lo = std::exp(b);
    }
    *choice = minimize_log(sd, SK_WGCV, omega, lo, hi, 2);
    choice->omega = omega;
  })
}
int kp_opt_objective(const kp_spectral* sd, double lambda, double* value) {
  KP_API(*value = spectral_value(sd, SK_OPT, lambda))
}
int kp_wgcv_objective(const kp_spectral* sd, double omega, double lambda, double* value) {
  KP_API(*value = spectral_value(sd, SK_WGCV, lambda, omega))
}
// discrepancy (regparam.cpp:288-327)
// Discrepancy principle for a batch of right-hand sides sharing the
// preconditioner factors (BASELINE C4): per image the spectral data of
// make_spectral_data (regparam.cpp:119-126) and discrepancy()'s root search
// (regparam.cpp:288-327, find_root :184-214, with the two-level look-ahead
// of find_root_batched), but every round evaluates the candidate lambdas of
// ALL still-open images in one batched reduction launch. Each image takes
// exactly the decisions, and gets exactly the lambda, of kp_discrepancy on
// its own spectral data (same per-lambda sums, same host decisions).
// status[i]: 0, or KP_ERR_NO_ROOT (no sign change in the bracket) /
// KP_ERR_RUNTIME (non-finite objective) with lambdas[i] = NaN.
// make_test_problem (deblur.cpp:201-229) for `batch` images on the device:
// x_true = the BASELINE blob image (seed image_seeds[i], `blobs` blobs; blob
// parameters drawn by the host Rng exactly as kpg_blob_image draws them),
// b_true = A x_true (this operator), noise from Rng(noise_seeds[i]).normal()
// scaled to noise_levels[i] * ||b_true|| (problem_dev.cu), b = b_true +
// noise. x_true / b / noise: batch * n^2 (host or device per
// device_pointers; noise optional); noise_norms: host, batch (optional).
int kp_generate_test_problems(const kp_operator* opc, int batch, const unsigned long long* image_seeds,
                              int blobs, const unsigned long long* noise_seeds, const double* noise_levels,
                              double* x_true, double* b, double* noise, double* noise_norms,
                              int device_pointers) {
  KP_API({
    auto* op = const_cast<kp_operator*>(opc);
    if (!op || batch < 1 || blobs < 0 || !image_seeds || !noise_seeds || !noise_levels || !x_true || !b)
      throw InvalidArgument("generate_test_problems: bad arguments");
    for (int i = 0; i < batch; ++i)
      if (noise_levels[i] < 0.0) throw InvalidArgument("make_test_problem: negative noise level");
    const int n = op->n;
    const size_t nn = size_t(n) * n, bnn = size_t(batch) * nn;
    std::vector<double> params(size_t(batch) * std::max(blobs, 1) * 4);
    for (int i = 0; i < batch; ++i) kpg_blob_params(n, image_seeds[i], blobs, params.data() + size_t(i) * blobs * 4);
    DBuf<double> dparams(params.size()), dlev(batch), dnorm(batch);
    DBuf<uint64_t> dseeds(batch);
    dparams.upload(params.data(), params.size());
    dlev.upload(noise_levels, batch);
    KP_CUDA(cudaMemcpyAsync(dseeds.p, noise_seeds, batch * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx().stream));
    const bool dev = device_pointers != 0;
    DBuf<double> own_x, own_b, own_e, bt(bnn);
    double* dx = dev ? x_true : (own_x.alloc(bnn), own_x.p);
    double* db = dev ? b : (own_b.alloc(bnn), own_b.p);
    double* de = (dev && noise) ? noise : (own_e.alloc(bnn), own_e.p);
    blob_images_dev(n, batch, blobs, dparams.p, dx);
    op_apply_batch(op, batch, dx, bt.p, false, nullptr, nullptr, nullptr, nullptr);  // b_true = A x_true
    rng_normals_dev(dseeds.p, batch, long(nn), de);
    add_noise_dev(batch, nn, dlev.p, bt.p, de, db, dnorm.p);
    if (!dev) {
      KP_CUDA(cudaMemcpyAsync(x_true, dx, bnn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
      KP_CUDA(cudaMemcpyAsync(b, db, bnn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
      if (noise) KP_CUDA(cudaMemcpyAsync(noise, de, bnn * sizeof(double), cudaMemcpyDeviceToHost, ctx().stream));
    }
    if (noise_norms) dnorm.download(noise_norms, batch);
    sync();
  })
}
// std::mt19937_64 on the device (test hook): count raw outputs per seed
int kp_rng_raw(const unsigned long long* seeds, int batch, long count, unsigned long long* out) {
  KP_API({
    if (!seeds || !out || batch < 1 || count < 0) throw InvalidArgument("rng_raw: bad arguments");
    DBuf<uint64_t> ds(batch), dout(size_t(batch) * count);
    KP_CUDA(cudaMemcpyAsync(ds.p, seeds, batch * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx().stream));
    mt19937_64_raw(ds.p, batch, count, dout.p);
    KP_CUDA(cudaMemcpyAsync(out, dout.p, size_t(batch) * count * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            ctx().stream));
    sync();
  })
}

int kp_discrepancy_batch(const kp_precond* p, int batch, const double* b, const double* noise_norms,
                         double eta, double* lambdas, int* status) {
  return kp_discrepancy_batch_ex(p, batch, b, noise_norms, eta, lambdas, status, 0);
}
int kp_discrepancy_batch_ex(const kp_precond* p, int batch, const double* b, const double* noise_norms,
                            double eta, double* lambdas, int* status, int device_pointers) {
  KP_API({
    if (!p || !b || !noise_norms || !lambdas || !status || batch < 1)
      throw InvalidArgument("discrepancy_batch: bad arguments");
    if (!(eta > 0.0)) throw InvalidArgument("discrepancy: eta must be positive");
    for (int i = 0; i < batch; ++i)
      if (!(noise_norms[i] > 0.0)) throw InvalidArgument("discrepancy: noise_norm must be positive");
    const int n = p->n;
    const size_t nn = size_t(n) * n;
    auto& sh = *p->sh;
    // spectral data of every image (b_hat = vec(U_c^T B U_r), one image at a time)
    DBuf<double> bhat(size_t(batch) * nn);
    {
      DBuf<double> db;
      if (!device_pointers) db.alloc(nn);
      for (int i = 0; i < batch; ++i) {
        if (device_pointers) {  // b already in device memory: project in place
          project_dev(n, sh.d_u_c.p, sh.d_u_r.p, b + size_t(i) * nn, bhat.p + size_t(i) * nn);
        } else {
          db.upload(b + size_t(i) * nn, nn);
          project_dev(n, sh.d_u_c.p, sh.d_u_r.p, db.p, bhat.p + size_t(i) * nn);
        }
      }
    }
    {
      std::lock_guard<std::mutex> lk(sh.lazy_mu);
      if (!sh.have_range) {
        sh.smax = sh.s_r[0] * sh.s_c[0];
        sh.smin = std::numeric_limits<double>::infinity();
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) {
            sh.smin = std::min(sh.smin, sh.s_r[j] * sh.s_c[i]);
            sh.smax = std::max(sh.smax, sh.s_r[j] * sh.s_c[i]);
          }
        sh.have_range = true;
      }
    }
    if (!(sh.smax > 0.0)) throw InvalidArgument("spectral data: all singular values zero");
    // evaluate the gap for per-image lambda lists (m values each) of the images in `act`
    auto gaps = [&](const std::vector<int>& act, const std::vector<double>& lam, int m,
                    std::vector<double>& out) {
      const int B = int(act.size());
      DBuf<double> dl(size_t(B) * m), sums(size_t(B) * m * 2);
      DBuf<int> didx(B);
      dl.upload(lam.data(), size_t(B) * m);
      KP_CUDA(cudaMemcpyAsync(didx.p, act.data(), B * sizeof(int), cudaMemcpyHostToDevice, ctx().stream));
      spectral_sums(SK_RESID, sh.d_s_r.p, sh.d_s_c.p, bhat.p, nullptr, n, dl.p, m, 0.0, sums.p, B, didx.p);
      std::vector<double> hsum(size_t(B) * m * 2);
      sums.download(hsum.data(), hsum.size());
      sync();
      out.resize(size_t(B) * m);
      for (int q = 0; q < B; ++q) {
        const double eps = eta * noise_norms[act[q]];
        for (int c = 0; c < m; ++c) out[size_t(q) * m + c] = hsum[(size_t(q) * m + c) * 2] - eps * eps;
      }
    };
    const double lo = 1e-10 * sh.smax, hi = sh.smax;
    std::vector<int> all(batch);
    for (int i = 0; i < batch; ++i) all[i] = i, status[i] = 0, lambdas[i] = std::nan("");
    // endpoints: gap(lo), gap(hi) as kp_discrepancy evaluates them (one value per launch width 1)
    std::vector<double> glo, ghi;
    gaps(all, std::vector<double>(batch, lo), 1, glo);
    gaps(all, std::vector<double>(batch, hi), 1, ghi);
    struct Walk {
      double a, b, flo;
      bool open;
    };
    std::vector<Walk> w(batch);
    std::vector<int> act;
    for (int i = 0; i < batch; ++i) {
      if (ghi[i] < 0.0 || glo[i] > 0.0) {
        status[i] = KP_ERR_NO_ROOT;
        continue;
      }
      if (glo[i] == 0.0) { lambdas[i] = lo; continue; }
      if (ghi[i] == 0.0) { lambdas[i] = hi; continue; }
      act.push_back(i);
    }
    // find_root_batched's opening evaluation of the log-bracket ends (width 2)
    const double ulo = std::log(lo), uhi = std::log(hi);
    if (!act.empty()) {
      std::vector<double> l(act.size() * 2), fe;
      for (size_t q = 0; q < act.size(); ++q) l[2 * q] = std::exp(ulo), l[2 * q + 1] = std::exp(uhi);
      gaps(act, l, 2, fe);
      std::vector<int> keep;
      for (size_t q = 0; q < act.size(); ++q) {
        const int i = act[q];
        const double flo = fe[2 * q], fhi = fe[2 * q + 1];
        if (std::isnan(flo) || std::isnan(fhi) || !std::isfinite(flo) || !std::isfinite(fhi)) {
          status[i] = KP_ERR_RUNTIME;
          continue;
        }
        if (flo == 0.0) { lambdas[i] = std::exp(ulo); continue; }
        if (fhi == 0.0) { lambdas[i] = std::exp(uhi); continue; }
        if ((flo > 0.0) == (fhi > 0.0)) { status[i] = KP_ERR_NO_ROOT; continue; }
        w[i] = Walk{ulo, uhi, flo, true};
        keep.push_back(i);
      }
      act.swap(keep);
    }
    const double tol = 1e-12;
    auto open = [&](double a, double b) { return b - a > tol * (1.0 + 0.5 * (std::abs(a) + std::abs(b))); };
    constexpr int LEVELS = 2, NODES = (1 << LEVELS) - 1;
    for (int i : act)
      if (!open(w[i].a, w[i].b)) lambdas[i] = std::exp(w[i].a + 0.5 * (w[i].b - w[i].a)), w[i].open = false;
    act.erase(std::remove_if(act.begin(), act.end(), [&](int i) { return !w[i].open; }), act.end());
    while (!act.empty()) {
      const size_t B = act.size();
      std::vector<double> nm(B * NODES), l(B * NODES), fv;
      for (size_t q = 0; q < B; ++q) {
        double na[NODES], nb[NODES];
        na[0] = w[act[q]].a, nb[0] = w[act[q]].b;
        for (int k = 0; k < NODES; ++k) {
          nm[q * NODES + k] = na[k] + 0.5 * (nb[k] - na[k]);
          if (2 * k + 2 < NODES) {
            na[2 * k + 1] = na[k], nb[2 * k + 1] = nm[q * NODES + k];
            na[2 * k + 2] = nm[q * NODES + k], nb[2 * k + 2] = nb[k];
          }
          l[q * NODES + k] = std::exp(nm[q * NODES + k]);
        }
      }
      gaps(act, l, NODES, fv);
      std::vector<int> keep;
      for (size_t q = 0; q < B; ++q) {
        const int i = act[q];
        Walk& wk = w[i];
        int node = 0;
        bool done = false;
        for (int level = 0; level < LEVELS && !done; ++level) {
          if (!open(wk.a, wk.b)) break;
          const double m = wk.a + 0.5 * (wk.b - wk.a);
          if (m <= wk.a || m >= wk.b) { lambdas[i] = std::exp(wk.a + 0.5 * (wk.b - wk.a)); done = true; break; }
          const double fm = fv[q * NODES + node];
          if (!std::isfinite(fm)) { status[i] = KP_ERR_RUNTIME; done = true; break; }
          if (fm == 0.0) { lambdas[i] = std::exp(m); done = true; break; }
          if ((fm > 0.0) == (wk.flo > 0.0)) {
            wk.a = m, wk.flo = fm;
            node = 2 * node + 2;
          } else {
            wk.b = m;
            node = 2 * node + 1;
          }
        }
        if (done) continue;
        if (!open(wk.a, wk.b)) {
          lambdas[i] = std::exp(wk.a + 0.5 * (wk.b - wk.a));
          continue;
        }
        keep.push_back(i);
      }
      act.swap(keep);
    }
  })
}

int kp_discrepancy(const kp_spectral* sd, double noise_norm, double eta, kp_param_choice* choice) {
  KP_API({
    check_spectral(sd, false);  // regparam.cpp: validation order of discrepancy()
    if (!choice) throw InvalidArgument("discrepancy: null output");
    if (!(noise_norm > 0.0)) throw InvalidArgument("discrepancy: noise_norm must be positive");
    if (!(eta > 0.0)) throw InvalidArgument("discrepancy: eta must be positive");
    const double eps = eta * noise_norm;
    const double lo = 1e-10 * sd->smax, hi = sd->smax;
    const double glo = gap_value(sd, eps, lo), ghi = gap_value(sd, eps, hi);
    if (ghi < 0.0)
      throw NoRoot("no root; eta * noise_norm too large: the residual cannot reach it inside the bracket");
    if (glo > 0.0)
      throw NoRoot("no root; eta * noise_norm too small: the residual exceeds it everywhere in the bracket");
    double lambda;
    if (glo == 0.0) lambda = lo;
    else if (ghi == 0.0) lambda = hi;
    else
      lambda = std::exp(find_root_batched(
          [&](const double* us, int m, double* v) {
            std::vector<double> l(m);
            for (int q = 0; q < m; ++q) l[q] = std::exp(us[q]);
            spectral_values(sd, SK_RESID, l.data(), m, 0.0, eps, v);
          },
          std::log(lo), std::log(hi), 1e-12));
    kp_param_choice c{};
    c.lambda = lambda, c.method = 3, c.eta = eta, c.noise_norm = noise_norm;
    c.objective_value = gap_value(sd, eps, lambda);
    c.bracket_lo = lo, c.bracket_hi = hi, c.grid_index = -1;
    *choice = c;
  })
}

}  // extern "C"
