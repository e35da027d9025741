// Shared infrastructure for the sm_100a kernels and the C-ABI host layer:
// library context (device, stream), error capture, per-class launch timing.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace kp {

// Exceptions mapped to the C-ABI status codes (include/kronprec_b200.h).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NoRoot : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define KP_CUDA(expr)                                                        \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess)                                                   \
      throw ::kp::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// KC_PRECOND_AUX: gemm_f16x's row sign hashes and zero-sign fix-up launches
enum KernelClass {
  KC_OPERATOR = 0,
  KC_PRECOND = 1,
  KC_VECTOR = 2,
  KC_SPECTRAL = 3,
  KC_PRECOND_AUX = 4,
  KC_COUNT = 5
};

struct Ctx {
  int device = -1;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  bool profile = false;
  long long launches = 0;
  // timing: event pairs recorded around launches, per kernel class
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[KC_COUNT];
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  double total_ms[KC_COUNT] = {};
  long long count[KC_COUNT] = {};
  cudaEvent_t events[16] = {};
  // dynamic shared-memory limit already set per kernel on this thread's device
  std::unordered_map<const void*, size_t> smem_attr;
};

Ctx& ctx();            // lazily initialised on first use (device 0)
void ensure_init();
void init_pool(int device);
// Raise a kernel's dynamic shared-memory limit to `bytes` on the calling
// thread's device (cached per thread: no shared mutable state, and a thread
// per device sets it for every device it uses).
void set_smem_limit(const void* kernel, size_t bytes);  // keep freed pool blocks cached (release threshold = max)
void check_launch(const char* what);

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx().stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KP_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Programmatic dependent launch: every hot-path kernel starts with
// pdl_wait() (griddepcontrol.wait) before touching memory, and is launched
// with launch_pdl(), so consecutive kernels on the stream (and in the
// captured iteration graphs) overlap one kernel's launch with the previous
// one's tail while keeping full stream-order visibility of its results.
// (An explicit early griddepcontrol.launch_dependents after the wait was
// measured: C1 12.1k vs 12.8k it/s, C2 +1 %, C5 -0.5 % — not adopted.)
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
}

// RAII launch bracket: counts the launch and, when profiling, records events.
struct LaunchScope {
  int cls;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  explicit LaunchScope(int c);
  ~LaunchScope() noexcept(false);
};

// Device buffer with RAII.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;  // stream the block was allocated on (and is freed on)
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    free();
    // Stream-ordered pool allocation (the pool keeps freed blocks; see
    // init_pool), so per-call scratch costs no device synchronisation.
    if (count) {
      s = ctx().stream;
      KP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    }
    n = count;
  }
  void free() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    free();
    p = o.p, n = o.n, s = o.s;
    o.p = nullptr, o.n = 0;
    return *this;
  }
  void upload(const T* h, size_t count) {
    KP_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, ctx().stream));
  }
  void download(T* h, size_t count) const {
    KP_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, ctx().stream));
  }
};

inline unsigned cdiv(long a, long b) { return unsigned((a + b - 1) / b); }

}  // namespace kp
