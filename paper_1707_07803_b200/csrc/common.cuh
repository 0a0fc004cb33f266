// Shared plumbing for the sm_100a kernels: error handling, stream-ordered
// device buffers, small device helpers.  All matrices are FP64 and
// column-major ("F order", first index fastest), the layout of the
// reference's cores (mpo.py:17-23) and of every unfolding the sweeps use.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mpob {

// A precondition failure: maps to the reference's ValueError.
struct ValueError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// A CUDA failure: maps to RuntimeError.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Device allocation failure: maps to MemoryError (numpy's on the CPU path).
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed at %s:%d: %s", what, file, line, cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) throw OutOfMemory(buf);
  throw CudaError(buf);
}
#define CK(x) ::mpob::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::mpob::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Stream-ordered device buffer (cudaMallocAsync from the device's default
// pool, whose release threshold the context raises so freed blocks are
// recycled instead of returned to the driver between sweeps).
template <typename T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DBuf() { reset(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { reset(); p_ = o.p_; n_ = o.n_; s_ = o.s_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void alloc(size_t n, cudaStream_t s) {
    reset();
    s_ = s;
    n_ = n;
    if (n) {
      void* p = nullptr;
      CK(cudaMallocAsync(&p, n * sizeof(T), s));
      p_ = static_cast<T*>(p);
    }
  }
  void reset() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  cudaStream_t stream() const { return s_; }
  void set_stream(cudaStream_t s) { s_ = s; }   // the stream the free is ordered on

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int current_device() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return dev;
}

// Function attributes (dynamic shared-memory opt-ins) are per device: run a
// setup once for each device the calling thread targets (thread-safe).
constexpr int kMaxDevices = 64;
template <typename F>
inline void once_per_device(std::once_flag (&flags)[kMaxDevices], F&& fn) {
  std::call_once(flags[current_device() & (kMaxDevices - 1)], std::forward<F>(fn));
}

// Count of our own kernel launches (reported by bench.py as gpu_launches).
// MPO_CHECK builds (tools/build_variant.sh check <file> -DMPO_CHECK): device
// bounds checks on the indexing the deterministic-output argument relies on
// (compute-sanitizer is not available on the GPU pool); a violation traps.
#ifdef MPO_CHECK
#define MPO_DCHECK(cond)                                                            \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("MPO_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #cond, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define MPO_DCHECK(cond) do {} while (0)
#endif

extern unsigned long long g_launches;
inline void note_launch(int n = 1) { g_launches += (unsigned long long)n; }
// how each truncating R2L step was rounded (tests / diagnostics):
// 0 certificate (wide), 1 certificate (tall), 2 tail cut (wide), 3 tail cut
// (tall), 4 full SVD
extern unsigned long long g_round_paths[5];

}  // namespace mpob
