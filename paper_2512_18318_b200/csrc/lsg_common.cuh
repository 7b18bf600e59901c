// lsg_common.cuh -- shared host/device plumbing for liblsg.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "lsg.h"

namespace lsg {

// Exceptions carry the status the C ABI returns; they never cross the ABI.
struct Error : std::runtime_error {
  lsg_status code;
  Error(lsg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);

[[noreturn]] inline void fail(lsg_status code, const std::string& msg) { throw Error(code, msg); }
inline void invalid(const std::string& m) { fail(LSG_EINVAL, m); }
inline void logic(const std::string& m) { fail(LSG_ELOGIC, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(LSG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                        std::to_string(line) + ")");
}
#define LSG_CUDA(x) ::lsg::cuda_check((x), #x, __FILE__, __LINE__)
#define LSG_LAUNCHED(ctx) \
  do {                    \
    (ctx)->note_launch(); \
    LSG_CUDA(cudaGetLastError()); \
  } while (0)

struct Ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  std::atomic<int64_t> launches{0};
  void note_launch() { launches.fetch_add(1, std::memory_order_relaxed); }
  void sync() { LSG_CUDA(cudaStreamSynchronize(stream)); }
  int smem_optin = 0;  // sharedMemPerBlockOptin
  // device scratch for calls that stage a per-call table and synchronise
  // before returning (align.cu, face.cu): allocated at context creation
  // (kScratchInit covers ~25k segments per call); a larger call grows it once
  // (synchronising) -- the one exception to "compute calls do not allocate",
  // documented in lsg.h
  static constexpr size_t kScratchInit = 1 << 20;
  std::mutex scratch_mu;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* scratch_get(size_t bytes) {
    if (bytes > scratch_bytes) {
      if (scratch) {
        sync();
        LSG_CUDA(cudaFree(scratch));
        scratch = nullptr;
        scratch_bytes = 0;
      }
      LSG_CUDA(cudaMalloc(&scratch, bytes));
      scratch_bytes = bytes;
    }
    return scratch;
  }
};

// The context's scratch, held (mutex) until the call has synchronised its
// stream and returns.
struct ScratchLease {
  std::unique_lock<std::mutex> lk;
  void* p = nullptr;
  ScratchLease(Ctx* c, size_t bytes) : lk(c->scratch_mu) { p = c->scratch_get(bytes < 16 ? 16 : bytes); }
};

// Makes the context's device current for the calling host thread.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const Ctx* c) {
    cudaGetDevice(&prev);
    if (prev != c->device) LSG_CUDA(cudaSetDevice(c->device));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Device buffer owned by a handle (no allocation on compute paths).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) LSG_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

template <class T>
struct PinnedBuf {
  T* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) LSG_CUDA(cudaMallocHost(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

bool is_device_ptr(const void* p);

// Runs f, translating exceptions into the ABI status + thread-local message.
template <class F>
lsg_status guard(const char* name, F&& f) {
  // every C-ABI call is an NVTX range (name = the entry point), so an Nsight
  // timeline attributes host gaps and launches to the reference-facing calls
  struct Range {
    explicit Range(const char* n) { nvtxRangePushA(n); }
    ~Range() { nvtxRangePop(); }
  } range(name);
  try {
    f();
    return LSG_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("out of host memory");
    return LSG_ERUNTIME;
  } catch (const std::exception& e) {
    set_error(e.what());
    return LSG_ERUNTIME;
  }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lsg

struct lsg_ctx_s : lsg::Ctx {};
