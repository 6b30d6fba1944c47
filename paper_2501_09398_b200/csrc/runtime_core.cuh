// runtime_core.cuh — includes, error plumbing, Launch / Slab records, run-time loaded NCCL and CUPTI.
// Part of runtime.cu (one translation unit; included in order, not compiled alone).
#pragma once

#include <cuda_runtime.h>
#include <cupti_activity.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys, no-ops without a tool

#include <mutex>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/iterbatch_b200.h"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define IB_CUDA(call)                                                                           \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? IB_ENOMEM : IB_ECUDA,                       \
                  std::string(#call) + ": " + cudaGetErrorName(e_) + ": " + cudaGetErrorString(e_)); \
    }                                                                                           \
  } while (0)

#define IB_TRY(expr)       \
  do {                     \
    int rc_ = (expr);      \
    if (rc_ != IB_OK) return rc_; \
  } while (0)

// NVTX range for the lifetime of a scope (the build / launch phases the paper times).
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// Restores the caller's current device (torch and other libraries rely on it).
struct DeviceGuard {
  int saved = -1;
  DeviceGuard() { cudaGetDevice(&saved); }
  ~DeviceGuard() {
    if (saved >= 0) cudaSetDevice(saved);
  }
};

// A kernel launch with its argument values stored by value (graph nodes copy them at add time).
struct Launch {
  const void *func = nullptr;
  dim3 grid, block;
  size_t smem = 0;  // dynamic shared memory bytes
  int slab = 0;
  int step = 0;  // half-step index within an iteration (FDTD: 0 = H, 1 = E) for cross-slab ordering
  int nargs = 0;
  static constexpr int kMaxArgs = 24;
  alignas(16) unsigned char slot[kMaxArgs][16];
  void *ptr[kMaxArgs];
  void **args() {
    for (int i = 0; i < nargs; ++i) ptr[i] = slot[i];
    return ptr;
  }
};

template <typename A>
void put_args(Launch &L, A a) {
  static_assert(sizeof(A) <= 16, "kernel argument too large");
  std::memcpy(L.slot[L.nargs++], &a, sizeof(A));
}
template <typename A, typename... R>
void put_args(Launch &L, A a, R... rest) {
  put_args(L, a);
  put_args(L, rest...);
}
template <typename... Args>
Launch make_launch(const void *func, dim3 grid, dim3 block, int slab, Args... args) {
  static_assert(sizeof...(Args) <= Launch::kMaxArgs, "too many kernel arguments for Launch");
  Launch L;
  L.func = func;
  L.grid = grid;
  L.block = block;
  L.slab = slab;
  put_args(L, args...);
  return L;
}

struct Slab {
  int device = 0;
  int row_lo = 0, row_hi = 0;  // global rows owned [lo, hi)
  bool has_top = false, has_bot = false;
  void *buf[2] = {nullptr, nullptr};  // (rows_local + 2) planes each: halo, owned..., halo
  void *power = nullptr;              // rows_local planes
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // "iteration t done" double buffer for neighbours
  cudaEvent_t join = nullptr;              // fork/join of the slab streams
  int64_t fs = 0;  // FDTD slabs: lattice field stride (elements) of buf[0]
  int rows() const { return row_hi - row_lo; }
};

const char *env_str(const char *name) {
  const char *v = std::getenv(name);
  return (v && *v) ? v : nullptr;
}

int64_t env_int(const char *name, int64_t dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::strtoll(v, nullptr, 10);
}

// ---- NCCL, loaded at run time (no link dependency; the process may already hold torch's copy) --
struct NcclId { char internal[128]; };
struct Nccl {
  bool ok = false;
  std::string err;
  int (*GetUniqueId)(NcclId *) = nullptr;
  int (*CommInitRank)(void **, int, NcclId, int) = nullptr;
  int (*CommDestroy)(void *) = nullptr;
  int (*Send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*Recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
};
Nccl &nccl() {
  static Nccl n = [] {
    Nccl r;
    // The copy the process already holds (torch's), else IB_NCCL_LIB (the Python layer points it
    // at the wheel torch links against, so a later `import torch` finds a compatible NCCL), else
    // the loader's default. RTLD_LOCAL: never interpose NCCL symbols on other libraries.
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char *path = std::getenv("IB_NCCL_LIB");
    if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      r.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return r;
    }
    r.GetUniqueId = (int (*)(NcclId *))dlsym(h, "ncclGetUniqueId");
    r.CommInitRank = (int (*)(void **, int, NcclId, int))dlsym(h, "ncclCommInitRank");
    r.CommDestroy = (int (*)(void *))dlsym(h, "ncclCommDestroy");
    r.Send = (int (*)(const void *, size_t, int, int, void *, cudaStream_t))dlsym(h, "ncclSend");
    r.Recv = (int (*)(void *, size_t, int, int, void *, cudaStream_t))dlsym(h, "ncclRecv");
    r.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
    r.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
    r.GetErrorString = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
    r.ok = r.GetUniqueId && r.CommInitRank && r.CommDestroy && r.Send && r.Recv && r.GroupStart &&
           r.GroupEnd && r.GetErrorString;
    if (!r.ok) r.err = "libnccl.so.2 lacks a required symbol";
    return r;
  }();
  return n;
}
constexpr int kNcclInt8 = 0;  // ncclInt8: halo planes move as raw bytes

// ---- CUPTI activity tracing, loaded at run time (what nsys uses; no in-kernel instrumentation) -
struct Cupti {
  bool ok = false;
  std::string err;
  CUptiResult (*RegisterCallbacks)(CUpti_BuffersCallbackRequestFunc, CUpti_BuffersCallbackCompleteFunc) = nullptr;
  CUptiResult (*Enable)(CUpti_ActivityKind) = nullptr;
  CUptiResult (*Disable)(CUpti_ActivityKind) = nullptr;
  CUptiResult (*FlushAll)(uint32_t) = nullptr;
  CUptiResult (*GetNextRecord)(uint8_t *, size_t, CUpti_Activity **) = nullptr;
  CUptiResult (*GetTimestamp)(uint64_t *) = nullptr;
  std::mutex mu;
  std::vector<int64_t> kernels;  // (start, end) pairs of this library's solver kernels
};
Cupti &cupti() {
  static Cupti *c = [] {
    Cupti *r = new Cupti();
    void *h = dlopen("libcupti.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcupti.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r->err = std::string("dlopen(libcupti) failed: ") + dlerror();
      return r;
    }
    r->RegisterCallbacks = (decltype(r->RegisterCallbacks))dlsym(h, "cuptiActivityRegisterCallbacks");
    r->Enable = (decltype(r->Enable))dlsym(h, "cuptiActivityEnable");
    r->Disable = (decltype(r->Disable))dlsym(h, "cuptiActivityDisable");
    r->FlushAll = (decltype(r->FlushAll))dlsym(h, "cuptiActivityFlushAll");
    r->GetNextRecord = (decltype(r->GetNextRecord))dlsym(h, "cuptiActivityGetNextRecord");
    r->GetTimestamp = (decltype(r->GetTimestamp))dlsym(h, "cuptiGetTimestamp");
    r->ok = r->RegisterCallbacks && r->Enable && r->Disable && r->FlushAll && r->GetNextRecord &&
            r->GetTimestamp;
    if (!r->ok) r->err = "libcupti lacks a required symbol";
    return r;
  }();
  return *c;
}
void CUPTIAPI cupti_buffer_requested(uint8_t **buffer, size_t *size, size_t *max_records) {
  *size = 8u << 20;
  *buffer = (uint8_t *)aligned_alloc(8, *size);
  *max_records = 0;
}
void CUPTIAPI cupti_buffer_completed(CUcontext, uint32_t, uint8_t *buffer, size_t, size_t valid) {
  Cupti &c = cupti();
  CUpti_Activity *rec = nullptr;
  std::lock_guard<std::mutex> lock(c.mu);
  while (c.GetNextRecord(buffer, valid, &rec) == CUPTI_SUCCESS) {
    if (rec->kind != CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL && rec->kind != CUPTI_ACTIVITY_KIND_KERNEL) continue;
    const CUpti_ActivityKernel9 *k = (const CUpti_ActivityKernel9 *)rec;
    const char *n = k->name ? k->name : "";
    // the solver kernels live in namespace ib (mangled _ZN2ib...); utilities are not traced
    if (std::strncmp(n, "_ZN2ib", 6) != 0 || std::strstr(n, "k_flush")) continue;
    c.kernels.push_back((int64_t)k->start);
    c.kernels.push_back((int64_t)k->end);
  }
  free(buffer);
}

}  // namespace
