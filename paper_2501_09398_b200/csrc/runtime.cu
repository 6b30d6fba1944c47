// runtime.cu — C++ launch layer behind include/iterbatch_b200.h.
//
// Replaces the bodies of the reference drivers (pkg/src/iterbatch/workloads.py):
//   run_loop     workloads.py:442-450  -> ib_run_stream : N (2N for FDTD) launches from a C++ loop,
//                                                          i.e. Listing 1
//   run_batched  workloads.py:453-471  -> ib_graph_build + ib_graph_run : K iterations unrolled
//                                          into one CUDA graph, instantiated and uploaded once,
//                                          replayed I = N/K times (Listing 3)
//   time_workload workloads.py:479-505 -> ib_times: T_C (create/instantiate/upload) separated
//                                          from T_E (first launch .. sync)
//   _fill_slabs  workloads.py:60-69    -> axis-0 slab decomposition rows*g//P across devices,
//                                          halo planes pushed by the stencil kernel itself
// The state lives in HBM for the whole run; the boundary is crossed by ib_upload/ib_download.
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

struct ib_ctx {
  int solver = 0, dtype = 0, esize = 8;
  int64_t dims[3] = {1, 1, 1};
  int ndims = 1;
  double scalars[3] = {0, 0, 0};
  std::vector<Slab> slabs;
  void *field[6] = {};      // vector / fdtd device fields (single slab)
  void *field2[6] = {};     // fused fdtd: the second buffer of the ping-pong field pairs
  // fused fdtd: the padded lattice (two parities), fields at lat[p] + f*lat_fs elements, rows of
  // lat_pitch elements (nz+1 rounded up to 16 bytes); field/field2 point into it
  void *lat[2] = {nullptr, nullptr};
  int64_t lat_pitch = 0, lat_fs = 0;
  int64_t fshape[6][3] = {};
  int fndim[6] = {};
  int nfields = 0;
  int cur = 0;              // hotspot ping-pong parity: buf[cur] holds the current temperature
  int num_sms = 148;        // of slab 0's device
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaStream_t cap_stream = nullptr;  // used only for stream capture of single-slab graphs
  // graph state
  int64_t K = 0;
  int gflags = 0, gmode = 0;
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // indexed by start parity
  cudaGraphConditionalHandle cond[2] = {};
  int *d_counter = nullptr;  // WHILE-mode remaining-batch counter
  void *flush = nullptr;
  size_t flush_bytes = 0;
  // multi-process slab (ib_create_dist)
  int rank = 0, nranks = 1;
  void *comm = nullptr;  // ncclComm_t (NCCL exchange)
  // peer exchange (ib_ipc_attach): the stencil kernel stores its boundary planes straight into the
  // neighbour ranks' halo planes through CUDA IPC mappings; cross-process ordering by device-side
  // iteration counters (k_dist_wait / k_dist_signal, one pair per iteration inside the graph)
  unsigned long long *sync = nullptr;        // [0] my completed iterations, [1] up's, [2] down's
  void *peer_buf_up[2] = {nullptr, nullptr}, *peer_buf_dn[2] = {nullptr, nullptr};
  unsigned long long *peer_sync_up = nullptr, *peer_sync_dn = nullptr;
  int peer_rows_up = 0;  // the up neighbour's owned rows (locates its bottom halo plane)
  int peer_rows_dn = 0;  // the down neighbour's (FDTD: its lattice field stride)
  bool peer = false;
  bool dist() const { return nranks > 1; }
  int64_t lattice_pitch() const { return lat_pitch; }
  // tracing (CUPTI activity records; host events on the CUPTI timebase)
  bool tracing = false;
  int64_t trace_cap = 0;
  struct HostEv { int64_t t, kind, batch, kernel; };
  std::vector<HostEv> host_ev;
  void ev(int kind, int64_t batch = -1, int64_t kernel = -1);

  cudaStream_t stream() const { return slabs[0].stream; }
  bool ping_pong() const {
    return solver == IB_SOLVER_HOTSPOT2D || solver == IB_SOLVER_HOTSPOT3D ||
           solver == IB_SOLVER_FDTD_FUSED;
  }
  bool fdtd() const { return solver == IB_SOLVER_FDTD || solver == IB_SOLVER_FDTD_FUSED; }
  bool hotspot() const { return solver == IB_SOLVER_HOTSPOT2D || solver == IB_SOLVER_HOTSPOT3D; }
  void *fieldp(int f, int parity) const {  // device field f holding parity `parity`
    return (solver == IB_SOLVER_FDTD_FUSED && parity) ? field2[f] : field[f];
  }
  int64_t plane() const {  // elements per axis-0 plane (hotspot)
    return solver == IB_SOLVER_HOTSPOT3D ? dims[1] * dims[2] : dims[1];
  }
};

void ib_ctx::ev(int kind, int64_t batch, int64_t kernel) {
  if (!tracing) return;
  uint64_t t = 0;
  cupti().GetTimestamp(&t);
  host_ev.push_back({(int64_t)t, kind, batch, kernel});
}

namespace {

int64_t numel(const int64_t *s, int n) {
  int64_t r = 1;
  for (int i = 0; i < n; ++i) r *= s[i];
  return r;
}

// ---- per-iteration launch lists ----------------------------------------------------------------
int hotspot_rows_per_chunk(const ib_ctx *c, int rows) {
  int64_t rpc = env_int("IB_HOTSPOT_RPC", 0);
  if (rpc <= 0) {
    const int64_t want_threads = 148LL * 2048 * 2;
    int64_t chunks = (want_threads + c->plane() - 1) / c->plane();
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, rows));
    rpc = (rows + chunks - 1) / chunks;
    rpc = std::min<int64_t>(rpc, 64);
  }
  return (int)std::max<int64_t>(1, std::min<int64_t>(rpc, rows));
}

// Kernel variant for a hotspot grid. IB_HOTSPOT_KERNEL=scalar|vec|tma forces one (if legal).
//   vec    one 16-byte group per thread, every load independent: best for L2-resident grids
//   tma    cp.async.bulk plane-march pipeline: best once the state no longer fits in L2
//   scalar marching fallback for shapes the vector paths cannot take (M or L not a multiple of V)
enum class HotKernel { Scalar, Vec, Tma };

template <typename T>
int tma_groups(const ib_ctx *c) {  // G such that TM = G*V*256 holds whole y-rows; 0 = not possible
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int64_t L = d3 ? c->dims[2] : 1;
  for (int G : {2, 1, 4}) {
    const int64_t TM = (int64_t)G * V * 256;
    if (!d3 || (TM % L == 0 && L <= 1024)) return G;
  }
  return 0;
}

template <typename T>
HotKernel hotspot_variant(const ib_ctx *c, int rows) {
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int64_t M = c->plane();
  const int64_t L = d3 ? c->dims[2] : 1;
  const bool vec_ok = (M % V == 0) && (!d3 || L % V == 0) && rows <= 65535 &&
                      (int64_t)(rows + 2) * M < (1LL << 31);  // 32-bit offsets
  const bool tma_ok = vec_ok && tma_groups<T>(c) > 0 && rows >= 2;
  const char *force = env_str("IB_HOTSPOT_KERNEL");
  if (force) {
    if (!std::strcmp(force, "tma") && tma_ok) return HotKernel::Tma;
    if (!std::strcmp(force, "vec") && vec_ok) return HotKernel::Vec;
    if (!std::strcmp(force, "scalar")) return HotKernel::Scalar;
  }
  const int64_t state_bytes = 3 * M * c->dims[0] * (int64_t)sizeof(T);
  if (tma_ok && state_bytes >= (96LL << 20)) return HotKernel::Tma;
  if (vec_ok) return HotKernel::Vec;
  return HotKernel::Scalar;
}

template <typename T, bool D3>
const void *tma_fn(int G) {
  switch (G) {
    case 1: return (const void *)ib::k_hotspot_tma<T, D3, 1>;
    case 4: return (const void *)ib::k_hotspot_tma<T, D3, 4>;
    default: return (const void *)ib::k_hotspot_tma<T, D3, 2>;
  }
}

template <typename T, bool D3, int SH>
const void *vec_fn_r(int R) {
  return R >= 4 ? (const void *)ib::k_hotspot_vec<T, D3, 4, SH>
                : R == 2 ? (const void *)ib::k_hotspot_vec<T, D3, 2, SH> : (const void *)ib::k_hotspot_vec<T, D3, 1, SH>;
}
template <typename T>
const void *vec_fn(bool d3, int R, int sh) {
  if (d3) return sh == 2 ? vec_fn_r<T, true, 2>(R) : sh == 1 ? vec_fn_r<T, true, 1>(R) : vec_fn_r<T, true, 0>(R);
  return sh ? vec_fn_r<T, false, 1>(R) : vec_fn_r<T, false, 0>(R);
}

template <typename T>
void hotspot_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  constexpr int V = 16 / sizeof(T);
  const bool d3 = c->solver == IB_SOLVER_HOTSPOT3D;
  const int C = (int)c->dims[1];
  const int L = d3 ? (int)c->dims[2] : 1;
  const int64_t plane = c->plane();
  const T k = (T)c->scalars[0];
  const T loss = (T)(2.0 * (d3 ? 3 : 2));
  const int P = (int)c->slabs.size();
  const bool multi = P > 1 || c->dist();  // slab buffers carry halo planes
  for (int g = 0; g < P; ++g) {
    Slab &s = c->slabs[g];
    const int rows = s.rows();
    const int64_t off = multi ? plane : 0;  // first owned plane
    const T *src = (const T *)s.buf[parity] + off;
    T *dst = (T *)s.buf[parity ^ 1] + off;
    T *up = nullptr, *dn = nullptr;
    if (P > 1 && g > 0) {  // my first owned row -> upper neighbour's bottom halo
      Slab &n = c->slabs[g - 1];
      up = (T *)n.buf[parity ^ 1] + (int64_t)(n.rows() + 1) * plane;
    }
    if (P > 1 && g + 1 < P) {  // my last owned row -> lower neighbour's top halo
      Slab &n = c->slabs[g + 1];
      dn = (T *)n.buf[parity ^ 1];
    }
    if (c->dist() && c->peer) {  // the neighbour ranks' halo planes, through IPC mappings
      if (s.has_top) up = (T *)c->peer_buf_up[parity ^ 1] + (int64_t)(c->peer_rows_up + 1) * plane;
      if (s.has_bot) dn = (T *)c->peer_buf_dn[parity ^ 1];
    }
    const int top = (int)s.has_top, bot = (int)s.has_bot;
    dim3 block(256);
    switch (hotspot_variant<T>(c, rows)) {
      case HotKernel::Vec: {
        // rows per thread (R+2 row loads per R outputs): with the neighbour loads (no shuffles)
        // R = 1 — the most threads, the shortest per-thread chain — unless the grid would exceed
        // four waves (measured: Hotspot3D 512x512x8 R=1 4.41, R=2 4.57, R=4 4.67 us/iter;
        // Hotspot2D 1024^2 R=1 2.56, R=2 3.12); with shuffles R = 2 (below). IB_HOTSPOT_VEC_ROWS
        // overrides.
        int64_t R = env_int("IB_HOTSPOT_VEC_ROWS", 0);
        const int64_t threads_per_row = plane / V;
        // CTA shape: bx threads along a plane row (up to 256), by row-blocks, bx*by = IB_HOTSPOT_BLOCK.
        // 256 measured best in-graph (Hotspot3D 512^2x8: 4.45 / 4.79 / 6.20 us at 256 / 512 / 1024;
        // Hotspot2D 2.60 / 2.65 / 2.68) although an EMPTY kernel's launch floor falls with fewer,
        // bigger CTAs (tools/microbench_floor.cu): real CTAs retire at their slowest warp.
        // With shuffles and R = 2 (below), 2-D measured best at 512 threads (256 x 2 row-blocks:
        // 2.33 vs 2.43 us/iter at 256), 3-D at 256 (4.21; 512: 4.61).
        int64_t bs = env_int("IB_HOTSPOT_BLOCK", d3 ? 256 : 512);
        bs = std::max<int64_t>(32, std::min<int64_t>(1024, bs / 32 * 32));
        const int64_t bx = std::min<int64_t>(std::min<int64_t>(256, bs), (threads_per_row + 31) / 32 * 32);
        const int64_t by = std::max<int64_t>(1, bs / bx);
        const int64_t xblocks = (threads_per_row + bx - 1) / bx;
        if (R <= 0) {
          const int64_t slots = 1536LL * c->num_sms;  // resident threads at <= 40 registers
          R = 1;
          while (R < 4 && xblocks * bx * ((rows + R - 1) / R) > 4 * slots) R *= 2;
        }
        R = R >= 4 ? 4 : (R >= 2 ? 2 : 1);
        // warp shuffles for the in-row (2-D) / z (3-D) neighbours when every warp covers 32 groups
        // of one row and whole y-rows: 1 = those, 2 = also the y rows. IB_HOTSPOT_SHUFFLE overrides.
        const int64_t gl = d3 ? L / V : 1;
        // Measured in-graph with PDL (us/iter, two runs): Hotspot3D 512^2x8 R=1 4.47, R=1+sh1 4.36,
        // R=2+sh1 4.22-4.25, sh2 (y rows by 8 shuffles) 4.60-4.77; Hotspot2D 1024^2 R=1 2.61,
        // R=1+sh1 2.49, R=2+sh1 2.45. So z / row shuffles, and 2 rows per thread with them.
        int64_t sh = env_int("IB_HOTSPOT_SHUFFLE", 1);
        if (!(threads_per_row % 32 == 0 && bx % 32 == 0 && 32 % gl == 0)) sh = 0;
        if (sh && env_int("IB_HOTSPOT_VEC_ROWS", 0) <= 0 && rows >= 2 && R < 2) R = 2;
        const void *fn = vec_fn<T>(d3, (int)R, (int)std::min<int64_t>(sh, 2));
        dim3 grid((unsigned)xblocks, (unsigned)((rows + R * by - 1) / (R * by)));
        out.push_back(make_launch(fn, grid, dim3((unsigned)bx, (unsigned)by), g, src, dst, (const T *)s.power,
                                  rows, C, L, k, loss,
                                  top, bot, up, dn));
        break;
      }
      case HotKernel::Tma: {
        const int G = tma_groups<T>(c);
        const int TM = G * V * 256;
        const int H = d3 ? L : V;
        const int ns = (int)std::max<int64_t>(3, std::min<int64_t>(8, env_int("IB_TMA_STAGES", 4)));
        const size_t smem = (size_t)ns * (TM + 2 * H + TM) * sizeof(T) + (size_t)ns * 8;
        const void *fn = d3 ? tma_fn<T, true>(G) : tma_fn<T, false>(G);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t tiles = (plane + TM - 1) / TM;
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
        const int64_t slots = (int64_t)std::max(1, per_sm) * c->num_sms;
        int64_t rpc = env_int("IB_HOTSPOT_RPC", 0);
        if (rpc <= 0) rpc = std::max<int64_t>(16, std::min<int64_t>(128, (int64_t)rows * tiles / (12 * slots)));
        rpc = std::min<int64_t>(rpc, rows);
        dim3 grid((unsigned)tiles, (unsigned)((rows + rpc - 1) / rpc));
        Launch Lz = make_launch(fn, grid, block, g, src, dst, (const T *)s.power, rows, C, L, (int)rpc, ns,
                                k, loss, top, bot, up, dn);
        Lz.smem = smem;
        out.push_back(Lz);
        break;
      }
      default: {
        const void *fn = d3 ? (const void *)ib::k_hotspot<T, true> : (const void *)ib::k_hotspot<T, false>;
        const int rpc = hotspot_rows_per_chunk(c, rows);
        dim3 grid((unsigned)((plane + 255) / 256), (unsigned)((rows + rpc - 1) / rpc));
        out.push_back(make_launch(fn, grid, block, g, src, dst, (const T *)s.power, rows, C, L, rpc, k,
                                  loss, top, bot, up, dn));
      }
    }
  }
}

// Fused leapfrog (k_fdtd_lf): TJ y-rows per tile, NS-stage bulk-copy ring. The largest TJ (and
// then NS) whose ring lets two CTAs share an SM; the grid is one wave of resident CTAs and the
// (tile, plane) units are split evenly over it. IB_FDTD_TJ / IB_FDTD_STAGES override.
struct LfConfig {
  int tj = 0, ns = 0;
  size_t smem = 0;
};
inline size_t lf_smem(int tj, int ns, int64_t P, int es) {
  return (size_t)ns * (size_t)(3 * (tj + 2) + 3 * (tj + 1)) * (size_t)P * es + (size_t)ns * 8;
}
inline int lf_threads(const ib_ctx *c, int tj) {  // one thread per (row, 16-byte group)
  const int64_t groups = c->lat_pitch / (16 / c->esize);
  return (int)(((tj + 1) * groups + 31) / 32 * 32);
}
inline LfConfig lf_config(const ib_ctx *c) {
  // The kernel is bound by the bytes each SM keeps in flight, CTAs/SM x (NS-1) x stage bytes.
  // Measured at 256^3 binary32 (us/iter): TJ=4/NS=6/1 per SM 130.7, TJ=4/NS=5 137.3,
  // TJ=3/NS=4/2 per SM 138.5, TJ=3/NS=3/2 per SM 196, TJ=4/NS=3/2 per SM 171. So: 4-row tiles
  // with the deepest ring one CTA per SM holds (<= 6 stages), then 2 per SM, then smaller tiles.
  const int64_t P = c->lat_pitch;
  const int es = c->esize;
  const size_t cap = 227 * 1024, half = 113 * 1024;
  LfConfig cfg;
  const int64_t ftj = env_int("IB_FDTD_TJ", 0), fns = env_int("IB_FDTD_STAGES", 0);
  const struct { int tj; bool two; } order[] = {{4, false}, {3, true}, {4, true}, {2, true},
                                                 {3, false}, {2, false}, {1, true}, {1, false}};
  for (auto o : order) {
    if (ftj > 0 && o.tj != ftj) continue;
    if (lf_threads(c, o.tj) > ib::kLfMaxThreads) continue;
    for (int ns = 3; ns <= 8; ++ns) {
      if (fns > 0 && ns != fns) continue;
      const size_t sm = lf_smem(o.tj, ns, P, es);
      if (sm <= (o.two ? half : cap) && (fns > 0 || ns <= 6)) cfg = {o.tj, ns, sm};
    }
    if (cfg.tj && (cfg.ns >= 4 || fns > 0 || ftj > 0)) break;
    if (cfg.tj && o.tj == 1) break;
    if (cfg.tj && cfg.ns < 4) cfg = LfConfig{};  // too shallow: try the next shape
  }
  if (!cfg.tj) {  // nothing deep enough: take any shape that fits
    for (auto o : order) {
      if (lf_threads(c, o.tj) > ib::kLfMaxThreads) continue;
      const size_t sm = lf_smem(o.tj, 3, P, es);
      if (sm <= cap) { cfg = {o.tj, 3, sm}; break; }
    }
  }
  return cfg;
}

template <typename T, bool U, int M>
const void *lf_fn_m(int tj) {
  switch (tj) {
    case 1: return (const void *)ib::k_fdtd_lf<T, U, 1, M>;
    case 2: return (const void *)ib::k_fdtd_lf<T, U, 2, M>;
    case 3: return (const void *)ib::k_fdtd_lf<T, U, 3, M>;
    default: return (const void *)ib::k_fdtd_lf<T, U, 4, M>;
  }
}
template <typename T>
const void *lf_fn(bool unit, int tj, int mode) {
  if (unit) return mode == ib::kLfH ? lf_fn_m<T, true, ib::kLfH>(tj)
                   : mode == ib::kLfE ? lf_fn_m<T, true, ib::kLfE>(tj) : lf_fn_m<T, true, ib::kLfFused>(tj);
  return mode == ib::kLfH ? lf_fn_m<T, false, ib::kLfH>(tj)
         : mode == ib::kLfE ? lf_fn_m<T, false, ib::kLfE>(tj) : lf_fn_m<T, false, ib::kLfFused>(tj);
}

// One k_fdtd_lf launch of `mode` from lattice buffer `from` to `to` (equal for the in-place
// half-steps).
template <typename T>
Launch lf_launch(ib_ctx *c, int mode, void *from, void *to, int x0, int npl, int64_t fs, void *halo_h = nullptr,
                 int64_t fs_h = 0, void *halo_e = nullptr, int64_t fs_e = 0, int slab = 0) {
  const int nx = (int)c->dims[0], ny = (int)c->dims[1], nz = (int)c->dims[2];
  const T d = (T)c->scalars[0], ch = (T)c->scalars[1], ce = (T)c->scalars[2];
  const bool unit = c->scalars[0] == 1.0;
  const LfConfig cfg = lf_config(c);
  const void *fn = lf_fn<T>(unit, cfg.tj, mode);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem);
  const int threads = lf_threads(c, cfg.tj);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, cfg.smem);
  // Lockstep (tile, x-chunk) grid: as many x-chunks as the resident slots hold whole columns of
  // TJ-row tiles (256^3, TJ=4, 148 slots: 65 tiles x 2 chunks). Filling the spare slots with
  // shorter tiles (74 tiles of 3-4 rows x 2) measured slower (137 vs 131 us): more halo rows.
  // IB_FDTD_TILES (uneven rows, h <= TJ), IB_FDTD_CHUNKS, IB_FDTD_CTAS (even split) override.
  const int64_t slots = (int64_t)std::max(1, per_sm) * c->num_sms;
  const int64_t min_tiles = (ny + 1 + cfg.tj - 1) / cfg.tj;
  int64_t tiles = min_tiles;
  if (env_int("IB_FDTD_TILES", 0) >= min_tiles) tiles = std::min<int64_t>(ny + 1, env_int("IB_FDTD_TILES", 0));
  int64_t chunks = env_int("IB_FDTD_CHUNKS", 0);
  if (chunks <= 0) chunks = std::max<int64_t>(1, slots / tiles);
  chunks = std::min<int64_t>(chunks, npl);  // every chunk non-empty
  int64_t ctas = env_int("IB_FDTD_CTAS", 0);
  if (ctas <= 0) {
    ctas = tiles * chunks;  // one CTA per (tile, chunk): the kernel maps blockIdx.x to both
  } else {
    chunks = 0;  // even split of the tile-major unit list over `ctas` CTAs
    ctas = std::max<int64_t>(1, std::min(ctas, tiles * npl));
  }
  Launch L = make_launch(fn, dim3((unsigned)ctas), dim3((unsigned)threads), slab, (const T *)from, (T *)to, nx,
                         ny, nz, (int)c->lat_pitch, fs, x0, npl, (int)tiles, (int)chunks, cfg.ns, ch, ce, d,
                         (T *)halo_h, fs_h, (T *)halo_e, fs_e);
  L.smem = cfg.smem;
  L.step = mode == ib::kLfE ? 1 : 0;
  return L;
}

// FDTD, the reference's two half-steps (H then E, in place on the lattice): k_fdtd_lf in its H
// and E modes, or the lean one-thread-per-point kernels when the z rows are too long for the
// staged kernel's CTA (or IB_FDTD_KERNEL=lean).
template <typename T>
void fdtd_launches(ib_ctx *c, std::vector<Launch> &out) {
  const char *force = env_str("IB_FDTD_KERNEL");
  const bool lean = (force && !std::strcmp(force, "lean")) || lf_config(c).tj == 0;
  const int nx = (int)c->dims[0];
  const int P = (int)c->slabs.size();
  if (c->dist()) {  // one rank's slab; the neighbours' halo planes through IPC mappings
    const int64_t plane = (int64_t)(c->dims[1] + 1) * c->lattice_pitch();
    Slab &s = c->slabs[0];
    T *base = (T *)s.buf[0] + (int64_t)(1 - s.row_lo) * plane;
    void *hh = nullptr, *he = nullptr;
    int64_t fh = 0, fe = 0;
    if (c->peer && s.has_bot) {
      hh = c->peer_buf_dn[0];  // the down rank's top halo plane (its local 0)
      fh = (int64_t)(c->peer_rows_dn + 2) * plane;
    }
    if (c->peer && s.has_top) {
      he = (T *)c->peer_buf_up[0] + (int64_t)(c->peer_rows_up + 1) * plane;  // the up rank's bottom halo
      fe = (int64_t)(c->peer_rows_up + 2) * plane;
    }
    out.push_back(lf_launch<T>(c, ib::kLfH, base, base, s.row_lo, s.rows(), s.fs, hh, fh, nullptr, 0, 0));
    out.push_back(lf_launch<T>(c, ib::kLfE, base, base, s.row_lo, s.rows(), s.fs, nullptr, 0, he, fe, 0));
    return;
  }
  if (P > 1) {  // axis-0 slabs: every H launch, then every E launch, halo planes pushed in-kernel
    const int64_t plane = (int64_t)(c->dims[1] + 1) * c->lat_pitch;
    for (int step = 0; step < 2; ++step)
      for (int g = 0; g < P; ++g) {
        Slab &s = c->slabs[g];
        T *base = (T *)s.buf[0] + (int64_t)(1 - s.row_lo) * plane;  // global plane index -> buffer
        void *hh = nullptr, *he = nullptr;
        int64_t fh = 0, fe = 0;
        if (step == 0 && g + 1 < P) {
          hh = c->slabs[g + 1].buf[0];  // its top halo plane (local 0)
          fh = c->slabs[g + 1].fs;
        }
        if (step == 1 && g > 0) {
          Slab &n = c->slabs[g - 1];
          he = (T *)n.buf[0] + (int64_t)(n.rows() + 1) * plane;  // its bottom halo plane
          fe = n.fs;
        }
        out.push_back(lf_launch<T>(c, step == 0 ? ib::kLfH : ib::kLfE, base, base, s.row_lo, s.rows(), s.fs,
                                   hh, fh, he, fe, g));
      }
    return;
  }
  if (!lean) {
    out.push_back(lf_launch<T>(c, ib::kLfH, c->lat[0], c->lat[0], 0, nx + 1, c->lat_fs));
    out.push_back(lf_launch<T>(c, ib::kLfE, c->lat[0], c->lat[0], 0, nx + 1, c->lat_fs));
    return;
  }
  const int ny = (int)c->dims[1], nz = (int)c->dims[2];
  const T d = (T)c->scalars[0], ch = (T)c->scalars[1], ce = (T)c->scalars[2];
  const bool unit = c->scalars[0] == 1.0;
  dim3 b2(32, 8);
  dim3 grid((unsigned)((nz + 1 + 31) / 32), (unsigned)((ny + 1 + 7) / 8), (unsigned)(nx + 1));
  const void *fh = unit ? (const void *)ib::k_fdtd_h2<T, true> : (const void *)ib::k_fdtd_h2<T, false>;
  const void *fe = unit ? (const void *)ib::k_fdtd_e2<T, true> : (const void *)ib::k_fdtd_e2<T, false>;
  T *f = (T *)c->lat[0];
  out.push_back(make_launch(fh, grid, b2, 0, f, nx, ny, nz, (int)c->lat_pitch, c->lat_fs, ch, d));
  out.push_back(make_launch(fe, grid, b2, 0, f, nx, ny, nz, (int)c->lat_pitch, c->lat_fs, ce, d));
  out.back().step = 1;
}

// FDTD fused: one k_fdtd_lf launch per iteration, parity -> parity ^ 1.
template <typename T>
void fdtd_fused_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  out.push_back(lf_launch<T>(c, ib::kLfFused, c->lat[parity], c->lat[parity ^ 1], 0, (int)c->dims[0] + 1,
                             c->lat_fs));
}

void iteration_launches(ib_ctx *c, int parity, std::vector<Launch> &out) {
  out.clear();
  switch (c->solver) {
    case IB_SOLVER_VECTOR: {
      const int64_t n = c->dims[0];
      const double cc = c->scalars[0];
      // 128-thread CTAs measured best (1.21 / 1.23 / 1.24 / 1.40 us per iteration in a PDL graph at
      // 128 / 256 / 512 / 1024); IB_VECTOR_BLOCK overrides
      int64_t bs = env_int("IB_VECTOR_BLOCK", 128);
      bs = std::max<int64_t>(32, std::min<int64_t>(1024, bs / 32 * 32));
      if (c->dtype == IB_F32) {
        const int64_t threads = (n >> 2) + (n & 3);
        dim3 block((unsigned)bs), grid((unsigned)((threads + bs - 1) / bs));
        out.push_back(make_launch((const void *)ib::k_vector_f32, grid, block, 0,
                                  (float *)c->field[0], n, cc));
      } else {
        const int64_t threads = (n >> 1) + (n & 1);
        dim3 block((unsigned)bs), grid((unsigned)((threads + bs - 1) / bs));
        out.push_back(make_launch((const void *)ib::k_vector_f64, grid, block, 0,
                                  (double *)c->field[0], n, cc));
      }
      break;
    }
    case IB_SOLVER_HOTSPOT2D:
    case IB_SOLVER_HOTSPOT3D:
      if (c->dtype == IB_F32)
        hotspot_launches<float>(c, parity, out);
      else
        hotspot_launches<double>(c, parity, out);
      break;
    case IB_SOLVER_FDTD:
      if (c->dtype == IB_F32)
        fdtd_launches<float>(c, out);
      else
        fdtd_launches<double>(c, out);
      break;
    case IB_SOLVER_FDTD_FUSED:
      if (c->dtype == IB_F32)
        fdtd_fused_launches<float>(c, parity, out);
      else
        fdtd_fused_launches<double>(c, parity, out);
      break;
  }
}

int launch_one(Launch &L, cudaStream_t s, bool pdl) {
  if (!pdl) {
    IB_CUDA(cudaLaunchKernel(L.func, L.grid, L.block, L.args(), L.smem, s));
    return IB_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = L.grid;
  cfg.blockDim = L.block;
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  IB_CUDA(cudaLaunchKernelExC(&cfg, L.func, L.args()));
  return IB_OK;
}

// Halo exchange of a distributed slab after an iteration that wrote buf[parity]:
// send my first owned plane to rank-1 and receive its last into my top halo; the mirror with
// rank+1. One NCCL group, on the launch stream (captured into graphs like the kernels).
int nccl_exchange(ib_ctx *c, int parity, cudaStream_t st) {
  Nccl &n = nccl();
  Slab &s = c->slabs[0];
  const size_t pb = (size_t)(c->plane() * c->esize);
  char *b = (char *)s.buf[parity];
  auto chk = [&](int r, const char *what) {
    if (r != 0) return fail(IB_ECUDA, std::string(what) + ": " + n.GetErrorString(r));
    return IB_OK;
  };
  IB_TRY(chk(n.GroupStart(), "ncclGroupStart"));
  if (s.has_top) {
    IB_TRY(chk(n.Send(b + pb, pb, kNcclInt8, c->rank - 1, c->comm, st), "ncclSend(up)"));
    IB_TRY(chk(n.Recv(b, pb, kNcclInt8, c->rank - 1, c->comm, st), "ncclRecv(up)"));
  }
  if (s.has_bot) {
    IB_TRY(chk(n.Send(b + (size_t)s.rows() * pb, pb, kNcclInt8, c->rank + 1, c->comm, st), "ncclSend(down)"));
    IB_TRY(chk(n.Recv(b + (size_t)(s.rows() + 1) * pb, pb, kNcclInt8, c->rank + 1, c->comm, st), "ncclRecv(down)"));
  }
  IB_TRY(chk(n.GroupEnd(), "ncclGroupEnd"));
  return IB_OK;
}

int launch_dist_wait(ib_ctx *c, cudaStream_t st) {
  const int top = c->slabs[0].has_top, bot = c->slabs[0].has_bot;
  Launch L = make_launch((const void *)ib::k_dist_wait, dim3(1), dim3(1), 0, (const unsigned long long *)c->sync,
                         top, bot, (long long)env_int("IB_DIST_TIMEOUT_MS", 20000));
  return launch_one(L, st, false);
}
int launch_dist_signal(ib_ctx *c, cudaStream_t st) {
  Launch L = make_launch((const void *)ib::k_dist_signal, dim3(1), dim3(1), 0, c->sync, c->peer_sync_up,
                         c->peer_sync_dn);
  return launch_one(L, st, false);
}

// Enqueue `iters` iterations starting at `parity` onto the slab streams (also used under stream
// capture). Multi-slab: kernel(g,t) waits for kernel(g+-1,t-1) — RAW on the halo it reads and
// WAR on the halo it writes — through double-buffered events.
int enqueue_iterations(ib_ctx *c, int64_t iters, int parity, bool pdl, cudaStream_t single_stream,
                       int64_t *kernels, int64_t *launches) {
  std::vector<Launch> its[2];
  iteration_launches(c, 0, its[0]);
  if (c->ping_pong()) iteration_launches(c, 1, its[1]);
  const int P = (int)c->slabs.size();
  int steps = 1;  // half-steps per iteration (launches are listed step-major)
  for (const Launch &L : its[0]) steps = std::max(steps, L.step + 1);
  int par = parity;
  int64_t nk = 0;
  for (int64_t t = 0; t < iters; ++t) {
    std::vector<Launch> &v = c->ping_pong() ? its[par] : its[0];
    for (size_t q = 0; q < v.size(); ++q) {
      Launch &L = v[q];
      Slab &s = c->slabs[L.slab];
      cudaStream_t st = (P == 1 && single_stream) ? single_stream : s.stream;
      // phase = global half-step index; a slab's launch of phase f waits for its neighbours'
      // launches of phase f-1 (RAW on the halo it reads, WAR on the halo it writes)
      const int64_t f = t * steps + L.step;
      if (P > 1) {
        IB_CUDA(cudaSetDevice(s.device));
        if (f > 0) {
          if (L.slab > 0) IB_CUDA(cudaStreamWaitEvent(st, c->slabs[L.slab - 1].ev[(f - 1) & 1], 0));
          if (L.slab + 1 < P) IB_CUDA(cudaStreamWaitEvent(st, c->slabs[L.slab + 1].ev[(f - 1) & 1], 0));
        }
      }
      // PDL only chains kernels on the same stream; the very first launch has no predecessor.
      // Peer-exchange contexts never use it: the wait / signal kernels must not overlap the stencil.
      const bool use_pdl = pdl && P == 1 && (t > 0 || q > 0) && !c->peer;
      if (c->peer) IB_TRY(launch_dist_wait(c, st));  // neighbours done with the previous phase
      c->ev(single_stream ? IB_EV_NODE_ADDED : IB_EV_BASELINE_KERNEL_LAUNCHED, single_stream ? -1 : t,
            single_stream ? nk : (int64_t)q);
      IB_TRY(launch_one(L, st, use_pdl));
      if (P > 1) IB_CUDA(cudaEventRecord(s.ev[f & 1], st));
      if (c->peer) IB_TRY(launch_dist_signal(c, st));  // its halo planes went out with its stores
      ++nk;
    }
    if (c->dist()) {  // boundary planes of this iteration's output <-> neighbouring ranks
      cudaStream_t st = single_stream ? single_stream : c->slabs[0].stream;
      if (!c->peer) IB_TRY(nccl_exchange(c, par ^ 1, st));
    }
    if (c->ping_pong()) par ^= 1;
  }
  if (P > 1) IB_CUDA(cudaSetDevice(c->slabs[0].device));
  if (kernels) *kernels += nk;
  if (launches) *launches += nk;
  return IB_OK;
}

// Join all slab streams into slab 0's stream (or fork from it).
int join_into(ib_ctx *c, cudaStream_t root, bool fork) {
  if (c->slabs.size() == 1) return IB_OK;
  if (fork) {
    IB_CUDA(cudaSetDevice(c->slabs[0].device));
    IB_CUDA(cudaEventRecord(c->slabs[0].join, root));
  }
  for (size_t g = 1; g < c->slabs.size(); ++g) {
    Slab &s = c->slabs[g];
    IB_CUDA(cudaSetDevice(s.device));
    if (fork) {
      IB_CUDA(cudaStreamWaitEvent(s.stream, c->slabs[0].join, 0));
    } else {
      IB_CUDA(cudaEventRecord(s.join, s.stream));
      IB_CUDA(cudaSetDevice(c->slabs[0].device));
      IB_CUDA(cudaStreamWaitEvent(root, s.join, 0));
    }
  }
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  return IB_OK;
}

void free_graphs(ib_ctx *c) {
  for (int p = 0; p < 2; ++p) {
    if (c->exec[p]) cudaGraphExecDestroy(c->exec[p]);
    if (c->graph[p]) cudaGraphDestroy(c->graph[p]);
    c->exec[p] = nullptr;
    c->graph[p] = nullptr;
  }
  c->K = 0;
}

// Listing 3: cudaGraphCreate + a linear chain of cudaGraphAddKernelNode.
// With IB_FLAG_PDL the chain edges are programmatic (kernel t+1 may be resident before t ends).
int build_manual_chain(ib_ctx *c, cudaGraph_t graph, int64_t K, int parity, bool pdl,
                       cudaGraphNode_t *first, cudaGraphNode_t *last, int64_t *nodes) {
  std::vector<Launch> its[2];
  iteration_launches(c, 0, its[0]);
  if (c->ping_pong()) iteration_launches(c, 1, its[1]);
  cudaGraphNode_t prev = nullptr;
  int par = parity;
  for (int64_t t = 0; t < K; ++t) {
    std::vector<Launch> &v = c->ping_pong() ? its[par] : its[0];
    for (Launch &L : v) {
      cudaKernelNodeParams np = {};
      np.func = const_cast<void *>(L.func);
      np.gridDim = L.grid;
      np.blockDim = L.block;
      np.sharedMemBytes = (unsigned)L.smem;
      np.kernelParams = L.args();
      np.extra = nullptr;
      cudaGraphNode_t node;
      if (!prev) {
        IB_CUDA(cudaGraphAddKernelNode(&node, graph, nullptr, 0, &np));
        if (first) *first = node;
      } else if (!pdl) {
        IB_CUDA(cudaGraphAddKernelNode(&node, graph, &prev, 1, &np));
      } else {
        IB_CUDA(cudaGraphAddKernelNode(&node, graph, nullptr, 0, &np));
        cudaGraphEdgeData ed = {};
        ed.from_port = cudaGraphKernelNodePortProgrammatic;
        ed.type = cudaGraphDependencyTypeProgrammatic;
        IB_CUDA(cudaGraphAddDependencies_v2(graph, &prev, &node, &ed, 1));
      }
      prev = node;
      c->ev(IB_EV_NODE_ADDED, -1, *nodes);
      ++*nodes;
    }
    if (c->ping_pong()) par ^= 1;
  }
  if (last) *last = prev;
  return IB_OK;
}

}  // namespace

// Device-side tail of a WHILE body: decrement the remaining-batch counter and keep looping while
// batches remain (cudaGraphSetConditional, CUDA 12.4+ conditional nodes).
__global__ void k_while_tick(int *counter, cudaGraphConditionalHandle h) {
  int left = *counter - 1;
  *counter = left;
  cudaGraphSetConditional(h, left > 0 ? 1u : 0u);
}

namespace {

// Build one executable graph starting at `parity`.
int build_one(ib_ctx *c, int parity, ib_times *tm) {
  const bool pdl = (c->gflags & IB_FLAG_PDL) != 0;
  const bool wh = (c->gflags & IB_FLAG_WHILE) != 0;
  const int P = (int)c->slabs.size();
  int64_t nodes = 0;
  NvtxRange range("ib graph build (create + instantiate + upload)");
  c->ev(IB_EV_BUILD_STARTED);
  auto a = clk::now();
  cudaGraph_t g = nullptr;
  if (c->gmode == IB_BUILD_MANUAL && P == 1 && !c->dist()) {
    IB_CUDA(cudaGraphCreate(&g, 0));
    cudaGraph_t body = g;
    if (wh) {
      // graph = [WHILE node { K-chain ; tick }]; the counter is set before each launch.
      IB_CUDA(cudaGraphConditionalHandleCreate(&c->cond[parity], g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = c->cond[parity];
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t wnode;
      IB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &cp));
      body = cp.conditional.phGraph_out[0];
      ++nodes;
    }
    cudaGraphNode_t last = nullptr;
    IB_TRY(build_manual_chain(c, body, c->K, parity, pdl, nullptr, &last, &nodes));
    if (wh) {
      cudaKernelNodeParams np = {};
      int *cnt = c->d_counter;
      cudaGraphConditionalHandle h = c->cond[parity];
      void *args[2] = {&cnt, &h};
      np.func = (void *)k_while_tick;
      np.gridDim = dim3(1);
      np.blockDim = dim3(1);
      np.kernelParams = args;
      cudaGraphNode_t tick;
      IB_CUDA(cudaGraphAddKernelNode(&tick, body, &last, 1, &np));
      ++nodes;
    }
  } else {
    if (wh) return fail(IB_EINVAL, "IB_FLAG_WHILE requires IB_BUILD_MANUAL on a single slab");
    // Stream capture of exactly the stream-mode launch sequence.
    cudaStream_t root = (P == 1) ? c->cap_stream : c->slabs[0].stream;
    IB_CUDA(cudaSetDevice(c->slabs[0].device));
    IB_CUDA(cudaStreamBeginCapture(root, cudaStreamCaptureModeThreadLocal));
    int rc = join_into(c, root, true);
    int64_t kk = 0, ll = 0;
    if (rc == IB_OK) rc = enqueue_iterations(c, c->K, parity, pdl, P == 1 ? root : nullptr, &kk, &ll);
    if (rc == IB_OK) rc = join_into(c, root, false);
    cudaError_t e = cudaStreamEndCapture(root, &g);
    if (rc != IB_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    IB_CUDA(e);
    size_t n = 0;
    IB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    nodes += (int64_t)n;
  }
  auto b = clk::now();
  unsigned long long iflags = 0;
  if (c->gflags & IB_FLAG_DEVICE_LAUNCH) iflags |= cudaGraphInstantiateFlagDeviceLaunch;
  cudaGraphExec_t ex = nullptr;
  cudaError_t ie = cudaGraphInstantiateWithFlags(&ex, g, iflags);
  if (ie != cudaSuccess) {
    cudaGraphDestroy(g);
    return fail(IB_ECUDA, std::string("cudaGraphInstantiateWithFlags: ") + cudaGetErrorString(ie));
  }
  auto d = clk::now();
  c->ev(IB_EV_GRAPH_INSTANTIATED);
  if (!(c->gflags & IB_FLAG_NO_UPLOAD)) {
    IB_CUDA(cudaGraphUpload(ex, c->stream()));
    IB_CUDA(cudaStreamSynchronize(c->stream()));
  }
  auto e2 = clk::now();
  c->ev(IB_EV_GRAPH_UPLOADED);
  c->graph[parity] = g;
  c->exec[parity] = ex;
  if (tm) {
    tm->create_s += secs(a, b);
    tm->instantiate_s += secs(b, d);
    tm->upload_s += secs(d, e2);
    tm->build_s += secs(a, e2);
    tm->nodes += nodes;
  }
  return IB_OK;
}

int check_ctx(const ib_ctx *c) {
  if (!c) return fail(IB_EINVAL, "null context");
  return IB_OK;
}

}  // namespace

// ================================================================================================
// C ABI
// ================================================================================================
extern "C" {

int ib_abi_version(void) { return IB_ABI_VERSION; }

const char *ib_last_error(void) { return g_err.c_str(); }

int ib_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  if (count) *count = n;
  if (n == 0) return fail(IB_ENODEV, "no CUDA device visible");
  return IB_OK;
}

int ib_mem_info(int device, int64_t *free_bytes, int64_t *total_bytes) {
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(device));
  size_t f = 0, t = 0;
  IB_CUDA(cudaMemGetInfo(&f, &t));
  if (free_bytes) *free_bytes = (int64_t)f;
  if (total_bytes) *total_bytes = (int64_t)t;
  return IB_OK;
}

void ib_destroy(ib_ctx *c) {
  if (!c) return;
  DeviceGuard guard;
  if (!c->slabs.empty()) cudaSetDevice(c->slabs[0].device);
  free_graphs(c);
  if (c->comm) {
    nccl().CommDestroy(c->comm);
    c->comm = nullptr;
  }
  for (Slab &s : c->slabs) {
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (int p = 0; p < 2; ++p) {
      if (s.buf[p]) cudaFree(s.buf[p]);
      if (s.ev[p]) cudaEventDestroy(s.ev[p]);
    }
    if (s.power) cudaFree(s.power);
    if (s.join) cudaEventDestroy(s.join);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (!c->slabs.empty()) cudaSetDevice(c->slabs[0].device);
  if (c->lat[0] || c->lat[1]) {
    for (int p = 0; p < 2; ++p)
      if (c->lat[p]) cudaFree(c->lat[p]);
  } else {
    for (int f = 0; f < 6; ++f) {
      if (c->field[f]) cudaFree(c->field[f]);
      if (c->field2[f]) cudaFree(c->field2[f]);
    }
  }
  for (int p = 0; p < 2; ++p) {
    if (c->peer_buf_up[p]) cudaIpcCloseMemHandle(c->peer_buf_up[p]);
    if (c->peer_buf_dn[p]) cudaIpcCloseMemHandle(c->peer_buf_dn[p]);
  }
  if (c->peer_sync_up) cudaIpcCloseMemHandle(c->peer_sync_up);
  if (c->peer_sync_dn) cudaIpcCloseMemHandle(c->peer_sync_dn);
  if (c->sync) cudaFree(c->sync);
  if (c->d_counter) cudaFree(c->d_counter);
  if (c->tracing) {
    Cupti &cp = cupti();
    cp.Disable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
    cp.FlushAll(1);
    std::lock_guard<std::mutex> lock(cp.mu);
    cp.kernels.clear();
  }
  if (c->flush) cudaFree(c->flush);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

static int create_impl(ib_ctx *c, const int *devices, int ndevices) {
  const int P = ndevices;
  const bool hot = c->solver == IB_SOLVER_HOTSPOT2D || c->solver == IB_SOLVER_HOTSPOT3D;
  if (P > 1 && !hot && c->solver != IB_SOLVER_FDTD)
    return fail(IB_EINVAL, "multi-slab execution is defined for the hotspot solvers and the two-half-step FDTD");
  // axis-0 slabs: hotspot rows, or the FDTD lattice's nx+1 planes
  const int64_t rows = hot ? c->dims[0] : (c->solver == IB_SOLVER_FDTD && (P > 1 || c->nranks > 1) ? c->dims[0] + 1 : 1);
  if (P > rows) return fail(IB_EINVAL, "more slabs than rows along axis 0");
  c->slabs.resize(P);
  const bool dist = c->nranks > 1;
  if (dist && (P != 1 || !(hot || c->solver == IB_SOLVER_FDTD)))
    return fail(IB_EINVAL, "distributed contexts are single-slab hotspot or two-half-step FDTD grids");
  if (dist && c->nranks > rows) return fail(IB_EINVAL, "more ranks than rows along axis 0");
  for (int g = 0; g < P; ++g) {
    Slab &s = c->slabs[g];
    s.device = devices[g];
    const int64_t G = dist ? c->rank : g, NP = dist ? c->nranks : P;
    s.row_lo = (int)(rows * G / NP);  // workloads.py:65 bounds formula
    s.row_hi = (int)(rows * (G + 1) / NP);
    s.has_top = G > 0;
    s.has_bot = G + 1 < NP;
    IB_CUDA(cudaSetDevice(s.device));
    IB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    for (int p = 0; p < 2; ++p) IB_CUDA(cudaEventCreateWithFlags(&s.ev[p], cudaEventDisableTiming));
    IB_CUDA(cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming));
  }
  // peer access between neighbouring slabs on different devices (NVLink P2P stores)
  for (int g = 0; g + 1 < P; ++g) {
    int a = c->slabs[g].device, b = c->slabs[g + 1].device;
    if (a == b) continue;
    int ok = 0;
    IB_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
    if (!ok) return fail(IB_EINVAL, "devices " + std::to_string(a) + "," + std::to_string(b) + " lack peer access");
    for (int dir = 0; dir < 2; ++dir) {
      IB_CUDA(cudaSetDevice(dir ? b : a));
      cudaError_t e = cudaDeviceEnablePeerAccess(dir ? a : b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else IB_CUDA(e);
    }
  }
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->slabs[0].device));
  IB_CUDA(cudaEventCreate(&c->t0));
  IB_CUDA(cudaEventCreate(&c->t1));
  IB_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  IB_CUDA(cudaMalloc(&c->d_counter, sizeof(int)));
  if (dist) {
    IB_CUDA(cudaMalloc(&c->sync, 256));
    IB_CUDA(cudaMemset(c->sync, 0, 256));
  }
  const int es = c->esize;
  if (hot) {
    const int64_t plane = c->plane();
    for (Slab &s : c->slabs) {
      IB_CUDA(cudaSetDevice(s.device));
      const int64_t planes = s.rows() + (P > 1 || dist ? 2 : 0);
      for (int p = 0; p < 2; ++p) {
        IB_CUDA(cudaMalloc(&s.buf[p], (size_t)(planes * plane * es)));
        IB_CUDA(cudaMemset(s.buf[p], 0, (size_t)(planes * plane * es)));
      }
      IB_CUDA(cudaMalloc(&s.power, (size_t)(s.rows() * plane * es)));
      IB_CUDA(cudaMemset(s.power, 0, (size_t)(s.rows() * plane * es)));
    }
    IB_CUDA(cudaSetDevice(c->slabs[0].device));
  } else if (c->fdtd()) {
    // both FDTD solvers: the padded lattice (kernels.cuh, k_fdtd_lf); the fused leapfrog double
    // buffers it, the two half-steps update one copy in place
    const int64_t nx = c->dims[0], ny = c->dims[1], nz = c->dims[2];
    const int64_t v = 16 / es;
    c->lat_pitch = (nz + 1 + v - 1) / v * v;
    c->lat_fs = (nx + 1) * (ny + 1) * c->lat_pitch;
    const bool fused = c->solver == IB_SOLVER_FDTD_FUSED;
    if (fused && lf_config(c).tj == 0)
      return fail(IB_EINVAL, "fused fdtd: the z rows are too long for one CTA (threads or shared-memory ring); use the two-kernel solver");
    if (P > 1 || dist) {  // slabs / ranks: planes [lo, hi) plus one halo plane each side, in place
      if (lf_config(c).tj == 0)
        return fail(IB_EINVAL, "fdtd slabs need the staged kernel: the z rows are too long for one CTA");
      const int64_t plane = (ny + 1) * c->lat_pitch;
      for (Slab &s : c->slabs) {
        IB_CUDA(cudaSetDevice(s.device));
        s.fs = (int64_t)(s.rows() + 2) * plane;
        const size_t bb = (size_t)(6 * s.fs * es);
        IB_CUDA(cudaMalloc(&s.buf[0], bb));
        IB_CUDA(cudaMemset(s.buf[0], 0, bb));
      }
      IB_CUDA(cudaSetDevice(c->slabs[0].device));
      IB_CUDA(cudaDeviceSynchronize());
      return IB_OK;
    }
    const size_t b = (size_t)(6 * c->lat_fs * es);
    for (int p = 0; p < (fused ? 2 : 1); ++p) {
      IB_CUDA(cudaMalloc(&c->lat[p], b));
      IB_CUDA(cudaMemset(c->lat[p], 0, b));
    }
    for (int f = 0; f < 6; ++f) {
      c->field[f] = (char *)c->lat[0] + (size_t)(f * c->lat_fs * es);
      if (fused) c->field2[f] = (char *)c->lat[1] + (size_t)(f * c->lat_fs * es);
    }
  } else {
    for (int f = 0; f < c->nfields; ++f) {
      const size_t b = (size_t)(numel(c->fshape[f], c->fndim[f]) * es);
      IB_CUDA(cudaMalloc(&c->field[f], b));
      IB_CUDA(cudaMemset(c->field[f], 0, b));
    }
  }
  IB_CUDA(cudaDeviceSynchronize());
  return IB_OK;
}

static int create_common(ib_ctx **out, int solver, int dtype, const int64_t *dims, int ndims,
                         const double *scalars, int nscalars, const int *devices, int ndevices,
                         int rank, int nranks, const void *id128) {
  if (!out) return fail(IB_EINVAL, "out is null");
  *out = nullptr;
  if (solver < IB_SOLVER_VECTOR || solver > IB_SOLVER_FDTD_FUSED) return fail(IB_EINVAL, "unknown solver");
  if (dtype != IB_F32 && dtype != IB_F64) return fail(IB_EINVAL, "dtype must be IB_F32 or IB_F64");
  static const int want_nd[5] = {1, 2, 3, 3, 3};
  static const int want_ns[5] = {1, 1, 1, 3, 3};
  if (ndims != want_nd[solver] || !dims)
    return fail(IB_EINVAL, "solver expects " + std::to_string(want_nd[solver]) + " dims, got " + std::to_string(ndims));
  if (nscalars != want_ns[solver] || !scalars)
    return fail(IB_EINVAL, "solver expects " + std::to_string(want_ns[solver]) + " scalars");
  for (int i = 0; i < ndims; ++i)
    if (dims[i] < 1) return fail(IB_EINVAL, "dims must be >= 1");
  if (solver != IB_SOLVER_VECTOR) {
    for (int i = 0; i < ndims; ++i)
      if (dims[i] > (1LL << 30)) return fail(IB_EINVAL, "dimension too large");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(IB_ENODEV, "no CUDA device visible (this library has no CPU fallback)");
  }
  std::vector<int> devs;
  if (!devices || ndevices <= 0) {
    int d = 0;
    IB_CUDA(cudaGetDevice(&d));
    devs.push_back(d);
  } else {
    for (int i = 0; i < ndevices; ++i) {
      if (devices[i] < 0 || devices[i] >= ndev) return fail(IB_EINVAL, "device id out of range");
      devs.push_back(devices[i]);
    }
  }
  DeviceGuard guard;
  ib_ctx *c = new ib_ctx();
  c->solver = solver;
  c->dtype = dtype;
  c->esize = dtype == IB_F32 ? 4 : 8;
  c->ndims = ndims;
  for (int i = 0; i < ndims; ++i) c->dims[i] = dims[i];
  for (int i = 0; i < nscalars; ++i) c->scalars[i] = scalars[i];
  c->rank = rank;
  c->nranks = nranks;
  if ((solver == IB_SOLVER_FDTD || solver == IB_SOLVER_FDTD_FUSED) && !(scalars[0] > 0.0)) {
    delete c;
    return fail(IB_EINVAL, "cell_size must be positive");
  }
  if (solver == IB_SOLVER_VECTOR) {
    c->nfields = 1;
    c->fndim[0] = 1;
    c->fshape[0][0] = dims[0];
  } else if (solver == IB_SOLVER_FDTD || solver == IB_SOLVER_FDTD_FUSED) {
    const int64_t nx = dims[0], ny = dims[1], nz = dims[2];
    const int64_t sh[6][3] = {{nx, ny + 1, nz + 1}, {nx + 1, ny, nz + 1}, {nx + 1, ny + 1, nz},
                              {nx + 1, ny, nz},     {nx, ny + 1, nz},     {nx, ny, nz + 1}};
    c->nfields = 6;
    for (int f = 0; f < 6; ++f) {
      c->fndim[f] = 3;
      for (int a = 0; a < 3; ++a) c->fshape[f][a] = sh[f][a];
    }
    if ((nx + 1) > 65535) {
      delete c;
      return fail(IB_EINVAL, "fdtd nx must be < 65535");
    }
  } else {
    c->nfields = 2;
    for (int f = 0; f < 2; ++f) {
      c->fndim[f] = ndims;
      for (int a = 0; a < ndims; ++a) c->fshape[f][a] = dims[a];
    }
  }
  int rc = create_impl(c, devs.data(), (int)devs.size());
  if (rc == IB_OK && nranks > 1 && id128) {
    Nccl &n = nccl();
    if (!n.ok) {
      rc = fail(IB_ECUDA, n.err);
    } else {
      NcclId id;
      std::memcpy(id.internal, id128, sizeof(id.internal));
      cudaSetDevice(c->slabs[0].device);
      const int r = n.CommInitRank(&c->comm, nranks, id, rank);
      if (r != 0) {
        c->comm = nullptr;
        rc = fail(IB_ECUDA, std::string("ncclCommInitRank: ") + n.GetErrorString(r));
      }
    }
  }
  if (rc != IB_OK) {
    std::string msg = g_err;
    ib_destroy(c);
    g_err = msg;
    return rc;
  }
  *out = c;
  return IB_OK;
}

int ib_create(ib_ctx **out, int solver, int dtype, const int64_t *dims, int ndims,
              const double *scalars, int nscalars, const int *devices, int ndevices) {
  return create_common(out, solver, dtype, dims, ndims, scalars, nscalars, devices, ndevices, 0, 1,
                       nullptr);
}

int ib_nccl_unique_id(void *id128) {
  if (!id128) return fail(IB_EINVAL, "id buffer is null");
  Nccl &n = nccl();
  if (!n.ok) return fail(IB_ECUDA, n.err);
  NcclId id;
  const int r = n.GetUniqueId(&id);
  if (r != 0) return fail(IB_ECUDA, std::string("ncclGetUniqueId: ") + n.GetErrorString(r));
  std::memcpy(id128, id.internal, sizeof(id.internal));
  return IB_OK;
}

int ib_create_dist(ib_ctx **out, int solver, int dtype, const int64_t *dims, int ndims,
                   const double *scalars, int nscalars, int device, int rank, int nranks,
                   const void *id128) {
  if (solver != IB_SOLVER_HOTSPOT2D && solver != IB_SOLVER_HOTSPOT3D && solver != IB_SOLVER_FDTD)
    return fail(IB_EINVAL, "distributed contexts are defined for hotspot grids and the two-half-step FDTD");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(IB_EINVAL, "bad rank / nranks");
  if (solver == IB_SOLVER_FDTD && nranks > 1 && id128)
    return fail(IB_EINVAL, "distributed FDTD uses the peer exchange: pass id128 = NULL, then ib_ipc_attach");

  return create_common(out, solver, dtype, dims, ndims, scalars, nscalars, &device, 1, rank, nranks,
                       id128);
}

int ib_ipc_export(const ib_ctx *c, void *out, size_t bytes) {
  IB_TRY(check_ctx(c));
  if (!c->dist()) return fail(IB_EINVAL, "IPC export is for distributed (ib_create_dist) contexts");
  if (!out || bytes < IB_IPC_BYTES) return fail(IB_EINVAL, "IPC export needs IB_IPC_BYTES bytes");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  cudaIpcMemHandle_t h[3];
  std::memset(h, 0, sizeof(h));
  for (int p = 0; p < 2; ++p)
    if (c->slabs[0].buf[p]) IB_CUDA(cudaIpcGetMemHandle(&h[p], c->slabs[0].buf[p]));  // FDTD: one lattice
  IB_CUDA(cudaIpcGetMemHandle(&h[2], c->sync));
  std::memcpy(out, h, sizeof(h));
  return IB_OK;
}

int ib_ipc_attach(ib_ctx *c, const void *up, const void *dn) {
  IB_TRY(check_ctx(c));
  if (!c->dist()) return fail(IB_EINVAL, "IPC attach is for distributed (ib_create_dist) contexts");
  const Slab &s = c->slabs[0];
  if ((s.has_top && !up) || (s.has_bot && !dn))
    return fail(IB_EINVAL, "IPC attach needs the handles of every neighbour rank");
  if (c->peer) return fail(IB_ESTATE, "IPC peers already attached");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(s.device));
  auto open = [&](const void *blob, void **bufs, unsigned long long **sync) -> int {
    cudaIpcMemHandle_t h[3];
    std::memcpy(h, blob, sizeof(h));
    for (int p = 0; p < (c->fdtd() ? 1 : 2); ++p)
      IB_CUDA(cudaIpcOpenMemHandle(&bufs[p], h[p], cudaIpcMemLazyEnablePeerAccess));
    void *sp = nullptr;
    IB_CUDA(cudaIpcOpenMemHandle(&sp, h[2], cudaIpcMemLazyEnablePeerAccess));
    *sync = (unsigned long long *)sp;
    return IB_OK;
  };
  if (s.has_top) IB_TRY(open(up, c->peer_buf_up, &c->peer_sync_up));
  if (s.has_bot) IB_TRY(open(dn, c->peer_buf_dn, &c->peer_sync_dn));
  const int64_t rows = c->fdtd() ? c->dims[0] + 1 : c->dims[0];
  c->peer_rows_up = (int)(rows * c->rank / c->nranks - rows * (c->rank - 1) / c->nranks);
  c->peer_rows_dn = (int)(rows * (c->rank + 2) / c->nranks - rows * (c->rank + 1) / c->nranks);
  c->peer = true;
  return IB_OK;
}

int ib_slab_info(const ib_ctx *c, int64_t *lo, int64_t *hi, int *has_top, int *has_bot) {
  IB_TRY(check_ctx(c));
  const Slab &s = c->slabs[0];
  const bool sl = c->hotspot() || (c->fdtd() && c->dist());
  if (lo) *lo = sl ? s.row_lo : 0;
  if (hi) *hi = sl ? s.row_hi : c->dims[0];
  if (has_top) *has_top = c->nranks > 1 && s.has_top;
  if (has_bot) *has_bot = c->nranks > 1 && s.has_bot;
  return IB_OK;
}

int ib_num_fields(const ib_ctx *c) { return c ? c->nfields : 0; }

int ib_field_shape(const ib_ctx *c, int field, int64_t *shape3, int *ndim) {
  IB_TRY(check_ctx(c));
  if (field < 0 || field >= c->nfields) return fail(IB_EINVAL, "field index out of range");
  if (ndim) *ndim = c->fndim[field];
  if (shape3)
    for (int a = 0; a < 3; ++a) shape3[a] = a < c->fndim[field] ? c->fshape[field][a] : 1;
  return IB_OK;
}

int64_t ib_field_bytes(const ib_ctx *c, int field) {
  if (!c || field < 0 || field >= c->nfields) return -1;
  return numel(c->fshape[field], c->fndim[field]) * c->esize;
}

int64_t ib_iteration_bytes(const ib_ctx *c) {
  if (!c) return -1;
  const int64_t es = c->esize;
  switch (c->solver) {
    case IB_SOLVER_VECTOR: return 2 * c->dims[0] * es;
    case IB_SOLVER_HOTSPOT2D:
    case IB_SOLVER_HOTSPOT3D: return 3 * numel(c->dims, c->ndims) * es;
    case IB_SOLVER_FDTD: {
      int64_t e = 0, h = 0;
      for (int f = 0; f < 3; ++f) e += numel(c->fshape[f], 3);
      for (int f = 3; f < 6; ++f) h += numel(c->fshape[f], 3);
      return (e + 2 * h + h + 2 * e) * es;  // H half-step + E half-step
    }
    case IB_SOLVER_FDTD_FUSED: {
      int64_t n = 0;
      for (int f = 0; f < 6; ++f) n += numel(c->fshape[f], 3);
      return 2 * n * es;  // every field read once and written once
    }
  }
  return -1;
}

static int hotspot_copy(ib_ctx *c, int field, void *host, size_t bytes, bool up) {
  const int64_t plane = c->plane();
  const int64_t pb = plane * c->esize;
  const int P = (int)c->slabs.size();
  char *h = (char *)host;
  if (c->nranks > 1) {  // local window: [lo - top, hi + bot) up, [lo, hi) down (see header)
    Slab &s = c->slabs[0];
    IB_CUDA(cudaSetDevice(s.device));
    if (field == 1) {
      IB_CUDA(cudaMemcpyAsync(up ? s.power : host, up ? host : s.power, (size_t)(s.rows() * pb),
                              up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, s.stream));
    } else if (up) {
      char *dev = (char *)s.buf[c->cur] + (s.has_top ? 0 : pb);
      const size_t nb = (size_t)((s.rows() + s.has_top + s.has_bot) * pb);
      IB_CUDA(cudaMemcpyAsync(dev, h, nb, cudaMemcpyHostToDevice, s.stream));
    } else {
      IB_CUDA(cudaMemcpyAsync(h, (char *)s.buf[c->cur] + pb, (size_t)(s.rows() * pb),
                              cudaMemcpyDeviceToHost, s.stream));
    }
    IB_CUDA(cudaStreamSynchronize(s.stream));
    (void)bytes;
    return IB_OK;
  }
  for (int g = 0; g < P; ++g) {
    Slab &s = c->slabs[g];
    IB_CUDA(cudaSetDevice(s.device));
    const int64_t off = (P > 1) ? pb : 0;
    char *dev = field == 0 ? (char *)s.buf[c->cur] + off : (char *)s.power;
    const size_t nb = (size_t)(s.rows() * pb);
    if (up) {
      IB_CUDA(cudaMemcpyAsync(dev, h + s.row_lo * pb, nb, cudaMemcpyHostToDevice, s.stream));
      if (field == 0 && s.has_top)
        IB_CUDA(cudaMemcpyAsync((char *)s.buf[c->cur], h + (s.row_lo - 1) * pb, (size_t)pb,
                                cudaMemcpyHostToDevice, s.stream));
      if (field == 0 && s.has_bot)
        IB_CUDA(cudaMemcpyAsync((char *)s.buf[c->cur] + (int64_t)(s.rows() + 1) * pb,
                                h + (int64_t)s.row_hi * pb, (size_t)pb, cudaMemcpyHostToDevice, s.stream));
    } else {
      IB_CUDA(cudaMemcpyAsync(h + s.row_lo * pb, dev, nb, cudaMemcpyDeviceToHost, s.stream));
    }
  }
  (void)bytes;
  for (Slab &s : c->slabs) {
    IB_CUDA(cudaSetDevice(s.device));
    IB_CUDA(cudaStreamSynchronize(s.stream));
  }
  return IB_OK;
}

// FDTD slab / rank: the global planes of `field` a transfer moves — upload: the owned planes and
// the halo plane each side that exists, download: the owned planes; clipped to the field's extent.
static void fdtd_planes(const ib_ctx *c, const Slab &s, int field, bool up, int64_t *lo, int64_t *hi) {
  const int64_t n = c->fshape[field][0];
  *lo = std::min<int64_t>(up ? std::max<int64_t>(s.row_lo - 1, 0) : s.row_lo, n);
  *hi = std::min<int64_t>(up ? s.row_hi + 1 : s.row_hi, n);
  if (*hi < *lo) *hi = *lo;
}

static int xfer(ib_ctx *c, int field, void *host, size_t bytes, bool up) {
  IB_TRY(check_ctx(c));
  if (field < 0 || field >= c->nfields) return fail(IB_EINVAL, "field index out of range");
  if (!host) return fail(IB_EINVAL, "host pointer is null");
  int64_t want = ib_field_bytes(c, field);
  if (c->nranks > 1 && c->hotspot()) {
    const Slab &s = c->slabs[0];
    const int64_t pb = c->plane() * c->esize;
    want = (field == 0 && up) ? (s.rows() + s.has_top + s.has_bot) * pb : s.rows() * pb;
  } else if (c->nranks > 1) {  // FDTD rank: this field's planes of the window (see the header)
    int64_t lo, hi;
    fdtd_planes(c, c->slabs[0], field, up, &lo, &hi);
    want = (hi - lo) * c->fshape[field][1] * c->fshape[field][2] * c->esize;
  }
  if ((int64_t)bytes != want)
    return fail(IB_EINVAL, "field " + std::to_string(field) + " holds " + std::to_string(want) +
                               " bytes, got " + std::to_string(bytes));
  DeviceGuard guard;
  if (c->hotspot()) return hotspot_copy(c, field, host, bytes, up);
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  if (c->fdtd() && (c->slabs.size() > 1 || c->dist())) {  // slabs / ranks: owned (+ halo) planes
    const int64_t *sh = c->fshape[field];
    const size_t es = (size_t)c->esize;
    const int64_t plane = (c->dims[1] + 1) * c->lat_pitch;
    int64_t host0 = 0;  // global plane of the host buffer's first plane (a rank holds its window)
    if (c->dist()) {
      int64_t hi0;
      fdtd_planes(c, c->slabs[0], field, up, &host0, &hi0);
    }
    for (Slab &s : c->slabs) {
      IB_CUDA(cudaSetDevice(s.device));
      int64_t lo, hi;
      fdtd_planes(c, s, field, up, &lo, &hi);
      if (hi <= lo) continue;
      char *hbase = (char *)host + (size_t)((lo - host0) * sh[1] * sh[2]) * es;
      char *dbase = (char *)s.buf[0] + (size_t)(field * s.fs + (lo - s.row_lo + 1) * plane) * es;
      cudaMemcpy3DParms m = {};
      cudaPitchedPtr hp = make_cudaPitchedPtr(hbase, (size_t)sh[2] * es, (size_t)sh[2] * es, (size_t)sh[1]);
      cudaPitchedPtr dp = make_cudaPitchedPtr(dbase, (size_t)c->lat_pitch * es, (size_t)sh[2] * es,
                                              (size_t)(c->dims[1] + 1));
      m.srcPtr = up ? hp : dp;
      m.dstPtr = up ? dp : hp;
      m.extent = make_cudaExtent((size_t)sh[2] * es, (size_t)sh[1], (size_t)(hi - lo));
      m.kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
      IB_CUDA(cudaMemcpy3DAsync(&m, s.stream));
    }
    for (Slab &s : c->slabs) {
      IB_CUDA(cudaSetDevice(s.device));
      IB_CUDA(cudaStreamSynchronize(s.stream));
    }
    return IB_OK;
  }
  void *dev = c->fieldp(field, c->cur);
  if (c->fdtd()) {  // C-order host array <-> padded lattice
    const int64_t *sh = c->fshape[field];
    const size_t es = (size_t)c->esize;
    cudaMemcpy3DParms m = {};
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)sh[2] * es, (size_t)sh[2] * es, (size_t)sh[1]);
    cudaPitchedPtr dp = make_cudaPitchedPtr(dev, (size_t)c->lat_pitch * es, (size_t)sh[2] * es,
                                            (size_t)(c->dims[1] + 1));
    m.srcPtr = up ? hp : dp;
    m.dstPtr = up ? dp : hp;
    m.extent = make_cudaExtent((size_t)sh[2] * es, (size_t)sh[1], (size_t)sh[0]);
    m.kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    IB_CUDA(cudaMemcpy3DAsync(&m, c->stream()));
    IB_CUDA(cudaStreamSynchronize(c->stream()));
    return IB_OK;
  }
  if (up)
    IB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c->stream()));
  else
    IB_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream()));
  IB_CUDA(cudaStreamSynchronize(c->stream()));
  return IB_OK;
}

int ib_upload(ib_ctx *c, int field, const void *host, size_t bytes) {
  return xfer(c, field, const_cast<void *>(host), bytes, true);
}
int ib_download(ib_ctx *c, int field, void *host, size_t bytes) {
  return xfer(c, field, host, bytes, false);
}

int ib_sync(ib_ctx *c) {
  IB_TRY(check_ctx(c));
  DeviceGuard guard;
  for (Slab &s : c->slabs) {
    IB_CUDA(cudaSetDevice(s.device));
    IB_CUDA(cudaStreamSynchronize(s.stream));
  }
  return IB_OK;
}

static int sync_all(ib_ctx *c) {
  for (Slab &s : c->slabs) {
    IB_CUDA(cudaSetDevice(s.device));
    IB_CUDA(cudaStreamSynchronize(s.stream));
  }
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  return IB_OK;
}

int ib_run_stream(ib_ctx *c, int64_t iterations, int flags, ib_times *tm) {
  NvtxRange range("ib stream run (per-kernel launches)");
  IB_TRY(check_ctx(c));
  if (c->dist() && !c->comm && !c->peer)
    return fail(IB_ESTATE, "distributed context without an exchange: call ib_ipc_attach first");
  if (iterations < 0) return fail(IB_EINVAL, "total_iterations must be >= 0");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  ib_times t = {};
  const bool pdl = (flags & IB_FLAG_PDL) != 0;
  auto a = clk::now();
  IB_CUDA(cudaEventRecord(c->t0, c->stream()));
  IB_TRY(join_into(c, c->stream(), true));
  IB_TRY(enqueue_iterations(c, iterations, c->cur, pdl, nullptr, &t.kernels, &t.launches));
  if (c->peer && iterations > 0) IB_TRY(launch_dist_wait(c, c->stream()));
  IB_TRY(join_into(c, c->stream(), false));
  IB_CUDA(cudaEventRecord(c->t1, c->stream()));
  IB_CUDA(cudaEventSynchronize(c->t1));
  IB_TRY(sync_all(c));
  auto b = clk::now();
  float ms = 0;
  IB_CUDA(cudaEventElapsedTime(&ms, c->t0, c->t1));
  if (c->ping_pong() && (iterations & 1)) c->cur ^= 1;
  t.exec_s = secs(a, b);
  t.gpu_s = ms * 1e-3;
  if (tm) *tm = t;
  return IB_OK;
}

int ib_num_steps(const ib_ctx *c) { return c ? (c->solver == IB_SOLVER_FDTD ? 2 : 1) : 0; }

int ib_run_step(ib_ctx *c, int step, ib_times *tm) {
  IB_TRY(check_ctx(c));
  if (step < 0 || step >= ib_num_steps(c)) return fail(IB_EINVAL, "step index out of range");
  if (c->dist())
    return fail(IB_EINVAL, "per-step calls are not defined for distributed contexts (use ib_run_stream)");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  std::vector<Launch> v;
  iteration_launches(c, c->cur, v);
  ib_times t = {};
  auto a = clk::now();
  IB_CUDA(cudaEventRecord(c->t0, c->stream()));
  IB_TRY(join_into(c, c->stream(), true));
  for (Launch &L : v) {
    if (c->solver == IB_SOLVER_FDTD && L.step != step) continue;
    Slab &s = c->slabs[L.slab];
    IB_CUDA(cudaSetDevice(s.device));
    IB_TRY(launch_one(L, s.stream, false));
    ++t.kernels;
  }
  IB_TRY(join_into(c, c->stream(), false));
  IB_CUDA(cudaEventRecord(c->t1, c->stream()));
  IB_CUDA(cudaEventSynchronize(c->t1));
  IB_TRY(sync_all(c));
  auto b = clk::now();
  float ms = 0;
  IB_CUDA(cudaEventElapsedTime(&ms, c->t0, c->t1));
  if (c->ping_pong()) c->cur ^= 1;
  t.launches = t.kernels;
  t.exec_s = secs(a, b);
  t.gpu_s = ms * 1e-3;
  if (tm) *tm = t;
  return IB_OK;
}

int ib_graph_destroy(ib_ctx *c) {
  IB_TRY(check_ctx(c));
  DeviceGuard guard;
  cudaSetDevice(c->slabs[0].device);
  free_graphs(c);
  return IB_OK;
}

int64_t ib_graph_batch_size(const ib_ctx *c) { return c ? c->K : -1; }

int ib_graph_build(ib_ctx *c, int64_t batch_size, int build_mode, int flags, ib_times *tm) {
  IB_TRY(check_ctx(c));
  if (c->dist() && !c->comm && !c->peer)
    return fail(IB_ESTATE, "distributed context without an exchange: call ib_ipc_attach first");
  if (batch_size < 1) return fail(IB_EINVAL, "batch_size must be >= 1");
  if (build_mode != IB_BUILD_MANUAL && build_mode != IB_BUILD_CAPTURE)
    return fail(IB_EINVAL, "unknown build mode");
  if ((flags & IB_FLAG_DEVICE_LAUNCH) && c->slabs.size() > 1) {
    for (auto &s : c->slabs)
      if (s.device != c->slabs[0].device)
        return fail(IB_EINVAL, "device-launch graphs must live on one device");
  }
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  free_graphs(c);
  c->K = batch_size;
  c->gflags = flags;
  c->gmode = build_mode;
  ib_times t = {};
  size_t f0 = 0, f1 = 0, tot = 0;
  const bool meminfo = (flags & IB_FLAG_MEMINFO) != 0;
  if (meminfo) IB_CUDA(cudaMemGetInfo(&f0, &tot));
  int rc = build_one(c, c->cur, &t);
  if (rc == IB_OK && c->ping_pong() && (batch_size & 1)) rc = build_one(c, c->cur ^ 1, &t);
  if (rc != IB_OK) {
    std::string msg = g_err;
    free_graphs(c);
    g_err = msg;
    return rc;
  }
  if (meminfo) {
    IB_CUDA(cudaMemGetInfo(&f1, &tot));
    t.graph_bytes = (int64_t)f0 - (int64_t)f1;
  }
  if (tm) *tm = t;
  return IB_OK;
}

int ib_graph_run(ib_ctx *c, int64_t num_batches, ib_times *tm) {
  NvtxRange range("ib graph run (batch launches)");
  IB_TRY(check_ctx(c));
  if (num_batches < 0) return fail(IB_EINVAL, "num_batches must be >= 0");
  if (c->K < 1) return fail(IB_ESTATE, "no graph built: call ib_graph_build first");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  ib_times t = {};
  // the state parity may have moved since the build (e.g. an odd stream run): build lazily
  if (!c->exec[c->cur]) IB_TRY(build_one(c, c->cur, &t));
  if (c->ping_pong() && (c->K & 1) && !c->exec[c->cur ^ 1]) IB_TRY(build_one(c, c->cur ^ 1, &t));
  const bool wh = (c->gflags & IB_FLAG_WHILE) != 0;
  const int64_t per = c->K * (c->solver == IB_SOLVER_FDTD ? 2 : 1) * (int64_t)c->slabs.size();  // kernels / batch
  auto a = clk::now();
  IB_CUDA(cudaEventRecord(c->t0, c->stream()));
  if (num_batches > 0) {
    if (wh) {
      if (c->ping_pong() && (c->K & 1) && num_batches > 1)
        return fail(IB_EINVAL, "IB_FLAG_WHILE with an odd batch_size needs num_batches <= 1 (ping-pong parity)");
      int nb = (int)num_batches;
      IB_CUDA(cudaMemcpyAsync(c->d_counter, &nb, sizeof(int), cudaMemcpyHostToDevice, c->stream()));
      c->ev(IB_EV_GRAPH_LAUNCHED, 0);
      IB_CUDA(cudaGraphLaunch(c->exec[c->cur], c->stream()));
      t.launches = 1;
      if (c->ping_pong() && (c->K & 1)) c->cur ^= 1;
    } else {
      for (int64_t b = 0; b < num_batches; ++b) {
        c->ev(IB_EV_GRAPH_LAUNCHED, b);
        IB_CUDA(cudaGraphLaunch(c->exec[c->cur], c->stream()));
        if (c->ping_pong() && (c->K & 1)) c->cur ^= 1;
      }
      t.launches = num_batches;
    }
  }
  // peer exchange: the run ends when the neighbours are done too (their last halo stores into
  // this rank's planes have landed), so a following upload / download cannot race them
  if (c->peer && num_batches > 0) IB_TRY(launch_dist_wait(c, c->stream()));
  IB_CUDA(cudaEventRecord(c->t1, c->stream()));
  IB_CUDA(cudaEventSynchronize(c->t1));
  auto b = clk::now();
  float ms = 0;
  IB_CUDA(cudaEventElapsedTime(&ms, c->t0, c->t1));
  t.exec_s = secs(a, b);
  t.gpu_s = ms * 1e-3;
  t.kernels = per * num_batches;
  if (tm) *tm = t;
  return IB_OK;
}

int ib_run_batched(ib_ctx *c, int64_t batch_size, int64_t num_batches, int build_mode, int flags,
                   ib_times *tm) {
  IB_TRY(check_ctx(c));
  if (batch_size < 1) return fail(IB_EINVAL, "batch_size must be >= 1");
  if (num_batches < 0) return fail(IB_EINVAL, "num_batches must be >= 0");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  cudaEvent_t e0;
  IB_CUDA(cudaEventCreate(&e0));
  IB_CUDA(cudaEventRecord(e0, c->stream()));
  ib_times b = {}, r = {};
  int rc = ib_graph_build(c, batch_size, build_mode, flags, &b);
  if (rc == IB_OK) rc = ib_graph_run(c, num_batches, &r);
  if (rc != IB_OK) {
    cudaEventDestroy(e0);
    return rc;
  }
  float ms = 0;
  cudaError_t e = cudaEventElapsedTime(&ms, e0, c->t1);
  cudaEventDestroy(e0);
  IB_CUDA(e);
  free_graphs(c);
  if (tm) {
    *tm = b;
    tm->exec_s = r.exec_s;
    tm->gpu_s = ms * 1e-3;
    tm->kernels = r.kernels;
    tm->launches = r.launches;
    tm->build_s += r.build_s;  // lazily built parity executables, if any
  }
  return IB_OK;
}

int ib_run_peeled(ib_ctx *c, int64_t total, int64_t batch_size, int build_mode, int flags,
                  ib_times *tm) {
  IB_TRY(check_ctx(c));
  if (total < 0) return fail(IB_EINVAL, "total_iterations must be >= 0");
  if (batch_size < 1) return fail(IB_EINVAL, "batch_size must be >= 1");
  if (flags & IB_FLAG_WHILE) return fail(IB_EINVAL, "IB_FLAG_WHILE is not supported with peeling");
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  cudaEvent_t e0;
  IB_CUDA(cudaEventCreate(&e0));
  IB_CUDA(cudaEventRecord(e0, c->stream()));
  ib_times acc = {};
  const int64_t full = total / batch_size, rem = total % batch_size;
  int rc = IB_OK;
  for (int part = 0; part < 2 && rc == IB_OK; ++part) {
    const int64_t k = part == 0 ? batch_size : rem;
    const int64_t n = part == 0 ? full : 1;
    if (k == 0 || n == 0) continue;
    ib_times b = {}, r = {};
    rc = ib_graph_build(c, k, build_mode, flags, &b);
    if (rc == IB_OK) rc = ib_graph_run(c, n, &r);
    acc.create_s += b.create_s;
    acc.instantiate_s += b.instantiate_s;
    acc.upload_s += b.upload_s;
    acc.build_s += b.build_s + r.build_s;
    acc.exec_s += r.exec_s;
    acc.kernels += r.kernels;
    acc.launches += r.launches;
    acc.nodes += b.nodes;
  }
  if (rc != IB_OK) {
    cudaEventDestroy(e0);
    return rc;
  }
  IB_CUDA(cudaEventRecord(c->t1, c->stream()));
  IB_CUDA(cudaEventSynchronize(c->t1));
  float ms = 0;
  cudaError_t e = cudaEventElapsedTime(&ms, e0, c->t1);
  cudaEventDestroy(e0);
  IB_CUDA(e);
  free_graphs(c);
  acc.gpu_s = ms * 1e-3;
  if (tm) *tm = acc;
  return IB_OK;
}

int ib_host_alloc(void **ptr, size_t bytes) {
  if (!ptr) return fail(IB_EINVAL, "ptr is null");
  IB_CUDA(cudaMallocHost(ptr, bytes ? bytes : 1));
  return IB_OK;
}

int ib_host_free(void *ptr) {
  if (ptr) IB_CUDA(cudaFreeHost(ptr));
  return IB_OK;
}

uint64_t ib_fnv1a64(const void *data, size_t nbytes, uint64_t h) {
  const unsigned char *p = (const unsigned char *)data;
  for (size_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

uint64_t ib_fnv1a64_f64(const void *values, size_t n, int dtype, uint64_t h) {
  if (dtype == IB_F64) return ib_fnv1a64(values, n * 8, h);
  const float *f = (const float *)values;
  for (size_t i = 0; i < n; ++i) {
    const double d = (double)f[i];
    unsigned char b[8];
    std::memcpy(b, &d, 8);  // x86-64 is little-endian: these are the "<f8" bytes
    for (int q = 0; q < 8; ++q) {
      h ^= b[q];
      h *= 0x100000001b3ULL;
    }
  }
  return h;
}

int ib_trace_enable(ib_ctx *c, int64_t capacity) {
  IB_TRY(check_ctx(c));
  if (capacity < 0) return fail(IB_EINVAL, "capacity must be >= 0");
  if (capacity > 0 && c->slabs.size() > 1) return fail(IB_EINVAL, "tracing needs a single-slab context");
  Cupti &cp = cupti();
  if (!cp.ok) return fail(IB_ECUDA, cp.err);
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  IB_TRY(sync_all(c));
  static bool registered = false;
  if (!registered) {
    if (cp.RegisterCallbacks(cupti_buffer_requested, cupti_buffer_completed) != CUPTI_SUCCESS)
      return fail(IB_ECUDA, "cuptiActivityRegisterCallbacks failed");
    registered = true;
  }
  if (c->tracing) {
    cp.Disable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
    cp.FlushAll(1);
  }
  {
    std::lock_guard<std::mutex> lock(cp.mu);
    cp.kernels.clear();
  }
  c->host_ev.clear();
  c->tracing = false;
  c->trace_cap = 0;
  if (capacity == 0) return IB_OK;
  if (cp.Enable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS)
    return fail(IB_ECUDA, "cuptiActivityEnable(CONCURRENT_KERNEL) failed");
  c->tracing = true;
  c->trace_cap = capacity;
  return IB_OK;
}

int64_t ib_trace_kernels(ib_ctx *c, int64_t *out, int64_t capacity) {
  if (!c || !c->tracing) return fail(IB_ESTATE, "tracing is not enabled");
  DeviceGuard guard;
  cudaSetDevice(c->slabs[0].device);
  if (sync_all(c) != IB_OK) return IB_ECUDA;
  Cupti &cp = cupti();
  cp.FlushAll(1);
  std::lock_guard<std::mutex> lock(cp.mu);
  std::vector<std::pair<int64_t, int64_t>> k;
  for (size_t i = 0; i + 1 < cp.kernels.size(); i += 2) k.push_back({cp.kernels[i], cp.kernels[i + 1]});
  std::sort(k.begin(), k.end());
  const int64_t n = (int64_t)k.size();
  for (int64_t i = 0; out && i < std::min(n, capacity); ++i) {
    out[2 * i] = k[(size_t)i].first;
    out[2 * i + 1] = k[(size_t)i].second;
  }
  return n;
}

int64_t ib_trace_host_events(ib_ctx *c, int64_t *rows, int64_t capacity) {
  if (!c || !c->tracing) return fail(IB_ESTATE, "tracing is not enabled");
  const int64_t n = (int64_t)c->host_ev.size();
  for (int64_t i = 0; rows && i < std::min(n, capacity); ++i) {
    rows[4 * i] = c->host_ev[(size_t)i].t;
    rows[4 * i + 1] = c->host_ev[(size_t)i].kind;
    rows[4 * i + 2] = c->host_ev[(size_t)i].batch;
    rows[4 * i + 3] = c->host_ev[(size_t)i].kernel;
  }
  return n;
}

int ib_flush_l2(ib_ctx *c) {
  IB_TRY(check_ctx(c));
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  if (!c->flush) {
    int dev = c->slabs[0].device, l2 = 0;
    IB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    c->flush_bytes = std::max<size_t>((size_t)l2 * 2, 256u << 20);
    IB_CUDA(cudaMalloc(&c->flush, c->flush_bytes));
  }
  static uint32_t salt = 1;
  const int64_t n16 = (int64_t)(c->flush_bytes / 16);
  ib::k_flush<<<148 * 4, 512, 0, c->stream()>>>((uint4 *)c->flush, n16, salt++);
  IB_CUDA(cudaGetLastError());
  IB_CUDA(cudaStreamSynchronize(c->stream()));
  return IB_OK;
}

}  // extern "C"
