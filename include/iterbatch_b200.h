/*
 * iterbatch_b200.h — C ABI of the B200-native iteration-batching runtime.
 *
 * Drop-in boundary for the reference's solver API (Python, pkg/src/iterbatch/workloads.py).
 * The reference has no FFI: its plugin point is the step protocol
 *   step(state, workers) -> state                       (workloads.py:97,167,325,358)
 * driven by
 *   run_loop(program, state, total_iterations)          (workloads.py:442-450, Listing 1)
 *   run_batched(program, state, batch_size, num_batches)(workloads.py:453-471, Listings 2/3)
 *   time_workload(program, state, plan, order, repeats) (workloads.py:479-505)
 *   state_checksum(state)                               (workloads.py:508-525)
 * This library replaces the body of those calls with a per-RUN boundary (not per step):
 * upload once, launch N kernels (stream mode) or I graph launches of a K-iteration unrolled
 * CUDA graph (graph mode), download once. The Python mirror in
 * paper_2501_09398_b200/workloads.py binds these entry points with ctypes; see INTEGRATION.md.
 *
 * Conventions: every int-returning call returns IB_OK (0) or a negative IB_E* status; the
 * message for the last failure on the calling thread is ib_last_error(). No torch types,
 * plain pointers and sizes only. One context = one solver instance; not thread-safe.
 */
#ifndef ITERBATCH_B200_H
#define ITERBATCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IB_ABI_VERSION 1

/* status codes (the Python shim maps them to the reference's exception types) */
#define IB_OK 0
#define IB_EINVAL (-1)  /* bad argument            -> ValueError   (workloads.py:444-446,463-466) */
#define IB_ECUDA (-2)   /* CUDA runtime failure    -> RuntimeError */
#define IB_ENOMEM (-3)  /* device/host allocation  -> MemoryError  */
#define IB_ESTATE (-4)  /* call out of order (run before build, ...) -> RuntimeError */
#define IB_ENODEV (-5)  /* no CUDA device          -> RuntimeError (never a CPU fallback) */

/* solver families: one per reference step program (workloads.py:429-439, cli.py:202-207) */
#define IB_SOLVER_VECTOR 0    /* vector_scale_step  workloads.py:97-105  ; 1 kernel / iteration */
#define IB_SOLVER_HOTSPOT2D 1 /* hotspot_step 2-D   workloads.py:180-185 ; 1 kernel / iteration */
#define IB_SOLVER_HOTSPOT3D 2 /* hotspot_step 3-D   workloads.py:186-204 ; 1 kernel / iteration */
#define IB_SOLVER_FDTD 3      /* fdtd_h_step + fdtd_e_step workloads.py:325-413 ; 2 kernels / it. */
#define IB_SOLVER_FDTD_FUSED 4 /* the same leapfrog as ONE kernel per iteration (H then E fused, fields
                                  double-buffered: each field read and written once per iteration) */

/* arithmetic type of the device state */
#define IB_F32 0
#define IB_F64 1

/* graph construction (stream capture vs manual creation) */
#define IB_BUILD_MANUAL 0  /* cudaGraphCreate + cudaGraphAddKernelNode chain (Listing 3) */
#define IB_BUILD_CAPTURE 1 /* cudaStreamBeginCapture over the stream-mode launch sequence */

/* flags for ib_graph_build / ib_run_stream */
#define IB_FLAG_PDL 0x1           /* programmatic dependent launch edges between consecutive kernels */
#define IB_FLAG_DEVICE_LAUNCH 0x2 /* instantiate with cudaGraphInstantiateFlagDeviceLaunch (Listing 3) */
#define IB_FLAG_NO_UPLOAD 0x4     /* skip cudaGraphUpload (first launch pays the upload) */
#define IB_FLAG_WHILE 0x8         /* wrap the K-chain in a conditional WHILE node: one cudaGraphLaunch
                                     runs all num_batches batches (device-side loop, no host gap);
                                     an odd K on a ping-pong solver puts two batches in the body, the
                                     second (other buffer parity) inside an IF node */
#define IB_FLAG_MEMINFO 0x10      /* fill ib_times.graph_bytes from cudaMemGetInfo before/after the
                                     build (the paper's m_base/m_node probe; costs ~ms per call) */
#define IB_FLAG_PATCH 0x20        /* odd batch_size on a ping-pong solver: ONE executable whose kernel
                                     nodes are re-pointed (cudaGraphExecKernelNodeSetParams) before a
                                     launch that starts on the other buffer parity, instead of a second
                                     executable with the parity baked in (manual builds, one slab) */

/* Per-call timing record. Host times are steady-clock seconds; gpu_s is CUDA-event time on the
 * context's launch stream (first launch .. end of last kernel). */
typedef struct ib_times {
  double create_s;      /* graph create + node add (or capture) */
  double instantiate_s; /* cudaGraphInstantiate */
  double upload_s;      /* cudaGraphUpload + sync */
  double build_s;       /* T_C = create + instantiate + upload (Eq. 2) */
  double exec_s;        /* T_E host wall: first launch call .. stream synchronized (Eq. 3) */
  double gpu_s;         /* T_E on the device (CUDA events) */
  int64_t kernels;      /* kernels executed by the call */
  int64_t launches;     /* host launch API calls issued (kernel or graph launches) */
  int64_t nodes;        /* nodes in the built graph (build only) */
  int64_t graph_bytes;  /* device memory attributed to the instantiated+uploaded graph(s) */
} ib_times;

typedef struct ib_ctx ib_ctx;

/* ---- library / device --------------------------------------------------------------------- */
int ib_abi_version(void);
const char *ib_last_error(void);
int ib_device_count(int *count);
/* HBM bytes free/total on a device (used for the paper's memory model m_base/m_node). */
int ib_mem_info(int device, int64_t *free_bytes, int64_t *total_bytes);

/* ---- context -------------------------------------------------------------------------------
 * dims:    vector (N) ; hotspot2d (R, C) ; hotspot3d (R, C, L) ; fdtd (nx, ny, nz) cells.
 * scalars: vector  [c]              (VectorWorkload.scale_constant, workloads.py:77)
 *          hotspot [k]              (HotspotWorkload.diffusion_coefficient, workloads.py:120)
 *          fdtd    [d, c_h, c_e]    (cell_size; dt/mu0; dt/eps0 — workloads.py:327-328,364-365)
 *          Constants are passed in binary64 and rounded ONCE to the state dtype on the host,
 *          except the vector constant in IB_F32 which stays binary64 (v' = (float)((double)v*c)).
 * devices: one entry per slab; hotspot solvers partition axis 0 into ndevices slabs with the
 *          reference's bounds formula rows*g//P (workloads.py:65), IB_SOLVER_FDTD partitions the
 *          (nx+1)-plane lattice the same way. Each slab's kernel stores its boundary plane(s)
 *          straight into the neighbours' halo planes (peer pointers between devices); cross-slab
 *          ordering is graph edges. Device ids may repeat (several slabs on one GPU, same graph).
 *          Both FDTD solvers shard (the fused one ping-pongs each slab's planes). vector requires
 *          ndevices == 1. NULL/0 means {current device}.
 * Device layout: vector and hotspot fields are C-order like the reference's arrays; both FDTD
 *          solvers keep the six fields on one padded (nx+1) x (ny+1) x P lattice (P = nz+1
 *          rounded up to 16 bytes), converted by ib_upload / ib_download.
 */
int ib_create(ib_ctx **out, int solver, int dtype, const int64_t *dims, int ndims,
              const double *scalars, int nscalars, const int *devices, int ndevices);
void ib_destroy(ib_ctx *ctx);

/* Halo exchange of a multi-slab context (ib_create with ndevices > 1), SURVEY.md §8e:
 * IB_HALO_STORE (default, v2) — each slab's kernel stores its boundary planes straight into the
 * neighbours' halo planes; IB_HALO_COPY (v1) — the kernels write only their own slab and peer
 * cudaMemcpyAsync (UVA) copies of those planes follow each launch on the slab's stream (memcpy
 * nodes in the captured graph; FDTD: the H / E / fused planes each neighbour reads). Same results
 * bit for bit. Drops any built graph. EINVAL for distributed (ib_create_dist) contexts.
 * Single-slab contexts accept either and ignore it. */
#define IB_HALO_STORE 0
#define IB_HALO_COPY 1
int ib_set_halo_mode(ib_ctx *ctx, int mode);

/* Fields, in the reference's state_arrays() order (workloads.py:93,163,272):
 * vector: 0 values ; hotspot: 0 temperature, 1 power ; fdtd: 0 ex 1 ey 2 ez 3 hx 4 hy 5 hz.
 * Host buffers are C-contiguous in the context dtype; bytes must equal the full field size. */
int ib_num_fields(const ib_ctx *ctx);
int ib_field_shape(const ib_ctx *ctx, int field, int64_t *shape3, int *ndim);
int64_t ib_field_bytes(const ib_ctx *ctx, int field);
int ib_upload(ib_ctx *ctx, int field, const void *host, size_t bytes);
int ib_download(ib_ctx *ctx, int field, void *host, size_t bytes);
/* Bytes one iteration moves by the roofline convention (every array read once, written once). */
int64_t ib_iteration_bytes(const ib_ctx *ctx);
/* The kernels one iteration launches (the variant the runtime chose for this shape and device):
 * a JSON array of {"kernel", "grid", "block", "smem", "slab", "step"} (with IB_HALO_COPY each
 * launch is followed by {"memcpy_nodes", "slab", "step"}: the peer copies after it), NUL-terminated into buf
 * (truncated to cap). Returns the full length including the NUL, or a negative status. */
int64_t ib_describe(ib_ctx *ctx, char *buf, int64_t cap);

/* ---- stream mode: run_loop (Listing 1) ------------------------------------------------------- */
int ib_run_stream(ib_ctx *ctx, int64_t iterations, int flags, ib_times *times);
/* One step of the chain program, for the per-step API (vector_scale_step, hotspot_step,
 * fdtd_h_step = step 0, fdtd_e_step = step 1; workloads.py:97,167,325,358). */
int ib_run_step(ib_ctx *ctx, int step, ib_times *times);
int ib_num_steps(const ib_ctx *ctx);

/* ---- graph mode: run_batched (Listings 2/3) -------------------------------------------------
 * ib_graph_build unrolls batch_size iterations into one graph (2 nodes / iteration for fdtd;
 * P nodes / iteration for P slabs), instantiates and uploads it on the context's non-blocking
 * stream. Ping-pong parity: an even batch_size returns the buffers to their start parity, so one
 * executable is replayed; an odd batch_size gets a second executable with swapped buffers and the
 * two alternate (both are built and counted in T_C).
 * ib_graph_run launches the executable num_batches times (or once, with IB_FLAG_WHILE). */
int ib_graph_build(ib_ctx *ctx, int64_t batch_size, int build_mode, int flags, ib_times *times);
int ib_graph_run(ib_ctx *ctx, int64_t num_batches, ib_times *times);
int ib_graph_destroy(ib_ctx *ctx);
/* run_batched in one call: build (T_C) + num_batches launches (T_E) + destroy. times->gpu_s is
 * the CUDA-event interval from before the build to the end of the last kernel, i.e. the paper's
 * total T = T_C + T_E (Eq. 1) on the device clock; build_s / exec_s split it on the host clock. */
int ib_run_batched(ib_ctx *ctx, int64_t batch_size, int64_t num_batches, int build_mode,
                   int flags, ib_times *times);
/* Loop peeling (the reference rejects non-divisors, model.py:104-108): run
 * total_iterations as floor(N/K) replays of a K-iteration graph plus one graph of the N mod K
 * remainder iterations. Same timing convention as ib_run_batched (both builds inside gpu_s). */
int ib_run_peeled(ib_ctx *ctx, int64_t total_iterations, int64_t batch_size, int build_mode,
                  int flags, ib_times *times);
int64_t ib_graph_batch_size(const ib_ctx *ctx);

/* Device synchronisation of the context's streams. */
int ib_sync(ib_ctx *ctx);

/* ---- pinned host staging (used by the e2e path) -------------------------------------------- */
int ib_host_alloc(void **ptr, size_t bytes);
int ib_host_free(void *ptr);

/* ---- checksum (workloads.py:508-525) ---------------------------------------------------------
 * 64-bit FNV-1a, offset 0xcbf29ce484222325, prime 0x100000001b3, continued from h.
 * ib_fnv1a64_f64 hashes the little-endian binary64 bytes of n values given in the context dtype
 * (float values are widened exactly to binary64 first, as np.ascontiguousarray(a, "<f8") does). */
uint64_t ib_fnv1a64(const void *data, size_t nbytes, uint64_t h);
uint64_t ib_fnv1a64_f64(const void *values, size_t n, int dtype, uint64_t h);

/* ---- multi-process slabs (one process per GPU) -------------------------------
 * A distributed hotspot context owns the axis-0 slab [rows*rank//nranks, rows*(rank+1)//nranks)
 * of a global grid (dims = GLOBAL dims) on `device`, plus one halo plane per interior face. After
 * every iteration's stencil kernel the runtime exchanges boundary planes with rank-1 / rank+1 by
 * NCCL send/recv on the launch stream (libnccl.so.2 is dlopen'ed; graphs are stream-captured, so
 * the exchange is part of the iteration-batch graph). All ranks call ib_create_dist collectively
 * with the same 128-byte id from ib_nccl_unique_id on rank 0 (NCCL exchange), or with id128 =
 * NULL and then ib_ipc_attach (peer exchange, below).
 * For these contexts ib_upload takes the slab WITH its halo rows, i.e. global rows
 * [lo - has_top, hi + has_bot) for the temperature and [lo, hi) for the power; ib_download
 * returns the owned rows [lo, hi). ib_slab_info reports lo, hi, has_top, has_bot.
 * IB_SOLVER_FDTD and IB_SOLVER_FDTD_FUSED (peer exchange only; id128 must be NULL): a rank owns
 * planes [lo, hi) of the (nx+1)-plane lattice;
 * for every field ib_upload takes its global planes [lo - has_top, hi + has_bot) and ib_download
 * returns [lo, hi), both clipped to that field's own extent along axis 0 (nx or nx+1). */
int ib_nccl_unique_id(void *id128);
int ib_create_dist(ib_ctx **out, int solver, int dtype, const int64_t *dims, int ndims,
                   const double *scalars, int nscalars, int device, int rank, int nranks,
                   const void *id128);
int ib_slab_info(const ib_ctx *ctx, int64_t *lo, int64_t *hi, int *has_top, int *has_bot);

/* ---- peer halo exchange across processes (the NVLink-native alternative to NCCL) --------------
 * Create the context with ib_create_dist(..., id128 = NULL) (no NCCL communicator), export this
 * rank's buffers with ib_ipc_export (IB_IPC_BYTES of CUDA IPC handles: both temperature buffers
 * and a small counter block), hand them to the neighbour ranks (any host transport; the Python
 * layer uses torch.distributed), and ib_ipc_attach the handles of rank-1 (up) and rank+1 (down)
 * (NULL where there is none). From then on the stencil kernel stores its first / last owned
 * output plane straight into the neighbours' halo planes (NVLink peer stores); ordering across
 * processes is a pair of one-thread kernels per iteration (wait for the neighbours' completed-
 * iteration counters, publish this rank's), all inside the iteration-batch graph. A lost
 * neighbour traps after the wait timeout instead of hanging the device: ib_set_dist_timeout
 * (milliseconds, > 0; initial value IB_DIST_TIMEOUT_MS, default 120000). It applies to graphs
 * built afterwards (the timeout is a kernel argument baked into the graph's wait nodes).
 * A neighbour's first kernel of a run stores into this rank's halo planes, so the ranks must
 * synchronise (any host barrier) after ib_upload and before the next run; a run itself ends only
 * once the neighbours are done, so downloads need no barrier.
 * Replaces the NCCL group of ib_create_dist(id128 != NULL). SURVEY.md §8e, v2. */
#define IB_IPC_BYTES 192
int ib_ipc_export(const ib_ctx *ctx, void *out, size_t bytes);
int ib_ipc_attach(ib_ctx *ctx, const void *up_handles, const void *down_handles);
int ib_set_dist_timeout(ib_ctx *ctx, int64_t milliseconds);

/* ---- real traces (the reference's EventTrace schema, simulate.py:28-36, fileio.py:48) ---------
 * ib_trace_enable(ctx, capacity > 0) clears and arms tracing; 0 disarms. While armed (single-slab
 * contexts; one traced context per process at a time) CUPTI activity tracing (libcupti, dlopen'ed —
 * the mechanism nsys uses; the kernels carry no instrumentation) records every solver kernel's
 * [start, end] in ns, and the runtime logs host events on the same CUPTI timebase: node added (0),
 * graph instantiated (1), graph uploaded (2), graph launched (3), baseline kernel launched (7),
 * build started (100).
 * ib_trace_kernels returns the number of kernels recorded and copies [start_ns, end_ns] pairs;
 * ib_trace_host_events returns the number of host events and copies (t_ns, kind, batch, kernel). */
#define IB_EV_NODE_ADDED 0
#define IB_EV_GRAPH_INSTANTIATED 1
#define IB_EV_GRAPH_UPLOADED 2
#define IB_EV_GRAPH_LAUNCHED 3
#define IB_EV_BASELINE_KERNEL_LAUNCHED 7
#define IB_EV_BUILD_STARTED 100
int ib_trace_enable(ib_ctx *ctx, int64_t capacity);
int64_t ib_trace_kernels(ib_ctx *ctx, int64_t *start_end_ns, int64_t capacity);
int64_t ib_trace_host_events(ib_ctx *ctx, int64_t *rows4, int64_t capacity);

/* ---- L2 flush helper for benchmark hygiene (writes a buffer larger than L2) ----------------- */
int ib_flush_l2(ib_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* ITERBATCH_B200_H */
