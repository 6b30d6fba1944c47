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

#include "runtime_core.cuh"
#include "runtime_ctx.cuh"
#include "runtime_launches.cuh"
#include "runtime_graphs.cuh"

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
  if (P > 1 && !hot && !c->fdtd())
    return fail(IB_EINVAL, "multi-slab execution is defined for the hotspot and FDTD solvers");
  // axis-0 slabs: hotspot rows, or the FDTD lattice's nx+1 planes
  const int64_t rows = hot ? c->dims[0] : (c->fdtd() && (P > 1 || c->nranks > 1) ? c->dims[0] + 1 : 1);
  if (P > rows) return fail(IB_EINVAL, "more slabs than rows along axis 0");
  c->slabs.resize(P);
  const bool dist = c->nranks > 1;
  if (dist && (P != 1 || !(hot || c->fdtd())))
    return fail(IB_EINVAL, "distributed contexts are single-slab hotspot or FDTD grids");
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
    if (P > 1 || dist) {  // slabs / ranks: planes [lo, hi) plus one halo plane each side; the
      // two half-steps update one copy in place, the fused leapfrog ping-pongs two
      if (lf_config(c).tj == 0)
        return fail(IB_EINVAL, "fdtd slabs need the staged kernel: the z rows are too long for one CTA");
      const int64_t plane = (ny + 1) * c->lat_pitch;
      for (Slab &s : c->slabs) {
        IB_CUDA(cudaSetDevice(s.device));
        s.fs = (int64_t)(s.rows() + 2) * plane;
        const size_t bb = (size_t)(6 * s.fs * es);
        for (int p = 0; p < (fused ? 2 : 1); ++p) {
          IB_CUDA(cudaMalloc(&s.buf[p], bb));
          IB_CUDA(cudaMemset(s.buf[p], 0, bb));
        }
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
  c->dist_timeout_ms = std::max<int64_t>(1, env_int("IB_DIST_TIMEOUT_MS", 120000));
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
  if (solver == IB_SOLVER_VECTOR)
    return fail(IB_EINVAL, "distributed contexts are defined for hotspot grids and FDTD");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(IB_EINVAL, "bad rank / nranks");
  if ((solver == IB_SOLVER_FDTD || solver == IB_SOLVER_FDTD_FUSED) && nranks > 1 && id128)
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
    for (int p = 0; p < (c->solver == IB_SOLVER_FDTD ? 1 : 2); ++p)  // in-place FDTD: one lattice
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

int ib_set_dist_timeout(ib_ctx *c, int64_t ms) {
  IB_TRY(check_ctx(c));
  if (ms <= 0) return fail(IB_EINVAL, "the wait timeout must be > 0 ms");
  c->dist_timeout_ms = ms;
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

int64_t ib_describe(ib_ctx *c, char *buf, int64_t cap) {
  IB_TRY(check_ctx(c));
  DeviceGuard guard;
  IB_CUDA(cudaSetDevice(c->slabs[0].device));
  std::vector<Launch> v;
  iteration_launches(c, c->cur, v);
  std::string js = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    const Launch &L = v[i];
    const char *name = nullptr;
    if (cudaFuncGetName(&name, L.func) != cudaSuccess || !name) {
      cudaGetLastError();
      name = "?";
    }
    char row[640];
    std::snprintf(row, sizeof(row),
                  "%s{\"kernel\": \"%s\", \"grid\": [%u, %u, %u], \"block\": [%u, %u, %u], "
                  "\"smem\": %zu, \"slab\": %d, \"step\": %d}",
                  i ? ", " : "", name, L.grid.x, L.grid.y, L.grid.z, L.block.x, L.block.y, L.block.z,
                  L.smem, L.slab, L.step);
    js += row;
    if (copies_halos(c)) {  // IB_HALO_COPY: the peer copies that follow this launch
      const int P = (int)c->slabs.size();
      const int up = L.slab > 0, dn = L.slab + 1 < P;  // neighbours above / below
      const int n = c->hotspot() ? up + dn
                    : c->solver == IB_SOLVER_FDTD_FUSED ? 6 * dn + 3 * up
                    : (L.step == 0 ? 3 * dn : 3 * up);  // H: H fields down, E: E fields up
      std::snprintf(row, sizeof(row), ", {\"memcpy_nodes\": %d, \"slab\": %d, \"step\": %d}", n, L.slab, L.step);
      js += row;
    }
  }
  js += "]";
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>((size_t)cap - 1, js.size());
    std::memcpy(buf, js.data(), n);
    buf[n] = 0;
  }
  return (int64_t)js.size() + 1;
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
      char *dbase = (char *)s.buf[c->cur] + (size_t)(field * s.fs + (lo - s.row_lo + 1) * plane) * es;
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
    if (copies_halos(c)) IB_TRY(halo_copies(c, L.slab, c->cur ^ 1, L.step, s.stream));
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

int ib_set_halo_mode(ib_ctx *c, int mode) {
  IB_TRY(check_ctx(c));
  if (mode != IB_HALO_STORE && mode != IB_HALO_COPY)
    return fail(IB_EINVAL, "halo mode must be IB_HALO_STORE or IB_HALO_COPY");
  if (mode == IB_HALO_COPY && c->dist())
    return fail(IB_EINVAL, "IB_HALO_COPY applies to single-process slabs (ranks exchange by peer stores or NCCL)");
  if (c->halo_copy != (mode == IB_HALO_COPY)) {
    DeviceGuard guard;
    IB_CUDA(cudaSetDevice(c->slabs[0].device));
    IB_TRY(sync_all(c));
    free_graphs(c);  // the built graphs embed the other exchange
  }
  c->halo_copy = mode == IB_HALO_COPY;
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
  const bool patch = (flags & IB_FLAG_PATCH) != 0;
  if (patch && (build_mode != IB_BUILD_MANUAL || c->slabs.size() > 1 || c->dist() || (flags & IB_FLAG_WHILE)))
    return fail(IB_EINVAL, "IB_FLAG_PATCH needs a manual build on one slab, without IB_FLAG_WHILE");
  int rc;
  if (patch) {  // one executable (in exec[0]) built at the current parity, re-pointed as needed
    rc = build_one(c, c->cur, &t);
    if (rc == IB_OK && c->cur != 0) {
      c->exec[0] = c->exec[c->cur];
      c->graph[0] = c->graph[c->cur];
      c->exec[c->cur] = nullptr;
      c->graph[c->cur] = nullptr;
    }
    c->exec_parity = c->cur;
  } else {
    rc = build_one(c, c->cur, &t);
    if (rc == IB_OK && c->ping_pong() && (batch_size & 1)) rc = build_one(c, c->cur ^ 1, &t);
  }
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
  const bool patch = (c->gflags & IB_FLAG_PATCH) != 0;
  // the state parity may have moved since the build (e.g. an odd stream run): build lazily
  if (!patch && !c->exec[c->cur]) IB_TRY(build_one(c, c->cur, &t));
  if (!patch && c->ping_pong() && (c->K & 1) && !c->exec[c->cur ^ 1]) IB_TRY(build_one(c, c->cur ^ 1, &t));
  const bool wh = (c->gflags & IB_FLAG_WHILE) != 0;
  const int64_t per = c->K * (c->solver == IB_SOLVER_FDTD ? 2 : 1) * (int64_t)c->slabs.size();  // kernels / batch
  auto a = clk::now();
  IB_CUDA(cudaEventRecord(c->t0, c->stream()));
  if (num_batches > 0) {
    if (wh) {
      if (num_batches > INT32_MAX) return fail(IB_EINVAL, "IB_FLAG_WHILE: num_batches must fit the device counter");
      int nb = (int)num_batches;
      IB_CUDA(cudaMemcpyAsync(c->d_counter, &nb, sizeof(int), cudaMemcpyHostToDevice, c->stream()));
      c->ev(IB_EV_GRAPH_LAUNCHED, 0);
      IB_CUDA(cudaGraphLaunch(c->exec[c->cur], c->stream()));
      t.launches = 1;
      if (c->ping_pong() && (c->K & 1) && (num_batches & 1)) c->cur ^= 1;
    } else {
      for (int64_t b = 0; b < num_batches; ++b) {
        c->ev(IB_EV_GRAPH_LAUNCHED, b);
        if (patch) {
          if (c->ping_pong() && c->exec_parity != c->cur) IB_TRY(patch_exec_parity(c, c->cur));
          IB_CUDA(cudaGraphLaunch(c->exec[0], c->stream()));
        } else {
          IB_CUDA(cudaGraphLaunch(c->exec[c->cur], c->stream()));
        }
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
