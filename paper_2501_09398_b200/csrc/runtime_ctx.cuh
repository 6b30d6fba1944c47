// runtime_ctx.cuh — ib_ctx: one solver instance (device fields, slabs, graphs, exchange, tracing).
// Part of runtime.cu (one translation unit; included in order, not compiled alone).
#pragma once

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
  // IB_FLAG_PATCH: the single executable's kernel nodes in chain order, and the start parity its
  // node parameters currently encode
  std::vector<cudaGraphNode_t> kernel_nodes;
  int exec_parity = 0;
  cudaGraphConditionalHandle cond[2] = {};
  cudaGraphConditionalHandle cond_if[2] = {};  // odd-K WHILE: the IF node of the body's second batch
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
  int64_t dist_timeout_ms = 120000;  // k_dist_wait traps after this long (ib_set_dist_timeout)
  // single-process slabs: halo planes by cudaMemcpyPeerAsync after each kernel (IB_HALO_COPY)
  // instead of the kernel's own stores into the neighbours' halos
  bool halo_copy = false;
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
