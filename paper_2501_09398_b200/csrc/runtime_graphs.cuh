// runtime_graphs.cuh — stream-mode enqueue, cross-slab / cross-rank ordering, halo exchange, graph construction (manual chain, capture, WHILE node).
// Part of runtime.cu (one translation unit; included in order, not compiled alone).
#pragma once

namespace {

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
                         top, bot, (long long)c->dist_timeout_ms);
  return launch_one(L, st, false);
}
int launch_dist_signal(ib_ctx *c, cudaStream_t st) {
  Launch L = make_launch((const void *)ib::k_dist_signal, dim3(1), dim3(1), 0, c->sync, c->peer_sync_up,
                         c->peer_sync_dn);
  return launch_one(L, st, false);
}

// IB_HALO_COPY: the halo planes a slab's launch would have stored into its
// neighbours, moved by peer copies on the slab's stream right after the launch — cudaMemcpyAsync
// over UVA (peer access is enabled between slab devices; cudaMemcpyPeerAsync cannot be stream-
// captured), memcpy nodes in the graph, before the slab's "done" event, so the same phase edges
// order them. Slab buffers hold one halo plane each side: local plane 0, owned 1..rows, rows+1.
//   hotspot (ping-pong): my first / last owned output plane -> the neighbours' halos, buf[outpar]
//   FDTD H launch (in place): my last plane's H (fields 3..5) -> the next slab's lower halo
//   FDTD E launch (in place): my first plane's E (fields 0..2) -> the previous slab's upper halo
//   fused FDTD (ping-pong): my last plane's E and H -> the next slab's lower halo, my first
//                           plane's E -> the previous slab's upper halo, buf[outpar]
int halo_copies(ib_ctx *c, int g, int outpar, int step, cudaStream_t st) {
  const int P = (int)c->slabs.size();
  Slab &s = c->slabs[g];
  const size_t es = (size_t)c->esize;
  if (c->hotspot()) {
    const size_t pb = (size_t)c->plane() * es;
    const char *b = (const char *)s.buf[outpar];
    if (g > 0) {
      Slab &n = c->slabs[g - 1];
      IB_CUDA(cudaMemcpyAsync((char *)n.buf[outpar] + (size_t)(n.rows() + 1) * pb, b + pb, pb, cudaMemcpyDefault, st));
    }
    if (g + 1 < P) {
      Slab &n = c->slabs[g + 1];
      IB_CUDA(cudaMemcpyAsync(n.buf[outpar], b + (size_t)s.rows() * pb, pb, cudaMemcpyDefault, st));
    }
    return IB_OK;
  }
  const bool fused = c->solver == IB_SOLVER_FDTD_FUSED;
  const int buf = fused ? outpar : 0;
  const size_t pb = (size_t)(c->dims[1] + 1) * (size_t)c->lattice_pitch() * es;  // one field's plane
  auto copy = [&](Slab &n, int64_t nplane, int64_t myplane, int f0, int f1) -> int {
    for (int f = f0; f < f1; ++f)
      IB_CUDA(cudaMemcpyAsync((char *)n.buf[buf] + ((size_t)f * n.fs * es + (size_t)nplane * pb),
                              (const char *)s.buf[buf] + ((size_t)f * s.fs * es + (size_t)myplane * pb), pb,
                              cudaMemcpyDefault, st));
    return IB_OK;
  };
  if (g + 1 < P && (fused || step == 0))  // last plane -> next slab's lower halo (H; fused: E too)
    IB_TRY(copy(c->slabs[g + 1], 0, s.rows(), fused ? 0 : 3, 6));
  if (g > 0 && (fused || step == 1))  // first plane's E -> previous slab's upper halo
    IB_TRY(copy(c->slabs[g - 1], c->slabs[g - 1].rows() + 1, 1, 0, 3));
  return IB_OK;
}
bool copies_halos(const ib_ctx *c) { return c->halo_copy && c->slabs.size() > 1 && !c->dist(); }

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
      if (copies_halos(c)) IB_TRY(halo_copies(c, L.slab, par ^ 1, L.step, st));
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

// IB_FLAG_PATCH: re-point the single executable's kernel nodes so it starts at `parity`.
int patch_exec_parity(ib_ctx *c, int parity) {
  std::vector<Launch> its[2];
  iteration_launches(c, 0, its[0]);
  iteration_launches(c, 1, its[1]);
  const size_t per = its[0].size();
  for (size_t n = 0; n < c->kernel_nodes.size(); ++n) {
    const int64_t t = (int64_t)(n / per);
    Launch &L = its[(parity + t) & 1][n % per];
    cudaKernelNodeParams np = {};
    np.func = const_cast<void *>(L.func);
    np.gridDim = L.grid;
    np.blockDim = L.block;
    np.sharedMemBytes = (unsigned)L.smem;
    np.kernelParams = L.args();
    IB_CUDA(cudaGraphExecKernelNodeSetParams(c->exec[0], c->kernel_nodes[n], &np));
  }
  c->exec_parity = parity;
  return IB_OK;
}

void free_graphs(ib_ctx *c) {
  for (int p = 0; p < 2; ++p) {
    if (c->exec[p]) cudaGraphExecDestroy(c->exec[p]);
    if (c->graph[p]) cudaGraphDestroy(c->graph[p]);
    c->exec[p] = nullptr;
    c->graph[p] = nullptr;
  }
  c->kernel_nodes.clear();
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
      if (c->gflags & IB_FLAG_PATCH) c->kernel_nodes.push_back(node);
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

// Odd K on a ping-pong solver: the WHILE body holds two batches, the second (other start parity)
// inside an IF node. This tick ends the first: it runs the IF body only if batches remain, and
// stops the loop unless the IF body's own tick (k_while_tick) re-arms it.
__global__ void k_while_tick_half(int *counter, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  int left = *counter - 1;
  *counter = left;
  cudaGraphSetConditional(hi, left > 0 ? 1u : 0u);
  cudaGraphSetConditional(hw, 0u);
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
      // An odd K flips a ping-pong solver's parity every batch, and one executable bakes in one
      // start parity: the body then runs batch (parity) and, in an IF node, batch (parity ^ 1).
      const bool two = c->ping_pong() && (c->K & 1);
      int *cnt = c->d_counter;
      cudaGraphConditionalHandle hw = c->cond[parity], hi = {};
      cudaKernelNodeParams np = {};
      np.gridDim = dim3(1);
      np.blockDim = dim3(1);
      cudaGraphNode_t tick;
      if (!two) {
        void *args[2] = {&cnt, &hw};
        np.func = (void *)k_while_tick;
        np.kernelParams = args;
        IB_CUDA(cudaGraphAddKernelNode(&tick, body, &last, 1, &np));
        ++nodes;
      } else {
        IB_CUDA(cudaGraphConditionalHandleCreate(&c->cond_if[parity], g, 0, cudaGraphCondAssignDefault));
        hi = c->cond_if[parity];
        void *args[3] = {&cnt, &hw, &hi};
        np.func = (void *)k_while_tick_half;
        np.kernelParams = args;
        IB_CUDA(cudaGraphAddKernelNode(&tick, body, &last, 1, &np));
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hi;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        IB_CUDA(cudaGraphAddNode(&inode, body, &tick, 1, &ip));
        cudaGraph_t second = ip.conditional.phGraph_out[0];
        cudaGraphNode_t last2 = nullptr;
        IB_TRY(build_manual_chain(c, second, c->K, parity ^ 1, pdl, nullptr, &last2, &nodes));
        void *args2[2] = {&cnt, &hw};
        cudaKernelNodeParams np2 = np;
        np2.func = (void *)k_while_tick;
        np2.kernelParams = args2;
        cudaGraphNode_t tick2;
        IB_CUDA(cudaGraphAddKernelNode(&tick2, second, &last2, 1, &np2));
        nodes += 3;
      }
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
