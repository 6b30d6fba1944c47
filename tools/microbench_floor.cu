// Floor of a one-wave per-iteration kernel in a CUDA graph on B200 (diagnostic, not product):
// K back-to-back launches of (a) an empty kernel, (b) a 16-byte-per-thread read, (c) a read +
// write (copy), (d) three row reads + power + write (the Hotspot2D access pattern without the
// arithmetic), all with Hotspot2D 1024^2's grid (1024 x 256 threads, 4 floats each), captured with
// programmatic edges, ping-pong buffers L2-resident. Prints device us per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/floor tools/microbench_floor.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void pdl() {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__global__ void k_empty(const float4 *, float4 *, const float4 *, int) { pdl(); }
__global__ void k_read(const float4 *a, float4 *b, const float4 *, int n) {
  pdl();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float4 v = a[i];
  if (v.x == 12345.f) b[i] = v;  // keep the load
}
__global__ void k_copy(const float4 *a, float4 *b, const float4 *, int n) {
  pdl();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  b[i] = a[i];
}
__global__ void k_rows(const float4 *a, float4 *b, const float4 *p, int n) {
  pdl();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = 256;  // float4 per 1024-float row
  int up = i >= row ? i - row : i, dn = i + row < n ? i + row : i;
  float4 x = a[up], c = a[i], y = a[dn], q = p[i];
  b[i] = make_float4(x.x + c.x + y.x + q.x, x.y + c.y + y.y + q.y, x.z + c.z + y.z + q.z, x.w + c.w + y.w + q.w);
}

__global__ void k_scale(const float4 *a, float4 *b, const float4 *, int n) {
  pdl();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float4 v = a[i];
  const double c = 0.9999;
  b[i] = make_float4((float)(v.x * c), (float)(v.y * c), (float)(v.z * c), (float)(v.w * c));
}

// binary64 Hotspot2D 1024^2 pattern: double2 per thread (512 per 1024-double row), three row reads
// + power + write; RB rows per thread (RB+2 row reads for RB outputs)
template <int RB>
__global__ void k_rows64(const double2 *a, double2 *b, const double2 *p, int n) {
  pdl();
  const int row = 512, i0 = (blockIdx.x * blockDim.x + threadIdx.x);
  const int x = i0 % row, r0 = (i0 / row) * RB;
  double2 v[RB + 2];
#pragma unroll
  for (int q = 0; q < RB + 2; ++q) {
    int r = r0 - 1 + q;
    r = r < 0 ? 0 : (r > 1023 ? 1023 : r);
    v[q] = a[r * row + x];
  }
#pragma unroll
  for (int q = 0; q < RB; ++q) {
    const double2 w = p[(r0 + q) * row + x];
    b[(r0 + q) * row + x] = make_double2(v[q].x + v[q + 1].x + v[q + 2].x + w.x, v[q].y + v[q + 1].y + v[q + 2].y + w.y);
  }
}

int main() {
  const int n = 1024 * 1024 / 4, K = 100, reps = 20;
  float4 *a, *b, *p;
  cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&p, n * 16);
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16); cudaMemset(p, 0, n * 16);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void (*fns[4])(const float4 *, float4 *, const float4 *, int) = {k_empty, k_read, k_copy, k_rows};
  const char *names[4] = {"empty", "read 16B/thread", "copy", "3 rows + power + write"};
  for (int f = 0; f < 4; ++f) {
    for (int pdlon = 0; pdlon < 2; ++pdlon) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n / 256); cfg.blockDim = dim3(256); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = (pdlon && k > 0) ? 1 : 0;
        const float4 *src = (k & 1) ? b : a; float4 *dst = (k & 1) ? a : b;
        cudaLaunchKernelEx(&cfg, fns[f], src, dst, (const float4 *)p, n);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphUpload(ge, s);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-26s pdl=%d  %.3f us/launch\n", names[f], pdlon, 1000.f * ms / (reps * K));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  // empty-kernel floor vs grid shape (same thread count where possible)
  const int shapes[][2] = {{1024, 256}, {512, 512}, {256, 512}, {128, 1024}, {256, 1024}, {2048, 128}, {148, 1024}, {32, 128}, {1, 32}};
  for (auto sh : shapes) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sh[0]); cfg.blockDim = dim3(sh[1]); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = k > 0 ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_empty, (const float4 *)a, b, (const float4 *)p, n);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphUpload(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty grid %5d x %4d    pdl=1  %.3f us/launch\n", sh[0], sh[1], 1000.f * ms / (reps * K));
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  }
  // the skeleton's shape: 2^14 floats, 32 x 128 threads, one float4 each, in place
  {
    const int ns = 4096;
    const char *sn[4] = {"small empty", "small read", "small copy in place", "small scale (f64 mul) in place"};
    void (*sf[4])(const float4 *, float4 *, const float4 *, int) = {k_empty, k_read, k_copy, k_scale};
    for (int f = 0; f < 4; ++f) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ns / 128); cfg.blockDim = dim3(128); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = k > 0 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, sf[f], (const float4 *)a, a, (const float4 *)p, ns);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphUpload(ge, s);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-32s pdl=1  %.3f us/launch\n", sn[f], 1000.f * ms / (reps * K));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  // binary64 Hotspot2D 1024^2 access pattern (no arithmetic beyond the adds): the floor the
  // binary64 k_hotspot_vec runs against
  {
    const int n2 = 1024 * 1024 / 2;
    double2 *a2, *b2, *p2;
    cudaMalloc(&a2, n2 * 16); cudaMalloc(&b2, n2 * 16); cudaMalloc(&p2, n2 * 16);
    cudaMemset(a2, 0, n2 * 16); cudaMemset(b2, 0, n2 * 16); cudaMemset(p2, 0, n2 * 16);
    struct { const char *name; void (*fn)(const double2 *, double2 *, const double2 *, int); int rb, block; } v[] = {
        {"f64 3 rows + power + write, R=1, 256 thr", k_rows64<1>, 1, 256},
        {"f64 3 rows + power + write, R=1, 512 thr", k_rows64<1>, 1, 512},
        {"f64 4 rows + 2 power + 2 writes, R=2, 256", k_rows64<2>, 2, 256},
        {"f64 R=2, 512 thr", k_rows64<2>, 2, 512},
        {"f64 R=4, 256 thr", k_rows64<4>, 4, 256},
        {"f64 R=4, 128 thr", k_rows64<4>, 4, 128}};
    for (auto &c : v) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n2 / c.rb / c.block); cfg.blockDim = dim3(c.block); cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = k > 0 ? 1 : 0;
        const double2 *src = (k & 1) ? b2 : a2; double2 *dst = (k & 1) ? a2 : b2;
        cudaLaunchKernelEx(&cfg, c.fn, src, dst, (const double2 *)p2, n2);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphUpload(ge, s);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-44s pdl=1  %.3f us/launch\n", c.name, 1000.f * ms / (reps * K));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
