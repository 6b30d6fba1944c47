// L2 bandwidth on B200 for an L2-resident working set (diagnostic, not product): is a one-wave
// Hotspot2D launch (12.6 MB of algorithmic traffic, ~16 MB through L1/L2) bound by L2 bandwidth
// or by latency? (a) steady state: one long kernel re-reading an L2-resident buffer many times
// (no launch overhead); (b) per launch: K PDL-chained launches of a 16-byte/thread read of the
// buffer, grid = n/256 CTAs; (c) the same with R float4 per thread (fewer CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/microbench_l2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_steady(const float4 *__restrict__ a, float4 *__restrict__ out, int n, int passes) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = 0; p < passes; ++p)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      float4 v = __ldcg(a + i);  // L2 (bypass L1)
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x == 12345.f) out[0] = acc;
}
template <int R>
__global__ void k_read(const float4 *__restrict__ a, float4 *__restrict__ out, int n) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int base = blockIdx.x * blockDim.x * R + threadIdx.x;
  float4 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = a[base + r * blockDim.x];
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r) s += v[r].x + v[r].y + v[r].z + v[r].w;
  if (s == 12345.f) out[0] = v[0];
}
template <int R>
__global__ void k_copy(const float4 *__restrict__ a, float4 *__restrict__ b, int n) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int base = blockIdx.x * blockDim.x * R + threadIdx.x;
  float4 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = a[base + r * blockDim.x];
#pragma unroll
  for (int r = 0; r < R; ++r) b[base + r * blockDim.x] = v[r];
}

template <typename F>
static float per_launch(cudaStream_t s, F launch, int K, int reps) {
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < K; ++k) launch(k);
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
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  return 1000.f * ms / (reps * K);
}

int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  float4 *a, *b;
  const int nmax = 64 << 20 >> 4;  // 64 MB
  cudaMalloc(&a, nmax * 16); cudaMalloc(&b, nmax * 16);
  cudaMemset(a, 0, nmax * 16); cudaMemset(b, 0, nmax * 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mb : {4, 8, 16, 32}) {
    const int n = (mb << 20) >> 4;
    for (int ctas_per_sm : {2, 4, 8}) {
      const int passes = 200;
      k_steady<<<sms * ctas_per_sm, 256, 0, s>>>(a, b, n, 2);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      k_steady<<<sms * ctas_per_sm, 256, 0, s>>>(a, b, n, passes);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("steady  %2d MB  %4d x 256   %.2f TB/s\n", mb, sms * ctas_per_sm,
             (double)n * 16 * passes / (ms * 1e-3) / 1e12);
    }
  }
  const int K = 100, reps = 20;
  auto attr_launch = [&](int k, void *fn, dim3 grid, dim3 block, void **args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = k > 0 ? 1 : 0;
    cudaLaunchKernelExC(&cfg, fn, args);
  };
  for (int mb : {4, 8, 16}) {
    int n = (mb << 20) >> 4;
    for (int block : {256, 512, 1024}) {
      void *fr[3] = {(void *)k_read<1>, (void *)k_read<2>, (void *)k_read<4>};
      void *fc[3] = {(void *)k_copy<1>, (void *)k_copy<2>, (void *)k_copy<4>};
      for (int ri = 0; ri < 3; ++ri) {
        const int R = 1 << ri;
        dim3 grid(n / (block * R));
        float tr = per_launch(s, [&](int k) {
          const float4 *src = a; float4 *dst = b; int nn = n;
          void *args[3] = {&src, &dst, &nn};
          attr_launch(k, fr[ri], grid, dim3(block), args);
        }, K, reps);
        float tc = per_launch(s, [&](int k) {
          const float4 *src = (k & 1) ? b : a; float4 *dst = (k & 1) ? a : b; int nn = n;
          void *args[3] = {&src, &dst, &nn};
          attr_launch(k, fc[ri], grid, dim3(block), args);
        }, K, reps);
        printf("launch  %2d MB  %5d x %4d R=%d   read %.3f us (%.2f TB/s)   copy %.3f us (%.2f TB/s)\n",
               mb, grid.x, block, R, tr, (double)n * 16 / (tr * 1e-6) / 1e12, tc,
               2.0 * n * 16 / (tc * 1e-6) / 1e12);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
