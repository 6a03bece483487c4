// Diagnostics: per-kernel cost of back-to-back launches inside one CUDA graph,
// for kernel shapes like the LL kernels (148 x 512, cooperative attribute,
// dynamic shared memory, cold instruction/L2 cache after a flush).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lo tools/launch_overhead.cu -lcuda && /tmp/lo
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 1023) p[0] = 1;
}

__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && s[0] == 1) p[0] = 1;
}

__global__ void k_load(const int* q, int* p) {
  __shared__ int v;
  if (threadIdx.x == 0) v = *(volatile const int*)q;
  __syncthreads();
  if (v == 12345) p[0] = 1;
}

// large straight-line code: cold i-cache after an L2 flush
__global__ void k_bigcode(float* p, float a) {
  float x = threadIdx.x;
#pragma unroll
  for (int i = 0; i < 6000; ++i) x = x * a + (float)(i & 7);
  if (x == 1.2345f) p[0] = x;
}

template <class F>
float time_graph(const char* name, F launch, int per, cudaStream_t st, char* flush, size_t fb, int reps) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < per; ++i) launch(st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f, sum = 0.f;
  for (int r = 0; r < reps + 2; ++r) {
    if (flush) cudaMemsetAsync(flush, r & 0xFF, fb, st);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) { sum += ms; if (ms < best) best = ms; }
  }
  printf("%-34s %s per kernel: mean %7.2f us  best %7.2f us\n", name, flush ? "flushed" : "warm   ",
         1e3f * sum / reps / per, 1e3f * best / per);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best;
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int* d;
  CK(cudaMalloc(&d, 1 << 20));
  CK(cudaMemset(d, 0, 1 << 20));
  size_t fb = 256u << 20;
  char* flush;
  CK(cudaMalloc(&flush, fb));
  CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
  const int reps = 20;
  for (int f = 0; f < 2; ++f) {
    char* fl = f ? flush : nullptr;
    for (int per : {1, 10}) {
      printf("-- %d kernel(s) per graph\n", per);
      time_graph("empty 1x32", [&](cudaStream_t s) { k_empty<<<1, 32, 0, s>>>(d); }, per, st, fl, fb, reps);
      time_graph("empty 148x512", [&](cudaStream_t s) { k_empty<<<148, 512, 0, s>>>(d); }, per, st, fl, fb, reps);
      time_graph("empty 296x512", [&](cudaStream_t s) { k_empty<<<296, 512, 0, s>>>(d); }, per, st, fl, fb, reps);
      time_graph("empty 148x512 coop", [&](cudaStream_t s) {
        cudaLaunchConfig_t c = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        c.gridDim = 148; c.blockDim = 512; c.stream = s; c.attrs = at; c.numAttrs = 1;
        cudaLaunchKernelEx(&c, k_empty, d);
      }, per, st, fl, fb, reps);
      time_graph("smem 10KB 148x512", [&](cudaStream_t s) { k_smem<<<148, 512, 10 << 10, s>>>(d); }, per, st, fl, fb, reps);
      time_graph("smem 60KB 148x512", [&](cudaStream_t s) { k_smem<<<148, 512, 60 << 10, s>>>(d); }, per, st, fl, fb, reps);
      time_graph("alt smem 10/60KB 148x512", [&](cudaStream_t s) {
        static int i = 0;
        k_smem<<<148, 512, ((i++ & 1) ? 60 : 10) << 10, s>>>(d);
      }, per, st, fl, fb, reps);
      time_graph("one load 148x512", [&](cudaStream_t s) { k_load<<<148, 512, 0, s>>>(d + 1000, d); }, per, st, fl, fb, reps);
      time_graph("bigcode 148x512", [&](cudaStream_t s) { k_bigcode<<<148, 512, 0, s>>>((float*)d, 1.0001f); }, per, st, fl, fb, reps);
    }
  }
  return 0;
}
