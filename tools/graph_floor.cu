// Diagnostics: the floor under the bench's LL step — a CUDA graph of S steps,
// each [256 MB memset (L2 flush), 1-CTA kernel (the untimed barrier), event,
// kernel A (148 x 512), kernel B (148 x 512), event], timed between the two
// in-graph events like bench.py does.  A/B are empty, or do one dependent
// global load each; B optionally launched with programmatic dependent launch
// (PDL: B's CTAs start while A drains; B waits with griddepcontrol.wait).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gf tools/graph_floor.cu && /tmp/gf
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));                \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void k_barrier(int* p) {
  if (threadIdx.x == 0) p[1] += 1;
}

template <bool LOAD, bool PDL_WAIT, bool TRIGGER>
__global__ void __launch_bounds__(512) k_step(const int* q, int* p) {
  if (TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (PDL_WAIT) asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int v;
  if (LOAD) {
    if (threadIdx.x == 0) v = *(volatile const int*)(q + blockIdx.x * 64);
    __syncthreads();
    if (v == 12345) p[0] = 1;
  } else if (p && threadIdx.x == 1023) {
    p[0] = 1;
  }
}

template <class FA, class FB>
int run(const char* name, FA a, FB b, cudaStream_t st, char* flush, int* d) {
  const int S = 10;
  std::vector<cudaEvent_t> ev(2 * S);
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDefault));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < S; ++i) {
    cudaMemsetAsync(flush, i, 256u << 20, st);
    k_barrier<<<1, 64, 0, st>>>(d);
    cudaEventRecordWithFlags(ev[2 * i], st, cudaEventRecordExternal);
    a(st);
    b(st);
    cudaEventRecordWithFlags(ev[2 * i + 1], st, cudaEventRecordExternal);
  }
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  double sum = 0;
  int n = 0;
  for (int r = 0; r < 12; ++r) {
    CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    if (r < 2) continue;
    for (int i = 0; i < S; ++i) {
      float ms;
      cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]);
      sum += ms;
      ++n;
    }
  }
  printf("%-44s step (event to event): %6.2f us\n", name, 1e3 * sum / n);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return 0;
}

template <class K>
void launch_pdl(K kern, cudaStream_t s, const int* q, int* p) {
  cudaLaunchConfig_t c = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.gridDim = 148;
  c.blockDim = 512;
  c.stream = s;
  c.attrs = at;
  c.numAttrs = 1;
  cudaLaunchKernelEx(&c, kern, q, p);
}

int main() {
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  int* d;
  CK(cudaMalloc(&d, 4 << 20));
  CK(cudaMemset(d, 0, 4 << 20));
  char* flush;
  CK(cudaMalloc(&flush, 256u << 20));
  const int* q = d + 4096;
  run("empty A + empty B", [&](cudaStream_t s) { k_step<false, false, false><<<148, 512, 0, s>>>(q, d); },
      [&](cudaStream_t s) { k_step<false, false, false><<<148, 512, 0, s>>>(q, d); }, st, flush, d);
  run("load A + load B", [&](cudaStream_t s) { k_step<true, false, false><<<148, 512, 0, s>>>(q, d); },
      [&](cudaStream_t s) { k_step<true, false, false><<<148, 512, 0, s>>>(q, d); }, st, flush, d);
  run("load A + load B (PDL, B waits)", [&](cudaStream_t s) { k_step<true, false, false><<<148, 512, 0, s>>>(q, d); },
      [&](cudaStream_t s) { launch_pdl(k_step<true, true, false>, s, q, d); }, st, flush, d);
  run("load A (early trigger) + load B (PDL, waits)",
      [&](cudaStream_t s) { k_step<true, false, true><<<148, 512, 0, s>>>(q, d); },
      [&](cudaStream_t s) { launch_pdl(k_step<true, true, false>, s, q, d); }, st, flush, d);
  run("load A only", [&](cudaStream_t s) { k_step<true, false, false><<<148, 512, 0, s>>>(q, d); },
      [&](cudaStream_t s) {}, st, flush, d);
  run("nothing between the events", [&](cudaStream_t s) {}, [&](cudaStream_t s) {}, st, flush, d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
