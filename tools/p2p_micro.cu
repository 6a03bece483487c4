// Diagnostics: NVLink peer bandwidth on this box, kernel-driven — GPU 0
// writing into GPU 1 (push) vs GPU 0 reading from GPU 1 (pull), 16-B
// vector accesses, several bytes-in-flight settings; plus both GPUs pushing
// to each other at once.  Needs 2 GPUs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p2p tools/p2p_micro.cu && /tmp/p2p
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

template <int U>
__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t base = ((size_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n; base += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + (size_t)u * blockDim.x;
      if (i < n) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + (size_t)u * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

template <int U>
float run(const int4* src, int4* dst, size_t n, int grid, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_kernel<U><<<grid, 512, 0, s>>>(src, dst, n);
  cudaEventRecord(a, s);
  for (int r = 0; r < 5; ++r) copy_kernel<U><<<grid, 512, 0, s>>>(src, dst, n);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 512ull << 20, n = bytes / 16;
  int4 *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&a1, bytes));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaMemset(a1, 1, bytes));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  cudaStream_t s1;
  CK(cudaStreamCreate(&s1));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&a0, bytes));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMemset(a0, 1, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0;
  CK(cudaStreamCreate(&s0));
  for (int grid : {148, 296, 592}) {
    float push = run<8>(a0, b1, n, grid, s0);   // local read, remote write
    float pull = run<8>(a1, b0, n, grid, s0);   // remote read, local write
    float pull4 = run<4>(a1, b0, n, grid, s0);
    float pull16 = run<16>(a1, b0, n, grid, s0);
    float local = run<8>(a0, b0, n, grid, s0);
    printf("grid %4d: push %6.1f GB/s  pull(U8) %6.1f  pull(U4) %6.1f  pull(U16) %6.1f  local copy %7.1f GB/s(one way)\n",
           grid, bytes / push / 1e6, bytes / pull / 1e6, bytes / pull4 / 1e6, bytes / pull16 / 1e6,
           bytes / local / 1e6);
  }
  // both directions at once: 0 pushes to 1, 1 pushes to 0
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s0);
    for (int r = 0; r < 5; ++r) copy_kernel<8><<<296, 512, 0, s0>>>(a0, b1, n);
    CK(cudaSetDevice(1));
    for (int r = 0; r < 5; ++r) copy_kernel<8><<<296, 512, 0, s1>>>(a1, b0, n);
    CK(cudaSetDevice(0));
    cudaEventRecord(b, s0);
    cudaEventSynchronize(b);
    cudaStreamSynchronize(s1);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("bidirectional push: %6.1f GB/s per direction (GPU0 view)\n", bytes / (ms / 5) / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
