// Diagnostics: all-to-all NVLink bandwidth — every GPU reads (pull) or
// writes (push) an equal share from/to every peer at once, 16-B vector
// accesses, 8 in flight per thread.  The HT dispatch/combine traffic pattern
// without any of the protocol.  Reports remote GB/s per GPU.  2-8 GPUs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/a2a tools/a2a_micro.cu && /tmp/a2a
#include <cstdio>
#include <cstdint>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

struct Peers { int4* p[8]; };

// peer slot q of every GPU holds the bytes destined for GPU q; CTA b works on
// peer (me + 1 + b) % n first so every link is busy from the start
template <bool PULL>
__global__ void a2a_kernel(Peers src, Peers dst, int n, int me, size_t per) {
  const size_t nv = per / 16;
  for (int r = 0; r < n - 1; ++r) {
    const int q = (me + 1 + (blockIdx.x + r) % (n - 1)) % n;
    const int4* s = PULL ? src.p[q] + me * nv : src.p[me] + q * nv;  // pull: peer's slot for me
    int4* d = PULL ? dst.p[me] + q * nv : dst.p[q] + me * nv;        // push: my slot at the peer
    const size_t stride = (size_t)gridDim.x * blockDim.x * 8;
    for (size_t base = (size_t)blockIdx.x * blockDim.x * 8 + threadIdx.x; base < nv; base += stride) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const size_t i = base + (size_t)u * blockDim.x;
        if (i < nv) v[u] = s[i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const size_t i = base + (size_t)u * blockDim.x;
        if (i < nv) d[i] = v[u];
      }
    }
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) { printf("need 2+ GPUs\n"); return 0; }
  if (n > 8) n = 8;
  const size_t per = 256ull << 20;  // bytes per (src, dst) pair
  Peers src{}, dst{};
  std::vector<cudaStream_t> st(n);
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&src.p[g], per * n));
    CK(cudaMalloc(&dst.p[g], per * n));
    CK(cudaMemset(src.p[g], g, per * n));
    CK(cudaStreamCreate(&st[g]));
    for (int h = 0; h < n; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
  }
  for (int mode = 0; mode < 2; ++mode)
    for (int grid : {148, 296}) {
      std::vector<float> ms(n);
      std::vector<std::thread> th;
      for (int g = 0; g < n; ++g)
        th.emplace_back([&, g] {
          cudaSetDevice(g);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          for (int r = 0; r < 2; ++r)
            mode ? a2a_kernel<false><<<grid, 512, 0, st[g]>>>(src, dst, n, g, per)
                 : a2a_kernel<true><<<grid, 512, 0, st[g]>>>(src, dst, n, g, per);
          cudaStreamSynchronize(st[g]);
          cudaEventRecord(a, st[g]);
          for (int r = 0; r < 5; ++r)
            mode ? a2a_kernel<false><<<grid, 512, 0, st[g]>>>(src, dst, n, g, per)
                 : a2a_kernel<true><<<grid, 512, 0, st[g]>>>(src, dst, n, g, per);
          cudaEventRecord(b, st[g]);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms[g], a, b);
        });
      for (auto& t : th) t.join();
      float worst = 0;
      for (float m : ms) worst = worst > m ? worst : m;
      printf("n=%d %s grid %d: remote %.1f GB/s per GPU (slowest GPU)\n", n, mode ? "push" : "pull", grid,
             (double)per * (n - 1) / (worst / 5) / 1e6);
    }
  CK(cudaGetLastError());
  return 0;
}
