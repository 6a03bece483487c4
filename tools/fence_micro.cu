// Diagnostics: cost of the release step of a flag protocol on this system —
// fence.acq_rel.sys vs fence.acq_rel.gpu vs st.release.sys, after a few
// 16-B stores to local memory or to a peer GPU (NVLink), from every CTA.
// Reports the median per-CTA cycles of the release instruction.  2 GPUs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fm tools/fence_micro.cu && /tmp/fm
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

template <int MODE>
__global__ void release_kernel(int4* dst, uint64_t* flag, long long* cyc, int nstore) {
  if (threadIdx.x < 32) {
    for (int i = 0; i < nstore; ++i) dst[(blockIdx.x * nstore + i) * 32 + threadIdx.x] = make_int4(i, 1, 2, 3);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    if (MODE == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"(1ull) : "memory");
    } else if (MODE == 1) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"(1ull) : "memory");
    } else {
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"(1ull) : "memory");
    }
    // make the next instruction depend on completion of the release
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
}

int main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  int4 *loc, *rem = nullptr;
  uint64_t* flag;
  long long* cyc;
  cudaSetDevice(0);
  cudaMalloc(&loc, 64 << 20);
  cudaMalloc(&flag, 4096);
  cudaMalloc(&cyc, 148 * 8);
  if (ndev > 1) {
    cudaSetDevice(1);
    cudaMalloc(&rem, 64 << 20);
    cudaSetDevice(0);
    cudaDeviceEnablePeerAccess(1, 0);
  }
  const char* names[3] = {"fence.acq_rel.sys + st.relaxed.sys", "fence.acq_rel.gpu + st.relaxed.gpu",
                          "st.release.sys"};
  for (int target = 0; target < (rem ? 2 : 1); ++target)
    for (int nstore : {0, 1, 8, 64})
      for (int mode = 0; mode < 3; ++mode) {
        std::vector<long long> all;
        for (int rep = 0; rep < 5; ++rep) {
          int4* dst = target ? rem : loc;
          if (mode == 0) release_kernel<0><<<148, 256>>>(dst, flag, cyc, nstore);
          if (mode == 1) release_kernel<1><<<148, 256>>>(dst, flag, cyc, nstore);
          if (mode == 2) release_kernel<2><<<148, 256>>>(dst, flag, cyc, nstore);
          cudaDeviceSynchronize();
          std::vector<long long> h(148);
          cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
          if (rep) all.insert(all.end(), h.begin(), h.end());
        }
        std::sort(all.begin(), all.end());
        printf("%-6s stores/warp %3d  %-36s median %7lld cyc  p90 %7lld\n", target ? "PEER" : "local", nstore,
               names[mode], all[all.size() / 2], all[all.size() * 9 / 10]);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
