// Diagnostics: round-trip latency of a payload + flag handoff between two
// GPUs over NVLink, for each way of releasing the flag, and an ordering check
// (the receiver verifies every payload word after it acquired the flag).
//
// GPU0 (ping) CTA c: write `kb` KB of payload (every warp, 16-B stores) into
// GPU1's buffer, __syncthreads, release (mode), flag[c] = iter.  GPU1 (pong)
// CTA c: acquire flag[c] == iter, verify the chunk, then release a pong flag
// back into GPU0's memory.  GPU0 waits for the pong and starts the next
// iteration.  Reports the median round trip per CTA in microseconds and the
// number of payload words seen stale after the flag (ordering violations).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rm tools/release_micro.cu && /tmp/rm
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_acq_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// release modes (thread 0 after __syncthreads unless stated)
//  0 fence.acq_rel.sys + st.relaxed.sys
//  1 fence.acq_rel.gpu + st.relaxed.sys      (outside the PTX model for a peer observer)
//  2 st.release.sys
//  3 red.release.sys.add
//  4 every thread fence.acq_rel.sys, __syncthreads, thread 0 st.relaxed.sys
//  5 no fence, st.relaxed.sys                 (incorrect; isolates the fence cost)
template <int MODE>
__device__ __forceinline__ void release_flag(uint64_t* f, uint64_t v) {
  if (MODE == 4) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
  } else {
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  if (MODE == 0 || MODE == 4) {
    if (MODE == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  } else if (MODE == 1) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  } else if (MODE == 2) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  } else if (MODE == 3) {
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(f), "l"(1ull) : "memory");
  } else {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
  }
}

template <int MODE>
__global__ void __launch_bounds__(512) ping(int4* remote, uint64_t* rflag, uint64_t* pong, int words, int iters,
                                            float* rtt_us) {
  const int c = blockIdx.x;
  int4* chunk = remote + (size_t)c * words;
  for (int it = 1; it <= iters; ++it) {
    const uint64_t t0 = gtime();
    for (int i = threadIdx.x; i < words; i += blockDim.x) chunk[i] = make_int4(it, i, c, it ^ i);
    release_flag<MODE>(&rflag[c], (uint64_t)it);
    if (threadIdx.x == 0) {
      while (ld_acq_sys(&pong[c]) < (uint64_t)it) {
      }
      rtt_us[(size_t)c * iters + it - 1] = (gtime() - t0) * 1e-3f;
    }
    __syncthreads();
  }
}

template <int MODE>
__global__ void __launch_bounds__(512) pongk(const int4* local, const uint64_t* flag, uint64_t* rpong, int words,
                                             int iters, unsigned long long* bad) {
  const int c = blockIdx.x;
  const int4* chunk = local + (size_t)c * words;
  __shared__ int s_go;
  for (int it = 1; it <= iters; ++it) {
    if (threadIdx.x == 0) {
      // MODE 3 counts arrivals (+1 per iteration)
      while (ld_acq_sys(&flag[c]) < (uint64_t)it) {
      }
      s_go = 1;
    }
    __syncthreads();
    // the acquire by thread 0 + bar.sync orders these loads after it
    unsigned long long nb = 0;
    for (int i = threadIdx.x; i < words; i += blockDim.x) {
      int4 v;
      asm volatile("ld.relaxed.sys.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(&chunk[i]) : "memory");
      if (v.x != it || v.y != i || v.z != c || v.w != (it ^ i)) ++nb;
    }
    if (nb) atomicAdd(bad, nb);
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&rpong[c]), "l"((uint64_t)it) : "memory");
  }
}

template <int MODE>
void run(int ctas, int kb, int iters, int4* buf1, uint64_t* flag1, uint64_t* pong0, float* rtt0,
         unsigned long long* bad1, const char* name) {
  const int words = kb * 1024 / 16;
  cudaSetDevice(1);
  cudaMemset(flag1, 0, 4096);
  cudaMemset(bad1, 0, 8);
  cudaDeviceSynchronize();
  cudaSetDevice(0);
  cudaMemset(pong0, 0, 4096);
  cudaDeviceSynchronize();
  cudaSetDevice(1);
  pongk<MODE><<<ctas, 512>>>(buf1, flag1, pong0, words, iters, bad1);
  cudaSetDevice(0);
  ping<MODE><<<ctas, 512>>>(buf1, flag1, pong0, words, iters, rtt0);
  cudaDeviceSynchronize();
  cudaSetDevice(1);
  cudaDeviceSynchronize();
  unsigned long long nb = 0;
  cudaMemcpy(&nb, bad1, 8, cudaMemcpyDeviceToHost);
  cudaSetDevice(0);
  std::vector<float> h((size_t)ctas * iters);
  cudaMemcpy(h.data(), rtt0, h.size() * 4, cudaMemcpyDeviceToHost);
  // drop the first 10% of iterations (warm-up)
  std::vector<float> v;
  for (int c = 0; c < ctas; ++c)
    for (int it = iters / 10; it < iters; ++it) v.push_back(h[(size_t)c * iters + it]);
  std::sort(v.begin(), v.end());
  printf("ctas %3d  KB/cta %4d  %-44s rtt median %7.2f us  p90 %7.2f  stale words %llu  %s\n", ctas, kb, name,
         v[v.size() / 2], v[v.size() * 9 / 10], nb, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 1;
  }
  int4* buf1;
  uint64_t *flag1, *pong0;
  float* rtt0;
  unsigned long long* bad1;
  const int iters = 200;
  cudaSetDevice(1);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaMalloc(&buf1, (size_t)148 * 64 * 1024);
  cudaMalloc(&flag1, 4096);
  cudaMalloc(&bad1, 8);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&pong0, 4096);
  cudaMalloc(&rtt0, (size_t)148 * iters * 4);
  for (int ctas : {1, 148})
    for (int kb : {0, 1, 16, 64}) {
      run<5>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "no fence + st.relaxed.sys (incorrect)");
      run<1>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "fence.acq_rel.gpu + st.relaxed.sys");
      run<0>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "fence.acq_rel.sys + st.relaxed.sys");
      run<2>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "st.release.sys");
      run<3>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "red.release.sys.add");
      run<4>(ctas, kb, iters, buf1, flag1, pong0, rtt0, bad1, "all threads fence.acq_rel.sys");
    }
  return 0;
}
