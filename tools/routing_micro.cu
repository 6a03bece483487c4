// Diagnostics: cost of the LL dispatch routing pass shapes (148 x 512,
// b = 128 tokens, top-8 of 256 experts), per variant, from %globaltimer
// stamps of thread 0 of each CTA (median over CTAs, warm L2).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rm tools/routing_micro.cu && /tmp/rm
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() {
#ifdef USE_CLOCK
  return clock64();
#else
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
#endif
}

template <int V, int ITERS>
__global__ void __launch_bounds__(512) routing(const int64_t* topk, int b, int K, int E, int L, uint64_t Lm,
                                               uint64_t Km, uint64_t* st, int* sink) {
  extern __shared__ int sm[];
  const int W = (b + 31) >> 5, N = E / L;
  int* s_topk = sm;
  uint32_t* s_ebits = reinterpret_cast<uint32_t*>(s_topk + b * K);
  uint32_t* s_dbits = s_ebits + E * W;
  int* s_m = reinterpret_cast<int*>(s_dbits + N * W);
  int* s_q = s_m + E;
  __shared__ int s_bad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t t0, t1, t2, t3, t4;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
  t0 = gt();
  int64_t r0 = 0, r1 = 0;
  const int items = b * K;
  if ((int)threadIdx.x < items) r0 = __ldg(topk + threadIdx.x);
  if ((int)threadIdx.x + 512 < items) r1 = __ldg(topk + threadIdx.x + 512);
  for (int i = threadIdx.x; i < (E + N) * W + E + N; i += blockDim.x) reinterpret_cast<int*>(s_ebits)[i] = 0;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  t1 = gt();
  for (int i = threadIdx.x, r = 0; i < items; i += blockDim.x, ++r) {
    const int64_t e = r == 0 ? r0 : r1;
    if (e < 0 || e >= E) s_bad = 1;
    s_topk[i] = (int)e;
  }
  __syncthreads();
  t2 = gt();
  if (V >= 1) {
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
      const int t = (int)(((uint64_t)i * Km) >> 32);
      const int e = s_topk[i];
      const int rr = t * K, k = i - rr;
      bool dup = false;
#pragma unroll
      for (int j = 0; j < 7; ++j) dup |= j < k && s_topk[rr + j] == e;
      if (dup) s_bad = 1;
      if (V >= 2 && V < 20) atomicAdd(&s_m[e], 1);
      if (V >= 3 && V != 21) atomicOr(&s_ebits[e * W + (t >> 5)], 1u << (t & 31));
    }
  }
  __syncthreads();
  t3 = gt();
  if (V >= 20) {
    // design A pass B: m from popcounts, dbits by warp reduce
    const int E32 = (E + 31) & ~31;
    for (int e = threadIdx.x; e < E32; e += blockDim.x) {
      const int d = (int)(((uint64_t)e * Lm) >> 32);
      int m = 0;
      for (int w = 0; w < W; ++w) {
        const uint32_t v = e < E ? s_ebits[e * W + w] : 0u;
        m += __popc(v);
        const uint32_t r = __reduce_or_sync(0xffffffffu, v);
        if (lane == 0 && r) atomicOr(&s_dbits[d * W + w], r);
      }
      if (e < E) s_m[e] = m;
    }
  } else if (V >= 10) {
    // dbits pass variants: 10 = loads+magic only, 11 = + reduce_or, 12 = + atomicOr
    const int E32 = (E + 31) & ~31;
    uint32_t acc = 0;
    for (int w = 0; w < W; ++w)
      for (int e = threadIdx.x; e < E32; e += blockDim.x) {
        const uint32_t v = e < E ? s_ebits[e * W + w] : 0u;
        const int d = (int)(((uint64_t)e * Lm) >> 32);
        if (V == 10) acc |= v + d;
        if (V >= 11) {
          const uint32_t r = __reduce_or_sync(0xffffffffu, v);
          if (V == 11) acc |= r + d;
          if (V == 12 && lane == 0 && r) atomicOr(&s_dbits[d * W + w], r);
        }
      }
    if (acc == 0x12345) sink[1] = acc;
  } else if (V >= 4) {
    for (int tb = warp * 32; tb < b; tb += blockDim.x) {
      const int t = tb + lane;
      uint64_t mask = 0;
      if (t < b) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < K) mask |= 1ull << (int)(((uint64_t)s_topk[t * K + k] * Lm) >> 32);
      }
      uint64_t wm = ((uint64_t)__reduce_or_sync(0xffffffffu, (uint32_t)(mask >> 32)) << 32) |
                    __reduce_or_sync(0xffffffffu, (uint32_t)mask);
      for (; wm; wm &= wm - 1) {
        const int d = __ffsll(wm) - 1;
        const unsigned bal = __ballot_sync(0xffffffffu, (mask >> d) & 1);
        if (lane == 0) {
          s_dbits[d * W + (tb >> 5)] = bal;
          atomicAdd(&s_q[d], __popc(bal));
        }
      }
    }
  }
  __syncthreads();
  t4 = gt();
  __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint64_t* o = st + blockIdx.x * 8;
    o[0] = t0; o[1] = t1; o[2] = t2; o[3] = t3; o[4] = t4;
  }
  if (s_bad == 12345) sink[0] = s_m[3] + s_q[0];
}

int main() {
  const int b = 128, K = 8, E = 256;
  std::vector<int64_t> h(b * K);
  unsigned s = 1;
  for (int t = 0; t < b; ++t) {
    int used[256] = {0};
    for (int k = 0; k < K; ++k) {
      int e;
      do { s = s * 1103515245u + 12345u; e = (s >> 8) % E; } while (used[e]);
      used[e] = 1;
      h[t * K + k] = e;
    }
  }
  int64_t* d;
  uint64_t* st;
  int* sink;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&st, 148 * 8 * 8);
  cudaMalloc(&sink, 64);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  for (int L : {256, 64, 32}) {
    const int N = E / L, W = (b + 31) / 32;
    const uint64_t Lm = ((1ull << 32) + L - 1) / L, Km = ((1ull << 32) + K - 1) / K;
    const int smem = 4 * (b * K + (E + N) * W + E + N);
    printf("-- N=%d (L=%d)\n", N, L);
    auto run = [&](auto kern, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      std::vector<double> a(4, 0);
      for (int rep = 0; rep < 6; ++rep) {
        kern<<<148, 512, smem>>>(d, b, K, E, L, Lm, Km, st, sink);
        cudaDeviceSynchronize();
        std::vector<uint64_t> o(148 * 8);
        cudaMemcpy(o.data(), st, o.size() * 8, cudaMemcpyDeviceToHost);
        if (rep == 0) continue;
        for (int ph = 0; ph < 4; ++ph) {
          std::vector<double> v;
          for (int c = 0; c < 148; ++c) v.push_back((double)(o[c * 8 + ph + 1] - o[c * 8 + ph]));
          std::sort(v.begin(), v.end());
          a[ph] += v[74] / 5;
        }
      }
      printf("  %-28s zero %6.0f  pass1 %6.0f  pass2 %6.0f  tokens %6.0f ns\n", name, a[0], a[1], a[2], a[3]);
    };
    run(routing<0, 1>, "loads only"); run(routing<0, 2>, "loads only (2nd pass)");
    run(routing<1, 1>, "+dup check"); run(routing<1, 2>, "+dup check (2nd pass)");
    run(routing<2, 1>, "+atomicAdd s_m"); run(routing<2, 2>, "+atomicAdd s_m (2nd pass)");
    run(routing<3, 1>, "+atomicOr ebits"); run(routing<3, 2>, "+atomicOr ebits (2nd pass)");
    run(routing<4, 1>, "+dst ballots"); run(routing<4, 2>, "+dst ballots (2nd pass)");
    run(routing<10, 1>, "dbits loads+magic"); run(routing<10, 2>, "dbits loads+magic (2nd pass)");
    run(routing<11, 1>, "dbits +reduce_or"); run(routing<11, 2>, "dbits +reduce_or (2nd pass)");
    run(routing<12, 1>, "dbits +atomicOr"); run(routing<12, 2>, "dbits +atomicOr (2nd pass)");
    run(routing<20, 1>, "design A"); run(routing<20, 2>, "design A (2nd pass)");
    run(routing<21, 1>, "design A w/o ebits atomics"); run(routing<21, 2>, "design A w/o ebits atomics (2nd pass)");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
