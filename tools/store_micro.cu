// Diagnostics: cost of the LL dispatch own-row store pattern — 128 CTAs x
// 512 threads, each CTA writes one 7168-B row (448 x 16-B chunks) to 8
// rows of a [256 x 128 x 7168] B output (scattered over 235 MB) — vs the
// same bytes to contiguous rows; warm and after a 256 MB memset flush.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm tools/store_micro.cu && /tmp/sm
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(512) stores(uint8_t* out, const int* rows, int nch, uint64_t* st) {
  uint64_t t0 = gt();
  const int c = threadIdx.x;
  int4 v = make_int4(blockIdx.x, c, 1, 2);
  if (c < nch) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = rows[blockIdx.x * 8 + k];
      *reinterpret_cast<int4*>(out + (int64_t)r * 7168 + (int64_t)c * 16) = v;
    }
  }
  __syncthreads();
  uint64_t t1 = gt();
  if (threadIdx.x == 0) { st[blockIdx.x * 2] = t0; st[blockIdx.x * 2 + 1] = t1; }
}

int main() {
  const size_t nrows = 256 * 128;
  uint8_t* out;
  cudaMalloc(&out, nrows * 7168);
  char* flush;
  cudaMalloc(&flush, 256u << 20);
  int* rows;
  cudaMalloc(&rows, 128 * 8 * 4);
  uint64_t* st;
  cudaMalloc(&st, 148 * 2 * 8);
  std::vector<int> scat(128 * 8), cont(128 * 8);
  unsigned s = 7;
  for (int t = 0; t < 128; ++t)
    for (int k = 0; k < 8; ++k) {
      s = s * 1103515245u + 12345u;
      const int e = (s >> 8) % 256;
      scat[t * 8 + k] = e * 128 + t;  // expert-major row of (e, src 0, i = t)
      cont[t * 8 + k] = t * 8 + k;
    }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int pat = 0; pat < 3; ++pat)
    for (int fl = 0; fl < 2; ++fl) {
      const int nch = pat == 2 ? 0 : 448;
      cudaMemcpy(rows, pat == 1 ? cont.data() : scat.data(), 128 * 8 * 4, cudaMemcpyHostToDevice);
      double span = 0, ev = 0;
      for (int rep = 0; rep < 6; ++rep) {
        if (fl) cudaMemset(flush, rep, 256u << 20);
        cudaEventRecord(a);
        stores<<<128, 512>>>(out, rows, nch, st);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::vector<uint64_t> o(256);
        cudaMemcpy(o.data(), st, 256 * 8, cudaMemcpyDeviceToHost);
        uint64_t lo = ~0ull, hi = 0;
        for (int i = 0; i < 128; ++i) { lo = std::min(lo, o[2 * i]); hi = std::max(hi, o[2 * i + 1]); }
        if (rep) { span += (hi - lo) / 5.0; ev += ms * 1000 / 5.0; }
      }
      printf("%-11s %-8s CTA span %7.0f ns   event %7.2f us  (%.1f MB)\n", pat == 2 ? "no stores" : (pat ? "contiguous" : "scattered"),
             fl ? "flushed" : "warm", span, ev, 128 * 8 * 7168 / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
