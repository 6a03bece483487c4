// Block-wide routing layout in shared memory (used by K1 and, redundantly
// per CTA, by the fused LL dispatch kernel).  Bit-exact with the reference's
// integer loops:
//   m[e]        = m(e, self), tokens routed to e             ll.py:255-259
//   q[d]        = tokens touching rank d (dedup)              ht.py:305-307
//   slot[t, d]  = index of t among tokens touching d          ll.py:295-302
//   rank[t, k]  = index of t among tokens routed to e_tk      ll.py:383-399
// Warp w owns a contiguous token segment: pass 1 builds per-warp column
// histograms with shared atomics, pass 2 scans them across warps, pass 3
// walks each segment 32 tokens at a time and ranks an entry with a shared
// ballot word (popc of the lower lanes that hit the same column).
#pragma once
#include "common.cuh"

namespace epb {

struct BlockLayoutSmem {
  int* hist;        // [nwarps][E+N]
  uint32_t* ballot; // [nwarps][E+N]
  static size_t bytes(int nwarps, int E, int N) { return (size_t)nwarps * (E + N) * 8; }
};

// topk: b*K expert ids (already validated).  Outputs may live in shared or
// global memory.  Requires all threads of the block.
template <typename TopkT>
EPB_DEV void block_layout(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                          int32_t* m_out, int32_t* q_out, int32_t* rank_out, int32_t* slot_out,
                          uint64_t* mask_out) {
  const int C = E + N;
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nwarps * C; i += blockDim.x) {
    sm.hist[i] = 0;
    sm.ballot[i] = 0u;
  }
  __syncthreads();
  const int seg = (b + nwarps - 1) / nwarps;
  const int t0 = min(b, warp * seg), t1 = min(b, t0 + seg);
  int* h = sm.hist + warp * C;
  uint32_t* bw = sm.ballot + warp * C;
  for (int t = t0 + lane; t < t1; t += 32) {
    uint64_t mask = 0;
    for (int k = 0; k < K; ++k) {
      const int e = (int)topk[(int64_t)t * K + k];
      atomicAdd(&h[e], 1);
      mask |= 1ull << (e / L);
    }
    for (uint64_t mm = mask; mm; mm &= mm - 1) atomicAdd(&h[E + __ffsll(mm) - 1], 1);
    if (mask_out) mask_out[t] = mask;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int run = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int v = sm.hist[w * C + c];
      sm.hist[w * C + c] = run;
      run += v;
    }
    if (c < E) { if (m_out) m_out[c] = run; }
    else if (q_out) q_out[c - E] = run;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = t0; base < t1; base += 32) {
    const int t = base + lane;
    const bool act = t < t1;
    uint64_t mask = 0;
    if (act) {
      for (int k = 0; k < K; ++k) {
        const int e = (int)topk[(int64_t)t * K + k];
        mask |= 1ull << (e / L);
        atomicOr(&bw[e], 1u << lane);
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) atomicOr(&bw[E + __ffsll(mm) - 1], 1u << lane);
    }
    __syncwarp();
    if (act) {
      for (int k = 0; k < K; ++k) {
        const int e = (int)topk[(int64_t)t * K + k];
        rank_out[(int64_t)t * K + k] = h[e] + __popc(bw[e] & lt);
      }
      if (slot_out)
        for (int d = 0; d < N; ++d)
          slot_out[(int64_t)t * N + d] = ((mask >> d) & 1) ? h[E + d] + __popc(bw[E + d] & lt) : -1;
    }
    __syncwarp();
    if (act) {
      // the lowest lane hitting a column advances its running count
      for (int k = 0; k < K; ++k) {
        const int e = (int)topk[(int64_t)t * K + k];
        const uint32_t bits = bw[e];
        if ((bits & lt) == 0) h[e] += __popc(bits);
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) {
        const int c = E + __ffsll(mm) - 1;
        const uint32_t bits = bw[c];
        if ((bits & lt) == 0) h[c] += __popc(bits);
      }
    }
    __syncwarp();
    if (act) {
      for (int k = 0; k < K; ++k) bw[(int)topk[(int64_t)t * K + k]] = 0u;
      for (uint64_t mm = mask; mm; mm &= mm - 1) bw[E + __ffsll(mm) - 1] = 0u;
    }
    __syncwarp();
  }
  __syncthreads();
}

// row validation: ids in [0, E), distinct within a row (api.py:150-170)
template <typename TopkT>
EPB_DEV bool block_validate(const TopkT* topk, int b, int K, int E, int* s_bad) {
  (void)s_bad;
  bool bad = false;
  for (int t = threadIdx.x; t < b; t += blockDim.x) {
    for (int k = 0; k < K; ++k) {
      const int64_t e = (int64_t)topk[(int64_t)t * K + k];
      if (e < 0 || e >= E) { bad = true; break; }
      for (int j = 0; j < k; ++j)
        if ((int64_t)topk[(int64_t)t * K + j] == e) bad = true;
    }
  }
  return __syncthreads_or(bad) == 0;  // one verdict per block (a barrier)
}

}  // namespace epb
