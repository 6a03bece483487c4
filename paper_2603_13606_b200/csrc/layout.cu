// K1 routing_layout: one pass over topk_idx producing every integer the
// dispatch/combine kernels need, bit-exact with the reference's loops:
//   expert_count[e]   = m(e, self)                      ll.py:255-259, ht.py:299-304
//   rank_count[d]     = q(self, d) (tokens touching d)  ht.py:305-307
//   tok_slot[t, d]    = index of t among tokens touching d, ascending t
//                       (the optimized-layout slot order, ll.py:295-302)
//   tok_rank[t, k]    = index of t among tokens routed to e_tk, ascending t
//                       (filled[l] order, ll.py:383-399; HT (e, src, t) order,
//                       ht.py:567-580)
// plus validation (ids in range, distinct per row; api.py:150-170).
//
// One CTA.  Warp w owns a contiguous token segment; pass 1 builds per-warp
// histograms with shared atomics, pass 2 scans them across warps per column,
// pass 3 re-walks each segment 32 tokens at a time and ranks a lane's entry
// with a shared ballot word (popc of lower lanes that hit the same column).
#include "common.cuh"
#include "internal.h"

namespace epb {

__global__ void __launch_bounds__(1024)
routing_layout_kernel(const int64_t* __restrict__ topk, int b, int K, int E, int N, int L,
                      int32_t* m_out, int32_t* q_out, int32_t* tok_rank, int32_t* tok_slot,
                      int* err) {
  extern __shared__ int smem[];
  const int C = E + N;
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* hist = smem;                                                   // [nwarps][C]
  uint32_t* ballot = reinterpret_cast<uint32_t*>(smem + nwarps * C);  // [nwarps][C]
  __shared__ int s_bad;
  for (int i = threadIdx.x; i < nwarps * C; i += blockDim.x) {
    hist[i] = 0;
    ballot[i] = 0u;
  }
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();

  const int seg = (b + nwarps - 1) / nwarps;
  const int t0 = min(b, warp * seg), t1 = min(b, t0 + seg);
  int* h = hist + warp * C;
  uint32_t* bw = ballot + warp * C;

  // pass 1: validate + per-warp histograms
  for (int t = t0 + lane; t < t1; t += 32) {
    uint64_t mask = 0;
    bool ok = true;
    for (int k = 0; k < K; ++k) {
      const int64_t e = topk[(int64_t)t * K + k];
      if (e < 0 || e >= E) { ok = false; break; }
      for (int j = 0; j < k; ++j)
        if (topk[(int64_t)t * K + j] == e) ok = false;
      mask |= 1ull << (int)(e / L);
    }
    if (!ok) { s_bad = 1; continue; }
    for (int k = 0; k < K; ++k) atomicAdd(&h[(int)topk[(int64_t)t * K + k]], 1);
    for (uint64_t mm = mask; mm; mm &= mm - 1) atomicAdd(&h[E + __ffsll(mm) - 1], 1);
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicCAS(err, 0, EPB_INVALID_ARGUMENT);
    return;
  }
  // pass 2: exclusive scan over warps, per column
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int run = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int v = hist[w * C + c];
      hist[w * C + c] = run;
      run += v;
    }
    if (c < E) m_out[c] = run;
    else q_out[c - E] = run;
  }
  __syncthreads();
  // pass 3: ranks
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = t0; base < t1; base += 32) {
    const int t = base + lane;
    const bool act = t < t1;
    int ek[kMaxTopK];
    uint64_t mask = 0;
    if (act) {
      for (int k = 0; k < K; ++k) {
        ek[k] = (int)topk[(int64_t)t * K + k];
        mask |= 1ull << (ek[k] / L);
        atomicOr(&bw[ek[k]], 1u << lane);
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) atomicOr(&bw[E + __ffsll(mm) - 1], 1u << lane);
    }
    __syncwarp();
    if (act) {
      for (int k = 0; k < K; ++k)
        tok_rank[(int64_t)t * K + k] = h[ek[k]] + __popc(bw[ek[k]] & lt);
      for (int d = 0; d < N; ++d)
        tok_slot[(int64_t)t * N + d] =
            ((mask >> d) & 1) ? h[E + d] + __popc(bw[E + d] & lt) : -1;
    }
    __syncwarp();
    if (act) {
      // the lowest lane hitting a column advances its running count
      for (int k = 0; k < K; ++k) {
        const uint32_t bits = bw[ek[k]];
        if ((bits & lt) == 0) h[ek[k]] += __popc(bits);
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) {
        const int c = E + __ffsll(mm) - 1;
        const uint32_t bits = bw[c];
        if ((bits & lt) == 0) h[c] += __popc(bits);
      }
    }
    __syncwarp();
    if (act) {
      for (int k = 0; k < K; ++k) bw[ek[k]] = 0u;
      for (uint64_t mm = mask; mm; mm &= mm - 1) bw[E + __ffsll(mm) - 1] = 0u;
    }
    __syncwarp();
  }
}

}  // namespace epb

using namespace epb;

extern "C" int epb_routing_layout(epb_group* g, const int64_t* topk_idx, int32_t b,
                                  const epb_layout* lay, void* stream) {
  if (!g || !lay) return fail(EPB_INVALID_ARGUMENT, "null argument");
  if (b < 0 || b > g->cfg.max_tokens_per_rank)
    return fail(EPB_INVALID_ARGUMENT, "token count exceeds max_tokens_per_rank");
  const int E = g->cfg.num_experts, N = g->cfg.num_ranks, K = g->cfg.top_k;
  const int L = experts_per_rank(E, N);
  const int C = E + N;
  int warps = 32;
  while (warps > 1 && (size_t)warps * C * 8 > 200 * 1024) warps >>= 1;
  const size_t smem = (size_t)warps * C * 8;
  if (smem > 220 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "too many experts for routing_layout");
  EPB_CUDA(cudaFuncSetAttribute(routing_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  routing_layout_kernel<<<1, warps * 32, smem, as_stream(stream)>>>(
      topk_idx, b, K, E, N, L, lay->expert_count, lay->rank_count, lay->tok_rank, lay->tok_slot,
      g->d_err);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}
