// K1 routing_layout: validation + the integer layout of one rank's routing,
// written to global memory (HT handles, strict-mode LL handle validation).
// The arithmetic is block_layout (layout.cuh); the LL dispatch kernel runs
// the same routine per CTA in shared memory instead.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace epb {

__global__ void __launch_bounds__(1024)
routing_layout_kernel(const int64_t* __restrict__ topk, int b, int K, int E, int N, int L,
                      int32_t* m_out, int32_t* q_out, int32_t* tok_rank, int32_t* tok_slot, int* err) {
  extern __shared__ int smem[];
  const BlockLayoutSmem sm = BlockLayoutSmem::carve(smem, blockDim.x >> 5, E, N);
  if (!block_layout_checked(topk, b, K, E, N, L, sm, m_out, q_out, tok_rank, tok_slot) && threadIdx.x == 0)
    raise_err(err, EPB_INVALID_ARGUMENT);
}

// Multi-CTA form for large batches: (1) CTA c lays out tokens
// [c*chunk, (c+1)*chunk) alone (local ranks/slots, per-chunk column
// histogram); (2) exclusive prefix of every column over the chunks; (3) every
// rank/slot gets its chunk's base added.  Same integers as one block over all
// tokens: a column's order is ascending t, chunks are ascending t ranges.
__global__ void __launch_bounds__(256)
layout_chunk_kernel(const int64_t* __restrict__ topk, int b, int K, int E, int N, int L, int chunk, int32_t* hist,
                    int32_t* tok_rank, int32_t* tok_slot, int* err) {
  extern __shared__ int smem[];
  const int t0 = blockIdx.x * chunk, bc = min(chunk, b - t0);
  const int64_t* tk = topk + (int64_t)t0 * K;
  const BlockLayoutSmem sm = BlockLayoutSmem::carve(smem, blockDim.x >> 5, E, N);
  int32_t* h = hist + (int64_t)blockIdx.x * (E + N);
  if (!block_layout_checked(tk, bc, K, E, N, L, sm, h, h + E, tok_rank + (int64_t)t0 * K,
                            tok_slot + (int64_t)t0 * N) && threadIdx.x == 0)
    raise_err(err, EPB_INVALID_ARGUMENT);
}

// one warp per column: 32 chunks per step loaded at once, shuffle scan
__global__ void layout_prefix_kernel(int32_t* hist, int chunks, int E, int N, int32_t* m_out, int32_t* q_out) {
  const int C = E + N;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int c = blockIdx.x * wpb + (threadIdx.x >> 5); c < C; c += gridDim.x * wpb) {
    int carry = 0;
    for (int j0 = 0; j0 < chunks; j0 += 32) {
      const int j = j0 + lane;
      const int v = j < chunks ? hist[(int64_t)j * C + c] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (j < chunks) hist[(int64_t)j * C + c] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      if (c < E) m_out[c] = carry;
      else q_out[c - E] = carry;
    }
  }
}

__global__ void layout_fix_kernel(const int64_t* __restrict__ topk, int b, int K, int E, int N, int chunk,
                                  const int32_t* base, int32_t* tok_rank, int32_t* tok_slot) {
  const int C = E + N;
  const int64_t nk = (int64_t)b * K, nd = (int64_t)b * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk + nd; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nk) {
      const int t = (int)(i / K);
      const int64_t e = topk[i];
      if (e >= 0 && e < E) tok_rank[i] += base[(int64_t)(t / chunk) * C + (int)e];  // (invalid rows: error set)
    } else {
      const int64_t j = i - nk;
      const int t = (int)(j / N), d = (int)(j - (int64_t)t * N);
      const int v = tok_slot[j];
      if (v >= 0) tok_slot[j] = v + base[(int64_t)(t / chunk) * C + E + d];
    }
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
  if (b > 4 * kLayChunk && g->d_lay && lay->tok_slot) {
    const int chunks = (b + kLayChunk - 1) / kLayChunk;
    const int wpc = 4;  // warps per chunk CTA
    const size_t csm = BlockLayoutSmem::bytes(wpc, E, N);
    if (csm <= 200 * 1024) {
      cudaStream_t s = as_stream(stream);
      EPB_CUDA(cudaFuncSetAttribute(layout_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
      layout_chunk_kernel<<<chunks, wpc * 32, csm, s>>>(topk_idx, b, K, E, N, L, kLayChunk, g->d_lay, lay->tok_rank,
                                                         lay->tok_slot, g->d_err);
      EPB_LAUNCH_CHECK();
      layout_prefix_kernel<<<(E + N + 7) / 8, 256, 0, s>>>(g->d_lay, chunks, E, N, lay->expert_count,
                                                          lay->rank_count);
      EPB_LAUNCH_CHECK();
      const int64_t items = (int64_t)b * (K + N);
      layout_fix_kernel<<<(int)std::min<int64_t>(1184, (items + 255) / 256), 256, 0, s>>>(
          topk_idx, b, K, E, N, kLayChunk, g->d_lay, lay->tok_rank, lay->tok_slot);
      EPB_LAUNCH_CHECK();
      return EPB_OK;
    }
  }
  int warps = 32;
  while (warps > 1 && BlockLayoutSmem::bytes(warps, E, N) > 200 * 1024) warps >>= 1;
  const size_t smem = BlockLayoutSmem::bytes(warps, E, N);
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "too many experts for routing_layout");
  EPB_CUDA(cudaFuncSetAttribute(routing_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  routing_layout_kernel<<<1, warps * 32, smem, as_stream(stream)>>>(
      topk_idx, b, K, E, N, L, lay->expert_count, lay->rank_count, lay->tok_rank, lay->tok_slot, g->d_err);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}
