// K1 routing_layout: validation + the integer layout of one rank's routing,
// written to global memory (HT handles, strict-mode LL handle validation).
// The arithmetic is block_layout (layout.cuh); the LL dispatch kernel runs
// the same routine per CTA in shared memory instead.
#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace epb {

__global__ void __launch_bounds__(1024)
routing_layout_kernel(const int64_t* __restrict__ topk, int b, int K, int E, int N, int L,
                      int32_t* m_out, int32_t* q_out, int32_t* tok_rank, int32_t* tok_slot, int* err) {
  extern __shared__ int smem[];
  __shared__ int s_bad;
  if (!block_validate(topk, b, K, E, &s_bad)) {
    if (threadIdx.x == 0) atomicCAS(err, 0, EPB_INVALID_ARGUMENT);
    return;
  }
  BlockLayoutSmem sm;
  sm.hist = smem;
  sm.ballot = reinterpret_cast<uint32_t*>(smem + (blockDim.x >> 5) * (E + N));
  block_layout(topk, b, K, E, N, L, sm, m_out, q_out, tok_rank, tok_slot, nullptr);
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
