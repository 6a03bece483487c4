// High-Throughput dispatch/combine kernels (K5a meta, K5b dispatch, K6 combine).
//
// Reference semantics (epsim ht.py):
//  * metadata (ht.py:291-331): every rank all-gathers m_row[E] (tokens per
//    expert) and q_row[N] (dedup tokens per destination) before any payload;
//    receive shapes and the sorted-output offsets follow from them
//    (HTMeta.expert_offsets, ht.py:185-193).
//  * dispatch (ht.py:381-468, 553-583): one record per (token, destination
//    rank) = header + K f32 weights (+ the row); the receiver places a copy
//    of the row for every local expert it names, sorted by (local expert,
//    src, t).  The sender also writes, per k, the final output row on the
//    owner (offset(e, src) + rank of t within (e, src)), so placement is a
//    parallel scatter that never depends on arrival order.
//    B200 transport: PULL.  The sender converts its rows once into its own
//    window (`stage`, local HBM) and pushes only the small records; each
//    receiver reads every row it needs once over NVLink (peer loads measured
//    ~765 GB/s vs ~710 GB/s for peer stores on this system) and fans it out
//    to its local experts' output rows, so the NVLink transfer and the local
//    placement are one pass.  Rows a rank routes to its OWN experts never
//    leave: the sender writes them straight to their sorted positions.
//  * combine (ht.py:587-735): p = f32(w * y) from the f32 expert row; per
//    token, per node holding its experts (ascending), a partial = first p
//    then f32 adds in ascending k; out = f32(0 + partial_0) + partial_1 ...
//    Expert rows travel in their own dtype (f32, or bf16 which widens
//    exactly) and the home rank forms p, so the product is bit-identical.
//    Rows of the home's own experts are read in place, not copied.
//  * single-node transport only: the reference's rail FIFOs / forwarders
//    (ht.py:479-551) are out of scope on one NVSwitch domain, but the
//    hierarchical SUM ORDER is reproduced for any ranks_per_node.
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace epb {

constexpr int kHTThreads = 512;
constexpr int kHU = 8;  // 16-B loads in flight per lane in copies

EPB_DEV uint8_t* hpeer(const uint64_t* peers, int r) { return reinterpret_cast<uint8_t*>(peers[r]); }

EPB_DEV void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
EPB_DEV int4 ld_plain_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
EPB_DEV void st_plain_v4(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

// ---------------------------------------------------------------------------
// K5a: metadata all-gather over the windows
// ---------------------------------------------------------------------------
struct HTMetaSend {
  const int* err;  // a routing the layout kernel rejected sends nothing (validation before traffic)
  const int32_t* m;
  const int32_t* q;
  const uint64_t* peers;
  HTGeom g;
  int rank, parity;
  uint32_t tag;
  OpTrace ops;
};

// block-wide: this rank's row (m | q) into every peer's metadata slot, then
// one release and the per-source tags
EPB_DEV void meta_send_block(const HTMetaSend& p) {
  const HTGeom& g = p.g;
  const int C = g.E + g.N;
  const uint64_t row_off = g.meta + ((uint64_t)p.parity * g.N + p.rank) * C * 4;
  for (int i = threadIdx.x; i < g.N * C; i += blockDim.x) {
    const int d = i / C, c = i % C;
    const int32_t v = c < g.E ? p.m[c] : p.q[c - g.E];
    reinterpret_cast<int32_t*>(hpeer(p.peers, d) + row_off)[c] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    chaos_delay(g.chaos_ns, 0x41u);
    fence_release(g.sys_fence);  // one release covers every thread's row stores
    for (int d = 0; d < g.N; ++d) {
      uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, d) + g.meta_flag) + p.parity * g.N + p.rank;
      st_relaxed_sys_u64(flag, (uint64_t)p.tag);
      op_record(p.ops, EPB_OP_PUT, p.rank, d, row_off, 4ull * C);
      op_record(p.ops, EPB_OP_SIGNAL, p.rank, d, g.meta_flag + 8ull * (p.parity * g.N + p.rank), 8,
                p.parity * g.N + p.rank, p.tag);
    }
  }
  // the flags are out before any thread of the block starts waiting for the
  // peers' (the fused open waits next in the same block: a lane of warp 0
  // spinning on a peer's flag could otherwise starve thread 0's sends while
  // the peer's block does the same — a cross-GPU deadlock seen under
  // EPB_CHAOS_NS)
  __syncthreads();
}

__global__ void __launch_bounds__(256) ht_meta_send_kernel(HTMetaSend p) {
  if (*reinterpret_cast<const volatile int*>(p.err) != 0) return;
  meta_send_block(p);
}

struct HTMetaRecv {
  const uint8_t* win;
  int32_t* meta_out;
  int32_t* offsets;
  int32_t* recv_total;
  int* err;
  HTGeom g;
  uint64_t timeout_ns;
  int rank, parity;
  uint32_t tag;
};

// block-wide: wait for every source's row, then the group offsets and this
// rank's receive total (s_meta: [N*C + E] ints of shared memory)
EPB_DEV void meta_recv_block(const HTMetaRecv& p, int32_t* s_meta) {
  const HTGeom& g = p.g;
  const int N = g.N, E = g.E, C = E + N, L = g.L;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.meta_flag) + p.parity * N;
  bool fail = false;
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v;
    fail |= !wait_tag(&flags[s], p.tag, 0, 0xFFFFFFFFu, p.timeout_ns, p.err, &v);
  }
  if (__syncthreads_or(fail)) return;
  const int32_t* rows = reinterpret_cast<const int32_t*>(p.win + g.meta + (uint64_t)p.parity * N * C * 4);
  for (int i = threadIdx.x; i < N * C; i += blockDim.x) {
    const int32_t v = *reinterpret_cast<const volatile int32_t*>(&rows[i]);
    s_meta[i] = v;
    p.meta_out[i] = v;
  }
  __syncthreads();
  // offsets[e, s]: row of group (e, s) inside owner(e)'s sorted output
  // = (rows of earlier local experts of owner(e)) + (rows of e from src < s)
  int* s_col = s_meta + N * C;  // [E]: per-expert totals, then their per-owner exclusive scan
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int tot = 0;
    for (int s = 0; s < N; ++s) tot += s_meta[s * C + e];
    s_col[e] = tot;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int d = warp; d < N; d += blockDim.x >> 5) {  // one warp per owner: shuffle scan
    const int lo = d * L, hi = min(lo + L, E);
    int carry = 0;
    for (int b0 = lo; b0 < hi; b0 += 32) {
      const int e = b0 + lane;
      const int v = e < hi ? s_col[e] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (e < hi) s_col[e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (d == p.rank && lane == 0) *p.recv_total = carry;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int base = s_col[e];
    for (int s = 0; s < N; ++s) {
      p.offsets[e * N + s] = base;
      base += s_meta[s * C + e];
    }
  }
}

__global__ void __launch_bounds__(1024) ht_meta_recv_kernel(HTMetaRecv p) {
  extern __shared__ int32_t s_meta[];  // [N][C]
  meta_recv_block(p, s_meta);
}

// ---------------------------------------------------------------------------
// K1 + K5a fused: HTRank.open_round (ht.py:335-368) in ONE launch.  CTA c
// owns tokens [c*kLayChunk, (c+1)*kLayChunk): it validates them and builds
// per-warp column histograms (shared memory), writes the chunk's column
// totals, and after ONE grid barrier takes its chunk base per column from
// the totals of the earlier chunks and ranks its tokens (final ranks and
// slots, no fix-up pass).  CTA 0 also sums every chunk (m, q), sends this
// rank's metadata row before ranking its own chunk (the peers' rows travel
// meanwhile), then waits for every source's row and writes the receive
// shapes straight into host-mapped pinned memory, followed by the group's
// error word: the host reads the round's shapes after one stream
// synchronisation and no copy.  Top-k > 8 keeps the two-barrier form (chunk
// layouts, column prefix, chunk bases added).  Same integers as the
// three-kernel K1 + the K5a pair.  All CTAs are co-resident (cooperative
// launch); the barrier words are reset by the last CTA out.
struct HTOpen {
  const int64_t* topk;
  int b, K, L, chunk;  // tokens per CTA (one CTA: chunk = b)
  int32_t* hist;  // [grid][E+N] per-chunk column histograms, then their exclusive prefixes
  int32_t* tok_rank;
  int32_t* tok_slot;
  unsigned* bar;  // [2]: arrivals, exits
  HTMetaSend ms;  // m/q = the layout's outputs
  HTMetaRecv mr;  // meta_out / recv_total in host-mapped memory
  int32_t* host_err;
  uint64_t* stamps;  // optional [grid][16] %globaltimer checkpoints (diagnostics, epb_group_set_trace)
};

#define OPEN_STAMP(I) \
  do { if (p.stamps && threadIdx.x == 0) p.stamps[blockIdx.x * 16 + (I)] = globaltimer(); } while (0)

EPB_DEV void grid_arrive_wait(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) ht_open_kernel(HTOpen p) {
  extern __shared__ int smem[];
  const HTGeom& g = p.ms.g;
  const int E = g.E, N = g.N, C = E + N;
  const int G = gridDim.x;
  OPEN_STAMP(0);
  const int t0 = blockIdx.x * p.chunk, bc = max(0, min(p.chunk, p.b - t0));
  const int64_t* tk = p.topk + (int64_t)t0 * p.K;
  int32_t* h = p.hist + (int64_t)blockIdx.x * C;
  int32_t* ranks = p.tok_rank + (int64_t)t0 * p.K;
  int32_t* slots = p.tok_slot + (int64_t)t0 * N;
  const int nw = blockDim.x >> 5;
  const BlockLayoutSmem sm = BlockLayoutSmem::carve(smem, nw, E, N);
  uint64_t* lst = p.stamps ? p.stamps + blockIdx.x * 16 + 10 : nullptr;
  bool bad;
  if (G > 1 && p.K <= 8) {
    // (1) validated per-warp histograms of the chunk, its column totals out;
    // one grid barrier; (2) the chunk's base per column = the totals of the
    // earlier chunks (CTA 0 also sums all of them: m and q, and sends the
    // metadata row at once); (3) ranks and slots seeded with the bases
    if (!block_hist8(tk, bc, p.K, E, N, p.L, sm, h, lst) && threadIdx.x == 0)
      raise_err(p.mr.err, EPB_INVALID_ARGUMENT);
    OPEN_STAMP(1);
    grid_arrive_wait(p.bar, G);
    OPEN_STAMP(2);
    bad = *reinterpret_cast<const volatile int*>(p.mr.err) != 0;
    if (!bad) {
      int* s_base = smem + BlockLayoutSmem::bytes(nw, E, N) / 4;
      for (int c = threadIdx.x; c < C; c += blockDim.x) {
        int base = 0;
        for (int j = 0; j < (int)blockIdx.x; ++j) base += __ldcg(&p.hist[(int64_t)j * C + c]);
        s_base[c] = base;
        if (blockIdx.x == 0) {  // m and q: the totals over every chunk
          int tot = 0;
          for (int j = 0; j < G; ++j) tot += __ldcg(&p.hist[(int64_t)j * C + c]);
          if (c < E) const_cast<int32_t*>(p.ms.m)[c] = tot;
          else const_cast<int32_t*>(p.ms.q)[c - E] = tot;
        }
      }
      __syncthreads();
      OPEN_STAMP(3);
      if (blockIdx.x == 0) meta_send_block(p.ms);  // the peers' flags travel while the ranks are computed
      OPEN_STAMP(4);
      block_rank8(tk, bc, p.K, E, N, p.L, sm, s_base, nullptr, nullptr, ranks, slots, lst);
    }
  } else {
    // one chunk (final m / q directly), or top-k > 8: per-chunk layouts, a
    // column prefix over the chunks between two grid barriers, then the
    // chunk bases added to the ranks and slots
    int32_t* m_out = G == 1 ? const_cast<int32_t*>(p.ms.m) : h;
    int32_t* q_out = G == 1 ? const_cast<int32_t*>(p.ms.q) : h + E;
    if (!block_layout_checked(tk, bc, p.K, E, N, p.L, sm, m_out, q_out, ranks, slots, lst) && threadIdx.x == 0)
      raise_err(p.mr.err, EPB_INVALID_ARGUMENT);
    OPEN_STAMP(1);
    if (G > 1) grid_arrive_wait(p.bar, G);
    else __syncthreads();
    OPEN_STAMP(2);
    if (G > 1) {
      const int lane = threadIdx.x & 31;
      for (int c = blockIdx.x * nw + (threadIdx.x >> 5); c < C; c += G * nw) {
        int carry = 0;
        for (int j0 = 0; j0 < G; j0 += 32) {
          const int j = j0 + lane;
          const int v = j < G ? __ldcg(&p.hist[(int64_t)j * C + c]) : 0;
          int incl = v;
          for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
          }
          if (j < G) p.hist[(int64_t)j * C + c] = carry + incl - v;
          carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
          if (c < E) const_cast<int32_t*>(p.ms.m)[c] = carry;
          else const_cast<int32_t*>(p.ms.q)[c - E] = carry;
        }
      }
      grid_arrive_wait(p.bar, 2 * G);
    }
    OPEN_STAMP(3);
    bad = *reinterpret_cast<const volatile int*>(p.mr.err) != 0;
    if (!bad && bc > 0 && G > 1) {
      const int32_t* base = p.hist + (int64_t)blockIdx.x * C;
      for (int i = threadIdx.x; i < bc * p.K; i += blockDim.x) {
        const int e = (int)tk[i];
        ranks[i] += __ldcg(&base[e]);
      }
      for (int i = threadIdx.x; i < bc * N; i += blockDim.x) {
        const int v = slots[i];
        if (v >= 0) slots[i] = v + __ldcg(&base[E + i % N]);
      }
    }
    __syncthreads();
    if (blockIdx.x == 0 && !bad) meta_send_block(p.ms);
    OPEN_STAMP(4);
  }
  // (4) CTA 0: every source's metadata row, the offsets and the receive
  // shapes (a rejected routing sent nothing and waits for nothing)
  OPEN_STAMP(5);
  if (blockIdx.x == 0) {
    if (!bad) {
      OPEN_STAMP(6);
      meta_recv_block(p.mr, smem);
    }
    __syncthreads();
    OPEN_STAMP(7);
    if (threadIdx.x == 0) {
      __threadfence();
      *reinterpret_cast<volatile int32_t*>(p.host_err) = *reinterpret_cast<const volatile int*>(p.mr.err);
    }
  }
  OPEN_STAMP(8);
  // the last CTA out resets the barrier words for the next launch
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(p.bar + 1, 1u) == (unsigned)G - 1) {
    p.bar[0] = 0u;
    p.bar[1] = 0u;
  }
}

// ---------------------------------------------------------------------------
// K5b: dispatch
// ---------------------------------------------------------------------------
struct HTSend {
  const void* x;
  uint8_t* stage;          // own window: [B][RBp] wire rows
  const float* w;
  const int64_t* topk;
  const int32_t* q;
  const int32_t* tok_rank;
  const int32_t* tok_slot;
  const int32_t* offsets;  // [E, N]
  const uint64_t* peers;
  int* done;
  HTGeom g;
  int b, rank;
  int stage_ready;  // x IS this rank's stage region in the wire dtype
  uint32_t tag;
  OpTrace ops;
};

EPB_DEV void ht_publish_records(const HTSend& p, int d) {
  uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, d) + p.g.dflag) + p.rank;
  const uint64_t v = ((uint64_t)p.tag << 32) | (uint32_t)p.q[d];
  st_relaxed_sys_u64(flag, v);
  op_record(p.ops, EPB_OP_SIGNAL, p.rank, d, p.g.dflag + 8ull * p.rank, 8, 2 * p.g.N + p.rank, v);
}

// Send: (1) every token row, converted once to the wire dtype, into this
// rank's own stage (a flat streaming copy, 4 x 16 B in flight per thread);
// (2) one record (weights, header, output positions) per (token, rank it
// touches) — this rank included — into that rank's window, a warp per
// token; (3) per destination, the last CTA to finish publishes the flag
// (tag | record count) after a system-scope release.
template <int XT, int WT>
__global__ void __launch_bounds__(kHTThreads) ht_dispatch_send_kernel(HTSend p) {
  const HTGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L;
  const int me = p.rank;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // (1) stage (skipped when the caller wrote the tokens into the stage
  // region itself: zero-copy input)
  if (p.stage_ready) {
  } else if ((H % EPC) == 0 && g.RBp == H * (int)sizeof(uint16_t) * (WT == EPB_F32 ? 2 : 1)) {
    const int64_t nq = (int64_t)p.b * (H / EPC);
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    const uint8_t* xb = reinterpret_cast<const uint8_t*>(p.x);
    for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < nq; q0 += 4 * gs) {
      float f[4][EPC];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * gs;
        if (q < nq) load_elems_vec<XT, EPC>(xb, q * EPC, f[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * gs;
        if (q < nq) st_plain_v4(p.stage + q * 16, pack16<WT>(f[u]));
      }
    }
  } else {
    for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
      const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * XW;
      for (int el = threadIdx.x; el < H; el += blockDim.x)
        store_elem(p.stage + (int64_t)t * g.RBp, WT, el, load_elem(xrow, XT, el));
    }
  }
  // (2) records: lane k holds (e_k, w_k, pos_k), lane d < N (and d + 32)
  // the token's slot at rank d.  The record image [K f32 weights | t, K,
  // e[K], pos[K]] is the same for every destination: lane l builds its
  // 16-B piece once, then one vector store per lane per destination.
  const int nvec = g.rec_stride / 16;  // <= 25 (K <= 32)
  const int wq = g.WBp / 4;            // header word offset
  const int64_t rec0 = (int64_t)me * g.B;
  for (int t = blockIdx.x * nw + warp; t < p.b; t += gridDim.x * nw) {
    int e = 0, pos = 0;
    float wk = 0.0f;
    if (lane < K) {
      const int64_t i = (int64_t)t * K + lane;
      e = (int)p.topk[i];
      wk = p.w[i];
      pos = p.offsets[e * N + me] + p.tok_rank[i];
    }
    const int slot_lo = lane < N ? p.tok_slot[(int64_t)t * N + lane] : -1;
    const int slot_hi = lane + 32 < N ? p.tok_slot[(int64_t)t * N + lane + 32] : -1;
    uint32_t img[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int wi = 4 * lane + u;
      const int h = wi - wq;
      const int src = wi < wq ? wi : (h >= 2 && h < 2 + K ? h - 2 : (h >= 2 + K ? h - 2 - K : 0));
      const float wv = __shfl_sync(0xffffffffu, wk, src & 31);
      const int ev = __shfl_sync(0xffffffffu, e, src & 31);
      const int pv = __shfl_sync(0xffffffffu, pos, src & 31);
      uint32_t v = 0;
      if (wi < wq) v = wi < K ? __float_as_uint(wv) : 0u;
      else if (h == 0) v = (uint32_t)t;
      else if (h == 1) v = (uint32_t)K;
      else if (h < 2 + K) v = (uint32_t)ev;
      else if (h < 2 + 2 * K) v = (uint32_t)pv;
      img[u] = v;
    }
    const int4 piece = make_int4((int)img[0], (int)img[1], (int)img[2], (int)img[3]);
    for (int d = 0; d < N; ++d) {
      const int j = __shfl_sync(0xffffffffu, d < 32 ? slot_lo : slot_hi, d & 31);
      if (j < 0) continue;
      uint8_t* rec = hpeer(p.peers, d) + g.rec + (rec0 + j) * g.rec_stride;
      if (lane < nvec) st_plain_v4(rec + 16 * lane, piece);
      if (lane == 0) op_record(p.ops, EPB_OP_PUT, me, d, g.rec + (uint64_t)(rec0 + j) * g.rec_stride, 16ull * nvec);
    }
  }
  (void)L;
  // (3) publish: every CTA releases its stage rows and records at GPU scope
  // and counts in; the last one issues the rank's single system-scope
  // release (cumulative over all CTAs' stores) and flags every destination
  __syncthreads();
  if (threadIdx.x == 0) {
    chaos_delay(g.chaos_ns, 0x33u);
    fence_release(false);
    if (atomicAdd(p.done, 1) == (int)gridDim.x - 1) {
      *p.done = 0;
      fence_release(p.g.sys_fence);
      for (int d = 0; d < N; ++d)
        if (d != me) ht_publish_records(p, d);
    }
  }
}

struct HTRecv {
  const uint64_t* peers;  // rows are pulled from each source's stage
  const int32_t* q;       // this rank's own record count is q[rank]
  void* out;
  int32_t* origin;
  float* origin_w;
  const uint8_t* win;
  int* err;
  HTGeom g;
  uint64_t timeout_ns;
  int rank;
  uint32_t tag;
  OpTrace ops;
  int stages;  // bulk receive: ring depth per warp (<= kMaxStages)
};

// Receive: every record names a source token and the output rows of this
// rank's experts it feeds; the warp reads the header once, pulls the row
// from the source's stage (over NVLink, or locally for this rank's own
// tokens) once, and stores it to each of those rows (the local fan-out of
// ht.py:553-583).  Remote sources are visited in the order me+1, me+2, ...
// so every source's stage is read by a different receiver at a time; a
// share of the warps (1/N) handles this rank's own records concurrently.
template <int WT, int OT>
__global__ void __launch_bounds__(kHTThreads) ht_dispatch_recv_kernel(HTRecv p) {
  __shared__ int s_pre[kMaxRanks + 1], s_q[kMaxRanks];
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H, L = g.L;
  const int me = p.rank;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.dflag);
  bool fail = false;
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v = 0;
    if (s != me) fail |= !wait_tag(&flags[s], p.tag, 32, 0xFFFFFFFFu, p.timeout_ns, p.err, &v);
    s_q[s] = s == me ? p.q[me] : (int)(v & 0xFFFFFFFFu);
  }
  if (__syncthreads_or(fail)) return;
  // remote records interleaved over the sources in chunks of kRC: chunk c
  // reads source me+1+(c % (N-1)), its chunk c / (N-1), so every source's
  // stage is read by all receivers at an even rate for the whole phase
  constexpr int kRC = 32;
  __shared__ int s_maxq;
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int s2 = 0; s2 < N; ++s2)
      if (s2 != me) mx = max(mx, s_q[s2]);
    s_maxq = mx;
  }
  __syncthreads();
  const int lo = me * L, hi = min(lo + L, g.E);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // warps [0, sw) take this rank's own records, the rest the remote ones
  const int sw = N == 1 ? nw : max(1, nw / N);
  const bool self_warp = warp < sw;
  const int nrs = max(1, N - 1);
  const int rchunks = (s_maxq + kRC - 1) / kRC;
  const int items = self_warp ? 2 * s_q[me] : 2 * rchunks * nrs * kRC;
  const int wi = self_warp ? warp : warp - sw;
  const int wn = self_warp ? sw : nw - sw;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  constexpr int EPC = Elems<WT>::n;
  for (int f2 = wi * gridDim.x + blockIdx.x; f2 < items; f2 += gridDim.x * wn) {
    const int rj = f2 >> 1, half = f2 & 1;
    int s, j;
    if (self_warp) {
      s = me;
      j = rj;
    } else {
      const int c = rj / kRC, w = rj - c * kRC;
      s = (me + 1 + c % nrs) % N;
      j = (c / nrs) * kRC + w;
      if (j >= s_q[s]) continue;  // that source has fewer records
    }
    const uint8_t* rec = p.win + g.rec + ((int64_t)s * g.B + j) * g.rec_stride;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec + g.WBp);
    const uint8_t* row = hpeer(p.peers, s) + g.stage + (int64_t)hdr[0] * g.RBp;
    if (half == 0 && lane == 0)  // one record per row pulled from the source's stage
      op_record(p.ops, EPB_OP_GET, me, s, g.stage + (uint64_t)hdr[0] * g.RBp, (uint64_t)g.RB);
    int e = -1, pos = 0;
    if (lane < K) {
      e = (int)hdr[2 + lane];
      pos = (int)hdr[2 + K + lane];
    }
    const bool loc = lane < K && e >= lo && e < hi;
    const unsigned lm = __ballot_sync(0xffffffffu, loc);
    if (half == 0 && loc) {
      p.origin[(int64_t)pos * 4 + 0] = e;
      p.origin[(int64_t)pos * 4 + 1] = s;
      p.origin[(int64_t)pos * 4 + 2] = (int32_t)hdr[0];
      p.origin[(int64_t)pos * 4 + 3] = lane;
      p.origin_w[pos] = reinterpret_cast<const float*>(rec)[lane];
    }
    if ((H & 15) == 0) {
      const int nch = H / EPC;
      const int per = (nch + 1) / 2;
      const int c0 = half * per, c1 = min(nch, c0 + per);
      for (int base = c0; base < c1; base += 32 * kHU) {
        int4 v[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) v[u] = ld_plain_v4(row + (int64_t)c * 16);
        }
        for (unsigned mm = lm; mm; mm &= mm - 1) {
          const int kk = __ffs(mm) - 1;
          uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)__shfl_sync(0xffffffffu, pos, kk) * H * OW;
#pragma unroll
          for (int u = 0; u < kHU; ++u) {
            const int c = base + u * 32 + lane;
            if (c < c1) {
              if constexpr (OT == WT) {
                st_plain_v4(orow + (int64_t)c * 16, v[u]);
              } else {
                float fv[EPC];
                unpack16<WT>(v[u], fv);
                store_f32_chunk<OT, EPC>(orow, (int64_t)c * EPC, fv);
              }
            }
          }
        }
      }
    } else if (half == 0) {
      for (unsigned mm = lm; mm; mm &= mm - 1) {
        const int kk = __ffs(mm) - 1;
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)__shfl_sync(0xffffffffu, pos, kk) * H * OW;
        for (int el = lane; el < H; el += 32) store_elem(orow, OT, el, load_elem(row, WT, el));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Dispatch receive through the bulk-copy (TMA) engine: per warp, record
// half-rows are pulled with cp.async.bulk global->shared (completion on an
// mbarrier) into a 2-stage ring and written to every local expert's row with
// cp.async.bulk shared->global — no registers hold payload, so an SM keeps
// 2 x 8 half-rows (~112 KB at H=7168 bf16) in flight.  Same items and
// outputs as ht_dispatch_recv_kernel (wire-dtype output only).
// ---------------------------------------------------------------------------
constexpr int kBulkWarps = 8;
constexpr int kMaxStages = 4;  // row-load ring depth per warp (HTRecv::stages)

EPB_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
EPB_DEV void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
EPB_DEV void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
EPB_DEV bool mbar_try_wait(uint64_t* m, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(m)), "r"(parity)
      : "memory");
  return ok != 0;
}
EPB_DEV void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
EPB_DEV void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}
EPB_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
EPB_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
EPB_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(kBulkWarps * 32) ht_dispatch_recv_bulk_kernel(HTRecv p) {
  extern __shared__ __align__(128) uint8_t s_buf[];  // [warps][stages][hb] then [warps][kMaxStages] mbarriers
  __shared__ int s_ring[kBulkWarps][kMaxStages];       // item held by each stage, in issue order
  __shared__ int s_q[kMaxRanks];
  __shared__ int s_maxq;
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, L = g.L;
  const int me = p.rank;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t hb = (uint32_t)g.RBp / 2;
  const int S = p.stages;
  uint8_t* buf = s_buf + (size_t)warp * S * hb;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_buf + (size_t)nw * S * hb) + warp * kMaxStages;
  if (lane == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // the mbarrier initialisation
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.dflag);
  bool fail = false;
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v = 0;
    if (s != me) fail |= !wait_tag(&flags[s], p.tag, 32, 0xFFFFFFFFu, p.timeout_ns, p.err, &v);
    s_q[s] = s == me ? p.q[me] : (int)(v & 0xFFFFFFFFu);
  }
  if (__syncthreads_or(fail)) return;
  // the staged rows were acquired through generic loads; the bulk copies
  // read them through the async proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int s = 0; s < N; ++s) mx = max(mx, s_q[s]);
    s_maxq = mx;
  }
  __syncthreads();
  // items: (chunk of kRC records, round-robin over the sources me+1, ...,
  // me+N-1, me) x half rows
  constexpr int kRC = 32;
  const int rchunks = (s_maxq + kRC - 1) / kRC;
  const int items = 2 * rchunks * N * kRC;
  const int lo = me * L, hi = min(lo + L, g.E);
  auto resolve = [&](int f2, int& s, int& j) {
    const int rj = f2 >> 1, c = rj / kRC, w = rj - c * kRC;
    s = (me + 1 + c % N) % N;
    j = (c / N) * kRC + w;
    return j < s_q[s];
  };
  auto next_item = [&](int f2) {
    int s, j;
    for (; f2 < items; f2 += gridDim.x * nw)
      if (resolve(f2, s, j)) return f2;
    return items;
  };
  // an S-stage ring per warp: S-1 row loads in flight ahead of the item
  // being fanned out (the NVLink round trip is hidden behind S-1 items)
  uint32_t phase = 0u;  // bit st: parity of stage st's next completion
  auto issue = [&](int f2, int stg) {
    int s, j;
    resolve(f2, s, j);
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(p.win + g.rec + ((int64_t)s * g.B + j) * g.rec_stride + g.WBp);
    if (lane == 0) {
      const uint8_t* row = hpeer(p.peers, s) + g.stage + (int64_t)hdr[0] * g.RBp + (f2 & 1) * hb;
      mbar_expect_tx(&bar[stg], hb);
      bulk_load(buf + stg * hb, row, hb, &bar[stg]);
      s_ring[warp][stg] = f2;
    }
  };
  const int stride = gridDim.x * nw;
  int nxt = next_item(warp * gridDim.x + blockIdx.x);
  int head = 0, tail = 0;  // items fanned out / issued
  while (tail < S - 1 && nxt < items) {
    issue(nxt, tail % S);
    nxt = next_item(nxt + stride);
    ++tail;
  }
  while (head < tail) {
    const int stg = head % S;
    // the previous item's stores must have read its stage before it is refilled
    bulk_wait_read_all();
    __syncwarp();
    if (nxt < items) {
      issue(nxt, tail % S);
      nxt = next_item(nxt + stride);
      ++tail;
    }
    __syncwarp();
    const int cur = s_ring[warp][stg];
    int s, j;
    resolve(cur, s, j);
    const int half = cur & 1;
    const uint8_t* rec = p.win + g.rec + ((int64_t)s * g.B + j) * g.rec_stride;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec + g.WBp);
    if (half == 0 && lane == 0)  // one record per row pulled from the source's stage
      op_record(p.ops, EPB_OP_GET, me, s, g.stage + (uint64_t)hdr[0] * g.RBp, (uint64_t)g.RB);
    int e = -1, pos = 0;
    if (lane < K) {
      e = (int)hdr[2 + lane];
      pos = (int)hdr[2 + K + lane];
    }
    const bool loc = lane < K && e >= lo && e < hi;
    if (half == 0 && loc) {
      p.origin[(int64_t)pos * 4 + 0] = e;
      p.origin[(int64_t)pos * 4 + 1] = s;
      p.origin[(int64_t)pos * 4 + 2] = (int32_t)hdr[0];
      p.origin[(int64_t)pos * 4 + 3] = lane;
      p.origin_w[pos] = reinterpret_cast<const float*>(rec)[lane];
    }
    while (!mbar_try_wait(&bar[stg], (phase >> stg) & 1u)) {
    }
    phase ^= 1u << stg;
    if (loc) {
      bulk_store(reinterpret_cast<uint8_t*>(p.out) + (int64_t)pos * g.RBp + half * hb, buf + stg * hb, hb);
      bulk_commit();
    }
    ++head;
  }
  bulk_wait_all();
}

// ---------------------------------------------------------------------------
// K6: combine
// ---------------------------------------------------------------------------
struct HTCombSend {
  const void* y;
  const int* err;        // a failed validation (weights) aborts before any traffic
  const int32_t* origin;
  const int32_t* meta;  // [N][E+N] (m rows)
  const uint64_t* peers;
  int* done;
  // receive row table (filled here, read by the receive phase)
  const int64_t* topk;
  const int32_t* tok_rank;
  const int32_t* offsets;
  const uint8_t* win;
  uint64_t* row_ptr;
  HTGeom g;
  int rows, rank, in_dtype, b;
  int pull;  // expert rows are this rank's window region: homes pull them
  uint32_t tag;
  OpTrace ops;
};

EPB_DEV int ht_rows_to(const HTCombSend& p, int s) {
  const int C = p.g.E + p.g.N;
  const int lo = p.rank * p.g.L, hi = min(lo + p.g.L, p.g.E);
  int c = 0;
  for (int e = lo; e < hi; ++e) c += p.meta[s * C + e];
  return c;
}

EPB_DEV void ht_publish_comb(const HTCombSend& p, int s, int count) {
  uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, s) + p.g.cflag) + p.rank;
  const uint64_t v = ((uint64_t)p.tag << 32) | ((uint64_t)p.in_dtype << 28) | (uint32_t)count;
  st_relaxed_sys_u64(flag, v);
  op_record(p.ops, EPB_OP_SIGNAL, p.rank, s, p.g.cflag + 8ull * p.rank, 8, 3 * p.g.N + p.rank, v);
}

template <int IT>
__global__ void __launch_bounds__(kHTThreads) ht_combine_send_kernel(HTCombSend p) {
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H;
  const int me = p.rank;
  if (*reinterpret_cast<const volatile int*>(p.err) != 0) return;
  constexpr int ib = IT == EPB_F32 ? 4 : 2;
  const int bytes = H * ib;
  if (p.row_ptr) {
    // address of every (t, k) row the receive phase reduces: own experts'
    // rows in place in the expert output, the others in the combine slots
    const int L = g.L;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.b * K; i += gridDim.x * blockDim.x) {
      const int e = (int)p.topk[i];
      const uint64_t srow = (uint64_t)(p.offsets[e * N + me] + p.tok_rank[i]);  // row on owner(e)
      if (p.pull) {  // the owner's registered expert-output region, read over NVLink
        p.row_ptr[i] = reinterpret_cast<uint64_t>(hpeer(p.peers, e / L) + g.yout) + srow * g.yrow;
        if (e / L != me)  // the receive phase of this op reads it: one record per remote row
          op_record(p.ops, EPB_OP_GET, me, e / L, g.yout + srow * g.yrow, (uint64_t)bytes);
      }
      else
        p.row_ptr[i] = e / L == me ? reinterpret_cast<uint64_t>(p.y) + srow * bytes
                                   : reinterpret_cast<uint64_t>(p.win + g.crow + (int64_t)i * g.crow_stride);
    }
  }
  if (p.pull) {
    // nothing moves: announce that this rank's expert rows are complete
    // (written by earlier kernels on this stream) to every home rank
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      fence_release(p.g.sys_fence);
      for (int s2 = 0; s2 < N; ++s2)
        if (s2 != me) ht_publish_comb(p, s2, 0);
    }
    return;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nch = (bytes & 15) == 0 ? bytes / 16 : 0;
  // warp tasks: (row, half); rows of my own tokens stay (the home reads them in place)
  for (int task = warp * gridDim.x + blockIdx.x; task < 2 * p.rows; task += gridDim.x * nw) {
    const int r = task >> 1, half = task & 1;
    const int s = p.origin[(int64_t)r * 4 + 1];
    if (s == me) continue;
    const int t = p.origin[(int64_t)r * 4 + 2];
    const int k = p.origin[(int64_t)r * 4 + 3];
    uint8_t* dst = hpeer(p.peers, s) + g.crow + ((int64_t)t * K + k) * g.crow_stride;
    if (half == 0 && lane == 0)  // one record per expert row pushed to its token's home
      op_record(p.ops, EPB_OP_PUT, me, s, g.crow + (uint64_t)((int64_t)t * K + k) * g.crow_stride, (uint64_t)bytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.y) + (int64_t)r * bytes;
    if (nch) {
      const int per = (nch + 1) / 2;
      const int c0 = half * per, c1 = min(nch, c0 + per);
      for (int base = c0; base < c1; base += 32 * kHU) {
        int4 v[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) v[u] = ld_nc_v4(src + (int64_t)c * 16);
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) st_na_v4(dst + (int64_t)c * 16, v[u]);
        }
      }
    } else if (half == 0) {
      for (int c = lane; c < bytes / 2; c += 32)
        reinterpret_cast<uint16_t*>(dst)[c] = reinterpret_cast<const uint16_t*>(src)[c];
    }
  }
  // publish: one GPU-scope release per CTA, the last CTA's system-scope
  // release covers them all, then every home rank is flagged
  __syncthreads();
  if (threadIdx.x == 0) {
    chaos_delay(g.chaos_ns, 0x35u);
    fence_release(false);
    if (atomicAdd(p.done, 1) == (int)gridDim.x - 1) {
      *p.done = 0;
      fence_release(p.g.sys_fence);
      for (int s2 = 0; s2 < N; ++s2)
        if (s2 != me) ht_publish_comb(p, s2, ht_rows_to(p, s2));
    }
  }
}

struct HTCombRecv {
  int rows_local;            // every row is in this GPU's memory (push mode, or one rank)
  const int64_t* topk;
  const uint64_t* row_ptr;   // [b*K] from the send phase, or null
  const float* w;
  const void* y_local;       // this rank's expert rows [recv_total, H] (own tokens read in place)
  const int32_t* tok_rank;   // [b, K]
  const int32_t* offsets;    // [E, N]
  void* out;
  const uint8_t* win;
  int* err;
  HTGeom g;
  uint64_t timeout_ns;
  int b, rank, y_dtype;
  uint32_t tag;
};

// Single-node bf16 reduce with the row loads in flight through cp.async
// (shared memory, not registers): each warp keeps kCS tasks (token, 32
// chunks of 8 elements; K <= 8 rows of 512 B) in flight, so an SM has
// 16 warps x kCS x 4 KB of peer / local loads outstanding.  Each lane only
// consumes the chunks it copied itself: wait_group, no warp barrier.
// Order: acc = p_0, acc = fl(acc + p_k) ascending k, out = fl(0 + acc).
constexpr int kCS = 3;  // pipeline depth (tasks per warp in flight)

EPB_DEV void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
EPB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
EPB_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int OT>
EPB_DEV void ht_combine_reduce_async(const HTCombRecv& p, int K, int H, int warp, int lane, int nw) {
  extern __shared__ int4 s_stage[];  // [nw][kCS][8 rows][32 lanes]
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  int4* my = s_stage + (int64_t)warp * kCS * 8 * 32;
  const int nch = H / 8;
  const int segs = (nch + 31) / 32;
  const int tasks = p.b * segs;
  const int tstride = gridDim.x * nw;
  const int first = warp * gridDim.x + blockIdx.x;
  // per stage: lane k's weight, the task's token/chunk
  float sw[kCS];
  int st[kCS], sc[kCS];
  auto issue = [&](int task, int stg) {
    if (task < tasks) {
      const int t = task / segs, c = (task - t * segs) * 32 + lane;
      uint64_t row = 0;
      float w = 0.0f;
      if (lane < K) {
        row = p.row_ptr[(int64_t)t * K + lane];
        w = p.w[(int64_t)t * K + lane];
      }
      sw[stg] = w;
      st[stg] = t;
      sc[stg] = c;
      for (int k = 0; k < K; ++k) {
        const uint64_t rk = __shfl_sync(0xffffffffu, row, k);
        if (c < nch) cp_async16(&my[(stg * 8 + k) * 32 + lane], reinterpret_cast<const uint8_t*>(rk) + (int64_t)c * 16);
      }
    }
    cp_async_commit();  // (an empty group keeps the wait_group arithmetic uniform)
  };
#pragma unroll
  for (int i = 0; i < kCS - 1; ++i) issue(first + i * tstride, i);
  // stages rotate with the unrolled q, so every stage index is a constant
  for (int task0 = first; task0 < tasks; task0 += kCS * tstride) {
#pragma unroll
    for (int q = 0; q < kCS; ++q) {
      const int task = task0 + q * tstride;
      issue(task + (kCS - 1) * tstride, (q + kCS - 1) % kCS);
      cp_async_wait<kCS - 1>();  // this task's copies (this lane's) are in
      if (task < tasks) {
        const int t = st[q], c = sc[q];
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        for (int k = 0; k < K; ++k) {
          const float wk = __shfl_sync(0xffffffffu, sw[q], k);
          float y[8];
          unpack16<EPB_BF16>(my[(q * 8 + k) * 32 + lane], y);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float pk = __fmul_rn(wk, y[i]);
            acc[i] = k == 0 ? pk : __fadd_rn(acc[i], pk);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(0.0f, acc[i]);
        if (c < nch)
          store_f32_chunk<OT, 8>(reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * OW, (int64_t)c * 8, acc);
      }
    }
  }
  cp_async_wait<0>();
}

// 8 consecutive elements (chunk c) of a row in dtype IT, as f32
template <int IT>
EPB_DEV void ht_load8(const uint8_t* row, int c, float* y) {
  if constexpr (IT == EPB_F32) {
    unpack16<EPB_F32>(ld_plain_v4(row + (int64_t)c * 32), y);
    unpack16<EPB_F32>(ld_plain_v4(row + (int64_t)c * 32 + 16), y + 4);
  } else {
    unpack16<EPB_BF16>(ld_plain_v4(row + (int64_t)c * 16), y);
  }
}

template <int IT, int OT>
__global__ void __launch_bounds__(kHTThreads, 1) ht_combine_recv_kernel(HTCombRecv p) {
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H, L = g.L;
  const int me = p.rank;
  constexpr int YB = IT == EPB_F32 ? 4 : 2;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  if (__syncthreads_or(threadIdx.x == 0 && *reinterpret_cast<const volatile int*>(p.err) != 0)) return;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.cflag);
  bool fail = false;
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v = 0;
    if (s == me) continue;
    if (!wait_tag(&flags[s], p.tag, 32, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) { fail = true; continue; }
    // every rank must combine in the same dtype (the rows are raw bytes)
    if ((int)((v >> 28) & 0xF) != IT) { raise_err(p.err, EPB_TAG_MISMATCH); fail = true; }
  }
  if (__syncthreads_or(fail)) return;
  const uint8_t* crow = p.win + g.crow;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool one_node = g.rpn == N;
  if constexpr (IT == EPB_BF16) {
    // (cp.async from peer memory measured ~2.4x slower than register loads:
    // the async path only runs when every row is local)
    if (one_node && p.rows_local && p.row_ptr && K <= 8 && (H & 7) == 0) {
      ht_combine_reduce_async<OT>(p, K, H, warp, lane, nw);
      return;
    }
  }
  if ((H & 7) == 0 && K <= 32) {
    // warp tasks: (token, 32-chunk segment of 8 elements); lane = one chunk.
    // Lane k first resolves row k of the token (own expert rows are read in
    // place from the local expert output, others from the combine slots).
    const int nch = H / 8;
    const int segs = (nch + 31) / 32;
    const int tstride = gridDim.x * nw;
    int task = warp * gridDim.x + blockIdx.x;
    // lane k's row of a task's token: the send phase's table (one load,
    // prefetched a task ahead) or resolved from the routing
    uint64_t my_row = 0;
    float my_w = 0.0f;
    int my_node = 0;
    auto fetch = [&](int tk) {
      if (lane < K) {
        const int64_t i = (int64_t)tk * K + lane;
        my_w = p.w[i];
        if (p.row_ptr) my_row = p.row_ptr[i];
        if (!one_node || !p.row_ptr) {
          const int e = (int)p.topk[i];
          const int owner = e / L;
          my_node = owner / g.rpn;
          if (!p.row_ptr)
            my_row = owner == me
                ? reinterpret_cast<uint64_t>(p.y_local) + (uint64_t)(p.offsets[e * N + me] + p.tok_rank[i]) * H * YB
                : reinterpret_cast<uint64_t>(crow + i * g.crow_stride);
        }
      }
    };
    if (task < p.b * segs) fetch(task / segs);
    for (; task < p.b * segs; task += tstride) {
      const int t = task / segs, c = (task - t * segs) * 32 + lane;
      const uint64_t cur_row = my_row;
      const float cur_w = my_w;
      const int cur_node = my_node;
      if (task + tstride < p.b * segs) fetch((task + tstride) / segs);  // next task's rows, in flight now
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
      if (one_node) {
        // single node: acc = p_0 + p_1 + ... (first present as init), then
        // out = 0 + acc; all KB rows of a batch are in flight at once
        constexpr int KB = IT == EPB_F32 ? 4 : 8;  // rows in flight per lane
        constexpr int NV = IT == EPB_F32 ? 2 : 1;  // 16-B loads per 8-element chunk
        for (int k0 = 0; k0 < K; k0 += KB) {
          int4 v[KB][NV];
          float wk[KB];
#pragma unroll
          for (int u = 0; u < KB; ++u) {
            const uint64_t row = __shfl_sync(0xffffffffu, cur_row, (k0 + u) & 31);
            wk[u] = __shfl_sync(0xffffffffu, cur_w, (k0 + u) & 31);
            if (k0 + u < K && c < nch) {
#pragma unroll
              for (int q = 0; q < NV; ++q)
                v[u][q] = ld_plain_v4(reinterpret_cast<const uint8_t*>(row) + (int64_t)c * 16 * NV + 16 * q);
            }
          }
#pragma unroll
          for (int u = 0; u < KB; ++u) {
            const int k = k0 + u;
            if (k < K) {
              float y[8];
              if constexpr (IT == EPB_F32) {
                unpack16<EPB_F32>(v[u][0], y);
                unpack16<EPB_F32>(v[u][1], y + 4);
              } else {
                unpack16<EPB_BF16>(v[u][0], y);
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float pk = __fmul_rn(wk[u], y[i]);
                acc[i] = k == 0 ? pk : __fadd_rn(acc[i], pk);
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(0.0f, acc[i]);
      } else {
        // several nodes: ascending node, per node first-present then ascending k
        int prev = -1;
        for (;;) {
          int nd = 0x7fffffff;
          for (int k = 0; k < K; ++k) {
            const int n2 = __shfl_sync(0xffffffffu, cur_node, k);
            if (n2 > prev && n2 < nd) nd = n2;
          }
          if (nd == 0x7fffffff) break;
          float part[8];
          bool started = false;
          for (int k = 0; k < K; ++k) {
            const int n2 = __shfl_sync(0xffffffffu, cur_node, k);
            const uint64_t row = __shfl_sync(0xffffffffu, cur_row, k);
            const float wk = __shfl_sync(0xffffffffu, cur_w, k);
            if (n2 != nd) continue;
            float y[8];
            if (c < nch) ht_load8<IT>(reinterpret_cast<const uint8_t*>(row), c, y);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float pk = __fmul_rn(wk, y[i]);
              part[i] = started ? __fadd_rn(part[i], pk) : pk;
            }
            started = true;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], part[i]);
          prev = nd;
        }
      }
      if (c < nch) store_f32_chunk<OT, 8>(reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * OW, (int64_t)c * 8, acc);
    }
  } else {
    // hidden not a multiple of 8: element path, one CTA per token
    for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
      for (int el = threadIdx.x; el < H; el += blockDim.x) {
        float acc = 0.0f;
        int prev = -1;
        for (;;) {
          int nd = 0x7fffffff;
          for (int k = 0; k < K; ++k) {
            const int n2 = ((int)p.topk[(int64_t)t * K + k] / L) / g.rpn;
            if (n2 > prev && n2 < nd) nd = n2;
          }
          if (nd == 0x7fffffff) break;
          float part = 0.0f;
          bool started = false;
          for (int k = 0; k < K; ++k) {
            const int e = (int)p.topk[(int64_t)t * K + k];
            const int owner = e / L;
            if (owner / g.rpn != nd) continue;
            const uint8_t* row = owner == me
                ? reinterpret_cast<const uint8_t*>(p.y_local) +
                      (int64_t)(p.offsets[e * N + me] + p.tok_rank[(int64_t)t * K + k]) * H * YB
                : crow + ((int64_t)t * K + k) * g.crow_stride;
            const float pk = __fmul_rn(p.w[(int64_t)t * K + k], load_elem(row, IT, el));
            part = started ? __fadd_rn(part, pk) : pk;
            started = true;
          }
          acc = __fadd_rn(acc, part);
          prev = nd;
        }
        store_elem(reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * OW, OT, el, acc);
      }
    }
  }
}

__global__ void weights_equal_kernel(const float* a, const float* b, int64_t n, int* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (__float_as_uint(a[i]) != __float_as_uint(b[i]) && !(a[i] == b[i])) raise_err(err, EPB_INVALID_ARGUMENT);
}

}  // namespace epb

using namespace epb;

namespace {

uint32_t ht_tag(uint32_t round) { return (round % 0xFFFFFFFu) + 1u; }

int hsm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int check_ht(epb_group* g, int phases) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (g->cfg.algorithm != EPB_HT) return fail(EPB_HANDLE_STATE_ERROR, "group is not HT");
  if (!g->peers_ready) return fail(EPB_HANDLE_STATE_ERROR, "peer windows not mapped");
  if (phases < 1 || phases > 3) return fail(EPB_INVALID_ARGUMENT, "phases must be 1 (send), 2 (recv) or 3");
  return EPB_OK;
}

template <int XT, int WT>
cudaError_t launch_hsend(const HTSend& p, cudaStream_t s) {
  ht_dispatch_send_kernel<XT, WT><<<2 * hsm_count(), kHTThreads, 0, s>>>(p);
  return cudaGetLastError();
}

template <int XT>
cudaError_t launch_hsend_x(const HTSend& p, int out_dtype, cudaStream_t s) {
  (void)out_dtype;
  switch (p.g.wire) {
    case EPB_F32: return launch_hsend<XT, EPB_F32>(p, s);
    case EPB_BF16: return launch_hsend<XT, EPB_BF16>(p, s);
    default: return launch_hsend<XT, EPB_F16>(p, s);
  }
}

template <int WT, int OT>
cudaError_t launch_hrecv(const HTRecv& p, cudaStream_t s) {
  // wire-dtype output, half rows of 16-B multiples: the bulk-copy receive
  static const int bulk = [] { const char* v = getenv("EPB_HT_BULK"); return v ? atoi(v) : 1; }();
  // ring depth: EPB_HT_STAGES (default 2: 3 measured no faster at C3, N=1/2), as deep as 220 KB of
  // shared memory allows
  static const int want = [] { const char* v = getenv("EPB_HT_STAGES"); return v ? atoi(v) : 2; }();
  const size_t hb = (size_t)p.g.RBp / 2;
  int stages = std::max(2, std::min(want, kMaxStages));
  auto bytes = [&](int st) { return (size_t)kBulkWarps * st * hb + (size_t)kBulkWarps * kMaxStages * 8; };
  while (stages > 2 && bytes(stages) > 220 * 1024) --stages;
  const size_t bsm = bytes(stages);
  if (bulk && OT == WT && p.g.RB == p.g.RBp && (p.g.RBp % 32) == 0 && bsm <= 220 * 1024 && p.g.K <= 32) {
    cudaError_t e = cudaFuncSetAttribute(ht_dispatch_recv_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bsm);
    if (e != cudaSuccess) return e;
    HTRecv q = p;
    q.stages = stages;
    ht_dispatch_recv_bulk_kernel<<<bulk * hsm_count(), kBulkWarps * 32, bsm, s>>>(q);
    return cudaGetLastError();
  }
  ht_dispatch_recv_kernel<WT, OT><<<2 * hsm_count(), kHTThreads, 0, s>>>(p);
  return cudaGetLastError();
}

bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int epb_ht_meta_send(epb_group* g, uint32_t round, const epb_layout* lay, void* stream) {
  if (int rc = check_ht(g, 1)) return rc;
  HTMetaSend p;
  p.ops = OpTrace{g->op_ring, g->op_cap};
  p.err = g->d_err; p.m = lay->expert_count; p.q = lay->rank_count; p.peers = g->d_peers; p.g = g->ht;
  p.rank = g->rank; p.parity = round & 1; p.tag = ht_tag(round);
  ht_meta_send_kernel<<<1, 256, 0, as_stream(stream)>>>(p);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

int epb_ht_meta_recv(epb_group* g, uint32_t round, int32_t* meta_out, int32_t* offsets,
                     int32_t* recv_total, void* stream) {
  if (int rc = check_ht(g, 2)) return rc;
  HTMetaRecv p;
  p.win = g->window; p.meta_out = meta_out; p.offsets = offsets; p.recv_total = recv_total;
  p.err = g->d_err; p.g = g->ht; p.timeout_ns = g->timeout_ns; p.rank = g->rank;
  p.parity = round & 1; p.tag = ht_tag(round);
  const size_t smem = sizeof(int32_t) * (g->ht.N * (g->ht.E + g->ht.N) + g->ht.E);
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "metadata too large");
  EPB_CUDA(cudaFuncSetAttribute(ht_meta_recv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ht_meta_recv_kernel<<<1, 1024, smem, as_stream(stream)>>>(p);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

int epb_ht_open(epb_group* g, uint32_t round, const int64_t* topk_idx, int32_t b, const epb_layout* lay,
                int32_t* host_meta, int32_t* offsets, void* stream) {
  if (int rc = check_ht(g, 3)) return rc;
  if (!lay || !host_meta || !offsets) return fail(EPB_INVALID_ARGUMENT, "null argument");
  if (b < 0 || b > g->cfg.max_tokens_per_rank)
    return fail(EPB_INVALID_ARGUMENT, "token count exceeds max_tokens_per_rank");
  if (!g->d_lay || !lay->tok_slot) return fail(EPB_INVALID_ARGUMENT, "layout needs per-token slots");
  const int E = g->ht.E, N = g->ht.N;
  const int C = E + N;
  // 128-token chunks, 256 threads each (one chunk: no grid barriers).
  // EPB_OPEN_SINGLE=n lays out up to n tokens in one CTA of 1024 threads
  // instead (measured slower at 4096 tokens: 44 vs 5.5 us, the per-SM
  // shared-atomic rate bounds the layout passes; tools/ht_handle_profile.py)
  static const int kOpenSingle = [] {
    const char* e = getenv("EPB_OPEN_SINGLE");
    return e ? atoi(e) : 0;
  }();
  const bool single = b <= kOpenSingle;
  int thr = single ? 1024 : 256;
  while (thr > 128 && BlockLayoutSmem::bytes(thr / 32, E, N) > 200 * 1024) thr >>= 1;
  const size_t smem = std::max(BlockLayoutSmem::bytes(thr / 32, E, N) + sizeof(int32_t) * C,
                               sizeof(int32_t) * ((size_t)N * C + E));
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "metadata too large");
  HTOpen p;
  p.topk = topk_idx; p.b = b; p.K = g->cfg.top_k; p.L = g->ht.L;
  p.chunk = single ? std::max(1, b) : kLayChunk;
  const int grid = single ? 1 : (b + kLayChunk - 1) / kLayChunk;
  p.hist = g->d_lay; p.tok_rank = lay->tok_rank; p.tok_slot = lay->tok_slot;
  p.bar = reinterpret_cast<unsigned*>(g->d_scratch) + 8;
  p.ms.err = g->d_err; p.ms.m = lay->expert_count; p.ms.q = lay->rank_count; p.ms.peers = g->d_peers;
  p.ms.g = g->ht; p.ms.rank = g->rank; p.ms.parity = round & 1; p.ms.tag = ht_tag(round);
  p.ms.ops = OpTrace{g->op_ring, g->op_cap};
  p.mr.win = g->window; p.mr.meta_out = host_meta; p.mr.offsets = offsets; p.mr.recv_total = host_meta + N * C;
  p.mr.err = g->d_err; p.mr.g = g->ht; p.mr.timeout_ns = g->timeout_ns; p.mr.rank = g->rank;
  p.mr.parity = round & 1; p.mr.tag = ht_tag(round);
  p.host_err = host_meta + N * C + 1;
  p.stamps = g->trace;
  static std::mutex mu;
  struct OpenState { size_t smem = 0; int per_sm = 0, sms = 0; };
  static std::unordered_map<int, OpenState> state;  // per device: smem opted in, co-resident CTAs
  int dev = 0;
  EPB_CUDA(cudaGetDevice(&dev));
  int cap = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    OpenState& st = state[dev];
    if (st.smem < smem) {
      EPB_CUDA(cudaFuncSetAttribute(ht_open_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      EPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&st.per_sm, ht_open_kernel, 256, smem));
      EPB_CUDA(cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev));
      st.smem = smem;
    }
    cap = st.per_sm * st.sms;
  }
  if (!single && cap < grid) return fail(EPB_CAPACITY_EXCEEDED, "routing too large for one co-resident grid");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(thr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EPB_CUDA(cudaLaunchKernelEx(&cfg, ht_open_kernel, p));
  return EPB_OK;
}

int epb_ht_dispatch(epb_group* g, uint32_t round, int32_t phases, const epb_ht_dispatch_args* a, void* stream) {
  if (int rc = check_ht(g, phases)) return rc;
  const int wire = g->cfg.token_dtype;
  if (a->out_dtype != EPB_F32 && a->out_dtype != wire)
    return fail(EPB_TAG_MISMATCH, "dispatch output must be f32 or the wire dtype");
  if (!a16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (phases & 1) {
    if (a->num_tokens > 0 && !a16(a->x)) return fail(EPB_INVALID_ARGUMENT, "x must be 16-byte aligned");
    HTSend p;
    p.ops = OpTrace{g->op_ring, g->op_cap};
    p.x = a->x; p.w = a->weights; p.topk = a->topk_idx; p.q = a->rank_count; p.tok_rank = a->tok_rank;
    p.tok_slot = a->tok_slot; p.offsets = a->offsets; p.peers = g->d_peers;
    p.done = g->d_done; p.g = g->ht;
    p.b = a->num_tokens; p.rank = g->rank; p.tag = ht_tag(round);
    p.stage = g->window + g->ht.stage;
    p.stage_ready = a->x == p.stage && a->x_dtype == wire && g->ht.RB == g->ht.RBp;
    cudaError_t e;
    switch (a->x_dtype) {
      case EPB_F32: e = launch_hsend_x<EPB_F32>(p, a->out_dtype, s); break;
      case EPB_BF16: e = launch_hsend_x<EPB_BF16>(p, a->out_dtype, s); break;
      case EPB_F16: e = launch_hsend_x<EPB_F16>(p, a->out_dtype, s); break;
      default: return fail(EPB_TAG_MISMATCH, "HT dispatch input must be f32/bf16/f16");
    }
    if (e != cudaSuccess) return cuda_check(e, "ht_dispatch_send");
  }
  if (phases & 2) {
    HTRecv p;
    p.ops = OpTrace{g->op_ring, g->op_cap};
    p.peers = g->d_peers; p.q = a->rank_count; p.out = a->out; p.origin = a->origin; p.origin_w = a->origin_w;
    p.win = g->window; p.err = g->d_err;
    p.g = g->ht; p.timeout_ns = g->timeout_ns; p.rank = g->rank; p.tag = ht_tag(round);
    cudaError_t e;
    switch (wire) {
      case EPB_F32: e = launch_hrecv<EPB_F32, EPB_F32>(p, s); break;
      case EPB_BF16:
        e = a->out_dtype == EPB_F32 ? launch_hrecv<EPB_BF16, EPB_F32>(p, s) : launch_hrecv<EPB_BF16, EPB_BF16>(p, s);
        break;
      default:
        e = a->out_dtype == EPB_F32 ? launch_hrecv<EPB_F16, EPB_F32>(p, s) : launch_hrecv<EPB_F16, EPB_F16>(p, s);
    }
    if (e != cudaSuccess) return cuda_check(e, "ht_dispatch_recv");
  }
  return EPB_OK;
}

int epb_ht_combine(epb_group* g, uint32_t round, int32_t phases, const epb_ht_combine_args* a, void* stream) {
  if (int rc = check_ht(g, phases)) return rc;
  if (a->in_dtype != EPB_F32 && a->in_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine input f32|bf16");
  if (a->recv_total > 0 && !a16(a->expert_rows)) return fail(EPB_INVALID_ARGUMENT, "expert rows must be 16-byte aligned");
  if (a->expert_rows_in_window) {
    if (a->in_dtype != EPB_BF16 || !a->row_ptr || g->ht.yout_rows < (uint64_t)std::max(a->recv_total, 0) ||
        a->expert_rows != g->window + g->ht.yout)
      return fail(EPB_INVALID_ARGUMENT, "pulled combine needs bf16 rows in the window's expert-output region");
  }
  cudaStream_t s = as_stream(stream);
  if ((phases & 1) && a->dispatch_weights && a->num_tokens > 0) {
    // combine weights must equal the dispatched ones (ht.py:605-609)
    const int64_t n = (int64_t)a->num_tokens * g->cfg.top_k;
    weights_equal_kernel<<<(int)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, s>>>(
        a->weights, a->dispatch_weights, n, g->d_err);
    EPB_LAUNCH_CHECK();
  }
  if (phases & 1) {
    // the metadata rows of this round live in the window (parity = round & 1)
    HTCombSend p;
    p.ops = OpTrace{g->op_ring, g->op_cap};
    p.err = g->d_err;
    p.y = a->expert_rows; p.origin = a->origin;
    p.meta = reinterpret_cast<const int32_t*>(g->window + g->ht.meta +
                                              (uint64_t)(round & 1) * g->ht.N * (g->ht.E + g->ht.N) * 4);
    p.peers = g->d_peers; p.done = g->d_done + g->cfg.num_ranks; p.g = g->ht; p.rows = a->recv_total;
    p.rank = g->rank; p.in_dtype = a->in_dtype; p.tag = ht_tag(round);
    p.topk = a->topk_idx; p.tok_rank = a->tok_rank; p.offsets = a->offsets; p.win = g->window;
    p.row_ptr = a->row_ptr; p.b = a->num_tokens; p.pull = a->expert_rows_in_window;
    const int grid = 2 * hsm_count();
    if (a->in_dtype == EPB_F32) ht_combine_send_kernel<EPB_F32><<<grid, kHTThreads, 0, s>>>(p);
    else ht_combine_send_kernel<EPB_BF16><<<grid, kHTThreads, 0, s>>>(p);
    EPB_LAUNCH_CHECK();
  }
  if (phases & 2) {
    if (a->out_dtype != EPB_F32 && a->out_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine output f32|bf16");
    if (!a16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
    HTCombRecv p;
    p.rows_local = g->cfg.num_ranks == 1 || !a->expert_rows_in_window;
    p.topk = a->topk_idx; p.row_ptr = a->row_ptr; p.w = a->weights; p.y_local = a->expert_rows;
    p.tok_rank = a->tok_rank;
    p.offsets = a->offsets; p.out = a->out; p.win = g->window; p.err = g->d_err; p.g = g->ht;
    p.timeout_ns = g->timeout_ns; p.b = a->num_tokens; p.rank = g->rank; p.y_dtype = a->in_dtype;
    p.tag = ht_tag(round);
    const int grid = hsm_count();
    if (a->in_dtype == EPB_F32) {
      if (a->out_dtype == EPB_F32) ht_combine_recv_kernel<EPB_F32, EPB_F32><<<grid, kHTThreads, 0, s>>>(p);
      else ht_combine_recv_kernel<EPB_F32, EPB_BF16><<<grid, kHTThreads, 0, s>>>(p);
    } else {
      // cp.async staging of the bf16 reduce: [warps][kCS][8][32] x 16 B
      const int csm = (kHTThreads / 32) * kCS * 8 * 32 * 16;
      if (a->out_dtype == EPB_F32) {
        EPB_CUDA(cudaFuncSetAttribute(ht_combine_recv_kernel<EPB_BF16, EPB_F32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, csm));
        ht_combine_recv_kernel<EPB_BF16, EPB_F32><<<grid, kHTThreads, csm, s>>>(p);
      } else {
        EPB_CUDA(cudaFuncSetAttribute(ht_combine_recv_kernel<EPB_BF16, EPB_BF16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, csm));
        ht_combine_recv_kernel<EPB_BF16, EPB_BF16><<<grid, kHTThreads, csm, s>>>(p);
      }
    }
    EPB_LAUNCH_CHECK();
  }
  return EPB_OK;
}

int epb_weights_equal(epb_group* g, const float* a, const float* b, int64_t n, void* stream) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (n <= 0) return EPB_OK;
  const int grid = (int)std::min<int64_t>(1024, (n + 255) / 256);
  weights_equal_kernel<<<grid, 256, 0, as_stream(stream)>>>(a, b, n, g->d_err);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

}  // extern "C"
