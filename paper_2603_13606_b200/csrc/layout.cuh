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

constexpr int kIdsStride = 8 * 32 + 8;  // one warp's staged ids: 32 tokens x K<=8, one pad word per 32

struct BlockLayoutSmem {
  int* hist;        // [nwarps][E+N]
  uint32_t* ballot; // [nwarps][E+N]
  int* ids;         // [nwarps][kIdsStride] coalesced-load staging of expert ids
  __host__ __device__ static size_t bytes(int nwarps, int E, int N) {
    return (size_t)nwarps * (E + N) * 8 + (size_t)nwarps * kIdsStride * 4;
  }
  EPB_DEV static BlockLayoutSmem carve(int* base, int nwarps, int E, int N) {
    BlockLayoutSmem sm;
    sm.hist = base;
    sm.ballot = reinterpret_cast<uint32_t*>(base + nwarps * (E + N));
    sm.ids = base + 2 * nwarps * (E + N);
    return sm;
  }
};

// The ids of tokens [base, base + 32) (nt of them valid) loaded by the warp
// with coalesced loads (lane l reads elements l, l+32, ...), staged in shared
// memory with one pad word per 32 (conflict-free transposed reads), and
// returned per lane: lane i gets token base+i's K ids (K <= 8).
template <typename TopkT>
EPB_DEV void warp_ids8(const TopkT* topk, int base, int nt, int K, int* st, int (&ev)[8]) {
  const int lane = threadIdx.x & 31;
  const int n = nt * K;
  const TopkT* src = topk + (int64_t)base * K;
  TopkT v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = j * 32 + lane;
    v[j] = i < n ? src[i] : (TopkT)0;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = j * 32 + lane;
    // out-of-int-range ids are kept out of range as -1 (validation rejects them)
    const int64_t x = (int64_t)v[j];
    st[i + (i >> 5)] = (x < 0 || x > 0x7fffffff) ? -1 : (int)x;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = lane * K + k;
    ev[k] = k < K ? st[i + (i >> 5)] : 0;
  }
  __syncwarp();
}

// A lane's token's K expert ids: held in registers when K <= KM (one batch of
// independent loads per pass instead of a dependent load per use), read from
// memory otherwise (KM = 0).
template <int KM, typename TopkT>
struct TokenIds {
  int v[KM > 0 ? KM : 1];
  const TopkT* row;
  EPB_DEV void load(const TopkT* topk, int t, int K) {
    row = topk + (int64_t)t * K;
    if (KM > 0) {
#pragma unroll
      for (int k = 0; k < (KM > 0 ? KM : 1); ++k) v[k] = k < K ? (int)row[k] : 0;
    }
  }
  EPB_DEV int operator[](int k) const { return KM > 0 ? v[k] : (int)row[k]; }
};

#define EPB_FOR_K(k, KM, K) \
  _Pragma("unroll") for (int k = 0; k < ((KM) > 0 ? (KM) : (K)); ++k) if ((KM) == 0 || k < (K))

template <int KM, typename TopkT>
EPB_DEV void block_layout_k(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                            int32_t* m_out, int32_t* q_out, int32_t* rank_out, int32_t* slot_out,
                            uint64_t* mask_out, uint64_t* stamps = nullptr) {
#define LAY_STAMP(I) \
  do { if (stamps && threadIdx.x == 0) stamps[I] = globaltimer(); } while (0)
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
  TokenIds<KM, TopkT> ids;
  for (int t = t0 + lane; t < t1; t += 32) {
    ids.load(topk, t, K);
    uint64_t mask = 0;
    EPB_FOR_K(k, KM, K) {
      const int e = ids[k];
      atomicAdd(&h[e], 1);
      mask |= 1ull << (e / L);
    }
    for (uint64_t mm = mask; mm; mm &= mm - 1) atomicAdd(&h[E + __ffsll(mm) - 1], 1);
    if (mask_out) mask_out[t] = mask;
  }
  LAY_STAMP(0);
  __syncthreads();
  LAY_STAMP(1);
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
  LAY_STAMP(2);
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = t0; base < t1; base += 32) {
    const int t = base + lane;
    const bool act = t < t1;
    uint64_t mask = 0;
    if (act) {
      ids.load(topk, t, K);
      EPB_FOR_K(k, KM, K) {
        const int e = ids[k];
        mask |= 1ull << (e / L);
        atomicOr(&bw[e], 1u << lane);
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) atomicOr(&bw[E + __ffsll(mm) - 1], 1u << lane);
    }
    __syncwarp();
    if (act) {
      EPB_FOR_K(k, KM, K) {
        const int e = ids[k];
        rank_out[(int64_t)t * K + k] = h[e] + __popc(bw[e] & lt);
      }
      if (slot_out)
        for (int d = 0; d < N; ++d)
          slot_out[(int64_t)t * N + d] = ((mask >> d) & 1) ? h[E + d] + __popc(bw[E + d] & lt) : -1;
    }
    __syncwarp();
    if (act) {
      // the lowest lane hitting a column advances its running count
      EPB_FOR_K(k, KM, K) {
        const int e = ids[k];
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
      EPB_FOR_K(k, KM, K) bw[ids[k]] = 0u;
      for (uint64_t mm = mask; mm; mm &= mm - 1) bw[E + __ffsll(mm) - 1] = 0u;
    }
    __syncwarp();
  }
  LAY_STAMP(3);
  __syncthreads();
#undef LAY_STAMP
}

// topk: b*K expert ids (already validated).  Outputs may live in shared or
// global memory.  Requires all threads of the block.
template <typename TopkT>
EPB_DEV void block_layout(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                          int32_t* m_out, int32_t* q_out, int32_t* rank_out, int32_t* slot_out,
                          uint64_t* mask_out, uint64_t* stamps = nullptr) {
  if (K <= 8) block_layout_k<8>(topk, b, K, E, N, L, sm, m_out, q_out, rank_out, slot_out, mask_out, stamps);
  else block_layout_k<0>(topk, b, K, E, N, L, sm, m_out, q_out, rank_out, slot_out, mask_out, stamps);
}

// row validation: ids in [0, E), distinct within a row (api.py:150-170)
template <int KM, typename TopkT>
EPB_DEV bool rows_bad(const TopkT* topk, int b, int K, int E) {
  bool bad = false;
  for (int t = threadIdx.x; t < b; t += blockDim.x) {
    const TopkT* row = topk + (int64_t)t * K;
    if (KM > 0) {
      int64_t v[KM > 0 ? KM : 1];
#pragma unroll
      for (int k = 0; k < (KM > 0 ? KM : 1); ++k) v[k] = k < K ? (int64_t)row[k] : 0;
#pragma unroll
      for (int k = 0; k < (KM > 0 ? KM : 1); ++k) {
        if (k >= K) break;
        bad |= v[k] < 0 || v[k] >= E;
#pragma unroll
        for (int j = 0; j < k; ++j) bad |= v[j] == v[k];
      }
    } else {
      for (int k = 0; k < K; ++k) {
        const int64_t e = (int64_t)row[k];
        if (e < 0 || e >= E) { bad = true; break; }
        for (int j = 0; j < k; ++j)
          if ((int64_t)row[j] == e) bad = true;
      }
    }
  }
  return bad;
}

template <typename TopkT>
EPB_DEV bool block_validate(const TopkT* topk, int b, int K, int E, int* s_bad) {
  (void)s_bad;
  const bool bad = K <= 8 ? rows_bad<8>(topk, b, K, E) : rows_bad<0>(topk, b, K, E);
  return __syncthreads_or(bad) == 0;  // one verdict per block (a barrier)
}

// Validation (ids in [0, E), distinct within a row; api.py:150-170) fused
// with the layout for K <= 8: the expert ids are loaded once per pass, with
// coalesced loads, and a rejected routing writes no output.  Two halves so
// a multi-CTA caller can put a grid-wide exchange between them:
//   block_hist8: validation + per-warp column histograms (shared memory),
//                the block's column totals into `tot_out` (if given);
//                false for a rejected routing (one verdict per block);
//   block_rank8: exclusive scan of the histograms across warps seeded with
//                `col_base` (the counts of earlier blocks, or none), the
//                totals + base into m_out / q_out, then ranks and slots.
template <typename TopkT>
EPB_DEV bool block_hist8(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm, int32_t* tot_out,
                         uint64_t* stamps) {
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
  int* st = sm.ids + warp * kIdsStride;
  int ev[8];
  bool bad = false;
  for (int base = t0; base < t1; base += 32) {
    const int nt = min(32, t1 - base);
    warp_ids8(topk, base, nt, K, st, ev);
    if (lane < nt) {
      bool rb = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < K) {
          rb |= ev[k] < 0 || ev[k] >= E;
#pragma unroll
          for (int j = 0; j < k; ++j) rb |= ev[j] == ev[k];
        }
      }
      bad |= rb;
      if (!rb) {
        uint64_t mask = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k < K) {
            atomicAdd(&h[ev[k]], 1);
            mask |= 1ull << (ev[k] / L);
          }
        }
        for (uint64_t mm = mask; mm; mm &= mm - 1) atomicAdd(&h[E + __ffsll(mm) - 1], 1);
      }
    }
  }
  if (stamps && threadIdx.x == 0) stamps[0] = globaltimer();
  if (__syncthreads_or(bad)) return false;
  if (tot_out)
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      int tot = 0;
      for (int w = 0; w < nwarps; ++w) tot += sm.hist[w * C + c];
      tot_out[c] = tot;
    }
  return true;
}

template <typename TopkT>
EPB_DEV void block_rank8(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                         const int32_t* col_base, int32_t* m_out, int32_t* q_out, int32_t* rank_out,
                         int32_t* slot_out, uint64_t* stamps) {
  const int C = E + N;
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int run = col_base ? col_base[c] : 0;
    for (int w = 0; w < nwarps; ++w) {
      const int v = sm.hist[w * C + c];
      sm.hist[w * C + c] = run;
      run += v;
    }
    if (c < E) { if (m_out) m_out[c] = run; }
    else if (q_out) q_out[c - E] = run;
  }
  __syncthreads();
  if (stamps && threadIdx.x == 0) stamps[2] = globaltimer();
  const int seg = (b + nwarps - 1) / nwarps;
  const int t0 = min(b, warp * seg), t1 = min(b, t0 + seg);
  int* h = sm.hist + warp * C;
  uint32_t* bw = sm.ballot + warp * C;
  int* st = sm.ids + warp * kIdsStride;
  int ev[8];
  const uint32_t lt = (1u << lane) - 1u;
  for (int base = t0; base < t1; base += 32) {
    const int nt = min(32, t1 - base);
    warp_ids8(topk, base, nt, K, st, ev);
    const int t = base + lane;
    const bool act = lane < nt;
    uint64_t mask = 0;
    if (act) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < K) {
          mask |= 1ull << (ev[k] / L);
          atomicOr(&bw[ev[k]], 1u << lane);
        }
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) atomicOr(&bw[E + __ffsll(mm) - 1], 1u << lane);
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < K) rank_out[(int64_t)t * K + k] = h[ev[k]] + __popc(bw[ev[k]] & lt);
      if (slot_out)
        for (int d = 0; d < N; ++d)
          slot_out[(int64_t)t * N + d] = ((mask >> d) & 1) ? h[E + d] + __popc(bw[E + d] & lt) : -1;
    }
    __syncwarp();
    if (act) {
      // the lowest lane hitting a column advances its running count
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < K) {
          const uint32_t bits = bw[ev[k]];
          if ((bits & lt) == 0) h[ev[k]] += __popc(bits);
        }
      }
      for (uint64_t mm = mask; mm; mm &= mm - 1) {
        const int c = E + __ffsll(mm) - 1;
        const uint32_t bits = bw[c];
        if ((bits & lt) == 0) h[c] += __popc(bits);
      }
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < K) bw[ev[k]] = 0u;
      for (uint64_t mm = mask; mm; mm &= mm - 1) bw[E + __ffsll(mm) - 1] = 0u;
    }
    __syncwarp();
  }
  if (stamps && threadIdx.x == 0) stamps[3] = globaltimer();
  __syncthreads();
}

template <typename TopkT>
EPB_DEV bool block_layout_valid8(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                                 int32_t* m_out, int32_t* q_out, int32_t* rank_out, int32_t* slot_out,
                                 uint64_t* stamps) {
  if (!block_hist8(topk, b, K, E, N, L, sm, nullptr, stamps)) return false;
  block_rank8(topk, b, K, E, N, L, sm, nullptr, m_out, q_out, rank_out, slot_out, stamps);
  return true;
}

// validate + lay out; false (nothing written) for a rejected routing
template <typename TopkT>
EPB_DEV bool block_layout_checked(const TopkT* topk, int b, int K, int E, int N, int L, BlockLayoutSmem sm,
                                  int32_t* m_out, int32_t* q_out, int32_t* rank_out, int32_t* slot_out,
                                  uint64_t* stamps = nullptr) {
  if (K <= 8) return block_layout_valid8(topk, b, K, E, N, L, sm, m_out, q_out, rank_out, slot_out, stamps);
  __shared__ int s_unused;
  if (!block_validate(topk, b, K, E, &s_unused)) return false;
  block_layout(topk, b, K, E, N, L, sm, m_out, q_out, rank_out, slot_out, nullptr, stamps);
  return true;
}

}  // namespace epb
