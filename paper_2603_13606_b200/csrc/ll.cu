// Low-Latency dispatch / combine: two kernels per round (K2+K3 fused, K4a+K4b
// fused), each runnable as send-only, recv-only or both (cooperative launch).
//
// Reference semantics (epsim ll.py):
//  * dispatch send (ll.py:255-308): per destination rank d, the tokens that
//    touch d go, ascending t, into d's slots [src*B + j]; afterwards one
//    counter per (local expert of d, src) carries m(e, src) + 1.  Here the
//    counter word is (tag << 40) | (q << 20) | m, published with a release
//    fence after this rank's last slot store to d.  The tag (from the round
//    sequence) replaces the reference's counter reset (ll.py:351-353).
//  * dispatch recv (ll.py:310-400): wait for the counters, then place every
//    slot row at recv[l, src*B + i] for each local expert; i (the filled[l]
//    order) and j (the slot) are computed by the SENDER from its routing in
//    shared memory (ballot-free prefix counts over earlier tokens) and i is
//    carried in the slot header after the reference header fields.
//  * combine send (ll.py:404-462): each valid expert row (l, src, i) goes,
//    re-encoded in the combine wire dtype, to src's slot t*K + k; then one
//    flag per (expert rank -> home rank).
//  * combine recv (ll.py:464-507): out[t] = sum_k w[t,k] * y_k in f32,
//    ascending k from acc = 0, explicit __fmul_rn/__fadd_rn (no FMA).
//
// Latency design: routing layout, validation and the per-destination
// counts are computed inside the dispatch kernel from a shared-memory copy of
// topk_idx; copies keep 8 x 16 B loads in flight per lane before storing.
#include "common.cuh"
#include "internal.h"
#include "layout.cuh"

namespace epb {

constexpr int kPhaseSend = 1, kPhaseRecv = 2;
constexpr int kThreads = 256;
constexpr int kUnroll = 8;

EPB_DEV uint32_t ll_tag_of(uint32_t seq) { return (seq % 0xFFFFFFu) + 1u; }
EPB_DEV uint32_t ld_volatile_u32(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
EPB_DEV uint8_t* peer_base(const uint64_t* peers, int r) { return reinterpret_cast<uint8_t*>(peers[r]); }
EPB_DEV void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
EPB_DEV int4 ld_weak_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
EPB_DEV void st_weak_v4(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

// Warp-cooperative copy of nch 16-byte chunks, kUnroll loads in flight per lane.
EPB_DEV void warp_copy16(const uint8_t* src, uint8_t* dst, int nch, int lane) {
  for (int base = 0; base < nch; base += 32 * kUnroll) {
    int4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * 32 + lane;
      if (c < nch) v[u] = ld_weak_v4(src + (int64_t)c * 16);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * 32 + lane;
      if (c < nch) st_weak_v4(dst + (int64_t)c * 16, v[u]);
    }
  }
}

// The round sequence lives on the device (graph-replayable): the send phase
// reads the group counter; the last CTA to read it stores it into the
// handle word and advances the counter.  Recv-only launches read the handle.
EPB_DEV uint32_t ll_round_seq(uint32_t* dseq, int* drd, uint32_t* hseq, bool alloc) {
  __shared__ uint32_t s_seq;
  if (threadIdx.x == 0) {
    if (alloc) {
      const uint32_t seq = ld_volatile_u32(dseq);
      s_seq = seq;
      __threadfence();
      if (atomicAdd(drd, 1) == (int)gridDim.x - 1) {
        *drd = 0;
        *hseq = seq;
        *dseq = seq + 1;
      }
    } else {
      s_seq = ld_volatile_u32(hseq);
    }
  }
  __syncthreads();
  return s_seq;
}

// ===========================================================================
// dispatch
// ===========================================================================
struct LLDisp {
  const void* x;
  const float* x_scales;
  const int64_t* topk;
  uint32_t* hseq;
  void* out;
  float* out_scales;
  float* counts_f32;
  int32_t* counts_i32;
  int32_t* src_info;
  const uint64_t* peers;
  const uint8_t* win;
  int* done;
  int* err;
  uint32_t* dseq;
  int* drd;
  LLGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
};

// Convert elements [e0, e0 + EPC) of an input row (dtype XT) to f32.
template <int XT, int EPC>
EPB_DEV void load_input_chunk(const uint8_t* xrow, const float* xsc, int64_t e0, float* f) {
  load_elems_vec<XT, EPC>(xrow, e0, f);
  if constexpr (XT == EPB_FP8) {
    // fp8 input with block scales: dequantise (core.py:153-162); without
    // scales the codes are plain E4M3 values (implicit scale 1)
    if (xsc != nullptr) {
#pragma unroll
      for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], xsc[(e0 + i) >> 7]);
    }
  }
}

// counters of pairs (l, src = rank) at destination d
EPB_DEV void ll_publish_disp(const LLDisp& p, int d, const int* s_m, int qd, uint64_t parity_off,
                             uint32_t tag) {
  const LLGeom& g = p.g;
  uint64_t* ctr = reinterpret_cast<uint64_t*>(peer_base(p.peers, d) + parity_off + g.disp_ctr);
  for (int l = 0; l < g.L; ++l) {
    const int e = d * g.L + l;
    const uint64_t m = e < g.E ? (uint64_t)s_m[e] : 0ull;
    st_relaxed_sys(&ctr[l * g.N + p.rank], ((uint64_t)tag << 40) | ((uint64_t)qd << 20) | m);
  }
}

// copy one received slot row (WT, optional scales) to an output row (OT)
template <int WT, bool SC, int OT>
EPB_DEV void ll_copy_row(const LLGeom& g, const uint8_t* slot, uint8_t* orow, float* osc, int lane) {
  const int H = g.H;
  if ((H & 15) == 0) {
    constexpr int EPC = Elems<WT>::n;
    const int nch = H / EPC;
    if constexpr (OT == WT) {
      warp_copy16(slot, orow, nch, lane);
      if constexpr (SC) {
        const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
        for (int i = lane; i < H / 128; i += 32) osc[i] = sc[i];
      }
    } else {
      static_assert(OT == EPB_F32, "recv output is f32 or the wire dtype");
      const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
      for (int base = 0; base < nch; base += 32 * 4) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + u * 32 + lane;
          if (c < nch) v[u] = ld_weak_v4(slot + (int64_t)c * 16);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + u * 32 + lane;
          if (c < nch) {
            float f[EPC];
            unpack16<WT>(v[u], f);
            if constexpr (SC) {
              const float s = sc[(c * EPC) >> 7];
#pragma unroll
              for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], s);
            }
            store_f32_chunk<EPB_F32, EPC>(orow, (int64_t)c * EPC, f);
          }
        }
      }
    }
  } else {
    for (int el = lane; el < H; el += 32) {
      if constexpr (OT == WT) {
        if constexpr (OT == EPB_F32) reinterpret_cast<float*>(orow)[el] = reinterpret_cast<const float*>(slot)[el];
        else if constexpr (OT == EPB_FP8) orow[el] = slot[el];
        else reinterpret_cast<uint16_t*>(orow)[el] = reinterpret_cast<const uint16_t*>(slot)[el];
      } else {
        reinterpret_cast<float*>(orow)[el] = load_elem(slot, WT, el);
      }
    }
  }
}

template <int XT, int WT, bool SC, int OT>
__global__ void __launch_bounds__(kThreads) ll_dispatch_kernel(LLDisp p) {
  extern __shared__ int smem[];
  const LLGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L, E = g.E, B = g.B;
  const int b = p.b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t seq = ll_round_seq(p.dseq, p.drd, p.hseq, p.phases & kPhaseSend);
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;

  if (p.phases & kPhaseSend) {
    // shared: topk snapshot, layout outputs, per-warp histograms
    const int nwarps = blockDim.x >> 5;
    int* s_topk = smem;                              // [b*K]
    int* s_rank = s_topk + b * K;                    // [b*K]
    int* s_slot = s_rank + b * K;                    // [b*N]
    int* s_m = s_slot + b * N;                       // [E]
    int* s_q = s_m + E;                              // [N]
    BlockLayoutSmem lsm;
    lsm.hist = s_q + N;                              // [nwarps][E+N]
    lsm.ballot = reinterpret_cast<uint32_t*>(lsm.hist + nwarps * (E + N));
    __shared__ int s_bad;
    __shared__ int s_dst[kMaxRanks], s_j[kMaxRanks], s_nd;
    __shared__ uint32_t s_hdr[2 + 2 * kMaxTopK];
    for (int i = threadIdx.x; i < b * K; i += blockDim.x) s_topk[i] = (int)p.topk[i];
    __syncthreads();
    // validation before any traffic (api.py:150-170): every CTA reaches the
    // same verdict on the same routing, so no CTA sends anything on error
    if (!block_validate(p.topk, b, K, E, &s_bad)) {
      if (threadIdx.x == 0) atomicCAS(p.err, 0, EPB_INVALID_ARGUMENT);
      return;
    }
    block_layout(s_topk, b, K, E, N, L, lsm, s_m, s_q, s_rank, s_slot, nullptr);
    const uint64_t slot_off = parity_off + g.disp_slot;
    const int64_t slot_base = (int64_t)p.rank * B;
    for (int t = blockIdx.x; t < b; t += gridDim.x) {
      if (threadIdx.x == 0) {
        int nd = 0;
        for (int d = 0; d < N; ++d) {
          const int j = s_slot[t * N + d];
          if (j >= 0) { s_dst[nd] = d; s_j[nd] = j; ++nd; }
        }
        s_nd = nd;
        s_hdr[0] = (uint32_t)t;
        s_hdr[1] = (uint32_t)K;
      }
      if (threadIdx.x < K) {
        s_hdr[2 + threadIdx.x] = (uint32_t)s_topk[t * K + threadIdx.x];
        s_hdr[2 + K + threadIdx.x] = (uint32_t)s_rank[t * K + threadIdx.x];
      }
      __syncthreads();
      const int nd = s_nd;
      for (int w = threadIdx.x; w < 2 + 2 * K; w += blockDim.x)
        for (int i = 0; i < nd; ++i) {
          uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_base + s_j[i]) * g.slot_stride;
          reinterpret_cast<uint32_t*>(slot + g.RBp + g.SBp)[w] = s_hdr[w];
        }
      const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * dtype_width(XT);
      const float* xsc = p.x_scales ? p.x_scales + (int64_t)t * (H / 128) : nullptr;
      if ((H & 15) == 0) {
        constexpr int EPC = Elems<WT>::n;
        const int nch = H / EPC;
        for (int c = threadIdx.x; c < nch; c += blockDim.x) {
          float f[EPC];
          load_input_chunk<XT, EPC>(xrow, xsc, (int64_t)c * EPC, f);
          float scale = 0.0f;
          if constexpr (SC) {
            // block-128 = 8 consecutive 16-element chunks = 8 aligned lanes
            float amax = 0.0f;
#pragma unroll
            for (int i = 0; i < EPC; ++i) amax = fmaxf(amax, fabsf(f[i]));
            const unsigned gm = 0xFFu << (lane & 24);
            amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 1));
            amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 2));
            amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 4));
            scale = __fdiv_rn(amax, 448.0f);
            const float div = scale > 0.0f ? scale : 1.0f;
#pragma unroll
            for (int i = 0; i < EPC; ++i) f[i] = __fdiv_rn(f[i], div);
          }
          const int4 v = pack16<WT>(f);
          for (int i = 0; i < nd; ++i) {
            uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_base + s_j[i]) * g.slot_stride;
            st_na_v4(slot + (int64_t)c * 16, v);
            if constexpr (SC) {
              if ((c & 7) == 0) reinterpret_cast<float*>(slot + g.RBp)[c >> 3] = scale;
            }
          }
        }
      } else {
        // hidden not a multiple of 16: element path (scales need H % 128 == 0)
        for (int el = threadIdx.x; el < H; el += blockDim.x) {
          float f = load_elem(xrow, XT, el);
          if constexpr (XT == EPB_FP8) {
            if (xsc != nullptr) f = __fmul_rn(f, xsc[el >> 7]);
          }
          for (int i = 0; i < nd; ++i) {
            uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_base + s_j[i]) * g.slot_stride;
            store_elem(slot, WT, el, f);
          }
        }
      }
      __syncthreads();
      // completion: the last token to land at d publishes d's counters
      if (threadIdx.x < nd) {
        const int d = s_dst[threadIdx.x];
        fence_sys();
        const int old = atomicAdd(&p.done[d], 1);
        if (old == s_q[d] - 1) {
          p.done[d] = 0;
          fence_sys();
          ll_publish_disp(p, d, s_m, s_q[d], parity_off, tag);
        }
      }
      __syncthreads();
    }
    // destinations that receive nothing still get their (m = 0) counters
    if (blockIdx.x == 0)
      for (int d = threadIdx.x; d < N; d += blockDim.x)
        if (s_q[d] == 0) ll_publish_disp(p, d, s_m, 0, parity_off, tag);
  }

  if (p.phases & kPhaseRecv) {
    __shared__ int s_rq[kMaxRanks], s_pre[kMaxRanks + 1];
    __shared__ int s_fail;
    const int lo = p.rank * L;
    const int nloc = max(0, min(L, E - lo));
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    const uint64_t* ctr = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.disp_ctr);
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < L * N; i += blockDim.x) {
        int m = 0;
        if (i < nloc * N) {
          uint64_t v = 0;
          if (!wait_tag(&ctr[i], tag, 40, 0xFFFFFFu, p.timeout_ns, p.err, &v)) { s_fail = 1; continue; }
          m = (int)(v & 0xFFFFF);
        }
        p.counts_i32[i] = m;
        p.counts_f32[i] = (float)m;
      }
    }
    if (nloc == 0) return;
    if (threadIdx.x < N) {
      uint64_t v = 0;
      if (!wait_tag(&ctr[threadIdx.x], tag, 40, 0xFFFFFFu, p.timeout_ns, p.err, &v)) s_fail = 1;
      s_rq[threadIdx.x] = (int)((v >> 20) & 0xFFFFF);
    }
    __syncthreads();
    if (s_fail) return;
    if (threadIdx.x == 0) {
      int run = 0;
      for (int s = 0; s < N; ++s) { s_pre[s] = run; run += s_rq[s]; }
      s_pre[N] = run;
    }
    __syncthreads();
    const int items = s_pre[N] * K;
    const int nw = blockDim.x >> 5;
    const int ob = (OT == EPB_F32 ? 4 : dtype_width(OT));
    const int64_t orow_bytes = (int64_t)H * ob;
    for (int f = blockIdx.x * nw + warp; f < items; f += gridDim.x * nw) {
      const int sl = f / K, k = f - sl * K;
      int s = 0;
      while (s_pre[s + 1] <= sl) ++s;
      const int j = sl - s_pre[s];
      const uint8_t* slot = p.win + parity_off + g.disp_slot + ((int64_t)s * B + j) * g.slot_stride;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
      const int e = (int)hdr[2 + k];
      if (e < lo || e >= lo + nloc) continue;
      const int64_t row = (int64_t)(e - lo) * N * B + (int64_t)s * B + hdr[2 + K + k];
      if (lane == 0) p.src_info[row] = (int32_t)(hdr[0] * K + k);
      ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + row * orow_bytes,
                              SC ? p.out_scales + row * (H / 128) : nullptr, lane);
    }
  }
}

// ===========================================================================
// combine
// ===========================================================================
struct LLComb {
  const void* y;
  const int32_t* counts;
  const int32_t* src_info;
  const float* w;
  void* out;
  const uint32_t* hseq;
  const uint64_t* peers;
  const uint8_t* win;
  int* done;
  int* err;
  LLGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
};

template <int IT, int WT, int OT>
__global__ void __launch_bounds__(kThreads) ll_combine_kernel(LLComb p) {
  extern __shared__ int s_pre[];  // [L*N + 1]
  const LLGeom& g = p.g;
  const int N = g.N, L = g.L, B = g.B, H = g.H, K = g.K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __shared__ uint32_t s_seq;
  if (threadIdx.x == 0) s_seq = ld_volatile_u32(p.hseq);
  __syncthreads();
  const uint32_t seq = s_seq;
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
  constexpr int EPC = Elems<WT>::n;

  if (p.phases & kPhaseSend) {
    __shared__ int s_rows_to[kMaxRanks], s_cnt[kMaxRanks], s_wsum[kThreads / 32];
    const int P = L * N;
    if (threadIdx.x < N) { s_rows_to[threadIdx.x] = 0; s_cnt[threadIdx.x] = 0; }
    __syncthreads();
    // block-wide exclusive scan of the (l, src) counts
    const int per = (P + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per;
    int local = 0;
    for (int i = i0; i < min(P, i0 + per); ++i) {
      const int c = p.counts[i];
      local += c;
      if (c) atomicAdd(&s_rows_to[i % N], c);
    }
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w2 = 0; w2 < warp; ++w2) wbase += s_wsum[w2];
    int run = wbase + incl - local;
    for (int i = i0; i < min(P, i0 + per); ++i) {
      s_pre[i] = run;
      run += p.counts[i];
    }
    if (threadIdx.x == blockDim.x - 1) s_pre[P] = run;
    __syncthreads();
    const int total = s_pre[P];
    const int gw = blockIdx.x * nw + warp, tw = gridDim.x * nw;
    for (int r = gw; r < total; r += tw) {
      int lo_i = 0, hi_i = P;  // largest pair with s_pre[pair] <= r
      while (hi_i - lo_i > 1) {
        const int mid = (lo_i + hi_i) >> 1;
        if (s_pre[mid] <= r) lo_i = mid; else hi_i = mid;
      }
      const int pair = lo_i;
      const int l = pair / N, s = pair - l * N, i = r - s_pre[pair];
      const int64_t row = (int64_t)l * N * B + (int64_t)s * B + i;
      const int info = p.src_info[row];
      uint8_t* dst = peer_base(p.peers, s) + parity_off + g.comb_slot + (int64_t)info * g.comb_stride;
      const uint8_t* yrow = reinterpret_cast<const uint8_t*>(p.y) + row * H * dtype_width(IT);
      if ((H & 15) == 0) {
        const int nch = H / EPC;
        if constexpr (IT == WT) {
          for (int base = 0; base < nch; base += 32 * kUnroll) {
            int4 v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int c = base + u * 32 + lane;
              if (c < nch) v[u] = ld_nc_v4(yrow + (int64_t)c * 16);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int c = base + u * 32 + lane;
              if (c < nch) st_na_v4(dst + (int64_t)c * 16, v[u]);
            }
          }
        } else {
          for (int c = lane; c < nch; c += 32) {
            float f[EPC];
            load_elems_vec<IT, EPC>(yrow, (int64_t)c * EPC, f);
            st_na_v4(dst + (int64_t)c * 16, pack16<WT>(f));
          }
        }
      } else {
        for (int el = lane; el < H; el += 32) store_elem(dst, WT, el, load_elem(yrow, IT, el));
      }
      if (lane == 0) atomicAdd(&s_cnt[s], 1);
    }
    __syncthreads();
    if (threadIdx.x < N) {
      const int s = threadIdx.x;
      const int c = s_cnt[s];
      uint64_t* flag = reinterpret_cast<uint64_t*>(peer_base(p.peers, s) + parity_off + g.comb_ctr) + p.rank;
      if (c > 0) {
        fence_sys();
        const int old = atomicAdd(&p.done[s], c);
        if (old + c == s_rows_to[s]) {
          p.done[s] = 0;
          fence_sys();
          st_relaxed_sys(flag, (uint64_t)tag);
        }
      } else if (blockIdx.x == 0 && s_rows_to[s] == 0) {
        st_relaxed_sys(flag, (uint64_t)tag);
      }
    }
  }

  if (p.phases & kPhaseRecv) {
    __shared__ float s_w[kMaxTopK];
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.comb_ctr);
    if (threadIdx.x < N) {
      uint64_t v;
      if (!wait_tag(&flags[threadIdx.x], tag, 0, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) s_fail = 1;
    }
    __syncthreads();
    if (s_fail) return;
    const uint8_t* slots = p.win + parity_off + g.comb_slot;
    for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
      if (threadIdx.x < K) s_w[threadIdx.x] = p.w[(int64_t)t * K + threadIdx.x];
      __syncthreads();
      uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * dtype_width(OT);
      const uint8_t* tsl = slots + (int64_t)t * K * g.comb_stride;
      if ((H & 15) == 0) {
        for (int c = threadIdx.x; c < H / EPC; c += blockDim.x) {
          float acc[EPC];
#pragma unroll
          for (int i = 0; i < EPC; ++i) acc[i] = 0.0f;
          for (int k0 = 0; k0 < K; k0 += 8) {
            int4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k0 + u < K) v[u] = ld_weak_v4(tsl + (int64_t)(k0 + u) * g.comb_stride + (int64_t)c * 16);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (k0 + u < K) {
                float y[EPC];
                unpack16<WT>(v[u], y);
                const float wk = s_w[k0 + u];
#pragma unroll
                for (int i = 0; i < EPC; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(wk, y[i]));
              }
            }
          }
          store_f32_chunk<OT, EPC>(orow, (int64_t)c * EPC, acc);
        }
      } else {
        for (int el = threadIdx.x; el < H; el += blockDim.x) {
          float acc = 0.0f;
          for (int k = 0; k < K; ++k)
            acc = __fadd_rn(acc, __fmul_rn(s_w[k], load_elem(tsl + (int64_t)k * g.comb_stride, WT, el)));
          store_elem(orow, OT, el, acc);
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace epb

using namespace epb;

namespace {

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename Params>
cudaError_t launch(void (*kern)(Params), int grid, size_t smem, bool coop, const Params& p, cudaStream_t s) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (coop) {
    // both phases in one launch: CTAs in the receive phase wait on flags the
    // send phase of other CTAs writes, so all CTAs must be co-resident
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    grid = std::max(1, std::min(grid, per_sm * sm_count()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  kern<<<grid, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int XT, int WT, bool SC, int OT>
cudaError_t run_disp(const LLDisp& p, int grid, size_t smem, cudaStream_t s) {
  return launch(ll_dispatch_kernel<XT, WT, SC, OT>, grid, smem, p.phases == 3, p, s);
}

template <int XT, int WT, bool SC>
cudaError_t run_disp_o(const LLDisp& p, int out_dtype, int grid, size_t smem, cudaStream_t s) {
  if (out_dtype == EPB_F32 || WT == EPB_F32) return run_disp<XT, WT, SC, EPB_F32>(p, grid, smem, s);
  return run_disp<XT, WT, SC, WT>(p, grid, smem, s);
}

template <int XT>
cudaError_t run_disp_x(const LLDisp& p, int out_dtype, int grid, size_t smem, cudaStream_t s) {
  switch (p.g.wire) {
    case EPB_F32: return run_disp_o<XT, EPB_F32, false>(p, out_dtype, grid, smem, s);
    case EPB_BF16: return run_disp_o<XT, EPB_BF16, false>(p, out_dtype, grid, smem, s);
    case EPB_F16: return run_disp_o<XT, EPB_F16, false>(p, out_dtype, grid, smem, s);
    default:
      return p.g.scales ? run_disp_o<XT, EPB_FP8, true>(p, out_dtype, grid, smem, s)
                        : run_disp_o<XT, EPB_FP8, false>(p, out_dtype, grid, smem, s);
  }
}

template <int IT, int WT, int OT>
cudaError_t run_comb(const LLComb& p, int grid, size_t smem, cudaStream_t s) {
  return launch(ll_combine_kernel<IT, WT, OT>, grid, smem, p.phases == 3, p, s);
}

template <int IT, int WT>
cudaError_t run_comb_o(const LLComb& p, int out_dtype, int grid, size_t smem, cudaStream_t s) {
  return out_dtype == EPB_F32 ? run_comb<IT, WT, EPB_F32>(p, grid, smem, s)
                              : run_comb<IT, WT, EPB_BF16>(p, grid, smem, s);
}

template <int IT>
cudaError_t run_comb_w(const LLComb& p, int out_dtype, int grid, size_t smem, cudaStream_t s) {
  switch (p.g.cwire) {
    case EPB_F32: return run_comb_o<IT, EPB_F32>(p, out_dtype, grid, smem, s);
    case EPB_BF16: return run_comb_o<IT, EPB_BF16>(p, out_dtype, grid, smem, s);
    case EPB_F16: return run_comb_o<IT, EPB_F16>(p, out_dtype, grid, smem, s);
    default: return run_comb_o<IT, EPB_FP8>(p, out_dtype, grid, smem, s);
  }
}

int check_ll(epb_group* g, int phases) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (g->cfg.algorithm != EPB_LL) return fail(EPB_HANDLE_STATE_ERROR, "group is not LL");
  if (!g->peers_ready) return fail(EPB_HANDLE_STATE_ERROR, "peer windows not mapped");
  if (g->cfg.layout != EPB_LAYOUT_OPTIMIZED)
    return fail(EPB_INVALID_ARGUMENT, "legacy LL layout is not implemented on the GPU path");
  if (phases < 1 || phases > 3) return fail(EPB_INVALID_ARGUMENT, "phases must be 1 (send), 2 (recv) or 3");
  return EPB_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int epb_ll_dispatch(epb_group* g, uint32_t* hseq, int32_t phases, const epb_ll_dispatch_args* a,
                    void* stream) {
  if (int rc = check_ll(g, phases)) return rc;
  const int wire = g->cfg.token_dtype;
  const int b = a->num_tokens;
  if (b < 0 || b > g->cfg.max_tokens_per_rank)
    return fail(EPB_CAPACITY_EXCEEDED, "token count exceeds max_tokens_per_rank");
  if (phases & kPhaseSend) {
    if (b > 0 && !aligned16(a->x)) return fail(EPB_INVALID_ARGUMENT, "x must be 16-byte aligned");
    if (a->x_scales && g->cfg.hidden % 128) return fail(EPB_INVALID_ARGUMENT, "scaled fp8 input needs H % 128 == 0");
  }
  if (phases & kPhaseRecv) {
    if (a->out_dtype != EPB_F32 && a->out_dtype != wire)
      return fail(EPB_TAG_MISMATCH, "dispatch output must be f32 or the wire dtype");
    if (g->cfg.with_scales && a->out_dtype == wire && !a->out_scales)
      return fail(EPB_TAG_MISMATCH, "fp8 output with scales needs a SCALES output");
    if (!aligned16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  }
  LLDisp p;
  p.x = a->x; p.x_scales = a->x_scales; p.topk = a->topk_idx; p.hseq = hseq;
  p.out = a->out; p.out_scales = a->out_scales; p.counts_f32 = a->counts_f32; p.counts_i32 = a->counts_i32;
  p.src_info = a->src_info; p.peers = g->d_peers; p.win = g->window; p.done = g->d_done; p.err = g->d_err;
  p.dseq = reinterpret_cast<uint32_t*>(g->d_scratch); p.drd = g->d_scratch + 1;
  p.g = g->ll; p.timeout_ns = g->timeout_ns; p.b = b; p.rank = g->rank; p.phases = phases;
  const int recv_warps = (int)std::min<int64_t>(g->ll.n_disp * g->ll.K, 1 << 20);
  int grid = std::max(b, (recv_warps + 7) / 8);
  grid = std::max(1, std::min(grid, 2 * sm_count()));
  const int E = g->ll.E, N = g->ll.N, K = g->ll.K;
  const size_t smem = (phases & kPhaseSend)
      ? sizeof(int) * ((size_t)2 * b * K + (size_t)b * N + E + N) + BlockLayoutSmem::bytes(kThreads / 32, E, N)
      : 0;
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "LL batch too large for the fused dispatch kernel");
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  const int od = a->out_dtype;
  switch ((phases & kPhaseSend) ? a->x_dtype : wire) {
    case EPB_F32: e = run_disp_x<EPB_F32>(p, od, grid, smem, s); break;
    case EPB_BF16: e = run_disp_x<EPB_BF16>(p, od, grid, smem, s); break;
    case EPB_F16: e = run_disp_x<EPB_F16>(p, od, grid, smem, s); break;
    case EPB_FP8: e = run_disp_x<EPB_FP8>(p, od, grid, smem, s); break;
    default: return fail(EPB_INVALID_ARGUMENT, "x dtype");
  }
  if (e != cudaSuccess) return cuda_check(e, "ll_dispatch");
  return EPB_OK;
}

int epb_ll_combine(epb_group* g, const uint32_t* hseq, int32_t phases, const epb_ll_combine_args* a,
                   void* stream) {
  if (int rc = check_ll(g, phases)) return rc;
  const int b = a->num_tokens;
  if (b < 0 || b > g->cfg.max_tokens_per_rank) return fail(EPB_CAPACITY_EXCEEDED, "token count");
  if ((phases & kPhaseSend) && !aligned16(a->expert_out))
    return fail(EPB_INVALID_ARGUMENT, "expert_out must be 16-byte aligned");
  if (phases & kPhaseRecv) {
    if (a->out_dtype != EPB_F32 && a->out_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine output f32|bf16");
    if (!aligned16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  }
  if (a->in_dtype != EPB_F32 && a->in_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine input f32|bf16");
  LLComb p;
  p.y = a->expert_out; p.counts = a->counts_i32; p.src_info = a->src_info; p.w = a->weights; p.out = a->out;
  p.hseq = hseq; p.peers = g->d_peers; p.win = g->window; p.done = g->d_done + g->cfg.num_ranks;
  p.err = g->d_err; p.g = g->ll; p.timeout_ns = g->timeout_ns; p.b = b; p.rank = g->rank; p.phases = phases;
  const size_t smem = sizeof(int) * ((size_t)g->ll.L * g->ll.N + 1);
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "too many (expert, rank) pairs for combine");
  const int rows = g->ll.B * g->ll.K;  // upper bound of rows a rank returns (balanced)
  int grid = std::max(b, (rows + 7) / 8);
  grid = std::max(1, std::min(grid, 2 * sm_count()));
  cudaStream_t s = as_stream(stream);
  cudaError_t e = a->in_dtype == EPB_F32 ? run_comb_w<EPB_F32>(p, a->out_dtype, grid, smem, s)
                                         : run_comb_w<EPB_BF16>(p, a->out_dtype, grid, smem, s);
  if (e != cudaSuccess) return cuda_check(e, "ll_combine");
  return EPB_OK;
}

}  // extern "C"
