// Low-Latency dispatch/combine kernels (K2, K3, K4a, K4b).
//
// Reference semantics (epsim ll.py):
//  * dispatch send (ll.py:289-308): for every destination rank d, the tokens
//    touching d are written, ascending t, into d's slots [src*B + j]; then one
//    counter per (local expert of d, src) carries m(e, src) + 1.  Here the
//    counter word is tagged: (tag << 40) | (q << 20) | m, written with
//    release semantics after this rank's last slot store to d; the tag
//    replaces the reset (ll.py:351-353) so parities are reused race-free.
//  * dispatch recv (ll.py:310-400): wait for all (l, src) counters, then fan
//    every slot out to recv[l, src*B + i] for each local expert it hits;
//    i (the filled[l] order) is precomputed by the sender's routing layout
//    and carried in the slot header next to the reference header fields.
//  * combine send (ll.py:404-462): each valid expert row (l, src, i) is
//    re-encoded in the token dtype (FP8: implicit scale 1) into src's combine
//    slot t*K + k; then constant-tag counters per local expert.
//  * combine recv (ll.py:464-507): out[t] = sum_k w[t,k] * y_k in f32,
//    ascending k, acc starts at 0, no FMA (explicit __fmul_rn/__fadd_rn).
#include "common.cuh"
#include "internal.h"

namespace epb {

struct LLSend {
  const void* x;
  const float* x_scales;
  const int64_t* topk;
  const int32_t* m;
  const int32_t* q;
  const int32_t* tok_rank;
  const int32_t* tok_slot;
  const uint64_t* peers;
  int* done;
  int* err;
  uint32_t* dseq;       // group round counter (device)
  int* drd;             // arrivals of CTAs that read dseq
  uint32_t* hseq;       // out: this round's sequence (handle-owned)
  LLGeom g;
  int b, rank;
};

// Round sequence numbers live on the device so a captured CUDA graph can be
// replayed: the dispatch-send kernel reads the group counter, the last CTA
// to read it stores it into the handle's word and advances the counter;
// every later kernel of the round derives tag and parity from that word.
EPB_DEV uint32_t ll_tag_of(uint32_t seq) { return (seq % 0xFFFFFFu) + 1u; }
EPB_DEV uint32_t ld_volatile_u32(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }

EPB_DEV uint8_t* peer_base(const uint64_t* peers, int r) {
  return reinterpret_cast<uint8_t*>(peers[r]);
}

EPB_DEV void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// counters of pair (l, src=rank) at destination d: m(e, rank) with the tag
EPB_DEV void ll_write_disp_counters(const LLSend& p, int d, int lane, int nlanes, uint64_t parity_off,
                                    uint32_t tag) {
  const LLGeom& g = p.g;
  uint64_t* ctr = reinterpret_cast<uint64_t*>(peer_base(p.peers, d) + parity_off + g.disp_ctr);
  const uint64_t qd = (uint64_t)p.q[d];
  for (int l = lane; l < g.L; l += nlanes) {
    const int e = d * g.L + l;
    const uint64_t m = e < g.E ? (uint64_t)p.m[e] : 0ull;
    st_relaxed_sys(&ctr[l * g.N + p.rank], ((uint64_t)tag << 40) | (qd << 20) | m);
  }
}

// Convert elements [e0, e0 + EPC) of input row (dtype XT) to f32.
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

template <int XT, int WT, bool SC>
__global__ void __launch_bounds__(256) ll_dispatch_send_kernel(LLSend p) {
  __shared__ int s_dst[kMaxRanks], s_j[kMaxRanks], s_nd;
  __shared__ uint32_t s_hdr[2 + 2 * kMaxTopK];
  const LLGeom& g = p.g;
  const int t = blockIdx.x;
  const int K = g.K, N = g.N, H = g.H;
  __shared__ uint32_t s_seq;
  if (threadIdx.x == 0) {
    const uint32_t seq = ld_volatile_u32(p.dseq);
    s_seq = seq;
    __threadfence();
    if (atomicAdd(p.drd, 1) == (int)gridDim.x - 1) {
      *p.drd = 0;
      *p.hseq = seq;
      *p.dseq = seq + 1;
    }
  }
  __syncthreads();
  const uint32_t tag = ll_tag_of(s_seq);
  const uint64_t parity_off = (uint64_t)(s_seq & 1) * g.parity_bytes;
  if (t < p.b) {
    if (threadIdx.x == 0) {
      int nd = 0;
      for (int d = 0; d < N; ++d) {
        const int j = p.tok_slot[(int64_t)t * N + d];
        if (j >= 0) { s_dst[nd] = d; s_j[nd] = j; ++nd; }
      }
      s_nd = nd;
      s_hdr[0] = (uint32_t)t;
      s_hdr[1] = (uint32_t)K;
    }
    if (threadIdx.x < K) {
      s_hdr[2 + threadIdx.x] = (uint32_t)p.topk[(int64_t)t * K + threadIdx.x];
      s_hdr[2 + K + threadIdx.x] = (uint32_t)p.tok_rank[(int64_t)t * K + threadIdx.x];
    }
    __syncthreads();
    const int nd = s_nd;
    const uint64_t slot_off = parity_off + g.disp_slot;
    const int64_t slot_idx = (int64_t)p.rank * g.B;
    // header words
    for (int w = threadIdx.x; w < 2 + 2 * K; w += blockDim.x) {
      for (int i = 0; i < nd; ++i) {
        uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_idx + s_j[i]) * g.slot_stride;
        reinterpret_cast<uint32_t*>(slot + g.RBp + g.SBp)[w] = s_hdr[w];
      }
    }
    const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * dtype_width(XT);
    const float* xsc = p.x_scales ? p.x_scales + (int64_t)t * (H / 128) : nullptr;
    if ((H & 15) == 0) {
      constexpr int EPC = Elems<WT>::n;
      const int nch = H / EPC;
      const int lane = threadIdx.x & 31;
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
          uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_idx + s_j[i]) * g.slot_stride;
          st_na_v4(slot + (int64_t)c * 16, v);
          if constexpr (SC) {
            if ((c & 7) == 0) reinterpret_cast<float*>(slot + g.RBp)[c >> 3] = scale;
          }
        }
      }
    } else {
      // unaligned hidden: element path (no scales possible: H % 128 != 0)
      for (int el = threadIdx.x; el < H; el += blockDim.x) {
        float f = load_elem(xrow, XT, el);
        if constexpr (XT == EPB_FP8) {
          if (xsc != nullptr) f = __fmul_rn(f, xsc[el >> 7]);
        }
        for (int i = 0; i < nd; ++i) {
          uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (slot_idx + s_j[i]) * g.slot_stride;
          store_elem(slot, WT, el, f);
        }
      }
    }
    __syncthreads();
    // completion: the last CTA to finish a token for d publishes d's counters
    if (threadIdx.x < 32) {
      for (int i = 0; i < nd; ++i) {
        const int d = s_dst[i];
        int last = 0;
        if (threadIdx.x == 0) {
          fence_sys();
          const int old = atomicAdd(&p.done[d], 1);
          last = (old == p.q[d] - 1);
          if (last) p.done[d] = 0;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          fence_sys();
          ll_write_disp_counters(p, d, threadIdx.x, 32, parity_off, tag);
        }
      }
    }
  }
  // ranks this rank sends nothing to still get their (m = 0) counters
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    for (int d = 0; d < N; ++d)
      if (p.q[d] == 0) ll_write_disp_counters(p, d, threadIdx.x, 32, parity_off, tag);
  }
}

// ---------------------------------------------------------------------------
struct LLRecv {
  void* out;
  float* out_scales;
  float* counts_f32;
  int32_t* counts_i32;
  int32_t* src_info;
  const uint8_t* win;
  int* err;
  const uint32_t* hseq;
  LLGeom g;
  uint64_t timeout_ns;
  int rank;
};

// copy one received wire row (WT, optional scales) to an output row (OT)
template <int WT, bool SC, int OT>
EPB_DEV void ll_copy_row(const LLGeom& g, const uint8_t* slot, uint8_t* orow, float* osc, int lane) {
  const int H = g.H;
  if ((H & 15) == 0) {
    constexpr int EPC = Elems<WT>::n;
    const int nch = H / EPC;
    if constexpr (OT == WT) {
      for (int c = lane; c < nch; c += 32) st_v4(orow + (int64_t)c * 16, ld_v4(slot + (int64_t)c * 16));
      if constexpr (SC) {
        const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
        for (int i = lane; i < H / 128; i += 32) osc[i] = sc[i];
      }
    } else {
      static_assert(OT == EPB_F32, "recv output is f32 or the wire dtype");
      const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
      for (int c = lane; c < nch; c += 32) {
        float f[EPC];
        unpack16<WT>(ld_v4(slot + (int64_t)c * 16), f);
        if constexpr (SC) {
          const float s = sc[(c * EPC) >> 7];
#pragma unroll
          for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], s);
        }
#pragma unroll
        for (int q = 0; q < EPC / 4; ++q)
          st_v4(orow + ((int64_t)c * EPC + q * 4) * 4,
                make_int4(__float_as_int(f[4 * q]), __float_as_int(f[4 * q + 1]),
                          __float_as_int(f[4 * q + 2]), __float_as_int(f[4 * q + 3])));
      }
    }
  } else {
    for (int el = lane; el < H; el += 32) {
      float f = load_elem(slot, WT, el);
      if constexpr (OT == WT) {
        if constexpr (OT == EPB_F32) reinterpret_cast<float*>(orow)[el] = f;
        else if constexpr (OT == EPB_FP8) orow[el] = slot[el];
        else reinterpret_cast<uint16_t*>(orow)[el] = reinterpret_cast<const uint16_t*>(slot)[el];
      } else {
        reinterpret_cast<float*>(orow)[el] = f;
      }
    }
  }
}

template <int WT, bool SC, int OT>
__global__ void __launch_bounds__(256) ll_dispatch_recv_kernel(LLRecv p) {
  __shared__ int s_q[kMaxRanks], s_pre[kMaxRanks + 1];
  __shared__ int s_fail;
  const LLGeom& g = p.g;
  const int N = g.N, L = g.L, K = g.K, B = g.B;
  const int lo = p.rank * L;
  const int nloc = max(0, min(L, g.E - lo));
  if (threadIdx.x == 0) s_fail = 0;
  if (threadIdx.x < N) s_q[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t seq = ld_volatile_u32(p.hseq);
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
  const uint64_t* ctr = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.disp_ctr);
  for (int i = threadIdx.x; i < nloc * N; i += blockDim.x) {
    uint64_t v = 0;
    if (!wait_tag(&ctr[i], tag, 40, 0xFFFFFFu, p.timeout_ns, p.err, &v)) {
      s_fail = 1;
      continue;
    }
    const int l = i / N, s = i % N;
    if (l == 0) s_q[s] = (int)((v >> 20) & 0xFFFFF);
    if (blockIdx.x == 0) {
      const int m = (int)(v & 0xFFFFF);
      p.counts_i32[i] = m;
      p.counts_f32[i] = (float)m;
    }
  }
  if (blockIdx.x == 0) {
    for (int i = nloc * N + threadIdx.x; i < L * N; i += blockDim.x) {
      p.counts_i32[i] = 0;
      p.counts_f32[i] = 0.0f;
    }
  }
  __syncthreads();
  if (s_fail) return;
  if (threadIdx.x == 0) {
    int run = 0;
    for (int s = 0; s < N; ++s) { s_pre[s] = run; run += s_q[s]; }
    s_pre[N] = run;
  }
  __syncthreads();
  const int total = s_pre[N];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int ob = (OT == EPB_F32 ? 4 : dtype_width(OT));
  const int64_t orow_bytes = (int64_t)g.H * ob;
  for (int f = blockIdx.x * nw + warp; f < total; f += gridDim.x * nw) {
    int s = 0;
    while (s_pre[s + 1] <= f) ++s;
    const int j = f - s_pre[s];
    const uint8_t* slot = p.win + parity_off + g.disp_slot + ((int64_t)s * B + j) * g.slot_stride;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
    const uint32_t t = hdr[0];
    for (int k = 0; k < K; ++k) {
      const int e = (int)hdr[2 + k];
      if (e < lo || e >= lo + nloc) continue;
      const int l = e - lo;
      const int64_t row = (int64_t)l * N * B + (int64_t)s * B + hdr[2 + K + k];
      if (lane == 0) p.src_info[row] = (int32_t)(t * K + k);
      ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + row * orow_bytes,
                              SC ? p.out_scales + row * (g.H / 128) : nullptr, lane);
    }
  }
}

// ---------------------------------------------------------------------------
struct LLCombSend {
  const void* y;
  const int32_t* counts;
  const int32_t* src_info;
  const uint64_t* peers;
  int* done;
  int* err;
  const uint32_t* hseq;
  LLGeom g;
  int rank;
};

EPB_DEV void ll_write_comb_counters(const LLCombSend& p, int s, uint64_t parity_off, uint32_t tag) {
  const LLGeom& g = p.g;
  uint64_t* ctr = reinterpret_cast<uint64_t*>(peer_base(p.peers, s) + parity_off + g.comb_ctr);
  const int lo = p.rank * g.L;
  const int hi = min(lo + g.L, g.E);
  for (int e = lo; e < hi; ++e) st_relaxed_sys(&ctr[e], (uint64_t)tag);
}

template <int IT, int WT>
__global__ void __launch_bounds__(256) ll_combine_send_kernel(LLCombSend p) {
  extern __shared__ int s_pre[];            // [L*N + 1]
  __shared__ int s_rows_to[kMaxRanks], s_cnt[kMaxRanks];
  const LLGeom& g = p.g;
  const int N = g.N, L = g.L, B = g.B, H = g.H;
  const int P = L * N;
  const uint32_t seq = ld_volatile_u32(p.hseq);
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
  if (threadIdx.x < N) { s_rows_to[threadIdx.x] = 0; s_cnt[threadIdx.x] = 0; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < P; ++i) {
      s_pre[i] = run;
      const int c = p.counts[i];
      run += c;
      s_rows_to[i % N] += c;
    }
    s_pre[P] = run;
  }
  __syncthreads();
  const int total = s_pre[P];
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(total, r0 + per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ib = dtype_width(IT);
  for (int r = r0 + warp; r < r1; r += nw) {
    int lo_i = 0, hi_i = P;  // largest pair with s_pre[pair] <= r
    while (hi_i - lo_i > 1) {
      const int mid = (lo_i + hi_i) >> 1;
      if (s_pre[mid] <= r) lo_i = mid; else hi_i = mid;
    }
    const int pair = lo_i;
    const int l = pair / N, s = pair % N, i = r - s_pre[pair];
    const int64_t row = (int64_t)l * N * B + (int64_t)s * B + i;
    const int info = p.src_info[row];
    uint8_t* dst = peer_base(p.peers, s) + parity_off + g.comb_slot + (int64_t)info * g.comb_stride;
    const uint8_t* yrow = reinterpret_cast<const uint8_t*>(p.y) + row * H * ib;
    if ((H & 15) == 0) {
      constexpr int EPC = Elems<WT>::n;
      for (int c = lane; c < H / EPC; c += 32) {
        float f[EPC];
        load_elems_vec<IT, EPC>(yrow, (int64_t)c * EPC, f);
        st_na_v4(dst + (int64_t)c * 16, pack16<WT>(f));
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
    if (c > 0) {
      fence_sys();
      const int old = atomicAdd(&p.done[s], c);
      if (old + c == s_rows_to[s]) {
        p.done[s] = 0;
        fence_sys();
        ll_write_comb_counters(p, s, parity_off, tag);
      }
    } else if (blockIdx.x == 0 && s_rows_to[s] == 0) {
      ll_write_comb_counters(p, s, parity_off, tag);
    }
  }
}

// ---------------------------------------------------------------------------
struct LLCombRecv {
  const float* w;
  void* out;
  const uint8_t* win;
  int* err;
  const uint32_t* hseq;
  LLGeom g;
  uint64_t timeout_ns;
  int b;
};

template <int WT, int OT>
__global__ void __launch_bounds__(256) ll_combine_recv_kernel(LLCombRecv p) {
  __shared__ float s_w[kMaxTopK];
  __shared__ int s_fail;
  const LLGeom& g = p.g;
  const int K = g.K, H = g.H;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  const uint32_t seq = ld_volatile_u32(p.hseq);
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
  const uint64_t* ctr = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.comb_ctr);
  for (int e = threadIdx.x; e < g.E; e += blockDim.x) {
    uint64_t v;
    if (!wait_tag(&ctr[e], tag, 0, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) return;
  const uint8_t* slots = p.win + parity_off + g.comb_slot;
  for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
    if (threadIdx.x < K) s_w[threadIdx.x] = p.w[(int64_t)t * K + threadIdx.x];
    __syncthreads();
    uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * dtype_width(OT);
    if ((H & 15) == 0) {
      constexpr int EPC = Elems<WT>::n;
      for (int c = threadIdx.x; c < H / EPC; c += blockDim.x) {
        float acc[EPC];
#pragma unroll
        for (int i = 0; i < EPC; ++i) acc[i] = 0.0f;
        for (int k = 0; k < K; ++k) {
          float y[EPC];
          unpack16<WT>(ld_v4(slots + ((int64_t)t * K + k) * g.comb_stride + (int64_t)c * 16), y);
          const float wk = s_w[k];
#pragma unroll
          for (int i = 0; i < EPC; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(wk, y[i]));
        }
        store_f32_chunk<OT, EPC>(orow, (int64_t)c * EPC, acc);
      }
    } else {
      for (int el = threadIdx.x; el < H; el += blockDim.x) {
        float acc = 0.0f;
        for (int k = 0; k < K; ++k)
          acc = __fadd_rn(acc, __fmul_rn(s_w[k], load_elem(slots + ((int64_t)t * K + k) * g.comb_stride, WT, el)));
        store_elem(orow, OT, el, acc);
      }
    }
    __syncthreads();
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

template <int XT, int WT, bool SC>
cudaError_t launch_send(const LLSend& p, cudaStream_t s) {
  ll_dispatch_send_kernel<XT, WT, SC><<<max(p.b, 1), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <int XT>
cudaError_t launch_send_x(const LLSend& p, cudaStream_t s) {
  switch (p.g.wire) {
    case EPB_F32: return launch_send<XT, EPB_F32, false>(p, s);
    case EPB_BF16: return launch_send<XT, EPB_BF16, false>(p, s);
    case EPB_F16: return launch_send<XT, EPB_F16, false>(p, s);
    default:
      return p.g.scales ? launch_send<XT, EPB_FP8, true>(p, s) : launch_send<XT, EPB_FP8, false>(p, s);
  }
}

template <int WT, bool SC, int OT>
cudaError_t launch_recv(const LLRecv& p, int grid, cudaStream_t s) {
  ll_dispatch_recv_kernel<WT, SC, OT><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <int WT, bool SC>
cudaError_t launch_recv_w(const LLRecv& p, int out_dtype, int grid, cudaStream_t s) {
  if (out_dtype == EPB_F32) return launch_recv<WT, SC, EPB_F32>(p, grid, s);
  return launch_recv<WT, SC, WT>(p, grid, s);
}

template <int IT, int WT>
cudaError_t launch_csend(const LLCombSend& p, int grid, size_t smem, cudaStream_t s) {
  ll_combine_send_kernel<IT, WT><<<grid, 256, smem, s>>>(p);
  return cudaGetLastError();
}

template <int IT>
cudaError_t launch_csend_i(const LLCombSend& p, int grid, size_t smem, cudaStream_t s) {
  switch (p.g.cwire) {
    case EPB_F32: return launch_csend<IT, EPB_F32>(p, grid, smem, s);
    case EPB_BF16: return launch_csend<IT, EPB_BF16>(p, grid, smem, s);
    case EPB_F16: return launch_csend<IT, EPB_F16>(p, grid, smem, s);
    default: return launch_csend<IT, EPB_FP8>(p, grid, smem, s);
  }
}

template <int WT, int OT>
cudaError_t launch_crecv(const LLCombRecv& p, cudaStream_t s) {
  ll_combine_recv_kernel<WT, OT><<<max(1, min(p.b, 4 * sm_count())), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <int WT>
cudaError_t launch_crecv_w(const LLCombRecv& p, int out_dtype, cudaStream_t s) {
  return out_dtype == EPB_F32 ? launch_crecv<WT, EPB_F32>(p, s) : launch_crecv<WT, EPB_BF16>(p, s);
}

int check_ll(epb_group* g) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (g->cfg.algorithm != EPB_LL) return fail(EPB_HANDLE_STATE_ERROR, "group is not LL");
  if (!g->peers_ready) return fail(EPB_HANDLE_STATE_ERROR, "peer windows not mapped");
  if (g->cfg.layout != EPB_LAYOUT_OPTIMIZED)
    return fail(EPB_INVALID_ARGUMENT, "legacy LL layout is not implemented on the GPU path");
  return EPB_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int epb_ll_dispatch_send(epb_group* g, uint32_t* hseq, const void* x, int32_t x_dtype,
                         const float* x_scales, const int64_t* topk_idx, const epb_layout* lay,
                         void* stream) {
  if (int rc = check_ll(g)) return rc;
  if (!lay) return fail(EPB_INVALID_ARGUMENT, "null layout");
  if (x_scales && g->cfg.hidden % 128) return fail(EPB_INVALID_ARGUMENT, "scaled fp8 input needs H % 128 == 0");
  if (lay->num_tokens > 0 && !aligned16(x)) return fail(EPB_INVALID_ARGUMENT, "x must be 16-byte aligned");
  LLSend p;
  p.x = x; p.x_scales = x_scales; p.topk = topk_idx; p.m = lay->expert_count; p.q = lay->rank_count;
  p.tok_rank = lay->tok_rank; p.tok_slot = lay->tok_slot; p.peers = g->d_peers; p.done = g->d_done;
  p.err = g->d_err; p.g = g->ll; p.b = lay->num_tokens; p.rank = g->rank;
  p.dseq = reinterpret_cast<uint32_t*>(g->d_scratch); p.drd = g->d_scratch + 1; p.hseq = hseq;
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  switch (x_dtype) {
    case EPB_F32: e = launch_send_x<EPB_F32>(p, s); break;
    case EPB_BF16: e = launch_send_x<EPB_BF16>(p, s); break;
    case EPB_F16: e = launch_send_x<EPB_F16>(p, s); break;
    case EPB_FP8: e = launch_send_x<EPB_FP8>(p, s); break;
    default: return fail(EPB_INVALID_ARGUMENT, "x dtype");
  }
  if (e != cudaSuccess) return cuda_check(e, "ll_dispatch_send");
  return EPB_OK;
}

int epb_ll_dispatch_recv(epb_group* g, const uint32_t* hseq, void* out, int32_t out_dtype, float* out_scales,
                         float* counts_f32, int32_t* counts_i32, int32_t* src_info, void* stream) {
  if (int rc = check_ll(g)) return rc;
  const int wire = g->cfg.token_dtype;
  if (out_dtype != EPB_F32 && out_dtype != wire)
    return fail(EPB_TAG_MISMATCH, "dispatch output must be f32 or the wire dtype");
  const bool sc = g->cfg.with_scales;
  if (sc && out_dtype == wire && !out_scales)
    return fail(EPB_TAG_MISMATCH, "fp8 output with scales needs a SCALES output");
  if (!aligned16(out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  LLRecv p;
  p.out = out; p.out_scales = out_scales; p.counts_f32 = counts_f32; p.counts_i32 = counts_i32;
  p.src_info = src_info; p.win = g->window; p.err = g->d_err; p.g = g->ll;
  p.hseq = hseq; p.timeout_ns = g->timeout_ns; p.rank = g->rank;
  const int grid = max(1, min(2 * sm_count(), (int)((g->ll.n_disp + 7) / 8)));
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  switch (wire) {
    case EPB_F32: e = launch_recv<EPB_F32, false, EPB_F32>(p, grid, s); break;
    case EPB_BF16: e = launch_recv_w<EPB_BF16, false>(p, out_dtype, grid, s); break;
    case EPB_F16: e = launch_recv_w<EPB_F16, false>(p, out_dtype, grid, s); break;
    default:
      e = sc ? launch_recv_w<EPB_FP8, true>(p, out_dtype, grid, s)
             : launch_recv_w<EPB_FP8, false>(p, out_dtype, grid, s);
  }
  if (e != cudaSuccess) return cuda_check(e, "ll_dispatch_recv");
  return EPB_OK;
}

int epb_ll_combine_send(epb_group* g, const uint32_t* hseq, const void* expert_out, int32_t in_dtype,
                        const int32_t* counts_i32, const int32_t* src_info, void* stream) {
  if (int rc = check_ll(g)) return rc;
  if (!aligned16(expert_out)) return fail(EPB_INVALID_ARGUMENT, "expert_out must be 16-byte aligned");
  LLCombSend p;
  p.y = expert_out; p.counts = counts_i32; p.src_info = src_info; p.peers = g->d_peers;
  p.done = g->d_done + g->cfg.num_ranks; p.err = g->d_err; p.g = g->ll;
  p.hseq = hseq; p.rank = g->rank;
  const int P = g->ll.L * g->ll.N;
  const size_t smem = sizeof(int) * (P + 1);
  const int grid = max(1, min(2 * sm_count(), (g->ll.B * g->ll.K + 7) / 8 + 1));
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  if (smem > 48 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "too many (expert, rank) pairs for combine");
  switch (in_dtype) {
    case EPB_F32: e = launch_csend_i<EPB_F32>(p, grid, smem, s); break;
    case EPB_BF16: e = launch_csend_i<EPB_BF16>(p, grid, smem, s); break;
    default: return fail(EPB_TAG_MISMATCH, "combine input must be f32 or bf16");
  }
  if (e != cudaSuccess) return cuda_check(e, "ll_combine_send");
  return EPB_OK;
}

int epb_ll_combine_recv(epb_group* g, const uint32_t* hseq, const float* weights, int32_t b, void* out,
                        int32_t out_dtype, void* stream) {
  if (int rc = check_ll(g)) return rc;
  if (b < 0 || b > g->cfg.max_tokens_per_rank) return fail(EPB_CAPACITY_EXCEEDED, "token count");
  if (out_dtype != EPB_F32 && out_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine output f32|bf16");
  if (!aligned16(out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  LLCombRecv p;
  p.w = weights; p.out = out; p.win = g->window; p.err = g->d_err; p.g = g->ll;
  p.hseq = hseq; p.timeout_ns = g->timeout_ns; p.b = b;
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  switch (g->ll.cwire) {
    case EPB_F32: e = launch_crecv_w<EPB_F32>(p, out_dtype, s); break;
    case EPB_BF16: e = launch_crecv_w<EPB_BF16>(p, out_dtype, s); break;
    case EPB_F16: e = launch_crecv_w<EPB_F16>(p, out_dtype, s); break;
    default: e = launch_crecv_w<EPB_FP8>(p, out_dtype, s); break;
  }
  if (e != cudaSuccess) return cuda_check(e, "ll_combine_recv");
  return EPB_OK;
}

}  // extern "C"
