// Low-Latency dispatch / combine: two kernels per round (K2+K3 fused, K4a+K4b
// fused), each runnable as send-only, recv-only or both (one cooperative
// launch).  Every LL launch uses the same fixed grid (kLLGrid CTAs) on every
// rank, so a receiver knows how many per-CTA flags each peer publishes.
//
// Reference semantics (epsim ll.py):
//  * dispatch send (ll.py:255-308): per destination rank d, the tokens that
//    touch d go, ascending t, into d's slots [src*B + j]; the receiver learns
//    m(e, src) per (local expert, src) pair (the reference's counter value
//    m + 1).  Here CTA 0 of the source writes the tagged count words
//    (tag << 40) | (q << 20) | m and every source CTA publishes one tagged
//    flag per destination after a release fence; the tag (from the round
//    sequence) replaces the reference's counter reset (ll.py:351-353).
//  * dispatch recv (ll.py:310-400): after all flags of all sources, every
//    slot row goes to recv[l, src*B + i] for each local expert; i (the
//    filled[l] order) and j (the slot) are prefix counts the SENDER computes
//    over its earlier tokens, i travels in the slot header after the
//    reference header fields (layout.py:282-295).
//  * combine send (ll.py:404-462): each valid expert row (l, src, i) goes,
//    in the combine wire dtype, to src's slot t*K + k.
//  * combine recv (ll.py:464-507): out[t] = sum_k w[t,k] * y_k in f32,
//    ascending k from acc = 0, explicit __fmul_rn/__fadd_rn (no FMA).
//
// Latency design (B200): the token row is prefetched into registers at
// kernel start so its DRAM latency hides behind the routing pass; routing
// validation, counts and prefix ranks are one parallel shared-memory pass;
// flags replace atomics; copies keep 8 x 16 B loads in flight per lane;
// fences/flags use GPU scope when every rank lives on this GPU.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace epb {

constexpr int kPhaseSend = 1, kPhaseRecv = 2;
constexpr int kThreads = 512;
constexpr int kUnroll = 8;
constexpr int kParts = 4;  // combine send: warps per row

// diagnostics: thread 0 of each CTA stamps the global timer at checkpoints
#define LL_STAMP(P, I)                                                                    \
  do {                                                                                   \
    if ((P).trace && threadIdx.x == 0) (P).trace[blockIdx.x * 16 + (I)] = globaltimer(); \
  } while (0)

EPB_DEV uint32_t ll_tag_of(uint32_t seq) { return (seq % 0xFFFFFFu) + 1u; }
// round counters: written by an earlier kernel (visible at the kernel
// boundary) and not again until every CTA has read them — a relaxed GPU-scope
// load suffices (a volatile, i.e. system-scope, load measured ~2 us slower)
EPB_DEV uint32_t ld_round_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
EPB_DEV uint8_t* peer_base(const uint64_t* peers, int r) { return reinterpret_cast<uint8_t*>(peers[r]); }

// (the release fence itself: fence_release in common.cuh)
EPB_DEV void st_flag(uint64_t* p, uint64_t v, bool sys) {
  if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
EPB_DEV uint64_t ld_flag(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// spin until the low 32 bits equal `tag` (bounded; records TransportClosed)
EPB_DEV bool wait_flag(const uint64_t* f, uint32_t tag, bool sys, uint64_t timeout_ns, int* err) {
  uint64_t start = 0;
  for (int spins = 0;; ++spins) {
    if ((uint32_t)ld_flag(f, sys) == tag) return true;
    if ((spins & 31) != 31) continue;
    if (*(volatile int*)err != 0) return false;
    if (spins == 63) start = globaltimer();
    if (spins > 64 && (spins & 255) == 255 && globaltimer() - start > timeout_ns) {
      atomicCAS(err, 0, EPB_TRANSPORT_CLOSED);
      return false;
    }
  }
}
EPB_DEV int4 ld_weak_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
EPB_DEV void st_weak_v4(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

// Warp-cooperative copy of chunks [c0, c1) (16 B each), kUnroll loads in flight per lane.
EPB_DEV void warp_copy16(const uint8_t* src, uint8_t* dst, int c0, int c1, int lane) {
  for (int base = c0; base < c1; base += 32 * kUnroll) {
    int4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * 32 + lane;
      if (c < c1) v[u] = ld_weak_v4(src + (int64_t)c * 16);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = base + u * 32 + lane;
      if (c < c1) st_weak_v4(dst + (int64_t)c * 16, v[u]);
    }
  }
}

// Block-wide exclusive scan of val(0..P-1) into s_pre[0..P] (s_pre[P] =
// total); all threads call it; ends with a block barrier.
template <class F>
EPB_DEV void block_exclusive_scan(int P, F val, int* s_pre, int* s_wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (P + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per;
  int local = 0;
  for (int i = i0; i < min(P, i0 + per); ++i) local += val(i);
  int incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  int run = incl - local;
  for (int w2 = 0; w2 < warp; ++w2) run += s_wsum[w2];
  for (int i = i0; i < min(P, i0 + per); ++i) {
    s_pre[i] = run;
    run += val(i);
  }
  if (threadIdx.x == blockDim.x - 1) s_pre[P] = run;
  __syncthreads();
}

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
  int32_t* self_row;     // [b*K] row of (t, k) in this rank's output if e_tk is local, else -1
  int32_t* owner_row;    // [b*K] row of (t, k) in e_tk's owner's output (pulled combine), nullable
  const uint64_t* peers;
  const uint8_t* win;
  int* err;
  uint32_t* dseq;
  int* drd;
  uint64_t* trace;
  LLGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
  bool sys;
};

// copy one received slot row (WT, optional scales) to an output row (OT)
// (part `part` of `parts` equal chunk ranges; the scales go with part 0)
template <int WT, bool SC, int OT>
EPB_DEV void ll_copy_row(const LLGeom& g, const uint8_t* slot, uint8_t* orow, float* osc, int lane, int part,
                         int parts) {
  const int H = g.H;
  if ((H & 15) == 0) {
    constexpr int EPC = Elems<WT>::n;
    const int nch = H / EPC;
    const int per = (nch + parts - 1) / parts;
    const int c0 = part * per, c1 = min(nch, c0 + per);
    if constexpr (OT == WT) {
      warp_copy16(slot, orow, c0, c1, lane);
      if constexpr (SC) {
        const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
        if (part == 0)
          for (int i = lane; i < H / 128; i += 32) osc[i] = sc[i];
      }
    } else {
      static_assert(OT == EPB_F32, "recv output is f32 or the wire dtype");
      const float* sc = reinterpret_cast<const float*>(slot + g.RBp);
      for (int base = c0; base < c1; base += 32 * 4) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) v[u] = ld_weak_v4(slot + (int64_t)c * 16);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) {
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
    if (part != 0) return;
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
  const int K = g.K, N = g.N, H = g.H, L = g.L, E = g.E, B = g.B, G = g.grid;
  const int b = p.b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool sys = p.sys;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : (XT == EPB_FP8 ? 1 : 2);
  constexpr int NV = (EPC * XW) >= 16 ? (EPC * XW) / 16 : 0;  // 16-B input loads per chunk
  const bool vec = (H & 15) == 0;
  const int nch = vec ? H / EPC : 0;
  constexpr int OB = OT == EPB_F32 ? 4 : (OT == EPB_FP8 ? 1 : 2);  // output element bytes

  // split: warps 1.. quantise a token's chunks (<= 2 each, in registers)
  // while warp 0 resolves its destinations; else every thread loops
  const int nq = (int)blockDim.x - 32;
  const bool split = vec && nch <= 2 * nq;
  const int c_first = split ? (int)threadIdx.x - 32 : (int)threadIdx.x;  // first chunk of this thread
  // prefetch this CTA's first token chunk: its DRAM latency overlaps the
  // routing pass below
  int4 xr[NV > 0 ? NV : 1];
  const bool pre = (p.phases & kPhaseSend) && NV > 0 && vec && (int)blockIdx.x < b && c_first >= 0 && c_first < nch;
  if (pre) {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.x) +
                         ((int64_t)blockIdx.x * H + (int64_t)c_first * EPC) * XW;
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) xr[v] = ld_nc_v4(src + 16 * v);
  }
  // prefetch this thread's first two routing items (t*K + k) and, for
  // top-k <= 8, the routing row of token t = threadIdx.x (validation)
  int64_t rid0 = 0, rid1 = 0;
  int64_t row[8];
  const bool row_pre = (p.phases & kPhaseSend) && K <= 8 && (int)threadIdx.x < b;
  if (p.phases & kPhaseSend) {
    const int i0 = (int)threadIdx.x, i1 = i0 + (int)blockDim.x;
    if (i0 < b * K) rid0 = __ldg(p.topk + i0);
    if (i1 < b * K) rid1 = __ldg(p.topk + i1);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) row[k] = (row_pre && k < K) ? __ldg(p.topk + (int64_t)threadIdx.x * K + k) : -1 - k;
  LL_STAMP(p, 0);
  // round sequence: thread 0 issues the load now; it lands in shared memory
  // at the first block barrier after the routing pass (send) or right away
  __shared__ uint32_t s_seq;
  uint32_t seq_ld = 0;
  if (threadIdx.x == 0) seq_ld = ld_round_u32((p.phases & kPhaseSend) ? p.dseq : p.hseq);
  uint32_t seq = 0, tag = 0;
  uint64_t parity_off = 0;
  // per-expert token counts of this round (send phase; the fused receive
  // takes its own-rank counts from here)
  int* s_m = nullptr;

  if (p.phases & kPhaseSend) {
    // shared: routing snapshot, per-expert and per-destination token bitmaps
    // (bit t' of word t'/32), per-expert / per-destination counts
    const int W = (b + 31) >> 5;
    int* s_topk = smem;                                                        // [b*K]
    uint32_t* s_ebits = reinterpret_cast<uint32_t*>(s_topk + b * K);           // [E][W]
    uint32_t* s_dbits = s_ebits + E * W;                                       // [N][W]
    s_m = reinterpret_cast<int*>(s_dbits + N * W);                             // [E]
    int* s_q = s_m + E;                                                        // [N]
    __shared__ int s_bad, s_nd;
    // per destination entry: rank and absolute slot index in its window
    // (optimized: one slot per (token, dst) at src*B + j; legacy: one slot
    // per (token, expert) at ((e - dL)*N + src)*B + i)
    __shared__ int s_dst[kMaxRanks], s_j[kMaxRanks];
    __shared__ int s_self[kMaxTopK];  // output row of (t, k) for this rank's own experts, else -1
    __shared__ uint32_t s_hdr[2 + 2 * kMaxTopK];
    for (int i = threadIdx.x; i < E * W; i += blockDim.x) s_ebits[i] = 0;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    LL_STAMP(p, 8);
    // routing (api.py:150-170).  Rows: range check and distinct experts,
    // from registers (one token per thread).  Items (t, k), one per thread
    // per pass (coalesced): snapshot and the token bitmap of each expert.
    // No value-returning atomics and no dependent shared-memory chains on
    // this path: each link of such a chain costs ~30+ cycles.
    for (int t = threadIdx.x; t < b; t += blockDim.x) {
      bool ok = true;
      if (K <= 8) {
        int64_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (t == (int)threadIdx.x && row_pre) ? row[k] : (k < K ? p.topk[(int64_t)t * K + k] : -1 - k);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ok &= k >= K || (v[k] >= 0 && v[k] < E);
#pragma unroll
          for (int j = 0; j < k; ++j) ok &= v[j] != v[k];
        }
      } else {
        for (int k = 0; k < K; ++k) {
          const int64_t e = p.topk[(int64_t)t * K + k];
          ok &= e >= 0 && e < E;
          for (int j = 0; j < k; ++j) ok &= p.topk[(int64_t)t * K + j] != e;
        }
      }
      if (!ok) s_bad = 1;
    }
    const int items = b * K;
    for (int i = threadIdx.x, r = 0; i < items; i += blockDim.x, ++r) {
      const int64_t e = r == 0 ? rid0 : (r == 1 ? rid1 : p.topk[i]);
      const int t = (int)(((uint64_t)i * g.Kmagic) >> 32);
      s_topk[i] = (int)e;
      if (e >= 0 && e < E) atomicOr(&s_ebits[(int)e * W + (t >> 5)], 1u << (t & 31));
    }
    __syncthreads();
    LL_STAMP(p, 13);
    // per expert (threads [0, E)): token count = popcount of its bitmap;
    // per destination word (threads [E, E + N*W)): OR of its experts' words
    for (int u = threadIdx.x; u < E + N * W; u += blockDim.x) {
      if (u < E) {
        int m = 0;
        if (W <= 16) {
#pragma unroll
          for (int w = 0; w < 16; ++w) m += w < W ? __popc(s_ebits[u * W + min(w, W - 1)]) : 0;
        } else {
          for (int w = 0; w < W; ++w) m += __popc(s_ebits[u * W + w]);
        }
        s_m[u] = m;
      } else {
        const int d = (u - E) / W, w = (u - E) - d * W;
        const int e0 = d * L, e1 = min(E, e0 + L);
        uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
        int e = e0;
        for (; e + 4 <= e1; e += 4) {
          o0 |= s_ebits[e * W + w];
          o1 |= s_ebits[(e + 1) * W + w];
          o2 |= s_ebits[(e + 2) * W + w];
          o3 |= s_ebits[(e + 3) * W + w];
        }
        for (; e < e1; ++e) o0 |= s_ebits[e * W + w];
        s_dbits[d * W + w] = o0 | o1 | o2 | o3;
      }
    }
    LL_STAMP(p, 10);
    uint32_t arrived = 0;
    if (threadIdx.x == 0) {
      s_seq = seq_ld;
      LL_STAMP(p, 11);
      // every CTA has read the round counter (its value is consumed above,
      // so the read is complete): arrive now, act on the result at the end
      // of the send phase (the round trip overlaps it)
      arrived = atomicAdd(reinterpret_cast<unsigned*>(p.drd), 1u);
      LL_STAMP(p, 12);
    }
    __syncthreads();
    seq = s_seq;
    tag = ll_tag_of(seq);
    parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
    LL_STAMP(p, 1);
    // the last CTA to arrive records the round in the handle word and
    // advances the group counter (all CTAs have read it)
    auto commit_round = [&]() {
      if (threadIdx.x == 0 && arrived == (uint32_t)gridDim.x - 1) {
        *p.drd = 0;
        *p.hseq = seq;
        *p.dseq = seq + 1;
      }
    };
    if (s_bad) {
      // validation before any traffic: every CTA reaches the same verdict
      if (threadIdx.x == 0) atomicCAS(p.err, 0, EPB_INVALID_ARGUMENT);
      commit_round();
      return;
    }
    LL_STAMP(p, 2);
    // tokens per destination (count words), read at the publish below
    for (int d = threadIdx.x; d < N; d += blockDim.x) {
      int q = 0;
      for (int w = 0; w < W; ++w) q += __popc(s_dbits[d * W + w]);
      s_q[d] = q;
    }
    const uint64_t slot_off = parity_off + g.disp_slot;
    const bool legacy = g.layout == EPB_LAYOUT_LEGACY;
    // one token chunk: input (prefetched for the CTA's first token) ->
    // f32 -> optional block-128 FP8 scale (x / scale, correctly rounded) ->
    // 16-B wire image
    auto quantize = [&](int t, int c, const uint8_t* xrow, const float* xsc, int4& v, float& scale) {
      float f[EPC];
      if (pre && t == (int)blockIdx.x && c == c_first) {
        if constexpr (NV > 0) {
          constexpr int PER = 16 / XW;  // input elements per 16-B load
#pragma unroll
          for (int u = 0; u < NV; ++u) unpack16<XT>(xr[u], f + u * PER);
          if constexpr (XT == EPB_FP8) {
            if (xsc != nullptr) {
#pragma unroll
              for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], xsc[((int64_t)c * EPC + i) >> 7]);
            }
          }
        }
      } else {
        load_input_chunk<XT, EPC>(xrow, xsc, (int64_t)c * EPC, f);
      }
      scale = 0.0f;
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
      v = pack16<WT>(f);
    };
    // chunk c to every destination slot and every own-expert output row
    auto emit = [&](int c, const int4& v, float scale, int nd) {
      for (int i = 0; i < nd; ++i) {
        uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (int64_t)s_j[i] * g.slot_stride;
        st_na_v4(slot + (int64_t)c * 16, v);
        if constexpr (SC) {
          if ((c & 7) == 0) reinterpret_cast<float*>(slot + g.RBp)[c >> 3] = scale;
        }
      }
      for (int k = 0; k < K; ++k) {
        const int srow = s_self[k];
        if (srow < 0) continue;
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)srow * H * OB;
        if constexpr (OT == WT) {
          st_v4(orow + (int64_t)c * 16, v);
          if constexpr (SC) {
            if ((c & 7) == 0) p.out_scales[(int64_t)srow * (H / 128) + (c >> 3)] = scale;
          }
        } else {
          float fw[EPC];  // the f32 image of what a slot would carry
          unpack16<WT>(v, fw);
          if constexpr (SC) {
#pragma unroll
            for (int i = 0; i < EPC; ++i) fw[i] = __fmul_rn(fw[i], scale);
          }
          store_f32_chunk<EPB_F32, EPC>(orow, (int64_t)c * EPC, fw);
        }
      }
    };
    for (int t = blockIdx.x; t < b; t += G) {
      const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * XW;
      const float* xsc = p.x_scales ? p.x_scales + (int64_t)t * (H / 128) : nullptr;
      int4 qv[2];
      float qs[2] = {0.0f, 0.0f};
      if (split && warp > 0) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int c = c_first + r * nq;
          if (c < nch) quantize(t, c, xrow, xsc, qv[r], qs[r]);
        }
      }
      if (warp == 0) {
        // lane k: i = #{t' < t routed to e_tk} (popc of e's bitmap below t)
        // and, for its owner d_k, j = #{t' < t touching d_k}; lanes keep the
        // first occurrence of each destination
        const uint32_t below = (1u << (t & 31)) - 1u;
        const int wt = t >> 5;
        int e = -1, d = -1, ci = 0, cj = 0;
        if (lane < K) {
          e = s_topk[t * K + lane];
          d = (int)(((uint64_t)e * g.Lmagic) >> 32);
          if (W <= 16) {
#pragma unroll
            for (int w = 0; w < 16; ++w) {
              const int wc = min(w, W - 1);
              const uint32_t mk = w < wt ? 0xFFFFFFFFu : (w == wt ? below : 0u);
              ci += __popc(s_ebits[e * W + wc] & mk);
              cj += __popc(s_dbits[d * W + wc] & mk);
            }
          } else {
            for (int w = 0; w < wt; ++w) {
              ci += __popc(s_ebits[e * W + w]);
              cj += __popc(s_dbits[d * W + w]);
            }
            ci += __popc(s_ebits[e * W + wt] & below);
            cj += __popc(s_dbits[d * W + wt] & below);
          }
        }
        // rows for this rank's own experts skip the window: they go straight
        // to the expert-major output (and the combine reads them in place)
        const bool mine = lane < K && d == p.rank;
        bool first = lane < K && !mine;
        if (!legacy) {  // optimized: one slot per destination (dedup)
          for (int j = 0; j < K; ++j) {
            const int dj = __shfl_sync(0xffffffffu, d, j);
            first &= !(j < lane && dj == d);
          }
        }
        const unsigned fm = __ballot_sync(0xffffffffu, first);
        if (lane < K) {
          s_hdr[2 + lane] = (uint32_t)e;
          s_hdr[2 + K + lane] = (uint32_t)ci;
          const int srow = mine ? (e - p.rank * L) * N * B + p.rank * B + ci : -1;
          s_self[lane] = srow;
          if (p.self_row) p.self_row[(int64_t)t * K + lane] = srow;
          if (p.owner_row) p.owner_row[(int64_t)t * K + lane] = (e - d * L) * N * B + p.rank * B + ci;
          if (mine) p.src_info[srow] = t * K + lane;
          if (first) {
            const int pos = __popc(fm & ((1u << lane) - 1u));
            s_dst[pos] = d;
            s_j[pos] = legacy ? ((e - d * L) * N + p.rank) * B + ci : p.rank * B + cj;
          }
        }
        if (lane == 0) {
          s_nd = __popc(fm);
          s_hdr[0] = (uint32_t)t;
          s_hdr[1] = (uint32_t)K;
        }
      }
      __syncthreads();
      LL_STAMP(p, 9);
      const int nd = s_nd;
      for (int w = threadIdx.x; w < 2 + 2 * K; w += blockDim.x)
        for (int i = 0; i < nd; ++i) {
          uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (int64_t)s_j[i] * g.slot_stride;
          reinterpret_cast<uint32_t*>(slot + g.RBp + g.SBp)[w] = s_hdr[w];
        }
      if (split) {
        if (warp > 0) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int c = c_first + r * nq;
            if (c < nch) emit(c, qv[r], qs[r], nd);
          }
        }
      } else if (vec) {
        for (int c = threadIdx.x; c < nch; c += blockDim.x) {
          int4 v;
          float scale;
          quantize(t, c, xrow, xsc, v, scale);
          emit(c, v, scale, nd);
        }
      } else {
        // hidden not a multiple of 16: element path (scales need H % 128 == 0)
        for (int el = threadIdx.x; el < H; el += blockDim.x) {
          float f = load_elem(xrow, XT, el);
          if constexpr (XT == EPB_FP8) {
            if (xsc != nullptr) f = __fmul_rn(f, xsc[el >> 7]);
          }
          for (int i = 0; i < nd; ++i) {
            uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (int64_t)s_j[i] * g.slot_stride;
            store_elem(slot, WT, el, f);
          }
          for (int k = 0; k < K; ++k) {
            const int srow = s_self[k];
            if (srow < 0) continue;
            uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)srow * H * OB;
            uint32_t wire = 0;
            store_elem(&wire, WT, 0, f);
            if constexpr (OT == WT) store_elem(orow, WT, el, load_elem(&wire, WT, 0));
            else reinterpret_cast<float*>(orow)[el] = load_elem(&wire, WT, 0);
          }
        }
      }
      __syncthreads();
    }
    LL_STAMP(p, 3);
    commit_round();
    __syncthreads();  // s_q
    // publish: CTA 0 writes the count words of every (local expert, src)
    // pair at every destination; then every CTA fences and flags each
    // destination (a receiver waits for all grid CTAs of all sources)
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < N * L; i += blockDim.x) {
        const int d = i / L, l = i - d * L, e = d * L + l;
        uint64_t* ctr = reinterpret_cast<uint64_t*>(peer_base(p.peers, d) + parity_off + g.disp_ctr);
        const uint64_t m = e < E ? (uint64_t)s_m[e] : 0ull;
        ctr[l * N + p.rank] = ((uint64_t)tag << 40) | ((uint64_t)s_q[d] << 20) | m;
      }
    }
    __syncthreads();
    // (no flags to self: own rows went straight to the output and the fused
    // receive reads its own counts from shared memory)
    if ((int)threadIdx.x < N && (int)threadIdx.x != p.rank) {
      fence_release(g.sys_fence);
      uint64_t* flag = reinterpret_cast<uint64_t*>(peer_base(p.peers, threadIdx.x) + parity_off + g.disp_flag) +
                       (int64_t)p.rank * G + blockIdx.x;
      st_flag(flag, (uint64_t)tag, sys);
    }
    LL_STAMP(p, 4);
  }

  if (p.phases & kPhaseRecv) {
    __shared__ int s_rq[kMaxRanks], s_pre[kMaxRanks + 1];
    __shared__ int s_fail;
    LL_STAMP(p, 5);
    const int lo = p.rank * L;
    const int nloc = max(0, min(L, E - lo));
    if (threadIdx.x == 0) {
      s_fail = 0;
      if (!(p.phases & kPhaseSend)) s_seq = seq_ld;
    }
    __syncthreads();
    if (!(p.phases & kPhaseSend)) {
      seq = s_seq;
      tag = ll_tag_of(seq);
      parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
    }
    // every CTA of every peer source (no flags from self)
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.disp_flag);
    for (int i = threadIdx.x; i < N * G; i += blockDim.x)
      if (i / G != p.rank && !wait_flag(&flags[i], tag, sys, p.timeout_ns, p.err)) s_fail = 1;
    __syncthreads();
    if (s_fail) return;
    LL_STAMP(p, 6);
    const volatile uint64_t* ctr = reinterpret_cast<const volatile uint64_t*>(p.win + parity_off + g.disp_ctr);
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < L * N; i += blockDim.x) {
        const int l = i / N, s = i - l * N;
        int m = 0;
        if (i < nloc * N) {
          // own counts: this launch's routing pass (fused) or the earlier
          // send launch's count word (split phases, stream-ordered)
          m = (s == p.rank && s_m != nullptr) ? s_m[lo + l] : (int)(ctr[i] & 0xFFFFF);
        }
        p.counts_i32[i] = m;
        p.counts_f32[i] = (float)m;
      }
    }
    if (nloc == 0) return;
    const int ob = (OT == EPB_F32 ? 4 : dtype_width(OT));
    const int64_t orow_bytes = (int64_t)H * ob;
    const int nw = blockDim.x >> 5;
    if (g.layout == EPB_LAYOUT_LEGACY) {
      // legacy (ll.py:362-376): slot (l*N + r)*B + i holds recv[l, r*B + i]
      // — the same linear index; rows of remote pairs, prefix over pairs
      __shared__ int s_wsum[kThreads / 32];
      int* s_pp = smem;  // [L*N + 1] (the send phase is done with it)
      __syncthreads();
      block_exclusive_scan(nloc * N, [&](int i) { return i % N == p.rank ? 0 : (int)(ctr[i] & 0xFFFFF); }, s_pp,
                           s_wsum);
      const int rows = s_pp[nloc * N];
      for (int f2 = warp * gridDim.x + blockIdx.x; f2 < 2 * rows; f2 += gridDim.x * nw) {
        const int r = f2 >> 1, half = f2 & 1;
        int lo_i = 0, hi_i = nloc * N;  // largest pair with s_pp[pair] <= r
        while (hi_i - lo_i > 1) {
          const int mid = (lo_i + hi_i) >> 1;
          if (s_pp[mid] <= r) lo_i = mid; else hi_i = mid;
        }
        const int64_t lin = (int64_t)lo_i * B + (r - s_pp[lo_i]);
        const uint8_t* slot = p.win + parity_off + g.disp_slot + lin * g.slot_stride;
        if (lane == 0 && half == 0) {
          const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
          const int e = lo + lo_i / N;
          int k = 0;
          while (k < K - 1 && (int)hdr[2 + k] != e) ++k;
          p.src_info[lin] = (int32_t)(hdr[0] * K + k);
        }
        ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + lin * orow_bytes,
                                SC ? p.out_scales + lin * (H / 128) : nullptr, lane, half, 2);
      }
      LL_STAMP(p, 7);
      return;
    }
    // own rows were placed by the send phase; only remote slots remain
    if ((int)threadIdx.x < N) s_rq[threadIdx.x] = (int)threadIdx.x == p.rank ? 0 : (int)((ctr[threadIdx.x] >> 20) & 0xFFFFF);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int s = 0; s < N; ++s) { s_pre[s] = run; run += s_rq[s]; }
      s_pre[N] = run;
    }
    __syncthreads();
    // warp tasks (slot, half row): the header is read once, the row loaded
    // once and stored to every local expert the slot names (the fan-out of
    // ll.py:378-400); CTA-major order spreads the tasks over every SM
    const int nslots = s_pre[N];
    const bool fan = (H & 15) == 0;
    constexpr int EPC = Elems<WT>::n;
    for (int f2 = warp * gridDim.x + blockIdx.x; f2 < 2 * nslots; f2 += gridDim.x * nw) {
      const int sl = f2 >> 1, half = f2 & 1;
      int s = 0;
      while (s_pre[s + 1] <= sl) ++s;
      const int j = sl - s_pre[s];
      const uint8_t* slot = p.win + parity_off + g.disp_slot + ((int64_t)s * B + j) * g.slot_stride;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
      int e = -1, ci = 0;
      if (lane < K) {
        e = (int)hdr[2 + lane];
        ci = (int)hdr[2 + K + lane];
      }
      const bool loc = lane < K && e >= lo && e < lo + nloc;
      const int my_orow = (e - lo) * N * B + s * B + ci;
      const unsigned lm = __ballot_sync(0xffffffffu, loc);
      if (half == 0 && loc) p.src_info[my_orow] = (int32_t)(hdr[0] * K + lane);
      if (!fan) {
        for (unsigned mm = lm; mm; mm &= mm - 1) {
          const int64_t row = __shfl_sync(0xffffffffu, my_orow, __ffs(mm) - 1);
          ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + row * orow_bytes,
                                  SC ? p.out_scales + row * (H / 128) : nullptr, lane, half, 2);
        }
        continue;
      }
      const int nch = H / EPC;
      const int per = (nch + 1) / 2;
      const int c0 = half * per, c1 = min(nch, c0 + per);
      for (int base = c0; base < c1; base += 32 * kUnroll) {
        int4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int c = base + u * 32 + lane;
          if (c < c1) v[u] = ld_weak_v4(slot + (int64_t)c * 16);
        }
        float sc_c[kUnroll];
        if constexpr (SC && OT != WT) {
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int c = base + u * 32 + lane;
            sc_c[u] = c < c1 ? reinterpret_cast<const float*>(slot + g.RBp)[(c * EPC) >> 7] : 0.0f;
          }
        }
        for (unsigned mm = lm; mm; mm &= mm - 1) {
          const int64_t row = __shfl_sync(0xffffffffu, my_orow, __ffs(mm) - 1);
          uint8_t* o = reinterpret_cast<uint8_t*>(p.out) + row * orow_bytes;
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int c = base + u * 32 + lane;
            if (c < c1) {
              if constexpr (OT == WT) {
                st_weak_v4(o + (int64_t)c * 16, v[u]);
              } else {
                float f[EPC];
                unpack16<WT>(v[u], f);
                if constexpr (SC) {
#pragma unroll
                  for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], sc_c[u]);
                }
                store_f32_chunk<EPB_F32, EPC>(o, (int64_t)c * EPC, f);
              }
            }
          }
        }
      }
      if constexpr (SC && OT == WT) {
        if (half == 0) {
          for (unsigned mm = lm; mm; mm &= mm - 1) {
            const int64_t row = __shfl_sync(0xffffffffu, my_orow, __ffs(mm) - 1);
            for (int i = lane; i < H / 128; i += 32)
              p.out_scales[row * (H / 128) + i] = reinterpret_cast<const float*>(slot + g.RBp)[i];
          }
        }
      }
    }
    LL_STAMP(p, 7);
  }
}

// ===========================================================================
// combine
// ===========================================================================
struct LLComb {
  const void* y;
  const int32_t* counts;
  const int32_t* src_info;
  const int32_t* self_row;  // [b*K] from the dispatch: rows of own experts are read in place
  const int64_t* topk;      // [b*K] routing (legacy layout: slot e*B + t)
  const int32_t* owner_row; // [b*K] from the dispatch: row of (t, k) on e_tk's owner
  int pull;                 // expert outputs live in every rank's window: homes pull them
  const float* w;
  void* out;
  const uint32_t* hseq;
  const uint64_t* peers;
  const uint8_t* win;
  int* err;
  uint64_t* trace;
  LLGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
  bool sys;
};

template <int IT, int WT, int OT>
__global__ void __launch_bounds__(kThreads) ll_combine_kernel(LLComb p) {
  extern __shared__ int s_pre[];  // [L*N + 1]
  const LLGeom& g = p.g;
  const int N = g.N, L = g.L, B = g.B, H = g.H, K = g.K, G = g.grid;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool sys = p.sys;
  LL_STAMP(p, 0);
  __shared__ uint32_t s_seq;
  __shared__ int s_wsum[kThreads / 32];
  // the round load is in flight while the send phase loads its counts
  uint32_t seq_ld = 0;
  if (threadIdx.x == 0) seq_ld = ld_round_u32(p.hseq);
  constexpr int EPC = Elems<WT>::n;
  const bool vec = (H & 15) == 0;
  const int nch = vec ? H / EPC : 0;
  // rows of this rank's own source tokens never travel: only N > 1 sends
  const bool send = (p.phases & kPhaseSend) && N > 1 && !p.pull;
  const int P = L * N;
  const int per = (P + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per;
  int local = 0;
  if (send) {
    // counts of the (l, src) pairs, own-source pairs excluded
    for (int i = i0; i < min(P, i0 + per); ++i) local += (i % N == p.rank) ? 0 : p.counts[i];
  }
  if (threadIdx.x == 0) s_seq = seq_ld;
  __syncthreads();
  const uint32_t seq = s_seq;
  const uint32_t tag = ll_tag_of(seq);
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;

  if (send) {
    // block-wide exclusive scan of the remote (l, src) counts
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
      run += (i % N == p.rank) ? 0 : p.counts[i];
    }
    if (threadIdx.x == blockDim.x - 1) s_pre[P] = run;
    __syncthreads();
    LL_STAMP(p, 1);
    const int total = s_pre[P];
    const int part = (nch + kParts - 1) / kParts;
    const int tasks = vec ? total * kParts : total;
    for (int task = blockIdx.x * nw + warp; task < tasks; task += gridDim.x * nw) {
      const int r = vec ? task / kParts : task;
      const int q = vec ? task - r * kParts : 0;
      int lo_i = 0, hi_i = P;  // largest pair with s_pre[pair] <= r
      while (hi_i - lo_i > 1) {
        const int mid = (lo_i + hi_i) >> 1;
        if (s_pre[mid] <= r) lo_i = mid; else hi_i = mid;
      }
      const int pair = lo_i;
      const int l = pair / N, s = pair - l * N, i = r - s_pre[pair];
      if (s == p.rank) continue;  // own tokens: the home reads these rows in place
      const int64_t row = (int64_t)l * N * B + (int64_t)s * B + i;
      const int info = p.src_info[row];
      // optimized slot t*K + k (layout.py:108-110); legacy e*B + t (ll.py:433-436)
      const int64_t cs = g.layout == EPB_LAYOUT_LEGACY
                             ? (int64_t)(p.rank * L + l) * B + (int64_t)(((uint64_t)info * g.Kmagic) >> 32)
                             : (int64_t)info;
      uint8_t* dst = peer_base(p.peers, s) + parity_off + g.comb_slot + cs * g.comb_stride;
      const uint8_t* yrow = reinterpret_cast<const uint8_t*>(p.y) + row * H * dtype_width(IT);
      if (vec) {
        const int c0 = q * part, c1 = min(nch, c0 + part);
        if constexpr (IT == WT) {
          for (int base = c0; base < c1; base += 32 * kUnroll) {
            int4 v[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int c = base + u * 32 + lane;
              if (c < c1) v[u] = ld_nc_v4(yrow + (int64_t)c * 16);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int c = base + u * 32 + lane;
              if (c < c1) st_na_v4(dst + (int64_t)c * 16, v[u]);
            }
          }
        } else {
          for (int c = c0 + lane; c < c1; c += 32) {
            float f[EPC];
            load_elems_vec<IT, EPC>(yrow, (int64_t)c * EPC, f);
            st_na_v4(dst + (int64_t)c * 16, pack16<WT>(f));
          }
        }
      } else {
        for (int el = lane; el < H; el += 32) store_elem(dst, WT, el, load_elem(yrow, IT, el));
      }
    }
    __syncthreads();
    LL_STAMP(p, 2);
    if ((int)threadIdx.x < N && (int)threadIdx.x != p.rank) {
      fence_release(g.sys_fence);
      uint64_t* flag = reinterpret_cast<uint64_t*>(peer_base(p.peers, threadIdx.x) + parity_off + g.comb_flag) +
                       (int64_t)p.rank * G + blockIdx.x;
      st_flag(flag, (uint64_t)tag, sys);
    }
    LL_STAMP(p, 3);
  } else if ((p.phases & kPhaseSend) && N > 1 && p.pull) {
    // pulled combine: nothing moves; announce that this rank's expert
    // outputs (written by earlier kernels on this stream) are complete
    if ((int)threadIdx.x < N && (int)threadIdx.x != p.rank) {
      fence_release(g.sys_fence);
      uint64_t* flag = reinterpret_cast<uint64_t*>(peer_base(p.peers, threadIdx.x) + parity_off + g.comb_flag) +
                       (int64_t)p.rank * G + blockIdx.x;
      st_flag(flag, (uint64_t)tag, sys);
    }
  }

  if (p.phases & kPhaseRecv) {
    __shared__ float s_w[kMaxTopK];
    __shared__ int s_fail;
    LL_STAMP(p, 4);
    const uint8_t* slots = p.win + parity_off + g.comb_slot;
    constexpr int kSeg = 64;  // 16-B chunks per warp task (2 per lane)
    const int segs = vec ? (nch + kSeg - 1) / kSeg : 0;
    const int tasks = p.b * segs;
    const int tstride = gridDim.x * nw;
    int task = warp * gridDim.x + blockIdx.x;
    // lane k of a warp task: row k of the token — this rank's own expert row
    // (read in place from the expert output) or its combine slot — and w_k;
    // the first task's rows are resolved before the flag wait
    const bool legacy = g.layout == EPB_LAYOUT_LEGACY;
    int my_self = -1, my_slot = 0;
    uint64_t my_pull = 0;  // pulled combine: the row in its owner's window
    float my_w = 0.0f;
    auto fetch = [&](int tk) {  // lane k's row of token tk
      if (lane < K) {
        const int64_t i = (int64_t)tk * K + lane;
        my_w = p.w[i];
        if (p.pull) {
          const int e = (int)p.topk[i];
          const int owner = (int)(((uint64_t)e * g.Lmagic) >> 32);
          my_pull = reinterpret_cast<uint64_t>(peer_base(p.peers, owner) + g.yout) + (uint64_t)p.owner_row[i] * g.yrow;
        } else {
          my_self = p.self_row ? p.self_row[i] : -1;
          my_slot = legacy ? (int)p.topk[i] * B + tk : tk * K + lane;
        }
      }
    };
    if (vec && task < tasks) fetch(task / segs);
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.comb_flag);
    for (int i = threadIdx.x; i < N * G; i += blockDim.x)
      if (i / G != p.rank && !wait_flag(&flags[i], tag, sys, p.timeout_ns, p.err)) s_fail = 1;
    __syncthreads();
    if (s_fail) return;
    LL_STAMP(p, 5);
    if (vec) {
      for (; task < tasks; task += tstride) {
        const int t = task / segs, sg = task - t * segs;
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * dtype_width(OT);
        const int cbase = sg * kSeg + lane;
        const bool ok0 = cbase < nch, ok1 = cbase + 32 < nch;
        const uint8_t* my_row =
            p.pull ? reinterpret_cast<const uint8_t*>(my_pull)
                   : (my_self >= 0 ? reinterpret_cast<const uint8_t*>(p.y) + (int64_t)my_self * H * dtype_width(IT)
                                   : slots + (int64_t)my_slot * g.comb_stride);
        const bool my_in_y = !p.pull && my_self >= 0;
        float acc0[EPC], acc1[EPC];
#pragma unroll
        for (int i = 0; i < EPC; ++i) acc0[i] = acc1[i] = 0.0f;
        for (int k0 = 0; k0 < K; k0 += 8) {
          // all row pointers first, then 16 loads in flight per lane
          const uint8_t* rp[8];
          bool iny[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            rp[u] = reinterpret_cast<const uint8_t*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_row), (k0 + u) & 31));
            iny[u] = __shfl_sync(0xffffffffu, my_in_y, (k0 + u) & 31);
          }
          int4 v0[8], v1[8];
          if constexpr (IT == WT) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (k0 + u < K) {
                if (ok0) v0[u] = ld_weak_v4(rp[u] + (int64_t)cbase * 16);
                if (ok1) v1[u] = ld_weak_v4(rp[u] + (int64_t)(cbase + 32) * 16);
              }
            }
          } else {
            // own rows hold the input dtype: rounded through the wire dtype
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (k0 + u < K) {
                if (iny[u]) {
                  float f[EPC];
                  if (ok0) { load_elems_vec<IT, EPC>(rp[u], (int64_t)cbase * EPC, f); v0[u] = pack16<WT>(f); }
                  if (ok1) { load_elems_vec<IT, EPC>(rp[u], (int64_t)(cbase + 32) * EPC, f); v1[u] = pack16<WT>(f); }
                } else {
                  if (ok0) v0[u] = ld_weak_v4(rp[u] + (int64_t)cbase * 16);
                  if (ok1) v1[u] = ld_weak_v4(rp[u] + (int64_t)(cbase + 32) * 16);
                }
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (k0 + u < K) {
              const float wk = __shfl_sync(0xffffffffu, my_w, (k0 + u) & 31);
              float y[EPC];
              unpack16<WT>(v0[u], y);
#pragma unroll
              for (int i = 0; i < EPC; ++i) acc0[i] = __fadd_rn(acc0[i], __fmul_rn(wk, y[i]));
              unpack16<WT>(v1[u], y);
#pragma unroll
              for (int i = 0; i < EPC; ++i) acc1[i] = __fadd_rn(acc1[i], __fmul_rn(wk, y[i]));
            }
          }
        }
        // the next task's rows (their loads overlap these stores)
        const int nt = task + tstride;
        if (nt < tasks) fetch(nt / segs);
        if (ok0) store_f32_chunk<OT, EPC>(orow, (int64_t)cbase * EPC, acc0);
        if (ok1) store_f32_chunk<OT, EPC>(orow, (int64_t)(cbase + 32) * EPC, acc1);
      }
    } else {
      for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
        __syncthreads();
        if ((int)threadIdx.x < K) s_w[threadIdx.x] = p.w[(int64_t)t * K + threadIdx.x];
        __syncthreads();
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * dtype_width(OT);
        for (int el = threadIdx.x; el < H; el += blockDim.x) {
          float acc = 0.0f;
          for (int k = 0; k < K; ++k) {
            const int sr = p.self_row && !p.pull ? p.self_row[(int64_t)t * K + k] : -1;
            float y;
            if (p.pull) {
              const int e = (int)p.topk[(int64_t)t * K + k];
              const uint8_t* row = peer_base(p.peers, (int)(((uint64_t)e * g.Lmagic) >> 32)) + g.yout +
                                   (uint64_t)p.owner_row[(int64_t)t * K + k] * g.yrow;
              y = load_elem(row, WT, el);
            } else if (sr >= 0) {
              uint32_t wire = 0;  // own expert row, rounded through the wire dtype
              store_elem(&wire, WT, 0,
                         load_elem(reinterpret_cast<const uint8_t*>(p.y) + (int64_t)sr * H * dtype_width(IT), IT, el));
              y = load_elem(&wire, WT, 0);
            } else {
              const int64_t cs = legacy ? p.topk[(int64_t)t * K + k] * B + t : (int64_t)t * K + k;
              y = load_elem(slots + cs * g.comb_stride, WT, el);
            }
            acc = __fadd_rn(acc, __fmul_rn(s_w[k], y));
          }
          store_elem(orow, OT, el, acc);
        }
      }
    }
    LL_STAMP(p, 6);
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

// EPB_COOP=0 launches the fused kernels without the cooperative attribute
// (co-residency then rests on grid <= SMs x occupancy, checked below)
bool coop_attr_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EPB_COOP");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename Params>
cudaError_t launch(void (*kern)(Params), int grid, size_t smem, bool coop, const Params& p, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024));
  if (e != cudaSuccess) return e;
  if (coop) {
    // both phases in one launch: CTAs in the receive phase wait on flags the
    // send phase of other CTAs writes, so all CTAs must be co-resident
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm * sm_count() < grid) return cudaErrorCooperativeLaunchTooLarge;
    if (!coop_attr_enabled()) {
      kern<<<grid, kThreads, smem, s>>>(p);
      return cudaGetLastError();
    }
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
cudaError_t run_disp(const LLDisp& p, size_t smem, cudaStream_t s) {
  return launch(ll_dispatch_kernel<XT, WT, SC, OT>, p.g.grid, smem, p.phases == 3, p, s);
}

template <int XT, int WT, bool SC>
cudaError_t run_disp_o(const LLDisp& p, int out_dtype, size_t smem, cudaStream_t s) {
  if (out_dtype == EPB_F32 || WT == EPB_F32) return run_disp<XT, WT, SC, EPB_F32>(p, smem, s);
  return run_disp<XT, WT, SC, WT>(p, smem, s);
}

template <int XT>
cudaError_t run_disp_x(const LLDisp& p, int out_dtype, size_t smem, cudaStream_t s) {
  switch (p.g.wire) {
    case EPB_F32: return run_disp_o<XT, EPB_F32, false>(p, out_dtype, smem, s);
    case EPB_BF16: return run_disp_o<XT, EPB_BF16, false>(p, out_dtype, smem, s);
    case EPB_F16: return run_disp_o<XT, EPB_F16, false>(p, out_dtype, smem, s);
    default:
      return p.g.scales ? run_disp_o<XT, EPB_FP8, true>(p, out_dtype, smem, s)
                        : run_disp_o<XT, EPB_FP8, false>(p, out_dtype, smem, s);
  }
}

template <int IT, int WT, int OT>
cudaError_t run_comb(const LLComb& p, size_t smem, cudaStream_t s) {
  return launch(ll_combine_kernel<IT, WT, OT>, p.g.grid, smem, p.phases == 3, p, s);
}

template <int IT, int WT>
cudaError_t run_comb_o(const LLComb& p, int out_dtype, size_t smem, cudaStream_t s) {
  return out_dtype == EPB_F32 ? run_comb<IT, WT, EPB_F32>(p, smem, s) : run_comb<IT, WT, EPB_BF16>(p, smem, s);
}

template <int IT>
cudaError_t run_comb_w(const LLComb& p, int out_dtype, size_t smem, cudaStream_t s) {
  switch (p.g.cwire) {
    case EPB_F32: return run_comb_o<IT, EPB_F32>(p, out_dtype, smem, s);
    case EPB_BF16: return run_comb_o<IT, EPB_BF16>(p, out_dtype, smem, s);
    case EPB_F16: return run_comb_o<IT, EPB_F16>(p, out_dtype, smem, s);
    default: return run_comb_o<IT, EPB_FP8>(p, out_dtype, smem, s);
  }
}

int check_ll(epb_group* g, int phases) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (g->cfg.algorithm != EPB_LL) return fail(EPB_HANDLE_STATE_ERROR, "group is not LL");
  if (!g->peers_ready) return fail(EPB_HANDLE_STATE_ERROR, "peer windows not mapped");
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
  p.src_info = a->src_info; p.self_row = a->self_row; p.owner_row = a->owner_row;
  p.peers = g->d_peers; p.win = g->window; p.err = g->d_err;
  p.dseq = reinterpret_cast<uint32_t*>(g->d_scratch); p.drd = g->d_scratch + 1; p.trace = g->trace;
  p.g = g->ll; p.timeout_ns = g->timeout_ns; p.b = b; p.rank = g->rank; p.phases = phases;
  p.sys = g->sys_scope;
  const int E = g->ll.E, N = g->ll.N, K = g->ll.K;
  const size_t W = (size_t)(b + 31) / 32;
  size_t smem = (phases & kPhaseSend) ? sizeof(int) * ((size_t)b * K + (E + N) * W + E + N) : 0;
  if ((phases & kPhaseRecv) && g->cfg.layout == EPB_LAYOUT_LEGACY)  // receive: pair prefix [L*N + 1]
    smem = std::max(smem, sizeof(int) * ((size_t)g->ll.L * N + 1));
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "LL batch too large for the fused dispatch kernel");
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  const int od = a->out_dtype;
  switch ((phases & kPhaseSend) ? a->x_dtype : wire) {
    case EPB_F32: e = run_disp_x<EPB_F32>(p, od, smem, s); break;
    case EPB_BF16: e = run_disp_x<EPB_BF16>(p, od, smem, s); break;
    case EPB_F16: e = run_disp_x<EPB_F16>(p, od, smem, s); break;
    case EPB_FP8: e = run_disp_x<EPB_FP8>(p, od, smem, s); break;
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
  if ((phases & kPhaseRecv) && g->cfg.layout == EPB_LAYOUT_LEGACY && b > 0 && !a->topk)
    return fail(EPB_INVALID_ARGUMENT, "legacy layout combine needs the routing (topk)");
  p.y = a->expert_out; p.counts = a->counts_i32; p.src_info = a->src_info; p.self_row = a->self_row;
  p.topk = a->topk; p.w = a->weights; p.out = a->out;
  p.owner_row = a->owner_row; p.pull = a->expert_out_in_window;
  if (p.pull && (a->in_dtype != EPB_BF16 || g->ll.cwire != EPB_BF16 || !a->topk || !a->owner_row ||
                 g->ll.yout_rows == 0 || a->expert_out != g->window + g->ll.yout))
    return fail(EPB_INVALID_ARGUMENT, "pulled combine needs bf16 rows in the window's expert-output region");
  p.hseq = hseq; p.peers = g->d_peers; p.win = g->window; p.err = g->d_err; p.trace = g->trace;
  p.g = g->ll; p.timeout_ns = g->timeout_ns; p.b = b; p.rank = g->rank; p.phases = phases;
  p.sys = g->sys_scope;
  const size_t smem = sizeof(int) * ((size_t)g->ll.L * g->ll.N + 1);
  if (smem > 200 * 1024) return fail(EPB_CAPACITY_EXCEEDED, "too many (expert, rank) pairs for combine");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = a->in_dtype == EPB_F32 ? run_comb_w<EPB_F32>(p, a->out_dtype, smem, s)
                                         : run_comb_w<EPB_BF16>(p, a->out_dtype, smem, s);
  if (e != cudaSuccess) return cuda_check(e, "ll_combine");
  return EPB_OK;
}

}  // extern "C"
