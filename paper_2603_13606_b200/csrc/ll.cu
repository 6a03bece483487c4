// Low-Latency dispatch / combine: two kernels per round (K2+K3 fused, K4a+K4b
// fused), each runnable as send-only, recv-only or both (one cooperative
// launch when peers are other GPUs).  Every LL launch of a group uses the same
// grid on every rank: a receiver expects one arrival per source CTA.
//
// Reference semantics (epsim ll.py):
//  * dispatch send (ll.py:255-308): per destination rank d, the tokens that
//    touch d go, ascending t, into d's slots [src*B + j]; the receiver learns
//    m(e, src) per (local expert, src) pair (the reference's counter value
//    m + 1).  Here one CTA of the source writes a count row (m of each of d's
//    experts, then q = slots) into d's window, and once every source CTA has
//    stored, the source adds one arrival to d's counter for it after a
//    system-scope release.  Arrivals are cumulative per parity, so round seq
//    is complete at (seq>>1)+1: the counter never needs the reference's
//    reset (ll.py:351-353).
//  * dispatch recv (ll.py:310-400): every slot row goes to recv[l, src*B + i]
//    for each local expert; i (the filled[l] order) and j (the slot) are
//    prefix counts the SENDER computes over its earlier tokens, i travels in
//    the slot header after the reference header fields (layout.py:282-295).
//    Each receiving warp waits only for the source of its own task, so slots
//    of early sources are placed while later sources are still sending.
//  * combine send (ll.py:404-462): each valid expert row (l, src, i) goes,
//    in the combine wire dtype, to src's slot t*K + k.
//  * combine recv (ll.py:464-507): out[t] = sum_k w[t,k] * y_k in f32,
//    ascending k from acc = 0, explicit __fmul_rn/__fadd_rn (no FMA); a warp
//    waits only for the owners of its token's experts.
//
// Latency design (B200): the token row is prefetched into registers at
// kernel start; the routing snapshot is one coalesced load into shared
// memory; a CTA computes only its own tokens' positions (prefix counts over
// the earlier tokens, warp reductions) while its warps quantise; one release
// fence per rank (system scope when peers are other GPUs; the last CTA to finish), then one arrival per destination; receivers
// poll N counters, not per-CTA flags.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "internal.h"

namespace epb {

constexpr int kPhaseSend = 1, kPhaseRecv = 2;
constexpr int kThreads = 512;
constexpr int kUnroll = 8;
constexpr int kParts = 4;  // combine send: warps per row
constexpr uint32_t kPoison = 0xFFFFFFFFu;  // count row of a source whose routing was rejected

// diagnostics: thread 0 of each CTA stamps the global timer at checkpoints
#define LL_STAMP(P, I)                                                                    \
  do {                                                                                   \
    if ((P).trace && threadIdx.x == 0) (P).trace[blockIdx.x * 16 + (I)] = globaltimer(); \
  } while (0)

// round counters: written by an earlier kernel (visible at the kernel
// boundary) and not again until every CTA has read them — a relaxed GPU-scope
// load suffices (a volatile, i.e. system-scope, load measured ~2 us slower)
EPB_DEV uint32_t ld_round_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
EPB_DEV uint8_t* peer_base(const uint64_t* peers, int r) { return reinterpret_cast<uint8_t*>(peers[r]); }

// Programmatic dependent launch: the LL kernels are launched so that the
// next kernel's grid is scheduled while this one drains; each kernel first
// waits for its predecessors to complete (their writes visible), then lets
// its own dependents start launching.  Without the launch attribute both
// instructions are no-ops.
EPB_DEV void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

EPB_DEV uint64_t ld_acq(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// one arrival (the caller released first: fence_release, then these)
EPB_DEV void red_arrive(uint64_t* p, uint64_t v, bool sys) {
  if (sys) asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// spin until *c >= need (bounded; records TransportClosed).  Acquire: what
// the arriving CTAs stored before their release is visible afterwards.
EPB_DEV bool wait_arrivals(const uint64_t* c, uint64_t need, bool sys, uint64_t timeout_ns, int* err) {
  uint64_t start = 0;
  for (int spins = 0;; ++spins) {
    if (ld_acq(c, sys) >= need) return true;
    if ((spins & 31) != 31) continue;
    if (*(volatile int*)err != 0) return false;
    if (spins == 63) start = globaltimer();
    if (spins > 64 && (spins & 255) == 255 && globaltimer() - start > timeout_ns) {
      raise_err(err, EPB_TRANSPORT_CLOSED);
      return false;
    }
  }
}
// Publish this rank's part of a round: each round adds `grid` to every
// peer's arrival counter for this rank, after a system-scope release that
// covers every payload store of the round.  Two schemes, chosen per launch
// by the sender alone (the receiver only waits for grid*(rounds)):
//  * W <= direct_max storing CTAs (EPB_LL_DIRECT, default 0): each of CTAs
//    0..W-1 releases its own stores and adds 1; CTA grid-1 (which is not
//    one of them) releases and adds grid - W for itself and the idle CTAs
//    (W = 0, the pulled combine's announcement: CTA grid-1 alone);
//  * otherwise every CTA releases at GPU scope and counts in at a local
//    counter; the last one issues the rank's single system-scope release
//    (cumulative over all CTAs' stores: each CTA's GPU-scope release is
//    acquired by the last CTA's RMW on the counter) and adds grid.
// Concurrent system-scope fences from every SM measured several us; the
// per-CTA scheme measured no faster than the last-CTA chain even at 1-4
// tokens (N=2: 35.6 vs 32.8 us at 4 tokens), hence direct_max = 0.
// All threads call.  `done`: this kind's local counter (reset by the last).
EPB_DEV void ll_arrive(const uint64_t* peers, uint64_t off, int N, int me, bool fence_sys, bool sys,
                       unsigned* done, uint32_t chaos_ns, int W, const OpTrace& ops, uint32_t sig_base,
                       int direct_max) {
  __syncthreads();
  if (threadIdx.x != 0 || N == 1) return;
  const int G = gridDim.x, c = blockIdx.x;
  uint64_t add = 0;
  if (W <= direct_max && W < G) {
    add = c < W ? 1ull : (c == G - 1 ? (uint64_t)(G - W) : 0ull);
    if (add == 0) return;
    chaos_delay(chaos_ns, 0x53u);
    fence_release(fence_sys);
  } else {
    chaos_delay(chaos_ns, 0x51u);
    fence_release(false);
    if (atomicAdd(done, 1u) != (unsigned)G - 1) return;
    *done = 0u;  // next use is a later kernel (stream order)
    fence_release(fence_sys);
    add = (uint64_t)G;
  }
  for (int d = 0; d < N; ++d)
    if (d != me) {
      red_arrive(reinterpret_cast<uint64_t*>(peer_base(peers, d) + off) + me, add, sys);
      op_record(ops, EPB_OP_SIGNAL, me, d, off + 8ull * me, 8, sig_base + me, add);
    }
}

// warp: wait until every source in `need` (bit per rank) has arrived; bits
// already seen are cached in `seen`.  Lane 0 polls; __syncwarp orders the
// other lanes' later loads after its acquire.
EPB_DEV bool warp_wait_sources(uint64_t need, uint64_t& seen, const uint64_t* ctr, uint64_t target, bool sys,
                               uint64_t timeout_ns, int* err, int lane) {
  need &= ~seen;
  bool ok = true;
  while (need) {
    const int s = __ffsll((long long)need) - 1;
    if (lane == 0) ok = wait_arrivals(&ctr[s], target, sys, timeout_ns, err);
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) return false;
    seen |= 1ull << s;
    need &= need - 1;
  }
  __syncwarp();
  return true;
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
  uint32_t* dseq;  // [grid] round sequence: CTA c reads and advances its own copy
  unsigned* done;  // local CTA-completion counter of the send phase (ll_arrive)
  uint64_t* trace;
  OpTrace ops;
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

// the exact quotient for the rare near-midpoint elements: one out-of-line
// copy of the IEEE division sequence instead of one per unrolled element
__device__ __noinline__ float div_rn_call(float a, float b) { return __fdiv_rn(a, b); }

// f32 values of one 16-B wire chunk -> the wire image (block-128 FP8 scale
// over 8 aligned lanes; `scale` = the block's scale, 0 for non-FP8 wires)
template <int WT, bool SC>
EPB_DEV int4 wire_chunk(float* f, float& scale, int lane) {
  constexpr int EPC = Elems<WT>::n;
  scale = 0.0f;
  if constexpr (SC) {
    float amax = 0.0f;
#pragma unroll
    for (int i = 0; i < EPC; ++i) amax = fmaxf(amax, fabsf(f[i]));
    const unsigned gm = 0xFFu << (lane & 24);
    amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 2));
    amax = fmaxf(amax, __shfl_xor_sync(gm, amax, 4));
    scale = __fdiv_rn(amax, 448.0f);
    const float div = scale > 0.0f ? scale : 1.0f;
    // fl32(x / div) without 16 IEEE division sequences: q = x * rcp(div),
    // then one exact-residual correction (Markstein), correctly rounded for
    // |x|, div in [2^-100, 2^100] (checked against IEEE division on 10^9
    // random pairs, tools/div_check.c); the sign of a zero quotient follows
    // x.  Anything outside that range takes the out-of-line IEEE division.
    const float r = __frcp_rn(div);
    bool slow = div < 0x1p-100f || div > 0x1p100f;
#pragma unroll
    for (int i = 0; i < EPC; ++i) slow |= f[i] != 0.0f && fabsf(f[i]) < 0x1p-100f;
    if (!slow) {
#pragma unroll
      for (int i = 0; i < EPC; ++i) {
        const float q = __fmul_rn(f[i], r);
        const float res = __fmaf_rn(-q, div, f[i]);
        f[i] = copysignf(__fmaf_rn(res, r, q), f[i]);
      }
    } else {
      float tmp[EPC];
#pragma unroll
      for (int i = 0; i < EPC; ++i) tmp[i] = f[i];
#pragma unroll 1
      for (int i = 0; i < EPC; ++i) tmp[i] = div_rn_call(tmp[i], div);
#pragma unroll
      for (int i = 0; i < EPC; ++i) f[i] = tmp[i];
    }
  }
  return pack16<WT>(f);
}

// chunk c of an input row as f32 (from prefetched registers when given)
template <int XT, int EPC, int NV>
EPB_DEV void input_chunk(const int4* pre, const uint8_t* xrow, const float* xsc, int c, float* f) {
  if (pre != nullptr) {
    if constexpr (NV > 0) {
      constexpr int XW = XT == EPB_F32 ? 4 : (XT == EPB_FP8 ? 1 : 2);
      constexpr int PER = 16 / XW;
#pragma unroll
      for (int u = 0; u < NV; ++u) unpack16<XT>(pre[u], f + u * PER);
      if constexpr (XT == EPB_FP8) {
        if (xsc != nullptr) {
#pragma unroll
          for (int i = 0; i < EPC; ++i) f[i] = __fmul_rn(f[i], xsc[((int64_t)c * EPC + i) >> 7]);
        }
      }
      return;
    }
  }
  load_input_chunk<XT, EPC>(xrow, xsc, (int64_t)c * EPC, f);
}

EPB_DEV int sel8(const int* v, int i) {
  int r = v[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) r = i == k ? v[k] : r;
  return r;
}

// parts per token and work units (token, part) of the fast send path: a
// small batch spreads each token over up to 8 CTAs (chunk ranges are
// multiples of 8 chunks, the FP8 blocks)
EPB_DEV int fast_parts(int b, int G, int nch) {
  int P = b > 0 ? G / b : 1;
  return max(1, min(min(P, 8), max(1, nch / 8)));
}
EPB_DEV int fast_units(int b, int G, int nch) { return b * fast_parts(b, G, nch); }

// Send phase, fast path (top-k <= 8, batch <= block size, hidden % 16 == 0).
// Thread tau holds routing row tau in registers: validation, the earlier-
// token prefix counts of the CTA's token and the counting CTA's histograms
// need no shared-memory staging.  Work units are (token, part): a small
// batch spreads each token over up to 8 CTAs so few warps per SM quantise
// (latency, not throughput, bounds a decode step).  One barrier (which also
// reduces the validation verdict) separates the position pass from the
// stores; every warp derives the destination list itself.
// Returns the routing verdict (true = rejected, nothing was sent).
template <int XT, int WT, bool SC, int OT>
EPB_DEV bool ll_send_fast(const LLDisp& p, int* smem, uint32_t seq_ld, uint32_t& seq, uint64_t& parity_off) {
  const LLGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L, E = g.E, B = g.B, G = gridDim.x;
  const int b = p.b, me = p.rank, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5, BD = blockDim.x;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : (XT == EPB_FP8 ? 1 : 2);
  constexpr int NV = (EPC * XW) >= 16 ? (EPC * XW) / 16 : 0;
  constexpr int OB = OT == EPB_F32 ? 4 : (OT == EPB_FP8 ? 1 : 2);
  const int nch = H / EPC;
  const bool legacy = g.layout == EPB_LAYOUT_LEGACY;
  const int lo = me * L;
  const int nloc = max(0, min(L, E - lo));
  const int P = fast_parts(b, G, nch);
  const int per = ((nch + P - 1) / P + 7) & ~7;
  const int units = b * P;
  __shared__ int s_part[kThreads / 32][16];  // per-warp prefix partials (i of k, then j of k)
  __shared__ uint32_t s_seq2;
  const uint64_t L_magic = g.Lmagic;
  auto owner_of = [&](int e) { return (int)(((uint64_t)(uint32_t)e * L_magic) >> 32); };

  // chunks per thread held in registers (one 16-element FP8 chunk covers
  // H <= 8192 at 512 threads; 8-element wires take two); wider rows finish
  // in a loop that quantises as it stores
  constexpr int CPT = EPC >= 16 ? 1 : 2;
  // first unit's input chunks, prefetched (their DRAM latency overlaps the
  // routing loads and the position pass)
  int4 xr[CPT][NV > 0 ? NV : 1];
  bool xpre[CPT];
#pragma unroll
  for (int r = 0; r < CPT; ++r) xpre[r] = false;
  {
    const int u = blockIdx.x;
    if (NV > 0 && u < units) {
      const int t = u / P, c0 = (u - t * P) * per, c1 = min(nch, c0 + per);
#pragma unroll
      for (int r = 0; r < CPT; ++r) {
        const int c = c0 + tid + r * BD;
        if (c < c1) {
          const uint8_t* src = reinterpret_cast<const uint8_t*>(p.x) + ((int64_t)t * H + (int64_t)c * EPC) * XW;
#pragma unroll
          for (int v = 0; v < (NV > 0 ? NV : 1); ++v) xr[r][v] = ld_nc_v4(src + 16 * v);
          xpre[r] = true;
        }
      }
    }
  }
  // this thread's routing row (token tid): range, distinctness, owners
  int rw[8];
  bool row_ok = true;
  uint64_t own = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    rw[k] = -1 - k;
    if (tid < b && k < K) {
      const int64_t v = __ldg(p.topk + (int64_t)tid * K + k);
      const bool in = v >= 0 && v < E;
      row_ok &= in;
      rw[k] = in ? (int)v : -100;
    }
  }
#pragma unroll
  for (int k = 1; k < 8; ++k)
#pragma unroll
    for (int j = 0; j < k; ++j) row_ok &= rw[j] != rw[k];
  if (tid < b && row_ok) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < K) own |= 1ull << owner_of(rw[k]);
  }
  if (tid == 0) {
    // every CTA advances its own copy of the round sequence (the copies move
    // in lockstep, no cross-CTA atomics); CTA 0 records it in the handle
    s_seq2 = seq_ld;
    p.dseq[blockIdx.x] = seq_ld + 1;
    if (blockIdx.x == 0) *p.hseq = seq_ld;
  }
  LL_STAMP(p, 8);
  bool bad = false;
  for (int it = 0, u = blockIdx.x;; ++it, u += G) {
    const bool has = u < units;
    int t = 0, c0 = 0, c1 = 0;
    if (has) {
      t = u / P;
      c0 = (u - t * P) * per;
      c1 = min(nch, c0 + per);
    }
    int et[8];  // token t's experts (broadcast loads)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      et[k] = -2 - k;
      if (has && k < K) {
        const int64_t v = __ldg(p.topk + (int64_t)t * K + k);
        et[k] = (v >= 0 && v < E) ? (int)v : 0;
      }
    }
    const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * XW;
    const float* xsc = p.x_scales ? p.x_scales + (int64_t)t * (H / 128) : nullptr;
    int4 qv[CPT];
    float qs[CPT];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const int c = c0 + tid + r * BD;
      qs[r] = 0.0f;
      if (has && c < c1) {
        float f[EPC];
        input_chunk<XT, EPC, NV>(it == 0 && xpre[r] ? xr[r] : nullptr, xrow, xsc, c, f);
        qv[r] = wire_chunk<WT, SC>(f, qs[r], lane);
      }
    }
    LL_STAMP(p, 9);
    // prefix partials: i_k = #{t' < t routed to e_tk}, j_k = #{t' < t
    // touching owner(e_tk)} over this thread's token t' = tid
    uint32_t hit_i = 0, hit_j = 0;
    if (has && tid < t) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < K) {
          bool in = false;
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) in |= rw[k2] == et[k];
          hit_i |= (uint32_t)in << k;
          hit_j |= (uint32_t)((own >> owner_of(et[k])) & 1ull) << k;
        }
      }
    }
    int my_i = 0, my_j = 0;
    if (has && warp * 32 < t) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k < K) {
          const int ci = __reduce_add_sync(0xffffffffu, (hit_i >> k) & 1u);
          const int cj = __reduce_add_sync(0xffffffffu, (hit_j >> k) & 1u);
          if (lane == k) {
            my_i = ci;
            my_j = cj;
          }
        }
      }
    }
    if (lane < 8) {
      s_part[warp][lane] = my_i;
      s_part[warp][8 + lane] = my_j;
    }
    if (it == 0) {
      bad = __syncthreads_or(tid < b && !row_ok) != 0;
      seq = s_seq2;
      parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
    } else {
      __syncthreads();
    }
    if (!has || bad) break;
    chaos_delay(g.chaos_ns, 0x17u + it);
    LL_STAMP(p, 10);
    // destinations of token t (every warp derives them): lanes k < K
    int e = -1, d = -1, ci = 0, cj = 0;
    if (lane < K) {
      e = sel8(et, lane);
      d = owner_of(e);
      const int wl = (t + 31) >> 5;  // warps that held earlier tokens
      for (int w = 0; w < wl; ++w) {
        ci += s_part[w][lane];
        cj += s_part[w][8 + lane];
      }
    }
    const bool mine = lane < K && d == me;
    bool first = lane < K && !mine;
    if (!legacy) {  // optimized: one slot per destination rank (dedup)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int dj = __shfl_sync(0xffffffffu, d, j);
        first &= !(j < lane && dj == d);
      }
    }
    const unsigned fm = __ballot_sync(0xffffffffu, first);
    const unsigned mm = __ballot_sync(0xffffffffu, mine);
    const int jslot = legacy ? ((e - d * L) * N + me) * B + ci : me * B + cj;
    const int srow = mine ? (e - lo) * N * B + me * B + ci : -1;
    const uint64_t slot_off = parity_off + g.disp_slot;
    if (c0 == 0 && warp == 0) {
      // part 0: routing metadata and the slot headers (t, K, ids, ranks)
      if (lane < K) {
        if (p.self_row) p.self_row[(int64_t)t * K + lane] = srow;
        if (p.owner_row) p.owner_row[(int64_t)t * K + lane] = (e - d * L) * N * B + me * B + ci;
        if (mine) p.src_info[srow] = t * K + lane;
      }
      const int ve = __shfl_sync(0xffffffffu, e, max(0, min(31, lane - 2)));
      const int vc = __shfl_sync(0xffffffffu, ci, max(0, min(31, lane - 2 - K)));
      const uint32_t word = lane == 0 ? (uint32_t)t : lane == 1 ? (uint32_t)K : lane < 2 + K ? (uint32_t)ve : (uint32_t)vc;
      for (unsigned m = fm; m; m &= m - 1) {
        const int ln = __ffs(m) - 1;
        const int dd = __shfl_sync(0xffffffffu, d, ln), jj = __shfl_sync(0xffffffffu, jslot, ln);
        if (lane < 2 + 2 * K)
          reinterpret_cast<uint32_t*>(peer_base(p.peers, dd) + slot_off + (int64_t)jj * g.slot_stride + g.RBp +
                                      g.SBp)[lane] = word;
      }
    }
    // chunk c to every destination slot and every own-expert output row
    auto emit = [&](int c, bool ok, const int4& v, float scale) {
      for (unsigned m = fm; m; m &= m - 1) {
        const int ln = __ffs(m) - 1;
        const int dd = __shfl_sync(0xffffffffu, d, ln), jj = __shfl_sync(0xffffffffu, jslot, ln);
        if (ok) {
          uint8_t* slot = peer_base(p.peers, dd) + slot_off + (int64_t)jj * g.slot_stride;
          st_na_v4(slot + (int64_t)c * 16, v);
          if constexpr (SC) {
            if ((c & 7) == 0) reinterpret_cast<float*>(slot + g.RBp)[c >> 3] = scale;
          }
        }
      }
      for (unsigned m = mm; m; m &= m - 1) {
        const int sr = __shfl_sync(0xffffffffu, srow, __ffs(m) - 1);
        if (ok) {
          uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)sr * H * OB;
          if constexpr (OT == WT) {
            st_v4(orow + (int64_t)c * 16, v);
            if constexpr (SC) {
              if ((c & 7) == 0) p.out_scales[(int64_t)sr * (H / 128) + (c >> 3)] = scale;
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
      }
    };
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const int c = c0 + tid + r * BD;
      emit(c, c < c1, qv[r], qs[r]);
    }
    // chunks beyond CPT per thread (very wide rows): quantise as they go
    for (int cb = c0 + CPT * BD + warp * 32; cb < c1; cb += BD) {
      const int c = cb + lane;
      int4 v = make_int4(0, 0, 0, 0);
      float scale = 0.0f;
      float f[EPC];
      if (c < c1) input_chunk<XT, EPC, NV>(nullptr, xrow, xsc, c, f);
      else {
#pragma unroll
        for (int i = 0; i < EPC; ++i) f[i] = 0.0f;
      }
      v = wire_chunk<WT, SC>(f, scale, lane);
      emit(c, c < c1, v, scale);
    }
    LL_STAMP(p, 2);
    if (u + G >= units) break;
    __syncthreads();  // s_part reuse by the next unit
  }
  LL_STAMP(p, 3);
  if ((int)blockIdx.x == G - 1) {
    // the counting CTA: m(e) and q(d) over the batch (ll.py:255-259,
    // :292-296) -> a count row into every peer's window (m of the peer's
    // experts, then q), own counts straight to the counts output
    int* s_m = smem;    // [E]
    int* s_q = smem + E;  // [N]
#pragma unroll 1
    for (int e2 = tid; e2 < E; e2 += BD) s_m[e2] = 0;
    if (tid < N) s_q[tid] = 0;
    __syncthreads();
    if (!bad && tid < b) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < K) atomicAdd(&s_m[rw[k]], 1);
      for (uint64_t o = own; o; o &= o - 1) atomicAdd(&s_q[__ffsll((long long)o) - 1], 1);
    }
    __syncthreads();
    const int R = L + 1;
#pragma unroll 1
    for (int i = tid; i < N * R; i += BD) {
      const int d2 = i / R, l = i - d2 * R;
      if (d2 == me) continue;
      const uint32_t v = bad ? kPoison : (l < L ? (d2 * L + l < E ? (uint32_t)s_m[d2 * L + l] : 0u) : (uint32_t)s_q[d2]);
      reinterpret_cast<uint32_t*>(peer_base(p.peers, d2) + parity_off + g.cnt_row)[me * R + l] = v;
    }

#pragma unroll 1
    for (int l = tid; l < L; l += BD) {
      const int m = l < nloc && !bad ? s_m[lo + l] : 0;
      p.counts_i32[l * N + me] = m;
      p.counts_f32[l * N + me] = (float)m;
    }
    if (bad && tid == 0) raise_err(p.err, EPB_INVALID_ARGUMENT);
  }
  (void)nw;
  return bad;
}

// FAST: the decode hot path only (ll_send_fast + the optimized-layout vector
// receive) — a compact kernel keeps the instruction footprint small (cold
// i-cache after an L2 flush was the largest stall of the combined kernel);
// everything else (top-k > 8, batches above the block size, unaligned
// hidden, the legacy layout, op-traced launches) runs the general kernel.
template <int XT, int WT, bool SC, int OT, bool FAST>
__global__ void __launch_bounds__(kThreads) ll_dispatch_kernel(LLDisp p) {
  extern __shared__ int smem[];
  pdl_enter();
  const LLGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L, E = g.E, B = g.B, G = gridDim.x;
  const int b = p.b, me = p.rank;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool sys = p.sys;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : (XT == EPB_FP8 ? 1 : 2);
  constexpr int NV = (EPC * XW) >= 16 ? (EPC * XW) / 16 : 0;  // 16-B input loads per chunk
  const bool vec = (H & 15) == 0;
  const int nch = vec ? H / EPC : 0;
  constexpr int OB = OT == EPB_F32 ? 4 : (OT == EPB_FP8 ? 1 : 2);  // output element bytes
  const bool legacy = g.layout == EPB_LAYOUT_LEGACY;
  const int lo = me * L;
  const int nloc = max(0, min(L, E - lo));

  // split: warps 1.. quantise a token's chunks (<= 2 each, in registers)
  // while the position pass runs; else every thread loops
  const int nq = (int)blockDim.x - 32;
  const bool split = vec && nch <= 2 * nq;
  const int c_first = split ? (int)threadIdx.x - 32 : (int)threadIdx.x;  // first chunk of this thread
  // prefetch this CTA's first token chunk: its DRAM latency overlaps the
  // routing load and the position pass
  int4 xr[NV > 0 ? NV : 1];
  const bool pre = !FAST && (p.phases & kPhaseSend) && NV > 0 && vec && (int)blockIdx.x < b && c_first >= 0 &&
                   c_first < nch;
  if (pre) {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.x) +
                         ((int64_t)blockIdx.x * H + (int64_t)c_first * EPC) * XW;
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) xr[v] = ld_nc_v4(src + 16 * v);
  }
  LL_STAMP(p, 0);
  // round sequence: thread 0 issues the load now; it lands in shared memory
  // at the first block barrier
  __shared__ uint32_t s_seq;
  uint32_t seq_ld = 0;
  if (threadIdx.x == 0) seq_ld = ld_round_u32((p.phases & kPhaseSend) ? p.dseq + blockIdx.x : p.hseq);
  uint32_t seq = 0;
  uint64_t parity_off = 0;

  if constexpr (FAST) {
    if (p.phases & kPhaseSend) {
      const bool bad = ll_send_fast<XT, WT, SC, OT>(p, smem, seq_ld, seq, parity_off);
      // publish: one system-scope release per rank, one arrival per destination
      ll_arrive(p.peers, parity_off + g.d_arr, N, me, g.sys_fence, sys, p.done, g.chaos_ns,
                fast_units(p.b, gridDim.x, g.H / Elems<WT>::n), OpTrace{nullptr, 0u}, 0u, g.direct_max);
      LL_STAMP(p, 4);
      if (bad) return;
    }
  } else if (p.phases & kPhaseSend) {
    int* s_topk = smem;           // [b*K] routing snapshot (-1 = id out of range)
    int* s_m = s_topk + b * K;    // [E] per-expert token counts (counting CTA)
    int* s_q = s_m + E;           // [N] tokens per destination (counting CTA)
    __shared__ int s_nd;
    __shared__ int s_cnt[2 * kMaxTopK];  // this token's prefix counts: i per k, then j per k
    // per destination entry: rank and absolute slot index in its window
    // (optimized: one slot per (token, dst) at src*B + j; legacy: one slot
    // per (token, expert) at ((e - dL)*N + src)*B + i)
    __shared__ int s_dst[kMaxRanks], s_j[kMaxRanks];
    __shared__ int s_self[kMaxTopK];  // output row of (t, k) for this rank's own experts, else -1
    __shared__ uint32_t s_hdr[2 + 2 * kMaxTopK];
    const int items = b * K;
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
      const int64_t e = __ldg(p.topk + i);
      s_topk[i] = (e >= 0 && e < E) ? (int)e : -1;
    }
    if ((int)threadIdx.x < 2 * kMaxTopK) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LL_STAMP(p, 8);
    // routing validation (api.py:150-170): ids in range, distinct per row;
    // every CTA reaches the same verdict before any traffic
    bool row_bad = false;
    for (int t = threadIdx.x; t < b; t += blockDim.x) {
      bool ok = true;
      for (int k = 0; k < K; ++k) {
        const int e = s_topk[t * K + k];
        ok &= e >= 0;
        for (int j = 0; j < k; ++j) ok &= s_topk[t * K + j] != e;
      }
      row_bad |= !ok;
    }
    if (threadIdx.x == 0) {
      // the round: every CTA advances its own copy of the sequence (all
      // copies move in lockstep, no cross-CTA atomics); CTA 0 records it in
      // the handle word for the receive launch and the combine
      s_seq = seq_ld;
      p.dseq[blockIdx.x] = seq_ld + 1;
      if (blockIdx.x == 0) *p.hseq = seq_ld;
    }
    const bool bad = __syncthreads_or(row_bad) != 0;
    LL_STAMP(p, 1);
    seq = s_seq;
    parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
    const uint64_t slot_off = parity_off + g.disp_slot;

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
      v = wire_chunk<WT, SC>(f, scale, lane);
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
    for (int t = blockIdx.x; !bad && t < b; t += G) {
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
        if (p.trace && threadIdx.x == 32) p.trace[blockIdx.x * 16 + 9] = globaltimer();
      }
      // positions of token t: i_k = #{t' < t routed to e_tk} (ll.py:383-399)
      // and j_k = #{t' < t touching owner(e_tk)} (ll.py:292-296), one
      // earlier token per thread, warp reductions, shared atomics per warp
      for (int base = warp * 32; base < t; base += (int)blockDim.x) {
        const int tp = base + lane;
        uint32_t hit_i = 0, hit_j = 0;
        if (tp < t) {
          if (K <= 8) {  // both rows in registers
            int rw[8], et[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              rw[k] = k < K ? s_topk[tp * K + k] : -1;
              et[k] = k < K ? s_topk[t * K + k] : -2;
            }
            uint64_t own = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k < K) own |= 1ull << (int)(((uint64_t)rw[k] * g.Lmagic) >> 32);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              bool in = false;
#pragma unroll
              for (int k2 = 0; k2 < 8; ++k2) in |= rw[k2] == et[k];
              hit_i |= (uint32_t)in << k;
              if (k < K) hit_j |= (uint32_t)((own >> (int)(((uint64_t)et[k] * g.Lmagic) >> 32)) & 1ull) << k;
            }
          } else {
            uint64_t own = 0;
            for (int k2 = 0; k2 < K; ++k2) own |= 1ull << (int)(((uint64_t)s_topk[tp * K + k2] * g.Lmagic) >> 32);
            for (int k = 0; k < K; ++k) {
              const int e = s_topk[t * K + k];
              bool in = false;
              for (int k2 = 0; k2 < K; ++k2) in |= s_topk[tp * K + k2] == e;
              hit_i |= (uint32_t)in << k;
              hit_j |= (uint32_t)((own >> (int)(((uint64_t)e * g.Lmagic) >> 32)) & 1ull) << k;
            }
          }
        }
        int my_i = 0, my_j = 0;
        for (int k = 0; k < K; ++k) {
          const int ci = __reduce_add_sync(0xffffffffu, (hit_i >> k) & 1u);
          const int cj = __reduce_add_sync(0xffffffffu, (hit_j >> k) & 1u);
          if (lane == k) { my_i = ci; my_j = cj; }
        }
        if (lane < K) {
          atomicAdd(&s_cnt[lane], my_i);
          atomicAdd(&s_cnt[kMaxTopK + lane], my_j);
        }
      }
      if (warp == 0) LL_STAMP(p, 10);
      __syncthreads();
      if (warp == 0) {
        int e = -1, d = -1, ci = 0, cj = 0;
        if (lane < K) {
          e = s_topk[t * K + lane];
          d = (int)(((uint64_t)e * g.Lmagic) >> 32);
          ci = s_cnt[lane];
          cj = s_cnt[kMaxTopK + lane];
          s_cnt[lane] = 0;  // ready for the next token (read above by this lane only)
          s_cnt[kMaxTopK + lane] = 0;
        }
        // rows for this rank's own experts skip the window: they go straight
        // to the expert-major output (and the combine reads them in place)
        const bool mine = lane < K && d == me;
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
          const int srow = mine ? (e - lo) * N * B + me * B + ci : -1;
          s_self[lane] = srow;
          if (p.self_row) p.self_row[(int64_t)t * K + lane] = srow;
          if (p.owner_row) p.owner_row[(int64_t)t * K + lane] = (e - d * L) * N * B + me * B + ci;
          if (mine) p.src_info[srow] = t * K + lane;
          if (first) {
            const int pos = __popc(fm & ((1u << lane) - 1u));
            s_dst[pos] = d;
            s_j[pos] = legacy ? ((e - d * L) * N + me) * B + ci : me * B + cj;
          }
        }
        if (lane == 0) {
          s_nd = __popc(fm);
          s_hdr[0] = (uint32_t)t;
          s_hdr[1] = (uint32_t)K;
        }
      }
      __syncthreads();
      LL_STAMP(p, 2);
      const int nd = s_nd;
      for (int w = threadIdx.x; w < 2 + 2 * K; w += blockDim.x)
        for (int i = 0; i < nd; ++i) {
          uint8_t* slot = peer_base(p.peers, s_dst[i]) + slot_off + (int64_t)s_j[i] * g.slot_stride;
          reinterpret_cast<uint32_t*>(slot + g.RBp + g.SBp)[w] = s_hdr[w];
        }
      if (threadIdx.x == 0)  // one record per (token, destination): row, scales, header
        for (int i = 0; i < nd; ++i)
          op_record(p.ops, EPB_OP_PUT, me, s_dst[i], slot_off + (uint64_t)s_j[i] * g.slot_stride,
                    (uint64_t)g.RBp + g.SBp + 4ull * (2 + 2 * K));
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
    if ((int)blockIdx.x == G - 1) {
      // the counting CTA: m(e) per expert and q(d) per destination over the
      // whole batch (ll.py:255-259, :292-296) -> a count row into every
      // peer's window (m of the peer's experts, then q), own counts straight
      // to the counts output
      for (int e = threadIdx.x; e < E; e += blockDim.x) s_m[e] = 0;
      for (int d = threadIdx.x; d < N; d += blockDim.x) s_q[d] = 0;
      __syncthreads();
      if (!bad) {
        for (int t = threadIdx.x; t < b; t += blockDim.x) {
          uint64_t own = 0;
          for (int k = 0; k < K; ++k) {
            const int e = s_topk[t * K + k];
            atomicAdd(&s_m[e], 1);
            own |= 1ull << (int)(((uint64_t)e * g.Lmagic) >> 32);
          }
          for (; own; own &= own - 1) atomicAdd(&s_q[__ffsll((long long)own) - 1], 1);
        }
      }
      __syncthreads();
      const int R = L + 1;
      for (int i = threadIdx.x; i < N * R; i += blockDim.x) {
        const int d = i / R, l = i - d * R;
        if (d == me) continue;
        const uint32_t v = bad ? kPoison : (l < L ? (d * L + l < E ? (uint32_t)s_m[d * L + l] : 0u) : (uint32_t)s_q[d]);
        reinterpret_cast<uint32_t*>(peer_base(p.peers, d) + parity_off + g.cnt_row)[me * R + l] = v;
      }
      if (threadIdx.x == 0)
        for (int d = 0; d < N; ++d)
          if (d != me) op_record(p.ops, EPB_OP_PUT, me, d, parity_off + g.cnt_row + 4ull * me * R, 4ull * R);
      for (int l = threadIdx.x; l < L; l += blockDim.x) {
        const int m = l < nloc && !bad ? s_m[lo + l] : 0;
        p.counts_i32[l * N + me] = m;
        p.counts_f32[l * N + me] = (float)m;
      }
      if (bad && threadIdx.x == 0) raise_err(p.err, EPB_INVALID_ARGUMENT);
    }
    // publish: one release per CTA, one arrival per destination
    ll_arrive(p.peers, parity_off + g.d_arr, N, me, g.sys_fence, sys, p.done, g.chaos_ns, G, p.ops, (seq & 1) * N, g.direct_max);
    LL_STAMP(p, 4);
    if (bad) return;
  }

  if (p.phases & kPhaseRecv) {
    LL_STAMP(p, 5);
    if (!(p.phases & kPhaseSend)) {
      if (threadIdx.x == 0) s_seq = seq_ld;
      __syncthreads();
      seq = s_seq;
      parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
    }
    if (N == 1) return;  // own rows and counts were placed by the send phase
    const uint64_t target = (uint64_t)G * ((seq >> 1) + 1);
    const uint64_t* arr = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.d_arr);
    const uint32_t* crows = reinterpret_cast<const uint32_t*>(p.win + parity_off + g.cnt_row);
    const int R = L + 1;
    const int nsrc = N - 1;
    const int ob = (OT == EPB_F32 ? 4 : dtype_width(OT));
    const int64_t orow_bytes = (int64_t)H * ob;
    if (!FAST && legacy) {
      // legacy (ll.py:362-376): slot (l*N + r)*B + i holds recv[l, r*B + i]
      // — the same linear index; per source, rows of its pairs by prefix
      __shared__ int s_wsum[kThreads / 32];
      __shared__ int s_ok;
      int* s_pp = smem;  // [L + 1] (the send phase is done with it)
      for (int so = 0; so < nsrc; ++so) {
        const int s = (me + 1 + so) % N;
        __syncthreads();
        if (threadIdx.x == 0) s_ok = wait_arrivals(&arr[s], target, sys, p.timeout_ns, p.err);
        __syncthreads();
        if (!s_ok) return;
        const uint32_t* crow = crows + s * R;
        if (crow[L] == kPoison) {
          if (threadIdx.x == 0) raise_err(p.err, EPB_TRANSPORT_CLOSED);
          return;
        }
        if ((int)blockIdx.x == s % G)
          for (int l = threadIdx.x; l < L; l += blockDim.x) {
            const int m = l < nloc ? (int)crow[l] : 0;
            p.counts_i32[l * N + s] = m;
            p.counts_f32[l * N + s] = (float)m;
          }
        block_exclusive_scan(nloc, [&](int l) { return (int)crow[l]; }, s_pp, s_wsum);
        const int rows = s_pp[nloc];
        for (int f2 = warp * gridDim.x + blockIdx.x; f2 < 2 * rows; f2 += gridDim.x * nw) {
          const int r = f2 >> 1, half = f2 & 1;
          int lo_i = 0, hi_i = nloc;  // largest l with s_pp[l] <= r
          while (hi_i - lo_i > 1) {
            const int mid = (lo_i + hi_i) >> 1;
            if (s_pp[mid] <= r) lo_i = mid; else hi_i = mid;
          }
          const int64_t lin = ((int64_t)lo_i * N + s) * B + (r - s_pp[lo_i]);
          const uint8_t* slot = p.win + parity_off + g.disp_slot + lin * g.slot_stride;
          if (lane == 0 && half == 0) {
            const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
            const int e = lo + lo_i;
            int k = 0;
            while (k < K - 1 && (int)hdr[2 + k] != e) ++k;
            p.src_info[lin] = (int32_t)(hdr[0] * K + k);
          }
          ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + lin * orow_bytes,
                                  SC ? p.out_scales + lin * (H / 128) : nullptr, lane, half, 2);
        }
      }
      LL_STAMP(p, 7);
      return;
    }
    // warp tasks (source, slot j, quarter row), sources interleaved so a warp's
    // successive tasks visit different sources; each warp waits only for
    // its task's source.  The header is read once, the row loaded once and
    // stored to every local expert the slot names (the fan-out of
    // ll.py:378-400).  Task (s, 0, 0) also writes the counts of pairs (l, s).
    const bool fan = (H & 15) == 0;
    uint64_t seen = 0;
    constexpr int kRP = 4;  // row parts per slot: 4 x B x (N-1) warp tasks
    const int tasks = kRP * B * nsrc;
    for (int f2 = warp * gridDim.x + blockIdx.x; f2 < tasks; f2 += gridDim.x * nw) {
      const int part = f2 % kRP, r = f2 / kRP;
      const int j = r / nsrc, so = r - j * nsrc;
      const int s = me + 1 + so < N ? me + 1 + so : me + 1 + so - N;
      if (!warp_wait_sources(1ull << s, seen, arr, target, sys, p.timeout_ns, p.err, lane)) return;
      if (f2 == (int)blockIdx.x) LL_STAMP(p, 6);  // warp 0's first arrival seen
      // the slot count, the slot header and the first batch of the row are
      // loaded together (one round trip; slot (s, j) exists even when the
      // source sent fewer slots — those loads are then simply unused)
      const uint32_t* crow = crows + s * R;
      const uint8_t* slot = p.win + parity_off + g.disp_slot + ((int64_t)s * B + j) * g.slot_stride;
      const uint32_t* hdr = reinterpret_cast<const uint32_t*>(slot + g.RBp + g.SBp);
      const int nch2 = H / EPC;
      const int per = (nch2 + kRP - 1) / kRP;
      const int c0 = part * per, c1 = min(nch2, c0 + per);
      int4 v0[kUnroll];
      if (FAST || fan) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c < c1) v0[u] = ld_weak_v4(slot + (int64_t)c * 16);
        }
      }
      const uint32_t q = crow[L];
      int e = -1, ci = 0;
      if (lane < K) {
        e = (int)hdr[2 + lane];
        ci = (int)hdr[2 + K + lane];
      }
      const uint32_t tok = hdr[0];
      if (q == kPoison) {
        if (lane == 0) raise_err(p.err, EPB_TRANSPORT_CLOSED);
        return;
      }
      if (j == 0 && part == 0)
        for (int l = lane; l < L; l += 32) {
          const int m = l < nloc ? (int)crow[l] : 0;
          p.counts_i32[l * N + s] = m;
          p.counts_f32[l * N + s] = (float)m;
        }
      if (j >= (int)q) continue;
      const bool loc = lane < K && e >= lo && e < lo + nloc;
      const int my_orow = (e - lo) * N * B + s * B + ci;
      const unsigned lm = __ballot_sync(0xffffffffu, loc);
      if (part == 0 && loc) p.src_info[my_orow] = (int32_t)(tok * K + lane);
      if (!FAST && !fan) {
        for (unsigned mm = lm; mm; mm &= mm - 1) {
          const int64_t row = __shfl_sync(0xffffffffu, my_orow, __ffs(mm) - 1);
          ll_copy_row<WT, SC, OT>(g, slot, reinterpret_cast<uint8_t*>(p.out) + row * orow_bytes,
                                  SC ? p.out_scales + row * (H / 128) : nullptr, lane, part, kRP);
        }
        continue;
      }
      for (int base = c0; base < c1; base += 32 * kUnroll) {
        int4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int c = base + u * 32 + lane;
          if (base == c0) v[u] = v0[u];
          else if (c < c1) v[u] = ld_weak_v4(slot + (int64_t)c * 16);
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
        if (part == 0) {
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
  unsigned* done;  // local CTA-completion counter of the send phase (ll_arrive)
  uint64_t* trace;
  OpTrace ops;
  LLGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
  bool sys;
};

// VEC: hidden % 16 == 0 (the vector paths only; the element paths are a
// separate instantiation, keeping the hot kernel's code small)
template <int IT, int WT, int OT, bool VEC>
__global__ void __launch_bounds__(kThreads) ll_combine_kernel(LLComb p) {
  extern __shared__ int s_pre[];  // [L*N + 1]
  pdl_enter();
  const LLGeom& g = p.g;
  const int N = g.N, L = g.L, B = g.B, H = g.H, K = g.K, G = gridDim.x;
  const int me = p.rank;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool sys = p.sys;
  LL_STAMP(p, 0);
  __shared__ uint32_t s_seq;
  __shared__ int s_wsum[kThreads / 32];
  // the round load is in flight while the send phase loads its counts
  uint32_t seq_ld = 0;
  if (threadIdx.x == 0 && N > 1) seq_ld = ld_round_u32(p.hseq);
  constexpr int EPC = Elems<WT>::n;
  constexpr bool vec = VEC;
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
  // (one rank: every row is this rank's own, read in place — no slots, no
  // round parity, no barrier)
  uint32_t seq = 0;
  if (N > 1) {
    if (threadIdx.x == 0) s_seq = seq_ld;
    __syncthreads();
    seq = s_seq;
  }
  const uint64_t parity_off = (uint64_t)(seq & 1) * g.parity_bytes;
  int send_ctas = 0;  // CTAs that store rows this round (task t of the first pass goes to CTA t / warps)

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
    send_ctas = min((int)gridDim.x, ((vec ? total * kParts : total) + nw - 1) / nw);
    chaos_delay(g.chaos_ns, 0x2Bu);
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
      if (lane == 0 && q == 0)  // one record per (token, k) row pushed to its home
        op_record(p.ops, EPB_OP_PUT, me, s, parity_off + g.comb_slot + (uint64_t)cs * g.comb_stride,
                  (uint64_t)H * dtype_width(WT));
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
    LL_STAMP(p, 2);
  }
  if ((p.phases & kPhaseSend) && N > 1) {
    // one release per CTA, one arrival per home rank (pulled combine: the
    // expert outputs were written by earlier kernels on this stream — the
    // arrival announces them)
    ll_arrive(p.peers, parity_off + g.c_arr, N, me, g.sys_fence, sys, p.done, g.chaos_ns, send_ctas, p.ops,
              2 * N + (seq & 1) * N, g.direct_max);
    LL_STAMP(p, 3);
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
    int my_self = -1, my_slot = 0, my_owner = me;
    uint64_t my_pull = 0;  // pulled combine: the row in its owner's window
    float my_w = 0.0f;
    auto fetch = [&](int tk) {  // lane k's row of token tk
      if (lane < K) {
        const int64_t i = (int64_t)tk * K + lane;
        my_w = p.w[i];
        const int e = (int)p.topk[i];
        my_owner = (int)(((uint64_t)e * g.Lmagic) >> 32);
        if (p.pull) {
          my_pull = reinterpret_cast<uint64_t>(peer_base(p.peers, my_owner) + g.yout) + (uint64_t)p.owner_row[i] * g.yrow;
        } else {
          my_self = p.self_row ? p.self_row[i] : -1;
          my_slot = legacy ? e * B + tk : tk * K + lane;
        }
      }
    };
    if (vec && task < tasks) fetch(task / segs);
    const uint64_t target = (uint64_t)G * ((seq >> 1) + 1);
    const uint64_t* arr = reinterpret_cast<const uint64_t*>(p.win + parity_off + g.c_arr);
    uint64_t seen = 0;
    LL_STAMP(p, 5);
    if (vec) {
      for (; task < tasks; task += tstride) {
        const int t = task / segs, sg = task - t * segs;
        // the owners of this token's experts must have arrived (rows pushed
        // into our slots, or, pulled, their expert outputs announced)
        if (N > 1) {
          const uint64_t bit = (lane < K && my_owner != me) ? 1ull << my_owner : 0ull;
          const uint64_t need = (uint64_t)__reduce_or_sync(0xffffffffu, (uint32_t)bit) |
                                ((uint64_t)__reduce_or_sync(0xffffffffu, (uint32_t)(bit >> 32)) << 32);
          if (!warp_wait_sources(need, seen, arr, target, sys, p.timeout_ns, p.err, lane)) return;
          if (task == (int)blockIdx.x) LL_STAMP(p, 7);  // warp 0's first token's sources seen
        }
        uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + (int64_t)t * H * dtype_width(OT);
        const int cbase = sg * kSeg + lane;
        if (p.pull && sg == 0 && lane < K && my_owner != me)  // one record per (token, k) row pulled
          op_record(p.ops, EPB_OP_GET, me, my_owner,
                    g.yout + (uint64_t)p.owner_row[(int64_t)t * K + lane] * g.yrow, (uint64_t)H * dtype_width(WT));
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
      // element path (hidden not a multiple of 16): every source first
      if (threadIdx.x == 0) {
        s_fail = 0;
        for (int s2 = 0; s2 < N; ++s2)
          if (s2 != me && !wait_arrivals(&arr[s2], target, sys, p.timeout_ns, p.err)) s_fail = 1;
      }
      __syncthreads();
      if (s_fail) return;
      for (int t = blockIdx.x; t < p.b; t += gridDim.x) {
        __syncthreads();
        if ((int)threadIdx.x < K) {
          s_w[threadIdx.x] = p.w[(int64_t)t * K + threadIdx.x];
          const int k = threadIdx.x;
          const int e = (int)p.topk[(int64_t)t * K + k];
          const int ow = (int)(((uint64_t)e * g.Lmagic) >> 32);
          if (p.pull && ow != me)
            op_record(p.ops, EPB_OP_GET, me, ow, g.yout + (uint64_t)p.owner_row[(int64_t)t * K + k] * g.yrow,
                      (uint64_t)H * dtype_width(WT));
        }
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

// EPB_PDL=0 launches the LL kernels without programmatic dependent launch
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("EPB_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
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

// per-kernel launch state, set up once: the dynamic shared memory opt-in and
// the co-residency check of the cooperative launch (cudaFuncSetAttribute and
// the occupancy query cost several microseconds of host time per call)
struct KernState {
  size_t smem_set = 0;  // dynamic shared memory opted in so far
  size_t occ_smem = 0;  // smem the occupancy was computed for
  int per_sm = -1;
};
std::mutex g_kern_mu;
std::unordered_map<uint64_t, KernState> g_kern;  // key: kernel address ^ device (attributes are per device)

template <typename Params>
cudaError_t launch(void (*kern)(Params), int grid, size_t smem, bool coop, const Params& p, cudaStream_t s) {
  int per_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_kern_mu);
    KernState& ks = g_kern[reinterpret_cast<uint64_t>(kern) ^ ((uint64_t)dev << 56)];
    const size_t want = std::max<size_t>(smem, 48 * 1024);
    if (want > ks.smem_set) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
      if (e != cudaSuccess) return e;
      ks.smem_set = want;
    }
    if (coop && (ks.per_sm < 0 || smem > ks.occ_smem)) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ks.per_sm, kern, kThreads, smem);
      if (e != cudaSuccess) return e;
      ks.occ_smem = smem;
    }
    per_sm = ks.per_sm;
  }
  if (coop) {
    // both phases in one launch: CTAs in the receive phase wait on arrivals
    // other GPUs' CTAs publish, so all CTAs must be co-resident
    if (per_sm * sm_count() < grid) return cudaErrorCooperativeLaunchTooLarge;
    if (!coop_attr_enabled()) {
      // co-residency from grid <= SMs x occupancy alone: may overlap its
      // predecessor's drain like the unfused launches
      if (!pdl_enabled()) {
        kern<<<grid, kThreads, smem, s>>>(p);
        return cudaGetLastError();
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, kern, p);
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
  if (pdl_enabled()) {
    // not cooperative: let this grid be scheduled while its predecessor
    // drains (it waits for the predecessor's completion in pdl_enter)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  kern<<<grid, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int XT, int WT, bool SC, int OT>
cudaError_t run_disp(const LLDisp& p, size_t smem, cudaStream_t s) {
  // fused send + receive across GPUs: receivers spin on arrivals from peer
  // GPUs' CTAs, which must all be resident -> cooperative launch
  const bool coop = p.phases == 3 && p.g.N > 1;
  // (an op-traced launch takes the general kernel: the decode kernel
  // carries no trace code)
  const bool fast = p.g.K <= 8 && p.b <= kThreads && (p.g.H & 15) == 0 && p.g.layout == EPB_LAYOUT_OPTIMIZED &&
                    p.ops.ring == nullptr;
  return fast ? launch(ll_dispatch_kernel<XT, WT, SC, OT, true>, p.g.grid, smem, coop, p, s)
              : launch(ll_dispatch_kernel<XT, WT, SC, OT, false>, p.g.grid, smem, coop, p, s);
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
  const bool coop = p.phases == 3 && p.g.N > 1;
  return (p.g.H & 15) == 0 ? launch(ll_combine_kernel<IT, WT, OT, true>, p.g.grid, smem, coop, p, s)
                           : launch(ll_combine_kernel<IT, WT, OT, false>, p.g.grid, smem, coop, p, s);
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
  p.dseq = g->d_seq; p.done = reinterpret_cast<unsigned*>(g->d_scratch) + 4; p.trace = g->trace;
  p.ops.ring = g->op_ring; p.ops.cap = g->op_cap;
  p.g = g->ll; p.timeout_ns = g->timeout_ns; p.b = b; p.rank = g->rank; p.phases = phases;
  p.sys = g->sys_scope;
  const int E = g->ll.E, N = g->ll.N, K = g->ll.K;
  // send: routing snapshot [b*K] + per-expert / per-destination counts;
  // legacy receive: per-source expert prefix [L + 1]
  size_t smem = (phases & kPhaseSend) ? sizeof(int) * ((size_t)b * K + E + N) : 0;
  if ((phases & kPhaseRecv) && g->cfg.layout == EPB_LAYOUT_LEGACY)
    smem = std::max(smem, sizeof(int) * ((size_t)g->ll.L + 1));
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
  p.ops.ring = g->op_ring; p.ops.cap = g->op_cap;
  p.done = reinterpret_cast<unsigned*>(g->d_scratch) + 5;
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
