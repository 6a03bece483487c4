// High-Throughput dispatch/combine kernels (K5a meta, K5b dispatch, K6 combine).
//
// Reference semantics (epsim ht.py):
//  * metadata (ht.py:291-331): every rank all-gathers m_row[E] (tokens per
//    expert) and q_row[N] (dedup tokens per destination) before any payload;
//    receive shapes and the sorted-output offsets follow from them
//    (HTMeta.expert_offsets, ht.py:185-193).
//  * dispatch (ht.py:381-468, 553-583): one record per (token, destination
//    rank) = header + K f32 weights + row; the receiver places a copy of the
//    row for every local expert it names, sorted by (local expert, src, t).
//    The sender also writes, per k, the final output row on the owner
//    (offset(e, src) + rank of t within (e, src)), so placement is a parallel
//    scatter that never depends on arrival order.  Rows a rank routes to its
//    OWN experts skip the window: the sender writes them straight to their
//    sorted output position.
//  * combine (ht.py:587-735): p = f32(w * y) from the f32 expert row; per
//    token, per node holding its experts (ascending), a partial = first p
//    then f32 adds in ascending k; out = f32(0 + partial_0) + partial_1 ...
//    Expert rows travel in their own dtype (f32, or bf16 which widens
//    exactly) and the home rank forms p, so the product is bit-identical.
//    Rows of the home's own experts are read in place, not copied.
//  * single-node transport only: the reference's rail FIFOs / forwarders
//    (ht.py:479-551) are out of scope on one NVSwitch domain, but the
//    hierarchical SUM ORDER is reproduced for any ranks_per_node.
#include "common.cuh"
#include "internal.h"

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
  const int32_t* m;
  const int32_t* q;
  const uint64_t* peers;
  HTGeom g;
  int rank, parity;
  uint32_t tag;
};

__global__ void __launch_bounds__(256) ht_meta_send_kernel(HTMetaSend p) {
  const HTGeom& g = p.g;
  const int C = g.E + g.N;
  const uint64_t row_off = g.meta + ((uint64_t)p.parity * g.N + p.rank) * C * 4;
  for (int i = threadIdx.x; i < g.N * C; i += blockDim.x) {
    const int d = i / C, c = i % C;
    const int32_t v = c < g.E ? p.m[c] : p.q[c - g.E];
    reinterpret_cast<int32_t*>(hpeer(p.peers, d) + row_off)[c] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < g.N) {
    fence_sys();
    uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, threadIdx.x) + g.meta_flag) +
                     p.parity * g.N + p.rank;
    st_relaxed_sys_u64(flag, (uint64_t)p.tag);
  }
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

__global__ void __launch_bounds__(1024) ht_meta_recv_kernel(HTMetaRecv p) {
  extern __shared__ int32_t s_meta[];  // [N][C]
  __shared__ int s_fail;
  const HTGeom& g = p.g;
  const int N = g.N, E = g.E, C = E + N, L = g.L;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.meta_flag) + p.parity * N;
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v;
    if (!wait_tag(&flags[s], p.tag, 0, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) return;
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

// ---------------------------------------------------------------------------
// K5b: dispatch
// ---------------------------------------------------------------------------
struct HTDisp {
  const void* x;
  const float* w;
  const int64_t* topk;
  const int32_t* tok_rank;
  const int32_t* tok_slot;
  const int32_t* offsets;  // [E, N]
  const uint64_t* peers;
  const uint8_t* win;
  void* out;               // own sorted output
  int32_t* origin;
  float* origin_w;
  int* err;
  HTGeom g;
  uint64_t timeout_ns;
  int b, rank, phases;
  uint32_t tag;
};

constexpr int kFlush = 4;  // sender CTAs publish progress every kFlush tokens

// dispatch flag word: (tag << 40) | (tokens of the source << 20) | tokens done by the CTA
EPB_DEV void ht_publish_progress(const HTDisp& p, int c, int done) {
  if ((int)threadIdx.x < p.g.N && (int)threadIdx.x != p.rank) {
    fence_sys();
    uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, threadIdx.x) + p.g.dflag) +
                     (int64_t)p.rank * kHTSendCTAs + c;
    st_relaxed_sys_u64(flag, ((uint64_t)p.tag << 40) | ((uint64_t)p.b << 20) | (uint64_t)done);
  }
}

// wait until sender CTA c of this source has published this round and either
// advanced past `processed` or finished; backs off so the spinning receivers
// leave the memory system to the incoming records.  ~0 on timeout / error.
EPB_DEV uint64_t ht_wait_progress(const uint64_t* f, uint32_t tag, int c, int processed, uint64_t timeout_ns,
                                  int* err) {
  uint64_t start = 0;
  for (int spins = 0;; ++spins) {
    const uint64_t v = ld_acquire_sys(f);
    if ((uint32_t)(v >> 40) == tag) {
      const int bs = (int)((v >> 20) & 0xFFFFF), done = (int)(v & 0xFFFFF);
      const int n_c = c < bs ? (bs - c + kHTSendCTAs - 1) / kHTSendCTAs : 0;
      if (done > processed || done >= n_c) return v;
    }
    if (*(volatile int*)err != 0) return ~0ull;
    if (spins == 0) start = globaltimer();
    else if ((spins & 63) == 0 && globaltimer() - start > timeout_ns) {
      atomicCAS(err, 0, EPB_TRANSPORT_CLOSED);
      return ~0ull;
    }
    __nanosleep(200);
  }
}

// K5b: one cooperative launch, two roles.
//  * sender CTA c (< kHTSendCTAs) owns tokens t = c, c + kHTSendCTAs, ...;
//    each goes once to every remote rank it touches, into that rank's record
//    slot [src][t] (header carries the round tag), and straight into this
//    rank's own sorted output for its local experts.  Afterwards the CTA
//    fences and raises flag [src][c] at every remote rank.
//  * receiver CTAs walk the (src, sender CTA) pairs: once a pair's flag is up
//    its records are scattered to their sorted positions while other pairs
//    are still in flight, so the HBM scatter overlaps the NVLink transfer.
template <int XT, int WT, int OT>
__global__ void __launch_bounds__(kHTThreads) ht_dispatch_kernel(HTDisp p) {
  constexpr int kTB = 16;
  const HTGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L, B = g.B;
  const int me = p.rank;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : 2;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  const bool sender = (int)blockIdx.x < kHTSendCTAs;
  if (sender && (p.phases & 1)) {
    __shared__ int s_e[kTB][kMaxTopK], s_pos[kTB][kMaxTopK];
    __shared__ float s_w[kTB][kMaxTopK];
    __shared__ int s_go[kTB][kMaxRanks];
    const int c0 = blockIdx.x;
    const int G = kHTSendCTAs;
    for (int base = c0; base < p.b; base += G * kTB) {
      __syncthreads();
      for (int idx = threadIdx.x; idx < kTB * K; idx += blockDim.x) {
        const int i = idx / K, k = idx - i * K, t = base + i * G;
        if (t >= p.b) continue;
        const int e = (int)p.topk[(int64_t)t * K + k];
        const int pos = p.offsets[e * N + me] + p.tok_rank[(int64_t)t * K + k];
        const float wk = p.w[(int64_t)t * K + k];
        s_e[i][k] = e;
        s_pos[i][k] = pos;
        s_w[i][k] = wk;
        if (e / L == me) {
          p.origin[(int64_t)pos * 4 + 0] = e;
          p.origin[(int64_t)pos * 4 + 1] = me;
          p.origin[(int64_t)pos * 4 + 2] = t;
          p.origin[(int64_t)pos * 4 + 3] = k;
          p.origin_w[pos] = wk;
        }
      }
      for (int idx = threadIdx.x; idx < kTB * N; idx += blockDim.x) {
        const int i = idx / N, d = idx - i * N, t = base + i * G;
        s_go[i][d] = (t < p.b && d != me && p.tok_slot[(int64_t)t * N + d] >= 0) ? 1 : 0;
      }
      __syncthreads();
      for (int i = 0; i < kTB; ++i) {
        const int t = base + i * G;
        if (t >= p.b) break;
        if (i > 0 && (i & (kFlush - 1)) == 0) {
          // progress: tokens [0, done) of this CTA are complete at every destination
          __syncthreads();
          ht_publish_progress(p, c0, (base - c0) / G + i);
        }
        const int64_t slot = (int64_t)me * B + t;
        // record: [row][K weights][tag, t, K, ids[K], positions[K]]
        const int words = K + 3 + 2 * K;
        for (int idx = threadIdx.x; idx < N * words; idx += blockDim.x) {
          const int d = idx / words, wd = idx - d * words;
          if (!s_go[i][d]) continue;
          uint8_t* rec = hpeer(p.peers, d) + g.rec + slot * g.rec_stride;
          if (wd < K) {
            reinterpret_cast<float*>(rec + g.RBp)[wd] = s_w[i][wd];
          } else {
            const int h = wd - K;
            const uint32_t v = h == 0 ? p.tag : h == 1 ? (uint32_t)t : h == 2 ? (uint32_t)K
                               : h < 3 + K ? (uint32_t)s_e[i][h - 3] : (uint32_t)s_pos[i][h - 3 - K];
            reinterpret_cast<uint32_t*>(rec + g.RBp + g.WBp)[h] = v;
          }
        }
        const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * XW;
        if ((H & 15) == 0) {
          for (int c = threadIdx.x; c < H / EPC; c += blockDim.x) {
            float f[EPC];
            load_elems_vec<XT, EPC>(xrow, (int64_t)c * EPC, f);
            const int4 v = pack16<WT>(f);
            for (int d = 0; d < N; ++d)
              if (s_go[i][d]) st_na_v4(hpeer(p.peers, d) + g.rec + slot * g.rec_stride + (int64_t)c * 16, v);
            float fw[EPC];
            unpack16<WT>(v, fw);  // the wire image, exactly what a record carries
            for (int k = 0; k < K; ++k)
              if (s_e[i][k] / L == me)
                store_f32_chunk<OT, EPC>(reinterpret_cast<uint8_t*>(p.out) + (int64_t)s_pos[i][k] * H * OW,
                                         (int64_t)c * EPC, fw);
          }
        } else {
          for (int el = threadIdx.x; el < H; el += blockDim.x) {
            const float f = load_elem(xrow, XT, el);
            for (int d = 0; d < N; ++d)
              if (s_go[i][d]) store_elem(hpeer(p.peers, d) + g.rec + slot * g.rec_stride, WT, el, f);
            const float fw = WT == EPB_F32 ? f
                             : (WT == EPB_BF16 ? bf16_widen(bf16_bits_rne(f)) : f16_widen(f16_bits_rne(f)));
            for (int k = 0; k < K; ++k)
              if (s_e[i][k] / L == me)
                store_elem(reinterpret_cast<uint8_t*>(p.out) + (int64_t)s_pos[i][k] * H * OW, OT, el, fw);
          }
        }
      }
    }
    __syncthreads();
    ht_publish_progress(p, c0, c0 < p.b ? (p.b - c0 + G - 1) / G : 0);
    return;
  }
  if (!sender && (p.phases & 2)) {
    // receiver CTAs: items = (sender CTA c, remote src), c-major; one CTA per
    // item, its warps split the (token, k) copies of every published step
    __shared__ uint64_t s_v;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nrc = (int)gridDim.x - kHTSendCTAs;
    const int lo = me * L, hi = min(lo + L, g.E);
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.dflag);
    for (int item = (int)blockIdx.x - kHTSendCTAs; item < kHTSendCTAs * N; item += nrc) {
      const int c = item / N, s = item - c * N;
      if (s == me) continue;
      const uint64_t* flag = &flags[(int64_t)s * kHTSendCTAs + c];
      int processed = 0;
      for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_v = ht_wait_progress(flag, p.tag, c, processed, p.timeout_ns, p.err);
        __syncthreads();
        const uint64_t v = s_v;
        if (v == ~0ull) return;
        const int bs = (int)((v >> 20) & 0xFFFFF);  // tokens of source s
        const int done = (int)(v & 0xFFFFF);
        const int n_c = c < bs ? (bs - c + kHTSendCTAs - 1) / kHTSendCTAs : 0;
        const int ntok = max(0, min(done, n_c) - processed);
        for (int f = warp; f < ntok * K; f += nw) {
          const int i = processed + f / K, k = f - (f / K) * K;
          const int t = c + i * kHTSendCTAs;
          const uint8_t* rec = p.win + g.rec + ((int64_t)s * B + t) * g.rec_stride;
          const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec + g.RBp + g.WBp);
          if (hdr[0] != p.tag) continue;  // t does not touch this rank this round
          const int e = (int)hdr[3 + k];
          if (e < lo || e >= hi) continue;
          const int64_t pos = hdr[3 + K + k];
          if (lane == 0) {
            p.origin[pos * 4 + 0] = e;
            p.origin[pos * 4 + 1] = s;
            p.origin[pos * 4 + 2] = t;
            p.origin[pos * 4 + 3] = k;
            p.origin_w[pos] = reinterpret_cast<const float*>(rec + g.RBp)[k];
          }
          uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + pos * H * OW;
          if ((H & 15) == 0) {
            const int nch = H / EPC;
            for (int bb = 0; bb < nch; bb += 32 * kHU) {
              int4 q[kHU];
#pragma unroll
              for (int u = 0; u < kHU; ++u) {
                const int cc = bb + u * 32 + lane;
                if (cc < nch) q[u] = ld_plain_v4(rec + (int64_t)cc * 16);
              }
#pragma unroll
              for (int u = 0; u < kHU; ++u) {
                const int cc = bb + u * 32 + lane;
                if (cc < nch) {
                  if constexpr (OT == WT) {
                    st_plain_v4(orow + (int64_t)cc * 16, q[u]);
                  } else {
                    float fv[EPC];
                    unpack16<WT>(q[u], fv);
                    store_f32_chunk<OT, EPC>(orow, (int64_t)cc * EPC, fv);
                  }
                }
              }
            }
          } else {
            for (int el = lane; el < H; el += 32) store_elem(orow, OT, el, load_elem(rec, WT, el));
          }
        }
        processed = max(processed, min(done, n_c));
        if (processed >= n_c) break;
      }
    }
  }
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
  HTGeom g;
  int rows, rank, in_dtype;
  uint32_t tag;
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
  st_relaxed_sys_u64(flag, ((uint64_t)p.tag << 32) | ((uint64_t)p.in_dtype << 28) | (uint32_t)count);
}

template <int IT>
__global__ void __launch_bounds__(kHTThreads) ht_combine_send_kernel(HTCombSend p) {
  __shared__ int s_cnt[kMaxRanks];
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H;
  const int me = p.rank;
  if (*reinterpret_cast<const volatile int*>(p.err) != 0) return;
  if ((int)threadIdx.x < N) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int ib = IT == EPB_F32 ? 4 : 2;
  const int bytes = H * ib;
  const int nch = (bytes & 15) == 0 ? bytes / 16 : 0;
  // warp tasks: (row, half); rows of my own tokens stay (the home reads them in place)
  for (int task = warp * gridDim.x + blockIdx.x; task < 2 * p.rows; task += gridDim.x * nw) {
    const int r = task >> 1, half = task & 1;
    const int s = p.origin[(int64_t)r * 4 + 1];
    if (s == me) continue;
    const int t = p.origin[(int64_t)r * 4 + 2];
    const int k = p.origin[(int64_t)r * 4 + 3];
    uint8_t* dst = hpeer(p.peers, s) + g.crow + ((int64_t)t * K + k) * g.crow_stride;
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
    if (lane == 0 && half == 0) atomicAdd(&s_cnt[s], 1);
  }
  __syncthreads();
  if ((int)threadIdx.x < N && (int)threadIdx.x != me) {
    const int s = threadIdx.x;
    const int c = s_cnt[s];
    const int want = ht_rows_to(p, s);
    if (c > 0) {
      fence_sys();
      const int old = atomicAdd(&p.done[s], c);
      if (old + c == want) {
        p.done[s] = 0;
        fence_sys();
        ht_publish_comb(p, s, want);
      }
    } else if (blockIdx.x == 0 && want == 0) {
      ht_publish_comb(p, s, 0);
    }
  }
}

struct HTCombRecv {
  const int64_t* topk;
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
__global__ void __launch_bounds__(kHTThreads, 2) ht_combine_recv_kernel(HTCombRecv p) {
  __shared__ int s_fail;
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H, L = g.L;
  const int me = p.rank;
  constexpr int YB = IT == EPB_F32 ? 4 : 2;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  if (threadIdx.x == 0) s_fail = *reinterpret_cast<const volatile int*>(p.err) != 0;
  __syncthreads();
  if (s_fail) return;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.cflag);
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v = 0;
    if (s == me) continue;
    if (!wait_tag(&flags[s], p.tag, 32, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) { s_fail = 1; continue; }
    // every rank must combine in the same dtype (the rows are raw bytes)
    if ((int)((v >> 28) & 0xF) != IT) { atomicCAS(p.err, 0, EPB_TAG_MISMATCH); s_fail = 1; }
  }
  __syncthreads();
  if (s_fail) return;
  const uint8_t* crow = p.win + g.crow;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool one_node = g.rpn == N;
  if ((H & 7) == 0 && K <= 32) {
    // warp tasks: (token, 32-chunk segment of 8 elements); lane = one chunk.
    // Lane k first resolves row k of the token (own expert rows are read in
    // place from the local expert output, others from the combine slots).
    const int nch = H / 8;
    const int segs = (nch + 31) / 32;
    for (int task = warp * gridDim.x + blockIdx.x; task < p.b * segs; task += gridDim.x * nw) {
      const int t = task / segs, c = (task - t * segs) * 32 + lane;
      uint64_t my_row = 0;
      float my_w = 0.0f;
      int my_node = 0;
      if (lane < K) {
        const int e = (int)p.topk[(int64_t)t * K + lane];
        const int owner = e / L;
        my_node = owner / g.rpn;
        my_w = p.w[(int64_t)t * K + lane];
        my_row = owner == me
            ? reinterpret_cast<uint64_t>(p.y_local) +
                  (uint64_t)(p.offsets[e * N + me] + p.tok_rank[(int64_t)t * K + lane]) * H * YB
            : reinterpret_cast<uint64_t>(crow + ((int64_t)t * K + lane) * g.crow_stride);
      }
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
      if (one_node) {
        // single node: acc = p_0 + p_1 + ... (first present as init), then
        // out = 0 + acc; all KB rows of a batch are in flight at once
        constexpr int KB = IT == EPB_F32 ? 2 : 4;
        constexpr int NV = IT == EPB_F32 ? 2 : 1;  // 16-B loads per 8-element chunk
        for (int k0 = 0; k0 < K; k0 += KB) {
          int4 v[KB][NV];
          float wk[KB];
#pragma unroll
          for (int u = 0; u < KB; ++u) {
            const uint64_t row = __shfl_sync(0xffffffffu, my_row, (k0 + u) & 31);
            wk[u] = __shfl_sync(0xffffffffu, my_w, (k0 + u) & 31);
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
            const int n2 = __shfl_sync(0xffffffffu, my_node, k);
            if (n2 > prev && n2 < nd) nd = n2;
          }
          if (nd == 0x7fffffff) break;
          float part[8];
          bool started = false;
          for (int k = 0; k < K; ++k) {
            const int n2 = __shfl_sync(0xffffffffu, my_node, k);
            const uint64_t row = __shfl_sync(0xffffffffu, my_row, k);
            const float wk = __shfl_sync(0xffffffffu, my_w, k);
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
    if (__float_as_uint(a[i]) != __float_as_uint(b[i]) && !(a[i] == b[i])) atomicCAS(err, 0, EPB_INVALID_ARGUMENT);
}

}  // namespace epb

using namespace epb;

namespace {

uint32_t ht_tag(uint32_t round) { return (round % 0xFFFFFFu) + 1u; }  // fits the 24-bit flag field

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

int ht_coop_grid(void (*kern)(HTDisp)) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHTThreads, 0);
  return per_sm * hsm_count();
}

template <int XT, int WT, int OT>
cudaError_t launch_hdisp(const HTDisp& p, cudaStream_t s) {
  auto kern = ht_dispatch_kernel<XT, WT, OT>;
  const int grid = kHTSendCTAs + kHTRecvCTAs;
  if (p.phases == 3) {
    // sender and receiver CTAs wait on each other's flags: all co-resident
    if (ht_coop_grid(kern) < grid) return cudaErrorCooperativeLaunchTooLarge;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kHTThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  }
  kern<<<grid, kHTThreads, 0, s>>>(p);
  return cudaGetLastError();
}

template <int XT, int WT>
cudaError_t launch_hdisp_o(const HTDisp& p, int out_dtype, cudaStream_t s) {
  return out_dtype == EPB_F32 ? launch_hdisp<XT, WT, EPB_F32>(p, s) : launch_hdisp<XT, WT, WT>(p, s);
}

template <int XT>
cudaError_t launch_hdisp_x(const HTDisp& p, int out_dtype, cudaStream_t s) {
  switch (p.g.wire) {
    case EPB_F32: return launch_hdisp<XT, EPB_F32, EPB_F32>(p, s);
    case EPB_BF16: return launch_hdisp_o<XT, EPB_BF16>(p, out_dtype, s);
    default: return launch_hdisp_o<XT, EPB_F16>(p, out_dtype, s);
  }
}

bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int epb_ht_meta_send(epb_group* g, uint32_t round, const epb_layout* lay, void* stream) {
  if (int rc = check_ht(g, 1)) return rc;
  HTMetaSend p;
  p.m = lay->expert_count; p.q = lay->rank_count; p.peers = g->d_peers; p.g = g->ht;
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

int epb_ht_dispatch(epb_group* g, uint32_t round, int32_t phases, const epb_ht_dispatch_args* a, void* stream) {
  if (int rc = check_ht(g, phases)) return rc;
  const int wire = g->cfg.token_dtype;
  if (a->out_dtype != EPB_F32 && a->out_dtype != wire)
    return fail(EPB_TAG_MISMATCH, "dispatch output must be f32 or the wire dtype");
  if (!a16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
  if ((phases & 1) && a->num_tokens > 0 && !a16(a->x)) return fail(EPB_INVALID_ARGUMENT, "x must be 16-byte aligned");
  HTDisp p;
  p.x = a->x; p.w = a->weights; p.topk = a->topk_idx; p.tok_rank = a->tok_rank; p.tok_slot = a->tok_slot;
  p.offsets = a->offsets; p.peers = g->d_peers; p.win = g->window; p.out = a->out; p.origin = a->origin;
  p.origin_w = a->origin_w; p.err = g->d_err; p.g = g->ht; p.timeout_ns = g->timeout_ns; p.b = a->num_tokens;
  p.rank = g->rank; p.phases = phases; p.tag = ht_tag(round);
  cudaStream_t s = as_stream(stream);
  cudaError_t e;
  switch (a->x_dtype) {
    case EPB_F32: e = launch_hdisp_x<EPB_F32>(p, a->out_dtype, s); break;
    case EPB_BF16: e = launch_hdisp_x<EPB_BF16>(p, a->out_dtype, s); break;
    case EPB_F16: e = launch_hdisp_x<EPB_F16>(p, a->out_dtype, s); break;
    default: return fail(EPB_TAG_MISMATCH, "HT dispatch input must be f32/bf16/f16");
  }
  if (e != cudaSuccess) return cuda_check(e, "ht_dispatch");
  return EPB_OK;
}

int epb_ht_combine(epb_group* g, uint32_t round, int32_t phases, const epb_ht_combine_args* a, void* stream) {
  if (int rc = check_ht(g, phases)) return rc;
  if (a->in_dtype != EPB_F32 && a->in_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine input f32|bf16");
  if (a->recv_total > 0 && !a16(a->expert_rows)) return fail(EPB_INVALID_ARGUMENT, "expert rows must be 16-byte aligned");
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
    p.err = g->d_err;
    p.y = a->expert_rows; p.origin = a->origin;
    p.meta = reinterpret_cast<const int32_t*>(g->window + g->ht.meta +
                                              (uint64_t)(round & 1) * g->ht.N * (g->ht.E + g->ht.N) * 4);
    p.peers = g->d_peers; p.done = g->d_done + g->cfg.num_ranks; p.g = g->ht; p.rows = a->recv_total;
    p.rank = g->rank; p.in_dtype = a->in_dtype; p.tag = ht_tag(round);
    const int grid = 2 * hsm_count();
    if (a->in_dtype == EPB_F32) ht_combine_send_kernel<EPB_F32><<<grid, kHTThreads, 0, s>>>(p);
    else ht_combine_send_kernel<EPB_BF16><<<grid, kHTThreads, 0, s>>>(p);
    EPB_LAUNCH_CHECK();
  }
  if (phases & 2) {
    if (a->out_dtype != EPB_F32 && a->out_dtype != EPB_BF16) return fail(EPB_TAG_MISMATCH, "combine output f32|bf16");
    if (!a16(a->out)) return fail(EPB_INVALID_ARGUMENT, "out must be 16-byte aligned");
    HTCombRecv p;
    p.topk = a->topk_idx; p.w = a->weights; p.y_local = a->expert_rows; p.tok_rank = a->tok_rank;
    p.offsets = a->offsets; p.out = a->out; p.win = g->window; p.err = g->d_err; p.g = g->ht;
    p.timeout_ns = g->timeout_ns; p.b = a->num_tokens; p.rank = g->rank; p.y_dtype = a->in_dtype;
    p.tag = ht_tag(round);
    const int grid = 2 * hsm_count();
    if (a->in_dtype == EPB_F32) {
      if (a->out_dtype == EPB_F32) ht_combine_recv_kernel<EPB_F32, EPB_F32><<<grid, kHTThreads, 0, s>>>(p);
      else ht_combine_recv_kernel<EPB_F32, EPB_BF16><<<grid, kHTThreads, 0, s>>>(p);
    } else {
      if (a->out_dtype == EPB_F32) ht_combine_recv_kernel<EPB_BF16, EPB_F32><<<grid, kHTThreads, 0, s>>>(p);
      else ht_combine_recv_kernel<EPB_BF16, EPB_BF16><<<grid, kHTThreads, 0, s>>>(p);
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
