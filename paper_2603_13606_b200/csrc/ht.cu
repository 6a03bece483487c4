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
struct HTSend {
  const void* x;
  const float* w;
  const int64_t* topk;
  const int32_t* q;
  const int32_t* tok_rank;
  const int32_t* tok_slot;
  const int32_t* offsets;  // [E, N]
  const uint64_t* peers;
  void* out;               // own sorted output (self rows land here directly)
  int32_t* origin;
  float* origin_w;
  int* done;
  HTGeom g;
  int b, rank;
  uint32_t tag;
};

EPB_DEV void ht_publish_records(const HTSend& p, int d) {
  uint64_t* flag = reinterpret_cast<uint64_t*>(hpeer(p.peers, d) + p.g.dflag) + p.rank;
  st_relaxed_sys_u64(flag, ((uint64_t)p.tag << 32) | (uint32_t)p.q[d]);
}

template <int XT, int WT, int OT>
__global__ void __launch_bounds__(kHTThreads) ht_dispatch_send_kernel(HTSend p) {
  // a CTA owns tokens blockIdx.x + i*gridDim.x; their routing metadata is
  // gathered for kTB tokens at once (one latency for the batch), then rows
  // move token by token
  constexpr int kTB = 16;
  __shared__ int s_e[kTB][kMaxTopK], s_pos[kTB][kMaxTopK];
  __shared__ float s_w[kTB][kMaxTopK];
  __shared__ int s_j[kTB][kMaxRanks];
  __shared__ int s_cnt[kMaxRanks];
  const HTGeom& g = p.g;
  const int K = g.K, N = g.N, H = g.H, L = g.L, G = gridDim.x;
  const int me = p.rank;
  constexpr int EPC = Elems<WT>::n;
  constexpr int XW = XT == EPB_F32 ? 4 : 2;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  const int64_t rec0 = (int64_t)me * g.B;
  if ((int)threadIdx.x < N) s_cnt[threadIdx.x] = 0;
  for (int base = blockIdx.x; base < p.b; base += G * kTB) {
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
      int j = -1;
      if (t < p.b && d != me) j = p.tok_slot[(int64_t)t * N + d];
      s_j[i][d] = j;
    }
    __syncthreads();
    if ((int)threadIdx.x < N)
      for (int i = 0; i < kTB; ++i) s_cnt[threadIdx.x] += s_j[i][threadIdx.x] >= 0;
    for (int i = 0; i < kTB; ++i) {
      const int t = base + i * G;
      if (t >= p.b) break;
      // record header (reference fields + output positions) and weights
      const int words = K + 2 + 2 * K;
      for (int idx = threadIdx.x; idx < N * words; idx += blockDim.x) {
        const int d = idx / words, wd = idx - d * words;
        if (s_j[i][d] < 0) continue;
        uint8_t* rec = hpeer(p.peers, d) + g.rec + (rec0 + s_j[i][d]) * g.rec_stride;
        if (wd < K) {
          reinterpret_cast<float*>(rec + g.RBp)[wd] = s_w[i][wd];
        } else {
          const int h = wd - K;
          const uint32_t v = h == 0 ? (uint32_t)t : h == 1 ? (uint32_t)K
                             : h < 2 + K ? (uint32_t)s_e[i][h - 2] : (uint32_t)s_pos[i][h - 2 - K];
          reinterpret_cast<uint32_t*>(rec + g.RBp + g.WBp)[h] = v;
        }
      }
      const uint8_t* xrow = reinterpret_cast<const uint8_t*>(p.x) + (int64_t)t * H * XW;
      if ((H & 15) == 0) {
        for (int c = threadIdx.x; c < H / EPC; c += blockDim.x) {
          float f[EPC];
          load_elems_vec<XT, EPC>(xrow, (int64_t)c * EPC, f);
          const int4 v = pack16<WT>(f);
          for (int d = 0; d < N; ++d) {
            const int j = s_j[i][d];
            if (j >= 0) st_na_v4(hpeer(p.peers, d) + g.rec + (rec0 + j) * g.rec_stride + (int64_t)c * 16, v);
          }
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
          for (int d = 0; d < N; ++d) {
            const int j = s_j[i][d];
            if (j >= 0) store_elem(hpeer(p.peers, d) + g.rec + (rec0 + j) * g.rec_stride, WT, el, f);
          }
          const float fw = WT == EPB_F32 ? f : (WT == EPB_BF16 ? bf16_widen(bf16_bits_rne(f)) : f16_widen(f16_bits_rne(f)));
          for (int k = 0; k < K; ++k)
            if (s_e[i][k] / L == me)
              store_elem(reinterpret_cast<uint8_t*>(p.out) + (int64_t)s_pos[i][k] * H * OW, OT, el, fw);
        }
      }
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < N && (int)threadIdx.x != me) {
    const int d = threadIdx.x;
    const int c = s_cnt[d];
    if (c > 0) {
      fence_sys();
      const int old = atomicAdd(&p.done[d], c);
      if (old + c == p.q[d]) {
        p.done[d] = 0;
        fence_sys();
        ht_publish_records(p, d);
      }
    } else if (blockIdx.x == 0 && p.q[d] == 0) {
      ht_publish_records(p, d);
    }
  }
}

struct HTRecv {
  void* out;
  int32_t* origin;
  float* origin_w;
  const uint8_t* win;
  int* err;
  HTGeom g;
  uint64_t timeout_ns;
  int rank;
  uint32_t tag;
};

template <int WT, int OT>
__global__ void __launch_bounds__(kHTThreads) ht_dispatch_recv_kernel(HTRecv p) {
  __shared__ int s_pre[kMaxRanks + 1], s_q[kMaxRanks];
  __shared__ int s_fail;
  const HTGeom& g = p.g;
  const int N = g.N, K = g.K, H = g.H, L = g.L;
  const int me = p.rank;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(p.win + g.dflag);
  for (int s = threadIdx.x; s < N; s += blockDim.x) {
    uint64_t v = 0;
    if (s != me && !wait_tag(&flags[s], p.tag, 32, 0xFFFFFFFFu, p.timeout_ns, p.err, &v)) s_fail = 1;
    s_q[s] = s == me ? 0 : (int)(v & 0xFFFFFFFFu);  // own rows were placed by the sender
  }
  __syncthreads();
  if (s_fail) return;
  if (threadIdx.x == 0) {
    int run = 0;
    for (int s = 0; s < N; ++s) { s_pre[s] = run; run += s_q[s]; }
    s_pre[N] = run;
  }
  __syncthreads();
  const int items = s_pre[N] * K;  // (record, k); non-local k exit at once
  const int lo = me * L, hi = min(lo + L, g.E);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int OW = OT == EPB_F32 ? 4 : 2;
  constexpr int EPC = Elems<WT>::n;
  for (int f = warp * gridDim.x + blockIdx.x; f < items; f += gridDim.x * nw) {
    const int rj = f / K, k = f - rj * K;
    int s = 0;
    while (s_pre[s + 1] <= rj) ++s;
    const int j = rj - s_pre[s];
    const uint8_t* rec = p.win + g.rec + ((int64_t)s * g.B + j) * g.rec_stride;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(rec + g.RBp + g.WBp);
    const int e = (int)hdr[2 + k];
    if (e < lo || e >= hi) continue;
    const int64_t pos = hdr[2 + K + k];
    if (lane == 0) {
      p.origin[pos * 4 + 0] = e;
      p.origin[pos * 4 + 1] = s;
      p.origin[pos * 4 + 2] = (int32_t)hdr[0];
      p.origin[pos * 4 + 3] = k;
      p.origin_w[pos] = reinterpret_cast<const float*>(rec + g.RBp)[k];
    }
    uint8_t* orow = reinterpret_cast<uint8_t*>(p.out) + pos * H * OW;
    if ((H & 15) == 0) {
      const int nch = H / EPC;
      for (int base = 0; base < nch; base += 32 * kHU) {
        int4 v[kHU];
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int c = base + u * 32 + lane;
          if (c < nch) v[u] = ld_plain_v4(rec + (int64_t)c * 16);
        }
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int c = base + u * 32 + lane;
          if (c < nch) {
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
    } else {
      for (int el = lane; el < H; el += 32) store_elem(orow, OT, el, load_elem(rec, WT, el));
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

template <int XT, int WT, int OT>
cudaError_t launch_hsend(const HTSend& p, cudaStream_t s) {
  const int grid = std::max(1, std::min(p.b, 2 * hsm_count()));
  ht_dispatch_send_kernel<XT, WT, OT><<<grid, kHTThreads, 0, s>>>(p);
  return cudaGetLastError();
}

template <int XT, int WT>
cudaError_t launch_hsend_o(const HTSend& p, int out_dtype, cudaStream_t s) {
  return out_dtype == EPB_F32 ? launch_hsend<XT, WT, EPB_F32>(p, s) : launch_hsend<XT, WT, WT>(p, s);
}

template <int XT>
cudaError_t launch_hsend_x(const HTSend& p, int out_dtype, cudaStream_t s) {
  switch (p.g.wire) {
    case EPB_F32: return launch_hsend<XT, EPB_F32, EPB_F32>(p, s);
    case EPB_BF16: return launch_hsend_o<XT, EPB_BF16>(p, out_dtype, s);
    default: return launch_hsend_o<XT, EPB_F16>(p, out_dtype, s);
  }
}

template <int WT, int OT>
cudaError_t launch_hrecv(const HTRecv& p, cudaStream_t s) {
  ht_dispatch_recv_kernel<WT, OT><<<2 * hsm_count(), kHTThreads, 0, s>>>(p);
  return cudaGetLastError();
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
  cudaStream_t s = as_stream(stream);
  if (phases & 1) {
    if (a->num_tokens > 0 && !a16(a->x)) return fail(EPB_INVALID_ARGUMENT, "x must be 16-byte aligned");
    HTSend p;
    p.x = a->x; p.w = a->weights; p.topk = a->topk_idx; p.q = a->rank_count; p.tok_rank = a->tok_rank;
    p.tok_slot = a->tok_slot; p.offsets = a->offsets; p.peers = g->d_peers; p.out = a->out;
    p.origin = a->origin; p.origin_w = a->origin_w; p.done = g->d_done; p.g = g->ht;
    p.b = a->num_tokens; p.rank = g->rank; p.tag = ht_tag(round);
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
    p.out = a->out; p.origin = a->origin; p.origin_w = a->origin_w; p.win = g->window; p.err = g->d_err;
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
