// Physical window geometry (host + device).
//
// The reference sizes one window per rank (ll.py:107-121, ht.py:167-174).
// Here each payload slot is padded to 16-byte multiples so every row moves
// with 16-B vector stores / bulk copies; `logical_bytes` keeps the
// reference's number for footprint/buffer-report parity (layout.py:164-194).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/epb200.h"

namespace epb {

constexpr int kMaxRanksHost = 64;
// LL kernels run a rank-independent grid (default one 512-thread CTA per
// B200 SM, co-resident for the cooperative fused launch; EPB_LL_CTAS picks a
// smaller one so LL can share the GPU with compute) — every rank must use
// the same value: a receiver expects one arrival per source CTA
constexpr int kLLGrid = 148;

inline size_t a16(size_t x) { return (x + 15) / 16 * 16; }
inline size_t a256(size_t x) { return (x + 255) / 256 * 256; }
inline int width_of(int dt) { return dt == EPB_F32 ? 4 : (dt == EPB_FP8 ? 1 : 2); }

// LL, per parity:
//   [count rows: N src x (L+1) u32]   row src = m of each of this rank's local
//                                     experts from src, then q (slots from src)
//   [dispatch arrivals: N src u64][combine arrivals: N src u64]
//   [disp slots: n_disp x slot_stride]                      (256-aligned)
//   [comb slots: n_comb x comb_stride]
// slot = [row RBp][scales SBp][hdr: t, kcount, K ids, K ranks (HBp)]
// Arrivals are cumulative: every CTA of a source adds 1 per round after a
// release, so round seq on parity seq&1 is complete at grid*((seq>>1)+1).
struct LLGeom {
  int N, E, L, K, H, B, wire, cwire, scales, layout;
  int RB, RBp, SB, SBp, HB, HBp, CB;
  int slot_stride, comb_stride;
  int64_t n_disp, n_comb;
  uint64_t cnt_row, d_arr, c_arr, disp_slot, comb_slot;  // offsets within a parity
  int grid;  // CTAs of every LL launch (the same on every rank: receivers expect `grid` arrivals)
  uint64_t Lmagic;  // ceil(2^32 / L): owner rank e / L = (e * Lmagic) >> 32 (exact for e * L < 2^32)
  uint64_t Kmagic;  // ceil(2^32 / K): token of a routing item i / K (i * K < 2^32)
  uint64_t parity_bytes, window_bytes, logical_bytes;
  uint64_t barrier;  // [N] u64 device-barrier flags (after both parities)
  uint64_t yout, yout_rows, yrow;  // registered expert-output region [L][N*B] bf16 rows (expert_out_window)
  int sys_fence;                   // release fences at system scope (peers on other GPUs)
  uint32_t chaos_ns;               // stress mode: random delays before stores / releases (EPB_CHAOS_NS)
  int direct_max;                  // ll_arrive: per-CTA arrivals up to this many storing CTAs (EPB_LL_DIRECT)
};

// HT:
//   [meta rows: 2 x N x (E+N) u32][meta flags: 2 x N u64]
//   [dispatch flags: N u64][combine flags: N u64]
//   [stage: B x RBp]  this rank's token rows in the wire dtype; receivers
//                     pull the rows they need from it over NVLink
//   [records: N x B x rec_stride]   rec = [w: K f32][hdr + pos]
//   [combine rows: B x K x crow_stride]  (f32 capacity: 4H)
struct HTGeom {
  int N, E, L, K, H, B, rpn, wire;
  int RB, RBp, WBp, HBp, rec_stride, crow_stride;
  uint64_t meta, meta_flag, dflag, cflag, stage, rec, crow;
  uint64_t yout, yout_rows, yrow;  // registered expert-output region (expert_out_window)
  int sys_fence;                   // release fences at system scope (peers on other GPUs)
  uint32_t chaos_ns;               // stress mode: random delays before stores / releases (EPB_CHAOS_NS)
  uint64_t window_bytes, logical_bytes;
  uint64_t barrier;  // [N] u64 device-barrier flags
};

inline int experts_per_rank(int e, int n) { return (e + n - 1) / n; }

constexpr int kLayChunk = 128;  // tokens per CTA of the multi-CTA routing layout (K1)

inline void make_ll_geom(const epb_config& c, LLGeom& g) {
  g.N = c.num_ranks; g.E = c.num_experts; g.L = experts_per_rank(c.num_experts, c.num_ranks);
  g.K = c.top_k; g.H = c.hidden; g.B = c.max_tokens_per_rank; g.wire = c.token_dtype;
  g.scales = c.with_scales; g.layout = c.layout;
  g.cwire = c.combine_dtype < 0 ? c.token_dtype : c.combine_dtype;
  g.CB = c.hidden * width_of(g.cwire);
  g.RB = c.hidden * width_of(c.token_dtype);
  g.RBp = (int)a16(g.RB);
  g.SB = c.with_scales ? (c.hidden / 128) * 4 : 0;
  g.SBp = (int)a16(g.SB);
  g.HB = 8 + 4 * c.top_k;
  g.HBp = (int)a16(g.HB + 4 * c.top_k);
  g.slot_stride = g.RBp + g.SBp + g.HBp;
  g.Lmagic = ((1ull << 32) + (uint64_t)g.L - 1) / (uint64_t)g.L;
  g.Kmagic = ((1ull << 32) + (uint64_t)g.K - 1) / (uint64_t)g.K;
  g.comb_stride = (int)a16(g.CB);
  const int64_t pairs = (int64_t)g.L * g.N;
  if (c.layout == EPB_LAYOUT_LEGACY) {
    g.n_disp = pairs * g.B;
    g.n_comb = (int64_t)g.E * g.B;
  } else {
    g.n_disp = (int64_t)g.N * g.B;
    g.n_comb = (int64_t)g.B * g.K;
  }
  g.grid = kLLGrid;
  g.cnt_row = 0;
  g.d_arr = a16((uint64_t)g.N * (g.L + 1) * 4);
  g.c_arr = g.d_arr + (uint64_t)g.N * 8;
  g.disp_slot = a256(g.c_arr + (uint64_t)g.N * 8);
  g.comb_slot = a256(g.disp_slot + (uint64_t)g.n_disp * g.slot_stride);
  g.parity_bytes = a256(g.comb_slot + (uint64_t)g.n_comb * g.comb_stride);
  g.yrow = a16(2 * (uint64_t)c.hidden);
  g.yout_rows = c.expert_out_window ? (uint64_t)g.L * g.N * g.B : 0;
  g.yout = 2 * g.parity_bytes;
  g.barrier = a256(g.yout + g.yout_rows * g.yrow);
  g.window_bytes = a256(g.barrier + (uint64_t)g.N * 8);
  // reference ll_regions (ll.py:58-121)
  const uint64_t ref_slot = (uint64_t)(g.HB + g.RB + g.SB);
  const uint64_t ref_parity = pairs * 8 + (uint64_t)g.E * 8 + g.n_disp * ref_slot +
                              g.n_comb * (uint64_t)g.CB;
  g.logical_bytes = 2 * ref_parity;
}

inline void make_ht_geom(const epb_config& c, HTGeom& g) {
  g.N = c.num_ranks; g.E = c.num_experts; g.L = experts_per_rank(c.num_experts, c.num_ranks);
  g.K = c.top_k; g.H = c.hidden; g.B = c.max_tokens_per_rank; g.rpn = c.ranks_per_node;
  g.wire = c.token_dtype;
  g.RB = c.hidden * width_of(c.token_dtype);
  g.RBp = (int)a16(g.RB);
  g.WBp = (int)a16(4 * c.top_k);
  g.HBp = (int)a16(8 + 8 * c.top_k);
  g.rec_stride = g.WBp + g.HBp;  // record = weights + header/positions; the row stays in `stage`
  g.crow_stride = (int)a16(4 * (size_t)c.hidden);
  g.meta = 0;
  g.meta_flag = a256((uint64_t)2 * g.N * (g.E + g.N) * 4);
  g.dflag = g.meta_flag + 2 * g.N * 8;
  g.cflag = g.dflag + g.N * 8;
  g.stage = a256(g.cflag + g.N * 8);
  g.rec = a256(g.stage + (uint64_t)g.B * g.RBp);
  g.crow = a256(g.rec + (uint64_t)g.N * g.B * g.rec_stride);
  g.yrow = a16(2 * (uint64_t)c.hidden);
  g.yout_rows = c.expert_out_window ? (uint64_t)g.N * g.B * (uint64_t)std::min(g.K, g.L) : 0;
  g.yout = a256(g.crow + (uint64_t)g.B * g.K * g.crow_stride);
  g.barrier = a256(g.yout + g.yout_rows * g.yrow);
  g.window_bytes = a256(g.barrier + (uint64_t)g.N * 8);
  // reference ht_regions (ht.py:78-174)
  const int nodes = c.num_ranks / c.ranks_per_node;
  const uint64_t record = 8 + 4 * c.top_k + 4 * c.top_k + (uint64_t)g.RB +
                          (c.with_scales ? (c.hidden / 128) * 4 : 0);
  const uint64_t chunk = 8 + (uint64_t)c.ht_chunk_tokens * record;
  uint64_t b = 2ull * g.N * (g.E + g.N) * 4;
  b += (uint64_t)g.N * 8;
  b += (uint64_t)g.N * g.B * record;
  b += (uint64_t)(nodes - 1) * c.ht_fifo_depth * chunk;
  b += (uint64_t)c.ranks_per_node * nodes * 8;
  b += (uint64_t)nodes * g.B * g.K * (4 + 4 * (uint64_t)c.hidden);
  b += (uint64_t)nodes * g.B * 4 * (uint64_t)c.hidden;
  g.logical_bytes = b;
}

}  // namespace epb
