/*
 * epb200 — B200-native expert-parallel dispatch/combine (C ABI).
 *
 * Drop-in replacement for the engine/fabric layer of the reference simulator
 * `epsim` (arxiv 2603.13606, NCCL EP).  The reference's Python API layer
 * (pkg/src/epsim/api.py) maps onto these entry points one-to-one:
 *
 *   reference                                   | here
 *   --------------------------------------------+-------------------------------
 *   ll_regions / ht_regions (ll.py:107, ht.py:167)| epb_window_geometry
 *   Fabric.register_window (fabric.py:120)       | epb_group_create
 *   _Rendezvous.exchange (api.py:82-94)          | epb_group_ipc_desc + epb_group_open_peers
 *                                                |  (descriptors all-gathered by the host)
 *   per-token routing loops (ll.py:255-259,      | epb_routing_layout            (K1)
 *     292-296; ht.py:299-307; api.py:150-170)    |
 *   LLRank.dispatch send (ll.py:227-308)         | epb_ll_dispatch phase SEND    (K2)
 *   LLRank.complete_dispatch (ll.py:310-400)     | epb_ll_dispatch phase RECV    (K3)
 *   LLRank.combine (ll.py:404-462)               | epb_ll_combine phase SEND     (K4a)
 *   LLRank.complete_combine (ll.py:464-507)      | epb_ll_combine phase RECV     (K4b)
 *   HTRank.exchange_metadata (ht.py:291-331)     | epb_ht_meta_send / _recv      (K5a)
 *   HTRank.open_round (ht.py:335-368)            | epb_ht_open (K1 + K5a, one launch)
 *   HTRank.dispatch + _assemble (ht.py:381-583)  | epb_ht_dispatch               (K5b)
 *   HTRank.combine (ht.py:587-735)               | epb_ht_combine                (K6)
 *   quantize_block / dequantize_block            | epb_fp8_quantize / _dequantize (K7)
 *     (core.py:127-162)                          |
 *   fabric.shutdown / wait timeout               | epb_group_poll_error (device error word)
 *
 * Conventions
 *  - Every function returns 0 on success or an epb_status code whose order
 *    follows epsim.core.ErrorCode (core.py:21-28); epb_last_error() gives the
 *    detail string of the last failure on the calling thread.
 *  - All tensor pointers are DEVICE pointers; calls are asynchronous on the
 *    given stream (a cudaStream_t passed as void*).  The library never frees
 *    caller memory.
 *  - send/recv halves are separate launches so that N ranks emulated on ONE
 *    GPU never run two kernels that wait on each other: all ranks' sends are
 *    enqueued before any rank's recv.  With one process per GPU the recv
 *    half spins (acquire loads, bounded by a timeout) on flags the peers'
 *    send kernels store over NVLink.
 *  - Sequence tags replace the reference's counter resets (ll.py:351-353):
 *    every flag carries the round's tag, so double-buffer parities are reused
 *    without a reset race.
 */
#ifndef EPB200_H
#define EPB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- status codes: 1..7 = epsim ErrorCode order (core.py:21-28) -------- */
typedef enum {
  EPB_OK = 0,
  EPB_INVALID_ARGUMENT = 1,
  EPB_SHAPE_MISMATCH = 2,
  EPB_TAG_MISMATCH = 3,
  EPB_CONFIG_MISMATCH = 4,
  EPB_CAPACITY_EXCEEDED = 5,
  EPB_HANDLE_STATE_ERROR = 6,
  EPB_TRANSPORT_CLOSED = 7,
  EPB_CUDA_ERROR = 8
} epb_status;

/* element kinds (epsim Dtype, core.py:45-56) */
enum { EPB_F32 = 0, EPB_BF16 = 1, EPB_F16 = 2, EPB_FP8 = 3 };
enum { EPB_LL = 0, EPB_HT = 1 };
enum { EPB_LAYOUT_OPTIMIZED = 0, EPB_LAYOUT_LEGACY = 1 };

/* static group geometry (epsim EpConfig, core.py:325-383) */
typedef struct epb_config {
  int32_t algorithm;        /* EPB_LL | EPB_HT */
  int32_t num_ranks;
  int32_t ranks_per_node;
  int32_t num_experts;
  int32_t top_k;
  int32_t hidden;
  int32_t max_tokens_per_rank;
  int32_t token_dtype;      /* wire dtype, EPB_F32..EPB_FP8 */
  int32_t with_scales;      /* FP8 block-128 scales on the wire */
  int32_t layout;           /* LL slot layout */
  int32_t ht_chunk_tokens;  /* kept for fingerprint parity */
  int32_t ht_fifo_depth;
  int32_t combine_dtype;    /* LL combine wire dtype; -1 = token_dtype (reference) */
  int32_t expert_out_window; /* reserve a registered expert-output region in
                               the window (HT: N*B*min(K,L) bf16 rows; LL:
                               [L][N*B] bf16 rows, bf16 combine wire); a
                               combine whose input IS that region is pulled
                               by the token's home rank over NVLink */
} epb_config;

typedef struct epb_window_info {
  uint64_t physical_bytes;  /* bytes this library needs (16-B aligned slots) */
  uint64_t logical_bytes;   /* the reference's window_bytes (footprint parity) */
  uint64_t expert_out_offset; /* HT with expert_out_window: byte offset of the
                                 expert-output region in the window */
  uint64_t expert_out_rows;   /* its capacity in rows of hidden bf16 */
  uint64_t token_in_offset;   /* HT: byte offset of the token stage (this rank's
                                 rows in the wire dtype, read by the peers);
                                 a dispatch whose TOKENS input IS this region
                                 skips the stage copy (zero-copy input) */
  uint64_t token_in_rows;     /* its capacity in rows (max_tokens_per_rank); 0 for LL */
} epb_window_info;

/* per-handle routing layout; caller-owned device buffers (K1 outputs) */
typedef struct epb_layout {
  int32_t* expert_count;    /* [E]    m(e, self)                       */
  int32_t* rank_count;      /* [N]    q(self, d): tokens touching d    */
  int32_t* tok_rank;        /* [b*K]  rank of t among tokens -> e_tk    */
  int32_t* tok_slot;        /* [b*N]  dedup slot of t at rank d, or -1  */
  int32_t num_tokens;       /* b */
} epb_layout;

/* IPC descriptor exchanged by the host bootstrap (NCCL/gloo all-gather) */
typedef struct epb_ipc_desc {
  uint8_t handle[64];       /* cudaIpcMemHandle_t of the allocation     */
  uint64_t offset;          /* window offset inside that allocation     */
  uint64_t bytes;
  int32_t device;
  int32_t pid;
} epb_ipc_desc;

typedef struct epb_group epb_group;

int epb_version(void);
const char* epb_last_error(void);

int epb_window_geometry(const epb_config* cfg, epb_window_info* out);

/* window: device pointer of >= physical_bytes, or NULL to let the library
 * cudaMalloc it.  The window is zeroed on `stream`. */
int epb_group_create(const epb_config* cfg, int rank, void* window,
                     uint64_t window_bytes, void* stream, epb_group** out);
int epb_group_window(epb_group* g, void** window, uint64_t* bytes);
int epb_group_ipc_desc(epb_group* g, epb_ipc_desc* out);
/* process mode: open every peer's window through CUDA IPC */
int epb_group_open_peers(epb_group* g, const epb_ipc_desc* descs);
/* single-process emulation: peer windows are plain device pointers */
int epb_group_set_peers(epb_group* g, const uint64_t* peer_windows);
int epb_group_set_timeout(epb_group* g, uint64_t timeout_ns);
/* diagnostics: with a device buffer of >= grid*16 u64, LL kernels stamp
 * %globaltimer at phase checkpoints (thread 0 of each CTA); NULL disables */
int epb_group_set_trace(epb_group* g, uint64_t* trace);
/* device-side barrier over the peer windows (graph-capturable; one tiny
 * kernel: store epoch to every peer, wait for every peer's epoch) */
int epb_group_barrier(epb_group* g, void* stream);
/* reads (and with clear!=0 resets) the device error word; synchronises */
int epb_group_poll_error(epb_group* g, int clear, int32_t* code);
/* Op trace (the reference fabric's trace sink, fabric.py:83-111,186-201):
 * with a ring set, every transport kernel appends one record per window
 * transfer — a row record or count row stored into a peer's window (put), a
 * row read from a peer's window by a pulled transport (get), an arrival
 * counter add or flag store (signal).  ring: device memory of 4 + 4 *
 * capacity u64; ring[0] counts appended records (records past `capacity`
 * are dropped, the count still grows); record i = ring[4 + 4i ..]:
 *   w0 = op (1 put, 2 signal, 3 get) | window << 4 | src << 8 | dst << 20
 *        | signal_id << 32;  w1 = byte offset in dst's window;
 *   w2 = length in bytes;  w3 = signal value.
 * src is the initiating rank, dst the rank whose window is addressed.
 * Signal ids: LL dispatch arrivals parity*N + src, LL combine arrivals
 * 2N + parity*N + src; HT metadata flags parity*N + src, HT dispatch flags
 * 2N + src, HT combine flags 3N + src.  NULL ring: tracing off. */
int epb_group_set_op_trace(epb_group* g, uint64_t* ring, uint32_t capacity);
/* Host address of a pinned mirror of the error word: the kernel recording
 * a failure also writes its code there, so after synchronising the group's
 * streams a zero read means no failure was recorded (a nonzero one is
 * confirmed and cleared with epb_group_poll_error).  Valid until destroy. */
int epb_group_error_word(epb_group* g, const int32_t** host_word);
int epb_group_destroy(epb_group* g);

/* K1: validation + counts + dedup slots + per-expert ranks */
int epb_routing_layout(epb_group* g, const int64_t* topk_idx, int32_t b,
                       const epb_layout* lay, void* stream);

/* LL rounds are sequenced ON THE DEVICE (graph-replayable): the send phase
 * of a dispatch reads the group's round counter, stores it into *hseq (a
 * caller-owned device u32 per handle) and advances the counter; every later
 * launch of the round takes the same hseq.  Parity = seq & 1 (ll.py:250).
 *
 * phases: EPB_PHASE_SEND (1), EPB_PHASE_RECV (2) or both (3, one
 * cooperative launch; only valid when the peers run on other GPUs or N=1). */
enum { EPB_PHASE_SEND = 1, EPB_PHASE_RECV = 2, EPB_PHASE_BOTH = 3 };

typedef struct epb_ll_dispatch_args {
  const void* x;            /* send: [b, H] tokens, x_dtype (FP8 = codes)   */
  int32_t x_dtype;          /*   converted to the wire dtype in-kernel       */
  const float* x_scales;    /*   [b, H/128] for scaled FP8 input, else NULL  */
  const int64_t* topk_idx;  /*   [b, K]; validated + laid out in-kernel      */
  int32_t num_tokens;       /* b */
  void* out;                /* recv: [L, N*B, H] in out_dtype (F32 = the     */
  int32_t out_dtype;        /*   reference boundary, or the wire dtype)      */
  float* out_scales;        /*   [L, N*B, H/128] with a scaled FP8 wire      */
  float* counts_f32;        /*   [L, N] RECV_EXPERT_COUNTER                  */
  int32_t* counts_i32;      /*   [L, N] (combine input)                      */
  int32_t* src_info;        /*   [L, N*B] = t*K + k of each valid row        */
  int32_t* self_row;        /* send: [b, K] output row of (t, k) when e_tk is
                               this rank's own expert (placed directly, no
                               window hop), else -1; combine input           */
  int32_t* owner_row;       /* send, nullable: [b, K] row of (t, k) in the
                               dispatch output of e_tk's owner (pulled
                               combine input)                                */
} epb_ll_dispatch_args;

/* K2 + K3: LL dispatch (ll.py:227-400) */
int epb_ll_dispatch(epb_group* g, uint32_t* hseq, int32_t phases,
                    const epb_ll_dispatch_args* args, void* stream);

typedef struct epb_ll_combine_args {
  const void* expert_out;   /* send: [L, N*B, H] f32|bf16                    */
  int32_t in_dtype;
  const int32_t* counts_i32;/*   from the dispatch                          */
  const int32_t* src_info;
  const float* weights;     /* recv: [b, K] f32                              */
  int32_t num_tokens;
  void* out;                /*   [b, H] f32|bf16                             */
  int32_t out_dtype;
  const int32_t* self_row;  /* [b, K] from the dispatch (own rows read in place) */
  const int64_t* topk;      /* [b, K] routing of the handle; required by the
                               legacy layout (combine slot e*B + t,
                               ll.py:433-436), unused by the optimized one  */
  const int32_t* owner_row; /* [b, K] from the dispatch (pulled combine)      */
  int32_t expert_out_in_window; /* 1: expert_out is the window's expert-output
                               region; homes pull their rows over NVLink    */
} epb_ll_combine_args;

/* K4a + K4b: LL combine (ll.py:404-507) */
int epb_ll_combine(epb_group* g, const uint32_t* hseq, int32_t phases,
                   const epb_ll_combine_args* args, void* stream);

/* K5a: HT metadata all-gather over the windows */
int epb_ht_meta_send(epb_group* g, uint32_t round, const epb_layout* lay,
                     void* stream);
/* meta_out: [N, E+N] i32 (m rows then q rows); offsets: [E, N] i32 row
 * offset of group (e, src) on owner(e); recv_total: [1] i32 */
int epb_ht_meta_recv(epb_group* g, uint32_t round, int32_t* meta_out,
                     int32_t* offsets, int32_t* recv_total, void* stream);
/* K1 + K5a in one cooperative launch (HTRank.open_round, ht.py:335-368):
 * validation + routing layout into `lay` (tok_slot required), the metadata
 * all-gather and the group offsets [E, N].  host_meta: device-accessible
 * pinned host memory of N*(E+N) + 2 i32 = the metadata rows, the receive
 * total, then the group's error word, written by the kernel (read them
 * after synchronising `stream`; a nonzero error word means the round did
 * not open: poll and clear it with epb_group_poll_error).  Requires every
 * rank's kernel to be able to run concurrently (ranks on distinct GPUs, or
 * N = 1); ranks emulated on one GPU use the separate launches. */
int epb_ht_open(epb_group* g, uint32_t round, const int64_t* topk_idx, int32_t b,
                const epb_layout* lay, int32_t* host_meta, int32_t* offsets, void* stream);
/* K5b: HT dispatch (ht.py:381-583).  phases: SEND writes one record per
 * (token, remote destination) and places rows for this rank's own experts
 * directly in `out`; RECV waits for every source and scatters record rows to
 * their sorted (expert, src, token) positions.  BOTH = the two launches back
 * to back (peers on other GPUs). */
typedef struct epb_ht_dispatch_args {
  const void* x;             /* [b, H] f32|bf16|f16 */
  int32_t x_dtype;
  const float* weights;      /* [b, K] f32 (travel with the records) */
  const int64_t* topk_idx;   /* [b, K] */
  int32_t num_tokens;
  const int32_t* rank_count; /* K1 layout: q [N]        */
  const int32_t* tok_rank;   /*            [b*K]        */
  const int32_t* tok_slot;   /*            [b*N]        */
  const int32_t* offsets;    /* epb_ht_meta_recv [E, N] */
  void* out;                 /* [recv_total, H] f32 or the wire dtype */
  int32_t out_dtype;
  int32_t* origin;           /* [recv_total, 4] = (e, src, t, k) */
  float* origin_w;           /* [recv_total] */
} epb_ht_dispatch_args;
int epb_ht_dispatch(epb_group* g, uint32_t round, int32_t phases,
                    const epb_ht_dispatch_args* args, void* stream);

/* K6: HT combine (ht.py:587-735).  SEND moves expert rows of remote tokens
 * to their home's combine slots; RECV reduces in the reference's
 * (node, k) order, reading rows of its own tokens in place. */
typedef struct epb_ht_combine_args {
  const void* expert_rows;   /* [recv_total, H] f32|bf16, dispatch order */
  int32_t in_dtype;
  const int32_t* origin;     /* from the dispatch */
  int32_t recv_total;
  const int64_t* topk_idx;   /* [b, K] */
  const float* weights;      /* [b, K] f32 */
  int32_t num_tokens;
  const int32_t* tok_rank;   /* K1 layout [b*K] */
  const int32_t* offsets;    /* [E, N] */
  void* out;                 /* [b, H] f32|bf16 */
  int32_t out_dtype;
  const float* dispatch_weights; /* [b, K] weights given at dispatch, checked
                                    against `weights` before any traffic
                                    (ht.py:605-609); NULL skips the check */
  uint64_t* row_ptr;         /* [b*K] scratch: the send phase stores the
                                address of every (t, k) expert row the
                                receive reduces (own rows in place, others in
                                the combine slots); NULL: resolved inline */
  int32_t expert_rows_in_window; /* 1: expert_rows is the window's expert-
                                    output region (bf16); the receive pulls
                                    every row from its owner over NVLink */
} epb_ht_combine_args;
int epb_ht_combine(epb_group* g, uint32_t round, int32_t phases,
                   const epb_ht_combine_args* args, void* stream);
/* device-side check that combine weights equal the dispatched ones
 * (ht.py:605-609); sets EPB_INVALID_ARGUMENT in the error word */
int epb_weights_equal(epb_group* g, const float* a, const float* b, int64_t n,
                      void* stream);

/* K7: standalone block-128 FP8 (E4M3, reference tie rule) */
int epb_fp8_quantize(const void* x, int32_t x_dtype, int64_t rows, int32_t h,
                     uint8_t* codes, float* scales, void* stream);
int epb_fp8_dequantize(const uint8_t* codes, const float* scales, int64_t rows,
                       int32_t h, float* out, void* stream);
/* elementwise E4M3 encode without scales (combine-wire form) */
int epb_e4m3_encode(const float* x, int64_t n, uint8_t* codes, void* stream);
/* generic wire conversion f32<->dtype (NDTensor read_f32/write_f32) */
int epb_convert(const void* src, int32_t src_dtype, void* dst,
                int32_t dst_dtype, int64_t n, void* stream);
/* sets *flag (device int32) to 1 if any element is non-finite
 * (quantize_block's InvalidArgument check, core.py:143-144) */
int epb_check_finite(const float* x, int64_t n, int32_t* flag, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* EPB200_H */
