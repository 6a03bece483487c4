// Group lifecycle: window allocation, CUDA-IPC peer mapping, error word.
// Replaces epsim's Fabric.register_window + _Rendezvous (fabric.py:120-132,
// api.py:67-94, 256-319): the host all-gathers epb_ipc_desc records (over a
// torch.distributed group) and every rank maps every peer window once.
#include <cuda.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>

#include <string>

#include "common.cuh"
#include "internal.h"

namespace epb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(EPB_CUDA_ERROR, m);
}

static int validate_config(const epb_config* c) {
  if (!c) return fail(EPB_INVALID_ARGUMENT, "null config");
  if (c->num_ranks < 1 || c->num_ranks > kMaxRanksHost)
    return fail(EPB_INVALID_ARGUMENT, "num_ranks outside [1, 64]");
  if (c->top_k < 1 || c->top_k > c->num_experts || c->top_k > 32)
    return fail(EPB_INVALID_ARGUMENT, "top_k outside [1, min(E, 32)]");
  if (c->ranks_per_node < 1 || c->num_ranks % c->ranks_per_node)
    return fail(EPB_INVALID_ARGUMENT, "ranks_per_node must divide num_ranks");
  if (c->num_experts < c->num_ranks) return fail(EPB_INVALID_ARGUMENT, "num_experts < num_ranks");
  if (c->hidden < 1 || c->max_tokens_per_rank < 1)
    return fail(EPB_INVALID_ARGUMENT, "hidden / max_tokens_per_rank < 1");
  if (c->max_tokens_per_rank >= (1 << 20))
    return fail(EPB_INVALID_ARGUMENT, "max_tokens_per_rank must be < 2^20");
  if (c->token_dtype < EPB_F32 || c->token_dtype > EPB_FP8)
    return fail(EPB_INVALID_ARGUMENT, "token_dtype");
  if (c->with_scales && (c->token_dtype != EPB_FP8 || c->hidden % 128))
    return fail(EPB_INVALID_ARGUMENT, "with_scales requires fp8 and hidden % 128 == 0");
  if (c->algorithm == EPB_HT && c->token_dtype == EPB_FP8)
    return fail(EPB_INVALID_ARGUMENT, "fp8 token dtype is not supported by the HT algorithm");
  if (c->algorithm != EPB_LL && c->algorithm != EPB_HT)
    return fail(EPB_INVALID_ARGUMENT, "algorithm");
  if (c->combine_dtype < -1 || c->combine_dtype > EPB_FP8)
    return fail(EPB_INVALID_ARGUMENT, "combine_dtype");
  if (c->layout != EPB_LAYOUT_OPTIMIZED && c->layout != EPB_LAYOUT_LEGACY)
    return fail(EPB_INVALID_ARGUMENT, "layout");
  if (c->expert_out_window && c->hidden % 8)
    return fail(EPB_INVALID_ARGUMENT, "expert_out_window needs hidden % 8 == 0");
  if (c->expert_out_window && c->algorithm == EPB_LL &&
      (c->combine_dtype < 0 ? c->token_dtype : c->combine_dtype) != EPB_BF16)
    return fail(EPB_INVALID_ARGUMENT, "LL expert_out_window needs a bf16 combine wire");
  return EPB_OK;
}

// Device-side barrier over the peer windows: every rank stores the epoch in
// slot [rank] of every peer's barrier array, then waits until all N slots of
// its own array show it.  Used to align ranks outside timed regions and as a
// graph-capturable alternative to a host barrier.
__global__ void group_barrier_kernel(const uint64_t* peers, uint64_t off, int n, int rank, uint32_t* epoch_ctr,
                                     int* err, uint64_t timeout_ns, int sys) {
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(epoch_ctr) + 1;
    *epoch_ctr = s_epoch;
  }
  __syncthreads();
  const uint32_t ep = s_epoch;
  if ((int)threadIdx.x < n) {
    uint64_t* slot = reinterpret_cast<uint64_t*>(peers[threadIdx.x] + off) + rank;
    if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"((uint64_t)ep) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(slot), "l"((uint64_t)ep) : "memory");
    const uint64_t* mine = reinterpret_cast<const uint64_t*>(peers[rank] + off) + threadIdx.x;
    uint64_t v;
    wait_tag(mine, ep, 0, 0xFFFFFFFFu, timeout_ns, err, &v);
  }
}

}  // namespace epb

using namespace epb;

extern "C" {

int epb_group_barrier(epb_group* g, void* stream) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (!g->peers_ready) return fail(EPB_HANDLE_STATE_ERROR, "peer windows not mapped");
  const uint64_t off = g->cfg.algorithm == EPB_LL ? g->ll.barrier : g->ht.barrier;
  group_barrier_kernel<<<1, 64, 0, as_stream(stream)>>>(g->d_peers, off, g->cfg.num_ranks, g->rank,
                                                         reinterpret_cast<uint32_t*>(g->d_scratch) + 2, g->d_err,
                                                         g->timeout_ns, g->sys_scope ? 1 : 0);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}


int epb_version(void) { return 1; }

const char* epb_last_error(void) { return g_last_error.c_str(); }

int epb_window_geometry(const epb_config* cfg, epb_window_info* out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  out->expert_out_offset = 0;
  out->expert_out_rows = 0;
  out->token_in_offset = 0;
  out->token_in_rows = 0;
  if (cfg->algorithm == EPB_LL) {
    LLGeom g;
    make_ll_geom(*cfg, g);
    out->physical_bytes = g.window_bytes;
    out->logical_bytes = g.logical_bytes;
    out->expert_out_offset = g.yout;
    out->expert_out_rows = g.yout_rows;
  } else {
    HTGeom g;
    make_ht_geom(*cfg, g);
    out->physical_bytes = g.window_bytes;
    out->logical_bytes = g.logical_bytes;
    out->expert_out_offset = g.yout;
    out->expert_out_rows = g.yout_rows;
    out->token_in_offset = g.stage;
    out->token_in_rows = (uint64_t)g.B;
  }
  return EPB_OK;
}

int epb_group_create(const epb_config* cfg, int rank, void* window, uint64_t window_bytes,
                     void* stream, epb_group** out) {
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (rank < 0 || rank >= cfg->num_ranks) return fail(EPB_INVALID_ARGUMENT, "rank out of range");
  epb_group* g = new epb_group();
  g->cfg = *cfg;
  g->rank = rank;
  make_ll_geom(*cfg, g->ll);
  make_ht_geom(*cfg, g->ht);
  // release fences: system scope whenever a peer window lives on another GPU
  // (epb_group_open_peers); GPU scope only while every rank is on this GPU.
  // EPB_SYS_FENCE=1 forces system scope everywhere; EPB_SYS_FENCE=0 forces
  // GPU scope even across GPUs (outside the PTX memory model: measurement only)
  {
    const char* f = getenv("EPB_SYS_FENCE");
    g->fence_override = f ? (atoi(f) != 0 ? 1 : 0) : -1;
    g->ll.sys_fence = g->ht.sys_fence = g->fence_override == 1 ? 1 : 0;
  }
  g->ll.chaos_ns = g->ht.chaos_ns = 0;
  if (const char* c = getenv("EPB_CHAOS_NS")) g->ll.chaos_ns = g->ht.chaos_ns = (uint32_t)strtoul(c, nullptr, 10);
  g->ll.direct_max = 0;  // last-CTA publish at every batch size (direct arrivals measured no faster)
  if (const char* c = getenv("EPB_LL_DIRECT")) g->ll.direct_max = atoi(c);
  // LL grid (identical on every rank: receivers count one arrival per
  // source CTA); EPB_LL_CTAS < 148 leaves SMs free for concurrent compute
  if (const char* c = getenv("EPB_LL_CTAS")) {
    const int v = atoi(c);
    if (v >= 1 && v <= kLLGrid) g->ll.grid = v;
  }
  const uint64_t need = cfg->algorithm == EPB_LL ? g->ll.window_bytes : g->ht.window_bytes;
  cudaGetDevice(&g->device);
  cudaStream_t s = as_stream(stream);
  auto cleanup = [&](int code) {
    if (g->owns_window && g->window) cudaFree(g->window);
    if (g->d_peers) cudaFree(g->d_peers);
    if (g->d_err) cudaFree(g->d_err);
    if (g->d_done) cudaFree(g->d_done);
    if (g->d_scratch) cudaFree(g->d_scratch);
    if (g->d_seq) cudaFree(g->d_seq);
    if (g->d_lay) cudaFree(g->d_lay);
    if (g->h_err) cudaFreeHost(g->h_err);
    delete g;
    return code;
  };
  if (window) {
    if (window_bytes < need)
      return cleanup(fail(EPB_CAPACITY_EXCEEDED, "window smaller than the physical geometry"));
    if (reinterpret_cast<uintptr_t>(window) % 256)
      return cleanup(fail(EPB_INVALID_ARGUMENT, "window must be 256-byte aligned"));
    g->window = reinterpret_cast<uint8_t*>(window);
    g->window_bytes = window_bytes;
  } else {
    cudaError_t e = cudaMalloc(&g->window, need);
    if (e != cudaSuccess) return cleanup(cuda_check(e, "cudaMalloc(window)"));
    g->owns_window = true;
    g->window_bytes = need;
  }
  const int n = cfg->num_ranks;
  const int l = experts_per_rank(cfg->num_experts, n);
  cudaError_t e = cudaMalloc(&g->d_peers, sizeof(uint64_t) * n);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_err, sizeof(int) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_done, sizeof(int) * 4 * n);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_scratch, sizeof(int) * (8 * n + 2 * l * n + 64));
  if (e == cudaSuccess) e = cudaMalloc(&g->d_seq, sizeof(uint32_t) * kLLGrid);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->d_seq, 0, sizeof(uint32_t) * kLLGrid, s);
  if (e == cudaSuccess)
    e = cudaMalloc(&g->d_lay, sizeof(int) * (size_t)((cfg->max_tokens_per_rank + kLayChunk - 1) / kLayChunk) *
                                  (cfg->num_experts + n));
  if (e == cudaSuccess) e = cudaMemsetAsync(g->window, 0, g->window_bytes, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->d_err, 0, sizeof(int) * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->d_done, 0, sizeof(int) * 4 * n, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g->d_scratch, 0, sizeof(int) * (8 * n + 2 * l * n + 64), s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  // host mirror of the error word (raise_err, common.cuh): its device
  // address lives in d_err[2..3]
  if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&g->h_err), 16, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    g->h_err[0] = 0;
    void* dp = nullptr;
    e = cudaHostGetDevicePointer(&dp, g->h_err, 0);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_err + 2, &dp, sizeof(dp), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return cleanup(cuda_check(e, "group setup"));
  if (const char* t = getenv("EPB_TIMEOUT_MS")) g->timeout_ns = strtoull(t, nullptr, 10) * 1000000ull;
  // a single rank is its own peer
  if (n == 1) {
    uint64_t self = reinterpret_cast<uint64_t>(g->window);
    e = cudaMemcpy(g->d_peers, &self, sizeof(self), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cleanup(cuda_check(e, "peer table"));
    g->peers_ready = true;
  }
  *out = g;
  return EPB_OK;
}

int epb_group_window(epb_group* g, void** window, uint64_t* bytes) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  *window = g->window;
  *bytes = g->window_bytes;
  return EPB_OK;
}

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

int epb_group_ipc_desc(epb_group* g, epb_ipc_desc* out) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  memset(out, 0, sizeof(*out));
  void* base = g->window;
  if (!g->owns_window) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    EPB_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn) return fail(EPB_CUDA_ERROR, "cuMemGetAddressRange unavailable");
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (((PFN_getAddressRange)fn)(&b, &sz, reinterpret_cast<CUdeviceptr>(g->window)) != CUDA_SUCCESS)
      return fail(EPB_CUDA_ERROR, "cuMemGetAddressRange failed");
    base = reinterpret_cast<void*>(b);
  }
  g->alloc_base = base;
  cudaIpcMemHandle_t h;
  EPB_CUDA(cudaIpcGetMemHandle(&h, base));
  memcpy(out->handle, &h, sizeof(h));
  out->offset = reinterpret_cast<uint8_t*>(g->window) - reinterpret_cast<uint8_t*>(base);
  out->bytes = g->window_bytes;
  out->device = g->device;
  out->pid = (int32_t)getpid();
  return EPB_OK;
}

int epb_group_open_peers(epb_group* g, const epb_ipc_desc* descs) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  const int n = g->cfg.num_ranks;
  std::vector<uint64_t> ptrs(n);
  for (int r = 0; r < n; ++r) {
    if (r == g->rank) {
      ptrs[r] = reinterpret_cast<uint64_t>(g->window);
      continue;
    }
    if (descs[r].bytes < g->window_bytes)
      return fail(EPB_CONFIG_MISMATCH, "peer window smaller than ours");
    cudaIpcMemHandle_t h;
    memcpy(&h, descs[r].handle, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_check(e, "cudaIpcOpenMemHandle");
    g->ipc_opened.push_back(p);
    ptrs[r] = reinterpret_cast<uint64_t>(p) + descs[r].offset;
  }
  EPB_CUDA(cudaMemcpy(g->d_peers, ptrs.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice));
  g->peers_ready = true;
  g->sys_scope = true;
  g->ll.sys_fence = g->ht.sys_fence = g->fence_override == 0 ? 0 : 1;
  return EPB_OK;
}

int epb_group_set_peers(epb_group* g, const uint64_t* peer_windows) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  // one process driving several GPUs: a peer window on another device is
  // reached through peer access (UVA pointers), and ordering towards it
  // needs system-scope releases, exactly as for CUDA-IPC peers
  for (int r = 0; r < g->cfg.num_ranks; ++r) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, reinterpret_cast<const void*>(peer_windows[r])) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (at.type == cudaMemoryTypeDevice && at.device != g->device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_check(e, "cudaDeviceEnablePeerAccess");
      g->sys_scope = true;
    }
  }
  if (g->sys_scope) g->ll.sys_fence = g->ht.sys_fence = g->fence_override == 0 ? 0 : 1;
  EPB_CUDA(cudaMemcpy(g->d_peers, peer_windows, sizeof(uint64_t) * g->cfg.num_ranks,
                      cudaMemcpyHostToDevice));
  g->peers_ready = true;
  return EPB_OK;
}

int epb_group_set_trace(epb_group* g, uint64_t* trace) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  g->trace = trace;
  return EPB_OK;
}

int epb_group_set_timeout(epb_group* g, uint64_t timeout_ns) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  g->timeout_ns = timeout_ns;
  return EPB_OK;
}

int epb_group_poll_error(epb_group* g, int clear, int32_t* code) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  int v = 0;
  EPB_CUDA(cudaMemcpy(&v, g->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  *code = v;
  if (clear && v) {
    EPB_CUDA(cudaMemset(g->d_err, 0, sizeof(int)));
    reinterpret_cast<volatile int*>(g->h_err)[0] = 0;
  }
  return EPB_OK;
}

int epb_group_set_op_trace(epb_group* g, uint64_t* ring, uint32_t capacity) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  if (ring && capacity == 0) return fail(EPB_INVALID_ARGUMENT, "op trace capacity must be positive");
  g->op_ring = reinterpret_cast<unsigned long long*>(ring);
  g->op_cap = ring ? capacity : 0;
  return EPB_OK;
}

int epb_group_error_word(epb_group* g, const int32_t** host_word) {
  if (!g || !host_word) return fail(EPB_INVALID_ARGUMENT, "null argument");
  *host_word = g->h_err;
  return EPB_OK;
}

int epb_group_destroy(epb_group* g) {
  if (!g) return fail(EPB_INVALID_ARGUMENT, "null group");
  cudaDeviceSynchronize();
  for (void* p : g->ipc_opened) cudaIpcCloseMemHandle(p);
  if (g->owns_window) cudaFree(g->window);
  cudaFree(g->d_peers);
  cudaFree(g->d_err);
  cudaFree(g->d_done);
  cudaFree(g->d_scratch);
  cudaFree(g->d_seq);
  cudaFree(g->d_lay);
  cudaFreeHost(g->h_err);
  delete g;
  return EPB_OK;
}

}  // extern "C"
