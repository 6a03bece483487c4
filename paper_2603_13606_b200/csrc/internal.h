// Library-internal state shared by the translation units.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/epb200.h"
#include "geometry.h"

struct epb_group {
  epb_config cfg;
  int rank;
  int device;
  uint8_t* window = nullptr;
  uint64_t window_bytes = 0;
  bool owns_window = false;
  void* alloc_base = nullptr;   // allocation holding `window` (for IPC)
  uint64_t* d_peers = nullptr;  // [N] window bases as seen from this GPU
  std::vector<void*> ipc_opened;
  int* d_err = nullptr;         // device error word [4]: code, -, mirror address
  int* h_err = nullptr;         // mapped pinned host mirror of the code (raise_err)
  int* d_done = nullptr;        // [2*N] arrival counters (dispatch, combine)
  int* d_scratch = nullptr;     // [8*N + 2*L*N + 64] small per-call state
  uint32_t* d_seq = nullptr;    // [kLLGrid] LL round sequence, one copy per dispatch CTA
  int* d_lay = nullptr;         // [ceil(B / kLayChunk)][E+N] per-chunk routing histograms (K1)
  epb::LLGeom ll;
  epb::HTGeom ht;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  uint64_t* trace = nullptr;    // optional [grid][16] globaltimer stamps (diagnostics)
  unsigned long long* op_ring = nullptr;  // optional op trace ring (epb_group_set_op_trace)
  uint32_t op_cap = 0;
  bool peers_ready = false;
  bool sys_scope = false;       // peers on other GPUs: system-scope fences/flags
  int fence_override = -1;      // EPB_SYS_FENCE: -1 auto, 0 GPU scope, 1 system scope
};

namespace epb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace epb

#define EPB_CUDA(call)                                          \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return epb::cuda_check(_e, #call);   \
  } while (0)

#define EPB_LAUNCH_CHECK() EPB_CUDA(cudaGetLastError())
