// Shared device primitives: memory-ordering PTX, wire codecs, geometry.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>

#include "../../include/epb200.h"

#define EPB_DEV __device__ __forceinline__

namespace epb {

constexpr int kMaxRanks = 64;
constexpr int kMaxTopK = 32;

// ---------------------------------------------------------------------------
// memory ordering (flags cross NVLink: system scope)
// ---------------------------------------------------------------------------
EPB_DEV uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
EPB_DEV void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
EPB_DEV void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// Release before a flag that a peer acquires.  `sys`: the peer may run on
// another GPU, so the fence must be system scope (a GPU-scope fence orders
// nothing for an observer outside this GPU in the PTX memory model).  The
// flag-writing thread issues it after a block barrier, so by cumulativity it
// covers the payload stores of every thread of the CTA.  GPU scope is used
// only while all ranks share this GPU (N = 1 or emulated ranks).
EPB_DEV void fence_release(bool sys) {
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// Stress mode (EPB_CHAOS_NS > 0): a pseudo-random __nanosleep in [0, ns)
// before payload stores and before releases, so CTAs, warps and ranks
// interleave differently every round (the analogue of the reference
// fabric's seeded delivery reordering, fabric.py:203-245).
EPB_DEV void chaos_delay(uint32_t ns, uint32_t salt) {
  if (ns == 0) return;
  uint32_t x;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(x));
  x ^= salt * 0x9E3779B9u + (blockIdx.x << 16) + threadIdx.x;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  __nanosleep(x % ns);
}
EPB_DEV uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// streaming 16-B load of read-once inputs (never window data)
EPB_DEV int4 ld_nc_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
EPB_DEV int4 ld_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
EPB_DEV void st_v4(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}
// store that should not linger in L2 (payload written once, read by a peer)
EPB_DEV void st_na_v4(void* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Bounded spin on a tagged flag.  Returns false (and records
// EPB_TRANSPORT_CLOSED, the analogue of fabric.py:284-291) on timeout.
// Op trace: the B200 counterpart of the reference fabric's per-op log
// (fabric.py:104-111, one CSV line per put / signal / lsa_store).  When a
// ring is registered (epb_group_set_op_trace) the transport kernels append
// one 32-byte record per window transfer they perform: a row record or
// count row stored into a peer's window (PUT), a row read from a peer's
// window (GET: pulled transports), an arrival counter add or flag store
// (SIGNAL).  ring[0] counts appended records (beyond `cap` they are
// dropped, the count keeps growing); record i is ring[4 + 4i .. 4i + 7]:
//   w0 = op | window << 4 | src << 8 | dst << 20 | signal_id << 32
//   w1 = byte offset in dst's window, w2 = length, w3 = signal value.
// A null ring costs one uniform branch per site.
enum { EPB_OP_PUT = 1, EPB_OP_SIGNAL = 2, EPB_OP_GET = 3 };
struct OpTrace {
  unsigned long long* ring;
  uint32_t cap;
};
EPB_DEV void op_record(const OpTrace& t, int op, int src, int dst, uint64_t off, uint64_t len, uint32_t sig = 0,
                       uint64_t value = 0) {
  if (t.ring == nullptr) return;
  const unsigned long long i = atomicAdd(t.ring, 1ull);
  if (i >= t.cap) return;
  unsigned long long* r = t.ring + 4 + 4 * i;
  r[0] = (unsigned long long)op | ((unsigned long long)(src & 0xfff) << 8) |
         ((unsigned long long)(dst & 0xfff) << 20) | ((unsigned long long)sig << 32);
  r[1] = off;
  r[2] = len;
  r[3] = value;
}

// Record the first failure in the group's error word err[0].  err[2..3]
// hold the device address of a mapped pinned host mirror (or 0): the winner
// also writes the code there, so the host learns "no failure" from one host
// read after a synchronisation instead of a device->host copy.
EPB_DEV void raise_err(int* err, int code) {
  if (atomicCAS(err, 0, code) == 0) {
    int* mirror = reinterpret_cast<int*>(*reinterpret_cast<volatile unsigned long long*>(err + 2));
    if (mirror != nullptr) {
      __threadfence_system();
      *reinterpret_cast<volatile int*>(mirror) = code;
    }
  }
}

EPB_DEV bool wait_tag(const uint64_t* flag, uint32_t tag, int shift, uint32_t mask,
                      uint64_t timeout_ns, int* err, uint64_t* value_out) {
  uint64_t start = 0;
  int spins = 0;
  while (true) {
    uint64_t v = ld_acquire_sys(flag);
    if ((uint32_t)((v >> shift) & mask) == tag) {
      *value_out = v;
      return true;
    }
    if (*(volatile int*)err != 0) return false;
    if (++spins == 64) start = globaltimer();
    if (spins > 64 && (spins & 255) == 0) {
      if (globaltimer() - start > timeout_ns) {
        raise_err(err, EPB_TRANSPORT_CLOSED);
        return false;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// wire codecs — bit-exact with epsim core.py
// ---------------------------------------------------------------------------
// E4M3 value of a code; NaN codes decode to +0.0 (core.py:95-96)
EPB_DEV float e4m3_value(uint32_t c) {
  const uint32_t e = (c >> 3) & 0xF, m = c & 7;
  if (e == 15 && m == 7) return 0.0f;
  float v = (e == 0) ? __fmul_rn((float)m, 0x1p-9f)
                     : __uint_as_float(((e + 120u) << 23) | (m << 20));
  return (c & 0x80) ? -v : v;
}

// nearest E4M3 of clamp(|x|, 448); exact midpoints resolve to the SMALLER
// magnitude (searchsorted side="left" over midpoints, core.py:109-120), sign
// from signbit.  Hardware cvt.rn.satfinite is RNE, so a tie that RNE sent to
// the larger neighbour is stepped down one code.
//
// An exact midpoint is recognised from the bits: in the normal range
// [2^-6, 448] it has fraction bit 19 set and bits 18..0 clear; in the
// subnormal range it is an odd multiple of 2^-10.  Clearing that half-step
// (bit 19, or subtracting 2^-10) gives the lower neighbour exactly, which
// the hardware RNE conversion then encodes without rounding.
EPB_DEV float e4m3_tie_down(float x) {
  const float a = fminf(fabsf(x), 448.0f);
  const uint32_t u = __float_as_uint(a);
  if (a >= 0x1p-6f) {
    if ((u & 0xFFFFFu) == 0x80000u) return __uint_as_float(u & ~0x80000u);
  } else {
    const float s = a * 1024.0f;  // exact (power of two)
    if (s == truncf(s) && (((int)s) & 1)) return __fsub_rn(a, 0x1p-10f);
  }
  return a;
}

EPB_DEV uint32_t e4m3_encode(float x) {
  const __nv_fp8_storage_t c = __nv_cvt_float_to_fp8(e4m3_tie_down(x), __NV_SATFINITE, __NV_E4M3);
  return ((uint32_t)c & 0x7F) | (signbit(x) ? 0x80u : 0u);
}

// two codes at once (one cvt.rn.satfinite.e4m3x2.f32): lo = x0, hi = x1
EPB_DEV uint32_t e4m3_encode2(float x0, float x1) {
  const __nv_fp8x2_storage_t c =
      __nv_cvt_float2_to_fp8x2(make_float2(e4m3_tie_down(x0), e4m3_tie_down(x1)), __NV_SATFINITE, __NV_E4M3);
  return ((uint32_t)c & 0x7F7Fu) | (signbit(x0) ? 0x80u : 0u) | (signbit(x1) ? 0x8000u : 0u);
}

EPB_DEV uint16_t bf16_bits_rne(float x) {
  uint32_t u = __float_as_uint(x);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
EPB_DEV float bf16_widen(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
EPB_DEV uint16_t f16_bits_rne(float x) { return __half_as_ushort(__float2half_rn(x)); }
EPB_DEV float f16_widen(uint16_t h) { return __half2float(__ushort_as_half(h)); }

EPB_DEV int dtype_width(int dt) { return dt == EPB_F32 ? 4 : (dt == EPB_FP8 ? 1 : 2); }

// load element i of a row of dtype dt as f32 (fp8 without scale)
EPB_DEV float load_elem(const void* base, int dt, int64_t i) {
  switch (dt) {
    case EPB_F32: return reinterpret_cast<const float*>(base)[i];
    case EPB_BF16: return bf16_widen(reinterpret_cast<const uint16_t*>(base)[i]);
    case EPB_F16: return f16_widen(reinterpret_cast<const uint16_t*>(base)[i]);
    default: return e4m3_value(reinterpret_cast<const uint8_t*>(base)[i]);
  }
}
EPB_DEV void store_elem(void* base, int dt, int64_t i, float v) {
  switch (dt) {
    case EPB_F32: reinterpret_cast<float*>(base)[i] = v; break;
    case EPB_BF16: reinterpret_cast<uint16_t*>(base)[i] = bf16_bits_rne(v); break;
    case EPB_F16: reinterpret_cast<uint16_t*>(base)[i] = f16_bits_rne(v); break;
    default: reinterpret_cast<uint8_t*>(base)[i] = (uint8_t)e4m3_encode(v); break;
  }
}

// ---------------------------------------------------------------------------
// 16-byte chunk codecs.  A "chunk" is 16 bytes of one row in some dtype:
// 4 f32, 8 bf16/f16 or 16 fp8 elements.
// ---------------------------------------------------------------------------
template <int DT> struct Elems;
template <> struct Elems<EPB_F32> { static constexpr int n = 4; };
template <> struct Elems<EPB_BF16> { static constexpr int n = 8; };
template <> struct Elems<EPB_F16> { static constexpr int n = 8; };
template <> struct Elems<EPB_FP8> { static constexpr int n = 16; };

template <int DT>
EPB_DEV void unpack16(const int4& v, float* f) {
  const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
  if constexpr (DT == EPB_F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(w[i]);
  } else if constexpr (DT == EPB_BF16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = bf16_widen((uint16_t)(w[i] & 0xFFFF));
      f[2 * i + 1] = bf16_widen((uint16_t)(w[i] >> 16));
    }
  } else if constexpr (DT == EPB_F16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = f16_widen((uint16_t)(w[i] & 0xFFFF));
      f[2 * i + 1] = f16_widen((uint16_t)(w[i] >> 16));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = e4m3_value((w[i >> 2] >> (8 * (i & 3))) & 0xFF);
  }
}

template <int DT>
EPB_DEV int4 pack16(const float* f) {
  uint32_t w[4];
  if constexpr (DT == EPB_F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __float_as_uint(f[i]);
  } else if constexpr (DT == EPB_BF16) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = (uint32_t)bf16_bits_rne(f[2 * i]) | ((uint32_t)bf16_bits_rne(f[2 * i + 1]) << 16);
  } else if constexpr (DT == EPB_F16) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = (uint32_t)f16_bits_rne(f[2 * i]) | ((uint32_t)f16_bits_rne(f[2 * i + 1]) << 16);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = e4m3_encode2(f[4 * i], f[4 * i + 1]) | (e4m3_encode2(f[4 * i + 2], f[4 * i + 3]) << 16);
  }
  return make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
}

// load `n` elements starting at element e0 of a row in dtype DT as f32.
// n = Elems<OUT>::n; reads n*width bytes (16-B aligned multiples).
template <int DT, int N>
EPB_DEV void load_elems_vec(const void* row, int64_t e0, float* f) {
  constexpr int per = Elems<DT>::n;
  static_assert(N % per == 0 || per % N == 0, "chunk mismatch");
  if constexpr (N >= per) {
#pragma unroll
    for (int c = 0; c < N / per; ++c) {
      const char* p = reinterpret_cast<const char*>(row) + (e0 + c * per) * (16 / per);
      int4 v = ld_nc_v4(p);
      unpack16<DT>(v, f + c * per);
    }
  } else {
    // fewer elements than a 16-B chunk of DT (e.g. 4 f32 out of fp8 input)
    const uint8_t* p = reinterpret_cast<const uint8_t*>(row);
#pragma unroll
    for (int i = 0; i < N; ++i) f[i] = load_elem(p, DT, e0 + i);
  }
}

// store EPC f32 values as elements [e0, e0+EPC) of a row in dtype OT
// (f32 or bf16/f16); e0*width must be 16-B aligned when EPC*width >= 16.
template <int OT, int EPC>
EPB_DEV void store_f32_chunk(uint8_t* row, int64_t e0, const float* f) {
  if constexpr (OT == EPB_F32) {
#pragma unroll
    for (int q = 0; q < EPC / 4; ++q)
      st_v4(row + (e0 + 4 * q) * 4, make_int4(__float_as_int(f[4 * q]), __float_as_int(f[4 * q + 1]),
                                             __float_as_int(f[4 * q + 2]), __float_as_int(f[4 * q + 3])));
  } else if constexpr (EPC >= 8) {
#pragma unroll
    for (int q = 0; q < EPC / 8; ++q) st_v4(row + (e0 + 8 * q) * 2, pack16<OT>(f + 8 * q));
  } else {
    uint16_t* o = reinterpret_cast<uint16_t*>(row) + e0;
#pragma unroll
    for (int i = 0; i < EPC; ++i) o[i] = OT == EPB_BF16 ? bf16_bits_rne(f[i]) : f16_bits_rne(f[i]);
  }
}

EPB_DEV size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace epb
