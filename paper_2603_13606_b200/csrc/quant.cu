// K7: standalone block-128 FP8 quantisation and the elementwise wire codecs
// (epsim core.py:114-178).  The dispatch kernel fuses the same arithmetic;
// these entry points serve the tagged-tensor boundary (SCALES inputs,
// read_f32/write_f32 of device tensors) and the codec parity tests.
#include "common.cuh"
#include "internal.h"

namespace epb {

// one warp per 128-element block: 4 elements per lane
template <int XT>
__global__ void fp8_quantize_kernel(const void* x, int64_t nblocks, uint8_t* codes, float* scales) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t blk = gw; blk < nblocks; blk += nw) {
    const int64_t e0 = blk * 128 + lane * 4;
    float f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = load_elem(x, XT, e0 + i);
    float amax = fmaxf(fmaxf(fabsf(f[0]), fabsf(f[1])), fmaxf(fabsf(f[2]), fabsf(f[3])));
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = __fdiv_rn(amax, 448.0f);
    const float div = scale > 0.0f ? scale : 1.0f;
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) w |= e4m3_encode(__fdiv_rn(f[i], div)) << (8 * i);
    reinterpret_cast<uint32_t*>(codes)[blk * 32 + lane] = w;
    if (lane == 0) scales[blk] = scale;
  }
}

__global__ void fp8_dequantize_kernel(const uint8_t* codes, const float* scales, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn(e4m3_value(codes[i]), scales[i >> 7]);
}

__global__ void e4m3_encode_kernel(const float* x, int64_t n, uint8_t* codes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    codes[i] = (uint8_t)e4m3_encode(x[i]);
}

__global__ void convert_kernel(const void* src, int sdt, void* dst, int ddt, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    store_elem(dst, ddt, i, load_elem(src, sdt, i));
}

__global__ void nonfinite_kernel(const float* x, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) atomicExch(flag, 1);
}

inline int grid_for(int64_t n, int per_block) {
  int64_t g = (n + per_block - 1) / per_block;
  return (int)(g < 1 ? 1 : (g > 4096 ? 4096 : g));
}

}  // namespace epb

using namespace epb;

extern "C" {

int epb_fp8_quantize(const void* x, int32_t x_dtype, int64_t rows, int32_t h, uint8_t* codes, float* scales,
                     void* stream) {
  if (h % 128) return fail(EPB_INVALID_ARGUMENT, "hidden not a multiple of 128");
  const int64_t nblocks = rows * (h / 128);
  if (nblocks == 0) return EPB_OK;
  cudaStream_t s = as_stream(stream);
  const int grid = grid_for(nblocks, 8);
  switch (x_dtype) {
    case EPB_F32: fp8_quantize_kernel<EPB_F32><<<grid, 256, 0, s>>>(x, nblocks, codes, scales); break;
    case EPB_BF16: fp8_quantize_kernel<EPB_BF16><<<grid, 256, 0, s>>>(x, nblocks, codes, scales); break;
    case EPB_F16: fp8_quantize_kernel<EPB_F16><<<grid, 256, 0, s>>>(x, nblocks, codes, scales); break;
    default: return fail(EPB_INVALID_ARGUMENT, "quantize input dtype");
  }
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

int epb_fp8_dequantize(const uint8_t* codes, const float* scales, int64_t rows, int32_t h, float* out,
                       void* stream) {
  if (h % 128) return fail(EPB_INVALID_ARGUMENT, "hidden not a multiple of 128");
  const int64_t n = rows * h;
  if (n == 0) return EPB_OK;
  fp8_dequantize_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(codes, scales, n, out);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

int epb_e4m3_encode(const float* x, int64_t n, uint8_t* codes, void* stream) {
  if (n == 0) return EPB_OK;
  e4m3_encode_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, n, codes);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

int epb_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n, void* stream) {
  if (n == 0) return EPB_OK;
  convert_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(src, src_dtype, dst, dst_dtype, n);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

// returns 1 in *flag (device int) when any element is non-finite
int epb_check_finite(const float* x, int64_t n, int32_t* flag, void* stream) {
  if (n == 0) return EPB_OK;
  nonfinite_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, n, flag);
  EPB_LAUNCH_CHECK();
  return EPB_OK;
}

}  // extern "C"
