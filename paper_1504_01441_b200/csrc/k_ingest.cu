// Ingest and output formats of the file path:
// fileio.load_png's integer -> [0, 1] float conversion fused with
// pipeline.as_rgb's grey -> RGB repeat, fileio.save_png's 8-bit
// quantisation, and metering.choose_reference's mean luminance. Decoding the
// PNG container itself (zlib) stays on the host; only raw 8/16-bit samples
// cross PCIe -- 4x (2x) fewer bytes than the float32 frames.
#include "hdr_common.cuh"
#include "hdr_internal.h"

namespace hdr {

// fileio.load_png (fileio.py:21-41): f32(clip(f64(v) / 255 or 65535)),
// then as_rgb (pipeline.py:112-115) for one-channel input. Each thread
// converts 4 pixels (16-byte / 8-byte loads of the raw samples when aligned).
template <class T, int C>
__global__ void __launch_bounds__(256) decode_kernel(const T* __restrict__ in, int64_t npx,
                                                     double scale, float* __restrict__ out) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < npx; i += stride) {
    float v[3];
#pragma unroll
    for (int c = 0; c < C; ++c) v[c] = (float)fmin(fmax((double)in[i * C + c] / scale, 0.0), 1.0);
    float* o = out + 3 * i;
    o[0] = v[0];
    o[1] = C == 3 ? v[1] : v[0];
    o[2] = C == 3 ? v[2] : v[0];
  }
}

void launch_decode(const void* in, int64_t npx, int channels, int bits, float* out,
                   cudaStream_t s) {
  int64_t blocks = std::min<int64_t>((npx + 255) / 256, 148 * 16);
  if (blocks < 1) return;
  double scale = bits == 16 ? 65535.0 : 255.0;
  if (bits == 16) {
    if (channels == 3)
      klaunch(decode_kernel<uint16_t, 3>, (unsigned)blocks, 256, 0, s, (const uint16_t*)in, npx, scale, out);
    else
      klaunch(decode_kernel<uint16_t, 1>, (unsigned)blocks, 256, 0, s, (const uint16_t*)in, npx, scale, out);
  } else {
    if (channels == 3)
      klaunch(decode_kernel<uint8_t, 3>, (unsigned)blocks, 256, 0, s, (const uint8_t*)in, npx, scale, out);
    else
      klaunch(decode_kernel<uint8_t, 1>, (unsigned)blocks, 256, 0, s, (const uint8_t*)in, npx, scale, out);
  }
}

// fileio.save_png (fileio.py:44-53): clip(floor(f64(x) * 255 + 0.5), 0, 255)
// as uint8, 16 values per thread (four 16-byte loads, one 16-byte store).
__global__ void __launch_bounds__(256) encode_u8_kernel(const float* __restrict__ x, int64_t n,
                                                        uint8_t* __restrict__ out) {
  pdl_wait();
  auto q = [](float v) -> uint32_t {
    double d = floor(fma((double)v, 255.0, 0.5));  // exact: v*255 fits in 53 bits
    return (uint32_t)fmin(fmax(d, 0.0), 255.0);
  };
  int64_t nv = n / 16;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool vec = ((uintptr_t)x & 15) == 0 && ((uintptr_t)out & 15) == 0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (; i < nv; i += stride) {
      const float4* p = reinterpret_cast<const float4*>(x) + 4 * i;
      uint32_t wds[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float4 f = __ldcs(p + k);
        wds[k] = q(f.x) | q(f.y) << 8 | q(f.z) << 16 | q(f.w) << 24;
      }
      reinterpret_cast<uint4*>(out)[i] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
    }
    i = 16 * nv + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  }
  for (; i < n; i += stride) out[i] = (uint8_t)q(x[i]);
}

void launch_encode_u8(const float* x, int64_t n, uint8_t* out, cudaStream_t s) {
  int64_t blocks = std::min<int64_t>((n / 16 + 255) / 256 + 1, 148 * 8);
  klaunch(encode_u8_kernel, (unsigned)blocks, 256, 0, s, x, n, out);
}

// metering.choose_reference's mean_lum (metering.py:46-48): mean of
// image.luminance over the frame, accumulated in f64 (numpy accumulates the
// float32 luminance pairwise in float32; the two agree to ~1e-7 relative,
// which only matters for a tie-break between equal exposures).
// luminance of pixel i (RGB) or the grey value itself (channels == 1: the
// reference meters grey images directly, metering.py:28,47)
__device__ __forceinline__ float meter_value(const float* img, int channels, int64_t i) {
  if (channels == 1) return img[i];
  const float* p = img + 3 * i;
  float y = fadd(fadd(fmul(0.299f, p[0]), fmul(0.587f, p[1])), fmul(0.114f, p[2]));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

__global__ void __launch_bounds__(256) mean_lum_kernel(const float* __restrict__ img, int channels,
                                                       int64_t n, double* __restrict__ out) {
  pdl_wait();
  __shared__ double part[8];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += (double)meter_value(img, channels, i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += part[k];
    atomicAdd(out, t / (double)n);
  }
}

void launch_mean_luminance(const float* img, int channels, int64_t n, double* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 4);
  if (blocks < 1) return;
  klaunch(mean_lum_kernel, (unsigned)blocks, 256, 0, s, img, channels, n, out);
}

// metering.select_offset's statistic (metering.py:28-29): the number of
// pixels whose image.luminance is below dark_level. numpy 2 compares the
// float32 luminance with the Python float cast to float32 (NEP 50), so the
// compare is in f32 (the caller passes f32(dark_level)).
__global__ void __launch_bounds__(256) dark_count_kernel(const float* __restrict__ img, int channels,
                                                         int64_t n, float dark,
                                                         unsigned long long* out) {
  pdl_wait();
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt += meter_value(img, channels, i) < dark ? 1ull : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

void launch_dark_count(const float* img, int channels, int64_t n, float dark,
                       unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 4);
  if (blocks < 1) return;
  klaunch(dark_count_kernel, (unsigned)blocks, 256, 0, s, img, channels, n, dark, out);
}

}  // namespace hdr
