// Sparse-to-dense flow: splat (K9) and the densify-finalise fused with the
// bilinear backward warp, luminance of the warped frame and its histogram
// (K11 + K12). The domain-transform filter (K10) is in k_dtfilter.cu.
#include "hdr_common.cuh"
#include "hdr_internal.h"
#include "hdr_planes.cuh"

namespace hdr {

// ---------------------------------------------------------------- K9
// densify.build_sparse_maps (densify.py:38-56): collisions keep the lowest
// (score, index). Single block, four phases separated by block barriers;
// only the touched pixels of the scratch key/index planes are initialised.
__device__ __forceinline__ unsigned long long ordered_bits(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__device__ __forceinline__ bool splat_pixel(const double* r, int w, int h, int64_t* p) {
  double xf = rint(r[0]), yf = rint(r[1]);  // int(round()) is half-even
  if (!(xf >= 0 && xf < w && yf >= 0 && yf < h)) return false;
  *p = (int64_t)yf * w + (int64_t)xf;
  return true;
}

__global__ void __launch_bounds__(1024) splat_kernel(const double* __restrict__ m,
                                                     const int32_t* __restrict__ count,
                                                     int m_static, int w, int h, DtPlanes maps,
                                                     unsigned long long* __restrict__ key,
                                                     int32_t* __restrict__ idx,
                                                     int32_t* __restrict__ status) {
  pdl_wait();
  int n = count ? *count : m_static;
  int64_t p;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!splat_pixel(m + 5 * (int64_t)i, w, h, &p)) {
      if (status) atomicExch(status, 1);
      continue;
    }
    key[p] = ~0ULL;
    idx[p] = 0x7fffffff;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (splat_pixel(m + 5 * (int64_t)i, w, h, &p))
      atomicMin(&key[p], ordered_bits(m[5 * (int64_t)i + 4]));
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (splat_pixel(m + 5 * (int64_t)i, w, h, &p) && key[p] == ordered_bits(m[5 * (int64_t)i + 4]))
      atomicMin(&idx[p], i);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double* r = m + 5 * (int64_t)i;
    if (!splat_pixel(r, w, h, &p) || idx[p] != i) continue;
    stp(maps, 0, p, r[2] - r[0]);
    stp(maps, 1, p, r[3] - r[1]);
    stp(maps, 2, p, 1.0);
  }
}

void launch_splat(const double* matches, const int32_t* count, int m_static, int w, int h,
                  DtPlanes maps, uint64_t* scratch_key, int32_t* scratch_idx, int32_t* status,
                  cudaStream_t s) {
  int64_t P = (int64_t)w * h;
  for (int k = 0; k < 3; ++k)
    cudaMemsetAsync(maps.p[k], 0, P * (maps.f64[k] ? 8 : 4), s);
  klaunch(splat_kernel, 1, 1024, 0, s, matches, count, m_static, w, h, maps,
                                  reinterpret_cast<unsigned long long*>(scratch_key), scratch_idx,
                                  status);
}

// densify.build_sparse_maps in CSR-by-row form for the first domain-transform
// row pass (dt_rows_first_kernel): the same collision rule as splat_kernel,
// then the winners bucketed by row (count, block-wide exclusive scan over the
// h + 1 row starts, scatter; the order inside a row is irrelevant, the x are
// distinct). Single block: a pair has at most one weeded match per tile.
__global__ void __launch_bounds__(1024) splat_rows_kernel(
    const double* __restrict__ m, const int32_t* __restrict__ count, int m_static, int w, int h,
    unsigned long long* __restrict__ key, int32_t* __restrict__ idx, int32_t* __restrict__ row_count,
    int32_t* __restrict__ row_start, SparseEntry* __restrict__ entries, int32_t* __restrict__ status) {
  pdl_wait();
  __shared__ int32_t part[1024];
  int n = count ? *count : m_static;
  int64_t p;
  for (int i = threadIdx.x; i <= h; i += blockDim.x) row_count[i] = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (!splat_pixel(m + 5 * (int64_t)i, w, h, &p)) {
      if (status) atomicExch(status, 1);
      continue;
    }
    key[p] = ~0ULL;
    idx[p] = 0x7fffffff;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (splat_pixel(m + 5 * (int64_t)i, w, h, &p))
      atomicMin(&key[p], ordered_bits(m[5 * (int64_t)i + 4]));
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (splat_pixel(m + 5 * (int64_t)i, w, h, &p) && key[p] == ordered_bits(m[5 * (int64_t)i + 4]))
      atomicMin(&idx[p], i);
  __syncthreads();
  // winners take a slot in their row (kept in key[p], no longer needed)
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (splat_pixel(m + 5 * (int64_t)i, w, h, &p) && idx[p] == i)
      key[p] = (unsigned long long)atomicAdd(&row_count[p / w], 1);
  __syncthreads();
  // exclusive scan of row_count[0..h) -> row_start[0..h]: contiguous chunks
  // per thread, a block scan of the chunk sums
  const int per = (h + blockDim.x) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(h, b0 + per);
  int32_t sum = 0;
  for (int i = b0; i < b1; ++i) sum += row_count[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    int32_t v = threadIdx.x >= (unsigned)off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = part[threadIdx.x] - sum;
  for (int i = b0; i < b1; ++i) {
    row_start[i] = run;
    run += row_count[i];
  }
  if (threadIdx.x == blockDim.x - 1) row_start[h] = part[threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double* r = m + 5 * (int64_t)i;
    if (!splat_pixel(r, w, h, &p) || idx[p] != i) continue;
    int y = (int)(p / w);
    SparseEntry e;
    e.x = (int)(p - (int64_t)y * w);
    e.pad = 0;
    e.u = r[2] - r[0];
    e.v = r[3] - r[1];
    entries[row_start[y] + (int)key[p]] = e;
  }
}

void launch_splat_rows(const double* matches, const int32_t* count, int m_static, int w, int h,
                       uint64_t* scratch_key, int32_t* scratch_idx, int32_t* row_count,
                       int32_t* row_start, SparseEntry* entries, int32_t* status, cudaStream_t s) {
  klaunch(splat_rows_kernel, 1, 1024, 0, s, matches, count, m_static, w, h,
                                       reinterpret_cast<unsigned long long*>(scratch_key),
                                       scratch_idx, row_count, row_start, entries, status);
}

// ---------------------------------------------------------------- K11/K12
__global__ void hflow_kernel(const double* __restrict__ Hd, int w, int h, float* __restrict__ flow) {
  pdl_wait();
  __shared__ double H[9];
  if (threadIdx.x < 9) H[threadIdx.x] = Hd[threadIdx.x];
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)w * h) return;
  int x = (int)(i % w), y = (int)(i / w);
  float u, v;
  h_pixel_flow(H, x, y, w, h, &u, &v);
  reinterpret_cast<float2*>(flow)[i] = make_float2(u, v);
}

void launch_hflow(const double* H, int w, int h, float* flow, cudaStream_t s) {
  int64_t n = (int64_t)w * h;
  klaunch(hflow_kernel, (unsigned)((n + 255) / 256), 256, 0, s, H, w, h, flow);
}

__device__ __forceinline__ float luma3(float r, float g, float b) {
  float y = fadd(fadd(fmul(0.299f, r), fmul(0.587f, g)), fmul(0.114f, b));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

__device__ __forceinline__ uint32_t quant3(float x) {
  float v = floorf(fadd(fmul(x, 255.0f), 0.5f));
  return (uint32_t)fminf(fmaxf(v, 0.0f), 255.0f);
}

// densify_flow finalise (densify.py:134-142) + warp_image (densify.py:145-174)
// + luminance(warped) -> quantised histogram for make_ssim (pipeline.py:168).
// do_flow = false: flow is an input (warp_image alone); src = null: no warp.
__global__ void __launch_bounds__(256) finalize_warp_kernel(
    DtPlanes smooth, const double* __restrict__ fallback, const int32_t* __restrict__ has_fb,
    int w, int h, double floor_, const float* __restrict__ src, int channels,
    float* __restrict__ flow, float* __restrict__ warped, uint8_t* __restrict__ valid,
    uint8_t* __restrict__ qw, uint32_t* __restrict__ hist, bool do_flow) {
  pdl_wait();
  __shared__ uint32_t sh[kBins];
  __shared__ double H[9];
  __shared__ int use_fb;
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) use_fb = (fallback && (!has_fb || *has_fb)) ? 1 : 0;
  __syncthreads();
  if (threadIdx.x < 9 && use_fb) H[threadIdx.x] = fallback[threadIdx.x];
  __syncthreads();
  int64_t P = (int64_t)w * h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(i % w), y = (int)(i / w);
    float fu, fv;
    if (do_flow) {
      double n = ldp(smooth, 2, i);
      if (n > floor_) {
        fu = (float)(ldp(smooth, 0, i) / n);
        fv = (float)(ldp(smooth, 1, i) / n);
      } else if (use_fb) {
        h_pixel_flow(H, x, y, w, h, &fu, &fv);
      } else {
        fu = 0.0f;
        fv = 0.0f;
      }
      reinterpret_cast<float2*>(flow)[i] = make_float2(fu, fv);
      if (!src) continue;
    } else {
      float2 f = reinterpret_cast<const float2*>(flow)[i];
      fu = f.x;
      fv = f.y;
    }
    double sx = dadd((double)x, (double)fu), sy = dadd((double)y, (double)fv);
    bool ok = sx >= 0.0 && sx <= (double)(w - 1) && sy >= 0.0 && sy <= (double)(h - 1);
    double cx = fmin(fmax(sx, 0.0), (double)(w - 1));
    double cy = fmin(fmax(sy, 0.0), (double)(h - 1));
    int x0 = (int)floor(cx), y0 = (int)floor(cy);
    int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
    double fx = dsub(cx, (double)x0), fy = dsub(cy, (double)y0);
    double gx = dsub(1.0, fx), gy = dsub(1.0, fy);
    const float* s00 = src + ((int64_t)y0 * w + x0) * channels;
    const float* s01 = src + ((int64_t)y0 * w + x1) * channels;
    const float* s10 = src + ((int64_t)y1 * w + x0) * channels;
    const float* s11 = src + ((int64_t)y1 * w + x1) * channels;
    float o[3] = {0.0f, 0.0f, 0.0f};  // the first three channels, for the luminance
    for (int k = 0; k < channels; ++k) {
      double top = dadd(dmul((double)s00[k], gx), dmul((double)s01[k], fx));
      double bot = dadd(dmul((double)s10[k], gx), dmul((double)s11[k], fx));
      float v = (float)dadd(dmul(top, gy), dmul(bot, fy));
      if (k < 3) o[k] = v;
      warped[i * channels + k] = v;
    }
    valid[i] = ok ? 1 : 0;
    if (qw) {
      float lum = channels == 3 ? luma3(o[0], o[1], o[2]) : luma3(o[0], o[0], o[0]);
      uint32_t q = quant3(lum);
      qw[i] = (uint8_t)q;
      unsigned peers = __match_any_sync(__activemask(), q);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh[q], (uint32_t)__popc(peers));
    }
  }
  if (!qw) return;
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// warp_image (densify.py:145-174) + luminance(warped) -> quantised histogram,
// flow given. Blocks sweep 256-pixel row segments (grid-stride), so each
// thread's (x, y) comes without a per-pixel division and the block histogram
// is flushed once per block.
// Rows [y0, y1) of the (w, h) frame (the whole frame for the pair; a row
// band of it for the banded pair); hist may be null (halo rows of a band).
__global__ void __launch_bounds__(256) warp_kernel(const float* __restrict__ flow, int w, int h,
                                                   const float* __restrict__ src,
                                                   float* __restrict__ warped,
                                                   uint8_t* __restrict__ valid,
                                                   uint8_t* __restrict__ qw,
                                                   uint32_t* __restrict__ hist, int y0, int y1) {
  pdl_wait();
  // one histogram per warp (plain shared atomics; see luma_hist_kernel)
  __shared__ uint32_t sh[8][kBins];
  for (int i = threadIdx.x; i < 8 * kBins; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t* mine = sh[threadIdx.x >> 5];
  // row / segment indices advance without a division per step
  const int segs = (w + 255) >> 8;
  const int dq = gridDim.x / segs, dr = gridDim.x - dq * segs;
  int y = y0 + (int)blockIdx.x / segs, seg = blockIdx.x - (y - y0) * segs;
  // the flow of the next work item is loaded before this one's gathers are
  // issued (software pipelining: its DRAM latency hides behind them)
  auto flow_at = [&](int yy, int ss) {
    const int xx = ss * 256 + threadIdx.x;
    return yy < y1 && xx < w ? __ldcs(reinterpret_cast<const float2*>(flow) + (int64_t)yy * w + xx)
                             : make_float2(0.0f, 0.0f);
  };
#ifndef HDR_WARP_PREFETCH
#define HDR_WARP_PREFETCH 1
#endif
  float2 fnext = HDR_WARP_PREFETCH ? flow_at(y, seg) : make_float2(0.0f, 0.0f);
  for (; y < y1; y += dq, seg += dr) {
    if (seg >= segs) { seg -= segs; ++y; if (y >= y1) break; }
#if HDR_WARP_PREFETCH
    const float2 f = fnext;
    {
      int yn = y + dq, sn = seg + dr;
      if (sn >= segs) { sn -= segs; ++yn; }
      fnext = flow_at(yn, sn);
    }
#endif
    int x = seg * 256 + threadIdx.x;
    if (x >= w) continue;
    int64_t i = (int64_t)y * w + x;
#if !HDR_WARP_PREFETCH
    float2 f = __ldcs(reinterpret_cast<const float2*>(flow) + i);
#endif
    double sx = dadd((double)x, (double)f.x), sy = dadd((double)y, (double)f.y);
    const double wm = (double)(w - 1), hm = (double)(h - 1);
    bool ok = sx >= 0.0 && sx <= wm && sy >= 0.0 && sy <= hm;
    // np.clip of a finite value: compare + select (f64 fmin/fmax cost ~7
    // instructions each here)
    double cx = sx < 0.0 ? 0.0 : (sx > wm ? wm : sx);
    double cy = sy < 0.0 ? 0.0 : (sy > hm ? hm : sy);
    int x0 = (int)floor(cx), y0 = (int)floor(cy);
    double fx = dsub(cx, (double)x0), fy = dsub(cy, (double)y0);
    double gx = dsub(1.0, fx), gy = dsub(1.0, fy);
    // 32-bit element offsets (3 w h < 2^31 for any frame the context holds)
    const int o00 = 3 * (y0 * w + x0);
    const int dxo = x0 + 1 < w ? 3 : 0, dyo = y0 + 1 < h ? 3 * w : 0;
    const float* s00 = src + o00;
    const float* s01 = s00 + dxo;
    const float* s10 = s00 + dyo;
    const float* s11 = s10 + dxo;
    float o[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double top = dadd(dmul((double)__ldg(s00 + k), gx), dmul((double)__ldg(s01 + k), fx));
      double bot = dadd(dmul((double)__ldg(s10 + k), gx), dmul((double)__ldg(s11 + k), fx));
      o[k] = (float)dadd(dmul(top, gy), dmul(bot, fy));
    }
    float* wo = warped + 3 * i;
    wo[0] = o[0]; wo[1] = o[1]; wo[2] = o[2];
    valid[i] = ok ? 1 : 0;
    uint32_t q = quant3(luma3(o[0], o[1], o[2]));
    qw[i] = (uint8_t)q;
    atomicAdd(&mine[q], 1u);
  }
  if (!hist) return;
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) t += sh[w8][b];
    if (t) atomicAdd(&hist[b], t);
  }
}

void launch_warp_rows(const float* flow, int w, int h, int y0, int y1, const float* src, float* warped,
                      uint8_t* valid, uint8_t* qw, uint32_t* hist, cudaStream_t s) {
  if (y1 <= y0) return;
  int64_t work = (int64_t)((w + 255) / 256) * (y1 - y0);
  int64_t cap = 148 * 12;
  int64_t blocks = work < cap ? work : cap;
  klaunch(warp_kernel, (unsigned)blocks, 256, 0, s, flow, w, h, src, warped, valid, qw, hist, y0, y1);
}

void launch_warp(const float* flow, int w, int h, const float* src, float* warped, uint8_t* valid,
                 uint8_t* qw, uint32_t* hist, cudaStream_t s) {
  if (3 * (int64_t)w * h >= ((int64_t)1 << 31)) {  // beyond the 32-bit offsets of warp_kernel
    DtPlanes none{{nullptr, nullptr, nullptr}, {0, 0, 0}, 0};
    launch_finalize_warp(none, nullptr, nullptr, w, h, 0.0, src, 3, const_cast<float*>(flow), warped, valid,
                         qw, hist, false, s);
    return;
  }
  int64_t work = (int64_t)((w + 255) / 256) * h;
#ifndef HDR_WARP_BLOCKS_PER_SM
#define HDR_WARP_BLOCKS_PER_SM 12
#endif
  int64_t cap = 148 * HDR_WARP_BLOCKS_PER_SM;
  int64_t blocks = work < cap ? work : cap;
  klaunch(warp_kernel, (unsigned)blocks, 256, 0, s, flow, w, h, src, warped, valid, qw, hist, 0, h);
}

void launch_finalize_warp(DtPlanes smooth, const double* fallback, const int32_t* has_fallback,
                          int w, int h, double floor_, const float* src, int channels, float* flow,
                          float* warped, uint8_t* valid, uint8_t* qw, uint32_t* hist_w,
                          bool do_flow, cudaStream_t s) {
  int64_t P = (int64_t)w * h;
  int64_t blocks = (P + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  klaunch(finalize_warp_kernel, (unsigned)blocks, 256, 0, s, smooth, fallback, has_fallback, w, h,
                                                        floor_, src, channels, flow, warped,
                                                        valid, qw, hist_w, do_flow);
}

}  // namespace hdr
