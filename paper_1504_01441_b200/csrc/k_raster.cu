// Raster stages: luminance + quantise + histograms (K1), CDF-matching LUT
// (K2), 2x2 box pyramid (K3), FP64 summed-area table (K4) and quadrant
// cornerness with per-tile argmax (K5).
//
// Bit-exactness discipline: every f32/f64 op
// that numpy rounds separately is written with the _rn intrinsics in the
// reference's evaluation order, so no FMA contraction can change a bit.
#include "hdr_common.cuh"
#include "hdr_internal.h"
#include "hdr_scan.cuh"

namespace hdr {

// ---------------------------------------------------------------- K1
// image.luminance (image.py:23-29): ((.299R + .587G) + .114B), clip [0,1]
__device__ __forceinline__ float luma(float r, float g, float b) {
  float y = fadd(fadd(fmul(0.299f, r), fmul(0.587f, g)), fmul(0.114f, b));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

// image.quantize_256 (image.py:91-93): floor(x*255 + .5) in f32, clip, u8
__device__ __forceinline__ uint32_t quant(float x) {
  float v = floorf(fadd(fmul(x, 255.0f), 0.5f));
  v = fminf(fmaxf(v, 0.0f), 255.0f);
  return (uint32_t)v;
}

// warp-aggregated shared-memory histogram update
__device__ __forceinline__ void hist_add(uint32_t* sh, uint32_t bin) {
  unsigned peers = __match_any_sync(__activemask(), bin);
  int lane = threadIdx.x & 31;
  if (lane == __ffs(peers) - 1) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
}

constexpr int kHistWarps = 8;

// 4 pixels per thread: 3 x float4 of interleaved RGB in, float4 lum + uchar4 q out.
__global__ void __launch_bounds__(256) luma_hist_kernel(const float* __restrict__ rgb,
                                                        int64_t n, float* __restrict__ lum,
                                                        uint8_t* __restrict__ q,
                                                        uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kHistWarps][kBins];
  for (int i = threadIdx.x; i < kHistWarps * kBins; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  uint32_t* mine = sh[(threadIdx.x >> 5) % kHistWarps];
  int64_t groups = n >> 2;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
    const float4* p = reinterpret_cast<const float4*>(rgb + 12 * g);
    float4 a = __ldcs(p), b = __ldcs(p + 1), c = __ldcs(p + 2);
    float y0 = luma(a.x, a.y, a.z), y1 = luma(a.w, b.x, b.y);
    float y2 = luma(b.z, b.w, c.x), y3 = luma(c.y, c.z, c.w);
    uint32_t q0 = quant(y0), q1 = quant(y1), q2 = quant(y2), q3 = quant(y3);
    if (lum) reinterpret_cast<float4*>(lum)[g] = make_float4(y0, y1, y2, y3);
    if (q) reinterpret_cast<uchar4*>(q)[g] = make_uchar4(q0, q1, q2, q3);
    if (hist) { hist_add(mine, q0); hist_add(mine, q1); hist_add(mine, q2); hist_add(mine, q3); }
  }
  // tail (n % 4 pixels), handled by block 0
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t i = (groups << 2) + threadIdx.x;
    float y = luma(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
    uint32_t v = quant(y);
    if (lum) lum[i] = y;
    if (q) q[i] = (uint8_t)v;
    if (hist) atomicAdd(&mine[v], 1u);
  }
  if (!hist) return;
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kHistWarps; ++w) s += sh[w][b];
    if (s) atomicAdd(&hist[b], s);
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  int cap = 148 * 8;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

void launch_luma_hist(const float* rgb, int64_t n, float* lum, uint8_t* q, uint32_t* hist,
                      cudaStream_t s) {
  luma_hist_kernel<<<grid_for((n >> 2) + 1, 256), 256, 0, s>>>(rgb, n, lum, q, hist);
}

void launch_luminance(const float* rgb, int64_t n, float* lum, cudaStream_t s) {
  luma_hist_kernel<<<grid_for((n >> 2) + 1, 256), 256, 0, s>>>(rgb, n, lum, nullptr, nullptr);
}

// histogram of quantize_256(x) for a strided single-channel view
__global__ void hist_plain_kernel(const float* __restrict__ x, int64_t n, int32_t stride,
                                  uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    hist_add(sh, quant(x[i * stride]));
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

void launch_hist_plain(const float* x, int64_t n, int32_t stride, uint32_t* hist,
                       cudaStream_t s) {
  hist_plain_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, stride, hist);
}

// ---------------------------------------------------------------- K2
// image._match_channel (image.py:96-106): cdf = cumsum(bincount)/size (f64),
// lut = searchsorted(cdf_ref, cdf_src, 'left') capped at 255, then f32 k/255.
__global__ void __launch_bounds__(256) lut_kernel(const uint32_t* __restrict__ hs,
                                                  int64_t ns, const uint32_t* __restrict__ hr,
                                                  int64_t nr, float* __restrict__ lut) {
  __shared__ double cdf_s[kBins], cdf_r[kBins];
  __shared__ long long ws[kBins], wr[kBins];
  int t = threadIdx.x;
  ws[t] = hs[t];
  wr[t] = hr[t];
  __syncthreads();
  // inclusive scans (Hillis-Steele over 256 entries, exact in int64)
  for (int off = 1; off < kBins; off <<= 1) {
    long long a = t >= off ? ws[t - off] : 0, b = t >= off ? wr[t - off] : 0;
    __syncthreads();
    ws[t] += a;
    wr[t] += b;
    __syncthreads();
  }
  cdf_s[t] = (double)ws[t] / (double)ns;
  cdf_r[t] = (double)wr[t] / (double)nr;
  __syncthreads();
  double v = cdf_s[t];
  int lo = 0, hi = kBins;  // first j with cdf_r[j] >= v
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cdf_r[mid] < v) lo = mid + 1; else hi = mid;
  }
  int j = lo < kBins - 1 ? lo : kBins - 1;
  lut[t] = __fdiv_rn((float)j, 255.0f);
}

void launch_lut(const uint32_t* hist_src, int64_t n_src, const uint32_t* hist_ref,
                int64_t n_ref, float* lut, cudaStream_t s) {
  lut_kernel<<<1, kBins, 0, s>>>(hist_src, n_src, hist_ref, n_ref, lut);
}

__global__ void apply_lut_q_kernel(const uint8_t* __restrict__ q, int64_t n,
                                   const float* __restrict__ lut, float* __restrict__ out) {
  __shared__ float t[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) t[i] = lut[i];
  __syncthreads();
  int64_t groups = n >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
    uchar4 v = reinterpret_cast<const uchar4*>(q)[g];
    reinterpret_cast<float4*>(out)[g] = make_float4(t[v.x], t[v.y], t[v.z], t[v.w]);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    int64_t i = (groups << 2) + threadIdx.x;
    out[i] = t[q[i]];
  }
}

void launch_apply_lut_q(const uint8_t* q, int64_t n, const float* lut, float* out,
                        cudaStream_t s) {
  apply_lut_q_kernel<<<grid_for((n >> 2) + 1, 256), 256, 0, s>>>(q, n, lut, out);
}

__global__ void apply_lut_f_kernel(const float* __restrict__ x, int64_t n, int32_t stride,
                                   const float* __restrict__ lut, float* __restrict__ out) {
  __shared__ float t[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) t[i] = lut[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i * stride] = t[quant(x[i * stride])];
}

void launch_apply_lut_f(const float* x, int64_t n, int32_t stride, const float* lut,
                        float* out, cudaStream_t s) {
  apply_lut_f_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, stride, lut, out);
}

// ---------------------------------------------------------------- K3
// image.downsample (image.py:61-68): (((a+b)+c)+d) * 0.25f, odd edge dropped.
// blockIdx.z selects one of two same-shaped images (reference and source
// pyramids are built in the same launch).
__global__ void downsample2_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                   int w, int h, float* __restrict__ oa,
                                   float* __restrict__ ob) {
  const float* in = blockIdx.z ? b : a;
  float* out = blockIdx.z ? ob : oa;
  if (!in) return;
  int ow = w / 2, oh = h / 2;
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= ow || y >= oh) return;
  const float* r0 = in + (int64_t)(2 * y) * w + 2 * x;
  const float* r1 = r0 + w;
  float a0, a1, b0, b1;
  if ((w & 1) == 0) {  // rows start 8-byte aligned: vector loads
    float2 u = *reinterpret_cast<const float2*>(r0);
    float2 v = *reinterpret_cast<const float2*>(r1);
    a0 = u.x; a1 = u.y; b0 = v.x; b1 = v.y;
  } else {
    a0 = r0[0]; a1 = r0[1]; b0 = r1[0]; b1 = r1[1];
  }
  out[(int64_t)y * ow + x] = fmul(fadd(fadd(fadd(a0, a1), b0), b1), 0.25f);
}

void launch_downsample2(const float* a, const float* b, int w, int h, float* oa, float* ob,
                        cudaStream_t s) {
  dim3 blk(32, 8);
  dim3 grd(ceil_div(w / 2, 32), ceil_div(h / 2, 8), 2);
  downsample2_kernel<<<grd, blk, 0, s>>>(a, b, w, h, oa, ob);
}

// ---------------------------------------------------------------- K4
// image.integral (image.py:32-44): cumsum down each column in f64 (pass 1),
// then along each row (pass 2) — numpy's sequential order, bit for bit.
__global__ void sat_cols_kernel(const float* __restrict__ img, int w, int h,
                                double* __restrict__ t) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t w1 = w + 1;
  if (x == 0) t[0] = 0.0;
  if (x >= w) return;
  t[x + 1] = 0.0;
  double acc = 0.0;
  const float* p = img + x;
  double* o = t + w1 + x + 1;
  int y = 0;
  for (; y + 8 <= h; y += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(p + (int64_t)(y + k) * w);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc = dadd(acc, (double)v[k]);
      o[(int64_t)(y + k) * w1] = acc;
    }
  }
  for (; y < h; ++y) {
    acc = dadd(acc, (double)p[(int64_t)y * w]);
    o[(int64_t)y * w1] = acc;
  }
}

// pass 2: one warp per 32 rows, 32x32 tiles staged through shared memory so
// both the loads and the stores stay coalesced; lane r scans row r.
__global__ void __launch_bounds__(32) sat_rows_kernel(double* __restrict__ t, int w, int h) {
  __shared__ double tile[32][33];
  int lane = threadIdx.x;
  int row0 = blockIdx.x * 32 + 1;  // table rows 1..h
  int64_t w1 = w + 1;
  if (row0 + lane <= h) t[(int64_t)(row0 + lane) * w1] = 0.0;
  double acc = 0.0;
  for (int c0 = 1; c0 <= w; c0 += 32) {
    for (int r = 0; r < 32; ++r) {
      int row = row0 + r, col = c0 + lane;
      tile[r][lane] = (row <= h && col <= w) ? t[(int64_t)row * w1 + col] : 0.0;
    }
    __syncwarp();
    int ncol = min(32, w - c0 + 1);
    for (int c = 0; c < ncol; ++c) {
      acc = dadd(acc, tile[lane][c]);
      tile[lane][c] = acc;
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r) {
      int row = row0 + r, col = c0 + lane;
      if (row <= h && col <= w) t[(int64_t)row * w1 + col] = tile[r][lane];
    }
    __syncwarp();
  }
}

void launch_integral(const float* img, int w, int h, double* table, cudaStream_t s) {
  sat_cols_kernel<<<ceil_div(w, 128), 128, 0, s>>>(img, w, h, table);
  sat_rows_kernel<<<ceil_div(h, 32), 32, 0, s>>>(table, w, h);
}

// ---------------------------------------------------------------- K5
// matcher._quadrant_diffs + detect_corners (matcher.py:37-105). One block per
// tile; candidate (lx, ly) sits at t0 + spacing/2 + k*spacing.
__device__ __forceinline__ double box(const double* t, int64_t w1, int x0, int y0, int x1,
                                      int y1) {
  // ((t[y1,x1] - t[y0,x1]) - t[y1,x0]) + t[y0,x0]   (image.py:58)
  return dadd(dsub(dsub(t[y1 * w1 + x1], t[y0 * w1 + x1]), t[y1 * w1 + x0]), t[y0 * w1 + x0]);
}

__global__ void __launch_bounds__(256) detect_kernel(const double* __restrict__ t, int w,
                                                     int h, int tile, double threshold,
                                                     int half, TileCorner* __restrict__ out) {
  int tiles_x = ceil_div(w, tile);
  int tid_tile = blockIdx.x;
  int t0x = (tid_tile % tiles_x) * tile, t0y = (tid_tile / tiles_x) * tile;
  int sp = tile / 16 > 1 ? tile / 16 : 1;
  int first = sp / 2;
  int limx = min(tile, w - t0x), limy = min(tile, h - t0y);
  int nx = limx > first ? (limx - first + sp - 1) / sp : 0;
  int ny = limy > first ? (limy - first + sp - 1) / sp : 0;
  int64_t w1 = w + 1;
  double area = (double)(half * half);
  double best = -1.0;
  int best_i = 0x7fffffff;
  for (int i = threadIdx.x; i < nx * ny; i += blockDim.x) {
    int lx = i % nx, ly = i / nx;
    int x = t0x + first + lx * sp, y = t0y + first + ly * sp;
    if (x < half || x > w - half || y < half || y > h - half) continue;
    double tl = box(t, w1, x - half, y - half, x, y) / area;
    double tr = box(t, w1, x, y - half, x + half, y) / area;
    double br = box(t, w1, x, y, x + half, y + half) / area;
    double bl = box(t, w1, x - half, y, x, y + half) / area;
    double d0 = fabs(dsub(tr, tl)), d1 = fabs(dsub(br, tr));
    double d2 = fabs(dsub(bl, br)), d3 = fabs(dsub(tl, bl));
    double lo = fmin(fmin(d0, d1), fmin(d2, d3));
    if (!(lo > threshold)) continue;
    double c = dadd(dadd(dadd(d0, d1), d2), d3);
    if (c > best || (c == best && i < best_i)) { best = c; best_i = i; }
  }
  // block argmax: highest score, ties to the lowest row-major candidate
  for (int off = 16; off; off >>= 1) {
    double ob = __shfl_down_sync(0xffffffff, best, off);
    int oi = __shfl_down_sync(0xffffffff, best_i, off);
    if (ob > best || (ob == best && oi < best_i)) { best = ob; best_i = oi; }
  }
  __shared__ double sb[8];
  __shared__ int si[8];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sb[warp] = best; si[warp] = best_i; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sb[k] > best || (sb[k] == best && si[k] < best_i)) { best = sb[k]; best_i = si[k]; }
    TileCorner tc;
    if (best_i == 0x7fffffff) {
      tc.x = -1; tc.y = -1; tc.score = 0.0;
    } else {
      tc.x = t0x + first + (best_i % nx) * sp;
      tc.y = t0y + first + (best_i / nx) * sp;
      tc.score = best;
    }
    out[tid_tile] = tc;
  }
}

void launch_detect(const double* table, int w, int h, int tile, double threshold, int half,
                   TileCorner* tiles, cudaStream_t s) {
  int nt = ceil_div(w, tile) * ceil_div(h, tile);
  detect_kernel<<<nt, 256, 0, s>>>(table, w, h, tile, threshold, half, tiles);
}

__global__ void __launch_bounds__(1024) compact_corners_kernel(const TileCorner* __restrict__ tiles,
                                                               int ntiles, double* __restrict__ out,
                                                               int32_t* __restrict__ count) {
  __shared__ int scratch[32];
  int base = 0;
  for (int c0 = 0; c0 < ntiles; c0 += blockDim.x) {
    int i = c0 + threadIdx.x;
    int flag = (i < ntiles && tiles[i].x >= 0) ? 1 : 0;
    int total;
    int pos = block_exclusive_scan(flag, scratch, &total);
    if (flag) {
      TileCorner tc = tiles[i];
      double* r = out + 3 * (int64_t)(base + pos);
      r[0] = tc.x; r[1] = tc.y; r[2] = tc.score;
    }
    base += total;
  }
  if (threadIdx.x == 0) *count = base;
}

void launch_compact_corners(const TileCorner* tiles, int ntiles, double* corners,
                            int32_t* count, cudaStream_t s) {
  compact_corners_kernel<<<1, 1024, 0, s>>>(tiles, ntiles, corners, count);
}

}  // namespace hdr
