// Raster stages: luminance + quantise + histograms (K1), CDF-matching LUT
// (K2), 2x2 box pyramid (K3), FP64 summed-area lattice (K4) and quadrant
// cornerness with per-tile argmax (K5).
//
// Bit-exactness discipline: every f32/f64 op
// that numpy rounds separately is written with the _rn intrinsics in the
// reference's evaluation order, so no FMA contraction can change a bit.
#include "hdr_common.cuh"
#include "hdr_internal.h"

#include <algorithm>
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
  pdl_wait();
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
    if (hist) {
      // plain shared atomics into the warp's own histogram: measured faster
      // than warp-aggregated __match_any_sync updates, whose MATCH
      // instructions saturated the ADU pipe (raster stage 106 -> 80 us)
      atomicAdd(&mine[q0], 1u);
      atomicAdd(&mine[q1], 1u);
      atomicAdd(&mine[q2], 1u);
      atomicAdd(&mine[q3], 1u);
    }
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
#ifndef HDR_RASTER_BLOCKS_PER_SM
#define HDR_RASTER_BLOCKS_PER_SM 4
#endif
  int cap = 148 * HDR_RASTER_BLOCKS_PER_SM;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

void launch_luma_hist(const float* rgb, int64_t n, float* lum, uint8_t* q, uint32_t* hist,
                      cudaStream_t s) {
  klaunch(luma_hist_kernel, grid_for((n >> 2) + 1, 256), 256, 0, s, rgb, n, lum, q, hist);
}

void launch_luminance(const float* rgb, int64_t n, float* lum, cudaStream_t s) {
  klaunch(luma_hist_kernel, grid_for((n >> 2) + 1, 256), 256, 0, s, rgb, n, lum, nullptr, nullptr);
}

// histogram of quantize_256(x) for a strided single-channel view
__global__ void hist_plain_kernel(const float* __restrict__ x, int64_t n, int32_t stride,
                                  uint32_t* __restrict__ hist) {
  pdl_wait();
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
  klaunch(hist_plain_kernel, grid_for(n, 256), 256, 0, s, x, n, stride, hist);
}

// ---------------------------------------------------------------- K2
// image._match_channel (image.py:96-106): cdf = cumsum(bincount)/size (f64),
// lut = searchsorted(cdf_ref, cdf_src, 'left') capped at 255, then f32 k/255.
__global__ void __launch_bounds__(256) lut_kernel(const uint32_t* __restrict__ hs,
                                                  int64_t ns, const uint32_t* __restrict__ hr,
                                                  int64_t nr, float* __restrict__ lut) {
  pdl_wait();
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
  klaunch(lut_kernel, 1, kBins, 0, s, hist_src, n_src, hist_ref, n_ref, lut);
}

__global__ void apply_lut_q_kernel(const uint8_t* __restrict__ q, int64_t n,
                                   const float* __restrict__ lut, float* __restrict__ out) {
  pdl_wait();
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
  klaunch(apply_lut_q_kernel, grid_for((n >> 2) + 1, 256), 256, 0, s, q, n, lut, out);
}

__global__ void apply_lut_f_kernel(const float* __restrict__ x, int64_t n, int32_t stride,
                                   const float* __restrict__ lut, float* __restrict__ out) {
  pdl_wait();
  __shared__ float t[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) t[i] = lut[i];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i * stride] = t[quant(x[i * stride])];
}

void launch_apply_lut_f(const float* x, int64_t n, int32_t stride, const float* lut,
                        float* out, cudaStream_t s) {
  klaunch(apply_lut_f_kernel, grid_for(n, 256), 256, 0, s, x, n, stride, lut, out);
}

// ---------------------------------------------------------------- K3
// image.downsample (image.py:61-68): (((a+b)+c)+d) * 0.25f, odd edge dropped.
// blockIdx.z selects one of two same-shaped images (reference and source
// pyramids are built in the same launch).
__global__ void downsample2_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                   int w, int h, float* __restrict__ oa,
                                   float* __restrict__ ob) {
  pdl_wait();
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
  klaunch(downsample2_kernel, grd, blk, 0, s, a, b, w, h, oa, ob);
}

// ---------------------------------------------------------------- K4
// image.integral (image.py:32-44) restricted to the lattice the detector
// reads. numpy fixes the rounding order: a sequential f64 cumsum down each
// column (pass 1), then a sequential cumsum along each row (pass 2), so
// both passes keep that order exactly; they only skip *storing* entries no
// quadrant sum will read. Table row Y / column X live at rowmap[Y] /
// colmap[X] (-1 = not needed); identity maps give the full table.
constexpr int kSatPrefetch = 32;

// Exactness certificate. Every partial sum numpy forms (image.py:42-43) and
// every rect_sum difference (image.py:58) is a sum of a subset of the
// level's samples. If all samples are multiples of 2^qmin and their total is
// below 2^(52+qmin), all of those values are representable in f64, every
// addition is exact, and ANY summation order reproduces numpy's bits.
__device__ __forceinline__ int log2_quantum(float v) {
  uint32_t u = __float_as_uint(v) & 0x7fffffffu;
  if (u == 0) return 1 << 20;
  uint32_t e = u >> 23, m = u & 0x7fffffu;
  uint32_t M = e ? (m | 0x800000u) : m;
  return (e ? (int)e - 150 : -149) + __ffs(M) - 1;
}

__device__ __forceinline__ bool level_exact(const SatBatch& b, int l) {
  if (!b.qmin) return false;
  double s = b.sums[l];
  if (!(s > 0.0)) return s == 0.0;
  int q = b.qmin[l];
  // s * (1 + 2^-30) bounds the rounding of the f64 reduction itself
  return ilogb(s * (1.0 + 9.3e-10)) + 1 <= 52 + q;
}

__global__ void __launch_bounds__(256) level_stats_kernel(SatBatch b) {
  pdl_wait();
  const SatLevel& L = b.lv[blockIdx.y];
  int64_t n = (int64_t)L.w * L.h;
  int qm = 1 << 20;
  double acc = 0.0;
  // eight independent loads per thread per step (the level is streamed once)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += 8 * stride) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t i = base + k * stride;
      v[k] = i < n ? __ldg(L.img + i) : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      qm = min(qm, log2_quantum(v[k]));
      acc += (double)fabsf(v[k]);
    }
  }
  for (int off = 16; off; off >>= 1) {
    qm = min(qm, __shfl_down_sync(0xffffffff, qm, off));
    acc += __shfl_down_sync(0xffffffff, acc, off);
  }
  __shared__ int sq[8];
  __shared__ double sa[8];
  int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sq[warp] = qm; sa[warp] = acc; }
  __syncthreads();
  if (threadIdx.x == 0) {  // one atomic pair per block
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) { qm = min(qm, sq[k]); acc += sa[k]; }
    atomicMin(&b.qmin[blockIdx.y], qm);
    atomicAdd(&b.sums[blockIdx.y], acc);
  }
}

void launch_level_stats(const SatBatch& b, int max_pixels, cudaStream_t s, bool precleared) {
  if (!precleared) {
    cudaMemsetAsync(b.sums, 0, sizeof(double) * 5, s);
    cudaMemsetAsync(b.qmin, 0x3f, sizeof(int32_t) * 5, s);  // large positive
  }
  // two blocks per SM per level: each thread streams its share in steps of
  // eight independent loads, and a level costs only ~300 same-address atomics
  int bx = std::min(grid_for(max_pixels, 256), 148 * 2);
  dim3 g(bx, b.n);
  klaunch(level_stats_kernel, g, 256, 0, s, b);
}

__global__ void __launch_bounds__(32) sat_cols_kernel(SatBatch b) {
  pdl_wait();
  const SatLevel& L = b.lv[blockIdx.y];
  if (level_exact(b, blockIdx.y)) return;  // the tile-local detector handles it
  int x = blockIdx.x * 32 + threadIdx.x;
  if (blockIdx.x * 32 >= L.w) return;
  bool live = x < L.w;
  const float* col = L.img + (live ? x : 0);
  int64_t w = L.w;
  int h = L.h;
  float cur[kSatPrefetch];
#pragma unroll
  for (int k = 0; k < kSatPrefetch; ++k) cur[k] = (live && k < h) ? __ldg(col + k * w) : 0.0f;
  double acc = 0.0;
  for (int y0 = 0; y0 < h; y0 += kSatPrefetch) {
    float nxt[kSatPrefetch];
#pragma unroll
    for (int k = 0; k < kSatPrefetch; ++k) {
      int y = y0 + kSatPrefetch + k;
      nxt[k] = (live && y < h) ? __ldg(col + (int64_t)y * w) : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < kSatPrefetch; ++k) {
      int y = y0 + k;
      if (y < h) {
        acc = dadd(acc, (double)cur[k]);
        int ri = L.rowmap[y + 1];
        if (ri >= 0 && live) L.ctab[(int64_t)ri * w + x] = acc;
      }
    }
#pragma unroll
    for (int k = 0; k < kSatPrefetch; ++k) cur[k] = nxt[k];
  }
}

// pass 2: one warp per 32 stored rows; lane r scans row r. 32x32 tiles are
// staged through shared memory so the global loads stay coalesced, and the
// next tile is prefetched into registers while the current one is scanned.
__global__ void __launch_bounds__(32) sat_rows_kernel(SatBatch b) {
  pdl_wait();
  const SatLevel& L = b.lv[blockIdx.y];
  if (level_exact(b, blockIdx.y)) return;
  __shared__ double tile[32][33];
  int lane = threadIdx.x;
  int r0 = blockIdx.x * 32;
  if (r0 >= L.nrows) return;
  int myr = r0 + lane;
  bool live = myr < L.nrows;
  int Y = live ? L.rowlist[myr] : -1;
  int64_t w = L.w;
  double* out = L.ltab + (int64_t)myr * L.ncols;
  if (live && L.colmap[0] >= 0) out[L.colmap[0]] = 0.0;
  auto load = [&](int c0, int r) -> double {
    int rr = r0 + r, c = c0 + lane;
    if (rr >= L.nrows || c >= L.w) return 0.0;
    return L.rowlist[rr] == 0 ? 0.0 : L.ctab[(int64_t)rr * w + c];
  };
  double pre[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) pre[r] = load(0, r);
  double acc = 0.0;
  for (int c0 = 0; c0 < L.w; c0 += 32) {
#pragma unroll
    for (int r = 0; r < 32; ++r) tile[r][lane] = pre[r];
    __syncwarp();
    if (c0 + 32 < L.w) {
#pragma unroll
      for (int r = 0; r < 32; ++r) pre[r] = load(c0 + 32, r);
    }
    int n = min(32, L.w - c0);
    for (int c = 0; c < n; ++c) {
      acc = dadd(acc, tile[lane][c]);
      int ci = L.colmap[c0 + c + 1];
      if (ci >= 0 && live) out[ci] = (Y == 0) ? 0.0 : acc;
    }
    __syncwarp();
  }
}

void launch_sat(const SatBatch& b, int max_w, int max_rows, cudaStream_t s) {
  dim3 g1(ceil_div(max_w, 32), b.n), g2(ceil_div(max_rows, 32), b.n);
  klaunch(sat_cols_kernel, g1, 32, 0, s, b);
  klaunch(sat_rows_kernel, g2, 32, 0, s, b);
}

// ---------------------------------------------------------------- K5
// matcher._quadrant_diffs + detect_corners (matcher.py:37-105). One block per
// tile (all pyramid levels in one launch); candidate (lx, ly) sits at
// t0 + spacing/2 + k*spacing.
struct LatticeView {
  const double* t;
  const int32_t* rm;
  const int32_t* cm;
  int ncols;
  __device__ __forceinline__ double at(int Y, int X) const {
    return t[(int64_t)rm[Y] * ncols + cm[X]];
  }
};

__device__ __forceinline__ double box(const LatticeView& v, int x0, int y0, int x1, int y1) {
  // ((t[y1,x1] - t[y0,x1]) - t[y1,x0]) + t[y0,x0]   (image.py:58)
  return dadd(dsub(dsub(v.at(y1, x1), v.at(y0, x1)), v.at(y1, x0)), v.at(y0, x0));
}

template <bool EXACT>
__global__ void __launch_bounds__(256) detect_kernel(SatBatch b, DetectParams dp) {
  pdl_wait();
  extern __shared__ double local_sat[];
  int lev = 0;
  while (lev + 1 < b.n && (int)blockIdx.x >= b.lv[lev + 1].tile_base) ++lev;
  if ((dp.exact_ok && level_exact(b, lev)) != EXACT) return;
  const SatLevel& L = b.lv[lev];
  int w = L.w, h = L.h, tile = dp.tile, half = dp.half;
  int tiles_x = ceil_div(w, tile);
  int tid_tile = blockIdx.x - L.tile_base;
  int t0x = (tid_tile % tiles_x) * tile, t0y = (tid_tile / tiles_x) * tile;
  int sp = tile / 16 > 1 ? tile / 16 : 1;
  int first = sp / 2;
  int limx = min(tile, w - t0x), limy = min(tile, h - t0y);
  int nx = limx > first ? (limx - first + sp - 1) / sp : 0;
  int ny = limy > first ? (limy - first + sp - 1) / sp : 0;
  // Exact path: the quadrant sums straight from the pixels, separably. Under
  // the level's exactness certificate (every partial sum of the level is
  // exactly representable) any summation order gives numpy's SAT
  // differences bit for bit, so the sums are formed in parallel: candidate
  // x's quadrant columns start at x - half (m < nx) or x (m = nx + lx), rows
  // likewise; H[r][m] sums `half` pixels of row r from column start m, V[n][m]
  // sums `half` rows of H -- tl = V[ly][lx], tr = V[ly][nx+lx],
  // bl = V[ny+ly][lx], br = V[ny+ly][nx+lx] (image.py:47-58).
  double* Vs = local_sat;                                   // [2ny][2nx]
  double* Hs = local_sat + 32 * 32;                         // [rows][2nx]
  float* img_s = reinterpret_cast<float*>(Hs + (tile + 2 * half) * 32);  // [rows][cols]
  const int ry0 = t0y + first - half, rx0 = t0x + first - half;
  const int rows = ny > 0 ? (ny - 1) * sp + 2 * half : 0;
  const int cols = nx > 0 ? (nx - 1) * sp + 2 * half : 0;
  const int NX = 2 * nx, NY = 2 * ny;
  if (EXACT && nx > 0 && ny > 0) {
    // rows by warp, columns by lane: no integer division per element, and
    // all of a thread's loads are issued before the first store
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    // groups of 4 rows x 3 column steps: 12 loads in flight per thread
    for (int rb = wid; rb < rows; rb += 4 * nwarp) {
      float v[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        int r = rb + (k / 3) * nwarp, c = lane + (k % 3) * 32;
        int y = ry0 + r, x = rx0 + c;
        v[k] = (r < rows && c < cols && y >= 0 && y < h && x >= 0 && x < w)
                   ? __ldg(L.img + (int64_t)y * w + x) : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        int r = rb + (k / 3) * nwarp, c = lane + (k % 3) * 32;
        if (r < rows && c < cols) img_s[r * cols + c] = v[k];
      }
    }
    for (int r = wid; r < rows; r += nwarp)  // columns beyond 96 (tile + 2 half > 96)
      for (int c = lane + 96; c < cols; c += 32) {
        int y = ry0 + r, x = rx0 + c;
        img_s[r * cols + c] = (y >= 0 && y < h && x >= 0 && x < w) ? L.img[(int64_t)y * w + x] : 0.0f;
      }
    __syncthreads();
    // H[r][m]: warp per row, lane per column start (NX <= 32)
    for (int r = wid; r < rows; r += nwarp)
      if (lane < NX) {
        int c0 = lane < nx ? lane * sp : (lane - nx) * sp + half;
        const float* row = img_s + r * cols + c0;
        double acc = 0.0;
        for (int k = 0; k < half; ++k) acc += (double)row[k];
        Hs[r * NX + lane] = acc;
      }
    __syncthreads();
    for (int n = wid; n < NY; n += nwarp)
      if (lane < NX) {
        int q0 = n < ny ? n * sp : (n - ny) * sp + half;
        double acc = 0.0;
        for (int k = 0; k < half; ++k) acc += Hs[(q0 + k) * NX + lane];
        Vs[n * NX + lane] = acc;
      }
    __syncthreads();
  }
  LatticeView v{L.ltab, L.rowmap, L.colmap, L.ncols};
  // ((t[y1,x1] - t[y0,x1]) - t[y1,x0]) + t[y0,x0]   (image.py:58)
  auto box = [&](int x0, int y0, int x1, int y1) -> double {
    return dadd(dsub(dsub(v.at(y1, x1), v.at(y0, x1)), v.at(y1, x0)), v.at(y0, x0));
  };
  double area = (double)(half * half);
  double best = -1.0;
  int best_i = 0x7fffffff;
  // candidate (lx, ly) = (tid & 15, tid >> 4): nx, ny <= 16 (tile / 16 spacing)
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    int lx = t & 15, ly = t >> 4;
    if (lx >= nx || ly >= ny) continue;
    int i = ly * nx + lx;  // row-major candidate index (tie-break order)
    int x = t0x + first + lx * sp, y = t0y + first + ly * sp;
    if (x < half || x > w - half || y < half || y > h - half) continue;
    double tl, tr, br, bl;
    if (EXACT) {
      tl = Vs[ly * NX + lx] / area;
      tr = Vs[ly * NX + nx + lx] / area;
      bl = Vs[(ny + ly) * NX + lx] / area;
      br = Vs[(ny + ly) * NX + nx + lx] / area;
    } else {
      tl = box(x - half, y - half, x, y) / area;
      tr = box(x, y - half, x + half, y) / area;
      br = box(x, y, x + half, y + half) / area;
      bl = box(x - half, y, x, y + half) / area;
    }
    double d0 = fabs(dsub(tr, tl)), d1 = fabs(dsub(br, tr));
    double d2 = fabs(dsub(bl, br)), d3 = fabs(dsub(tl, bl));
    double lo = fmin(fmin(d0, d1), fmin(d2, d3));
    if (!(lo > dp.threshold)) continue;
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
    L.tiles[tid_tile] = tc;
  }
}

// V [32][32] + H [tile + 2 half][32] doubles + the pixel region (f32)
size_t detect_exact_smem(int tile, int half) {
  size_t side = (size_t)tile + 2 * (size_t)half;
  return (32 * 32 + side * 32) * sizeof(double) + side * side * sizeof(float);
}

void init_raster_attributes() { allow_max_dynamic_smem(detect_kernel<true>); }

void launch_detect(const SatBatch& b, int total_tiles, const DetectParams& dp, cudaStream_t s) {
  if (dp.exact_ok)
    klaunch(detect_kernel<true>, total_tiles, 256, detect_exact_smem(dp.tile, dp.half), s, b, dp);
  klaunch(detect_kernel<false>, total_tiles, 256, 0, s, b, dp);
}

__global__ void __launch_bounds__(1024) compact_corners_kernel(const TileCorner* __restrict__ tiles,
                                                               int ntiles, double* __restrict__ out,
                                                               int32_t* __restrict__ count) {
  pdl_wait();
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
  klaunch(compact_corners_kernel, 1, 1024, 0, s, tiles, ntiles, corners, count);
}

}  // namespace hdr

namespace hdr {

// matcher.cornerness (matcher.py:51-61) for n points of a dense (h+1, w+1)
// f64 integral table: out[2i] = C = ((d0 + d1) + d2) + d3, out[2i+1] = min.
__global__ void cornerness_kernel(const double* __restrict__ t, int w1, const int32_t* __restrict__ xy,
                                  int n, int half, double* __restrict__ out) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x = xy[2 * i], y = xy[2 * i + 1];
  auto rect = [&](int x0, int y0, int x1, int y1) {  // image.py:58
    return dadd(dsub(dsub(t[(int64_t)y1 * w1 + x1], t[(int64_t)y0 * w1 + x1]), t[(int64_t)y1 * w1 + x0]),
                t[(int64_t)y0 * w1 + x0]);
  };
  double area = (double)(half * half);
  double tl = rect(x - half, y - half, x, y) / area, tr = rect(x, y - half, x + half, y) / area;
  double br = rect(x, y, x + half, y + half) / area, bl = rect(x - half, y, x, y + half) / area;
  double d0 = fabs(dsub(tr, tl)), d1 = fabs(dsub(br, tr)), d2 = fabs(dsub(bl, br)), d3 = fabs(dsub(tl, bl));
  out[2 * i] = dadd(dadd(dadd(d0, d1), d2), d3);
  out[2 * i + 1] = fmin(fmin(d0, d1), fmin(d2, d3));
}

void launch_cornerness(const double* table, int w1, const int32_t* xy, int n, int half, double* out,
                       cudaStream_t s) {
  if (n > 0) klaunch(cornerness_kernel, (n + 127) / 128, 128, 0, s, table, w1, xy, n, half, out);
}

}  // namespace hdr
