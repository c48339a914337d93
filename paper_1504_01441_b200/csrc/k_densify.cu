// Sparse-to-dense flow: splat (K9), domain-transform recursive filter (K10),
// densify-finalise fused with the bilinear backward warp, luminance of the
// warped frame and its histogram (K11 + K12).
#include "hdr_common.cuh"
#include "hdr_internal.h"

namespace hdr {

// ---------------------------------------------------------------- K9
// densify.build_sparse_maps (densify.py:38-56): collisions keep the lowest
// (score, index). Single block, four phases separated by block barriers.
__device__ __forceinline__ unsigned long long ordered_bits(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__global__ void __launch_bounds__(1024) splat_kernel(const double* __restrict__ m,
                                                     const int32_t* __restrict__ count,
                                                     int m_static, int w, int h,
                                                     double* __restrict__ pu,
                                                     double* __restrict__ pv,
                                                     double* __restrict__ pn,
                                                     unsigned long long* __restrict__ key,
                                                     int32_t* __restrict__ idx,
                                                     int32_t* __restrict__ status) {
  int n = count ? *count : m_static;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xr = m[5 * (int64_t)i], yr = m[5 * (int64_t)i + 1];
    double xf = rint(xr), yf = rint(yr);  // int(round()) half-even
    if (!(xf >= 0 && xf < w && yf >= 0 && yf < h)) {
      if (status) atomicExch(status, 1);
      continue;
    }
    int64_t p = (int64_t)yf * w + (int64_t)xf;
    key[p] = ~0ULL;
    idx[p] = 0x7fffffff;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xf = rint(m[5 * (int64_t)i]), yf = rint(m[5 * (int64_t)i + 1]);
    if (!(xf >= 0 && xf < w && yf >= 0 && yf < h)) continue;
    atomicMin(&key[(int64_t)yf * w + (int64_t)xf], ordered_bits(m[5 * (int64_t)i + 4]));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double xf = rint(m[5 * (int64_t)i]), yf = rint(m[5 * (int64_t)i + 1]);
    if (!(xf >= 0 && xf < w && yf >= 0 && yf < h)) continue;
    int64_t p = (int64_t)yf * w + (int64_t)xf;
    if (key[p] == ordered_bits(m[5 * (int64_t)i + 4])) atomicMin(&idx[p], i);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double* r = m + 5 * (int64_t)i;
    double xf = rint(r[0]), yf = rint(r[1]);
    if (!(xf >= 0 && xf < w && yf >= 0 && yf < h)) continue;
    int64_t p = (int64_t)yf * w + (int64_t)xf;
    if (idx[p] != i) continue;
    pu[p] = r[2] - r[0];
    pv[p] = r[3] - r[1];
    pn[p] = 1.0;
  }
}

void launch_splat(const double* matches, const int32_t* count, int m_static, int w, int h,
                  double* pu, double* pv, double* pn, uint64_t* scratch_key,
                  int32_t* scratch_idx, int32_t* status, cudaStream_t s) {
  size_t plane = (size_t)w * h * sizeof(double);
  cudaMemsetAsync(pu, 0, plane, s);
  cudaMemsetAsync(pv, 0, plane, s);
  cudaMemsetAsync(pn, 0, plane, s);
  splat_kernel<<<1, 1024, 0, s>>>(matches, count, m_static, w, h, pu, pv, pn,
                                  reinterpret_cast<unsigned long long*>(scratch_key),
                                  scratch_idx, status);
}

// ---------------------------------------------------------------- K10
// densify.dt_filter (densify.py:78-113). One pass = forward+backward along
// rows, then forward+backward along columns, every step
//   b[i] += a * (b[i-1] - b[i])            (densify.py:69-75)
// with a = exp(c_i * (1 + (sigma_s/sigma_r) |g[i+1] - g[i]|)).
// Both axes are split into chunks; a chunk's effect on the carry is the
// affine map (A, B) of its zero-carry run, chunks are linked by composing
// those maps, and each chunk is then re-run with its true carry-in using the
// reference's own update formula.
constexpr int kPlanes = 3;

struct Affine {
  double A;
  double B[kPlanes];
};

__device__ __forceinline__ Affine compose(const Affine& first, const Affine& then) {
  Affine r;
  r.A = then.A * first.A;
#pragma unroll
  for (int k = 0; k < kPlanes; ++k) r.B[k] = then.A * first.B[k] + then.B[k];
  return r;
}

__device__ __forceinline__ Affine shfl_up_aff(const Affine& v, int off) {
  Affine r;
  r.A = __shfl_up_sync(0xffffffff, v.A, off);
#pragma unroll
  for (int k = 0; k < kPlanes; ++k) r.B[k] = __shfl_up_sync(0xffffffff, v.B[k], off);
  return r;
}

__device__ __forceinline__ double dt_coef(float g0, float g1, double ratio, double c) {
  double d = 1.0 + ratio * fabs((double)g1 - (double)g0);
  return exp(c * d);
}

// Row pass: one block per row, the row's planes resident in shared memory.
template <int K>
__global__ void __launch_bounds__(256) dt_rows_kernel(const float* __restrict__ guide,
                                                      double* __restrict__ planes, int w, int h,
                                                      double ratio, double c) {
  extern __shared__ double sm[];
  double* xs = sm;            // K * w
  double* av = sm + K * w;    // w (a between i and i+1; av[w-1] = 0)
  __shared__ Affine wsum[32];
  int y = blockIdx.x;
  int64_t P = (int64_t)w * h;
  const float* g = guide + (int64_t)y * w;
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) xs[k * w + i] = planes[k * P + (int64_t)y * w + i];
    av[i] = (i + 1 < w) ? dt_coef(g[i], g[i + 1], ratio, c) : 0.0;
  }
  __syncthreads();
  int T = blockDim.x;
  int L = (w + T - 1) / T;
  int s0 = threadIdx.x * L, s1 = min(w, s0 + L);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
  for (int dir = 0; dir < 2; ++dir) {
    // segment map with zero carry
    Affine m;
    m.A = 1.0;
#pragma unroll
    for (int k = 0; k < K; ++k) m.B[k] = 0.0;
    if (dir == 0) {
      for (int i = s0; i < s1; ++i) {
        double a = i > 0 ? av[i - 1] : 0.0;
        m.A *= a;
#pragma unroll
        for (int k = 0; k < K; ++k) { double x = xs[k * w + i]; m.B[k] = x + a * (m.B[k] - x); }
      }
    } else {
      for (int i = s1 - 1; i >= s0; --i) {
        double a = av[i];
        m.A *= a;
#pragma unroll
        for (int k = 0; k < K; ++k) { double x = xs[k * w + i]; m.B[k] = x + a * (m.B[k] - x); }
      }
    }
    // exclusive scan of segment maps in processing order
    int rank = dir == 0 ? threadIdx.x : T - 1 - threadIdx.x;
    (void)rank;
    Affine inc = m;
    if (dir == 0) {
      for (int off = 1; off < 32; off <<= 1) {
        Affine o = shfl_up_aff(inc, off);
        if (lane >= off) inc = compose(o, inc);
      }
    } else {
      for (int off = 1; off < 32; off <<= 1) {
        Affine o;
        o.A = __shfl_down_sync(0xffffffff, inc.A, off);
#pragma unroll
        for (int k = 0; k < K; ++k) o.B[k] = __shfl_down_sync(0xffffffff, inc.B[k], off);
        if (lane + off < 32) inc = compose(o, inc);
      }
    }
    if ((dir == 0 && lane == 31) || (dir == 1 && lane == 0)) wsum[warp] = inc;
    __syncthreads();
    // carry into this thread's segment: all earlier segments (in scan order)
    Affine pre;
    pre.A = 1.0;
#pragma unroll
    for (int k = 0; k < K; ++k) pre.B[k] = 0.0;
    if (dir == 0) {
      for (int j = 0; j < warp; ++j) pre = compose(pre, wsum[j]);
      Affine o = shfl_up_aff(inc, 1);
      if (lane > 0) pre = compose(pre, o);
    } else {
      for (int j = nw - 1; j > warp; --j) pre = compose(pre, wsum[j]);
      Affine o;
      o.A = __shfl_down_sync(0xffffffff, inc.A, 1);
#pragma unroll
      for (int k = 0; k < K; ++k) o.B[k] = __shfl_down_sync(0xffffffff, inc.B[k], 1);
      if (lane < 31) pre = compose(pre, o);
    }
    __syncthreads();
    // re-run with the true carry (pre.B = value just before the segment)
    double prev[K];
#pragma unroll
    for (int k = 0; k < K; ++k) prev[k] = pre.B[k];
    if (dir == 0) {
      for (int i = s0; i < s1; ++i) {
        double a = i > 0 ? av[i - 1] : 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          double x = xs[k * w + i];
          double v = x + a * (prev[k] - x);
          xs[k * w + i] = v;
          prev[k] = v;
        }
      }
    } else {
      for (int i = s1 - 1; i >= s0; --i) {
        double a = av[i];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          double x = xs[k * w + i];
          double v = x + a * (prev[k] - x);
          xs[k * w + i] = v;
          prev[k] = v;
        }
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < w; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) planes[k * P + (int64_t)y * w + i] = xs[k * w + i];
}

// Column pass, three kernels per direction over (column, row-chunk) threads.
constexpr int kChunk = 64;

template <int K>
__device__ __forceinline__ double col_coef(const float* g, int64_t w, int y, int x, int h,
                                           double ratio, double c) {
  return (y + 1 < h) ? dt_coef(g[(int64_t)y * w + x], g[(int64_t)(y + 1) * w + x], ratio, c) : 0.0;
}

// phase 1: zero-carry map of each chunk -> carry[(chunk, col)]
template <int K>
__global__ void dt_cols_local(const float* __restrict__ guide, const double* __restrict__ planes,
                              int w, int h, double ratio, double c, int dir,
                              double* __restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y;
  if (x >= w) return;
  int64_t P = (int64_t)w * h;
  int r0 = ch * kChunk, r1 = min(h, r0 + kChunk);
  double A = 1.0, B[K];
#pragma unroll
  for (int k = 0; k < K; ++k) B[k] = 0.0;
  if (dir == 0) {
    for (int y = r0; y < r1; ++y) {
      double a = y > 0 ? col_coef<K>(guide, w, y - 1, x, h, ratio, c) : 0.0;
      A *= a;
#pragma unroll
      for (int k = 0; k < K; ++k) { double v = planes[k * P + (int64_t)y * w + x]; B[k] = v + a * (B[k] - v); }
    }
  } else {
    for (int y = r1 - 1; y >= r0; --y) {
      double a = col_coef<K>(guide, w, y, x, h, ratio, c);
      A *= a;
#pragma unroll
      for (int k = 0; k < K; ++k) { double v = planes[k * P + (int64_t)y * w + x]; B[k] = v + a * (B[k] - v); }
    }
  }
  int nch = gridDim.y;
  double* o = carry + ((int64_t)ch * w + x) * (K + 1);
  o[0] = A;
#pragma unroll
  for (int k = 0; k < K; ++k) o[1 + k] = B[k];
  (void)nch;
}

// phase 2: per column, link chunks in scan order; carry becomes carry-in
template <int K>
__global__ void dt_cols_link(int w, int nch, int dir, double* __restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  double cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k) cur[k] = 0.0;
  for (int t = 0; t < nch; ++t) {
    int ch = dir == 0 ? t : nch - 1 - t;
    double* o = carry + ((int64_t)ch * w + x) * (K + 1);
    double A = o[0];
    double nxt[K];
#pragma unroll
    for (int k = 0; k < K; ++k) nxt[k] = A * cur[k] + o[1 + k];
#pragma unroll
    for (int k = 0; k < K; ++k) { o[1 + k] = cur[k]; cur[k] = nxt[k]; }
  }
}

// phase 3: re-run each chunk from its carry-in, in place
template <int K>
__global__ void dt_cols_apply(const float* __restrict__ guide, double* __restrict__ planes, int w,
                              int h, double ratio, double c, int dir,
                              const double* __restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y;
  if (x >= w) return;
  int64_t P = (int64_t)w * h;
  int r0 = ch * kChunk, r1 = min(h, r0 + kChunk);
  const double* o = carry + ((int64_t)ch * w + x) * (K + 1);
  double prev[K];
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = o[1 + k];
  if (dir == 0) {
    for (int y = r0; y < r1; ++y) {
      double a = y > 0 ? col_coef<K>(guide, w, y - 1, x, h, ratio, c) : 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double* p = planes + k * P + (int64_t)y * w + x;
        double v = *p;
        v = v + a * (prev[k] - v);
        *p = v;
        prev[k] = v;
      }
    }
  } else {
    for (int y = r1 - 1; y >= r0; --y) {
      double a = col_coef<K>(guide, w, y, x, h, ratio, c);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double* p = planes + k * P + (int64_t)y * w + x;
        double v = *p;
        v = v + a * (prev[k] - v);
        *p = v;
        prev[k] = v;
      }
    }
  }
}

template <int K>
static void dt_filter_k(const float* guide, double* planes, int w, int h, double sigma_s,
                        double sigma_r, int passes, double* carry, cudaStream_t s) {
  double ratio = sigma_s / sigma_r;
  double root = sqrt(2.0);
  double den = sqrt(pow(4.0, passes) - 1.0);
  size_t row_smem = (size_t)(K + 1) * w * sizeof(double);
  int nch = ceil_div(h, kChunk);
  dim3 cg(ceil_div(w, 128), nch);
  for (int i = 1; i <= passes; ++i) {
    double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;
    double c = -root / sigma_i;
    if (w > 1) dt_rows_kernel<K><<<h, 256, row_smem, s>>>(guide, planes, w, h, ratio, c);
    if (h > 1) {
      for (int dir = 0; dir < 2; ++dir) {
        dt_cols_local<K><<<cg, 128, 0, s>>>(guide, planes, w, h, ratio, c, dir, carry);
        dt_cols_link<K><<<ceil_div(w, 128), 128, 0, s>>>(w, nch, dir, carry);
        dt_cols_apply<K><<<cg, 128, 0, s>>>(guide, planes, w, h, ratio, c, dir, carry);
      }
    }
  }
}

void init_densify_attributes() {
  int cap = 227 * 1024;
  cudaFuncSetAttribute(dt_rows_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
  cudaFuncSetAttribute(dt_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
  cudaFuncSetAttribute(dt_rows_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

void launch_dt_filter(const float* guide, double* planes, int k, int w, int h, double sigma_s,
                      double sigma_r, int passes, double* carry, cudaStream_t s) {
  switch (k) {
    case 1: dt_filter_k<1>(guide, planes, w, h, sigma_s, sigma_r, passes, carry, s); break;
    case 2: dt_filter_k<2>(guide, planes, w, h, sigma_s, sigma_r, passes, carry, s); break;
    default: dt_filter_k<3>(guide, planes, w, h, sigma_s, sigma_r, passes, carry, s); break;
  }
}

// ---------------------------------------------------------------- K11/K12
// geometry.homography_pixel_flow (geometry.py:124-135) at one pixel, f32.
__device__ __forceinline__ void h_pixel_flow(const double* H, int x, int y, int w, int h,
                                             float* fu, float* fv) {
  double xn, yn, nx, ny;
  to_norm((double)x, (double)y, w, h, &xn, &yn);
  double den = apply_h(H, xn, yn, &nx, &ny);
  bool bad = fabs(den) < 1e-12;
  double safe = bad ? 1.0 : den;
  double px, py;
  from_norm(nx / safe, ny / safe, w, h, &px, &py);
  *fu = bad ? 0.0f : (float)dsub(px, (double)x);
  *fv = bad ? 0.0f : (float)dsub(py, (double)y);
}

__global__ void hflow_kernel(const double* __restrict__ Hd, int w, int h, float* __restrict__ flow) {
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
  hflow_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(H, w, h, flow);
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
// do_flow = false: flow is an input (warp_image alone).
__global__ void __launch_bounds__(256) finalize_warp_kernel(
    const double* __restrict__ smooth, const double* __restrict__ fallback,
    const int32_t* __restrict__ has_fb, int w, int h, double floor_,
    const float* __restrict__ src, int channels, float* __restrict__ flow,
    float* __restrict__ warped, uint8_t* __restrict__ valid, uint8_t* __restrict__ qw,
    uint32_t* __restrict__ hist, bool do_flow) {
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
      double n = smooth[2 * P + i];
      if (n > floor_) {
        fu = (float)(smooth[i] / n);
        fv = (float)(smooth[P + i] / n);
      } else if (use_fb) {
        h_pixel_flow(H, x, y, w, h, &fu, &fv);
      } else {
        fu = 0.0f;
        fv = 0.0f;
      }
      reinterpret_cast<float2*>(flow)[i] = make_float2(fu, fv);
      if (!warped) continue;
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
    float o[3];
    for (int k = 0; k < channels; ++k) {
      double top = dadd(dmul((double)s00[k], gx), dmul((double)s01[k], fx));
      double bot = dadd(dmul((double)s10[k], gx), dmul((double)s11[k], fx));
      o[k] = (float)dadd(dmul(top, gy), dmul(bot, fy));
      warped[i * channels + k] = o[k];
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

void launch_finalize_warp(const double* smooth, const double* fallback,
                          const int32_t* has_fallback, int w, int h, double floor_,
                          const float* src, int channels, float* flow, float* warped,
                          uint8_t* valid, uint8_t* qw, uint32_t* hist_w, bool do_flow,
                          cudaStream_t s) {
  int64_t P = (int64_t)w * h;
  int64_t blocks = (P + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  finalize_warp_kernel<<<(unsigned)blocks, 256, 0, s>>>(smooth, fallback, has_fallback, w, h,
                                                        floor_, src, channels, flow, warped,
                                                        valid, qw, hist_w, do_flow);
}

}  // namespace hdr
