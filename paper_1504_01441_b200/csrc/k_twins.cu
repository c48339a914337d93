// Stage twins outside the pair's hot path: the general forms of reference
// functions whose pair-pipeline kernels are specialised (single-channel f32
// guide, <= 3 planes, rows that fit in shared memory, RGB frames), plus the
// small geometry/raster helpers a user of the reference calls directly.
//
//   dt_rows_seq / dt_cols_seq  densify.dt_filter (densify.py:59-113) for any
//                              guide (f32 or f64, any channel count), any
//                              plane count and any width: one thread per
//                              (line, plane) runs the reference's recursion
//                              (densify.py:69-75) sequentially, so results
//                              follow numpy's rounding step for step. The
//                              f32 single-channel instance is also the pair
//                              pipeline's row pass for rows too wide for the
//                              shared-memory row kernels.
//   rect_sum                   image.rect_sum (image.py:47-58), batched.
//   quantize_256               image.quantize_256 (image.py:91-93).
//   downsample_ch              image.downsample (image.py:61-68), interleaved
//                              channels, f32 or f64 input.
//   apply_homography           geometry.apply_homography (geometry.py:80-93).
//   transfer_error             geometry.symmetric_transfer_error
//                              (geometry.py:96-115).
#include "hdr_common.cuh"
#include "hdr_geom.cuh"
#include "hdr_internal.h"
#include "hdr_planes.cuh"

namespace hdr {

// ---------------------------------------------------------------- dt_filter
// sum over channels of |g1 - g0| in f64 with numpy's pairwise summation
// (np.abs(np.diff(g)).sum(axis=2), densify.py:63-64): a plain running sum
// from 0 below 8 terms, eight interleaved partial sums from 8 on
template <typename GT>
__device__ __forceinline__ double absdiff_sum(const GT* g0, const GT* g1, int C) {
  auto term = [&](int i) { return fabs(dsub((double)g1[i], (double)g0[i])); };
  if (C < 8) {
    double s = 0.0;
    for (int i = 0; i < C; ++i) s = dadd(s, term(i));
    return s;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = term(j);
  int i = 8;
  for (; i < C - (C % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], term(i + j));
  double s = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < C; ++i) s = dadd(s, term(i));
  return s;
}

// exp(c * (1 + ratio * sum|dg|)), separately rounded as numpy evaluates it
// (densify.py:65-66 and :105-106)
template <typename GT>
__device__ __forceinline__ double seq_coef(const GT* g0, const GT* g1, int C, double ratio,
                                           double c) {
  return exp(dmul(c, dadd(1.0, dmul(ratio, absdiff_sum(g0, g1, C)))));
}

// b[i] += a * (b[i-1] - b[i])
__device__ __forceinline__ double seq_step(double x, double prev, double a) {
  return dadd(x, dmul(a, dsub(prev, x)));
}

template <typename GT>
__global__ void __launch_bounds__(128) dt_rows_seq_kernel(const GT* __restrict__ guide, int C,
                                                          DtPlanes P, int w, int h, double ratio,
                                                          double c) {
  pdl_wait();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)h * P.k) return;
  const int k = (int)(t / h), y = (int)(t - (int64_t)k * h);
  const int64_t row = (int64_t)y * w;
  const GT* g = guide + row * C;
  double prev = ldp(P, k, row);
  for (int i = 1; i < w; ++i) {
    prev = seq_step(ldp(P, k, row + i), prev, seq_coef(g + (int64_t)(i - 1) * C, g + (int64_t)i * C, C, ratio, c));
    stp(P, k, row + i, prev);
  }
  for (int i = w - 2; i >= 0; --i) {
    prev = seq_step(ldp(P, k, row + i), prev, seq_coef(g + (int64_t)i * C, g + (int64_t)(i + 1) * C, C, ratio, c));
    stp(P, k, row + i, prev);
  }
}

template <typename GT>
__global__ void __launch_bounds__(128) dt_cols_seq_kernel(const GT* __restrict__ guide, int C,
                                                          DtPlanes P, int w, int h, double ratio,
                                                          double c) {
  pdl_wait();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)w * P.k) return;
  const int k = (int)(t / w), x = (int)(t - (int64_t)k * w);
  const int64_t W = w, WC = (int64_t)w * C;
  const GT* g = guide + (int64_t)x * C;
  double prev = ldp(P, k, x);
  for (int y = 1; y < h; ++y) {
    prev = seq_step(ldp(P, k, y * W + x), prev, seq_coef(g + (y - 1) * WC, g + y * WC, C, ratio, c));
    stp(P, k, y * W + x, prev);
  }
  for (int y = h - 2; y >= 0; --y) {
    prev = seq_step(ldp(P, k, y * W + x), prev, seq_coef(g + y * WC, g + (y + 1) * WC, C, ratio, c));
    stp(P, k, y * W + x, prev);
  }
}

void launch_dt_rows_seq(const float* guide, const DtPlanes& P, int w, int h, double ratio, double c,
                        cudaStream_t s) {
  int64_t n = (int64_t)h * P.k;
  klaunch(dt_rows_seq_kernel<float>, (unsigned)((n + 127) / 128), 128, 0, s, guide, 1, P, w, h, ratio, c);
}

// the whole filter, densify.py:96-113 (sigma_i and c per pass as dt_filter_k)
template <typename GT>
static void dt_filter_seq(const GT* guide, int C, const DtPlanes& P, int w, int h, double sigma_s,
                          double sigma_r, int passes, cudaStream_t s) {
  const double ratio = sigma_s / sigma_r;
  const double root = sqrt(2.0);
  const double den = sqrt(pow(4.0, passes) - 1.0);
  for (int i = 1; i <= passes; ++i) {
    double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;
    double c = -root / sigma_i;
    if (w > 1) {
      int64_t n = (int64_t)h * P.k;
      klaunch(dt_rows_seq_kernel<GT>, (unsigned)((n + 127) / 128), 128, 0, s, guide, C, P, w, h, ratio, c);
    }
    if (h > 1) {
      int64_t n = (int64_t)w * P.k;
      klaunch(dt_cols_seq_kernel<GT>, (unsigned)((n + 127) / 128), 128, 0, s, guide, C, P, w, h, ratio, c);
    }
  }
}

void launch_dt_filter_general(const double* guide, int C, const DtPlanes& P, int w, int h,
                              double sigma_s, double sigma_r, int passes, cudaStream_t s) {
  dt_filter_seq<double>(guide, C, P, w, h, sigma_s, sigma_r, passes, s);
}

// ---------------------------------------------------------------- rect_sum
// table[y1, x1] - table[y0, x1] - table[y1, x0] + table[y0, x0], left to right
// (image.py:58); a query outside the table or with x0 > x1 / y0 > y1 raises
// in the reference (image.py:54-57): it sets *bad and reads nothing
__global__ void rect_sum_kernel(const double* __restrict__ t, int64_t w1, int64_t h1,
                                const int64_t* __restrict__ q, int64_t n, double* __restrict__ out,
                                int32_t* __restrict__ bad) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t x0 = q[i], y0 = q[n + i], x1 = q[2 * n + i], y1 = q[3 * n + i];
  if (x0 < 0 || y0 < 0 || x0 > x1 || y0 > y1 || x1 >= w1 || y1 >= h1) {
    atomicExch(bad, 1);
    return;
  }
  out[i] = dadd(dsub(dsub(t[y1 * w1 + x1], t[y0 * w1 + x1]), t[y1 * w1 + x0]), t[y0 * w1 + x0]);
}

void launch_rect_sum(const double* table, int64_t w1, int64_t h1, const int64_t* q, int64_t n,
                     double* out, int32_t* bad, cudaStream_t s) {
  if (n <= 0) return;
  klaunch(rect_sum_kernel, (unsigned)((n + 255) / 256), 256, 0, s, table, w1, h1, q, n, out, bad);
}

// ---------------------------------------------------------------- quantize_256
// clip(floor(x * 255.0 + 0.5), 0, 255) as uint8 (image.py:91-93): f32 inputs
// stay f32 (numpy's weak Python-float scalars), f64 inputs are f64
template <typename T>
__global__ void quantize_kernel(const T* __restrict__ x, int64_t n, uint8_t* __restrict__ out) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    T v;
    if constexpr (sizeof(T) == 4) v = floorf(fadd(fmul(x[i], 255.0f), 0.5f));
    else v = floor(dadd(dmul(x[i], 255.0), 0.5));
    // NaN clips to NaN in numpy and casts to 0 on x86; keep that
    out[i] = v != v ? 0 : (uint8_t)(v < (T)0 ? (T)0 : (v > (T)255 ? (T)255 : v));
  }
}

void launch_quantize(const void* x, bool f64, int64_t n, uint8_t* out, cudaStream_t s) {
  if (n <= 0) return;
  int64_t b = (n + 255) / 256;
  unsigned blocks = (unsigned)(b < 148 * 16 ? b : 148 * 16);
  if (f64) klaunch(quantize_kernel<double>, blocks, 256, 0, s, (const double*)x, n, out);
  else klaunch(quantize_kernel<float>, blocks, 256, 0, s, (const float*)x, n, out);
}

// ---------------------------------------------------------------- downsample
// (((v00 + v01) + v10) + v11) * 0.25 per channel of an interleaved (h, w, C)
// image, odd trailing row/column dropped (image.py:61-68). f32 input: f32
// arithmetic; f64 input: f64 arithmetic, then astype(float32).
template <typename T>
__global__ void downsample_ch_kernel(const T* __restrict__ in, int w, int h, int C,
                                     float* __restrict__ out) {
  pdl_wait();
  const int ow = w / 2, oh = h / 2;
  int64_t n = (int64_t)ow * oh * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int ch = (int)(i % C);
    int64_t p = i / C;
    int x = (int)(p % ow), y = (int)(p / ow);
    const T* r0 = in + ((int64_t)(2 * y) * w + 2 * x) * C + ch;
    const T* r1 = r0 + (int64_t)w * C;
    if constexpr (sizeof(T) == 4)
      out[i] = fmul(fadd(fadd(fadd(r0[0], r0[C]), r1[0]), r1[C]), 0.25f);
    else
      out[i] = (float)dmul(dadd(dadd(dadd(r0[0], r0[C]), r1[0]), r1[C]), 0.25);
  }
}

void launch_downsample_ch(const void* in, bool f64, int w, int h, int C, float* out, cudaStream_t s) {
  int64_t n = (int64_t)(w / 2) * (h / 2) * C;
  if (n <= 0) return;
  int64_t b = (n + 255) / 256;
  unsigned blocks = (unsigned)(b < 148 * 16 ? b : 148 * 16);
  if (f64) klaunch(downsample_ch_kernel<double>, blocks, 256, 0, s, (const double*)in, w, h, C, out);
  else klaunch(downsample_ch_kernel<float>, blocks, 256, 0, s, (const float*)in, w, h, C, out);
}

// ---------------------------------------------------------------- geometry
// apply_homography (geometry.py:80-93); *bad = 1 if any |denom| < 1e-12
__global__ void apply_h_kernel(const double* __restrict__ H, const double* __restrict__ pts, int64_t n,
                               double* __restrict__ out, int32_t* __restrict__ bad) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double Hs[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) Hs[k] = H[k];
  double nx, ny;
  double den = apply_h(Hs, pts[2 * i], pts[2 * i + 1], &nx, &ny);
  if (!(fabs(den) >= 1e-12)) atomicExch(bad, 1);
  out[2 * i] = nx / den;
  out[2 * i + 1] = ny / den;
}

void launch_apply_homography(const double* H, const double* pts, int64_t n, double* out, int32_t* bad,
                             cudaStream_t s) {
  if (n <= 0) return;
  klaunch(apply_h_kernel, (unsigned)((n + 255) / 256), 256, 0, s, H, pts, n, out, bad);
}

// symmetric_transfer_error (geometry.py:107-115): hypot(fwd, bwd) with
// h_inv = np.linalg.inv(h) (LU with partial pivoting, inv3); *bad = 1 when h
// is exactly singular (numpy raises LinAlgError)
__global__ void transfer_error_kernel(const double* __restrict__ H, const double* __restrict__ rp,
                                      const double* __restrict__ sp, int64_t n,
                                      double* __restrict__ out, int32_t* __restrict__ bad) {
  pdl_wait();
  __shared__ double Hs[18];
  __shared__ int okinv;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 9; ++k) Hs[k] = H[k];
    okinv = inv3(Hs, Hs + 9);
    if (!okinv && blockIdx.x == 0) *bad = 1;
  }
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !okinv) return;
  double f = transfer_dist(Hs, rp[2 * i], rp[2 * i + 1], sp[2 * i], sp[2 * i + 1]);
  double b = transfer_dist(Hs + 9, sp[2 * i], sp[2 * i + 1], rp[2 * i], rp[2 * i + 1]);
  out[i] = hypot(f, b);
}

void launch_transfer_error(const double* H, const double* rp, const double* sp, int64_t n, double* out,
                           int32_t* bad, cudaStream_t s) {
  unsigned blocks = n > 0 ? (unsigned)((n + 255) / 256) : 1;
  klaunch(transfer_error_kernel, blocks, 256, 0, s, H, rp, sp, n, out, bad);
}

}  // namespace hdr
