// Domain-transform recursive filter (K10): densify.dt_filter, densify.py:78-113.
//
// One pass = a forward+backward sweep along every row, then along every
// column; each step is the reference's update (densify.py:69-75)
//   b[i] += a * (b[i-1] - b[i]),   a = exp(c_pass * (1 + (sigma_s/sigma_r)|g[i+1]-g[i]|)).
//
// Rows: one block per row, the row resident in shared memory; the row is cut
//   into per-thread segments whose zero-carry effects are affine maps, the
//   maps are scanned across the block, and each segment is re-run from its
//   true carry with the reference formula. HBM: one read + one write.
// Columns: 32-row chunks. `agg` reads a chunk once and reduces it to the
//   affine data both directions need (forward map A,B and the backward
//   sums Z0 = sum (1-a_i) prod_{j<i} a_j y0_i, R for the carry's own
//   response, Q = prod a_i); `link` runs the two carry chains per column;
//   `apply` re-runs each chunk forward from its carry (writing y in place,
//   L2-resident) and backward from its carry (overwriting with z). HBM: two
//   reads + one write, instead of re-reading per direction.
// Planes may be stored f32 or f64 (DtPlanes::f64); all arithmetic is f64.
#include "hdr_common.cuh"
#include "hdr_internal.h"
#include "hdr_planes.cuh"

namespace hdr {

// a between samples with guide values g0, g1 (densify.py:59-66, :105-106)
__device__ __forceinline__ double dt_coef(float g0, float g1, double ratio, double c) {
  return exp(c * (1.0 + ratio * fabs((double)g1 - (double)g0)));
}

template <int K>
struct Aff {
  double A;
  double B[K];
};

template <int K>
__device__ __forceinline__ Aff<K> compose(const Aff<K>& first, const Aff<K>& then) {
  Aff<K> r;
  r.A = then.A * first.A;
#pragma unroll
  for (int k = 0; k < K; ++k) r.B[k] = then.A * first.B[k] + then.B[k];
  return r;
}

template <int K>
__device__ __forceinline__ Aff<K> shfl_aff(const Aff<K>& v, int off, bool up) {
  Aff<K> r;
  r.A = up ? __shfl_up_sync(0xffffffff, v.A, off) : __shfl_down_sync(0xffffffff, v.A, off);
#pragma unroll
  for (int k = 0; k < K; ++k)
    r.B[k] = up ? __shfl_up_sync(0xffffffff, v.B[k], off) : __shfl_down_sync(0xffffffff, v.B[k], off);
  return r;
}

// ---------------------------------------------------------------- rows
constexpr int kRowThreads = 256;

template <int K>
__global__ void __launch_bounds__(kRowThreads) dt_rows_kernel(const float* __restrict__ guide,
                                                              DtPlanes P, int w, int h,
                                                              double ratio, double c) {
  extern __shared__ double sm[];
  double* xs = sm;          // K * w
  double* av = sm + K * w;  // a between i and i+1; av[w-1] = 0
  __shared__ Aff<K> wsum[kRowThreads / 32];
  int y = blockIdx.x;
  int64_t row = (int64_t)y * w;
  const float* g = guide + row;
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) xs[k * w + i] = ldp(P, k, row + i);
    av[i] = (i + 1 < w) ? dt_coef(g[i], g[i + 1], ratio, c) : 0.0;
  }
  __syncthreads();
  const int T = blockDim.x;
  int L = (w + T - 1) / T;
  int s0 = threadIdx.x * L, s1 = min(w, s0 + L);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
#pragma unroll 1
  for (int dir = 0; dir < 2; ++dir) {
    // zero-carry map of this thread's segment
    Aff<K> m;
    m.A = 1.0;
#pragma unroll
    for (int k = 0; k < K; ++k) m.B[k] = 0.0;
    for (int t = 0; t < s1 - s0; ++t) {
      int i = dir == 0 ? s0 + t : s1 - 1 - t;
      double a = dir == 0 ? (i > 0 ? av[i - 1] : 0.0) : av[i];
      m.A *= a;
#pragma unroll
      for (int k = 0; k < K; ++k) { double x = xs[k * w + i]; m.B[k] = x + a * (m.B[k] - x); }
    }
    // inclusive scan of segment maps in processing order
    bool up = dir == 0;
    Aff<K> inc = m;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Aff<K> o = shfl_aff(inc, off, up);
      if (up ? lane >= off : lane + off < 32) inc = compose(o, inc);
    }
    if (lane == (up ? 31 : 0)) wsum[warp] = inc;
    __syncthreads();
    Aff<K> pre;
    pre.A = 1.0;
#pragma unroll
    for (int k = 0; k < K; ++k) pre.B[k] = 0.0;
    if (up) {
      for (int j = 0; j < warp; ++j) pre = compose(pre, wsum[j]);
    } else {
      for (int j = nw - 1; j > warp; --j) pre = compose(pre, wsum[j]);
    }
    Aff<K> o = shfl_aff(inc, 1, up);
    if (up ? lane > 0 : lane < 31) pre = compose(pre, o);
    __syncthreads();
    // re-run from the true carry (pre.B = the value just before the segment)
    double prev[K];
#pragma unroll
    for (int k = 0; k < K; ++k) prev[k] = pre.B[k];
    for (int t = 0; t < s1 - s0; ++t) {
      int i = dir == 0 ? s0 + t : s1 - 1 - t;
      double a = dir == 0 ? (i > 0 ? av[i - 1] : 0.0) : av[i];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double x = xs[k * w + i];
        double v = x + a * (prev[k] - x);
        xs[k * w + i] = v;
        prev[k] = v;
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < w; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) stp(P, k, row + i, xs[k * w + i]);
}

// ---------------------------------------------------------------- columns
constexpr int kColChunk = 32;

// coefficient between rows y and y+1 of column x (0 past the last row)
__device__ __forceinline__ double col_a(const float* g, int64_t w, int h, int y, int x,
                                        double ratio, double c) {
  return (y >= 0 && y + 1 < h) ? dt_coef(g[(int64_t)y * w + x], g[(int64_t)(y + 1) * w + x], ratio, c)
                               : 0.0;
}

// Aggregates, field-major: agg[f][chunk][col], f = A, Q, R, B[K], Z0[K]
template <int K>
__global__ void __launch_bounds__(64) dt_cols_agg(const float* __restrict__ guide, DtPlanes P,
                                                  int w, int h, double ratio, double c,
                                                  double* __restrict__ agg) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y, nch = gridDim.y;
  if (x >= w) return;
  int r0 = ch * kColChunk, r1 = min(h, r0 + kColChunk);
  double y0[K], z0[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { y0[k] = 0.0; z0[k] = 0.0; }
  double Pp = 1.0, R = 0.0, pref = 1.0;
  double a_prev = col_a(guide, w, h, r0 - 1, x, ratio, c);
#pragma unroll 8
  for (int y = r0; y < r1; ++y) {
    int64_t i = (int64_t)y * w + x;
    Pp *= a_prev;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double xv = ldp(P, k, i);
      y0[k] = xv + a_prev * (y0[k] - xv);
    }
    double a = col_a(guide, w, h, y, x, ratio, c);
    double wgt = (1.0 - a) * pref;
#pragma unroll
    for (int k = 0; k < K; ++k) z0[k] += wgt * y0[k];
    R += wgt * Pp;
    pref *= a;
    a_prev = a;
  }
  int64_t F = (int64_t)nch * w, o = (int64_t)ch * w + x;
  agg[o] = Pp;
  agg[F + o] = pref;
  agg[2 * F + o] = R;
#pragma unroll
  for (int k = 0; k < K; ++k) { agg[(3 + k) * F + o] = y0[k]; agg[(3 + K + k) * F + o] = z0[k]; }
}

// carries per column, field-major carry[f][chunk][col]: C_b[K] (value above
// chunk b), then D_b[K] (value below chunk b)
template <int K>
__global__ void dt_cols_link(int w, int nch, const double* __restrict__ agg,
                             double* __restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  int64_t F = (int64_t)nch * w;
  double C[K];
#pragma unroll
  for (int k = 0; k < K; ++k) C[k] = 0.0;
#pragma unroll 4
  for (int b = 0; b < nch; ++b) {
    int64_t o = (int64_t)b * w + x;
    double A = agg[o];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      carry[k * F + o] = C[k];
      C[k] = A * C[k] + agg[(3 + k) * F + o];
    }
  }
  double D[K];
#pragma unroll
  for (int k = 0; k < K; ++k) D[k] = 0.0;
#pragma unroll 4
  for (int b = nch - 1; b >= 0; --b) {
    int64_t o = (int64_t)b * w + x;
    double Q = agg[F + o], R = agg[2 * F + o];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      carry[(K + k) * F + o] = D[k];
      D[k] = agg[(3 + K + k) * F + o] + carry[k * F + o] * R + Q * D[k];  // z_s = Z0 + C*R + Q*D
    }
  }
}

// Re-run each chunk from its carries with the reference update formula. The
// forward values and the coefficients stay in shared memory (private to the
// thread's column) for the backward sweep: HBM sees one read and one write.
constexpr int kColThreads = 64;

template <int K>
__global__ void __launch_bounds__(kColThreads) dt_cols_apply(const float* __restrict__ guide,
                                                             DtPlanes P, int w, int h,
                                                             double ratio, double c,
                                                             const double* __restrict__ carry) {
  extern __shared__ double colbuf[];  // [K + 1][kColChunk][kColThreads]
  int tx = threadIdx.x;
  int x = blockIdx.x * blockDim.x + tx;
  int ch = blockIdx.y, nch = gridDim.y;
  if (x >= w) return;
  int r0 = ch * kColChunk, r1 = min(h, r0 + kColChunk);
  int64_t F = (int64_t)nch * w, o = (int64_t)ch * w + x;
  auto Y = [&](int k, int r) -> double& { return colbuf[(k * kColChunk + r) * kColThreads + tx]; };
  double prev[K];
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = carry[k * F + o];
  double a_prev = col_a(guide, w, h, r0 - 1, x, ratio, c);
#pragma unroll 8
  for (int y = r0; y < r1; ++y) {
    int64_t i = (int64_t)y * w + x;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double xv = ldp(P, k, i);
      double v = xv + a_prev * (prev[k] - xv);
      prev[k] = v;
      Y(k, y - r0) = v;
    }
    double a = col_a(guide, w, h, y, x, ratio, c);
    Y(K, y - r0) = a;
    a_prev = a;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = carry[(K + k) * F + o];
#pragma unroll 8
  for (int y = r1 - 1; y >= r0; --y) {
    int64_t i = (int64_t)y * w + x;
    double a = Y(K, y - r0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double yv = Y(k, y - r0);
      double v = yv + a * (prev[k] - yv);
      prev[k] = v;
      stp(P, k, i, v);
    }
  }
}

template <int K>
static void dt_filter_k(const float* guide, DtPlanes P, int w, int h, double sigma_s,
                        double sigma_r, int passes, double* scratch, cudaStream_t s) {
  double ratio = sigma_s / sigma_r;
  double root = sqrt(2.0);
  double den = sqrt(pow(4.0, passes) - 1.0);
  size_t row_smem = (size_t)(K + 1) * w * sizeof(double);
  int nch = ceil_div(h, kColChunk);
  double* agg = scratch;
  double* carry = agg + (int64_t)nch * w * (3 + 2 * K);
  dim3 cg(ceil_div(w, kColThreads), nch);
  size_t col_smem = (size_t)(K + 1) * kColChunk * kColThreads * sizeof(double);
  for (int i = 1; i <= passes; ++i) {
    double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;  // densify.py:104
    double c = -root / sigma_i;
    if (w > 1) dt_rows_kernel<K><<<h, kRowThreads, row_smem, s>>>(guide, P, w, h, ratio, c);
    if (h > 1) {
      dt_cols_agg<K><<<cg, kColThreads, 0, s>>>(guide, P, w, h, ratio, c, agg);
      dt_cols_link<K><<<ceil_div(w, 64), 64, 0, s>>>(w, nch, agg, carry);
      dt_cols_apply<K><<<cg, kColThreads, col_smem, s>>>(guide, P, w, h, ratio, c, carry);
    }
  }
}

int64_t dt_scratch_doubles(int w, int h, int k) {
  int nch = ceil_div(h, kColChunk);
  return (int64_t)nch * w * (3 + 2 * k) + (int64_t)nch * w * 2 * k + (int64_t)w * h + 64;
}

void init_densify_attributes() {
  allow_max_dynamic_smem(dt_rows_kernel<1>);
  allow_max_dynamic_smem(dt_rows_kernel<2>);
  allow_max_dynamic_smem(dt_rows_kernel<3>);
  allow_max_dynamic_smem(dt_cols_apply<1>);
  allow_max_dynamic_smem(dt_cols_apply<2>);
  allow_max_dynamic_smem(dt_cols_apply<3>);
}

void launch_dt_filter(const float* guide, DtPlanes P, int w, int h, double sigma_s, double sigma_r,
                      int passes, double* scratch, cudaStream_t s) {
  switch (P.k) {
    case 1: dt_filter_k<1>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, s); break;
    case 2: dt_filter_k<2>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, s); break;
    default: dt_filter_k<3>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, s); break;
  }
}

}  // namespace hdr
