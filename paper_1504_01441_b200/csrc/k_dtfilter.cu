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
// Columns: 16-row chunks held in registers. `agg` reads a chunk once and
//   reduces it to the affine data both directions need (forward map A,B and
//   the backward sums Z0 = sum (1-a_i) prod_{j<i} a_j y0_i, R for the
//   carry's own response, Q = prod a_i); `link` links the chunks of each
//   column with warp scans of affine maps; `apply` re-runs each chunk forward
//   from its upper carry and backward from its lower carry with the
//   reference formula. HBM: two reads + one write per column sweep pair.
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

// Row pass for w <= kRowThreads * kRowSeg: each thread's segment
// coefficients live in registers (shared memory holds only the planes, so
// three blocks fit per SM), and the two directions are separate static loops.
constexpr int kRowSeg = 16;

template <int K>
__device__ __forceinline__ void row_block_scan(Aff<K>& inc, bool up, Aff<K>* wsum, int lane, int warp,
                                               int nw, Aff<K>& pre) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    Aff<K> o = shfl_aff(inc, off, up);
    if (up ? lane >= off : lane + off < 32) inc = compose(o, inc);
  }
  if (lane == (up ? 31 : 0)) wsum[warp] = inc;
  __syncthreads();
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
}

template <int K>
__global__ void __launch_bounds__(kRowThreads) dt_rows_reg_kernel(const float* __restrict__ guide,
                                                                  DtPlanes P, int w, int h,
                                                                  double ratio, double c) {
  extern __shared__ double xs[];  // K * w
  __shared__ Aff<K> wsum[kRowThreads / 32];
  int y = blockIdx.x;
  int64_t row = (int64_t)y * w;
  for (int i = threadIdx.x; i < w; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) xs[k * w + i] = ldp(P, k, row + i);
  const int L = (w + kRowThreads - 1) / kRowThreads;
  int s0 = threadIdx.x * L, n = min(w, s0 + L) - s0;
  // af[j] couples samples s0-1+j and s0+j (0 outside the row)
  const float* g = guide + row;
  float gv[kRowSeg + 2];
#pragma unroll
  for (int j = 0; j < kRowSeg + 2; ++j) {
    int i = s0 - 1 + j;
    gv[j] = (j <= n + 1 && i >= 0 && i < w) ? g[i] : 0.0f;
  }
  double af[kRowSeg + 1];
#pragma unroll
  for (int j = 0; j <= kRowSeg; ++j) {
    int i = s0 - 1 + j;
    af[j] = (j <= n && i >= 0 && i + 1 < w) ? dt_coef(gv[j], gv[j + 1], ratio, c) : 0.0;
  }
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kRowThreads >> 5;
  // ---- forward
  Aff<K> m;
  m.A = 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = 0.0;
#pragma unroll
  for (int j = 0; j < kRowSeg; ++j)
    if (j < n) {
      double a = af[j];
      m.A *= a;
#pragma unroll
      for (int k = 0; k < K; ++k) { double x = xs[k * w + s0 + j]; m.B[k] = x + a * (m.B[k] - x); }
    }
  Aff<K> pre;
  row_block_scan<K>(m, true, wsum, lane, warp, nw, pre);
  double prev[K];
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = pre.B[k];
#pragma unroll
  for (int j = 0; j < kRowSeg; ++j)
    if (j < n) {
      double a = af[j];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double x = xs[k * w + s0 + j];
        prev[k] = x + a * (prev[k] - x);
        xs[k * w + s0 + j] = prev[k];
      }
    }
  // ---- backward
  m.A = 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = 0.0;
#pragma unroll
  for (int j = kRowSeg - 1; j >= 0; --j)
    if (j < n) {
      double a = af[j + 1];
      m.A *= a;
#pragma unroll
      for (int k = 0; k < K; ++k) { double x = xs[k * w + s0 + j]; m.B[k] = x + a * (m.B[k] - x); }
    }
  row_block_scan<K>(m, false, wsum, lane, warp, nw, pre);
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = pre.B[k];
#pragma unroll
  for (int j = kRowSeg - 1; j >= 0; --j)
    if (j < n) {
      double a = af[j + 1];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double x = xs[k * w + s0 + j];
        prev[k] = x + a * (prev[k] - x);
        xs[k * w + s0 + j] = prev[k];
      }
    }
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) stp(P, k, row + i, xs[k * w + i]);
}

// ---------------------------------------------------------------- columns
// 16-row chunks, thread per (column, chunk), the chunk held in registers: all
// 16 x K samples and 18 guide values are loaded up front (the loads carry no
// dependency, so each thread has ~60 requests in flight), then swept.
constexpr int kColChunk = 16;
constexpr int kColThreads = 64;

template <int K>
struct ColChunk {
  double x[K][kColChunk];
  double a[kColChunk + 1];  // a[j] couples rows r0-1+j and r0+j (a[0] links to the chunk above)
  int n;                    // valid rows in this chunk
};

template <int K>
__device__ __forceinline__ void load_chunk(const float* __restrict__ guide, const DtPlanes& P,
                                           int w, int h, int x, int r0, double ratio, double c,
                                           ColChunk<K>& ck) {
  ck.n = min(kColChunk, h - r0);
  float g[kColChunk + 2];
#pragma unroll
  for (int j = 0; j < kColChunk + 2; ++j) {
    int y = r0 - 1 + j;
    g[j] = (y >= 0 && y < h) ? __ldg(guide + (int64_t)y * w + x) : 0.0f;
  }
#pragma unroll
  for (int j = 0; j < kColChunk; ++j)
#pragma unroll
    for (int k = 0; k < K; ++k)
      ck.x[k][j] = (j < ck.n) ? ldp(P, k, (int64_t)(r0 + j) * w + x) : 0.0;
#pragma unroll
  for (int j = 0; j <= kColChunk; ++j) {
    int y = r0 - 1 + j;  // coefficient between rows y and y+1
    ck.a[j] = (y >= 0 && y + 1 < h && j <= ck.n) ? dt_coef(g[j], g[j + 1], ratio, c) : 0.0;
  }
}

// Aggregates, field-major agg[f][chunk][col], f = A, Q, R, B[K], Z0[K]:
// forward zero-carry map y_end = A*C + B, and z_start = Z0 + C*R + Q*D.
template <int K>
__global__ void __launch_bounds__(kColThreads) dt_cols_agg(const float* __restrict__ guide,
                                                           DtPlanes P, int w, int h, double ratio,
                                                           double c, double* __restrict__ agg) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y, nch = gridDim.y;
  if (x >= w) return;
  ColChunk<K> ck;
  load_chunk<K>(guide, P, w, h, x, ch * kColChunk, ratio, c, ck);
  double y0[K], z0[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { y0[k] = 0.0; z0[k] = 0.0; }
  double Pp = 1.0, R = 0.0, pref = 1.0;
#pragma unroll
  for (int j = 0; j < kColChunk; ++j) {
    if (j < ck.n) {
      double ap = ck.a[j], an = ck.a[j + 1];
      Pp *= ap;
#pragma unroll
      for (int k = 0; k < K; ++k) y0[k] = ck.x[k][j] + ap * (y0[k] - ck.x[k][j]);
      double wgt = (1.0 - an) * pref;
#pragma unroll
      for (int k = 0; k < K; ++k) z0[k] += wgt * y0[k];
      R += wgt * Pp;
      pref *= an;
    }
  }
  int64_t F = (int64_t)nch * w, o = (int64_t)ch * w + x;
  agg[o] = Pp;
  agg[F + o] = pref;
  agg[2 * F + o] = R;
#pragma unroll
  for (int k = 0; k < K; ++k) { agg[(3 + k) * F + o] = y0[k]; agg[(3 + K + k) * F + o] = z0[k]; }
}

// Carry chains. A block owns 32 columns; thread (cx, g) composes the affine
// maps of chunk group g (a run of `per` consecutive chunks) of column cx, the
// groups are linked by a Hillis-Steele scan over g in shared memory, then
// each thread emits its chunks' carries. All global accesses are coalesced
// across the 32 columns. carry[f][chunk][col]: C_b[K] (above), D_b[K] (below).
constexpr int kLinkGroups = 32;

template <int K>
__global__ void __launch_bounds__(1024) dt_cols_link(int w, int nch, const double* __restrict__ agg,
                                                     double* __restrict__ carry) {
  __shared__ Aff<K> maps[kLinkGroups][33];
  int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  int x = blockIdx.x * 32 + cx;
  bool live = x < w;
  int64_t F = (int64_t)nch * w;
  int per = (nch + kLinkGroups - 1) / kLinkGroups;
  int b0 = min(nch, g * per), b1 = min(nch, b0 + per);
  // ---- forward: y_end(b) = A_b C_b + B_b
  Aff<K> m;
  m.A = 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = 0.0;
  if (live)
    for (int b = b0; b < b1; ++b) {
      int64_t o = (int64_t)b * w + x;
      Aff<K> t;
      t.A = agg[o];
#pragma unroll
      for (int k = 0; k < K; ++k) t.B[k] = agg[(3 + k) * F + o];
      m = compose(m, t);
    }
  maps[g][cx] = m;
  __syncthreads();
  for (int off = 1; off < kLinkGroups; off <<= 1) {
    Aff<K> o = maps[g >= off ? g - off : 0][cx];
    __syncthreads();
    if (g >= off) maps[g][cx] = compose(o, maps[g][cx]);
    __syncthreads();
  }
  double C[K];
#pragma unroll
  for (int k = 0; k < K; ++k) C[k] = g ? maps[g - 1][cx].B[k] : 0.0;
  if (live)
    for (int b = b0; b < b1; ++b) {
      int64_t o = (int64_t)b * w + x;
      double A = agg[o];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        carry[k * F + o] = C[k];
        C[k] = A * C[k] + agg[(3 + k) * F + o];
      }
    }
  __syncthreads();
  // ---- backward: z_start(b) = Q_b D_b + (Z0_b + C_b R_b), from the bottom
  m.A = 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = 0.0;
  if (live)
    for (int b = b1 - 1; b >= b0; --b) {
      int64_t o = (int64_t)b * w + x;
      Aff<K> t;
      t.A = agg[F + o];
      double Rb = agg[2 * F + o];
#pragma unroll
      for (int k = 0; k < K; ++k) t.B[k] = agg[(3 + K + k) * F + o] + carry[k * F + o] * Rb;
      m = compose(m, t);
    }
  maps[g][cx] = m;
  __syncthreads();
  for (int off = 1; off < kLinkGroups; off <<= 1) {
    Aff<K> o = maps[g + off < kLinkGroups ? g + off : g][cx];
    __syncthreads();
    if (g + off < kLinkGroups) maps[g][cx] = compose(o, maps[g][cx]);
    __syncthreads();
  }
  double D[K];
#pragma unroll
  for (int k = 0; k < K; ++k) D[k] = g + 1 < kLinkGroups ? maps[g + 1][cx].B[k] : 0.0;
  if (live)
    for (int b = b1 - 1; b >= b0; --b) {
      int64_t o = (int64_t)b * w + x;
      double Q = agg[F + o], Rb = agg[2 * F + o];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        carry[(K + k) * F + o] = D[k];
        D[k] = Q * D[k] + agg[(3 + K + k) * F + o] + carry[k * F + o] * Rb;
      }
    }
}

// Re-run each chunk from its carries with the reference update formula,
// forward then backward, entirely in registers: one read, one write.
// FINAL (last pass of the pair path, K == 3 planes pu, pv, n): instead of
// storing the planes, finish densify_flow (densify.py:134-142) in registers
// and write the f32 flow: ratio where n > floor, else the homography flow.
template <int K, bool FINAL>
__global__ void __launch_bounds__(kColThreads) dt_cols_apply(const float* __restrict__ guide,
                                                             DtPlanes P, int w, int h,
                                                             double ratio, double c,
                                                             const double* __restrict__ carry,
                                                             DtFlowOut fo) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y, nch = gridDim.y;
  if (x >= w) return;
  int r0 = ch * kColChunk;
  int64_t F = (int64_t)nch * w, o = (int64_t)ch * w + x;
  double prev[K];
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = carry[k * F + o];
  ColChunk<K> ck;
  load_chunk<K>(guide, P, w, h, x, r0, ratio, c, ck);
#pragma unroll
  for (int j = 0; j < kColChunk; ++j)
    if (j < ck.n) {
      double ap = ck.a[j];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double xv = ck.x[k][j];
        prev[k] = xv + ap * (prev[k] - xv);
        ck.x[k][j] = prev[k];
      }
    }
#pragma unroll
  for (int k = 0; k < K; ++k) prev[k] = carry[(K + k) * F + o];
#pragma unroll
  for (int j = kColChunk - 1; j >= 0; --j)
    if (j < ck.n) {
      double an = ck.a[j + 1];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double yv = ck.x[k][j];
        prev[k] = yv + an * (prev[k] - yv);
        ck.x[k][j] = prev[k];
      }
    }
  if (FINAL) {
    bool use_fb = fo.fallback && (!fo.has_fb || *fo.has_fb);
    double H[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) H[i] = use_fb ? fo.fallback[i] : 0.0;
#pragma unroll
    for (int j = 0; j < kColChunk; ++j)
      if (j < ck.n) {
        double nv = ck.x[K - 1][j];
        float fu = 0.0f, fv = 0.0f;
        if (nv > fo.floor_) {
          fu = (float)(ck.x[0][j] / nv);
          fv = (float)(ck.x[K > 2 ? 1 : 0][j] / nv);
        } else if (use_fb) {
          h_pixel_flow(H, x, r0 + j, w, h, &fu, &fv);
        }
        reinterpret_cast<float2*>(fo.flow)[(int64_t)(r0 + j) * w + x] = make_float2(fu, fv);
      }
    return;
  }
#pragma unroll
  for (int j = 0; j < kColChunk; ++j)
    if (j < ck.n)
#pragma unroll
      for (int k = 0; k < K; ++k) stp(P, k, (int64_t)(r0 + j) * w + x, ck.x[k][j]);
}

template <int K>
static bool dt_filter_k(const float* guide, DtPlanes P, int w, int h, double sigma_s,
                        double sigma_r, int passes, double* scratch, const DtFlowOut& fo,
                        cudaStream_t s) {
  bool finalized = false;
  double ratio = sigma_s / sigma_r;
  double root = sqrt(2.0);
  double den = sqrt(pow(4.0, passes) - 1.0);
  size_t row_smem = (size_t)(K + 1) * w * sizeof(double);
  int nch = ceil_div(h, kColChunk);
  double* agg = scratch;
  double* carry = agg + (int64_t)nch * w * (3 + 2 * K);
  dim3 cg(ceil_div(w, kColThreads), nch);
  for (int i = 1; i <= passes; ++i) {
    double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;  // densify.py:104
    double c = -root / sigma_i;
    if (w > 1) {
      if (w <= kRowThreads * kRowSeg)
        dt_rows_reg_kernel<K><<<h, kRowThreads, (size_t)K * w * sizeof(double), s>>>(guide, P, w, h,
                                                                                    ratio, c);
      else
        dt_rows_kernel<K><<<h, kRowThreads, row_smem, s>>>(guide, P, w, h, ratio, c);
    }
    if (h > 1) {
      dt_cols_agg<K><<<cg, kColThreads, 0, s>>>(guide, P, w, h, ratio, c, agg);
      dt_cols_link<K><<<ceil_div(w, 32), 1024, 0, s>>>(w, nch, agg, carry);
      if (i == passes && fo.flow && K == 3) {
        dt_cols_apply<K, true><<<cg, kColThreads, 0, s>>>(guide, P, w, h, ratio, c, carry, fo);
        finalized = true;
      } else {
        dt_cols_apply<K, false><<<cg, kColThreads, 0, s>>>(guide, P, w, h, ratio, c, carry, fo);
      }
    }
  }
  return finalized;
}

int64_t dt_scratch_doubles(int w, int h, int k) {
  int nch = ceil_div(h, kColChunk);
  return (int64_t)nch * w * (3 + 2 * k) + (int64_t)nch * w * 2 * k + (int64_t)w * h + 64;
}

void init_densify_attributes() {
  allow_max_dynamic_smem(dt_rows_kernel<1>);
  allow_max_dynamic_smem(dt_rows_kernel<2>);
  allow_max_dynamic_smem(dt_rows_kernel<3>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<1>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<2>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<3>);
}

bool launch_dt_filter(const float* guide, DtPlanes P, int w, int h, double sigma_s, double sigma_r,
                      int passes, double* scratch, cudaStream_t s, const DtFlowOut* fo) {
  DtFlowOut none{nullptr, nullptr, 0.0, nullptr};
  const DtFlowOut& f = fo ? *fo : none;
  switch (P.k) {
    case 1: return dt_filter_k<1>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s);
    case 2: return dt_filter_k<2>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s);
    default: return dt_filter_k<3>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s);
  }
}

}  // namespace hdr
