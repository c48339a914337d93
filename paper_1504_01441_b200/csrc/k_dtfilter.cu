// Domain-transform recursive filter (K10): densify.dt_filter, densify.py:78-113.
//
// One pass = a forward+backward sweep along every row, then along every
// column; each step is the reference's update (densify.py:69-75)
//   b[i] += a * (b[i-1] - b[i]),   a = exp(c_pass * (1 + (sigma_s/sigma_r)|g[i+1]-g[i]|)).
// Sweeps are cut into segments whose zero-carry effects are affine maps; the
// maps are linked by scans and every segment is re-run from its true carry
// with the reference formula (results differ from the sequential recursion
// only by rounding, ~1e-16 relative).
//
// Rows (dt_rows_bulk_kernel): one CTA per row, the K plane rows and the guide
//   row moved by bulk copies into shared memory, 512 threads x <= 8 samples,
//   block scans of the segment maps. The pair's first row pass
//   (dt_rows_first_kernel) builds its rows from the CSR splat instead of
//   reading dense splat planes and writes sample-free rows as zeros.
// Columns (dt_cols_cluster, the default): a cluster of 8 CTAs owns a band of
//   columns over the full height, each CTA a row range, each thread 8 rows of
//   one column in registers; chunk maps are scanned inside the CTA and linked
//   across the cluster through DSMEM, and the next band is prefetched by
//   cp.async into per-thread shared-memory slots. The last pass writes the
//   f32 flow (densify_flow) instead of the planes.
// Columns fallback (tall images, test hook): `agg` reduces 8-row chunks to
//   the affine data both directions need (forward map A,B and the backward
//   sums Z0 = sum (1-a_i) prod_{j<i} a_j y0_i, R, Q = prod a_i), `link` links
//   the chunks of each column, `apply` re-runs each chunk from its carries.
// Planes may be stored f32 or f64 (DtPlanes::f64); all arithmetic is f64.
#include "hdr_common.cuh"
#include "hdr_internal.h"
#include "hdr_planes.cuh"
#include "hdr_bulk.cuh"

#include <cooperative_groups.h>
#include <algorithm>
#include <type_traits>

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

template <int K>
__device__ __forceinline__ Aff<K> shfl_aff_idx(const Aff<K>& v, int src) {
  Aff<K> r;
  r.A = __shfl_sync(0xffffffff, v.A, src);
#pragma unroll
  for (int k = 0; k < K; ++k) r.B[k] = __shfl_sync(0xffffffff, v.B[k], src);
  return r;
}

#ifndef HDR_ROW_SCAN_SHFL
#define HDR_ROW_SCAN_SHFL 1
#endif

// ---------------------------------------------------------------- rows
// Row-sweep block size / max segment: 512 x 8 measured best for batch
// throughput (897 pairs/s vs 873 at 256 x 16 and 886 at 384 x 8); 384 x 8
// gives the lowest single-pair latency (1.64 ms). Overridable at build time.
#ifndef HDR_ROW_THREADS
#define HDR_ROW_THREADS 512
#endif
// 9, not 8: widths in (3584, 4096] (12MP is 4000) then take 9-sample odd
// segments instead of 8-sample even ones whose half-warp loads conflict
// (kbench dt at 4000x3000: 2267 -> 1295 us for the three-pass filter; 5MP
// unchanged, its segments are 7)
#ifndef HDR_ROW_SEG
#define HDR_ROW_SEG 9
#endif
constexpr int kRowThreads = HDR_ROW_THREADS;

template <int K>
__global__ void __launch_bounds__(kRowThreads) dt_rows_kernel(const float* __restrict__ guide,
                                                              DtPlanes P, int w, int h,
                                                              double ratio, double c) {
  pdl_wait();
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
constexpr int kRowSeg = HDR_ROW_SEG;

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
#if HDR_ROW_SCAN_SHFL
  {
    // the other warps' totals composed by a shuffle scan over lanes (lane j
    // holds wsum[j]; 5 steps) instead of a serial fold of up to nw - 1
    // dependent shared loads + compositions per thread
    Aff<K> t = pre;
    if (lane < nw) t = wsum[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      Aff<K> u = shfl_aff(t, off, up);
      if (up ? lane >= off : lane + off < 32) t = compose(u, t);
    }
    const int src = up ? warp - 1 : warp + 1;
    Aff<K> v = shfl_aff_idx(t, src < 0 ? 0 : src);
    if (up ? warp > 0 : warp + 1 < nw) pre = v;
  }
#else
  if (up) {
    for (int j = 0; j < warp; ++j) pre = compose(pre, wsum[j]);
  } else {
    for (int j = nw - 1; j > warp; --j) pre = compose(pre, wsum[j]);
  }
#endif
  Aff<K> o = shfl_aff(inc, 1, up);
  if (up ? lane > 0 : lane < 31) pre = compose(pre, o);
  __syncthreads();
}

template <int K>
__global__ void __launch_bounds__(kRowThreads) dt_rows_reg_kernel(const float* __restrict__ guide,
                                                                  DtPlanes P, int w, int h,
                                                                  double ratio, double c) {
  pdl_wait();
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

// One row swept forward then backward in shared memory: xs holds the K plane
// rows, gs the guide row; 256 threads each own a segment of ceil(w/256)
// samples (coefficients in registers), segments linked by block scans of
// affine maps, then re-run with the reference update.
template <int K>
__device__ __forceinline__ void row_sweep_smem(double* xs, const float* gs, int w, double ratio,
                                               double c, Aff<K>* wsum) {
#ifndef HDR_ROW_ODD_SEG
#define HDR_ROW_ODD_SEG 1
#endif
  int L = (w + kRowThreads - 1) / kRowThreads;
  // an odd segment length puts a half-warp's segment starts on 16 distinct
  // 8-byte bank pairs (an even one shares them two or four ways)
  if (HDR_ROW_ODD_SEG && !(L & 1) && L < kRowSeg) ++L;
  int s0 = threadIdx.x * L, n = max(0, min(w, s0 + L) - s0);
  // af[j] couples samples s0-1+j and s0+j (0 outside the row)
  double af[kRowSeg + 1];
#pragma unroll
  for (int j = 0; j <= kRowSeg; ++j) {
    int i = s0 - 1 + j;
    af[j] = (j <= n && i >= 0 && i + 1 < w) ? dt_coef(gs[i], gs[i + 1], ratio, c) : 0.0;
  }
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
}

// the swept row back to HBM (one bulk copy per plane)
template <int K>
__device__ __forceinline__ void store_row_bulk(const DtPlanes& P, int64_t row, const double* xs, int w) {
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      bulk_store(reinterpret_cast<double*>(P.p[k]) + row, xs + k * w, (uint32_t)w * 8);
    bulk_commit();
    bulk_wait_read();
  }
}

// Row pass with the row moved by bulk copies: one thread issues the K plane
// rows and the guide row (one cp.async.bulk each) and the results go back the
// same way, so the 256 threads only compute. Needs all planes f64 and
// 16-byte aligned rows (w % 4 == 0, aligned bases); w <= kRowThreads*kRowSeg.
template <int K>
#ifdef HDR_ROW_MIN_BLOCKS
#define HDR_ROW_BOUNDS kRowThreads, HDR_ROW_MIN_BLOCKS
#else
#define HDR_ROW_BOUNDS kRowThreads
#endif
__global__ void __launch_bounds__(HDR_ROW_BOUNDS) dt_rows_bulk_kernel(const float* __restrict__ guide,
                                                                   DtPlanes P, int w, int h,
                                                                   double ratio, double c) {
  pdl_wait();
  extern __shared__ __align__(16) double xs[];  // K * w planes, then w guide floats
  float* gs = reinterpret_cast<float*>(xs + K * w);
  __shared__ Aff<K> wsum[kRowThreads / 32];
  __shared__ uint64_t bar;
  int y = blockIdx.x;
  int64_t row = (int64_t)y * w;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)(K * w * 8 + w * 4));
#pragma unroll
    for (int k = 0; k < K; ++k)
      bulk_load(xs + k * w, reinterpret_cast<const double*>(P.p[k]) + row, (uint32_t)w * 8, &bar);
    bulk_load(gs, guide + row, (uint32_t)w * 4, &bar);
  }
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(&bar, 0);
  row_sweep_smem<K>(xs, gs, w, ratio, c, wsum);
  store_row_bulk<K>(P, row, xs, w);
}

// First row pass straight from the splat (densify.py:38-56 + the first
// horizontal sweep): the planes before it are zero except one (u, v, 1)
// sample per weeded match, so a row is built in shared memory from its
// samples (CSR by row, DtSparse) instead of being read, and a row without
// samples -- most of them: corners sit on a 4-px candidate lattice -- stays
// zero through the sweep and is written as zeros without any compute. The
// planes need no initialisation (this writes every sample). K == 3 (pu, pv, n).
__global__ void __launch_bounds__(kRowThreads) dt_rows_first_kernel(const float* __restrict__ guide,
                                                                    DtPlanes P, int w, int h,
                                                                    double ratio, double c,
                                                                    DtSparse sp, bool zero_rows) {
  pdl_wait();
  constexpr int K = 3;
  extern __shared__ __align__(16) double xs[];  // K * w planes, then w guide floats
  float* gs = reinterpret_cast<float*>(xs + K * w);
  __shared__ Aff<K> wsum[kRowThreads / 32];
  __shared__ uint64_t bar;
  int y = blockIdx.x;
  int64_t row = (int64_t)y * w;
  const int e0 = sp.row_start[y], e1 = sp.row_start[y + 1];
  if (e0 == e1) {
    // the column sweep that follows skips rows without samples when it can
    // (dt_cols_cluster's zrows); otherwise the zeros are written
    if (!zero_rows) return;
    const double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(P.p[k]) + row);
      for (int i = threadIdx.x; i < w / 2; i += blockDim.x) __stcs(d + i, z);
    }
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)(w * 4));
    bulk_load(gs, guide + row, (uint32_t)w * 4, &bar);
  }
  for (int i = threadIdx.x; i < K * w; i += blockDim.x) xs[i] = 0.0;
  __syncthreads();
  for (int e = e0 + (int)threadIdx.x; e < e1; e += blockDim.x) {
    const SparseEntry& t = sp.entries[e];
    xs[t.x] = t.u;
    xs[w + t.x] = t.v;
    xs[2 * w + t.x] = 1.0;
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  row_sweep_smem<K>(xs, gs, w, ratio, c, wsum);
  // plain 16-byte stores (not a bulk copy): this pass is the first write of
  // the planes, and compute-sanitizer's initcheck does not track TMA stores
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double2* d = reinterpret_cast<double2*>(reinterpret_cast<double*>(P.p[k]) + row);
    const double2* q = reinterpret_cast<const double2*>(xs + k * w);
    for (int i = threadIdx.x; i < w / 2; i += blockDim.x) d[i] = q[i];
  }
}

static bool rows_bulk_ok(const float* guide, const DtPlanes& P, int w) {
  if (w % 4 || w > kRowThreads * kRowSeg || (reinterpret_cast<uintptr_t>(guide) & 15)) return false;
  for (int k = 0; k < P.k; ++k)
    if (!P.f64[k] || (reinterpret_cast<uintptr_t>(P.p[k]) & 15)) return false;
  return true;
}

// ---------------------------------------------------------------- columns
// 8-row chunks, thread per (column, chunk), the chunk held in registers: all
// 8 x K samples and 10 guide values are loaded up front (the loads carry no
// dependency, so each thread has ~34 requests in flight), then swept. 16-row
// chunks held twice the registers (apply 255 + spill, agg 154) at a quarter
// of the occupancy and ran slower: 5MP, 3 passes, 725 us (16) / 647 (8) /
// 672 (4, where the link's serial chain over 486 chunks takes 40 us a pass).
#ifndef HDR_COL_CHUNK
#define HDR_COL_CHUNK 8
#endif
constexpr int kColChunk = HDR_COL_CHUNK;
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

// Aggregates, chunk-major agg[chunk][f][col], f = A, Q, R, B[K], Z0[K]:
// forward zero-carry map y_end = A*C + B, and z_start = Z0 + C*R + Q*D.
// ch0: first chunk of the launch (a row band's chunks; 0 for the whole
// image), nch: chunks of the whole image (the agg layout)
template <int K>
#ifndef HDR_AGG_MIN_BLOCKS
#define HDR_AGG_MIN_BLOCKS 1
#endif
#ifndef HDR_APPLY_MIN_BLOCKS
#define HDR_APPLY_MIN_BLOCKS 8
#endif
__global__ void __launch_bounds__(kColThreads, HDR_AGG_MIN_BLOCKS) dt_cols_agg(const float* __restrict__ guide,
                                                           DtPlanes P, int w, int h, double ratio,
                                                           double c, double* __restrict__ agg,
                                                           int ch0, int nch) {
  pdl_wait();
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = ch0 + (int)blockIdx.y;
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
  // chunk-major: a run of chunks (a row band) is one contiguous block
  double* a = agg + (int64_t)ch * (3 + 2 * K) * w + x;
  a[0] = Pp;
  a[w] = pref;
  a[2 * w] = R;
#pragma unroll
  for (int k = 0; k < K; ++k) { a[(3 + k) * w] = y0[k]; a[(3 + K + k) * w] = z0[k]; }
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
  pdl_wait();
  __shared__ Aff<K> maps[kLinkGroups][33];
  int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  int x = blockIdx.x * 32 + cx;
  bool live = x < w;
  int64_t F = (int64_t)nch * w;
  // agg[chunk][field][col] (chunk-major, see dt_cols_agg)
  auto AG = [&](int f, int b) { return ((int64_t)b * (3 + 2 * K) + f) * w + x; };
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
      t.A = agg[AG(0, b)];
#pragma unroll
      for (int k = 0; k < K; ++k) t.B[k] = agg[AG(3 + k, b)];
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
      double A = agg[AG(0, b)];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        carry[k * F + o] = C[k];
        C[k] = A * C[k] + agg[AG(3 + k, b)];
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
      t.A = agg[AG(1, b)];
      double Rb = agg[AG(2, b)];
#pragma unroll
      for (int k = 0; k < K; ++k) t.B[k] = agg[AG(3 + K + k, b)] + carry[k * F + o] * Rb;
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
      double Q = agg[AG(1, b)], Rb = agg[AG(2, b)];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        carry[(K + k) * F + o] = D[k];
        D[k] = Q * D[k] + agg[AG(3 + K + k, b)] + carry[k * F + o] * Rb;
      }
    }
}

// Re-run each chunk from its carries with the reference update formula,
// forward then backward, entirely in registers: one read, one write.
// FINAL (last pass of the pair path, K == 3 planes pu, pv, n): instead of
// storing the planes, finish densify_flow (densify.py:134-142) in registers
// and write the f32 flow: ratio where n > floor, else the homography flow.
template <int K, bool FINAL>
__global__ void __launch_bounds__(kColThreads, HDR_APPLY_MIN_BLOCKS) dt_cols_apply(const float* __restrict__ guide,
                                                             DtPlanes P, int w, int h,
                                                             double ratio, double c,
                                                             const double* __restrict__ carry,
                                                             DtFlowOut fo, int ch0, int nch) {
  pdl_wait();
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = ch0 + (int)blockIdx.y;
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

// ---------------------------------------------------------------- columns, cluster-resident
// One column sweep pair (down then up) in a single kernel. A cluster of kCL
// CTAs owns a band of `bw` columns over the full image height: CTA `rank`
// holds rows [rank*RP, (rank+1)*RP), split into G = kCT / bw groups of kSR
// rows; thread (col, grp) keeps its kSR x K samples and kSR+1 coefficients in
// registers from load to store. The chunk aggregates of dt_cols_agg are
// linked by a Hillis-Steele scan over the groups in shared memory and across
// the cluster through distributed shared memory (one barrier.cluster per
// direction), so a sweep pair costs one HBM read and one write of the planes
// instead of agg + link + apply's two reads, one write and the carry traffic.
#ifndef HDR_COL_CLUSTER
#define HDR_COL_CLUSTER 8
#endif
constexpr int kCL = HDR_COL_CLUSTER;  // CTAs per cluster (8: portable maximum)
#ifndef HDR_COL_THREADS_LOG2
#define HDR_COL_THREADS_LOG2 8
#endif
#ifndef HDR_COL_ROWS
#define HDR_COL_ROWS 8
#endif
constexpr int kCT = 1 << HDR_COL_THREADS_LOG2;  // threads per CTA (256: two CTAs per SM)
constexpr int kCTLog2 = HDR_COL_THREADS_LOG2;
constexpr int kSR = HDR_COL_ROWS;    // rows per thread
constexpr int kMaxBw = kCT / 8 < 32 ? kCT / 8 : 32;  // widest band (cluster arrays)

namespace cg = cooperative_groups;

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Cluster barrier for data exchanged through shared memory only: the release
// fence is restricted to this CTA's shared-memory writes (MEMBAR.CTA instead
// of the GPU-scope MEMBAR that barrier.cluster.arrive.release emits, which
// also waits for the thread's in-flight cp.async prefetches and global
// stores); peers read the published values through DSMEM after the wait.
#ifndef HDR_COL_SMEM_SYNC
#define HDR_COL_SMEM_SYNC 1
#endif
__device__ __forceinline__ void cluster_sync_smem() {
#if HDR_COL_SMEM_SYNC
  asm volatile(
      "fence.release.sync_restrict::shared::cta.cluster;\n"
      "barrier.cluster.arrive.relaxed.aligned;\n"
      "barrier.cluster.wait.aligned;\n"
      "fence.acquire.sync_restrict::shared::cluster.cluster;\n" ::: "memory");
#else
  cluster_arrive();
  cluster_wait();
#endif
}


// prefetch slots of one thread: element (k, j) at pfx[(k * kSR + j) * kCT + tid]
// (consecutive threads, consecutive words: conflict-free), guide j at
// pfg[j * kCT + tid]
template <int K>
constexpr size_t cols_pf_smem() {
  return sizeof(double) * K * kSR * kCT + sizeof(float) * (kSR + 2) * kCT;
}

// Scan of the groups' affine maps inside a CTA (thread = (group, column),
// lane = sub * bw + col): warp shuffles over the groups of a warp, then the
// warps' totals through shared memory -- two block barriers per scan.
// up: m becomes the inclusive prefix (groups above and this one) and ex the
// exclusive prefix; !up: the same as suffixes (groups below).
template <int K>
__device__ __forceinline__ void scan_groups(Aff<K>& m, bool up, int bw_log2,
                                            Aff<K> (*wsc)[kMaxBw], Aff<K>& ex) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int bw = 1 << bw_log2, col = lane & (bw - 1), sub = lane >> bw_log2, Gw = 32 >> bw_log2;
  for (int off = 1; off < Gw; off <<= 1) {
    Aff<K> o = shfl_aff(m, off << bw_log2, up);
    if (up ? sub >= off : sub + off < Gw) m = compose(o, m);
  }
  Aff<K> e = shfl_aff(m, bw, up);  // exclusive within the warp
  if (up ? sub == 0 : sub == Gw - 1) {
    e.A = 1.0;
#pragma unroll
    for (int k = 0; k < K; ++k) e.B[k] = 0.0;
  }
  if (up ? sub == Gw - 1 : sub == 0) wsc[warp][col] = m;
  __syncthreads();
  Aff<K> pre;  // the other warps' totals, composed in sweep order
  pre.A = 1.0;
#pragma unroll
  for (int k = 0; k < K; ++k) pre.B[k] = 0.0;
  if (up) {
    for (int q = 0; q < warp; ++q) pre = compose(pre, wsc[q][col]);
  } else {
    for (int q = nw - 1; q > warp; --q) pre = compose(pre, wsc[q][col]);
  }
  ex = compose(pre, e);
  m = compose(pre, m);
  __syncthreads();  // wsc is reused by the next scan
}

// PF: the band's samples arrive by cp.async into per-thread shared-memory
// slots issued one band ahead (needs f64 planes and dynamic shared memory of
// cols_pf_smem<K>()), so HBM reads of band b+1 overlap the link, apply and
// store phases of band b; otherwise plain loads at the top of each band.
template <int K, bool FINAL, bool PF>
#ifndef HDR_COL_MIN_BLOCKS
#define HDR_COL_MIN_BLOCKS (kCT <= 256 ? 2 : 1)
#endif
__global__ void __cluster_dims__(kCL, 1, 1) __launch_bounds__(kCT, HDR_COL_MIN_BLOCKS)
    dt_cols_cluster(const float* __restrict__ guide, DtPlanes P, int w, int h, double ratio,
                    double c, int bw_log2, DtFlowOut fo, const int32_t* __restrict__ zrows) {
  pdl_wait();
  __shared__ Aff<K> wsc[kCT / 32][kMaxBw];  // per-warp totals of the group scans
  // per-column CTA totals read by the cluster peers, double-buffered by band
  // parity: band b+2 reuses band b's buffer only after two cluster barriers,
  // by which time every peer has read it, so bands need no closing barrier
  __shared__ Aff<K> ctaF2[2][kMaxBw], ctaB2[2][kMaxBw];
  __shared__ double cin[kMaxBw][K], din[kMaxBw][K];
  __shared__ Aff<K> remote[kCL][kMaxBw];
  extern __shared__ __align__(16) double pfx[];
  float* pfg = reinterpret_cast<float*>(pfx + K * kSR * kCT);
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int bw = 1 << bw_log2, G = kCT >> bw_log2;
  const int col = threadIdx.x & (bw - 1), grp = threadIdx.x >> bw_log2;
  const int RP = ceil_div(h, kCL);
  const int nbands = ceil_div(w, bw);
  const int r0 = rank * RP + grp * kSR;
  const int rend = min(h, (rank + 1) * RP);
  const int nrows = max(0, min(kSR, rend - r0));
  // zrows (the CSR row starts of the pair's first pass, PF only): rows without
  // a splat sample are exactly zero after the first row sweep and were not
  // written, so they are neither loaded nor read (bit j = row r0 + j)
  uint32_t zmask = 0;
  if (PF && zrows)
    for (int j = 0; j < nrows; ++j)
      if (__ldg(zrows + r0 + j) == __ldg(zrows + r0 + j + 1)) zmask |= 1u << j;
  // the thread's first row of every plane (band 0); a band adds band << bw_log2
  const int64_t o0 = (int64_t)r0 * w + col;
  // guide rows r0-1 .. r0+nrows that exist: j in [jg0, jg1)
  const int jg0 = r0 == 0 ? 1 : 0, jg1 = min(nrows + 2, h - r0 + 1);
  auto prefetch = [&](int band) {
    const int x = (band << bw_log2) + col;
    if (band >= nbands || x >= w) return;
    const int64_t o = o0 + (band << bw_log2);
    const float* gp = guide + (o - w);
#pragma unroll
    for (int j = 0; j < kSR + 2; ++j)
      if (j >= jg0 && j < jg1) cp_async4(pfg + j * kCT + threadIdx.x, gp + (int64_t)j * w);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double* pk = reinterpret_cast<const double*>(P.p[k]) + o;
#pragma unroll
      for (int j = 0; j < kSR; ++j)
        if (j < nrows && !((zmask >> j) & 1u)) cp_async8(pfx + (k * kSR + j) * kCT + threadIdx.x, pk + (int64_t)j * w);
    }
    cp_async_commit();
  };
  if (PF) prefetch(blockIdx.y);
  // persistent: the grid holds as many clusters as can be co-resident and
  // each walks bands (no cluster-launch fragmentation between waves)
  int parity = 0;
  for (int band = blockIdx.y; band < nbands; band += gridDim.y, parity ^= 1) {
  Aff<K>* ctaF = ctaF2[parity];
  Aff<K>* ctaB = ctaB2[parity];
  const int x = (band << bw_log2) + col;
  const bool live = x < w;
  const int n = live ? nrows : 0;
  // ---- load (all requests issued before the first use)
  double xv[K][kSR];
  double a[kSR + 1];  // a[j] couples rows r0-1+j and r0+j
  {
    float g[kSR + 2];
    if (PF) cp_async_wait_all();  // this thread's slots for this band have landed
#pragma unroll
    for (int j = 0; j < kSR + 2; ++j) {
      int y = r0 - 1 + j;
      bool ok = live && j <= n + 1 && y >= 0 && y < h;
      g[j] = ok ? (PF ? pfg[j * kCT + threadIdx.x] : __ldg(guide + (int64_t)y * w + x)) : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < kSR; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k)
        xv[k][j] = (j < n && !((zmask >> j) & 1u)) ? (PF ? pfx[(k * kSR + j) * kCT + threadIdx.x]
                                                        : ldp(P, k, (int64_t)(r0 + j) * w + x))
                                                   : 0.0;
#pragma unroll
    for (int j = 0; j <= kSR; ++j) {
      int y = r0 - 1 + j;
      a[j] = (n > 0 && j <= n && y >= 0 && y + 1 < h) ? dt_coef(g[j], g[j + 1], ratio, c) : 0.0;
    }
  }
  // ---- chunk aggregates (see dt_cols_agg)
  double Pp = 1.0, R = 0.0, Q = 1.0;
  double y0[K], z0[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { y0[k] = 0.0; z0[k] = 0.0; }
#pragma unroll
  for (int j = 0; j < kSR; ++j)
    if (j < n) {
      double ap = a[j], an = a[j + 1];
      Pp *= ap;
#pragma unroll
      for (int k = 0; k < K; ++k) y0[k] = xv[k][j] + ap * (y0[k] - xv[k][j]);
      double wgt = (1.0 - an) * Q;
#pragma unroll
      for (int k = 0; k < K; ++k) z0[k] += wgt * y0[k];
      R += wgt * Pp;
      Q *= an;
    }
  // every sample of this band is in registers and consumed: refill the
  // slots with the next band while this one is linked, applied and stored
  if (PF) prefetch(band + gridDim.y);
  // ---- forward link: inclusive scan over groups, then across the cluster
  Aff<K> m;
  m.A = Pp;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = y0[k];
  Aff<K> ex;  // exclusive prefix of this group within the CTA
  scan_groups<K>(m, true, bw_log2, wsc, ex);
  if (grp == G - 1) ctaF[col] = m;
  cluster_sync_smem();
  // gather the lower ranks' totals for this column (one remote load per thread)
  for (int q = grp; q < rank; q += G) remote[q][col] = *cl.map_shared_rank(&ctaF[col], q);
  __syncthreads();
  double C[K];
  if (grp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) C[k] = 0.0;
    for (int q = 0; q < rank; ++q) {
      const Aff<K>& t = remote[q][col];
#pragma unroll
      for (int k = 0; k < K; ++k) C[k] = t.A * C[k] + t.B[k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) cin[col][k] = C[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) C[k] = ex.A * cin[col][k] + ex.B[k];
  // ---- backward link: suffix scan of z_start(g) = Q_g z_start(g+1) + (Z0_g + C_g R_g)
  m.A = Q;
#pragma unroll
  for (int k = 0; k < K; ++k) m.B[k] = z0[k] + C[k] * R;
  Aff<K> sx;  // suffix from the groups below this one within the CTA
  scan_groups<K>(m, false, bw_log2, wsc, sx);
  if (grp == 0) ctaB[col] = m;
  cluster_sync_smem();
  for (int q = rank + 1 + grp; q < kCL; q += G) remote[q][col] = *cl.map_shared_rank(&ctaB[col], q);
  __syncthreads();
  double D[K];
  if (grp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) D[k] = 0.0;
    for (int q = kCL - 1; q > rank; --q) {
      const Aff<K>& t = remote[q][col];
#pragma unroll
      for (int k = 0; k < K; ++k) D[k] = t.A * D[k] + t.B[k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) din[col][k] = D[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) D[k] = sx.A * din[col][k] + sx.B[k];
  // ---- apply: forward from C, backward from D, with the reference update
  if (n > 0) {
    double prev[K];
#pragma unroll
    for (int k = 0; k < K; ++k) prev[k] = C[k];
#pragma unroll
    for (int j = 0; j < kSR; ++j)
      if (j < n) {
        double ap = a[j];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          double v = xv[k][j];
          prev[k] = v + ap * (prev[k] - v);
          xv[k][j] = prev[k];
        }
      }
#pragma unroll
    for (int k = 0; k < K; ++k) prev[k] = D[k];
#pragma unroll
    for (int j = kSR - 1; j >= 0; --j)
      if (j < n) {
        double an = a[j + 1];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          double v = xv[k][j];
          prev[k] = v + an * (prev[k] - v);
          xv[k][j] = prev[k];
        }
      }
    if (FINAL) {
      bool use_fb = fo.fallback && (!fo.has_fb || *fo.has_fb);
#pragma unroll
      for (int j = 0; j < kSR; ++j)
        if (j < n) {
          double nv = xv[K - 1][j];
          float fu = 0.0f, fv = 0.0f;
          if (nv > fo.floor_) {
            // one reciprocal: the f64 quotient differs by at most an ulp,
            // far below the f32 rounding of the flow
            double inv = 1.0 / nv;
            fu = (float)(xv[0][j] * inv);
            fv = (float)(xv[K > 2 ? 1 : 0][j] * inv);
          } else if (use_fb) {
            h_pixel_flow(fo.fallback, x, r0 + j, w, h, &fu, &fv);
          }
          reinterpret_cast<float2*>(fo.flow)[(int64_t)(r0 + j) * w + x] = make_float2(fu, fv);
        }
    } else if (PF) {
      // every plane is f64 on the prefetch path
      const int64_t o = o0 + (band << bw_log2);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double* pk = reinterpret_cast<double*>(P.p[k]) + o;
#pragma unroll
        for (int j = 0; j < kSR; ++j)
          if (j < n) pk[(int64_t)j * w] = xv[k][j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < kSR; ++j)
        if (j < n)
#pragma unroll
          for (int k = 0; k < K; ++k) stp(P, k, (int64_t)(r0 + j) * w + x, xv[k][j]);
    }
  }
  }
  // no CTA may leave while a peer can still read its shared memory
  cluster_arrive();
  cluster_wait();
}

// co-resident clusters of a cluster-kernel instantiation (0 = query failed)
template <int K, bool FINAL, bool PF>
static int max_clusters() {
  static int n = -1;
  if (n < 0) {
    size_t smem = PF ? cols_pf_smem<K>() : 0;
    if (kCL > 8)  // clusters beyond the portable 8 CTAs must be opted into
      cudaFuncSetAttribute(dt_cols_cluster<K, FINAL, PF>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (PF && cudaFuncSetAttribute(dt_cols_cluster<K, FINAL, PF>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return n = 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCL, 1024);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = smem;
    int v = 0;
    if (cudaOccupancyMaxActiveClusters(&v, dt_cols_cluster<K, FINAL, PF>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      v = 0;
    }
    n = v;
  }
  return n;
}

// test hook: 0 turns the cp.async band prefetch of the cluster kernel off
static bool g_cols_prefetch = true;
// clusters launched = co-resident maximum / g_cols_grid_div (tuning hook)
static int g_cols_grid_div = 1;

template <int K, bool FINAL>
static void launch_cols_cluster(const float* guide, const DtPlanes& P, int w, int h, double ratio,
                                double c, int bl, const DtFlowOut& fo, cudaStream_t s,
                                const int32_t* zrows = nullptr) {
  int nb = ceil_div(w, 1 << bl);
  bool pf = g_cols_prefetch;
  for (int k = 0; k < P.k; ++k)
    if (!P.f64[k]) pf = false;
  int mc = pf ? max_clusters<K, FINAL, true>() : 0;
  if (pf && mc > 0) {
    if (g_cols_grid_div > 1) mc = std::max(1, mc / g_cols_grid_div);
    dim3 cgrid(kCL, std::min(nb, mc));
    klaunch(dt_cols_cluster<K, FINAL, true>, cgrid, kCT, cols_pf_smem<K>(), s, guide, P, w, h, ratio, c, bl, fo,
                                                                          zrows);
    return;
  }
  mc = max_clusters<K, FINAL, false>();
  dim3 cgrid(kCL, mc > 0 ? std::min(nb, mc) : nb);
  klaunch(dt_cols_cluster<K, FINAL, false>, cgrid, kCT, 0, s, guide, P, w, h, ratio, c, bl, fo, nullptr);
}

// log2 of the cluster kernel's band width for this height, or -1 (too tall)
static int cluster_bw_log2(int h) {
  int rp = ceil_div(h, kCL);
  int g = ceil_div(rp, kSR), gl = 0;
  while ((1 << gl) < g) ++gl;
  while ((kCT >> gl) > kMaxBw) ++gl;  // bw <= kMaxBw
  int bl = kCTLog2 - gl;
  return bl >= 1 ? bl : -1;
}

// dynamic shared memory dt_rows_kernel<K> may take (set by init_densify_attributes)
static int g_rows_smem_max[4] = {0, 0, 0, 0};

// test hook: 0 selects the agg/link/apply column path
static bool g_cols_cluster = true;
// test hook: 0 makes the sparse-first row pass write its sample-free rows
// (zeros) instead of letting the first column sweep skip them
static bool g_skip_zero_rows = true;

// c of pass i (densify.py:104-106)
static double dt_pass_c(double sigma_s, int passes, int i) {
  double den = sqrt(pow(4.0, passes) - 1.0);
  double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;
  return -sqrt(2.0) / sigma_i;
}

// one horizontal sweep pair over h rows (any row set: rows are independent)
template <int K>
static void rows_pass(const float* guide, const DtPlanes& P, int w, int h, double ratio, double c,
                      cudaStream_t s) {
  size_t row_smem = (size_t)(K + 1) * w * sizeof(double);
  if (rows_bulk_ok(guide, P, w))
    klaunch(dt_rows_bulk_kernel<K>, h, kRowThreads, (size_t)K * w * sizeof(double) + (size_t)w * 4, s,
            guide, P, w, h, ratio, c);
  else if (w <= kRowThreads * kRowSeg)
    klaunch(dt_rows_reg_kernel<K>, h, kRowThreads, (size_t)K * w * sizeof(double), s, guide, P, w, h, ratio, c);
  else if (row_smem <= (size_t)g_rows_smem_max[K])
    klaunch(dt_rows_kernel<K>, h, kRowThreads, row_smem, s, guide, P, w, h, ratio, c);
  else
    launch_dt_rows_seq(guide, P, w, h, ratio, c, s);
}

// ---- row-band pieces of the filter: a band of whole
// chunks [ch0, ch1) runs its rows and its column chunks locally; only the
// chunk aggregates cross bands (the caller sums them over the ranks), and
// link + apply then give every band exactly the single-GPU agg/link/apply
// result.
int64_t dt_band_agg_doubles(int w, int h, int k) { return (int64_t)ceil_div(h, kColChunk) * w * (3 + 2 * k); }
int dt_band_chunk_rows() { return kColChunk; }

template <int K>
static void band_rows_k(const float* guide, const DtPlanes& P, int w, int h, int y0, int y1, double sigma_s,
                        double sigma_r, int passes, int i, cudaStream_t s) {
  if (w <= 1 || y1 <= y0) return;
  DtPlanes B = P;
  for (int k = 0; k < K; ++k)
    B.p[k] = P.f64[k] ? (void*)((double*)P.p[k] + (int64_t)y0 * w) : (void*)((float*)P.p[k] + (int64_t)y0 * w);
  rows_pass<K>(guide + (int64_t)y0 * w, B, w, y1 - y0, sigma_s / sigma_r, dt_pass_c(sigma_s, passes, i), s);
}

template <int K>
static void band_agg_k(const float* guide, const DtPlanes& P, int w, int h, int y0, int y1, double sigma_s,
                       double sigma_r, int passes, int i, double* agg, cudaStream_t s) {
  int nch = ceil_div(h, kColChunk), ch0 = y0 / kColChunk, ch1 = ceil_div(y1, kColChunk);
  if (h <= 1 || ch1 <= ch0) return;
  dim3 cg(ceil_div(w, kColThreads), ch1 - ch0);
  klaunch(dt_cols_agg<K>, cg, kColThreads, 0, s, guide, P, w, h, sigma_s / sigma_r, dt_pass_c(sigma_s, passes, i),
          agg, ch0, nch);
}

template <int K>
static void band_apply_k(const float* guide, const DtPlanes& P, int w, int h, int y0, int y1, double sigma_s,
                         double sigma_r, int passes, int i, const double* agg, double* carry,
                         const DtFlowOut& fo, cudaStream_t s) {
  int nch = ceil_div(h, kColChunk), ch0 = y0 / kColChunk, ch1 = ceil_div(y1, kColChunk);
  if (h <= 1 || ch1 <= ch0) return;
  double ratio = sigma_s / sigma_r, c = dt_pass_c(sigma_s, passes, i);
  klaunch(dt_cols_link<K>, ceil_div(w, 32), 1024, 0, s, w, nch, agg, carry);
  dim3 cg(ceil_div(w, kColThreads), ch1 - ch0);
  if (fo.flow && K == 3)
    klaunch(dt_cols_apply<K, true>, cg, kColThreads, 0, s, guide, P, w, h, ratio, c, (const double*)carry, fo,
            ch0, nch);
  else
    klaunch(dt_cols_apply<K, false>, cg, kColThreads, 0, s, guide, P, w, h, ratio, c, (const double*)carry, fo,
            ch0, nch);
}

void launch_dt_band(int op, const float* guide, const DtPlanes& P, int w, int h, int y0, int y1,
                    double sigma_s, double sigma_r, int passes, int i, double* agg, double* carry,
                    const DtFlowOut* fo, cudaStream_t s) {
  DtFlowOut none{nullptr, nullptr, 0.0, nullptr};
  const DtFlowOut& f = fo ? *fo : none;
  auto go = [&](auto kk) {
    constexpr int K = decltype(kk)::value;
    if (op == 0) band_rows_k<K>(guide, P, w, h, y0, y1, sigma_s, sigma_r, passes, i, s);
    else if (op == 1) band_agg_k<K>(guide, P, w, h, y0, y1, sigma_s, sigma_r, passes, i, agg, s);
    else band_apply_k<K>(guide, P, w, h, y0, y1, sigma_s, sigma_r, passes, i, agg, carry, f, s);
  };
  switch (P.k) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    default: go(std::integral_constant<int, 3>{}); break;
  }
}

template <int K>
static bool dt_filter_k(const float* guide, DtPlanes P, int w, int h, double sigma_s,
                        double sigma_r, int passes, double* scratch, const DtFlowOut& fo,
                        cudaStream_t s, KProbe* kr, KProbe* kc, const DtSparse* sp) {
  bool finalized = false;
  double ratio = sigma_s / sigma_r;
  double root = sqrt(2.0);
  double den = sqrt(pow(4.0, passes) - 1.0);
  size_t row_smem = (size_t)(K + 1) * w * sizeof(double);
  int nch = ceil_div(h, kColChunk);
  double* agg = scratch;
  double* carry = agg + (int64_t)nch * w * (3 + 2 * K);
  dim3 cg(ceil_div(w, kColThreads), nch);
  // the first column sweep reads the sparse-first rows through the CSR row
  // starts (rows without samples stay unwritten) when it runs the prefetching
  // cluster kernel; decided here so the row pass knows whether to write zeros
  const int bl0 = cluster_bw_log2(h);
  bool skip_zero = sp && K == 3 && h > 1 && bl0 >= 0 && g_cols_cluster && g_cols_prefetch && g_skip_zero_rows;
  for (int k = 0; k < P.k; ++k)
    if (!P.f64[k]) skip_zero = false;
  if (skip_zero)
    skip_zero = (passes == 1 && fo.flow) ? max_clusters<K, true, true>() > 0 : max_clusters<K, false, true>() > 0;
  for (int i = 1; i <= passes; ++i) {
    double sigma_i = sigma_s * sqrt(3.0) * pow(2.0, passes - i) / den;  // densify.py:104
    double c = -root / sigma_i;
    if (w > 1) {
      kprobe_mark(kr, 0, s);
      if (i == 1 && sp && K == 3)
        klaunch(dt_rows_first_kernel, h, kRowThreads, (size_t)3 * w * sizeof(double) + (size_t)w * 4, s, 
            guide, P, w, h, ratio, c, *sp, !skip_zero);
      else if (rows_bulk_ok(guide, P, w))
        klaunch(dt_rows_bulk_kernel<K>, h, kRowThreads, (size_t)K * w * sizeof(double) + (size_t)w * 4, s, 
            guide, P, w, h, ratio, c);
      else if (w <= kRowThreads * kRowSeg)
        klaunch(dt_rows_reg_kernel<K>, h, kRowThreads, (size_t)K * w * sizeof(double), s, guide, P, w, h,
                                                                                    ratio, c);
      else if (row_smem <= (size_t)g_rows_smem_max[K])
        klaunch(dt_rows_kernel<K>, h, kRowThreads, row_smem, s, guide, P, w, h, ratio, c);
      else  // rows wider than shared memory: the sequential twin (k_twins.cu)
        launch_dt_rows_seq(guide, P, w, h, ratio, c, s);
      kprobe_mark(kr, 1, s);
    }
    int bl = cluster_bw_log2(h);
    bool fin_pass = i == passes && fo.flow && K == 3;
    if (h > 1) kprobe_mark(kc, 0, s);
    if (h > 1 && bl >= 0 && g_cols_cluster) {
      const int32_t* zr = (i == 1 && skip_zero) ? sp->row_start : nullptr;
      if (fin_pass) {
        launch_cols_cluster<K, true>(guide, P, w, h, ratio, c, bl, fo, s, zr);
        finalized = true;
      } else {
        launch_cols_cluster<K, false>(guide, P, w, h, ratio, c, bl, fo, s, zr);
      }
    } else if (h > 1) {
      klaunch(dt_cols_agg<K>, cg, kColThreads, 0, s, guide, P, w, h, ratio, c, agg, 0, nch);
      klaunch(dt_cols_link<K>, ceil_div(w, 32), 1024, 0, s, w, nch, agg, carry);
      if (i == passes && fo.flow && K == 3) {
        klaunch(dt_cols_apply<K, true>, cg, kColThreads, 0, s, guide, P, w, h, ratio, c, carry, fo, 0, nch);
        finalized = true;
      } else {
        klaunch(dt_cols_apply<K, false>, cg, kColThreads, 0, s, guide, P, w, h, ratio, c, carry, fo, 0, nch);
      }
    }
    if (h > 1) kprobe_mark(kc, 1, s);
  }
  return finalized;
}

int64_t dt_scratch_doubles(int w, int h, int k) {
  int nch = ceil_div(h, kColChunk);
  return (int64_t)nch * w * (3 + 2 * k) + (int64_t)nch * w * 2 * k + (int64_t)w * h + 64;
}

void dt_set_cluster_columns(bool on) { g_cols_cluster = on; }
void dt_set_cols_prefetch(bool on) { g_cols_prefetch = on; }
void dt_set_skip_zero_rows(bool on) { g_skip_zero_rows = on; }
void dt_set_cols_grid_div(int d) { g_cols_grid_div = d < 1 ? 1 : d; }

void init_densify_attributes() {
  g_rows_smem_max[1] = allow_max_dynamic_smem(dt_rows_kernel<1>);
  g_rows_smem_max[2] = allow_max_dynamic_smem(dt_rows_kernel<2>);
  g_rows_smem_max[3] = allow_max_dynamic_smem(dt_rows_kernel<3>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<1>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<2>);
  allow_max_dynamic_smem(dt_rows_reg_kernel<3>);
  allow_max_dynamic_smem(dt_rows_bulk_kernel<1>);
  allow_max_dynamic_smem(dt_rows_bulk_kernel<2>);
  allow_max_dynamic_smem(dt_rows_bulk_kernel<3>);
  allow_max_dynamic_smem(dt_rows_first_kernel);
}

bool dt_sparse_first_ok(const float* guide, const DtPlanes& P, int w) {
  return P.k == 3 && w > 1 && rows_bulk_ok(guide, P, w);
}

bool launch_dt_filter(const float* guide, DtPlanes P, int w, int h, double sigma_s, double sigma_r,
                      int passes, double* scratch, cudaStream_t s, const DtFlowOut* fo,
                      KProbe* kr, KProbe* kc, const DtSparse* sp) {
  DtFlowOut none{nullptr, nullptr, 0.0, nullptr};
  const DtFlowOut& f = fo ? *fo : none;
  switch (P.k) {
    case 1: return dt_filter_k<1>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s, kr, kc, sp);
    case 2: return dt_filter_k<2>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s, kr, kc, sp);
    default: return dt_filter_k<3>(guide, P, w, h, sigma_s, sigma_r, passes, scratch, f, s, kr, kc, sp);
  }
}

}  // namespace hdr
