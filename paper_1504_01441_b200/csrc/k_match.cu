// Sparse registration: per-corner SSD search (K6), ordered compaction,
// union-of-inliers weeding with the reference's Philox sampler (K7) and the
// least-squares homography that seeds the next finer level (K8).
//
// Everything stays on the device: counts are device words, grids are sized
// for the tile count (the maximum number of corners) and idle blocks exit,
// so the coarse-to-fine chain of matcher.pyramidal_match (matcher.py:221-263)
// runs without a host round trip and can be captured in one CUDA graph.
#ifdef HDR_FINISH_TIMING
#include <cstdio>
// debug build only: clock64 stamps of finish_level's phases (thread 0)
__device__ long long g_fit_stamps[8];
#define FIT_STAMP(i) \
  if (threadIdx.x == 0) g_fit_stamps[i] = clock64()
#else
#define FIT_STAMP(i) (void)0
#endif
#include "hdr_common.cuh"
#include "hdr_geom.cuh"
#include "hdr_warpfit.cuh"
#include "hdr_internal.h"
#include "hdr_scan.cuh"

namespace hdr {

// ---------------------------------------------------------------- K6
struct SsdKey {
  double score;
  long long d2;
  int cy, cx;
};

// ssd_match tie rule (matcher.py:136-142): min score, then d2, then y, then x
__device__ __forceinline__ bool key_less(const SsdKey& a, const SsdKey& b) {
  if (a.score != b.score) return a.score < b.score;
  if (a.d2 != b.d2) return a.d2 < b.d2;
  if (a.cy != b.cy) return a.cy < b.cy;
  return a.cx < b.cx;
}

__device__ __forceinline__ SsdKey shfl_key(const SsdKey& k, int off) {
  SsdKey o;
  o.score = __shfl_down_sync(0xffffffff, k.score, off);
  o.d2 = __shfl_down_sync(0xffffffff, k.d2, off);
  o.cy = __shfl_down_sync(0xffffffff, k.cy, off);
  o.cx = __shfl_down_sync(0xffffffff, k.cx, off);
  return o;
}

#ifndef HDR_SSD_STRIP
#define HDR_SSD_STRIP 4
#endif
#ifndef HDR_SSD_THREADS
#define HDR_SSD_THREADS 128
#endif
constexpr int kSsdStrip = HDR_SSD_STRIP;      // candidate windows per thread (one row)
constexpr int kSsdThreads = HDR_SSD_THREADS;  // threads per corner

// Block-cooperative exhaustive search; returns true on thread 0 with the
// winner in *best. Window bounds must already be clamped and non-empty.
__device__ bool ssd_search(const float* __restrict__ ref, const float* __restrict__ src,
                           int w, int xr, int yr, int xi, int yi, int cx0, int cx1, int cy0,
                           int cy1, int patch, double* smem, SsdKey* best) {
  int hp = patch / 2;
  int nx = cx1 - cx0 + 1, ny = cy1 - cy0 + 1;
  int sw = nx + patch - 1, sh = ny + patch - 1;
  double* T = smem;
  double* S = smem + patch * patch;
  // staging: rows by warp, columns by lane (no integer division per element),
  // and batches of 8 loads in flight per thread before the stores -- a
  // load -> store chain per element serialises on DRAM latency
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    auto stage = [&](const float* img, int y0, int x0, int rows, int cols, double* dst) {
      const int cstep = (cols + 31) >> 5;  // column steps per row (<= 3 for a 41-wide window)
      const int items = ((rows + nwarp - 1 - wid) / nwarp) * cstep;  // this lane's (row, col) pairs
      for (int b = 0; b < items; b += 8) {
        float v[8];
        int idx[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          int it = b + k;
          int r = wid + (it / cstep) * nwarp, c = lane + (it % cstep) * 32;
          bool ok = it < items && r < rows && c < cols;
          idx[k] = ok ? r * cols + c : -1;
          v[k] = ok ? __ldg(img + (int64_t)(y0 + r) * w + (x0 + c)) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (idx[k] >= 0) dst[idx[k]] = (double)v[k];
      }
    };
    stage(ref, yr - hp, xr - hp, patch, patch, T);
    stage(src, cy0 - hp, cx0 - hp, sh, sw, S);
  }
  __syncthreads();
  SsdKey k;
  k.score = INFINITY; k.d2 = 0x7fffffffffffffffLL; k.cy = 0x7fffffff; k.cx = 0x7fffffff;
  // each thread sweeps a 1xSW strip of candidate windows, sliding an SW-wide
  // register window along the source row: per tap one shared load of S and
  // one (broadcast) of T feed SW FMAs. Every window keeps the same row-major
  // tap order, so identical windows tie exactly as in the reference.
  constexpr int SW = kSsdStrip;
  int nstrip = (nx + SW - 1) / SW;
  for (int t = threadIdx.x; t < nstrip * ny; t += blockDim.x) {
    int oy = t / nstrip, ox = (t - oy * nstrip) * SW;
    double acc[SW];
#pragma unroll
    for (int j = 0; j < SW; ++j) acc[j] = 0.0;
    for (int ky = 0; ky < patch; ++ky) {
      const double* srow = S + (oy + ky) * sw + ox;
      const double* trow = T + ky * patch;
      double win[SW];
#pragma unroll
      for (int j = 0; j < SW - 1; ++j) win[j] = srow[j];
      for (int kx = 0; kx < patch; ++kx) {
        win[SW - 1] = srow[kx + SW - 1];
        double tv = trow[kx];
#pragma unroll
        for (int j = 0; j < SW; ++j) {
          double d = win[j] - tv;
          acc[j] = fma(d, d, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < SW - 1; ++j) win[j] = win[j + 1];
      }
    }
#pragma unroll
    for (int j = 0; j < SW; ++j) {
      if (ox + j >= nx) break;
      SsdKey cand;
      cand.score = acc[j];
      cand.cx = cx0 + ox + j;
      cand.cy = cy0 + oy;
      long long dx = cand.cx - xi, dy = cand.cy - yi;
      cand.d2 = dx * dx + dy * dy;
      if (key_less(cand, k)) k = cand;
    }
  }
  for (int off = 16; off; off >>= 1) {
    SsdKey o = shfl_key(k, off);
    if (key_less(o, k)) k = o;
  }
  __shared__ SsdKey part[32];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) part[warp] = k;
  __syncthreads();
  if (threadIdx.x != 0) return false;
  for (int i = 1; i < (int)((blockDim.x + 31) >> 5); ++i)
    if (key_less(part[i], k)) k = part[i];
  *best = k;
  return true;
}

// matcher._match_level body (matcher.py:186-207) for one detector tile.
__global__ void __launch_bounds__(256) ssd_tiles_kernel(const TileCorner* __restrict__ tiles,
                                                        const float* __restrict__ ref,
                                                        const float* __restrict__ src, int w,
                                                        int h, const double* __restrict__ hpred,
                                                        int radius, int patch,
                                                        MatchRow* __restrict__ rows,
                                                        uint8_t* __restrict__ flags) {
  pdl_wait();
  extern __shared__ double smem[];
  int slot = blockIdx.x;
  TileCorner tc = tiles[slot];
  int hp = patch / 2;
  bool ok = tc.x >= 0;
  int x = tc.x, y = tc.y, xi = 0, yi = 0;
  if (ok && !(hp <= x && x <= w - 1 - hp && hp <= y && y <= h - 1 - hp)) ok = false;
  if (ok) {
    double H[9];
    for (int i = 0; i < 9; ++i) H[i] = hpred[i];
    double xn, yn, nx, ny;
    to_norm((double)x, (double)y, w, h, &xn, &yn);
    double den = apply_h(H, xn, yn, &nx, &ny);
    if (fabs(den) < 1e-12) {
      ok = false;
    } else {
      double px, py;
      from_norm(nx / den, ny / den, w, h, &px, &py);
      if (!(isfinite(px) && isfinite(py))) ok = false;
      else if (fabs(px) > 8.0 * w || fabs(py) > 8.0 * h) ok = false;
      else { xi = (int)rint(px); yi = (int)rint(py); }  // Python round(): half-even
    }
  }
  int cx0 = max(xi - radius, hp), cx1 = min(xi + radius, w - 1 - hp);
  int cy0 = max(yi - radius, hp), cy1 = min(yi + radius, h - 1 - hp);
  if (ok && (cx0 > cx1 || cy0 > cy1)) ok = false;
  if (!ok) {
    if (threadIdx.x == 0) flags[slot] = 0;
    return;
  }
  SsdKey best;
  if (ssd_search(ref, src, w, x, y, xi, yi, cx0, cx1, cy0, cy1, patch, smem, &best)) {
    MatchRow r;
    r.v[0] = x; r.v[1] = y; r.v[2] = best.cx; r.v[3] = best.cy; r.v[4] = best.score;
    rows[slot] = r;
    flags[slot] = 1;
  }
}

// matcher.ssd_match for explicit (x_ref, y_ref, x_init, y_init) points.
__global__ void __launch_bounds__(256) ssd_points_kernel(const float* __restrict__ ref,
                                                         const float* __restrict__ src, int w,
                                                         int h, const int32_t* __restrict__ pts,
                                                         int radius, int patch,
                                                         double* __restrict__ out,
                                                         uint8_t* __restrict__ found) {
  pdl_wait();
  extern __shared__ double smem[];
  int i = blockIdx.x;
  int hp = patch / 2;
  int xr = pts[4 * i], yr = pts[4 * i + 1], xi = pts[4 * i + 2], yi = pts[4 * i + 3];
  if (!(hp <= xr && xr <= w - 1 - hp && hp <= yr && yr <= h - 1 - hp)) {
    if (threadIdx.x == 0) found[i] = 2;  // reference raises ValueError
    return;
  }
  int cx0 = max(xi - radius, hp), cx1 = min(xi + radius, w - 1 - hp);
  int cy0 = max(yi - radius, hp), cy1 = min(yi + radius, h - 1 - hp);
  if (cx0 > cx1 || cy0 > cy1) {
    if (threadIdx.x == 0) found[i] = 0;
    return;
  }
  SsdKey best;
  if (ssd_search(ref, src, w, xr, yr, xi, yi, cx0, cx1, cy0, cy1, patch, smem, &best)) {
    out[3 * i] = best.cx; out[3 * i + 1] = best.cy; out[3 * i + 2] = best.score;
    found[i] = 1;
  }
}

static size_t ssd_smem(int radius, int patch) {
  size_t side = 2 * (size_t)radius + patch;
  return (side * side + (size_t)patch * patch + 8) * sizeof(double);
}

constexpr int kSsdMaxSmem = 200 * 1024;

static void init_finish_attributes();

void init_match_attributes() {
  allow_max_dynamic_smem(ssd_tiles_kernel);
  allow_max_dynamic_smem(ssd_points_kernel);
  init_finish_attributes();
}

void launch_ssd_tiles(const TileCorner* tiles, int ntiles, const float* ref, const float* src,
                      int w, int h, const double* hpred, int radius, int patch, MatchRow* rows,
                      uint8_t* flags, cudaStream_t s) {
  size_t bytes = ssd_smem(radius, patch);
  klaunch(ssd_tiles_kernel, ntiles, kSsdThreads, bytes, s, tiles, ref, src, w, h, hpred, radius, patch, rows,
                                              flags);
}

void launch_ssd_points(const float* ref, const float* src, int w, int h, const int32_t* pts,
                       int n, int radius, int patch, double* out, uint8_t* found,
                       cudaStream_t s) {
  if (n <= 0) return;
  size_t bytes = ssd_smem(radius, patch);
  klaunch(ssd_points_kernel, n, kSsdThreads, bytes, s, ref, src, w, h, pts, radius, patch, out, found);
}

// ordered compaction of per-slot rows (tile order is the reference's corner
// order, matcher.py:97-104 -> :187)
// mask / witness (may be null): the weeding arrays of the n rows that follow,
// cleared here so the pair needs no memset node between this kernel and
// weed_kernel (a memset would also break the programmatic launch chain)
__global__ void __launch_bounds__(1024) compact_rows_kernel(const MatchRow* __restrict__ rows,
                                                            const uint8_t* __restrict__ flags,
                                                            int nslots, MatchRow* __restrict__ out,
                                                            int32_t* __restrict__ count,
                                                            double* __restrict__ out_copy,
                                                            uint32_t* __restrict__ mask,
                                                            int32_t* __restrict__ witness) {
  pdl_wait();
  if (mask) {
    for (int i = threadIdx.x; i < (nslots + 31) / 32 + 1; i += blockDim.x) mask[i] = 0u;
    for (int i = threadIdx.x; i < nslots + 1; i += blockDim.x) witness[i] = 0;
  }
  __shared__ int scratch[32];
  int base = 0;
  for (int c0 = 0; c0 < nslots; c0 += blockDim.x) {
    int i = c0 + threadIdx.x;
    int f = (i < nslots && flags[i] == 1) ? 1 : 0;
    int total;
    int pos = block_exclusive_scan(f, scratch, &total);
    if (f) {
      MatchRow r = rows[i];
      out[base + pos] = r;
      if (out_copy)
        for (int k = 0; k < 5; ++k) out_copy[5 * (int64_t)(base + pos) + k] = r.v[k];
    }
    base += total;
  }
  if (threadIdx.x == 0) *count = base;
}

void launch_compact_rows(const MatchRow* rows, const uint8_t* flags, int nslots, MatchRow* out,
                         int32_t* count, double* out_copy, cudaStream_t s, uint32_t* mask,
                         int32_t* witness) {
  klaunch(compact_rows_kernel, 1, 1024, 0, s, rows, flags, nslots, out, count, out_copy, mask, witness);
}

// ---------------------------------------------------------------- K7
__device__ __forceinline__ void norm_row(const MatchRow& r, int w, int h, double* p) {
  to_norm(r.v[0], r.v[1], w, h, &p[0], &p[1]);
  to_norm(r.v[2], r.v[3], w, h, &p[2], &p[3]);
}

__device__ __forceinline__ int weed_delta(int n, int delta) {
  if (delta >= 0) return delta;
  int d = (int)ceil(0.15 * (double)n);  // weeding.default_delta (weeding.py:30-32)
  return d > 12 ? d : 12;
}

// One block per RANSAC iteration (weeding.py:69-89). Warp 0 draws with
// resampling (weeding.py:74-84; every lane runs the same Philox stream) and
// fits the four-point homography spread over its lanes (warp_fit4); then the
// whole block tests the symmetric transfer error of every match against it
// and OR-s an accepted inlier set into the reliable mask. One kernel per
// level instead of a fit kernel + a count kernel with the fits in between.
__global__ void __launch_bounds__(256) weed_kernel(const MatchRow* __restrict__ rows,
                                                   const int32_t* __restrict__ count, int w, int h,
                                                   double eps, int delta, const uint64_t* __restrict__ keys,
                                                   uint32_t* __restrict__ mask, int32_t* __restrict__ witness,
                                                   int32_t* __restrict__ grey) {
  pdl_wait();
  __shared__ WarpFitSmem wsm;
  __shared__ double Hs[18];
  __shared__ int okf;
  const int it = blockIdx.x, lane = threadIdx.x & 31;
  const int n = *count;
  if (n < 4) return;
  if (threadIdx.x < 32) {
    Philox g;
    philox_init(&g, keys[2 * it], keys[2 * it + 1]);
    double H[9];
    int g_local = 0;
    bool ok = false;
    for (int r = 0; r < kMaxResample && !ok; ++r) {
      int idx[4];
      choice4(&g, n, idx);
      double px[4], py[4], qx[4], qy[4];
      for (int k = 0; k < 4; ++k) {
        double p[4];
        norm_row(rows[idx[k]], w, h, p);
        px[k] = p[0]; py[k] = p[1]; qx[k] = p[2]; qy[k] = p[3];
      }
      ok = warp_fit4(px, py, qx, qy, H, &g_local, &wsm) == 0;
    }
    double Hi[9];
    ok = ok && inv3(H, Hi);
    if (lane == 0) {
      if (g_local) atomicAdd(grey, g_local);
      for (int k = 0; k < 9; ++k) { Hs[k] = H[k]; Hs[9 + k] = Hi[k]; }
      okf = ok;
    }
  }
  __syncthreads();
  if (!okf) return;
  int total = 0;
  uint32_t bits = 0;  // inlier bits of this thread's first 32 chunks
  for (int c0 = 0, k = 0; c0 < n; c0 += blockDim.x, ++k) {
    int i = c0 + threadIdx.x;
    bool in = false;
    if (i < n) {
      double p[4];
      norm_row(rows[i], w, h, p);
      in = is_inlier(Hs, Hs + 9, p[0], p[1], p[2], p[3], eps);
    }
    if (in && k < 32) bits |= 1u << k;
    total += __syncthreads_count(in);
  }
  if (total <= weed_delta(n, delta)) return;
  for (int c0 = 0, k = 0; c0 < n; c0 += blockDim.x, ++k) {
    int i = c0 + threadIdx.x;
    bool in;
    if (k < 32) {
      in = (bits >> k) & 1u;
    } else {
      in = false;
      if (i < n) {
        double p[4];
        norm_row(rows[i], w, h, p);
        in = is_inlier(Hs, Hs + 9, p[0], p[1], p[2], p[3], eps);
      }
    }
    unsigned word = __ballot_sync(0xffffffff, in);
    if (lane == 0 && word) atomicOr(&mask[i >> 5], word);
    if (in) atomicMax(&witness[i], total);
  }
}

void launch_weed(const MatchRow* rows, const int32_t* count, int n_static, int w, int h,
                 int iterations, double eps, const uint64_t* keys, int delta, uint32_t* mask,
                 int32_t* witness, int32_t* grey, cudaStream_t s, bool cleared) {
  if (!cleared) {
    cudaMemsetAsync(mask, 0, sizeof(uint32_t) * ((n_static + 31) / 32 + 1), s);
    cudaMemsetAsync(witness, 0, sizeof(int32_t) * (n_static + 1), s);
  }
  klaunch(weed_kernel, iterations, 256, 0, s, rows, count, w, h, eps, delta, keys, mask, witness, grey);
}

// ---------------------------------------------------------------- K8
constexpr int kFitCache = 4096;  // weeded points held in shared memory by finish_level
constexpr int kCompactWords = 2048;  // mask words (65536 rows) whose prefix finish_level keeps in shared memory
// the bits of mask word k that are rows below n
__device__ __forceinline__ uint32_t word_bits(int k, int n) {
  int r = n - 32 * k;
  return r >= 32 ? 0xffffffffu : (1u << r) - 1u;
}

// entry k of DLT row r (0 or 1) of correspondence p -> q (geometry.py:51-63)
__device__ __forceinline__ double dlt_entry(int r, int k, double px, double py, double qx,
                                            double qy) {
  int lo = r ? 3 : 0;
  if (k == lo) return -px;
  if (k == lo + 1) return -py;
  if (k == lo + 2) return -1.0;
  double q = r ? qy : qx;
  if (k == 6) return px * q;
  if (k == 7) return py * q;
  if (k == 8) return q;
  return 0.0;
}
// Block-wide least-squares DLT (geometry.fit_homography for n >= 4) over
// points fetched by `get(i, p)` (p = ref x, ref y, src x, src y).
template <class Get>
__device__ int block_fit(int n, Get get, double* H, int32_t* grey) {

  __shared__ double red[32][6];
  __shared__ double bc[6];
  __shared__ int status;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nw = (blockDim.x + 31) >> 5;
  __shared__ WarpFitSmem wfs;
  if (n == 4) {
    if (warp == 0) {
      double px[4], py[4], qx[4], qy[4];
      for (int k = 0; k < 4; ++k) {
        double p[4];
        get(k, p);
        px[k] = p[0]; py[k] = p[1]; qx[k] = p[2]; qy[k] = p[3];
      }
      int g = 0;
      double Hl[9];
      int st = warp_fit4(px, py, qx, qy, Hl, &g, &wfs);
      if (lane == 0) {
        status = st;
        for (int k = 0; k < 9; ++k) H[k] = Hl[k];
        if (g && grey) atomicAdd(grey, g);
      }
    }
    __syncthreads();
    return status;
  }
  // centroids
  double s[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double p[4];
    get(i, p);
    for (int k = 0; k < 4; ++k) s[k] += p[k];
  }
  for (int k = 0; k < 4; ++k)
    for (int off = 16; off; off >>= 1) s[k] += __shfl_down_sync(0xffffffff, s[k], off);
  if (lane == 0)
    for (int k = 0; k < 4; ++k) red[warp][k] = s[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) {
      double a = 0.0;
      for (int j = 0; j < nw; ++j) a += red[j][k];
      bc[k] = a / (double)n;
    }
  }
  __syncthreads();
  FIT_STAMP(2);
  // mean distances to the centroids
  double md[2] = {0, 0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double p[4];
    get(i, p);
    md[0] += hypot(p[0] - bc[0], p[1] - bc[1]);
    md[1] += hypot(p[2] - bc[2], p[3] - bc[3]);
  }
  for (int k = 0; k < 2; ++k)
    for (int off = 16; off; off >>= 1) md[k] += __shfl_down_sync(0xffffffff, md[k], off);
  __syncthreads();
  if (lane == 0) { red[warp][0] = md[0]; red[warp][1] = md[1]; }
  __syncthreads();
  __shared__ double tr[3], ts[3];
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int j = 0; j < nw; ++j) { a += red[j][0]; b += red[j][1]; }
    a /= (double)n;
    b /= (double)n;
    status = (a < 1e-12 || b < 1e-12) ? 2 : 0;
#ifdef HDR_DEBUG_FIT
    printf("block_fit: n=%d md=%g %g c=%g %g %g %g\n", n, a, b, bc[0], bc[1], bc[2], bc[3]);
#endif
    double sr = sqrt(2.0) / a, ss = sqrt(2.0) / b;
    tr[0] = sr; tr[1] = -sr * bc[0]; tr[2] = -sr * bc[1];
    ts[0] = ss; ts[1] = -ss * bc[2]; ts[2] = -ss * bc[3];
  }
  __syncthreads();
  FIT_STAMP(3);
  if (status) return status;
  // Gram matrix of the conditioned DLT rows. With p~ = (px, py, 1), rows are
  // r0 = [-p~, 0, qx p~], r1 = [0, -p~, qy p~], so G is assembled from 24 sums
  // S_w = sum w p~ p~^T (6 unique entries each) for w in {1, qx, qy, qx^2+qy^2}.
  double acc[24];
#pragma unroll
  for (int k = 0; k < 24; ++k) acc[k] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double p[4];
    get(i, p);
    double px = (p[0] - bc[0]) * tr[0], py = (p[1] - bc[1]) * tr[0];
    double qx = (p[2] - bc[2]) * ts[0], qy = (p[3] - bc[3]) * ts[0];
    double mono[6] = {px * px, px * py, px, py * py, py, 1.0};
    double wts[4] = {1.0, qx, qy, qx * qx + qy * qy};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 6; ++b) acc[6 * a + b] += wts[a] * mono[b];
  }
  __shared__ double gsh[8][24];
  __shared__ double g45s[45];
#pragma unroll
  for (int k = 0; k < 24; ++k) {
    double v = acc[k];
    for (int off = 16; off; off >>= 1) v += __shfl_down_sync(0xffffffff, v, off);
    if (lane == 0) gsh[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double S[24];
    for (int k = 0; k < 24; ++k) {
      double v = 0.0;
      for (int j = 0; j < nw; ++j) v += gsh[j][k];
      S[k] = v;
    }
    // unique (i <= j) entries of the 3x3 blocks, monomial order above
    const int mi[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
    double G[9][9];
    for (int i = 0; i < 9; ++i)
      for (int j = 0; j < 9; ++j) G[i][j] = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        int m = mi[i][j];
        G[i][j] = G[3 + i][3 + j] = S[m];
        G[i][6 + j] = G[6 + j][i] = -S[6 + m];
        G[3 + i][6 + j] = G[6 + j][3 + i] = -S[12 + m];
        G[6 + i][6 + j] = S[18 + m];
      }
    int k = 0;
    for (int i = 0; i < 9; ++i)
      for (int j = i; j < 9; ++j) g45s[k++] = G[i][j];
    int g = 0;
    FIT_STAMP(4);
    status = fit_from_gram(g45s, tr, ts, H, &g);
    FIT_STAMP(5);
    if (g && grey) atomicAdd(grey, g);
  }
  __syncthreads();
  return status;
}

// Close one pyramid level (matcher.py:247-260): compact the weeded set in
// index order (np.flatnonzero), record level_counts, fit the LSQ H and hand
// it to the next finer level; level 0 also fills the user-visible outputs.
__global__ void __launch_bounds__(256, 1) finish_level_kernel(
    const MatchRow* __restrict__ raw, const int32_t* __restrict__ raw_count,
    const uint32_t* __restrict__ mask, int w, int h, int level, MatchRow* __restrict__ weeded,
    int32_t* __restrict__ weeded_count, int64_t* __restrict__ kept_idx,
    double* __restrict__ hpred, double* __restrict__ homography, int32_t* __restrict__ info,
    double* __restrict__ out_matches, double* __restrict__ out_raw, int32_t* grey) {
  pdl_wait();
  FIT_STAMP(0);
  extern __shared__ double pts_cache[];  // normalised (rx, ry, sx, sy) of the weeded set
  __shared__ int scratch[32];
  __shared__ int word_base[kCompactWords];
  int n = *raw_count;
  int m = 0;
  bool cached = n <= kFitCache;
  auto put_row = [&](int i, int pos) {
    const MatchRow rw = raw[i];
    weeded[pos] = rw;
    if (cached) norm_row(rw, w, h, pts_cache + 4 * pos);
    if (kept_idx) kept_idx[pos] = i;
    if (out_matches)
      for (int k = 0; k < 5; ++k) out_matches[5 * (int64_t)pos + k] = rw.v[k];
  };
  if (n >= 4) {
    // np.flatnonzero order: the exclusive prefix of the mask words' popcounts
    // (thread t owns the contiguous words [t W, t W + W)) goes to shared
    // memory, then every kept row r lands at word_base[r / 32] + (set bits
    // below r in its word), rows dealt out one per thread so all of a
    // thread's row loads are independent and in flight together
    const int nw = (n + 31) >> 5;
    const int W = (nw + blockDim.x - 1) / blockDim.x;
    const int w0 = min(nw, (int)threadIdx.x * W), w1 = min(nw, w0 + W);
    const bool in_smem = nw <= kCompactWords;
    int cnt = 0;
    for (int k = w0; k < w1; ++k) cnt += __popc(mask[k] & word_bits(k, n));
    int pos = block_exclusive_scan(cnt, scratch, &m);
    if (in_smem) {
      for (int k = w0; k < w1; ++k) {
        word_base[k] = pos;
        pos += __popc(mask[k] & word_bits(k, n));
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t mw = mask[i >> 5];
        if (!((mw >> (i & 31)) & 1u)) continue;
        put_row(i, word_base[i >> 5] + __popc(mw & ((1u << (i & 31)) - 1u)));
      }
    } else {
      for (int k = w0; k < w1; ++k)
        for (uint32_t b = mask[k] & word_bits(k, n); b; b &= b - 1) put_row(32 * k + __ffs(b) - 1, pos++);
    }
  }
  if (threadIdx.x == 0) {
    *weeded_count = m;
    if (info) {
      info[3 + 2 * level] = n;
      info[4 + 2 * level] = m;
      if (level == 0) { info[16] = m; info[17] = n; }
    }
  }
  if (m < 4) return;
  __shared__ double Hs[9];
  const MatchRow* wr = weeded;
  auto get = [&](int i, double* p) {
    if (cached) {
      const double* q = pts_cache + 4 * i;
      p[0] = q[0]; p[1] = q[1]; p[2] = q[2]; p[3] = q[3];
    } else {
      norm_row(wr[i], w, h, p);
    }
  };
  __syncthreads();  // weeded rows / cached points visible block-wide
  FIT_STAMP(1);
  int st = block_fit(m, get, Hs, grey);
  FIT_STAMP(6);
#ifdef HDR_FINISH_TIMING
  if (threadIdx.x == 0)
    printf("finish L%d n=%d m=%d compact %lld centroid %lld md %lld gram %lld solve %lld tail %lld\n", level, n, m,
           g_fit_stamps[1] - g_fit_stamps[0], g_fit_stamps[2] - g_fit_stamps[1], g_fit_stamps[3] - g_fit_stamps[2],
           g_fit_stamps[4] - g_fit_stamps[3], g_fit_stamps[5] - g_fit_stamps[4], g_fit_stamps[6] - g_fit_stamps[5]);
#endif

  if (threadIdx.x == 0 && st == 0) {
    for (int k = 0; k < 9; ++k) hpred[k] = Hs[k];
    if (level == 0 && homography) {
      for (int k = 0; k < 9; ++k) homography[k] = Hs[k];
      if (info) info[1] = 1;
    }
  }
}

void launch_finish_level(const MatchRow* raw, const int32_t* raw_count, const uint32_t* mask,
                         int w, int h, int level, MatchRow* weeded, int32_t* weeded_count,
                         int64_t* kept_idx, double* hpred, double* homography, int32_t* info,
                         double* out_matches, double* out_raw, int32_t* grey, cudaStream_t s) {
  (void)out_raw;
  klaunch(finish_level_kernel, 1, 256, kFitCache * 4 * sizeof(double), s, raw, raw_count, mask, w, h, level, weeded, weeded_count,
                                        kept_idx, hpred, homography, info, out_matches, out_raw,
                                        grey);
}

// matcher.fit_matches_homography over device rows (count on the device)
__global__ void __launch_bounds__(256) fit_rows_kernel(const MatchRow* __restrict__ rows,
                                                       const int32_t* __restrict__ count, int w,
                                                       int h, double* __restrict__ H,
                                                       int32_t* __restrict__ status) {
  pdl_wait();
  int n = *count;
  if (n < 4) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  __shared__ double Hs[9];
  auto get = [&](int i, double* p) { norm_row(rows[i], w, h, p); };
  int st = block_fit(n, get, Hs, nullptr);
  if (threadIdx.x == 0) {
    *status = st;
    if (st == 0)
      for (int k = 0; k < 9; ++k) H[k] = Hs[k];
  }
}

void launch_fit_rows(const MatchRow* rows, const int32_t* count, int w, int h, double* H,
                     int32_t* status, cudaStream_t s) {
  klaunch(fit_rows_kernel, 1, 256, 0, s, rows, count, w, h, H, status);
}

// geometry.fit_homography on explicit point arrays
__global__ void __launch_bounds__(256) fit_points_kernel(const double* __restrict__ rp,
                                                         const double* __restrict__ sp, int n,
                                                         double* __restrict__ H,
                                                         int32_t* __restrict__ status) {
  pdl_wait();
  __shared__ double Hs[9];
  auto get = [&](int i, double* p) {
    p[0] = rp[2 * i]; p[1] = rp[2 * i + 1]; p[2] = sp[2 * i]; p[3] = sp[2 * i + 1];
  };
  int st = block_fit(n, get, Hs, nullptr);
  if (threadIdx.x == 0) {
    *status = st;
    if (st == 0)
      for (int k = 0; k < 9; ++k) H[k] = Hs[k];
  }
}

void launch_fit_points(const double* ref_pts, const double* src_pts, int n, double* H,
                       int32_t* status, cudaStream_t s) {
  klaunch(fit_points_kernel, 1, 256, 0, s, ref_pts, src_pts, n, H, status);
}

__global__ void inlier_mask_kernel(const double* __restrict__ H, const double* __restrict__ rp,
                                   const double* __restrict__ sp, int n, double eps,
                                   uint8_t* __restrict__ mask) {
  pdl_wait();
  __shared__ double Hs[18];
  __shared__ int okinv;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 9; ++k) Hs[k] = H[k];
    okinv = inv3(Hs, Hs + 9);
  }
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  mask[i] = okinv ? is_inlier(Hs, Hs + 9, rp[2 * i], rp[2 * i + 1], sp[2 * i], sp[2 * i + 1], eps)
                  : 0;
}

void launch_inlier_mask(const double* H, const double* ref_pts, const double* src_pts, int n,
                        double eps, uint8_t* mask, cudaStream_t s) {
  if (n <= 0) return;
  klaunch(inlier_mask_kernel, ceil_div(n, 256), 256, 0, s, H, ref_pts, src_pts, n, eps, mask);
}

__global__ void set_identity_kernel(double* h) {
  pdl_wait();
  int i = threadIdx.x;
  if (i < 9) h[i] = (i % 4 == 0) ? 1.0 : 0.0;
}

void launch_set_identity(double* h, cudaStream_t s) { klaunch(set_identity_kernel, 1, 32, 0, s, h); }

static void init_finish_attributes() { allow_max_dynamic_smem(finish_level_kernel); }

}  // namespace hdr
