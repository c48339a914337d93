// Warp-level form of the four-point fit of weeding's RANSAC hypotheses
// (geometry.fit_homography with n = 4, geometry.py:35-77; the serial
// __host__ __device__ fit4 in hdr_geom.cuh backs the host test hook): the
// pivoted Householder QR of the 9x8 matrix A^T with one COLUMN per lane.
//
// With a column per lane, the column norms and Householder dot products are
// lane-local sums in fit4's own order, so every result is bit-identical to
// fit4; the lanes only exchange the pivot (an argmax) and the current
// Householder vector. The step loop stays rolled: fit4 fully unrolled is
// ~10k straight-line instructions run once per hypothesis, and one thread per
// hypothesis spent most of its time on instruction-cache misses (ncu:
// no_instruction 45% of weed_fit's stalls); a warp per hypothesis with the
// rolled loop took weed_fit from ~37 to ~25 us per level.
//
// Measured and not kept: the same treatment of the least-squares solve
// (fit_from_gram, a column of the 9x9 Cholesky per lane, inverse iteration
// by every lane): its chain of dependent shuffles, selects, sqrt and
// reciprocal costs ~1.6k cycles per Cholesky step and ~7.8k per inverse
// iteration (clock64 trace), ~46k cycles against ~25k for the serial form.
//
// Every lane of the warp calls it and receives the same status and H.
#pragma once
#include "hdr_geom.cuh"

namespace hdr {

constexpr unsigned kFull = 0xffffffffu;

// Per-warp shared scratch of the solvers.
struct WarpFitSmem {
  double L[81];     // Cholesky factor by columns / R of the QR grey zone
  double rdiag[8], beta[8], s[8], il[9];
  int perm[9];
};

// x[k] for a runtime k over a register array (predicated selects)
template <int N>
__device__ __forceinline__ double pick(const double (&x)[N], int k) {
  double v = x[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (i == k) v = x[i];
  return v;
}

// first maximum (lowest index on ties) of v over the lanes, as (value, index)
__device__ __forceinline__ void warp_argmax(double& v, int& idx, int width) {
  for (int o = width >> 1; o; o >>= 1) {
    double ov = __shfl_xor_sync(kFull, v, o);
    int oi = __shfl_xor_sync(kFull, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
}

__device__ __noinline__ void jacobi8_device(double* a, double* s) { jacobi_singular_values(a, 8, s); }

// geometry.fit_homography for n = 4 (fit4 in hdr_geom.cuh).
__device__ __noinline__ int warp_fit4(const double* px_in, const double* py_in, const double* qx_in,
                                      const double* qy_in, double* H, int* grey, WarpFitSmem* sm) {
  const int lane = threadIdx.x & 31;
  double px[4], py[4], qx[4], qy[4], tr[3], ts[3];
#pragma unroll
  for (int i = 0; i < 4; ++i) { px[i] = px_in[i]; py[i] = py_in[i]; qx[i] = qx_in[i]; qy[i] = qy_in[i]; }
  if (!hartley(px, py, 4, tr)) return 2;
  if (!hartley(qx, qy, 4, ts)) return 2;
  // column c = lane of M = A^T: row 2i (c even) or 2i+1 (c odd) of A
  const int c = lane < 8 ? lane : 7;
  double M[9];
  {
    const int i = c >> 1;
    double p0 = px[0], p1 = py[0], q0 = qx[0], q1 = qy[0];
#pragma unroll
    for (int t = 1; t < 4; ++t)
      if (t == i) { p0 = px[t]; p1 = py[t]; q0 = qx[t]; q1 = qy[t]; }
    double r0[9], r1[9];
    dlt_rows(p0, p1, q0, q1, r0, r1);
#pragma unroll
    for (int r = 0; r < 9; ++r) M[r] = (c & 1) ? r1[r] : r0[r];
  }
#pragma unroll 1
  for (int k = 0; k < 8; ++k) {
    double cn = 0.0;
#pragma unroll
    for (int r = 0; r < 9; ++r)
      if (r >= k) cn += M[r] * M[r];
    double best = (lane < 8 && lane >= k) ? cn : -1.0;
    int piv = lane < 8 ? lane : 31;
    warp_argmax(best, piv, 32);
    const int src = lane == k ? piv : (lane == piv ? k : lane);
#pragma unroll
    for (int r = 0; r < 9; ++r) M[r] = __shfl_sync(kFull, M[r], src);
    const double nrm = sqrt(best);
    const double mkk = __shfl_sync(kFull, pick(M, k), k);
    const double alpha = (mkk > 0.0) ? -nrm : nrm;
    if (lane == k)
#pragma unroll
      for (int r = 0; r < 9; ++r)
        if (r == k) M[r] -= alpha;
    double v[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) v[r] = __shfl_sync(kFull, M[r], k);
    double vv = 0.0;
#pragma unroll
    for (int r = 0; r < 9; ++r)
      if (r >= k) vv += v[r] * v[r];
    const double bk = (vv > 0.0) ? 2.0 / vv : 0.0;
    if (lane == 0) { sm->beta[k] = bk; sm->rdiag[k] = alpha; }
    if (lane > k && lane < 8) {
      double d = 0.0;
#pragma unroll
      for (int r = 0; r < 9; ++r)
        if (r >= k) d += v[r] * M[r];
      d *= bk;
#pragma unroll
      for (int r = 0; r < 9; ++r)
        if (r >= k) M[r] -= d * v[r];
    }
  }
  __syncwarp();
  const double ratio = fabs(sm->rdiag[6]) / fabs(sm->rdiag[0]);
  bool degenerate = !(ratio > 1e-9);
  if (ratio > 1e-13 && ratio < 1e-6) {
    // grey zone (rare): exact singular values of R by one lane
    if (lane < 8)
#pragma unroll
      for (int i = 0; i < 8; ++i) sm->L[i * 8 + lane] = (lane > i) ? M[i] : (lane == i ? sm->rdiag[i] : 0.0);
    __syncwarp();
    if (lane == 0) {
      jacobi8_device(sm->L, sm->s);
      if (grey) ++*grey;
    }
    __syncwarp();
    degenerate = sm->s[6] <= 1e-9 * sm->s[0];
    __syncwarp();
  }
  if (degenerate) return 2;
  // null vector = Q e_9 = H0 H1 ... H7 e_9 (every lane, the same order)
  double y[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) y[r] = r == 8 ? 1.0 : 0.0;
#pragma unroll 1
  for (int k = 7; k >= 0; --k) {
    double v[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) v[r] = __shfl_sync(kFull, M[r], k);
    double d = 0.0;
#pragma unroll
    for (int r = 0; r < 9; ++r)
      if (r >= k) d += v[r] * y[r];
    d *= sm->beta[k];
#pragma unroll
    for (int r = 0; r < 9; ++r)
      if (r >= k) y[r] -= d * v[r];
  }
  return finish_h(y, tr, ts, H);
}

}  // namespace hdr
