// Small dense geometry kernels shared by the weeding and least-squares paths,
// written once as __host__ __device__ code (the host copy backs the test hooks).
//
//  * Philox4x64-10 + numpy's bounded-integer and choice(replace=False)
//    samplers (weeding.py:62-84).
//  * Hartley-conditioned DLT fits with the reference's DegenerateFit rules
//    (geometry.py:22-77).
//  * 3x3 inverse / determinant and the symmetric transfer test
//    (geometry.py:96-121).
#pragma once
#include "hdr_common.cuh"

namespace hdr {

// ------------------------------------------------------------------ Philox
struct Philox {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
  int has32;
  uint32_t u32;
};

HD void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

HD void philox_init(Philox* g, uint64_t k0, uint64_t k1) {
  g->ctr[0] = g->ctr[1] = g->ctr[2] = g->ctr[3] = 0;
  g->key[0] = k0;
  g->key[1] = k1;
  g->pos = 4;  // empty buffer: the first draw bumps the counter to 1
  g->has32 = 0;
  g->u32 = 0;
}

HD void philox_block(const uint64_t* ctr, const uint64_t* key, uint64_t* out) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

HD uint64_t philox_next64(Philox* g) {
  if (g->pos < 4) return g->buf[g->pos++];
  if (++g->ctr[0] == 0)
    if (++g->ctr[1] == 0)
      if (++g->ctr[2] == 0) ++g->ctr[3];
  philox_block(g->ctr, g->key, g->buf);
  g->pos = 1;
  return g->buf[0];
}

// low half first, then the high half of the same 64-bit draw
HD uint32_t philox_next32(Philox* g) {
  if (g->has32) {
    g->has32 = 0;
    return g->u32;
  }
  uint64_t v = philox_next64(g);
  g->has32 = 1;
  g->u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// numpy random_bounded_uint64(off=0, rng, use_masked=0) for rng < 2^32-1:
// Lemire's multiply-shift with rejection.
HD uint32_t bounded32(Philox* g, uint32_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFu) return philox_next32(g);
  uint32_t excl = rng + 1u;
  uint64_t m = (uint64_t)philox_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (uint64_t)philox_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// Generator.choice(n, 4, replace=False): Floyd's algorithm over
// j = n-4 .. n-1 then a Fisher-Yates shuffle of the 4 picks.
HD void choice4(Philox* g, int n, int* idx) {
  for (int k = 0; k < 4; ++k) {
    int j = n - 4 + k;
    int v = (int)bounded32(g, (uint32_t)j);
    bool seen = false;
    for (int t = 0; t < k; ++t) seen |= (idx[t] == v);
    idx[k] = seen ? j : v;
  }
  for (int i = 3; i >= 1; --i) {
    int j = (int)bounded32(g, (uint32_t)i);
    int t = idx[i];
    idx[i] = idx[j];
    idx[j] = t;
  }
}

// ------------------------------------------------------------------ 3x3
HD double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

// LU with partial pivoting (LAPACK dgesv against I, as np.linalg.inv).
// Returns false for an exactly singular matrix (numpy raises LinAlgError).
HD bool inv3(const double* m, double* out) {
  double a[9];
  int piv[3] = {0, 1, 2};
  for (int i = 0; i < 9; ++i) a[i] = m[i];
  for (int k = 0; k < 3; ++k) {
    int p = k;
    double best = fabs(a[3 * k + k]);
    for (int i = k + 1; i < 3; ++i)
      if (fabs(a[3 * i + k]) > best) { best = fabs(a[3 * i + k]); p = i; }
    if (best == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < 3; ++j) { double t = a[3 * k + j]; a[3 * k + j] = a[3 * p + j]; a[3 * p + j] = t; }
      int t = piv[k]; piv[k] = piv[p]; piv[p] = t;
    }
    double r = 1.0 / a[3 * k + k];
    for (int i = k + 1; i < 3; ++i) {
      a[3 * i + k] *= r;
      for (int j = k + 1; j < 3; ++j) a[3 * i + j] -= a[3 * i + k] * a[3 * k + j];
    }
  }
  for (int c = 0; c < 3; ++c) {
    double x[3];
    for (int i = 0; i < 3; ++i) x[i] = (piv[i] == c) ? 1.0 : 0.0;
    for (int i = 1; i < 3; ++i)
      for (int j = 0; j < i; ++j) x[i] -= a[3 * i + j] * x[j];
    for (int i = 2; i >= 0; --i) {
      for (int j = i + 1; j < 3; ++j) x[i] -= a[3 * i + j] * x[j];
      x[i] /= a[3 * i + i];
    }
    for (int i = 0; i < 3; ++i) out[3 * i + c] = x[i];
  }
  return true;
}

HD void matmul3(const double* a, const double* b, double* c) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = dadd(dadd(dmul(a[3 * i], b[j]), dmul(a[3 * i + 1], b[3 + j])),
                          dmul(a[3 * i + 2], b[6 + j]));
}

// geometry._transfer_distance (geometry.py:96-104) for one pair.
HD double transfer_dist(const double* H, double x, double y, double tx, double ty) {
  double nx, ny;
  double den = apply_h(H, x, y, &nx, &ny);
  if (!(fabs(den) >= 1e-12)) return INFINITY;
  return hypot(dsub(nx / den, tx), dsub(ny / den, ty));
}

// geometry.inlier_mask: hypot(fwd, bwd) < eps
HD bool is_inlier(const double* H, const double* Hinv, double px, double py, double qx,
                  double qy, double eps) {
  double f = transfer_dist(H, px, py, qx, qy);
  double b = transfer_dist(Hinv, qx, qy, px, py);
  return hypot(f, b) < eps;
}

// ------------------------------------------------------------------ fits
// geometry._hartley_transform (geometry.py:22-32) on n points, in place;
// t = (s, tx, ty) of T = [[s, 0, tx], [0, s, ty], [0, 0, 1]].
HD bool hartley(double* x, double* y, int n, double* t) {
  double cx = 0.0, cy = 0.0;
  for (int i = 0; i < n; ++i) { cx = dadd(cx, x[i]); cy = dadd(cy, y[i]); }
  cx /= (double)n;
  cy /= (double)n;
  double md = 0.0;
  for (int i = 0; i < n; ++i) {
    x[i] = dsub(x[i], cx);
    y[i] = dsub(y[i], cy);
    md = dadd(md, hypot(x[i], y[i]));
  }
  md /= (double)n;
  if (md < 1e-12) return false;  // "coincident points"
  double s = sqrt(2.0) / md;
  for (int i = 0; i < n; ++i) { x[i] = dmul(x[i], s); y[i] = dmul(y[i], s); }
  t[0] = s;
  t[1] = dmul(-s, cx);
  t[2] = dmul(-s, cy);
  return true;
}

// DLT rows of correspondence (p -> q), geometry.py:51-63.
HD void dlt_rows(double px, double py, double qx, double qy, double* r0, double* r1) {
  r0[0] = -px; r0[1] = -py; r0[2] = -1.0; r0[3] = 0.0; r0[4] = 0.0; r0[5] = 0.0;
  r0[6] = dmul(px, qx); r0[7] = dmul(py, qx); r0[8] = qx;
  r1[0] = 0.0; r1[1] = 0.0; r1[2] = 0.0; r1[3] = -px; r1[4] = -py; r1[5] = -1.0;
  r1[6] = dmul(px, qy); r1[7] = dmul(py, qy); r1[8] = qy;
}

// Singular values of a small square matrix by one-sided Jacobi (columns of
// a, n x n row-major, destroyed); sorted descending into s.
HD void jacobi_singular_values(double* a, int n, double* s) {
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = 0; r < n; ++r) {
          double u = a[r * n + p], v = a[r * n + q];
          al += u * u; be += v * v; ga += u * v;
        }
        if (ga == 0.0) continue;
        double rel = fabs(ga) / sqrt(al * be);
        if (!(rel > 1e-17)) continue;
        off = fmax(off, rel);
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < n; ++r) {
          double u = a[r * n + p], v = a[r * n + q];
          a[r * n + p] = c * u - sn * v;
          a[r * n + q] = sn * u + c * v;
        }
      }
    if (off < 1e-16) break;
  }
  for (int j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int r = 0; r < n; ++r) acc += a[r * n + j] * a[r * n + j];
    s[j] = sqrt(acc);
  }
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && s[j] > s[j - 1]; --j) { double t = s[j]; s[j] = s[j - 1]; s[j - 1] = t; }
}

// Finish a conditioned null vector h (9): H = inv(T_src) h T_ref, then the
// h33 and determinant rules (geometry.py:71-76). Returns 0 or 2 (degenerate).
HD int finish_h(const double* hc, const double* tr, const double* ts, double* H) {
  double Tr[9] = {tr[0], 0.0, tr[1], 0.0, tr[0], tr[2], 0.0, 0.0, 1.0};
  // inverse of [[s,0,a],[0,s,b],[0,0,1]] = [[1/s,0,-a/s],[0,1/s,-b/s],[0,0,1]]
  double is = 1.0 / ts[0];
  double Tsi[9] = {is, 0.0, -ts[1] * is, 0.0, is, -ts[2] * is, 0.0, 0.0, 1.0};
  double tmp[9], h[9];
  matmul3(Tsi, hc, tmp);
  matmul3(tmp, Tr, h);
  if (fabs(h[8]) < 1e-12) return 2;
  double d = h[8];
  for (int i = 0; i < 9; ++i) H[i] = h[i] / d;
  if (fabs(det3(H)) <= 1e-12) return 2;
  return 0;
}

// Four-point DLT (geometry.fit_homography with n = 4).
// The null vector of the 8x9 system is the 9th column of Q in a pivoted
// Householder QR of A^T (9x8); |R66| / |R00| is the rank-revealing estimate
// of the reference's s[-2] / s[0] test (for n = 4, s[-2] is the 7th of 8
// singular values, geometry.py:67). Estimates inside the grey zone
// [1e-13, 1e-6] are settled with exact singular values of R (Jacobi).
// Returns 0 ok, 2 degenerate; *grey counts grey-zone decisions.
HD int fit4(const double* px_in, const double* py_in, const double* qx_in,
            const double* qy_in, double* H, int* grey) {
  double px[4], py[4], qx[4], qy[4], tr[3], ts[3];
  for (int i = 0; i < 4; ++i) { px[i] = px_in[i]; py[i] = py_in[i]; qx[i] = qx_in[i]; qy[i] = qy_in[i]; }
  if (!hartley(px, py, 4, tr)) return 2;
  if (!hartley(qx, qy, 4, ts)) return 2;
  // M = A^T, 9 rows x 8 columns; column c = row c of A
  double M[9][8];
  for (int i = 0; i < 4; ++i) {
    double r0[9], r1[9];
    dlt_rows(px[i], py[i], qx[i], qy[i], r0, r1);
    for (int k = 0; k < 9; ++k) { M[k][2 * i] = r0[k]; M[k][2 * i + 1] = r1[k]; }
  }
  // Fully unrolled so every index is static and M lives in registers; the
  // Householder vector of step k is kept in M[k..8][k], R's diagonal in rdiag.
  double beta[8], rdiag[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double best = -1.0;
    int piv = k;
#pragma unroll
    for (int c = k; c < 8; ++c) {
      double cn = 0.0;
#pragma unroll
      for (int r = k; r < 9; ++r) cn += M[r][c] * M[r][c];
      if (cn > best) { best = cn; piv = c; }
    }
#pragma unroll
    for (int c = k + 1; c < 8; ++c)
      if (c == piv) {
#pragma unroll
        for (int r = 0; r < 9; ++r) { double t = M[r][k]; M[r][k] = M[r][c]; M[r][c] = t; }
      }
    double nrm = sqrt(best);
    double alpha = (M[k][k] > 0.0) ? -nrm : nrm;
    M[k][k] -= alpha;
    double vv = 0.0;
#pragma unroll
    for (int r = k; r < 9; ++r) vv += M[r][k] * M[r][k];
    beta[k] = (vv > 0.0) ? 2.0 / vv : 0.0;
    rdiag[k] = alpha;
#pragma unroll
    for (int c = k + 1; c < 8; ++c) {
      double d = 0.0;
#pragma unroll
      for (int r = k; r < 9; ++r) d += M[r][k] * M[r][c];
      d *= beta[k];
#pragma unroll
      for (int r = k; r < 9; ++r) M[r][c] -= d * M[r][k];
    }
  }
  double ratio = fabs(rdiag[6]) / fabs(rdiag[0]);
  bool degenerate = !(ratio > 1e-9);
  if (ratio > 1e-13 && ratio < 1e-6) {
    // grey zone: exact singular values of R (8x8 upper) decide
    double R[64], s[8];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) R[i * 8 + j] = (j > i) ? M[i][j] : (j == i ? rdiag[i] : 0.0);
    jacobi_singular_values(R, 8, s);
    degenerate = s[6] <= 1e-9 * s[0];
    if (grey) ++*grey;
  }
  if (degenerate) return 2;
  // null vector = Q e_9 = H0 H1 ... H7 e_9
  double y[9] = {0, 0, 0, 0, 0, 0, 0, 0, 1.0};
#pragma unroll
  for (int k = 7; k >= 0; --k) {
    double d = 0.0;
#pragma unroll
    for (int r = k; r < 9; ++r) d += M[r][k] * y[r];
    d *= beta[k];
#pragma unroll
    for (int r = k; r < 9; ++r) y[r] -= d * M[r][k];
  }
  return finish_h(y, tr, ts, H);
}

// Cyclic Jacobi eigen-decomposition of a symmetric 9x9 (row-major, destroyed);
// eigenvalues into w, eigenvectors as columns of v.
HD void jacobi_eig9(double* a, double* w, double* v) {
  for (int i = 0; i < 81; ++i) v[i] = (i % 10 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 50; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < 9; ++p) {
      diag += a[p * 9 + p] * a[p * 9 + p];
      for (int q = p + 1; q < 9; ++q) off += a[p * 9 + q] * a[p * 9 + q];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 9; ++q) {
        double apq = a[p * 9 + q];
        if (apq == 0.0) continue;
        double app = a[p * 9 + p], aqq = a[q * 9 + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 9; ++k) {  // columns p, q
          double akp = a[k * 9 + p], akq = a[k * 9 + q];
          a[k * 9 + p] = c * akp - s * akq;
          a[k * 9 + q] = s * akp + c * akq;
        }
        for (int k = 0; k < 9; ++k) {  // rows p, q
          double apk = a[p * 9 + k], aqk = a[q * 9 + k];
          a[p * 9 + k] = c * apk - s * aqk;
          a[q * 9 + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 9; ++k) {
          double vkp = v[k * 9 + p], vkq = v[k * 9 + q];
          v[k * 9 + p] = c * vkp - s * vkq;
          v[k * 9 + q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 9; ++i) w[i] = a[i * 9 + i];
}

// Least-squares DLT for n >= 5 from the Gram matrix G = A^T A (upper
// triangle packed row-major, 45 entries) in conditioned coordinates.
// The rank rule s[-2] <= 1e-9 s[0] is applied on sqrt(eigenvalues); below
// ~1e-8 the Gram form cannot resolve it (documented in DESIGN.md).
//
// The smallest eigenvector comes from inverse iteration on G + sigma*I
// (sigma = 1e-13 max diag keeps exact fits, lambda_min = 0, well posed)
// through a diagonally pivoted Cholesky factor; the pivots double as the
// rank estimate (d7 ~ lambda7 within a small factor).
HD int fit_from_gram(const double* g45, const double* tr, const double* ts, double* H,
                     int* grey) {
  // The matrix lives as its packed lower triangle A[i (i + 1) / 2 + j], j <= i,
  // with every loop unrolled so each index is a constant: a 9x9 array with
  // the pivot swaps as selects was put in local memory by the compiler, and
  // the factorisation and the iterations ran from there (~25-60k cycles per
  // fit; the arithmetic below is the same, operation for operation).
  double A[45];
#define HDR_A(i, j) A[(i) * ((i) + 1) / 2 + (j)]
  {
    int k = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) { HDR_A(j, i) = g45[k]; ++k; }
  }
  double dmax = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) dmax = fmax(dmax, HDR_A(i, i));
#ifdef HDR_DEBUG_FIT
  printf("gram in: g0=%g g1=%g g44=%g dmax=%g\n", g45[0], g45[1], g45[44], dmax);
#endif
  if (!(dmax > 0.0)) return 2;
  double sigma = 1e-13 * dmax;
#pragma unroll
  for (int i = 0; i < 9; ++i) HDR_A(i, i) += sigma;
  int perm[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) perm[i] = i;
  double piv[9], il[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) {
    int p = c;
    double best = HDR_A(c, c);
#pragma unroll
    for (int i = c + 1; i < 9; ++i)
      if (HDR_A(i, i) > best) { best = HDR_A(i, i); p = i; }
    // symmetric swap of c and p: rows of the finished columns j < c (the
    // factor) and the trailing symmetric block; (p, c) stays. Selects over
    // the candidates: a branch per candidate measured ~20% slower (one thread
    // walks this code, and the branchy form is longer)
#pragma unroll
    for (int q = c + 1; q < 9; ++q) {
      const bool sw = q == p;
      auto swp = [sw](double& x, double& y) {
        double t0 = x, t1 = y;
        x = sw ? t1 : t0;
        y = sw ? t0 : t1;
      };
#pragma unroll
      for (int j = 0; j < c; ++j) swp(HDR_A(c, j), HDR_A(q, j));
      swp(HDR_A(c, c), HDR_A(q, q));
#pragma unroll
      for (int k = c + 1; k < q; ++k) swp(HDR_A(k, c), HDR_A(q, k));
#pragma unroll
      for (int k = q + 1; k < 9; ++k) swp(HDR_A(k, c), HDR_A(k, q));
      int t0 = perm[c], t1 = perm[q];
      perm[c] = sw ? t1 : t0;
      perm[q] = sw ? t0 : t1;
    }
    double d = HDR_A(c, c);
    piv[c] = d;
    if (!(d > 0.0)) return 2;
    double l = sqrt(d);
    HDR_A(c, c) = l;
    il[c] = 1.0 / l;
#pragma unroll
    for (int i = c + 1; i < 9; ++i) HDR_A(i, c) *= il[c];
#pragma unroll
    for (int i = c + 1; i < 9; ++i)
#pragma unroll
      for (int j = c + 1; j <= i; ++j) HDR_A(i, j) -= HDR_A(i, c) * HDR_A(j, c);
  }
  // rank rule s[-2] <= 1e-9 s[0]: resolvable in Gram precision only down to
  // ~1e-7 relative singular values; d7 - sigma estimates s7^2
  double s7sq = fmax(piv[7] - sigma, 0.0), s0sq = piv[0] - sigma;
  if (grey && s7sq > 1e-13 * s0sq && s7sq < 1e-10 * s0sq) ++*grey;
  if (s7sq <= 1e-13 * s0sq) return 2;
  double v[9], y[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) v[i] = 1.0 / 3.0;
  // (G + sigma I) has condition ~1e13, so successive iterates jitter at
  // ~1e-15..1e-14 once converged: stop at 1e-13 (H to ~1e-13 relative)
  for (int it = 0; it < 30; ++it) {
#pragma unroll
    for (int i = 0; i < 9; ++i) {  // L y = v
      double s = v[i];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= HDR_A(i, j) * y[j];
      y[i] = s * il[i];
    }
#pragma unroll
    for (int i = 8; i >= 0; --i) {  // L^T z = y (z into y)
      double s = y[i];
#pragma unroll
      for (int j = i + 1; j < 9; ++j) s -= HDR_A(j, i) * y[j];
      y[i] = s * il[i];
    }
    double nrm = 0.0, sgn = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) { nrm += y[i] * y[i]; sgn += y[i] * v[i]; }
    nrm = 1.0 / sqrt(nrm);
    if (sgn < 0) nrm = -nrm;
    double diff = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      double z = y[i] * nrm;
      diff = fmax(diff, fabs(z - v[i]));
      v[i] = z;
    }
    if (diff < 1e-13) break;
  }

  double hc[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) hc[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = 0; j < 9; ++j)
      if (perm[i] == j) hc[j] = v[i];
#undef HDR_A
  return finish_h(hc, tr, ts, H);
}

}  // namespace hdr
