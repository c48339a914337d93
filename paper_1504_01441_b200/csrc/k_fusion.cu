// Merge inputs: SSIM registration-trust map (K13) and the per-stage quality /
// fusion-weight kernels (K14); the pyramid blend itself is in k_merge.cu.
//
// Storage is f32 (images, weights, pyramid levels); SSIM moments and the
// weight products are evaluated in f64 like the reference
// (fusion.py:34-77); the 5-tap pyramid arithmetic is f32. Tolerances:
// SURVEY.md §8(a) a19-a22 (SSIM <= 1e-4, composite <= 1e-3).
#include "hdr_common.cuh"
#include "hdr_internal.h"

namespace hdr {

// ---------------------------------------------------------------- K13
constexpr int kSsimTW = 32, kSsimTH = 16, kMaxRad = 15;

__device__ __forceinline__ float lumf(float r, float g, float b) {
  float y = fadd(fadd(fmul(0.299f, r), fmul(0.587f, g)), fmul(0.114f, b));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

// fusion.ssim_map (fusion.py:34-64): separable reflect blurs along axis 0
// then axis 1 of a, b, a^2, b^2, ab; scipy's symmetric-kernel accumulation
// order x0*w0 + sum_{j=r..1} (x[-j] + x[+j]) * w[j].
// b = lut_b[qb] when qb != nullptr (the warped frame's equalised luminance).
__global__ void __launch_bounds__(kSsimTW * 8) ssim_kernel(
    const float* __restrict__ a, const float* __restrict__ b, const uint8_t* __restrict__ qb,
    const float* __restrict__ lut_b, int w, int h, int r, const double* __restrict__ taps,
    float* __restrict__ out) {
  pdl_wait();
  extern __shared__ double sm[];
  const int EW = kSsimTW + 2 * r, EH = kSsimTH + 2 * r;
  float* sa = reinterpret_cast<float*>(sm);  // EH x EW
  float* sb = sa + EH * EW;
  double* V = sm + ((2 * EH * EW + 1) / 2);  // 5 x kSsimTH x EW
  __shared__ double k[2 * kMaxRad + 1];
  __shared__ float lut[kBins];
  int tid = threadIdx.x, nt = blockDim.x;
  if (tid < 2 * r + 1) k[tid] = taps[tid];
  if (qb)
    for (int i = tid; i < kBins; i += nt) lut[i] = lut_b[i];
  __syncthreads();
  int x0 = blockIdx.x * kSsimTW - r, y0 = blockIdx.y * kSsimTH - r;
  for (int i = tid; i < EH * EW; i += nt) {
    int ly = i / EW, lx = i % EW;
    int gy = reflect_index(y0 + ly, h), gx = reflect_index(x0 + lx, w);
    int64_t p = (int64_t)gy * w + gx;
    sa[i] = a[p];
    sb[i] = qb ? lut[qb[p]] : b[p];
  }
  __syncthreads();
  // vertical (axis 0)
  const int SV = kSsimTH * EW;
  for (int i = tid; i < SV; i += nt) {
    int oy = i / EW, lx = i % EW;
    int c = (oy + r) * EW + lx;
    double va = sa[c], vb = sb[c];
    // FMA-contracted (the SSIM bar is 1e-4; scipy's exact order is not needed)
    double m0 = va * k[r], m1 = vb * k[r];
    double m2 = (va * va) * k[r], m3 = (vb * vb) * k[r], m4 = (va * vb) * k[r];
    for (int j = r; j >= 1; --j) {
      double ua = sa[c - j * EW], ub = sb[c - j * EW], da = sa[c + j * EW], db = sb[c + j * EW];
      double kj = k[r + j];
      m0 = fma(ua + da, kj, m0);
      m1 = fma(ub + db, kj, m1);
      m2 = fma(fma(ua, ua, da * da), kj, m2);
      m3 = fma(fma(ub, ub, db * db), kj, m3);
      m4 = fma(fma(ua, ub, da * db), kj, m4);
    }
    V[0 * SV + i] = m0; V[1 * SV + i] = m1; V[2 * SV + i] = m2; V[3 * SV + i] = m3;
    V[4 * SV + i] = m4;
  }
  __syncthreads();
  // horizontal (axis 1) + SSIM formula
  for (int i = tid; i < kSsimTW * kSsimTH; i += nt) {
    int oy = i / kSsimTW, ox = i % kSsimTW;
    int gx = blockIdx.x * kSsimTW + ox, gy = blockIdx.y * kSsimTH + oy;
    if (gx >= w || gy >= h) continue;
    double m[5];
    int c = oy * EW + ox + r;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double* row = V + q * SV;
      double acc = row[c] * k[r];
      for (int j = r; j >= 1; --j) acc = fma(row[c - j] + row[c + j], k[r + j], acc);
      m[q] = acc;
    }
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double mu_a = m[0], mu_b = m[1];
    double var_a = m[2] - mu_a * mu_a, var_b = m[3] - mu_b * mu_b, cov = m[4] - mu_a * mu_b;
    double s = ((2.0 * mu_a * mu_b + C1) * (2.0 * cov + C2)) /
               ((mu_a * mu_a + mu_b * mu_b + C1) * (var_a + var_b + C2));
    s = fmin(fmax(s, -1.0), 1.0);
    out[(int64_t)gy * w + gx] = (float)s;
  }
}

template <int R>
__global__ void ssim_fixed_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                  const uint8_t* __restrict__ qb, const float* __restrict__ lut_b,
                                  int w, int h, const double* __restrict__ taps,
                                  float* __restrict__ out, int ty0);

void init_fusion_attributes() {
  allow_max_dynamic_smem(ssim_fixed_kernel<5>);
  allow_max_dynamic_smem(ssim_kernel);
}

// Specialised for a compile-time radius (the default 11-tap window): 32x32
// outputs per 32x8 block, each thread owning one column and 4 rows, so all
// tap loops unroll and no index needs a division.
constexpr int kS2 = 32;
// rows per vertical work item of ssim_fixed_kernel: E x 32/VR items over 256
// threads (VR = 4: 336 items, two rounds, the second 31% busy; VR = 2: 672
// items, three rounds, 88% busy, ~1.7x the staged-sample products per output)
#ifndef HDR_SSIM_VROWS
#define HDR_SSIM_VROWS 4
#endif
constexpr int VR = HDR_SSIM_VROWS;

// chunk permutation of ssim_fixed_kernel's vertical-pass rows (radius 5:
// 21 chunks of 16 bytes; found by exhaustive search, see the horizontal pass)
__device__ __forceinline__ int ssim_chunk(int k) { return (unsigned)(k - 8) < 8u ? k ^ 1 : k; }
#ifndef HDR_SSIM_SWIZZLE
#define HDR_SSIM_SWIZZLE 1
#endif
#ifndef HDR_SSIM_STAGE_INC
#define HDR_SSIM_STAGE_INC 1
#endif

template <int R>
#ifndef HDR_SSIM_MIN_BLOCKS
#define HDR_SSIM_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(256, HDR_SSIM_MIN_BLOCKS) ssim_fixed_kernel(
    const float* __restrict__ a, const float* __restrict__ b, const uint8_t* __restrict__ qb,
    const float* __restrict__ lut_b, int w, int h, const double* __restrict__ taps,
    float* __restrict__ out, int ty0) {
  pdl_wait();
  constexpr int E = kS2 + 2 * R;  // staged rows/cols incl. halo
  constexpr bool SWZ = HDR_SSIM_SWIZZLE && R == 5;
  const int by = ty0 + (int)blockIdx.y;  // tile row (ty0 > 0: a row band's tiles)
  __shared__ float sa[E][E + 1], sb[E][E + 1];
  __shared__ int rows[E], cols[E];
  __shared__ float lut[kBins];
  extern __shared__ double V[];  // [5][kS2][E]
  int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  int x0 = blockIdx.x * kS2 - R, y0 = by * kS2 - R;
  double k[2 * R + 1];
#pragma unroll
  for (int j = 0; j <= 2 * R; ++j) k[j] = taps[j];
  if (tid < E) { rows[tid] = reflect_index(y0 + tid, h); cols[tid] = reflect_index(x0 + tid, w); }
  if (qb)
    for (int i = tid; i < kBins; i += 256) lut[i] = lut_b[i];
  __syncthreads();
  {
    // all of this thread's global loads are issued before the first store
    // (the staged tile is E*E = 1764 samples: 7 per thread)
    constexpr int NE = (E * E + 255) / 256;
    float va[NE];
    uint32_t vq[NE];
#if HDR_SSIM_STAGE_INC
    // (r, cc) of i = tid + 256 it advance without a division (256 = DR E + DC)
    constexpr int DR = 256 / E, DC = 256 - DR * E;
    const int r00 = tid / E, c00 = tid - r00 * E;
    {
      int r = r00, cc = c00;
#pragma unroll
      for (int it = 0; it < NE; ++it) {
        bool ok = tid + it * 256 < E * E;
        int64_t p = ok ? (int64_t)rows[r] * w + cols[cc] : 0;
        va[it] = ok ? __ldg(a + p) : 0.0f;
        vq[it] = qb ? (ok ? (uint32_t)__ldg(qb + p) : 0u) : __float_as_uint(ok ? __ldg(b + p) : 0.0f);
        r += DR; cc += DC;
        if (cc >= E) { cc -= E; ++r; }
        r = min(r, E - 1);
      }
    }
    {
      int r = r00, cc = c00;
#pragma unroll
      for (int it = 0; it < NE; ++it) {
        if (tid + it * 256 >= E * E) break;
        sa[r][cc] = va[it];
        sb[r][cc] = qb ? lut[vq[it]] : __uint_as_float(vq[it]);
        r += DR; cc += DC;
        if (cc >= E) { cc -= E; ++r; }
      }
    }
#else
#pragma unroll
    for (int it = 0; it < NE; ++it) {
      int i = tid + it * 256;
      int r = i / E, cc = i - r * E;
      bool ok = i < E * E;
      int64_t p = ok ? (int64_t)rows[r] * w + cols[cc] : 0;
      va[it] = ok ? __ldg(a + p) : 0.0f;
      vq[it] = qb ? (ok ? (uint32_t)__ldg(qb + p) : 0u) : __float_as_uint(ok ? __ldg(b + p) : 0.0f);
    }
#pragma unroll
    for (int it = 0; it < NE; ++it) {
      int i = tid + it * 256;
      if (i >= E * E) break;
      int r = i / E, cc = i - r * E;
      sa[r][cc] = va[it];
      sb[r][cc] = qb ? lut[vq[it]] : __uint_as_float(vq[it]);
    }
#endif
  }
  __syncthreads();
  // vertical (axis 0): work item (rg, c) produces rows VR rg .. VR rg + VR-1 of staged
  // column c from 14 staged samples (sliding); the E x 8 items are dealt out
  // flat over the 256 threads, so the second round runs 3 warps, not 8
  for (int item = tid; item < E * (kS2 / VR); item += 256) {
    const int rg = item / E, c = item - rg * E;
    // the products of each staged sample are formed once (not once per tap
    // that reads it): same roundings, ~25% fewer f64 instructions
    double va[VR + 2 * R], vb[VR + 2 * R], vaa[VR + 2 * R], vbb[VR + 2 * R], vab[VR + 2 * R];
#pragma unroll
    for (int j = 0; j < VR + 2 * R; ++j) {
      va[j] = sa[VR * rg + j][c];
      vb[j] = sb[VR * rg + j][c];
      vaa[j] = va[j] * va[j];
      vbb[j] = vb[j] * vb[j];
      vab[j] = va[j] * vb[j];
    }
#pragma unroll
    for (int q = 0; q < VR; ++q) {
      double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
      for (int j = 0; j <= 2 * R; ++j) {
        m0 = fma(va[q + j], k[j], m0);
        m1 = fma(vb[q + j], k[j], m1);
        m2 = fma(vaa[q + j], k[j], m2);
        m3 = fma(vbb[q + j], k[j], m3);
        m4 = fma(vab[q + j], k[j], m4);
      }
      int oy = VR * rg + q;
      const int cs = SWZ ? (ssim_chunk(c >> 1) << 1) | (c & 1) : c;
      V[(0 * kS2 + oy) * E + cs] = m0;
      V[(1 * kS2 + oy) * E + cs] = m1;
      V[(2 * kS2 + oy) * E + cs] = m2;
      V[(3 * kS2 + oy) * E + cs] = m3;
      V[(4 * kS2 + oy) * E + cs] = m4;
    }
  }
  __syncthreads();
  // horizontal (axis 1): thread owns 4 consecutive outputs of one row
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  int oy = tid >> 3, ox0 = (tid & 7) * 4;
  int gy = by * kS2 + oy;
  double m[5][4];
  // the 8 lanes of a row read 16-byte chunks 32 bytes apart (two lanes per
  // bank group: lanes l and l + 4 are 128 bytes apart). SWZ: the vertical
  // pass stored chunk k of every row at ssim_chunk(k) (chunks 8..15 swapped in
  // pairs), a permutation under which the 8 lanes' chunks of every step fall
  // in 8 distinct bank groups -- one wavefront per row without the lane-
  // dependent rotation (and its 2 x 7 x 5 double selects) used otherwise.
  constexpr int NC = (4 + 2 * R) / 2;  // 16-byte chunks per thread (7)
  static_assert((4 + 2 * R) % 2 == 0 && E % 2 == 0, "16-byte chunks");
  const int rot = SWZ ? 0 : (tid >> 2) & 1;
  int pst[NC];
#pragma unroll
  for (int st = 0; st < NC; ++st) pst[st] = SWZ ? ssim_chunk((ox0 >> 1) + st) : (ox0 >> 1) + st;
#pragma unroll
  for (int mm = 0; mm < 5; ++mm) {
    const double2* row2 = reinterpret_cast<const double2*>(V + (mm * kS2 + oy) * E);
    double2 r[NC];
    if (SWZ) {
#pragma unroll
      for (int st = 0; st < NC; ++st) r[st] = row2[pst[st]];
    } else {
#pragma unroll
      for (int st = 0; st < NC; ++st) r[st] = row2[(ox0 >> 1) + (st + rot == NC ? 0 : st + rot)];
    }
    double v[4 + 2 * R];
#pragma unroll
    for (int t = 0; t < NC; ++t) {
      double2 cv = rot ? r[(t + NC - 1) % NC] : r[t];
      v[2 * t] = cv.x;
      v[2 * t + 1] = cv.y;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j <= 2 * R; ++j) acc = fma(v[q + j], k[j], acc);
      m[mm][q] = acc;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int gx = blockIdx.x * kS2 + ox0 + q;
    if (gx >= w || gy >= h) continue;
    double mu_a = m[0][q], mu_b = m[1][q];
    double var_a = m[2][q] - mu_a * mu_a, var_b = m[3][q] - mu_b * mu_b;
    double cov = m[4][q] - mu_a * mu_b;
    double sc = ((2.0 * mu_a * mu_b + C1) * (2.0 * cov + C2)) /
                ((mu_a * mu_a + mu_b * mu_b + C1) * (var_a + var_b + C2));
    out[(int64_t)gy * w + gx] = (float)fmin(fmax(sc, -1.0), 1.0);
  }
}

// rows [y0, y1) of the SSIM map (y0 a multiple of 32; radius 5 only): a row
// band's tiles
bool launch_ssim_rows(const float* a, const uint8_t* qb, const float* lut_b, int w, int h, int y0, int y1,
                      int window, const double* taps, float* out, cudaStream_t s) {
  if (y1 <= y0) return true;  // an empty band (the last ranks of a short frame)
  if (window / 2 != 5 || y0 % kS2) return false;
  size_t vb = 5 * (size_t)kS2 * (kS2 + 10) * sizeof(double);
  dim3 grd(ceil_div(w, kS2), ceil_div(y1, kS2) - y0 / kS2);
  klaunch(ssim_fixed_kernel<5>, grd, dim3(32, 8), vb, s, a, (const float*)nullptr, qb, lut_b, w, h, taps, out,
          y0 / kS2);
  return true;
}

void launch_ssim(const float* a, const float* b_or_null, const uint8_t* qb, const float* lut_b,
                 int w, int h, int window, const double* taps, float* out, cudaStream_t s) {
  int r = window / 2;
  if (r == 5) {
    size_t vb = 5 * (size_t)kS2 * (kS2 + 10) * sizeof(double);
    dim3 grd(ceil_div(w, kS2), ceil_div(h, kS2));
    klaunch(ssim_fixed_kernel<5>, grd, dim3(32, 8), vb, s, a, b_or_null, qb, lut_b, w, h, taps, out, 0);
    return;
  }
  int EW = kSsimTW + 2 * r, EH = kSsimTH + 2 * r;
  size_t bytes = ((2 * EH * EW + 1) / 2) * sizeof(double) + 5 * (size_t)kSsimTH * EW * sizeof(double);
  dim3 grd(ceil_div(w, kSsimTW), ceil_div(h, kSsimTH));
  klaunch(ssim_kernel, grd, kSsimTW * 8, bytes, s, a, b_or_null, qb, lut_b, w, h, r, taps, out);
}

// ---------------------------------------------------------------- K14
// fusion.quality_weights (fusion.py:67-77) at one pixel, f64.
__device__ __forceinline__ double quality(const float* __restrict__ rgb, int w, int h, int x,
                                          int y) {
  auto L = [&](int yy, int xx) -> double {
    const float* p = rgb + ((int64_t)reflect_index(yy, h) * w + reflect_index(xx, w)) * 3;
    return (double)lumf(p[0], p[1], p[2]);
  };
  double c0 = L(y, x);
  // ndimage.laplace: correlate1d([1,-2,1]) along axis 0, += along axis 1
  double lap0 = dadd(dmul(c0, -2.0), dadd(L(y - 1, x), L(y + 1, x)));
  double lap1 = dadd(dmul(c0, -2.0), dadd(L(y, x - 1), L(y, x + 1)));
  double con = fabs(dadd(lap0, lap1));
  const float* p = rgb + ((int64_t)y * w + x) * 3;
  double r = p[0], g = p[1], b = p[2];
  double mean = dadd(dadd(r, g), b) / 3.0;
  double dr = r - mean, dg = g - mean, db = b - mean;
  double var = dadd(dadd(dmul(dr, dr), dmul(dg, dg)), dmul(db, db)) / 3.0;
  double sat = sqrt(var);
  double er = r - 0.5, eg = g - 0.5, eb = b - 0.5;
  double ssum = dadd(dadd(dmul(er, er), dmul(eg, eg)), dmul(eb, eb));
  double ex = exp(-ssum / (2.0 * 0.2 * 0.2));
  return dadd(dmul(dmul(con, sat), ex), 1e-12);
}

__global__ void quality_kernel(const float* __restrict__ rgb, int w, int h, float* __restrict__ out) {
  pdl_wait();
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  out[(int64_t)y * w + x] = (float)quality(rgb, w, h, x, y);
}

void launch_quality(const float* rgb, int w, int h, float* out, cudaStream_t s) {
  dim3 blk(32, 8), grd(ceil_div(w, 32), ceil_div(h, 8));
  klaunch(quality_kernel, grd, blk, 0, s, rgb, w, h, out);
}

// fusion.fusion_weights (fusion.py:117-128)
__global__ void fusion_weights_kernel(const float* __restrict__ ref, const float* __restrict__ warped,
                                      const float* __restrict__ ssim,
                                      const uint8_t* __restrict__ valid, int w, int h,
                                      float* __restrict__ wr, float* __restrict__ ws) {
  pdl_wait();
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  int64_t i = (int64_t)y * w + x;
  double qr = quality(ref, w, h, x, y);
  double qs = quality(warped, w, h, x, y);
  double sv = fmin(fmax((double)ssim[i], 0.0), 1.0);
  double vs = dmul(dmul(qs, sv), valid[i] ? 1.0 : 0.0);
  double tot = dadd(qr, vs);
  wr[i] = (float)(qr / tot);
  ws[i] = (float)(vs / tot);
}

void launch_fusion_weights(const float* ref, const float* warped, const float* ssim,
                           const uint8_t* valid, int w, int h, float* wr, float* ws,
                           cudaStream_t s) {
  dim3 blk(32, 8), grd(ceil_div(w, 32), ceil_div(h, 8));
  klaunch(fusion_weights_kernel, grd, blk, 0, s, ref, warped, ssim, valid, w, h, wr, ws);
}

}  // namespace hdr

namespace hdr {

// ---------------------------------------------------------------- pyramid twins
// fusion._blur5 / _pyr_down / _pyr_up (fusion.py:80-93) in f64 on (h, w, c)
// interleaved arrays, for the stage-level gaussian_pyramid /
// laplacian_pyramid / collapse_pyramid APIs (the pair path fuses these into
// k_merge.cu's kernels). scipy's symmetric correlate1d accumulates
// x0*w0, then (x-2 + x+2)*w2, then (x-1 + x+1)*w1, each op rounded
// separately; that order is kept so the results match bit for bit.
__device__ __forceinline__ double sym5(double xm2, double xm1, double x0, double xp1, double xp2,
                                       double w0, double w1, double w2) {
  double t = dmul(x0, w0);
  t = dadd(t, dmul(dadd(xm2, xp2), w2));
  return dadd(t, dmul(dadd(xm1, xp1), w1));
}

// out (oh, ow, c) = blur5(in)[::2, ::2]
__global__ void pyr_down_kernel(const double* __restrict__ in, int w, int h, int c,
                                double* __restrict__ out, int ow, int oh) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)ow * oh * c) return;
  int k = (int)(i % c);
  int64_t p = i / c;
  int x = (int)(p % ow), y = (int)(p / ow);
  double v[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {  // axis 0 at row 2y for the 5 columns axis 1 reads
    int xx = reflect_index(2 * x - 2 + j, w);
    double r[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) r[q] = in[((int64_t)reflect_index(2 * y - 2 + q, h) * w + xx) * c + k];
    v[j] = sym5(r[0], r[1], r[2], r[3], r[4], 6.0 / 16, 4.0 / 16, 1.0 / 16);
  }
  out[i] = sym5(v[0], v[1], v[2], v[3], v[4], 6.0 / 16, 4.0 / 16, 1.0 / 16);
}

// out (h, w, c) = 2x-gain blur5 of in (ch, cw, c) zero-inserted on the fine
// grid; with `base`: out = base - up (laplacian_pyramid) for sign < 0, or
// base + up (collapse_pyramid) for sign > 0, one rounding like numpy's
__global__ void pyr_up_kernel(const double* __restrict__ in, int cw, int ch, int c,
                              double* __restrict__ out, int w, int h,
                              const double* __restrict__ base, int sign) {
  pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)w * h * c) return;
  int k = (int)(i % c);
  int64_t p = i / c;
  int x = (int)(p % w), y = (int)(p / w);
  auto up = [&](int yy, int xx) -> double {  // zero-inserted fine sample
    return ((yy | xx) & 1) ? 0.0 : in[((int64_t)(yy >> 1) * cw + (xx >> 1)) * c + k];
  };
  double v[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    int xx = reflect_index(x - 2 + j, w);
    double r[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) r[q] = up(reflect_index(y - 2 + q, h), xx);
    v[j] = sym5(r[0], r[1], r[2], r[3], r[4], 12.0 / 16, 8.0 / 16, 2.0 / 16);
  }
  double u = sym5(v[0], v[1], v[2], v[3], v[4], 12.0 / 16, 8.0 / 16, 2.0 / 16);
  out[i] = !base ? u : (sign < 0 ? dsub(base[i], u) : dadd(base[i], u));
}

void launch_pyr_down(const double* in, int w, int h, int c, double* out, cudaStream_t s) {
  int ow = (w + 1) / 2, oh = (h + 1) / 2;
  int64_t n = (int64_t)ow * oh * c;
  if (n > 0) klaunch(pyr_down_kernel, (unsigned)((n + 255) / 256), 256, 0, s, in, w, h, c, out, ow, oh);
}

void launch_pyr_up(const double* in, int cw, int ch, int c, double* out, int w, int h,
                   const double* base, int sign, cudaStream_t s) {
  int64_t n = (int64_t)w * h * c;
  if (n > 0)
    klaunch(pyr_up_kernel, (unsigned)((n + 255) / 256), 256, 0, s, in, cw, ch, c, out, w, h, base, sign);
}

}  // namespace hdr
