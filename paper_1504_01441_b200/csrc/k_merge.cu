// Laplacian-pyramid exposure fusion (K14 + K15), fusion.py:96-157, as four
// tiled kernels:
//   weights_down0  quality weights of both frames (fusion.py:67-77), the
//                  SSIM/validity trust and normalisation (fusion.py:117-128)
//                  for a 36x36 level-0 tile, written for the owned 32x32 and
//                  immediately blurred + decimated into level 1 of the
//                  8-channel Gaussian pyramid (ref RGB, warped RGB, W_ref,
//                  W_src) -- the weights never make a separate HBM round trip
//                  before the first reduction;
//   down           the same 5-tap reflect blur + [::2, ::2] for levels >= 1;
//   collapse       C_k = W_ref (G_ref - up G_ref') + W_src (G_src - up G_src')
//                  + up C'  (the blend of laplacian_pyramid terms and
//                  collapse_pyramid folded together); level 0 reads the
//                  interleaved inputs and writes the clipped composite.
// up() is _pyr_up (fusion.py:89-93): zero-insert on the fine grid, 2x-gain
// 5-tap blur, scipy 'reflect' on the fine grid -- evaluated separably from a
// shared-memory staging of the horizontally up-sampled rows.
// Arithmetic is f32 (the composite tolerance is 1e-3).
#include "hdr_common.cuh"
#include "hdr_internal.h"

namespace hdr {

__constant__ float kK5[5] = {1.0f / 16, 4.0f / 16, 6.0f / 16, 4.0f / 16, 1.0f / 16};
__constant__ float kK5x2[5] = {2.0f / 16, 8.0f / 16, 12.0f / 16, 8.0f / 16, 2.0f / 16};

__device__ __forceinline__ float lum_f(float r, float g, float b) {
  float y = fadd(fadd(fmul(0.299f, r), fmul(0.587f, g)), fmul(0.114f, b));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

// contrast x saturation x well-exposedness + 1e-12 (fusion.py:67-77).
// The laplacian and the channel std stay f64 as in the reference: for grey or
// clipped pixels the true std is exactly 0 there (3v * (1/3) rounds back to v),
// while an f32 mean leaves ~1e-8 of std, which outweighs the 1e-12 floor and
// changes the blend weights completely. Only the exposedness exp is f32.
__device__ __forceinline__ double quality_d(double lap, float r, float g, float b) {
  const double third = 1.0 / 3.0;
  double R = r, G = g, B = b;
  double mean = ((R + G) + B) * third;
  double dr = R - mean, dg = G - mean, db = B - mean;
  double sat = sqrt(((dr * dr + dg * dg) + db * db) * third);
  float er = r - 0.5f, eg = g - 0.5f, eb = b - 0.5f;
  double ex = (double)__expf(-(er * er + eg * eg + eb * eb) * 12.5f);
  return fabs(lap) * sat * ex + 1e-12;
}

// ---------------------------------------------------------------- weights + level 1
constexpr int kOT = 16;           // level-1 outputs per tile side
constexpr int kRT = 2 * kOT + 4;  // level-0 region incl. the 2-px blur halo (36)
constexpr int kLT = kRT + 2;      // + 1-px laplacian halo (38)

__global__ void __launch_bounds__(256) weights_down0_kernel(
    const float* __restrict__ ref, const float* __restrict__ warped, const float* __restrict__ ssim,
    const uint8_t* __restrict__ valid, int w, int h, float* __restrict__ wr_out,
    float* __restrict__ ws_out, float* __restrict__ g1, int ow, int oh) {
  extern __shared__ float smf[];
  float (*lr)[kLT] = reinterpret_cast<float (*)[kLT]>(smf);
  float (*lw)[kLT] = reinterpret_cast<float (*)[kLT]>(smf + kLT * kLT);
  // ref rgb, warped rgb, w_ref, w_src
  float (*px)[kRT][kRT + 1] = reinterpret_cast<float (*)[kRT][kRT + 1]>(smf + 2 * kLT * kLT);
  float (*V)[kOT][kRT] = reinterpret_cast<float (*)[kOT][kRT]>(smf + 2 * kLT * kLT + 8 * kRT * (kRT + 1));
  __shared__ int ridx[kLT], cidx[kLT];
  int tid = threadIdx.x, nt = blockDim.x;
  int Y0 = blockIdx.y * kOT, X0 = blockIdx.x * kOT;
  int vy0 = 2 * Y0 - 3, vx0 = 2 * X0 - 3;  // virtual origin of the 38x38 lum tile
  if (tid < kLT) {
    ridx[tid] = reflect_index(vy0 + tid, h);
    cidx[tid] = reflect_index(vx0 + tid, w);
  }
  __syncthreads();
  for (int i = tid; i < kLT * kLT; i += nt) {
    int ly = i / kLT, lx = i - ly * kLT;
    int64_t p = ((int64_t)ridx[ly] * w + cidx[lx]) * 3;
    float r0 = ref[p], r1 = ref[p + 1], r2 = ref[p + 2];
    float w0 = warped[p], w1 = warped[p + 1], w2 = warped[p + 2];
    lr[ly][lx] = lum_f(r0, r1, r2);
    lw[ly][lx] = lum_f(w0, w1, w2);
    if (ly >= 1 && ly <= kRT && lx >= 1 && lx <= kRT) {
      int ty = ly - 1, tx = lx - 1;
      px[0][ty][tx] = r0; px[1][ty][tx] = r1; px[2][ty][tx] = r2;
      px[3][ty][tx] = w0; px[4][ty][tx] = w1; px[5][ty][tx] = w2;
    }
  }
  __syncthreads();
  for (int i = tid; i < kRT * kRT; i += nt) {
    int ty = i / kRT, tx = i - ty * kRT;
    int ly = ty + 1, lx = tx + 1;
    // ndimage.laplace: [1,-2,1] along axis 0, += along axis 1 (exact in f64)
    double cr = lr[ly][lx], cw = lw[ly][lx];
    double lapr = ((double)lr[ly - 1][lx] + lr[ly + 1][lx] - 2.0 * cr) +
                  ((double)lr[ly][lx - 1] + lr[ly][lx + 1] - 2.0 * cr);
    double lapw = ((double)lw[ly - 1][lx] + lw[ly + 1][lx] - 2.0 * cw) +
                  ((double)lw[ly][lx - 1] + lw[ly][lx + 1] - 2.0 * cw);
    double qr = quality_d(lapr, px[0][ty][tx], px[1][ty][tx], px[2][ty][tx]);
    double qs = quality_d(lapw, px[3][ty][tx], px[4][ty][tx], px[5][ty][tx]);
    int64_t p = (int64_t)ridx[ly] * w + cidx[lx];
    double sv = fmin(fmax((double)ssim[p], 0.0), 1.0);
    qs = valid[p] ? qs * sv : 0.0;
    double inv = 1.0 / (qr + qs);
    float a = (float)(qr * inv), b = (float)(qs * inv);
    px[6][ty][tx] = a;
    px[7][ty][tx] = b;
    // owned level-0 pixels: rows/cols [2Y0, 2Y0 + 32) of the real image
    int ry = vy0 + ly, rx = vx0 + lx;
    if (ty >= 2 && ty < 2 + 2 * kOT && tx >= 2 && tx < 2 + 2 * kOT && ry < h && rx < w) {
      wr_out[p] = a;
      ws_out[p] = b;
    }
  }
  __syncthreads();
  // vertical 5-tap + decimation: V[c][oy][tx] (region row 2*oy + i)
  for (int i = tid; i < 8 * kOT * kRT; i += nt) {
    int c = i / (kOT * kRT), r = i - c * (kOT * kRT);
    int oy = r / kRT, tx = r - oy * kRT;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < 5; ++k) acc += kK5[k] * px[c][2 * oy + k][tx];
    V[c][oy][tx] = acc;
  }
  __syncthreads();
  int64_t OP = (int64_t)ow * oh;
  for (int i = tid; i < 8 * kOT * kOT; i += nt) {
    int c = i >> 8, r = i & 255;  // kOT * kOT = 256
    int oy = r >> 4, ox = r & 15;
    int Y = Y0 + oy, X = X0 + ox;
    if (Y >= oh || X >= ow) continue;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < 5; ++k) acc += kK5[k] * V[c][oy][2 * ox + k];
    g1[c * OP + (int64_t)Y * ow + X] = acc;
  }
}

// ---------------------------------------------------------------- levels >= 1
// all 8 channels staged at once: 2 barriers per tile instead of 3 per channel
constexpr size_t kDownSmem = sizeof(float) * (8 * kRT * (kRT + 1) + 8 * kOT * kRT);

__global__ void __launch_bounds__(256) down_kernel(const float* __restrict__ in, int w, int h,
                                                   float* __restrict__ out, int ow, int oh) {
  extern __shared__ float smd[];
  float (*tile)[kRT][kRT + 1] = reinterpret_cast<float (*)[kRT][kRT + 1]>(smd);
  float (*V)[kOT][kRT] = reinterpret_cast<float (*)[kOT][kRT]>(smd + 8 * kRT * (kRT + 1));
  __shared__ int ridx[kRT], cidx[kRT];
  int tid = threadIdx.x, nt = blockDim.x;
  int Y0 = blockIdx.y * kOT, X0 = blockIdx.x * kOT;
  int vy0 = 2 * Y0 - 2, vx0 = 2 * X0 - 2;
  if (tid < kRT) {
    ridx[tid] = reflect_index(vy0 + tid, h);
    cidx[tid] = reflect_index(vx0 + tid, w);
  }
  __syncthreads();
  int64_t P = (int64_t)w * h, OP = (int64_t)ow * oh;
  for (int i = tid; i < 8 * kRT * kRT; i += nt) {
    int c = i / (kRT * kRT), r = i - c * (kRT * kRT);
    int ty = r / kRT, tx = r - ty * kRT;
    tile[c][ty][tx] = in[c * P + (int64_t)ridx[ty] * w + cidx[tx]];
  }
  __syncthreads();
  for (int i = tid; i < 8 * kOT * kRT; i += nt) {
    int c = i / (kOT * kRT), r = i - c * (kOT * kRT);
    int oy = r / kRT, tx = r - oy * kRT;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < 5; ++k) acc += kK5[k] * tile[c][2 * oy + k][tx];
    V[c][oy][tx] = acc;
  }
  __syncthreads();
  for (int i = tid; i < 8 * kOT * kOT; i += nt) {
    int c = i >> 8, r = i & 255;
    int oy = r >> 4, ox = r & 15;
    int Y = Y0 + oy, X = X0 + ox;
    if (Y >= oh || X >= ow) continue;
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < 5; ++k) acc += kK5[k] * V[c][oy][2 * ox + k];
    out[c * OP + (int64_t)Y * ow + X] = acc;
  }
}

// ---------------------------------------------------------------- collapse
constexpr int kFT = 32;           // fine outputs per tile side
constexpr int kFV = kFT + 4;      // virtual fine rows/cols incl. the 2-px halo
constexpr int kCT = kFT / 2 + 3;  // coarse rows/cols the tile can touch (19)
constexpr size_t kCollapseSmem = sizeof(float) * (9 * kCT * kCT + 9 * kFV * (kFT + 1));

// 9 coarse channels: G_ref 0-2, G_src 3-5 (gc, planar 8-ch level), C 6-8 (cc)
template <bool LEVEL0>
__global__ void __launch_bounds__(256) collapse_kernel(
    const float* __restrict__ g, const float* __restrict__ ref, const float* __restrict__ warped,
    const float* __restrict__ wr, const float* __restrict__ ws, int w, int h,
    const float* __restrict__ gc, const float* __restrict__ cc, int cw, int ch,
    float* __restrict__ out) {
  extern __shared__ float smc[];
  float (*C)[kCT][kCT] = reinterpret_cast<float (*)[kCT][kCT]>(smc);
  float (*Hs)[kFV][kFT + 1] = reinterpret_cast<float (*)[kFV][kFT + 1]>(smc + 9 * kCT * kCT);
  __shared__ int frow[kFV], fcol[kFV];  // local coarse index of each virtual fine row/col, -1 = odd
  int tid = threadIdx.x, nt = blockDim.x;
  int y0 = blockIdx.y * kFT, x0 = blockIdx.x * kFT;
  int cy0 = max(0, y0 / 2 - 1), cx0 = max(0, x0 / 2 - 1);
  if (tid < kFV) {
    int R = reflect_index(y0 - 2 + tid, h);
    frow[tid] = (R & 1) ? -1 : (R >> 1) - cy0;
    int Rx = reflect_index(x0 - 2 + tid, w);
    fcol[tid] = (Rx & 1) ? -1 : (Rx >> 1) - cx0;
  }
  int64_t CP = (int64_t)cw * ch;
  if (gc) {
    for (int i = tid; i < 9 * kCT * kCT; i += nt) {
      int c = i / (kCT * kCT), r = i - c * (kCT * kCT);
      int yy = r / kCT, xx = r - yy * kCT;
      int Y = min(cy0 + yy, ch - 1), X = min(cx0 + xx, cw - 1);
      int64_t p = (int64_t)Y * cw + X;
      C[c][yy][xx] = c < 6 ? gc[c * CP + p] : cc[(c - 6) * CP + p];
    }
  }
  __syncthreads();
  // horizontal up-sampling of the virtual rows y0-2 .. y0+33
  for (int i = tid; i < kFV * kFT; i += nt) {
    int v = i >> 5, x = i & 31;
    int cr = frow[v];
    float acc[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] = 0.0f;
    if (cr >= 0 && gc) {
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        int cc2 = fcol[x + j];
        if (cc2 < 0) continue;
#pragma unroll
        for (int c = 0; c < 9; ++c) acc[c] += kK5x2[j] * C[c][cr][cc2];
      }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) Hs[c][v][x] = acc[c];
  }
  __syncthreads();
  int64_t P = (int64_t)w * h;
  for (int i = tid; i < kFT * kFT; i += nt) {
    int yy = i >> 5, x = i & 31;
    int Y = y0 + yy, X = x0 + x;
    if (Y >= h || X >= w) continue;
    float u[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      float acc = 0.0f;
#pragma unroll
      for (int k = 0; k < 5; ++k) acc += kK5x2[k] * Hs[c][yy + k][x];
      u[c] = acc;
    }
    int64_t p = (int64_t)Y * w + X;
    if (LEVEL0) {
      float a = wr[p], b = ws[p];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float v = a * (ref[3 * p + k] - u[k]) + b * (warped[3 * p + k] - u[3 + k]) + u[6 + k];
        out[3 * p + k] = fminf(fmaxf(v, 0.0f), 1.0f);
      }
    } else {
      float a = g[6 * P + p], b = g[7 * P + p];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        out[k * P + p] = a * (g[k * P + p] - u[k]) + b * (g[(3 + k) * P + p] - u[3 + k]) + u[6 + k];
    }
  }
}

// top of the pyramid: C = w_ref * G_ref + w_src * G_src (laps[-1] = gp[-1])
__global__ void fuse_top_kernel(const float* __restrict__ g, int w, int h, float* __restrict__ c) {
  int64_t P = (int64_t)w * h;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  float a = g[6 * P + i], b = g[7 * P + i];
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k * P + i] = a * g[k * P + i] + b * g[(3 + k) * P + i];
}

constexpr size_t kW0Smem = sizeof(float) * (2 * kLT * kLT + 8 * kRT * (kRT + 1) + 8 * kOT * kRT);

void init_merge_attributes() {
  cudaFuncSetAttribute(weights_down0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kW0Smem);
  cudaFuncSetAttribute(down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDownSmem);
  cudaFuncSetAttribute(collapse_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kCollapseSmem);
  cudaFuncSetAttribute(collapse_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kCollapseSmem);
}

void launch_weights_down0(const float* ref, const float* warped, const float* ssim,
                          const uint8_t* valid, int w, int h, float* wr, float* ws, float* g1,
                          int ow, int oh, cudaStream_t s) {
  dim3 grd(ceil_div(ow, kOT), ceil_div(oh, kOT));
  weights_down0_kernel<<<grd, 256, kW0Smem, s>>>(ref, warped, ssim, valid, w, h, wr, ws, g1, ow, oh);
}

void launch_fuse_down(const float* in, int w, int h, float* out, int ow, int oh, cudaStream_t s) {
  dim3 grd(ceil_div(ow, kOT), ceil_div(oh, kOT));
  down_kernel<<<grd, 256, kDownSmem, s>>>(in, w, h, out, ow, oh);
}

void launch_fuse_top(const float* g, int w, int h, float* c, cudaStream_t s) {
  int64_t P = (int64_t)w * h;
  fuse_top_kernel<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(g, w, h, c);
}

void launch_fuse_collapse(const float* g, int w, int h, const float* gc, const float* cc, int cw,
                          int ch, float* c, cudaStream_t s) {
  dim3 grd(ceil_div(w, kFT), ceil_div(h, kFT));
  collapse_kernel<false><<<grd, 256, kCollapseSmem, s>>>(g, nullptr, nullptr, nullptr, nullptr, w, h, gc, cc,
                                             cw, ch, c);
}

void launch_fuse_collapse0(const float* ref, const float* warped, const float* wr, const float* ws,
                           int w, int h, const float* gc, const float* cc, int cw, int ch,
                           float* out, cudaStream_t s) {
  dim3 grd(ceil_div(w, kFT), ceil_div(h, kFT));
  collapse_kernel<true><<<grd, 256, kCollapseSmem, s>>>(nullptr, ref, warped, wr, ws, w, h, gc, cc, cw, ch,
                                            out);
}

}  // namespace hdr
