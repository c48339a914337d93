// Laplacian-pyramid exposure fusion (K14 + K15), fusion.py:96-157, for NF
// frames (NF = 2: the reference's fuse; NF > 2: the k-way generalisation of
// frame 0 is the reference, weights normalised over all
// frames), as four tiled kernels:
//   weights_down0  quality weights of every frame (fusion.py:67-77), the
//                  SSIM/validity trust and normalisation (fusion.py:117-128)
//                  for a 36x36 level-0 tile; for the owned 32x32 it writes
//                  the sources' weights and the level-0 blend of the frames
//                  B0 = sum_f w_f I_f (into the composite buffer), and it
//                  blurs + decimates the tile into level 1 of the 4*NF-channel
//                  Gaussian pyramid (RGB of every frame, then the NF weights)
//                  -- the weights never make a separate HBM round trip before
//                  the first reduction;
//   down           the same 5-tap reflect blur + [::2, ::2] for levels >= 1;
//   collapse       C_k = sum_f W_f (G_f - up G_f') + up C'  (the blend of
//                  laplacian_pyramid terms and collapse_pyramid folded
//                  together); level 0 is B0 - sum_f w_f up G_f' + up C',
//                  clipped: it reads B0 and NF-1 weight planes instead of
//                  every frame and weight (55 -> 31 B/px of level-0 traffic
//                  plus the coarse tiles), w_0 = 1 - sum_{f>0} w_f.
// Arithmetic is f32 (the composite tolerance is 1e-3).
#include "hdr_common.cuh"
#include "hdr_internal.h"
#include "hdr_bulk.cuh"

#include <algorithm>

namespace hdr {

__constant__ float kK5[5] = {1.0f / 16, 4.0f / 16, 6.0f / 16, 4.0f / 16, 1.0f / 16};
__constant__ float kK5x2[5] = {2.0f / 16, 8.0f / 16, 12.0f / 16, 8.0f / 16, 2.0f / 16};

__device__ __forceinline__ float lum_f(float r, float g, float b) {
  float y = fadd(fadd(fmul(0.299f, r), fmul(0.587f, g)), fmul(0.114f, b));
  return fminf(fmaxf(y, 0.0f), 1.0f);
}

// contrast x saturation x well-exposedness + 1e-12 (fusion.py:67-77).
// The laplacian is formed in f64 as in the reference: it is then exact (a sum
// of a few f32 values), so a flat neighbourhood gets exactly 0 contrast like
// numpy's. The channel std uses the pairwise form var = ((r-g)^2 + (g-b)^2 +
// (b-r)^2) / 9 in f32: it is exactly 0 for a grey pixel, as numpy's f64 std
// is (an f32 MEAN would leave ~1e-8 of std there, which outweighs the 1e-12
// floor and changes the blend weights completely), and within ~1e-7 relative
// of it otherwise. Everything after the laplacian -- sqrt, exp, products,
// normalisation -- is f32: relative error ~1e-7 on a weight moves the
// composite by ~1e-7, far inside the 1e-3 bar.
#ifndef HDR_SAT_APPROX
#define HDR_SAT_APPROX 1
#endif
__device__ __forceinline__ float quality_f(double lap, float r, float g, float b) {
  float d0 = r - g, d1 = g - b, d2 = b - r;
#if HDR_SAT_APPROX
  // MUFU square root (~2 ulp; exactly 0 at 0): the IEEE-rounded sqrt was 8% of
  // the weights pass's instructions, and the weights carry no bit-exact bar
  float sat, var = (d0 * d0 + d1 * d1 + d2 * d2) * (1.0f / 9.0f);
  asm("sqrt.approx.f32 %0, %1;" : "=f"(sat) : "f"(var));
#else
  float sat = __fsqrt_rn((d0 * d0 + d1 * d1 + d2 * d2) * (1.0f / 9.0f));
#endif
  float er = r - 0.5f, eg = g - 0.5f, eb = b - 0.5f;
  float ex = __expf(-(er * er + eg * eg + eb * eb) * 12.5f);
  return fabsf((float)lap) * sat * ex + 1e-12f;
}

// ndimage.laplace at the centre of a 3x3 neighbourhood, f64 (exact)
__device__ __forceinline__ double lap5(float n, float s, float w_, float e, float c) {
  double cc = c;
  return (((double)n + s) - 2.0 * cc) + (((double)w_ + e) - 2.0 * cc);
}

// ---------------------------------------------------------------- weights + level 1
constexpr int kOT = 16;           // level-1 outputs per tile side
constexpr int kRT = 2 * kOT + 4;  // level-0 region incl. the 2-px blur halo (36)
constexpr int kLT = kRT + 2;      // + 1-px laplacian halo (38)
constexpr int kRP = kRT + 1;      // padded row pitch of the staged region
// row pitch of the vertical-pass rows V: odd, so the two q rows a warp's
// horizontal pass reads (16 lanes each, stride 2) fall on disjoint banks
constexpr int kVP = kRT + 1;

// 5-tap blur + [::2, ::2] of NC staged channels px[c][36][kRP] into a 16x16
// level-1 tile, four channels at a time: vertical into V[4][16][37], then
// horizontal to global. V needs only 2368 floats, so it can alias the
// luminance tiles of weights_down (the occupancy limit is shared memory).
#ifndef HDR_DOWN_SLIDE
#define HDR_DOWN_SLIDE 1
#endif
template <int NC>
__device__ __forceinline__ void down_tile(const float* px, float* V, int tid, int Y0, int X0,
                                          float* __restrict__ out, int ow, int oh) {
  int P = ow * oh;
#pragma unroll 1
  for (int quad = 0; quad < NC / 4; ++quad) {
    const float* src = px + quad * 4 * kRT * kRP;
    // 4 * 16 * 36 = 2304 = 9 * 256 vertical outputs (q = c * 16 + oy): the
    // first 32 columns of every q with a warp per q and a lane per column
    // (consecutive words, no bank conflicts -- dealing the 36 columns out
    // flat put two q rows 74 words apart into one warp: 2.3 wavefronts per
    // load), then the last 4 columns of all 64 q rows in one round
#if HDR_DOWN_SLIDE
    // one task per (channel, column): the column's 35 input rows are read
    // from shared memory once into registers and its 16 outputs formed from
    // them (2.2 shared loads per output instead of 5: the weights pass was
    // bound by the L1/shared pipe, ncu l1tex 81%); 144 of the 256 threads
    if (tid < 4 * kRT) {
      const int c = tid / kRT, x = tid - c * kRT;
      const float* col = src + c * kRT * kRP + x;
      float in[2 * kOT + 3];
#pragma unroll
      for (int r = 0; r < 2 * kOT + 3; ++r) in[r] = col[r * kRP];
#pragma unroll
      for (int oy = 0; oy < kOT; ++oy) {
        float acc = kK5[0] * in[2 * oy];
#pragma unroll
        for (int k = 1; k < 5; ++k) acc += kK5[k] * in[2 * oy + k];
        V[(c * kOT + oy) * kVP + x] = acc;
      }
    }
#else
    auto vert = [&](int q, int x) {
      int c = q >> 4, oy = q & 15;
      const float* col = src + (c * kRT + 2 * oy) * kRP + x;
      float acc = kK5[0] * col[0];
#pragma unroll
      for (int k = 1; k < 5; ++k) acc += kK5[k] * col[k * kRP];
      V[q * kVP + x] = acc;
    };
#pragma unroll 2
    for (int q = tid >> 5; q < 4 * kOT; q += 8) vert(q, tid & 31);
    // remainder: warp w takes channel w/2, rows oy = 2k + (w&1), k = lane/4,
    // and columns 32 + lane%4 -- the 8 rows sit 20 banks apart, so the 32
    // lanes hit 32 distinct banks
    {
      const int wp = tid >> 5, ln = tid & 31;
      vert(16 * (wp >> 1) + 2 * (ln >> 2) + (wp & 1), 32 + (ln & 3));
    }
#endif
    __syncthreads();
    // 4 * 16 * 16 = 1024 = 4 * 256 horizontal outputs
#pragma unroll
    for (int i = tid; i < 4 * kOT * kOT; i += 256) {
      int q = i >> 4, ox = i & 15;
      int c = q >> 4, oy = q & 15;
      int Y = Y0 + oy, X = X0 + ox;
      const float* row = V + q * kVP + 2 * ox;
      float acc = kK5[0] * row[0];
#pragma unroll
      for (int k = 1; k < 5; ++k) acc += kK5[k] * row[k];
      if (Y < oh && X < ow) out[(quad * 4 + c) * P + Y * ow + X] = acc;
    }
    __syncthreads();
  }
}

#ifndef HDR_W0_MIN_BLOCKS
#define HDR_W0_MIN_BLOCKS 3
#endif
template <int NF>
__global__ void __launch_bounds__(256, NF == 2 ? HDR_W0_MIN_BLOCKS : 2) weights_down_kernel(FuseFrames<NF> fr, int w, int h,
                                                          float* __restrict__ g1, int ow, int oh,
                                                          float* __restrict__ b0) {
  pdl_wait();
  extern __shared__ float smf[];
  float* lum = smf;                    // [NF][38][38] luminance of every frame
  float* px = smf + NF * kLT * kLT;    // [4NF][36][37]: RGB of every frame, then the weights
  float* V = smf;                      // [4][16][37], aliases the luminance after the weights
  __shared__ int ridx[kLT], cidx[kLT];
  int tid = threadIdx.x;
  int Y0 = blockIdx.y * kOT, X0 = blockIdx.x * kOT;
  int vy0 = 2 * Y0 - 3, vx0 = 2 * X0 - 3;  // virtual origin of the 38x38 lum tile
  if (tid < kLT) {
    ridx[tid] = reflect_index(vy0 + tid, h);
    cidx[tid] = reflect_index(vx0 + tid, w);
  }
  __syncthreads();
  // every global load of the tile is issued before the first use: the SSIM
  // and validity of the weight pass (6 per thread and source frame) and the
  // RGB of all frames (6 x 3NF per thread)
  constexpr int kNW = (kRT * kRT + 255) / 256;  // 6
  constexpr int kNL = (kLT * kLT + 255) / 256;  // 6
  float svv[NF - 1][kNW];
  uint8_t vdd[NF - 1][kNW];
  {
    int ty = tid / kRT, tx = tid - ty * kRT;
#pragma unroll
    for (int it = 0; it < kNW; ++it) {
      int i = tid + it * 256;
      int p = ridx[min(ty + 1, kLT - 1)] * w + cidx[tx + 1];
#pragma unroll
      for (int f = 1; f < NF; ++f) {
        svv[f - 1][it] = i < kRT * kRT ? __ldg(fr.ssim[f] + p) : 0.0f;
        vdd[f - 1][it] = i < kRT * kRT ? __ldg(fr.valid[f] + p) : 0;
      }
      tx += 4; ty += 7;  // 256 = 7 * 36 + 4
      if (tx >= kRT) { tx -= kRT; ++ty; }
    }
  }
  {
    float rgb[kNL][3 * NF];
    int ly = tid / kLT, lx = tid - ly * kLT;
    int lys[kNL], lxs[kNL];
#pragma unroll
    for (int it = 0; it < kNL; ++it) {
      int i = tid + it * 256;
      lys[it] = ly; lxs[it] = lx;
      int p = (ridx[min(ly, kLT - 1)] * w + cidx[lx]) * 3;
      bool ok = i < kLT * kLT;
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int k = 0; k < 3; ++k) rgb[it][3 * f + k] = ok ? __ldg(fr.img[f] + p + k) : 0.0f;
      lx += 28; ly += 6;  // 256 = 6 * 38 + 28
      if (lx >= kLT) { lx -= kLT; ++ly; }
    }
#pragma unroll
    for (int it = 0; it < kNL; ++it) {
      int i = tid + it * 256;
      if (i >= kLT * kLT) break;
#pragma unroll
      for (int f = 0; f < NF; ++f)
        lum[f * kLT * kLT + i] = lum_f(rgb[it][3 * f], rgb[it][3 * f + 1], rgb[it][3 * f + 2]);
      if ((unsigned)(lys[it] - 1) < (unsigned)kRT && (unsigned)(lxs[it] - 1) < (unsigned)kRT) {
        float* d = px + (lys[it] - 1) * kRP + (lxs[it] - 1);
#pragma unroll
        for (int c = 0; c < 3 * NF; ++c) d[c * kRT * kRP] = rgb[it][c];
      }
    }
  }
  __syncthreads();
  {
    int ty = tid / kRT, tx = tid - ty * kRT;
#pragma unroll
    for (int it = 0; it < kNW; ++it) {
      int i = tid + it * 256;
      if (i >= kRT * kRT) break;
      int c = (ty + 1) * kLT + tx + 1;
      float* d = px + ty * kRP + tx;
      float q[NF];
      float tot = 0.0f;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const float* L = lum + f * kLT * kLT;
        double lap = lap5(L[c - kLT], L[c + kLT], L[c - 1], L[c + 1], L[c]);
        q[f] = quality_f(lap, d[(3 * f) * kRT * kRP], d[(3 * f + 1) * kRT * kRP],
                         d[(3 * f + 2) * kRT * kRP]);
        if (f > 0) {
          // source frames: x clip(SSIM, 0, 1) x validity (fusion.py:124-125)
          float sv = fminf(fmaxf(svv[f - 1][it], 0.0f), 1.0f);
          q[f] = vdd[f - 1][it] ? q[f] * sv : 0.0f;
        }
        tot = f == 0 ? q[0] : tot + q[f];
      }
      float inv = __frcp_rn(tot);
      // owned level-0 pixels: rows/cols [2Y0, 2Y0 + 32) of the real image
      bool own = (unsigned)(ty - 2) < 2u * kOT && (unsigned)(tx - 2) < 2u * kOT &&
                 vy0 + ty + 1 < h && vx0 + tx + 1 < w;
      int p = own ? ridx[ty + 1] * w + cidx[tx + 1] : 0;
      float bl[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        float wf = q[f] * inv;
        d[(3 * NF + f) * kRT * kRP] = wf;
        // the sources' weights for the collapse (w_0 = 1 - their sum there)
        if (own && f > 0) fr.wout[f][p] = wf;
#pragma unroll
        for (int k = 0; k < 3; ++k) bl[k] = f == 0 ? wf * d[k * kRT * kRP] : bl[k] + wf * d[(3 * f + k) * kRT * kRP];
      }
      // level 0's blend of the frames, B0 = sum_f w_f I_f: the level-0 term of
      // the Laplacian blend is B0 - sum_f w_f up(G1_f), so the collapse reads
      // B0 (12 B/px) instead of every frame (12 NF B/px)
      if (own)
#pragma unroll
        for (int k = 0; k < 3; ++k) b0[3 * p + k] = bl[k];
      tx += 4; ty += 7;
      if (tx >= kRT) { tx -= kRT; ++ty; }
    }
  }
  __syncthreads();
  down_tile<4 * NF>(px, V, tid, Y0, X0, g1, ow, oh);
}

// ---------------------------------------------------------------- levels >= 1
// 4 channels per CTA (blockIdx.z picks the group of the level's 4 NF
// channels): 31 KB of shared memory, so 7 CTAs fit per SM where the 8-channel
// tile (52 KB) fitted 4
template <int NF>
constexpr size_t down_smem() { return sizeof(float) * (4 * kRT * kRP + 4 * kOT * kVP); }

template <int NF>
__global__ void __launch_bounds__(256) down_kernel(const float* __restrict__ in, int w, int h,
                                                   float* __restrict__ out, int ow, int oh) {
  pdl_wait();
  constexpr int NC = 4;
  in += (int64_t)blockIdx.z * NC * w * h;
  out += (int64_t)blockIdx.z * NC * ow * oh;
  extern __shared__ float smd[];
  float* tile = smd;                // [NC][36][37]
  float* V = smd + NC * kRT * kRP;  // [4][16][37]
  __shared__ int ridx[kRT], cidx[kRT];
  int tid = threadIdx.x;
  int Y0 = blockIdx.y * kOT, X0 = blockIdx.x * kOT;
  int vy0 = 2 * Y0 - 2, vx0 = 2 * X0 - 2;
  if (tid < kRT) {
    ridx[tid] = reflect_index(vy0 + tid, h);
    cidx[tid] = reflect_index(vx0 + tid, w);
  }
  __syncthreads();
  int P = w * h;
  {
    // the whole region gathered by cp.async: every sample of every channel
    // in flight at once (register loads in dependent rounds left the small
    // levels latency-bound at ~8 us per launch)
    int ty = tid / kRT, tx = tid - ty * kRT;  // 256 = 7 * 36 + 4
#pragma unroll 1
    for (int i = tid; i < kRT * kRT; i += 256) {
      const float* sp = in + ridx[ty] * w + cidx[tx];
      float* dp = tile + ty * kRP + tx;
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async4(dp + c * kRT * kRP, sp + (int64_t)c * P);
      tx += 4; ty += 7;
      if (tx >= kRT) { tx -= kRT; ++ty; }
    }
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();
  down_tile<NC>(tile, V, tid, Y0, X0, out, ow, oh);
}

// ---------------------------------------------------------------- collapse
constexpr int kFT = 32;           // fine outputs per tile side
constexpr int kCT = kFT / 2 + 3;  // coarse rows/cols the tile can touch (19)
constexpr size_t kCollapseSmem = sizeof(float) * (9 * kCT * kCT + 9 * kCT * kFT);

// Polyphase form of up(): fine sample y gets 2 * K5[j] * coarse(R/2) for the
// taps j whose reflected fine index R = reflect(y - 2 + j) is even -- at most
// three distinct coarse rows. tap_rows() lists them (local coarse index and
// the summed weight; unused slots carry weight 0 and index 0).
__device__ __forceinline__ void tap_rows(int y, int n, int c0, int* idx, float* wt) {
  int k = 0;
#pragma unroll
  for (int t = 0; t < 3; ++t) { idx[t] = 0; wt[t] = 0.0f; }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    int R = reflect_index(y - 2 + j, n);
    if (R & 1) continue;
    int cr = (R >> 1) - c0;
    if (k > 0 && idx[k - 1] == cr) { wt[k - 1] += kK5x2[j]; continue; }
    if (k > 1 && idx[k - 2] == cr) { wt[k - 2] += kK5x2[j]; continue; }
    idx[k] = cr; wt[k] = kK5x2[j]; ++k;
  }
}

template <int NF>
constexpr size_t collapse_smem() {
  return sizeof(float) * (((3 * (NF + 1) * kCT * kCT + 3) & ~3) + 3 * (NF + 1) * kCT * kFT);
}

// 3NF + 3 coarse channels: G_f RGB (gc, the planar 4NF-channel level), C (cc)
#ifndef HDR_COLLAPSE_MIN_BLOCKS
#define HDR_COLLAPSE_MIN_BLOCKS 4
#endif
#ifndef HDR_COLLAPSE0_DIFF
#define HDR_COLLAPSE0_DIFF 1
#endif
#ifndef HDR_COLLAPSE_DIFF
#define HDR_COLLAPSE_DIFF 1
#endif
template <bool LEVEL0, int NF>
#ifndef HDR_COLLAPSE0_MIN_BLOCKS
#define HDR_COLLAPSE0_MIN_BLOCKS HDR_COLLAPSE_MIN_BLOCKS
#endif
__global__ void __launch_bounds__(256, LEVEL0 ? HDR_COLLAPSE0_MIN_BLOCKS : HDR_COLLAPSE_MIN_BLOCKS) collapse_kernel(const float* __restrict__ g, FuseFrames<NF> fr,
                                                      int w, int h, const float* __restrict__ gc,
                                                      const float* __restrict__ cc, int cw, int ch,
                                                      float* __restrict__ out) {
  pdl_wait();
  constexpr int NCH = 3 * (NF + 1);
  // up-sample coarse differences (3 NF channels) instead of the 3 NF + 3
  // coarse channels: level 0 (HDR_COLLAPSE0_DIFF) and the coarser levels
  // (HDR_COLLAPSE_DIFF), see the gather below
  constexpr bool DIFF = LEVEL0 ? HDR_COLLAPSE0_DIFF : HDR_COLLAPSE_DIFF;
  extern __shared__ float smc[];
  float* C = smc;                      // [NCH][19][19] coarse tile
  float* Hc = smc + ((NCH * kCT * kCT + 3) & ~3);  // [NCH][19][32] up-sampled along x (16B aligned)
  __shared__ int vr[kFT][3], hc[kFT][3];
  __shared__ float vw[kFT][3], hw[kFT][3];
  int tid = threadIdx.x;
  int y0 = blockIdx.y * kFT, x0 = blockIdx.x * kFT;
  int cy0 = max(0, y0 / 2 - 1), cx0 = max(0, x0 / 2 - 1);
  if (tid < kFT) {
    tap_rows(y0 + tid, h, cy0, vr[tid], vw[tid]);
  } else if (tid < 2 * kFT) {
    tap_rows(x0 + tid - kFT, w, cx0, hc[tid - kFT], hw[tid - kFT]);
  }
  int CP = cw * ch;
  if (gc) {  // null for a single-level pyramid: up() of nothing is 0
    // gathered by cp.async, every request in flight at once
    int yy = tid / kCT, xx = tid - yy * kCT;  // 256 = 13 * 19 + 9
    for (int i = tid; i < kCT * kCT; i += 256) {
      int p = min(cy0 + yy, ch - 1) * cw + min(cx0 + xx, cw - 1);
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        cp_async4(C + c * kCT * kCT + i, c < 3 * NF ? gc + c * CP + p : cc + (c - 3 * NF) * CP + p);
      xx += 9; yy += 13;
      if (xx >= kCT) { xx -= kCT; ++yy; }
    }
    cp_async_commit();
    cp_async_wait_all();
    if (DIFF) {
      // up() is linear, so the level-0 term B0 - sum_f w_f up(G_f) + up(C)
      // with w_0 = 1 - sum_{f>0} w_f is B0 + up(C - G_0) - sum_{f>0} w_f
      // up(G_f - G_0) (and a coarser level's sum_f W_f (G_f - up G'_f) +
      // up C' likewise, the blurred normalised weights summing to 1): the
      // differences are formed on the coarse samples this thread copied (its
      // own cp.async landed), and only 3 NF channels are up-sampled instead
      // of 3 NF + 3
      for (int i = tid; i < kCT * kCT; i += 256) {
        float g0[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) g0[k] = C[k * kCT * kCT + i];
#pragma unroll
        for (int k = 0; k < 3; ++k) C[k * kCT * kCT + i] = C[(3 * NF + k) * kCT * kCT + i] - g0[k];
#pragma unroll
        for (int f = 1; f < NF; ++f)
#pragma unroll
          for (int k = 0; k < 3; ++k) C[(3 * f + k) * kCT * kCT + i] -= g0[k];
      }
    }
  }
  __syncthreads();
  // channels up-sampled: the level-0 kernel needs 3 NF (differences above)
  constexpr int NU = DIFF ? 3 * NF : NCH;
  // horizontal: Hc[c][r][x] for the 19 coarse rows and the 32 fine columns
  for (int i = tid; i < kCT * kFT; i += 256) {
    int r = i >> 5, x = i & 31;
    int j0 = hc[x][0], j1 = hc[x][1], j2 = hc[x][2];
    float w0 = hw[x][0], w1 = hw[x][1], w2 = hw[x][2];
#pragma unroll
    for (int c = 0; c < NU; ++c) {
      const float* row = C + (c * kCT + r) * kCT;
      Hc[(c * kCT + r) * kFT + x] = gc ? w0 * row[j0] + w1 * row[j1] + w2 * row[j2] : 0.0f;
    }
  }
  __syncthreads();
  int P = w * h;
  // each thread: 4 consecutive pixels of one row (the 32x32 tile = 256 x 4),
  // so the up-sampled rows are read as float4 and, where the layout allows,
  // the frames / weights / output move as 16-byte vectors
  const int yy = tid >> 3, xq = (tid & 7) * 4;
  const int Y = y0 + yy, X = x0 + xq;
  if (Y >= h || X >= w) return;
  const int r0 = vr[yy][0], r1 = vr[yy][1], r2 = vr[yy][2];
  const float w0 = vw[yy][0], w1 = vw[yy][1], w2 = vw[yy][2];
  float u[NCH][4];
#pragma unroll
  for (int c = 0; c < NU; ++c) {
    const float* col = Hc + c * kCT * kFT + xq;
    float4 a = *reinterpret_cast<const float4*>(col + r0 * kFT);
    float4 b = *reinterpret_cast<const float4*>(col + r1 * kFT);
    float4 d = *reinterpret_cast<const float4*>(col + r2 * kFT);
    u[c][0] = w0 * a.x + w1 * b.x + w2 * d.x;
    u[c][1] = w0 * a.y + w1 * b.y + w2 * d.y;
    u[c][2] = w0 * a.z + w1 * b.z + w2 * d.z;
    u[c][3] = w0 * a.w + w1 * b.w + w2 * d.w;
  }
  const int p = Y * w + X;
  const bool full = X + 3 < w;
  // vector I/O needs 16-byte aligned rows: w % 4 == 0 (and P % 4 == 0 for
  // the planar levels); the bases are 256-byte aligned allocations
  bool aligned = ((uintptr_t)out & 15) == 0;
  if (LEVEL0) {
#pragma unroll
    for (int f = 1; f < NF; ++f) aligned = aligned && ((uintptr_t)fr.wout[f] & 15) == 0;
  } else {
    aligned = aligned && ((uintptr_t)g & 15) == 0;
  }
  const bool vec = full && aligned && (w & 3) == 0 && (LEVEL0 || (P & 3) == 0);
  float wt[NF][4];
#pragma unroll
  for (int f = (LEVEL0 || DIFF) ? 1 : 0; f < NF; ++f) {
    const float* wp = LEVEL0 ? fr.wout[f] + p : g + (3 * NF + f) * P + p;
    if (vec) {
      float4 t = __ldg(reinterpret_cast<const float4*>(wp));
      wt[f][0] = t.x; wt[f][1] = t.y; wt[f][2] = t.z; wt[f][3] = t.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) wt[f][j] = X + j < w ? __ldg(wp + j) : 0.0f;
    }
  }
  float o[3][4];
  if (LEVEL0) {
    // composite = B0 - sum_f w_f up(G1_f) + up(C1), w_0 = 1 - sum_{f>0} w_f
    // (B0 = sum_f w_f I_f, written by weights_down into `out`)
    float b[3][4];
    float* op = out + 3 * p;
    if (vec) {
      float4 t0 = *reinterpret_cast<const float4*>(op);
      float4 t1 = *(reinterpret_cast<const float4*>(op) + 1);
      float4 t2 = *(reinterpret_cast<const float4*>(op) + 2);
      float v12[12] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w, t2.x, t2.y, t2.z, t2.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) b[k][j] = v12[3 * j + k];
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) b[k][j] = X + j < w ? op[3 * j + k] : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#if HDR_COLLAPSE0_DIFF
      // u[k] = up(C - G_0), u[3f + k] = up(G_f - G_0)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float v = b[k][j] + u[k][j];
#pragma unroll
        for (int f = 1; f < NF; ++f) v -= wt[f][j] * u[3 * f + k][j];
        o[k][j] = fminf(fmaxf(v, 0.0f), 1.0f);
      }
#else
      float w0 = 1.0f;
#pragma unroll
      for (int f = 1; f < NF; ++f) w0 -= wt[f][j];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        float v = w0 * u[k][j];
#pragma unroll
        for (int f = 1; f < NF; ++f) v += wt[f][j] * u[3 * f + k][j];
        o[k][j] = fminf(fmaxf(b[k][j] - v + u[3 * NF + k][j], 0.0f), 1.0f);
      }
#endif
    }
    if (vec) {
      float4* o4 = reinterpret_cast<float4*>(op);
      o4[0] = make_float4(o[0][0], o[1][0], o[2][0], o[0][1]);
      o4[1] = make_float4(o[1][1], o[2][1], o[0][2], o[1][2]);
      o4[2] = make_float4(o[2][2], o[0][3], o[1][3], o[2][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (X + j < w)
#pragma unroll
          for (int k = 0; k < 3; ++k) op[3 * j + k] = o[k][j];
    }
    return;
  }
  float gv[NF][3][4];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float* gp = g + (3 * f + k) * P + p;
      if (vec) {
        float4 t = __ldg(reinterpret_cast<const float4*>(gp));
        gv[f][k][0] = t.x; gv[f][k][1] = t.y; gv[f][k][2] = t.z; gv[f][k][3] = t.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) gv[f][k][j] = X + j < w ? __ldg(gp + j) : 0.0f;
      }
    }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (DIFF) {
        // W_0 = 1 - sum_{f>0} W_f (the blurred normalised weights sum to 1):
        // C = G_0 + up(C' - G'_0) + sum_{f>0} W_f ((G_f - G_0) - up(G'_f - G'_0))
        float v = gv[0][k][j] + u[k][j];
#pragma unroll
        for (int f = 1; f < NF; ++f) v += wt[f][j] * ((gv[f][k][j] - gv[0][k][j]) - u[3 * f + k][j]);
        o[k][j] = v;
      } else {
        float v = 0.0f;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          v = f == 0 ? wt[0][j] * (gv[0][k][j] - u[k][j]) : v + wt[f][j] * (gv[f][k][j] - u[3 * f + k][j]);
        o[k][j] = v + u[3 * NF + k][j];
      }
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float* op = out + k * P + p;
    if (vec) {
      *reinterpret_cast<float4*>(op) = make_float4(o[k][0], o[k][1], o[k][2], o[k][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (X + j < w) op[j] = o[k][j];
    }
  }
}

// top of the pyramid: C = sum_f w_f * G_f (laps[-1] = gp[-1])
template <int NF>
__global__ void fuse_top_kernel(const float* __restrict__ g, int w, int h, float* __restrict__ c) {
  pdl_wait();
  int64_t P = (int64_t)w * h;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float v = 0.0f;
#pragma unroll
    for (int f = 0; f < NF; ++f) v = f == 0 ? g[(3 * NF) * P + i] * g[k * P + i]
                                           : v + g[(3 * NF + f) * P + i] * g[(3 * f + k) * P + i];
    c[k * P + i] = v;
  }
}

template <int NF>
constexpr size_t weights_smem() { return sizeof(float) * (NF * kLT * kLT + 4 * NF * kRT * kRP); }
static_assert(4 * kOT * kVP <= 2 * kLT * kLT, "V aliases the luminance tiles");

template <int NF>
static void init_merge_nf() {
  cudaFuncSetAttribute(weights_down_kernel<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)weights_smem<NF>());
  cudaFuncSetAttribute(down_kernel<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<NF>());
  cudaFuncSetAttribute(collapse_kernel<true, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)collapse_smem<NF>());
  cudaFuncSetAttribute(collapse_kernel<false, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)collapse_smem<NF>());
}

void init_merge_attributes() {
  init_merge_nf<2>();
  init_merge_nf<3>();
  init_merge_nf<4>();
}

template <int NF>
static void launch_fuse_nf(const FuseFrames<NF>& fr, const FusePyramid& py, cudaStream_t s,
                           KProbe* kp_w0, KProbe* kp_c0) {
  const int L = py.levels;
  const Dims* d = py.dims;
  // level 1 always has storage (py.g[1]): with a single-level pyramid the
  // weights pass still runs its reduction there and the collapse ignores it
  const Dims d1 = L > 1 ? d[1] : Dims{(d[0].w + 1) / 2, (d[0].h + 1) / 2};
  kprobe_mark(kp_w0, 0, s);
  dim3 g0(ceil_div(d1.w, kOT), ceil_div(d1.h, kOT));
  klaunch(weights_down_kernel<NF>, g0, dim3(256), weights_smem<NF>(), s, fr, d[0].w, d[0].h, py.g[1], d1.w,
          d1.h, py.out);
  kprobe_mark(kp_w0, 1, s);
  if (L == 1) {
    dim3 gf(ceil_div(d[0].w, kFT), ceil_div(d[0].h, kFT));
    klaunch(collapse_kernel<true, NF>, gf, dim3(256), collapse_smem<NF>(), s, (const float*)nullptr, fr,
               d[0].w, d[0].h, (const float*)nullptr, (const float*)nullptr, 0, 0, py.out);
    return;
  }
  for (int k = 1; k + 1 < L; ++k) {
    dim3 gk(ceil_div(d[k + 1].w, kOT), ceil_div(d[k + 1].h, kOT), NF);
    klaunch(down_kernel<NF>, gk, dim3(256), down_smem<NF>(), s, (const float*)py.g[k], d[k].w, d[k].h,
            py.g[k + 1], d[k + 1].w, d[k + 1].h);
  }
  int64_t Pt = (int64_t)d[L - 1].w * d[L - 1].h;
  klaunch(fuse_top_kernel<NF>, dim3((unsigned)((Pt + 255) / 256)), dim3(256), 0, s, (const float*)py.g[L - 1],
          d[L - 1].w, d[L - 1].h, py.c[L - 1]);
  for (int k = L - 2; k >= 1; --k) {
    dim3 gk(ceil_div(d[k].w, kFT), ceil_div(d[k].h, kFT));
    klaunch(collapse_kernel<false, NF>, gk, dim3(256), collapse_smem<NF>(), s, (const float*)py.g[k], fr,
               d[k].w, d[k].h, (const float*)py.g[k + 1], (const float*)py.c[k + 1], d[k + 1].w, d[k + 1].h,
               py.c[k]);
  }
  kprobe_mark(kp_c0, 0, s);
  dim3 gf(ceil_div(d[0].w, kFT), ceil_div(d[0].h, kFT));
  klaunch(collapse_kernel<true, NF>, gf, dim3(256), collapse_smem<NF>(), s, (const float*)nullptr, fr, d[0].w,
             d[0].h, (const float*)py.g[1], (const float*)py.c[1], d[1].w, d[1].h, py.out);
  kprobe_mark(kp_c0, 1, s);
}

void launch_fuse(int nf, const FuseFrameSet& fs, const FusePyramid& py, cudaStream_t s,
                 KProbe* kp_w0, KProbe* kp_c0) {
  auto pack = [&](auto fr) {
    for (int f = 0; f < (int)(sizeof(fr.img) / sizeof(fr.img[0])); ++f) {
      fr.img[f] = fs.img[f];
      fr.ssim[f] = fs.ssim[f];
      fr.valid[f] = fs.valid[f];
      fr.wout[f] = fs.wout[f];
    }
    return fr;
  };
  switch (nf) {
    case 2: launch_fuse_nf<2>(pack(FuseFrames<2>{}), py, s, kp_w0, kp_c0); break;
    case 3: launch_fuse_nf<3>(pack(FuseFrames<3>{}), py, s, kp_w0, kp_c0); break;
    default: launch_fuse_nf<4>(pack(FuseFrames<4>{}), py, s, kp_w0, kp_c0); break;
  }
}

}  // namespace hdr
