// Internal launcher declarations shared between the kernel translation units
// and the C-ABI layer (hdr_api.cu). Every launcher only enqueues work.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hdr {

// Kernel probes (hdr_ctx_set_kernel_probes): events recorded on the launching
// stream around successive launches of one kernel family, so a caller can
// time individual kernels inside a pair (or a replayed pair graph).
constexpr int kMaxKProbeLaunches = 8;
struct KProbe {
  cudaEvent_t ev[2 * kMaxKProbeLaunches];
  int n;     // launches to bracket (0 = off)
  int next;  // next launch index
};
// records ev[2*next + end] (end = 0 before, 1 after) if armed; after the
// closing mark `next` advances. Safe while the stream is being captured.
void kprobe_mark(KProbe* p, int end, cudaStream_t s);

// per-tile detector output: x < 0 means "no corner in this tile"
struct TileCorner {
  int32_t x, y;
  double score;
};

// one raw/weeded match row (x_ref, y_ref, x_src, y_src, score)
struct MatchRow {
  double v[5];
};

void init_match_attributes();
void init_densify_attributes();
void init_fusion_attributes();
void init_raster_attributes();

// ---- k_raster.cu
void launch_luma_hist(const float* rgb, int64_t n, float* lum, uint8_t* q,
                      uint32_t* hist, cudaStream_t s);
void launch_hist_plain(const float* x, int64_t n, int32_t stride, uint32_t* hist,
                       cudaStream_t s);
void launch_lut(const uint32_t* hist_src, int64_t n_src, const uint32_t* hist_ref,
                int64_t n_ref, float* lut, cudaStream_t s);
void launch_apply_lut_q(const uint8_t* q, int64_t n, const float* lut, float* out,
                        cudaStream_t s);
void launch_apply_lut_f(const float* x, int64_t n, int32_t stride, const float* lut,
                        float* out, cudaStream_t s);
void launch_luminance(const float* rgb, int64_t n, float* lum, cudaStream_t s);
void launch_downsample2(const float* a, const float* b, int w, int h, float* oa,
                        float* ob, cudaStream_t s);
// One pyramid level of the lattice summed-area table + corner detector.
struct SatLevel {
  const float* img;
  int w, h;
  const int32_t* rowmap;   // h+1 entries: stored row index of table row Y, or -1
  const int32_t* colmap;   // w+1 entries
  const int32_t* rowlist;  // nrows entries: Y of each stored row (ascending)
  double* ctab;            // pass-1 column sums of stored rows, [nrows][w]
  double* ltab;            // lattice table, [nrows][ncols]
  int nrows, ncols;
  TileCorner* tiles;       // per-tile detector output
  int tile_base;           // first block of this level in the detect grid
};
struct SatBatch {
  SatLevel lv[5];
  int n;
  // Exactness certificate per level (k_raster.cu K4): when every partial sum
  // of numpy's cumsums is exactly representable, any summation order gives
  // numpy's bits and the detector takes the tile-local path. null = never.
  int32_t* qmin;   // min log2 quantum of the level's nonzero samples
  double* sums;    // sum of the level's samples
};
struct DetectParams {
  int tile, half;
  double threshold;
  int exact_ok;    // tile region fits the tile-local kernel's shared memory
};
// precleared: sums = 0 and qmin = 0x3f3f3f3f already (the pair's first kernel)
void launch_level_stats(const SatBatch& b, int max_pixels, cudaStream_t s, bool precleared = false);
void launch_sat(const SatBatch& b, int max_w, int max_rows, cudaStream_t s);
void launch_detect(const SatBatch& b, int total_tiles, const DetectParams& dp, cudaStream_t s);
size_t detect_exact_smem(int tile, int half);
void launch_cornerness(const double* table, int w1, const int32_t* xy, int n, int half, double* out,
                       cudaStream_t s);
void launch_compact_corners(const TileCorner* tiles, int ntiles, double* corners,
                            int32_t* count, cudaStream_t s);

// ---- k_match.cu
void launch_ssd_tiles(const TileCorner* tiles, int ntiles, const float* ref,
                      const float* src, int w, int h, const double* hpred, int radius,
                      int patch, MatchRow* rows, uint8_t* flags, cudaStream_t s);
void launch_ssd_points(const float* ref, const float* src, int w, int h,
                       const int32_t* pts, int n, int radius, int patch, double* out,
                       uint8_t* found, cudaStream_t s);
// mask / witness: when given, the weeding arrays for nslots rows are cleared
// too (launch_weed(..., cleared = true) then skips its memsets)
void launch_compact_rows(const MatchRow* rows, const uint8_t* flags, int nslots,
                         MatchRow* out, int32_t* count, double* out_copy,
                         cudaStream_t s, uint32_t* mask = nullptr, int32_t* witness = nullptr);
void launch_weed(const MatchRow* rows, const int32_t* count, int n_static, int w,
                 int h, int iterations, double eps, const uint64_t* keys, int delta,
                 uint32_t* mask, int32_t* witness, int32_t* grey, cudaStream_t s,
                 bool cleared = false);
// compaction of the weeded set + least-squares H (+ level bookkeeping)
void launch_finish_level(const MatchRow* raw, const int32_t* raw_count,
                         const uint32_t* mask, int w, int h, int level,
                         MatchRow* weeded, int32_t* weeded_count, int64_t* kept_idx,
                         double* hpred, double* homography, int32_t* info,
                         double* out_matches, double* out_raw, int32_t* grey,
                         cudaStream_t s);
void launch_fit_rows(const MatchRow* rows, const int32_t* count, int w, int h,
                     double* H, int32_t* status, cudaStream_t s);
void launch_fit_points(const double* ref_pts, const double* src_pts, int n, double* H,
                       int32_t* status, cudaStream_t s);
void launch_inlier_mask(const double* H, const double* ref_pts, const double* src_pts,
                        int n, double eps, uint8_t* mask, cudaStream_t s);
void launch_set_identity(double* h, cudaStream_t s);

// ---- k_densify.cu / k_dtfilter.cu
// Up to three H x W planes, each f32 or f64 (see hdr_planes.cuh).
struct DtPlanes {
  void* p[3];
  int f64[3];
  int k;
};
void launch_splat(const double* matches, const int32_t* count, int m_static, int w,
                  int h, DtPlanes maps, uint64_t* scratch_key, int32_t* scratch_idx,
                  int32_t* status, cudaStream_t s);
int64_t dt_scratch_doubles(int w, int h, int k);
void dt_set_cluster_columns(bool on);
void dt_set_cols_prefetch(bool on);
void dt_set_skip_zero_rows(bool on);
void dt_set_cols_grid_div(int d);  // 0 auto, 1..3 force a band shape, -1 off
// optional fused densify-finalise for the last column pass (K == 3)
struct DtFlowOut {
  const double* fallback;   // 3x3 H or null
  const int32_t* has_fb;    // device flag gating fallback (null = use if non-null)
  double floor_;
  float* flow;              // (h, w, 2)
};
// sparse splat maps in CSR-by-row form: row y's samples are
// entries[row_start[y] .. row_start[y+1]) (collision winners only)
struct SparseEntry {
  int32_t x, pad;
  double u, v;
};
struct DtSparse {
  const int32_t* row_start;  // h + 1
  const SparseEntry* entries;
};
// splat winners -> CSR rows (no dense planes); row_start needs h + 1 ints,
// row_count h + 1 ints of scratch, entries up to m rows
void launch_splat_rows(const double* matches, const int32_t* count, int m_static, int w, int h,
                       uint64_t* scratch_key, int32_t* scratch_idx, int32_t* row_count,
                       int32_t* row_start, SparseEntry* entries, int32_t* status, cudaStream_t s);
// the first row pass can consume the CSR splat directly (K == 3, f64 rows)
bool dt_sparse_first_ok(const float* guide, const DtPlanes& P, int w);
// returns true when the flow was written (planes then hold pre-final values);
// with `first`, the planes' initial content is ignored: pass 1 builds its
// rows from the CSR splat (see dt_sparse_first_ok)
bool launch_dt_filter(const float* guide, DtPlanes planes, int w, int h, double sigma_s,
                      double sigma_r, int passes, double* scratch, cudaStream_t s,
                      const DtFlowOut* fo = nullptr, KProbe* kp_rows = nullptr,
                      KProbe* kp_cols = nullptr, const DtSparse* first = nullptr);
// row-band pieces of dt_filter: op 0 = the band's row
// sweeps, 1 = its column-chunk aggregates into agg (the whole image's layout),
// 2 = link the (rank-summed) agg and apply the band's chunks (+ the flow when
// fo->flow, K == 3). Bands are whole chunks of dt_band_chunk_rows() rows.
void launch_dt_band(int op, const float* guide, const DtPlanes& P, int w, int h, int y0, int y1,
                    double sigma_s, double sigma_r, int passes, int i, double* agg, double* carry,
                    const DtFlowOut* fo, cudaStream_t s);
int64_t dt_band_agg_doubles(int w, int h, int k);
int dt_band_chunk_rows();
// ---- k_twins.cu (general stage twins)
// f32 single-channel guide, one row pass of any width (sequential per row)
void launch_dt_rows_seq(const float* guide, const DtPlanes& P, int w, int h, double ratio, double c,
                        cudaStream_t s);
// the whole filter for an f64 guide of C interleaved channels, <= 3 planes
void launch_dt_filter_general(const double* guide, int C, const DtPlanes& P, int w, int h,
                              double sigma_s, double sigma_r, int passes, cudaStream_t s);
// q = (x0[n], y0[n], x1[n], y1[n]) int64; *bad = 1 on an out-of-range query
void launch_rect_sum(const double* table, int64_t w1, int64_t h1, const int64_t* q, int64_t n,
                     double* out, int32_t* bad, cudaStream_t s);
void launch_quantize(const void* x, bool f64, int64_t n, uint8_t* out, cudaStream_t s);
void launch_downsample_ch(const void* in, bool f64, int w, int h, int C, float* out, cudaStream_t s);
void launch_apply_homography(const double* H, const double* pts, int64_t n, double* out, int32_t* bad,
                             cudaStream_t s);
void launch_transfer_error(const double* H, const double* rp, const double* sp, int64_t n, double* out,
                           int32_t* bad, cudaStream_t s);
void launch_hflow(const double* H, int w, int h, float* flow, cudaStream_t s);
void launch_warp_rows(const float* flow, int w, int h, int y0, int y1, const float* src, float* warped,
                      uint8_t* valid, uint8_t* qw, uint32_t* hist, cudaStream_t s);
bool launch_ssim_rows(const float* a, const uint8_t* qb, const float* lut_b, int w, int h, int y0, int y1,
                      int window, const double* taps, float* out, cudaStream_t s);
void launch_warp(const float* flow, int w, int h, const float* src, float* warped, uint8_t* valid,
                 uint8_t* qw, uint32_t* hist, cudaStream_t s);
void launch_finalize_warp(DtPlanes smooth, const double* fallback,
                          const int32_t* has_fallback, int w, int h, double floor_,
                          const float* src, int channels, float* flow, float* warped,
                          uint8_t* valid, uint8_t* qw, uint32_t* hist_w,
                          bool do_flow, cudaStream_t s);

// ---- k_ingest.cu
void launch_decode(const void* in, int64_t npx, int channels, int bits, float* out,
                   cudaStream_t s);
void launch_encode_u8(const float* x, int64_t n, uint8_t* out, cudaStream_t s);
void launch_mean_luminance(const float* img, int channels, int64_t n, double* out, cudaStream_t s);
void launch_dark_count(const float* img, int channels, int64_t n, float dark,
                       unsigned long long* out, cudaStream_t s);

// ---- k_fusion.cu
void launch_ssim(const float* a, const float* b_or_null, const uint8_t* qb,
                 const float* lut_b, int w, int h, int window, const double* taps,
                 float* out, cudaStream_t s);
void launch_quality(const float* rgb, int w, int h, float* out, cudaStream_t s);
void launch_fusion_weights(const float* ref, const float* warped, const float* ssim,
                           const uint8_t* valid, int w, int h, float* wr, float* ws,
                           cudaStream_t s);
// fusion._pyr_down / _pyr_up twins (f64, (h, w, c) interleaved)
void launch_pyr_down(const double* in, int w, int h, int c, double* out, cudaStream_t s);
void launch_pyr_up(const double* in, int cw, int ch, int c, double* out, int w, int h,
                   const double* base, int sign, cudaStream_t s);
// ---- k_merge.cu: Laplacian-pyramid fusion of NF = 2..4 frames (frame 0 is
// the reference); level k >= 1 holds 4*NF planar channels (RGB of every
// frame, then the NF weights) in g[k] and the 3 collapse channels in c[k].
constexpr int kMaxFuseFrames = 4;
struct Dims {
  int w, h;
};
template <int NF>
struct FuseFrames {
  const float* img[NF];      // (h, w, 3) interleaved; [0] = reference, [f] = warped source f
  const float* ssim[NF];     // [f >= 1]: (h, w)
  const uint8_t* valid[NF];  // [f >= 1]: (h, w)
  float* wout[NF];           // normalised level-0 weights (h, w)
};
struct FuseFrameSet {
  const float* img[kMaxFuseFrames];
  const float* ssim[kMaxFuseFrames];
  const uint8_t* valid[kMaxFuseFrames];
  float* wout[kMaxFuseFrames];
};
struct FusePyramid {
  int levels;
  Dims dims[32];
  float* g[32];   // g[0] unused; g[1] must exist even for levels == 1
  float* c[32];
  float* out;     // composite (h, w, 3), clipped
};
void init_merge_attributes();
void launch_fuse(int nf, const FuseFrameSet& fs, const FusePyramid& py, cudaStream_t s,
                 KProbe* kp_w0 = nullptr, KProbe* kp_c0 = nullptr);

}  // namespace hdr
