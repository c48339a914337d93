/*
 * hdrb200.h — C ABI of libhdrb200.so, the sm_100a register+merge path.
 *
 * The reference (`hdrflow`, pure Python) has no FFI; its drop-in boundary is
 * the set of Python functions in pkg/src/hdrflow/{pipeline,image,matcher,
 * weeding,geometry,densify,fusion}.py. Each export below is the GPU twin of
 * one of those functions (cited per entry) so a binding (ctypes, see
 * INTEGRATION.md) can replace them one for one. All array arguments are
 * DEVICE pointers (caller-owned, row-major, C-contiguous); work is enqueued
 * on the context's stream. No torch types cross this boundary.
 *
 * Error convention: every entry returns an int status.
 */
#ifndef HDRB200_H
#define HDRB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HDR_OK = 0,
  HDR_ERR_INVALID = 1,      /* ValueError (bad shape / precondition)        */
  HDR_ERR_DEGENERATE = 2,   /* geometry.DegenerateFit (geometry.py:18)      */
  HDR_ERR_REGISTRATION = 3, /* pipeline.RegistrationError (pipeline.py:27)  */
  HDR_ERR_CONFIG = 4,       /* pipeline.ConfigError (pipeline.py:31)        */
  HDR_ERR_CUDA = 5,         /* RuntimeError from the CUDA runtime           */
  HDR_ERR_EMPTY = 6,        /* "no result" (ssd_match returns None)         */
  HDR_ERR_SINGULAR = 7      /* numpy.linalg.LinAlgError (np.linalg.inv)     */
};

/* Mirror of PipelineParams (pipeline.py:35-57); delta < 0 means None. */
typedef struct hdr_params {
  int32_t tile;
  int32_t quadrant_half;
  int32_t radius;
  int32_t patch;
  int32_t max_levels;
  int32_t iterations;
  int32_t coarse_iterations;
  int32_t delta;
  int32_t passes;
  int32_t ssim_window;
  int32_t workers;
  int32_t _pad;
  double threshold;
  double eps_px;
  double sigma_s;
  double sigma_r;
  double ssim_sigma;
  double normalization_floor;
  uint64_t seed;
} hdr_params;

/* Caller-owned device outputs of one register_and_fuse call
 * (RegistrationOutput, pipeline.py:99-109). `ssim` is float32 on the device
 * (the host wrapper widens to float64). `info` receives int32 words:
 *   [0] status (HDR_OK or HDR_ERR_REGISTRATION)
 *   [1] 1 if `homography` is valid (MatchResult.homography is not None)
 *   [2] number of pyramid levels L
 *   [3 + 2*l], [4 + 2*l]  level_counts[l] = (raw, weeded), l < L
 *   [16] number of weeded level-0 matches, [17] number of raw level-0 matches
 *   [18] diagnostic: fits whose rank test fell in the grey zone
 * `matches`/`raw_matches` hold up to hdr_max_matches() rows of 5 float64. */
typedef struct hdr_outputs {
  float* composite;   /* (H, W, 3) */
  float* flow;        /* (H, W, 2) */
  float* warped;      /* (H, W, 3) */
  uint8_t* valid;     /* (H, W)    */
  float* ssim;        /* (H, W)    */
  double* matches;    /* (max, 5)  */
  double* raw_matches;/* (max, 5)  */
  double* homography; /* 3x3       */
  int32_t* info;      /* 32 words  */
} hdr_outputs;

#define HDR_INFO_WORDS 32

typedef struct hdr_ctx hdr_ctx;

/* ---- context / params ------------------------------------------------- */
void hdr_params_default(hdr_params* p);
/* PipelineParams.validate (pipeline.py:59-87): HDR_OK or HDR_ERR_CONFIG with
 * the reference's message copied into msg. */
int hdr_params_validate(const hdr_params* p, char* msg, size_t msg_len);
/* Allocates the whole workspace for images up to width x height once; the
 * hot path never allocates. `stream` is a cudaStream_t (NULL = legacy). */
int hdr_ctx_create(int32_t width, int32_t height, void* stream, hdr_ctx** out);
int hdr_ctx_destroy(hdr_ctx* ctx);
int hdr_ctx_set_stream(hdr_ctx* ctx, void* stream);
int32_t hdr_max_matches(int32_t width, int32_t height, int32_t tile);
const char* hdr_last_error(void);
/* Implementation switches for testing equivalent kernel paths (process-wide;
 * no reference counterpart). "dt_cluster_columns": 1 (default) = one
 * cluster-resident kernel per column sweep pair, 0 = chunk agg/link/apply.
 * "dt_sparse_first": 1 (default) = the pair's first domain-transform row pass
 * builds its rows from the CSR splat (no dense splat planes), 0 = dense splat.
 * "dt_cols_grid_div": d >= 1 (default 1) = launch 1/d of the co-resident
 * column-sweep clusters (tuning: SM sharing with concurrent pairs).
 * "dt_cols_prefetch": 1 (default) = the cluster column kernel prefetches the
 * next band by cp.async, 0 = plain loads.
 * "dt_skip_zero_rows": 1 (default) = with the sparse first row pass, rows
 * without splat samples are left unwritten and the first (prefetching
 * cluster) column sweep treats them as zero, 0 = they are written as zeros.
 * Returns HDR_ERR_INVALID for an unknown name. */
int hdr_set_option(const char* name, int64_t value);
/* Blocks until the context's stream drains; returns HDR_ERR_CUDA on a
 * sticky or asynchronous CUDA error. */
int hdr_ctx_sync(hdr_ctx* ctx);

/* ---- whole pair (pipeline.register_and_fuse, pipeline.py:174-198) -------
 * ref/src: (H, W, 3) float32 in [0,1]. Fully asynchronous, no host sync,
 * CUDA-graph capturable; the registration verdict lands in out->info[0]. */
int hdr_register_and_fuse(hdr_ctx* ctx, const hdr_params* p, int32_t width,
                          int32_t height, const float* ref, const float* src,
                          const hdr_outputs* out);
/* Captures the whole pair into a CUDA graph bound to these pointers and
 * replays it (first call per (ctx, shape, pointers, params) instantiates). */
int hdr_register_and_fuse_graph(hdr_ctx* ctx, const hdr_params* p, int32_t width,
                                int32_t height, const float* ref, const float* src,
                                const hdr_outputs* out);

/* Stage probes: when set, the pair pipeline records events[2*s] before and
 * events[2*s+1] after stage s on the context stream (cudaEvent_t handles;
 * NULL disables). Stages: 0 luminance/histograms/LUT/pyramids, 1 SAT +
 * corners, 2 coarse-to-fine match/weed/fit chain, 3 splat + domain-transform
 * filter, 4 densify-finalise + warp, 5 SSIM, 6 fusion. Probes are baked into
 * graphs captured while they are set. */
#define HDR_NUM_STAGES 7
int hdr_ctx_set_probes(hdr_ctx* ctx, void* const* events);
/* Kernel probes: events[2*j] / events[2*j+1] are recorded on the context
 * stream before / after the j-th launch (j < n <= 8) of one kernel family
 * inside each pair (register_and_fuse, eager or graph: baked into graphs
 * captured while set; n = 0 or events = NULL disarms). Families: */
#define HDR_KP_DT_ROWS 0         /* domain-transform row sweeps (one per pass)  */
#define HDR_KP_DT_COLS 1         /* domain-transform column sweeps (per pass)   */
#define HDR_KP_WARP 2            /* warp_image + luminance histogram            */
#define HDR_KP_SSIM 3            /* ssim_map                                    */
#define HDR_KP_FUSE_WEIGHTS0 4   /* fusion weights + first pyramid reduction    */
#define HDR_KP_FUSE_COLLAPSE0 5  /* level-0 blend + collapse -> composite       */
#define HDR_NUM_KPROBES 6
int hdr_ctx_set_kernel_probes(hdr_ctx* ctx, int32_t kernel, void* const* events, int32_t n);
/* Kernel nodes in the most recently instantiated pair graph of ctx. */
int32_t hdr_ctx_graph_kernels(hdr_ctx* ctx);

/* ---- file path: raw PNG samples ------------------------
 * The PNG container is decoded on the host; only the raw 8- or 16-bit
 * samples cross PCIe. hdr_decode_image is fileio.load_png's scaling
 * (fileio.py:21-41: f32(clip(v / (2^bits - 1)))) fused with pipeline.as_rgb
 * (pipeline.py:112-115): raw (h, w[, channels]) -> rgb (h, w, 3) f32.
 * hdr_encode_u8 is fileio.save_png's quantisation (fileio.py:44-53):
 * clip(floor(x * 255 + 0.5), 0, 255) of n floats. hdr_mean_luminance is
 * metering.choose_reference's tie-break statistic (metering.py:46-48) over n
 * pixels of an RGB (channels 3: luminance) or grey (channels 1: the value
 * itself) image, written to one device double. */
int hdr_decode_image(hdr_ctx* ctx, const void* raw, int32_t width, int32_t height,
                     int32_t channels, int32_t bits, float* rgb);
int hdr_encode_u8(hdr_ctx* ctx, const float* img, int64_t n, uint8_t* out);
int hdr_mean_luminance(hdr_ctx* ctx, const float* img, int32_t channels, int64_t n, double* out);
/* metering.select_offset's statistic (metering.py:28-29): the number of the n
 * pixels whose luminance (channels 3) or value (channels 1) is < dark_level
 * (compared in f32, as numpy 2 does), written to one device uint64. */
int hdr_dark_count(hdr_ctx* ctx, const float* img, int32_t channels, int64_t n, float dark_level,
                   uint64_t* out);
/* pipeline.run_hdr's compute (pipeline.py:267-282) on raw samples: decode
 * both frames into context-owned RGB buffers, register_and_fuse them
 * (use_graph != 0: the cached pair graph), and, when composite_u8 is not
 * NULL, write save_png's 8-bit composite (h, w, 3) next to out->composite. */
int hdr_register_and_fuse_raw(hdr_ctx* ctx, const hdr_params* p, int32_t width,
                              int32_t height, const void* ref_raw, const void* src_raw,
                              int32_t channels, int32_t bits, int32_t use_graph,
                              const hdr_outputs* out, uint8_t* composite_u8);

/* ---- per-stage twins ---------------------------------------------------- */
/* image.luminance (image.py:23-29): rgb (n,3) -> lum (n). */
int hdr_luminance(hdr_ctx* ctx, const float* rgb, int64_t n, float* lum);
/* image.match_histogram (image.py:96-122), one channel: src (n_src) mapped
 * onto ref's histogram; channel c of interleaved data via stride. */
int hdr_match_histogram(hdr_ctx* ctx, const float* src, int64_t n_src,
                        const float* ref, int64_t n_ref, int32_t stride,
                        float* out);
/* image.build_pyramid (image.py:71-88): levels[0] = img (not copied); writes
 * levels 1.. into out_levels[] (device buffers of (h>>l) x (w>>l) floats);
 * returns the count in *n_levels. */
int hdr_build_pyramid(hdr_ctx* ctx, const float* img, int32_t width, int32_t height,
                      int32_t max_levels, int32_t min_dim, float** out_levels,
                      int32_t* n_levels);
/* image.integral (image.py:32-44): (h+1, w+1) float64 summed-area table. */
int hdr_integral(hdr_ctx* ctx, const float* img, int32_t width, int32_t height,
                 double* table);
/* image.rect_sum (image.py:47-58): n queries q = (x0[n], y0[n], x1[n], y1[n])
 * int64 against a (h1, w1) float64 table; HDR_ERR_INVALID ("rectangle bounds
 * out of range") if any query is out of range. Synchronous. */
int hdr_rect_sum(hdr_ctx* ctx, const double* table, int32_t w1, int32_t h1, const int64_t* q,
                 int64_t n, double* out);
/* image.quantize_256 (image.py:91-93): n samples (f32, or f64 when is_f64)
 * -> uint8. */
int hdr_quantize_256(hdr_ctx* ctx, const void* x, int32_t is_f64, int64_t n, uint8_t* out);
/* image.downsample (image.py:61-68): (h, w, channels) interleaved, f32 (or
 * f64 when is_f64) -> (h/2, w/2, channels) float32. */
int hdr_downsample(hdr_ctx* ctx, const void* img, int32_t is_f64, int32_t width, int32_t height,
                   int32_t channels, float* out);
/* matcher.cornerness (matcher.py:51-61) at n points xy (n, 2) int32 of an
 * image whose (h+1, w+1) f64 integral table is given (callers check the
 * half-neighbourhood bounds): out (n, 2) = (cornerness, min contrast). */
int hdr_cornerness(hdr_ctx* ctx, const double* table, int32_t width, int32_t height,
                   const int32_t* xy, int32_t n, int32_t half, double* out);
/* matcher.detect_corners (matcher.py:64-105): rows (x, y, score) in tile
 * order; *count (host) receives n. corners needs room for ntiles rows. */
int hdr_detect_corners(hdr_ctx* ctx, const float* lum, int32_t width, int32_t height,
                       int32_t tile, double threshold, int32_t half,
                       double* corners, int32_t* count);
/* matcher.ssd_match (matcher.py:108-143) for n points at once:
 * pts (n, 4) int32 (x_ref, y_ref, x_init, y_init) -> out (n, 3) float64
 * (x_src, y_src, score), found[i] = 0 where the reference returns None. */
int hdr_ssd_match(hdr_ctx* ctx, const float* ref, const float* src, int32_t width,
                  int32_t height, const int32_t* pts, int32_t n, int32_t radius,
                  int32_t patch, double* out, uint8_t* found);
/* matcher._match_level (matcher.py:181-210): detect + predict through
 * h_pred (device 3x3) + SSD; raw (ntiles, 5); *count (host) = rows. */
int hdr_match_level(hdr_ctx* ctx, const hdr_params* p, const float* lum_ref,
                    const float* lum_src, int32_t width, int32_t height,
                    const double* h_pred, double* raw, int32_t* count);
/* weeding.weed (weeding.py:100-111): matches (n, 5); kept (n) int64 sorted
 * indices, *n_kept (host); witness (n) int64. seed is WeedParams.seed. */
int hdr_weed(hdr_ctx* ctx, const double* matches, int32_t n, int32_t width,
             int32_t height, int32_t iterations, double eps, uint64_t seed,
             int32_t delta, int64_t* kept, int32_t* n_kept, int64_t* witness);
/* matcher.fit_matches_homography (matcher.py:213-218): least-squares H over
 * (n, 5) matches; h (3x3, device). HDR_ERR_DEGENERATE on DegenerateFit. */
int hdr_fit_matches_homography(hdr_ctx* ctx, const double* matches, int32_t n,
                               int32_t width, int32_t height, double* h);
/* geometry.fit_homography (geometry.py:35-77): ref_pts/src_pts (n, 2). */
int hdr_fit_homography(hdr_ctx* ctx, const double* ref_pts, const double* src_pts,
                       int32_t n, double* h);
/* geometry.apply_homography (geometry.py:80-93): pts (n, 2) -> out (n, 2);
 * HDR_ERR_INVALID ("point maps to infinity") if any |denominator| < 1e-12.
 * Synchronous. */
int hdr_apply_homography(hdr_ctx* ctx, const double* h, const double* pts, int64_t n,
                         double* out);
/* geometry.symmetric_transfer_error (geometry.py:107-115): (n) float64;
 * HDR_ERR_SINGULAR if h is exactly singular (np.linalg.inv raises).
 * Synchronous. */
int hdr_symmetric_transfer_error(hdr_ctx* ctx, const double* h, const double* ref_pts,
                                 const double* src_pts, int64_t n, double* out);
/* geometry.inlier_mask (geometry.py:118-121). */
int hdr_inlier_mask(hdr_ctx* ctx, const double* h, const double* ref_pts,
                    const double* src_pts, int32_t n, double eps, uint8_t* mask);
/* geometry.homography_pixel_flow (geometry.py:124-135): flow (h, w, 2). */
int hdr_homography_flow(hdr_ctx* ctx, const double* h, int32_t width, int32_t height,
                        float* flow);
/* pipeline.match_stack (pipeline.py:122-130): RGB pair -> level-0 weeded and
 * raw matches, H, level counts (info words as in hdr_outputs). */
int hdr_match_stack(hdr_ctx* ctx, const hdr_params* p, int32_t width, int32_t height,
                    const float* ref, const float* src, double* matches,
                    double* raw_matches, double* homography, int32_t* info);
/* densify.build_sparse_maps (densify.py:38-56): (m, 5) -> pu, pv, n planes
 * (h, w) float64; collisions keep the lowest (score, index). */
int hdr_sparse_maps(hdr_ctx* ctx, const double* matches, int32_t m, int32_t width,
                    int32_t height, double* pu, double* pv, double* n);
/* densify.dt_filter (densify.py:78-113): guide (h, w) f32, planes (k, h, w)
 * float64 planar (any k; the planes are filtered three at a time), filtered
 * in place. Any width: rows wider than the shared-memory row kernels take
 * the sequential row twin. */
int hdr_dt_filter(hdr_ctx* ctx, const float* guide, double* planes, int32_t k,
                  int32_t width, int32_t height, double sigma_s, double sigma_r,
                  int32_t passes);
/* densify.dt_filter for a general guide (densify.py:59-66: the domain
 * distances sum |diff| over the guide's channels): guide (h, w, channels)
 * float64 interleaved, planes (k, h, w) float64, filtered in place by the
 * reference's sequential recursion, one thread per (line, plane). */
int hdr_dt_filter_general(hdr_ctx* ctx, const double* guide, int32_t channels, double* planes,
                          int32_t k, int32_t width, int32_t height, double sigma_s,
                          double sigma_r, int32_t passes);
/* densify.densify_flow (densify.py:116-142): filtered planes (3, h, w) ->
 * flow (h, w, 2) f32; fallback = device 3x3 or NULL. */
int hdr_densify_finalize(hdr_ctx* ctx, const double* smooth, int32_t width,
                         int32_t height, const double* fallback, double floor_,
                         float* flow);
/* densify.warp_image (densify.py:145-174): src (h, w, c), any c >= 1. */
int hdr_warp_image(hdr_ctx* ctx, const float* src, int32_t channels, int32_t width,
                   int32_t height, const float* flow, float* warped, uint8_t* valid);
/* fusion.ssim_map (fusion.py:34-64): a, b (h, w) f32 -> ssim (h, w) f32. */
int hdr_ssim_map(hdr_ctx* ctx, const float* a, const float* b, int32_t width,
                 int32_t height, int32_t window, double sigma, float* out);
/* pipeline.make_ssim (pipeline.py:165-171). */
int hdr_make_ssim(hdr_ctx* ctx, const float* lum_ref, const float* warped,
                  int32_t width, int32_t height, int32_t window, double sigma,
                  float* out);
/* fusion.quality_weights (fusion.py:67-77): rgb (h, w, 3) -> (h, w) f32. */
int hdr_quality_weights(hdr_ctx* ctx, const float* rgb, int32_t width, int32_t height,
                        float* out);
/* n-frame stack (n = 2..4, BASELINE config "5MP
 * three-exposure stack"): frames[0] is the reference (pick it with
 * metering.choose_reference); each source f >= 1 is registered to it exactly
 * as register_and_fuse does up to the SSIM map (outs[f-1] receives its flow,
 * warped frame, validity, SSIM, matches, H and info words; composite may be
 * NULL there), then the n frames are blended by hdr_fuse_stack into
 * `composite`. A source that fails to register leaves info[0] =
 * HDR_ERR_REGISTRATION in its outputs (the caller raises, as the reference
 * would for that pair). */
int hdr_register_and_fuse_stack(hdr_ctx* ctx, const hdr_params* p, int32_t n, int32_t width,
                                int32_t height, const float* const* frames,
                                const hdr_outputs* const* outs, float* composite);
/* k-way fusion of an n-frame stack (n = 2..4): frames[0]
 * is the reference, frames[1..n-1] the warped sources with their SSIM
 * (ssim[f-1]) and validity (valid[f-1]); the weights are fusion.py:117-128's
 * generalised to n frames (w_0 = q(ref), w_f = q(warped_f) clip(ssim_f, 0, 1)
 * valid_f, each divided by their sum) and blended through fusion.py:96-157's
 * pyramids. n = 2 is exactly hdr_fuse. Arrays of device pointers live on
 * the host. */
int hdr_fuse_stack(hdr_ctx* ctx, int32_t n, const float* const* frames, const float* const* ssim,
                   const uint8_t* const* valid, int32_t width, int32_t height, int32_t levels,
                   float* out);
/* fusion.fusion_weights (fusion.py:117-128): normalised (w_ref, w_src),
 * each (h, w) f32; valid is 0/1 per pixel. */
int hdr_fusion_weights(hdr_ctx* ctx, const float* ref, const float* warped, const float* ssim,
                       const uint8_t* valid, int32_t width, int32_t height, float* w_ref,
                       float* w_src);
/* fusion._pyr_down (fusion.py:85-86): in (h, w, ch) f64 -> out
 * (ceil(h/2), ceil(w/2), ch): 5-tap reflect blur, then [::2, ::2]. */
int hdr_pyr_down(hdr_ctx* ctx, const double* in, int32_t width, int32_t height, int32_t ch,
                 double* out);
/* fusion._pyr_up (fusion.py:89-93): in (ch_h, ch_w, ch) f64, the ceil-half
 * of (height, width) -> out (height, width, ch): zero-insert, 2x-gain blur.
 * With base (height, width, ch): out = base - up for sign < 0 (a
 * laplacian_pyramid level, fusion.py:103-107) or base + up for sign > 0 (a
 * collapse_pyramid step, fusion.py:110-114); base may alias out. */
int hdr_pyr_up(hdr_ctx* ctx, const double* in, int32_t coarse_width, int32_t coarse_height,
               int32_t ch, int32_t width, int32_t height, const double* base, int32_t sign,
               double* out);
/* fusion.fuse (fusion.py:135-157): levels <= 0 selects the default. */
int hdr_fuse(hdr_ctx* ctx, const float* ref, const float* warped, const float* ssim,
             const uint8_t* valid, int32_t width, int32_t height, int32_t levels,
             float* out);

/* ---- row-band pieces of one pair across ranks ---------
 * paper_1504_01441_b200/banded.py runs one giant pair over N GPUs: the
 * registration is replicated, every rank owns the rows [y0, y1) of a band
 * (a multiple of hdr_band_rows_multiple() rows), and these entries do that
 * band's share of densify_flow (densify.py:116-142), warp_image
 * (densify.py:145-174) and make_ssim (pipeline.py:165-171); the caller sums
 * the column-chunk aggregates and the warped-luminance histogram over the
 * ranks (NCCL all-reduce) between them. */
int32_t hdr_band_rows_multiple(void);
/* doubles of the dt_filter chunk-aggregate buffer for (w, h) and k planes */
int64_t hdr_band_agg_doubles(int32_t width, int32_t height, int32_t k);
/* op 0: the band's row sweeps of pass pass_i; op 1: its column-chunk
 * aggregates into agg (chunk-major: chunk c's aggregates are the
 * hdr_band_agg_doubles(width, 16, k) doubles at c times that offset, so a
 * band's chunks form one block; gather the blocks over the ranks next);
 * op 2: link the whole agg and re-run the band's chunks, writing the
 * planes -- or, when flow != NULL (last pass, k = 3), the f32 flow with the
 * homography fallback below `floor_` (fallback/has_fb as hdr_densify_finalize). */
int hdr_band_dt(hdr_ctx* ctx, int32_t op, const float* guide, double* planes, int32_t k, int32_t width,
                int32_t height, int32_t y0, int32_t y1, double sigma_s, double sigma_r, int32_t passes,
                int32_t pass_i, double* agg, const double* fallback, const int32_t* has_fb, double floor_,
                float* flow);
/* warp_image of rows [y0, y1) of full-size buffers (+ the quantised warped
 * luminance and, when hist != NULL, its 256-bin histogram added to hist). */
int hdr_band_warp(hdr_ctx* ctx, const float* flow, int32_t width, int32_t height, int32_t y0, int32_t y1,
                  const float* src, float* warped, uint8_t* valid, uint8_t* qw, uint32_t* hist);
/* make_ssim rows [y0, y1): hist_w = the whole frame's warped-luminance
 * histogram (summed over ranks), qw valid on [y0 - 5, y1 + 5). */
int hdr_band_ssim(hdr_ctx* ctx, const float* lum_ref, const uint8_t* qw, const uint32_t* hist_w, int32_t width,
                  int32_t height, int32_t y0, int32_t y1, int32_t window, double sigma, float* out);

/* Tool: with hdr_set_option("trace", 1) every launch is bracketed by events;
 * writes "kernel<TAB>microseconds" lines for the launches since, then clears
 * them (synchronises the device). */
int hdr_trace_dump(char* buf, int64_t cap);

/* ---- host-side helpers (no GPU work) ------------------------------------ */
/* matcher.level_seed (matcher.py:146-149). */
uint32_t hdr_level_seed(uint64_t seed, int32_t level);
/* Philox keys of weeding._iteration_rng (weeding.py:62-66):
 * keys[2*i], keys[2*i+1] = SeedSequence(seed, spawn_key=(i,)).generate_state(2, u64). */
int hdr_iteration_keys(uint64_t seed, int32_t iterations, uint64_t* keys);
/* Test hook: the device sampler's own code run on the host —
 * Generator(Philox(key)).choice(n, 4, replace=False) repeated `draws` times
 * on one stream; out (draws, 4). */
int hdr_choice4_host(const uint64_t* key, int32_t n, int32_t draws, int64_t* out);
/* Test hook: the device DLT fit (geometry.fit_homography) run on the host
 * with HOST pointers; returns HDR_OK / HDR_ERR_DEGENERATE / HDR_ERR_INVALID. */
int hdr_fit_homography_host(const double* ref_pts, const double* src_pts, int32_t n,
                            double* h);

#ifdef __cplusplus
}
#endif
#endif
