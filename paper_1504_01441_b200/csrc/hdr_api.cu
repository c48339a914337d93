// C ABI of libhdrb200.so: context/workspace, the device-resident pair
// pipeline (pipeline.register_and_fuse, pipeline.py:174-198), CUDA-graph
// replay, per-stage twins, and the host-side SeedSequence key schedule.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <cstring>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hdrb200.h"
#include "hdr_common.cuh"
#include "hdr_geom.cuh"
#include "hdr_internal.h"
#include "hdr_scan.cuh"

using namespace hdr;

// ------------------------------------------------------------ errors
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(HDR_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

static int check_launch() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return fail(HDR_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return HDR_OK;
}

extern "C" const char* hdr_last_error(void) { return g_err.c_str(); }

namespace hdr {
bool g_pdl = true;
bool g_trace = false;
struct TraceRec {
  const void* kern;
  cudaEvent_t ev[2];
};
static std::vector<TraceRec> g_trace_recs;
void trace_launch(const void* kern, cudaStream_t s, int end) {
  if (!end) {
    TraceRec r{kern, {nullptr, nullptr}};
    cudaEventCreate(&r.ev[0]);
    cudaEventCreate(&r.ev[1]);
    g_trace_recs.push_back(r);
  }
  cudaEventRecord(g_trace_recs.back().ev[end], s);
}
}

// Tool: per-launch device times since tracing was switched on (one line per
// launch, "name<TAB>microseconds"), then the records are cleared. Needs the
// traced work finished (synchronises the device).
extern "C" int hdr_trace_dump(char* buf, int64_t cap) {
  cudaDeviceSynchronize();
  std::string out;
  for (auto& r : hdr::g_trace_recs) {
    const char* name = nullptr;
    if (cudaFuncGetName(&name, r.kern) != cudaSuccess || !name) name = "?";
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, r.ev[0], r.ev[1]);
    out += std::string(name) + "\t" + std::to_string(ms * 1e3) + "\n";
    cudaEventDestroy(r.ev[0]);
    cudaEventDestroy(r.ev[1]);
  }
  hdr::g_trace_recs.clear();
  cudaGetLastError();
  if ((int64_t)out.size() + 1 > cap) return HDR_ERR_INVALID;
  memcpy(buf, out.c_str(), out.size() + 1);
  return HDR_OK;
}

// test hook: 0 sends the pair through the dense splat + first row pass
static bool g_sparse_first = true;

extern "C" int hdr_set_option(const char* name, int64_t value) {
  if (name && std::string(name) == "dt_cluster_columns") {
    hdr::dt_set_cluster_columns(value != 0);
    return HDR_OK;
  }
  if (name && std::string(name) == "dt_sparse_first") {
    g_sparse_first = value != 0;
    return HDR_OK;
  }
  if (name && std::string(name) == "dt_cols_grid_div") {
    hdr::dt_set_cols_grid_div((int)value);
    return HDR_OK;
  }
  if (name && std::string(name) == "trace") {
    hdr::g_trace = value != 0;
    return HDR_OK;
  }
  if (name && std::string(name) == "pdl") {
    hdr::g_pdl = value != 0;
    return HDR_OK;
  }
  if (name && std::string(name) == "dt_cols_prefetch") {
    hdr::dt_set_cols_prefetch(value != 0);
    return HDR_OK;
  }
  if (name && std::string(name) == "dt_skip_zero_rows") {
    hdr::dt_set_skip_zero_rows(value != 0);
    return HDR_OK;
  }
  return fail(HDR_ERR_INVALID, std::string("unknown option: ") + (name ? name : "(null)"));
}

// ------------------------------------------------------------ SeedSequence
// numpy.random.SeedSequence (numpy/random/bit_generator.pyx), host side.
namespace {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                   MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;

void words_of(uint64_t v, std::vector<uint32_t>& out) {
  if (v == 0) { out.push_back(0); return; }
  while (v) { out.push_back((uint32_t)v); v >>= 32; }
}

void seedseq_pool(uint64_t entropy, uint64_t spawn, uint32_t pool[4]) {
  std::vector<uint32_t> run, sp, ent;
  words_of(entropy, run);
  words_of(spawn, sp);
  while (run.size() < 4) run.push_back(0);  // spawn key present: pad run entropy
  ent = run;
  ent.insert(ent.end(), sp.begin(), sp.end());
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
}

void seedseq_state(const uint32_t pool[4], int n, uint32_t* out) {
  uint32_t hc = INIT_B;
  for (int i = 0; i < n; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hc;
    hc *= MULT_B;
    v *= hc;
    v ^= v >> 16;
    out[i] = v;
  }
}
}  // namespace

extern "C" uint32_t hdr_level_seed(uint64_t seed, int32_t level) {
  uint32_t pool[4], s;
  seedseq_pool(seed, (uint64_t)level, pool);
  seedseq_state(pool, 1, &s);
  return s;
}

extern "C" int hdr_iteration_keys(uint64_t seed, int32_t iterations, uint64_t* keys) {
  if (iterations < 0 || (!keys && iterations)) return fail(HDR_ERR_INVALID, "bad key request");
  for (int i = 0; i < iterations; ++i) {
    uint32_t pool[4], st[4];
    seedseq_pool(seed, (uint64_t)i, pool);
    seedseq_state(pool, 4, st);
    keys[2 * i] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    keys[2 * i + 1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  }
  return HDR_OK;
}

extern "C" int hdr_choice4_host(const uint64_t* key, int32_t n, int32_t draws, int64_t* out) {
  if (n < 4) return fail(HDR_ERR_INVALID, "n must be >= 4");
  Philox g;
  philox_init(&g, key[0], key[1]);
  for (int d = 0; d < draws; ++d) {
    int idx[4];
    choice4(&g, n, idx);
    for (int k = 0; k < 4; ++k) out[4 * d + k] = idx[k];
  }
  return HDR_OK;
}

extern "C" int hdr_fit_homography_host(const double* rp, const double* sp, int32_t n, double* H) {
  if (n < 4) return fail(HDR_ERR_INVALID, "need at least 4 point pairs");
  if (n == 4) {
    double px[4], py[4], qx[4], qy[4];
    for (int i = 0; i < 4; ++i) { px[i] = rp[2 * i]; py[i] = rp[2 * i + 1]; qx[i] = sp[2 * i]; qy[i] = sp[2 * i + 1]; }
    int g = 0;
    return fit4(px, py, qx, qy, H, &g) ? fail(HDR_ERR_DEGENERATE, "degenerate correspondence set")
                                       : HDR_OK;
  }
  // same arithmetic as block_fit's least-squares branch, serially
  double c[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) { c[0] += rp[2 * i]; c[1] += rp[2 * i + 1]; c[2] += sp[2 * i]; c[3] += sp[2 * i + 1]; }
  for (int k = 0; k < 4; ++k) c[k] /= n;
  double md0 = 0, md1 = 0;
  for (int i = 0; i < n; ++i) {
    md0 += hypot(rp[2 * i] - c[0], rp[2 * i + 1] - c[1]);
    md1 += hypot(sp[2 * i] - c[2], sp[2 * i + 1] - c[3]);
  }
  md0 /= n;
  md1 /= n;
  if (md0 < 1e-12 || md1 < 1e-12) return fail(HDR_ERR_DEGENERATE, "coincident points");
  double sr = sqrt(2.0) / md0, ss = sqrt(2.0) / md1;
  double tr[3] = {sr, -sr * c[0], -sr * c[1]}, ts[3] = {ss, -ss * c[2], -ss * c[3]};
  double g45[45] = {0};
  for (int i = 0; i < n; ++i) {
    double r0[9], r1[9];
    dlt_rows((rp[2 * i] - c[0]) * sr, (rp[2 * i + 1] - c[1]) * sr, (sp[2 * i] - c[2]) * ss,
             (sp[2 * i + 1] - c[3]) * ss, r0, r1);
    int k = 0;
    for (int a = 0; a < 9; ++a)
      for (int b = a; b < 9; ++b) { g45[k] += r0[a] * r0[b] + r1[a] * r1[b]; ++k; }
  }
  int g = 0;
  return fit_from_gram(g45, tr, ts, H, &g) ? fail(HDR_ERR_DEGENERATE, "degenerate correspondence set")
                                          : HDR_OK;
}

// ------------------------------------------------------------ params
extern "C" void hdr_params_default(hdr_params* p) {
  memset(p, 0, sizeof(*p));
  p->tile = 64;
  p->threshold = 4.0 / 255.0;
  p->quadrant_half = 8;
  p->radius = 10;
  p->patch = 21;
  p->max_levels = 5;
  p->iterations = 256;
  p->coarse_iterations = 64;
  p->delta = -1;
  p->eps_px = 2.0;
  p->sigma_s = 400.0;
  p->sigma_r = 0.2;
  p->passes = 3;
  p->ssim_window = 11;
  p->ssim_sigma = 1.5;
  p->normalization_floor = 1e-4;
  p->seed = 0;
  p->workers = 1;
}

extern "C" int hdr_params_validate(const hdr_params* p, char* msg, size_t len) {
  struct Rule { bool ok; const char* text; };
  const Rule rules[] = {  // PipelineParams.validate order (pipeline.py:60-87)
      {p->tile >= 16, "tile must be >= 16"},
      {p->threshold > 0, "threshold must be positive"},
      {p->quadrant_half >= 2, "quadrant_half must be >= 2"},
      {p->radius >= 1, "radius must be >= 1"},
      {p->patch >= 3 && p->patch % 2 == 1, "patch must be odd and >= 3"},
      {1 <= p->max_levels && p->max_levels <= kMaxLevels, "max_levels must be in [1, 5]"},
      {p->iterations >= 1, "iterations must be >= 1"},
      {p->coarse_iterations >= 1, "coarse_iterations must be >= 1"},
      {p->delta < 0 || p->delta >= 4, "delta must be >= 4"},
      {p->eps_px > 0, "eps_px must be positive"},
      {p->sigma_s > 0, "sigma_s must be positive"},
      {p->sigma_r > 0, "sigma_r must be positive"},
      {p->passes >= 1, "passes must be >= 1"},
      {p->ssim_window >= 3 && p->ssim_window % 2 == 1, "ssim_window must be odd and >= 3"},
      {p->ssim_sigma > 0, "ssim_sigma must be positive"},
      {p->normalization_floor > 0, "normalization_floor must be positive"},
      {p->workers >= 1, "workers must be >= 1"},
      {p->workers >= 1 && p->iterations % p->workers == 0, "iterations must be divisible by workers"},
      {p->workers >= 1 && p->coarse_iterations % p->workers == 0,
       "coarse_iterations must be divisible by workers"},
  };
  for (const Rule& r : rules)
    if (!r.ok) {
      if (msg && len) snprintf(msg, len, "%s", r.text);
      return fail(HDR_ERR_CONFIG, r.text);
    }
  return HDR_OK;
}

// ------------------------------------------------------------ geometry of a call
// image.build_pyramid level dims (image.py:71-88)
static int pyramid_dims(int w, int h, int max_levels, Dims* d) {
  d[0] = {w, h};
  int n = 1;
  while (n < max_levels) {
    int nw = d[n - 1].w / 2, nh = d[n - 1].h / 2;
    if (std::min(nw, nh) < 100) break;
    d[n++] = {nw, nh};
  }
  return n;
}

// fusion.default_fusion_levels (fusion.py:131-132): max(1, floor(log2 min) - 1)
static int fusion_levels_default(int w, int h) {
  int m = std::min(w, h);
  int lg = 31 - __builtin_clz((unsigned)m);
  return std::max(1, lg - 1);
}

// fusion.gaussian_pyramid dims: ceil halving while len < levels and min >= 2
static int fusion_dims(int w, int h, int levels, std::vector<Dims>& d) {
  d.clear();
  d.push_back({w, h});
  while ((int)d.size() < levels && std::min(d.back().w, d.back().h) >= 2)
    d.push_back({(d.back().w + 1) / 2, (d.back().h + 1) / 2});
  return (int)d.size();
}

static int64_t round4(int64_t n) { return (n + 3) & ~int64_t(3); }

// floats of a fusion pyramid of nf frames: levels 1.. (level 1 also for a
// single-level pyramid) x (4 nf Gaussian + 3 collapse channels)
static int64_t fusion_floats(const std::vector<Dims>& fd, int nf) {
  int64_t n = 0;
  for (size_t k = 1; k < std::max<size_t>(fd.size(), 2); ++k) {
    Dims d = k < fd.size() ? fd[k] : Dims{(fd[0].w + 1) / 2, (fd[0].h + 1) / 2};
    n += round4(4 * nf * (int64_t)d.w * d.h) + 64 + round4(3 * (int64_t)d.w * d.h) + 64;
  }
  return n;
}

static void fusion_layout(const std::vector<Dims>& fd, int nf, float* base, FusePyramid& py) {
  py.levels = (int)fd.size();
  float* q = base;
  for (size_t k = 0; k < std::max<size_t>(fd.size(), 2) && k < 32; ++k) {
    Dims d = k < fd.size() ? fd[k] : Dims{(fd[0].w + 1) / 2, (fd[0].h + 1) / 2};
    py.dims[k] = d;
    py.g[k] = py.c[k] = nullptr;
    if (k == 0) continue;
    int64_t n = (int64_t)d.w * d.h;
    py.g[k] = q;  // every region starts 16-byte aligned (vector I/O in collapse)
    q += round4(4 * nf * n) + 64;
    py.c[k] = q;
    q += round4(3 * n) + 64;
  }
}

static int ntiles_of(int w, int h, int tile) { return ceil_div(w, tile) * ceil_div(h, tile); }

// ------------------------------------------------------------ context
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  uint64_t used = 0;            // LRU stamp
};

struct KeySet {
  uint64_t* keys = nullptr;     // kMaxLevels x iters x 2
  int iters = 0;
};

constexpr size_t kMaxGraphs = 32;     // cached pair graphs per context
constexpr size_t kMaxParamSets = 8;   // cached key / tap sets per context

struct hdr_ctx {
  int W = 0, H = 0;
  int device = 0;               // the CUDA device the workspace lives on
  int64_t P = 0;
  cudaStream_t stream = nullptr;
  // raster
  float* lum_ref = nullptr;
  uint8_t* q_src = nullptr;
  float* eq_src = nullptr;
  float* pyr = nullptr;         // levels 1.. of both pyramids
  uint32_t* hist = nullptr;     // [ref, src, warped, scratch] x 256
  float* lut = nullptr;         // [src, warped, scratch] x 256
  double* ctab = nullptr;       // lattice SAT pass-1 rows, all levels
  double* ltab = nullptr;       // lattice SAT, all levels
  int64_t ctab_cap = 0, ltab_cap = 0;
  std::map<std::string, int32_t*> lattice_maps;  // device rowmap|colmap|rowlist
  TileCorner* tiles = nullptr;  // all levels
  int64_t tiles_cap = 0;
  // matching
  MatchRow* slot_rows = nullptr;
  uint8_t* slot_flags = nullptr;
  MatchRow* raw = nullptr;
  MatchRow* weeded = nullptr;
  int64_t rows_cap = 0;
  int32_t* counters = nullptr;  // 0 raw, 1 weeded, 2 splat status, 3 grey, 4 fit status
  uint32_t* mask = nullptr;
  int32_t* witness = nullptr;
  int64_t* kept = nullptr;
  double* hpred = nullptr;      // 9 + 9 scratch
  // Philox keys + RANSAC fit scratch per (seed, iterations, coarse_iterations)
  // and Gaussian taps per (window, sigma): every parameter set owns its own
  // buffers, so a captured graph always replays against the contents it was
  // captured with (evicting a set destroys the graphs first)
  std::map<std::tuple<uint64_t, int, int>, KeySet> keysets;
  KeySet* keyset = nullptr;     // the current call's
  std::map<std::pair<int, double>, double*> tapsets;
  // densify
  void* planes = nullptr;       // pu, pv, n: f64 planes (24 B per pixel)
  double* carry = nullptr;      // domain-transform aggregates / carries / coefficients
  uint64_t* splat_key = nullptr;
  int32_t* splat_idx = nullptr;
  int32_t* splat_rows = nullptr;    // row counts (H + 1) then row starts (H + 1)
  SparseEntry* splat_entries = nullptr;
  uint8_t* qw = nullptr;
  // merge
  float* wr = nullptr;
  float* ws = nullptr;
  float* fpyr = nullptr;
  int64_t fpyr_cap = 0;
  double* taps = nullptr;       // the current call's 31 taps (owned by tapsets)
  int32_t* info_scratch = nullptr;
  int32_t* stats_q = nullptr;   // exactness certificate per level (K4)
  double* stats_s = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t probes[2 * HDR_NUM_STAGES] = {};
  bool probing = false;
  KProbe kprobes[HDR_NUM_KPROBES] = {};
  float* frames = nullptr;      // decoded ref + src RGB frames of the raw-sample path (lazy)
  float* fstack = nullptr;      // k-way fusion: pyramid (4 NF + 3 ch / level) + NF weights (lazy)
  int64_t fstack_cap = 0;
  int32_t graph_kernels = 0;
  std::map<std::string, GraphEntry> graphs;
  uint64_t graph_clock = 0;
  std::vector<void*> allocs;
};

// Every entry point runs on its context's device (the caller's current device
// may differ: lazy allocations and launches would otherwise land on the wrong
// GPU), restoring the caller's device on return.
struct CtxDevice {
  int prev = -1;
  explicit CtxDevice(const hdr_ctx* c) {
    if (!c) return;
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; return; }
    if (prev != c->device) cudaSetDevice(c->device);
    else prev = -1;
  }
  ~CtxDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
static cudaError_t ctx_alloc(hdr_ctx* c, T** p, size_t count) {
  size_t bytes = std::max<size_t>(count * sizeof(T), 256);
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e == cudaSuccess) {
    c->allocs.push_back(q);
    *p = reinterpret_cast<T*>(q);
  }
  return e;
}

extern "C" int32_t hdr_max_matches(int32_t width, int32_t height, int32_t tile) {
  return ntiles_of(width, height, std::max(16, tile));
}

extern "C" int hdr_ctx_destroy(hdr_ctx* c) {
  CtxDevice dg_(c);
  if (!c) return HDR_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& kv : c->keysets) {
    cudaFree(kv.second.keys);
  }
  for (auto& kv : c->tapsets) cudaFree(kv.second);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->frames) cudaFree(c->frames);
  if (c->fstack) cudaFree(c->fstack);
  delete c;
  return HDR_OK;
}

static void init_kernel_attributes();

extern "C" int hdr_ctx_create(int32_t width, int32_t height, void* stream, hdr_ctx** out) {
  if (!out || width < 1 || height < 1) return fail(HDR_ERR_INVALID, "bad context size");
  static std::once_flag once;
  std::call_once(once, init_kernel_attributes);
  hdr_ctx* c = new hdr_ctx();
  if (cudaGetDevice(&c->device) != cudaSuccess) {
    delete c;
    return fail(HDR_ERR_CUDA, "no current CUDA device");
  }
  c->W = width;
  c->H = height;
  c->P = (int64_t)width * height;
  c->stream = (cudaStream_t)stream;
  int64_t P = c->P;
  Dims d[kMaxLevels];
  int64_t pyr_sum = 0;
  {
    int w = width, h = height;
    for (int l = 1; l < kMaxLevels; ++l) { w /= 2; h /= 2; pyr_sum += (int64_t)w * h + 64; }
  }
  (void)d;
  int64_t tiles_total = 0;
  {
    int w = width, h = height;
    for (int l = 0; l < kMaxLevels; ++l) { tiles_total += ntiles_of(std::max(w, 1), std::max(h, 1), 16); w /= 2; h /= 2; }
  }
  c->tiles_cap = tiles_total;
  c->rows_cap = ntiles_of(width, height, 16) + 32;
  std::vector<Dims> fd;
  fusion_dims(width, height, 64, fd);
  int64_t fsum = fusion_floats(fd, 2);
  c->fpyr_cap = fsum;
  cudaError_t e = cudaSuccess;
#define ALLOC(ptr, n) \
  if (e == cudaSuccess) e = ctx_alloc(c, &c->ptr, (size_t)(n))
  ALLOC(lum_ref, P);
  ALLOC(q_src, P + 16);
  ALLOC(eq_src, P);
  ALLOC(pyr, 2 * pyr_sum);
  ALLOC(hist, 4 * kBins);
  ALLOC(lut, 3 * kBins);
  {
    int64_t cs = 0, ls = 0;
    int w = width, h = height;
    for (int l = 0; l < kMaxLevels && w >= 1 && h >= 1; ++l) {
      cs += (int64_t)(h + 1) * w + 64;
      ls += (int64_t)(h + 1) * (w + 1) + 64;
      w /= 2;
      h /= 2;
    }
    c->ctab_cap = cs;
    c->ltab_cap = ls;
  }
  ALLOC(ctab, c->ctab_cap);
  ALLOC(ltab, c->ltab_cap);
  ALLOC(tiles, tiles_total);
  ALLOC(slot_rows, c->rows_cap);
  ALLOC(slot_flags, c->rows_cap);
  ALLOC(raw, c->rows_cap);
  ALLOC(weeded, c->rows_cap);
  ALLOC(counters, 16);
  ALLOC(mask, c->rows_cap / 32 + 2);
  ALLOC(witness, c->rows_cap + 1);
  ALLOC(kept, c->rows_cap);
  ALLOC(hpred, 32);
  if (e == cudaSuccess) e = ctx_alloc(c, reinterpret_cast<double**>(&c->planes), 3 * P + 64);
  ALLOC(carry, dt_scratch_doubles(width, height, 3));
  ALLOC(splat_key, P);
  ALLOC(splat_idx, P);
  ALLOC(splat_rows, 2 * ((int64_t)height + 1) + 8);
  ALLOC(splat_entries, c->rows_cap);
  ALLOC(qw, P + 16);
  ALLOC(wr, P);
  ALLOC(ws, P);
  ALLOC(fpyr, fsum + 64);
  ALLOC(info_scratch, HDR_INFO_WORDS);
  ALLOC(stats_q, 8);
  ALLOC(stats_s, 8);
#undef ALLOC
  if (e != cudaSuccess) {
    hdr_ctx_destroy(c);
    return fail(HDR_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return HDR_OK;
}

extern "C" int hdr_ctx_set_stream(hdr_ctx* c, void* stream) {
  CtxDevice dg_(c);
  if (!c) return fail(HDR_ERR_INVALID, "null context");
  c->stream = (cudaStream_t)stream;
  return HDR_OK;
}

extern "C" int hdr_ctx_set_probes(hdr_ctx* c, void* const* events) {
  CtxDevice dg_(c);
  if (!c) return fail(HDR_ERR_INVALID, "null context");
  c->probing = events != nullptr;
  for (int i = 0; i < 2 * HDR_NUM_STAGES; ++i)
    c->probes[i] = events ? (cudaEvent_t)events[i] : nullptr;
  return HDR_OK;
}

extern "C" int32_t hdr_ctx_graph_kernels(hdr_ctx* c) {
  CtxDevice dg_(c); return c ? c->graph_kernels : -1; }

extern "C" int hdr_ctx_set_kernel_probes(hdr_ctx* c, int32_t kernel, void* const* events,
                                         int32_t n) {
  CtxDevice dg_(c);
  if (!c) return fail(HDR_ERR_INVALID, "null context");
  if (kernel < 0 || kernel >= HDR_NUM_KPROBES) return fail(HDR_ERR_INVALID, "unknown kernel probe");
  if (n < 0 || n > kMaxKProbeLaunches || (n > 0 && !events))
    return fail(HDR_ERR_INVALID, "kernel probes: 0 <= n <= 8 launches");
  KProbe& k = c->kprobes[kernel];
  k = KProbe{};
  k.n = events ? n : 0;
  for (int i = 0; i < 2 * k.n; ++i) k.ev[i] = (cudaEvent_t)events[i];
  return HDR_OK;
}

namespace hdr {
void kprobe_mark(KProbe* p, int end, cudaStream_t s) {
  if (!p || p->next >= p->n) return;
  cudaEvent_t e = p->ev[2 * p->next + end];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
  if (end) ++p->next;
}
}  // namespace hdr

// Stage boundaries of the pair: an NVTX range per stage on the host timeline
// (nsys / ncu NVTX filtering; free when no tool is attached) and, with probes
// set, CUDA events recorded on the stream (hdr_ctx_set_probes).
static const char* const kStageNames[7] = {"hdr:raster", "hdr:corners", "hdr:match_chain", "hdr:dt_filter",
                                           "hdr:finalize_warp", "hdr:ssim", "hdr:fuse"};
static void probe(hdr_ctx* c, int stage, int end) {
  if (end) nvtxRangePop();
  else nvtxRangePushA(kStageNames[stage]);
  if (!c->probing) return;
  cudaEvent_t e = c->probes[2 * stage + end];
  if (!e) return;
  // while capturing, External makes it a real event-record node (replays
  // time it); outside capture the flag is not accepted
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
  else
    cudaEventRecord(e, c->stream);
}

extern "C" int hdr_ctx_sync(hdr_ctx* c) {
  CtxDevice dg_(c);
  if (!c) return fail(HDR_ERR_INVALID, "null context");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaGetLastError());
  return HDR_OK;
}

static void drop_graphs(hdr_ctx* c) {
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);  // in-flight launches finish first
  c->graphs.clear();
}

// Parameter-set caches are bounded; evicting one frees buffers that cached
// graphs (and queued work) may reference, so both go first.
template <class Map, class Free>
static int evict_if_full(hdr_ctx* c, Map& m, Free free_fn) {
  if (m.size() < kMaxParamSets) return HDR_OK;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  drop_graphs(c);
  for (auto& kv : m) free_fn(kv.second);
  m.clear();
  return HDR_OK;
}

// Philox keys for every level (weeding._iteration_rng, weeding.py:62-66,
// seeded per level by matcher.level_seed, matcher.py:146-149) and the RANSAC
// fit scratch, one set per (seed, iterations, coarse_iterations).
static int ensure_keys(hdr_ctx* c, const hdr_params* p) {
  auto key = std::make_tuple(p->seed, p->iterations, p->coarse_iterations);
  auto it = c->keysets.find(key);
  if (it != c->keysets.end()) {
    c->keyset = &it->second;
    return HDR_OK;
  }
  int rc = evict_if_full(c, c->keysets, [](KeySet& k) { cudaFree(k.keys); });
  if (rc) return rc;
  KeySet ks;
  ks.iters = std::max(p->iterations, p->coarse_iterations);
  CUDA_TRY(cudaMalloc(&ks.keys, sizeof(uint64_t) * 2 * (size_t)ks.iters * kMaxLevels));
  std::vector<uint64_t> host(2 * (size_t)ks.iters * kMaxLevels, 0);
  for (int l = 0; l < kMaxLevels; ++l) {
    int n = l == 0 ? p->iterations : p->coarse_iterations;
    hdr_iteration_keys(hdr_level_seed(p->seed, l), n, host.data() + 2 * (size_t)ks.iters * l);
  }
  // a fresh buffer no queued work reads: a plain blocking upload suffices
  cudaError_t e = cudaMemcpy(ks.keys, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(ks.keys);
    return fail(HDR_ERR_CUDA, std::string("key upload: ") + cudaGetErrorString(e));
  }
  c->keyset = &(c->keysets[key] = ks);
  return HDR_OK;
}

// fusion._gaussian_kernel (fusion.py:28-31), one tap set per (window, sigma)
static int ensure_taps(hdr_ctx* c, int window, double sigma) {
  int r = window / 2;
  if (r > 15) return fail(HDR_ERR_INVALID, "ssim_window above 31 is not supported");
  auto key = std::make_pair(window, sigma);
  auto it = c->tapsets.find(key);
  if (it != c->tapsets.end()) {
    c->taps = it->second;
    return HDR_OK;
  }
  int rc = evict_if_full(c, c->tapsets, [](double* t) { cudaFree(t); });
  if (rc) return rc;
  double k[31], sum = 0.0;
  for (int i = -r; i <= r; ++i) {
    double x = (double)i / sigma;
    k[i + r] = exp(-0.5 * (x * x));
  }
  for (int i = 0; i < 2 * r + 1; ++i) sum += k[i];
  for (int i = 0; i < 2 * r + 1; ++i) k[i] /= sum;
  double* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(double) * 32));
  cudaError_t e = cudaMemcpy(d, k, sizeof(double) * (2 * r + 1), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return fail(HDR_ERR_CUDA, std::string("taps upload: ") + cudaGetErrorString(e));
  }
  c->tapsets[key] = d;
  c->taps = d;
  return HDR_OK;
}

static float* pyr_level(hdr_ctx* c, const Dims* d, int l, int which) {
  // levels 1.. of [ref, src], packed after each other
  float* base = c->pyr;
  for (int k = 1; k < l; ++k) base += 2 * ((int64_t)d[k].w * d[k].h + 64);
  return base + which * ((int64_t)d[l].w * d[l].h + 64);
}

// Table rows/columns the detector reads (matcher.py:75-87): {g-half, g, g+half}
// for every candidate coordinate g that passes the fit test; `full` keeps all.
static void lattice_axis(int n, int tile, int half, bool full, std::vector<char>& need) {
  need.assign(n + 1, full ? 1 : 0);
  if (full) return;
  int sp = std::max(1, tile / 16), first = sp / 2;
  for (int t0 = 0; t0 < n; t0 += tile) {
    int lim = std::min(tile, n - t0);
    for (int o = first; o < lim; o += sp) {
      int g = t0 + o;
      if (g >= half && g <= n - half) need[g - half] = need[g] = need[g + half] = 1;
    }
  }
}

struct LatticeInfo {
  const int32_t* rowmap;
  const int32_t* colmap;
  const int32_t* rowlist;
  int nrows, ncols;
};

// Device maps for one level, built on the host once per (w, h, tile, half).
static int lattice_maps(hdr_ctx* c, int w, int h, int tile, int half, bool full, LatticeInfo* out) {
  char key[96];
  snprintf(key, sizeof key, "%d,%d,%d,%d,%d", w, h, tile, half, (int)full);
  std::vector<char> rn, cn;
  lattice_axis(h, tile, half, full, rn);
  lattice_axis(w, tile, half, full, cn);
  std::vector<int32_t> rowmap(h + 1, -1), colmap(w + 1, -1), rowlist;
  int nc = 0;
  for (int X = 0; X <= w; ++X)
    if (cn[X]) colmap[X] = nc++;
  for (int Y = 0; Y <= h; ++Y)
    if (rn[Y]) {
      rowmap[Y] = (int)rowlist.size();
      rowlist.push_back(Y);
    }
  int nr = (int)rowlist.size();
  auto it = c->lattice_maps.find(key);
  int32_t* dev;
  if (it != c->lattice_maps.end()) {
    dev = it->second;
  } else {
    std::vector<int32_t> host;
    host.insert(host.end(), rowmap.begin(), rowmap.end());
    host.insert(host.end(), colmap.begin(), colmap.end());
    host.insert(host.end(), rowlist.begin(), rowlist.end());
    host.push_back(0);
    CUDA_TRY(cudaMalloc(&dev, host.size() * sizeof(int32_t)));
    c->allocs.push_back(dev);
    CUDA_TRY(cudaMemcpy(dev, host.data(), host.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    c->lattice_maps[key] = dev;
  }
  out->rowmap = dev;
  out->colmap = dev + (h + 1);
  out->rowlist = dev + (h + 1) + (w + 1);
  out->nrows = nr;
  out->ncols = nc;
  return HDR_OK;
}

// Fill a SatBatch for n levels of images (lum[l], dims d[l]) carving ctab /
// ltab from the context; tiles[l] receive the detector output.
static int sat_batch(hdr_ctx* c, int n, const float* const* lum, const Dims* d, int tile,
                     int half, bool full, TileCorner* const* tiles, double* ltab_override,
                     SatBatch* b, int* max_w, int* max_rows, int* total_tiles) {
  b->n = n;
  b->qmin = full ? nullptr : c->stats_q;  // full tables always take numpy's order
  b->sums = full ? nullptr : c->stats_s;
  int64_t co = 0, lo = 0;
  *max_w = *max_rows = *total_tiles = 0;
  for (int l = 0; l < n; ++l) {
    LatticeInfo li;
    int rc = lattice_maps(c, d[l].w, d[l].h, tile, half, full, &li);
    if (rc) return rc;
    SatLevel& L = b->lv[l];
    L.img = lum[l];
    L.w = d[l].w;
    L.h = d[l].h;
    L.rowmap = li.rowmap;
    L.colmap = li.colmap;
    L.rowlist = li.rowlist;
    L.nrows = li.nrows;
    L.ncols = li.ncols;
    L.ctab = c->ctab + co;
    L.ltab = ltab_override ? ltab_override : c->ltab + lo;
    co += (int64_t)li.nrows * d[l].w + 64;
    lo += (int64_t)li.nrows * li.ncols + 64;
    if (co > c->ctab_cap || (!ltab_override && lo > c->ltab_cap))
      return fail(HDR_ERR_INVALID, "image larger than the lattice workspace");
    L.tiles = tiles ? tiles[l] : nullptr;
    L.tile_base = *total_tiles;
    *total_tiles += ntiles_of(d[l].w, d[l].h, tile);
    *max_w = std::max(*max_w, d[l].w);
    *max_rows = std::max(*max_rows, li.nrows);
  }
  return HDR_OK;
}

static DetectParams detect_params(int tile, int half, double threshold) {
  DetectParams dp{tile, half, threshold, 0};
  dp.exact_ok = detect_exact_smem(tile, half) <= 200 * 1024;
  return dp;
}

static TileCorner* tiles_level(hdr_ctx* c, const Dims* d, int l, int tile) {
  TileCorner* t = c->tiles;
  for (int k = 0; k < l; ++k) t += ntiles_of(d[k].w, d[k].h, tile);
  return t;
}

static DtPlanes f64_planes(double* a, double* b, double* n, int k) {
  DtPlanes pl;
  pl.p[0] = a; pl.p[1] = b; pl.p[2] = n;
  pl.f64[0] = pl.f64[1] = pl.f64[2] = 1;
  pl.k = k;
  return pl;
}

// The pair path's planes are all f64: with f32 flow numerators the flow moves
// by ~1e-6 px, which flips warp_image's validity test on pixels whose sample
// lands exactly on the frame edge (integer shifts) and the fusion spreads each
// flip over ~70 composite pixels. f64 keeps the flow within
// ~1e-13 of the reference before its f32 cast.
static DtPlanes pair_planes(hdr_ctx* c, int64_t P) {
  double* d = reinterpret_cast<double*>(c->planes);
  return f64_planes(d, d + P, d + 2 * P, 3);
}

// ------------------------------------------------------------ kernels used by the pipeline only
// The pair's first kernel: info words, and the per-pair accumulators
// (histograms, counters, the exactness certificate's per-level min/sum)
// cleared here rather than by memset nodes, which would break the
// programmatic launch chain.
__global__ void info_init_kernel(int32_t* info, int levels, uint32_t* hist, int32_t* counters,
                                 int32_t* stats_q, double* stats_s, double* hpred) {
  pdl_wait();
  int i = threadIdx.x;
  if (i < HDR_INFO_WORDS) info[i] = (i == 2) ? levels : 0;
  if (i < 9) hpred[i] = (i % 4 == 0) ? 1.0 : 0.0;  // the coarsest level predicts with identity
  for (int j = i; j < 4 * kBins; j += blockDim.x) hist[j] = 0u;
  if (i < 16) counters[i] = 0;
  if (i < 5) {
    stats_q[i] = 0x3f3f3f3f;  // large positive: atomicMin identity
    stats_s[i] = 0.0;
  }
}

// the registration verdict (pipeline.py:185-187) and the grey-zone count
__global__ void status_kernel(const int32_t* weeded_count, int32_t* info, const int32_t* grey) {
  pdl_wait();
  if (threadIdx.x == 0) {
    info[0] = (*weeded_count >= 4) ? HDR_OK : HDR_ERR_REGISTRATION;
    info[18] = *grey;
  }
}

static int check_ptr_align(const void* p, size_t a, const char* what) {
  if (((uintptr_t)p) % a) return fail(HDR_ERR_INVALID, std::string(what) + " must be 16-byte aligned");
  return HDR_OK;
}

// The whole matching chain (pipeline.match_stack, pipeline.py:122-130) on
// device-resident RGB inputs. info words as documented in hdrb200.h.
static int enqueue_match(hdr_ctx* c, const hdr_params* p, int w, int h, const float* ref,
                         const float* src, double* out_matches, double* out_raw,
                         double* out_h, int32_t* info) {
  cudaStream_t s = c->stream;
  int64_t P = (int64_t)w * h;
  Dims d[kMaxLevels];
  int L = pyramid_dims(w, h, p->max_levels, d);
  probe(c, 0, 0);
  klaunch(info_init_kernel, 1, 256, 0, s, info, L, c->hist, c->counters, c->stats_q, c->stats_s, c->hpred);
  launch_luma_hist(ref, P, c->lum_ref, nullptr, c->hist, s);
  launch_luma_hist(src, P, nullptr, c->q_src, c->hist + kBins, s);
  launch_lut(c->hist + kBins, P, c->hist, P, c->lut, s);
  launch_apply_lut_q(c->q_src, P, c->lut, c->eq_src, s);
  const float* lref[kMaxLevels];
  const float* lsrc[kMaxLevels];
  lref[0] = c->lum_ref;
  lsrc[0] = c->eq_src;
  for (int l = 1; l < L; ++l) {
    float* a = pyr_level(c, d, l, 0);
    float* b = pyr_level(c, d, l, 1);
    launch_downsample2(lref[l - 1], lsrc[l - 1], d[l - 1].w, d[l - 1].h, a, b, s);
    lref[l] = a;
    lsrc[l] = b;
  }
  probe(c, 0, 1);
  probe(c, 1, 0);
  {
    SatBatch sb;
    TileCorner* tl[kMaxLevels];
    for (int l = 0; l < L; ++l) tl[l] = tiles_level(c, d, l, p->tile);
    int mw, mr, nt;
    int rc = sat_batch(c, L, lref, d, p->tile, p->quadrant_half, false, tl, nullptr, &sb, &mw, &mr, &nt);
    if (rc) return rc;
    int maxpx = d[0].w * d[0].h;
    launch_level_stats(sb, maxpx, s, true);
    launch_sat(sb, mw, mr, s);
    launch_detect(sb, nt, detect_params(p->tile, p->quadrant_half, p->threshold), s);
  }
  probe(c, 1, 1);
  probe(c, 2, 0);
  int32_t* raw_count = c->counters + 0;
  int32_t* weeded_count = c->counters + 1;
  int32_t* grey = c->counters + 3;
  for (int l = L - 1; l >= 0; --l) {
    int nt = ntiles_of(d[l].w, d[l].h, p->tile);
    launch_ssd_tiles(tiles_level(c, d, l, p->tile), nt, lref[l], lsrc[l], d[l].w, d[l].h,
                     c->hpred, p->radius, p->patch, c->slot_rows, c->slot_flags, s);
    launch_compact_rows(c->slot_rows, c->slot_flags, nt, c->raw, raw_count,
                        l == 0 ? out_raw : nullptr, s, c->mask, c->witness);
    int iters = l == 0 ? p->iterations : p->coarse_iterations;
    double eps = 2.0 * p->eps_px / (double)d[l].w;  // MatcherParams.weed_params
    launch_weed(c->raw, raw_count, nt, d[l].w, d[l].h, iters, eps,
                c->keyset->keys + 2 * (size_t)c->keyset->iters * l, p->delta, c->mask, c->witness, grey, s,
                true);
    launch_finish_level(c->raw, raw_count, c->mask, d[l].w, d[l].h, l, c->weeded, weeded_count,
                        nullptr, c->hpred, out_h, info, l == 0 ? out_matches : nullptr, nullptr,
                        grey, s);
  }
  klaunch(status_kernel, 1, 32, 0, s, weeded_count, info, (const int32_t*)grey);
  probe(c, 2, 1);
  return check_launch();
}

// fusion.fuse (fusion.py:135-157) for nf frames from `base` (pyramid) and
// `wout` (nf level-0 weight planes)
static int enqueue_fuse_frames(hdr_ctx* c, int nf, const FuseFrameSet& fs, int w, int h, int levels,
                               float* base, float* out) {
  if (levels <= 0) levels = fusion_levels_default(w, h);
  std::vector<Dims> fd;
  fusion_dims(w, h, levels, fd);
  FusePyramid py{};
  fusion_layout(fd, nf, base, py);
  py.out = out;
  launch_fuse(nf, fs, py, c->stream, &c->kprobes[HDR_KP_FUSE_WEIGHTS0],
              &c->kprobes[HDR_KP_FUSE_COLLAPSE0]);
  return check_launch();
}

static int enqueue_fuse(hdr_ctx* c, const float* ref, const float* warped, const float* ssim,
                        const uint8_t* valid, int w, int h, int levels, float* out) {
  FuseFrameSet fs{};
  fs.img[0] = ref;
  fs.img[1] = warped;
  fs.ssim[1] = ssim;
  fs.valid[1] = valid;
  fs.wout[0] = c->wr;
  fs.wout[1] = c->ws;
  return enqueue_fuse_frames(c, 2, fs, w, h, levels, c->fpyr, out);
}

static int enqueue_pair(hdr_ctx* c, const hdr_params* p, int w, int h, const float* ref,
                        const float* src, const hdr_outputs* o, bool fuse = true) {
  cudaStream_t s = c->stream;
  for (KProbe& k : c->kprobes) k.next = 0;
  int64_t P = (int64_t)w * h;
  int rc = enqueue_match(c, p, w, h, ref, src, o->matches, o->raw_matches, o->homography, o->info);
  if (rc) return rc;
  int32_t* weeded_count = c->counters + 1;
  // make_flow (pipeline.py:153-162): splat, filter, ratio + H fallback
  probe(c, 3, 0);
  DtPlanes pl = pair_planes(c, P);
  // the last column pass finishes densify_flow in registers and writes the
  // f32 flow directly (the smoothed planes never make a final round trip)
  DtFlowOut fo{o->homography, o->info + 1, p->normalization_floor, o->flow};
  DtSparse sp{c->splat_rows + (h + 1), c->splat_entries};
  const bool sparse_first = g_sparse_first && dt_sparse_first_ok(c->lum_ref, pl, w);
  if (sparse_first)  // the first row pass builds its rows from the CSR splat
    launch_splat_rows(o->matches, weeded_count, 0, w, h, c->splat_key, c->splat_idx, c->splat_rows,
                      c->splat_rows + (h + 1), c->splat_entries, c->counters + 2, s);
  else
    launch_splat(o->matches, weeded_count, 0, w, h, pl, c->splat_key, c->splat_idx, c->counters + 2, s);
  bool flow_done = launch_dt_filter(c->lum_ref, pl, w, h, p->sigma_s, p->sigma_r, p->passes,
                                    c->carry, s, &fo, &c->kprobes[HDR_KP_DT_ROWS],
                                    &c->kprobes[HDR_KP_DT_COLS], sparse_first ? &sp : nullptr);
  probe(c, 3, 1);
  probe(c, 4, 0);
  // warp_image + luminance(warped) histogram (pipeline.py:192, :168)
  kprobe_mark(&c->kprobes[HDR_KP_WARP], 0, s);
  if (flow_done)
    launch_warp(o->flow, w, h, src, o->warped, o->valid, c->qw, c->hist + 2 * kBins, s);
  else
    launch_finalize_warp(pl, o->homography, o->info + 1, w, h, p->normalization_floor, src, 3,
                         o->flow, o->warped, o->valid, c->qw, c->hist + 2 * kBins, true, s);
  kprobe_mark(&c->kprobes[HDR_KP_WARP], 1, s);
  probe(c, 4, 1);
  probe(c, 5, 0);
  // make_ssim (pipeline.py:165-171)
  launch_lut(c->hist + 2 * kBins, P, c->hist, P, c->lut + kBins, s);
  kprobe_mark(&c->kprobes[HDR_KP_SSIM], 0, s);
  launch_ssim(c->lum_ref, nullptr, c->qw, c->lut + kBins, w, h, p->ssim_window, c->taps, o->ssim, s);
  kprobe_mark(&c->kprobes[HDR_KP_SSIM], 1, s);
  probe(c, 5, 1);
  if (!fuse) return check_launch();
  probe(c, 6, 0);
  // fusion.fuse (pipeline.py:193)
  rc = enqueue_fuse(c, ref, o->warped, o->ssim, o->valid, w, h, 0, o->composite);
  probe(c, 6, 1);
  return rc;
}

// lattice maps are uploaded with a blocking copy: build them before any capture
static int ensure_lattice(hdr_ctx* c, const hdr_params* p, int w, int h) {
  Dims d[kMaxLevels];
  int L = pyramid_dims(w, h, p->max_levels, d);
  for (int l = 0; l < L; ++l) {
    LatticeInfo li;
    int rc = lattice_maps(c, d[l].w, d[l].h, p->tile, p->quadrant_half, false, &li);
    if (rc) return rc;
  }
  return HDR_OK;
}

static int check_pair_args(hdr_ctx* c, const hdr_params* p, int w, int h, const float* ref,
                           const float* src, const hdr_outputs* o, bool need_composite = true) {
  if (!c || !p || !o) return fail(HDR_ERR_INVALID, "null argument");
  char msg[128];
  int rc = hdr_params_validate(p, msg, sizeof msg);
  if (rc) return rc;
  if (w > c->W || h > c->H || w < 1 || h < 1)
    return fail(HDR_ERR_INVALID, "image larger than the context workspace");
  if (std::min(w, h) < 100) return fail(HDR_ERR_INVALID, "input below 100 pixels in one dimension");
  if (ntiles_of(w, h, p->tile) > c->rows_cap) return fail(HDR_ERR_INVALID, "too many tiles");
  size_t side = 2 * (size_t)p->radius + p->patch;
  if ((side * side + (size_t)p->patch * p->patch) * 8 > 200 * 1024)
    return fail(HDR_ERR_INVALID, "radius/patch search window exceeds shared memory");
  if (!ref || !src || (need_composite && !o->composite) || !o->flow || !o->warped || !o->valid || !o->ssim ||
      !o->matches || !o->raw_matches || !o->homography || !o->info)
    return fail(HDR_ERR_INVALID, "null buffer");
  rc = check_ptr_align(ref, 16, "ref");
  if (!rc) rc = check_ptr_align(src, 16, "src");
  if (rc) return rc;
  rc = ensure_keys(c, p);
  if (!rc) rc = ensure_taps(c, p->ssim_window, p->ssim_sigma);
  if (!rc) rc = ensure_lattice(c, p, w, h);
  return rc;
}

extern "C" int hdr_register_and_fuse(hdr_ctx* c, const hdr_params* p, int32_t w, int32_t h,
                                     const float* ref, const float* src, const hdr_outputs* o) {
  CtxDevice dg_(c);
  int rc = check_pair_args(c, p, w, h, ref, src, o);
  if (rc) return rc;
  return enqueue_pair(c, p, w, h, ref, src, o);
}

#define NEED(cond, msg) \
  if (!(cond)) return fail(HDR_ERR_INVALID, msg)

// ------------------------------------------------------------ file path
static int check_raw(int channels, int bits) {
  if (channels != 1 && channels != 3) return fail(HDR_ERR_INVALID, "channels must be 1 or 3");
  if (bits != 8 && bits != 16) return fail(HDR_ERR_INVALID, "bits must be 8 or 16");
  return HDR_OK;
}

extern "C" int hdr_decode_image(hdr_ctx* c, const void* raw, int32_t w, int32_t h,
                                int32_t channels, int32_t bits, float* rgb) {
  CtxDevice dg_(c);
  NEED(c && raw && rgb, "null argument");
  int rc = check_raw(channels, bits);
  if (rc) return rc;
  launch_decode(raw, (int64_t)w * h, channels, bits, rgb, c->stream);
  return check_launch();
}

extern "C" int hdr_encode_u8(hdr_ctx* c, const float* img, int64_t n, uint8_t* out) {
  CtxDevice dg_(c);
  NEED(c && img && out, "null argument");
  launch_encode_u8(img, n, out, c->stream);
  return check_launch();
}

extern "C" int hdr_dark_count(hdr_ctx* c, const float* img, int32_t channels, int64_t n,
                              float dark_level, uint64_t* out) {
  CtxDevice dg_(c);
  NEED(c && img && out, "null argument");
  NEED(channels >= 1, "channels must be >= 1");
  launch_dark_count(img, channels, n, dark_level, reinterpret_cast<unsigned long long*>(out),
                    c->stream);
  return check_launch();
}

extern "C" int hdr_mean_luminance(hdr_ctx* c, const float* img, int32_t channels, int64_t n,
                                  double* out) {
  CtxDevice dg_(c);
  NEED(c && img && out, "null argument");
  NEED(channels >= 1, "channels must be >= 1");
  launch_mean_luminance(img, channels, n, out, c->stream);
  return check_launch();
}

extern "C" int hdr_register_and_fuse_graph(hdr_ctx* c, const hdr_params* p, int32_t w, int32_t h,
                                           const float* ref, const float* src,
                                           const hdr_outputs* o);

extern "C" int hdr_register_and_fuse_raw(hdr_ctx* c, const hdr_params* p, int32_t w, int32_t h,
                                         const void* ref_raw, const void* src_raw,
                                         int32_t channels, int32_t bits, int32_t use_graph,
                                         const hdr_outputs* o, uint8_t* composite_u8) {
  CtxDevice dg_(c);
  NEED(c && ref_raw && src_raw, "null argument");
  int rc = check_raw(channels, bits);
  if (rc) return rc;
  if (w > c->W || h > c->H || w < 1 || h < 1)
    return fail(HDR_ERR_INVALID, "image larger than the context workspace");
  if (!c->frames) CUDA_TRY(cudaMalloc(&c->frames, 2 * 3 * (size_t)c->P * sizeof(float)));
  int64_t P = (int64_t)w * h;
  float* ref = c->frames;
  float* src = c->frames + 3 * (size_t)c->P;
  launch_decode(ref_raw, P, channels, bits, ref, c->stream);
  launch_decode(src_raw, P, channels, bits, src, c->stream);
  rc = use_graph ? hdr_register_and_fuse_graph(c, p, w, h, ref, src, o)
                 : hdr_register_and_fuse(c, p, w, h, ref, src, o);
  if (rc) return rc;
  if (composite_u8) launch_encode_u8(o->composite, 3 * P, composite_u8, c->stream);
  return check_launch();
}

extern "C" int hdr_register_and_fuse_graph(hdr_ctx* c, const hdr_params* p, int32_t w, int32_t h,
                                           const float* ref, const float* src,
                                           const hdr_outputs* o) {
  CtxDevice dg_(c);
  int rc = check_pair_args(c, p, w, h, ref, src, o);
  if (rc) return rc;
  char key[768];
  int kn = snprintf(key, sizeof key, "%d,%d,%p,%p,%p,%p,%p,%p,%p,%p,%p,%p,%p|%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%a,%a,%a,%a,%a,%a,%llu",
           w, h, (const void*)ref, (const void*)src, (void*)o->composite, (void*)o->flow,
           (void*)o->warped, (void*)o->valid, (void*)o->ssim, (void*)o->matches,
           (void*)o->raw_matches, (void*)o->homography, (void*)o->info, p->tile, p->quadrant_half,
           p->radius, p->patch, p->max_levels, p->iterations, p->coarse_iterations, p->delta,
           p->passes, p->ssim_window, p->threshold, p->eps_px, p->sigma_s, p->sigma_r,
           p->ssim_sigma, p->normalization_floor, (unsigned long long)p->seed);
  std::string kkey(key, kn > 0 ? std::min(kn, (int)sizeof key - 1) : 0);
  char pk[32];
  if (c->probing)
    for (int i = 0; i < 2 * HDR_NUM_STAGES; ++i) {
      snprintf(pk, sizeof pk, ",%p", (void*)c->probes[i]);
      kkey += pk;
    }
  for (const KProbe& k : c->kprobes)
    for (int i = 0; i < 2 * k.n; ++i) {
      snprintf(pk, sizeof pk, ";%p", (void*)k.ev[i]);
      kkey += pk;
    }
  if (c->graphs.size() >= kMaxGraphs && !c->graphs.count(kkey)) {
    auto lru = c->graphs.begin();
    for (auto it = c->graphs.begin(); it != c->graphs.end(); ++it)
      if (it->second.used < lru->second.used) lru = it;
    if (lru->second.exec) cudaGraphExecDestroy(lru->second.exec);
    c->graphs.erase(lru);
  }
  GraphEntry& g = c->graphs[kkey];
  g.used = ++c->graph_clock;
  if (!g.exec) {
    // capture on the context's private stream (the caller's may be the
    // legacy default stream, which cannot be captured); replay on theirs
    cudaGraph_t graph = nullptr;
    if (!c->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = c->stream;
    c->stream = c->cap_stream;
    cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      c->stream = user;
      c->graphs.erase(kkey);
      return fail(HDR_ERR_CUDA, std::string("begin capture: ") + cudaGetErrorString(e));
    }
    rc = enqueue_pair(c, p, w, h, ref, src, o);
    e = cudaStreamEndCapture(c->stream, &graph);
    c->stream = user;
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      c->graphs.erase(kkey);
      return rc;
    }
    if (e != cudaSuccess) {
      c->graphs.erase(kkey);
      return fail(HDR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    }
    size_t nodes = 0;
    cudaGraphGetNodes(graph, nullptr, &nodes);
    std::vector<cudaGraphNode_t> list(nodes);
    if (nodes) cudaGraphGetNodes(graph, list.data(), &nodes);
    int32_t kernels = 0;
    for (auto nd : list) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kernels;
    }
    c->graph_kernels = kernels;
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      c->graphs.erase(kkey);
      return fail(HDR_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
  }
  CUDA_TRY(cudaGraphLaunch(g.exec, c->stream));
  return HDR_OK;
}

// ------------------------------------------------------------ per-stage twins
extern "C" int hdr_luminance(hdr_ctx* c, const float* rgb, int64_t n, float* lum) {
  CtxDevice dg_(c);
  NEED(c && rgb && lum, "null argument");
  NEED(n >= 0, "bad size");
  int rc = check_ptr_align(rgb, 16, "rgb");
  if (!rc) rc = check_ptr_align(lum, 16, "lum");
  if (rc) return rc;
  if (n) launch_luminance(rgb, n, lum, c->stream);
  return check_launch();
}

extern "C" int hdr_match_histogram(hdr_ctx* c, const float* src, int64_t n_src, const float* ref,
                                   int64_t n_ref, int32_t stride, float* out) {
  CtxDevice dg_(c);
  NEED(c && src && ref && out, "null argument");
  NEED(n_src > 0 && n_ref > 0 && stride >= 1, "bad size");
  cudaStream_t s = c->stream;
  uint32_t* hs = c->hist + 3 * kBins;
  uint32_t* hr = c->hist + 2 * kBins;
  CUDA_TRY(cudaMemsetAsync(hr, 0, sizeof(uint32_t) * 2 * kBins, s));
  launch_hist_plain(src, n_src, stride, hs, s);
  launch_hist_plain(ref, n_ref, stride, hr, s);
  launch_lut(hs, n_src, hr, n_ref, c->lut + 2 * kBins, s);
  launch_apply_lut_f(src, n_src, stride, c->lut + 2 * kBins, out, s);
  return check_launch();
}

extern "C" int hdr_build_pyramid(hdr_ctx* c, const float* img, int32_t w, int32_t h,
                                 int32_t max_levels, int32_t min_dim, float** out_levels,
                                 int32_t* n_levels) {
  CtxDevice dg_(c);
  NEED(c && img && out_levels && n_levels, "null argument");
  if (std::min(w, h) < min_dim)
    return fail(HDR_ERR_INVALID, "input below " + std::to_string(min_dim) + " pixels in one dimension");
  int L = 1, cw = w, ch = h;
  const float* prev = img;
  while (L < max_levels) {
    int nw = cw / 2, nh = ch / 2;
    if (std::min(nw, nh) < min_dim || std::min(nw, nh) < 1) break;
    NEED(out_levels[L], "missing level buffer");
    launch_downsample2(prev, nullptr, cw, ch, out_levels[L], nullptr, c->stream);
    prev = out_levels[L];
    cw = nw;
    ch = nh;
    ++L;
  }
  *n_levels = L;
  return check_launch();
}

extern "C" int hdr_integral(hdr_ctx* c, const float* img, int32_t w, int32_t h, double* table) {
  CtxDevice dg_(c);
  NEED(c && img && table && w >= 1 && h >= 1, "bad argument");
  NEED(w <= c->W && h <= c->H, "image larger than the workspace");
  SatBatch sb;
  Dims d[1] = {{w, h}};
  const float* lum[1] = {img};
  int mw, mr, nt;
  int rc = sat_batch(c, 1, lum, d, 16, 2, true, nullptr, table, &sb, &mw, &mr, &nt);
  if (rc) return rc;
  launch_sat(sb, mw, mr, c->stream);
  return check_launch();
}

// detect_corners on one level into c->tiles (shared by the per-stage entries)
static int detect_one(hdr_ctx* c, const float* lum, int w, int h, int tile, double threshold,
                      int half) {
  NEED(w <= c->W && h <= c->H, "image larger than the workspace");
  SatBatch sb;
  Dims d[1] = {{w, h}};
  const float* lv[1] = {lum};
  TileCorner* tl[1] = {c->tiles};
  int mw, mr, nt;
  int rc = sat_batch(c, 1, lv, d, tile, half, false, tl, nullptr, &sb, &mw, &mr, &nt);
  if (rc) return rc;
  launch_level_stats(sb, w * h, c->stream);
  launch_sat(sb, mw, mr, c->stream);
  launch_detect(sb, nt, detect_params(tile, half, threshold), c->stream);
  return HDR_OK;
}

extern "C" int hdr_detect_corners(hdr_ctx* c, const float* lum, int32_t w, int32_t h, int32_t tile,
                                  double threshold, int32_t half, double* corners, int32_t* count) {
  CtxDevice dg_(c);
  NEED(c && lum && corners && count, "null argument");
  if (tile < 16) return fail(HDR_ERR_INVALID, "tile must be >= 16");
  NEED((int64_t)(w + 1) * (h + 1) <= (int64_t)(c->W + 1) * (c->H + 1), "image larger than the workspace");
  int nt = ntiles_of(w, h, tile);
  NEED(nt <= c->tiles_cap, "too many tiles");
  cudaStream_t s = c->stream;
  int rc = detect_one(c, lum, w, h, tile, threshold, half);
  if (rc) return rc;
  launch_compact_corners(c->tiles, nt, corners, c->counters + 5, s);
  CUDA_TRY(cudaMemcpyAsync(count, c->counters + 5, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return check_launch();
}

extern "C" int hdr_ssd_match(hdr_ctx* c, const float* ref, const float* src, int32_t w, int32_t h,
                             const int32_t* pts, int32_t n, int32_t radius, int32_t patch,
                             double* out, uint8_t* found) {
  CtxDevice dg_(c);
  NEED(c && ref && src && pts && out && found, "null argument");
  NEED(radius >= 1 && patch >= 3 && patch % 2 == 1, "bad radius/patch");
  size_t side = 2 * (size_t)radius + patch;
  NEED((side * side + (size_t)patch * patch) * 8 <= 200 * 1024, "search window exceeds shared memory");
  launch_ssd_points(ref, src, w, h, pts, n, radius, patch, out, found, c->stream);
  return check_launch();
}

extern "C" int hdr_match_level(hdr_ctx* c, const hdr_params* p, const float* lum_ref,
                               const float* lum_src, int32_t w, int32_t h, const double* h_pred,
                               double* raw, int32_t* count) {
  CtxDevice dg_(c);
  NEED(c && p && lum_ref && lum_src && h_pred && raw && count, "null argument");
  if (p->tile < 16) return fail(HDR_ERR_INVALID, "tile must be >= 16");
  int nt = ntiles_of(w, h, p->tile);
  NEED(nt <= c->rows_cap, "too many tiles");
  NEED((int64_t)(w + 1) * (h + 1) <= (int64_t)(c->W + 1) * (c->H + 1), "image larger than the workspace");
  cudaStream_t s = c->stream;
  int rc = detect_one(c, lum_ref, w, h, p->tile, p->threshold, p->quadrant_half);
  if (rc) return rc;
  launch_ssd_tiles(c->tiles, nt, lum_ref, lum_src, w, h, h_pred, p->radius, p->patch, c->slot_rows,
                   c->slot_flags, s);
  launch_compact_rows(c->slot_rows, c->slot_flags, nt, c->raw, c->counters + 0, raw, s);
  CUDA_TRY(cudaMemcpyAsync(count, c->counters + 0, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return check_launch();
}

__global__ void rows_from_matrix_kernel(const double* m, int n, MatchRow* rows, int32_t* count) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *count = n;
  if (i >= n) return;
  MatchRow r;
  for (int k = 0; k < 5; ++k) r.v[k] = m[5 * (int64_t)i + k];
  rows[i] = r;
}

__global__ void widen_kept_kernel(const uint32_t* mask, const int32_t* wit, int n, int64_t* kept,
                                  int32_t* n_kept, int64_t* witness) {
  pdl_wait();
  // single block: ordered compaction of the reliable mask
  __shared__ int scratch[32];
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    int i = c0 + threadIdx.x;
    int f = i < n ? (int)((mask[i >> 5] >> (i & 31)) & 1u) : 0;
    int total;
    int pos = hdr::block_exclusive_scan(f, scratch, &total);
    if (f) kept[base + pos] = i;
    if (i < n && witness) witness[i] = wit[i];
    base += total;
  }
  if (threadIdx.x == 0) *n_kept = base;
}

extern "C" int hdr_weed(hdr_ctx* c, const double* matches, int32_t n, int32_t w, int32_t h,
                        int32_t iterations, double eps, uint64_t seed, int32_t delta, int64_t* kept,
                        int32_t* n_kept, int64_t* witness) {
  CtxDevice dg_(c);
  NEED(c && matches && kept && n_kept, "null argument");
  if (n < 4) return fail(HDR_ERR_INVALID, "need at least 4 matches to weed");
  if (iterations < 1) return fail(HDR_ERR_INVALID, "iterations must be >= 1");
  if (delta >= 0 && delta < 4) return fail(HDR_ERR_INVALID, "delta must be >= 4");
  if (!(eps > 0)) return fail(HDR_ERR_INVALID, "eps must be positive");
  NEED(n <= c->rows_cap, "too many matches for the workspace");
  cudaStream_t s = c->stream;
  // keys for this exact (seed, iterations): weeding._iteration_rng
  std::vector<uint64_t> host(2 * (size_t)iterations);
  hdr_iteration_keys(seed, iterations, host.data());
  uint64_t* dkeys = nullptr;
  CUDA_TRY(cudaMallocAsync(&dkeys, host.size() * sizeof(uint64_t), s));
  CUDA_TRY(cudaMemcpyAsync(dkeys, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  klaunch(rows_from_matrix_kernel, ceil_div(n, 256), 256, 0, s, matches, n, c->raw, c->counters + 0);
  launch_weed(c->raw, c->counters + 0, n, w, h, iterations, eps, dkeys, delta, c->mask, c->witness,
              c->counters + 3, s);
  klaunch(widen_kept_kernel, 1, 1024, 0, s, c->mask, c->witness, n, kept, c->counters + 6, witness);
  CUDA_TRY(cudaMemcpyAsync(n_kept, c->counters + 6, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaFreeAsync(dkeys, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return check_launch();
}

static int fit_status_to_rc(int32_t st) {
  if (st == 0) return HDR_OK;
  if (st == 1) return fail(HDR_ERR_INVALID, "need at least 4 point pairs");
  return fail(HDR_ERR_DEGENERATE, "degenerate correspondence set");
}

extern "C" int hdr_fit_matches_homography(hdr_ctx* c, const double* matches, int32_t n, int32_t w,
                                          int32_t h, double* H) {
  CtxDevice dg_(c);
  NEED(c && matches && H, "null argument");
  if (n < 4) return fail(HDR_ERR_INVALID, "need at least 4 point pairs");
  NEED(n <= c->rows_cap, "too many matches for the workspace");
  cudaStream_t s = c->stream;
  klaunch(rows_from_matrix_kernel, ceil_div(n, 256), 256, 0, s, matches, n, c->raw, c->counters + 0);
  launch_fit_rows(c->raw, c->counters + 0, w, h, H, c->counters + 4, s);
  int32_t st = 0;
  CUDA_TRY(cudaMemcpyAsync(&st, c->counters + 4, sizeof st, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  int rc = check_launch();
  return rc ? rc : fit_status_to_rc(st);
}

extern "C" int hdr_fit_homography(hdr_ctx* c, const double* ref_pts, const double* src_pts,
                                  int32_t n, double* H) {
  CtxDevice dg_(c);
  NEED(c && ref_pts && src_pts && H, "null argument");
  if (n < 4) return fail(HDR_ERR_INVALID, "need at least 4 point pairs");
  cudaStream_t s = c->stream;
  launch_fit_points(ref_pts, src_pts, n, H, c->counters + 4, s);
  int32_t st = 0;
  CUDA_TRY(cudaMemcpyAsync(&st, c->counters + 4, sizeof st, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  int rc = check_launch();
  return rc ? rc : fit_status_to_rc(st);
}

extern "C" int hdr_inlier_mask(hdr_ctx* c, const double* H, const double* ref_pts,
                               const double* src_pts, int32_t n, double eps, uint8_t* mask) {
  CtxDevice dg_(c);
  NEED(c && H && ref_pts && src_pts && mask, "null argument");
  launch_inlier_mask(H, ref_pts, src_pts, n, eps, mask, c->stream);
  return check_launch();
}

extern "C" int hdr_homography_flow(hdr_ctx* c, const double* H, int32_t w, int32_t h, float* flow) {
  CtxDevice dg_(c);
  NEED(c && H && flow, "null argument");
  launch_hflow(H, w, h, flow, c->stream);
  return check_launch();
}

extern "C" int hdr_match_stack(hdr_ctx* c, const hdr_params* p, int32_t w, int32_t h,
                               const float* ref, const float* src, double* matches,
                               double* raw_matches, double* homography, int32_t* info) {
  CtxDevice dg_(c);
  NEED(c && p && ref && src && matches && raw_matches && homography && info, "null argument");
  char msg[128];
  int rc = hdr_params_validate(p, msg, sizeof msg);
  if (rc) return rc;
  if (std::min(w, h) < 100) return fail(HDR_ERR_INVALID, "input below 100 pixels in one dimension");
  NEED((int64_t)w * h <= c->P && (int64_t)(w + 1) * (h + 1) <= (int64_t)(c->W + 1) * (c->H + 1),
       "image larger than the workspace");
  NEED(ntiles_of(w, h, p->tile) <= c->rows_cap, "too many tiles");
  rc = check_ptr_align(ref, 16, "ref");
  if (!rc) rc = check_ptr_align(src, 16, "src");
  if (!rc) rc = ensure_keys(c, p);
  if (!rc) rc = ensure_lattice(c, p, w, h);
  if (rc) return rc;
  return enqueue_match(c, p, w, h, ref, src, matches, raw_matches, homography, info);
}

extern "C" int hdr_sparse_maps(hdr_ctx* c, const double* matches, int32_t m, int32_t w, int32_t h,
                               double* pu, double* pv, double* n) {
  CtxDevice dg_(c);
  NEED(c && pu && pv && n && (m == 0 || matches), "null argument");
  NEED((int64_t)w * h <= c->P, "image larger than the workspace");
  cudaStream_t s = c->stream;
  CUDA_TRY(cudaMemsetAsync(c->counters + 2, 0, sizeof(int32_t), s));
  DtPlanes pl = f64_planes(pu, pv, n, 3);
  launch_splat(matches, nullptr, m, w, h, pl, c->splat_key, c->splat_idx, c->counters + 2, s);
  int32_t st = 0;
  CUDA_TRY(cudaMemcpyAsync(&st, c->counters + 2, sizeof st, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  int rc = check_launch();
  if (rc) return rc;
  if (st) return fail(HDR_ERR_INVALID, "match reference position out of bounds");
  return HDR_OK;
}

extern "C" int hdr_dt_filter(hdr_ctx* c, const float* guide, double* planes, int32_t k, int32_t w,
                             int32_t h, double sigma_s, double sigma_r, int32_t passes) {
  CtxDevice dg_(c);
  NEED(c && guide && planes && w >= 1 && h >= 1, "null argument");
  if (!(sigma_s > 0) || !(sigma_r > 0)) return fail(HDR_ERR_INVALID, "sigma_s and sigma_r must be positive");
  if (passes < 1) return fail(HDR_ERR_INVALID, "passes must be >= 1");
  NEED(k >= 1, "at least one data plane");
  NEED(dt_scratch_doubles(w, h, 3) <= dt_scratch_doubles(c->W, c->H, 3), "image larger than the workspace");
  int64_t P = (int64_t)w * h;
  // planes share the guide's coefficients and never interact: groups of three
  for (int k0 = 0; k0 < k; k0 += 3) {
    int kk = std::min(3, k - k0);
    double* b = planes + (int64_t)k0 * P;
    DtPlanes pl = f64_planes(b, b + P, b + 2 * P, kk);
    launch_dt_filter(guide, pl, w, h, sigma_s, sigma_r, passes, c->carry, c->stream);
  }
  return check_launch();
}

extern "C" int hdr_dt_filter_general(hdr_ctx* c, const double* guide, int32_t channels, double* planes,
                                     int32_t k, int32_t w, int32_t h, double sigma_s, double sigma_r,
                                     int32_t passes) {
  CtxDevice dg_(c);
  NEED(c && guide && planes && w >= 1 && h >= 1, "null argument");
  if (!(sigma_s > 0) || !(sigma_r > 0)) return fail(HDR_ERR_INVALID, "sigma_s and sigma_r must be positive");
  if (passes < 1) return fail(HDR_ERR_INVALID, "passes must be >= 1");
  NEED(k >= 1 && channels >= 1, "at least one data plane and one guide channel");
  int64_t P = (int64_t)w * h;
  for (int k0 = 0; k0 < k; k0 += 3) {
    int kk = std::min(3, k - k0);
    double* b = planes + (int64_t)k0 * P;
    DtPlanes pl = f64_planes(b, b + P, b + 2 * P, kk);
    launch_dt_filter_general(guide, channels, pl, w, h, sigma_s, sigma_r, passes, c->stream);
  }
  return check_launch();
}

// one status word of the context read back synchronously (stage twins whose
// reference raises on a data-dependent condition)
static int status_word(hdr_ctx* c, int32_t* st) {
  CUDA_TRY(cudaMemcpyAsync(st, c->counters + 2, sizeof *st, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return check_launch();
}

extern "C" int hdr_rect_sum(hdr_ctx* c, const double* table, int32_t w1, int32_t h1, const int64_t* q,
                            int64_t n, double* out) {
  CtxDevice dg_(c);
  NEED(c && table && (n == 0 || (q && out)) && w1 >= 1 && h1 >= 1, "null argument");
  CUDA_TRY(cudaMemsetAsync(c->counters + 2, 0, sizeof(int32_t), c->stream));
  launch_rect_sum(table, w1, h1, q, n, out, c->counters + 2, c->stream);
  int32_t st = 0;
  int rc = status_word(c, &st);
  if (rc) return rc;
  if (st) return fail(HDR_ERR_INVALID, "rectangle bounds out of range");
  return HDR_OK;
}

extern "C" int hdr_quantize_256(hdr_ctx* c, const void* x, int32_t is_f64, int64_t n, uint8_t* out) {
  CtxDevice dg_(c);
  NEED(c && (n == 0 || (x && out)), "null argument");
  launch_quantize(x, is_f64 != 0, n, out, c->stream);
  return check_launch();
}

extern "C" int hdr_downsample(hdr_ctx* c, const void* img, int32_t is_f64, int32_t w, int32_t h,
                              int32_t channels, float* out) {
  CtxDevice dg_(c);
  NEED(c && img && out && channels >= 1, "null argument");
  if (h < 2 || w < 2) return fail(HDR_ERR_INVALID, "image too small to downsample");
  launch_downsample_ch(img, is_f64 != 0, w, h, channels, out, c->stream);
  return check_launch();
}

extern "C" int hdr_apply_homography(hdr_ctx* c, const double* H, const double* pts, int64_t n, double* out) {
  CtxDevice dg_(c);
  NEED(c && H && (n == 0 || (pts && out)), "null argument");
  CUDA_TRY(cudaMemsetAsync(c->counters + 2, 0, sizeof(int32_t), c->stream));
  launch_apply_homography(H, pts, n, out, c->counters + 2, c->stream);
  int32_t st = 0;
  int rc = status_word(c, &st);
  if (rc) return rc;
  if (st) return fail(HDR_ERR_INVALID, "point maps to infinity");
  return HDR_OK;
}

extern "C" int hdr_symmetric_transfer_error(hdr_ctx* c, const double* H, const double* ref_pts,
                                            const double* src_pts, int64_t n, double* out) {
  CtxDevice dg_(c);
  NEED(c && H && (n == 0 || (ref_pts && src_pts && out)), "null argument");
  CUDA_TRY(cudaMemsetAsync(c->counters + 2, 0, sizeof(int32_t), c->stream));
  launch_transfer_error(H, ref_pts, src_pts, n, out, c->counters + 2, c->stream);
  int32_t st = 0;
  int rc = status_word(c, &st);
  if (rc) return rc;
  if (st) return fail(HDR_ERR_SINGULAR, "Singular matrix");
  return HDR_OK;
}

// ---- row-band pieces of the pair (paper_1504_01441_b200/banded.py)
extern "C" int32_t hdr_band_rows_multiple(void) { return 32; }

extern "C" int64_t hdr_band_agg_doubles(int32_t w, int32_t h, int32_t k) {
  return hdr::dt_band_agg_doubles(w, h, k);
}

extern "C" int hdr_band_dt(hdr_ctx* c, int32_t op, const float* guide, double* planes, int32_t k, int32_t w,
                           int32_t h, int32_t y0, int32_t y1, double sigma_s, double sigma_r, int32_t passes,
                           int32_t pass_i, double* agg, const double* fallback, const int32_t* has_fb,
                           double floor_, float* flow) {
  CtxDevice dg_(c);
  NEED(c && guide && planes && k >= 1 && k <= 3 && w >= 1 && h >= 1, "bad argument");
  NEED(op >= 0 && op <= 2 && pass_i >= 1 && pass_i <= passes, "bad band operation");
  NEED(0 <= y0 && y0 <= y1 && y1 <= h && y0 % dt_band_chunk_rows() == 0 &&
           (y1 == h || y1 % dt_band_chunk_rows() == 0),
       "band rows must be whole chunks");
  NEED(op == 0 || agg, "null aggregate buffer");
  NEED(dt_scratch_doubles(w, h, k) <= dt_scratch_doubles(c->W, c->H, 3), "image larger than the workspace");
  int64_t P = (int64_t)w * h;
  DtPlanes pl = f64_planes(planes, planes + P, planes + 2 * P, k);
  DtFlowOut fo{fallback, has_fb, floor_, flow};
  double* carry = c->carry + hdr::dt_band_agg_doubles(w, h, k);
  launch_dt_band(op, guide, pl, w, h, y0, y1, sigma_s, sigma_r, passes, pass_i, agg, carry, &fo, c->stream);
  return check_launch();
}

extern "C" int hdr_band_warp(hdr_ctx* c, const float* flow, int32_t w, int32_t h, int32_t y0, int32_t y1,
                             const float* src, float* warped, uint8_t* valid, uint8_t* qw, uint32_t* hist) {
  CtxDevice dg_(c);
  NEED(c && flow && src && warped && valid && qw && 0 <= y0 && y0 <= y1 && y1 <= h, "bad argument");
  NEED(3 * (int64_t)w * h < ((int64_t)1 << 31), "frame too large for the banded warp");
  launch_warp_rows(flow, w, h, y0, y1, src, warped, valid, qw, hist, c->stream);
  return check_launch();
}

extern "C" int hdr_band_ssim(hdr_ctx* c, const float* lum_ref, const uint8_t* qw, const uint32_t* hist_w,
                             int32_t w, int32_t h, int32_t y0, int32_t y1, int32_t window, double sigma,
                             float* out) {
  CtxDevice dg_(c);
  NEED(c && lum_ref && qw && hist_w && out && 0 <= y0 && y0 <= y1 && y1 <= h, "bad argument");
  NEED((int64_t)w * h <= c->P, "image larger than the workspace");
  int rc = ensure_taps(c, window, sigma);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  int64_t P = (int64_t)w * h;
  uint32_t* hr = c->hist + 3 * kBins;
  CUDA_TRY(cudaMemsetAsync(hr, 0, sizeof(uint32_t) * kBins, s));
  launch_hist_plain(lum_ref, P, 1, hr, s);
  launch_lut(hist_w, P, hr, P, c->lut + 2 * kBins, s);
  if (!launch_ssim_rows(lum_ref, qw, c->lut + 2 * kBins, w, h, y0, y1, window, c->taps, out, s))
    return fail(HDR_ERR_INVALID, "banded SSIM needs an 11-tap window and 32-row band starts");
  return check_launch();
}

extern "C" int hdr_densify_finalize(hdr_ctx* c, const double* smooth, int32_t w, int32_t h,
                                    const double* fallback, double floor_, float* flow) {
  CtxDevice dg_(c);
  NEED(c && smooth && flow, "null argument");
  // the fused kernel with the warp outputs switched off
  int64_t P = (int64_t)w * h;
  DtPlanes pl = f64_planes(const_cast<double*>(smooth), const_cast<double*>(smooth) + P,
                           const_cast<double*>(smooth) + 2 * P, 3);
  launch_finalize_warp(pl, fallback, nullptr, w, h, floor_, nullptr, 1, flow, nullptr, nullptr,
                       nullptr, nullptr, true, c->stream);
  return check_launch();
}

extern "C" int hdr_warp_image(hdr_ctx* c, const float* src, int32_t channels, int32_t w, int32_t h,
                              const float* flow, float* warped, uint8_t* valid) {
  CtxDevice dg_(c);
  NEED(c && src && flow && warped && valid, "null argument");
  NEED(channels >= 1, "channels must be >= 1");
  if (channels == 3 && (int64_t)w * h <= c->P) {
    // the pair pipeline's kernel (its luminance histogram lands in scratch)
    launch_warp(flow, w, h, src, warped, valid, c->qw, c->hist + 2 * kBins, c->stream);
    return check_launch();
  }
  DtPlanes none = f64_planes(nullptr, nullptr, nullptr, 0);
  launch_finalize_warp(none, nullptr, nullptr, w, h, 0.0, src, channels,
                       const_cast<float*>(flow), warped, valid, nullptr, nullptr, false, c->stream);
  return check_launch();
}

extern "C" int hdr_ssim_map(hdr_ctx* c, const float* a, const float* b, int32_t w, int32_t h,
                            int32_t window, double sigma, float* out) {
  CtxDevice dg_(c);
  NEED(c && a && b && out, "null argument");
  if (window % 2 != 1) return fail(HDR_ERR_INVALID, "window must be odd");
  int rc = ensure_taps(c, window, sigma);
  if (rc) return rc;
  launch_ssim(a, b, nullptr, nullptr, w, h, window, c->taps, out, c->stream);
  return check_launch();
}

extern "C" int hdr_make_ssim(hdr_ctx* c, const float* lum_ref, const float* warped, int32_t w,
                             int32_t h, int32_t window, double sigma, float* out) {
  CtxDevice dg_(c);
  NEED(c && lum_ref && warped && out, "null argument");
  int64_t P = (int64_t)w * h;
  NEED(P <= c->P, "image larger than the workspace");
  int rc = ensure_taps(c, window, sigma);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  uint32_t* hw = c->hist + 2 * kBins;
  uint32_t* hr = c->hist + 3 * kBins;
  CUDA_TRY(cudaMemsetAsync(hw, 0, sizeof(uint32_t) * 2 * kBins, s));
  launch_luma_hist(warped, P, nullptr, c->qw, hw, s);
  launch_hist_plain(lum_ref, P, 1, hr, s);
  launch_lut(hw, P, hr, P, c->lut + 2 * kBins, s);
  launch_ssim(lum_ref, nullptr, c->qw, c->lut + 2 * kBins, w, h, window, c->taps, out, s);
  return check_launch();
}

extern "C" int hdr_quality_weights(hdr_ctx* c, const float* rgb, int32_t w, int32_t h, float* out) {
  CtxDevice dg_(c);
  NEED(c && rgb && out, "null argument");
  launch_quality(rgb, w, h, out, c->stream);
  return check_launch();
}

extern "C" int hdr_fusion_weights(hdr_ctx* c, const float* ref, const float* warped,
                                  const float* ssim, const uint8_t* valid, int32_t w, int32_t h,
                                  float* w_ref, float* w_src) {
  CtxDevice dg_(c);
  NEED(c && ref && warped && ssim && valid && w_ref && w_src, "null argument");
  launch_fusion_weights(ref, warped, ssim, valid, w, h, w_ref, w_src, c->stream);
  return check_launch();
}

extern "C" int hdr_cornerness(hdr_ctx* c, const double* table, int32_t w, int32_t h,
                              const int32_t* xy, int32_t n, int32_t half, double* out) {
  CtxDevice dg_(c);
  NEED(c && table && xy && out, "null argument");
  NEED(half >= 1 && w >= 1 && h >= 1, "bad arguments");
  launch_cornerness(table, w + 1, xy, n, half, out, c->stream);
  return check_launch();
}

extern "C" int hdr_pyr_down(hdr_ctx* c, const double* in, int32_t w, int32_t h, int32_t ch,
                            double* out) {
  CtxDevice dg_(c);
  NEED(c && in && out, "null argument");
  NEED(w >= 1 && h >= 1 && ch >= 1, "empty image");
  launch_pyr_down(in, w, h, ch, out, c->stream);
  return check_launch();
}

extern "C" int hdr_pyr_up(hdr_ctx* c, const double* in, int32_t cw, int32_t cht, int32_t ch,
                          int32_t w, int32_t h, const double* base, int32_t sign, double* out) {
  CtxDevice dg_(c);
  NEED(c && in && out, "null argument");
  NEED(w >= 1 && h >= 1 && ch >= 1 && cw == (w + 1) / 2 && cht == (h + 1) / 2,
       "coarse shape must be the ceil-half of the fine shape");
  launch_pyr_up(in, cw, cht, ch, out, w, h, base, sign, c->stream);
  return check_launch();
}

extern "C" int hdr_fuse(hdr_ctx* c, const float* ref, const float* warped, const float* ssim,
                        const uint8_t* valid, int32_t w, int32_t h, int32_t levels, float* out) {
  CtxDevice dg_(c);
  NEED(c && ref && warped && ssim && valid && out, "null argument");
  NEED((int64_t)w * h <= c->P, "image larger than the workspace");
  std::vector<Dims> fd;
  fusion_dims(w, h, levels > 0 ? levels : fusion_levels_default(w, h), fd);
  NEED(fusion_floats(fd, 2) <= c->fpyr_cap, "fusion pyramid larger than the workspace");
  return enqueue_fuse(c, ref, warped, ssim, valid, w, h, levels, out);
}

extern "C" int hdr_fuse_stack(hdr_ctx* c, int32_t n, const float* const* frames,
                              const float* const* ssim, const uint8_t* const* valid, int32_t w,
                              int32_t h, int32_t levels, float* out);

extern "C" int hdr_register_and_fuse_stack(hdr_ctx* c, const hdr_params* p, int32_t n,
                                           int32_t w, int32_t h, const float* const* frames,
                                           const hdr_outputs* const* outs, float* composite) {
  CtxDevice dg_(c);
  NEED(c && p && frames && outs && composite, "null argument");
  NEED(n >= 2 && n <= kMaxFuseFrames, "stacks take 2..4 frames");
  const float* warped[kMaxFuseFrames] = {};
  const float* ssim[kMaxFuseFrames] = {};
  const uint8_t* valid[kMaxFuseFrames] = {};
  warped[0] = frames[0];
  for (int f = 1; f < n; ++f) {
    NEED(outs[f - 1], "null outputs");
    int rc = check_pair_args(c, p, w, h, frames[0], frames[f], outs[f - 1], false);
    if (rc) return rc;
    // register_and_fuse up to the SSIM map (pipeline.py:183-192), per source
    rc = enqueue_pair(c, p, w, h, frames[0], frames[f], outs[f - 1], false);
    if (rc) return rc;
    warped[f] = outs[f - 1]->warped;
    ssim[f - 1] = outs[f - 1]->ssim;
    valid[f - 1] = outs[f - 1]->valid;
  }
  return hdr_fuse_stack(c, n, warped, ssim, valid, w, h, 0, composite);
}

extern "C" int hdr_fuse_stack(hdr_ctx* c, int32_t n, const float* const* frames,
                              const float* const* ssim, const uint8_t* const* valid, int32_t w,
                              int32_t h, int32_t levels, float* out) {
  CtxDevice dg_(c);
  NEED(c && frames && out, "null argument");
  NEED(n >= 2 && n <= kMaxFuseFrames, "stack fusion takes 2..4 frames");
  NEED(n == 2 || (ssim && valid), "null argument");
  NEED((int64_t)w * h <= c->P && w >= 1 && h >= 1, "image larger than the workspace");
  FuseFrameSet fs{};
  for (int f = 0; f < n; ++f) {
    NEED(frames[f], "null frame");
    fs.img[f] = frames[f];
    if (f > 0) {
      NEED(ssim[f - 1] && valid[f - 1], "null ssim/valid");
      fs.ssim[f] = ssim[f - 1];
      fs.valid[f] = valid[f - 1];
    }
  }
  std::vector<Dims> fd;
  fusion_dims(w, h, levels > 0 ? levels : fusion_levels_default(w, h), fd);
  int64_t need = fusion_floats(fd, n) + (int64_t)n * (round4((int64_t)w * h) + 64);
  if (need > c->fstack_cap) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->fstack) cudaFree(c->fstack);
    c->fstack = nullptr;
    c->fstack_cap = 0;
    CUDA_TRY(cudaMalloc(&c->fstack, need * sizeof(float)));
    c->fstack_cap = need;
  }
  float* wbase = c->fstack + fusion_floats(fd, n);
  for (int f = 0; f < n; ++f) fs.wout[f] = wbase + (int64_t)f * (round4((int64_t)w * h) + 64);
  return enqueue_fuse_frames(c, n, fs, w, h, levels, c->fstack, out);
}

// ------------------------------------------------------------ attributes
static void init_kernel_attributes() {
  hdr::init_match_attributes();
  hdr::init_densify_attributes();
  hdr::init_fusion_attributes();
  hdr::init_merge_attributes();
  hdr::init_raster_attributes();
}
