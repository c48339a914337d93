// Shared helpers for libhdrb200 (sm_100a). Functions marked HD compile for
// both the device and the host (the host copies back the test hooks).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define HD __host__ __device__ __forceinline__

namespace hdr {

constexpr int kMaxLevels = 5;     // image.py:13
constexpr int kBins = 256;        // image.py:15
constexpr int kMaxResample = 10;  // weeding.py:27

// scipy.ndimage mode='reflect' (half-sample symmetric: d c b a | a b c d | d c b a)
// for any excursion (period 2n). SURVEY.md Appendix A.7.
HD int reflect_index(int i, int n) {
  if (n == 1) return 0;
  int p = 2 * n;
  i %= p;
  if (i < 0) i += p;
  return i < n ? i : p - 1 - i;
}

HD int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Separately rounded arithmetic: numpy never contracts a*b+c into an FMA
// (SURVEY.md A.1); nvcc would, so parity-critical expressions use these.
HD float fmul(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fmul_rn(a, b);
#else
  return a * b;
#endif
}
HD float fadd(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fadd_rn(a, b);
#else
  return a + b;
#endif
}
HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
HD double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

// image.to_normalized (image.py:125-129): ((2x - W) / W, (2y - H) / W), f64.
HD void to_norm(double x, double y, int w, int h, double* xn, double* yn) {
  double fw = (double)w;
  *xn = dsub(dmul(2.0, x), (double)w) / fw;
  *yn = dsub(dmul(2.0, y), (double)h) / fw;
}

// image.from_normalized (image.py:132-136).
HD void from_norm(double xn, double yn, int w, int h, double* x, double* y) {
  double fw = (double)w;
  *x = dadd(dmul(xn, fw), (double)w) / 2.0;
  *y = dadd(dmul(yn, fw), (double)h) / 2.0;
}

// Opt a kernel into the largest dynamic shared memory the device allows
// (opt-in limit minus the kernel's static shared memory).
template <class K>
inline int allow_max_dynamic_smem(K kernel) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) return 0;
  int bytes = optin - (int)fa.sharedSizeBytes;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return 0;
  return bytes;
}

// Programmatic dependent launch (PDL): with g_pdl every kernel is launched
// with programmatic stream serialisation, so its launch and CTA rasterisation
// overlap the tail of the previous kernel on the stream; pdl_wait() (the
// first statement of every kernel) then waits for that kernel's completion
// and memory flush. No kernel triggers its dependents early: measured, an
// early griddepcontrol.launch_dependents made the graph-replayed pair slower
// (1.46 -> 1.52 ms), while the implicit trigger at grid end takes the
// stream-launched pair from 1.59 to 1.46 ms and leaves the graph at 1.45.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// every kernel of the library is launched through klaunch and starts with
// pdl_wait(); hdr_set_option("pdl", 0) turns the attribute off
extern bool g_pdl;
// launch tracing (hdr_set_option("trace", 1)): events around every launch,
// read back with hdr_trace_dump (tools only; it breaks PDL overlap)
extern bool g_trace;
void trace_launch(const void* kern, cudaStream_t s, int end);

template <typename... KArgs, typename... Args>
inline cudaError_t klaunch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                           Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  if (g_trace) trace_launch((const void*)kern, s, 0);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (g_trace) trace_launch((const void*)kern, s, 1);
  return e;
}

// Apply a row-major 3x3 H to (x, y), numpy operation order:
// ((h0*x + h1*y) + h2) / ((h6*x + h7*y) + h8). Returns the denominator.
HD double apply_h(const double* H, double x, double y, double* mx, double* my) {
  double den = dadd(dadd(dmul(H[6], x), dmul(H[7], y)), H[8]);
  *mx = dadd(dadd(dmul(H[0], x), dmul(H[1], y)), H[2]);
  *my = dadd(dadd(dmul(H[3], x), dmul(H[4], y)), H[5]);
  return den;
}

// geometry.homography_pixel_flow (geometry.py:124-135) at one pixel, f32.
HD void h_pixel_flow(const double* H, int x, int y, int w, int h, float* fu, float* fv) {
  double xn, yn, nx, ny;
  to_norm((double)x, (double)y, w, h, &xn, &yn);
  double den = apply_h(H, xn, yn, &nx, &ny);
  bool bad = fabs(den) < 1e-12;
  double safe = bad ? 1.0 : den;
  double px, py;
  from_norm(nx / safe, ny / safe, w, h, &px, &py);
  *fu = bad ? 0.0f : (float)dsub(px, (double)x);
  *fv = bad ? 0.0f : (float)dsub(py, (double)y);
}

}  // namespace hdr
