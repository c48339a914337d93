// Experiment (not product): would the column sweep be cheaper as a row sweep
// over a transposed copy? Times the row kernel in place, a row kernel whose
// output is written transposed (plain 8-byte stores, sectors merged in L2),
// the same over the transposed image (a "column" pass), and the cluster
// column kernel, all on 3 f64 planes.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//     -I paper_1504_01441_b200/csrc scripts/exp/exp_transpose.cu \
//     -L paper_1504_01441_b200 -lhdrb200 -Xlinker -rpath=$PWD/paper_1504_01441_b200 -o /tmp/exp_t
#include "../../paper_1504_01441_b200/csrc/k_dtfilter.cu"
#include <cstdio>
#include <vector>

namespace hdr {
template <int K, int MODE>
__global__ void __launch_bounds__(kRowThreads) dt_rows_T_kernel(const float* __restrict__ guide,
                                                                DtPlanes P, DtPlanes Q, int w, int h,
                                                                double ratio, double c) {
  extern __shared__ __align__(16) double xs[];
  float* gs = reinterpret_cast<float*>(xs + K * w);
  __shared__ Aff<K> wsum[kRowThreads / 32];
  __shared__ uint64_t bar;
  int y = blockIdx.x;
  int64_t row = (int64_t)y * w;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)(K * w * 8 + w * 4));
#pragma unroll
    for (int k = 0; k < K; ++k)
      bulk_load(xs + k * w, reinterpret_cast<const double*>(P.p[k]) + row, (uint32_t)w * 8, &bar);
    bulk_load(gs, guide + row, (uint32_t)w * 4, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  row_sweep_smem<K>(xs, gs, w, ratio, c, wsum);
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double* d = reinterpret_cast<double*>(Q.p[k]) + (int64_t)i * h + y;
      if (MODE == 0) *d = xs[k * w + i];
      else __stcg(d, xs[k * w + i]);
    }
}
}  // namespace hdr

using namespace hdr;

int main() {
  const int W = 2592, H = 1944, K = 3;
  size_t P = (size_t)W * H;
  float* g;
  float* gT;
  double *a, *b;
  cudaMalloc(&g, P * 4);
  cudaMalloc(&gT, P * 4);
  cudaMalloc(&a, P * 8 * K);
  cudaMalloc(&b, P * 8 * K);
  std::vector<float> hg(P);
  for (size_t i = 0; i < P; ++i) hg[i] = (float)((i * 2654435761u) % 1000) / 1000.0f;
  cudaMemcpy(g, hg.data(), P * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(gT, hg.data(), P * 4, cudaMemcpyHostToDevice);
  cudaMemset(a, 0, P * 8 * K);
  cudaMemset(b, 0, P * 8 * K);
  DtPlanes A{}, B{};
  A.k = B.k = K;
  for (int k = 0; k < K; ++k) {
    A.p[k] = a + k * P; B.p[k] = b + k * P;
    A.f64[k] = B.f64[k] = true;
  }
  init_densify_attributes();
  size_t smw = (size_t)K * W * 8 + W * 4, smh = (size_t)K * H * 8 + H * 4;
  cudaFuncSetAttribute(dt_rows_T_kernel<3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(dt_rows_T_kernel<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double ratio = 400.0 / 0.2, c = -0.01;
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 3; ++i) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.1f us  (%s)\n", name, ms / 20 * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  DtFlowOut none{nullptr, nullptr, 0.0, nullptr};
  int bl = cluster_bw_log2(H);
  timeit("rows in place (bulk)", [&] { dt_rows_bulk_kernel<3><<<H, kRowThreads, smw>>>(g, A, W, H, ratio, c); });
  timeit("rows -> transposed (st)", [&] { dt_rows_T_kernel<3, 0><<<H, kRowThreads, smw>>>(g, A, B, W, H, ratio, c); });
  timeit("rows -> transposed (st.cg)", [&] { dt_rows_T_kernel<3, 1><<<H, kRowThreads, smw>>>(g, A, B, W, H, ratio, c); });
  timeit("T rows (cols) -> normal (st)", [&] { dt_rows_T_kernel<3, 0><<<W, kRowThreads, smh>>>(gT, B, A, H, W, ratio, c); });
  timeit("cols cluster", [&] { launch_cols_cluster<3, false>(g, A, W, H, ratio, c, bl, none, 0); });
  return 0;
}
