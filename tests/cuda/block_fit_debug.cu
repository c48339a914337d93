// Debug harness: the library's block-wide fit kernel on random points, with
// hdr_geom's debug prints enabled.
#define HDR_DEBUG_FIT 1
#include <cstdio>
#include "../../paper_1504_01441_b200/csrc/k_match.cu"
int main() {
  int n = 6;
  double p[12] = {-0.9, -0.5, 0.3, -0.7, 0.8, 0.6, -0.2, 0.9, 0.1, 0.1, 0.5, -0.3};
  double q[12];
  for (int i = 0; i < 6; ++i) { q[2*i] = 1.01*p[2*i] + 0.02*p[2*i+1] + 0.03; q[2*i+1] = -0.01*p[2*i] + 0.99*p[2*i+1] - 0.02; }
  double *dp, *dq, *dH; int* dst;
  cudaMalloc(&dp, 96); cudaMalloc(&dq, 96); cudaMalloc(&dH, 72); cudaMalloc(&dst, 4);
  cudaMemcpy(dp, p, 96, cudaMemcpyHostToDevice); cudaMemcpy(dq, q, 96, cudaMemcpyHostToDevice);
  hdr::launch_fit_points(dp, dq, n, dH, dst, 0);
  int st = -1; double H[9];
  cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost); cudaMemcpy(H, dH, 72, cudaMemcpyDeviceToHost);
  printf("status %d err %s H00 %g\n", st, cudaGetErrorString(cudaGetLastError()), H[0]);
  return 0;
}
