// Debug harness: run hdr::fit_from_gram on host and device with the same input.
#include <cstdio>
#include "../../paper_1504_01441_b200/csrc/hdr_geom.cuh"
using namespace hdr;

__global__ void k(const double* g45, const double* tr, const double* ts, double* H, int* st) {
  int g = 0;
  *st = fit_from_gram(g45, tr, ts, H, &g);
}

int main() {
  // 6 points, affine map
  double p[12] = {-0.9, -0.5, 0.3, -0.7, 0.8, 0.6, -0.2, 0.9, 0.1, 0.1, 0.5, -0.3};
  double q[12];
  for (int i = 0; i < 6; ++i) { q[2*i] = 1.01*p[2*i] + 0.02*p[2*i+1] + 0.03; q[2*i+1] = -0.01*p[2*i] + 0.99*p[2*i+1] - 0.02; }
  double c[4] = {0,0,0,0};
  int n = 6;
  for (int i = 0; i < n; ++i) { c[0]+=p[2*i]; c[1]+=p[2*i+1]; c[2]+=q[2*i]; c[3]+=q[2*i+1]; }
  for (int k2 = 0; k2 < 4; ++k2) c[k2] /= n;
  double m0=0,m1=0;
  for (int i = 0; i < n; ++i) { m0 += hypot(p[2*i]-c[0], p[2*i+1]-c[1]); m1 += hypot(q[2*i]-c[2], q[2*i+1]-c[3]); }
  m0/=n; m1/=n;
  double sr = sqrt(2.0)/m0, ss = sqrt(2.0)/m1;
  double tr[3] = {sr, -sr*c[0], -sr*c[1]}, ts[3] = {ss, -ss*c[2], -ss*c[3]};
  double g45[45] = {0};
  for (int i = 0; i < n; ++i) {
    double r0[9], r1[9];
    dlt_rows((p[2*i]-c[0])*sr, (p[2*i+1]-c[1])*sr, (q[2*i]-c[2])*ss, (q[2*i+1]-c[3])*ss, r0, r1);
    int kk = 0;
    for (int a = 0; a < 9; ++a) for (int b = a; b < 9; ++b) { g45[kk] += r0[a]*r0[b] + r1[a]*r1[b]; ++kk; }
  }
  double Hh[9]; int gh = 0;
  int sh = fit_from_gram(g45, tr, ts, Hh, &gh);
  double *dg, *dtr, *dts, *dH; int* dst;
  cudaMalloc(&dg, 45*8); cudaMalloc(&dtr, 24); cudaMalloc(&dts, 24); cudaMalloc(&dH, 72); cudaMalloc(&dst, 4);
  cudaMemcpy(dg, g45, 45*8, cudaMemcpyHostToDevice); cudaMemcpy(dtr, tr, 24, cudaMemcpyHostToDevice); cudaMemcpy(dts, ts, 24, cudaMemcpyHostToDevice);
  k<<<1,1>>>(dg, dtr, dts, dH, dst);
  double Hd[9]; int sd = -1;
  cudaMemcpy(Hd, dH, 72, cudaMemcpyDeviceToHost); cudaMemcpy(&sd, dst, 4, cudaMemcpyDeviceToHost);
  printf("host st=%d device st=%d err=%s\n", sh, sd, cudaGetErrorString(cudaGetLastError()));
  for (int i = 0; i < 9; ++i) printf("%d % .17g % .17g\n", i, Hh[i], Hd[i]);
  return 0;
}
