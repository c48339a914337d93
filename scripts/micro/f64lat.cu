// Dependent-chain latency of FP64 ops on this GPU (one thread), cycles/op.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b, z = 1.0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, y, z);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x + y;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 200; ++i) x = sqrt(x) + 1.0;
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 200; ++i) x = 1.0 / x + 1.0;
  long long t4 = clock64();
  float f = (float)a;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) f = fmaf(f, (float)y, 1.0f);
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31);
  long long t6 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, c, 0.999, 0.5); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 0.999, 0.5); cudaDeviceSynchronize();
  printf("cycles/op: dfma %.1f dadd %.1f sqrt+add %.1f rcp+add %.1f ffma %.1f shfl64 %.1f\n", c[0] / 1000.0, c[1] / 1000.0,
         c[2] / 200.0, c[3] / 200.0, c[4] / 1000.0, c[5] / 1000.0);
}
