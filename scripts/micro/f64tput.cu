// FP64 / FP32 FMA throughput per SM (many independent chains, full occupancy).
#include <cstdio>
template <typename T>
__global__ void k(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms = 148, blocks = sms * 8, threads = 256, iters = 4096;
  double* od; float* of;
  cudaMalloc(&od, sizeof(double) * blocks * threads);
  cudaMalloc(&of, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<double><<<blocks, threads>>>(od, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)blocks * threads * iters * 8;
    printf("f64: %.2f TFMA/s = %.1f FMA/clk/SM at 1.965 GHz\n", fma / ms / 1e9, fma / (ms * 1e-3) / 1.965e9 / sms);
    cudaEventRecord(e0);
    k<float><<<blocks, threads>>>(of, iters, 0.999999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("f32: %.2f TFMA/s = %.1f FMA/clk/SM\n", fma / ms / 1e9, fma / (ms * 1e-3) / 1.965e9 / sms);
  }
}
