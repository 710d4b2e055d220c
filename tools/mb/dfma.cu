// FP64 FMA throughput: 8 independent DFMA chains per thread, all SMs busy.
#include <cstdio>
__global__ void k(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = x0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    const int iters = 20000, threads = 256;
    k<<<sms * blocks_per_sm, threads>>>(o, 100, 0.999999, 1e-9);
    cudaEventRecord(e0);
    k<<<sms * blocks_per_sm, threads>>>(o, iters, 0.999999, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)threads * sms * blocks_per_sm;
    printf("%d CTAs/SM (%d warps/SM): %.2f TFLOP/s fp64 FMA, %.3f warp-DFMA per SM-clock @1.965GHz\n",
           blocks_per_sm, blocks_per_sm * 8, fl / ms / 1e9, fl / 2 / 32 / (ms * 1e-3) / sms / 1.965e9);
  }
}
