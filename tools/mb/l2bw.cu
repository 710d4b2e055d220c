// L2-resident read bandwidth: repeatedly sum a buffer of S MB (fits in L2).
#include <cstdio>
__global__ void rd(const double2 *p, size_t n, double *out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcg(p + i); acc += v.x + v.y;
  }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mb : {16, 32, 65, 100, 116, 400}) {
    size_t bytes = (size_t)mb << 20; double2 *p; double *o; cudaMalloc(&p, bytes); cudaMalloc(&o, 8);
    cudaMemset(p, 0, bytes);
    size_t n = bytes / sizeof(double2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) rd<<<sms * 8, 256>>>(p, n, o);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) rd<<<sms * 8, 256>>>(p, n, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%4d MB: %.2f TB/s (%.2f us per pass)\n", mb, bytes * 20.0 / (ms / 1e3) / 1e12, ms * 1000 / 20);
    cudaFree(p); cudaFree(o);
  }
}
