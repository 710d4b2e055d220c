#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long *slots, double *out) {
  cg::grid_group g = cg::this_grid();
  __shared__ double r;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicMax(&slots[i % 3], (unsigned long long)(blockIdx.x + i));
    g.sync();
    if (threadIdx.x == 0) r = (double)__ldcg(&slots[i % 3]);
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = r;
}
// hand-rolled barrier: monotonically increasing counter
__global__ void k2(int iters, unsigned int *ctr, double *out) {
  __shared__ double r;
  const unsigned int nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int target = (i + 1) * nb;
      unsigned int v;
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
      r = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = r;
}
int main() {
  unsigned long long *slots; double *out; unsigned int *ctr;
  cudaMalloc(&slots, 64); cudaMalloc(&out, 8); cudaMalloc(&ctr, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {256, 512, 1024}) {
    int iters = 2000;
    void *args[] = {&iters, &slots, &out};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)k, sms, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, sms, threads, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaMemset(ctr, 0, 4);
    void *args2[] = {&iters, &ctr, &out};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k2, sms, threads, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    printf("threads %d: cg grid.sync %.3f us/iter, hand barrier %.3f us/iter (%s)\n", threads, ms*1000/iters, ms2*1000/iters, cudaGetErrorString(cudaGetLastError()));
  }
}
