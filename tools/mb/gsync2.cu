// Grid barrier variants for the operator sweeps (one CTA per SM, all
// co-resident): the flat hand-rolled counter (op_barrier) vs a two-level
// barrier over thread-block clusters (hardware cluster barrier, then one
// arrival per cluster on the global counter).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gsync2 tools/mb/gsync2.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void flat(int iters, unsigned int *ctr, double *out) {
  __shared__ double r;
  const unsigned int nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int target = (i + 1) * nb, v;
      __threadfence();
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
      r = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = r;
}

__global__ void clustered(int iters, unsigned int *ctr, double *out) {
  __shared__ double r;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned int ncl = gridDim.x / cl.num_blocks();
  for (int i = 0; i < iters; ++i) {
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      unsigned int target = (i + 1) * ncl, v;
      __threadfence();
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
      r = v;
    }
    cl.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = r;
}

int main() {
  double *out; unsigned int *ctr;
  cudaMalloc(&out, 8); cudaMalloc(&ctr, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {512}) {
    cudaMemset(ctr, 0, 4);
    void *args[] = {(void *)&iters, &ctr, &out};
    cudaLaunchCooperativeKernel((void *)flat, sms, threads, args, 0, 0);
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)flat, sms, threads, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("flat counter, %d CTAs: %.3f us/barrier (%s)\n", sms, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
    for (int cs : {2, 4}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms); cfg.blockDim = dim3(threads);
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
      cfg.attrs = at; cfg.numAttrs = 2;
      cudaMemset(ctr, 0, 4);
      cudaError_t e = cudaLaunchKernelEx(&cfg, clustered, iters, ctr, out);
      cudaDeviceSynchronize();
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(a);
      e = cudaLaunchKernelEx(&cfg, clustered, iters, ctr, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("cluster %d (%d clusters): %.3f us/barrier (launch %s, %s)\n", cs, sms / cs, ms * 1000 / iters,
             cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
    }
  }
}
