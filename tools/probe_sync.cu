#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_sync_only(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) { cl.sync(); acc += 1.0; }
  if (threadIdx.x == 0) out[blockIdx.x] = acc + sm[0];
}
__global__ void k_arrive_wait(int iters, double* out) {
  extern __shared__ double sm[];
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    acc += 1.0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc + sm[0];
}
__global__ void k_dsmem(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  sm[threadIdx.x] = threadIdx.x;
  double acc = 0;
  cl.sync();
  for (int i = 0; i < iters; ++i) {
    double* rem = cl.map_shared_rank(sm, (cl.block_rank() + 1 + (i & 3)) % cl.num_blocks());
    acc += rem[(threadIdx.x + i) & 511];
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
template <typename K>
void run(const char* name, K k, int C, int thr, int nclus) {
  size_t smem = 64 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1; cfg.blockDim = dim3(thr); cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(C * nclus);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  cudaLaunchKernelEx(&cfg, k, 100, out);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-12s C=%2d thr=%4d clusters=%2d: %.3f us/iter (%s)\n", name, C, thr, nclus, ms * 1e3 / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}
int main() {
  for (int C : {16, 8, 4})
    for (int thr : {128, 512, 1024}) run("sync", k_sync_only, C, thr, C == 16 ? 7 : (C == 8 ? 15 : 33));
  run("arrive/wait", k_arrive_wait, 16, 512, 7);
  run("dsmem-ld", k_dsmem, 16, 512, 7);
  run("dsmem-ld", k_dsmem, 8, 512, 15);
}
