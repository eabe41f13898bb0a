// Probe: 16-CTA cluster residency, cluster.sync cost, FP64 add/mul rate.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  double acc = threadIdx.x;
  sm[threadIdx.x] = acc;
  for (int i = 0; i < iters; ++i) {
    cl.sync();
    double* rem = cl.map_shared_rank(sm, (cl.block_rank() + 1) % cl.num_blocks());
    acc += rem[threadIdx.x];
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

__global__ void k_fp64(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.5, c1 = 0.25, c2 = 0.125, c3 = 0.0625;
  for (int i = 0; i < iters; ++i) {
    c0 = c0 * b + a; c1 = c1 * b + a; c2 = c2 * b + a; c3 = c3 * b + a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}

int main() {
  int C = 16, threads = 512;
  size_t smem = 210 * 1024;
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
  for (int cs : {16, 8, 4}) {
    at[0].val.clusterDim.x = cs;
    cfg.gridDim = dim3(cs * 64);
    int nc = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k_sync, &cfg);
    printf("cluster %d x %d thr, %zu KB smem: max active clusters %d (%s)\n", cs, threads,
           smem / 1024, nc, cudaGetErrorString(e));
  }
  double* out; cudaMalloc(&out, 1 << 24);
  at[0].val.clusterDim.x = 16;
  cfg.gridDim = dim3(16 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_sync, 10000, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("8 clusters of 16: 10000 cluster.sync+DSMEM: %.3f ms -> %.3f us each (%s)\n", ms,
           ms * 1e3 / 10000, cudaGetErrorString(e ? e : cudaGetLastError()));
  }
  // FP64 FMA-free? (b*c + a with --fmad=false -> DMUL + DADD)
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_fp64<<<148 * 4, 512>>>(20000, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * 4 * 512 * 20000 * 8;
    printf("fp64 mul+add: %.2f Tops/s\n", ops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
