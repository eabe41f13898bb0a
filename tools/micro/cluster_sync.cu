// Microbenchmark: cost of the cluster solver's synchronisation patterns on
// one 16-CTA cluster (512 threads, 1 CTA/SM), clock64 cycles per iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cs tools/micro/cluster_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr int T = 512;

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(T, 1) k(long long* out, int mode, int nst) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  __shared__ double* peers[16];
  __shared__ double scratch[128];
  __shared__ uint64_t mbar2[2];
  if (threadIdx.x < 16) peers[threadIdx.x] = cl.map_shared_rank(sm, threadIdx.x);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar2[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  double acc = threadIdx.x;
  long long t0 = 0;
  for (int it = 0; it < 40; ++it) {
    if (it == 8) t0 = clock64();
    if (mode == 0) {
      cl.sync();
    } else if (mode == 1) {
      // nst remote stores per thread spread over all peers, then sync
      for (int j = 0; j < nst; ++j) {
        const int dst = (threadIdx.x + j * 7 + rank) & 15;
        peers[dst][(threadIdx.x * nst + j) & 8191] = acc + j;
      }
      cl.sync();
    } else if (mode == 2) {
      // the same stores to the own CTA through the cluster window
      for (int j = 0; j < nst; ++j) peers[rank][(threadIdx.x * nst + j) & 8191] = acc + j;
      cl.sync();
    } else if (mode == 3) {
      // plain local shared stores
      for (int j = 0; j < nst; ++j) sm[(threadIdx.x * nst + j) & 8191] = acc + j;
      cl.sync();
    } else if (mode == 4) {
      // block sum of 3 values + cluster exchange + sum (cl_cluster_sum3 shape)
      double w[3] = {acc, acc + 1, acc + 2};
      for (int q = 0; q < 3; ++q)
        for (int o = 16; o > 0; o >>= 1) w[q] += __shfl_down_sync(0xffffffffu, w[q], o);
      const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
      __syncthreads();
      if (l == 0)
        for (int q = 0; q < 3; ++q) scratch[q * 16 + wi] = w[q];
      __syncthreads();
      if (threadIdx.x < 32) {
        for (int q = 0; q < 3; ++q) {
          double t = threadIdx.x < 16 ? scratch[q * 16 + threadIdx.x] : 0.0;
          for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
          t = __shfl_sync(0xffffffffu, t, 0);
          if (threadIdx.x < 16) peers[threadIdx.x][8192 + ((it * 3 + q) & 15) * 16 + rank] = t;
        }
      }
      cl.sync();
      if (threadIdx.x < 32) {
        for (int q = 0; q < 3; ++q) {
          double t = threadIdx.x < 16 ? sm[8192 + ((it * 3 + q) & 15) * 16 + threadIdx.x] : 0.0;
          for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
          if (threadIdx.x == 0) scratch[48 + q] = t;
        }
      }
      __syncthreads();
      acc += scratch[48] * 1e-30;
    } else if (mode == 5) {
      // split barrier: arrive.release ... wait.acquire with nothing between
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 6) {
      // relaxed arrive (no release fence)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    } else if (mode == 7) {
      // remote stores + fence.acq_rel.cluster + relaxed arrive
      for (int j = 0; j < nst; ++j) {
        const int dst = (threadIdx.x + j * 7 + rank) & 15;
        peers[dst][(threadIdx.x * nst + j) & 8191] = acc + j;
      }
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 8) {
      __syncthreads();
    } else if (mode == 10) {
      // remote stores, fence by the writers, relaxed arrive, acquire wait
      for (int j = 0; j < nst; ++j) {
        const int dst = (threadIdx.x + j * 7 + rank) & 15;
        peers[dst][(threadIdx.x * nst + j) & 8191] = acc + j;
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (mode == 11) {
      // st.async remote stores completing on the destination's mbarrier; each
      // CTA waits on its own mbarrier for the bytes it receives (no barrier)
      // two barriers alternating by iteration: a producer can run at most one
      // iteration ahead of any consumer (it waits for everyone's bytes)
      const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar2[it & 1]);
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(T * nst * 8) : "memory");
      for (int j = 0; j < nst; ++j) {
        const int dst = (threadIdx.x + j * 7 + rank) & 15;
        const unsigned la = (unsigned)__cvta_generic_to_shared(sm + (((it & 1) * T * nst + threadIdx.x * nst + j) & 8191));
        unsigned ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(dst));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mb), "r"(dst));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(acc + j), "r"(rb) : "memory");
      }
      unsigned ok = 0;
      for (long spin = 0; !ok && spin < (1L << 24); ++spin) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(mb), "r"((unsigned)((it >> 1) & 1)) : "memory");
      }
      if (!ok) out[100] = 1;  // timed out
    } else if (mode == 9) {
      // sum3 with tagged 16-byte DSMEM words polled by the consumers instead
      // of a cluster barrier (two parity buffers of [3][16] {value, tag})
      double w[3] = {acc, acc + 1, acc + 2};
      for (int q = 0; q < 3; ++q)
        for (int o = 16; o > 0; o >>= 1) w[q] += __shfl_down_sync(0xffffffffu, w[q], o);
      const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
      if (l == 0)
        for (int q = 0; q < 3; ++q) scratch[q * 16 + wi] = w[q];
      __syncthreads();
      const double tag = (double)(it + 1);
      double* box = sm + 8192 + 256 + (it & 1) * 96;  // [3][16][2]
      if (threadIdx.x < 48) {
        const int q = threadIdx.x >> 4, dst = threadIdx.x & 15;
        double t = 0.0;
        for (int i = 0; i < 16; ++i) t += scratch[q * 16 + i];
        double* rb = peers[dst] + 8192 + 256 + (it & 1) * 96 + (q * 16 + rank) * 2;
        unsigned long long ra;
        asm volatile("cvta.to.shared.u64 %0, %1;" : "=l"(ra) : "l"(rb));
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"l"(ra), "d"(t), "d"(tag) : "memory");
      }
      if (threadIdx.x < 48) {
        const int q = threadIdx.x >> 4, src = threadIdx.x & 15;
        const double* mine = box + (q * 16 + src) * 2;
        double v, g;
        do {
          asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(g) : "r"((unsigned)__cvta_generic_to_shared(mine)) : "memory");
        } while (g != tag);
        scratch[48 + threadIdx.x] = v;
      }
      __syncthreads();
      if (threadIdx.x < 3) {
        double t = 0.0;
        for (int i = 0; i < 16; ++i) t += scratch[48 + threadIdx.x * 16 + i];
        scratch[96 + threadIdx.x] = t;
      }
      __syncthreads();
      acc += scratch[96] * 1e-30;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[rank] = (t1 - t0) / 32;
  if (acc == -1.0) out[99] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 128 * sizeof(long long));
  if (getenv("MODE_MIN")) { }
  const size_t smem = (8192 + 512) * 8;
  cudaMemset(d, 0, 128 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"cl.sync only", "remote st + sync", "own-window st + sync", "local st + sync",
                         "sum3 pattern", "arrive.rel/wait.acq", "arrive.relaxed/wait",
                         "remote st + rel/acq", "__syncthreads", "sum3 tagged polling", "remote st + fence + relaxed", "st.async + mbarrier"};
  for (int mode = 0; mode < 12; ++mode) {
    for (int nst : {0, 2, 7}) {
      if ((mode == 0 || mode == 4 || mode == 5 || mode == 6 || mode == 8 || mode == 9) && nst) continue;
      k<<<16, T, smem>>>(d, mode, nst);
      long long h[16];
      cudaError_t e = cudaMemcpy(h, d, 16 * sizeof(long long), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long mx = 0, mn = 1LL << 60;
      for (int i = 0; i < 16; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; }
      printf("%-24s stores/thread %d: %lld..%lld cycles/iter\n", names[mode], nst, mn, mx);
      fflush(stdout);
    }
  }
  return 0;
}
