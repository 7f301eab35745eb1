// Microbenchmark: cost of one grid-wide barrier (no work between barriers),
// one CTA per SM, cooperative launch.  Variants:
//   0  every CTA: bar.sync; thread 0 atom.add.release.gpu on one word, spin on
//      ld.acquire.gpu until bit 31 flips; bar.sync            (the sweeps' and legs' barrier)
//   1  as 0 but each CTA first writes 64 scattered doubles (the release has
//      stores to drain, as in a sweep step)
//   2  hierarchical: barrier.cluster (clusters of C CTAs), one atomic per
//      cluster (its rank-0 CTA), that CTA polls, barrier.cluster again
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_flat(unsigned* bar, int iters, int stores, double* junk) {
  unsigned old = 0;
  for (int it = 0; it < iters; ++it) {
    if (stores && threadIdx.x < 64) junk[((size_t)blockIdx.x * 64 + threadIdx.x) * 97 % (1 << 22)] += 1.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while (((cur ^ old) & 0x80000000u) == 0);
    }
    __syncthreads();
  }
}

__global__ void k_hier(unsigned* bar, int iters, int stores, double* junk) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned nclus = gridDim.x / cl.num_blocks();
  const bool lead = cl.block_rank() == 0;
  const unsigned cid = blockIdx.x / cl.num_blocks();
  unsigned old = 0;
  for (int it = 0; it < iters; ++it) {
    if (stores && threadIdx.x < 64) junk[((size_t)blockIdx.x * 64 + threadIdx.x) * 97 % (1 << 22)] += 1.0;
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (lead && threadIdx.x == 0) {
      const unsigned inc = cid == 0 ? 0x80000000u - (nclus - 1) : 1u;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(bar), "r"(inc) : "memory");
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      } while (((cur ^ old) & 0x80000000u) == 0);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

int main() {
  unsigned* bar;
  double* junk;
  cudaMalloc(&bar, 4);
  cudaMemset(bar, 0, 4);
  cudaMalloc(&junk, 8 << 22);
  cudaMemset(junk, 0, 8 << 22);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int stores = 0; stores < 2; ++stores) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k_flat, bar, iters, stores, junk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("flat  G=%d stores=%d: %.3f us per barrier (%s)\n", sms, stores, 1e3 * ms / iters,
                           cudaGetErrorString(cudaGetLastError()));
    }
    for (int C : {2, 4}) {
      const int G = sms / C * C;
      for (int rep = 0; rep < 3; ++rep) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = C;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, k_hier, &cfg);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_hier, bar, iters, stores, junk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2)
          printf("hier  C=%d G=%d (max active clusters %d) stores=%d: %.3f us per barrier (%s / %s)\n", C, G, ncl, stores,
                 1e3 * ms / iters, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
