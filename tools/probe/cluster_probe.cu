// Microbenchmark: cost of barriers available to a latency-bound wavefront sweep.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_cluster_sync(int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) { v = v * 1.0000001 + 1.0; cl.sync(); }
  if (v == 123.0) out[0] = v;
}
__global__ void k_cluster_sync_mem(int iters, double* buf, double* out) {
  // phase: each thread writes one global value, barrier, reads a neighbour's
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank() * blockDim.x + threadIdx.x;
  const int n = cl.num_blocks() * blockDim.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    buf[g] = acc + i;
    cl.sync();
    acc += buf[(g * 7 + 13) % n];
    cl.sync();
  }
  if (acc == 1.5) out[0] = acc;
}
__global__ void k_block_sync(int iters, double* out) {
  double v = threadIdx.x;
  for (int i = 0; i < iters; ++i) { v = v * 1.0000001 + 1.0; __syncthreads(); }
  if (v == 123.0) out[0] = v;
}
__global__ void k_chain(const int* __restrict__ idx, int iters, int* out) {
  // dependent L2 load chain latency
  int j = threadIdx.x;
  for (int i = 0; i < iters; ++i) j = idx[j];
  if (j == -5) out[0] = j;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 24);
  double* buf; cudaMalloc(&buf, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int C : {2, 4, 8, 16}) for (int T : {256, 512, 1024}) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(C); cfg.blockDim = dim3(T);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_cluster_sync_mem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int iters = 2000;
    cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, d); cudaDeviceSynchronize();
    cudaEventRecord(a); cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    float ms2;
    cudaEventRecord(a); cudaLaunchKernelEx(&cfg, k_cluster_sync_mem, iters, buf, d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms2, a, b);
    printf("cluster %2d x %4d threads: cluster.sync %.3f us; write+sync+read+sync %.3f us  (%s)\n", C, T, ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  for (int T : {256, 512, 1024}) {
    int iters = 20000;
    k_block_sync<<<1, T>>>(iters, d); cudaDeviceSynchronize();
    cudaEventRecord(a); k_block_sync<<<1, T>>>(iters, d); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("__syncthreads %4d threads: %.4f us\n", T, ms * 1e3 / iters);
  }
  // dependent load chain: small table (L1/L2-resident) and large (HBM)
  for (int sz : {1024, 1 << 20, 1 << 26}) {
    int* idx; cudaMalloc(&idx, (size_t)sz * 4);
    int* h = new int[sz];
    for (int i = 0; i < sz; ++i) h[i] = (int)(((long long)i * 7919 + 104729) % sz);
    cudaMemcpy(idx, h, (size_t)sz * 4, cudaMemcpyHostToDevice);
    int iters = 10000; int* o; cudaMalloc(&o, 4);
    k_chain<<<1, 32>>>(idx, iters, o); cudaDeviceSynchronize();
    cudaEventRecord(a); k_chain<<<1, 32>>>(idx, iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent load chain, table %d ints: %.1f ns per load\n", sz, ms * 1e6 / iters);
  }
  return 0;
}
