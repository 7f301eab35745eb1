// Microbenchmarks that shape the solver design: grid barrier latency, graph-launch
// latency, FP64 DGEMM throughput (cuBLAS), L2-resident streaming bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cublas_v2.h>
namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
__device__ unsigned int bar_count = 0;
__device__ volatile unsigned int bar_gen = 0;
__global__ void k_mybar(int iters, int* out) {
  unsigned int nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int gen = bar_gen;
      __threadfence();
      unsigned int t = atomicAdd(&bar_count, 1);
      if (t == nb - 1) { bar_count = 0; __threadfence(); bar_gen = gen + 1; }
      else { while (bar_gen == gen) { } }
      __threadfence();
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
__global__ void k_empty(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = 1; }
__global__ void k_stream(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i] * 1.0000001;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c0 = 0.1, c1 = 0.2, c2 = 0.3, c3 = 0.4, c4=0.5,c5=0.6,c6=0.7,c7=0.8;
  for (int i = 0; i < iters; ++i) {
    c0 = fma(a, b, c0); c1 = fma(a, b, c1); c2 = fma(a, b, c2); c3 = fma(a, b, c3);
    c4 = fma(a, b, c4); c5 = fma(a, b, c5); c6 = fma(a, b, c6); c7 = fma(a, b, c7);
  }
  if (c0+c1+c2+c3+c4+c5+c6+c7 == 1234.5) out[0] = 1;
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d L2 %d MB smem/block optin %zu clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  int* d_out; CK(cudaMalloc(&d_out, 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bps : {1, 2, 4}) for (int th : {256, 512}) {
    int nb = p.multiProcessorCount * bps; int iters = 2000;
    void* args[] = {&iters, &d_out};
    CK(cudaLaunchCooperativeKernel((void*)k_gridsync, nb, th, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)k_gridsync, nb, th, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync blocks=%d threads=%d: %.3f us/sync\n", nb, th, ms * 1000 / iters);
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)k_mybar, nb, th, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("custom barrier blocks=%d threads=%d: %.3f us/sync\n", nb, th, ms * 1000 / iters);
  }
  // graph of empty kernels
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; ++i) k_empty<<<148, 256, 0, s>>>(d_out);
  cudaStreamEndCapture(s, &g); CK(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEventRecord(e0, s); for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(e1, s);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("graph kernel node: %.3f us/launch\n", ms * 1000 / 2000);
  cudaEventRecord(e0, s); for (int r = 0; r < 2000; ++r) k_empty<<<148, 256, 0, s>>>(d_out); cudaEventRecord(e1, s);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("stream launch empty: %.3f us/launch\n", ms * 1000 / 2000);
  // streaming bandwidth at several sizes (L2 resident vs HBM)
  for (size_t mb : {8, 32, 64, 4096}) {
    size_t n = mb * 1024 * 1024 / 8; double *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
    cudaMemset(a, 0, n * 8);
    k_stream<<<p.multiProcessorCount * 8, 256>>>(a, b, n); cudaDeviceSynchronize();
    int reps = mb > 1000 ? 5 : 50;
    cudaEventRecord(e0); for (int r = 0; r < reps; ++r) k_stream<<<p.multiProcessorCount * 8, 256>>>(a, b, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("stream copy %zu MB: %.1f GB/s (%.2f us/launch)\n", mb, 2.0 * n * 8 * reps / (ms * 1e6), ms * 1000 / reps);
    cudaFree(a); cudaFree(b);
  }
  // DFMA throughput
  {
    int iters = 100000; k_dfma<<<p.multiProcessorCount * 8, 256>>>((double*)d_out, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<<<p.multiProcessorCount * 8, 256>>>((double*)d_out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)p.multiProcessorCount * 8 * 256;
    printf("DFMA: %.2f TFLOP/s\n", flops / (ms * 1e9));
  }
  // cuBLAS DGEMM
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {2048, 4096, 8192}) {
    double *A, *B, *C; CK(cudaMalloc(&A, (size_t)n * n * 8)); CK(cudaMalloc(&B, (size_t)n * n * 8)); CK(cudaMalloc(&C, (size_t)n * n * 8));
    cudaMemset(A, 0, (size_t)n*n*8); cudaMemset(B, 0, (size_t)n*n*8);
    double one = 1.0, zero = 0.0;
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("cuBLAS DGEMM n=%d: %.2f TFLOP/s\n", n, 5 * 2.0 * n * (double)n * n / (ms * 1e9));
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  size_t fr, tot; cudaMemGetInfo(&fr, &tot); printf("mem free %.1f GB total %.1f GB\n", fr / 1e9, tot / 1e9);
  return 0;
}
