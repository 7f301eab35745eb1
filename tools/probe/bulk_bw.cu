// Microbenchmark: global -> shared streaming bandwidth of cp.async.bulk
// (non-tensor TMA) per CTA, with a ring of S stages of B bytes, one CTA per
// SM, one producer lane, consumers only release (no compute).  Compared with
// plain coalesced LDG.128 streaming of the same buffer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_par(uint32_t bar, uint32_t par) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(par) : "memory");
  } while (!done);
}

__global__ void k_bulk(const char* src, size_t per_cta, int S, int B, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)S * B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * per_cta;
  const int64_t n = per_cta / B;
  if (warp == 0) {
    if (lane) return;
    for (int64_t p = 0; p < n; ++p) {
      const int s = (int)(p % S);
      const uint32_t r = (uint32_t)(p / S);
      wait_par(su32(bars + S + s), (r & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bars + s)), "r"(B) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + (size_t)s * B)), "l"(base + p * B), "r"(B), "r"(su32(bars + s)) : "memory");
    }
    return;
  }
  // consumer warps: warp w takes pieces w-1, w-1+nc, ...
  const int nc = (blockDim.x >> 5) - 1;
  double acc = 0;
  for (int64_t p = warp - 1; p < n; p += nc) {
    const int s = (int)(p % S);
    wait_par(su32(bars + s), (uint32_t)((p / S) & 1));
    acc += reinterpret_cast<const double*>(sm + (size_t)s * B)[lane];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bars + S + s)) : "memory");
  }
  if (acc == 12345.0) sink[0] = acc;
}

__global__ void k_ldg(const double2* src, size_t n2, double* sink) {
  double2 acc{0, 0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(src + i);
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 12345.0) sink[0] = acc.y;
}

int main() {
  const size_t bytes = (size_t)8 << 30;
  char* buf; double* sink;
  cudaMalloc(&buf, bytes); cudaMalloc(&sink, 8);
  cudaMemset(buf, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  k_ldg<<<sms * 4, 512>>>((const double2*)buf, bytes / 16, sink);
  cudaEventRecord(e0); k_ldg<<<sms * 4, 512>>>((const double2*)buf, bytes / 16, sink); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("LDG.128 stream: %.1f GB/s\n", bytes / ms / 1e6);
  const int cfgs[][3] = {{24, 8192, 13}, {12, 16384, 13}, {6, 32768, 7}, {4, 49152, 5}, {2, 98304, 3}, {24, 8192, 5}, {48, 4096, 13}};
  for (auto& c : cfgs) {
    const int S = c[0], B = c[1], warps = c[2];
    const size_t per = (bytes / sms) / B * B;
    const size_t smem = (size_t)S * B + 16 * S;
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bulk<<<sms, 32 * warps, smem>>>(buf, per, S, B, sink);
    cudaEventRecord(e0); k_bulk<<<sms, 32 * warps, smem>>>(buf, per, S, B, sink); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("bulk S=%2d B=%6d consumers=%2d: %.1f GB/s %s\n", S, B, warps - 1, per * sms / ms / 1e6, cudaGetErrorString(err));
  }
  return 0;
}
