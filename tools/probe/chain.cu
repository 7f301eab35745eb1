// Store -> remote-poll latency along a chain of warps on different SMs:
// warp i spins (ld.relaxed.gpu) on slot[i-1], then stores slot[i]
// (st.relaxed.gpu).  Prints ns per hop.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 chain.cu -o chain
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

template <int kMode>
__global__ void chain(unsigned long long* slot, int hops, int stride, unsigned long long epoch, long long* out) {
  // block b, warp 0 handles hops h with h % gridDim.x == b  (consecutive hops on different SMs)
  if (threadIdx.x != 0) return;
  long long t0 = 0;
  for (int h = blockIdx.x; h < hops; h += gridDim.x) {
    if (h > 0) {
      const unsigned long long* p = slot + (size_t)(h - 1) * stride;
      if (kMode == 0) while (ldr(p) != epoch) {}
      else while (ldv(p) != epoch) {}
    }
    if (h == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (kMode == 0) str(slot + (size_t)h * stride, epoch);
    else *(volatile unsigned long long*)(slot + (size_t)h * stride) = epoch;
    if (h == hops - 1) {
      long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      out[0] = t1;
    }
    if (h == 0) out[1] = t0;
  }
}

int main() {
  const int hops = 4096, stride = 32;
  unsigned long long* slot;
  long long* out;
  cudaMalloc(&slot, sizeof(unsigned long long) * hops * stride);
  cudaMalloc(&out, 16);
  cudaMemset(slot, 0, sizeof(unsigned long long) * hops * stride);
  for (int mode = 0; mode < 2; ++mode)
    for (int grid : {2, 16, 148}) {
      for (int rep = 0; rep < 3; ++rep) {
        const unsigned long long epoch = 1000 + mode * 100 + grid * 3 + rep;
        if (mode == 0) chain<0><<<grid, 32>>>(slot, hops, stride, epoch, out);
        else chain<1><<<grid, 32>>>(slot, hops, stride, epoch, out);
        cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        if (rep == 2) printf("mode %s grid %3d: %.1f ns per hop\n", mode ? "volatile" : "relaxed.gpu", grid,
                             (double)(h[0] - h[1]) / (hops - 1));
      }
    }
  return 0;
}
