// chain.cu plus, per hop, the flow leg's patch arithmetic: 16 __shfl_sync + a
// 16-deep DFMA chain (and optionally 32 spin-free loads) between the wait and
// the store.  Distinguishes memory latency from instruction-path effects.
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

template <int kWork>
__global__ void chain(unsigned long long* slot, int hops, int stride, unsigned long long epoch, long long* out,
                      const double* binv, double* sink) {
  const int lane = threadIdx.x & 31;
  long long t0 = 0;
  double acc = 0.0;
  for (int h = blockIdx.x; h < hops; h += gridDim.x) {
    if (h > 0 && lane == 0) {
      const unsigned long long* p = slot + (size_t)(h - 1) * stride;
      while (ldr(p) < epoch) {
      }
    }
    __syncwarp();
    if (h == 0 && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (kWork) {
      double v = (double)(lane + h);
      double d = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c) d = fma(binv[lane * 16 + c], __shfl_sync(0xffffffffu, v, c), d);
      acc += d;
      if (d == 1.2345e300) sink[lane] = d;
    }
    if (lane == 0) str(slot + (size_t)h * stride, epoch + (acc == 1.2345e300));
    if (h == hops - 1 && lane == 0) {
      long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      out[0] = t1;
    }
    if (h == 0 && lane == 0) out[1] = t0;
  }
}

int main() {
  const int hops = 4096, stride = 32;
  unsigned long long* slot;
  long long* out;
  double *binv, *sink;
  cudaMalloc(&slot, sizeof(unsigned long long) * hops * stride);
  cudaMalloc(&out, 16);
  cudaMalloc(&binv, 8 * 512);
  cudaMalloc(&sink, 8 * 32);
  cudaMemset(binv, 0, 8 * 512);
  cudaMemset(slot, 0, sizeof(unsigned long long) * hops * stride);
  unsigned long long epoch = 1;
  for (int work = 0; work < 2; ++work)
    for (int grid : {2, 148, 592}) {
      for (int rep = 0; rep < 3; ++rep, ++epoch) {
        if (work) chain<1><<<grid, 32>>>(slot, hops, stride, epoch, out, binv, sink);
        else chain<0><<<grid, 32>>>(slot, hops, stride, epoch, out, binv, sink);
        cudaDeviceSynchronize();
        long long hh[2];
        cudaMemcpy(hh, out, 16, cudaMemcpyDeviceToHost);
        if (rep == 2) printf("work %d grid %3d: %.1f ns per hop\n", work, grid, (double)(hh[0] - hh[1]) / (hops - 1));
      }
    }
  return 0;
}
