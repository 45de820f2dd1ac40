// Does reading back data written as partial 32-byte sectors cost a DRAM
// round trip on B200?  Kernel W writes a 1 MB array either with full-sector
// coalesced stores (mode 0) or as two interleaved passes of 8-byte stores from
// different warps (mode 1: every sector written by two partial stores), or
// mode 1 followed by an L2 prefetch of every line (mode 2); kernel R (next
// launch) reads it with plain loads and records per-warp latency.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void w(double* x, int n, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (mode == 0) {
    if (i < n) x[i] = i * 1.5;
  } else {
    // thread i writes element 2*(i%half)+parity with parity from the block half
    const int half = n / 2;
    const int j = i % half, par = i / half;
    if (i < n) x[2 * j + par] = (2 * j + par) * 1.5;
    if (mode == 2 && i < n && (i % 16) == 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(x + 2 * j));
  }
}

__global__ void r(const double* x, int n, unsigned long long* lat, double* sink) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long t0 = gt();
  double v = 0;
  for (int k = 0; k < 8; ++k) {
    const int idx = (i * 8 + k * 32) % n;
    v += __ldcg(x + idx);
  }
  sink[i] = v;
  const unsigned long long t1 = gt();
  if ((threadIdx.x & 31) == 0) lat[i / 32] = t1 - t0;
}

int main() {
  const int n = 1 << 17;  // 1 MB
  double *x, *sink;
  unsigned long long* lat;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&sink, n * 8);
  cudaMalloc(&lat, (n / 32) * 8);
  static unsigned long long h[1 << 12];
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      w<<<n / 256, 256>>>(x, n, mode);
      r<<<n / 256, 256>>>(x, n, lat, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(h, lat, (n / 32) * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0, sum = 0;
      for (int k = 0; k < n / 32; ++k) {
        mx = h[k] > mx ? h[k] : mx;
        sum += h[k];
      }
      printf("mode %d rep %d: read latency per warp avg %.0f ns max %llu ns\n", mode, rep,
             double(sum) / (n / 32), mx);
    }
  }
  return 0;
}
