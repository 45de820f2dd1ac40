// Latency of the M-step's tree helpers (csrc/fold_trees.cuh) in isolation:
// one warp, partials in global memory (L2-resident), cycles per call.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_05018_b200/csrc/fold_trees.cuh"

using namespace dpmrf_b200;

__global__ void k(const double* p, uint32_t cnt, int reps, long long* cyc, double* out) {
  __shared__ double q[kTreeScratch];
  double acc = 0;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) acc += warp_tree<true>(p + r * 8, cnt, q);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / reps;
    out[0] = acc;
  }
}

int main() {
  double *p, *out;
  long long* c;
  cudaMalloc(&p, (1 << 20) * 8);
  cudaMemset(p, 0, (1 << 20) * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&c, 64);
  for (uint32_t cnt : {32u, 50u, 200u, 256u, 300u, 1024u}) {
    k<<<1, 32>>>(p, cnt, 4, c, out);
    k<<<1, 32>>>(p, cnt, 16, c, out);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("warp_tree cnt %4u: %lld cycles/call\n", cnt, h);
  }
  return 0;
}
