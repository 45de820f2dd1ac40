// microbench.cu -- latency probes that shape the optimization-phase design on
// B200: dependent DADD chain, dependent LDS->DADD chain, cooperative grid
// barrier cost vs grid size, and back-to-back empty kernels in a CUDA graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cooperative_groups.h>
#include "../paper_1809_05018_b200/csrc/common.cuh"
#include <chrono>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

__global__ void dadd_chain(double* out, double x, int n, long long* cycles) {
  double acc = x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x);
  const long long t1 = clock64();
  out[0] = acc;
  cycles[0] = t1 - t0;
}

// Dependent FP64 op chains: DFMA, DMUL, correctly rounded div / sqrt.
template <int kOp>
__global__ void fp64_chain(double* out, double x, int n, long long* cycles) {
  double acc = x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (kOp == 0) acc = __fma_rn(acc, x, 1e-300);
    if (kOp == 1) acc = __dmul_rn(acc, x);
    if (kOp == 2) acc = __ddiv_rn(x, acc);
    if (kOp == 3) acc = __dsqrt_rn(acc);
    if (kOp == 4) acc = log(acc + 2.0);
    if (kOp == 5) acc = dpmrf_b200::log_cr(acc + 2.0);
  }
  const long long t1 = clock64();
  out[0] = acc;
  cycles[0] = t1 - t0;
}

__global__ void lds_chain(double* out, int n, long long* cycles) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  if (threadIdx.x) return;
  double acc = 0.0;
  const long long t0 = clock64();
  for (int r = 0; r < n / 1024; ++r)
#pragma unroll 8
    for (int i = 0; i < 1024; ++i) acc = __dadd_rn(acc, s[i]);
  const long long t1 = clock64();
  out[0] = acc;
  cycles[0] = t1 - t0;
}

// The leaf-fold chain as k_leaf_fold runs it: 8 lanes of one warp, each a
// 1023-add dependent chain over its own shared-memory row (stride 1025),
// next 16 operands loaded while the current 16 adds retire.
__global__ void leaf_chain_smem(double* out, long long* cycles) {
  __shared__ double s[4 * 1025];  // (48 KB static limit: 4 rows)
  for (int i = threadIdx.x; i < 4 * 1025; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  if (threadIdx.x >= 4) return;
  const double* v = s + threadIdx.x * 1025;
  const long long t0 = clock64();
  constexpr int kG = 16;
  double acc = v[0], cur[kG], nxt[kG];
  unsigned i = 1;
#pragma unroll
  for (int j = 0; j < kG; ++j) cur[j] = v[i + j];
  while (i + 2 * kG <= 1024) {
#pragma unroll
    for (int j = 0; j < kG; ++j) nxt[j] = v[i + kG + j];
#pragma unroll
    for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
#pragma unroll
    for (int j = 0; j < kG; ++j) cur[j] = nxt[j];
    i += kG;
  }
#pragma unroll
  for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
  i += kG;
  for (; i < 1024; ++i) acc = __dadd_rn(acc, v[i]);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

// The M-step's fold_span (common path of the fold kernels) on 2 lanes of a
// one-warp block; cycles AND globaltimer ns (-> the SM clock during the chain).
__device__ __noinline__ double dpmrf_probe_fold(const double* v, uint32_t i, uint32_t end, double acc) {
  constexpr int kG = 16;
  double cur[kG], nxt[kG];
  if (i + kG <= end) {
#pragma unroll
    for (int j = 0; j < kG; ++j) cur[j] = v[i + j];
    while (i + 2 * kG <= end) {
#pragma unroll
      for (int j = 0; j < kG; ++j) nxt[j] = v[i + kG + j];
#pragma unroll
      for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
#pragma unroll
      for (int j = 0; j < kG; ++j) cur[j] = nxt[j];
      i += kG;
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
    i += kG;
  }
  for (; i < end; ++i) acc = __dadd_rn(acc, v[i]);
  return acc;
}

__global__ void fold_span_probe(double* out, long long* cycles) {
  __shared__ __align__(16) double s[2][1026];
  for (int i = threadIdx.x; i < 2 * 1026; i += blockDim.x) (&s[0][0])[i] = 1.0 + i * 1e-9;
  __syncwarp();
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long t0 = clock64();
  double acc = 0.0;
  if (threadIdx.x < 2) {
    const double* v = s[threadIdx.x];
    acc = dpmrf_probe_fold(v, 1, 1024, v[0]);
  }
  const long long t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    cycles[0] = t1 - t0;
    cycles[1] = (long long)(g1 - g0);
  }
}

// Same chain with operands already in registers (the DADD-latency floor).
__global__ void leaf_chain_regs(double* out, long long* cycles) {
  if (threadIdx.x >= 8) return;
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = 1.0 + (threadIdx.x * 32 + j) * 1e-9;
  const long long t0 = clock64();
  double acc = r[0];
  for (int rep = 0; rep < 32; ++rep)
#pragma unroll
    for (int j = 0; j < 32; ++j) acc = __dadd_rn(acc, r[j]);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

__global__ void grid_barriers(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) sink[0] = iters;
}

// Hand-rolled grid barrier: one release-add per block on a monotone counter,
// thread 0 spins with acquire loads until the counter reaches the epoch target.
__device__ __forceinline__ void flag_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void flag_barriers(int iters, unsigned* ctr) {
  for (int i = 0; i < iters; ++i) flag_barrier(ctr, (i + 1u) * gridDim.x);
}

__global__ void wide_empty(int* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1;
}

__global__ void empty_kernel(int* sink) {
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] += 1;
}

int main() {
  double* d;
  long long* c;
  int* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&c, 64);
  cudaMalloc(&sink, 64);
  long long h;
  const int n = 1 << 20;
  int l2 = 0, persist = 0, window = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&window, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  printf("L2 %d MB, max persisting L2 %d MB, max access-policy window %d MB\n", l2 >> 20,
         persist >> 20, window >> 20);
  dadd_chain<<<1, 1>>>(d, 1e-9, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.2f cycles/op\n", double(h) / n);
  {
    const char* names[] = {"DFMA", "DMUL", "__ddiv_rn", "__dsqrt_rn", "log (libdevice)", "log_cr"};
    const int ns[] = {n, n, 1 << 14, 1 << 14, 1 << 12, 1 << 10};
    for (int op = 0; op < 6; ++op) {
      switch (op) {
        case 0: fp64_chain<0><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
        case 1: fp64_chain<1><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
        case 2: fp64_chain<2><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
        case 3: fp64_chain<3><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
        case 4: fp64_chain<4><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
        case 5: fp64_chain<5><<<1, 1>>>(d, 1.0000001, ns[op], c); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("dependent %s: %.2f cycles/op\n", names[op], double(h) / ns[op]);
    }
  }
  {
    long long hc[2];
    for (int rep = 0; rep < 3; ++rep) {
      fold_span_probe<<<1, 32>>>(d, c);
      cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
      printf("fold_span 1023 adds: %lld cycles, %lld ns -> %.0f MHz, %.2f cycles/add\n", hc[0], hc[1],
             1e3 * hc[0] / double(hc[1]), hc[0] / 1023.0);
    }
  }
  lds_chain<<<1, 256>>>(d, n, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent LDS+DADD fold (unroll 8): %.2f cycles/element\n", double(h) / n);
  leaf_chain_smem<<<1, 256>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("leaf chain (4 lanes, smem rows, 16-deep prefetch): %.2f cycles/add\n", double(h) / 1023);
  leaf_chain_regs<<<1, 32>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("leaf chain (8 lanes, register operands): %.2f cycles/add\n", double(h) / 1024);
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, grid_barriers, 256, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocks : {sms, 2 * sms, 4 * sms, per * sms}) {
    int iters = 1000;
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)grid_barriers, blocks, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)grid_barriers, blocks, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync with %d blocks x 256: %.2f us/barrier\n", blocks, ms * 1e3 / iters);
  }
  for (int threads : {512, 1024}) {
    int iters = 1000;
    void* args[] = {&iters, &sink};
    cudaLaunchCooperativeKernel((void*)grid_barriers, sms, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)grid_barriers, sms, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync with %d blocks x %d: %.2f us/barrier\n", sms, threads, ms * 1e3 / iters);
  }
  unsigned* ctr;
  cudaMalloc(&ctr, 64);
  for (int blocks : {sms, 4 * sms, 8 * sms}) {
    int iters = 1000;
    cudaMemset(ctr, 0, 64);
    void* args[] = {&iters, &ctr};
    cudaLaunchCooperativeKernel((void*)flag_barriers, blocks, 256, args, 0, 0);
    cudaMemset(ctr, 0, 64);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)flag_barriers, blocks, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("flag barrier with %d blocks x 256: %.2f us/barrier\n", blocks, ms * 1e3 / iters);
  }
  // 1000 dependent empty kernels captured in a graph
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 1000; ++i) empty_kernel<<<1, 32, 0, s>>>(sink);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("graph of 1000 tiny kernels: %.2f us/kernel\n", ms);
  cudaEventRecord(a, s);
  for (int i = 0; i < 1000; ++i) empty_kernel<<<1, 32, 0, s>>>(sink);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("stream of 1000 tiny kernels: %.2f us/kernel\n", ms);
  for (int blocks : {sms * 8, 1600}) {
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 1000; ++i) wide_empty<<<blocks, 256, 0, s>>>(sink);
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    cudaGraphLaunch(ge2, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge2, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of 1000 empty kernels x %d blocks x 256: %.2f us/kernel\n", blocks, ms);
  }
  // host round trip: launch + sync of one tiny kernel + 8-byte D2H
  long long* hp;
  cudaMallocHost(&hp, 64);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000; ++i) {
    empty_kernel<<<1, 32, 0, s>>>(sink);
    cudaMemcpyAsync(hp, c, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  }
  auto t1 = std::chrono::steady_clock::now();
  printf("host round trip (launch + D2H + sync): %.2f us\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000);
  return 0;
}
