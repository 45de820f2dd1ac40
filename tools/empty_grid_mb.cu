#include <cstdio>
#include <cstdint>
__global__ void k_flag(const uint8_t* f, uint32_t n, uint32_t* out) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  if (i < n && f[i]) atomicAdd(out, 1u);
}
__global__ void k_tile(const uint8_t* tilef, uint32_t* out) {
  __shared__ int go;
  if (threadIdx.x == 0) go = tilef[blockIdx.x];
  __syncthreads();
  if (go) atomicAdd(out, 1u);
}
__global__ void k_vec(const uint4* f, uint32_t n16, uint32_t* out) {
  const uint32_t i = blockIdx.x * 256 + threadIdx.x;
  if (i < n16) { uint4 v = f[i]; if (v.x | v.y | v.z | v.w) atomicAdd(out, 1u); }
}
int main() {
  const uint32_t n = 16u << 20;  // 16.4 M items (D: vertices + hoods)
  uint8_t* f; uint32_t* out; cudaMalloc(&f, n); cudaMemset(f, 0, n); cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a); for (int i = 0; i < 20; ++i) k_flag<<<n / 256, 256>>>(f, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("per-item flag, %u blocks: %.2f us\n", n / 256, ms * 1000 / 20);
    cudaEventRecord(a); for (int i = 0; i < 20; ++i) k_tile<<<n / 256, 256>>>(f, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("per-tile flag, %u blocks: %.2f us\n", n / 256, ms * 1000 / 20);
    cudaEventRecord(a); for (int i = 0; i < 20; ++i) k_vec<<<n / 16 / 256, 256>>>((const uint4*)f, n / 16, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("16 flags/thread, %u blocks: %.2f us\n", n / 16 / 256, ms * 1000 / 20);
  }
  return 0;
}
