// Reference point only (not product code): time CUB's onesweep radix sort of
// 67M (uint32 key, uint32 value) pairs over 22 key bits, as a target for the
// hand-written stable passes in csrc/radix.cuh.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
__global__ void fill(uint32_t* k, uint32_t* v, size_t n, int bits) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) { uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15; k[i] = h & ((1u << bits) - 1); v[i] = (uint32_t)i; }
}
int main() {
  size_t n = 1ull << 26; int bits = 22;
  uint32_t *k0, *k1, *v0, *v1; cudaMalloc(&k0, n*4); cudaMalloc(&k1, n*4); cudaMalloc(&v0, n*4); cudaMalloc(&v1, n*4);
  fill<<<1184,256>>>(k0, v0, n, bits);
  void* tmp = nullptr; size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, bits);
  cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bb : {22, 16, 11, 8}) {
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, bb);
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("CUB SortPairs n=%zu bits=%d: %.3f ms (%.1f Gpairs/s)\n", n, bb, best, n / best / 1e6);
  }
  return 0;
}
