// Reference point (not product code): CUB's onesweep radix sort on this GPU
// for the two sorts of a C2 frame - 3.8 M (tile id, splat) pairs over 11
// key bits and 0.36 M (depth key, index) pairs over 31 bits.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a cub_sort_bench.cu -o cub_sort_bench
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>

static float time_sort(uint32_t n, int bits, bool clustered) {
  std::vector<uint32_t> hk(n), hv(n);
  std::mt19937 rng(1);
  for (uint32_t i = 0; i < n; ++i) {
    hk[i] = clustered ? (uint32_t)((i / 11 + (rng() % 61)) % 2040) : (rng() & ((1u << bits) - 1));
    hv[i] = i;
  }
  uint32_t *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, 4 * n); cudaMalloc(&k1, 4 * n); cudaMalloc(&v0, 4 * n); cudaMalloc(&v1, 4 * n);
  cudaMemcpy(k0, hk.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(v0, hv.data(), 4 * n, cudaMemcpyHostToDevice);
  cub::DoubleBuffer<uint32_t> dk(k0, k1), dv(v0, v1);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, bits);
  void* tmp; cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, 0, bits);
  cudaEventRecord(a);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, 0, bits);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(tmp);
  return 1e3f * ms / reps;
}

int main() {
  printf("cub SortPairs 3.8M x 11 bits (clustered tiles): %.1f us\n", time_sort(3800000, 11, true));
  printf("cub SortPairs 3.8M x 11 bits (uniform):         %.1f us\n", time_sort(3800000, 11, false));
  printf("cub SortPairs 0.36M x 31 bits:                   %.1f us\n", time_sort(360000, 31, false));
  return 0;
}
