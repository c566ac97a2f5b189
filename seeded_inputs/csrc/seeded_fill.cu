// Seeded counter-based input generator on the device (bench/test utility).
//
// Independent CUDA implementation of the generator documented in
// seeded_inputs/__init__.py (SplitMix64 counter hash).
// It holds no arithmetic of the allreduce method and is never called by the
// product path (paper_2508_13397_b200/); tests and bench.py use it to fill
// multi-GiB buffers in HBM without a host round trip.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// dtype: 0 int32, 1 float32, 2 bfloat16 (bits).  dist: 0 signed, 1 positive,
// 2 full, 3 ones, 4 ramp.
__device__ __forceinline__ uint32_t value_bits(uint64_t u, uint64_t i, int dtype, int dist) {
  if (dist == 3) return dtype == 0 ? 1u : (dtype == 1 ? 0x3F800000u : 0x3F80u);
  if (dist == 4) {
    if (dtype == 0) return (uint32_t)(i % 4096);
    if (dtype == 1) return __float_as_uint((float)(i % 4096));
    return __float_as_uint((float)(i % 256)) >> 16;
  }
  if (dtype == 0) {
    if (dist == 2) return (uint32_t)(u >> 32);
    int32_t v = (int32_t)((u >> 43) & ((1ull << 21) - 1)) - (1 << 20);
    return (uint32_t)v;
  }
  if (dtype == 1) {
    if (dist == 1) {
      uint32_t m = (uint32_t)((u >> 41) & 0x7FFFFFull);
      return 0x3F800000u | m;  // 1 + m * 2^-23, exact
    }
    int32_t m = (int32_t)((u >> 40) & 0xFFFFFFull) - (1 << 23);
    return __float_as_uint((float)m * 0x1p-23f);  // exact: |m| < 2^24
  }
  uint32_t mant = (uint32_t)((u >> 49) & 0x7F);
  if (dist == 1) return (127u << 7) | mant;
  uint32_t sign = (uint32_t)(u >> 63);
  uint32_t exp = 119u + (uint32_t)((u >> 56) & 7);
  return (sign << 15) | (exp << 7) | mant;
}

__global__ void fill_kernel(void* dst, uint64_t n, uint64_t start, int dtype, int dist,
                            uint64_t key) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    uint64_t i = start + j;
    uint32_t b = value_bits(mix64(key ^ i), i, dtype, dist);
    if (dtype == 2)
      reinterpret_cast<uint16_t*>(dst)[j] = (uint16_t)b;
    else
      reinterpret_cast<uint32_t*>(dst)[j] = b;
  }
}

}  // namespace

extern "C" {

// Fill dst[0..n) with elements [start, start+n) of rank `rank`'s seeded buffer.
// Returns 0 on success, a cudaError_t value otherwise.
int seeded_fill(void* dst, uint64_t n, uint64_t start, int dtype, int dist, uint64_t seed,
                int rank, void* stream) {
  if (n == 0) return 0;
  if (dtype < 0 || dtype > 2 || dist < 0 || dist > 4) return (int)cudaErrorInvalidValue;
  uint64_t key = mix64(seed ^ ((uint64_t)(rank + 1) * 0x9E3779B97F4A7C15ull));
  int threads = 256;
  uint64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  fill_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(dst, n, start, dtype, dist,
                                                                      key);
  return (int)cudaGetLastError();
}

}  // extern "C"
