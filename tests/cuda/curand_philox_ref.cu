// Test-only helper (P13): raw Philox4x32-10 words from cuRAND's own device function
// curand_Philox4x32_10(uint4 ctr, uint2 key) (curand_philox4x32_x.h), with the same
// counter/key mapping as reading A-11, to check libssi's generator bit for bit.
#include <curand_philox4x32_x.h>
#include <stdint.h>

__global__ void ref_words(uint64_t seed, uint64_t sid, int64_t n, uint4* out) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    uint4 c = make_uint4(uint32_t(p), uint32_t(uint64_t(p) >> 32), uint32_t(sid), uint32_t(sid >> 32));
    uint2 k = make_uint2(uint32_t(seed), uint32_t(seed >> 32));
    out[p] = curand_Philox4x32_10(c, k);
  }
}

extern "C" int curand_ref_words(uint64_t seed, uint64_t sid, int64_t n, void* out) {
  ref_words<<<256, 256>>>(seed, sid, n, static_cast<uint4*>(out));
  return int(cudaDeviceSynchronize());
}
