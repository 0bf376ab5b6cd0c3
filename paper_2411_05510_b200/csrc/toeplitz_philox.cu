// A2 block-Toeplitz assembly (Eq. 6) and A3 Philox Gaussian sketch
// (Eq. 14; generator reading A-11).
#include "covariance.cuh"

namespace ssi {
namespace {

// T[r*l+a][c*l+b] = R[(i+r-c)-1][a][b]. One thread writes two adjacent columns of a
// row (16-byte store when aligned); pure store-bandwidth kernel, R stays in L2.
// One CTA per row of T: row (r, a) is the concatenation over block columns c of the rows
// R_{i+r-c}[a][:] (Eq. 6), i.e. i contiguous copies of l doubles -- streamed as 16-byte vectors
// (l even and aligned rows; a scalar loop otherwise). Write-bound (m^2 doubles).
__global__ void __launch_bounds__(256) toeplitz_kernel(const double* __restrict__ R, int l, int i,
                                                       double* __restrict__ T, int64_t ldT, int vec) {
  const int row = blockIdx.x;
  const int r = row / l, a = row - r * l;
  const int64_t ll = int64_t(l) * l;
  double* dst = T + int64_t(row) * ldT;
  const double* src0 = R + int64_t(i + r - 1) * ll + int64_t(a) * l;   // block column c = 0
  if (vec) {
    const int hl = l >> 1, np = hl * i;
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int c = e / hl, k = e - c * hl;
      const double2 v = __ldg(reinterpret_cast<const double2*>(src0 - int64_t(c) * ll) + k);
      __stcs(reinterpret_cast<double2*>(dst + int64_t(c) * l) + k, v);
    }
  } else {
    const int m = l * i;
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
      const int c = e / l, b = e - c * l;
      dst[e] = __ldg(src0 - int64_t(c) * ll + b);
    }
  }
}

// Philox4x32-10 (Salmon et al. SC'11): M0 = 0xD2511F53, M1 = 0xCD9E8D57,
// Weyl key increments 0x9E3779B9, 0xBB67AE85.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ uint4 pair_words(uint64_t p, uint64_t seed, uint64_t sid) {
  return philox4x32_10(make_uint4(uint32_t(p), uint32_t(p >> 32), uint32_t(sid), uint32_t(sid >> 32)),
                       make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
}

__global__ void philox_words_kernel(uint64_t seed, uint64_t sid, int64_t n, uint4* out) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    out[p] = pair_words(uint64_t(p), seed, sid);
}

// Omega (m x k col-major, ld): element e = col*m + row, pair p = e/2;
// u = (53-bit word + 0.5) * 2^-53; Box-Muller in FP64: even e -> r cos, odd e -> r sin.
__global__ void sketch_kernel(int m, int k, uint64_t seed, uint64_t sid, double* omega, int64_t ld) {
  const int64_t n = int64_t(m) * k;
  const int64_t np = (n + 1) / 2;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < np;
       p += int64_t(gridDim.x) * blockDim.x) {
    const uint4 w = pair_words(uint64_t(p), seed, sid);
    const uint64_t a = (uint64_t(w.x) | (uint64_t(w.y) << 32)) >> 11;
    const uint64_t b = (uint64_t(w.z) | (uint64_t(w.w) << 32)) >> 11;
    const double u1 = (double(a) + 0.5) * 0x1.0p-53;
    const double u2 = (double(b) + 0.5) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(2.0 * 3.141592653589793 * u2, &sn, &cs);   // same argument rounding as the oracle
    const int64_t e0 = 2 * p;
    const double val[2] = {rad * cs, rad * sn};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int64_t e = e0 + q;
      if (e < n) omega[(e % m) + (e / m) * ld] = val[q];
    }
  }
}

}  // namespace

ssi_status toeplitz_launch(const double* R, int l, int i, double* T, int64_t ldT, cudaStream_t s) {
  const int64_t m = int64_t(l) * i;
  if (m > 2147483647) {
    set_last_error("ssi_toeplitz: m = %lld too large", (long long)m);
    return SSI_ERR_INVALID_ARG;
  }
  const int vec = ((l & 1) == 0 && (ldT & 1) == 0 && ((reinterpret_cast<uintptr_t>(R) | reinterpret_cast<uintptr_t>(T)) & 15) == 0) ? 1 : 0;
  toeplitz_kernel<<<unsigned(m), 256, 0, s>>>(R, l, i, T, ldT, vec);
  return launch_check("toeplitz_kernel");
}

ssi_status sketch_launch(int m, int k, uint64_t seed, uint64_t sid, double* omega, int64_t ldo,
                         cudaStream_t s) {
  const int64_t np = (int64_t(m) * k + 1) / 2;
  int64_t blocks = (np + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  sketch_kernel<<<int(blocks), 256, 0, s>>>(m, k, seed, sid, omega, ldo);
  return launch_check("sketch_kernel");
}

ssi_status philox_words_launch(uint64_t seed, uint64_t sid, int64_t n, uint32_t* words,
                               cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  philox_words_kernel<<<int(blocks), 256, 0, s>>>(seed, sid, n, reinterpret_cast<uint4*>(words));
  return launch_check("philox_words_kernel");
}

}  // namespace ssi
