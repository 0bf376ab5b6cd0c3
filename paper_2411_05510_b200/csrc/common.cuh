// Shared device/host helpers of libssi.so (sm_100a). No method arithmetic lives here.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/ssi.h"

namespace ssi {

// ---------------------------------------------------------------- workspace layout
// Every ws starts with a 256-byte header whose first int32 is the device status word.
constexpr size_t kWsHeader = 256;
constexpr size_t kWsAlign = 256;

// Carves aligned sub-buffers out of a caller workspace. With base == nullptr it only
// counts bytes, so the *_ws() size queries and the real carving share one code path.
struct Carver {
  char* base;
  size_t off;
  explicit Carver(void* b) : base(static_cast<char*>(b)), off(kWsHeader) {}
  template <typename T>
  T* take(size_t n) {
    off = (off + kWsAlign - 1) / kWsAlign * kWsAlign;
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  size_t bytes() const { return (off + kWsAlign - 1) / kWsAlign * kWsAlign; }
};

__device__ __forceinline__ void set_status(int32_t* st, int32_t code) {
  if (st) atomicMax(st, code);
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_{z<n} p[z * stride] in the fixed order z = 0, 1, ... (deterministic split-K reduction);
// loads are issued eight at a time so the L2 latency overlaps instead of chaining.
__device__ __forceinline__ double ordered_sum(const double* __restrict__ p, int64_t stride, int n) {
  double s = 0.0;
  int z = 0;
  for (; z + 8 <= n; z += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(p + int64_t(z + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; z < n; ++z) s += __ldg(p + int64_t(z) * stride);
  return s;
}

// FP64 reciprocal / rsqrt: hardware approximation refined by Newton steps to full precision
// (a few ulp), inline (no call to the IEEE division / sqrt slow-path subroutines).
__device__ __forceinline__ double fast_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  return fma(r, fma(-d, r, 1.0), r);
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double hx = 0.5 * x;
  r = r * fma(-hx * r, r, 1.5);
  r = r * fma(-hx * r, r, 1.5);
  return r * fma(-hx * r, r, 1.5);
}

// ---------------------------------------------------------------- FP64 tensor core
// mma.sync m8n8k4 f64 (SASS DMMA.8x8x4). Fragments (PTX ISA, m8n8k4 .f64):
//   A 8x4 row : lane holds A[lane>>2][lane&3]
//   B 4x8 col : lane holds B[lane&3][lane>>2]
//   C 8x8     : lane holds C[lane>>2][2*(lane&3) + {0,1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace ssi

// ---------------------------------------------------------------- host-side error state
namespace ssi {
void set_last_error(const char* fmt, ...);
ssi_status launch_check(const char* what);
}  // namespace ssi

#define SSI_REQUIRE(cond, code, ...)          \
  do {                                        \
    if (!(cond)) {                            \
      ::ssi::set_last_error(__VA_ARGS__);     \
      return (code);                          \
    }                                         \
  } while (0)

#define SSI_TRY(expr)                  \
  do {                                 \
    ssi_status _s = (expr);            \
    if (_s != SSI_OK) return _s;       \
  } while (0)
