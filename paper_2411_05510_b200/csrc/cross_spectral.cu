// Cross-spectral product of SSI_COV_SPECTRAL (cov_spectral.cu) with three real products per
// complex one (Gauss): for every frequency f and channel pair (b, a),
//   G_ab(f) = sum_s Ye_{s,a}(f) conj(X_{s,b}(f))
//   T1 = sum_s Xr Yr,  T2 = sum_s Xi Yi,  T3 = sum_s (Xr + Xi)(Yi - Yr)
//   Re G = T1 + T2,   Im G = T3 + T1 - T2
// i.e. 6 lp^2 S flops per frequency instead of 8 lp^2 S for the complex-stacked real GEMM.
// One CTA owns a 64 (b) x 64 (a) tile of one frequency and keeps the three accumulators in
// registers (FP64 DMMA m8n8k4, 8 warps as 2 x 4, warp tile 32 x 16); the operand tiles (16
// segments x 64 channels of interleaved (Re, Im) pairs) are staged by cp.async in a 2-stage ring
// and read as 16-byte (Re, Im) fragments; the sums Xr + Xi and Yi - Yr are formed on the
// fragments. The epilogue writes Re G and Im G (optionally adding to
// them: segment chunks accumulate in a fixed order).
#include "cov_spectral.cuh"

namespace ssi {
namespace {

constexpr int XT = 64;            // tile (b) x (a)
constexpr int XS = 16;            // segments per stage
constexpr int XP = 2 * XT + 4;    // smem pitch of a segment's (Re, Im) x 64 channels: P = 4 (mod 16)
                                  // puts the 8 lanes of a quarter-warp 16-byte fragment load on
                                  // distinct bank groups
constexpr int XNT = 256;
constexpr int XST = 2;            // stages
constexpr int XSTAGE = 2 * XS * XP;   // A segments + B segments per stage

struct XArgs {
  const double* A;   // X spectra  [f][s][lp][Re, Im]
  const double* B;   // Ye spectra [f][s][lp][Re, Im]
  int64_t sF;        // per-frequency stride of A and B (2 S_capacity lp)
  int64_t nseg;      // segments in this chunk
  int lp;
  double* G;         // [f][2][lp][lp]: element (b, a) of part q at f*2lp^2 + q*lp^2 + b + a*lp
  int accum;
};

__device__ __forceinline__ void cpa16(double* dst, const double* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

// stage: segments [s0, s0 + 16) of A (channels b0..b0+63) and B (channels a0..a0+63), one 16-byte
// (Re, Im) piece per channel: 1 KB contiguous per segment and operand
__device__ __forceinline__ void x_load(const XArgs& g, double* st, const double* Af, const double* Bf, int64_t s0,
                                       int b0, int a0) {
  const int tid = threadIdx.x;
  double* As = st;
  double* Bs = st + XS * XP;
#pragma unroll
  for (int q = 0; q < 4; ++q) {           // 16 segments x 64 pieces per operand
    const int p = tid + q * XNT;
    const int sg = p >> 6, c = p & 63;
    const int64_t seg = s0 + sg;
    const bool rv = seg < g.nseg;
    const bool va = rv && b0 + c < g.lp, vb = rv && a0 + c < g.lp;
    cpa16(As + sg * XP + 2 * c, va ? Af + (seg * g.lp + b0 + c) * 2 : Af, va);
    cpa16(Bs + sg * XP + 2 * c, vb ? Bf + (seg * g.lp + a0 + c) * 2 : Bf, vb);
  }
}

__global__ void __launch_bounds__(XNT, 2) cross3m_kernel(XArgs g) {
  extern __shared__ __align__(16) double xs[];
  const int b0 = blockIdx.x * XT, a0 = blockIdx.y * XT;
  const int64_t f = blockIdx.z;
  const double* Af = g.A + f * g.sF;
  const double* Bf = g.B + f * g.sF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int r8 = lane >> 2, kq = lane & 3;
  double t1[4][2][2], t2[4][2][2], t3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;
  const int nst = int((g.nseg + XS - 1) / XS);
  x_load(g, xs, Af, Bf, 0, b0, a0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int it = 0; it < nst; ++it) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (it + 1 < nst) x_load(g, xs + ((it + 1) % XST) * XSTAGE, Af, Bf, int64_t(it + 1) * XS, b0, a0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* As = xs + (it % XST) * XSTAGE;
    const double* Bs = As + XS * XP;
#pragma unroll
    for (int k4 = 0; k4 < XS; k4 += 4) {
      const int s = k4 + kq;                                  // this lane's segment (k index)
      double ar[4], ai[4], as[4], br[2], bi[2], bd[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(As + s * XP + 2 * (wm + 8 * i + r8));
        ar[i] = v.x; ai[i] = v.y;
        as[i] = ar[i] + ai[i];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(Bs + s * XP + 2 * (wn + 8 * j + r8));
        br[j] = v.x; bi[j] = v.y;
        bd[j] = bi[j] - br[j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma884(t1[i][j][0], t1[i][j][1], ar[i], br[j]);
          dmma884(t2[i][j][0], t2[i][j][1], ai[i], bi[j]);
          dmma884(t3[i][j][0], t3[i][j][1], as[i], bd[j]);
        }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  const int64_t lp2 = int64_t(g.lp) * g.lp;
  double* Gre = g.G + f * 2 * lp2;
  double* Gim = Gre + lp2;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = b0 + wm + 8 * i + r8;
        const int a = a0 + wn + 8 * j + 2 * kq + e;
        if (b < g.lp && a < g.lp) {
          const double re = t1[i][j][e] + t2[i][j][e];
          const double im = t3[i][j][e] + (t1[i][j][e] - t2[i][j][e]);
          const int64_t o = b + int64_t(a) * g.lp;
          Gre[o] = g.accum ? Gre[o] + re : re;
          Gim[o] = g.accum ? Gim[o] + im : im;
        }
      }
}

}  // namespace

ssi_status cross_spectral_3m(const double* A, const double* B, int64_t sF, int64_t nseg, int lp, int nfreq,
                             double* G, bool accumulate, cudaStream_t s) {
  if (nfreq < 1 || nfreq > 65535 || (lp & 1)) {
    set_last_error("cross_spectral_3m: bad sizes (nfreq %d, lp %d)", nfreq, lp);
    return SSI_ERR_INVALID_ARG;
  }
  XArgs g{A, B, sF, nseg, lp, G, accumulate ? 1 : 0};
  const size_t smem = sizeof(double) * XST * XSTAGE;
  cudaFuncSetAttribute(cross3m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const dim3 grid(unsigned((lp + XT - 1) / XT), unsigned((lp + XT - 1) / XT), unsigned(nfreq));
  cross3m_kernel<<<grid, XNT, smem, s>>>(g);
  return launch_check("cross3m_kernel");
}

}  // namespace ssi
