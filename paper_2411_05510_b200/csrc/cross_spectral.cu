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
// Measured alternative (-DSSI_CROSS_TMA=1, cross3m_tma_kernel): the same tile and fragment order, but each stage's
// 32 segment rows (1 KB each, contiguous in HBM) are moved by the bulk-copy engine
// (cp.async.bulk ... mbarrier::complete_tx) into a 3-stage ring with a full / empty mbarrier
// pair per slot: warp 0 refills the slot the CTA finished one iteration earlier, so two
// stages are in flight behind the one the warps multiply, and no thread computes addresses
// or issues per-16-byte copies. Segments past the chunk's end are not copied; warp 0 zeroes
// their rows (both operands) before it posts the stage, so stale shared memory never reaches
// the sums.
// Parity-green, but 1.564 ms against the cp.async kernel's 1.513 ms per c3 launch (CUPTI, 4
// alternating calls each) and 125.4 vs 126.9 records/s: its warps stall on the full barrier
// (22 % of samples, profiles/cross3m_tma_r02.ncu-rep) because a slot is refilled only after the
// slowest warp released it; the 2-stage cp.async ring with 16 warps per SM hides the same
// latency. Kept for the A/B; DESIGN.md §6 A1. -DSSI_CROSS_TMA=2: the warp whose release
// completes a slot (a shared counter) refills it at once, so no warp waits on an empty barrier.
#include "cov_spectral.cuh"

#ifndef SSI_CROSS_TMA
#define SSI_CROSS_TMA 0
#endif

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

// ---------------------------------------------------------------- bulk-copy (TMA) variant
constexpr int XSTT = 3;           // ring depth
constexpr int XBAR_OFF = XSTT * XSTAGE;   // barriers after the ring (doubles)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "XW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra XW_%=;\n}" ::"r"(su32(b)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

// warp 0: stage st of the chunk into ring slot st % XSTT (lane j < 16 copies segment j of A,
// lane 16 + j segment j of B); lane 0 posts the byte count first.
__device__ __forceinline__ void x_issue(const XArgs& g, double* xs, uint64_t* full, const double* Af,
                                        const double* Bf, int st, int b0, int a0, int lane) {
  const int slot = st % XSTT;
  const int64_t s0 = int64_t(st) * XS;
  const int nv = int(g.nseg - s0 < XS ? g.nseg - s0 : XS);
  const int wa = min(XT, g.lp - b0), wb = min(XT, g.lp - a0);
  if (nv < XS) {   // the chunk's last stage: zero the rows past its end (both operands)
    double* z = xs + slot * XSTAGE;
    for (int r = nv; r < XS; ++r)
      for (int c = lane; c < XT; c += 32) {
        *reinterpret_cast<double2*>(z + r * XP + 2 * c) = make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(z + XS * XP + r * XP + 2 * c) = make_double2(0.0, 0.0);
      }
  }
  __syncwarp();
  if (lane == 0) bar_expect(&full[slot], uint32_t(nv * (wa + wb) * 16));
  __syncwarp();
  const int sg = lane & 15;
  if (sg < nv) {
    double* dst = xs + slot * XSTAGE + (lane >> 4) * (XS * XP) + sg * XP;
    const double* src = (lane < 16 ? Af + ((s0 + sg) * g.lp + b0) * 2 : Bf + ((s0 + sg) * g.lp + a0) * 2);
    bulk_g2s(dst, src, uint32_t((lane < 16 ? wa : wb) * 16), &full[slot]);
  }
}

// LASTW: the warp whose release completes a slot refills it (a shared counter per slot) instead
// of warp 0 waiting on the slot's empty barrier
template <bool LASTW>
__global__ void __launch_bounds__(XNT, 2) cross3m_tma_kernel(XArgs g) {
  extern __shared__ __align__(16) double xs[];
  uint64_t* full = reinterpret_cast<uint64_t*>(xs + XBAR_OFF);
  uint64_t* empty = full + XSTT;
  int* cnt = reinterpret_cast<int*>(empty + XSTT);
  const int b0 = blockIdx.x * XT, a0 = blockIdx.y * XT;
  const int64_t f = blockIdx.z;
  const double* Af = g.A + f * g.sF;
  const double* Bf = g.B + f * g.sF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  const int r8 = lane >> 2, kq = lane & 3;
  const int nst = int((g.nseg + XS - 1) / XS);
  if (tid == 0) {
    for (int i = 0; i < XSTT; ++i) {
      bar_init(&full[i], 1);
      bar_init(&empty[i], XNT / 32);
      cnt[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int st = 0; st < min(XSTT, nst); ++st) x_issue(g, xs, full, Af, Bf, st, b0, a0, lane);
  double t1[4][2][2], t2[4][2][2], t3[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;
  for (int it = 0; it < nst; ++it) {
    // refill the slot every warp released one iteration ago (stage it - 1 + XSTT)
    if (!LASTW && warp == 0 && it > 0 && it - 1 + XSTT < nst) {
      bar_wait(&empty[(it - 1) % XSTT], uint32_t(((it - 1) / XSTT) & 1));
      x_issue(g, xs, full, Af, Bf, it - 1 + XSTT, b0, a0, lane);
    }
    const int slot = it % XSTT;
    bar_wait(&full[slot], uint32_t((it / XSTT) & 1));
    const double* As = xs + slot * XSTAGE;
    const double* Bs = As + XS * XP;
#pragma unroll
    for (int k4 = 0; k4 < XS; k4 += 4) {
      const int s = k4 + kq;
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
    __syncwarp();
    if (LASTW) {
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&cnt[slot], 1) == XNT / 32 - 1;
        if (last) cnt[slot] = 0;
        __threadfence_block();
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last && it + XSTT < nst) x_issue(g, xs, full, Af, Bf, it + XSTT, b0, a0, lane);
    } else if (lane == 0) {
      bar_arrive(&empty[slot]);
    }
  }
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
  const dim3 grid(unsigned((lp + XT - 1) / XT), unsigned((lp + XT - 1) / XT), unsigned(nfreq));
#if !SSI_CROSS_TMA
  const size_t smem = sizeof(double) * XST * XSTAGE;
  cudaFuncSetAttribute(cross3m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cross3m_kernel<<<grid, XNT, smem, s>>>(g);
  return launch_check("cross3m_kernel");
#else
  // bulk copies need 16-byte aligned global rows: (Re, Im) doubles at 16-byte aligned bases
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) {
    set_last_error("cross_spectral_3m: spectra not 16-byte aligned");
    return SSI_ERR_INVALID_ARG;
  }
  const size_t smem = sizeof(double) * XBAR_OFF + 3 * XSTT * sizeof(uint64_t);
  constexpr bool lastw = SSI_CROSS_TMA == 2;
  cudaFuncSetAttribute(cross3m_tma_kernel<lastw>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cross3m_tma_kernel<lastw><<<grid, XNT, smem, s>>>(g);
  return launch_check("cross3m_tma_kernel");
#endif
}

}  // namespace ssi
