// A1, SSI_COV_INT8X3: lagged output covariances (§2.1) on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM), exact integer arithmetic.
//
// Slicing (pre-pass). Per channel a, e_a = ceil(log2 max_t |y_a|) + 1, so x = y 2^-e_a lies in
// [-1/2, 1/2]. Three int8 slices in base B = 254 (|d| <= 127):
//     d1 = rint(B x), d2 = rint(B (B x - d1)), d3 = rint(B (B (B x - d1) - d2))
// give y = 2^e_a (d1/B + d2/B^2 + d3/B^3) + r, |r| <= 2^e_a / (2 B^3) (every step exact in FP64
// for FP32 records). The product y_{t+k,a} y_{t,b} keeps the eight slice products of weight
// w = i + j <= 5 (dropping d3 d3 / B^6); they are summed EXACTLY in int32 per weight class
// (|sum| < 2^31 for chunks of <= 43520 samples) and promoted once per chunk:
//     C = 2^(e_a + e_b) (acc2/B^2 + acc3/B^3 + acc4/B^4 + acc5/B^5)   (FP64, ~1e-16 rel.)
// The error is the slicing remainder r and the dropped d3 d3 term (measured on c3).
//
// Tiling. Output rows are (lag, channel) pairs, columns are channels b. The lag-shifted
// operand A is loaded MN-major: a 16-channel group as a time column [t][16 B] (TMA box of
// KT + 16 samples starting at t0 + k0, any k0). An MN-major SWIZZLE_NONE descriptor with
// LBO = 128 B (K groups of 8 samples) and SBO = 16 B (16-row MN groups) makes row group g
// read the same column g samples later, so ONE M = 128 MMA covers 16 channels x 8 consecutive
// lags; a second descriptor 8 samples further covers the next 8 lags (two "units" per CTA).
// B (un-shifted record, N = 64 channels) is a K-major 128B-swizzled TMA tile whose time
// start is always 16-aligned. TMEM: 2 units x 4 weights x 64 int32 columns = 512. The three slice
// products of one A slice run as ONE MMA over the concatenated B slices (N = 192), so each A slice
// is read from shared memory once per K-step (3 MMAs per unit instead of 8).
// Warp 0 issues TMA, warp 1 issues tcgen05.mma, all four warps drain TMEM at the end.
// (TMA on this driver faults for 1-byte boxes whose innermost start is not 16-B aligned and
// for boxes entirely out of bounds; the layout above never issues either.)
#include <cuda.h>

#include "cov_i8.cuh"

namespace ssi {
namespace {

constexpr int KT = 128;                 // time samples per K-block (= one 128 B row of B)
constexpr int LPU = 8;                  // lags per unit (8 row groups of 16 channels)
constexpr int UNITS = 2;                // units per CTA: lags k0 .. k0 + 15
constexpr int AW = KT + UNITS * LPU;    // A window samples (144)
constexpr int A_SLICE_BYTES = AW * 16;                       // 2304
constexpr int A_BYTES = 3 * A_SLICE_BYTES;                   // 6912
constexpr int A_PAD = (A_BYTES + 1023) / 1024 * 1024;        // 7168 (B stays 1024-aligned)
constexpr int MAX_STAGES = 6;
constexpr int SMEM_CAP = 232448;        // 227 KB dynamic shared memory per CTA
constexpr int NT = 128;
constexpr int BLK_PER_CHUNK_MAX = 340;                       // 43520 samples -> exact int32
constexpr int NW = 4;                                        // weight classes 2..5
constexpr double kBase = 254.0;

struct I8Geom {
  int l, nb;               // channels, B tile width
  int64_t Tpad;
  int lag_lo, lag_hi;
  int lag_blocks;          // ceil(L / 16)
  int64_t t_grid0;         // 16-aligned start of the time grid
  int64_t nblk;            // K-blocks over [t_grid0, t_end)
  int bpc;                 // K-blocks per chunk
  int stages;              // smem ring depth
};

__host__ __device__ inline int b_bytes(int nb) { return 3 * nb * KT; }
__host__ __device__ inline int stage_bytes(int nb) { return A_PAD + b_bytes(nb); }

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// tcgen05 shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 at bit 46, layout type [61,64) (0 none, 2 128B swizzle).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t((saddr & 0x3FFFF) >> 4)) | (uint64_t(lbo >> 4) << 16) | (uint64_t(sbo >> 4) << 32) |
         (1ull << 46) | (uint64_t(layout) << 61);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(z)
      : "memory");
}

// ---------------------------------------------------------------- pre-pass
template <typename T>
__global__ void chan_max_kernel(const T* __restrict__ Y, int64_t N, int l, int64_t ldY,
                                unsigned long long* __restrict__ mx, int32_t* status) {
  const int a = blockIdx.y * 32 + (threadIdx.x & 31);
  if (a >= l) return;
  double m = 0.0;
  bool bad = false;
  for (int64_t t = blockIdx.x * 8 + (threadIdx.x >> 5); t < N; t += int64_t(gridDim.x) * 8) {
    const double v = double(Y[t * ldY + a]);
    bad |= !isfinite(v);
    m = fmax(m, fabs(v));
  }
  if (bad) set_status(status, SSI_ERR_NONFINITE);
  atomicMax(mx + a, __double_as_longlong(m));      // non-negative doubles order as integers
}

__global__ void chan_exp_kernel(const unsigned long long* __restrict__ mx, int l, int* __restrict__ e) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= l) return;
  const double m = __longlong_as_double(mx[a]);
  int ex = 0;
  if (m > 0.0) { frexp(m, &ex); ex += 1; }    // m < 2^(ex-1)  ->  |y| 2^-ex < 1/2
  e[a] = ex;
}

// Tile of 128 samples x 32 channels: reads Y (time-major), writes
//   DA[s][cg][t][16]   (channel-group time columns, whole record, zero past N)
//   DB[s][a][t]        (channel rows, zero outside [t_begin, t_end))
// The slices are staged twice in shared memory, time-major ([s][t][a], rows of 48 B) and
// channel-major ([s][a][t], rows of 144 B), so both outputs are packed with 16-byte loads.
constexpr int TT_LD = 48, TA_LD = KT + 16;
template <typename T>
__global__ void __launch_bounds__(256) slice_kernel(const T* __restrict__ Y, int64_t N, int l, int64_t ldY,
                                                   int64_t Tpad, int64_t t_begin, int64_t t_end,
                                                   const int* __restrict__ e, int8_t* __restrict__ DA,
                                                   int8_t* __restrict__ DB) {
  __shared__ __align__(16) int8_t tt_tile[3][KT][TT_LD];    // [s][t][a]
  __shared__ __align__(16) int8_t ta_tile[3][32][TA_LD];    // [s][a][t]
  const int64_t t0 = int64_t(blockIdx.x) * KT;
  const int a0 = blockIdx.y * 32;
  const int tid = threadIdx.x;
  const int ncg = l / 16;
  const int lane = tid & 31;
  const bool ch_ok = a0 + lane < l;
  const double scale = ldexp(1.0, ch_ok ? -e[a0 + lane] : 0);
  for (int tg = tid >> 5; tg < KT / 4; tg += 8) {            // lane = channel, 4 samples per thread
    uint32_t packed[3] = {0u, 0u, 0u};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int tt = 4 * tg + u;
      const int64_t t = t0 + tt;
      int8_t d[3] = {0, 0, 0};
      if (ch_ok && t < N) {
        // rint by the 1.5 * 2^52 trick (round to nearest even, |v| < 2^51): the rounded value as
        // a double and, in the low word, as an integer -- full-rate DADDs instead of FRND / F2I
        constexpr double kMagic = 6755399441055744.0;
        const double x = double(Y[t * ldY + a0 + lane]) * scale;     // exact: power of two
        const double s1 = kBase * x;
        const double m1 = s1 + kMagic, r1 = m1 - kMagic;
        const double s2 = kBase * (s1 - r1);
        const double m2 = s2 + kMagic, r2 = m2 - kMagic;
        const double m3 = kBase * (s2 - r2) + kMagic;
        d[0] = int8_t(__double2loint(m1)); d[1] = int8_t(__double2loint(m2)); d[2] = int8_t(__double2loint(m3));
      }
      const bool in_shard = t >= t_begin && t < t_end;
#pragma unroll
      for (int sl = 0; sl < 3; ++sl) {
        tt_tile[sl][tt][lane] = d[sl];
        if (in_shard) packed[sl] |= uint32_t(uint8_t(d[sl])) << (8 * u);
      }
    }
#pragma unroll
    for (int sl = 0; sl < 3; ++sl) *reinterpret_cast<uint32_t*>(&ta_tile[sl][lane][4 * tg]) = packed[sl];
  }
  __syncthreads();
  // DA: (s, channel group of 2, t of 128) -> 16 bytes
  for (int q = tid; q < 3 * 2 * KT; q += 256) {
    const int sl = q / (2 * KT), rem = q % (2 * KT), g = rem / KT, tt = rem % KT;
    const int cg = a0 / 16 + g;
    if (cg >= ncg) continue;
    const uint4 v = *reinterpret_cast<const uint4*>(&tt_tile[sl][tt][16 * g]);
    *reinterpret_cast<uint4*>(DA + ((int64_t(sl) * ncg + cg) * Tpad + t0 + tt) * 16) = v;
  }
  // DB: (s, a, 16-byte piece of 8)
  for (int q = tid; q < 3 * 32 * 8; q += 256) {
    const int sl = q / 256, rem = q % 256, a = rem / 8, c = rem % 8;
    if (a0 + a >= l) continue;
    const uint4 v = *reinterpret_cast<const uint4*>(&ta_tile[sl][a][16 * c]);
    *reinterpret_cast<uint4*>(DB + (int64_t(sl) * l + a0 + a) * Tpad + t0 + 16 * c) = v;
  }
}

// ---------------------------------------------------------------- main tcgen05 kernel
// blockIdx.x = (lag block, channel group, b tile), blockIdx.y = time chunk.
__global__ void __launch_bounds__(NT, 1)
cov_i8_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, I8Geom g,
              const int* __restrict__ e, double* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int SB = stage_bytes(g.nb);
  const int STAGES = g.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncg = g.l / 16, nbt = g.l / g.nb;
  int u = blockIdx.x;
  const int bt = u % nbt; u /= nbt;
  const int cg = u % ncg; u /= ncg;
  const int lb = u;                                   // lag block: lags k0 .. k0 + 8 UNITS - 1
  const int k0 = g.lag_lo + lb * (UNITS * LPU);
  const int b0 = bt * g.nb;
  const int chunk = blockIdx.y;
  const int64_t blk0 = int64_t(chunk) * g.bpc;
  int64_t nblk = g.nblk - blk0;
  if (nblk > g.bpc) nblk = g.bpc;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // TMEM: UNITS x 4 weights x nb <= 512 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // weight class 3 (first written by an accumulating MMA) starts at zero: each warp clears its
  // 32 TMEM lanes of the class-3 columns of every unit
  {
    const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
    for (int un = 0; un < UNITS; ++un)
      for (int c0 = 0; c0 < g.nb; c0 += 16)
        tmem_st16_zero(lane_base + uint32_t((un * NW + 3) * g.nb + c0));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (nblk > 0) {
    if (warp == 0 && lane == 0) {
      // ---------------- TMA producer (stage index and phase kept incrementally)
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < nblk; ++it) {
        mbar_wait(empty + s, ph ^ 1);
        uint8_t* A = smem + s * SB;
        uint8_t* B = A + A_PAD;
        const int64_t t0 = g.t_grid0 + (blk0 + it) * KT;
        mbar_expect_tx(full + s, A_BYTES + b_bytes(g.nb));
        tma_load_4d(A, &mapA, full + s, 0, int(t0 + k0), cg, 0);
        tma_load_3d(B, &mapB, full + s, int(t0), b0, 0);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    } else if (warp == 1 && lane == 0) {
      // ---------------- MMA issuer: per K-step and unit, three MMAs, one per A slice, each over
      // the B slices concatenated along N (they are adjacent in shared memory): A_i x [B_0 B_1 B_2]
      // lands in weight classes i, i+1, i+2 (adjacent TMEM column blocks of nb); A_2 takes
      // [B_0 B_1] only (d3 d3 dropped). 8 slice products, 3 MMAs, each A slice read once.
      // idesc: S32 accum, signed int8 A/B, A MN-major (bit 15), B K-major, N>>3, M>>4
      const uint32_t idesc_base = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (uint32_t(128 >> 4) << 24);
      const uint32_t idesc3 = idesc_base | (uint32_t((3 * g.nb) >> 3) << 17);
      const uint32_t idesc2 = idesc_base | (uint32_t((2 * g.nb) >> 3) << 17);
      // descriptors of stage 0; a stage / slice / K offset adds (bytes >> 4) to the start-address
      // field (addresses < 256 KB: the 14-bit field never carries)
      const uint32_t abase0 = smem_u32(smem);
      const uint64_t ad0 = umma_desc(abase0, 128, 16, 0);
      const uint64_t bd0 = umma_desc(abase0 + A_PAD, 16, 1024, 2);
      const uint32_t sb16 = uint32_t(SB) >> 4;
      int s = 0;
      uint32_t ph = 0;
      for (int64_t it = 0; it < nblk; ++it) {
        mbar_wait(full + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t ads = ad0 + uint64_t(uint32_t(s) * sb16);
        const uint64_t bds = bd0 + uint64_t(uint32_t(s) * sb16);
#pragma unroll
        for (int j = 0; j < KT / 32; ++j) {
          const uint64_t bd = bds + uint64_t(uint32_t((32 * j) >> 4));
#pragma unroll
          for (int un = 0; un < UNITS; ++un) {
            const uint32_t tcol = tmem + uint32_t(un * NW * g.nb);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              // A slice q, K offset 32 j samples, unit offset 8 un samples (16 B each)
              const uint64_t ad = ads + uint64_t((q * A_SLICE_BYTES + (32 * j + LPU * un) * 16) >> 4);
              const bool init = (it == 0 && j == 0 && q == 0);   // classes 0..2 (class 3 pre-zeroed)
              umma_i8(tcol + uint32_t(q * g.nb), ad, bd, q < 2 ? idesc3 : idesc2, init ? 0u : 1u);
            }
          }
        }
        umma_commit(empty + s);      // frees the smem stage when these MMAs complete
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      umma_commit(done);
    }
    // ---------------- epilogue: TMEM -> registers -> FP64 partial sums
    mbar_wait(done, 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = warp * 32 + lane;               // TMEM lane
    const int a = cg * 16 + (row & 15);
    const double sa = ldexp(1.0, e[a]);
    const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
    for (int un = 0; un < UNITS; ++un) {
      const int lag = k0 + un * LPU + (row >> 4);
      const bool valid = lag <= g.lag_hi;
      double* out = partial + ((int64_t(chunk) * (g.lag_hi - g.lag_lo + 1) + (lag - g.lag_lo)) * g.l + a) * g.l + b0;
      for (int c0 = 0; c0 < g.nb; c0 += 16) {
        int32_t v2[16], v3[16], v4[16], v5[16];
        const uint32_t col = uint32_t(un * NW * g.nb + c0);
        tmem_ld16(lane_base + col, v2);
        tmem_ld16(lane_base + col + uint32_t(g.nb), v3);
        tmem_ld16(lane_base + col + uint32_t(2 * g.nb), v4);
        tmem_ld16(lane_base + col + uint32_t(3 * g.nb), v5);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        double sb[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) sb[c] = ldexp(1.0, __ldg(e + b0 + c0 + c));
        if (valid) {
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            double r[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              constexpr double i2 = 1.0 / (kBase * kBase), i3 = i2 / kBase, i4 = i3 / kBase, i5 = i4 / kBase;
              const double acc = ((double(v5[c + h]) * i5 + double(v4[c + h]) * i4) + double(v3[c + h]) * i3) +
                                 double(v2[c + h]) * i2;
              r[h] = acc * sa * sb[c + h];
            }
            *reinterpret_cast<double2*>(out + c0 + c) = make_double2(r[0], r[1]);
          }
        }
      }
    }
  } else {
    const int row = warp * 32 + lane;
    const int a = cg * 16 + (row & 15);
    for (int un = 0; un < UNITS; ++un) {
      const int lag = k0 + un * LPU + (row >> 4);
      if (lag > g.lag_hi) continue;
      double* out = partial + ((int64_t(chunk) * (g.lag_hi - g.lag_lo + 1) + (lag - g.lag_lo)) * g.l + a) * g.l + b0;
      for (int c = 0; c < g.nb; ++c) out[c] = 0.0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void cov_i8_finalize(const double* __restrict__ part, int nchunks, int64_t per, int l, int lag_lo,
                                int64_t N, int normalize, double* __restrict__ R) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < per; e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    s = ordered_sum(part + e, per, nchunks);
    if (normalize) s /= double(N - (lag_lo + int(e / (int64_t(l) * l))));
    R[e] = s;
  }
}

// ---------------------------------------------------------------- host helpers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// B tile width nb: 64 channels if l % 64 == 0, else l itself (l % 16 == 0, l <= 64). The slice
// products of one A slice are merged into one MMA over the concatenated B slices (N = 3 nb <= 256),
// and TMEM holds UNITS x 4 weight classes x nb <= 512 columns.
int pick_nb(int l) {
  if (l % 64 == 0) return 64;
  if (l % 16 == 0 && l <= 64) return l;
  return 0;
}

struct I8Plan {
  int64_t Tpad, t_grid0, nblk;
  int nb, lag_blocks, bpc, nchunks;
  size_t da_bytes, db_bytes, part_elems;
};

I8Plan plan(int64_t N, int l, int lag_lo, int lag_hi, int64_t t_begin, int64_t t_end) {
  I8Plan p;
  p.Tpad = (N + lag_hi + 2 * KT + 32 + KT - 1) / KT * KT;
  p.nb = pick_nb(l);
  const int L = lag_hi - lag_lo + 1;
  p.lag_blocks = (L + UNITS * LPU - 1) / (UNITS * LPU);
  p.t_grid0 = t_begin / 16 * 16;
  p.nblk = (t_end - p.t_grid0 + KT - 1) / KT;
  if (p.nblk < 1) p.nblk = 1;
  const int64_t units = int64_t(p.lag_blocks) * (l / 16) * (l / (p.nb ? p.nb : 1));
  int64_t nchunks = (148 * 6 + units - 1) / units;     // ~6 waves of CTAs
  const int64_t minch = (p.nblk + BLK_PER_CHUNK_MAX - 1) / BLK_PER_CHUNK_MAX;
  if (nchunks < minch) nchunks = minch;
  if (nchunks > p.nblk) nchunks = p.nblk;
  p.bpc = int((p.nblk + nchunks - 1) / nchunks);
  p.nchunks = int((p.nblk + p.bpc - 1) / p.bpc);
  p.da_bytes = size_t(3) * p.Tpad * l;
  p.db_bytes = size_t(3) * p.Tpad * l;
  p.part_elems = size_t(p.nchunks) * L * l * l;
  return p;
}

}  // namespace

bool cov_i8_supported(int l, int n_lags, int64_t ldY, int dtype) {
  (void)n_lags; (void)ldY; (void)dtype;
  return pick_nb(l) > 0 && l <= 4096;
}

void cov_i8_carve(Carver& c, int64_t N, int l, int lag_lo, int lag_hi) {
  const I8Plan p = plan(N, l, lag_lo, lag_hi, 0, N);
  c.take<unsigned long long>(l);
  c.take<int>(l);
  c.take<int8_t>(p.da_bytes);
  c.take<int8_t>(p.db_bytes);
  // a shard never needs more chunks than the full record
  c.take<double>(p.part_elems);
}

ssi_status cov_i8(const void* Y, int dtype, int64_t N, int l, int64_t ldY, int lag_lo, int lag_hi,
                  int64_t t_begin, int64_t t_end, int normalize, double* R, void* ws, int32_t* status,
                  cudaStream_t s) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    set_last_error("cov_i8: cuTensorMapEncodeTiled unavailable");
    return SSI_ERR_CUDA;
  }
  const I8Plan p0 = plan(N, l, lag_lo, lag_hi, 0, N);
  const I8Plan p = plan(N, l, lag_lo, lag_hi, t_begin, t_end);
  Carver c(ws);
  unsigned long long* mx = c.take<unsigned long long>(l);
  int* e = c.take<int>(l);
  int8_t* DA = c.take<int8_t>(p0.da_bytes);
  int8_t* DB = c.take<int8_t>(p0.db_bytes);
  double* part = c.take<double>(p0.part_elems);
  if (p.part_elems > p0.part_elems) {
    set_last_error("cov_i8: internal plan mismatch");
    return SSI_ERR_WORKSPACE;
  }
  // 1. per-channel power-of-two scales over the whole record (every time shard agrees)
  if (cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * l, s) != cudaSuccess) return launch_check("cov_i8 memset");
  {
    dim3 grid(592, (l + 31) / 32);
    if (dtype == SSI_F32) {
      chan_max_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(Y), N, l, ldY, mx, status);
    } else {
      chan_max_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(Y), N, l, ldY, mx, status);
    }
    SSI_TRY(launch_check("chan_max_kernel"));
    chan_exp_kernel<<<(l + 127) / 128, 128, 0, s>>>(mx, l, e);
    SSI_TRY(launch_check("chan_exp_kernel"));
  }
  // 2. slices
  {
    dim3 grid(unsigned(p.Tpad / KT), (l + 31) / 32);
    if (dtype == SSI_F32)
      slice_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(Y), N, l, ldY, p.Tpad, t_begin, t_end, e, DA, DB);
    else
      slice_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(Y), N, l, ldY, p.Tpad, t_begin, t_end, e, DA, DB);
    SSI_TRY(launch_check("slice_kernel"));
  }
  // 3. tensor maps: A = DA[s][cg][t][16] (box 16 ch x AW samples x 1 group x 3 slices),
  //    B = DB[s][a][t] (box 128 samples x nb channels x 3 slices, 128B swizzle)
  CUtensorMap mapA, mapB;
  {
    const int ncg = l / 16;
    const cuuint64_t dims[4] = {16, cuuint64_t(p.Tpad), cuuint64_t(ncg), 3};
    const cuuint64_t strides[3] = {16, cuuint64_t(16) * p.Tpad, cuuint64_t(16) * p.Tpad * ncg};
    const cuuint32_t box[4] = {16, AW, 1, 3};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mapA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, DA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_last_error("cov_i8: encoding the A tensor map failed");
      return SSI_ERR_CUDA;
    }
  }
  {
    const cuuint64_t dims[3] = {cuuint64_t(p.Tpad), cuuint64_t(l), 3};
    const cuuint64_t strides[2] = {cuuint64_t(p.Tpad), cuuint64_t(p.Tpad) * l};
    const cuuint32_t box[3] = {KT, cuuint32_t(p.nb), 3};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&mapB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, DB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_last_error("cov_i8: encoding the B tensor map failed");
      return SSI_ERR_CUDA;
    }
  }
  // 4. tcgen05 contraction + fixed-order chunk reduction
  int stages = int((SMEM_CAP - 1024 - 256) / stage_bytes(p.nb));
  if (stages > MAX_STAGES) stages = MAX_STAGES;
  I8Geom g{l, p.nb, p.Tpad, lag_lo, lag_hi, p.lag_blocks, p.t_grid0, p.nblk, p.bpc, stages};
  const size_t smem = size_t(stages) * stage_bytes(p.nb) + 1024 + 256;
  cudaFuncSetAttribute(cov_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  dim3 grid(unsigned(p.lag_blocks * (l / 16) * (l / p.nb)), unsigned(p.nchunks));
  cov_i8_kernel<<<grid, NT, smem, s>>>(mapA, mapB, g, e, part);
  SSI_TRY(launch_check("cov_i8_kernel"));
  const int L = lag_hi - lag_lo + 1;
  const int64_t per = int64_t(L) * l * l;
  int blocks = int((per + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  cov_i8_finalize<<<blocks, 256, 0, s>>>(part, p.nchunks, per, l, lag_lo, N, normalize, R);
  return launch_check("cov_i8_finalize");
}

}  // namespace ssi
