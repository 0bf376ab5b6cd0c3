// Tall-skinny FP64 DMMA GEMM for the RSVD passes T*Omega, T^T*Q, T*Z (Eqs. 14-15, PAPER.md:
// 223-231): M = m (11520), N = k (220), K = m. A CTA owns a 64 x 224 tile, so T is streamed
// from HBM exactly once per pass and X (m x k, 20 MB) is served from L2. 8 warps as 2 (M) x 4
// (N), warp tile 32 x 56 = 4 x 7 m8n8k4 DMMA tiles; operands staged by cp.async (16 B) in a
// 3-stage ring; split-K chosen so tiles x splits fill whole waves of the 148 SMs.
#include <cmath>

#include "gemm_f64.cuh"

namespace ssi {
namespace {

// N-tile widths: 224 (the RSVD panels, k <= 224), 128 and 64 (the narrow DFT products; a
// smaller tile also fits 2-3 CTAs per SM).
constexpr int BM = 64, BN = 224, BK = 16, NT = 256, STAGES = 3;
#ifndef TALL64_ST
#define TALL64_ST 3
#endif
#ifndef TALL64_MINB
#define TALL64_MINB 4
#endif
#ifndef TALL128_ST
#define TALL128_ST 3
#endif
#ifndef TALL128_MINB
#define TALL128_MINB 2
#endif
#ifndef TALL224_ST
#define TALL224_ST 2
#endif
#ifndef TALL224_MINB
#define TALL224_MINB 2
#endif
constexpr int LDK = BK + 4;            // k-contiguous rows (A row-major, B): 20 doubles
constexpr int LDM = BM + 4;            // m-contiguous rows (A col-major): 68 doubles
// per-stage tile sizes: A is BM x BK (k-contiguous rows) or BK x BM (m-contiguous rows); B is
// TBN x BK (k-contiguous)
template <bool AROW> constexpr int a_elems() { return AROW ? BM * LDK : BK * LDM; }
template <int TBN> constexpr int b_elems() { return TBN * LDK; }
template <bool AROW, int TBN> constexpr int stage_elems() { return a_elems<AROW>() + b_elems<TBN>(); }
template <bool AROW, int TBN, int ST> constexpr size_t tall_smem() {
  return size_t(ST) * stage_elems<AROW, TBN>() * sizeof(double);
}

__device__ __forceinline__ void cp16n(double* dst, const double* src, int nbytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) { cp16n(dst, src, valid ? 16 : 0); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct TallArgs {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* out;       // partial base (split z at z * M * N, col-major ld M) or C
  int64_t ldo;
  int64_t kchunk;
  int64_t sA, sB, sO;   // batch strides (blockIdx.z); 0 when unbatched
  int mode;             // 0 plain / batched; 1 lower-triangular tiles of a square C (blockIdx.x
                        // = triangular tile index, TBN = BM); 2 upper-triangular B (N tile
                        // blockIdx.z only needs K rows [0, n0 + TBN))
  const int* run_if;    // conditional launch (run_enabled), nullptr = always
};

template <bool AROW, int TBN>
__device__ __forceinline__ void load_stage(const TallArgs& g, double* st, int64_t m0, int64_t k0, int64_t ke) {
  const int tid = threadIdx.x;
  double* As = st;
  double* Bs = st + a_elems<AROW>();
  // A: 64 x 16 doubles = 512 16-byte pieces, 2 per thread
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int p = tid + q * NT;
    if (AROW) {                      // row i: 16 k-contiguous doubles = 8 pieces
      const int i = p >> 3, kk = (p & 7) * 2;
      const int64_t gi = m0 + i, gk = k0 + kk;
      const bool ok = gi < g.M && gk < ke;
      cp16(As + i * LDK + kk, ok ? g.A + gi * g.lda + gk : g.A, ok);
    } else {                         // k-row kk: 64 m-contiguous doubles = 32 pieces
      const int kk = p >> 5, i = (p & 31) * 2;
      const int64_t gi = m0 + i, gk = k0 + kk;
      const bool ok = gi < g.M && gk < ke;
      cp16(As + kk * LDM + i, ok ? g.A + gi + gk * g.lda : g.A, ok);
    }
  }
  // B: TBN columns x 16 k-contiguous doubles = 8 TBN pieces, TBN / 32 per thread
#pragma unroll
  for (int q = 0; q < TBN / 32; ++q) {
    const int p = tid + q * NT;
    const int j = p >> 3, kk = (p & 7) * 2;
    const int64_t gk = k0 + kk;
    const bool ok = j < g.N && gk < ke;
    cp16(Bs + j * LDK + kk, ok ? g.B + gk + int64_t(j) * g.ldb : g.B, ok);
  }
}

template <bool AROW, int TBN, int ST = STAGES, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) gemm_tall_kernel(TallArgs g) {
  constexpr int WN = TBN / 4;          // warp tile N (56 / 32 / 16)
  constexpr int NJ = WN / 8;           // m8n8k4 tiles per warp along N
  constexpr int STAGE_ELEMS = stage_elems<AROW, TBN>();
  extern __shared__ __align__(16) double sm[];
  if (!run_enabled(g.run_if)) return;
  int64_t m0 = int64_t(blockIdx.x) * BM, n0 = 0;
  double* out = g.out + int64_t(blockIdx.y) * g.M * g.N;   // split-K slab (or C)
  if (g.mode == 0) {
    if (blockIdx.z) {
      g.A += int64_t(blockIdx.z) * g.sA;
      g.B += int64_t(blockIdx.z) * g.sB;
      out += int64_t(blockIdx.z) * g.sO;
    }
  } else {
    if (g.mode == 1) {
      const int t = int(blockIdx.x);
      int ti = int((sqrtf(8.0f * float(t) + 1.0f) - 1.0f) * 0.5f);
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      while (ti * (ti + 1) / 2 > t) --ti;
      const int tj = t - ti * (ti + 1) / 2;
      m0 = int64_t(ti) * BM;
      n0 = int64_t(tj) * TBN;
    } else {
      n0 = int64_t(blockIdx.z) * TBN;
      if (n0 + TBN < g.K) g.K = n0 + TBN;
    }
    g.B += n0 * g.ldb;
    out += n0 * g.ldo;
    g.N = (g.N - n0 < TBN) ? g.N - n0 : TBN;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * WN;
  const int64_t kb = int64_t(blockIdx.y) * g.kchunk;
  const int64_t ke = kb + g.kchunk < g.K ? kb + g.kchunk : g.K;
  const int nst = int((ke - kb + BK - 1) / BK);

  double acc[4][NJ][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nst) load_stage<AROW, TBN>(g, sm + s * STAGE_ELEMS, m0, kb + s * BK, ke);
    cp_commit();
  }
  for (int it = 0; it < nst; ++it) {
    cp_wait<ST - 2>();
    __syncthreads();
    {
      const int nx = it + ST - 1;
      if (nx < nst) load_stage<AROW, TBN>(g, sm + (nx % ST) * STAGE_ELEMS, m0, kb + int64_t(nx) * BK, ke);
      cp_commit();
    }
    const double* As = sm + (it % ST) * STAGE_ELEMS;
    const double* Bs = As + a_elems<AROW>();
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[4], bf[NJ];
      const int kq = k4 + (lane & 3), r8 = lane >> 2;
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = AROW ? As[(wm + 8 * i + r8) * LDK + kq] : As[kq * LDM + wm + 8 * i + r8];
#pragma unroll
      for (int j = 0; j < NJ; ++j) bf[j] = Bs[(wn + 8 * j + r8) * LDK + kq];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = m0 + wm + 8 * i + (lane >> 2);
        const int64_t c = wn + 8 * j + 2 * (lane & 3) + e;
        if (r < g.M && c < g.N) out[r + c * g.ldo] = acc[i][j][e];
      }
}

__global__ void tall_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ part, double* __restrict__ C,
                            int64_t ldc, const int* run_if = nullptr) {
  if (!run_enabled(run_if)) return;
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    s = ordered_sum(part + e, total, splits);
    C[(e % M) + (e / M) * ldc] = s;
  }
}

template <bool AROW, int TBN, int ST = STAGES, int MINB = 1>
ssi_status launch_one(dim3 grid, const TallArgs& g, cudaStream_t s) {
  constexpr size_t smem = tall_smem<AROW, TBN, ST>();
  cudaFuncSetAttribute(gemm_tall_kernel<AROW, TBN, ST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  gemm_tall_kernel<AROW, TBN, ST, MINB><<<grid, NT, smem, s>>>(g);
  return launch_check("gemm_tall_kernel");
}

// narrowest N tile that covers N
ssi_status launch_tall(bool arow, int64_t N, dim3 grid, const TallArgs& g, cudaStream_t s) {
  if (N <= 64)
    return arow ? launch_one<true, 64, TALL64_ST, TALL64_MINB>(grid, g, s)
                : launch_one<false, 64, TALL64_ST, TALL64_MINB>(grid, g, s);
  if (N <= 128)
    return arow ? launch_one<true, 128, TALL128_ST, TALL128_MINB>(grid, g, s)
                : launch_one<false, 128, TALL128_ST, TALL128_MINB>(grid, g, s);
  return arow ? launch_one<true, 224, TALL224_ST, TALL224_MINB>(grid, g, s)
              : launch_one<false, 224, TALL224_ST, TALL224_MINB>(grid, g, s);
}

int tall_splits(int64_t M, int64_t K) {
  const int64_t tiles = (M + BM - 1) / BM;
  // smallest split count whose tile count is within 3% of a whole number of waves
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 64; ++s) {
    if (K / s < 4 * BK) break;
    const double units = double(tiles * s);
    const double waves = units / 148.0;
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff + 0.03) { best_eff = eff; best = s; }
  }
  return best;
}

}  // namespace

size_t gemm_tall_partial_elems(int64_t M, int64_t N, int64_t K) {
  const int s = tall_splits(M, K);
  return s > 1 ? size_t(s) * size_t(M) * size_t(N) : 0;
}

size_t gemm_tall_partial_elems_upto(int64_t M, int64_t N) {
  // the split count is not monotone in M: take the maximum over every square size <= M so a
  // workspace sized for the largest lag of a sweep serves every smaller one
  size_t best = 0;
  for (int64_t m = 1; m <= M; ++m) {
    const size_t e = gemm_tall_partial_elems(m, N, m);
    if (e > best) best = e;
  }
  return best;
}

ssi_status gemm_tall(int64_t M, int64_t N, int64_t K, bool a_rowmajor, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc, double* partial, cudaStream_t s) {
  if (N > BN) {
    set_last_error("gemm_tall: N = %lld > %d", (long long)N, BN);
    return SSI_ERR_INVALID_ARG;
  }
  const int splits = tall_splits(M, K);
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int z = int((K + kchunk - 1) / kchunk);
  TallArgs g{M, N, K, A, lda, B, ldb, z > 1 ? partial : C, z > 1 ? M : ldc, kchunk, 0, 0, 0, 0};
  dim3 grid(unsigned((M + BM - 1) / BM), unsigned(z));
  SSI_TRY(launch_tall(a_rowmajor, N, grid, g, s));
  if (z > 1) {
    const int64_t tot = M * N;
    int blocks = int((tot + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    tall_reduce<<<blocks, 256, 0, s>>>(M, N, z, partial, C, ldc);
    SSI_TRY(launch_check("tall_reduce"));
  }
  return SSI_OK;
}

// C (n x n, col-major, ldc) lower triangle (64 x 64 tiles on and below the diagonal) of
// op(A) (n x K) * B (K x n); split-K over whole waves with a fixed-order reduction.
ssi_status gemm_tall_syrk_lower(int64_t n, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
                                double* C, int64_t ldc, double* partial, cudaStream_t s, const int* run_if) {
  const int nt = int((n + BM - 1) / BM);
  const int tiles = nt * (nt + 1) / 2;
  int splits = 1;
  for (int sp = 1; sp <= 64; ++sp) {                       // ~3 CTAs per SM (61 KB smem each)
    if (K / sp < 4 * BK) break;
    splits = sp;
    if (tiles * sp >= 3 * 148) break;
  }
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int z = int((K + kchunk - 1) / kchunk);
  TallArgs g{n, n, K, A, lda, B, ldb, z > 1 ? partial : C, z > 1 ? n : ldc, kchunk, 0, 0, 0, 1, run_if};
  {
    const ssi_status st = launch_one<true, 64, TALL64_ST, TALL64_MINB>(dim3(unsigned(tiles), unsigned(z)), g, s);
    if (st != SSI_OK) return st;
  }
  if (z > 1) {
    const int64_t tot = n * n;
    int blocks = int((tot + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    tall_reduce<<<blocks, 256, 0, s>>>(n, n, z, partial, C, ldc, run_if);
    SSI_TRY(launch_check("tall_reduce"));
  }
  return SSI_OK;
}

// C (M x N, col-major) = A (M x K, col-major) * B (K x N, col-major, upper triangular: B(k, j) = 0
// for k > j): N tiles of 64, tile j0 reads only K rows [0, j0 + 64); no split-K.
ssi_status gemm_tall_triu(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double* C, int64_t ldc, cudaStream_t s, const int* run_if) {
  const int64_t kchunk = (K + BK - 1) / BK * BK;
  TallArgs g{M, N, K, A, lda, B, ldb, C, ldc, kchunk, 0, 0, 0, 2, run_if};
  return launch_one<false, 64, TALL64_ST, TALL64_MINB>(dim3(unsigned((M + BM - 1) / BM), 1u, unsigned((N + 63) / 64)), g, s);
}

ssi_status gemm_tall_batched(int64_t M, int64_t N, int64_t K, bool a_rowmajor, const double* A, int64_t lda,
                             int64_t sA, const double* B, int64_t ldb, int64_t sB, double* C, int64_t ldc,
                             int64_t sC, int batch, cudaStream_t s) {
  if (N > BN || batch < 1 || batch > 65535) {
    set_last_error("gemm_tall_batched: N = %lld > %d or bad batch %d", (long long)N, BN, batch);
    return SSI_ERR_INVALID_ARG;
  }
  const int64_t kchunk = (K + BK - 1) / BK * BK;
  TallArgs g{M, N, K, A, lda, B, ldb, C, ldc, kchunk, sA, sB, sC, 0};
  dim3 grid(unsigned((M + BM - 1) / BM), 1u, unsigned(batch));
  return launch_tall(a_rowmajor, N, grid, g, s);
}

}  // namespace ssi
