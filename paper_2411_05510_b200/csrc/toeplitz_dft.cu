// Block-Toeplitz products without forming T (north star (b): "exploit its block-Toeplitz
// structure"; Eq. 6). With B_d = R_{i+d} (d = r - c in [-(i-1), i-1]),
//     (T X)_r   = sum_c B_{r-c}   X_c          (block convolution)
//     (T^T X)_c = sum_r B_{r-c}^T X_r          (block correlation)
// where X_c = X[c*l : (c+1)*l, :]. Both are exact circular convolutions of period P = 2i-1
// (the 2i-1 block lags are distinct mod P), so with the length-P DFT along the block index
//     hat(TX)_f = hatB_f hatX_f,   hat(T^T X)_f = hatB_f^H hatX_f,   hatB_f = sum_d B_d w^{fd},
// w = exp(-2 pi i / P). All data are real, so only f = 0 .. (P-1)/2 = i-1 are formed (F = i).
// The complex products are real GEMMs on the 2l x 2l real form [[Re, -Im], [Im, Re]] of hatB_f
// (batched FP64 DMMA, gemm_tall_batched); T^T uses the transpose of the same storage.
// Per pass: 2 F (2l)^2 k flop in the products (3.9e9 at c3 vs 2 m^2 k = 5.8e10 for explicit T)
// plus two DFTs of 2 F i l k flop each; T (1.06 GB at c3) is never read.
#include <cmath>

#include "gemm_f64.cuh"
#include "toeplitz_dft.cuh"

#ifndef SSI_BT_SPEC_GEMM
#define SSI_BT_SPEC_GEMM 1   // 0: the direct-sum spectrum kernel for every shape (A/B)
#endif

namespace ssi {
namespace {

constexpr int DT = 256;          // threads per CTA (8 warps)
constexpr int DW = DT / 32;

// cos / sin of 2 pi t / P for t in [0, P): shared-memory table
__device__ __forceinline__ void twiddles(int P, double* cs, double* sn) {
  for (int t = threadIdx.x; t < P; t += blockDim.x) {
    double s, c;
    sincospi(2.0 * double(t) / double(P), &s, &c);
    cs[t] = c;
    sn[t] = s;
  }
}

// hatB_f for f in [0, F), written as the real 2l x 2l block form, row-major:
//   [a][b] = [l+a][l+b] = Re hatB_f[a][b],  [l+a][b] = Im,  [a][l+b] = -Im.
// CTA: 32 consecutive (a, b) elements (lanes) x 8 warps over f. R: [>= 2i-1][l][l] row-major.
__global__ void __launch_bounds__(DT) bt_spectrum_kernel(const double* __restrict__ R, int l, int i,
                                                         double* __restrict__ Bb) {
  extern __shared__ __align__(16) double sm[];
  const int P = 2 * i - 1, F = i;
  double* cs = sm;
  double* sn = cs + P;
  double* rs = sn + P;                    // [P][32]: rs[(d + i - 1)*32 + lane] = B_d[e]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ll = int64_t(l) * l;
  const int64_t e = int64_t(blockIdx.x) * 32 + lane;
  const bool ok = e < ll;
  twiddles(P, cs, sn);
  for (int d = warp; d < P; d += DW) rs[d * 32 + lane] = ok ? R[int64_t(d) * ll + e] : 0.0;
  __syncthreads();
  if (!ok) return;
  const int a = int(e / l), b = int(e % l);
  const int64_t L2 = 2 * int64_t(l);
  for (int f = warp; f < F; f += DW) {
    double re = 0.0, im = 0.0;
    // d = -(i-1) .. i-1, phase t = f d mod P, starting at f (P - (i-1)) mod P
    int t = int((int64_t(f) * (P - (i - 1))) % P);
    for (int dd = 0; dd < P; ++dd) {
      const double v = rs[dd * 32 + lane];
      re = fma(v, cs[t], re);
      im = fma(-v, sn[t], im);
      t += f;
      if (t >= P) t -= P;
    }
    double* blk = Bb + int64_t(f) * L2 * L2;
    blk[int64_t(a) * L2 + b] = re;
    blk[int64_t(l + a) * L2 + (l + b)] = re;
    blk[int64_t(l + a) * L2 + b] = im;
    blk[int64_t(a) * L2 + (l + b)] = -im;
  }
}

// hatX_f = sum_{c<i} X_c w^{fc}: Xh[j][f][0:l] = Re, Xh[j][f][l:2l] = Im (per f a 2l x k
// col-major matrix, ld 2l F). CTA: 32 rows a of one column j; 8 warps over f. (Odd l; for even l
// the forward and inverse DFTs run as batched DMMA GEMMs against the tables of bt_tables_kernel.)
__global__ void __launch_bounds__(DT) bt_forward_kernel(const double* __restrict__ X, int64_t ldx, int l, int i,
                                                        int k, double* __restrict__ Xh) {
  extern __shared__ __align__(16) double sm[];
  const int P = 2 * i - 1, F = i;
  double* cs = sm;
  double* sn = cs + P;
  double* xs = sn + P;                    // [i][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a = blockIdx.x * 32 + lane;
  const int j = blockIdx.y;
  const bool ok = a < l;
  twiddles(P, cs, sn);
  const double* xc = X + int64_t(j) * ldx;
  for (int c = warp; c < i; c += DW) xs[c * 32 + lane] = ok ? xc[int64_t(c) * l + a] : 0.0;
  __syncthreads();
  if (!ok) return;
  const int64_t L2 = 2 * int64_t(l);
  for (int f = warp; f < F; f += DW) {
    double re = 0.0, im = 0.0;
    int t = 0;
    for (int c = 0; c < i; ++c) {
      const double v = xs[c * 32 + lane];
      re = fma(v, cs[t], re);
      im = fma(-v, sn[t], im);
      t += f;
      if (t >= P) t -= P;
    }
    double* o = Xh + (int64_t(j) * F + f) * L2;
    o[a] = re;
    o[l + a] = im;
  }
}

// Y_r = (1/P) [Re hatY_0 + 2 sum_{f=1}^{F-1} (Re hatY_f cos(2 pi r f / P) - Im hatY_f sin(...))],
// r in [0, i): Y[r*l + a + j*ldy]. CTA: 32 rows a of one column j; 8 warps over r.
__global__ void __launch_bounds__(DT) bt_inverse_kernel(const double* __restrict__ Yh, int l, int i, int k,
                                                        double* __restrict__ Y, int64_t ldy) {
  extern __shared__ __align__(16) double sm[];
  const int P = 2 * i - 1, F = i;
  double* cs = sm;
  double* sn = cs + P;
  double* ys = sn + P;                    // [F][2][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a = blockIdx.x * 32 + lane;
  const int j = blockIdx.y;
  const bool ok = a < l;
  twiddles(P, cs, sn);
  const int64_t L2 = 2 * int64_t(l);
  for (int f = warp; f < F; f += DW) {
    const double* src = Yh + (int64_t(j) * F + f) * L2;
    ys[(2 * f) * 32 + lane] = ok ? src[a] : 0.0;
    ys[(2 * f + 1) * 32 + lane] = ok ? src[l + a] : 0.0;
  }
  __syncthreads();
  if (!ok) return;
  const double invP = 1.0 / double(P);
  for (int r = warp; r < i; r += DW) {
    double acc = 0.0;
    int t = r;
    if (t >= P) t -= P;
    for (int f = 1; f < F; ++f) {
      acc = fma(ys[(2 * f) * 32 + lane], cs[t], acc);
      acc = fma(-ys[(2 * f + 1) * 32 + lane], sn[t], acc);
      t += r;
      if (t >= P) t -= P;
    }
    Y[int64_t(r) * l + a + int64_t(j) * ldy] = fma(2.0, acc, ys[lane]) * invP;
  }
}

size_t smem_twiddle(int i) { return sizeof(double) * 2 * size_t(2 * i - 1); }

// DFT matrices of the GEMM form (l even): Ft (i x 2F col-major, ld ldF): Ft[c][2f] = cos(2 pi f c/P),
// Ft[c][2f+1] = -sin(...); Gt (2F x i col-major): Gt[2f][r] = w_f cos(2 pi r f/P)/P,
// Gt[2f+1][r] = -w_f sin(2 pi r f/P)/P, w_0 = 1, w_f = 2 (f >= 1).
__global__ void bt_tables_kernel(int i, int ldF, double* __restrict__ Ft, double* __restrict__ Gt) {
  const int P = 2 * i - 1, F = i;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < F * i; e += gridDim.x * blockDim.x) {
    const int f = e / i, c = e % i;            // (f, c) for Ft; (f, r = c) for Gt
    const int t = int((int64_t(f) * c) % P);
    double sn, cs;
    sincospi(2.0 * double(t) / double(P), &sn, &cs);
    Ft[c + int64_t(2 * f) * ldF] = cs;
    Ft[c + int64_t(2 * f + 1) * ldF] = -sn;
    const double w = (f == 0 ? 1.0 : 2.0) / double(P);
    Gt[2 * f + int64_t(c) * 2 * F] = w * cs;
    Gt[2 * f + 1 + int64_t(c) * 2 * F] = -w * sn;
    if (c == 0 && ldF > i) {               // zero pad row (read in 16-byte pairs by the GEMM)
      for (int cc = i; cc < ldF; ++cc) { Ft[cc + int64_t(2 * f) * ldF] = 0.0; Ft[cc + int64_t(2 * f + 1) * ldF] = 0.0; }
    }
  }
}

// Spectrum as a GEMM (l even, k >= l): Z (l^2 x 2F, col-major) = R (l^2 x P) Wb (P x 2F),
// Wb[dd][2f] = cos(2 pi t / P), Wb[dd][2f + 1] = -sin(2 pi t / P), t = f (dd - (i - 1)) mod P
// (dd = d + i - 1 indexes R_{i+d}); ld P + 1 with a zero pad row (16-byte k pairs).
__global__ void bt_wspec_kernel(int i, double* __restrict__ Wb) {
  const int P = 2 * i - 1, F = i, ld = P + 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ld * 2 * F; e += gridDim.x * blockDim.x) {
    const int dd = e % ld, kk = e / ld, f = kk >> 1;
    double v = 0.0;
    if (dd < P) {
      const int t = int((int64_t(f) * (dd - (i - 1) + P)) % P);
      double sn, cs;
      sincospi(2.0 * double(t) / double(P), &sn, &cs);
      v = (kk & 1) ? -sn : cs;
    }
    Wb[e] = v;
  }
}

// Z (l^2 x 2F) -> the real 2l x 2l block form of bt_spectrum_kernel
__global__ void bt_scatter_kernel(const double* __restrict__ Z, int l, int F, double* __restrict__ Bb) {
  const int64_t ll = int64_t(l) * l, L2 = 2 * int64_t(l);
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < ll * F; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = q % ll, f = q / ll;
    const int a = int(e / l), b = int(e % l);
    const double re = Z[e + 2 * f * ll], im = Z[e + (2 * f + 1) * ll];
    double* blk = Bb + f * L2 * L2;
    blk[int64_t(a) * L2 + b] = re;
    blk[int64_t(l + a) * L2 + (l + b)] = re;
    blk[int64_t(l + a) * L2 + b] = im;
    blk[int64_t(a) * L2 + (l + b)] = -im;
  }
}

}  // namespace

size_t bt_spectrum_elems(int l, int i) { return size_t(i) * 4 * size_t(l) * l; }
int bt_ldF(int i) { return (i + 1) & ~1; }
size_t bt_table_elems(int i) { return size_t(bt_ldF(i)) * 2 * i + size_t(2 * i) * i + size_t(2 * i) * (2 * i); }
size_t bt_freq_elems(int l, int i, int k) { return size_t(i) * 2 * size_t(l) * k; }

ssi_status bt_spectrum(const double* R, int l, int i, double* Bb, double* tables, cudaStream_t s, double* Z) {
  bt_tables_kernel<<<unsigned((i * i + 255) / 256), 256, 0, s>>>(i, bt_ldF(i), tables,
                                                              tables + size_t(bt_ldF(i)) * 2 * i);
  SSI_TRY(launch_check("bt_tables_kernel"));
  if (SSI_BT_SPEC_GEMM && Z && l % 2 == 0 && 2 * i <= kTallMaxN && (reinterpret_cast<uintptr_t>(R) & 15) == 0) {
    // Z (l^2 x 2F) = R (l^2 x P) Wb (P x 2F) on the DMMA pipe, then the block form
    double* Wb = tables + size_t(bt_ldF(i)) * 2 * i + size_t(2 * i) * i;
    const int P = 2 * i - 1, F = i;
    const int64_t ll = int64_t(l) * l;
    bt_wspec_kernel<<<unsigned((2 * i * 2 * i + 255) / 256), 256, 0, s>>>(i, Wb);
    SSI_TRY(launch_check("bt_wspec_kernel"));
    SSI_TRY(gemm_tall_batched(ll, 2 * F, P, false, R, ll, 0, Wb, P + 1, 0, Z, ll, 0, 1, s));
    int blocks = int((ll * F + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    bt_scatter_kernel<<<blocks, 256, 0, s>>>(Z, l, F, Bb);
    return launch_check("bt_scatter_kernel");
  }
  const int P = 2 * i - 1;
  const size_t smem = smem_twiddle(i) + sizeof(double) * size_t(P) * 32;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(bt_spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int64_t ll = int64_t(l) * l;
  bt_spectrum_kernel<<<unsigned((ll + 31) / 32), DT, smem, s>>>(R, l, i, Bb);
  return launch_check("bt_spectrum_kernel");
}

bool bt_gemm_form(int l, int i) { return l % 2 == 0 && 2 * i <= kTallMaxN; }

ssi_status bt_apply(const double* Bb, const double* tables, int l, int i, int k, bool trans, const double* X,
                    int64_t ldx, double* Y, int64_t ldy, double* Xh, double* Yh, cudaStream_t s) {
  const int F = i;
  const int64_t L2 = 2 * int64_t(l);
  const bool gemm_form = bt_gemm_form(l, i) && ldx % 2 == 0 && ldy % 2 == 0 &&
                         (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  // frequency-domain layout: per column j, F blocks of (Re[l], Im[l]): hatX[j][f][part][a]
  const int64_t ldh = L2 * F;                 // column stride of one frequency's 2l x k matrix
  if (gemm_form) {
    // hatX(:, (f, part)) of column j = X_j (l x i, col-major ld l) * Ft (i x 2F)
    const double* Ft = tables;
    SSI_TRY(gemm_tall_batched(l, 2 * F, i, false, X, l, ldx, Ft, bt_ldF(i), 0, Xh, l, ldh, k, s));
  } else {
    const size_t smem_f = smem_twiddle(i) + sizeof(double) * size_t(i) * 32;
    if (smem_f > 48 * 1024)
      cudaFuncSetAttribute(bt_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_f));
    const dim3 grid(unsigned((l + 31) / 32), unsigned(k));
    bt_forward_kernel<<<grid, DT, smem_f, s>>>(X, ldx, l, i, k, Xh);
    SSI_TRY(launch_check("bt_forward_kernel"));
  }
  // hatY_f = Bblk_f hatX_f (T X) or Bblk_f^T hatX_f (T^T X), in column chunks of <= 224
  for (int j0 = 0; j0 < k; j0 += kTallMaxN) {
    const int nj = k - j0 < kTallMaxN ? k - j0 : kTallMaxN;
    SSI_TRY(gemm_tall_batched(L2, nj, L2, !trans, Bb, L2, L2 * L2, Xh + j0 * ldh, ldh, L2,
                              Yh + j0 * ldh, ldh, L2, F, s));
  }
  if (gemm_form) {
    // Y_j (l x i, col-major ld l) = hatY_j (l x 2F) * Gt (2F x i)
    const double* Gt = tables + size_t(bt_ldF(i)) * 2 * i;
    return gemm_tall_batched(l, i, 2 * F, false, Yh, l, ldh, Gt, 2 * F, 0, Y, l, ldy, k, s);
  }
  const size_t smem_i = smem_twiddle(i) + sizeof(double) * size_t(F) * 2 * 32;
  if (smem_i > 48 * 1024)
    cudaFuncSetAttribute(bt_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_i));
  const dim3 grid(unsigned((l + 31) / 32), unsigned(k));
  bt_inverse_kernel<<<grid, DT, smem_i, s>>>(Yh, l, i, k, Y, ldy);
  return launch_check("bt_inverse_kernel");
}

}  // namespace ssi
