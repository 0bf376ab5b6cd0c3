// A13: hard criteria + 3D soft criteria (§2.1; Eq. (stabcriteria3D),
// PAPER.md:283-291 §2.3 step ii; readings A-17..A-21). One launch for all lags, one CTA
// per model order, one warp per pole; MAC over the l mode-shape components.
#include "rsvd.cuh"
#include "cluster.cuh"

namespace ssi {
namespace {

constexpr int NT = 256, NW = NT / 32;

__device__ __forceinline__ bool hard_ok(const ssi_pole_table& t, int64_t e, const ssi_criteria& c) {
  return t.xi[e] <= c.xi_max && t.mpc[e] > c.mpc_min && t.mpd[e] < c.mpd_max;
}

// 1 - MAC <= alpha_mac, MAC = |a^H b|^2 / (|a|^2 |b|^2); warp-collective.
__device__ bool mac_ok(const double* a, const double* b, int l, double alpha) {
  const int lane = threadIdx.x & 31;
  double re = 0.0, im = 0.0, na = 0.0, nb = 0.0;
  for (int i = lane; i < l; i += 32) {
    const double ar = a[2 * i], ai = a[2 * i + 1], br = b[2 * i], bi = b[2 * i + 1];
    re += ar * br + ai * bi;   // conj(a) b
    im += ar * bi - ai * br;
    na += ar * ar + ai * ai;
    nb += br * br + bi * bi;
  }
  re = warp_sum(re); im = warp_sum(im); na = warp_sum(na); nb = warp_sum(nb);
  const double mac = (re * re + im * im) / (na * nb);
  return (1.0 - mac) <= alpha;
}

// One launch for every lag: CTA (order o, lag g = blockIdx.y); the tables travel by value in a
// kernel-parameter TableSet (no host-to-device copy; at most SSI_MAX_LAGS lags per launch).
__global__ void __launch_bounds__(NT) stab_kernel(TableSet ts, int g0, ssi_criteria c, uint8_t* flags,
                                                  int32_t* stable_count) {
  __shared__ int cnt;
  const int o = blockIdx.x;
  const int gl = blockIdx.y, g = g0 + gl;
  const ssi_pole_table& cur = ts.t[gl];
  const ssi_pole_table& prev = ts.t[gl > 0 ? gl - 1 : SSI_MAX_LAGS - 1];   // slot MAX-1: lag g0 - 1
  const int has_prev = g > 0;
  flags += int64_t(gl) * cur.n_orders * cur.cap;
  stable_count += int64_t(gl) * cur.n_orders;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cap = cur.cap, l = cur.l;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int n_here = cur.count[o] > 0 ? cur.count[o] : 0;
  for (int sl = warp; sl < cap; sl += NW) {
    uint8_t flag = 0;
    const int64_t e = int64_t(o) * cap + sl;
    if (sl < n_here && hard_ok(cur, e, c)) {
      flag = 1;
      const double f = cur.f[e], xi = cur.xi[e];
      const double* sh = cur.shape + e * l * 2;
      // neighbors: (g, o-1) in cur, then (g-1, o) in prev
      for (int axis = 0; axis < 2 && flag == 1; ++axis) {
        const ssi_pole_table* t = axis == 0 ? &cur : &prev;
        const int oo = axis == 0 ? o - 1 : o;
        if (oo < 0 || (axis == 1 && !has_prev)) continue;
        const int nn = t->count[oo] > 0 ? t->count[oo] : 0;
        for (int q = 0; q < nn; ++q) {
          const int64_t eq = int64_t(oo) * cap + q;
          if (!hard_ok(*t, eq, c)) continue;
          const double fq = t->f[eq], xq = t->xi[eq];
          const double df = fabs(f - fq) / fmax(f, fq);
          const double dxi = fabs(xi - xq) / fmax(xi, xq);
          if (!(df <= c.alpha_f && dxi <= c.alpha_xi)) continue;
          if (mac_ok(sh, t->shape + eq * l * 2, l, c.alpha_mac)) { flag = 2; break; }
        }
      }
    }
    if (lane == 0) {
      flags[e] = flag;
      if (flag == 2) atomicAdd(&cnt, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) stable_count[o] = cnt;
}

}  // namespace

ssi_status stab3d_run(const ssi_pole_table* tables, int n_lags, const ssi_criteria& crit,
                      uint8_t* flags, int32_t* stable_count, cudaStream_t s) {
  const int no = tables[0].n_orders, cap = tables[0].cap;
  // lags in groups of SSI_MAX_LAGS - 1; the last slot carries the group's predecessor lag
  for (int g0 = 0; g0 < n_lags; g0 += SSI_MAX_LAGS - 1) {
    const int ng = n_lags - g0 < SSI_MAX_LAGS - 1 ? n_lags - g0 : SSI_MAX_LAGS - 1;
    TableSet ts;
    for (int j = 0; j < SSI_MAX_LAGS; ++j) ts.t[j] = tables[g0 + (j < ng ? j : 0)];
    ts.t[SSI_MAX_LAGS - 1] = tables[g0 > 0 ? g0 - 1 : 0];
    stab_kernel<<<dim3(unsigned(no), unsigned(ng)), NT, 0, s>>>(ts, g0, crit, flags + int64_t(g0) * no * cap,
                                                                stable_count + int64_t(g0) * no);
    SSI_TRY(launch_check("stab_kernel"));
  }
  return SSI_OK;
}

}  // namespace ssi
