// push.cuh — Eq. 2: the implicit predictor-corrector
// velocity and position update of ONE particle.  The single implementation
// used by every kernel that moves a particle: the tiled mover (field samples
// from the TMA-staged box), the basic mover and the inflow injection (samples
// from the global field window).
//
//   v~   = gamma^n v^n + k E(x-bar)                    k = (q/m) dt / 2     (R7)
//   a    = k B(x-bar) / (c gamma~)                                           (R8)
//   v-bar = (v~ + v~ x a + (v~ . a) a) / (gamma~ (1 + a . a))               (R4, R6)
//   x-bar = x^n + v-bar dt / 2
// n_iter times (R2), the first field sample at x^n (R1); then
//   x^{n+1} = x^n + v-bar dt,   v^{n+1} = 2 v-bar - v^n                      (gamma == 1, R3)
// or, relativistic (REL = 1, NEXT-1, R5): gamma~ starts at gamma^n; each
// iterate u = 2 gamma~ v-bar - gamma^n v^n, gamma^{n+1} = sqrt(1 + u.u / c^2),
// gamma~ = (gamma^n + gamma^{n+1}) / 2; v^{n+1} = u / gamma^{n+1}.
//
// Positions are in cell units (h_d = dt / (2 Delta_d)).  `sample(xb, EB)`
// returns the PRE-SCALED fields at cell-unit position xb: EB[0..2] = k E,
// EB[3..5] = k B / c, and whether the sample was clamped to the window (R11).
#pragma once
#include "pic_internal.cuh"

namespace pic {

// 1/D for D >= 1 (D = 1 + |a|^2 of Eq. 2): MUFU.RCP64H seed + two Newton steps
// (error well below 1 ulp of the 1e-12 parity budget; no IEEE slow path).
__device__ __forceinline__ double rcp_ge1(double D) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(D));
  double e = fma(-D, r, 1.0);
  r = fma(r, e, r);
  e = fma(-D, r, 1.0);
  return fma(r, e, r);
}

// NIT > 0: compile-time iteration count (fully unrolled); NIT == 0: n_iter.
template <int NIT, int REL, class Sample>
__device__ __forceinline__ bool push_eq2(const double xn[3], const double vn[3], const double h[3], double c,
                                         int n_iter, const Sample &sample, double xnew[3], double vnew[3]) {
  const int nit = NIT > 0 ? NIT : n_iter;
  double xb[3] = {xn[0], xn[1], xn[2]};
  double vb[3] = {vn[0], vn[1], vn[2]};
  bool clamped = false;
  if constexpr (REL == 0) {
#pragma unroll
    for (int it = 0; it < nit; ++it) {
      double EB[6];
      clamped |= sample(xb, EB);
      // v~ = v^n + k E ; a = k B / c ; v-bar = (v~ + v~ x a + (v~ . a) a) / (1 + a . a)
      const double vt0 = vn[0] + EB[0], vt1 = vn[1] + EB[1], vt2 = vn[2] + EB[2];
      const double a0 = EB[3], a1 = EB[4], a2 = EB[5];
      const double dot = fma(vt0, a0, fma(vt1, a1, vt2 * a2));
      const double invD = rcp_ge1(fma(a0, a0, fma(a1, a1, fma(a2, a2, 1.0))));
      vb[0] = fma(dot, a0, fma(vt1, a2, fma(-vt2, a1, vt0))) * invD;
      vb[1] = fma(dot, a1, fma(vt2, a0, fma(-vt0, a2, vt1))) * invD;
      vb[2] = fma(dot, a2, fma(vt0, a1, fma(-vt1, a0, vt2))) * invD;
#pragma unroll
      for (int d = 0; d < 3; ++d) xb[d] = fma(vb[d], h[d], xn[d]);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      xnew[d] = fma(vb[d], 2.0 * h[d], xn[d]);
      vnew[d] = fma(2.0, vb[d], -vn[d]);
    }
  } else {
    const double ic2 = 1.0 / (c * c);
    const double gn = 1.0 / sqrt(1.0 - (vn[0] * vn[0] + vn[1] * vn[1] + vn[2] * vn[2]) * ic2);
    double gt = gn, g1 = gn, u1[3] = {gn * vn[0], gn * vn[1], gn * vn[2]};
#pragma unroll
    for (int it = 0; it < nit; ++it) {
      double EB[6];
      clamped |= sample(xb, EB);
      const double igt = 1.0 / gt;
      const double vt0 = fma(gn, vn[0], EB[0]), vt1 = fma(gn, vn[1], EB[1]), vt2 = fma(gn, vn[2], EB[2]);
      const double a0 = EB[3] * igt, a1 = EB[4] * igt, a2 = EB[5] * igt;
      const double dot = fma(vt0, a0, fma(vt1, a1, vt2 * a2));
      const double invD = rcp_ge1(fma(a0, a0, fma(a1, a1, fma(a2, a2, 1.0)))) * igt;
      vb[0] = fma(dot, a0, fma(vt1, a2, fma(-vt2, a1, vt0))) * invD;
      vb[1] = fma(dot, a1, fma(vt2, a0, fma(-vt0, a2, vt1))) * invD;
      vb[2] = fma(dot, a2, fma(vt0, a1, fma(-vt1, a0, vt2))) * invD;
#pragma unroll
      for (int d = 0; d < 3; ++d) u1[d] = fma(2.0 * gt, vb[d], -gn * vn[d]);
      g1 = sqrt(fma(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2], ic2, 1.0));
      gt = 0.5 * (gn + g1);
#pragma unroll
      for (int d = 0; d < 3; ++d) xb[d] = fma(vb[d], h[d], xn[d]);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      xnew[d] = fma(vb[d], 2.0 * h[d], xn[d]);
      vnew[d] = u1[d] / g1;
    }
  }
  return clamped;
}

// Pre-scaled samples from the global field window (R11 clamp, R12 weights).
struct WindowSampler {
  const Geom *g;
  const double *F;
  double ks, ks_c;
  __device__ __forceinline__ bool operator()(const double xb[3], double EB[6]) const {
    const bool cl = sample_window(*g, F, xb, EB);
#pragma unroll
    for (int m = 0; m < 6; ++m) EB[m] *= (m < 3) ? ks : ks_c;
    return cl;
  }
};

}  // namespace pic
