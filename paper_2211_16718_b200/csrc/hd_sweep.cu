// hd_sweep.cu -- fused WENO5 (state + flux) / Roe / flux-difference sweeps.
//
// Replaces kernels.py:68-204 (hyper_sweep) together with the flux arrays
// upwind.py:116-127 (_flux_components) that the reference materialises per
// dimension: here f(u) is formed on the fly when a point enters the window.
//
// Execution model: one thread marches one segment [c0, c1) of one grid line
// along the sweep axis, holding a 5-point register window of the state and
// flux (u0..u4, f1..f4; f0 == u_{1+dim}).  At cell c the window (c-2..c+2)
// yields the RIGHT reconstruction at c-1/2 and the LEFT reconstruction at
// c+1/2 (the reference's mirrored stencils, K:104-123, share this window), so
// each window is evaluated once and each interface flux once (the reference's
// fprev carry, K:197-203).  The Roe flux at c-1/2 combines the carried left
// state with the fresh right state.
//
// y/z sweeps: lanes are consecutive x columns -> every window load and every
// inc read-modify-write is a fully coalesced 256-byte warp access.
// x sweep: lanes are consecutive y rows; each lane walks its row sequentially
// (sector reuse through L1).
#include <cstring>

#include "hd_device.cuh"

namespace hd {

// ---------------------------------------------------------------------------
// WENO5 reconstructions
// ---------------------------------------------------------------------------

// kernels.py:25-57, exact operation order.
__device__ __forceinline__ double recon5_exact(double f0, double f1, double f2, double f3,
                                               double f4, double eps, int power) {
  const double t1 = xa(xs(f0, xm(2.0, f1)), f2);
  const double s1 = xa(xs(f0, xm(4.0, f1)), xm(3.0, f2));
  const double b1 = xa(xm(C13_12, xm(t1, t1)), xm(0.25, xm(s1, s1)));
  const double t2 = xa(xs(f1, xm(2.0, f2)), f3);
  const double s2 = xs(f1, f3);
  const double b2 = xa(xm(C13_12, xm(t2, t2)), xm(0.25, xm(s2, s2)));
  const double t3 = xa(xs(f2, xm(2.0, f3)), f4);
  const double s3 = xa(xs(xm(3.0, f2), xm(4.0, f3)), f4);
  const double b3 = xa(xm(C13_12, xm(t3, t3)), xm(0.25, xm(s3, s3)));
  const double d1 = xa(eps, b1), d2 = xa(eps, b2), d3 = xa(eps, b3);
  double e1 = d1, e2 = d2, e3 = d3;
  for (int q = 0; q < power - 1; ++q) {
    e1 = xm(e1, d1);
    e2 = xm(e2, d2);
    e3 = xm(e3, d3);
  }
  const double a1 = xd(0.1, e1), a2 = xd(0.6, e2), a3 = xd(0.3, e3);
  const double asum = xa(xa(a1, a2), a3);
  const double w1 = xd(a1, asum), w2 = xd(a2, asum), w3 = xd(a3, asum);
  const double c1 = xa(xs(xm(C1_3, f0), xm(C7_6, f1)), xm(C11_6, f2));
  const double c2 = xa(xa(xm(-C1_6, f1), xm(C5_6, f2)), xm(C1_3, f3));
  const double c3 = xs(xa(xm(C1_3, f2), xm(C5_6, f3)), xm(C1_6, f4));
  return xa(xa(xm(w1, c1), xm(w2, c2)), xm(w3, c3));
}

// Both reconstructions of one 5-point window q0..q4 (centred on cell c):
//   left  = value at c+1/2 (stencil q0..q4),
//   right = value at c-1/2 (mirrored stencil q4..q0).
// The mirrored stencil has the same smoothness indicators in reverse order
// (weno.py:9-11), so beta/eps terms are computed once; the three normalised
// weights of each side share one reciprocal:
//   w_k = (g_k / e_k) / sum_j (g_j / e_j) = g_k prod_{j!=k} e_j / sum_j g_j prod_{i!=j} e_i.
__device__ __forceinline__ void recon_pair_d(double D0, double D1, double D2, double D3, double q2,
                                             double eps, int power, double& left, double& right);

template <bool EXACT>
__device__ __forceinline__ void recon_pair(double q0, double q1, double q2, double q3, double q4,
                                           double eps, int power, double& left, double& right) {
  if constexpr (EXACT) {
    left = recon5_exact(q0, q1, q2, q3, q4, eps, power);
    right = recon5_exact(q4, q3, q2, q1, q0, eps, power);
  } else {
    recon_pair_d(q1 - q0, q2 - q1, q3 - q2, q4 - q3, q2, eps, power, left, right);
  }
}

// The fast pair from the window's first differences D_i = q_{i+1} - q_i and its
// centre q2 (a marching window can carry the differences instead of the values).
__device__ __forceinline__ void recon_pair_d(double D0, double D1, double D2, double D3, double q2,
                                             double eps, int power, double& left, double& right) {
  {
    // Everything in first differences D_i = q_{i+1} - q_i of the window:
    //   beta_k = 13/12 t_k^2 + 1/4 s_k^2 with t1 = D1-D0, s1 = 3D1-D0, t2 = D2-D1,
    //   s2 = -(D1+D2), t3 = D3-D2, s3 = D3-3D2 (scaled by 12; the common factor
    //   cancels in the normalised weights once eps is scaled too), and since the
    //   weights sum to one each value is q2 + sum_k w_k (c_k - q2), with
    //   6 (c_k - q2) = 5D1-2D0, D1+2D2, 4D2-D3 (left) and 2D3-5D2, -(D2+2D1),
    //   D0-4D1 (right).
    // expanded: 12 beta1 = 13 t1^2 + 3 s1^2 = 4 (10 D1^2 - 11 D0 D1 + 4 D0^2), and
    // likewise 3 beta2 = 4 D1^2 - 5 D1 D2 + 4 D2^2, 3 beta3 = 10 D2^2 - 11 D2 D3 + 4 D3^2;
    // all three (and eps) scaled by the common factor 3/4, which cancels in the
    // normalised weights, and factored so every constant is exact and each
    // indicator is two FMAs on a shared square:
    //   d1 = D0 (D0 - 2.75 D1) + 2.5 D1^2,  d2 = D1 (D1 - 1.25 D2) + D2^2,
    //   d3 = D3 (D3 - 2.75 D2) + 2.5 D2^2   (11 FP64 operations instead of 16)
    const double S1 = D1 * D1, S2 = D2 * D2;
    const double epsq = 0.75 * eps;
    const double d1 = fma(D0, fma(-2.75, D1, D0), fma(2.5, S1, epsq));
    const double d2 = fma(D1, fma(-1.25, D2, D1), S2 + epsq);
    const double d3 = fma(D3, fma(-2.75, D2, D3), fma(2.5, S2, epsq));
    double e1 = d1, e2 = d2, e3 = d3;
    for (int q = 0; q < power - 1; ++q) {
      e1 *= d1;
      e2 *= d2;
      e3 *= d3;
    }
    const double e12 = e1 * e2, e13 = e1 * e3, e23 = e2 * e3;
    // left: weights (0.1/e1, 0.6/e2, 0.3/e3) ~ (e23, 6 e13, 3 e12), corrections
    // (c_k - q2) = (5D1-2D0)/6, (D1+2D2)/6, (4D2-D3)/6; the 1/6 goes into the
    // numerator's weights (6 e13 / 6 = e13, 3 e12 / 6 = e12 / 2) except for the
    // first term, whose correction takes it (5/6 D1 - 1/3 D0), so the normaliser
    // is two FMAs on the products: 13 operations per side instead of 14.5
    const double al1 = fma(5.0 / 6.0, D1, (-1.0 / 3.0) * D0), al2 = fma(2.0, D2, D1),
                 al3 = fma(4.0, D2, -D3);
    const double numl = fma(e23, al1, fma(e13, al2, (0.5 * e12) * al3));
    left = fma(numl, frcp_weights(fma(6.0, e13, fma(3.0, e12, e23))), q2);
    // right (mirrored): (0.1/e3, 0.6/e2, 0.3/e1) ~ (e12, 6 e13, 3 e23), corrections
    // (2D3-5D2)/6, -(D2+2D1)/6, (D0-4D1)/6
    const double ar1 = fma(-5.0 / 6.0, D2, (1.0 / 3.0) * D3), ar2 = fma(2.0, D1, D2),
                 ar3 = fma(-4.0, D1, D0);
    const double numr = fma(e12, ar1, fma(-e13, ar2, (0.5 * e23) * ar3));
    right = fma(numr, frcp_weights(fma(6.0, e13, fma(3.0, e23, e12))), q2);
  }
}

// kernels.py:60-65
template <bool EXACT>
__device__ __forceinline__ double entropy_fixed(double lam, double delta) {
  const double mag = fabs(lam);
  if (delta > 0.0 && mag < delta) {
    if constexpr (EXACT) return xd(xa(xm(lam, lam), xm(delta, delta)), xm(2.0, delta));
    return (lam * lam + delta * delta) / (2.0 * delta);
  }
  return mag;
}

// ---------------------------------------------------------------------------
// Roe interface flux (kernels.py:125-195)
// ---------------------------------------------------------------------------
template <int DIM, bool EXACT>
__device__ __forceinline__ void roe_flux(const double (&uL)[NV], const double (&uR)[NV],
                                         const double (&fl)[NV], const double (&fr)[NV],
                                         const Phys& ph, double (&flux)[NV]) {
  constexpr int mn = 1 + DIM, mt1 = 1 + (DIM + 1) % 3, mt2 = 1 + (DIM + 2) % 3;
  const double gm1 = ph.gm1;
  if constexpr (EXACT) {
    const double rl = uL[0];
    const double il = xd(1.0, rl);
    const double vxl = xm(uL[1], il), vyl = xm(uL[2], il), vzl = xm(uL[3], il);
    const double pl = xm(gm1, xs(uL[4], xm(xm(0.5, rl), xa(xa(xm(vxl, vxl), xm(vyl, vyl)), xm(vzl, vzl)))));
    const double rr = uR[0];
    const double ir = xd(1.0, rr);
    const double vxr = xm(uR[1], ir), vyr = xm(uR[2], ir), vzr = xm(uR[3], ir);
    const double pr = xm(gm1, xs(uR[4], xm(xm(0.5, rr), xa(xa(xm(vxr, vxr), xm(vyr, vyr)), xm(vzr, vzr)))));
    const double sl = xsqrt(rl), sr = xsqrt(rr);
    const double isw = xd(1.0, xa(sl, sr));
    const double ua = xm(xa(xm(sl, vxl), xm(sr, vxr)), isw);
    const double va = xm(xa(xm(sl, vyl), xm(sr, vyr)), isw);
    const double wa = xm(xa(xm(sl, vzl), xm(sr, vzr)), isw);
    const double Hl = xm(xa(uL[4], pl), il);
    const double Hr = xm(xa(uR[4], pr), ir);
    const double Ha = xm(xa(xm(sl, Hl), xm(sr, Hr)), isw);
    const double q2 = xa(xa(xm(ua, ua), xm(va, va)), xm(wa, wa));
    const double a2 = xm(gm1, xs(Ha, xm(0.5, q2)));
    const double aa = xsqrt(a2);
    double vn, vt1, vt2;
    if (DIM == 0) { vn = ua; vt1 = va; vt2 = wa; }
    else if (DIM == 1) { vn = va; vt1 = wa; vt2 = ua; }
    else { vn = wa; vt1 = ua; vt2 = va; }
    const double dr = xs(uR[0], uL[0]);
    const double dmn = xs(uR[mn], uL[mn]);
    const double dt1 = xs(uR[mt1], uL[mt1]);
    const double dt2 = xs(uR[mt2], uL[mt2]);
    const double dE = xs(uR[4], uL[4]);
    const double b1 = xd(gm1, a2);
    const double b2 = xm(xm(0.5, b1), q2);
    const double ia = xd(1.0, aa);
    const double b1vt1dt1 = xm(xm(b1, vt1), dt1), b1vt2dt2 = xm(xm(b1, vt2), dt2);
    const double b1dE = xm(b1, dE);
    const double s1 = xm(0.5, xa(xs(xs(xs(xm(xa(b2, xm(vn, ia)), dr), xm(xa(xm(b1, vn), ia), dmn)),
                                       b1vt1dt1), b1vt2dt2), b1dE));
    const double s2 = xs(xa(xa(xa(xm(xs(1.0, b2), dr), xm(xm(b1, vn), dmn)), b1vt1dt1), b1vt2dt2), b1dE);
    const double s3 = xa(xm(-vt1, dr), dt1);
    const double s4 = xa(xm(-vt2, dr), dt2);
    const double s5 = xm(0.5, xa(xs(xs(xs(xm(xs(b2, xm(vn, ia)), dr), xm(xs(xm(b1, vn), ia), dmn)),
                                       b1vt1dt1), b1vt2dt2), b1dE));
    const double lam_n = entropy_fixed<true>(vn, ph.delta);
    const double k1 = xm(entropy_fixed<true>(xs(vn, aa), ph.delta), s1);
    const double k2 = xm(lam_n, s2);
    const double k3 = xm(lam_n, s3);
    const double k4 = xm(lam_n, s4);
    const double k5 = xm(entropy_fixed<true>(xa(vn, aa), ph.delta), s5);
    const double diss_r = xa(xa(k1, k2), k5);
    const double diss_n = xa(xa(xm(k1, xs(vn, aa)), xm(k2, vn)), xm(k5, xa(vn, aa)));
    const double diss_1 = xa(xa(xa(xm(k1, vt1), xm(k2, vt1)), k3), xm(k5, vt1));
    const double diss_2 = xa(xa(xa(xm(k1, vt2), xm(k2, vt2)), k4), xm(k5, vt2));
    const double diss_E = xa(xa(xa(xa(xm(k1, xs(Ha, xm(vn, aa))), xm(k2, xm(0.5, q2))), xm(k3, vt1)),
                                xm(k4, vt2)), xm(k5, xa(Ha, xm(vn, aa))));
    flux[0] = xs(xm(0.5, xa(fl[0], fr[0])), xm(0.5, diss_r));
    flux[1] = xm(0.5, xa(fl[1], fr[1]));
    flux[2] = xm(0.5, xa(fl[2], fr[2]));
    flux[3] = xm(0.5, xa(fl[3], fr[3]));
    flux[4] = xs(xm(0.5, xa(fl[4], fr[4])), xm(0.5, diss_E));
    flux[mn] = xs(flux[mn], xm(0.5, diss_n));
    flux[mt1] = xs(flux[mt1], xm(0.5, diss_1));
    flux[mt2] = xs(flux[mt2], xm(0.5, diss_2));
  } else {
    // rsqrt-based: 1/rho = (rho^-1/2)^2, sqrt(rho) = rho * rho^-1/2
    const double rl = uL[0], rr = uR[0];
    const double isl = rsqrt(rl), isr = rsqrt(rr);
    const double il = isl * isl, ir = isr * isr;
    const double sl = rl * isl, sr = rr * isr;
    // kinetic energy 0.5*rho*|v|^2 = 0.5*|m|^2/rho
    const double pl = gm1 * (uL[4] - (0.5 * il) * (uL[1] * uL[1] + uL[2] * uL[2] + uL[3] * uL[3]));
    const double pr = gm1 * (uR[4] - (0.5 * ir) * (uR[1] * uR[1] + uR[2] * uR[2] + uR[3] * uR[3]));
    const double isw = frcp(sl + sr);
    // sl*v_l = m_l * isl (since m = rho v): saves the velocity products
    const double ua = (uL[1] * isl + uR[1] * isr) * isw;
    const double va = (uL[2] * isl + uR[2] * isr) * isw;
    const double wa = (uL[3] * isl + uR[3] * isr) * isw;
    // sl*H_l = (E_l + p_l) * isl
    const double Ha = ((uL[4] + pl) * isl + (uR[4] + pr) * isr) * isw;
    const double q2 = ua * ua + va * va + wa * wa;
    const double a2 = gm1 * (Ha - 0.5 * q2);
    const double ia = rsqrt(a2);
    const double aa = a2 * ia;
    double vn, vt1, vt2;
    if (DIM == 0) { vn = ua; vt1 = va; vt2 = wa; }
    else if (DIM == 1) { vn = va; vt1 = wa; vt2 = ua; }
    else { vn = wa; vt1 = ua; vt2 = va; }
    const double dr = uR[0] - uL[0];
    const double dmn = uR[mn] - uL[mn];
    const double dt1 = uR[mt1] - uL[mt1];
    const double dt2 = uR[mt2] - uL[mt2];
    const double dE = uR[4] - uL[4];
    const double b1 = gm1 * (ia * ia);
    const double b2 = 0.5 * b1 * q2;
    // common part of s1/s5: b2*dr - b1*(vn*dmn + vt1*dt1 + vt2*dt2 - dE)
    const double proj = vn * dmn + vt1 * dt1 + vt2 * dt2 - dE;
    const double common = b2 * dr - b1 * proj;
    const double acoustic = ia * (vn * dr - dmn);
    const double s1 = 0.5 * (common + acoustic);
    const double s5 = 0.5 * (common - acoustic);
    const double s2 = dr - common;  // (1-b2) dr + b1 (vn dmn + vt1 dt1 + vt2 dt2) - b1 dE
    const double s3 = dt1 - vt1 * dr;
    const double s4 = dt2 - vt2 * dr;
    const double lam_n = entropy_fixed<false>(vn, ph.delta);
    const double k1 = entropy_fixed<false>(vn - aa, ph.delta) * s1;
    const double k2 = lam_n * s2;
    const double k3 = lam_n * s3;
    const double k4 = lam_n * s4;
    const double k5 = entropy_fixed<false>(vn + aa, ph.delta) * s5;
    const double k15 = k1 + k5;
    const double k125 = k15 + k2;
    const double diss_r = k125;
    const double diss_n = k125 * vn + (k5 - k1) * aa;
    const double diss_1 = k125 * vt1 + k3;
    const double diss_2 = k125 * vt2 + k4;
    const double diss_E = k15 * Ha + (k5 - k1) * (vn * aa) + k2 * (0.5 * q2) + k3 * vt1 + k4 * vt2;
    flux[0] = 0.5 * ((fl[0] + fr[0]) - diss_r);
    flux[4] = 0.5 * ((fl[4] + fr[4]) - diss_E);
    flux[mn] = 0.5 * ((fl[mn] + fr[mn]) - diss_n);
    flux[mt1] = 0.5 * ((fl[mt1] + fr[mt1]) - diss_1);
    flux[mt2] = 0.5 * ((fl[mt2] + fr[mt2]) - diss_2);
  }
}

// ---------------------------------------------------------------------------
// Point decode + directional flux (physics.py:240-255, upwind.py:116-127)
// ---------------------------------------------------------------------------
template <int DIM, bool EXACT>
__device__ __forceinline__ void point_flux(const double (&u)[NV], double gm1, double (&f)[NV],
                                           double& inv_out, double (&prim)[4]) {
  double vx, vy, vz, p, inv;
  if constexpr (EXACT) {
    inv = xd(1.0, u[0]);
    vx = xm(u[1], inv);
    vy = xm(u[2], inv);
    vz = xm(u[3], inv);
    p = xm(gm1, xs(u[4], xm(xm(0.5, u[0]), xa(xa(xm(vx, vx), xm(vy, vy)), xm(vz, vz)))));
  } else {
    inv = frcp(u[0]);
    vx = u[1] * inv;
    vy = u[2] * inv;
    vz = u[3] * inv;
    p = gm1 * (u[4] - (0.5 * inv) * (u[1] * u[1] + u[2] * u[2] + u[3] * u[3]));
  }
  const double vd = DIM == 0 ? vx : (DIM == 1 ? vy : vz);
  f[0] = u[1 + DIM];
  if constexpr (EXACT) {
    f[1] = xm(u[1], vd);
    f[2] = xm(u[2], vd);
    f[3] = xm(u[3], vd);
    f[1 + DIM] = xa(f[1 + DIM], p);
    f[4] = xm(xa(u[4], p), vd);
  } else {
    f[1] = u[1] * vd;
    f[2] = u[2] * vd;
    f[3] = u[3] * vd;
    f[1 + DIM] += p;
    f[4] = (u[4] + p) * vd;
  }
  inv_out = inv;
  prim[0] = vx;
  prim[1] = vy;
  prim[2] = vz;
  prim[3] = p;
}

constexpr int SWEEP_THREADS = 64;
// Window placement and register cap per sweep direction (measured on B200 at
// 512^3, tools/sweep_bench.py):
//   y, z: window in shared memory, 6 blocks of 64 threads per SM (12 warps,
//         <= 168 registers, no spills) -- 7.3 ms vs 8.3 ms with a register window
//   x:    register window, 4 blocks per SM -- its lanes walk different rows, and
//         more resident warps thrash L1 (15.5 ms at 6 blocks vs 9.9 ms)
// x: 4 blocks/SM with a register window; y: 6 blocks/SM with the window in the
// shared ring; z (UPDATE role, flux window in the ring): 4 blocks/SM and up to 255
// registers -- 9.7 -> 9.25 ms at 512^3 (6 blocks: spills; 4 without the window: 11.4)
constexpr int SWEEP_MIN_BLOCKS_X = 4, SWEEP_MIN_BLOCKS_Y = 6, SWEEP_MIN_BLOCKS_Z = 4;
template <int DIM> struct SweepCfg {
  static constexpr bool smem_window = DIM != 0;
  static constexpr int min_blocks =
      DIM == 0 ? SWEEP_MIN_BLOCKS_X : (DIM == 1 ? SWEEP_MIN_BLOCKS_Y : SWEEP_MIN_BLOCKS_Z);
};

// What a sweep does besides -dF/dx (the fast-mode stage pipeline, hd_api.cu):
//   ROLE_PLAIN  inc (-)= dF/dx
//   ROLE_VISC   y sweep: also adds the x and y viscous flux divergence
//               D_x F_x + D_y F_y (viscous.py:119-120) of the cell it writes
//   ROLE_UPDATE z sweep, last kernel of a stage: adds D_z F_z and feeds the
//               finished increment to the RK stage update (timeint.py:168-193)
//               instead of storing it; the new stage state goes out with its face
//               images (into the z neighbours' ghost planes in peer mode)
// The flux group differentiated along the sweep rides in the shared ring with the
// window (one HBM read per value); the y sweep reads D_x's stencil directly.
// ROLE_UPDATE_DIAG: ROLE_UPDATE of the last stage with the diagnostics of the new
// state folded in (hd_arm_reduce) -- a separate instantiation, so the other stages'
// update kernel carries none of its registers
// ROLE_RK4_*: ROLE_UPDATE specialised to the stages of the classical RK4 tableau
// (timeint.py:181-193), so no run-time flag, predicated load or unused operand
// remains: A = stage 0 (acc = k, no accumulator read), B = stages 1, 2 (acc += 2k),
// C = stage 3 (u + dt/6 (acc + k), no accumulator write), C_DIAG = C with the
// diagnostics.  ROLE_UPDATE / ROLE_UPDATE_DIAG stay the generic (TVD-RK3) path.
constexpr int ROLE_PLAIN = 0, ROLE_VISC = 1, ROLE_UPDATE = 2, ROLE_UPDATE_DIAG = 3;
constexpr int ROLE_RK4_A = 4, ROLE_RK4_B = 5, ROLE_RK4_C = 6, ROLE_RK4_C_DIAG = 7;

struct SweepArgs {
  Geo geo;
  Phys ph;
  const double* u;
  double* inc;
  double inv_dx;
  int seg;          // segment length
  int accumulate;   // 0: inc = 0 - d ; 1: inc -= d
  int check;        // latch positivity of interior points
  unsigned long long* err;
  int64_t tag;
  // ROLE_VISC / ROLE_UPDATE
  const double* vflux;  // 9 symmetric viscous flux fields (nullptr: inviscid)
  // ROLE_UPDATE
  RKArgs rk;
  // ROLE_UPDATE, last stage: diagnostics of the new state fused in (nullptr: off);
  // one partial (HD_RED_* layout) per warp
  double* fred;
  int64_t fred_tag;
  double rh[3];  // 1 / h
};

// Line geometry: thread -> interior coords of the line origin
template <int DIM>
__device__ __forceinline__ bool line_of(const SweepArgs& a, int& i, int& j, int& k) {
  const Geo& G = a.geo;
  if (DIM == 0) {
    j = blockIdx.x * blockDim.x + threadIdx.x;
    k = blockIdx.y * blockDim.y + threadIdx.y;
    i = 0;
    return j < G.n[1] && k < G.n[2];
  } else if (DIM == 1) {
    i = blockIdx.x * blockDim.x + threadIdx.x;
    k = blockIdx.y * blockDim.y + threadIdx.y;
    j = 0;
    return i < G.n[0] && k < G.n[2];
  } else {
    i = blockIdx.x * blockDim.x + threadIdx.x;
    j = blockIdx.y * blockDim.y + threadIdx.y;
    k = 0;
    return i < G.n[0] && j < G.n[1];
  }
}

// PW: WENO power fixed at compile time (2, the reference default), or 0 = read
// at run time.  A run-time exponent loop inside each of the 18 reconstructions
// of an interface splits the code into basic blocks the scheduler cannot
// interleave; the fixed form lets the independent variables overlap.
template <int DIM, bool EXACT, int ROLE, int PW>
__global__ void __launch_bounds__(SWEEP_THREADS, SweepCfg<DIM>::min_blocks) sweep_kernel(const SweepArgs a) {
  constexpr bool SMEM_WINDOW = SweepCfg<DIM>::smem_window;
  int li, lj, lk;
  if (!line_of<DIM>(a, li, lj, lk)) return;
  const Geo& G = a.geo;
  const int64_t base = G.idx(li, lj, lk);
  const int seg_id = blockIdx.z;
  const int nd = G.n[DIM];
  const int c0 = seg_id * a.seg;
  if (c0 >= nd) return;
  const int c1 = min(c0 + a.seg, nd);
  const int64_t sd = G.stride(DIM);
  const int64_t np = G.npts;
  const double* __restrict__ u = a.u + base;
  double* __restrict__ inc = a.inc + base;
  const double gm1 = a.ph.gm1, eps = a.ph.eps;
  const int power = PW ? PW : a.ph.power;

  // Window in shared memory (SMEM_WINDOW): a 5-slot ring per thread, slot =
  // position mod 5, 9 values per point (u0..u4, f1..f4; f0 == u_{1+dim});
  // consecutive threads hold consecutive doubles, so every access is bank-
  // conflict free, and the 45-double window stays out of the register file.
  // Otherwise a register window: point w holds line position c - 2 + w.
  // The VISC/UPDATE roles keep a second ring: the viscous flux group F_dim
  // (differentiated along the sweep), so D_dim F_dim reads each flux value from
  // HBM once (y 8.28 -> 8.06 ms, z 9.7 -> 9.25 ms at 512^3 against stencil loads).
  // Its values go global -> shared with cp.async, one iteration ahead: loaded
  // into registers instead, their scoreboard was shared with loads issued late in
  // the previous iteration and the store into the ring stalled on them (ncu: 20%
  // of the y sweep's and 24% of the z sweep's warp samples).
  constexpr bool VROLE = ROLE != ROLE_PLAIN;
  constexpr bool UPD = ROLE >= ROLE_UPDATE;
  constexpr bool DIAG = (ROLE == ROLE_UPDATE_DIAG || ROLE == ROLE_RK4_C_DIAG) && !EXACT;
  constexpr bool RK4S = ROLE >= ROLE_RK4_A;  // a specialised RK4 stage
  constexpr bool READ_ACC = ROLE == ROLE_RK4_B || ROLE == ROLE_RK4_C || ROLE == ROLE_RK4_C_DIAG;
  constexpr bool FWIN = VROLE && SMEM_WINDOW;
  constexpr int FS = 6;  // flux ring slots: positions c-3 .. c+2 at iteration c
  __shared__ double ring[SMEM_WINDOW ? 5 * 9 * SWEEP_THREADS : 1];
  __shared__ double fring[FWIN ? FS * 4 * SWEEP_THREADS : 1];
  double* const mine = ring + threadIdx.y * 32 + threadIdx.x;
  double* const fmine = fring + threadIdx.y * 32 + threadIdx.x;
  auto slot = [&](int m) -> double* { return mine + ((m + 5) % 5) * (9 * SWEEP_THREADS); };
  auto fslot = [&](int m) -> double* { return fmine + ((m + FS) % FS) * (4 * SWEEP_THREADS); };
  double wu[5][NV], wf[5][NV];
  const bool fwin = FWIN && a.vflux;
  // flux group at position m -> fslot(m); one cp.async group per position
  auto fissue = [&](int m) {
    if (fwin) {
      double* sp = fslot(m);
#pragma unroll
      for (int r = 0; r < 4; ++r)
        cp_async8(sp + r * SWEEP_THREADS, a.vflux + (int64_t)vf_field(DIM, r + 1) * np + base + (int64_t)m * sd);
    }
    cp_async_commit();
  };

  // raw loads are issued one iteration before the point enters the window
  // (and the inc read of a cell at the top of the iteration that writes it),
  // so HBM/L2 latency hides behind a full window of FP64 work
  auto fetch = [&](int m, double (&dst)[NV]) {
    const double* q = u + (int64_t)m * sd;
#pragma unroll
    for (int v = 0; v < NV; ++v) dst[v] = __ldg(q + v * np);
  };
  auto ingest = [&](int m, const double (&src)[NV], double (&uu)[NV], double (&ff)[NV]) {
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = src[v];
    double inv, pv[4];
    point_flux<DIM, EXACT>(uu, gm1, ff, inv, pv);
    if constexpr (SMEM_WINDOW) {
      double* sp = slot(m);
#pragma unroll
      for (int v = 0; v < NV; ++v) sp[v * SWEEP_THREADS] = uu[v];
#pragma unroll
      for (int v = 1; v < NV; ++v) sp[(NV - 1 + v) * SWEEP_THREADS] = ff[v];
    }
    if (a.check && m >= 0 && m < nd) {
      const int code = !(uu[0] > 0.0) ? 1 : (!(pv[3] > 0.0) ? 2 : 0);
      if (code)
        latch_error(a.err, a.tag, code,
                    first_image(G, DIM == 0 ? m : li, DIM == 1 ? m : lj, DIM == 2 ? m : lk));
    }
  };

  double pre[NV];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    fetch(c0 - 3 + w, pre);
    ingest(c0 - 3 + w, pre, wu[w + 1], wf[w + 1]);
  }
  fetch(c0 + 1, pre);
  if constexpr (FWIN)
    for (int m = c0 - 2; m <= c0; ++m) fissue(m);

  double lu[NV], lf[NV];  // left states at c-1/2 (carried)
  // fused diagnostics of the new state (ROLE_UPDATE, last stage)
  double diag[9] = {-INFINITY, -INFINITY, -INFINITY, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double fprev[NV];
  for (int c = c0 - 1; c <= c1; ++c) {
    // shift; position c+2 enters from the prefetch buffer
    if constexpr (!SMEM_WINDOW) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          wu[w][v] = wu[w + 1][v];
          wf[w][v] = wf[w + 1][v];
        }
      }
    }
    ingest(c + 2, pre, wu[4], wf[4]);
    if (c < c1) fetch(c + 3, pre);
    if constexpr (FWIN) {
      if (c < c1) fissue(c + 2);
      else cp_async_commit();  // keep one group per iteration
    }
    const bool wr = c > c0;
    // y sweep: pull the next cell's D_x stencil lines (x group) into L1 a window
    // ahead (8.05 -> 7.92 ms at 512^3)
    if constexpr (ROLE == ROLE_VISC) {
      if (a.vflux && c < c1) {
        const int64_t qn = base + (int64_t)c * sd;
#pragma unroll
        for (int r = 1; r < NV; ++r)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.vflux + (int64_t)vf_field(0, r) * np + qn));
      }
    }
    double* q = inc + (int64_t)(c - 1) * sd;
    // ROLE_UPDATE: the RK inputs of cell c-1 (base state, accumulator) are
    // loaded here, a full window of FP64 work before the update consumes them
    double ru0[NV], racc[NV];
    if constexpr (UPD) {
      const int64_t qo = base + (int64_t)(c - 1) * sd;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        ru0[v] = wr ? a.rk.u[qo + v * np] : 0.0;
        if constexpr (RK4S) racc[v] = (READ_ACC && wr) ? a.rk.acc[qo + v * np] : 0.0;
        else racc[v] = (wr && a.rk.rd_acc) ? a.rk.acc[qo + v * np] : 0.0;
      }
    }
    double old[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) old[v] = (wr && a.accumulate) ? q[v * np] : 0.0;
    // reconstructions of window c: ru/rf at c-1/2, nu/nf at c+1/2
    double ru[NV], rf[NV], nu[NV], nf[NV];
    if constexpr (SMEM_WINDOW) {
      const double* w0 = slot(c - 2);
      const double* w1 = slot(c - 1);
      const double* w2 = slot(c);
      const double* w3 = slot(c + 1);
      // position c+2 was ingested this iteration: its values are still in registers
#pragma unroll
      for (int v = 0; v < 2 * NV - 1; ++v) {
        double l, r;
        const double q4 = v < NV ? wu[4][v] : wf[4][v - NV + 1];
        recon_pair<EXACT>(w0[v * SWEEP_THREADS], w1[v * SWEEP_THREADS], w2[v * SWEEP_THREADS],
                          w3[v * SWEEP_THREADS], q4, eps, power, l, r);
        if (v < NV) { nu[v] = l; ru[v] = r; }
        else { nf[v - NV + 1] = l; rf[v - NV + 1] = r; }
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        recon_pair<EXACT>(wu[0][v], wu[1][v], wu[2][v], wu[3][v], wu[4][v], eps, power, nu[v], ru[v]);
#pragma unroll
      for (int v = 1; v < NV; ++v)
        recon_pair<EXACT>(wf[0][v], wf[1][v], wf[2][v], wf[3][v], wf[4][v], eps, power, nf[v], rf[v]);
    }
    nf[0] = nu[1 + DIM];
    rf[0] = ru[1 + DIM];
    if (c >= c0) {
      double flux[NV];
      roe_flux<DIM, EXACT>(lu, ru, lf, rf, a.ph, flux);
      if (wr) {
        double val[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          // accumulate: inc -= d ; first sweep of an RHS: inc = 0 - d (upwind.py:181-182)
          if constexpr (EXACT) val[v] = xs(old[v], xm(xs(flux[v], fprev[v]), a.inv_dx));
          else val[v] = old[v] - (flux[v] - fprev[v]) * a.inv_dx;
        }
        if (fwin) {
          // y sweep: D_x F_x from row loads (x neighbours share the lanes' lines);
          // then D_dim F_dim from the window, positions c-3 .. c+1
          if constexpr (ROLE == ROLE_VISC)
            add_viscous_divergence<EXACT>(a.vflux, G, base + (int64_t)(c - 1) * sd, 1, val);
          cp_async_wait<1>();  // position c+1 landed (c+2 may be in flight)
          const double* m2 = fslot(c - 3);
          const double* m1 = fslot(c - 2);
          const double* p1 = fslot(c);
          const double* p2 = fslot(c + 1);
          const double coef = 1.0 / (12.0 * G.h[DIM]);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int o = r * SWEEP_THREADS;
            val[r + 1] += (8.0 * (p1[o] - m1[o]) + (m2[o] - p2[o])) * coef;
          }
        }
        if constexpr (ROLE == ROLE_VISC) {
#pragma unroll
          for (int v = 0; v < NV; ++v) q[v * np] = val[v];
        } else if constexpr (UPD) {
          int ci = li, cj = lj, ck = lk;
          if (DIM == 0) ci = c - 1;
          else if (DIM == 1) cj = c - 1;
          else ck = c - 1;
          double out[NV];
          if constexpr (RK4S)
            rk4_store<ROLE == ROLE_RK4_A ? 0 : (ROLE == ROLE_RK4_B ? 1 : 2)>(a.rk, G, ci, cj, ck, val, ru0, racc, out);
          else rk_store_pre(a.rk, G, ci, cj, ck, val, ru0, racc, out);
          if constexpr (DIAG) {
            const int code = diag_fast(out, a.ph.gamma, a.rh[0], a.rh[1], a.rh[2], diag);
            if (code) latch_error(a.err, a.fred_tag, code, G.idx(ci, cj, ck));
          }
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) q[v * np] = val[v];
        }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) fprev[v] = flux[v];
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      lu[v] = nu[v];
      lf[v] = nf[v];
    }
  }
  if constexpr (DIAG) {
    // deterministic warp tree; one partial per warp (the launcher guarantees full warps)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int c = 0; c < 3; ++c) diag[c] = dmax_nan(diag[c], __shfl_down_sync(0xffffffffu, diag[c], off));
#pragma unroll
      for (int c = 3; c < 9; ++c) diag[c] += __shfl_down_sync(0xffffffffu, diag[c], off);
    }
    if (threadIdx.x == 0) {
      const int64_t w = ((int64_t)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) *
                            blockDim.y + threadIdx.y;
#pragma unroll
      for (int c = 0; c < 9; ++c) a.fred[w * 9 + c] = diag[c];
    }
  }
  // peer stores (this line segment held boundary planes) performed before the kernel ends
  if (UPD && DIM == 2 && G.peer_any &&
      ((G.peer[2] && (c0 < G.g || c1 > nd - G.g)) || touches_peer(G, li, lj, G.g)))
    __threadfence_system();
}

// ---------------------------------------------------------------------------
// x sweep with shared-memory staging.  A warp owns 32 consecutive y rows of one
// z plane and marches them along x together; x is the contiguous axis, so the
// plain kernel's per-lane loads and stores touch 32 different rows (one sector
// per lane: partial-sector writes, L1 thrash).  Here the warp moves 4-point
// chunks of all 32 rows with cp.async (lane l copies row 8i + l/4, position
// l%4: 32 contiguous bytes of each of 8 rows per instruction), in a ring of XB
// buffers filled XB-1 chunks ahead, and its increments go out through an 8-cell
// ring in groups aligned to each row's 32-byte sectors (XO below).
// ---------------------------------------------------------------------------
// Chunks of XC = 4 positions per row; staging tiles have row pitch XC + 1
// doubles (odd: conflict-free 64-bit access).  Chunks of 2 with a shared-memory
// window ring measured slower at 512^3 (149-165 vs 141 ms/step).
constexpr int XC = 4;
constexpr int XS_PAD = XC + 1;
// Staging ring depth: with 2 buffers (one chunk = 4 cells ahead) the chunk waits
// are ~23% of the x sweep's warp samples (ncu, 256^3), yet 3 buffers (51 KB of
// dynamic shared memory per block, same 4 blocks/SM) measured slower: 8.5 -> 10.3
// ms at 512^3
constexpr int XB = 2;
// Output ring of XO = 8 cells per row (pitch XO + 1, odd): a flush writes each
// row's increments in groups that start on a 32-byte sector boundary of that row
// (rows of n_x + 2g doubles alternate between two sector phases), so every
// group is one full sector instead of two partial ones -- ncu at 512^3: L2 write
// sectors 335.5M -> see DESIGN.md section 8.
constexpr int XO = 8;
constexpr int XO_PAD = XO + 1;

template <bool EXACT, int PW>
__global__ void __launch_bounds__(SWEEP_THREADS, SWEEP_MIN_BLOCKS_X) sweep_x_staged_kernel(const SweepArgs a) {
  constexpr int WARPS = SWEEP_THREADS / 32;
  __shared__ double xin[WARPS][XB][NV][32 * XS_PAD];
  __shared__ double xout[WARPS][NV][32 * XO_PAD];
  const Geo& G = a.geo;
  const int lane = threadIdx.x, w = threadIdx.y;
  const int j0 = blockIdx.x * 32;  // launch guarantees n_y % 32 == 0
  const int k = blockIdx.y * WARPS + w;
  if (k >= G.n[2]) return;  // warp-uniform
  const int nd = G.n[0];
  const int c0 = blockIdx.z * a.seg;
  if (c0 >= nd) return;
  const int c1 = min(c0 + a.seg, nd);
  const int64_t np = G.npts;
  const int64_t row0 = G.idx(0, j0, k);  // cell x = 0 of row j0
  const int64_t sy = G.sy;
  const int64_t base = row0 + (int64_t)lane * sy;  // this lane's row
  const double gm1 = a.ph.gm1, eps = a.ph.eps;
  const int power = PW ? PW : a.ph.power;
  const int p0 = c0 - 3;  // first position entering the window

  // chunk t holds positions p0 + XC t .. p0 + XC t + XC-1 of all 32 rows; lane l
  // copies row (32/XC) i + l/XC, position l % XC (consecutive lanes: consecutive x)
  constexpr int RPI = 32 / XC;  // rows per copy instruction
  auto issue = [&](int t) {
    const int buf = t % XB;
    const int xo = lane % XC;
    const int p = p0 + XC * t + xo;
    if (p <= c1 + 2) {
#pragma unroll
      for (int i = 0; i < XC; ++i) {
        const int r = RPI * i + lane / XC;
        const double* src = a.u + row0 + (int64_t)r * sy + p;
#pragma unroll
        for (int v = 0; v < NV; ++v) cp_async8(&xin[w][buf][v][r * XS_PAD + xo], src + v * np);
      }
    }
    cp_async_commit();
  };
  auto take = [&](int p, double (&uu)[NV], double (&ff)[NV]) {
    const int q = p - p0;
    const double* s = &xin[w][(q / XC) % XB][0][lane * XS_PAD + (q % XC)];
#pragma unroll
    for (int v = 0; v < NV; ++v) uu[v] = s[v * 32 * XS_PAD];
    double inv, pv[4];
    point_flux<0, EXACT>(uu, gm1, ff, inv, pv);
    if (a.check && p >= 0 && p < nd) {
      const int code = !(uu[0] > 0.0) ? 1 : (!(pv[3] > 0.0) ? 2 : 0);
      if (code) latch_error(a.err, a.tag, code, first_image(G, p, j0 + lane, k));
    }
  };
  // out: cell c0 + i staged in ring slot i % XO; flush t writes, per row, the
  // XC = 4 cells [L, L + 4) with L = 4t + e - (e ? 4 : 0), e = cells before the
  // row's first sector boundary -- after flush t every cell < 4t + e of the row
  // is written, the ring holds cells 4t-3 .. 4t+3 while a flush reads them.
  // inc = old - d, coalesced: 4 lanes fill one sector of one row.
  const int seg_len = c1 - c0;
  auto flush = [&](int t) {
    __syncwarp();
    const int xo = lane % XC;
#pragma unroll
    for (int i = 0; i < XC; ++i) {
      const int r = RPI * i + lane / XC;
      double* row = a.inc + row0 + (int64_t)r * sy + c0;
      const int e = (int)((0u - (unsigned)((uintptr_t)row >> 3)) & 3u);
      const int cell = XC * t + e - (e ? XC : 0) + xo;
      if (cell >= 0 && cell < seg_len) {
        double* dst = row + cell;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double d = xout[w][v][r * XO_PAD + (cell % XO)];
          const double old = a.accumulate ? dst[v * np] : 0.0;
          if constexpr (EXACT) dst[v * np] = xs(old, d);
          else dst[v * np] = old - d;
        }
      }
    }
    __syncwarp();
  };

  // Register window.  Exact: the five positions c-2 .. c+2 (wu/wf[0..4]).  Fast:
  // the differences D0..D2 of positions c-2 .. c+1 and the value at c+1 -- four
  // values per variable instead of five; each position difference is formed once
  // (not four times), and the centre is q2 = q(c+1) - D2: 2 instead of 4 FP64
  // operations per reconstruction pair and 18 fewer registers.
  double wu[EXACT ? 5 : 4][NV], wf[EXACT ? 5 : 4][NV];
  // Entering chunk t (its first position is consumed): wait for it -- it was
  // issued when chunk t-XB+1 was entered, later chunks may still be in flight --
  // then issue chunk t+XB-1 into the buffer chunk t-1 has vacated.  Positions
  // p0 .. p0+3 fill the window first.
#pragma unroll
  for (int t = 0; t < XB - 1; ++t) issue(t);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q % XC == 0) {
      cp_async_wait<XB - 2>();
      __syncwarp();
      issue(q / XC + XB - 1);
    }
    if constexpr (EXACT) {
      take(p0 + q, wu[q + 1], wf[q + 1]);
    } else {
      // wu[3] holds the newest value; wu[q-1] = its difference to the previous one
      double nu_[NV], nf_[NV];
      take(p0 + q, nu_, nf_);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (q > 0) {  // never contracted with the flux products: segment-split invariant
          wu[q - 1][v] = __dsub_rn(nu_[v], wu[3][v]);
          wf[q - 1][v] = __dsub_rn(nf_[v], wf[3][v]);
        }
        wu[3][v] = nu_[v];
        wf[3][v] = nf_[v];
      }
    }
  }

  double lu[NV], lf[NV], fprev[NV];
  for (int c = c0 - 1; c <= c1; ++c) {
    const int p = c + 2;
    if ((p - p0) % XC == 0) {
      cp_async_wait<XB - 2>();
      __syncwarp();
      issue((p - p0) / XC + XB - 1);
    }
    double ru[NV], rf[NV], nu[NV], nf[NV];
    if constexpr (EXACT) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          wu[q][v] = wu[q + 1][v];
          wf[q][v] = wf[q + 1][v];
        }
      take(p, wu[4], wf[4]);
#pragma unroll
      for (int v = 0; v < NV; ++v)
        recon_pair<EXACT>(wu[0][v], wu[1][v], wu[2][v], wu[3][v], wu[4][v], eps, power, nu[v], ru[v]);
#pragma unroll
      for (int v = 1; v < NV; ++v)
        recon_pair<EXACT>(wf[0][v], wf[1][v], wf[2][v], wf[3][v], wf[4][v], eps, power, nf[v], rf[v]);
    } else {
      double qu[NV], qf[NV];
      take(p, qu, qf);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double D3 = __dsub_rn(qu[v], wu[3][v]);
        recon_pair_d(wu[0][v], wu[1][v], wu[2][v], D3, __dsub_rn(wu[3][v], wu[2][v]), eps, power, nu[v],
                     ru[v]);
        wu[0][v] = wu[1][v];
        wu[1][v] = wu[2][v];
        wu[2][v] = D3;
        wu[3][v] = qu[v];
      }
#pragma unroll
      for (int v = 1; v < NV; ++v) {
        const double D3 = __dsub_rn(qf[v], wf[3][v]);
        recon_pair_d(wf[0][v], wf[1][v], wf[2][v], D3, __dsub_rn(wf[3][v], wf[2][v]), eps, power, nf[v],
                     rf[v]);
        wf[0][v] = wf[1][v];
        wf[1][v] = wf[2][v];
        wf[2][v] = D3;
        wf[3][v] = qf[v];
      }
    }
    nf[0] = nu[1];
    rf[0] = ru[1];
    if (c >= c0) {
      double flux[NV];
      roe_flux<0, EXACT>(lu, ru, lf, rf, a.ph, flux);
      if (c > c0) {
        const int i = c - 1 - c0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double d;
          if constexpr (EXACT) d = xm(xs(flux[v], fprev[v]), a.inv_dx);
          else d = (flux[v] - fprev[v]) * a.inv_dx;
          xout[w][v][lane * XO_PAD + (i % XO)] = d;
        }
        if (i % XC == XC - 1) flush(i / XC);
        if (i == seg_len - 1) {
          if (i % XC != XC - 1) flush(i / XC);
          flush(i / XC + 1);
        }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) fprev[v] = flux[v];
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      lu[v] = nu[v];
      lf[v] = nf[v];
    }
  }
  cp_async_wait<0>();
}

template <int DIM, bool EXACT, int ROLE>
static int launch_dim(const hd_plan* p, const SweepArgs& a, int nseg, cudaStream_t s) {
  const Geo& G = p->geo;
  constexpr int BY = SWEEP_THREADS / 32;
  dim3 block(32, BY, 1), grid;
  if (DIM == 0) grid = dim3((G.n[1] + 31) / 32, (G.n[2] + BY - 1) / BY, nseg);
  else if (DIM == 1) grid = dim3((G.n[0] + 31) / 32, (G.n[2] + BY - 1) / BY, nseg);
  else grid = dim3((G.n[0] + 31) / 32, (G.n[1] + BY - 1) / BY, nseg);
  // exact z sweep: the run-time exponent loop measured faster (34.8 vs 39.0 ms at 512^3)
  if (a.ph.power == 2 && !(EXACT && DIM == 2))
    sweep_kernel<DIM, EXACT, ROLE, (EXACT && DIM == 2) ? 0 : 2><<<grid, block, 0, s>>>(a);
  else sweep_kernel<DIM, EXACT, ROLE, 0><<<grid, block, 0, s>>>(a);
  hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

// Resident warps per SM of the fast-mode kernel each axis launches in a step
// (staged x sweep, y VISC, z RK4 stage), queried once per process.
static int sweep_warps_per_sm(int dim) {
  static int cached[3] = {0, 0, 0};
  if (cached[dim] > 0) return cached[dim];
  int blocks = 0;
  cudaError_t e;
  if (dim == 0) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sweep_x_staged_kernel<false, 2>, SWEEP_THREADS, 0);
  else if (dim == 1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sweep_kernel<1, false, ROLE_VISC, 2>, SWEEP_THREADS, 0);
  else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sweep_kernel<2, false, ROLE_RK4_B, 2>, SWEEP_THREADS, 0);
  if (e != cudaSuccess || blocks < 1) {
    (void)cudaGetLastError();
    return SWEEP_THREADS / 32 * SweepCfg<0>::min_blocks;  // not cached: retry next launch
  }
  return cached[dim] = blocks * (SWEEP_THREADS / 32);
}

void sweep_occupancy_warm() {
  for (int d = 0; d < 3; ++d) (void)sweep_warps_per_sm(d);
}

// Segments per line.  A segment of L cells costs about L + SEG_RESTART cells of
// work (the window refill and the extra interface flux at its start), and a
// launch of W waves of resident warps takes about ceil(W) wave times, since the
// warps of a sweep march in step and a partial last wave idles the rest of the
// SMs; pick the count minimising ceil(W) (L + SEG_RESTART) among those giving at
// least two waves (below that the schedulers lack warps to hide latency: a
// single 86 %-full wave of the y sweep measured 7 % slower than 2.9 waves of
// shorter segments).  Measured per axis (tools/gpu/seg_probe.py) it matches the
// round-1 rule at 512^3 and 256^3 and beats it on small blocks: 128^3 2.59 ->
// 2.46 ms per step (x sweep -4 %, y -4 %, z sweep -9 %), -3 % on 256x256x64.
constexpr int SEG_RESTART = 8;
constexpr int SEG_MIN_WAVES = 2;
static int model_segments(int64_t lines, int n, int64_t warp_slots) {
  int best = 1;
  double best_cost = 0.0;
  bool best_full = false;
  const int max_seg = n / 8 > 0 ? n / 8 : 1;
  for (int ns = 1; ns <= max_seg; ++ns) {
    const int len = (n + ns - 1) / ns;
    if (ns > 1 && (n + len - 1) / len != ns) continue;  // same split as a smaller count
    const int64_t warps = (lines + 31) / 32 * ns;
    const int64_t waves = (warps + warp_slots - 1) / warp_slots;
    const bool full = warps >= SEG_MIN_WAVES * warp_slots;
    const double cost = (double)waves * (len + SEG_RESTART);
    if (ns == 1 || (full && !best_full) || (full == best_full && cost < best_cost)) {
      best = ns;
      best_cost = cost;
      best_full = full;
    }
  }
  return best;
}

static SweepArgs make_args(const hd_plan* p, int dim, const double* u, double* inc, int accumulate,
                           int check, int64_t tag, int& nseg) {
  const Geo& G = p->geo;
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.geo = G;
  a.ph = p->phys;
  a.u = u;
  a.inc = inc;
  a.inv_dx = 1.0 / G.h[dim];  // upwind.py:204
  a.accumulate = accumulate;
  a.check = check;
  a.err = (unsigned long long*)(p->ws + p->off[HD_BUF_ERR]);
  a.tag = tag;
  const int64_t lines = (int64_t)G.n[0] * G.n[1] * G.n[2] / G.n[dim];
  if (p->opt[HD_OPT_SWEEP_WAVES] > 0) {
    // the round-1 rule: enough independent lines to fill this many waves of
    // 148 SMs x 256 threads
    const int64_t target = (int64_t)p->sm_count * 256 * p->opt[HD_OPT_SWEEP_WAVES];
    nseg = (int)((target + lines - 1) / lines);
    if (nseg < 1) nseg = 1;
    if (nseg > G.n[dim] / 8) nseg = G.n[dim] / 8 > 0 ? G.n[dim] / 8 : 1;
  } else {
    nseg = model_segments(lines, G.n[dim], (int64_t)p->sm_count * sweep_warps_per_sm(dim));
  }
  // HD_OPT_SEGMENTS (tests: results must not depend on the split)
  if (p->opt[HD_OPT_SEGMENTS] >= 1 && p->opt[HD_OPT_SEGMENTS] <= G.n[dim]) nseg = (int)p->opt[HD_OPT_SEGMENTS];
  a.seg = (G.n[dim] + nseg - 1) / nseg;
  nseg = (G.n[dim] + a.seg - 1) / a.seg;
  return a;
}

int launch_sweep(const hd_plan* p, int dim, const double* u, double* inc, int accumulate, int check,
                 int64_t tag, cudaStream_t s) {
  if (dim < 0 || dim > 2) return HD_E_ARG;
  int nseg;
  SweepArgs a = make_args(p, dim, u, inc, accumulate, check, tag, nseg);
  const bool exact = p->mode == HD_MODE_EXACT;
  if (dim == 0 && p->geo.n[1] % 32 == 0 && p->opt[HD_OPT_X_STAGED]) {
    constexpr int BY = SWEEP_THREADS / 32;
    const Geo& G = p->geo;
    dim3 block(32, BY, 1), grid(G.n[1] / 32, (G.n[2] + BY - 1) / BY, nseg);
    auto kern = exact ? (a.ph.power == 2 ? sweep_x_staged_kernel<true, 2> : sweep_x_staged_kernel<true, 0>)
                      : (a.ph.power == 2 ? sweep_x_staged_kernel<false, 2> : sweep_x_staged_kernel<false, 0>);
    kern<<<grid, block, 0, s>>>(a);
    hd::count_launches(1);
    return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
  }
  switch (dim * 2 + (exact ? 1 : 0)) {
    case 0: return launch_dim<0, false, ROLE_PLAIN>(p, a, nseg, s);
    case 1: return launch_dim<0, true, ROLE_PLAIN>(p, a, nseg, s);
    case 2: return launch_dim<1, false, ROLE_PLAIN>(p, a, nseg, s);
    case 3: return launch_dim<1, true, ROLE_PLAIN>(p, a, nseg, s);
    case 4: return launch_dim<2, false, ROLE_PLAIN>(p, a, nseg, s);
    default: return launch_dim<2, true, ROLE_PLAIN>(p, a, nseg, s);
  }
}

int launch_sweep_visc(const hd_plan* p, const double* u, double* inc, const double* vflux,
                      int64_t tag, cudaStream_t s) {
  int nseg;
  SweepArgs a = make_args(p, 1, u, inc, 1, 0, tag, nseg);
  a.vflux = vflux;
  if (p->mode == HD_MODE_EXACT) return HD_E_UNSUPPORTED;  // exact mode runs the unfused stage
  return launch_dim<1, false, ROLE_VISC>(p, a, nseg, s);
}

int launch_sweep_update(const hd_plan* p, const double* u_stage, double* inc, const double* vflux,
                        int scheme, int stage, double* u, const double* dt_dev,
                        int64_t tag, cudaStream_t s, double* red_out, int64_t red_tag, int* fused) {
  int nseg;
  SweepArgs a = make_args(p, 2, u_stage, inc, 1, 0, tag, nseg);
  a.vflux = vflux;
  a.rk = make_rk(p, scheme, stage, u, dt_dev);
  if (p->mode == HD_MODE_EXACT) return HD_E_UNSUPPORTED;  // exact mode runs the unfused stage
  // the last stage can fold the diagnostics of the new state in (hd_arm_reduce):
  // full warps only (n_x % 32, n_y % 2), and room for one partial per warp
  const Geo& G = p->geo;
  const int64_t warps = (int64_t)(G.n[0] / 32) * G.n[1] * nseg;
  if (fused) *fused = 0;
  const bool rk4 = scheme == HD_SCHEME_RK4;
  if (red_out && a.rk.to_u && G.n[0] % 32 == 0 && G.n[1] % 2 == 0 &&
      warps <= fused_red_capacity(p->geom)) {
    a.fred = (double*)(p->ws + p->off[HD_BUF_FRED]);
    a.fred_tag = red_tag;
    for (int d = 0; d < 3; ++d) a.rh[d] = 1.0 / G.h[d];
    int rc = rk4 ? launch_dim<2, false, ROLE_RK4_C_DIAG>(p, a, nseg, s)
                 : launch_dim<2, false, ROLE_UPDATE_DIAG>(p, a, nseg, s);
    if (!rc) rc = launch_reduce_finish(a.fred, (int)warps, red_out, s);
    if (!rc && fused) *fused = 1;
    return rc;
  }
  if (rk4) {
    if (stage == 0) return launch_dim<2, false, ROLE_RK4_A>(p, a, nseg, s);
    if (stage < 3) return launch_dim<2, false, ROLE_RK4_B>(p, a, nseg, s);
    return launch_dim<2, false, ROLE_RK4_C>(p, a, nseg, s);
  }
  return launch_dim<2, false, ROLE_UPDATE>(p, a, nseg, s);
}

// ---------------------------------------------------------------------------
// kernels.py:68-204 hyper_sweep with the reference's own argument list: a slab of
// lines [a_lo, a_hi) x [0, nb) from base0 with strides (sd, sa, sb), the flux
// components taken from the caller's array f (upwind.py:116-127 output), exact
// IEEE arithmetic in the reference order.  One thread per line, one interface at
// a time -- the compatibility entry for a caller that keeps the reference's
// run_slabs loop (upwind.py:30-45, 185-212); the fused sweeps above are the
// fast path.
// ---------------------------------------------------------------------------
struct LineArgs {
  const double* u;
  const double* f;
  double* inc;
  int64_t npts, base0, sd, sa, sb, nd, nb, a_lo, a_hi;
  double inv_dx, eps;
  int power;
  Phys ph;
};

template <int DIM>
__global__ void hyper_sweep_lines_kernel(const LineArgs a) {
  const int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nlines = (a.a_hi - a.a_lo) * a.nb;
  if (line >= nlines) return;
  const int64_t ia = a.a_lo + line / a.nb, ib = line % a.nb;
  const int64_t base = a.base0 + ia * a.sa + ib * a.sb;
  double fprev[NV];
  for (int64_t m = -1; m < a.nd; ++m) {
    const int64_t c = base + m * a.sd;
    double uL[NV], uR[NV], fL[NV], fR[NV], flux[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double* qu = a.u + v * a.npts + c;
      const double* qf = a.f + v * a.npts + c;
      const int64_t s = a.sd;
      uL[v] = recon5_exact(qu[-2 * s], qu[-s], qu[0], qu[s], qu[2 * s], a.eps, a.power);
      uR[v] = recon5_exact(qu[3 * s], qu[2 * s], qu[s], qu[0], qu[-s], a.eps, a.power);
      fL[v] = recon5_exact(qf[-2 * s], qf[-s], qf[0], qf[s], qf[2 * s], a.eps, a.power);
      fR[v] = recon5_exact(qf[3 * s], qf[2 * s], qf[s], qf[0], qf[-s], a.eps, a.power);
    }
    roe_flux<DIM, true>(uL, uR, fL, fR, a.ph, flux);
    if (m >= 0) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double* q = a.inc + v * a.npts + c;
        *q = xs(*q, xm(xs(flux[v], fprev[v]), a.inv_dx));
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) fprev[v] = flux[v];
  }
}

}  // namespace hd

extern "C" int hd_hyper_sweep_lines(const double* u, const double* f, double* inc, int64_t npts,
                                    int64_t base0, int64_t sd, int64_t sa, int64_t sb, int64_t nd,
                                    int64_t nb, int64_t a_lo, int64_t a_hi, int dim, double inv_dx,
                                    double gamma, double eps, int power, double delta, void* stream) {
  using namespace hd;
  if (!u || !f || !inc || dim < 0 || dim > 2 || npts < 1 || nd < 0 || nb < 0 || a_hi < a_lo || power < 1)
    return HD_E_ARG;
  const int64_t nlines = (a_hi - a_lo) * nb;
  if (nlines == 0 || nd == 0) return HD_OK;
  LineArgs a;
  a.u = u;
  a.f = f;
  a.inc = inc;
  a.npts = npts;
  a.base0 = base0;
  a.sd = sd;
  a.sa = sa;
  a.sb = sb;
  a.nd = nd;
  a.nb = nb;
  a.a_lo = a_lo;
  a.a_hi = a_hi;
  a.inv_dx = inv_dx;
  a.eps = eps;
  a.power = power;
  a.ph.gamma = gamma;
  a.ph.gm1 = gamma - 1.0;  // kernels.py:84
  a.ph.delta = delta;
  a.ph.eps = eps;
  a.ph.power = power;
  a.ph.prandtl = 0.0;
  a.ph.mu = 0.0;
  const int threads = 128;
  const unsigned blocks = (unsigned)((nlines + threads - 1) / threads);
  cudaStream_t s = (cudaStream_t)stream;
  if (dim == 0) hyper_sweep_lines_kernel<0><<<blocks, threads, 0, s>>>(a);
  else if (dim == 1) hyper_sweep_lines_kernel<1><<<blocks, threads, 0, s>>>(a);
  else hyper_sweep_lines_kernel<2><<<blocks, threads, 0, s>>>(a);
  count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

