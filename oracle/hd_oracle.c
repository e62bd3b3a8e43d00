/*
 * hd_oracle.c -- CPU restatement of the hitdns reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2211_16718_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product never links or calls it.
 *
 * Every routine restates one reference function operation-for-operation, in
 * the same association order, so that (compiled with -ffp-contract=off, no
 * -ffast-math) it reproduces the numba/numpy reference bit-for-bit:
 *
 *   or_recon5          pkg/src/hitdns/kernels.py:25-57   (_recon5)
 *   or_entropy_fixed   pkg/src/hitdns/kernels.py:60-65   (_entropy_fixed)
 *   or_hyper_sweep     pkg/src/hitdns/kernels.py:68-204  (hyper_sweep)
 *   or_central_diff4   pkg/src/hitdns/kernels.py:207-227 (central_diff4)
 *   or_fill_ghosts     pkg/src/hitdns/grid.py:211-251    (_wrap_axis, fill_ghosts_*)
 *   or_decode          pkg/src/hitdns/physics.py:240-255 (decode_primitives)
 *   or_flux_components pkg/src/hitdns/upwind.py:116-127  (_flux_components)
 *   or_hyperbolic_rhs  pkg/src/hitdns/upwind.py:163-213  (hyperbolic_rhs)
 *   or_parabolic_rhs   pkg/src/hitdns/viscous.py:54-121  (parabolic_rhs)
 *   or_rhs             pkg/src/hitdns/timeint.py:141-158 (make_rhs.rhs)
 *   or_rk4_step        pkg/src/hitdns/timeint.py:181-193 (rk4_step)
 *   or_rk3_step        pkg/src/hitdns/timeint.py:168-178 (rk3_tvd_step)
 *   or_max_signal      pkg/src/hitdns/timeint.py:110-131 (max_signal via cons_to_prim)
 *   or_enstrophy       the north star's enstrophy (the reference has none) from the
 *                      reference's own operators: velocities as physics.py:249-252
 *                      (decode_primitives), derivatives as viscous.py:23-51
 *                      (central_derivative_4 -> kernels.py:221-226)
 *
 * Parity is pinned by tests/test_oracle_golden.py against fixtures produced by
 * running the reference itself (tests/golden/make_golden.py).
 *
 * Threading: OpenMP over the outermost loop only; every output element is
 * computed by exactly one thread with a fixed operation order, so results are
 * bitwise independent of the thread count (as run_slabs is, upwind.py:30-45).
 *
 * Error convention: functions that decode states return 0 on success,
 * 1 for a nonpositive density, 2 for a nonpositive pressure (the two
 * InvalidStateError cases of physics.py:47-55), with the first offending flat
 * point index in *where.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NV 5

/* WENO literals, weno.py:28-33 (Python doubles) */
static const double C_13_12 = 13.0 / 12.0;
static const double C_1_3 = 1.0 / 3.0;
static const double C_7_6 = 7.0 / 6.0;
static const double C_11_6 = 11.0 / 6.0;
static const double C_1_6 = 1.0 / 6.0;
static const double C_5_6 = 5.0 / 6.0;

/* kernels.py:25-57 */
static inline double or_recon5(double f0, double f1, double f2, double f3, double f4,
                               double eps, int power) {
  double t1 = (f0 - 2.0 * f1) + f2;
  double s1 = (f0 - 4.0 * f1) + 3.0 * f2;
  double b1 = C_13_12 * (t1 * t1) + 0.25 * (s1 * s1);
  double t2 = (f1 - 2.0 * f2) + f3;
  double s2 = f1 - f3;
  double b2 = C_13_12 * (t2 * t2) + 0.25 * (s2 * s2);
  double t3 = (f2 - 2.0 * f3) + f4;
  double s3 = (3.0 * f2 - 4.0 * f3) + f4;
  double b3 = C_13_12 * (t3 * t3) + 0.25 * (s3 * s3);
  double d1 = eps + b1, d2 = eps + b2, d3 = eps + b3;
  double e1 = d1, e2 = d2, e3 = d3;
  for (int q = 0; q < power - 1; ++q) {
    e1 = e1 * d1;
    e2 = e2 * d2;
    e3 = e3 * d3;
  }
  double a1 = 0.1 / e1, a2 = 0.6 / e2, a3 = 0.3 / e3;
  double asum = (a1 + a2) + a3;
  double w1 = a1 / asum, w2 = a2 / asum, w3 = a3 / asum;
  double c1 = (C_1_3 * f0 - C_7_6 * f1) + C_11_6 * f2;
  double c2 = ((-C_1_6) * f1 + C_5_6 * f2) + C_1_3 * f3;
  double c3 = (C_1_3 * f2 + C_5_6 * f3) - C_1_6 * f4;
  return (w1 * c1 + w2 * c2) + w3 * c3;
}

/* kernels.py:60-65 */
static inline double or_entropy_fixed(double lam, double delta) {
  double mag = fabs(lam);
  if (delta > 0.0 && mag < delta) return (lam * lam + delta * delta) / (2.0 * delta);
  return mag;
}

/* kernels.py:68-204: one slab [a_lo, a_hi) of lines along the stride-sd axis. */
void or_hyper_sweep(const double* u, const double* f, double* inc, int64_t npts,
                    int64_t base0, int64_t sd, int64_t sa, int64_t sb, int64_t nd,
                    int64_t nb, int64_t a_lo, int64_t a_hi, int dim, double inv_dx,
                    double gamma, double eps, int power, double delta) {
  const double gm1 = gamma - 1.0;
  const int mn = 1 + dim, mt1 = 1 + (dim + 1) % 3, mt2 = 1 + (dim + 2) % 3;
  const int64_t o0 = 0, o1 = npts, o2 = 2 * npts, o3 = 3 * npts, o4 = 4 * npts;
#pragma omp parallel for schedule(static)
  for (int64_t ia = a_lo; ia < a_hi; ++ia) {
    double uL[NV], uR[NV], flux[NV], fprev[NV] = {0, 0, 0, 0, 0};
    for (int64_t ib = 0; ib < nb; ++ib) {
      const int64_t base = base0 + ia * sa + ib * sb;
      for (int64_t m = -1; m < nd; ++m) {
        const int64_t c = base + m * sd;
        const int64_t i0 = c - 2 * sd, i1 = c - sd, i2 = c, i3 = c + sd, i4 = c + 2 * sd,
                      i5 = c + 3 * sd;
        for (int v = 0; v < NV; ++v) {
          const int64_t o = v * npts;
          uL[v] = or_recon5(u[o + i0], u[o + i1], u[o + i2], u[o + i3], u[o + i4], eps, power);
          uR[v] = or_recon5(u[o + i5], u[o + i4], u[o + i3], u[o + i2], u[o + i1], eps, power);
        }
        double fl[NV], fr[NV];
        const int64_t oo[NV] = {o0, o1, o2, o3, o4};
        for (int v = 0; v < NV; ++v) {
          const int64_t o = oo[v];
          fl[v] = or_recon5(f[o + i0], f[o + i1], f[o + i2], f[o + i3], f[o + i4], eps, power);
        }
        for (int v = 0; v < NV; ++v) {
          const int64_t o = oo[v];
          fr[v] = or_recon5(f[o + i5], f[o + i4], f[o + i3], f[o + i2], f[o + i1], eps, power);
        }
        /* decode the reconstructed interface states (kernels.py:126-137) */
        const double rl = uL[0];
        const double il = 1.0 / rl;
        const double vxl = uL[1] * il, vyl = uL[2] * il, vzl = uL[3] * il;
        const double pl = gm1 * (uL[4] - (0.5 * rl) * ((vxl * vxl + vyl * vyl) + vzl * vzl));
        const double rr = uR[0];
        const double ir = 1.0 / rr;
        const double vxr = uR[1] * ir, vyr = uR[2] * ir, vzr = uR[3] * ir;
        const double pr = gm1 * (uR[4] - (0.5 * rr) * ((vxr * vxr + vyr * vyr) + vzr * vzr));
        /* density-weighted average (kernels.py:140-151) */
        const double sl = sqrt(rl), sr = sqrt(rr);
        const double isw = 1.0 / (sl + sr);
        const double ua = (sl * vxl + sr * vxr) * isw;
        const double va = (sl * vyl + sr * vyr) * isw;
        const double wa = (sl * vzl + sr * vzr) * isw;
        const double Hl = (uL[4] + pl) * il;
        const double Hr = (uR[4] + pr) * ir;
        const double Ha = (sl * Hl + sr * Hr) * isw;
        const double q2 = (ua * ua + va * va) + wa * wa;
        const double a2 = gm1 * (Ha - 0.5 * q2);
        const double aa = sqrt(a2);
        double vn, vt1, vt2;
        if (dim == 0) { vn = ua; vt1 = va; vt2 = wa; }
        else if (dim == 1) { vn = va; vt1 = wa; vt2 = ua; }
        else { vn = wa; vt1 = ua; vt2 = va; }
        /* characteristic strengths (kernels.py:160-173) */
        const double dr = uR[0] - uL[0];
        const double dmn = uR[mn] - uL[mn];
        const double dt1 = uR[mt1] - uL[mt1];
        const double dt2 = uR[mt2] - uL[mt2];
        const double dE = uR[4] - uL[4];
        const double b1 = gm1 / a2;
        const double b2 = (0.5 * b1) * q2;
        const double ia_ = 1.0 / aa;
        const double s1 = 0.5 * (((((b2 + vn * ia_) * dr - (b1 * vn + ia_) * dmn) - (b1 * vt1) * dt1) -
                                  (b1 * vt2) * dt2) + b1 * dE);
        const double s2 = (((((1.0 - b2) * dr + (b1 * vn) * dmn) + (b1 * vt1) * dt1) + (b1 * vt2) * dt2) -
                           b1 * dE);
        const double s3 = (-vt1) * dr + dt1;
        const double s4 = (-vt2) * dr + dt2;
        const double s5 = 0.5 * (((((b2 - vn * ia_) * dr - (b1 * vn - ia_) * dmn) - (b1 * vt1) * dt1) -
                                  (b1 * vt2) * dt2) + b1 * dE);
        const double k1 = or_entropy_fixed(vn - aa, delta) * s1;
        const double k2 = or_entropy_fixed(vn, delta) * s2;
        const double k3 = or_entropy_fixed(vn, delta) * s3;
        const double k4 = or_entropy_fixed(vn, delta) * s4;
        const double k5 = or_entropy_fixed(vn + aa, delta) * s5;
        /* dissipation X|L|Xinv du (kernels.py:182-186) */
        const double diss_r = (k1 + k2) + k5;
        const double diss_n = (k1 * (vn - aa) + k2 * vn) + k5 * (vn + aa);
        const double diss_1 = ((k1 * vt1 + k2 * vt1) + k3) + k5 * vt1;
        const double diss_2 = ((k1 * vt2 + k2 * vt2) + k4) + k5 * vt2;
        const double diss_E = (((k1 * (Ha - vn * aa) + k2 * (0.5 * q2)) + k3 * vt1) + k4 * vt2) +
                              k5 * (Ha + vn * aa);
        flux[0] = 0.5 * (fl[0] + fr[0]) - 0.5 * diss_r;
        flux[1] = 0.5 * (fl[1] + fr[1]);
        flux[2] = 0.5 * (fl[2] + fr[2]);
        flux[3] = 0.5 * (fl[3] + fr[3]);
        flux[4] = 0.5 * (fl[4] + fr[4]) - 0.5 * diss_E;
        flux[mn] -= 0.5 * diss_n;
        flux[mt1] -= 0.5 * diss_1;
        flux[mt2] -= 0.5 * diss_2;
        if (m >= 0) {
          for (int v = 0; v < NV; ++v) inc[oo[v] + c] -= (flux[v] - fprev[v]) * inv_dx;
        }
        for (int v = 0; v < NV; ++v) fprev[v] = flux[v];
      }
    }
  }
}

/* kernels.py:207-227.  src is (gz, gy, gx) with ghost width g; dst is
 * (nz+2og, ny+2og, nx+2og); writes dst interior for k in [k_lo, k_hi). */
void or_central_diff4(const double* src, double* dst, int di, int dj, int dk, int g, int og,
                      int nx, int ny, int nz, int k_lo, int k_hi, double coef) {
  const int64_t sgx = nx + 2 * g, sgy = ny + 2 * g;
  const int64_t dgx = nx + 2 * og, dgy = ny + 2 * og;
#pragma omp parallel for schedule(static)
  for (int k = k_lo; k < k_hi; ++k) {
    const int zc = g + k;
    for (int j = 0; j < ny; ++j) {
      const int yc = g + j;
      for (int i = 0; i < nx; ++i) {
        const int xc = g + i;
#define S(z, y, x) src[((int64_t)(z) * sgy + (y)) * sgx + (x)]
        const double val = (((-S(zc + 2 * dk, yc + 2 * dj, xc + 2 * di)) +
                             8.0 * S(zc + dk, yc + dj, xc + di)) -
                            8.0 * S(zc - dk, yc - dj, xc - di)) +
                           S(zc - 2 * dk, yc - 2 * dj, xc - 2 * di);
#undef S
        dst[((int64_t)(og + k) * dgy + (og + j)) * dgx + (og + i)] = val * coef;
      }
    }
  }
}

/* grid.py:211-251: periodic wrap of one (gz,gy,gx) array; x, then y, then z,
 * each copying the full extent of the other axes. */
void or_fill_ghosts_array(double* a, int nx, int ny, int nz, int g) {
  const int64_t gx = nx + 2 * g, gy = ny + 2 * g, gz = nz + 2 * g;
  for (int64_t k = 0; k < gz; ++k)
    for (int64_t j = 0; j < gy; ++j) {
      double* row = a + (k * gy + j) * gx;
      for (int q = 0; q < g; ++q) {
        row[q] = row[nx + q];
        row[nx + g + q] = row[g + q];
      }
    }
  for (int64_t k = 0; k < gz; ++k) {
    double* pl = a + k * gy * gx;
    for (int q = 0; q < g; ++q) {
      memcpy(pl + (int64_t)q * gx, pl + (int64_t)(ny + q) * gx, gx * sizeof(double));
      memcpy(pl + (int64_t)(ny + g + q) * gx, pl + (int64_t)(g + q) * gx, gx * sizeof(double));
    }
  }
  const int64_t plane = gx * gy;
  for (int q = 0; q < g; ++q) {
    memcpy(a + q * plane, a + (int64_t)(nz + q) * plane, plane * sizeof(double));
    memcpy(a + (int64_t)(nz + g + q) * plane, a + (int64_t)(g + q) * plane, plane * sizeof(double));
  }
}

void or_fill_ghosts(double* u, int nx, int ny, int nz, int g) {
  const int64_t npts = (int64_t)(nx + 2 * g) * (ny + 2 * g) * (nz + 2 * g);
  for (int v = 0; v < NV; ++v) or_fill_ghosts_array(u + v * npts, nx, ny, nz, g);
}

/* physics.py:240-255 over the full ghosted extent.  prim = rho,u,v,w,p. */
int or_decode(const double* U, double* prim, int64_t npts, double gamma, int64_t* where) {
  const double gm1 = gamma - 1.0;
  for (int64_t p = 0; p < npts; ++p)
    if (!(U[p] > 0.0)) { *where = p; return 1; }
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npts; ++p) {
    const double rho = U[p];
    const double inv = 1.0 / rho;
    const double u = U[npts + p] * inv, v = U[2 * npts + p] * inv, w = U[3 * npts + p] * inv;
    prim[p] = rho;
    prim[npts + p] = u;
    prim[2 * npts + p] = v;
    prim[3 * npts + p] = w;
    prim[4 * npts + p] = gm1 * (U[4 * npts + p] - (0.5 * rho) * ((u * u + v * v) + w * w));
  }
  for (int64_t p = 0; p < npts; ++p)
    if (!(prim[4 * npts + p] > 0.0)) { *where = p; return 2; }
  return 0;
}

/* upwind.py:116-127 */
void or_flux_components(const double* U, const double* prim, double* F, int64_t npts, int dim) {
  const double* vd = prim + (1 + dim) * npts;
  const double* p = prim + 4 * npts;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < npts; ++q) {
    F[q] = U[(1 + dim) * npts + q];
    F[npts + q] = U[npts + q] * vd[q];
    F[2 * npts + q] = U[2 * npts + q] * vd[q];
    F[3 * npts + q] = U[3 * npts + q] * vd[q];
    F[(1 + dim) * npts + q] += p[q];
    F[4 * npts + q] = (U[4 * npts + q] + p[q]) * vd[q];
  }
}

typedef struct {
  int n[3];
  double length[3];
  int g;
  double gamma, prandtl, mu_eff, eps, delta;
  int power;
} or_geom;

static double or_spacing(const or_geom* G, int d) { return G->length[d] / (double)G->n[d]; }

/* upwind.py:163-213.  U ghosts must be filled; accumulates into inc.
 * prim/F are caller scratch of 5*npts each. */
int or_hyperbolic_rhs(const or_geom* G, const double* U, double* inc, double* prim, double* F,
                      int64_t* where) {
  const int nx = G->n[0], ny = G->n[1], nz = G->n[2], g = G->g;
  const int64_t gx = nx + 2 * g, gy = ny + 2 * g, gz = nz + 2 * g;
  const int64_t npts = gx * gy * gz;
  int rc = or_decode(U, prim, npts, G->gamma, where);
  if (rc) return rc;
  const int64_t sx = 1, sy = gx, sz = gx * gy;
  const int64_t base0 = g * sz + g * sy + g * sx;
  const int64_t geo[3][6] = {{sx, sz, sy, nx, nz, ny}, {sy, sz, sx, ny, nz, nx}, {sz, sy, sx, nz, ny, nx}};
  for (int dim = 0; dim < 3; ++dim) {
    or_flux_components(U, prim, F, npts, dim);
    const double inv_dx = 1.0 / or_spacing(G, dim);
    or_hyper_sweep(U, F, inc, npts, base0, geo[dim][0], geo[dim][1], geo[dim][2], geo[dim][3],
                   geo[dim][5], 0, geo[dim][4], dim, inv_dx, G->gamma, G->eps, G->power, G->delta);
  }
  return 0;
}

/* viscous.py:54-121.  Accumulates into inc.  work: scratch of >= 26*npts. */
int or_parabolic_rhs(const or_geom* G, const double* U, double* inc, double* work, int64_t* where) {
  const double mu = G->mu_eff;
  if (mu == 0.0) return 0;
  const int nx = G->n[0], ny = G->n[1], nz = G->n[2], g = G->g;
  const int64_t gx = nx + 2 * g, gy = ny + 2 * g, gz = nz + 2 * g;
  const int64_t npts = gx * gy * gz;
  const int64_t nint = (int64_t)nx * ny * nz;
  const double gamma = G->gamma;
  double* prim = work;                 /* 5*npts */
  double* T = work + 5 * npts;         /* npts */
  double* grad = T + npts;             /* 12 interior arrays: grad[i][j] (9), gradT[j] (3) */
  double* scratch = grad + 12 * nint;  /* 4*npts */
  double* dtmp = scratch + 4 * npts;   /* nint */
  int rc = or_decode(U, prim, npts, gamma, where);
  if (rc) return rc;
  for (int64_t q = 0; q < npts; ++q) T[q] = (gamma * prim[4 * npts + q]) / prim[q];
  const int off[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      or_central_diff4(prim + (1 + i) * npts, grad + (3 * i + j) * nint, off[j][0], off[j][1],
                       off[j][2], g, 0, nx, ny, nz, 0, nz, 1.0 / (12.0 * or_spacing(G, j)));
  for (int j = 0; j < 3; ++j)
    or_central_diff4(T, grad + (9 + j) * nint, off[j][0], off[j][1], off[j][2], g, 0, nx, ny, nz,
                     0, nz, 1.0 / (12.0 * or_spacing(G, j)));
  const double q_coef = (-mu) / ((gamma - 1.0) * G->prandtl);
  const double two_thirds = 2.0 / 3.0;
  memset(scratch, 0, 4 * npts * sizeof(double));
#define GR(i, j) grad[(3 * (i) + (j)) * nint + q]
  for (int d = 0; d < 3; ++d) {
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nint; ++q) {
      const int64_t i = q % nx, j = (q / nx) % ny, k = q / ((int64_t)nx * ny);
      const int64_t pg = ((k + g) * gy + (j + g)) * gx + (i + g);
      const double div = (GR(0, 0) + GR(1, 1)) + GR(2, 2);
      const double ttd = two_thirds * div;
      double tau[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          tau[a][b] = (a == b) ? mu * (2.0 * GR(a, a) - ttd)
                               : (a < b ? mu * (GR(a, b) + GR(b, a)) : mu * (GR(b, a) + GR(a, b)));
      const double qd = q_coef * grad[(9 + d) * nint + q];
      const double uu = prim[npts + pg], vv = prim[2 * npts + pg], ww = prim[3 * npts + pg];
      const double wk = ((uu * tau[0][d] + vv * tau[1][d]) + ww * tau[2][d]) - qd;
      scratch[0 * npts + pg] = tau[0][d];
      scratch[1 * npts + pg] = tau[1][d];
      scratch[2 * npts + pg] = tau[2][d];
      scratch[3 * npts + pg] = wk;
    }
    for (int r = 0; r < 4; ++r) or_fill_ghosts_array(scratch + r * npts, nx, ny, nz, g);
    for (int r = 0; r < 4; ++r) {
      or_central_diff4(scratch + r * npts, dtmp, off[d][0], off[d][1], off[d][2], g, 0, nx, ny,
                       nz, 0, nz, 1.0 / (12.0 * or_spacing(G, d)));
      double* dst = inc + (1 + r) * npts;
#pragma omp parallel for schedule(static)
      for (int64_t q = 0; q < nint; ++q) {
        const int64_t i = q % nx, j = (q / nx) % ny, k = q / ((int64_t)nx * ny);
        const int64_t pg = ((k + g) * gy + (j + g)) * gx + (i + g);
        dst[pg] += dtmp[q];
      }
    }
  }
#undef GR
  return 0;
}

static int64_t or_npts(const or_geom* G) {
  return (int64_t)(G->n[0] + 2 * G->g) * (G->n[1] + 2 * G->g) * (G->n[2] + 2 * G->g);
}

/* Scratch size (doubles) for or_rhs / steppers. */
int64_t or_work_size(const or_geom* G) {
  const int64_t npts = or_npts(G);
  const int64_t nint = (int64_t)G->n[0] * G->n[1] * G->n[2];
  return 5 * npts + 5 * npts + (5 * npts + npts + 12 * nint + 4 * npts + nint);
}

/* timeint.py:152-156: sync ghosts of U in place; inc = hyperbolic + parabolic. */
int or_rhs(const or_geom* G, double* U, double* inc, double* work, int64_t* where) {
  const int64_t npts = or_npts(G);
  or_fill_ghosts(U, G->n[0], G->n[1], G->n[2], G->g);
  memset(inc, 0, 5 * npts * sizeof(double));
  int rc = or_hyperbolic_rhs(G, U, inc, work, work + 5 * npts, where);
  if (rc) return rc;
  return or_parabolic_rhs(G, U, inc, work + 10 * npts, where);
}

/* timeint.py:181-193.  U updated in place.  Returns 10*stage + rc on failure. */
int or_rk4_step(const or_geom* G, double* U, double dt, double* work, int64_t* where) {
  const int64_t N = 5 * or_npts(G);
  double* k = (double*)malloc(4 * N * sizeof(double));
  double* us = (double*)malloc(N * sizeof(double));
  if (!k || !us) { free(k); free(us); return -1; }
  const double half = 0.5 * dt;
  int rc = 0;
  for (int s = 0; s < 4 && !rc; ++s) {
    double* ks = k + s * N;
    if (s == 0) {
      rc = or_rhs(G, U, ks, work, where);
    } else {
      const double c = (s == 3) ? dt : half;
      const double* kp = k + (s - 1) * N;
#pragma omp parallel for schedule(static)
      for (int64_t q = 0; q < N; ++q) us[q] = U[q] + c * kp[q];
      rc = or_rhs(G, us, ks, work, where);
    }
    if (rc) rc = 10 * s + rc;
  }
  if (!rc) {
    const double c6 = dt / 6.0;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < N; ++q)
      U[q] = U[q] + c6 * (((k[q] + 2.0 * k[N + q]) + 2.0 * k[2 * N + q]) + k[3 * N + q]);
  }
  free(k);
  free(us);
  return rc;
}

/* timeint.py:168-178 */
int or_rk3_step(const or_geom* G, double* U, double dt, double* work, int64_t* where) {
  const int64_t N = 5 * or_npts(G);
  double* r = (double*)malloc(N * sizeof(double));
  double* u1 = (double*)malloc(N * sizeof(double));
  double* u2 = (double*)malloc(N * sizeof(double));
  if (!r || !u1 || !u2) { free(r); free(u1); free(u2); return -1; }
  int rc = or_rhs(G, U, r, work, where);
  if (!rc) {
    for (int64_t q = 0; q < N; ++q) u1[q] = U[q] + dt * r[q];
    rc = or_rhs(G, u1, r, work, where);
    if (rc) rc += 10;
  }
  if (!rc) {
    for (int64_t q = 0; q < N; ++q) u2[q] = 0.75 * U[q] + 0.25 * (u1[q] + dt * r[q]);
    rc = or_rhs(G, u2, r, work, where);
    if (rc) rc += 20;
  }
  if (!rc) {
    const double c13 = 1.0 / 3.0, c23 = 2.0 / 3.0;
    for (int64_t q = 0; q < N; ++q) U[q] = c13 * U[q] + c23 * (u2[q] + dt * r[q]);
  }
  free(r); free(u1); free(u2);
  return rc;
}

/* timeint.py:110-131 + physics.py:58-71,87-89: interior CFL signal.
 * mode 0 = "max", 1 = "sum".  out[0] = signal, out[1] = max wavespeed. */
int or_max_signal(const or_geom* G, const double* U, int mode, double* out, int64_t* where) {
  const int nx = G->n[0], ny = G->n[1], nz = G->n[2], g = G->g;
  const int64_t gx = nx + 2 * g, gy = ny + 2 * g;
  const int64_t npts = or_npts(G);
  const double gamma = G->gamma;
  const double h[3] = {or_spacing(G, 0), or_spacing(G, 1), or_spacing(G, 2)};
  double sig = -INFINITY, wav = -INFINITY;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t p = ((int64_t)(k + g) * gy + (j + g)) * gx + (i + g);
        if (!(U[p] > 0.0)) { *where = p; return 1; }
      }
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t p = ((int64_t)(k + g) * gy + (j + g)) * gx + (i + g);
        const double rho = U[p];
        const double v0 = U[npts + p] / rho, v1 = U[2 * npts + p] / rho, v2 = U[3 * npts + p] / rho;
        const double kin = (0.5 * rho) * ((v0 * v0 + v1 * v1) + v2 * v2);
        const double pr = (gamma - 1.0) * (U[4 * npts + p] - kin);
        if (!(pr > 0.0)) { *where = p; return 2; }
        const double a = sqrt((gamma * pr) / rho);
        const double s0 = (fabs(v0) + a) / h[0], s1 = (fabs(v1) + a) / h[1], s2 = (fabs(v2) + a) / h[2];
        const double s = mode == 1 ? (s0 + s1) + s2 : fmax(fmax(s0, s1), s2);
        if (s > sig || isnan(s)) sig = s;
        const double vm = fmax(fmax(fabs(v0), fabs(v1)), fabs(v2)) + a;
        if (vm > wav || isnan(vm)) wav = vm;
      }
  out[0] = sig;
  out[1] = wav;
  return 0;
}

/* Sum over the interior of 0.5 |curl v|^2 with v = m * (1/rho) and the
 * 4th-order central difference ((-s2 + 8 s1) - 8 s-1) + s-2) * (1/(12h)).
 * Ghosts of U must be filled.  Per-plane partial sums added in plane order
 * (bitwise independent of the thread count). */
double or_enstrophy(const or_geom* G, const double* U) {
  const int nx = G->n[0], ny = G->n[1], nz = G->n[2], g = G->g;
  const int64_t gx = nx + 2 * g, gy = ny + 2 * g;
  const int64_t npts = or_npts(G);
  const int64_t st[3] = {1, gx, gx * gy};
  double coef[3];
  for (int d = 0; d < 3; ++d) coef[d] = 1.0 / (12.0 * or_spacing(G, d));
  double* plane = (double*)calloc((size_t)nz, sizeof(double));
  if (!plane) return NAN;
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k) {
    double acc = 0.0;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int64_t p = ((int64_t)(k + g) * gy + (j + g)) * gx + (i + g);
        double gr[3][3];
        for (int a = 0; a < 3; ++a)
          for (int d = 0; d < 3; ++d) {
            double v[5];
            for (int o = -2; o <= 2; ++o) {
              if (!o) continue;
              const int64_t q = p + o * st[d];
              v[o + 2] = U[(1 + a) * npts + q] * (1.0 / U[q]);
            }
            gr[a][d] = (((-v[4] + 8.0 * v[3]) - 8.0 * v[1]) + v[0]) * coef[d];
          }
        const double wx = gr[2][1] - gr[1][2], wy = gr[0][2] - gr[2][0], wz = gr[1][0] - gr[0][1];
        acc += 0.5 * ((wx * wx + wy * wy) + wz * wz);
      }
    plane[k] = acc;
  }
  double s = 0.0;
  for (int k = 0; k < nz; ++k) s += plane[k];
  free(plane);
  return s;
}

/* Full-step driver for the CPU baseline: `steps` RK4 (scheme 4) or RK3 (3)
 * steps with CFL (cfl > 0) or fixed dt.  dts[steps] receives each dt. */
int or_advance(const or_geom* G, double* U, int scheme, double cfl, double dt_fixed, int steps,
               double* dts, int64_t* where) {
  double* work = (double*)malloc(or_work_size(G) * sizeof(double));
  if (!work) return -1;
  int rc = 0;
  for (int s = 0; s < steps && !rc; ++s) {
    double dt = dt_fixed;
    if (cfl > 0.0) {
      double out[2];
      rc = or_max_signal(G, U, 0, out, where);
      if (rc) { rc = 100 + rc; break; }
      if (!isfinite(out[0]) || out[0] <= 0.0) { rc = 103; break; }
      dt = cfl / out[0];
    }
    if (dts) dts[s] = dt;
    rc = scheme == 3 ? or_rk3_step(G, U, dt, work, where) : or_rk4_step(G, U, dt, work, where);
  }
  free(work);
  return rc;
}

int or_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (the reference arm uses every host thread even
 * when a launcher such as torchrun exported OMP_NUM_THREADS=1). */
void or_set_num_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
