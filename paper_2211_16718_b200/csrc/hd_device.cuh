// hd_device.cuh -- device helpers shared by the sweep and field kernels.
#pragma once

#include "hd_internal.cuh"

namespace hd {

// ((-s[+2] + 8 s[+1]) - 8 s[-1]) + s[-2], times coef (kernels.py:221-226)
template <bool EXACT>
__device__ __forceinline__ double cd4(const double* __restrict__ s, int64_t st, double coef) {
  const double p2 = __ldg(s + 2 * st), p1 = __ldg(s + st), m1 = __ldg(s - st),
               m2 = __ldg(s - 2 * st);
  if constexpr (EXACT) return xm(xa(xs(xa(-p2, xm(8.0, p1)), xm(8.0, m1)), m2), coef);
  return (8.0 * (p1 - m1) + (m2 - p2)) * coef;
}

// ---- cp.async (LDGSTS): global -> shared without staging through registers ----
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// the same stencil on values already in registers / shared memory; the fast
// form rounds the derivative itself (no contraction into its consumers), so a
// kernel variant that uses it twice (flux kernel + enstrophy) computes the same
// fluxes bit for bit
template <bool EXACT>
__device__ __forceinline__ double cd4v(double m2, double m1, double p1, double p2, double coef) {
  if constexpr (EXACT) return xm(xa(xs(xa(-p2, xm(8.0, p1)), xm(8.0, m1)), m2), coef);
  return __dmul_rn(8.0 * (p1 - m1) + (m2 - p2), coef);
}

// Writes v at interior point (i,j,k) of field f and at its periodic images
// along the axes in `mask` (only those that wrap locally).
__device__ __forceinline__ void store_with_images(double* f, const Geo& G, int i, int j, int k,
                                                  int mask, double v) {
  int ox[3], oy[3], oz[3];
  int nx = 1, ny = 1, nz = 1;
  ox[0] = 0; oy[0] = 0; oz[0] = 0;
  const int g = G.g;
  if (mask & 1) {
    if (i + G.n[0] < G.n[0] + g) ox[nx++] = G.n[0];
    if (i - G.n[0] >= -g) ox[nx++] = -G.n[0];
  }
  if (mask & 2) {
    if (j + G.n[1] < G.n[1] + g) oy[ny++] = G.n[1];
    if (j - G.n[1] >= -g) oy[ny++] = -G.n[1];
  }
  if (mask & 4) {
    if (k + G.n[2] < G.n[2] + g) oz[nz++] = G.n[2];
    if (k - G.n[2] >= -g) oz[nz++] = -G.n[2];
  }
  for (int c = 0; c < nz; ++c)
    for (int b = 0; b < ny; ++b)
      for (int a = 0; a < nx; ++a) f[G.idx(i + ox[a], j + oy[b], k + oz[c])] = v;
}

// axes whose face images kernels write: locally periodic axes, and split axes
// whose images go to the neighbours' ghost planes (peer stores, Geo::peer)
__device__ __forceinline__ int periodic_mask(const Geo& G) {
  return ((G.periodic[0] || G.peer[0]) ? 1 : 0) | ((G.periodic[1] || G.peer[1]) ? 2 : 0) |
         ((G.periodic[2] || G.peer[2]) ? 4 : 0);
}

__device__ __forceinline__ double dmax_nan(double a, double b) {
  // numpy max propagates NaN
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b);
}

// Fast-mode diagnostics of one conserved state (timeint.py:100-131 with one
// reciprocal of rho): folds it into acc = {signal max, signal sum, wavespeed,
// mass, mx, my, mz, energy, KE}; returns 1 / 2 for a nonpositive density /
// pressure, else 0.  Shared by reduce_kernel<fast> and the fused z sweep.
__device__ __forceinline__ int diag_fast(const double (&c)[5], double gamma, double rh0, double rh1,
                                         double rh2, double (&acc)[9]) {
  const double rho = c[0], m1 = c[1], m2 = c[2], m3 = c[3], E = c[4];
  const double inv = frcp(rho);
  const double v0 = m1 * inv, v1 = m2 * inv, v2 = m3 * inv;
  const double p = (gamma - 1.0) * (E - (0.5 * inv) * (m1 * m1 + m2 * m2 + m3 * m3));
  const double a = sqrt(gamma * p * inv);
  const double s0 = (fabs(v0) + a) * rh0, s1 = (fabs(v1) + a) * rh1, s2 = (fabs(v2) + a) * rh2;
  acc[0] = dmax_nan(acc[0], dmax_nan(dmax_nan(s0, s1), s2));
  acc[1] = dmax_nan(acc[1], (s0 + s1) + s2);
  acc[2] = dmax_nan(acc[2], dmax_nan(dmax_nan(fabs(v0), fabs(v1)), fabs(v2)) + a);
  acc[3] += rho;
  acc[4] += m1;
  acc[5] += m2;
  acc[6] += m3;
  acc[7] += E;
  acc[8] += 0.5 * ((v0 * v0 + v1 * v1) + v2 * v2);
  return !(rho > 0.0) ? 1 : (!(p > 0.0) ? 2 : 0);
}

// does the point (i,j,k) have a face image that lands in a neighbour's buffer?
__device__ __forceinline__ bool touches_peer(const Geo& G, int i, int j, int k) {
  const int g = G.g;
  return (G.peer[0] && (i < g || i >= G.n[0] - g)) || (G.peer[1] && (j < g || j >= G.n[1] - g)) ||
         (G.peer[2] && (k < g || k >= G.n[2] - g));
}



// v at interior (i,j,k) plus its face images along the axes in `mask`
// (stencils here are axis-aligned: edges and corners are never read).
__device__ __forceinline__ void store_face_images(double* f, const Geo& G, int i, int j, int k,
                                                  int mask, double v) {
  f[G.idx(i, j, k)] = v;
  const int g = G.g;
  // peer axes: the image lands in the neighbour's buffer (peer_lo/hi deltas)
  if (mask & 1) {
    if (i < g) f[G.idx(i + G.n[0], j, k) + G.peer_lo[0]] = v;
    if (i >= G.n[0] - g) f[G.idx(i - G.n[0], j, k) + G.peer_hi[0]] = v;
  }
  if (mask & 2) {
    if (j < g) f[G.idx(i, j + G.n[1], k) + G.peer_lo[1]] = v;
    if (j >= G.n[1] - g) f[G.idx(i, j - G.n[1], k) + G.peer_hi[1]] = v;
  }
  if (mask & 4) {
    if (k < g) f[G.idx(i, j, k + G.n[2]) + G.peer_lo[2]] = v;
    if (k >= G.n[2] - g) f[G.idx(i, j, k - G.n[2]) + G.peer_hi[2]] = v;
  }
}

// Symmetric viscous-flux storage: tau is symmetric, so the 3 x 4 flux
// components F_d = (tau_0d, tau_1d, tau_2d, work_d) of viscous.py:112-116 are
// held as 9 fields; each is differentiated along the axes listed:
//   0 tau00 {x}   1 tau01 {x,y}   2 tau11 {y}   3 w0 {x}   4 w1 {y}
//   5 tau02 {x,z} 6 tau12 {y,z}   7 tau22 {z}   8 w2 {z}
// Fields 5..8 (everything differentiated along z) are contiguous: the z halo
// exchange of a decomposed run moves exactly that group.
constexpr int VF_N = 9;
constexpr int VF_ZGROUP = 5;
__device__ __forceinline__ int vf_field(int d, int row) {  // F_d[row-1]
  constexpr int tab[3][4] = {{0, 1, 5, 3}, {1, 2, 6, 4}, {5, 6, 7, 8}};
  return tab[d][row - 1];
}
__host__ __device__ __forceinline__ int vf_axes(int f) {
  constexpr int tab[9] = {1, 3, 2, 1, 2, 5, 6, 4, 4};
  return tab[f];
}


// ---------------------------------------------------------------------------
// RK stage update (timeint.py:168-193), per point and variable
// ---------------------------------------------------------------------------
struct RKArgs {
  int scheme, stage;
  double* u;         // step base state (in/out for the last stage)
  const double* stage_in;  // this stage's input state (RK3 stages 1, 2 combine it)
  double* stage_out;       // next stage state (ping-pong half of the STAGE buffer)
  double* acc;       // RK4 accumulator
  const double* dt;  // device dt
  // fast mode: out = a0 u + a1 stage_in + dt (kc k + ka acc); acc' = b0 acc + b1 k
  double a0, a1, kc, ka, b0, b1;
  int rd_us, rd_acc, wr_acc, to_u;
};

template <bool EXACT>
__device__ __forceinline__ void rk_point(const RKArgs& r, double dt, int64_t off, double k,
                                         double& out, bool& to_u) {
  const double u0 = r.u[off];
  if (r.scheme == HD_SCHEME_RK4) {
    if constexpr (EXACT) {
      const double half = xm(0.5, dt);
      switch (r.stage) {
        case 0: r.acc[off] = k; out = xa(u0, xm(half, k)); to_u = false; break;
        case 1: r.acc[off] = xa(r.acc[off], xm(2.0, k)); out = xa(u0, xm(half, k)); to_u = false; break;
        case 2: r.acc[off] = xa(r.acc[off], xm(2.0, k)); out = xa(u0, xm(dt, k)); to_u = false; break;
        default: out = xa(u0, xm(xd(dt, 6.0), xa(r.acc[off], k))); to_u = true; break;
      }
    } else {
      const double half = 0.5 * dt;
      switch (r.stage) {
        case 0: r.acc[off] = k; out = u0 + half * k; to_u = false; break;
        case 1: r.acc[off] = r.acc[off] + 2.0 * k; out = u0 + half * k; to_u = false; break;
        case 2: r.acc[off] = r.acc[off] + 2.0 * k; out = u0 + dt * k; to_u = false; break;
        default: out = u0 + (dt * (1.0 / 6.0)) * (r.acc[off] + k); to_u = true; break;
      }
    }
  } else {  // TVD-RK3
    if constexpr (EXACT) {
      switch (r.stage) {
        case 0: out = xa(u0, xm(dt, k)); to_u = false; break;
        case 1: out = xa(xm(0.75, u0), xm(0.25, xa(r.stage_in[off], xm(dt, k)))); to_u = false; break;
        default:
          out = xa(xm(1.0 / 3.0, u0), xm(2.0 / 3.0, xa(r.stage_in[off], xm(dt, k)))); to_u = true; break;
      }
    } else {
      switch (r.stage) {
        case 0: out = u0 + dt * k; to_u = false; break;
        case 1: out = 0.75 * u0 + 0.25 * (r.stage_in[off] + dt * k); to_u = false; break;
        default: out = (1.0 / 3.0) * u0 + (2.0 / 3.0) * (r.stage_in[off] + dt * k); to_u = true; break;
      }
    }
  }
}

template <bool EXACT>
__device__ __forceinline__ void rk_store(const RKArgs& r, const Geo& G, int i, int j, int k,
                                         const double (&kv)[NV]) {
  // Only face images are written: every consumer of a stage state reads its
  // ghosts along one axis at a time (sweeps, gradients), never edges/corners.
  const double dt = *r.dt;
  const int64_t q = G.idx(i, j, k);
  const int pm = periodic_mask(G);
  if constexpr (EXACT) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double out;
      bool to_u;
      rk_point<true>(r, dt, q + v * G.npts, kv[v], out, to_u);
      store_face_images((to_u ? r.u : r.stage_out) + v * G.npts, G, i, j, k, pm, out);
    }
  } else {
    const double kcd = r.kc * dt, kad = r.ka * dt;
    double* dst = r.to_u ? r.u : r.stage_out;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int64_t off = q + v * G.npts;
      const double kk = kv[v];
      double w = kcd * kk, accv = 0.0;
      if (r.rd_acc) {
        accv = r.acc[off];
        w = fma(kad, accv, w);
      }
      double out = fma(r.a0, r.u[off], w);
      if (r.rd_us) out = fma(r.a1, r.stage_in[off], out);
      if (r.wr_acc) r.acc[off] = fma(r.b0, accv, r.b1 * kk);
      store_face_images(dst + v * G.npts, G, i, j, k, pm, out);
    }
  }
}

// fast-mode RK update with the base state and accumulator already in registers
// Index deltas of the face images of interior point (i,j,k) along the axes in
// `mask` (at most one per axis once n >= 2g; z images land in the neighbours'
// buffers in peer mode); returns how many.
__device__ __forceinline__ int face_image_deltas(const Geo& G, int i, int j, int k, int mask,
                                                 int64_t (&dl)[6]) {
  int nd = 0;
  const int g = G.g;
  // both images of an axis when the block is thinner than 2g along it
  if (mask & 1) {
    if (i < g) dl[nd++] = G.n[0] + G.peer_lo[0];
    if (i >= G.n[0] - g) dl[nd++] = -(int64_t)G.n[0] + G.peer_hi[0];
  }
  if (mask & 2) {
    if (j < g) dl[nd++] = (int64_t)G.n[1] * G.sy + G.peer_lo[1];
    if (j >= G.n[1] - g) dl[nd++] = -(int64_t)G.n[1] * G.sy + G.peer_hi[1];
  }
  if (mask & 4) {
    if (k < g) dl[nd++] = (int64_t)G.n[2] * G.sz + G.peer_lo[2];
    if (k >= G.n[2] - g) dl[nd++] = -(int64_t)G.n[2] * G.sz + G.peer_hi[2];
  }
  return nd;
}

// N fields (stride npts) at flat point q and its face images
template <int N>
__device__ __forceinline__ void store_point_images(double* f, int64_t np, int64_t q, int nd,
                                                   const int64_t (&dl)[6], const double (&v)[N]) {
#pragma unroll
  for (int c = 0; c < N; ++c) f[q + c * np] = v[c];
  for (int t = 0; t < nd; ++t)
#pragma unroll
    for (int c = 0; c < N; ++c) f[q + dl[t] + c * np] = v[c];
}

__device__ __forceinline__ void rk_store_pre(const RKArgs& r, const Geo& G, int i, int j, int k,
                                             const double (&kv)[NV], const double (&u0)[NV],
                                             const double (&acc)[NV], double (&outv)[NV]) {
  const double dt = *r.dt;
  const int64_t q = G.idx(i, j, k);
  const double kcd = r.kc * dt, kad = r.ka * dt;
  double* dst = r.to_u ? r.u : r.stage_out;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int64_t off = q + v * G.npts;
    double out = fma(r.a0, u0[v], fma(kad, acc[v], kcd * kv[v]));
    if (r.rd_us) out = fma(r.a1, r.stage_in[off], out);
    if (r.wr_acc) r.acc[off] = fma(r.b0, acc[v], r.b1 * kv[v]);
    outv[v] = out;
  }
  int64_t dl[6];
  const int nd = face_image_deltas(G, i, j, k, periodic_mask(G), dl);
  store_point_images<NV>(dst, G.npts, q, nd, dl, outv);
}

// rk_store_pre for the classical RK4 tableau with the stage kind fixed at compile
// time: K = 0 stage 0 (acc = k), 1 stages 1-2 (acc += 2k), 2 stage 3 (u + dt/6 (acc + k)).
// The same roundings as the generic path: out = u0 + (kad acc + round(kcd k)).
template <int K>  // 0, 1, 2 only
__device__ __forceinline__ void rk4_store(const RKArgs& r, const Geo& G, int i, int j, int k,
                                          const double (&kv)[NV], const double (&u0)[NV],
                                          const double (&acc)[NV], double (&outv)[NV]) {
  static_assert(K >= 0 && K <= 2, "RK4 stage kind");
  const double dt = *r.dt;
  const int64_t q = G.idx(i, j, k);
  const double kcd = r.kc * dt;
  double* dst = K == 2 ? r.u : r.stage_out;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double kk = __dmul_rn(kcd, kv[v]);
    if constexpr (K == 2) {
      outv[v] = __dadd_rn(u0[v], fma(r.ka * dt, acc[v], kk));
    } else {
      outv[v] = __dadd_rn(u0[v], kk);
      r.acc[q + v * G.npts] = K == 0 ? kv[v] : fma(1.0, acc[v], 2.0 * kv[v]);
    }
  }
  int64_t dl[6];
  const int nd = face_image_deltas(G, i, j, k, periodic_mask(G), dl);
  store_point_images<NV>(dst, G.npts, q, nd, dl, outv);
}

RKArgs make_rk(const hd_plan* p, int scheme, int stage, double* u, const double* dt_dev);

// kv[row] += D_d F_d[row-1] for the dims in dmask, in the order d = 0, 1, 2 and
// rows 1..4 (viscous.py:112-120).
template <bool EXACT>
__device__ __forceinline__ void add_viscous_divergence(const double* __restrict__ vf, const Geo& G,
                                                       int64_t q, int dmask, double (&kv)[NV]) {
  const int64_t np = G.npts;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (!(dmask & (1 << d))) continue;
    const int64_t st = G.stride(d);
    const double coef = 1.0 / (12.0 * G.h[d]);
#pragma unroll
    for (int row = 1; row < NV; ++row) {
      const double dv = cd4<EXACT>(vf + (int64_t)vf_field(d, row) * np + q, st, coef);
      if constexpr (EXACT) kv[row] = xa(kv[row], dv);
      else kv[row] += dv;
    }
  }
}

}  // namespace hd
