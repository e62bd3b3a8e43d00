// hd_field.cu -- ghost fill, viscous terms, RK stage updates, reductions.
//
//   fill_ghosts_kernel   grid.py:211-251   (_wrap_axis x -> y -> z, full extents)
//   prims_kernel         physics.py:240-255 + viscous.py:80-81 (u, v, w, T = gamma p / rho)
//   gradflux_kernel      viscous.py:86-116 (12 central gradients -> tau, q -> 9 flux fields,
//                        periodic images along the flux's own axis = the sync_scalars it needs)
//   divergence_kernel    viscous.py:119-120 (inc[1..4] += D_d F_d, d = 0, 1, 2), fused with
//                        the RK stage update timeint.py:168-193
//   rk_update_kernel     timeint.py:168-193 when mu == 0 (viscous.py:72-73 short-circuit)
//   central_diff4_kernel kernels.py:207-227 (stand-alone, for the operator API)
//   reduce kernels       timeint.py:100-131 (CFL signal, totals, max wavespeed, KE)
#include <cuda.h>

#include "hd_device.cuh"

namespace hd {

// ---------------------------------------------------------------------------
// periodic ghost fill: one launch per axis, x then y then z (grid.py:241-243)
// ---------------------------------------------------------------------------
__global__ void fill_axis_kernel(double* f, int nfields, Geo G, int axis) {
  const int g = G.g;
  const int64_t e0 = G.gn[0], e1 = G.gn[1], e2 = G.gn[2];
  // slab: 2g positions along `axis`, full ghosted extent of the others
  int64_t ea = 2 * g, eb, ec;
  if (axis == 0) { eb = e1; ec = e2; }
  else if (axis == 1) { eb = e0; ec = e2; }
  else { eb = e0; ec = e1; }
  const int64_t per_field = ea * eb * ec;
  const int64_t total = per_field * nfields;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fld = t / per_field;
    int64_t r = t - fld * per_field;
    // fastest index: the contiguous axis among (b, c, a) ordering chosen for coalescing
    int64_t a, b, c;
    if (axis == 0) {  // a = x ghost pos (fastest), b = y, c = z
      a = r % ea; r /= ea; b = r % eb; c = r / eb;
    } else {          // b = x (fastest), a = ghost pos, c = other
      b = r % eb; r /= eb; a = r % ea; c = r / ea;
    }
    const int n = G.n[axis];
    const int64_t dst_pos = a < g ? a : (a - g) + n + g;      // [0,g) or [n+g, n+2g)
    const int64_t src_pos = a < g ? a + n : (a - g) + g;      // n + q   or g + q
    int64_t dx, dy, dz, sx, sy, sz;
    if (axis == 0) { dx = dst_pos; sx = src_pos; dy = sy = b; dz = sz = c; }
    else if (axis == 1) { dy = dst_pos; sy = src_pos; dx = sx = b; dz = sz = c; }
    else { dz = dst_pos; sz = src_pos; dx = sx = b; dy = sy = c; }
    double* base = f + fld * G.npts;
    base[(dz * e1 + dy) * e0 + dx] = base[(sz * e1 + sy) * e0 + sx];
  }
}

int launch_fill_ghosts(const hd_plan* p, double* f, int nfields, int axis_mask, cudaStream_t s) {
  const Geo& G = p->geo;
  for (int axis = 0; axis < 3; ++axis) {
    if (!(axis_mask & (1 << axis)) || !G.periodic[axis]) continue;
    int64_t others = axis == 0 ? (int64_t)G.gn[1] * G.gn[2]
                               : (axis == 1 ? (int64_t)G.gn[0] * G.gn[2] : (int64_t)G.gn[0] * G.gn[1]);
    int64_t total = (int64_t)2 * G.g * others * nfields;
    int blocks = (int)((total + 255) / 256);
    if (blocks > p->sm_count * 16) blocks = p->sm_count * 16;
    if (blocks < 1) blocks = 1;
    fill_axis_kernel<<<blocks, 256, 0, s>>>(f, nfields, G, axis); hd::count_launches(1);
  }
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

// ---------------------------------------------------------------------------
// primitives for the viscous terms over the ghosted box
// ---------------------------------------------------------------------------
template <bool EXACT>
__global__ void prims_kernel(const double* __restrict__ u, double* __restrict__ prim, Geo G,
                             Phys ph, int64_t q_lo, int64_t q_hi) {
  const int64_t np = G.npts;
  for (int64_t q = q_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < q_hi;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double rho = __ldg(u + q), m1 = __ldg(u + np + q), m2 = __ldg(u + 2 * np + q),
                 m3 = __ldg(u + 3 * np + q), E = __ldg(u + 4 * np + q);
    double vx, vy, vz, T;
    if constexpr (EXACT) {
      const double inv = xd(1.0, rho);
      vx = xm(m1, inv);
      vy = xm(m2, inv);
      vz = xm(m3, inv);
      const double p = xm(ph.gm1, xs(E, xm(xm(0.5, rho), xa(xa(xm(vx, vx), xm(vy, vy)), xm(vz, vz)))));
      T = xd(xm(ph.gamma, p), rho);
    } else {
      const double inv = frcp(rho);
      vx = m1 * inv;
      vy = m2 * inv;
      vz = m3 * inv;
      const double p = ph.gm1 * (E - (0.5 * inv) * (m1 * m1 + m2 * m2 + m3 * m3));
      T = ph.gamma * p * inv;
    }
    prim[q] = vx;
    prim[np + q] = vy;
    prim[2 * np + q] = vz;
    prim[3 * np + q] = T;
  }
}

static int prims_range(const hd_plan* p, const double* u, int64_t q_lo, int64_t q_hi,
                       cudaStream_t s) {
  if (q_hi <= q_lo) return HD_OK;
  double* prim = (double*)(p->ws + p->off[HD_BUF_PRIM]);
  int64_t want = (q_hi - q_lo + 255) / 256;
  int blocks = (int)(want < p->sm_count * 8 ? want : p->sm_count * 8);
  if (p->mode == HD_MODE_EXACT)
    prims_kernel<true><<<blocks, 256, 0, s>>>(u, prim, p->geo, p->phys, q_lo, q_hi);
  else
    prims_kernel<false><<<blocks, 256, 0, s>>>(u, prim, p->geo, p->phys, q_lo, q_hi);
  hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int launch_prims(const hd_plan* p, const double* u, cudaStream_t s) {
  return prims_range(p, u, 0, p->geo.npts, s);
}

// ghosted z planes [z_lo, z_hi), full x-y extent (decomposed runs: exchanged ghosts)
int launch_prims_planes(const hd_plan* p, const double* u, int z_lo, int z_hi, cudaStream_t s) {
  return prims_range(p, u, (int64_t)z_lo * p->geo.sz, (int64_t)z_hi * p->geo.sz, s);
}


// ---------------------------------------------------------------------------
// viscous fluxes: 12 gradients -> tau, heat flux -> F_d = (tau_0d, tau_1d, tau_2d, work_d),
// stored symmetrically as 9 fields (hd_device.cuh VF_*)
// ---------------------------------------------------------------------------
// viscous.py:92-116 at one point: stress, heat flux, the 9 symmetric flux values
template <bool EXACT>
__device__ __forceinline__ void viscous_flux_point(const double (&gr)[3][3], const double (&gT)[3],
                                                   const double (&vel)[3], double mu, double q_coef,
                                                   double (&val)[VF_N]) {
  double tau[3][3];
  if constexpr (EXACT) {
    const double div = xa(xa(gr[0][0], gr[1][1]), gr[2][2]);
    const double ttd = xm(2.0 / 3.0, div);
#pragma unroll
    for (int a = 0; a < 3; ++a) tau[a][a] = xm(mu, xs(xm(2.0, gr[a][a]), ttd));
    tau[0][1] = tau[1][0] = xm(mu, xa(gr[0][1], gr[1][0]));
    tau[0][2] = tau[2][0] = xm(mu, xa(gr[0][2], gr[2][0]));
    tau[1][2] = tau[2][1] = xm(mu, xa(gr[1][2], gr[2][1]));
  } else {
    const double div = gr[0][0] + gr[1][1] + gr[2][2];
    const double ttd = (2.0 / 3.0) * div;
#pragma unroll
    for (int a = 0; a < 3; ++a) tau[a][a] = mu * (2.0 * gr[a][a] - ttd);
    tau[0][1] = tau[1][0] = mu * (gr[0][1] + gr[1][0]);
    tau[0][2] = tau[2][0] = mu * (gr[0][2] + gr[2][0]);
    tau[1][2] = tau[2][1] = mu * (gr[1][2] + gr[2][1]);
  }
  double w[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if constexpr (EXACT) {
      const double qd = xm(q_coef, gT[d]);
      w[d] = xs(xa(xa(xm(vel[0], tau[0][d]), xm(vel[1], tau[1][d])), xm(vel[2], tau[2][d])), qd);
    } else {
      w[d] = vel[0] * tau[0][d] + vel[1] * tau[1][d] + vel[2] * tau[2][d] - q_coef * gT[d];
    }
  }
  val[0] = tau[0][0];
  val[1] = tau[0][1];
  val[2] = tau[1][1];
  val[3] = w[0];
  val[4] = w[1];
  val[5] = tau[0][2];
  val[6] = tau[1][2];
  val[7] = tau[2][2];
  val[8] = w[2];
}

template <bool EXACT>
__global__ void __launch_bounds__(128) gradflux_kernel(const double* __restrict__ prim,
                                                       double* __restrict__ vf, Geo G, double mu,
                                                       double q_coef) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= G.n[0] || j >= G.n[1]) return;
  const int64_t np = G.npts;
  const int64_t q = G.idx(i, j, k);
  const int64_t st[3] = {1, G.sy, G.sz};
  double coef[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) coef[d] = 1.0 / (12.0 * G.h[d]);
  double gr[3][3], gT[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int d = 0; d < 3; ++d) gr[a][d] = cd4<EXACT>(prim + a * np + q, st[d], coef[d]);
#pragma unroll
  for (int d = 0; d < 3; ++d) gT[d] = cd4<EXACT>(prim + 3 * np + q, st[d], coef[d]);
  const double vel[3] = {__ldg(prim + q), __ldg(prim + np + q), __ldg(prim + 2 * np + q)};
  double val[VF_N];
  viscous_flux_point<EXACT>(gr, gT, vel, mu, q_coef, val);
  const int pm = periodic_mask(G);
#pragma unroll
  for (int f = 0; f < VF_N; ++f)
    store_face_images(vf + (int64_t)f * np, G, i, j, k, pm & vf_axes(f), val[f]);
  if (G.peer_any && touches_peer(G, i, j, k)) __threadfence_system();
}

// ---------------------------------------------------------------------------
// enstrophy 0.5 |curl v|^2 (north-star diagnostic; the reference's operators:
// v = m * (1/rho) as physics.py:249-252, D_d as viscous.py:23-51)
// ---------------------------------------------------------------------------
// gr[a][d] = d v_a / d x_d
__device__ __forceinline__ double enstrophy_point(const double (&gr)[3][3]) {
  const double wx = gr[2][1] - gr[1][2], wy = gr[0][2] - gr[2][0], wz = gr[1][0] - gr[0][1];
  return 0.5 * ((wx * wx + wy * wy) + wz * wz);
}

// sum of v over the block in a fixed order (warp tree, then warps in order)
// -> partial[slot]; every thread of the block must call it
__device__ __forceinline__ void block_sum_store(double v, double* partial, int64_t slot) {
  __shared__ double sh[32];
  const int t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthreads = blockDim.x * blockDim.y * blockDim.z;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((t & 31) == 0) sh[t >> 5] = v;
  __syncthreads();
  if (t == 0) {
    double s = sh[0];
    for (int w = 1; w < nthreads / 32; ++w) s += sh[w];
    partial[slot] = s;
  }
}

__global__ void sum_finish_kernel(const double* partial, int n, double* out) {
  double v = 0.0;  // one warp, fixed order
  for (int b = threadIdx.x; b < n; b += 32) v += partial[b];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if (threadIdx.x == 0) *out = v;
}

constexpr int ENS_THREADS = 256, ENS_BLOCKS_MAX = 2048;

// stand-alone pass: one warp per x row, the 6 off-diagonal velocity gradients
// from the neighbours' conserved values (IEEE 1/rho, as decode_primitives)
__global__ void __launch_bounds__(ENS_THREADS) enstrophy_kernel(const double* __restrict__ u, Geo G,
                                                                double* partial) {
  const int64_t np = G.npts;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rows = (int64_t)G.n[1] * G.n[2];
  const int64_t st[3] = {1, G.sy, G.sz};
  double coef[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) coef[d] = 1.0 / (12.0 * G.h[d]);
  auto vel = [&](int64_t q, int c) { return __dmul_rn(__ldg(u + (1 + c) * np + q), __ddiv_rn(1.0, __ldg(u + q))); };
  auto D = [&](int64_t q, int c, int d) {
    return cd4v<true>(vel(q - 2 * st[d], c), vel(q - st[d], c), vel(q + st[d], c), vel(q + 2 * st[d], c),
                      coef[d]);
  };
  double acc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)(ENS_THREADS / 32) + warp; r < rows;
       r += (int64_t)gridDim.x * (ENS_THREADS / 32)) {
    const int64_t row0 = G.idx(0, (int)(r % G.n[1]), (int)(r / G.n[1]));
    for (int i = lane; i < G.n[0]; i += 32) {
      const int64_t q = row0 + i;
      double gr[3][3] = {{0.0, D(q, 0, 1), D(q, 0, 2)}, {D(q, 1, 0), 0.0, D(q, 1, 2)},
                         {D(q, 2, 0), D(q, 2, 1), 0.0}};
      acc += enstrophy_point(gr);
    }
  }
  block_sum_store(acc, partial, blockIdx.x);
}

int64_t ens_capacity(const hd_geom& g) {
  // z-marching flux kernel: tiles x z segments (<= tiles + 8 x 512 SMs), or the stand-alone pass
  const int64_t tiles = (int64_t)((g.n[0] + 31) / 32) * ((g.n[1] + 7) / 8);
  return tiles + 4096 > ENS_BLOCKS_MAX ? tiles + 4096 : ENS_BLOCKS_MAX;
}

// defined after the z-marching flux kernel
// gradflux with z marching (blocks of 32 x 8 columns): the z stencil comes from
// a per-thread register queue of 5 planes (each prims value is loaded once per
// column), the x/y stencils from a shared-memory plane tile with a 2-point halo.
// Needs n_x % 32 == 0 and n_y % 8 == 0 (else gradflux_kernel).
// 32 x 8 tiles, 2 blocks/SM, ~4 waves (32x16 and 16x16 tiles measured slower)
constexpr int GZ_TX = 32, GZ_TY = 8, GZ_H = 2, GZ_MINB = 2, GZ_WAVES = 4;
constexpr int GZ_PX = GZ_TX + 2 * GZ_H, GZ_PY = GZ_TY + 2 * GZ_H;

// fast-mode viscous primitives (u, v, w, T) from the 5 conserved values (the
// prims_kernel formula; viscous.py:80-81)
__device__ __forceinline__ void prims_of(const double (&c)[5], double gamma, double gm1,
                                         double (&pv)[4]) {
  const double inv = frcp(c[0]);
  pv[0] = c[1] * inv;
  pv[1] = c[2] * inv;
  pv[2] = c[3] * inv;
  pv[3] = gamma * (gm1 * (c[4] - (0.5 * inv) * (c[1] * c[1] + c[2] * c[2] + c[3] * c[3]))) * inv;
}

// FROM_U (fast mode): `src` is the conserved state and every loaded point is
// converted to primitives on the fly (no primitive fields in HBM); else `src`
// holds the 4 primitive fields.
// ENS: 1 = also the enstrophy of the state from the velocity gradients it forms
// (one partial per block into ens_partial); 2 = only that (no flux fields)
template <bool EXACT, bool FROM_U, int ENS>
__global__ void __launch_bounds__(GZ_TX * GZ_TY, GZ_MINB) gradflux_zm_kernel(
    const double* __restrict__ prim, double* __restrict__ vf, Geo G, double mu, double q_coef,
    int zseg, double gamma, double* ens_partial) {
  // two plane tiles (double-buffered: one barrier per plane); every load is
  // issued one plane before it is needed (z queue: plane k+3; ring: plane k+1)
  __shared__ double tile[2][4][GZ_PY][GZ_PX];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i = blockIdx.x * GZ_TX + tx, j = blockIdx.y * GZ_TY + ty;
  const int k0 = blockIdx.z * zseg;
  const int k1 = min(k0 + zseg, G.n[2]);
  const int64_t np = G.npts;
  const int64_t sz = G.sz;
  double coef[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) coef[d] = 1.0 / (12.0 * G.h[d]);
  // z queue: qz[f][w] = prims field f at plane k - 2 + w of this column
  // raw loads (NF fields) are issued one plane ahead and converted when used
  constexpr int NF = FROM_U ? 5 : 4;
  double qz[4][5], nq[NF];
  const int64_t col = G.idx(i, j, 0);
  const double gm1 = gamma - 1.0;
  auto load = [&](int64_t q, double (&v)[NF]) {
#pragma unroll
    for (int f = 0; f < NF; ++f) v[f] = __ldg(prim + f * np + q);
  };
  auto prims = [&](const double (&v)[NF], double (&pv)[4]) {
    if constexpr (FROM_U) {
      prims_of(v, gamma, gm1, pv);
    } else {
#pragma unroll
      for (int f = 0; f < 4; ++f) pv[f] = v[f];
    }
  };
#pragma unroll
  for (int w = 1; w < 5; ++w) {
    double v[NF], pv[4];
    load(col + (int64_t)(k0 - 3 + w) * sz, v);
    prims(v, pv);
#pragma unroll
    for (int f = 0; f < 4; ++f) qz[f][w] = pv[f];
  }
  load(col + (int64_t)(k0 + 2) * sz, nq);
  // halo ring of the plane tile (minus the never-read corners): <= 1 point per thread
  const int r = ty * GZ_TX + tx;
  int px = 0, py = 0;
  bool has_ring = r < GZ_PX * GZ_PY - GZ_TX * GZ_TY;
  if (has_ring) {  // ring index -> (px, py): rows above/below the tile, then side columns
    if (r < 2 * GZ_H * GZ_PX) {
      py = r / GZ_PX;
      px = r % GZ_PX;
      if (py >= GZ_H) py += GZ_TY;
    } else {
      const int s = r - 2 * GZ_H * GZ_PX;
      py = GZ_H + s / (2 * GZ_H);
      px = s % (2 * GZ_H);
      if (px >= GZ_H) px += GZ_TX;
    }
    has_ring = !((px < GZ_H || px >= GZ_H + GZ_TX) && (py < GZ_H || py >= GZ_H + GZ_TY));
  }
  const int64_t rcol = G.idx(blockIdx.x * GZ_TX + px - GZ_H, blockIdx.y * GZ_TY + py - GZ_H, 0);
  double rv[NF];
  if (has_ring) load(rcol + (int64_t)k0 * sz, rv);
  double ens = 0.0;
  for (int k = k0; k < k1; ++k) {
    const int b = k & 1;
    double pq[4], pr[4];
    prims(nq, pq);
    if (has_ring) prims(rv, pr);
#pragma unroll
    for (int f = 0; f < 4; ++f) {
#pragma unroll
      for (int w = 0; w < 4; ++w) qz[f][w] = qz[f][w + 1];
      qz[f][4] = pq[f];
      tile[b][f][ty + GZ_H][tx + GZ_H] = qz[f][2];
      if (has_ring) tile[b][f][py][px] = pr[f];
    }
    if (k + 1 < k1) {
      load(col + (int64_t)(k + 3) * sz, nq);
      if (has_ring) load(rcol + (int64_t)(k + 1) * sz, rv);
    }
    __syncthreads();
    double gr[3][3], gT[3];
    const int cx = tx + GZ_H, cy = ty + GZ_H;
    double (*tl)[GZ_PY][GZ_PX] = tile[b];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double gx = cd4v<EXACT>(tl[f][cy][cx - 2], tl[f][cy][cx - 1], tl[f][cy][cx + 1],
                                     tl[f][cy][cx + 2], coef[0]);
      const double gy = cd4v<EXACT>(tl[f][cy - 2][cx], tl[f][cy - 1][cx], tl[f][cy + 1][cx],
                                     tl[f][cy + 2][cx], coef[1]);
      const double gz = cd4v<EXACT>(qz[f][0], qz[f][1], qz[f][3], qz[f][4], coef[2]);
      if (f < 3) {
        gr[f][0] = gx;
        gr[f][1] = gy;
        gr[f][2] = gz;
      } else {
        gT[0] = gx;
        gT[1] = gy;
        gT[2] = gz;
      }
    }
    const double vel[3] = {qz[0][2], qz[1][2], qz[2][2]};
    if constexpr (ENS != 0) ens += enstrophy_point(gr);
    if constexpr (ENS == 2) continue;
    double val[VF_N];
    viscous_flux_point<EXACT>(gr, gT, vel, mu, q_coef, val);
    // each field gets face images only along the axes it is differentiated along
    // (z images into the neighbours' ghost planes in peer mode)
    const int pm = periodic_mask(G);
    const int g = G.g;
    const int64_t q = G.idx(i, j, k);
    const bool xl = (pm & 1) && i < g, xh = (pm & 1) && i >= G.n[0] - g;
    const bool yl = (pm & 2) && j < g, yh = (pm & 2) && j >= G.n[1] - g;
    const bool zl = (pm & 4) && k < g, zh = (pm & 4) && k >= G.n[2] - g;
    const int64_t dy = (int64_t)G.n[1] * G.sy, dz = (int64_t)G.n[2] * sz;
#pragma unroll
    for (int f = 0; f < VF_N; ++f) {
      double* F = vf + (int64_t)f * np + q;
      const double v = val[f];
      F[0] = v;
      const int axes = vf_axes(f);
      if (axes & 1) {
        if (xl) F[G.n[0] + G.peer_lo[0]] = v;
        if (xh) F[-G.n[0] + G.peer_hi[0]] = v;
      }
      if (axes & 2) {
        if (yl) F[dy + G.peer_lo[1]] = v;
        if (yh) F[-dy + G.peer_hi[1]] = v;
      }
      if (axes & 4) {
        if (zl) F[dz + G.peer_lo[2]] = v;
        if (zh) F[-dz + G.peer_hi[2]] = v;
      }
    }
  }
  // peer stores performed before the kernel ends (threads that made any)
  if (G.peer_any && ((G.peer[2] && (k0 < G.g || k1 > G.n[2] - G.g)) ||
                     touches_peer(G, i, j, G.g)))
    __threadfence_system();
  if constexpr (ENS != 0)
    block_sum_store(ens, ens_partial, ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
}


// ---------------------------------------------------------------------------
// z-marching flux kernel fed by TMA (fast mode, primitives from the state).
// The same tile march as gradflux_zm_kernel, but the raw state arrives as one
// 4D TMA box per plane -- (38 x, 12 y, 1 z, 5 variables): the 32 x 8 tile plus
// its 2-point halo, widened by one column on each side so the box starts on a
// 16-byte boundary (a tensor load whose innermost start coordinate is not
// 16-byte aligned raises an illegal instruction on B200; tools/gpu/tma_bisect*.cu)
// -- into a ring of GT_S shared-memory slots, tracked by one
// mbarrier per slot (expect_tx / complete_tx).  Thread 0 refills the slot of
// plane k with plane k + 4 right after iteration k's barrier, so every load is
// in flight ~2 planes ahead with no registers held and no per-thread address
// arithmetic; the threads only convert (their centre of plane k+2 into the
// register z queue, the halo ring of plane k into the primitive tile) and
// compute.  One barrier per plane, as before: it also retires the raw slot.
// ---------------------------------------------------------------------------
constexpr int GT_BX = GZ_PX + 2;  // box width: x - 3 .. x + 34 of the tile, 304 B rows
// Tile shape and ring depth of the TMA kernel: 32 x 8 tiles, a 4-plane ring, 2
// blocks/SM (3.64 ms per launch at 512^3 against 3.93 for the register-prefetch
// kernel).  32 x 16 tiles with a 5-plane ring at 1 block of 16 warps/SM (more
// bytes in flight, 17% less halo) measured 3.91 ms (tools/gpu/flux_probe.py).
template <int TY_, int S_> struct GtCfg {
  static constexpr int TY = TY_, S = S_, PY = TY + 2 * GZ_H;
  static constexpr int MINB = TY <= 8 ? 2 : 1;
  static constexpr int BOX = NV * PY * GT_BX;          // doubles per box
  static constexpr int SLOT = (BOX + 15) / 16 * 16;    // slots 128-byte aligned (TMA destination)
  struct Smem {
    double raw[S][SLOT];
    double tile[2][4][PY][GZ_PX];  // primitive planes, double-buffered
    unsigned long long full[S];    // mbarriers
  };
};
using GtSmall = GtCfg<8, 4>;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            int c3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

template <int ENS, class C>
__global__ void __launch_bounds__(GZ_TX * C::TY, C::MINB) gradflux_tma_kernel(
    const __grid_constant__ CUtensorMap tm, double* __restrict__ vf, Geo G, double mu, double q_coef,
    int zseg, double gamma, double* ens_partial) {
  constexpr int TY = C::TY, PY = C::PY, GT_S = C::S;
  constexpr unsigned BOX_BYTES = C::BOX * 8;
  extern __shared__ __align__(128) unsigned char gt_smem[];
  typename C::Smem& S = *reinterpret_cast<typename C::Smem*>(gt_smem);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * GZ_TX + tx;
  const int i = blockIdx.x * GZ_TX + tx, j = blockIdx.y * TY + ty;
  const int k0 = blockIdx.z * zseg;
  const int k1 = min(k0 + zseg, G.n[2]);
  const int g = G.g;
  const int p0 = k0 - 2, plast = k1 + 1;  // planes the z stencils touch
  // box origin (ghosted coordinates): x one column left of the halo, even, so the
  // row start is 16-byte aligned (n_x % 32 == 0, g = 3 -> 32 bx + g - 3)
  const int bx = blockIdx.x * GZ_TX - GZ_H - 1 + g, by = blockIdx.y * TY - GZ_H + g;
  double coef[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) coef[d] = 1.0 / (12.0 * G.h[d]);
  const double gm1 = gamma - 1.0;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    for (int s = 0; s < GT_S; ++s) mbar_init(&S.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int p) {  // thread 0
    const int s = (p - p0) % GT_S;
    mbar_expect_tx(&S.full[s], BOX_BYTES);
    tma_load_4d(&S.raw[s][0], &tm, bx, by, p + g, 0, &S.full[s]);
  };
  auto wait_plane = [&](int p) {
    const int r = p - p0;
    mbar_wait(&S.full[r % GT_S], (unsigned)((r / GT_S) & 1));
  };
  auto prims_at = [&](int p, int py, int px, double (&pv)[4]) {
    const int s = (p - p0) % GT_S;
    double c[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) c[v] = S.raw[s][(v * PY + py) * GT_BX + px + 1];
    prims_of(c, gamma, gm1, pv);
  };
  if (tid == 0)
    for (int p = p0; p < p0 + GT_S && p <= plast; ++p) issue(p);
  // z queue: qz[f][w] = primitive f at plane k - 2 + w of this column
  double qz[4][5];
#pragma unroll
  for (int w = 1; w < 5; ++w) {
    const int p = k0 - 3 + w;
    wait_plane(p);
    double pv[4];
    prims_at(p, ty + GZ_H, tx + GZ_H, pv);
#pragma unroll
    for (int f = 0; f < 4; ++f) qz[f][w] = pv[f];
  }
  // halo ring of the primitive tile (minus the never-read corners): <= 1 point per thread
  const int r = tid;
  int px = 0, py = 0;
  bool has_ring = r < GZ_PX * PY - GZ_TX * TY;
  if (has_ring) {
    if (r < 2 * GZ_H * GZ_PX) {
      py = r / GZ_PX;
      px = r % GZ_PX;
      if (py >= GZ_H) py += TY;
    } else {
      const int s = r - 2 * GZ_H * GZ_PX;
      py = GZ_H + s / (2 * GZ_H);
      px = s % (2 * GZ_H);
      if (px >= GZ_H) px += GZ_TX;
    }
    has_ring = !((px < GZ_H || px >= GZ_H + GZ_TX) && (py < GZ_H || py >= GZ_H + TY));
  }
  __syncthreads();  // planes k0-2 and k0-1 were needed for their centres only
  if (tid == 0) {
    if (k0 + GT_S - 2 <= plast) issue(k0 + GT_S - 2);
    if (k0 + GT_S - 1 <= plast) issue(k0 + GT_S - 1);
  }
  const int pm = periodic_mask(G);
  const int64_t np = G.npts, sz = G.sz;
  const int64_t dy = (int64_t)G.n[1] * G.sy, dz = (int64_t)G.n[2] * sz;
  double ens = 0.0;
  for (int k = k0; k < k1; ++k) {
    const int b = k & 1;
    wait_plane(k + 2);
    double pq[4];
    prims_at(k + 2, ty + GZ_H, tx + GZ_H, pq);
    double pr[4];
    if (has_ring) prims_at(k, py, px, pr);  // plane k arrived two iterations ago
#pragma unroll
    for (int f = 0; f < 4; ++f) {
#pragma unroll
      for (int w = 0; w < 4; ++w) qz[f][w] = qz[f][w + 1];
      qz[f][4] = pq[f];
      S.tile[b][f][ty + GZ_H][tx + GZ_H] = qz[f][2];
      if (has_ring) S.tile[b][f][py][px] = pr[f];
    }
    __syncthreads();
    // every thread is done with raw plane k: its slot takes plane k + S
    if (tid == 0 && k + GT_S <= plast) issue(k + GT_S);
    double gr[3][3], gT[3];
    const int cx = tx + GZ_H, cy = ty + GZ_H;
    double (*tl)[PY][GZ_PX] = S.tile[b];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double gx = cd4v<false>(tl[f][cy][cx - 2], tl[f][cy][cx - 1], tl[f][cy][cx + 1],
                                    tl[f][cy][cx + 2], coef[0]);
      const double gy = cd4v<false>(tl[f][cy - 2][cx], tl[f][cy - 1][cx], tl[f][cy + 1][cx],
                                    tl[f][cy + 2][cx], coef[1]);
      const double gz = cd4v<false>(qz[f][0], qz[f][1], qz[f][3], qz[f][4], coef[2]);
      if (f < 3) {
        gr[f][0] = gx;
        gr[f][1] = gy;
        gr[f][2] = gz;
      } else {
        gT[0] = gx;
        gT[1] = gy;
        gT[2] = gz;
      }
    }
    if constexpr (ENS != 0) ens += enstrophy_point(gr);
    if constexpr (ENS == 2) continue;
    const double vel[3] = {qz[0][2], qz[1][2], qz[2][2]};
    double val[VF_N];
    viscous_flux_point<false>(gr, gT, vel, mu, q_coef, val);
    const int64_t q = G.idx(i, j, k);
    const bool xl = (pm & 1) && i < g, xh = (pm & 1) && i >= G.n[0] - g;
    const bool yl = (pm & 2) && j < g, yh = (pm & 2) && j >= G.n[1] - g;
    const bool zl = (pm & 4) && k < g, zh = (pm & 4) && k >= G.n[2] - g;
#pragma unroll
    for (int f = 0; f < VF_N; ++f) {
      double* F = vf + (int64_t)f * np + q;
      const double v = val[f];
      F[0] = v;
      const int axes = vf_axes(f);
      if (axes & 1) {
        if (xl) F[G.n[0] + G.peer_lo[0]] = v;
        if (xh) F[-G.n[0] + G.peer_hi[0]] = v;
      }
      if (axes & 2) {
        if (yl) F[dy + G.peer_lo[1]] = v;
        if (yh) F[-dy + G.peer_hi[1]] = v;
      }
      if (axes & 4) {
        if (zl) F[dz + G.peer_lo[2]] = v;
        if (zh) F[-dz + G.peer_hi[2]] = v;
      }
    }
  }
  if (ENS != 2 && G.peer_any &&
      ((G.peer[2] && (k0 < G.g || k1 > G.n[2] - G.g)) || touches_peer(G, i, j, G.g)))
    __threadfence_system();
  if constexpr (ENS != 0)
    block_sum_store(ens, ens_partial, ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult st;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &st) != cudaSuccess ||
        st != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)f;
  }();
  return fn;
}

// The state u as a 4D tensor (x, y, z, variable) for TMA; false when the
// geometry or alignment does not allow it (odd extents: 8-byte rows are not
// 16-byte strides)
static bool state_tensor_map(const hd_plan* p, const double* u, int py, CUtensorMap* tm) {
  const Geo& G = p->geo;
  EncodeTiledFn enc = encode_tiled_fn();
  // 16-byte aligned rows and box origins: even ghosted x extent, g odd (origin
  // 32 bx + g - 3 even), 16-byte aligned base
  if (!enc || (G.gn[0] % 2) || ((G.g - 3) % 2) || ((uintptr_t)u % 16)) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)G.gn[0], (cuuint64_t)G.gn[1], (cuuint64_t)G.gn[2], NV};
  const cuuint64_t strides[3] = {(cuuint64_t)G.sy * 8, (cuuint64_t)G.sz * 8, (cuuint64_t)G.npts * 8};
  const cuuint32_t box[4] = {GT_BX, (cuuint32_t)py, 1, NV};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)u, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ENS, class C>
static bool launch_flux_tma_cfg(const hd_plan* p, const double* u, dim3 grid, dim3 block, int zseg,
                                double* partial, cudaStream_t s) {
  CUtensorMap tm;
  if (!state_tensor_map(p, u, C::PY, &tm)) return false;
  // the dynamic shared-memory opt-in is per device context: once per device
  static bool attr[64] = {};
  const int dev = p->device >= 0 && p->device < 64 ? p->device : 0;
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(gradflux_tma_kernel<ENS, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(typename C::Smem)) != cudaSuccess)
      return false;
    attr[dev] = true;
  }
  const double mu = p->phys.mu;
  const double q_coef = (-mu) / ((p->phys.gamma - 1.0) * p->phys.prandtl);  // viscous.py:107
  double* vf = (double*)(p->ws + p->off[HD_BUF_VFLUX]);
  gradflux_tma_kernel<ENS, C><<<grid, block, sizeof(typename C::Smem), s>>>(tm, vf, p->geo, mu, q_coef,
                                                                            zseg, p->phys.gamma, partial);
  return true;
}

static int zm_grid_ty(const hd_plan* p, int ty, int minb, dim3& grid, dim3& block);

// the TMA flux kernel on its own grid (*nblk: the ENS partial count); false when
// the state cannot be mapped (the caller falls back to the register-prefetch kernel)
template <int ENS>
static bool launch_flux_tma(const hd_plan* p, const double* u, double* partial, int64_t* nblk,
                            cudaStream_t s) {
  dim3 grid, block;
  const int zseg = zm_grid_ty(p, GtSmall::TY, GtSmall::MINB, grid, block);
  *nblk = (int64_t)grid.x * grid.y * grid.z;
  if (ENS && *nblk > ens_capacity(p->geom)) return false;
  return launch_flux_tma_cfg<ENS, GtSmall>(p, u, grid, block, zseg, partial, s);
}

// grid of the z-marching flux kernel: enough z segments for ~4 waves of 2 blocks
// per SM; returns the segment length
static int zm_grid_ty(const hd_plan* p, int ty, int minb, dim3& grid, dim3& block) {
  const Geo& G = p->geo;
  const int64_t cols = (int64_t)(G.n[0] / GZ_TX) * (G.n[1] / ty);
  int nseg = (int)((p->sm_count * minb * GZ_WAVES + cols - 1) / cols);
  nseg = nseg < 1 ? 1 : (nseg > G.n[2] ? G.n[2] : nseg);
  const int zseg = (G.n[2] + nseg - 1) / nseg;
  nseg = (G.n[2] + zseg - 1) / zseg;
  block = dim3(GZ_TX, ty, 1);
  grid = dim3(G.n[0] / GZ_TX, G.n[1] / ty, nseg);
  return zseg;
}

static int zm_grid(const hd_plan* p, dim3& grid, dim3& block) {
  return zm_grid_ty(p, GZ_TY, GZ_MINB, grid, block);
}

int launch_enstrophy(const hd_plan* p, const double* u, double* out, cudaStream_t s) {
  const Geo& G = p->geo;
  double* partial = (double*)(p->ws + p->off[HD_BUF_ENS]);
  if (G.n[0] % GZ_TX == 0 && G.n[1] % GZ_TY == 0 && p->opt[HD_OPT_FLUX_ZMARCH]) {
    // the flux kernel's z march without the flux fields: the state read once
    dim3 grid, block;
    const int zseg = zm_grid(p, grid, block);
    const int64_t nblk = (int64_t)grid.x * grid.y * grid.z;
    int64_t tb = 0;
    if (p->opt[HD_OPT_FLUX_TMA] && launch_flux_tma<2>(p, u, partial, &tb, s)) {
      sum_finish_kernel<<<1, 32, 0, s>>>(partial, (int)tb, out);
      hd::count_launches(2);
      return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
    }
    if (nblk <= ens_capacity(p->geom)) {
      gradflux_zm_kernel<false, true, 2><<<grid, block, 0, s>>>(u, nullptr, G, 0.0, 0.0, zseg,
                                                                p->phys.gamma, partial);
      sum_finish_kernel<<<1, 32, 0, s>>>(partial, (int)nblk, out);
      hd::count_launches(2);
      return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
    }
  }
  const int64_t rows = (int64_t)G.n[1] * G.n[2];
  int blocks = (int)((rows + ENS_THREADS / 32 - 1) / (ENS_THREADS / 32));
  if (blocks > ENS_BLOCKS_MAX) blocks = ENS_BLOCKS_MAX;
  enstrophy_kernel<<<blocks, ENS_THREADS, 0, s>>>(u, G, partial);
  sum_finish_kernel<<<1, 32, 0, s>>>(partial, blocks, out);
  hd::count_launches(2);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int launch_gradflux(const hd_plan* p, const double* u, cudaStream_t s, double* ens_out,
                    int* ens_folded) {
  const Geo& G = p->geo;
  if (ens_folded) *ens_folded = 0;
  const double* prim = (const double*)(p->ws + p->off[HD_BUF_PRIM]);
  const bool exact = p->mode == HD_MODE_EXACT;
  double* vf = (double*)(p->ws + p->off[HD_BUF_VFLUX]);
  const double mu = p->phys.mu;
  const double q_coef = (-mu) / ((p->phys.gamma - 1.0) * p->phys.prandtl);  // viscous.py:107
  if (G.n[0] % GZ_TX == 0 && G.n[1] % GZ_TY == 0 && p->opt[HD_OPT_FLUX_ZMARCH]) {
    dim3 grid, block;
    const int zseg = zm_grid(p, grid, block);
    const double gamma = p->phys.gamma;
    const int64_t nblk = (int64_t)grid.x * grid.y * grid.z;
    double* ep = (double*)(p->ws + p->off[HD_BUF_ENS]);
    const bool ens = ens_out && nblk <= ens_capacity(p->geom);
    // fast mode from the state: the TMA-fed kernel when the state maps to a tensor
    int64_t tb = 0;
    if (!exact && u && p->opt[HD_OPT_FLUX_TMA] &&
        (ens_out ? launch_flux_tma<1>(p, u, ep, &tb, s) : launch_flux_tma<0>(p, u, ep, &tb, s))) {
      if (ens_out) {
        sum_finish_kernel<<<1, 32, 0, s>>>(ep, (int)tb, ens_out);
        hd::count_launches(1);
        if (ens_folded) *ens_folded = 1;
      }
      hd::count_launches(1);
      return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
    }
    if (ens) {
      if (exact)
        gradflux_zm_kernel<true, false, 1><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef, zseg, gamma, ep);
      else if (u)
        gradflux_zm_kernel<false, true, 1><<<grid, block, 0, s>>>(u, vf, G, mu, q_coef, zseg, gamma, ep);
      else
        gradflux_zm_kernel<false, false, 1><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef, zseg, gamma, ep);
      sum_finish_kernel<<<1, 32, 0, s>>>(ep, (int)nblk, ens_out);
      hd::count_launches(1);
      if (ens_folded) *ens_folded = 1;
    } else if (exact) {
      gradflux_zm_kernel<true, false, 0><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef, zseg, gamma, ep);
    } else if (u) {
      gradflux_zm_kernel<false, true, 0><<<grid, block, 0, s>>>(u, vf, G, mu, q_coef, zseg, gamma, ep);
    } else {
      gradflux_zm_kernel<false, false, 0><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef, zseg, gamma, ep);
    }
    hd::count_launches(1);
    return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
  }
  if (u && !exact) {  // point-wise fallback reads primitives: make them first
    const int rc = launch_prims(p, u, s);
    if (rc) return rc;
  }
  dim3 block(32, 4, 1), grid((G.n[0] + 31) / 32, (G.n[1] + 3) / 4, G.n[2]);
  if (p->mode == HD_MODE_EXACT)
    gradflux_kernel<true><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef);
  else
    gradflux_kernel<false><<<grid, block, 0, s>>>(prim, vf, G, mu, q_coef);
  hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

// inc_out[r] = ((inc_in[r] + D0 F0[r]) + D1 F1[r]) + D2 F2[r] for the d's in dmask;
// then either store, or apply the RK stage update.
template <bool EXACT>
__global__ void __launch_bounds__(128) divergence_kernel(const double* __restrict__ vf,
                                                         const double* inc_in, double* inc_out,
                                                         Geo G, int dmask, int update, RKArgs r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = blockIdx.z;
  if (i >= G.n[0] || j >= G.n[1]) return;
  const int64_t np = G.npts;
  const int64_t q = G.idx(i, j, k);
  double kv[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) kv[v] = inc_in[q + v * np];
  add_viscous_divergence<EXACT>(vf, G, q, dmask, kv);
  if (update) {
    rk_store<EXACT>(r, G, i, j, k, kv);
    if (G.peer_any && touches_peer(G, i, j, k)) __threadfence_system();
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) inc_out[q + v * np] = kv[v];
  }
}

// Stage states ping-pong between the two halves of the STAGE buffer so a fused
// sweep never overwrites points other threads still read: stage s reads half
// (s-1)%2 (u for s = 0) and writes half s%2; the last stage writes u.
double* stage_buffer(const hd_plan* p, int scheme, int stage, double* u) {
  const int last = (scheme == HD_SCHEME_RK3 ? 3 : 4) - 1;
  if (stage >= last) return u;
  return (double*)(p->ws + p->off[HD_BUF_STAGE]) + (stage % 2) * NV * p->geo.npts;
}

RKArgs make_rk(const hd_plan* p, int scheme, int stage, double* u, const double* dt_dev) {
  RKArgs r;
  r.scheme = scheme;
  r.stage = stage;
  r.u = u;
  r.stage_in = stage == 0 ? u : stage_buffer(p, scheme, stage - 1, u);
  r.stage_out = stage_buffer(p, scheme, stage, u);
  r.acc = (double*)(p->ws + p->off[HD_BUF_ACC]);
  r.dt = dt_dev;
  // fast-mode coefficients of the same tableaux (timeint.py:168-193)
  r.a0 = 1.0; r.a1 = 0.0; r.kc = 0.0; r.ka = 0.0; r.b0 = 0.0; r.b1 = 0.0;
  r.rd_us = 0; r.rd_acc = 0; r.wr_acc = 0; r.to_u = 0;
  if (scheme == HD_SCHEME_RK4) {
    switch (stage) {
      case 0: r.kc = 0.5; r.b1 = 1.0; r.wr_acc = 1; break;                       // acc = k1
      case 1: r.kc = 0.5; r.b0 = 1.0; r.b1 = 2.0; r.rd_acc = r.wr_acc = 1; break;  // acc += 2 k2
      case 2: r.kc = 1.0; r.b0 = 1.0; r.b1 = 2.0; r.rd_acc = r.wr_acc = 1; break;  // acc += 2 k3
      default: r.kc = r.ka = 1.0 / 6.0; r.rd_acc = 1; r.to_u = 1; break;          // u + dt/6 (acc + k4)
    }
  } else {
    switch (stage) {
      case 0: r.kc = 1.0; break;
      case 1: r.a0 = 0.75; r.a1 = 0.25; r.kc = 0.25; r.rd_us = 1; break;
      default: r.a0 = 1.0 / 3.0; r.a1 = 2.0 / 3.0; r.kc = 2.0 / 3.0; r.rd_us = 1; r.to_u = 1; break;
    }
  }
  return r;
}

int launch_divergence(const hd_plan* p, int dims_mask, const double* inc_in, double* inc_out,
                      int update, int scheme, int stage, double* u, const double* dt_dev,
                      cudaStream_t s) {
  const Geo& G = p->geo;
  const double* vf = (const double*)(p->ws + p->off[HD_BUF_VFLUX]);
  RKArgs r = make_rk(p, scheme, stage, u, dt_dev);
  dim3 block(32, 4, 1), grid((G.n[0] + 31) / 32, (G.n[1] + 3) / 4, G.n[2]);
  if (p->mode == HD_MODE_EXACT)
    divergence_kernel<true><<<grid, block, 0, s>>>(vf, inc_in, inc_out, G, dims_mask, update, r);
  else
    divergence_kernel<false><<<grid, block, 0, s>>>(vf, inc_in, inc_out, G, dims_mask, update, r);
  hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int launch_rk_update(const hd_plan* p, const double* inc, int scheme, int stage, double* u,
                     const double* dt_dev, cudaStream_t s) {
  return launch_divergence(p, 0, inc, nullptr, 1, scheme, stage, u, dt_dev, s);
}

// ---------------------------------------------------------------------------
// central_diff4 with the reference's own argument list (kernels.py:207-227)
// ---------------------------------------------------------------------------
__global__ void central_diff4_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                     int di, int dj, int dk, int g, int og, int nx, int ny,
                                     int nz, int k_lo, int k_hi, double coef) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const int k = k_lo + blockIdx.z;
  if (i >= nx || j >= ny || k >= k_hi) return;
  const int64_t sgx = nx + 2 * g, sgy = ny + 2 * g;
  const int64_t dgx = nx + 2 * og, dgy = ny + 2 * og;
  const int64_t c = ((int64_t)(g + k) * sgy + (g + j)) * sgx + (g + i);
  const int64_t st = di + dj * sgx + dk * sgx * sgy;
  dst[((int64_t)(og + k) * dgy + (og + j)) * dgx + (og + i)] = cd4<true>(src + c, st, coef);
}

// ---------------------------------------------------------------------------
// state reduction: CFL signal (max & sum modes), max wavespeed, totals, KE
// ---------------------------------------------------------------------------
constexpr int RED_BLOCKS_MAX = 2048;
constexpr int RED_THREADS = 256;

// EXACT: the reference's true divisions and sqrt (dt bitwise equal to the
// reference); fast: one reciprocal of rho and multiplications by 1/h (dt within
// a few ulp)
template <bool EXACT>
__global__ void __launch_bounds__(RED_THREADS) reduce_kernel(const double* __restrict__ u, Geo G,
                                                             double gamma, double* partial,
                                                             unsigned long long* err, int64_t tag) {
  const int64_t np = G.npts;
  const double ih0 = G.h[0], ih1 = G.h[1], ih2 = G.h[2];
  const double rh0 = 1.0 / G.h[0], rh1 = 1.0 / G.h[1], rh2 = 1.0 / G.h[2];
  double smax = -INFINITY, ssum = -INFINITY, wmax = -INFINITY;
  double sums[6] = {0, 0, 0, 0, 0, 0};
  // one warp per x row (lanes stride x: coalesced, no per-point index division)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rows = (int64_t)G.n[1] * G.n[2];
  const int64_t wstride = (int64_t)gridDim.x * (RED_THREADS / 32);
  for (int64_t r = blockIdx.x * (int64_t)(RED_THREADS / 32) + warp; r < rows; r += wstride) {
  const int64_t row0 = G.idx(0, (int)(r % G.n[1]), (int)(r / G.n[1]));
  for (int i = lane; i < G.n[0]; i += 32) {
    const int64_t q = row0 + i;
    const double rho = u[q], m1 = u[np + q], m2 = u[2 * np + q], m3 = u[3 * np + q],
                 E = u[4 * np + q];
    // physics.py:58-71 cons_to_prim (true division), 87-89 sound speed
    double v0, v1, v2, p, a, s0, s1, s2;
    if constexpr (EXACT) {
      v0 = xd(m1, rho), v1 = xd(m2, rho), v2 = xd(m3, rho);
      const double kin = xm(xm(0.5, rho), xa(xa(xm(v0, v0), xm(v1, v1)), xm(v2, v2)));
      p = xm(gamma - 1.0, xs(E, kin));
      a = xsqrt(xd(xm(gamma, p), rho));
      s0 = xd(xa(fabs(v0), a), ih0), s1 = xd(xa(fabs(v1), a), ih1), s2 = xd(xa(fabs(v2), a), ih2);
    } else {
      const double inv = frcp(rho);
      v0 = m1 * inv, v1 = m2 * inv, v2 = m3 * inv;
      p = (gamma - 1.0) * (E - (0.5 * inv) * (m1 * m1 + m2 * m2 + m3 * m3));
      a = sqrt(gamma * p * inv);
      s0 = (fabs(v0) + a) * rh0, s1 = (fabs(v1) + a) * rh1, s2 = (fabs(v2) + a) * rh2;
    }
    if (!(rho > 0.0)) latch_error(err, tag, 1, q);
    else if (!(p > 0.0)) latch_error(err, tag, 2, q);
    smax = dmax_nan(smax, dmax_nan(dmax_nan(s0, s1), s2));
    ssum = dmax_nan(ssum, xa(xa(s0, s1), s2));
    wmax = dmax_nan(wmax, xa(dmax_nan(dmax_nan(fabs(v0), fabs(v1)), fabs(v2)), a));
    sums[0] += rho;
    sums[1] += m1;
    sums[2] += m2;
    sums[3] += m3;
    sums[4] += E;
    sums[5] += 0.5 * ((v0 * v0 + v1 * v1) + v2 * v2);
  }
  }
  // deterministic block tree: warp shuffles, then warp leaders in order
  __shared__ double sh[RED_THREADS / 32][9];
  double vals[9] = {smax, ssum, wmax, sums[0], sums[1], sums[2], sums[3], sums[4], sums[5]};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) vals[c] = dmax_nan(vals[c], __shfl_down_sync(0xffffffffu, vals[c], off));
#pragma unroll
    for (int c = 3; c < 9; ++c) vals[c] += __shfl_down_sync(0xffffffffu, vals[c], off);
  }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 9; ++c) sh[warp][c] = vals[c];
  __syncthreads();
  if (threadIdx.x == 0) {
    double out[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) out[c] = sh[0][c];
    for (int w = 1; w < RED_THREADS / 32; ++w) {
      for (int c = 0; c < 3; ++c) out[c] = dmax_nan(out[c], sh[w][c]);
      for (int c = 3; c < 9; ++c) out[c] += sh[w][c];
    }
    for (int c = 0; c < 9; ++c) partial[blockIdx.x * 9 + c] = out[c];
  }
}

__global__ void reduce_finish_kernel(const double* partial, int nblocks, double* out) {
  // one warp; fixed order
  const int lane = threadIdx.x;
  double vals[9];
  for (int c = 0; c < 3; ++c) vals[c] = -INFINITY;
  for (int c = 3; c < 9; ++c) vals[c] = 0.0;
  for (int b = lane; b < nblocks; b += 32) {
    for (int c = 0; c < 3; ++c) vals[c] = dmax_nan(vals[c], partial[b * 9 + c]);
    for (int c = 3; c < 9; ++c) vals[c] += partial[b * 9 + c];
  }
  for (int off = 16; off > 0; off >>= 1) {
    for (int c = 0; c < 3; ++c) vals[c] = dmax_nan(vals[c], __shfl_down_sync(0xffffffffu, vals[c], off));
    for (int c = 3; c < 9; ++c) vals[c] += __shfl_down_sync(0xffffffffu, vals[c], off);
  }
  if (lane == 0)
    for (int c = 0; c < 9; ++c) out[c] = vals[c];
}

int launch_reduce_finish(const double* partial, int nparts, double* out, cudaStream_t s) {
  reduce_finish_kernel<<<1, 32, 0, s>>>(partial, nparts, out);
  hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

int64_t fused_red_capacity(const hd_geom& g) {
  // z-sweep warps: (n_x / 32) x n_y lines x segments (make_args caps them at n_z / 8)
  const int64_t seg = g.n[2] / 8 > 1 ? g.n[2] / 8 : 1;
  return (int64_t)((g.n[0] + 31) / 32) * g.n[1] * seg;
}

int launch_reduce(const hd_plan* p, const double* u, double* out, int64_t tag, cudaStream_t s) {
  const Geo& G = p->geo;
  const int64_t rows = (int64_t)G.n[1] * G.n[2];  // one warp per x row
  int blocks = (int)((rows + RED_THREADS / 32 - 1) / (RED_THREADS / 32));
  if (blocks > RED_BLOCKS_MAX) blocks = RED_BLOCKS_MAX;
  double* partial = (double*)(p->ws + p->off[HD_BUF_RED]);
  unsigned long long* err = (unsigned long long*)(p->ws + p->off[HD_BUF_ERR]);
  if (p->mode == HD_MODE_EXACT)
    reduce_kernel<true><<<blocks, RED_THREADS, 0, s>>>(u, G, p->phys.gamma, partial, err, tag);
  else
    reduce_kernel<false><<<blocks, RED_THREADS, 0, s>>>(u, G, p->phys.gamma, partial, err, tag);
  hd::count_launches(1);
  reduce_finish_kernel<<<1, 32, 0, s>>>(partial, blocks, out); hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

// ---------------------------------------------------------------------------
// step bookkeeping (timeint.py:133-138, 224-237)
// ---------------------------------------------------------------------------
__global__ void set_dt_kernel(const double* red, int cfl_mode, double cfl, double dt_fixed,
                              double t_final, double* ctx, unsigned long long* err, int64_t tag) {
  double dt = dt_fixed;
  if (cfl > 0.0) {
    const double sig = red ? red[cfl_mode == 1 ? HD_RED_SIGNAL_SUM : HD_RED_SIGNAL_MAX] : 0.0;
    if (!(isfinite(sig) && sig > 0.0)) {
      latch_error(err, tag, 3, 0);
      dt = 0.0;
    } else {
      dt = __ddiv_rn(cfl, sig);
    }
  }
  if (t_final >= 0.0) dt = fmin(dt, __dsub_rn(t_final, ctx[HD_CTX_T]));
  ctx[HD_CTX_DT] = dt;
}

__global__ void commit_time_kernel(double* ctx) {
  ctx[HD_CTX_T] = __dadd_rn(ctx[HD_CTX_T], ctx[HD_CTX_DT]);
}

__global__ void fp64_probe_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-7;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int it = 0; it < iters; ++it) {
    x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
    x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
}

}  // namespace hd

using namespace hd;

extern "C" int hd_central_diff4(const double* src, double* dst, int di, int dj, int dk, int g,
                                int og, int nx, int ny, int nz, int k_lo, int k_hi, double coef,
                                void* stream) {
  if (!src || !dst || nx < 1 || ny < 1 || nz < 1 || k_hi <= k_lo) return k_hi == k_lo ? HD_OK : HD_E_ARG;
  dim3 block(32, 4, 1), grid((nx + 31) / 32, (ny + 3) / 4, k_hi - k_lo);
  central_diff4_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(src, dst, di, dj, dk, g, og, nx,
                                                                   ny, nz, k_lo, k_hi, coef); hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

extern "C" int hd_set_dt(hd_plan* p, const double* red, int cfl_mode, double cfl, double dt_fixed,
                         double t_final, double* ctx, int64_t tag, void* stream) {
  if (!p || !ctx) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  set_dt_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(
      red, cfl_mode, cfl, dt_fixed, t_final, ctx,
      (unsigned long long*)(p->ws + p->off[HD_BUF_ERR]), tag); hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

extern "C" int hd_commit_time(hd_plan* p, double* ctx, void* stream) {
  if (!p || !ctx) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  commit_time_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(ctx); hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}

extern "C" int hd_fp64_probe(double* out, int blocks, int threads, int iters, void* stream) {
  fp64_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters); hd::count_launches(1);
  return cudaGetLastError() == cudaSuccess ? HD_OK : HD_E_CUDA;
}
