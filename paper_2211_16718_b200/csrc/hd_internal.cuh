// hd_internal.cuh -- shared definitions of the libhd.so kernels (sm_100a).
//
// Arithmetic policies
//   EXACT: every operation is an explicit IEEE round-to-nearest intrinsic
//          (__dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn: never contracted into
//          DFMA) in the reference's association order, so results are
//          bitwise equal to the numba/numpy reference.
//   FAST:  algebraically rearranged (shared smoothness indicators, one
//          reciprocal per reconstruction pair, rsqrt-based Roe averages,
//          DFMA contraction).  Parity bar: 1e-10 relative L2 per conserved
//          variable after N steps (BASELINE.json north_star).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hd.h"

namespace hd {

constexpr int NV = 5;

// weno.py:28-33 literals (Python doubles; constant-folded identically).
constexpr double C13_12 = 13.0 / 12.0;
constexpr double C1_3 = 1.0 / 3.0;
constexpr double C7_6 = 7.0 / 6.0;
constexpr double C11_6 = 11.0 / 6.0;
constexpr double C1_6 = 1.0 / 6.0;
constexpr double C5_6 = 5.0 / 6.0;

// ---- exact IEEE primitives (never fused) --------------------------------------
__device__ __forceinline__ double xa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xs(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xsqrt(double a) { return __dsqrt_rn(a); }

// ---- fast reciprocal: MUFU.RCP64H seed + two Newton steps (~1 ulp) ----------
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Reciprocal for the WENO weight normalisation: one Newton step.  It only
// scales the correction term sum_k w_k (c_k - q2) (recon_pair), so its relative
// error enters the reconstructed value scaled by |c_k - q2| / |q2|.  Measured on
// B200 (tools/gpu/approx_acc.cu, log-uniform inputs): the MUFU seed is good to
// 9.9e-7, one Newton step to 9.9e-13, two to the IEEE result -- which is why the
// flux inputs (frcp) take two.
__device__ __forceinline__ double frcp_weights(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
}

// Geometry of one plan, passed by value to every kernel.
struct Geo {
  int n[3];     // interior extents (x, y, z)
  int gn[3];    // ghosted extents
  int g;
  int64_t npts; // ghosted points per field
  int64_t sy, sz;  // strides of y and z in points (sx = 1)
  double h[3];  // spacing
  int periodic[3];
  // peer images (hd_peer_attach3): per axis, element deltas from a local
  // buffer to the same buffer of the lower / upper neighbour, mapped into this
  // process; peer[d] = 1 when axis d's face images go to the neighbours
  int peer[3];
  int64_t peer_lo[3], peer_hi[3];
  int peer_any;

  __host__ __device__ int64_t idx(int i, int j, int k) const {  // interior coords, may be in ghosts
    return ((int64_t)(k + g) * gn[1] + (j + g)) * gn[0] + (i + g);
  }
  __host__ __device__ int64_t stride(int d) const { return d == 0 ? 1 : (d == 1 ? sy : sz); }
};

// Flat index of the first copy, in C (z, y, x) order over the ghosted box, of
// interior point (i,j,k): along a locally periodic axis the top g layers also
// sit in the low ghost layers.  The reference's decode_primitives checks the
// whole filled box and reports np.argwhere's first hit (physics.py:47-55,
// 240-255), so a stage error latches this index (min over offending points).
__device__ __forceinline__ int64_t first_image(const Geo& G, int i, int j, int k) {
  if (G.periodic[0] && i >= G.n[0] - G.g) i -= G.n[0];
  if (G.periodic[1] && j >= G.n[1] - G.g) j -= G.n[1];
  if (G.periodic[2] && k >= G.n[2] - G.g) k -= G.n[2];
  return G.idx(i, j, k);
}

struct Phys {
  double gamma, gm1, prandtl, mu;  // mu = effective viscosity (mu * visc_scale)
  double eps, delta;
  int power;
};

// Error latch: key = (tag << 36) | (code << 34) | point, min wins; ~0 = none.
__device__ __forceinline__ void latch_error(unsigned long long* key, int64_t tag, int code,
                                            int64_t point) {
  unsigned long long v = ((unsigned long long)tag << 36) | ((unsigned long long)code << 34) |
                         ((unsigned long long)point & ((1ull << 34) - 1));
  atomicMin(key, v);
}

}  // namespace hd

// Host-side plan (opaque to C callers).
struct hd_plan {
  hd_geom geom;
  hd_gas gas;
  hd_weno weno;
  int mode;
  hd::Geo geo;
  hd::Phys phys;
  char* ws;
  int64_t ws_bytes;
  int64_t off[HD_NBUF];
  int device;
  int sm_count;
  void* timer;  // per-kernel event timer (hd_timer_enable), owned
  char* peer_lo[3];  // neighbours' workspaces mapped here (hd_peer_attach3), not owned
  char* peer_hi[3];
  double* red_out;   // armed diagnostics of the next step's result (hd_arm_reduce)
  int64_t red_tag;
  double* ens_out;   // armed enstrophy of the next step's start state (hd_arm_enstrophy)
  int64_t opt[HD_OPT_N];  // hd_plan_set_option
};

namespace hd {
// number of kernels this library has launched (hd_launch_counter)
void count_launches(int n);
// launchers implemented in the .cu files
// occupancy queries behind the sweep segment model, done once per process at plan
// creation (never first inside a stream capture)
void sweep_occupancy_warm();
int launch_sweep(const hd_plan* p, int dim, const double* u, double* inc, int accumulate,
                 int check, int64_t tag, cudaStream_t s);
// fused stage pipeline (fast mode): y sweep + x/y viscous divergence; z sweep +
// z viscous divergence + RK update + primitives of the new stage state
int launch_sweep_visc(const hd_plan* p, const double* u, double* inc, const double* vflux,
                      int64_t tag, cudaStream_t s);
// red_out != nullptr on the last stage: fold the diagnostics of the new state
// in when possible (*fused = 1), else the caller reduces separately
int launch_sweep_update(const hd_plan* p, const double* u_stage, double* inc, const double* vflux,
                        int scheme, int stage, double* u, const double* dt_dev,
                        int64_t tag, cudaStream_t s, double* red_out = nullptr, int64_t red_tag = 0,
                        int* fused = nullptr);
int launch_reduce_finish(const double* partial, int nparts, double* out, cudaStream_t s);
// partial slots of HD_BUF_FRED (one per z-sweep warp of the segment heuristic)
int64_t fused_red_capacity(const hd_geom& g);
int launch_prims_planes(const hd_plan* p, const double* u, int z_lo, int z_hi, cudaStream_t s);
int launch_fill_ghosts(const hd_plan* p, double* f, int nfields, int axis_mask, cudaStream_t s);
int launch_prims(const hd_plan* p, const double* u, cudaStream_t s);
// viscous flux fields; fast mode with u != nullptr derives the primitives from
// the conserved state u on the fly, else they are read from HD_BUF_PRIM.
// ens_out != nullptr: also the enstrophy of that state when the z-marching
// kernel runs (*ens_folded = 1), else the caller runs launch_enstrophy
int launch_gradflux(const hd_plan* p, const double* u, cudaStream_t s, double* ens_out = nullptr,
                    int* ens_folded = nullptr);
// enstrophy sum of a state (ghosts valid) into *out
int launch_enstrophy(const hd_plan* p, const double* u, double* out, cudaStream_t s);
// partial slots of HD_BUF_ENS
int64_t ens_capacity(const hd_geom& g);
// divergence (+ optional RK update).  dims_mask: which d's divergence to add;
// update: 0 = store inc, else RK stage update with scheme/stage.
int launch_divergence(const hd_plan* p, int dims_mask, const double* inc_in, double* inc_out,
                      int update, int scheme, int stage, double* u, const double* dt_dev,
                      cudaStream_t s);
int launch_rk_update(const hd_plan* p, const double* inc, int scheme, int stage, double* u,
                     const double* dt_dev, cudaStream_t s);
int launch_reduce(const hd_plan* p, const double* u, double* out, int64_t tag, cudaStream_t s);
// the buffer holding the output of RK stage `stage` (u for the last one; hd_field.cu)
double* stage_buffer(const hd_plan* p, int scheme, int stage, double* u);
}  // namespace hd
