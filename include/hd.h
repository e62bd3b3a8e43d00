/*
 * hd.h -- C ABI of libhd.so, the B200 (sm_100a) hot path of the hitdns
 * compressible Navier-Stokes solver: WENO5 + Roe hyperbolic sweeps,
 * 4th-order central viscous terms, RK4/RK3 stage updates, CFL and
 * diagnostic reductions.
 *
 * Conventions (identical to the reference FieldSet, pkg/src/hitdns/grid.py:1-21):
 *   - a state is one flat fp64 buffer of 5 * total_points doubles, layout
 *     COMPONENT_CONTIGUOUS (var * total_points + point), x fastest, with
 *     `ghost` ghost layers on each side of each axis;
 *   - variables are [rho, rho*u, rho*v, rho*w, E].
 * All pointers are DEVICE pointers owned by the caller (torch); no call
 * allocates device memory except hd_plan_create (host-side plan struct).
 * Every compute call is asynchronous on the given cudaStream_t (passed as
 * void*, 0 = legacy default stream) and returns 0 or a negative HD_E* code.
 * Invalid states (rho <= 0 or p <= 0, physics.py:47-55) are not returned by
 * the call: they are latched in a device error key read by hd_error_read().
 */
#ifndef HD_H_
#define HD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HD_ABI_VERSION 3

/* status codes */
#define HD_OK 0
#define HD_E_ARG -1      /* bad argument / geometry */
#define HD_E_CUDA -2     /* a CUDA launch or API call failed */
#define HD_E_WORKSPACE -3 /* workspace missing or too small */
#define HD_E_UNSUPPORTED -4

/* arithmetic modes */
#define HD_MODE_FAST 0  /* FMA, one reciprocal per WENO reconstruction, shared betas */
#define HD_MODE_EXACT 1 /* reference operation order, no contraction: bitwise equal to the reference */

/* steppers (timeint.py:196 STEPPERS) */
#define HD_SCHEME_RK3 3
#define HD_SCHEME_RK4 4

/* stage parts (hd_stage_part): one RK stage, split around the halo seam.
 * Call in this order; between LOCAL and HALO the exchanged ghosts of the stage
 * input must arrive (LOCAL reads x ghosts only: a y/z exchange may still be in
 * flight), before MID the x/y ghosts of the viscous flux groups they
 * differentiate, before UPDATE the z ghosts of the z-flux group (fields 5..8
 * of HD_BUF_VFLUX). */
#define HD_PART_LOCAL 1   /* x sweep (exact: + y sweep) */
#define HD_PART_HALO 2    /* exact: z sweep + primitives + viscous fluxes;
                             fast: viscous fluxes from the state (primitives on the fly) */
#define HD_PART_MID 4     /* fast: y sweep + D_x F_x + D_y F_y */
#define HD_PART_UPDATE 8  /* fast: z sweep + D_z F_z + RK update;
                             exact: viscous divergence + RK update */
#define HD_PART_ALL 15

/* plan options (hd_plan_set_option); results never depend on them (tests) */
#define HD_OPT_SEGMENTS 0      /* sweep segments per line: 0 = automatic (>= 6 waves), else fixed */
#define HD_OPT_X_STAGED 1      /* 1 (default): cp.async-staged x sweep when n_y % 32 == 0; 0: plain */
#define HD_OPT_FLUX_ZMARCH 2   /* 1 (default): z-marching viscous flux kernel when the tiles fit; 0: pointwise */
#define HD_OPT_FLUX_TMA 3      /* 1 (default): fast-mode flux kernel fed by TMA when the state maps to a tensor */
#define HD_OPT_SWEEP_WAVES 4   /* automatic sweep segments: 0 (default) = wave-quantisation model; k > 0 = lines x segments >= k waves of 256 threads/SM */
#define HD_OPT_N 5

/* workspace buffers (hd_plan_buffer) */
#define HD_BUF_STAGE 0 /* 10 fields: RK stage states, ping-pong halves (stage s writes half s%2) */
#define HD_BUF_ACC 1   /* 5 fields: RK4 accumulator */
#define HD_BUF_INC 2   /* 5 fields: RHS increment */
#define HD_BUF_PRIM 3  /* 4 fields: u, v, w, T */
#define HD_BUF_VFLUX 4 /* 9 fields: symmetric viscous fluxes tau00 tau01 tau11 w0 w1 | tau02 tau12 tau22 w2 */
#define HD_BUF_RED 5   /* reduction partials + results */
#define HD_BUF_CTX 6   /* step context: t, dt, ... */
#define HD_BUF_ERR 7   /* error key (uint64) */
#define HD_BUF_STATE 8 /* 5 fields: march state of a peer-attached plan (hd_peer_attach) */
#define HD_BUF_SYNC 9  /* 16 uint64: peer flags [axis][state|vflux][from lo|hi], timeout word */
#define HD_BUF_FRED 10 /* per-warp partials of the diagnostics fused into the last z sweep */
#define HD_BUF_ENS 11  /* per-block partials of the enstrophy reduction */
#define HD_NBUF 12

/* results of hd_reduce_state (doubles at HD_BUF_RED result slot) */
#define HD_RED_SIGNAL_MAX 0
#define HD_RED_SIGNAL_SUM 1
#define HD_RED_WAVESPEED 2
#define HD_RED_MASS 3     /* plain sums; multiply by cell volume */
#define HD_RED_MOMX 4
#define HD_RED_MOMY 5
#define HD_RED_MOMZ 6
#define HD_RED_ENERGY 7
#define HD_RED_KE 8       /* sum of 0.5*|m/rho|^2 */
#define HD_RED_ENSTROPHY 9 /* sum of 0.5*|curl(m/rho)|^2 -- written by hd_enstrophy /
                              hd_arm_enstrophy, not by hd_reduce_state */
#define HD_RED_N 10

/* context slots (doubles at HD_BUF_CTX) */
#define HD_CTX_T 0
#define HD_CTX_DT 1
#define HD_CTX_N 4

typedef struct hd_geom {
  int n[3];            /* interior cells per axis (x, y, z) of THIS rank's block */
  double length[3];    /* box length per axis of this block (spacing = length/n) */
  int ghost;           /* ghost width g >= 3 (grid.py:69-70) */
  int periodic[3];     /* 1: axis wraps locally; 0: ghosts come from a halo exchange */
} hd_geom;

typedef struct hd_gas {     /* physics.py:26-44 GasModel */
  double gamma, prandtl, mu, visc_scale;
} hd_gas;

typedef struct hd_weno {    /* weno.py:40-55 WenoParams + entropy-fix delta (kernels.py:60) */
  double epsilon;
  int power;
  double delta;
} hd_weno;

typedef struct hd_plan hd_plan;

int hd_abi_version(void);
const char* hd_status_string(int status);

/* Workspace bytes a plan needs (stage/acc/inc/prims/viscous fluxes/reductions). */
int64_t hd_workspace_bytes(const hd_geom* geom);

/* Create a plan on the current device.  `workspace` (device, >= hd_workspace_bytes,
 * 256-byte aligned) stays owned by the caller and must outlive the plan. */
int hd_plan_create(const hd_geom* geom, const hd_gas* gas, const hd_weno* weno, int mode,
                   void* workspace, int64_t workspace_bytes, hd_plan** out);
int hd_plan_destroy(hd_plan* plan);
/* Set a kernel-selection option (HD_OPT_*) of a plan; applies to later launches. */
int hd_plan_set_option(hd_plan* plan, int option, int64_t value);
/* Device pointer of a workspace buffer (HD_BUF_*). */
void* hd_plan_buffer(hd_plan* plan, int which);
int64_t hd_plan_total_points(const hd_plan* plan);

/* ---- field-level operators (reference public API) -------------------------- */

/* grid.py:236-251 fill_ghosts_periodic / fill_ghosts_array: periodic wrap of
 * `nfields` consecutive fields along the plan's locally periodic axes. */
int hd_fill_ghosts(hd_plan* plan, double* fields, int nfields, void* stream);

/* kernels.py:68-204 hyper_sweep over every interior line along `dim`, with the
 * flux components of upwind.py:116-127 formed on the fly from u.
 * accumulate=1: inc -= dF/dx; accumulate=0: inc = 0 - dF/dx (interior only). */
int hd_hyper_sweep(hd_plan* plan, int dim, const double* u, double* inc, int accumulate,
                   void* stream);

/* kernels.py:68-73 hyper_sweep with the reference's exact argument list, on device
 * buffers: accumulates -dF/dx of dimension `dim` into inc for the slab of lines
 * [a_lo, a_hi) x [0, nb) (line origin base0 + ia*sa + ib*sb, stride sd, nd cells),
 * reconstructing the caller's flux array f (upwind.py:116-127).  Exact IEEE
 * arithmetic, bitwise equal to the numba kernel: the one-for-one replacement
 * inside the reference's run_slabs loop (upwind.py:185-212). */
int hd_hyper_sweep_lines(const double* u, const double* f, double* inc, int64_t npts, int64_t base0,
                         int64_t sd, int64_t sa, int64_t sb, int64_t nd, int64_t nb, int64_t a_lo,
                         int64_t a_hi, int dim, double inv_dx, double gamma, double eps, int power,
                         double delta, void* stream);

/* upwind.py:163-213 hyperbolic_rhs: x, y, z sweeps; also latches positivity. */
int hd_hyperbolic_rhs(hd_plan* plan, const double* u, double* inc, int accumulate, void* stream);

/* viscous.py:54-121 parabolic_rhs: accumulates into inc rows 1..4. */
int hd_parabolic_rhs(hd_plan* plan, const double* u, double* inc, void* stream);
/* hd_parabolic_rhs in two halves around the flux-field halo of a decomposed
 * block (viscous.py:111-120, the sync_scalars of RankHalo): the 9 symmetric
 * viscous flux fields into HD_BUF_VFLUX (face images along the periodic axes),
 * then inc[1..4] += their divergence in the reference order. */
int hd_viscous_fluxes(hd_plan* plan, const double* u, void* stream);
int hd_viscous_divergence(hd_plan* plan, double* inc, void* stream);

/* kernels.py:207-227 central_diff4, same argument list. */
int hd_central_diff4(const double* src, double* dst, int di, int dj, int dk, int g, int og,
                     int nx, int ny, int nz, int k_lo, int k_hi, double coef, void* stream);

/* timeint.py:152-156 rhs(u): ghost fill of u, then hyperbolic + parabolic into inc. */
int hd_rhs(hd_plan* plan, double* u, double* inc, void* stream);

/* ---- steppers --------------------------------------------------------------- */

/* One full step (timeint.py:181-193 rk4_step / 168-178 rk3_tvd_step), u in
 * place, dt read from device memory.  Ghosts of u must be valid on entry and
 * are valid on exit (locally periodic axes).  `tag` identifies the step in
 * the error key. */
int hd_step(hd_plan* plan, int scheme, double* u, const double* dt_dev, int64_t tag, void* stream);

/* One part of one RK stage (decomposed runs).  Stage s reads u (s == 0) or
 * half (s-1)%2 of the workspace STAGE buffer; the UPDATE part writes the next
 * stage state into half s%2 (or u itself after the last stage). */
int hd_stage_part(hd_plan* plan, int scheme, int stage, int parts, double* u,
                  const double* dt_dev, int64_t tag, void* stream);

/* ---- reductions and step bookkeeping --------------------------------------- */

/* timeint.py:100-131: one pass over the interior producing HD_RED_* results
 * at `out` (device, HD_RED_N doubles).  Latches positivity (cons_to_prim). */
int hd_reduce_state(hd_plan* plan, const double* u, double* out, int64_t tag, void* stream);

/* Arm the diagnostics of the state the next completed step produces: the last
 * RK stage's UPDATE (hd_step or hd_stage_part) writes the hd_reduce_state
 * results of the new state to `out` with error tag `tag` -- folded into the z
 * sweep in fast mode (no extra pass over the state), a separate reduction
 * otherwise.  One-shot. */
int hd_arm_reduce(hd_plan* plan, double* out, int64_t tag);

/* Enstrophy of a state (the north star's third diagnostic; the reference has
 * none -- its operators define it): velocities decoded as physics.py:249-252
 * (v = m * (1/rho)), the 9 velocity gradients by the 4th-order central
 * difference of viscous.py:23-51, out[0] = sum over the interior of
 * 0.5 * |curl v|^2 (divide by the point count for the mean).  Ghosts of u
 * must be valid along every axis (faces only).  Deterministic order. */
int hd_enstrophy(hd_plan* plan, const double* u, double* out, void* stream);
/* One-shot: the next stage-0 HALO part (hd_step / hd_stage_part) writes the
 * enstrophy of its input state -- the state the step starts from -- to
 * `out`, folded into the viscous flux kernel that already forms those
 * gradients (fast and exact mode, mu > 0), else a separate hd_enstrophy pass. */
int hd_arm_enstrophy(hd_plan* plan, double* out);

/* timeint.py:133-138 + 224-237: ctx[DT] = cfl / signal (cfl > 0) or dt_fixed,
 * clipped to t_final - ctx[T] when t_final >= 0.  Latches a zero/non-finite
 * signal.  signal = red[HD_RED_SIGNAL_MAX] or [SUM] per cfl_mode (0/1). */
int hd_set_dt(hd_plan* plan, const double* red, int cfl_mode, double cfl, double dt_fixed,
              double t_final, double* ctx, int64_t tag, void* stream);
/* ctx[T] += ctx[DT] */
int hd_commit_time(hd_plan* plan, double* ctx, void* stream);

/* ---- errors ----------------------------------------------------------------- */

/* Error key: 0 = none, else (tag << 36) | (code << 34) | flat point index;
 * the smallest key wins (earliest tag, density before pressure, lowest index).
 * code 1 = nonpositive density, 2 = nonpositive pressure, 3 = bad CFL signal.
 * tag = step * 8 + slot: hd_step/hd_stage_part latch slot 1 + stage with
 * their `tag` argument as the step; hd_reduce_state / hd_set_dt latch their
 * `tag` verbatim (callers use slot 0 before a step, 7 after it). */
int hd_error_read(hd_plan* plan, uint64_t* key, void* stream);
int hd_error_clear(hd_plan* plan, void* stream);

/* ---- per-kernel timing ------------------------------------------------------- */
/* With the timer on, every launch of the stage pipeline and of hd_reduce_state is
 * bracketed by CUDA events on its stream; hd_timer_read synchronises, returns the
 * summed milliseconds and launch counts per kind (HD_TK_*) and resets. */
#define HD_TK_SWEEP_X 0
#define HD_TK_SWEEP_Y 1
#define HD_TK_SWEEP_Z 2
#define HD_TK_GRADFLUX 3
#define HD_TK_PRIMS 4
#define HD_TK_DIVERGENCE 5
#define HD_TK_REDUCE 6
#define HD_TK_N 7
int hd_timer_enable(hd_plan* plan, int on);
int hd_timer_read(hd_plan* plan, double* ms, int64_t* count, int nkinds);

/* Kernels launched by this library since load (monotonic; for launch accounting). */
int64_t hd_launch_counter(void);

/* ---- microbenchmark ---------------------------------------------------------- */
/* FP64 FMA throughput probe: iters DFMA per thread on `out` (blocks x threads). */
int hd_fp64_probe(double* out, int blocks, int threads, int iters, void* stream);

/* Device pointer of the buffer that receives the output of RK stage `stage`
 * (5 fields, ghosted; `u` for the last stage), i.e. the input of stage+1 --
 * what a decomposed driver exchanges between the stage parts. */
int hd_stage_buffer(hd_plan* plan, int scheme, int stage, double* u, void** out);

/* ---- single-operation entry points (the names of SURVEY.md 8b) --------------- */
/* classical RK4 step (timeint.py:181-193) = hd_step(plan, HD_SCHEME_RK4, u, dt, 0, 0). */
int hd_rk4_step(hd_plan* plan, double* u, const double* dt_dev, void* stream);
/* CFL signal of the interior (timeint.py:122-131) into out_dev[0]: mode 0 = max
 * over points and directions of (|v_d| + a)/h_d, 1 = max of the sum over d. */
int hd_max_signal(hd_plan* plan, const double* u, double* out_dev, int mode, void* stream);
/* Volume-weighted mass, momentum (3), energy (timeint.py:100-107) into out5_dev. */
int hd_totals(hd_plan* plan, const double* u, double* out5_dev, void* stream);
/* The latched error as flags: bit0 nonpositive density, bit1 nonpositive
 * pressure, bit2 bad CFL signal; *where = flat point index (or -1). */
int hd_error_flags(hd_plan* plan, int* flags, int64_t* where, void* stream);
/* Ghost layers of `fields` (nfields x total points): periodic axes wrap
 * (grid.py:236-251); on a peer-attached plan the boundary layers along the
 * split axes are stored into the neighbours' ghost layers (`fields` must be a
 * buffer of the plan workspace; order it with hd_peer_signal / hd_peer_wait). */
int hd_halo_exchange(hd_plan* plan, double* fields, int nfields, void* stream);

/* ---- peer halo over NVLink (block decompositions, one process per GPU) ------
 * Replaces the face exchange of the reference's RankHalo (decomp.py:183-241)
 * for a plan whose split axes are not periodic: with the workspaces of the
 * lower and upper neighbours along every split axis mapped into this process
 * (hd_ipc_open of their hd_ipc_handle), every kernel that writes a stage state
 * or a viscous flux field stores the values of its g boundary layers straight
 * into the neighbours' ghost layers (peer stores over NVLink; the same index
 * deltas as the periodic images).  Requires the march state to live in
 * HD_BUF_STATE.  Protocol per RK stage with a counter v (1, 2, ...), z split:
 *   LOCAL; hd_peer_wait(STATE, v-1); HALO; hd_peer_signal(VFLUX, v); MID;
 *   hd_peer_wait(VFLUX, v); UPDATE; hd_peer_signal(STATE, v)
 * -- the STATE wait before LOCAL when x is split, the VFLUX wait before MID
 * when x or y is split (the two halves of HD_BUF_STAGE make every
 * write-after-read safe). */
#define HD_PEER_STATE 0
#define HD_PEER_VFLUX 1
/* 64-byte IPC handle + byte offset of `ptr` inside its allocation. */
int hd_ipc_handle(const void* ptr, void* handle64, int64_t* offset);
/* Map a peer allocation (handle from hd_ipc_handle) into this process: *ptr =
 * mapped base + offset. */
int hd_ipc_open(const void* handle64, int64_t offset, void** ptr);
/* Unmap (pass the pointer hd_ipc_open returned and its offset). */
int hd_ipc_close(void* ptr, int64_t offset);
/* lo_ws[d] / hi_ws[d]: the neighbours' workspaces along axis d as mapped here
 * (may be equal: two blocks along d), NULL for an axis that is not split (it
 * must then be periodic); all NULL detaches.  Zeroes this plan's flags (call
 * before any peer can signal, then barrier). */
int hd_peer_attach3(hd_plan* plan, void* const* lo_ws, void* const* hi_ws, void* stream);
/* z slabs only: hd_peer_attach3 with lo/hi along z. */
int hd_peer_attach(hd_plan* plan, void* lo_ws, void* hi_ws, void* stream);
int hd_peer_signal(hd_plan* plan, int which, int64_t value, void* stream);
/* Stream waits until every neighbour signalled >= value (spins at most
 * ~30 s, then sets the timeout word of HD_BUF_SYNC and lets the stream go). */
int hd_peer_wait(hd_plan* plan, int which, int64_t value, void* stream);
/* 1 if a wait timed out since the attach. */
int hd_peer_timed_out(hd_plan* plan, int* out, void* stream);

/* Layout / traversal study (replaces kernels.py:292-329 bench_weights_lex /
 * bench_weights_tiled, driven by bench.py:102-140 run_case).  `data` holds the
 * (nx + 2 pad) * ny * nz points x 5 variables per `layout` (0 = INTERLEAVED,
 * 1 = COMPONENT_CONTIGUOUS, grid.py Layout); the three WENO weights of every
 * variable of every active point go to out[3 * (5 p + v) + 0..2] (point-major,
 * so all combinations are bitwise comparable).  traversal 0 = lexicographic
 * (one thread per active point, x fastest), 1 = (tx, ty) tiles per z plane;
 * *wasted = idle lanes of the tiling (0 for lex).  Async on `stream`. */
int hd_bench_weights(const double* data, int layout, int traversal, int nx, int ny, int nz, int pad,
                     int tx, int ty, double eps, int power, double* out, int64_t* wasted,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HD_H_ */
