// hd_api.cu -- extern "C" boundary of libhd.so (declared in include/hd.h).
//
// The reference's seams this boundary replaces (pkg/src/hitdns/):
//   hd_hyper_sweep     kernels.py:68-73   hyper_sweep(u, f, inc, ...)
//   hd_central_diff4   kernels.py:207-208 central_diff4(src, dst, ...)
//   hd_hyperbolic_rhs  upwind.py:163-170  hyperbolic_rhs(fields, gas, params, delta, workers, out)
//   hd_parabolic_rhs   viscous.py:54-60   parabolic_rhs(fields, gas, halo, workers, out)
//   hd_rhs             timeint.py:141-158 make_rhs(...) -> rhs(fields)
//   hd_step            timeint.py:168-193 rk3_tvd_step / rk4_step (STEPPERS, :196)
//   hd_stage_part      the same stages split around the halo seam grid.py:254-267 /
//                      decomp.py:183-241 (sync_fields / sync_scalars)
//   hd_reduce_state    timeint.py:100-131 conserved_totals / max_wavespeed_interior / max_signal
//   hd_set_dt          timeint.py:133-138 compute_dt + the t_final clip of :236-237
//   hd_fill_ghosts     grid.py:236-251    fill_ghosts_periodic / fill_ghosts_array
#include <atomic>
#include <cstring>
#include <new>
#include <utility>
#include <vector>

#include "hd_internal.cuh"

using namespace hd;

namespace {

std::atomic<int64_t> g_launches{0};
int64_t hd_launches_total() { return g_launches.load(); }

constexpr int64_t ALIGN = 256;
constexpr int64_t RED_BYTES = (2048 * 9 + 16) * 8;

int64_t align_up(int64_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

bool geom_ok(const hd_geom* g) {
  if (!g || g->ghost < 3) return false;
  for (int d = 0; d < 3; ++d) {
    if (g->n[d] < 1 || !(g->length[d] > 0.0)) return false;
    if (g->n[d] < g->ghost) return false;  // decomp.py:78-82 (local extent >= ghost width)
  }
  return true;
}

int64_t npts_of(const hd_geom* g) {
  return (int64_t)(g->n[0] + 2 * g->ghost) * (g->n[1] + 2 * g->ghost) * (g->n[2] + 2 * g->ghost);
}

void layout(const hd_geom* g, int64_t off[HD_NBUF], int64_t* total) {
  const int64_t f = npts_of(g) * 8;
  int64_t o = 0;
  const int64_t sizes[HD_NBUF] = {10 * f, 5 * f, 5 * f, 4 * f, 9 * f, RED_BYTES, 8 * HD_CTX_N, 64,
                                  5 * f, 128, fused_red_capacity(*g) * 9 * 8, ens_capacity(*g) * 8};
  for (int b = 0; b < HD_NBUF; ++b) {
    off[b] = o;
    o = align_up(o + sizes[b]);
  }
  *total = o;
}

cudaStream_t S(void* s) { return (cudaStream_t)s; }

double* buf(hd_plan* p, int which) { return (double*)(p->ws + p->off[which]); }

// exchanged axes must be a suffix (z, or y+z) so the exact accumulation order
// x, y, z of upwind.py:200 is kept when the local sweeps run first
bool parts_supported(const hd_plan* p) {
  const int* per = p->geo.periodic;
  if (!per[0] && (per[1] || per[2])) return false;
  if (!per[1] && per[2]) return false;
  return true;
}


// sweeps for the dims in `dmask`, in x, y, z order; the first sweep of the
// RHS overwrites inc (0 - d, upwind.py:181-182) unless `accumulate_first`.
int sweeps(hd_plan* p, int dmask, const double* us, double* inc, bool first_overwrites, int64_t tag,
           cudaStream_t s) {
  bool first = first_overwrites;
  for (int d = 0; d < 3; ++d) {
    if (!(dmask & (1 << d))) continue;
    int rc = launch_sweep(p, d, us, inc, first ? 0 : 1, d == 0 ? 1 : 0, tag, s);
    if (rc) return rc;
    first = false;
  }
  return HD_OK;
}

int nstages(int scheme) { return scheme == HD_SCHEME_RK3 ? 3 : 4; }

void timer_free(void* t);  // defined with the Timer below

// stage s > 0 reads the output buffer of stage s-1 (hd_field.cu stage_buffer)
const double* stage_input(hd_plan* p, int scheme, int stage, double* u) {
  return stage == 0 ? u : stage_buffer(p, scheme, stage - 1, u);
}

}  // namespace

extern "C" {

int hd_abi_version(void) { return HD_ABI_VERSION; }

int64_t hd_launch_counter(void) { return hd_launches_total(); }

const char* hd_status_string(int status) {
  switch (status) {
    case HD_OK: return "ok";
    case HD_E_ARG: return "invalid argument";
    case HD_E_CUDA: return "CUDA error";
    case HD_E_WORKSPACE: return "workspace missing or too small";
    case HD_E_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

int64_t hd_workspace_bytes(const hd_geom* geom) {
  if (!geom_ok(geom)) return HD_E_ARG;
  int64_t off[HD_NBUF], total;
  layout(geom, off, &total);
  return total;
}

int hd_plan_create(const hd_geom* geom, const hd_gas* gas, const hd_weno* weno, int mode,
                   void* workspace, int64_t workspace_bytes, hd_plan** out) {
  if (!out) return HD_E_ARG;
  *out = nullptr;
  if (!geom_ok(geom) || !gas || !weno) return HD_E_ARG;
  if (!(gas->gamma > 1.0) || !(gas->prandtl > 0.0) || gas->mu < 0.0) return HD_E_ARG;
  if (!(weno->epsilon > 0.0) || weno->power < 1) return HD_E_ARG;
  if (mode != HD_MODE_FAST && mode != HD_MODE_EXACT) return HD_E_ARG;
  int64_t off[HD_NBUF], total;
  layout(geom, off, &total);
  // workspace == NULL: geometry-only plan (ghost fills); compute calls then fail
  if (workspace && (workspace_bytes < total || ((uintptr_t)workspace % ALIGN))) return HD_E_WORKSPACE;
  hd_plan* p = new (std::nothrow) hd_plan;
  if (!p) return HD_E_ARG;
  std::memset(p, 0, sizeof(*p));
  p->geom = *geom;
  p->gas = *gas;
  p->weno = *weno;
  p->mode = mode;
  Geo& G = p->geo;
  G.g = geom->ghost;
  for (int d = 0; d < 3; ++d) {
    G.n[d] = geom->n[d];
    G.gn[d] = geom->n[d] + 2 * geom->ghost;
    G.h[d] = geom->length[d] / (double)geom->n[d];  // grid.py:73-74
    G.periodic[d] = geom->periodic[d] ? 1 : 0;
  }
  G.npts = npts_of(geom);
  G.sy = G.gn[0];
  G.sz = (int64_t)G.gn[0] * G.gn[1];
  Phys& ph = p->phys;
  ph.gamma = gas->gamma;
  ph.gm1 = gas->gamma - 1.0;
  ph.prandtl = gas->prandtl;
  ph.mu = gas->mu * gas->visc_scale;  // physics.py:42-44 effective_mu
  ph.eps = weno->epsilon;
  ph.power = weno->power;
  ph.delta = weno->delta;
  p->ws = (char*)workspace;
  p->ws_bytes = workspace_bytes;
  p->opt[HD_OPT_SEGMENTS] = 0;
  p->opt[HD_OPT_X_STAGED] = 1;
  p->opt[HD_OPT_FLUX_ZMARCH] = 1;
  p->opt[HD_OPT_FLUX_TMA] = 1;
  p->opt[HD_OPT_SWEEP_WAVES] = 0;  // 0: the wave-quantisation model (hd_sweep.cu)
  std::memcpy(p->off, off, sizeof(off));
  if (cudaGetDevice(&p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) {
    delete p;
    return HD_E_CUDA;
  }
  sweep_occupancy_warm();
  // error key starts at "none"; context zeroed
  if (p->ws && (cudaMemset(p->ws + p->off[HD_BUF_ERR], 0xff, 8) != cudaSuccess ||
      cudaMemset(p->ws + p->off[HD_BUF_CTX], 0, 8 * HD_CTX_N) != cudaSuccess)) {
    delete p;
    return HD_E_CUDA;
  }
  *out = p;
  return HD_OK;
}

int hd_plan_destroy(hd_plan* p) {
  if (p) timer_free(p->timer);
  delete p;
  return HD_OK;
}

int hd_plan_set_option(hd_plan* p, int option, int64_t value) {
  if (!p || option < 0 || option >= HD_OPT_N || value < 0) return HD_E_ARG;
  p->opt[option] = value;
  return HD_OK;
}

void* hd_plan_buffer(hd_plan* p, int which) {
  if (!p || !p->ws || which < 0 || which >= HD_NBUF) return nullptr;
  return p->ws + p->off[which];
}

int64_t hd_plan_total_points(const hd_plan* p) { return p ? p->geo.npts : HD_E_ARG; }

int hd_fill_ghosts(hd_plan* p, double* fields, int nfields, void* stream) {
  if (!p || !fields || nfields < 1) return HD_E_ARG;
  return launch_fill_ghosts(p, fields, nfields, 7, S(stream));
}

int hd_hyper_sweep(hd_plan* p, int dim, const double* u, double* inc, int accumulate, void* stream) {
  if (!p || !u || !inc || dim < 0 || dim > 2) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  return launch_sweep(p, dim, u, inc, accumulate ? 1 : 0, 0, 0, S(stream));
}

int hd_hyperbolic_rhs(hd_plan* p, const double* u, double* inc, int accumulate, void* stream) {
  if (!p || !u || !inc) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  return sweeps(p, 7, u, inc, !accumulate, 0, S(stream));
}

int hd_parabolic_rhs(hd_plan* p, const double* u, double* inc, void* stream) {
  if (!p || !u || !inc) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (p->phys.mu == 0.0) return HD_OK;  // viscous.py:72-73
  if (!parts_supported(p)) return HD_E_UNSUPPORTED;
  int rc = launch_prims(p, u, S(stream));
  if (!rc) rc = launch_gradflux(p, nullptr, S(stream));
  if (!rc) rc = launch_divergence(p, 7, inc, inc, 0, HD_SCHEME_RK4, 0, nullptr, nullptr, S(stream));
  return rc;
}

int hd_viscous_fluxes(hd_plan* p, const double* u, void* stream) {
  if (!p || !u) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (p->phys.mu == 0.0) return HD_OK;
  int rc = launch_prims(p, u, S(stream));
  if (!rc) rc = launch_gradflux(p, nullptr, S(stream));
  return rc;
}

int hd_viscous_divergence(hd_plan* p, double* inc, void* stream) {
  if (!p || !inc) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (p->phys.mu == 0.0) return HD_OK;
  return launch_divergence(p, 7, inc, inc, 0, HD_SCHEME_RK4, 0, nullptr, nullptr, S(stream));
}

int hd_rhs(hd_plan* p, double* u, double* inc, void* stream) {
  if (!p || !u || !inc) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  int rc = launch_fill_ghosts(p, u, 5, 7, S(stream));
  if (!rc) rc = sweeps(p, 7, u, inc, true, 0, S(stream));
  if (!rc) rc = hd_parabolic_rhs(p, u, inc, stream);
  return rc;
}

}  // extern "C"

// ---- per-kernel event timer (hd_timer_*): event pairs around each launch of the
// stage pipeline, summed per kernel kind on read.  Off by default (zero cost).
namespace {
struct Timer {
  bool on = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> used;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  ~Timer() {
    for (auto& u : used) {
      cudaEventDestroy(u.second.first);
      cudaEventDestroy(u.second.second);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};
Timer* timer_of(hd_plan* p) { return (Timer*)p->timer; }
void timer_free(void* t) { delete (Timer*)t; }

// run launch expression `fn` bracketed by events when the timer is on
template <class F>
int timed(hd_plan* p, int kind, cudaStream_t s, F fn) {
  Timer* t = timer_of(p);
  if (!t || !t->on) return fn();
  cudaEvent_t a = t->take(), b = t->take();
  cudaEventRecord(a, s);
  const int rc = fn();
  cudaEventRecord(b, s);
  t->used.push_back({kind, {a, b}});
  return rc;
}
}  // namespace

extern "C" {

int hd_timer_enable(hd_plan* p, int on) {
  if (!p) return HD_E_ARG;
  if (!p->timer) p->timer = new (std::nothrow) Timer;
  if (!p->timer) return HD_E_ARG;
  timer_of(p)->on = on != 0;
  return HD_OK;
}

int hd_timer_read(hd_plan* p, double* ms, int64_t* count, int nkinds) {
  if (!p || !ms || !count || nkinds < HD_TK_N) return HD_E_ARG;
  for (int k = 0; k < nkinds; ++k) {
    ms[k] = 0.0;
    count[k] = 0;
  }
  Timer* t = timer_of(p);
  if (!t) return HD_OK;
  for (auto& u : t->used) {
    if (cudaEventSynchronize(u.second.second) != cudaSuccess) return HD_E_CUDA;
    float f = 0.0f;
    cudaEventElapsedTime(&f, u.second.first, u.second.second);
    ms[u.first] += f;
    count[u.first] += 1;
    t->pool.push_back(u.second.first);
    t->pool.push_back(u.second.second);
  }
  t->used.clear();
  return HD_OK;
}

int hd_stage_part(hd_plan* p, int scheme, int stage, int parts, double* u, const double* dt_dev,
                  int64_t tag, void* stream) {
  if (!p || !u || (scheme != HD_SCHEME_RK3 && scheme != HD_SCHEME_RK4)) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (stage < 0 || stage >= nstages(scheme)) return HD_E_ARG;
  cudaStream_t s = S(stream);
  const double* us = stage_input(p, scheme, stage, u);
  double* inc = buf(p, HD_BUF_INC);
  const bool visc = p->phys.mu != 0.0;
  const int64_t t = tag * 8 + 1 + stage;  // slot 1..4: RK stage (0 = pre-step CFL, 7 = diagnostics)
  int rc = HD_OK;
  const bool exact = p->mode == HD_MODE_EXACT;
  double* vflux = visc ? buf(p, HD_BUF_VFLUX) : nullptr;
  // LOCAL: sweeps that read no z ghosts (a z-halo exchange of `us` can be in flight)
  if (parts & HD_PART_LOCAL) {
    rc = timed(p, HD_TK_SWEEP_X, s, [&] { return launch_sweep(p, 0, us, inc, 0, 1, t, s); });
    if (!rc && exact)
      rc = timed(p, HD_TK_SWEEP_Y, s, [&] { return launch_sweep(p, 1, us, inc, 1, 0, t, s); });
  }
  // HALO (reads every ghost of `us`)
  //   exact: z sweep, primitives of the whole box, viscous fluxes
  //   fast:  viscous fluxes straight from the state (primitives on the fly)
  // Stage 0 folds an armed enstrophy of its input (the step's start state) into
  // the flux kernel, which forms the velocity gradients anyway (hd_arm_enstrophy).
  if (!rc && (parts & HD_PART_HALO)) {
    double* ens = stage == 0 ? p->ens_out : nullptr;
    int folded = 0;
    if (exact) {
      rc = timed(p, HD_TK_SWEEP_Z, s, [&] { return launch_sweep(p, 2, us, inc, 1, 0, t, s); });
      if (!rc && visc) rc = timed(p, HD_TK_PRIMS, s, [&] { return launch_prims(p, us, s); });
      if (!rc && visc)
        rc = timed(p, HD_TK_GRADFLUX, s, [&] { return launch_gradflux(p, nullptr, s, ens, &folded); });
    } else if (visc) {
      rc = timed(p, HD_TK_GRADFLUX, s, [&] { return launch_gradflux(p, us, s, ens, &folded); });
    }
    if (!rc && ens && !folded)
      rc = timed(p, HD_TK_REDUCE, s, [&] { return launch_enstrophy(p, us, ens, s); });
    if (stage == 0) p->ens_out = nullptr;
  }
  // MID (fast): y sweep + D_x F_x + D_y F_y (no z ghosts of the fluxes read)
  if (!rc && (parts & HD_PART_MID) && !exact)
    rc = timed(p, HD_TK_SWEEP_Y, s, [&] { return launch_sweep_visc(p, us, inc, vflux, t, s); });
  // UPDATE (reads the z ghosts of the viscous z-flux group)
  //   exact: divergence in the viscous.py:112-120 order + RK update
  //   fast:  z sweep + D_z F_z + RK update
  if (!rc && (parts & HD_PART_UPDATE)) {
    if (!dt_dev) return HD_E_ARG;
    const bool last = stage == nstages(scheme) - 1;
    int fused = 0;
    // peer mode: the final stage's images land in the neighbours' HD_BUF_STATE
    if (p->geo.peer_any && u != buf(p, HD_BUF_STATE)) return HD_E_ARG;
    if (exact)
      rc = timed(p, HD_TK_DIVERGENCE, s, [&] {
        return launch_divergence(p, visc ? 7 : 0, inc, nullptr, 1, scheme, stage, u, dt_dev, s);
      });
    else
      rc = timed(p, HD_TK_SWEEP_Z, s, [&] {
        return launch_sweep_update(p, us, inc, vflux, scheme, stage, u, dt_dev, t, s,
                                   last ? p->red_out : nullptr, p->red_tag, &fused);
      });
    // armed diagnostics of the step's result that the update could not fold in
    if (!rc && last && p->red_out && !fused)
      rc = timed(p, HD_TK_REDUCE, s, [&] { return launch_reduce(p, u, p->red_out, p->red_tag, s); });
    if (last) p->red_out = nullptr;
  }
  return rc;
}

int hd_step(hd_plan* p, int scheme, double* u, const double* dt_dev, int64_t tag, void* stream) {
  if (!p || !u || !dt_dev) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (scheme != HD_SCHEME_RK3 && scheme != HD_SCHEME_RK4) return HD_E_ARG;
  for (int d = 0; d < 3; ++d)
    if (!p->geo.periodic[d]) return HD_E_UNSUPPORTED;  // decomposed runs use hd_stage_part
  // timeint.py:153: the rhs syncs the ghosts of its input first
  int rc = launch_fill_ghosts(p, u, 5, 7, S(stream));
  for (int st = 0; st < nstages(scheme) && !rc; ++st) {
    rc = hd_stage_part(p, scheme, st, HD_PART_ALL, u, dt_dev, tag, stream);
  }
  return rc;
}

int hd_arm_reduce(hd_plan* p, double* out, int64_t tag) {
  if (!p) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  p->red_out = out;
  p->red_tag = tag;
  return HD_OK;
}

int hd_arm_enstrophy(hd_plan* p, double* out) {
  if (!p) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  p->ens_out = out;
  return HD_OK;
}

int hd_enstrophy(hd_plan* p, const double* u, double* out, void* stream) {
  if (!p || !u || !out) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  return timed(p, HD_TK_REDUCE, S(stream), [&] { return launch_enstrophy(p, u, out, S(stream)); });
}

int hd_stage_buffer(hd_plan* p, int scheme, int stage, double* u, void** out) {
  if (!p || !u || !out || (scheme != HD_SCHEME_RK3 && scheme != HD_SCHEME_RK4)) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  if (stage < 0 || stage >= nstages(scheme)) return HD_E_ARG;
  *out = stage_buffer(p, scheme, stage, u);
  return HD_OK;
}

int hd_reduce_state(hd_plan* p, const double* u, double* out, int64_t tag, void* stream) {
  if (!p || !u || !out) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  return timed(p, HD_TK_REDUCE, S(stream), [&] { return launch_reduce(p, u, out, tag, S(stream)); });
}

int hd_error_read(hd_plan* p, uint64_t* key, void* stream) {
  if (!p || !key) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  unsigned long long v = 0;
  if (cudaMemcpyAsync(&v, p->ws + p->off[HD_BUF_ERR], 8, cudaMemcpyDeviceToHost, S(stream)) != cudaSuccess ||
      cudaStreamSynchronize(S(stream)) != cudaSuccess)
    return HD_E_CUDA;
  *key = (v == ~0ull) ? 0 : (uint64_t)v;
  return HD_OK;
}

int hd_error_clear(hd_plan* p, void* stream) {
  if (!p) return HD_E_ARG;
  if (!p->ws) return HD_E_WORKSPACE;
  return cudaMemsetAsync(p->ws + p->off[HD_BUF_ERR], 0xff, 8, S(stream)) == cudaSuccess ? HD_OK
                                                                                        : HD_E_CUDA;
}

}  // extern "C"

namespace hd {
void count_launches(int n) { g_launches += n; }
}  // namespace hd
