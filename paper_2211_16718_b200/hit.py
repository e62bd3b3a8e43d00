"""Isotropic-turbulence initial conditions and spectra (pkg/src/hitdns/hit.py).

Off the hot path (runs once before the march), but needed to run the
benchmark configurations.  Two backends of the same synthesis
(hit.py:93-139: seeded complex Gaussian modes -> Hermitian symmetrisation ->
shell mask -> solenoidal projection -> exact per-shell rescale -> inverse FFT):

* ``backend="numpy"`` -- host numpy, the reference's own random stream
  (PCG64 ``default_rng(seed)``) and pocketfft, so the IC is bit-identical to
  the reference's under the same numpy version (pinned by
  tests/golden/traj32.json ``ic_sha256``);
* ``backend="torch"`` -- the same algorithm in HBM with cuFFT and the torch
  Philox stream: statistically identical, not bit-identical; used for grids
  whose host synthesis would need tens of GB (512^3);
* :func:`synthesize_velocity_slab` / :func:`make_initial_condition_slab` --
  the same algorithm decomposed over the ranks of a z-slab run (1024^3, where
  neither one host nor one GPU can hold the global transform next to the
  solver): every mode comes from a counter-based generator keyed by its
  global wavevector, so a rank draws any mode -- and its conjugate partner --
  without communication; the shell energies are summed over ranks before the
  exact per-shell rescale; the inverse FFT runs over (kz, kx) on ky slabs,
  one all-to-all, then over ky on the z slabs the solver owns.  The field is
  the same for every rank count up to FFT round-off.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError
from .grid import TWO_PI, FieldSet, GridSpec, Layout, convert_layout


@dataclass(frozen=True)
class HitParams:
    """hit.py:34-45."""

    u0: float = 0.3
    k0: float = 4.0
    re_lambda: float = 50.0
    rho0: float = 1.0
    seed: int = 2024

    def __post_init__(self):
        if self.u0 <= 0.0 or self.k0 <= 0.0 or self.re_lambda <= 0.0 or self.rho0 <= 0.0:
            raise ConfigError("u0, k0, re_lambda, rho0 must all be positive")


def target_spectrum(k, u0: float = 0.3, k0: float = 4.0):
    """E(k) = 16 sqrt(2/pi) (u0^2/k0) (k/k0)^4 exp(-2 (k/k0)^2) (hit.py:48-52)."""
    k = np.asarray(k, dtype=np.float64)
    ratio = k / k0
    return 16.0 * math.sqrt(2.0 / math.pi) * (u0 * u0 / k0) * ratio**4 * np.exp(-2.0 * ratio * ratio)


def gradient_variance(u0: float = 0.3, k0: float = 4.0) -> float:
    return (2.0 / 15.0) * (15.0 / 8.0) * u0 * u0 * k0 * k0


def taylor_microscale(u0: float = 0.3, k0: float = 4.0) -> float:
    return 2.0 * u0 / math.sqrt(gradient_variance(u0, k0))


def viscosity_from_re_lambda(params: HitParams) -> float:
    """mu = rho0 u0 lambda / Re_lambda (hit.py:65-67); 0.006 for the defaults."""
    return params.rho0 * params.u0 * taylor_microscale(params.u0, params.k0) / params.re_lambda


def eddy_turnover_time(params: HitParams) -> float:
    return taylor_microscale(params.u0, params.k0) / params.u0


def _shells(n: int):
    """Integer wavevector components (z, y, x broadcast order) and shell index."""
    kk = np.fft.fftfreq(n, 1.0 / n)
    kz, ky, kx = kk[:, None, None], kk[None, :, None], kk[None, None, :]
    shell = np.floor(np.sqrt(kx * kx + ky * ky + kz * kz) + 0.5).astype(np.int64)
    return kx, ky, kz, shell


def _shell_scale(raw: np.ndarray, n: int, params: HitParams) -> np.ndarray:
    """sqrt(E(s) n^6 / raw(s)) on populated shells 1..n/2-1, else 0 (hit.py:125-134)."""
    scale = np.zeros(raw.shape[0], dtype=np.float64)
    norm = float(n) ** 6
    for s in range(1, n // 2):
        if raw[s] > 0.0:
            scale[s] = math.sqrt(target_spectrum(float(s), params.u0, params.k0) * norm / raw[s])
    return scale


def _synth_numpy(n: int, params: HitParams):
    kx, ky, kz, shell = _shells(n)
    rng = np.random.default_rng(params.seed)
    c = rng.standard_normal((3, n, n, n)) + 1j * rng.standard_normal((3, n, n, n))
    # conjugate partner of mode m sits at (n - m) % n on every axis
    mirror = np.roll(np.flip(c, axis=(1, 2, 3)), 1, axis=(1, 2, 3))
    c = 0.5 * (c + np.conj(mirror))
    c *= (shell >= 1) & (shell < n // 2)
    k2 = kx * kx + ky * ky + kz * kz
    kdot = (kx * c[0] + ky * c[1] + kz * c[2]) / np.where(k2 == 0.0, 1.0, k2)
    c[0] -= kx * kdot
    c[1] -= ky * kdot
    c[2] -= kz * kdot
    energy = 0.5 * (np.abs(c[0]) ** 2 + np.abs(c[1]) ** 2 + np.abs(c[2]) ** 2)
    raw = np.bincount(shell.ravel(), weights=energy.ravel(), minlength=n // 2)
    c *= _shell_scale(raw, n, params)[shell]
    return tuple(np.fft.ifftn(c[a]).real for a in range(3))


def _synth_torch(n: int, params: HitParams, device):
    kk = torch.fft.fftfreq(n, 1.0 / n, dtype=torch.float64, device=device)
    kz, ky, kx = kk[:, None, None], kk[None, :, None], kk[None, None, :]
    shell = torch.floor(torch.sqrt(kx * kx + ky * ky + kz * kz) + 0.5).to(torch.int64)
    gen = torch.Generator(device=device)
    gen.manual_seed(params.seed)
    vel = []
    c = torch.complex(torch.randn((3, n, n, n), generator=gen, dtype=torch.float64, device=device),
                      torch.randn((3, n, n, n), generator=gen, dtype=torch.float64, device=device))
    c = 0.5 * (c + torch.conj(torch.roll(torch.flip(c, dims=(1, 2, 3)), (1, 1, 1), dims=(1, 2, 3))))
    c *= ((shell >= 1) & (shell < n // 2)).to(torch.float64)
    k2 = kx * kx + ky * ky + kz * kz
    kdot = (kx * c[0] + ky * c[1] + kz * c[2]) / torch.where(k2 == 0.0, torch.ones_like(k2), k2)
    c[0] -= kx * kdot
    c[1] -= ky * kdot
    c[2] -= kz * kdot
    energy = 0.5 * (c.real ** 2 + c.imag ** 2).sum(dim=0)
    # shell sums on the host: numpy's sequential bincount is reproducible bit-for-bit
    # (torch.bincount with weights accumulates with atomics on the GPU: its order,
    # hence the IC's last bits, would change from run to run and across processes)
    raw = np.bincount(shell.reshape(-1).cpu().numpy(), weights=energy.reshape(-1).cpu().numpy(),
                      minlength=n // 2)
    scale = torch.from_numpy(_shell_scale(raw, n, params)).to(device)
    c *= scale[shell]
    del energy, kdot
    for a in range(3):
        vel.append(torch.fft.ifftn(c[a]).real.contiguous())
    del c
    return tuple(vel)


def synthesize_velocity(n: int, params: HitParams, backend: str = "numpy", device=None):
    """Divergence-free velocity on an n^3 grid matching the target spectrum (hit.py:93-139).
    Returns (u, v, w) in (z, y, x) order: numpy arrays, or device tensors for ``torch``."""
    if n < 4:
        raise ConfigError(f"need n >= 4 to hold at least one spectral shell, got {n}")
    if backend == "numpy":
        return _synth_numpy(n, params)
    if backend == "torch":
        return _synth_torch(n, params, device or torch.device("cuda"))
    raise ValueError(f"backend must be 'numpy' or 'torch', got {backend!r}")


# ---- slab-decomposed synthesis ------------------------------------------------------
def _i64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


_K_INDEX, _K_SEED, _K_STREAM = _i64(0x9E3779B97F4A7C15), _i64(0xD1B54A32D192ED03), _i64(0x8CB92BA72F3D8DD7)
_M1, _M2 = _i64(0xBF58476D1CE4E5B9), _i64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 (torch's >> is arithmetic)."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _uniform(index: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    """(0, 1] doubles, a pure function of (index, seed, stream): the splitmix64
    finaliser over a Weyl-mixed counter (int64 arithmetic wraps)."""
    offset = _i64((seed * _K_SEED + (stream + 1) * _K_STREAM) % (1 << 64))  # Python ints: wrap here
    z = index * _K_INDEX + offset
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    z = z ^ _srl(z, 31)
    return (_srl(z, 11).to(torch.float64) + 1.0) * (2.0 ** -53)


def _mode_draw(n: int, seed: int, comp: int, kz, ky, kx) -> torch.Tensor:
    """Standard complex normal of velocity component ``comp`` at the integer
    wavevector indices (kz, ky, kx) in [0, n) (broadcast int64 tensors)."""
    index = ((comp * n + kz) * n + ky) * n + kx
    r = torch.sqrt(-2.0 * torch.log(_uniform(index, seed, 0)))
    theta = (2.0 * math.pi) * _uniform(index, seed, 1)
    return torch.complex(r * torch.cos(theta), r * torch.sin(theta))


def _freq(idx: torch.Tensor, n: int) -> torch.Tensor:
    """fftfreq(n, 1/n) of integer indices: k for k < n/2, k - n above."""
    return torch.where(idx < (n + 1) // 2, idx, idx - n).to(torch.float64)


def _sum_over_ranks(x: torch.Tensor, group) -> torch.Tensor:
    """Rank-order sum of a small tensor over the group (deterministic)."""
    import torch.distributed as dist

    if group is None and not (dist.is_available() and dist.is_initialized()):
        return x
    world = dist.get_world_size(group)
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x.contiguous(), group=group)
    total = parts[0].clone()
    for part in parts[1:]:
        total += part
    return total


def synthesize_velocity_slab(n: int, params: HitParams, rank: int = 0, world: int = 1, group=None,
                             device=None, chunk: int = 32):
    """The rank's z slab (z in [rank n/world, (rank+1) n/world), all y, x) of the
    solenoidal HIT velocity (hit.py:93-139's algorithm with a counter-based mode
    generator); (u, v, w) tensors of shape (n/world, n, n).  Collective over
    ``group`` (all ranks call it); world = 1 runs it on one device."""
    if n < 4:
        raise ConfigError(f"need n >= 4 to hold at least one spectral shell, got {n}")
    if n % world:
        raise ConfigError(f"{world} ranks do not divide n = {n}")
    dev = torch.device(device) if device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
    span = n // world
    ky_lo = rank * span
    idx = torch.arange(n, dtype=torch.int64, device=dev)
    ky_i = idx[ky_lo:ky_lo + span][None, :, None]
    kx_i = idx[None, None, :]
    fy, fx = _freq(ky_i, n), _freq(kx_i, n)
    mirror = lambda i: (n - i) % n  # noqa: E731 - index of the conjugate partner
    c = torch.empty((3, n, span, n), dtype=torch.complex128, device=dev)
    raw = np.zeros(n, dtype=np.float64)
    # modes, Hermitian symmetrisation, shell mask, solenoidal projection and the
    # shell energies, chunk by chunk along kz (bounded temporaries)
    for z0 in range(0, n, chunk):
        kz_i = idx[z0:z0 + chunk][:, None, None]
        fz = _freq(kz_i, n)
        k2 = fx * fx + fy * fy + fz * fz
        shell = torch.floor(torch.sqrt(k2) + 0.5).to(torch.int64)
        keep = ((shell >= 1) & (shell < n // 2)).to(torch.float64)
        part = torch.stack([0.5 * (_mode_draw(n, params.seed, a, kz_i, ky_i, kx_i) +
                                   torch.conj(_mode_draw(n, params.seed, a, mirror(kz_i), mirror(ky_i),
                                                         mirror(kx_i))))
                            for a in range(3)]) * keep
        kdot = (fx * part[0] + fy * part[1] + fz * part[2]) / torch.where(k2 == 0.0, torch.ones_like(k2), k2)
        part[0] -= fx * kdot
        part[1] -= fy * kdot
        part[2] -= fz * kdot
        energy = 0.5 * (part.real ** 2 + part.imag ** 2).sum(dim=0)
        # host bincount: sequential, so the sums are reproducible bit for bit
        raw += np.bincount(shell.expand_as(energy).reshape(-1).cpu().numpy(),
                           weights=energy.reshape(-1).cpu().numpy(), minlength=n)[:n]
        c[:, z0:z0 + chunk] = part
        del part, kdot, energy
    raw = _sum_over_ranks(torch.from_numpy(raw).to(dev), group).cpu().numpy()
    scale = torch.from_numpy(_shell_scale(raw, n, params)).to(dev)
    for z0 in range(0, n, chunk):
        fz = _freq(idx[z0:z0 + chunk][:, None, None], n)
        shell = torch.floor(torch.sqrt(fx * fx + fy * fy + fz * fz) + 0.5).to(torch.int64)
        c[:, z0:z0 + chunk] *= scale[shell]
    vel = []
    for a in range(3):
        # (kz, ky slab, kx) -> (z, ky slab, x), then z slabs to their owners
        ca = torch.fft.ifft(torch.fft.ifft(c[a], dim=2), dim=0)
        if world > 1:
            import torch.distributed as dist

            send = torch.view_as_real(ca).contiguous()  # (P z-blocks x span, span, n, 2)
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send, group=group)
            # recv[r] = z block of this rank, ky slab of rank r -> (z, ky, x)
            ca = torch.view_as_complex(recv.view(world, span, span, n, 2).permute(1, 0, 2, 3, 4)
                                       .reshape(span, n, n, 2).contiguous())
        vel.append(torch.fft.ifft(ca, dim=1).real.contiguous())
        del ca
    del c
    return tuple(vel)


def compute_spectrum_slab(u, v, w, rank: int = 0, world: int = 1, group=None) -> "SpectrumTable":
    """compute_spectrum of a field held as z slabs (u, v, w: this rank's
    (n/world, n, n) tensors): forward FFT over (y, x) on the slab, one
    all-to-all to ky slabs, FFT over z; shell energies summed over ranks in rank
    order.  Every rank gets the table.  Collective over ``group``."""
    span, n = u.shape[0], u.shape[-1]
    dev = u.device
    idx = torch.arange(n, dtype=torch.int64, device=dev)
    fy = _freq(idx[rank * span:(rank + 1) * span][None, :, None], n)
    fx = _freq(idx[None, None, :], n)
    fz = _freq(idx[:, None, None], n)
    shell = torch.floor(torch.sqrt(fx * fx + fy * fy + fz * fz) + 0.5).to(torch.int64)
    energy = torch.zeros((n, span, n), dtype=torch.float64, device=dev)
    for comp in (u, v, w):
        a = torch.fft.fftn(comp, dim=(1, 2))  # (z slab, ky, kx)
        if world > 1:
            import torch.distributed as dist

            send = torch.view_as_real(a.reshape(span, world, span, n).permute(1, 0, 2, 3).contiguous())
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send, group=group)
            a = torch.view_as_complex(recv.reshape(n, span, n, 2))  # (z, ky slab, kx)
        a = torch.fft.fft(a, dim=0)
        energy += a.real ** 2 + a.imag ** 2
        del a
    energy /= 2.0 * float(n) ** 6
    binned = np.bincount(shell.expand_as(energy).reshape(-1).cpu().numpy(),
                         weights=energy.reshape(-1).cpu().numpy(), minlength=n)[:n]
    binned = _sum_over_ranks(torch.from_numpy(binned).to(dev), group).cpu().numpy()
    return SpectrumTable(np.arange(n, dtype=np.int64), binned, n)


def make_initial_condition_slab(spec: GridSpec, params: HitParams, layout, group=None,
                                gamma: float = 1.4, device=None) -> FieldSet:
    """The block of ``layout`` (a z-slab RankLayout of ``spec``, decomp.decompose)
    of the HIT initial condition, synthesised across the group's ranks
    (:func:`synthesize_velocity_slab`); rho0, p0 = rho0/gamma, ghosts zero."""
    n = spec.n[0]
    if spec.n[1] != n or spec.n[2] != n:
        raise ConfigError(f"initial condition needs a cubic grid, got n={spec.n}")
    if tuple(layout.dims[:2]) != (1, 1):
        raise ConfigError(f"slab synthesis needs z slabs (1, 1, P), got dims {layout.dims}")
    world = layout.dims[2]
    u, v, w = synthesize_velocity_slab(n, params, layout.coords[2], world, group, device)
    rho0, p0 = params.rho0, params.rho0 / gamma
    fields = FieldSet.zeros(layout.spec, Layout.COMPONENT_CONTIGUOUS, device=u.device)
    it = fields.interior()
    it[0] = rho0
    it[1] = rho0 * u
    it[2] = rho0 * v
    it[3] = rho0 * w
    it[4] = p0 / (gamma - 1.0) + 0.5 * rho0 * (u * u + v * v + w * w)
    return fields


@dataclass
class SpectrumTable:
    k: np.ndarray
    energy: np.ndarray
    grid_n: int

    @property
    def resolved_max(self) -> int:
        return self.grid_n // 2 - 1

    def total(self) -> float:
        return float(np.sum(self.energy))

    def rows(self):
        for s in range(1, self.resolved_max + 1):
            yield int(self.k[s]), float(self.energy[s])


def compute_spectrum(u, v, w) -> SpectrumTable:
    """Shell-binned KE spectrum (hit.py:164-176); accepts numpy arrays or tensors."""
    if isinstance(u, torch.Tensor):
        n = u.shape[-1]
        e = (torch.fft.fftn(u).abs() ** 2 + torch.fft.fftn(v).abs() ** 2 +
             torch.fft.fftn(w).abs() ** 2) / (2.0 * float(n) ** 6)
        kk = torch.fft.fftfreq(n, 1.0 / n, dtype=torch.float64, device=u.device)
        shell = torch.floor(torch.sqrt(kk[:, None, None] ** 2 + kk[None, :, None] ** 2 +
                                       kk[None, None, :] ** 2) + 0.5).to(torch.int64)
        binned = torch.bincount(shell.reshape(-1), weights=e.reshape(-1)).cpu().numpy()
        return SpectrumTable(np.arange(binned.shape[0], dtype=np.int64), binned, n)
    nz, ny, nx = u.shape[-3:]
    if not (nz == ny == nx):
        raise ConfigError(f"spectral routines need a cubic grid, got {u.shape[-3:]}")
    n = nx
    e = (np.abs(np.fft.fftn(u)) ** 2 + np.abs(np.fft.fftn(v)) ** 2 +
         np.abs(np.fft.fftn(w)) ** 2) / (2.0 * float(n) ** 6)
    _, _, _, shell = _shells(n)
    binned = np.bincount(shell.ravel(), weights=e.ravel(), minlength=int(shell.max()) + 1)
    return SpectrumTable(np.arange(binned.shape[0], dtype=np.int64), binned, n)


def spectral_divergence(u, v, w) -> float:
    """max over wavevectors of |k . c(k)| with c = fft / n^3 (hit.py:179-188): zero up
    to transform round-off for a solenoidal field.  numpy arrays or tensors."""
    if isinstance(u, torch.Tensor):
        n = u.shape[-1]
        kk = torch.fft.fftfreq(n, 1.0 / n, dtype=torch.float64, device=u.device)
        div = (kk[None, None, :] * torch.fft.fftn(u) + kk[None, :, None] * torch.fft.fftn(v) +
               kk[:, None, None] * torch.fft.fftn(w)) / float(n) ** 3
        return float(div.abs().max())
    n = u.shape[-1]
    kx, ky, kz, _ = _shells(n)
    div = (kx * np.fft.fftn(u) + ky * np.fft.fftn(v) + kz * np.fft.fftn(w)) / float(n) ** 3
    return float(np.max(np.abs(div)))


def velocity(fields: FieldSet):
    """Interior velocity (m/rho) tensors of a device FieldSet."""
    it = fields.interior()
    return it[1] / it[0], it[2] / it[0], it[3] / it[0]


def make_initial_condition(spec: GridSpec, params: HitParams, gamma: float = 1.4,
                           layout: Layout = Layout.COMPONENT_CONTIGUOUS, backend: str = "auto",
                           device=None) -> FieldSet:
    """Conserved HIT state at rho0, p0 = rho0/gamma, ghosts zero (hit.py:210-236).

    ``backend="auto"``: numpy (reference-bit-identical) up to 128^3, torch above."""
    if spec.n[0] != spec.n[1] or spec.n[1] != spec.n[2]:
        raise ConfigError(f"initial condition needs a cubic grid, got n={spec.n}")
    for d in range(3):
        if abs(spec.length[d] - TWO_PI) > 1e-12 * TWO_PI:
            raise ConfigError("initial condition assumes a 2*pi-periodic box")
    n = spec.n[0]
    if backend == "auto":
        backend = "numpy" if n <= 128 else "torch"
    rho0 = params.rho0
    p0 = rho0 / gamma
    fields = FieldSet.zeros(spec, Layout.COMPONENT_CONTIGUOUS, device=device)
    it = fields.interior()
    if backend == "numpy":
        u, v, w = synthesize_velocity(n, params, "numpy")
        body = np.empty((5, n, n, n))
        body[0] = rho0
        body[1] = rho0 * u
        body[2] = rho0 * v
        body[3] = rho0 * w
        body[4] = p0 / (gamma - 1.0) + 0.5 * rho0 * (u * u + v * v + w * w)
        it.copy_(torch.from_numpy(body))
    else:
        u, v, w = synthesize_velocity(n, params, "torch", fields.data.device)
        it[0] = rho0
        it[1] = rho0 * u
        it[2] = rho0 * v
        it[3] = rho0 * w
        it[4] = p0 / (gamma - 1.0) + 0.5 * rho0 * (u * u + v * v + w * w)
    if layout != Layout.COMPONENT_CONTIGUOUS:
        fields = convert_layout(fields, layout)
    return fields


def write_spectrum(path, table: SpectrumTable) -> None:
    """Two columns ``k E(k)``, one row per shell 1 <= k <= n/2-1 (hit.py:190-194)."""
    with open(path, "w") as fh:
        for k, e in table.rows():
            fh.write(f"{k} {e:.17e}\n")


def read_spectrum(path):
    """Inverse of :func:`write_spectrum`; ``#`` lines and blanks skipped (hit.py:197-208)."""
    ks, es = [], []
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            a, b = line.split()
            ks.append(int(a))
            es.append(float(b))
    return np.array(ks, dtype=np.int64), np.array(es)
