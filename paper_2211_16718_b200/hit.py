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
  whose host synthesis would need tens of GB (512^3, 1024^3).
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
