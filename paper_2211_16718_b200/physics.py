"""Gas model and parameter records (pkg/src/hitdns/physics.py:26-44, weno.py:40-55)."""

from __future__ import annotations

from dataclasses import dataclass

OPTIMAL_WEIGHTS = (0.1, 0.6, 0.3)  # weno.py:25
FIFTH_ORDER_COEFFS = (1.0 / 30.0, -13.0 / 60.0, 47.0 / 60.0, 27.0 / 60.0, -1.0 / 20.0)  # weno.py:37


@dataclass(frozen=True)
class GasModel:
    """Gas constants and viscosity knobs for one run (physics.py:26-44)."""

    gamma: float = 1.4
    prandtl: float = 0.72
    mu: float = 0.0
    visc_scale: float = 1.0

    def __post_init__(self):
        if self.gamma <= 1.0:
            raise ValueError(f"gamma must exceed 1, got {self.gamma}")
        if self.prandtl <= 0.0:
            raise ValueError(f"prandtl must be positive, got {self.prandtl}")
        if self.mu < 0.0:
            raise ValueError(f"mu must be nonnegative, got {self.mu}")

    @property
    def effective_mu(self) -> float:
        return self.mu * self.visc_scale


@dataclass(frozen=True)
class WenoParams:
    """Regularisation epsilon and the power applied to (eps + beta) (weno.py:40-55)."""

    epsilon: float = 1e-6
    power: int = 2

    def __post_init__(self):
        if self.epsilon <= 0.0:
            raise ValueError(f"epsilon must be positive, got {self.epsilon}")
        if int(self.power) != self.power or self.power < 1:
            raise ValueError(f"power must be a positive integer, got {self.power}")
        object.__setattr__(self, "power", int(self.power))


DEFAULT_PARAMS = WenoParams()


# ---- pointwise helpers (physics.py:47-255) -------------------------------------------
# Not on the hot path (the kernels decode states inline); the reference's utility API on
# device tensors, evaluated with the reference's operation order.  Arrays carry the
# variables in the last axis like the reference's numpy helpers.


def _dev(a):
    import torch

    from .grid import default_device

    if isinstance(a, torch.Tensor):
        return a.to(torch.float64)
    return torch.as_tensor(a, dtype=torch.float64, device=default_device())


def _check_positive(name: str, values) -> None:
    """physics.py:47-55."""
    import torch

    from .errors import InvalidStateError

    ok = values > 0.0
    if bool(ok.all()):
        return
    bad = torch.nonzero(~ok)
    first = tuple(int(x) for x in bad[0]) if bad.numel() else None
    raise InvalidStateError(f"nonpositive {name} (min {float(values.min()):.6e}) at array index {first}",
                            where=first)


def cons_to_prim(cons, gamma: float):
    """Conserved -> primitive (rho, u, v, w, p) in the last axis (physics.py:58-71)."""
    cons = _dev(cons)
    rho = cons[..., 0]
    _check_positive("density", rho)
    out = cons.clone()
    vel = cons[..., 1:4] / rho[..., None]
    out[..., 1:4] = vel
    kinetic = 0.5 * rho * (vel * vel).sum(-1)
    p = (gamma - 1.0) * (cons[..., 4] - kinetic)
    _check_positive("pressure", p)
    out[..., 4] = p
    return out


def prim_to_cons(prim, gamma: float):
    """physics.py:74-84."""
    prim = _dev(prim)
    rho, vel, p = prim[..., 0], prim[..., 1:4], prim[..., 4]
    out = prim.clone()
    out[..., 1:4] = rho[..., None] * vel
    out[..., 4] = p / (gamma - 1.0) + 0.5 * rho * (vel * vel).sum(-1)
    return out


def sound_speed(prim, gamma: float):
    prim = _dev(prim)
    return (gamma * prim[..., 4] / prim[..., 0]).sqrt()


def temperature(prim, gamma: float):
    """T = gamma p / rho (physics.py:92-95)."""
    prim = _dev(prim)
    return gamma * prim[..., 4] / prim[..., 0]


def convective_flux(cons, dim: int, gamma: float):
    """Inviscid flux along ``dim`` (physics.py:98-113)."""
    cons = _dev(cons)
    prim = cons_to_prim(cons, gamma)
    vd = prim[..., 1 + dim]
    p = prim[..., 4]
    out = cons.clone()
    out[..., 0] = prim[..., 0] * vd
    out[..., 1:4] = cons[..., 1:4] * vd[..., None]
    out[..., 1 + dim] += p
    out[..., 4] = (cons[..., 4] + p) * vd
    return out


def max_wavespeed(cons, dim: int, gamma: float):
    """|v_d| + a (physics.py:116-119)."""
    prim = cons_to_prim(cons, gamma)
    return prim[..., 1 + dim].abs() + sound_speed(prim, gamma)


def viscous_stress(grad_v, mu: float, visc_scale: float = 1.0):
    """tau_ij = mu (g_ij + g_ji - 2/3 div delta_ij) (physics.py:218-228)."""
    import torch

    g = _dev(grad_v)
    div = g.diagonal(dim1=-2, dim2=-1).sum(-1)
    tau = g + g.transpose(-2, -1)
    eye = torch.eye(3, dtype=torch.float64, device=g.device)
    tau = tau - (2.0 / 3.0) * div[..., None, None] * eye
    return mu * visc_scale * tau


def heat_flux(grad_T, mu: float, visc_scale: float, gamma: float, prandtl: float):
    """physics.py:231-234."""
    coeff = -mu * visc_scale / ((gamma - 1.0) * prandtl)
    return coeff * _dev(grad_T)


def decode_primitives(fields, gamma: float):
    """Ghosted (rho, u, v, w, p) of a COMPONENT_CONTIGUOUS FieldSet, positivity
    checked over the full ghosted extent (physics.py:240-255)."""
    view = fields.component_view()
    rho = view[0]
    _check_positive("density", rho)
    inv_rho = 1.0 / rho
    u = view[1] * inv_rho
    v = view[2] * inv_rho
    w = view[3] * inv_rho
    p = (gamma - 1.0) * (view[4] - 0.5 * rho * (u * u + v * v + w * w))
    _check_positive("pressure", p)
    return rho, u, v, w, p
