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
