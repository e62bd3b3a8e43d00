"""Viscous right-hand side on the GPU (mirrors pkg/src/hitdns/viscous.py).

``parabolic_rhs`` = primitives kernel -> gradient/flux kernel (12 central
gradients, stress and heat flux, 12 flux fields with their periodic images
along their own axis) -> divergence kernel adding D_d F_d into rows 1..4 in
the reference order d = 0, 1, 2 (viscous.py:112-120).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .grid import FieldSet, Layout
from .physics import GasModel
from .plan import _stream_ptr, get_plan

_OFFSETS = ((1, 0, 0), (0, 1, 0), (0, 0, 1))


def central_derivative_4(field: torch.Tensor, dim: int, spacing: float, ghost_width: int = 3,
                         workers: int = 1, out: torch.Tensor | None = None,
                         out_ghost: int = 0) -> torch.Tensor:
    """Fourth-order central derivative of a ghosted (z, y, x) device array
    (viscous.py:23-51) through hd_central_diff4 (kernels.py:207-227)."""
    L = _lib.load(require_cuda=True)
    g = ghost_width
    if field.dtype != torch.float64 or not field.is_cuda:
        raise ValueError("central_derivative_4 needs a float64 CUDA tensor")
    field = field.contiguous()
    nz, ny, nx = (s - 2 * g for s in field.shape)
    if out is None:
        out = torch.empty((nz, ny, nx), dtype=torch.float64, device=field.device)
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    di, dj, dk = _OFFSETS[dim]
    coef = 1.0 / (12.0 * spacing)
    _lib.check(L.hd_central_diff4(ctypes.c_void_p(field.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                  di, dj, dk, g, out_ghost, nx, ny, nz, 0, nz, coef, _stream_ptr()),
               "hd_central_diff4")
    return out


def parabolic_rhs(fields: FieldSet, gas: GasModel, halo=None, workers: int = 1,
                  out: FieldSet | None = None, mode: str | None = None) -> FieldSet:
    """Viscous + heat-conduction RHS, added into ``out`` when given (viscous.py:54-121).
    mu == 0 returns the untouched (zero) increment (viscous.py:72-73)."""
    if fields.layout != Layout.COMPONENT_CONTIGUOUS:
        raise ValueError("parabolic_rhs needs COMPONENT_CONTIGUOUS fields")
    if out is None:
        out = fields.like()
    if gas.effective_mu == 0.0:
        return out
    periodic = tuple(getattr(halo, "periodic", (True, True, True))) if halo is not None else (True,) * 3
    if periodic == (True, True, True):
        get_plan(fields.spec, gas, mode=mode).parabolic_rhs(fields.data, out.data)
        return out
    # a decomposed block (DistHalo): fluxes, their faces along the split axes, divergence
    from . import _lib
    from .plan import _ptr, _stream_ptr

    plan = get_plan(fields.spec, gas, mode=mode, periodic=periodic)
    _lib.check(plan.L.hd_viscous_fluxes(plan.h, _ptr(fields.data), _stream_ptr()), "hd_viscous_fluxes")
    halo.sync_flux_fields(plan.fields(_lib.HD_BUF_VFLUX, 9), fields.spec)
    _lib.check(plan.L.hd_viscous_divergence(plan.h, _ptr(out.data), _stream_ptr()), "hd_viscous_divergence")
    return out
