"""Hyperbolic right-hand side on the GPU (mirrors pkg/src/hitdns/upwind.py:163-213).

``hyperbolic_rhs`` keeps the reference signature; ``workers`` is accepted
and ignored (the CUDA grid replaces run_slabs, upwind.py:30-45).  The work is
three launches of the fused WENO5/Roe/flux-difference sweep kernel
(csrc/hd_sweep.cu), x then y then z, exactly the reference's accumulation
order (upwind.py:200).
"""

from __future__ import annotations

from .grid import FieldSet, Layout
from .physics import DEFAULT_PARAMS, GasModel, WenoParams
from .plan import get_plan


def _require_cc(fields: FieldSet, who: str) -> None:
    if fields.layout != Layout.COMPONENT_CONTIGUOUS:
        raise ValueError(f"{who} needs COMPONENT_CONTIGUOUS fields")


def hyperbolic_rhs(fields: FieldSet, gas: GasModel, params: WenoParams = DEFAULT_PARAMS,
                   delta: float = 0.0, workers: int = 1, out: FieldSet | None = None,
                   mode: str | None = None) -> FieldSet:
    """-div(F) over all three dimensions; ghosts of ``fields`` must be filled.
    Adds into ``out`` when given (upwind.py:163-181)."""
    _require_cc(fields, "hyperbolic_rhs")
    plan = get_plan(fields.spec, gas, params, delta, mode)
    accumulate = out is not None
    if out is None:
        out = fields.like()
    plan.hyperbolic_rhs(fields.data, out.data, accumulate)
    plan.raise_if_error(wrap_steps=False)
    return out


def hyper_sweep(fields: FieldSet, dim: int, inc: FieldSet, gas: GasModel = GasModel(),
                params: WenoParams = DEFAULT_PARAMS, delta: float = 0.0,
                mode: str | None = None) -> FieldSet:
    """One dimension's sweep, accumulating -dF/dx into ``inc`` (kernels.py:68-204)."""
    _require_cc(fields, "hyper_sweep")
    get_plan(fields.spec, gas, params, delta, mode).hyper_sweep(dim, fields.data, inc.data, True)
    return inc
