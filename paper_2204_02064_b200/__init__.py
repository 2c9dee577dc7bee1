"""B200-native PERKS stencil library (arXiv 2204.02064): the iterative explicit stencil time
loop as three sm_100a execution variants (host loop / persistent / PERKS) behind a C ABI
(include/perks/perks_stencil.h, libperks_stencil.so).

``Stencil`` and ``run`` load the CUDA library on first use and raise if it is missing — there
is no CPU fallback.  ``model`` (the paper's §4 performance model) is pure Python.
"""
__all__ = ["Stencil", "run", "run_group", "CG", "VARIANTS", "model", "build"]


def __getattr__(name):
    if name in ("Stencil", "run", "run_group"):
        from . import stencil

        return getattr(stencil, name)
    if name == "CG":
        from .cg import CG

        return CG
    if name == "VARIANTS":
        from ._lib import VARIANTS

        return VARIANTS
    raise AttributeError(name)


def build(verbose: bool = False) -> str:
    from ._build import build as _b

    return _b(verbose)
