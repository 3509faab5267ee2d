"""B200-native (sm_100a) PFEM hot path: explicit FE differentiation on P1 simplex meshes.

C-ABI: include/pfem.h (libpfem.so, built from csrc/ by ``build.py``).  This package is a
thin binding; it never falls back to CPU code and never imports ``oracle/``.
"""
from .core import (MODES, Material, Mesh, cg, energy, fma_peak, heat, lame, launch_count, newton,  # noqa: F401
                   pretrain_loss, residual, tangent_apply, tangent_diag)
from ._lib import LIB_PATH, PfemError, load  # noqa: F401

__all__ = ["Mesh", "Material", "energy", "heat", "pretrain_loss", "residual", "tangent_apply", "tangent_diag", "cg", "newton", "lame", "launch_count", "fma_peak",
           "PfemError", "load", "LIB_PATH", "MODES"]
