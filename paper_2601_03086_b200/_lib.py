"""ctypes binding of libpfem.so (include/pfem.h).  Argument marshalling only: every step
of the path runs in the CUDA kernels of csrc/.  There is no CPU fallback — if the
library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpfem.so")

PFEM_OK = 0
STATUS = {0: "PFEM_OK", -1: "PFEM_ERR_ARG", -2: "PFEM_ERR_DEGENERATE", -3: "PFEM_ERR_INVERTED",
          -4: "PFEM_ERR_NOT_CONVERGED", -5: "PFEM_ERR_BREAKDOWN", -6: "PFEM_ERR_CAPACITY",
          -7: "PFEM_ERR_CUDA", -8: "PFEM_ERR_NOT_PREPARED"}
F32, F64 = 0, 1
LINEAR, NEOHOOKEAN = 0, 1
LAME, YOUNG_POISSON, YOUNG_POISSON_PLANE_STRESS = 0, 1, 2
ASSEMBLE_CSR, ASSEMBLE_COLOUR = 0, 1


class pfem_mesh(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("n_nodes", C.c_int32), ("n_elems", C.c_int32), ("n_parts", C.c_int32),
        ("dtype", C.c_int32), ("block_elems", C.c_int32), ("elem_order", C.c_int32), ("geometry", C.c_int32),
        ("elem_type", C.c_int32),
        ("coords", C.c_void_p), ("conn", C.c_void_p), ("part_elem", C.c_void_p), ("part_node", C.c_void_p),
        ("grad", C.c_void_p), ("vol", C.c_void_p), ("csr_ptr", C.c_void_p), ("csr_ent", C.c_void_p),
        ("colour", C.c_void_p), ("colour_elems", C.c_void_p), ("colour_ptr", C.c_void_p),
        ("max_colours", C.c_int32),
        ("n_colours", C.c_int32), ("n_negative", C.c_int32), ("n_blocks", C.c_int32), ("n_occ", C.c_int32),
        ("plan", C.c_void_p),
    ]


class pfem_material(C.Structure):
    _fields_ = [("model", C.c_int32), ("kind", C.c_int32), ("p0", C.c_void_p), ("p1", C.c_void_p),
                ("stride0", C.c_int64), ("stride1", C.c_int64)]


class pfem_flags(C.Structure):
    _fields_ = [("n_inverted", C.c_int32), ("first_inverted", C.c_int32), ("n_nonfinite", C.c_int32),
                ("reserved", C.c_int32)]


class pfem_cg_report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("reserved", C.c_int32), ("rel_res0", C.c_double), ("rel_res_final", C.c_double),
                ("true_rel_res_final", C.c_double), ("bnorm", C.c_double)]


class pfem_newton_report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("cg_iterations", C.c_int32), ("res0", C.c_double), ("res_final", C.c_double)]


class PfemError(RuntimeError):
    def __init__(self, status: int, message: str, index: int):
        super().__init__(f"{STATUS.get(status, status)}: {message} (index {index})")
        self.status = status
        self.index = index


_lib = None

SIGNATURES = {
    "pfem_mesh_prepare": (C.c_int, [C.POINTER(pfem_mesh), C.c_void_p]),
    "pfem_mesh_release": (None, [C.POINTER(pfem_mesh)]),
    "pfem_plan_export": (C.c_int, [C.POINTER(pfem_mesh), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "pfem_workspace_bytes": (C.c_size_t, [C.POINTER(pfem_mesh), C.c_int32]),
    "pfem_lame": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "pfem_energy": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_int32, C.c_void_p, C.c_int64,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                              C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_residual": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_int32, C.c_void_p, C.c_int64,
                                C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_tangent_apply": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_int32, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                     C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_cg_workspace_bytes": (C.c_size_t, [C.POINTER(pfem_mesh)]),
    "pfem_cg": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(pfem_cg_report),
                          C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_pretrain_loss": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_int32, C.c_void_p,
                                     C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_heat_workspace_bytes": (C.c_size_t, [C.POINTER(pfem_mesh), C.c_int32]),
    "pfem_heat": (C.c_int, [C.POINTER(pfem_mesh), C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t,
                            C.c_void_p]),
    "pfem_tangent_diag": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "pfem_pcg": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_int32, C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_void_p,
                           C.POINTER(pfem_cg_report), C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_newton_workspace_bytes": (C.c_size_t, [C.POINTER(pfem_mesh)]),
    "pfem_newton": (C.c_int, [C.POINTER(pfem_mesh), C.POINTER(pfem_material), C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_double, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_void_p,
                              C.POINTER(pfem_newton_report), C.c_void_p, C.c_size_t, C.c_void_p]),
    "pfem_last_error": (C.c_char_p, []),
    "pfem_last_error_index": (C.c_int64, []),
    "pfem_abi_version": (C.c_int32, []),
    "pfem_launch_count": (C.c_int64, [C.c_int32]),
    "pfem_fma_peak": (C.c_int32, [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.c_void_p]),
}


def load(path: str = LIB_PATH):
    """Load libpfem.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libpfem.so not found at {path}; run `python -m paper_2601_03086_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int):
    if status != PFEM_OK:
        lib = load()
        raise PfemError(status, lib.pfem_last_error().decode(), lib.pfem_last_error_index())
