"""Boundary checks that need no GPU: the C-ABI library builds, loads, and exports every
symbol include/pfem.h declares; the binding refuses CPU tensors (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pfem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pfem_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("pfem_mesh_prepare", "pfem_energy", "pfem_residual", "pfem_tangent_apply", "pfem_cg"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2601_03086_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_loads_and_reports_abi_version():
    import paper_2601_03086_b200 as pf
    lib = pf.load()
    assert lib.pfem_abi_version() == 6
    assert lib.pfem_last_error() is not None


def test_binding_rejects_cpu_tensors():
    import torch
    import paper_2601_03086_b200 as pf
    with pytest.raises((ValueError, RuntimeError)):
        pf.Mesh(torch.zeros((3, 2), dtype=torch.float64), torch.zeros((1, 3), dtype=torch.int32))


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2601_03086_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "pfem_oracle" not in txt, f


def test_ctypes_structs_match_the_header_layout(tmp_path):
    """Every struct the binding mirrors has the header's size and field offsets: a C program
    compiled against include/pfem.h prints offsetof / sizeof, compared with ctypes."""
    import subprocess
    from paper_2601_03086_b200 import _lib as L
    structs = {"pfem_mesh": L.pfem_mesh, "pfem_material": L.pfem_material, "pfem_flags": L.pfem_flags,
               "pfem_cg_report": L.pfem_cg_report, "pfem_newton_report": L.pfem_newton_report}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pfem.h"', 'int main(void) {']
    for name, cls in structs.items():
        lines.append(f'    printf("{name} size %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'    printf("{name} {fname} %zu\\n", offsetof({name}, {fname}));')
    lines += ['    return 0;', '}']
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            parts = ln.split()
            got[(parts[0], parts[1])] = int(parts[2])
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert got[(name, fname)] == getattr(cls, fname).offset, (name, fname)


def test_fma_peak_rejects_bad_arguments_without_a_gpu():
    """pfem_fma_peak checks its arguments before touching the device (no compute call here)."""
    import paper_2601_03086_b200 as pf
    lib = pf.load()
    out = ctypes.c_double(0.0)   # PFEM_ERR_ARG = -1
    assert lib.pfem_fma_peak(7, 16, ctypes.byref(out), None) == -1
    assert lib.pfem_fma_peak(1, 0, ctypes.byref(out), None) == -1
    assert lib.pfem_fma_peak(1, 16, None, None) == -1
    assert b"pfem_fma_peak" in lib.pfem_last_error()
