"""CPU-side checks of the boundary: the shared library loads without a GPU
and exports every symbol include/cutfem_mg.h declares; the binding fails
loudly without the library; argument validation happens before device work."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_11608_b200", "libcutfem_mg.so")
HDR = os.path.join(ROOT, "include", "cutfem_mg.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"\b(cutfem_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("cutfem_setup_mesh", "cutfem_build_patches", "cutfem_apply_operator", "cutfem_smooth",
              "cutfem_vcycle", "cutfem_solve_cg_mg"):
        assert n in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    for n in declared():
        assert hasattr(lib, n), n


def test_binding_covers_every_symbol():
    from paper_2508_11608_b200 import cutfem
    assert set(cutfem.EXPORTED) == set(declared())


def test_argument_errors_without_gpu():
    from paper_2508_11608_b200 import cutfem
    lib = cutfem._lib
    out = ctypes.c_void_p()
    assert lib.cutfem_setup_mesh(None, None, ctypes.byref(out)) == 1
    prm = cutfem.make_params(-1, -1, 2, 2, 3, 7, 0, 0, 1)   # degree 7: rejected
    assert lib.cutfem_setup_mesh(ctypes.byref(prm), None, ctypes.byref(out)) == 1
    assert b"degree" in lib.cutfem_last_error()
    assert lib.cutfem_smooth(None, 0, None, None, 0, None) == 1
    assert lib.cutfem_apply_operator(None, 0, None, None, None) == 1
