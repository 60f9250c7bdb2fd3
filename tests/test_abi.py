"""The C-ABI library loads without a GPU and exports every symbol the public
header declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "stamg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(stamg_\w+)\s*\(", txt, re.M)))


def test_header_has_entry_points():
    syms = header_symbols()
    for must in ["stamg_create", "stamg_sweep", "stamg_apply_scatter", "stamg_apply_A", "stamg_coarse_gs",
                 "stamg_prolongate", "stamg_restrict", "stamg_mg_apply", "stamg_solve", "stamg_last_error"]:
        assert must in syms


def test_library_exports_all_symbols(stamg):
    lib = stamg.lib()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_last_error_is_empty_string_initially(stamg):
    assert isinstance(stamg.lib().stamg_last_error(), bytes)


def test_create_rejects_unsupported_problem_without_gpu(stamg):
    # validation runs on the host before any device call
    from paper_2010_04559_b200 import configs as cf
    # (3D / p0 / Lin problems run on the reference-shape path; a two-material 3D problem and
    # a 3D cone beam are outside both paths)
    spec = cf.reference_test_problem(2, 1.0, 1, 1, 1, 2, [1.0, 0.5, 0.2], 1.0, dim=3)
    spec.beam = cf.BEAM_CONE_X0
    try:
        stamg.Context(spec)
    except stamg.InvalidArgument as e:
        assert "beam" in str(e)
    else:  # pragma: no cover
        raise AssertionError("a 3D cone beam must be rejected")
    spec = cf.reference_test_problem(2, 1.0, 1, 0, 2, 2, [1.0, 0.5, 0.2], 1.0, dim=3)
    try:
        stamg.Context(spec)
    except stamg.InvalidArgument as e:
        assert "p must be 0 or 1" in str(e)
    else:  # pragma: no cover
        raise AssertionError("p = 2 must be rejected")
