"""The C-ABI library loads and exports every symbol include/fvr_b200.h
declares (no device calls: this runs on the CPU box)."""

import os
import re
import subprocess

import pytest

from paper_1809_06417_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fvr_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fvr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("fvr_render_rays", "fvr_count_hull_samples", "fvr_adjust_rays", "fvr_loop_render",
                     "fvr_loop_adjust", "fvr_loop_finalize", "fvr_loop_update", "fvr_ctmap_build",
                     "fvr_temp_lookup", "fvr_visual_hull_view", "fvr_last_error"):
        assert required in names


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared_functions()


def test_exports_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fvr_[a-z0-9_]+)\b", out))
    assert set(declared_functions()) <= exported


def test_library_is_built_for_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_error_string_without_gpu():
    lib = _lib.load()
    assert lib.fvr_abi_version() == 1
    # argument validation happens before any CUDA call
    g = _lib.FvrGrid()
    g.nx = 0
    rc = lib.fvr_count_hull_samples(None, None, 1, None, g, None, None)
    assert rc == _lib.FVR_ERR_INVALID
    assert b"voxel counts" in lib.fvr_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_render_plan_chunk_entries_without_gpu():
    """Units of the render plan are padded to whole 32-byte lane chunks of
    16-bit weight words (fvr_rplan.cuh kRpB); the engine reads the padding
    from the library, so a build with another chunk size stays consistent."""
    n = _lib.load().fvr_rplan_chunk_entries()
    assert n in (8, 16) and n & (n - 1) == 0


def test_ctypes_signatures_match_header():
    """Every prototype in include/fvr_b200.h has a ctypes signature with the
    same number of parameters (the compiler already ties the header to the
    definitions: extern "C" functions cannot overload)."""
    import re

    from paper_1809_06417_b200 import _lib

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    h = open(os.path.join(root, "include", "fvr_b200.h")).read()
    protos = {}
    for m in re.finditer(r"^(?:int|int64_t|const char\*)\s+(fvr_\w+)\(([^;]*?)\);", h, re.M | re.S):
        args = m.group(2).strip()
        protos[m.group(1)] = 0 if args in ("void", "") else args.count(",") + 1
    assert protos, "no prototypes parsed"
    assert sorted(set(protos) - set(_lib._SIGNATURES)) == []
    bad = {k: (len(v[1]), protos[k]) for k, v in _lib._SIGNATURES.items() if k in protos and len(v[1]) != protos[k]}
    assert bad == {}, bad
