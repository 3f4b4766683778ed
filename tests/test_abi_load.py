"""CPU-side checks of the boundary: the CUDA library builds for sm_100a, loads,
and exports every function include/gr.h declares (no compute calls: no GPU
here). Also checks the binding fails loudly when the library is missing."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gr_[a-z_]+)\s*\(", src)))


def test_header_declares_north_star_names():
    names = _declared()
    for required in ("gr_graph_create", "gr_bfs", "gr_sssp", "gr_graph_destroy", "gr_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1501_05387_b200 as gr
    lib = ctypes.CDLL(gr.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(gr.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", gr.LIB_PATH], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(r"\bT %s\b" % name, out), name


def test_library_is_sm100a():
    import paper_1501_05387_b200 as gr
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gr.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string_without_gpu():
    import paper_1501_05387_b200 as gr
    assert gr.gr_version().startswith("gr_b200")


def test_missing_library_fails_loudly(tmp_path):
    import paper_1501_05387_b200 as gr
    with pytest.raises(gr.GrError):
        old = gr._lib
        try:
            gr._lib = None
            gr.load(str(tmp_path / "nope.so"))
        finally:
            gr._lib = old
