"""The C-ABI library loads and exports every symbol include/xlfuse_b200.h
declares; host-only entry points behave (no GPU needed); the product never
reaches into oracle/."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2007_06000_b200 as X
from paper_2007_06000_b200 import _lib
from tests.conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "xlfuse_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xlf_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_lib.SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for s in header_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (xlf_\w+)", out))
    assert set(header_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_plumbing():
    L = _lib.lib()
    assert b"sm_100a" in L.xlf_version()
    h = ctypes.c_void_p()
    rc = L.xlf_graph_parse(b"name x\n", ctypes.byref(h))
    assert _lib.STATUS[rc] == "parse"
    assert L.xlf_last_error()
    rc = L.xlf_graph_parse(None, ctypes.byref(h))
    assert _lib.STATUS[rc] == "arg"


def test_engine_rejects_bad_arguments_without_gpu():
    L = _lib.lib()
    out = ctypes.c_void_p()
    rc = L.xlf_engine_create(None, 0, 1, 0, None, 0, 1, ctypes.byref(out))
    assert _lib.STATUS[rc] == "arg"


def test_engine_options_are_validated_without_gpu():
    """Planner / executor options come only through xlf_engine_create_ex's
    option string (the library reads no environment variables); an unknown
    key or a malformed value is refused before any device work."""
    g = X.Graph(open(X.graph_path("fire")).read())
    w = X.seeded_weights(g, 1)
    for bad in ("nonsense=1", "xbuf=two", "xbuf"):
        with pytest.raises(X.XlfError) as ei:
            X.Engine(g, w, "b200", "bf16", options=bad)
        assert ei.value.kind == "validation", bad
    with pytest.raises(X.XlfError) as ei:
        X.Engine(g, w, "b200", "int8")
    assert ei.value.kind == "arg"


def test_library_reads_no_environment():
    csrc = os.path.join(ROOT, "paper_2007_06000_b200", "csrc")
    for f in os.listdir(csrc):
        if f.endswith((".cpp", ".cu", ".hpp", ".cuh")):
            assert "getenv" not in open(os.path.join(csrc, f)).read(), f


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2007_06000_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
