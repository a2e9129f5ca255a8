"""The reference-side C++ binding (tests/cpp/fused_exec_b200.cpp, the code
INTEGRATION.md shows a maintainer adding to the reference) compiled against
the reference's own headers and run against the reference's own
run_fused_block: every fused block of the fixtures, planned by the
reference's tune() for its titan_xp model, must give bit-identical stored
tensors on the B200 (fp32_exact), and a foreign plan must be refused with
ErrorKind::validation (fused_exec.cpp:33-38)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "binding_test")
GRAPHS = ["a1", "a2", "b1", "c1", "residual", "inc3a", "squeezenet11"]


def test_integration_doc_shows_the_compiled_binding():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    src = open(os.path.join(ROOT, "tests", "cpp", "fused_exec_b200.cpp")).read()
    assert src.strip() in doc, "INTEGRATION.md must show tests/cpp/fused_exec_b200.cpp verbatim"


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent (GPU box)")
def test_binding_compiles_against_the_reference_headers():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_binding_matches_reference_run_fused_block():
    if not os.path.exists(BIN):
        pytest.skip("binding_test not built (needs the reference headers at build time)")
    from paper_2007_06000_b200 import graph_path
    dev = os.path.join(ROOT, "paper_2007_06000_b200", "devices", "b200.device")
    r = subprocess.run([BIN, "--device", dev] + [graph_path(g) for g in GRAPHS], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "MISMATCH" not in r.stdout and "wrong kind" not in r.stdout
    assert "bit-identical" in r.stdout
    assert "tune on b200" in r.stdout  # plans of the reference's tuner for the committed B200 device document
