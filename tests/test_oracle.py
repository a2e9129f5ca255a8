"""Pins the CPU oracle (oracle/xlf_oracle.c + oracle/oracle.py) before it is
trusted as the checker: against the golden vectors generated from the
unmodified reference (tests/golden/make_golden.py) and, when the reference
library is built here, against the reference itself."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R
from tests.conftest import graph_text

SMALL = ["a1", "a2", "b1", "c1", "fire", "inc3a", "merge", "residual", "straight"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


@pytest.mark.parametrize("name", SMALL + ["squeezenet11"])
def test_oracle_matches_reference_goldens(golden, name):
    ent = golden["ours"][name]
    g = O.load_graph(graph_text(name))
    w = O.seeded_weights(g, ent["seed"])
    assert sha(O.flat_weights(g, w)) == ent["weights"]["sha256"]
    x = O.seeded_batch(g, ent["seed"], ent["batch"])
    assert sha(x) == ent["input"]["sha256"]
    names = [l.name for l in g.layers]
    outs = O.run_batch(g, x, w, names, threads=4)
    for n in names:
        d = ent["outputs"][n]
        assert list(outs[n].shape) == d["shape"], n
        assert sha(outs[n]) == d["sha256"], f"{name}/{n} differs from the reference bit pattern"


def test_stream_random_access_matches_sequential():
    a = O.stream(42, 0, 1000)
    b = O.stream(42, 500, 500)
    assert np.array_equal(a[500:], b)
    assert O.stream(0, 0, 4).tolist() == O.stream(0x9E3779B97F4A7C15, 0, 4).tolist()  # seed 0 -> golden ratio
    assert a.min() >= -0.5 and a.max() < 0.5


def test_pool_zero_padding_semantics():
    # maxpool pads with 0.0 (not -inf), avg divides by the full window
    # (reference.cpp:73-83): an all-negative 2x2 map, 3x3/s1/p1 window.
    x = np.full((1, 2, 2), -1.0, np.float32)
    mx = O.pool(x, dict(kind="max", k=3, stride=1, pad=1))
    av = O.pool(x, dict(kind="avg", k=3, stride=1, pad=1))
    assert np.all(mx == 0.0)
    assert np.allclose(av, -4.0 / 9.0)


def test_compare_metric():
    a = np.array([1.0, 0.0, -2.0], np.float32)
    b = np.array([1.0, 1e-7, -2.5], np.float32)
    ma, mr = O.compare(a, b)
    assert ma == pytest.approx(0.5)
    assert mr == pytest.approx(0.2)  # |0.5| / 2.5; the 1e-7 pair is floored at 1e-6 -> 0.1


@pytest.mark.skipif(not R.available(), reason="reference library not built (oracle/_ref)")
@pytest.mark.parametrize("name", ["b1", "fire", "straight", "inc3a", "residual"])
def test_oracle_matches_reference_library(name):
    text = graph_text(name)
    g = O.load_graph(text)
    w = O.seeded_weights(g, 7)
    x = O.seeded_batch(g, 9, 2)
    for o in g.outputs:
        mine = O.run_batch(g, x, w, [o])[o]
        theirs = R.run(text, x, o, g.shape_of(o), weights=O.flat_weights(g, w))
        assert np.array_equal(mine, theirs)
        # and the reference's own fused interpreter agrees with its oracle
        sim = R.run(text, x, o, g.shape_of(o), weights=O.flat_weights(g, w), mode=1)
        assert np.array_equal(sim, theirs)


@pytest.mark.skipif(not R.available(), reason="reference library not built (oracle/_ref)")
def test_out_dim_truncates_like_the_reference():
    """conv_out_dim (graph.cpp:76-78) divides in C++ int arithmetic: a 3-wide
    pool over a 2-wide input gives width (2-3)/2+1 = 1, not floor's 0, and the
    window reads the zero padding beyond the edge."""
    text = ("name trunc\ninput {\n  name d\n  shape [5, 7, 2]\n}\n"
            "layer {\n  name p\n  kind pool\n  inputs [d]\n  pool max\n  kernel 3\n  stride 2\n}\n"
            "layer {\n  name c\n  kind conv\n  inputs [d]\n  out_channels 3\n  kernel [3, 3]\n  stride 2\n}\n"
            "output p\noutput c\n")
    g = O.load_graph(text)
    assert g.shape_of("p") == (5, 3, 1) and g.shape_of("c") == (3, 3, 1)
    w = O.seeded_weights(g, 3)
    x = O.seeded_batch(g, 4, 2)
    for o in ("p", "c"):
        mine = O.run_batch(g, x, w, [o])[o]
        theirs = R.run(text, x, o, g.shape_of(o), weights=O.flat_weights(g, w))
        assert np.array_equal(mine, theirs), o
    with pytest.raises(ValueError):
        O.load_graph(text.replace("shape [5, 7, 2]", "shape [5, 7, 0]"))
