"""GPU parity of the bf16 tensor-core path (tcgen05 implicit GEMM, fp32
accumulate in TMEM) against the fp32 CPU oracle: <= 1e-2 norm-wise
(max|d| / max|ref|, the BASELINE BF16 tolerance).  Activations
and weights are rounded to bf16 at every HBM / shared-memory hand-off."""
import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text
from tests.test_gpu_parity import EDGE, run

pytestmark = pytest.mark.gpu

TOL = 1e-2
SMALL = ["a1", "a2", "b1", "c1", "fire", "inc3a", "merge", "residual", "straight"]


@pytest.mark.parametrize("part", ["b200", "reference", "unfused"])
@pytest.mark.parametrize("name", SMALL)
def test_bf16_within_tolerance(name, part):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 2)
    ref = O.run_batch(og, x, w, og.outputs)
    out, e = run(name, O.flat_weights(og, w), 2, part, "bf16", x=x)
    for o in og.outputs:
        err = O.normwise(out[o], ref[o])
        assert err <= TOL, (name, part, o, err)


def test_bf16_squeezenet_b256_sampled():
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, 256)
    out, _ = run("squeezenet11", O.flat_weights(og, w), 256, "b200", "bf16", x=x)
    sample = [0, 131, 255]
    ref = O.run_batch(og, x[sample], w, ["pool10"], threads=3)["pool10"]
    got = out["pool10"][sample]
    assert O.normwise(got, ref) <= TOL
    # argmax identical (SURVEY finding 7: degenerate under this init, still required)
    assert np.array_equal(got.reshape(3, -1).argmax(1), ref.reshape(3, -1).argmax(1))


@pytest.mark.parametrize("name,batch", [("straight", 1), ("merge", 8), ("fire", 32), ("inc3a", 64)])
def test_bf16_baseline_configs(name, batch):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    out, _ = run(name, O.flat_weights(og, w), batch, "b200", "bf16", x=x)
    o = og.outputs[0]
    sample = sorted({0, batch // 2, batch - 1})
    ref = O.run_batch(og, x[sample], w, [o], threads=4)[o]
    assert O.normwise(out[o][sample], ref) <= TOL


@pytest.mark.parametrize("part", ["b200", "unfused"])
def test_bf16_edge_graph(part):
    og = O.load_graph(EDGE)
    w = O.seeded_weights(og, 11)
    x = O.seeded_batch(og, 13, 3)
    names = ["rect", "ap", "sum"]
    ref = O.run_batch(og, x, w, names)
    out, _ = run(EDGE, O.flat_weights(og, w), 3, part, "bf16", x=x, names=names)
    for n in names:
        assert O.normwise(out[n], ref[n]) <= TOL, (part, n)


def test_bf16_uses_tensor_cores():
    g = X.Graph(graph_text("fire"))
    plan = X.device_plan(g, "b200", 32, "bf16")
    assert [s["tag"] for s in plan["steps"]] == ["split"]


@pytest.mark.parametrize("name", ["fire", "inc3a", "merge", "straight"])
def test_bf16_autotuned_within_tolerance(name):
    """The measured-time tuner changes tiles / staging / weight residency /
    grid shape only: results stay within the bf16 tolerance."""
    import torch
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 4)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", "bf16", max_batch=4)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(4)
    chosen = e.autotune(4, reps=2, topk=3)
    assert chosen and all(c["us"] > 0 for c in chosen)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(4)
    ref = O.run_batch(og, x, w, og.outputs)
    for o in og.outputs:
        err = O.normwise(e.read(o, 4).cpu().numpy(), ref[o])
        assert err <= TOL, (name, o, err)


@pytest.mark.parametrize("chunks", ["1", "3", "4"])
def test_bf16_run_host_pipelined_matches_device_path(chunks, monkeypatch):
    """run_host pipelines H2D / compute / D2H over image chunks (bf16 plans):
    the result equals the device-resident forward of the same inputs."""
    import torch
    monkeypatch.setenv("XLF_E2E_CHUNKS", chunks)
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 7, 6)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", "bf16", max_batch=6)
    host = e.run_host(x, "pool10")
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(6)
    dev = e.read("pool10", 6).cpu().numpy()
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("name,batch", [("squeezenet11", 8), ("inc3a", 4), ("fire", 6)])
def test_bf16_forwards_are_bitwise_reproducible(name, batch):
    """Race detector: repeated forwards (graph and direct launches) over the
    same input give bit-identical tensors -- the persistent pipeline's
    barriers, TMEM reuse and staging buffers leave no timing dependence."""
    import torch
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", "bf16", max_batch=batch)
    names = [n for n in e.materialized() if n not in dict(g.inputs)]
    outs = []
    for r in range(4):
        e.set_input_seeded(42, batch)
        e.forward(batch, use_graph=(r % 2 == 0))
        outs.append({n: e.read(n, batch).clone() for n in names})
    torch.cuda.synchronize()
    for n in names:
        for o in outs[1:]:
            assert torch.equal(outs[0][n], o[n]), n


FORCED = [
    {"XLF_XBUF": "1", "XLF_WRES": "0"},
    {"XLF_XBUF": "2", "XLF_WRES": "1"},
    {"XLF_XBUF": "2", "XLF_TSETS": "2"},
    {"XLF_XBUF": "1", "XLF_WRES": "1", "XLF_CTAS": "1"},
    # the earlier synchronisation structure: shared TMEM columns for every
    # group, a tile's first group waiting for the previous tile's last unit,
    # staging buffers released by the epilogue warps (XLF_DBG bit 16)
    {"XLF_NO_TSEP": "1", "XLF_NO_PWAIT": "1", "XLF_DBG": "16"},
    {"XLF_NO_NALT": "1", "XLF_XBUF": "2"},
]


@pytest.mark.parametrize("env", FORCED, ids=lambda d: ",".join(f"{k[4:]}={v}" for k, v in d.items()))
@pytest.mark.parametrize("name", ["fire", "inc3a", "straight", "residual", "squeezenet11"])
def test_bf16_forced_configurations(name, env, monkeypatch):
    """Every staging / weight-residency / accumulator-set / occupancy mode the
    tuner may pick computes the same function (bf16 tolerance vs the oracle)."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    batch = 3
    x = O.seeded_batch(og, 5, batch)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", "bf16", max_batch=batch)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(batch)
    sample = [0, batch - 1]
    ref = O.run_batch(og, x[sample], w, og.outputs, threads=2)
    for o in og.outputs:
        err = O.normwise(e.read(o, batch).cpu().numpy()[sample], ref[o])
        assert err <= TOL, (name, env, o, err)


WIDE = "name wide\ninput {\n  name d\n  shape [64, 20, 20]\n}\n" + "".join(
    f"layer {{\n  name c{i}\n  kind conv\n  inputs [d]\n  out_channels {16 + 8 * i}\n  kernel [1, 1]\n  activation relu\n}}\n"
    for i in range(6)) + "layer {\n  name cat\n  kind concat\n  inputs [c0, c1, c2, c3, c4, c5]\n}\noutput cat\n"


def test_bf16_many_parallel_branches():
    """Six 1x1 branches on one input run as one multi-branch kernel whose MMA
    group holds more ops than it has per-op accumulator barriers (the last
    barrier covers the rest): results within the bf16 tolerance."""
    import torch
    og = O.load_graph(WIDE)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 3)
    g = X.Graph(WIDE)
    e = X.Engine(g, O.flat_weights(og, w), "b200", "bf16", max_batch=3)
    assert any(len(s["layers"]) >= 5 for s in e.steps), [s["layers"] for s in e.steps]
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(3)
    ref = O.run_batch(og, x, w, ["cat"])
    err = O.normwise(e.read("cat", 3).cpu().numpy(), ref["cat"])
    assert err <= TOL, err


def test_bf16_tuning_report_roundtrip():
    """A tuning report saved from one engine re-applied to a fresh engine of
    the same model gives the same step configurations and bit-identical
    results (the tuned plan as a reusable artifact)."""
    import json
    import torch
    g = X.load_graph(X.graph_path("fire"))
    w = X.seeded_weights(g, 42)
    a = X.Engine(g, w, "b200", "bf16", max_batch=8)
    a.set_input_seeded(42, 8)
    a.forward(8, use_graph=False)
    report = a.autotune(8, reps=2, topk=2)
    b = X.Engine(g, w, "b200", "bf16", max_batch=8)
    b.apply_tuning(json.dumps(report))  # default separators: ", " / ": "
    keys = ("tile", "nxb", "wres", "ring_slots", "epi_warps", "tsets")
    assert [{k: s[k] for k in keys} for s in a.steps] == [{k: s[k] for k in keys} for s in b.steps]
    outs = []
    for e in (a, b):
        e.set_input_seeded(42, 8)
        e.forward(8)
        outs.append(e.read(g.outputs[0], 8))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    with pytest.raises(X.XlfError):
        b.apply_tuning('[{"id": "nope", "tile": [4, 4]}]')
