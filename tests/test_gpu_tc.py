"""GPU parity of the tensor-core path (tcgen05 implicit GEMM, fp32 accumulate
in TMEM) against the fp32 CPU oracle, for both operand types:

* bf16 (tcgen05.mma kind::f16): <= 1e-2 norm-wise;
* TF32 (kind::tf32, fp32 storage rounded to TF32 once at each producer):
  <= 1e-3 norm-wise;

norm-wise = max|d| / max|ref| (the BASELINE tolerances; the
element-wise compare() is undefined at the ReLU kink).  Activations and
weights are rounded at every HBM / shared-memory hand-off."""
import os

import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text
from tests.test_gpu_parity import EDGE, he_weights, run, structured_inputs

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "tf32": 1e-3}
PRECS = ["bf16", "tf32"]
SMALL = ["a1", "a2", "b1", "c1", "fire", "inc3a", "merge", "residual", "straight"]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("part", ["b200", "reference", "unfused"])
@pytest.mark.parametrize("name", SMALL)
def test_tc_within_tolerance(name, part, prec):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 2)
    ref = O.run_batch(og, x, w, og.outputs)
    out, e = run(name, O.flat_weights(og, w), 2, part, prec, x=x)
    for o in og.outputs:
        err = O.normwise(out[o], ref[o])
        assert err <= TOL[prec], (name, part, o, err)


@pytest.mark.parametrize("prec", PRECS)
def test_tc_squeezenet_b256_sampled(prec):
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, 256)
    out, _ = run("squeezenet11", O.flat_weights(og, w), 256, "b200", prec, x=x)
    sample = [0, 131, 255]
    ref = O.run_batch(og, x[sample], w, ["pool10"], threads=3)["pool10"]
    got = out["pool10"][sample]
    assert O.normwise(got, ref) <= TOL[prec]


def decisive_argmax(got, ref, tol):
    """Argmax agreement under a norm-wise error bound: where the reference's
    top-1 / top-2 margin exceeds 2 * tol * max|ref| no result within the
    tolerance can flip the argmax, so those images MUST agree; returns
    (decisive mask, agreement on all images)."""
    ref, got = ref.reshape(len(ref), -1), got.reshape(len(got), -1)
    top2 = np.sort(ref, 1)[:, -2:]
    bound = tol * np.abs(ref).max()
    decisive = (top2[:, 1] - top2[:, 0]) > 2 * bound
    agree = got.argmax(1) == ref.argmax(1)
    return decisive, agree


@pytest.mark.parametrize("prec", PRECS)
def test_tc_squeezenet_autotuned_b256_argmax(prec):
    """The configuration bench.py times: SqueezeNet v1.1, 256 images, the
    measured-time tuned plan, with He-init weights and structured inputs so
    the argmax is non-degenerate; every image's logits against the fp32
    oracle (north_star: identical argmax on SqueezeNet logits)."""
    import torch
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = he_weights(og)
    x = structured_inputs(og, 256)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=256)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(256, use_graph=False)
    assert e.autotune(256, reps=2, topk=2)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(256)
    got = e.read("pool10", 256).cpu().numpy()
    ref = O.run_batch(og, x, w, ["pool10"], threads=os.cpu_count() or 1)["pool10"]
    assert O.normwise(got, ref) <= TOL[prec]
    decisive, agree = decisive_argmax(got, ref, TOL[prec])
    assert decisive.mean() > 0.5, "margin rule would be vacuous"
    assert agree[decisive].all(), np.nonzero(decisive & ~agree)
    # images whose top-2 margin is inside the error bound may flip; they
    # must be rare (bf16 measured: 6 of 256, all indecisive)
    assert agree.mean() >= 0.95, agree.mean()
    assert len(set(ref.reshape(256, -1).argmax(1).tolist())) > 1  # non-degenerate


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name,batch", [("straight", 1), ("merge", 8), ("fire", 32), ("inc3a", 64)])
def test_tc_baseline_configs(name, batch, prec):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    out, _ = run(name, O.flat_weights(og, w), batch, "b200", prec, x=x)
    o = og.outputs[0]
    sample = sorted({0, batch // 2, batch - 1})
    ref = O.run_batch(og, x[sample], w, [o], threads=4)[o]
    assert O.normwise(out[o][sample], ref) <= TOL[prec]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("part", ["b200", "unfused"])
def test_tc_edge_graph(part, prec):
    og = O.load_graph(EDGE)
    w = O.seeded_weights(og, 11)
    x = O.seeded_batch(og, 13, 3)
    names = ["rect", "ap", "sum"]
    ref = O.run_batch(og, x, w, names)
    out, _ = run(EDGE, O.flat_weights(og, w), 3, part, prec, x=x, names=names)
    for n in names:
        assert O.normwise(out[n], ref[n]) <= TOL[prec], (part, n)


@pytest.mark.parametrize("prec", PRECS)
def test_tc_uses_tensor_cores(prec):
    g = X.Graph(graph_text("fire"))
    # forced whole-block fusion: one split kernel; by default the cost model
    # may split the block into squeeze + expands (TF32 at batch 32)
    plan = X.device_plan(g, "b200", 32, prec, options={"always_fuse": 1})
    assert [s["tag"] for s in plan["steps"]] == ["split"]
    plan = X.device_plan(g, "b200", 32, prec)
    assert [s["tag"] for s in plan["steps"]] in (["split"], ["conv", "multi-branch"])


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["fire", "inc3a", "merge", "straight"])
def test_tc_autotuned_within_tolerance(name, prec):
    """The measured-time tuner changes tiles / staging / weight residency /
    grid shape only: results stay within tolerance."""
    import torch
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 4)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=4)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(4)
    chosen = e.autotune(4, reps=2, topk=3)
    assert chosen and all(c["us"] > 0 for c in chosen)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(4)
    ref = O.run_batch(og, x, w, og.outputs)
    for o in og.outputs:
        err = O.normwise(e.read(o, 4).cpu().numpy(), ref[o])
        assert err <= TOL[prec], (name, o, err)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_tc_run_host_pipelined_matches_device_path(chunks, prec):
    """run_host pipelines H2D / compute / D2H over image chunks (tensor-core
    plans): the result equals the device-resident forward of the same inputs."""
    import torch
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 7, 6)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=6, options={"e2e_chunks": chunks})
    host = e.run_host(x, "pool10")
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(6)
    dev = e.read("pool10", 6).cpu().numpy()
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name,batch", [("squeezenet11", 8), ("inc3a", 4), ("fire", 6)])
def test_tc_forwards_are_bitwise_reproducible(name, batch, prec):
    """Race detector: repeated forwards (graph and direct launches) over the
    same input give bit-identical tensors -- the persistent pipeline's
    barriers, TMEM reuse and staging buffers leave no timing dependence."""
    import torch
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", prec, max_batch=batch)
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
    {"xbuf": 1, "wres": 0},
    {"xbuf": 2, "wres": 1},
    {"xbuf": 2, "tsets": 2},
    {"xbuf": 1, "wres": 1, "ctas": 1},
    # the earlier synchronisation structure: shared TMEM columns for every
    # group, a tile's first group waiting for the previous tile's last unit,
    # staging buffers released by the epilogue warps
    {"no_tsep": 1, "no_pwait": 1, "xrel_epi": 1},
    {"no_nalt": 1, "xbuf": 2},
    # output channels split over the grid's y dimension (channel groups with
    # resident weight slices; two-stage blocks recompute their producer)
    {"nsplit": 2, "always_fuse": 1},
    {"nsplit": 4, "wres": 0},
    {"nsplit": 8, "xbuf": 2, "tsets": 2},
]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("opts", FORCED, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
@pytest.mark.parametrize("name", ["fire", "inc3a", "straight", "residual", "squeezenet11"])
def test_tc_forced_configurations(name, opts, prec):
    """Every staging / weight-residency / accumulator-set / occupancy mode the
    tuner may pick computes the same function (tolerance vs the oracle)."""
    import torch
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    batch = 3
    x = O.seeded_batch(og, 5, batch)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch, options=opts)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(batch)
    sample = [0, batch - 1]
    ref = O.run_batch(og, x[sample], w, og.outputs, threads=2)
    for o in og.outputs:
        err = O.normwise(e.read(o, batch).cpu().numpy()[sample], ref[o])
        assert err <= TOL[prec], (name, opts, o, err)


WIDE = "name wide\ninput {\n  name d\n  shape [64, 20, 20]\n}\n" + "".join(
    f"layer {{\n  name c{i}\n  kind conv\n  inputs [d]\n  out_channels {16 + 8 * i}\n  kernel [1, 1]\n  activation relu\n}}\n"
    for i in range(6)) + "layer {\n  name cat\n  kind concat\n  inputs [c0, c1, c2, c3, c4, c5]\n}\noutput cat\n"


@pytest.mark.parametrize("prec", PRECS)
def test_tc_many_parallel_branches(prec):
    """Six 1x1 branches on one input run as one multi-branch kernel whose MMA
    group holds more ops than it has per-op accumulator barriers (the last
    barrier covers the rest): results within tolerance."""
    import torch
    og = O.load_graph(WIDE)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 3)
    g = X.Graph(WIDE)
    # mb_pw=1: merge the 1x1 branches although each alone would run on the pointwise kernel
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=3, options="mb_pw=1")
    assert any(len(s["layers"]) >= 5 for s in e.steps), [s["layers"] for s in e.steps]
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(3)
    ref = O.run_batch(og, x, w, ["cat"])
    err = O.normwise(e.read("cat", 3).cpu().numpy(), ref["cat"])
    assert err <= TOL[prec], err


@pytest.mark.parametrize("prec", PRECS)
def test_tc_tuning_report_roundtrip(prec):
    """A tuning report saved from one engine re-applied to a fresh engine of
    the same model gives the same step configurations and bit-identical
    results (the tuned plan as a reusable artifact); malformed or infeasible
    reports are refused and leave the engine unchanged."""
    import json
    import torch
    g = X.load_graph(X.graph_path("fire"))
    w = X.seeded_weights(g, 42)
    # one fused split step (its expand3 op is the widest: a 1 KB ring chunk is
    # smaller than one of its K steps)
    # (the generic fused-block kernel's configurations: the fire kernel's are
    # covered by test_gpu_fire.py)
    a = X.Engine(g, w, "b200", prec, max_batch=8, options="always_fuse=1,no_fire=1")
    a.set_input_seeded(42, 8)
    a.forward(8, use_graph=False)
    report = a.autotune(8, reps=2, topk=2)
    b = X.Engine(g, w, "b200", prec, max_batch=8, options="always_fuse=1,no_fire=1")
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
    before = [{k: s[k] for k in keys} for s in b.steps]
    sid = report[0]["id"]
    bad = [
        ('[{"id": "nope", "tile": [4, 4]}]', "validation"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "nxb": 3}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "tsets": 3}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "wres": 0, "ring_slots": 0}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "wres": 0, "ring_slots": 99}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "wres": 0, "ring_chunk": 1024}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4], "epi_warps": 6}}]', "infeasible"),
        (f'[{{"id": "{sid}", "tile": [4, 4]}}, {{"id": "nope", "tile": [4, 4]}}]', "validation"),  # 2nd entry bad: nothing applied
    ]
    for text, kind in bad:
        with pytest.raises(X.XlfError) as ei:
            b.apply_tuning(text)
        assert ei.value.kind == kind, (text, ei.value)
        assert [{k: s[k] for k in keys} for s in b.steps] == before
    b.set_input_seeded(42, 8)
    b.forward(8)
    torch.cuda.synchronize()
    assert torch.equal(b.read(g.outputs[0], 8), outs[0])


@pytest.mark.parametrize("prec", PRECS)
def test_tc_rewritten_input_is_not_readable(prec):
    """The tensor-core plan holds SqueezeNet's input in a space-to-depth
    layout (conv1 rewritten to stride 1): reading it back is refused instead
    of writing a 16x112x112 tensor into a 3x224x224 buffer."""
    g = X.load_graph(X.graph_path("squeezenet11"))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", prec, max_batch=2)
    e.set_input_seeded(42, 2)
    e.forward(2)
    with pytest.raises(X.XlfError):
        e.read("data", 2)
    with pytest.raises(X.XlfError):
        e.read("pool10", 3)  # batch beyond max_batch


@pytest.mark.parametrize("prec", PRECS)
def test_stem_kernel_matches_generic_path(prec):
    """SqueezeNet conv1 + pool1 run by the stem kernel (kernels_stem.cu) vs the
    generic fused-block kernel (option no_stem=1): both within the tolerance
    of the oracle on pool1, for a batch whose bands straddle the persistent
    grid unevenly (37 images), and the TF32 stem bit-identical to the generic
    path (max commutes with the monotone bias / ReLU / rounding)."""
    import torch
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.flat_weights(og, O.seeded_weights(og, 42))
    g = X.Graph(text)
    outs = {}
    for opt in ("", "no_stem=1"):
        e = X.Engine(g, w, "b200", prec, max_batch=37, options=opt)
        assert ("stem" in [s["tag"] for s in e.steps]) == (opt == "")
        e.set_input_seeded(42, 37)
        e.forward(37)
        outs[opt] = e.read("pool1", 37).cpu().numpy()
    torch.cuda.synchronize()
    x = O.seeded_batch(og, 42, 37)[[0, 18, 36]]
    ref = O.run_batch(og, x, O.seeded_weights(og, 42), ["pool1"])["pool1"]
    for o in outs.values():
        assert O.normwise(o[[0, 18, 36]], ref) <= TOL[prec]
    if prec == "tf32":
        assert np.array_equal(outs[""], outs["no_stem=1"])


@pytest.mark.parametrize("prec", PRECS)
def test_nsplit_matches_unsplit(prec):
    """Channel groups compute the unsplit function: SqueezeNet logits with
    every splittable step forced to 2 / 4 groups equal the unsplit plan up to
    the summation order of the global-average-pool partial sums, which
    follows the tile choice (the per-element arithmetic is identical: same
    MMA K order, same epilogue)."""
    import torch
    g = X.load_graph(X.graph_path("squeezenet11"))
    w = X.seeded_weights(g, 42)
    outs = []
    for opt in ("nsplit=1", "nsplit=2", "nsplit=4"):
        e = X.Engine(g, w, "b200", prec, max_batch=5, options=opt)
        if opt != "nsplit=1":
            assert any(s["nsplit"] > 1 for s in e.steps), opt
        e.set_input_seeded(42, 5)
        e.forward(5)
        outs.append(e.read("pool10", 5).cpu().numpy())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert O.normwise(o, outs[0]) <= 1e-6


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("batch,opts", [(3, ""), (37, ""), (5, "nsplit=4"), (37, "pw_mc=1")])
def test_pointwise_gemm_kernel(prec, batch, opts):
    """1x1 convs through the pointwise GEMM kernel (kernels_pw.cu: pixels of
    all images as one M dimension, M tiles crossing image boundaries; conv10 +
    global average pool with per-warp, per-image partial sums) against the
    generic kernel (no_pw=1) and the oracle, at batches whose tiles straddle
    images unevenly; pw_mc=1 runs the channel groups of an M tile as one
    cluster with the input chunks multicast."""
    import torch
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = O.flat_weights(og, O.seeded_weights(og, 42))
    g = X.Graph(text)
    outs = {}
    for key in (opts, "no_pw=1"):  # (no_fire: the squeezes are pointwise steps of their own)
        opt = "no_fire=1" + ("," + key if key else "")
        e = X.Engine(g, w, "b200", prec, max_batch=batch, options=opt)
        tags = [s["tag"] for s in e.steps]
        assert ("pointwise+gap" in tags) == ("no_pw=1" not in opt), tags
        e.set_input_seeded(42, batch)
        e.forward(batch)
        outs[key] = {n: e.read(n, batch).cpu().numpy() for n in ("fire9_squeeze", "pool10")}
    torch.cuda.synchronize()
    sample = [0, batch - 1]
    x = O.seeded_batch(og, 42, batch)[sample]
    ref = O.run_batch(og, x, O.seeded_weights(og, 42), ["fire9_squeeze", "pool10"])
    # the network output against the oracle (the tolerance's scope); the deep
    # intermediate against the generic kernel: both paths accumulate the same
    # 20 layers of bf16 / TF32 rounding before it
    assert O.normwise(outs[opts]["pool10"][sample], ref["pool10"]) <= TOL[prec]
    for n in ("fire9_squeeze", "pool10"):
        assert O.normwise(outs[opts][n], outs["no_pw=1"][n]) <= TOL[prec], n
