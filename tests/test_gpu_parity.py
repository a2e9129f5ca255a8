"""GPU parity of the sm_100a path against the reference (via the C ABI).

* fp32_exact must be BIT-IDENTICAL to the reference's run_reference: compared
  against the sha256 of the reference's own outputs (tests/golden) and
  against the oracle on fresh inputs;
* fp32 (FFMA) within 1e-5 norm-wise (max|d| / max|ref|);
* full BASELINE sizes through size-independent properties (every image equals
  the same image run alone; sampled images equal the oracle).
"""
import hashlib

import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text

pytestmark = pytest.mark.gpu

SMALL = ["a1", "a2", "b1", "c1", "fire", "inc3a", "merge", "residual", "straight"]
PARTS = ["reference", "b200", "unfused"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def run(name_or_text, weights, batch, part, prec, seed=42, names=None, x=None):
    import torch
    text = graph_text(name_or_text) if "\n" not in name_or_text else name_or_text
    g = X.Graph(text)
    e = X.Engine(g, weights, part, prec, max_batch=batch)
    if x is None:
        e.set_input_seeded(seed, batch)
    else:
        e.set_input(torch.from_numpy(x).cuda())
    e.forward(batch)
    names = names or g.outputs
    out = {n: e.read(n, batch).cpu().numpy() for n in names if n in e.materialized()}
    torch.cuda.synchronize()
    return out, e


@pytest.mark.parametrize("part", PARTS)
@pytest.mark.parametrize("name", SMALL + ["squeezenet11"])
def test_fp32_exact_is_bitwise_the_reference(golden, name, part):
    ent = golden["ours"][name]
    g = X.Graph(graph_text(name))
    w = X.seeded_weights(g, ent["seed"])
    out, e = run(name, w, ent["batch"], part, "fp32_exact", seed=ent["seed"], names=[l["name"] for l in g.layers])
    checked = 0
    for n, a in out.items():
        assert sha(a) == ent["outputs"][n]["sha256"], f"{name}/{part}: {n} is not bit-identical to the reference"
        checked += 1
    assert checked >= len(g.outputs)


@pytest.mark.parametrize("name", SMALL)
def test_fp32_ffma_within_1e5(name):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, 2)
    ref = O.run_batch(og, x, w, og.outputs)
    for part in ("b200", "reference"):
        out, _ = run(name, O.flat_weights(og, w), 2, part, "fp32", x=x)
        for o in og.outputs:
            assert O.normwise(out[o], ref[o]) <= 1e-5, (name, part, o)


@pytest.mark.parametrize("name,batch", [("squeezenet11", 4), ("inc3a", 4), ("straight", 1), ("merge", 8), ("a1", 2)])
def test_fp32_autotuned_plans_stay_exact(golden, name, batch):
    """The fp32 tuner (tiles x register-blocked convs on / off, engine.cpp
    autotune_fp32) changes only the work split, never an output's
    accumulation order: fp32_exact stays bit-identical to the oracle and FFMA
    within 1e-5, and the report re-applies to a fresh engine unchanged."""
    import torch
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    ref = O.run_batch(og, x, w, og.outputs, threads=4)
    g = X.Graph(text)
    for prec in ("fp32_exact", "fp32"):
        e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch)
        e.set_input(torch.from_numpy(x).cuda())
        e.forward(batch, use_graph=False)
        report = e.autotune(batch, reps=1, topk=2)
        assert report and all(r["kernel"] == "fp32" and r["tried"] >= 1 for r in report)
        e.forward(batch)
        out = e.read(g.outputs[0], batch).cpu().numpy()
        r = ref[og.outputs[0]]
        if prec == "fp32_exact":
            assert np.array_equal(out, r), f"{name}: tuned fp32_exact plan differs from the oracle"
        else:
            assert O.normwise(out, r) <= 1e-5
        e2 = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch)
        e2.apply_tuning(report)
        key = lambda st: [(s["tile"], s.get("rb"), s.get("threads")) for s in st]  # noqa: E731
        assert key(e2.steps) == key(e.steps)
        e2.set_input(torch.from_numpy(x).cuda())
        e2.forward(batch)
        assert np.array_equal(e2.read(g.outputs[0], batch).cpu().numpy(), out)
        # the other CTA size and register blocking on the tuned tiles: same bits
        for rb, nt in ((0, 512), (1, 512), (1, 256)):
            alt = [dict(r, rb=rb, threads=nt) for r in report]
            e3 = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch)
            try:
                e3.apply_tuning(alt)
            except X.XlfError:
                continue  # a 512-thread CTA at this tile may exceed shared memory: reported, not run
            e3.set_input(torch.from_numpy(x).cuda())
            e3.forward(batch)
            assert np.array_equal(e3.read(g.outputs[0], batch).cpu().numpy(), out), (name, prec, rb, nt)
    torch.cuda.synchronize()


NONSQUARE = "name nonsquare\ninput {\n  name d\n  shape [12, 14, 14]\n}\n" + "".join(
    f"layer {{\n  name {n}\n  kind conv\n  inputs [{i}]\n  out_channels {c}\n  kernel [{kh}, {kw}]\n  pad 0\n  activation relu\n}}\n"
    for n, i, c, kh, kw in [("k31", "d", 16, 3, 1), ("k13", "k31", 24, 1, 3), ("k51", "k13", 16, 5, 1), ("k15", "k51", 8, 1, 5),
                            ("k35", "d", 16, 3, 5), ("k53", "k35", 8, 5, 3)]) + "output k15\noutput k53\n"


@pytest.mark.parametrize("part", ["b200", "unfused"])
def test_nonsquare_kernels_exact(part):
    """k x 1 / 1 x k / 3x5 / 5x3 convs (shapes outside the register-blocked
    instantiations, or inside with kh != kw): fp32_exact bit for bit, planner
    choice and every tuned variant."""
    import torch
    og = O.load_graph(NONSQUARE)
    w = O.seeded_weights(og, 4)
    x = O.seeded_batch(og, 6, 3)
    names = [l.name for l in og.layers]
    ref = O.run_batch(og, x, w, names)
    g = X.Graph(NONSQUARE)
    e = X.Engine(g, O.flat_weights(og, w), part, "fp32_exact", max_batch=3)
    e.set_input(torch.from_numpy(x).cuda())
    for tune in (False, True):
        if tune:
            e.autotune(3, reps=1, topk=2)
        e.forward(3)
        for n in names:
            if n in e.materialized():
                assert np.array_equal(e.read(n, 3).cpu().numpy(), ref[n]), (part, tune, n)
    torch.cuda.synchronize()


# BASELINE configs at their full batch: C1 straight N=1, C2 merge N=8,
# C3 fire N=32, C4 inception-3a N=64 (fp32 here; bf16/TF32 tolerance tests
# live with the tensor-core path).
@pytest.mark.parametrize("name,batch,sample", [("straight", 1, [0]), ("merge", 8, list(range(8))),
                                               ("fire", 32, [0, 13, 31]), ("inc3a", 64, [0, 42, 63])])
def test_baseline_configs_full_batch(name, batch, sample):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    out, _ = run(name, O.flat_weights(og, w), batch, "b200", "fp32_exact", x=x)
    o = og.outputs[0]
    ref = O.run_batch(og, x[sample], w, [o], threads=8)[o]
    assert np.array_equal(out[o][sample], ref)
    # every image equals the same image computed alone (batch independence)
    alone, _ = run(name, O.flat_weights(og, w), 1, "b200", "fp32_exact", x=x[batch - 1:batch])
    assert np.array_equal(out[o][batch - 1], alone[o][0])


def he_weights(og, seed=42):
    """Fan-in scaled weights so the logits (and their argmax) are not
    degenerate (SURVEY finding 7: U[-0.5,0.5) weights give class 288 for every
    input): He-uniform (bound sqrt(6/fan_in)) from the seeded stream, zero
    bias -- the signal survives SqueezeNet's 26 layers."""
    w = O.seeded_weights(og, seed)
    for l in og.layers:
        if l.kind == "conv":
            f, b = w[l.name]
            fan = f.shape[1] * f.shape[2] * f.shape[3]
            w[l.name] = ((f * np.float32(2.0 * np.sqrt(6.0 / fan))).astype(np.float32), (b * np.float32(0.0)).astype(np.float32))
    return w


def structured_inputs(og, n, seed=42):
    """Seeded noise plus a per-image, per-channel offset, so images differ in
    more than i.i.d. noise and the argmax varies."""
    c = og.inputs[0][1][0]
    x = O.seeded_batch(og, seed, n)
    return (x + (O.stream(7, 0, n * c).reshape(n, c, 1, 1) * 4.0)).astype(np.float32)


def test_squeezenet_b256_exact_sampled_and_argmax():
    text = graph_text("squeezenet11")
    og = O.load_graph(text)
    w = he_weights(og)
    flat = O.flat_weights(og, w)
    import torch
    g = X.Graph(text)
    e = X.Engine(g, flat, "b200", "fp32_exact", max_batch=256)
    x = structured_inputs(og, 256)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(256)
    logits = e.read("pool10", 256).cpu().numpy().reshape(256, 1000)
    sample = [0, 77, 255]
    ref = O.run_batch(og, x[sample], w, ["pool10"], threads=3)["pool10"].reshape(len(sample), 1000)
    assert np.array_equal(logits[sample], ref)
    assert np.array_equal(logits[sample].argmax(1), ref.argmax(1))
    assert len(set(np.argmax(logits, 1).tolist())) > 1  # non-degenerate
    torch.cuda.synchronize()


def test_partitions_agree_bitwise_on_squeezenet():
    text = graph_text("squeezenet11")
    g = X.Graph(text)
    w = X.seeded_weights(g, 1)
    outs = [run(text, w, 4, p, "fp32_exact", seed=2)[0]["pool10"] for p in PARTS]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


# ---------------------------------------------------------------- edge cases

EDGE = """name edge
input {
  name d
  shape [5, 9, 7]
}
layer {
  name s2
  kind conv
  inputs [d]
  out_channels 6
  kernel [3, 3]
  pad 1
  stride 2
  group 1
  bias false
  activation relu
}
layer {
  name dw
  kind conv
  inputs [s2]
  out_channels 6
  kernel [3, 3]
  pad 1
  stride 1
  group 6
  bias true
  activation none
}
layer {
  name rect
  kind conv
  inputs [s2]
  out_channels 3
  kernel [1, 3]
  pad 0
  stride 1
  group 1
  bias true
  activation relu
}
layer {
  name mp
  kind pool
  inputs [d]
  pool max
  kernel 3
  stride 1
  pad 1
}
layer {
  name ap
  kind pool
  inputs [mp]
  pool avg
  kernel 2
  stride 2
  pad 1
}
layer {
  name r
  kind relu
  inputs [dw]
}
layer {
  name sum
  kind add
  inputs [dw, r]
}
output rect
output sum
output ap
"""


@pytest.mark.parametrize("part", PARTS)
@pytest.mark.parametrize("batch", [1, 3])
def test_edge_graph_exact(part, batch):
    """Ragged tiles, stride 2, grouped/depthwise, 1x3 kernels, no-bias,
    no-relu, channels not a multiple of 4, pool padding on raw inputs,
    standalone relu and add (reference.cpp:92-124)."""
    og = O.load_graph(EDGE)
    w = O.seeded_weights(og, 11)
    x = O.seeded_batch(og, 13, batch)
    names = ["s2", "dw", "rect", "mp", "ap", "sum"]
    ref = O.run_batch(og, x, w, names)
    out, e = run(EDGE, O.flat_weights(og, w), batch, part, "fp32_exact", x=x, names=names)
    for n in out:
        assert np.array_equal(out[n], ref[n]), (part, n)
    for o in og.outputs:
        assert o in out


def test_random_graphs_exact():
    """Seeded random conv/pool chains and fire-like splits with random
    shapes, kernels, strides and pads: bit-exact vs the oracle."""
    rng = np.random.default_rng(1234)
    for trial in range(6):
        C, H, W = int(rng.integers(1, 20)), int(rng.integers(5, 30)), int(rng.integers(5, 30))
        k = int(rng.choice([1, 3, 5]))
        pad = int(rng.integers(0, k // 2 + 1))
        s1 = int(rng.choice([1, 1, 2]))
        sq, e1, e3 = int(rng.integers(1, 24)), int(rng.integers(1, 40)), int(rng.integers(1, 40))
        text = (f"name rnd{trial}\ninput {{\n  name d\n  shape [{C}, {H}, {W}]\n}}\n"
                f"layer {{\n  name c0\n  kind conv\n  inputs [d]\n  out_channels {sq}\n  kernel [{k}, {k}]\n  pad {pad}\n"
                f"  stride {s1}\n  activation relu\n}}\n"
                f"layer {{\n  name a\n  kind conv\n  inputs [c0]\n  out_channels {e1}\n  kernel [1, 1]\n  activation relu\n}}\n"
                f"layer {{\n  name b\n  kind conv\n  inputs [c0]\n  out_channels {e3}\n  kernel [3, 3]\n  pad 1\n  activation relu\n}}\n"
                f"layer {{\n  name cat\n  kind concat\n  inputs [a, b]\n}}\n"
                f"layer {{\n  name p\n  kind pool\n  inputs [cat]\n  pool max\n  kernel 3\n  stride 2\n}}\n"
                "output p\n")
        try:
            og = O.load_graph(text)
        except ValueError:  # non-positive output dimension: the reference rejects it too
            continue
        w = O.seeded_weights(og, trial)
        x = O.seeded_batch(og, trial + 100, 2)
        ref = O.run_batch(og, x, w, ["cat", "p"])
        for part in PARTS:
            out, e = run(text, O.flat_weights(og, w), 2, part, "fp32_exact", x=x, names=["cat", "p"])
            for n in out:
                assert np.array_equal(out[n], ref[n]), (trial, part, n, text)
            if part == "b200":  # every tuned fp32 variant (tile, register blocking, CTA size): same bits
                import torch
                e.autotune(2, reps=1, topk=2)
                e.set_input(torch.from_numpy(x).cuda())
                e.forward(2)
                for n in out:
                    assert np.array_equal(e.read(n, 2).cpu().numpy(), ref[n]), (trial, "tuned", n, text)
