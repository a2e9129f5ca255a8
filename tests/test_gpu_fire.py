"""GPU tests of the fire kernel (kernels_fire.cu): split blocks -- a 1x1
squeeze staged on chip as a zero-bordered plane, expand convs read at shifted
plane addresses -- in one persistent tcgen05 kernel.

* every SqueezeNet fire module's concat output against the generic
  fused-block kernel (option no_fire=1) and the network output against the
  CPU oracle, at batches whose units straddle the persistent grid unevenly;
* the result does not depend on the unit shape or channel split: G whole
  images, R-row bands and 1 / 2 / 4 channel groups give bit-identical outputs
  (same MMA K order, same epilogue arithmetic);
* BASELINE config 3 (fire, N=32) and the fire-module fixture against the
  oracle;
* the measured-time tuner's fire entries round-trip through a tuning report;
  malformed / infeasible entries are refused and change nothing."""
import json

import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text

pytestmark = pytest.mark.gpu

TOL = {"bf16": 1e-2, "tf32": 1e-3}
PRECS = ["bf16", "tf32"]
FIRES = [f"fire{i}_concat" for i in range(2, 10)]


def _engine(name, prec, batch, opts=""):
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    e = X.Engine(X.Graph(text), O.flat_weights(og, w), "b200", prec, max_batch=batch, options=opts)
    return e, og, w


def _run(e, batch, names):
    import torch
    e.set_input_seeded(42, batch)
    e.forward(batch)
    out = {n: e.read(n, batch).cpu().numpy() for n in names}
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("batch", [3, 37])
def test_fire_kernel_matches_generic_and_oracle(prec, batch):
    e, og, w = _engine("squeezenet11", prec, batch)
    fires = [s for s in e.steps if s["tag"] == "fire"]
    # bf16: all eight fire modules; TF32 (fp32 operands, twice the bytes): at least fire2-fire5
    assert len(fires) == 8 if prec == "bf16" else len(fires) >= 4, [s["tag"] for s in e.steps]
    out = _run(e, batch, FIRES + ["pool10"])
    ref_e, _, _ = _engine("squeezenet11", prec, batch, "no_fire=1")
    assert not any(s["tag"] == "fire" for s in ref_e.steps)
    ref_out = _run(ref_e, batch, FIRES + ["pool10"])
    for n in FIRES + ["pool10"]:
        assert np.isfinite(out[n]).all(), n
        assert O.normwise(out[n], ref_out[n]) <= TOL[prec], (n, O.normwise(out[n], ref_out[n]))
    sample = [0, batch - 1]
    x = O.seeded_batch(og, 42, batch)[sample]
    ref = O.run_batch(og, x, w, ["pool10"])["pool10"]
    assert O.normwise(out["pool10"][sample], ref) <= TOL[prec]


@pytest.mark.parametrize("prec", PRECS)
def test_fire_unit_shapes_are_bitwise_identical(prec):
    batch = 5
    base = None
    seen = set()
    for opts in ["fire_nsplit=1,fire_g=1,fire_r=55", "fire_nsplit=1,fire_r=8", "fire_nsplit=2,fire_r=4", "fire_nsplit=2,fire_g=2",
                 "fire_nsplit=2,fire_g=3", "fire_nsplit=4,fire_g=1", "fire_nsplit=4,fire_r=7", "",
                 # 64-byte squeeze-input chunks (SWIZZLE_64B stages): same K order, same bits
                 "fire_cb=64,fire_nsplit=1,fire_r=8", "fire_cb=64,fire_nsplit=2,fire_g=2", "fire_cb=64,fire_sqs=1", "fire_cb=64",
                 # two CTAs per SM (4 epilogue warps, 256 TMEM columns each)
                 "fire_cps=2", "fire_cps=2,fire_nsplit=1,fire_r=4", "fire_cps=2,fire_nsplit=2,fire_g=2", "fire_cps=2,fire_stage=1"]:
        e, _, _ = _engine("squeezenet11", prec, batch, opts)
        cb = "64" if "fire_cb=64" in opts else "any"
        cb += ",cps2" if "fire_cps=2" in opts else ""
        cb += ",staged" if "fire_stage=1" in opts else ""
        shapes = (cb,) + tuple((s["id"], s["tile"][0], s["nsplit"]) for s in e.steps if s["tag"] == "fire")
        if not shapes or shapes in seen:
            continue
        seen.add(shapes)
        out = _run(e, batch, FIRES)
        # compare the fire outputs of steps that ran on the fire kernel in both engines
        fired = {s["layers"][0].split("_")[0] + "_concat" for s in e.steps if s["tag"] == "fire"}
        if base is None:
            base, base_fired = out, fired
            continue
        for n in sorted(fired & base_fired):
            # the first fire module's input is identical in both engines; later ones
            # are identical as long as every earlier module ran on the fire kernel
            earlier = [f for f in FIRES[:FIRES.index(n)]]
            if all(f in fired and f in base_fired for f in earlier):
                assert np.array_equal(out[n], base[n]), (opts, n)
    assert len(seen) >= (9 if prec == "bf16" else 8)


@pytest.mark.parametrize("name,batch,prec", [("fire", 32, "bf16"), ("fire", 32, "tf32"), ("b1", 3, "bf16"), ("b1", 3, "tf32")])
def test_fire_blocks_against_oracle(name, batch, prec):
    e, og, w = _engine(name, prec, batch)
    assert any(s["tag"] == "fire" for s in e.steps), [s["tag"] for s in e.steps]
    outs = _run(e, batch, og.outputs)
    sample = sorted({0, batch - 1})
    x = O.seeded_batch(og, 42, batch)[sample]
    ref = O.run_batch(og, x, w, og.outputs)
    for o in og.outputs:
        assert O.normwise(outs[o][sample], ref[o]) <= TOL[prec], (o, O.normwise(outs[o][sample], ref[o]))


@pytest.mark.parametrize("prec", PRECS)
def test_fire_tuning_report_roundtrip(prec):
    import torch
    e, og, w = _engine("squeezenet11", prec, 8)
    e.set_input_seeded(42, 8)
    e.forward(8, use_graph=False)
    report = e.autotune(8, reps=2, topk=1)
    fire_entries = [r for r in report if r.get("kernel") == "fire"]
    assert fire_entries and all({"nsplit", "G", "R"} <= set(r) for r in fire_entries)
    b, _, _ = _engine("squeezenet11", prec, 8)
    b.apply_tuning(json.dumps(report))
    key = lambda eng: [(s["id"], s["tile"], s["nsplit"]) for s in eng.steps]  # noqa: E731
    assert key(e) == key(b)
    outs = []
    for eng in (e, b):
        eng.set_input_seeded(42, 8)
        eng.forward(8)
        outs.append(eng.read("pool10", 8))
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    before = key(b)
    sid = fire_entries[0]["id"]
    for text, kind in [(f'[{{"id": "{sid}", "kernel": "fire", "nsplit": 2}}]', "parse"),
                       (f'[{{"id": "{sid}", "kernel": "fire", "nsplit": 3, "G": 1, "R": 4}}]', "infeasible"),
                       (f'[{{"id": "{sid}", "kernel": "fire", "nsplit": 1, "G": 0, "R": 4}}]', "infeasible"),
                       (f'[{{"id": "{sid}", "kernel": "fire", "nsplit": 1, "G": 1, "R": 4, "cb": 32}}]', "infeasible"),
                       (f'[{{"id": "{sid}", "kernel": "fire", "nsplit": 1, "G": 1, "R": 4}}, {{"id": "nope", "tile": [4, 4]}}]', "validation")]:
        with pytest.raises(X.XlfError) as ei:
            b.apply_tuning(text)
        assert ei.value.kind == kind, (text, ei.value)
        assert key(b) == before
