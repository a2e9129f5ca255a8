"""Planner / tiling parity with the reference (host only).

Mirrors the reference's own tests (proj/tests/test_fusion.cpp,
test_tiling.cpp, test_cost_model.cpp) and checks block reports, plans and
modelled store counts against the golden outputs of the reference planner."""
import os
import re

import numpy as np
import pytest

import paper_2007_06000_b200 as X
from tests.conftest import REFERENCE_FIXTURES, graph_text

OURS = ["a1", "a2", "b1", "c1", "fire", "inc3a", "merge", "residual", "squeezenet11", "straight"]


def g_of(name):
    return X.Graph(graph_text(name))


def plan_geo(text):
    m = re.search(r"tile \[(\d+), (\d+)\]\n\s*grid \[(\d+), (\d+)\]", text)
    th, tw, gh, gw = map(int, m.groups())
    return (th, tw), (gh, gw)


@pytest.mark.parametrize("name", OURS)
def test_block_report_plans_and_store_tx_match_reference(golden, name):
    ent = golden["ours"][name]
    g = g_of(name)
    assert X.block_assignment_report(g) == ent["block_report"]
    for bid, text in ent["plans"].items():
        tile, grid = plan_geo(text)
        assert X.plan_tiling(g, bid, tile, grid) == text
        assert list(X.store_transactions(g, bid)) == ent["store_tx"][bid]


@pytest.mark.skipif(not os.path.isdir(REFERENCE_FIXTURES), reason="reference fixtures absent")
@pytest.mark.parametrize("name", ["a1", "a2", "b1", "c1", "inception", "residual", "squeezenet"])
def test_reference_fixtures(golden, name):
    ent = golden["reference_fixtures"][name]
    g = X.Graph(open(os.path.join(REFERENCE_FIXTURES, name + ".graph")).read())
    assert X.block_assignment_report(g) == ent["block_report"]
    for bid, text in ent["plans"].items():
        tile, grid = plan_geo(text)
        assert X.plan_tiling(g, bid, tile, grid) == text
        assert list(X.store_transactions(g, bid)) == ent["store_tx"][bid]


def test_seeded_weights_match_golden(golden):
    import hashlib
    for name in OURS:
        w = X.seeded_weights(g_of(name), 42)
        assert hashlib.sha256(w.tobytes()).hexdigest() == golden["ours"][name]["weights"]["sha256"]


def count(blocks, mode):
    return sum(b.mode == mode for b in blocks)


def test_classify_mode_three_modes():  # test_fusion.cpp:77-92
    r = X.classify_mode(g_of("a1"), ["conv1", "conv2"])
    assert r.accepted and r.mode == "straight"
    r = X.classify_mode(g_of("b1"), ["fire_squeeze", "fire_expand1", "fire_expand3"])
    assert r.accepted and r.mode == "split"
    r = X.classify_mode(g_of("c1"), ["branch_a", "branch_b", "join"])
    assert r.accepted and r.mode == "merge"


def test_classify_mode_rejections():  # test_fusion.cpp:94-104
    r = X.classify_mode(g_of("residual"), ["conv1", "conv2", "conv3"])
    assert not r.accepted and "depth" in r.reject_reason
    r = X.classify_mode(g_of("b1"), ["fire_expand1", "fire_expand3", "fire_concat"])
    assert not r.accepted and "unsupported" in r.reject_reason


def test_squeezenet_v11_partition():
    g = g_of("squeezenet11")
    blocks = X.detect_fusion_blocks(g)
    assert count(blocks, "split") == 8 and count(blocks, "straight") == 0 and count(blocks, "merge") == 0
    seen = [m for b in blocks for m in b.members]
    assert sorted(seen) == sorted(l["name"] for l in g.layers)  # partition covers every layer once
    b2 = X.detect_fusion_blocks(g, "b200")
    assert count(b2, "split") == 8
    # B200 adds the conv1 -> pool1 straight block the reference rejects (fusion.cpp:66-69)
    assert any(b.members == ["conv1", "pool1"] for b in b2)


def test_inception_partitions():
    g = g_of("inc3a")
    ref = X.detect_fusion_blocks(g)
    assert count(ref, "straight") == 2  # r3->b3, r5->b5 (SURVEY finding 3)
    b2 = X.detect_fusion_blocks(g, "b200")
    assert any(b.members == ["mp", "bp"] for b in b2)  # pool producer, B200 only
    plan = X.device_plan(g, "b200", 64)
    fused = [s for s in plan["steps"] if s["kind"] == "fused"]
    assert len(fused) == 1 and fused[0]["tag"] == "multi-branch"  # one kernel, concat elided
    assert not plan["tensors"]["r3"]["materialized"] and not plan["tensors"]["mp"]["materialized"]
    assert plan["tensors"]["b3"]["alloc"] == plan["tensors"]["concat"]["alloc"]
    assert plan["tensors"]["b3"]["coff"] == 64 and plan["tensors"]["bp"]["coff"] == 224


def test_straight_and_merge_configs_form_no_reference_block():  # SURVEY finding 3
    assert all(not b.fused() for b in X.detect_fusion_blocks(g_of("straight")))
    assert all(not b.fused() for b in X.detect_fusion_blocks(g_of("merge")))
    st = X.device_plan(g_of("straight"), "b200", 1)
    assert [s["tag"] for s in st["steps"]] == ["straight+pool"]
    mg = X.device_plan(g_of("merge"), "b200", 8)
    assert [s["tag"] for s in mg["steps"]] == ["multi-branch"]


def test_residual_partition():  # test_fusion.cpp:134-144
    blocks = X.detect_fusion_blocks(g_of("residual"))
    merge = [b for b in blocks if "join" in b.members][0]
    assert merge.mode == "merge" and merge.producer_stage == ["conv3", "conv4"]
    assert [b for b in blocks if "conv5" in b.members][0].mode == "unfused"


def test_escaping_intermediate_flag():  # test_fusion.cpp:155-166
    text = ("name t\ninput {\n  name d\n  shape [2, 8, 8]\n}\n"
            "layer {\n  name c1\n  kind conv\n  inputs [d]\n  out_channels 2\n  kernel [1, 1]\n}\n"
            "layer {\n  name c2\n  kind conv\n  inputs [c1]\n  out_channels 2\n  kernel [3, 3]\n  pad 1\n}\n"
            "layer {\n  name p\n  kind pool\n  inputs [c1]\n  pool max\n  kernel 2\n  stride 2\n}\n"
            "output c2\noutput p\n")
    b = [b for b in X.detect_fusion_blocks(X.Graph(text)) if "c1" in b.members][0]
    assert b.mode == "straight" and b.stores_intermediate


def test_relu_folding():  # test_fusion.cpp:29-71
    base = "name t\ninput {\n  name d\n  shape [2, 8, 8]\n}\n"
    g = X.Graph(base + "layer {\n  name c\n  kind conv\n  inputs [d]\n  out_channels 2\n  kernel [3, 3]\n  pad 1\n}\n"
                "layer {\n  name r\n  kind relu\n  inputs [c]\n}\noutput r\n")
    assert [l["name"] for l in g.layers] == ["c"] and g.layers[0]["conv"]["relu"] and g.outputs == ["c"]
    g = X.Graph(base + "layer {\n  name r\n  kind relu\n  inputs [d]\n}\noutput r\n")
    assert g.find_layer("r") is not None
    g = X.Graph(base + "layer {\n  name c\n  kind conv\n  inputs [d]\n  out_channels 2\n  kernel [1, 1]\n}\n"
                "layer {\n  name r\n  kind relu\n  inputs [c]\n}\n"
                "layer {\n  name s\n  kind add\n  inputs [c, r]\n}\noutput s\n")
    assert g.find_layer("r") is not None


def test_tiling_a1_and_b1_plans():  # test_tiling.cpp:141-176
    t = X.plan_tiling(g_of("a1"), "b0", (14, 14), (2, 2))
    assert "border 2" in t and "channels 16" in t and "logical [14, 14]" in t and "constant_memory" in t
    assert f"shared_bytes {16 * 18 * 19 * 4}" in t
    t = X.plan_tiling(g_of("b1"), "b0", (14, 14), (4, 4))
    assert "border 1" in t and "logical [14, 14]" in t
    assert int(re.search(r"replicated_elements (\d+)", t).group(1)) > 0


def test_infeasible_plan_reports_shared_memory():  # test_tiling.cpp:178-193
    with pytest.raises(X.XlfError) as ei:
        X.plan_tiling(g_of("c1"), "b0", (14, 14), (4, 4))
    assert ei.value.kind == "infeasible" and "shared" in str(ei.value)
    # a 7x7 tile of the same block fits B200 (227 KB per block), not Pascal (48 KB)
    assert "shared_bytes" in X.plan_tiling(g_of("c1"), "b0", (7, 7), (8, 8), device="b200")


def test_store_transactions_table2():  # test_cost_model.cpp:25-38 (paper Table 2)
    assert X.store_transactions(g_of("a1"), "b0")[0] == 6272
    assert X.store_transactions(g_of("b1"), "b0")[0] == 100352


def test_errors_carry_kinds():
    with pytest.raises(X.XlfError) as ei:
        X.Graph("name broken\ninput {\n  name d\n  shape [1, 2]\n}\noutput d\n")
    assert ei.value.kind == "parse"
    with pytest.raises(X.XlfError) as ei:
        X.plan_tiling(g_of("a1"), "b99", (1, 1), (28, 28))
    assert ei.value.kind == "validation"


def test_graph_round_trip():
    g = g_of("squeezenet11")
    g2 = X.Graph(g.serialize())
    assert g2.serialize() == g.serialize()
    assert g2.shape_of("pool10") == (1000, 1, 1)


@pytest.mark.parametrize("name", OURS)
@pytest.mark.parametrize("part", ["reference", "b200", "unfused"])
def test_device_plans_cover_every_layer(name, part):
    g = g_of(name)
    p = X.device_plan(g, part, 8)
    executed = [l for s in p["steps"] for l in s["layers"]]
    elided = {n for n, t in p["tensors"].items() if t["materialized"]} - set(executed) - {i for i, _ in g.inputs}
    assert len(executed) == len(set(executed))
    assert set(executed) | elided == {l["name"] for l in g.layers}
    for s in p["steps"]:
        if s["kind"] == "fused":
            assert 0 < s["smem_bytes"] <= 227 * 1024
    for o in g.outputs:
        assert p["tensors"][o]["materialized"]


def test_b200_cost_based_fusion_decisions():
    """bf16 B200 partition.  Split / straight blocks of a 1x1 reduce into
    stride-1 expand convs run on the fire kernel (kernels_fire.cu: squeeze
    plane on chip, whole-image or row-band units) and stay fused -- all eight
    SqueezeNet fire modules (not inception-3a's 1x1-reduce -> 3x3, whose
    weights would force 32-channel groups).  Without it
    (option no_fire=1) a fused block is kept only when the planner's model
    beats its layers as single kernels: inception's reduce -> 3x3 (221 KB of
    weights re-streamed per small fused tile) is split; option always_fuse
    keeps every block fused."""
    g = X.load_graph(X.graph_path("fire"))
    steps = X.device_plan(g, "b200", 32, "bf16")["steps"]
    assert [s["tag"] for s in steps] == ["split"]
    g = X.load_graph(X.graph_path("squeezenet11"))
    steps = X.device_plan(g, "b200", 256, "bf16")["steps"]
    fires = [s for s in steps if s["tag"] == "split"]
    assert len(fires) == 8 and all(len(s["layers"]) == 3 for s in fires), [s["layers"] for s in steps]
    steps = X.device_plan(g, "b200", 256, "bf16", options="no_fire=1")["steps"]
    assert any(s["layers"] == ["fire9_squeeze"] for s in steps)
    g = X.load_graph(X.graph_path("inc3a"))
    # the fire kernel would need 4 groups of 32 channels for inception's 3x3
    # (weights), which it does not take: the cost model splits the block
    steps = X.device_plan(g, "b200", 64, "bf16")["steps"]
    assert any(s["layers"] == ["b3"] for s in steps), [s["layers"] for s in steps]
    steps = X.device_plan(g, "b200", 64, "bf16", options="no_fire=1")["steps"]
    assert any(s["layers"] == ["b3"] for s in steps), [s["layers"] for s in steps]
    steps = X.device_plan(g, "b200", 64, "bf16", options="no_fire=1,always_fuse=1")["steps"]
    assert not any(s["layers"] == ["b3"] for s in steps)
    # the fp32 planner is unaffected (its kernels stage no weights)
    g = X.load_graph(X.graph_path("inc3a"))
    assert not any(s["layers"] == ["b3"] for s in X.device_plan(g, "b200", 64, "fp32")["steps"])


def test_b200_device_document_round_trips():
    """paper_2007_06000_b200/devices/b200.device is serialize_device(b200_spec)
    in the reference's format (device.cpp:38-90); parsing it gives it back, and
    the reference planner's plan_tiling accepts it as a device."""
    path = os.path.join(X.DEVICES, "b200.device")
    text = open(path).read()
    assert X.device_document("b200") in text
    assert X.device_document(text) == X.device_document("b200")
    g = X.load_graph(X.graph_path("b1"))
    b = [b for b in X.detect_fusion_blocks(g) if b.fused()][0]
    h, w = g.shape_of(b.consumer_stage[0])[1:]
    plan = X.plan_tiling(g, b.id, (11, 11), (-(-h // 11), -(-w // 11)), text)
    assert "b200" in plan
