"""Executor behaviour through the C ABI: CUDA-graph replay vs eager launches,
end-to-end host path, device-side seeded inputs, run_fused_block /
simulate_graph API, per-step execution, error behaviour."""
import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text

pytestmark = pytest.mark.gpu


def test_graph_replay_equals_eager_and_steps():
    import torch
    g = X.Graph(graph_text("squeezenet11"))
    w = X.seeded_weights(g, 42)
    e = X.Engine(g, w, "b200", "fp32", max_batch=4)
    e.set_input_seeded(42, 4)
    e.forward(4, use_graph=True)
    a = e.read("pool10", 4).cpu()
    e.forward(4, use_graph=False)
    b = e.read("pool10", 4).cpu()
    for i in range(len(e.steps)):
        e.run_step(i, 4)
    c = e.read("pool10", 4).cpu()
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(a, c)


@pytest.mark.parametrize("opts", ["", "e2e_ramp=0", "e2e_chunks=3"])
@pytest.mark.parametrize("prec", ["fp32_exact", "bf16"])
def test_run_host_matches_device_path(prec, opts):
    """run_host's chunked H2D / forward / D2H pipeline (half-size end chunks by
    default, equal chunks with e2e_ramp=0) equals the device path."""
    import torch
    g = X.Graph(graph_text("fire"))
    og = O.load_graph(graph_text("fire"))
    w = X.seeded_weights(g, 42)
    x = O.seeded_batch(og, 42, 7)
    e = X.Engine(g, w, "b200", prec, max_batch=7, options=opts)
    host = e.run_host(x, "fire3_concat")
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(7)
    dev = e.read("fire3_concat", 7).cpu().numpy()
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("prec", ["fp32_exact", "bf16"])
def test_device_seeded_input_is_the_reference_stream(prec):
    import torch
    g = X.Graph(graph_text("b1"))
    og = O.load_graph(graph_text("b1"))
    w = X.seeded_weights(g, 1)
    e1 = X.Engine(g, w, "unfused", prec, max_batch=2)
    e1.set_input_seeded(42, 2, first_image=3)
    e1.forward(2)
    e2 = X.Engine(g, w, "unfused", prec, max_batch=2)
    c, h, wd = og.inputs[0][1]
    x = O.stream(42, 3 * c * h * wd, 2 * c * h * wd).reshape(2, c, h, wd)
    e2.set_input(torch.from_numpy(x).cuda())
    e2.forward(2)
    assert torch.equal(e1.read("fire_concat", 2), e2.read("fire_concat", 2))


def test_run_fused_block_and_simulate_graph_api():
    import torch
    text = graph_text("b1")
    g = X.Graph(text)
    og = O.load_graph(text)
    w = X.seeded_weights(g, 42)
    x = O.seeded_batch(og, 42, 2)
    blk = [b for b in X.detect_fusion_blocks(g) if b.fused()][0]
    values = {"data": torch.from_numpy(x).cuda()}
    written = X.run_fused_block(g, blk, values, w)
    ref = O.run_batch(og, x, O.seeded_weights(og, 42), ["fire_expand1", "fire_expand3"])
    assert set(written) == {"fire_expand1", "fire_expand3"}
    for k in written:
        assert np.array_equal(values[k].cpu().numpy(), ref[k])
    sim = X.simulate_graph(g, torch.from_numpy(x).cuda(), w, "reference", "fp32_exact")
    full = O.run_batch(og, x, O.seeded_weights(og, 42), og.outputs)
    assert np.array_equal(sim["fire_concat"].cpu().numpy(), full["fire_concat"])


def test_errors_are_loud():
    g = X.Graph(graph_text("fire"))
    w = X.seeded_weights(g, 42)
    with pytest.raises(X.XlfError) as ei:
        X.Engine(g, w[:-5], "b200", "fp32", max_batch=1)
    assert ei.value.kind == "validation"
    e = X.Engine(g, w, "b200", "fp32", max_batch=2)
    with pytest.raises(X.XlfError):
        e.forward(3)
    with pytest.raises(X.XlfError) as ei:
        e.read("fire3_squeeze", 1)  # fused intermediate: never in HBM
    assert "intermediate" in str(ei.value)
