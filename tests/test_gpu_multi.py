"""Several GPUs in one process (MultiEngine / xlf_multi_*): one engine per
device slot, batch-sharded by xlf_shard, one native host worker thread and
stream per device.  The box has one B200, so the slots are [0, 0]: two
engines and two worker threads on the same GPU exercise the sharding, the
concurrent workers and the gather exactly as two GPUs would."""
import numpy as np
import pytest

import paper_2007_06000_b200 as X
from oracle import oracle as O
from tests.conftest import graph_text

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [("fp32_exact", 0.0), ("bf16", 1e-2), ("tf32", 1e-3)])
@pytest.mark.parametrize("batch", [4, 5])
def test_multi_run_host_matches_oracle(prec, tol, batch):
    text = graph_text("squeezenet11")
    g = X.Graph(text)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    m = X.MultiEngine(g, O.flat_weights(og, w), [0, 0], "b200", prec, max_batch_per_device=3)
    out, ms = m.run_host(x, "pool10")
    assert len(ms) == 2 and all(t > 0 for t in ms)
    ref = O.run_batch(og, x, w, ["pool10"])["pool10"]
    if prec == "fp32_exact":
        assert np.array_equal(out, ref)
    else:
        assert O.normwise(out, ref) <= tol
    # each slot's images are exactly its shard: a single engine on the same images agrees
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch)
    single = e.run_host(x, "pool10")
    if prec == "fp32_exact":
        assert np.array_equal(out, single)


def test_multi_time_seeded_and_autotune():
    g = X.load_graph(X.graph_path("squeezenet11"))
    m = X.MultiEngine(g, X.seeded_weights(g, 42), [0, 0], "b200", "bf16", max_batch_per_device=32)
    m.autotune(32, reps=2, topk=1)
    ms = m.time_seeded(42, 32, steps=3, warmup=3)
    assert len(ms) == 2 and all(t > 0 for t in ms)
    with pytest.raises(X.XlfError):
        m.time_seeded(42, 33)
