"""Fire steps: the tuner's choices (tune_verbose timings on stderr) and the
per-step times of the tuned engine vs forced unit shapes.

    python tests/probes/fire_tune.py [batch] [forced options...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2007_06000_b200 as X  # noqa: E402
from tests.probes.fire_sweep import time_steps  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    g = X.load_graph(X.graph_path("squeezenet11"))
    w = X.seeded_weights(g, 42)
    e = X.Engine(g, w, "b200", "bf16", max_batch=batch, options="tune_verbose=1")
    e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    rep = e.autotune(batch, reps=3, topk=3)
    for r in rep:
        if r.get("kernel") == "fire":
            print(r)
    idx = [i for i, s in enumerate(e.steps) if s["tag"] == "fire"]
    t = time_steps(e, batch, idx)
    print("tuned:", {e.steps[i]["id"]: round(t[i], 1) for i in idx})
    for opt in sys.argv[2:]:
        f = X.Engine(g, w, "b200", "bf16", max_batch=batch, options=opt)
        f.set_input_seeded(42, batch)
        f.forward(batch, use_graph=False)
        idx = [i for i, s in enumerate(f.steps) if s["tag"] == "fire"]
        t = time_steps(f, batch, idx)
        print(opt, {f.steps[i]["id"]: (round(t[i], 1), f.steps[i]["tile"][0], f.steps[i]["nsplit"]) for i in idx})


if __name__ == "__main__":
    main()
