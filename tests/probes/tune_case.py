"""Autotune one graph at a small batch and check it against the oracle
(debug aid; run under compute-sanitizer).

    python tests/probes/tune_case.py squeezenet11 8
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.conftest import graph_text  # noqa: E402


def main():
    name, batch = sys.argv[1], int(sys.argv[2])
    topk = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    part = sys.argv[4] if len(sys.argv) > 4 else "b200"
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, batch)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), part, "bf16", max_batch=batch)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(batch)
    for c in e.autotune(batch, reps=1, topk=topk):
        print(c, flush=True)
    e.set_input(torch.from_numpy(x).cuda())
    e.forward(batch)
    ref = O.run_batch(og, x[:2], w, og.outputs, threads=2)
    for o in og.outputs:
        print(o, "normwise", O.normwise(e.read(o, batch).cpu().numpy()[:2], ref[o]))


if __name__ == "__main__":
    main()
