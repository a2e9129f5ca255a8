"""Runs a graph's forward several times on the same input and reports the
steps whose outputs differ between runs (race detector for the kernels).

    python tests/probes/determinism.py squeezenet11 8 bf16
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    name, batch, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", prec, max_batch=batch)
    outs = []
    for r in range(4):
        e.set_input_seeded(42, batch)
        e.forward(batch, use_graph=(r % 2 == 0))
        outs.append({n: e.read(n, batch).clone() for n in e.materialized() if n not in dict(g.inputs)})
    torch.cuda.synchronize()
    bad = [n for n in outs[0] if any(not torch.equal(outs[0][n], o[n]) for o in outs[1:])]
    print("nondeterministic tensors:", bad or "none")


if __name__ == "__main__":
    main()
