"""Tuned forward time of one graph (device resident), e.g. to compare plan
variants selected by environment knobs.

    python tests/probes/block_time.py inc3a 64 b200
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    name, batch, part = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), part, "bf16", max_batch=batch)
    e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    e.autotune(batch, reps=3, topk=3)
    for _ in range(3):
        e.forward(batch)
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        e.forward(batch)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    print(name, part, "steps", [(s["id"], s["tag"]) for s in e.steps], "us", round(statistics.median(ts), 1))


if __name__ == "__main__":
    main()
