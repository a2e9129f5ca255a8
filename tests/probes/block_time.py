"""Median forward time of one graph under several engine option strings
(tuned as bench.py tunes), e.g. to compare a planner choice on and off.

    python tests/probes/block_time.py inc3a 64 bf16 "" no_fire=1 ...
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    name, batch, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    g = X.load_graph(X.graph_path(name))
    w = X.seeded_weights(g, 42)
    for opt in sys.argv[4:] or [""]:
        e = X.Engine(g, w, "b200", prec, max_batch=batch, options=opt)
        e.set_input_seeded(42, batch)
        e.forward(batch, use_graph=False)
        e.autotune(batch, reps=3, topk=3)
        for _ in range(3):
            e.forward(batch, use_graph=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            e.forward(batch, use_graph=True)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        print(f"{name} {prec} b{batch} [{opt}]: {statistics.median(ts):.1f} us;",
              [(s["id"], s["tag"], s.get("tile"), s.get("nsplit")) for s in e.steps])


if __name__ == "__main__":
    main()
