"""Per-step device time of a tuned bf16 engine (CUDA events around each step).

    python tests/probes/step_times.py inc3a 64 b200 [precision]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    name, batch, part = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    prec = sys.argv[4] if len(sys.argv) > 4 else "bf16"
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), part, prec, max_batch=batch)
    e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    e.autotune(batch, reps=3, topk=3)
    n = len(e.steps)
    st = torch.cuda.current_stream()
    for _ in range(3):
        for i in range(n):
            e.run_step(i, batch)
    reps = 10
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(reps)]
    for k in range(reps):
        ev[k][0].record(st)
        for i in range(n):
            e.run_step(i, batch)
            ev[k][i + 1].record(st)
    torch.cuda.synchronize()
    tot = 0
    for i, s in enumerate(e.steps):
        t = sum(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(reps)) / reps * 1000
        tot += t
        print(f"{s['id']:40s} {s['tag']:14s} {str(s['layers']):60s} {t:8.1f} us  tile {s['tile']} wres {s.get('wres')} slots {s.get('ring_slots')}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    main()
