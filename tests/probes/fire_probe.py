"""Fire kernel probe: SqueezeNet v1.1 through the b200 plan with and without
the fire kernel (option no_fire=1) -- every fire block's concat output vs
the CPU oracle on sampled images, then per-step device times.

    python tests/probes/fire_probe.py [batch] [precision] [options]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from oracle import oracle as O  # noqa: E402


def step_times(e, batch, reps=10):
    n = len(e.steps)
    st = torch.cuda.current_stream()
    for _ in range(3):
        for i in range(n):
            e.run_step(i, batch)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(reps)]
    for k in range(reps):
        ev[k][0].record(st)
        for i in range(n):
            e.run_step(i, batch)
            ev[k][i + 1].record(st)
    torch.cuda.synchronize()
    return [sum(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(reps)) / reps * 1000 for i in range(n)]


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
    opts = sys.argv[3] if len(sys.argv) > 3 else ""
    text = open(X.graph_path("squeezenet11")).read()
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    g = X.Graph(text)
    e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch, options=opts)
    e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    torch.cuda.synchronize()
    sample = sorted({0, batch // 2, batch - 1})
    x = O.seeded_batch(og, 42, batch)[sample]
    names = [f"fire{i}_concat" for i in range(2, 10)]
    ref = O.run_batch(og, x, w, names + ["pool10"])
    for n in names + ["pool10"]:
        try:
            out = e.read(n, batch).cpu().numpy()[sample]
        except Exception as ex:  # noqa: BLE001
            print(n, "unreadable", ex)
            continue
        print(f"{n:14s} normwise {O.normwise(out, ref[n]):.2e} finite {np.isfinite(out).all()}")
    t = step_times(e, batch)
    for s, us in zip(e.steps, t):
        print(f"{s['id']:44s} {s['tag']:14s} tile {s['tile']} nsplit {s['nsplit']} smem {s['smem_bytes']:6d} {us:8.1f} us")
    print(f"sum {sum(t):.1f} us")
    e.forward(batch)
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e.forward(batch)
    a.record(st)
    for _ in range(20):
        e.forward(batch)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"forward {ms * 1000:.1f} us  {batch / ms * 1000:.0f} img/s")


if __name__ == "__main__":
    main()
