"""Fire kernel unit-shape sweep: SqueezeNet v1.1 at batch 256, every fire
step timed (CUDA events, run_step) under forced channel splits / unit shapes.

    python tests/probes/fire_sweep.py [precision] [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def time_steps(e, batch, idx, reps=10):
    st = torch.cuda.current_stream()
    out = {}
    for i in idx:
        for _ in range(2):
            e.run_step(i, batch)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            e.run_step(i, batch)
        b.record(st)
        torch.cuda.synchronize()
        out[i] = a.elapsed_time(b) / reps * 1000
    return out


def main():
    prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    g = X.load_graph(X.graph_path("squeezenet11"))
    w = X.seeded_weights(g, 42)
    shapes = [("g", 1), ("r", 4), ("r", 7), ("r", 8), ("r", 14), ("r", 16), ("r", 28), ("g", 2), ("g", 3), ("g", 4)]
    best = {}
    for ns in (1, 2, 4):
        for kind, v in shapes:
            opt = f"fire_nsplit={ns},fire_{kind}={v}"
            try:
                e = X.Engine(g, w, "b200", prec, max_batch=batch, options=opt)
            except Exception as ex:  # noqa: BLE001
                print(opt, "engine failed:", ex)
                continue
            e.set_input_seeded(42, batch)
            e.forward(batch, use_graph=False)
            idx = [i for i, s in enumerate(e.steps) if s["tag"] == "fire"]
            t = time_steps(e, batch, idx)
            row = []
            for i in idx:
                s = e.steps[i]
                key = s["layers"][0].split("_")[0]
                row.append(f"{key}:{t[i]:.1f}({s['tile'][0]}x{s['tile'][1]})")
                if key not in best or t[i] < best[key][0]:
                    best[key] = (t[i], opt, s["tile"])
            print(opt, " ".join(row), flush=True)
            del e
    print("best:")
    for k, v in sorted(best.items()):
        print(f"  {k}: {v[0]:.1f} us  {v[1]}  unit {v[2]}")


if __name__ == "__main__":
    main()
