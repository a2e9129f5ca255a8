"""Fire kernel debugging aid: one fire-module graph through the fire kernel
under forced unit shapes, each output compared with the CPU oracle, with the
error located by row / column / channel group.

    python tests/probes/fire_debug.py [graph] [batch] [precision]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "b1"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
    text = open(X.graph_path(name)).read()
    og = O.load_graph(text)
    w = O.seeded_weights(og, 42)
    x = O.seeded_batch(og, 42, batch)
    out_name = og.outputs[0]
    ref = O.run_batch(og, x, w, [out_name])[out_name]
    g = X.Graph(text)
    H = ref.shape[2]
    cfgs = ["no_fire=1", "", "fire_nsplit=1,fire_g=1,fire_r=%d" % H, "fire_nsplit=1,fire_g=1,fire_r=8", "fire_nsplit=2,fire_g=1,fire_r=8",
            "fire_nsplit=1,fire_g=2", "fire_nsplit=4,fire_g=1,fire_r=4"]
    for opt in cfgs:
        try:
            e = X.Engine(g, O.flat_weights(og, w), "b200", prec, max_batch=batch, options=opt)
        except Exception as ex:  # noqa: BLE001
            print(f"[{opt}] engine: {ex}")
            continue
        st = [(s["tag"], s["tile"], s["nsplit"]) for s in e.steps]
        e.set_input(torch.from_numpy(x).cuda())
        e.forward(batch, use_graph=False)
        out = e.read(out_name, batch).cpu().numpy()
        torch.cuda.synchronize()
        err = np.abs(out - ref)
        scale = np.abs(ref).max()
        bad = err > 0.02 * scale
        print(f"[{opt}] steps {st} normwise {err.max() / scale:.2e} bad {bad.mean():.4f} finite {np.isfinite(out).all()}")
        if bad.any():
            C = ref.shape[1]
            print("   bad by image", [round(float(bad[n].mean()), 3) for n in range(batch)])
            print("   bad by channel group (16)", [round(float(bad[:, c:c + 16].mean()), 3) for c in range(0, C, 16)])
            r = bad.mean(axis=(0, 1, 3))
            print("   bad rows", [i for i in range(H) if r[i] > 0][:40], "max row frac", round(float(r.max()), 3))
            cfr = bad.mean(axis=(0, 1, 2))
            print("   bad cols", [i for i in range(ref.shape[3]) if cfr[i] > 0][:40])
            n, c, y, xx = np.argwhere(bad)[0]
            print("   first bad", (n, c, y, xx), "got", out[n, c, y, xx], "ref", ref[n, c, y, xx])


if __name__ == "__main__":
    main()
