"""Replays tests/test_gpu_parity.py::test_random_graphs_exact trial by trial
and reports every mismatch (debug aid; run under compute-sanitizer too).

    python tests/probes/random_graphs.py [trials] [prec]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from tests.test_gpu_parity import PARTS, run  # noqa: E402


def graph(rng, trial):
    C, H, W = int(rng.integers(1, 20)), int(rng.integers(5, 30)), int(rng.integers(5, 30))
    k = int(rng.choice([1, 3, 5]))
    pad = int(rng.integers(0, k // 2 + 1))
    s1 = int(rng.choice([1, 1, 2]))
    sq, e1, e3 = int(rng.integers(1, 24)), int(rng.integers(1, 40)), int(rng.integers(1, 40))
    return (f"name rnd{trial}\ninput {{\n  name d\n  shape [{C}, {H}, {W}]\n}}\n"
            f"layer {{\n  name c0\n  kind conv\n  inputs [d]\n  out_channels {sq}\n  kernel [{k}, {k}]\n  pad {pad}\n"
            f"  stride {s1}\n  activation relu\n}}\n"
            f"layer {{\n  name a\n  kind conv\n  inputs [c0]\n  out_channels {e1}\n  kernel [1, 1]\n  activation relu\n}}\n"
            f"layer {{\n  name b\n  kind conv\n  inputs [c0]\n  out_channels {e3}\n  kernel [3, 3]\n  pad 1\n  activation relu\n}}\n"
            f"layer {{\n  name cat\n  kind concat\n  inputs [a, b]\n}}\n"
            f"layer {{\n  name p\n  kind pool\n  inputs [cat]\n  pool max\n  kernel 3\n  stride 2\n}}\n"
            "output p\n")


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    prec = sys.argv[2] if len(sys.argv) > 2 else "fp32_exact"
    rng = np.random.default_rng(1234)
    bad = 0
    for trial in range(trials):
        text = graph(rng, trial)
        try:
            og = O.load_graph(text)
        except ValueError:
            continue
        w = O.seeded_weights(og, trial)
        x = O.seeded_batch(og, trial + 100, 2)
        ref = O.run_batch(og, x, w, ["c0", "cat", "p"])
        for part in PARTS:
            out, e = run(text, O.flat_weights(og, w), 2, part, prec, x=x, names=["c0", "cat", "p"])
            for n in out:
                d = np.abs(out[n] - ref[n])
                if d.max() > 0 or not np.array_equal(out[n], ref[n]):
                    bad += 1
                    idx = np.argwhere(d > 0)
                    print(f"MISMATCH trial {trial} {part} {n} shape {ref[n].shape} max|d| {d.max():.3g} "
                          f"count {len(idx)} first {idx[:4].tolist()}")
                    print("   ", " ".join(l.strip() for l in text.splitlines() if l.strip() and "{" not in l and "}" not in l))
                    print("    steps:", [(s["id"], s["tag"], s["tile"]) for s in e.steps])
            del e
    print("bad", bad)


if __name__ == "__main__":
    main()
