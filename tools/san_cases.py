"""Small forwards for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the product once, outputs read back through the ABI.

    compute-sanitizer --tool memcheck python tools/san_cases.py [precision ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402

CASES = [("squeezenet11", 2, "b200"), ("squeezenet11", 2, "unfused"), ("inc3a", 2, "b200"), ("residual", 2, "b200"),
         ("a2", 2, "b200"), ("c1", 2, "reference"), ("fire", 3, "b200")]


TUNE = os.environ.get("SAN_TUNE", "1") == "1"


def main():
    precs = sys.argv[1:] or ["bf16", "fp32_exact"]
    for prec in precs:
        for name, batch, part in CASES:
            g = X.load_graph(X.graph_path(name))
            e = X.Engine(g, X.seeded_weights(g, 42), part, prec, max_batch=batch)
            e.set_input_seeded(42, batch)
            e.forward(batch, use_graph=False)
            if TUNE and prec.startswith("fp32"):
                # the fp32 tuner launches every (tile, register blocking, 256 / 512 threads) candidate
                e.autotune(batch, reps=1, topk=1)
            e.forward(batch, use_graph=True)
            for n in e.materialized():
                if n in dict(g.inputs):
                    continue
                e.read(n, batch)
            torch.cuda.synchronize()
            print(f"ok {prec} {name} {part} b{batch}: {len(e.steps)} steps", flush=True)


if __name__ == "__main__":
    main()
