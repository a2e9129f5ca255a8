"""One graph through the engine vs the oracle (debug aid).

    python tests/probes/run_case.py a1 unfused bf16 2
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from tests.conftest import graph_text  # noqa: E402
from tests.test_gpu_parity import run  # noqa: E402


def main():
    name, part, prec, batch = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    text = graph_text(name)
    og = O.load_graph(text)
    w = O.seeded_weights(og, 3)
    x = O.seeded_batch(og, 5, batch)
    out, e = run(name, O.flat_weights(og, w), batch, part, prec, x=x)
    torch.cuda.synchronize()
    for s in e.steps:
        print(" ", s["id"], s["tag"], s["tile"], s.get("nxb"), s["smem_bytes"])
    sample = list(range(min(batch, 3)))
    ref = O.run_batch(og, x[sample], w, og.outputs, threads=3)
    for o in og.outputs:
        print(name, part, prec, o, "normwise", O.normwise(out[o][sample], ref[o]))


if __name__ == "__main__":
    main()
