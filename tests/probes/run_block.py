"""Runs one graph's forward a few times (profiling target for ncu).

    python tests/probes/run_block.py fire 32 bf16 b200 5 [tune|notune] [options]

With `tune`, the engine is autotuned first (as bench.py does) and only the
forwards run inside cudaProfilerStart/Stop: profile with
`ncu --profile-from-start off ...` to capture exactly the bench's kernels.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    name, batch, prec, part, reps = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
    tune = len(sys.argv) > 6 and sys.argv[6] == "tune"
    g = X.load_graph(X.graph_path(name))
    opts = sys.argv[7] if len(sys.argv) > 7 else ""
    e = X.Engine(g, X.seeded_weights(g, 42), part, prec, max_batch=batch, options=opts)
    e.set_input_seeded(42, batch)
    if tune:
        e.forward(batch, use_graph=False)
        e.autotune(batch, reps=3, topk=3)
        e.set_input_seeded(42, batch)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(reps):
        e.forward(batch, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    for s in e.steps:
        print(s["id"], s["tag"], s["tile"], s["smem_bytes"], s.get("nxb"), s.get("wres"), s.get("bytes_algorithmic"))


if __name__ == "__main__":
    main()
