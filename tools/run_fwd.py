"""One profiled forward of SqueezeNet (bf16 / TF32, batch B, autotuned like
bench.py) bracketed by cudaProfilerStart/Stop, for ncu --profile-from-start off.
usage: python tools/run_fwd.py PREC B [options]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2007_06000_b200 as X  # noqa: E402

prec, B = sys.argv[1], int(sys.argv[2])
opts = sys.argv[3] if len(sys.argv) > 3 else ""
g = X.load_graph(X.graph_path("squeezenet11"))
e = X.Engine(g, X.seeded_weights(g, 42), "b200", prec, max_batch=B, options=opts)
e.set_input_seeded(42, B)
e.forward(B, use_graph=False)
if prec in ("bf16", "tf32"):
    e.autotune(B, reps=3, topk=3)
e.set_input_seeded(42, B)
for _ in range(3):
    e.forward(B, use_graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
e.forward(B, use_graph=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("steps:", [(s["id"], s["tag"]) for s in e.steps])
