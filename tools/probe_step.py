"""Times every step of a SqueezeNet engine (CUDA events, batch B) under two
option sets and compares a tensor between them (norm-wise): A/B probe for a
kernel change.  usage: python tools/probe_step.py PREC B "optsA" "optsB" TENSOR"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2007_06000_b200 as X  # noqa: E402
from oracle import oracle as O  # noqa: E402

prec, B = sys.argv[1], int(sys.argv[2])
opts = [sys.argv[3], sys.argv[4]]
name = sys.argv[5]
g = X.load_graph(X.graph_path("squeezenet11"))
w = X.seeded_weights(g, 42)
outs = []
for o in opts:
    e = X.Engine(g, w, "b200", prec, max_batch=B, options=o)
    e.set_input_seeded(42, B)
    e.forward(B, use_graph=False)
    if prec in ("bf16", "tf32"):
        e.autotune(B, reps=3, topk=3)
    e.set_input_seeded(42, B)
    e.forward(B)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    res = []
    for i, s in enumerate(e.steps):
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            e.run_step(i, B)
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        res.append((s["id"], s["tag"], round(statistics.median(ts), 1)))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        e.forward(B)
    a.record(st)
    for _ in range(20):
        e.forward(B)
    b.record(st)
    b.synchronize()
    print(f"[{o}] forward {a.elapsed_time(b) / 20 * 1000:.1f} us  steps: {res}", flush=True)
    e.forward(B)
    outs.append(e.read(name, B).cpu().numpy())
    if len(outs) == 1:
        og = O.load_graph(open(X.graph_path("squeezenet11")).read())
        x = O.seeded_batch(og, 42, 2)
        ref = O.run_batch(og, x, O.seeded_weights(og, 42), [name])[name]
    print(f"[{o}] {name} vs oracle (2 images): normwise {O.normwise(outs[-1][:2], ref):.3e}", flush=True)
print("A vs B normwise", O.normwise(outs[0], outs[1]))
