mkdir -p gpurun_out
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2007_06000_b200 as X
g = X.load_graph(X.graph_path("squeezenet11"))
w = X.seeded_weights(g, 42)
for opt in ("", "fire_cb=64"):
    e = X.Engine(g, w, "b200", "tf32", max_batch=256, options=opt)
    e.set_input_seeded(42, 256); e.forward(256, use_graph=False); e.autotune(256, reps=3, topk=3)
    for _ in range(3): e.forward(256)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): e.forward(256)
    b.record(); torch.cuda.synchronize()
    print(f"[{opt}] {a.elapsed_time(b)/10:.3f} ms", [(s["id"], s["tag"]) for s in e.steps])
PY
