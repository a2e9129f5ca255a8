python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2007_06000_b200 as X
g = X.load_graph(X.graph_path("squeezenet11"))
w = X.seeded_weights(g, 42)
for topk in (3, 12):
    e = X.Engine(g, w, "b200", "bf16", max_batch=256)
    e.set_input_seeded(42, 256); e.forward(256, use_graph=False); rep = e.autotune(256, reps=3, topk=topk)
    st = torch.cuda.current_stream()
    for i, s in enumerate(e.steps):
        if s["tag"] != "pool": continue
        for _ in range(3): e.run_step(i, 256)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): e.run_step(i, 256)
        b.record(); torch.cuda.synchronize()
        r = [x for x in rep if x["id"] == s["id"]]
        print(f"topk {topk} {s['id']} {a.elapsed_time(b)/20*1000:.1f} us tried {r[0]['tried'] if r else '-'} tile {s['tile']} nxb {s['nxb']} ew {s['epi_warps']} grid_all {s['grid_all']}")
PY
