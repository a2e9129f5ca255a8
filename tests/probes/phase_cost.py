"""Per-step kernel time of a graph under the XLF_DBG phase-isolation switches
(bf16): 0 = normal, 1 = no HBM stores, 2 = no accumulator epilogue,
4 = no MMAs, 6 = neither.  Profiling aid only (outputs are wrong when set).

    python tests/probes/phase_cost.py squeezenet11 256 [dbg ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def step_times(name, batch, reps=10):
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", "bf16", max_batch=batch)
    e.set_input_seeded(42, batch)
    n = len(e.steps)
    for _ in range(3):
        e.forward(batch, use_graph=False)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(n + 1)] for _ in range(reps)]
    st = torch.cuda.current_stream()
    for k in range(reps):
        ev[k][0].record(st)
        for i in range(n):
            e.run_step(i, batch)
            ev[k][i + 1].record(st)
    torch.cuda.synchronize()
    t = [sum(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(reps)) / reps * 1000 for i in range(n)]
    return [f"{s['id']}:{s['tag']}" for s in e.steps], t


def main():
    name, batch = sys.argv[1], int(sys.argv[2])
    dbgs = [int(x) for x in sys.argv[3:]] or [0, 1, 2, 4, 6]
    cols = {}
    names = None
    for d in dbgs:
        os.environ["XLF_DBG"] = str(d)
        names, cols[d] = step_times(name, batch)
    print(f"{'step':50s}" + "".join(f"  dbg={d:<5d}" for d in dbgs))
    for i, nm in enumerate(names):
        print(f"{nm[:50]:50s}" + "".join(f"  {cols[d][i]:9.1f}" for d in dbgs))
    print(f"{'total':50s}" + "".join(f"  {sum(cols[d]):9.1f}" for d in dbgs))


if __name__ == "__main__":
    main()
