"""Measured HBM traffic of a forward, fused (B200 partition) vs unfused.

Profiling target (run under `ncu --profile-from-start off --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv`):

    python tools/ncu_dram.py run GRAPH BATCH PRECISION PARTITION

(the engine is autotuned first, as bench.py does;
only one forward runs inside cudaProfilerStart/Stop).  Summary of the logs:

    python tools/ncu_dram.py summarize OUT.json LOG.csv...   (file names: GRAPH_BATCH_PREC_PART.csv)
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(name, batch, prec, part):
    import torch

    import paper_2007_06000_b200 as X
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), part, prec, max_batch=batch)
    e.set_input_seeded(42, batch)
    if True:  # every precision is tuned, as bench.py does
        e.forward(batch, use_graph=False)
        e.autotune(batch, reps=3, topk=3)
        e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    e.forward(batch, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    for s in e.steps:
        print(s["id"], s["tag"], s["tile"], s["bytes_algorithmic"])


def parse(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[start]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    per = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        k = per.setdefault(r[idi], {"kernel": r[ki]})
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
        k[r[mi]] = v * scale
    return list(per.values())


def summarize(out, logs):
    res = {}
    for p in logs:
        f = os.path.basename(p)[:-4].split("_")
        name, batch, prec, part = f[0], f[1], "_".join(f[2:-1]), f[-1]
        ks = parse(p)
        rd = sum(k.get("dram__bytes_read.sum", 0) for k in ks)
        wr = sum(k.get("dram__bytes_write.sum", 0) for k in ks)
        us = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
        res.setdefault(f"{name}_b{batch}_{prec}", {})[part] = {"kernels": len(ks), "dram_read": int(rd), "dram_write": int(wr),
                                                              "dram_total": int(rd + wr), "ncu_us_sum": round(us, 2)}
    for k, v in res.items():
        if "b200" in v and "unfused" in v:
            v["dram_saved"] = v["unfused"]["dram_total"] - v["b200"]["dram_total"]
            v["dram_ratio_unfused_over_fused"] = round(v["unfused"]["dram_total"] / max(1, v["b200"]["dram_total"]), 3)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5])
    else:
        summarize(sys.argv[2], sys.argv[3:])
