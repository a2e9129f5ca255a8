"""Generates tests/golden/golden.json from the UNMODIFIED reference
(oracle/_ref/libxlfuse_ref.so, built from /root/reference/proj/src).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

What is frozen, per fixture graph (paper_2007_06000_b200/graphs/*.graph and
the reference's own fixtures under /root/reference/proj/fixtures/graphs):
  * inputs  : SeededStream(42), image n = elements [n*CHW, (n+1)*CHW)
  * weights : seeded_weights(g, 42) (tensor.cpp:42-62), sha256 of the stream
  * every layer output of run_reference (reference.cpp:126-142): shape,
    sha256 of the float32 bytes, float64 sum and 64 sampled values
  * block_assignment_report of the reference planner (fusion.cpp:228-256)
  * titan_xp-tuned plans of every fused block (serialize_plan, tiling.cpp:493)
  * modelled store transactions fused / unfused (cost_model.cpp:43-55)
The reference publishes no numeric goldens, so these are the
ones the oracle restatement and the GPU path are pinned to.
"""
import hashlib
import json
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

SEED = 42
OURS = os.path.join(ROOT, "paper_2007_06000_b200", "graphs")
THEIRS = "/root/reference/proj/fixtures/graphs"


def digest(a):
    a = np.ascontiguousarray(a, np.float32)
    rng = np.random.default_rng(0)
    idx = sorted(set(rng.integers(0, a.size, 64).tolist()))
    return {"shape": list(a.shape), "sha256": hashlib.sha256(a.tobytes()).hexdigest(),
            "sum": float(a.astype(np.float64).sum()), "sample_idx": idx,
            "sample": [float(v) for v in a.ravel()[idx]]}


def one(path, batch):
    text = open(path).read()
    g = O.load_graph(text)
    entry = {"batch": batch, "seed": SEED}
    w = R.seeded_weights(text, SEED)
    entry["weights"] = {"count": int(w.size), "sha256": hashlib.sha256(w.tobytes()).hexdigest()}
    c, h, wd = g.inputs[0][1]
    x = R.seeded_inputs(text, SEED, batch * c * h * wd).reshape(batch, c, h, wd)
    entry["input"] = digest(x)
    outs = {}
    for l in g.layers:
        r = R.run(text, x, l.name, l.shape, weights=w, mode=0, threads=os.cpu_count())
        outs[l.name] = digest(r)
    entry["outputs"] = outs
    entry["block_report"] = R.block_report(text)
    plans, tx = {}, {}
    for m in re.finditer(r"^block (b\d+) mode (\w+)", entry["block_report"], re.M):
        bid, mode = m.group(1), m.group(2)
        if mode == "unfused":
            continue
        plans[bid] = R.plan(text, bid)
        tx[bid] = list(R.store_tx(text, bid))
    entry["plans"] = plans
    entry["store_tx"] = tx
    return entry


def main():
    out = {"ours": {}, "reference_fixtures": {}}
    for f in sorted(os.listdir(OURS)):
        name = f[:-6]
        batch = 1 if name == "squeezenet11" else 2
        print("golden", name, flush=True)
        out["ours"][name] = one(os.path.join(OURS, f), batch)
    if os.path.isdir(THEIRS):
        for f in sorted(os.listdir(THEIRS)):
            text = open(os.path.join(THEIRS, f)).read()
            name = f[:-6]
            rep = R.block_report(text)
            entry = {"block_report": rep, "plans": {}, "store_tx": {}}
            for m in re.finditer(r"^block (b\d+) mode (\w+)", rep, re.M):
                if m.group(2) != "unfused":
                    entry["plans"][m.group(1)] = R.plan(text, m.group(1))
                    entry["store_tx"][m.group(1)] = list(R.store_tx(text, m.group(1)))
            out["reference_fixtures"][name] = entry
    with open(os.path.join(ROOT, "tests", "golden", "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
