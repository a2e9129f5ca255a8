"""Per-tile end times of the first CTAs of each bf16 step (XLF_TRACE=2):
shows the steady-state per-tile period of the persistent kernel.

    python tests/probes/trace_tiles.py squeezenet11 256
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["XLF_TRACE"] = "2"

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from paper_2007_06000_b200 import _lib  # noqa: E402


def main():
    name, batch = sys.argv[1], int(sys.argv[2])
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", "bf16", max_batch=batch)
    e.set_input_seeded(42, batch)
    for _ in range(3):
        e.forward(batch, use_graph=False)
    torch.cuda.synchronize()
    n = ctypes.c_size_t()
    for i, s in enumerate(e.steps):
        if s["kind"] != "fused":
            continue
        buf = (ctypes.c_ulonglong * 256)()
        if _lib.lib().xlf_engine_trace(e._h, i, buf, 256, ctypes.byref(n)) != 0:
            continue
        print(f"step {s['id']} {s['tag']} tile={s['tile']}")
        t0 = min(v for v in buf if v) if any(buf) else 0
        for cta in range(4):
            ev = [v for v in buf[cta * 32:(cta + 1) * 32] if v]
            print(f"  cta{cta}: " + " ".join(f"{(v - t0) / 1000:6.2f}" for v in ev[:16]))


if __name__ == "__main__":
    main()
