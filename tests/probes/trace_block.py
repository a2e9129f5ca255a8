"""Per-CTA phase timeline of the bf16 fused kernels (XLF_TRACE=1).

    XLF_TRACE=1 python tests/probes/trace_block.py fire 32
Prints, for the first CTAs of each bf16 step, microseconds from CTA start to:
X issued, X landed (MMA thread), each unit's accumulator-ready / done, end.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("XLF_TRACE", "1")

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from paper_2007_06000_b200 import _lib  # noqa: E402


def main():
    name, batch = sys.argv[1], int(sys.argv[2])
    part = sys.argv[3] if len(sys.argv) > 3 else "b200"
    g = X.load_graph(X.graph_path(name))
    e = X.Engine(g, X.seeded_weights(g, 42), part, "bf16", max_batch=batch)
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
        print(f"step {s['id']} {s['tag']} tile={s['tile']} smem={s['smem_bytes']}")
        for cta in range(8):
            ev = list(buf[cta * 32:(cta + 1) * 32])
            t0 = ev[0]
            if not t0:
                continue
            rel = lambda k: f"{(ev[k] - t0) / 1000:7.2f}" if ev[k] else "      -"
            units = " ".join(f"[{rel(4 + 2 * u)} {rel(5 + 2 * u)}]" for u in range(12) if ev[4 + 2 * u] or ev[5 + 2 * u])
            print(f"  cta{cta}: xland {rel(2)} g0 issue [{rel(29)} {rel(30)}] g1 issue [{rel(31)}] units {units} "
                  f"end {rel(3)}")


if __name__ == "__main__":
    main()
