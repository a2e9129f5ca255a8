"""Timeline of the fire kernel on CTA (0, 0) (engine option trace=1): per job
the MMA issuer's wait / issue / commit stamps, the epilogue's wait / done
stamps and the producer's ring stamps, relative to the first stamp.

    python tests/probes/fire_trace.py [layer-prefix] [batch] [options] [graph]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402
from paper_2007_06000_b200 import _lib  # noqa: E402

N = 1024
NAMES = {11: "mma sq wait", 21: "mma sq issue", 31: "mma sq commit", 12: "mma ex wait", 22: "mma ex issue", 32: "mma ex commit",
         23: "mma ex first issued", 24: "mma ex all issued",
         41: "epi sq wait", 51: "epi sq got", 61: "epi sq done", 42: "epi ex wait", 52: "epi ex got", 62: "epi ex done", 50: "tma"}


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "fire2"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    opts = "trace=1" + ("," + sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] else "")
    g = X.load_graph(X.graph_path(sys.argv[4] if len(sys.argv) > 4 else "squeezenet11"))
    e = X.Engine(g, X.seeded_weights(g, 42), "b200", "bf16", max_batch=batch, options=opts)
    e.set_input_seeded(42, batch)
    e.forward(batch, use_graph=False)
    idx = [i for i, s in enumerate(e.steps) if s["tag"] == "fire" and s["layers"][0].startswith(which)][0]
    for _ in range(3):
        e.run_step(idx, batch)
    torch.cuda.synchronize()
    print(e.steps[idx]["id"], e.steps[idx]["tile"], e.steps[idx]["nsplit"])
    buf = (ctypes.c_ulonglong * (3 * N * 2))()
    n = ctypes.c_size_t(0)
    assert _lib.lib().xlf_engine_trace(e._h, idx, buf, 3 * N * 2, ctypes.byref(n)) == 0
    ev = []
    for role in range(3):
        for k in range(N):
            c, t = buf[(role * N + k) * 2], buf[(role * N + k) * 2 + 1]
            if t == 0:
                break
            ev.append((t, role, c >> 32, c & 0xffffffff))
    ev.sort()
    t0 = ev[0][0]
    # per-kind averages: MMA issue -> commit, epilogue got -> done
    import collections
    start, dur = {}, collections.defaultdict(list)
    for t, role, code, i in ev:
        if code in (21, 22, 51, 52):
            start[(code % 10, code // 10, i)] = t
        elif code in (31, 32, 61, 62):
            k = (code % 10, code // 10 - 1, i)
            if k in start:
                dur[("sq" if code % 10 == 1 else "ex") + (" mma" if code < 40 else " epi")].append(t - start[k])
    for k, v in sorted(dur.items()):
        print(f"avg {k}: {sum(v) / len(v):.0f} ns over {len(v)}")
    if os.environ.get("SUMMARY"):
        print("span", (ev[-1][0] - t0) / 1000, "us")
        return
    last = {}
    for t, role, code, i in ev[:600]:
        dt = t - last.get(role, t)
        last[role] = t
        print(f"{(t - t0) / 1000:9.2f} us  {'  ' * 20 * role}{NAMES.get(code, code)} {i}  (+{dt} ns)")
    print("span", (ev[-1][0] - t0) / 1000, "us,", len(ev), "events")


if __name__ == "__main__":
    main()
