"""run_host (H2D + forward + D2H from pinned memory) img/s of tuned bf16
SqueezeNet at batch B under several engine option strings.

    python tests/probes/e2e_opts.py 256 "" "e2e_ramp=1" "e2e_chunks=6,e2e_ramp=1"
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2007_06000_b200 as X  # noqa: E402


def main():
    B = int(sys.argv[1])
    g = X.load_graph(X.graph_path("squeezenet11"))
    w = X.seeded_weights(g, 42)
    pin_in = torch.rand((B, 3, 224, 224), dtype=torch.float32).pin_memory()
    pin_out = torch.empty((B, 1000, 1, 1), dtype=torch.float32).pin_memory()
    f32p = ctypes.POINTER(ctypes.c_float)
    xp = ctypes.cast(pin_in.data_ptr(), f32p)
    op = ctypes.cast(pin_out.data_ptr(), f32p)
    L = X.api.lib()
    dev = torch.empty_like(pin_in, device="cuda")
    for _ in range(3):
        dev.copy_(pin_in, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        dev.copy_(pin_in, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"H2D alone: {ms:.3f} ms for {pin_in.numel() * 4 / 1e6:.0f} MB = {pin_in.numel() * 4 / ms / 1e6:.1f} GB/s (floor {B / ms * 1000:.0f} img/s)")
    del dev
    for opt in sys.argv[2:] or [""]:
        e = X.Engine(g, w, "b200", "bf16", max_batch=B, options=opt)
        e.set_input_seeded(42, B)
        e.forward(B, use_graph=False)
        e.autotune(B, reps=3, topk=3)
        for _ in range(3):
            X.api.check(L.xlf_engine_run_host(e._h, xp, B, b"pool10", op, None))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            X.api.check(L.xlf_engine_run_host(e._h, xp, B, b"pool10", op, None))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"[{opt}] {ms:.3f} ms/step = {B / ms * 1000:.0f} img/s", flush=True)
        del e


if __name__ == "__main__":
    main()
