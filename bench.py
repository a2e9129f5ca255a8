"""Benchmark of the B200 fused CNN inference path (BASELINE.json metric:
"fused-block us & SqueezeNet img/s at 1/2/4/8 B200; HBM bytes saved vs
unfused").

Headline (`value`): SqueezeNet v1.1 inference, 256 images per GPU (BASELINE
config 5), bf16 tensor-core path, images/s over all ranks, inputs resident in
HBM (generated on device from the reference's SeededStream), one step = one
forward of the whole partition (one CUDA-graph launch).  In the same run:

* `e2e`: the same through the C ABI with host buffers (H2D of the NCHW fp32
  input + D2H of the logits inside the timed region);
* `parity`: the timed (autotuned) configuration's logits of sampled images
  against the CPU oracle (norm-wise error, argmax);
* `arms`: SqueezeNet img/s of every arithmetic path (bf16, TF32, fp32 SIMT)
  for the fused B200 partition AND the unfused sm_100a kernels -- the
  paper's fused-vs-unfused comparison;
* `blocks`: BASELINE configs 1-4 (straight / merge / split / inception) in us
  per block at every precision, fused vs unfused, each with its roofline
  fraction (algorithmic bytes / FLOPs against the measured peaks): device
  time per block (`us_pipelined`, forwards back to back; `speedup`) and
  single-launch latency (`us_median`, one synchronised CUDA-graph launch;
  `speedup_latency`); inputs stay L2-resident between repetitions;
* `roofline`: the dominant kernel of the headline step;
* `cpu_baseline`: the reference's own CPU path on this box's cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision bf16|tf32|fp32|fp32_exact]
    python bench.py --impl reference ...   # the reference's own CPU path

Multi-GPU: one rank per GPU (torchrun; `--gpus N` without torchrun re-launches
itself under torch.distributed.run); the batch is sharded (rank r generates
images [r*256, (r+1)*256)), no collective on the data path; the step time is
the max over ranks.  The optional NCCL gather of the logits to rank 0 is
timed separately (`gather_ms`).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "fused-block µs & SqueezeNet img/s at 1/2/4/8 B200; HBM bytes saved vs unfused"
PER_GPU_BATCH = 256
BLOCK_CONFIGS = [  # (config, graph, batch, precisions) -- BASELINE.json configs[0..3]
    ("straight", "straight", 1, ("fp32", "tf32", "bf16")),   # C1 is an fp32 config
    ("merge", "merge", 8, ("fp32", "tf32", "bf16")),
    ("split", "fire", 32, ("fp32", "tf32", "bf16")),
    ("inception", "inc3a", 64, ("tf32", "bf16", "fp32")),    # C4 names bf16 / TF32
    ("depthwise", "a2", 64, ("fp32", "tf32", "bf16")),       # paper a.2: depthwise 3x3 -> 1x1
]
TC = ("bf16", "tf32")
DTYPE = {"bf16": "bf16", "tf32": "tf32", "fp32": "f32", "fp32_exact": "f32"}


def peaks():
    """(HBM GB/s, bf16 dense TF/s, source): MEASURED_PEAKS.json (driver-written,
    this pool's B200s) or the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def pipe_peak_tflops(prec, sm_mhz):
    """Peak of the pipe a precision computes on: tcgen05 bf16 (measured), TF32
    (half the bf16 rate: 32-byte K steps of 8 instead of 16 elements at the
    same instruction rate), fp32 SIMT FMA (148 SMs x 128 lanes x 2 FLOP x clock)."""
    _, bf16, _ = peaks()
    if prec == "bf16":
        return bf16, "tcgen05 kind::f16 (measured bf16 peak)"
    if prec == "tf32":
        return bf16 / 2, "tcgen05 kind::tf32 (half the measured bf16 peak)"
    return 148 * 128 * 2 * (sm_mhz or 1965) * 1e6 / 1e12, "fp32 FFMA (SIMT, 148 x 128 lanes)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, every
    10 ms through NVML (nvidia-ml-py) on a background thread."""

    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop = threading.Event()
        self.thread = None

    def _sample(self):
        N, h = self.nvml, self.handle
        self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        try:
            while not self.stop.is_set():
                self._sample()
                time.sleep(0.01)
        except Exception:
            pass

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.nvml, self.handle = N, N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.handle, N.NVML_CLOCK_SM))
            self._sample()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(sm), "source": "nvml, 10 ms"}


# ----------------------------------------------------------------------------- checker / CPU legs (oracle)

def cpu_reference_rate(images: int, threads: int):
    """images/s of the reference's own CPU path (run_reference per image,
    reference.cpp:126-142, OpenMP across images) on SqueezeNet v1.1, from
    oracle/_ref when the reference compiled here, else the oracle port."""
    from oracle import oracle as O
    from oracle import ref as R
    text = open(os.path.join(ROOT, "paper_2007_06000_b200", "graphs", "squeezenet11.graph")).read()
    og = O.load_graph(text)
    x = O.seeded_batch(og, 42, images)
    t0 = time.perf_counter()
    if R.available():
        R.run(text, x, "pool10", og.shape_of("pool10"), wseed=42, mode=0, threads=threads)
        kind = "reference"
    else:
        O.run_batch(og, x, O.seeded_weights(og, 42), ["pool10"], threads=threads)
        kind = "port"
    dt = time.perf_counter() - t0
    return images / dt, kind, dt


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_parity(logits, first_image, sample, tol):
    """Checker: the timed configuration's logits of `sample` images against
    the CPU oracle on the same inputs (SeededStream(42) images first_image+i)
    and weights (seeded_weights(42)).  Norm-wise error and argmax agreement."""
    import numpy as np

    from oracle import oracle as O
    text = open(os.path.join(ROOT, "paper_2007_06000_b200", "graphs", "squeezenet11.graph")).read()
    og = O.load_graph(text)
    c, h, w = og.inputs[0][1]
    chw = c * h * w
    x = np.stack([O.stream(42, (first_image + i) * chw, chw).reshape(c, h, w) for i in sample]).astype(np.float32)
    ref = O.run_batch(og, x, O.seeded_weights(og, 42), ["pool10"], threads=min(len(sample), os.cpu_count() or 1))["pool10"]
    got = logits[sample]
    err = O.normwise(got, ref)
    agree = (got.reshape(len(sample), -1).argmax(1) == ref.reshape(len(sample), -1).argmax(1))
    return {"images_checked": len(sample), "sample": list(map(int, sample)), "normwise": float(f"{err:.3e}"), "tol": tol,
            "within_tol": bool(err <= tol), "argmax_equal": int(agree.sum()),
            "note": "seeded_weights(42) logits: argmax is degenerate under this init (SURVEY finding 7); the non-degenerate "
                    "He-init argmax check of the same tuned configuration is tests/test_gpu_tc.py::test_tc_squeezenet_autotuned_b256_argmax"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step = threads  # one image per host thread per step
    for _ in range(args.warmup):
        cpu_reference_rate(per_step, threads)
    kinds, secs = set(), 0.0
    for _ in range(args.steps):
        _, k, dt = cpu_reference_rate(per_step, threads)
        kinds.add(k)
        secs += dt
    value = per_step * args.steps / secs
    kind = kinds.pop()
    line = {
        "impl": "reference", "metric": BASELINE_METRIC, "value": round(value, 3), "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * secs / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "squeezenet_v1.1 224x224, reference CPU run_reference (oracle/_ref)", "images_per_step": per_step,
                   "parallelism": f"openmp x{threads} over images"},
        "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": threads, "cpu": cpu_model(), "kind": kind,
                         "sample": f"{per_step} images per step x {args.steps} steps"},
        "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def make_engine(X, g, w, part, prec, B, device, tune=True, first_image=0):
    """Engine + seeded device inputs; plans measured-time tuned (tensor-core
    and fp32 SIMT steps; part of the product, before any timed region)."""
    e = X.Engine(g, w, part, prec, max_batch=B, device=device)
    e.set_input_seeded(42, B, first_image=first_image)
    info = None
    if tune:
        t0 = time.time()
        e.forward(B, use_graph=False)
        chosen = e.autotune(B, reps=3, topk=3)
        info = {"steps_tuned": len(chosen), "seconds": round(time.time() - t0, 2)}
        e.set_input_seeded(42, B, first_image=first_image)
    return e, info


def time_forwards(torch, e, B, steps, warmup, st):
    """ms per forward: `warmup` untimed, then `steps` back to back between two
    CUDA events on the launching stream."""
    for _ in range(warmup):
        e.forward(B, use_graph=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        e.forward(B, use_graph=True)
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / steps


def plan_work(steps, batch):
    """Algorithmic bytes (inputs once + stored outputs once per image + weights
    once per launch) and FLOPs (2 x MACs, no halo recompute) of a plan."""
    nbytes = sum(s["bytes_algorithmic"] * batch + s.get("weight_bytes", 0) for s in steps)
    flops = sum(2 * s["macs"] * batch for s in steps)
    return nbytes, flops


def roofline_frac(nbytes, flops, ms, prec, sm_mhz):
    hbm, _, src = peaks()
    pipe, pipe_name = pipe_peak_tflops(prec, sm_mhz)
    t_mem, t_pipe = nbytes / (hbm * 1e9), flops / (pipe * 1e12)
    bound = "hbm" if t_mem >= t_pipe else "pipe"
    return {"bound": bound, "pipe": pipe_name, "roofline_us": round(max(t_mem, t_pipe) * 1e6, 2),
            "frac": round(max(t_mem, t_pipe) / (ms * 1e-3), 4), "achieved_gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
            "achieved_tflops": round(flops / (ms * 1e-3) / 1e12, 2), "peak_gbs": hbm, "peak_tflops": round(pipe, 1),
            "peak_source": src}


def time_blocks(X, torch, sm_mhz, reps=20):
    """us per fused block (B200 partition) vs the unfused kernels of the same
    layers, BASELINE configs 1-4 at every precision, inputs resident; each
    with its roofline fraction and algorithmic HBM bytes saved."""
    out = {}
    st = torch.cuda.current_stream()
    for cfg, gname, batch, precs in BLOCK_CONFIGS:
        g = X.load_graph(X.graph_path(gname))
        w = X.seeded_weights(g, 42)
        res = {"batch": batch}
        for prec in precs:
            r = {}
            for part in ("b200", "unfused"):
                e, _ = make_engine(X, g, w, part, prec, batch, torch.cuda.current_device())
                for _ in range(3):
                    e.forward(batch, use_graph=True)
                torch.cuda.synchronize()
                ts = []
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                # latency: one forward (one CUDA-graph launch) per event pair, synchronised
                for _ in range(reps):
                    a.record(st)
                    e.forward(batch, use_graph=True)
                    b.record(st)
                    b.synchronize()
                    ts.append(a.elapsed_time(b) * 1000.0)
                # device time per block: `reps` forwards back to back between two
                # events (the graph launches overlap the previous forward's kernels)
                a.record(st)
                for _ in range(reps):
                    e.forward(batch, use_graph=True)
                b.record(st)
                b.synchronize()
                pipelined = a.elapsed_time(b) * 1000.0 / reps
                nbytes, flops = plan_work(e.steps, batch)
                r[part] = {"us_median": round(statistics.median(ts), 2), "us_min": round(min(ts), 2), "us_pipelined": round(pipelined, 2),
                           "kernels": e.launches_per_forward, "hbm_bytes_algorithmic": int(nbytes), "gflop": round(flops / 1e9, 4)}
                del e
            # speedup on device time per block (the paper's us/block); the
            # single-launch latency ratio (launch overhead included) beside it
            r["speedup"] = round(r["unfused"]["us_pipelined"] / r["b200"]["us_pipelined"], 3)
            r["speedup_latency"] = round(r["unfused"]["us_median"] / r["b200"]["us_median"], 3)
            r["hbm_bytes_saved_algorithmic"] = r["unfused"]["hbm_bytes_algorithmic"] - r["b200"]["hbm_bytes_algorithmic"]
            # roofline of the block: the fused minimum traffic / work at the measured device time
            r["roofline"] = roofline_frac(r["b200"]["hbm_bytes_algorithmic"], r["b200"]["gflop"] * 1e9, r["b200"]["us_pipelined"] / 1000.0,
                                          prec, sm_mhz)
            res[prec] = r
        out[cfg] = res
    return out


def relaunch_under_torchrun(args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "tf32", "fp32", "fp32_exact"])
    ap.add_argument("--no-blocks", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-arms", action="store_true", help="skip the other precisions / the unfused partition")
    ap.add_argument("--no-tune", action="store_true", help="skip the measured-time tuner (planner model only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2007_06000_b200 as X

    # one rank per GPU; with fewer GPUs than ranks (a dry run of the N-rank
    # path on a 1-GPU box) ranks share devices and the bookkeeping collectives
    # run on gloo -- the line says so in "backend"
    ngpu = torch.cuda.device_count()
    local = local % max(1, ngpu)
    torch.cuda.set_device(local)
    backend = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if ngpu >= world else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    coll_dev = "cuda" if backend != "gloo" else "cpu"

    g = X.load_graph(X.graph_path("squeezenet11"))
    w = X.seeded_weights(g, 42)
    B = PER_GPU_BATCH
    prec = args.precision
    from paper_2007_06000_b200 import dist as D
    first, _ = D.shard(rank, world, B)  # rank r's shard: images [r*B, (r+1)*B) of the seeded stream (no exchange)
    e, tune = make_engine(X, g, w, "b200", prec, B, local, tune=not args.no_tune, first_image=first)
    nsteps = len(e.steps)
    st = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_ms(ms):
        t = torch.tensor([ms], device=coll_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        e.forward(B, use_graph=True)
    barrier()

    # --- timed region: K forwards through the product path (one CUDA-graph
    # launch per forward; its kernels overlap prologues via programmatic
    # dependent launch), CUDA events on the launching stream.
    with ClockSampler(local) as clk:
        barrier()
        # profiler range = the timed forwards (`ncu --profile-from-start off`
        # captures exactly these launches, not the tuner's)
        torch.cuda.profiler.start()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.steps):
            e.forward(B, use_graph=True)
        t1.record(st)
        barrier()
        torch.cuda.profiler.stop()
    ms_per_step = max_ms(t0.elapsed_time(t1) / args.steps)
    clocks = clk.summary()

    # --- parity of the timed configuration (its logits, after the timed loop)
    logits = e.read("pool10", B).cpu().numpy()

    # --- optional final gather of the logits to rank 0 (NCCL), timed apart
    gather_ms = None
    if world > 1:
        lt = torch.from_numpy(logits).to(coll_dev)
        parts = [torch.empty_like(lt) for _ in range(world)]
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        dist.all_gather(parts, lt)
        b.record(st)
        barrier()
        gather_ms = max_ms(a.elapsed_time(b))

    # --- per-kernel durations for the roofline: the same K forwards again,
    # step by step with an event after every step (not part of `value`).
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nsteps + 1)] for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        evs[k][0].record(st)
        for i in range(nsteps):
            e.run_step(i, B)
            evs[k][i + 1].record(st)
    barrier()
    per_step_kernel_ms = [statistics.mean(evs[k][i].elapsed_time(evs[k][i + 1]) for k in range(args.steps))
                          for i in range(nsteps)]

    # --- e2e through the C ABI with host buffers (pinned), same metric.
    c, h, wd = g.inputs[0][1]
    pin_in = torch.empty((B, c, h, wd), dtype=torch.float32).pin_memory()
    x_np = pin_in.numpy()
    x_np[:] = np.random.default_rng(rank).random((B, c, h, wd), dtype=np.float32) - 0.5
    pin_out = torch.empty((B, 1000, 1, 1), dtype=torch.float32).pin_memory()
    out_np = pin_out.numpy()
    import ctypes
    f32p = ctypes.POINTER(ctypes.c_float)
    L = X.api.lib()

    def e2e_step():
        X.api.check(L.xlf_engine_run_host(e._h, x_np.ctypes.data_as(f32p), B, b"pool10", out_np.ctypes.data_as(f32p),
                                          X.api._stream_ptr(None)))

    for _ in range(2):
        e2e_step()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(3, min(args.steps, 10))
    a.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    b.record(st)
    barrier()
    e2e_ms = max_ms(a.elapsed_time(b) / e2e_steps)

    if rank == 0:
        sm_mhz = clocks["sm_mhz"]
        # --- the other arithmetic paths and the unfused partition (same workload, same K)
        arms = None
        if not args.no_arms:
            arms = {}
            for p2 in ("bf16", "tf32", "fp32"):
                for part in ("b200", "unfused"):
                    if p2 == prec and part == "b200":
                        arms[f"{p2}_{part}"] = {"images_per_s": round(B / (ms_per_step * 1e-3), 1), "ms_per_step": round(ms_per_step, 4),
                                                "launches": e.launches_per_forward, "headline": True}
                        continue
                    e2, _ = make_engine(X, g, w, part, p2, B, local, tune=not args.no_tune)
                    ms2 = time_forwards(torch, e2, B, args.steps, args.warmup, st)
                    arms[f"{p2}_{part}"] = {"images_per_s": round(B / (ms2 * 1e-3), 1), "ms_per_step": round(ms2, 4),
                                            "launches": e2.launches_per_forward}
                    del e2
            for p2 in ("bf16", "tf32", "fp32"):
                f, u = arms.get(f"{p2}_b200"), arms.get(f"{p2}_unfused")
                if f and u:
                    f["speedup_vs_unfused"] = round(f["images_per_s"] / u["images_per_s"], 3)
        blocks = None if args.no_blocks else time_blocks(X, torch, sm_mhz)
        hbm_peak, _, src = peaks()
        dom = max(range(nsteps), key=lambda i: per_step_kernel_ms[i])
        s = e.steps[dom]
        alg_bytes = s["bytes_algorithmic"] * B + s.get("weight_bytes", 0)
        achieved = alg_bytes / (per_step_kernel_ms[dom] * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(prec, {}).get(s["id"])
            except Exception:
                traffic = None
        flops = 2 * s["macs"] * B
        pipe, pipe_name = pipe_peak_tflops(prec, sm_mhz)
        cpu = None
        parity = None
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            rate, kind, dt = cpu_reference_rate(threads, threads)
            cpu = {"value": round(rate, 3), "unit": "images/s", "cores": threads, "cpu": cpu_model(), "kind": kind,
                   "sample": f"{threads} images of squeezenet_v1.1 224x224 ({dt:.1f} s)"}
            parity = oracle_parity(logits, first, [0, 37, 74, 111, 148, 185, 222, 255], X.api.TOLERANCE[prec])
        value = world * B / (ms_per_step * 1e-3)
        step_nbytes, step_flops = plan_work(e.steps, B)
        line = {
            "metric": BASELINE_METRIC,
            "value": round(value, 2),
            "unit": "images/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": DTYPE[prec],
            "precision": prec,
            "data": "synthetic (SeededStream(42) inputs generated on device, seeded_weights(42))",
            "config": {"workload": f"squeezenet_v1.1 224x224 inference, b200 partition, {prec}",
                       "batch_per_gpu": B, "global_batch": B * world, "parallelism": f"batch-sharded dp{world}, no collective",
                       "plan": [f"{st_['id']}:{st_['tag']}" for st_ in e.steps],
                       "l2": "no L2 flush needed: one forward moves > 1.4 GB through HBM (L2 126 MB), so each iteration starts "
                             "with its input evicted"},
            "e2e": {"value": round(world * B / (e2e_ms * 1e-3), 2), "unit": "images/s",
                    "h2d_bytes_per_step": int(B * c * h * wd * 4), "d2h_bytes_per_step": int(B * 1000 * 4),
                    "path": "xlf_engine_run_host (C ABI), pinned host buffers"},
            "roofline": {"bound": "hbm", "kernel": s["id"] + ":" + s["tag"], "achieved": round(achieved, 2),
                         "peak": hbm_peak, "peak_source": src, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": int(alg_bytes),
                         "launch_ms": round(per_step_kernel_ms[dom], 4),
                         "share_of_step": round(per_step_kernel_ms[dom] / sum(per_step_kernel_ms), 4),
                         "compute": {"pipe": pipe_name, "achieved_tflops": round(flops / (per_step_kernel_ms[dom] * 1e-3) / 1e12, 3),
                                     "peak_tflops": round(pipe, 2)},
                         "step": roofline_frac(step_nbytes, step_flops, ms_per_step, prec, sm_mhz)},
            "kernels_ms": {f"{st_['id']}:{st_['tag']}": round(t, 4) for st_, t in zip(e.steps, per_step_kernel_ms)},
            "parity": parity,
            "arms": arms,
            "cpu_baseline": cpu,
            "gpu_launches": args.steps * e.launches_per_forward,
            "clocks": clocks,
            "gather_ms": gather_ms,
            "backend": backend if world > 1 else None,
            "devices_visible": ngpu,
            "blocks": blocks,
            "autotune": tune,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
