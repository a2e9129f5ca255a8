"""Python face of the drop-in API.

Names, argument meaning and error behaviour follow the reference
(reference proj/include/xlfuse/*.hpp): ``Graph``, ``FusionBlock``,
``detect_fusion_blocks``, ``classify_mode``, ``plan_tiling``,
``run_fused_block``, ``simulate_graph``, ``seeded_weights``.  Everything is
computed by the C++ library / sm_100a kernels behind the C ABI
(include/xlfuse_b200.h); this module only marshals arguments.  Device
tensors are torch CUDA tensors (torch is plumbing for device memory and
streams); host tensors are numpy arrays.  Layouts at this boundary are the
reference's: NCHW float32 (CHW per image, images stacked).
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import TensorRef, XlfError, check, lib, text_call  # noqa: F401

PARTITIONS = {"reference": 0, "b200": 1, "unfused": 2}
PRECISIONS = {"fp32_exact": 0, "fp32": 1, "bf16": 2, "tf32": 3}
# norm-wise tolerance of each precision against the reference (north_star)
TOLERANCE = {"fp32_exact": 0.0, "fp32": 1e-5, "tf32": 1e-3, "bf16": 1e-2}


def _options(options) -> bytes:
    """Engine options (xlf_engine_create_ex): "k=v,..." text or a dict."""
    if options is None:
        return b""
    if isinstance(options, dict):
        options = ",".join(f"{k}={int(v) if isinstance(v, bool) else v}" for k, v in options.items())
    return options.encode()


@dataclass
class FusionBlock:
    """fusion.hpp:21-33."""
    id: str
    mode: str
    members: list
    producer_stage: list = field(default_factory=list)
    consumer_stage: list = field(default_factory=list)
    stores_intermediate: bool = False

    def fused(self) -> bool:
        return self.mode != "unfused"


@dataclass
class ModeResult:
    """fusion.hpp:41-46."""
    accepted: bool
    mode: str
    escaping_intermediate: bool
    reject_reason: str


class Graph:
    """A prepared graph: parse_graph + infer_shapes + fold_elementwise
    (graph.cpp:221-256, :405-417, fusion.cpp:24-51), owned by the C++ library."""

    def __init__(self, text: str):
        h = ctypes.c_void_p()
        check(lib().xlf_graph_parse(text.encode(), ctypes.byref(h)))
        self._h = h
        self.text = text
        info = json.loads(text_call(lib().xlf_graph_json, h))
        self.name = info["name"]
        self.inputs = [(i["name"], tuple(i["shape"])) for i in info["inputs"]]
        self.outputs = info["outputs"]
        self.layers = info["layers"]
        self._by_name = {l["name"]: l for l in self.layers}

    @classmethod
    def load(cls, path: str) -> "Graph":
        with open(path) as fh:
            return cls(fh.read())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._LIB is not None:
            lib().xlf_graph_destroy(h)
            self._h = None

    def find_layer(self, name):
        return self._by_name.get(name)

    def shape_of(self, name):
        for n, s in self.inputs:
            if n == name:
                return s
        return tuple(self._by_name[name]["shape"])

    def consumers_of(self, name):
        return [l["name"] for l in self.layers if name in l["inputs"]]

    def serialize(self) -> str:
        return text_call(lib().xlf_graph_serialize, self._h)

    def conv_weight_spans(self):
        """(layer, offset, filter_count, bias_count) in save_weights order."""
        out, pos = [], 0
        for l in self.layers:
            if l["kind"] != "conv":
                continue
            c = l["conv"]
            nf = c["out_channels"] * (c["in_channels"] // c["group"]) * c["kernel"][0] * c["kernel"][1]
            nb = c["out_channels"] if c["bias"] else 0
            out.append((l["name"], pos, nf, nb))
            pos += nf + nb
        return out


def parse_graph(text: str) -> Graph:
    return Graph(text)


def load_graph(path: str) -> Graph:
    return Graph.load(path)


def detect_fusion_blocks(g: Graph, partition: str = "reference") -> list:
    """fusion.cpp:147-226 (partition='reference'); 'b200' adds pool
    epilogues/prologues and all-reader splits; 'unfused' = one per layer."""
    raw = json.loads(text_call(lib().xlf_blocks_json, g._h, PARTITIONS[partition]))
    return [FusionBlock(**b) for b in raw]


def block_assignment_report(g: Graph, partition: str = "reference") -> str:
    return text_call(lib().xlf_block_report, g._h, PARTITIONS[partition])


def classify_mode(g: Graph, candidate) -> ModeResult:
    return ModeResult(**json.loads(text_call(lib().xlf_classify_mode, g._h, ",".join(candidate).encode())))


def plan_tiling(g: Graph, block_id: str, tile, grid, device: str = "titan_xp") -> str:
    """serialize_plan(plan_tiling(...)) text (tiling.cpp:240-419, :493-527)."""
    return text_call(lib().xlf_plan_tiling, g._h, block_id.encode(), tile[0], tile[1], grid[0], grid[1], device.encode())


def device_document(device: str = "b200") -> str:
    """serialize_device(parse_device / builtin spec) (device.cpp:38-90)."""
    return text_call(lib().xlf_device_document, device.encode())


def store_transactions(g: Graph, block_id: str):
    f, u = ctypes.c_longlong(), ctypes.c_longlong()
    check(lib().xlf_store_tx(g._h, block_id.encode(), ctypes.byref(f), ctypes.byref(u)))
    return f.value, u.value


def device_plan(g: Graph, partition: str = "b200", batch_hint: int = 1, precision: str = "fp32", options=None) -> dict:
    """Host-only device program (kernel steps, tiles, tensor placement)."""
    return json.loads(text_call(lib().xlf_device_plan_json_ex, g._h, PARTITIONS[partition], PRECISIONS[precision], batch_hint,
                                _options(options)))


def seeded_weights(g: Graph, seed: int) -> np.ndarray:
    """tensor.cpp:42-62, flattened in save_weights order (tensor.cpp:64-95)."""
    n = ctypes.c_size_t()
    check(lib().xlf_seeded_weights(g._h, seed, None, 0, ctypes.byref(n)))
    out = np.empty(n.value, np.float32)
    check(lib().xlf_seeded_weights(g._h, seed, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n.value, ctypes.byref(n)))
    return out


def _check_tensor(graph, x, name, device):
    import torch
    shape = graph.shape_of(name)
    ok = isinstance(x, torch.Tensor) and x.dtype == torch.float32 and x.dim() == 4 and tuple(x.shape[1:]) == tuple(shape)
    if not ok or (device and not (x.is_cuda and x.is_contiguous())):
        raise XlfError(8, f"input {name!r} must be a contiguous{' CUDA' if device else ''} float32 [batch, {shape[0]}, "
                          f"{shape[1]}, {shape[2]}] tensor, got {getattr(x, 'dtype', type(x))} {tuple(getattr(x, 'shape', ()))}")


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Engine:
    """Device executor (successor of simulate_graph, fused_exec.cpp:313-349)."""

    def __init__(self, g: Graph, weights: np.ndarray, partition: str = "b200", precision: str = "fp32_exact",
                 max_batch: int = 1, device: int = 0, options=None):
        self.graph = g
        if partition not in PARTITIONS or precision not in PRECISIONS:
            raise XlfError(8, f"unknown partition / precision {partition!r} / {precision!r}")
        w = np.ascontiguousarray(weights, np.float32)
        h = ctypes.c_void_p()
        check(lib().xlf_engine_create_ex(g._h, device, PARTITIONS[partition], PRECISIONS[precision],
                                         w.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), w.size, max_batch, _options(options),
                                         ctypes.byref(h)))
        self._h = h
        self.partition, self.precision, self.max_batch, self.device = partition, precision, max_batch, device
        self.info = json.loads(text_call(lib().xlf_engine_json, h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._LIB is not None:
            lib().xlf_engine_destroy(h)
            self._h = None

    @property
    def steps(self):
        return self.info["plan"]["steps"]

    @property
    def launches_per_forward(self) -> int:
        return lib().xlf_engine_launches_per_forward(self._h)

    def _check_input(self, x, name, device):
        _check_tensor(self.graph, x, name, device)

    def set_input(self, x, stream=None, name=None):
        """x: torch CUDA float32 NCHW [batch, C, H, W] (contiguous); `name`
        selects the graph input (default: the first)."""
        name = name or self.graph.inputs[0][0]
        self._check_input(x, name, True)
        check(lib().xlf_engine_set_input_named(self._h, name.encode(), ctypes.c_void_p(x.data_ptr()), x.shape[0],
                                               _stream_ptr(stream)))

    def set_input_seeded(self, seed: int, batch: int, first_image: int = 0, stream=None):
        check(lib().xlf_engine_set_input_seeded(self._h, seed, first_image, batch, _stream_ptr(stream)))

    def forward(self, batch: int, use_graph: bool = True, stream=None):
        check(lib().xlf_engine_forward(self._h, batch, int(use_graph), _stream_ptr(stream)))

    def run_step(self, index: int, batch: int, stream=None):
        check(lib().xlf_engine_run_step(self._h, index, batch, _stream_ptr(stream)))

    def read(self, name: str, batch: int, stream=None):
        import torch
        shape = self.graph.shape_of(name)
        out = torch.empty((batch,) + tuple(shape), dtype=torch.float32, device=f"cuda:{self.device}")
        check(lib().xlf_engine_read(self._h, name.encode(), ctypes.c_void_p(out.data_ptr()), batch, _stream_ptr(stream)))
        return out

    def run_host(self, x: np.ndarray, name: str, stream=None) -> np.ndarray:
        """End to end from host memory (H2D + forward + D2H), synchronous."""
        shape = self.graph.inputs[0][1]
        if not isinstance(x, np.ndarray) or x.dtype != np.float32 or x.ndim != 4 or tuple(x.shape[1:]) != tuple(shape):
            raise XlfError(8, f"run_host input must be a float32 [batch, {shape[0]}, {shape[1]}, {shape[2]}] array")
        x = np.ascontiguousarray(x)
        out = np.empty((x.shape[0],) + tuple(self.graph.shape_of(name)), np.float32)
        f32p = ctypes.POINTER(ctypes.c_float)
        check(lib().xlf_engine_run_host(self._h, x.ctypes.data_as(f32p), x.shape[0], name.encode(),
                                        out.ctypes.data_as(f32p), _stream_ptr(stream)))
        return out

    def autotune(self, batch: int = 0, reps: int = 3, topk: int = 4) -> list:
        """Measured-time tuning of the fused steps (bf16 / TF32 tensor-core, fp32 SIMT tiles; xlf_engine_autotune):
        returns the chosen configuration of every tuned step."""
        check(lib().xlf_engine_autotune(self._h, batch, reps, topk))
        self.info = json.loads(text_call(lib().xlf_engine_json, self._h))
        return json.loads(text_call(lib().xlf_engine_tune_report, self._h))

    def apply_tuning(self, report) -> None:
        """Re-applies a report autotune() returned (list or JSON text), e.g.
        saved from an earlier run on the same model / batch / GPU."""
        text = report if isinstance(report, str) else json.dumps(report)
        check(lib().xlf_engine_apply_tuning(self._h, text.encode()))
        self.info = json.loads(text_call(lib().xlf_engine_json, self._h))

    def materialized(self):
        return [n for n, t in self.info["plan"]["tensors"].items() if t["materialized"]]


def shard_range(batch: int, n: int, k: int):
    """(first, count) of device slot k of n for `batch` images (xlf_shard)."""
    f, c = ctypes.c_int(), ctypes.c_int()
    check(lib().xlf_shard(batch, n, k, ctypes.byref(f), ctypes.byref(c)))
    return f.value, c.value


class MultiEngine:
    """Several GPUs of one node in one process (xlf_multi_*): one engine per
    device, batch-sharded, one host worker thread + stream per device."""

    def __init__(self, g: Graph, weights: np.ndarray, devices, partition: str = "b200", precision: str = "bf16",
                 max_batch_per_device: int = 1, options=None):
        if partition not in PARTITIONS or precision not in PRECISIONS:
            raise XlfError(8, f"unknown partition / precision {partition!r} / {precision!r}")
        self.graph, self.devices = g, list(devices)
        w = np.ascontiguousarray(weights, np.float32)
        dev = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        check(lib().xlf_multi_create(g._h, dev, len(self.devices), PARTITIONS[partition], PRECISIONS[precision],
                                     w.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), w.size, max_batch_per_device, _options(options),
                                     ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._LIB is not None:
            lib().xlf_multi_destroy(h)
            self._h = None

    def autotune(self, batch_per_device: int = 0, reps: int = 3, topk: int = 3):
        check(lib().xlf_multi_autotune(self._h, batch_per_device, reps, topk))

    def run_host(self, x: np.ndarray, name: str):
        """(outputs NCHW, per-device ms): the batch split by shard_range."""
        shape = self.graph.inputs[0][1]
        if not isinstance(x, np.ndarray) or x.dtype != np.float32 or x.ndim != 4 or tuple(x.shape[1:]) != tuple(shape):
            raise XlfError(8, f"run_host input must be a float32 [batch, {shape[0]}, {shape[1]}, {shape[2]}] array")
        x = np.ascontiguousarray(x)
        out = np.empty((x.shape[0],) + tuple(self.graph.shape_of(name)), np.float32)
        ms = (ctypes.c_double * len(self.devices))()
        f32p = ctypes.POINTER(ctypes.c_float)
        check(lib().xlf_multi_run_host(self._h, x.ctypes.data_as(f32p), x.shape[0], name.encode(), out.ctypes.data_as(f32p), ms))
        return out, list(ms)

    def time_seeded(self, seed: int, batch_per_device: int, steps: int = 10, warmup: int = 3):
        ms = (ctypes.c_double * len(self.devices))()
        check(lib().xlf_multi_time_seeded(self._h, seed, batch_per_device, steps, warmup, ms))
        return list(ms)


def simulate_graph(g: Graph, x, weights: np.ndarray, partition: str = "b200", precision: str = "fp32_exact",
                   names=None):
    """Runs the whole schedule on the GPU (fused_exec.cpp:313-349 semantics);
    x: torch CUDA NCHW batch.  Returns {name: torch NCHW} for `names` (default:
    graph outputs)."""
    e = Engine(g, weights, partition, precision, max_batch=x.shape[0])
    e.set_input(x)
    e.forward(x.shape[0])
    names = names or g.outputs
    return {n: e.read(n, x.shape[0]) for n in names}


class Block:
    """One fused block on the GPU: the successor of run_fused_block
    (fused_exec.hpp:35-37, fused_exec.cpp:30-311) behind xlf_block_prepare /
    xlf_block_run.  ``plan``: a serialize_plan text (e.g. ``plan_tiling(...)``)
    whose tile geometry the kernel runs at; None = the B200 planner's tile."""

    def __init__(self, g: Graph, block, weights: np.ndarray, precision: str = "fp32_exact", partition: str = "reference",
                 plan: str | None = None, device: str = "b200", max_batch: int = 1, gpu: int = 0, options=None):
        if partition not in ("reference", "b200") or precision not in PRECISIONS:
            raise XlfError(8, f"unknown partition / precision {partition!r} / {precision!r}")
        bid = block.id if isinstance(block, FusionBlock) else str(block)
        w = np.ascontiguousarray(weights, np.float32)
        h = ctypes.c_void_p()
        check(lib().xlf_block_prepare(g._h, bid.encode(), PARTITIONS[partition], plan.encode() if plan else None, device.encode(), gpu,
                                      PRECISIONS[precision], w.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), w.size, max_batch,
                                      _options(options), ctypes.byref(h)))
        self._h = h
        self.graph, self.precision, self.max_batch, self.gpu = g, precision, max_batch, gpu
        self.info = json.loads(text_call(lib().xlf_block_json, h))
        self.inputs = [i["name"] for i in self.info["inputs"]]
        self.outputs = [o["name"] for o in self.info["outputs"]]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._LIB is not None:
            lib().xlf_block_destroy(h)
            self._h = None

    @staticmethod
    def ref(t, layout: str = "nchw", cstride: int = 0, coff: int = 0) -> _lib.TensorRef:
        """xlf_tensor_ref of a torch CUDA tensor: NCHW fp32, or NHWC in the
        block's element type (`cstride` elements per pixel, channel `coff`)."""
        if layout == "nchw":
            return _lib.TensorRef(t.data_ptr(), _lib.LAYOUT_NCHW_F32, 0, 0)
        return _lib.TensorRef(t.data_ptr(), _lib.LAYOUT_NHWC, cstride or int(t.shape[-1]), coff)

    def run(self, ins, outs, batch: int, stream=None) -> None:
        """ins / outs: xlf_tensor_ref lists in the order of self.inputs / self.outputs."""
        ai = (_lib.TensorRef * max(1, len(ins)))(*ins)
        ao = (_lib.TensorRef * max(1, len(outs)))(*outs)
        check(lib().xlf_block_run(self._h, ai, len(ins), ao, len(outs), batch, _stream_ptr(stream)))


def run_fused_block(g: Graph, block: FusionBlock, values: dict, weights: np.ndarray, precision: str = "fp32_exact",
                    plan: str | None = None, partition: str = "reference"):
    """fused_exec.cpp:30-311 on the GPU: reads the block's producer inputs by
    name from ``values`` (torch CUDA NCHW fp32, caller-owned) and inserts /
    overwrites its stored tensors (consumer outputs + escaping intermediates,
    cost_model.cpp:21-41) in ``values``, like the reference.  Returns the
    names written.  ``weights``: the whole graph's, save_weights order."""
    import torch
    if not block.fused():
        raise XlfError(6, "run_fused_block: block is not fused")
    ins = []
    for n in _block_inputs(g, block):
        if n not in values:
            raise XlfError(6, f"missing input tensor '{n}'")
        ins.append(values[n])
    batch = ins[0].shape[0]
    b = Block(g, block, weights, precision, partition, plan=plan, max_batch=batch, gpu=ins[0].device.index or 0)
    outs = {o: torch.empty((batch,) + tuple(g.shape_of(o)), dtype=torch.float32, device=ins[0].device) for o in b.outputs}
    for x, n in zip(ins, b.inputs):
        _check_tensor(g, x, n, True)
    b.run([Block.ref(x) for x in ins], [Block.ref(outs[o]) for o in b.outputs], batch)
    values.update(outs)
    return list(outs)


def _block_inputs(g: Graph, block: FusionBlock) -> list:
    """External inputs of a block in layer order (xlf_block_prepare's order)."""
    names = set(block.members)
    ext = []
    for l in g.layers:
        if l["name"] in names:
            for i in l["inputs"]:
                if i not in names and i not in ext:
                    ext.append(i)
    return ext
