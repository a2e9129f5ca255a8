"""CPU oracle for the xlfuse fused-block path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module; the product package never
does.  It is deliberately independent of the product: its own parser of the
reference's structured-text graph format, its own shape inference and
topological order, and the arithmetic of ``liboracle.so`` (xlf_oracle.c).

Sources followed (all under /root/reference/proj):
  textdoc format ............ src/textdoc.cpp:154-201 (parse), brackets/commas stripped
  parse_graph ............... src/graph.cpp:221-256
  conv_out_dim .............. src/graph.cpp:76-78
  infer_shapes / topo_order . src/graph.cpp:303-417 (stable Kahn, file order)
  fold_elementwise .......... src/fusion.cpp:24-51
  run_reference ............. src/reference.cpp:126-142
  seeded_inputs/weights ..... src/tensor.cpp:31-62

Parity of this module is pinned against the compiled reference
(oracle/_ref/libxlfuse_ref.so, see :mod:`oracle.ref`) and the committed
golden vectors in tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib() -> ctypes.CDLL:
    """Loads (building if needed) liboracle.so."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
        L = ctypes.CDLL(path)
        f32p = ctypes.POINTER(ctypes.c_float)
        L.xlo_stream_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, f32p, ctypes.c_size_t]
        L.xlo_weight_seed.argtypes = [ctypes.c_uint64]
        L.xlo_weight_seed.restype = ctypes.c_uint64
        L.xlo_conv.argtypes = [f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p, f32p] + [ctypes.c_int] * 7 + [f32p]
        L.xlo_pool.argtypes = [f32p] + [ctypes.c_int] * 7 + [f32p]
        L.xlo_relu.argtypes = [f32p, f32p, ctypes.c_size_t]
        L.xlo_add.argtypes = [f32p, f32p, f32p, ctypes.c_size_t]
        L.xlo_compare.argtypes = [f32p, f32p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


# ----------------------------------------------------------------------------- graph

@dataclass
class OLayer:
    name: str
    kind: str
    inputs: list
    conv: dict | None = None
    pool: dict | None = None
    shape: tuple | None = None  # (C, H, W)


@dataclass
class OGraph:
    name: str
    inputs: list = field(default_factory=list)  # [(name, (C,H,W))]
    layers: list = field(default_factory=list)
    outputs: list = field(default_factory=list)

    def find(self, n):
        for l in self.layers:
            if l.name == n:
                return l
        return None

    def shape_of(self, n):
        for nm, s in self.inputs:
            if nm == n:
                return s
        return self.find(n).shape

    def consumers_of(self, n):
        return [l.name for l in self.layers if n in l.inputs]


def _tokens(text):
    """textdoc.cpp:154-201 -- yields (key, values|None, depth-change)."""
    out = []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line == "}":
            out.append(("}", None))
            continue
        parts = line.split(None, 1)
        key = parts[0]
        rest = parts[1].strip() if len(parts) > 1 else ""
        if rest == "{":
            out.append((key, "{"))
        else:
            vals = [v for v in rest.replace("[", " ").replace("]", " ").replace(",", " ").split() if v]
            out.append((key, vals))
    return out


def parse_graph(text: str) -> OGraph:
    """graph.cpp:221-256 (structure only; the reference validates more)."""
    toks = _tokens(text)
    g = OGraph(name="")
    i = 0

    def section(i):
        d = {}
        i += 1
        while toks[i][0] != "}":
            k, v = toks[i]
            d[k] = v
            i += 1
        return d, i + 1

    while i < len(toks):
        k, v = toks[i]
        if v == "{":
            d, i = section(i)
            if k == "input":
                s = tuple(int(x) for x in d["shape"])
                g.inputs.append((d["name"][0], s))
            elif k == "layer":
                kind = d["kind"][0]
                L = OLayer(d["name"][0], kind, list(d["inputs"]))
                if kind == "conv":
                    kk = [int(x) for x in d["kernel"]]
                    kh, kw = (kk[0], kk[0]) if len(kk) == 1 else (kk[0], kk[1])
                    L.conv = dict(cout=int(d["out_channels"][0]), kh=kh, kw=kw,
                                  pad=int(d.get("pad", ["0"])[0]), stride=int(d.get("stride", ["1"])[0]),
                                  group=int(d.get("group", ["1"])[0]),
                                  bias=d.get("bias", ["true"])[0] == "true",
                                  relu=d.get("activation", ["none"])[0] == "relu")
                elif kind == "pool":
                    L.pool = dict(kind=d["pool"][0], k=int(d["kernel"][0]),
                                  stride=int(d.get("stride", ["1"])[0]), pad=int(d.get("pad", ["0"])[0]))
                g.layers.append(L)
            continue
        if k == "name":
            g.name = v[0]
        elif k == "output":
            g.outputs.append(v[0])
        i += 1
    return g


def out_dim(n, k, pad, stride):
    """graph.cpp:76-78 in C++ int arithmetic: the division truncates toward
    zero, so a window one cell wider than the padded input still yields 1."""
    q = n + 2 * pad - k
    return (q // stride if q >= 0 else -((-q) // stride)) + 1


def topo_order(g: OGraph):
    """graph.cpp:303-332: stable Kahn, first file-order layer with indegree 0."""
    names = {l.name for l in g.layers}
    indeg = {l.name: sum(1 for x in l.inputs if x in names) for l in g.layers}
    done, order = set(), []
    while len(order) < len(g.layers):
        for l in g.layers:
            if l.name not in done and indeg[l.name] == 0:
                done.add(l.name)
                order.append(l)
                for c in g.layers:
                    if l.name in c.inputs:
                        indeg[c.name] -= 1
                break
        else:
            raise ValueError("graph contains a cycle")
    return order


def infer_shapes(g: OGraph) -> OGraph:
    for l in topo_order(g):
        ins = [g.shape_of(x) for x in l.inputs]
        if l.kind == "conv":
            c = l.conv
            c["cin"] = ins[0][0]
            l.shape = (c["cout"], out_dim(ins[0][1], c["kh"], c["pad"], c["stride"]),
                       out_dim(ins[0][2], c["kw"], c["pad"], c["stride"]))
            if min(l.shape[1:]) < 1:  # graph.cpp:362-365
                raise ValueError(f"{l.name}: non-positive output dimension")
        elif l.kind == "pool":
            p = l.pool
            l.shape = (ins[0][0], out_dim(ins[0][1], p["k"], p["pad"], p["stride"]),
                       out_dim(ins[0][2], p["k"], p["pad"], p["stride"]))
            if min(l.shape[1:]) < 1:  # graph.cpp:374-375
                raise ValueError(f"{l.name}: non-positive output dimension")
        elif l.kind in ("relu", "add"):
            l.shape = ins[0]
        elif l.kind == "concat":
            l.shape = (sum(s[0] for s in ins), ins[0][1], ins[0][2])
    return g


def fold_elementwise(g: OGraph) -> OGraph:
    """fusion.cpp:24-51."""
    changed = True
    while changed:
        changed = False
        for i, r in enumerate(g.layers):
            if r.kind != "relu":
                continue
            p = g.find(r.inputs[0])
            if p is None or p.kind != "conv" or len(g.consumers_of(p.name)) != 1:
                continue
            p.conv["relu"] = True
            del g.layers[i]
            for l in g.layers:
                l.inputs = [p.name if x == r.name else x for x in l.inputs]
            g.outputs = [p.name if o == r.name else o for o in g.outputs]
            changed = True
            break
    return g


def load_graph(text_or_path: str) -> OGraph:
    text = text_or_path
    if "\n" not in text_or_path and os.path.exists(text_or_path):
        text = open(text_or_path).read()
    return fold_elementwise(infer_shapes(parse_graph(text)))


# ----------------------------------------------------------------------------- data

def stream(seed: int, first: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    lib().xlo_stream_fill(ctypes.c_uint64(seed), ctypes.c_uint64(first), _p(out), n)
    return out


def seeded_batch(g: OGraph, seed: int, batch: int) -> np.ndarray:
    """Image n = elements [n*CHW, (n+1)*CHW) of SeededStream(seed); image 0
    equals seeded_inputs(g, seed) (tensor.cpp:31-40)."""
    c, h, w = g.inputs[0][1]
    return stream(seed, 0, batch * c * h * w).reshape(batch, c, h, w)


def seeded_weights(g: OGraph, seed: int) -> dict:
    """tensor.cpp:42-62: stream seed ^ 0xabcdef1234567890, layers in FILE order,
    filter [oc][ic/g][kh][kw] then bias."""
    ws = lib().xlo_weight_seed(ctypes.c_uint64(seed))
    out, pos = {}, 0
    for l in g.layers:
        if l.kind != "conv":
            continue
        c = l.conv
        nf = c["cout"] * (c["cin"] // c["group"]) * c["kh"] * c["kw"]
        nb = c["cout"] if c["bias"] else 0
        v = stream(ws, pos, nf + nb)
        pos += nf + nb
        out[l.name] = (v[:nf].reshape(c["cout"], c["cin"] // c["group"], c["kh"], c["kw"]).copy(), v[nf:].copy())
    return out


def flat_weights(g: OGraph, w: dict) -> np.ndarray:
    """save_weights stream order (tensor.cpp:64-95)."""
    parts = []
    for l in g.layers:
        if l.kind == "conv":
            f, b = w[l.name]
            parts += [f.ravel(), b.ravel()]
    return np.concatenate(parts).astype(np.float32)


# ----------------------------------------------------------------------------- layers

def conv(x: np.ndarray, filt: np.ndarray, bias: np.ndarray, c: dict) -> np.ndarray:
    C, H, W = x.shape
    Ho, Wo = out_dim(H, c["kh"], c["pad"], c["stride"]), out_dim(W, c["kw"], c["pad"], c["stride"])
    out = np.empty((c["cout"], Ho, Wo), np.float32)
    x = np.ascontiguousarray(x, np.float32)
    f = np.ascontiguousarray(filt, np.float32)
    b = np.ascontiguousarray(bias, np.float32) if bias is not None and bias.size else None
    lib().xlo_conv(_p(x), C, H, W, _p(f), _p(b) if b is not None else None, c["cout"], c["kh"], c["kw"],
                   c["pad"], c["stride"], c["group"], int(c["relu"]), _p(out))
    return out


def pool(x: np.ndarray, p: dict) -> np.ndarray:
    C, H, W = x.shape
    Ho, Wo = out_dim(H, p["k"], p["pad"], p["stride"]), out_dim(W, p["k"], p["pad"], p["stride"])
    out = np.empty((C, Ho, Wo), np.float32)
    x = np.ascontiguousarray(x, np.float32)
    lib().xlo_pool(_p(x), C, H, W, 0 if p["kind"] == "max" else 1, p["k"], p["stride"], p["pad"], _p(out))
    return out


def run_layer(l: OLayer, ins: list, w: dict) -> np.ndarray:
    """reference.cpp:92-124."""
    if l.kind == "conv":
        f, b = w[l.name]
        return conv(ins[0], f, b, l.conv)
    if l.kind == "pool":
        return pool(ins[0], l.pool)
    if l.kind == "relu":
        x = np.ascontiguousarray(ins[0])
        out = np.empty_like(x)
        lib().xlo_relu(_p(x), _p(out), x.size)
        return out
    if l.kind == "add":
        a, b = np.ascontiguousarray(ins[0]), np.ascontiguousarray(ins[1])
        out = np.empty_like(a)
        lib().xlo_add(_p(a), _p(b), _p(out), a.size)
        return out
    if l.kind == "concat":
        return np.concatenate(ins, axis=0)
    raise ValueError(l.kind)


def run_reference(g: OGraph, image: np.ndarray, w: dict, keep=None) -> dict:
    """reference.cpp:126-142 for ONE image (CHW).  Returns name -> CHW tensor
    (all layers, or only ``keep`` plus what is still needed)."""
    vals = {g.inputs[0][0]: np.ascontiguousarray(image, np.float32)}
    for l in topo_order(g):
        vals[l.name] = run_layer(l, [vals[x] for x in l.inputs], w)
    if keep is not None:
        vals = {k: vals[k] for k in keep}
    return vals


def run_batch(g: OGraph, batch: np.ndarray, w: dict, names, threads: int = 1) -> dict:
    """Per-image oracle over a batch (images are independent; threads only
    parallelise across images, each image's arithmetic is serial)."""
    names = list(names)

    def one(i):
        return run_reference(g, batch[i], w, keep=names)

    if threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(one, range(batch.shape[0])))
    else:
        res = [one(i) for i in range(batch.shape[0])]
    return {n: np.stack([r[n] for r in res]) for n in names}


def compare(a: np.ndarray, b: np.ndarray):
    """reference.cpp:144-157 -> (max_abs, max_rel)."""
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    ma, mr = ctypes.c_double(), ctypes.c_double()
    lib().xlo_compare(_p(a), _p(b), a.size, ctypes.byref(ma), ctypes.byref(mr))
    return ma.value, mr.value


def normwise(a: np.ndarray, ref: np.ndarray) -> float:
    """max|a - ref| / max|ref| -- the norm-wise metric the BASELINE tolerances
    (1e-5 fp32 / 1e-3 TF32 / 1e-2 BF16) are stated against."""
    a = a.astype(np.float64)
    ref = ref.astype(np.float64)
    den = max(np.abs(ref).max(), 1e-30)
    return float(np.abs(a - ref).max() / den)
