"""ctypes wrapper over oracle/_ref/libxlfuse_ref.so -- the UNMODIFIED xlfuse
reference compiled from /root/reference/proj/src (see oracle/Makefile).

TEST INFRASTRUCTURE ONLY (tests/, golden generation, bench.py reference arm).
``available()`` is False on machines where the library was never built.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(HERE, "_ref", "libxlfuse_ref.so")
_LIB = None


def available() -> bool:
    return os.path.exists(PATH)


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(PATH)
        f32p = ctypes.POINTER(ctypes.c_float)
        szp = ctypes.POINTER(ctypes.c_size_t)
        L.xref_last_error.restype = ctypes.c_char_p
        L.xref_seeded_weights.argtypes = [ctypes.c_char_p, ctypes.c_uint64, f32p, ctypes.c_size_t, szp]
        L.xref_seeded_inputs.argtypes = [ctypes.c_char_p, ctypes.c_uint64, f32p, ctypes.c_size_t]
        L.xref_run.argtypes = [ctypes.c_char_p, f32p, ctypes.c_uint64, f32p, ctypes.c_int, ctypes.c_char_p, f32p,
                               ctypes.c_int, ctypes.c_int]
        L.xref_block_report.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, szp]
        L.xref_plan.argtypes = [ctypes.c_char_p, ctypes.c_char_p] + [ctypes.c_int] * 4 + [ctypes.c_char_p, ctypes.c_char_p,
                                                                                     ctypes.c_size_t, szp]
        L.xref_store_tx.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_longlong),
                                    ctypes.POINTER(ctypes.c_longlong)]
        _LIB = L
    return _LIB


def _chk(rc):
    if rc != 0:
        raise RuntimeError(lib().xref_last_error().decode())


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) if a is not None else None


def seeded_weights(text: str, seed: int) -> np.ndarray:
    n = ctypes.c_size_t()
    _chk(lib().xref_seeded_weights(text.encode(), seed, None, 0, ctypes.byref(n)))
    out = np.empty(n.value, np.float32)
    _chk(lib().xref_seeded_weights(text.encode(), seed, _p(out), n.value, ctypes.byref(n)))
    return out


def seeded_inputs(text: str, seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    _chk(lib().xref_seeded_inputs(text.encode(), seed, _p(out), n))
    return out


def run(text: str, inputs: np.ndarray, name: str, out_shape, weights: np.ndarray | None = None,
        wseed: int = 42, mode: int = 0, threads: int = 1) -> np.ndarray:
    """mode 0: run_reference per image; mode 1: simulate_graph (reference fused
    interpreter, reference planner, titan_xp-tuned plans)."""
    inputs = np.ascontiguousarray(inputs, np.float32)
    batch = inputs.shape[0]
    out = np.empty((batch,) + tuple(out_shape), np.float32)
    w = np.ascontiguousarray(weights, np.float32) if weights is not None else None
    _chk(lib().xref_run(text.encode(), _p(w), wseed, _p(inputs), batch, name.encode(), _p(out), mode, threads))
    return out


def _text(fn, *args):
    n = ctypes.c_size_t()
    _chk(fn(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _chk(fn(*args, buf, n.value, ctypes.byref(n)))
    return buf.value.decode()


def block_report(text: str) -> str:
    return _text(lib().xref_block_report, text.encode())


def plan(text: str, block_id: str, tile=(0, 0), grid=(0, 0), device="titan_xp") -> str:
    return _text(lib().xref_plan, text.encode(), block_id.encode(), tile[0], tile[1], grid[0], grid[1],
                 device.encode())


def store_tx(text: str, block_id: str):
    f, u = ctypes.c_longlong(), ctypes.c_longlong()
    _chk(lib().xref_store_tx(text.encode(), block_id.encode(), ctypes.byref(f), ctypes.byref(u)))
    return f.value, u.value
