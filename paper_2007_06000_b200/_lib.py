"""ctypes binding of the C ABI (include/xlfuse_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2007_06000_b200/csrc``).  There is no fallback: if the
library is missing every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxlfuse_b200.so")

# Every symbol include/xlfuse_b200.h declares (checked by tests/test_abi.py).
SYMBOLS = [
    "xlf_last_error", "xlf_version", "xlf_graph_parse", "xlf_graph_destroy", "xlf_graph_json", "xlf_graph_serialize",
    "xlf_block_report", "xlf_blocks_json", "xlf_classify_mode", "xlf_plan_tiling", "xlf_store_tx", "xlf_device_document", "xlf_device_plan_json", "xlf_device_plan_json_ex", "xlf_seeded_weights",
    "xlf_engine_create", "xlf_engine_create_ex", "xlf_engine_destroy", "xlf_engine_json", "xlf_engine_num_steps",
    "xlf_engine_launches_per_forward", "xlf_engine_set_input", "xlf_engine_set_input_named", "xlf_engine_set_input_seeded", "xlf_engine_forward",
    "xlf_engine_run_step", "xlf_engine_read", "xlf_engine_run_host", "xlf_engine_autotune", "xlf_engine_tune_report", "xlf_engine_apply_tuning",
    "xlf_engine_trace", "xlf_block_prepare", "xlf_block_json", "xlf_block_run", "xlf_block_destroy",
    "xlf_shard", "xlf_multi_create", "xlf_multi_destroy", "xlf_multi_autotune", "xlf_multi_run_host", "xlf_multi_time_seeded",
]


class TensorRef(ctypes.Structure):
    """xlf_tensor_ref: a caller-owned device tensor."""
    _fields_ = [("data", ctypes.c_void_p), ("layout", ctypes.c_int), ("cstride", ctypes.c_int), ("coff", ctypes.c_int)]


LAYOUT_NCHW_F32, LAYOUT_NHWC = 0, 1

STATUS = {0: "ok", 1: "io", 2: "parse", 3: "validation", 4: "infeasible", 5: "verification", 6: "internal", 7: "cuda",
          8: "arg"}


class XlfError(RuntimeError):
    """Mirrors xlfuse::Error (error.hpp:21-35): ``kind`` is the ErrorKind name."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.kind = STATUS.get(code, "internal")
        super().__init__(f"[{self.kind}] {message}")


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    c_char_pp = ctypes.c_char_p
    vp, sz, szp = ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)
    f32p = ctypes.POINTER(ctypes.c_float)
    L.xlf_last_error.restype = ctypes.c_char_p
    L.xlf_version.restype = ctypes.c_char_p
    L.xlf_graph_parse.argtypes = [c_char_pp, ctypes.POINTER(vp)]
    L.xlf_graph_destroy.argtypes = [vp]
    L.xlf_graph_destroy.restype = None
    for fn in ("xlf_graph_json", "xlf_graph_serialize"):
        getattr(L, fn).argtypes = [vp, ctypes.c_char_p, sz, szp]
    for fn in ("xlf_block_report", "xlf_blocks_json"):
        getattr(L, fn).argtypes = [vp, ctypes.c_int, ctypes.c_char_p, sz, szp]
    L.xlf_classify_mode.argtypes = [vp, c_char_pp, ctypes.c_char_p, sz, szp]
    L.xlf_plan_tiling.argtypes = [vp, c_char_pp] + [ctypes.c_int] * 4 + [c_char_pp, ctypes.c_char_p, sz, szp]
    L.xlf_device_document.argtypes = [c_char_pp, ctypes.c_char_p, sz, szp]
    L.xlf_store_tx.argtypes = [vp, c_char_pp, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]
    L.xlf_device_plan_json.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, sz, szp]
    L.xlf_device_plan_json_ex.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_char_pp, ctypes.c_char_p, sz, szp]
    L.xlf_seeded_weights.argtypes = [vp, ctypes.c_uint64, f32p, sz, szp]
    L.xlf_engine_create.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p, sz, ctypes.c_int, ctypes.POINTER(vp)]
    L.xlf_engine_create_ex.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p, sz, ctypes.c_int, c_char_pp, ctypes.POINTER(vp)]
    L.xlf_engine_destroy.argtypes = [vp]
    L.xlf_engine_destroy.restype = None
    L.xlf_engine_json.argtypes = [vp, ctypes.c_char_p, sz, szp]
    L.xlf_engine_num_steps.argtypes = [vp]
    L.xlf_engine_launches_per_forward.argtypes = [vp]
    L.xlf_engine_set_input.argtypes = [vp, vp, ctypes.c_int, vp]
    L.xlf_engine_set_input_named.argtypes = [vp, c_char_pp, vp, ctypes.c_int, vp]
    L.xlf_engine_set_input_seeded.argtypes = [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, vp]
    L.xlf_engine_forward.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
    L.xlf_engine_run_step.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
    L.xlf_engine_read.argtypes = [vp, c_char_pp, vp, ctypes.c_int, vp]
    L.xlf_engine_run_host.argtypes = [vp, f32p, ctypes.c_int, c_char_pp, f32p, vp]
    L.xlf_engine_autotune.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.xlf_engine_tune_report.argtypes = [vp, ctypes.c_char_p, sz, szp]
    L.xlf_engine_apply_tuning.argtypes = [vp, ctypes.c_char_p]
    L.xlf_engine_trace.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), sz, szp]
    L.xlf_block_prepare.argtypes = [vp, c_char_pp, ctypes.c_int, c_char_pp, c_char_pp, ctypes.c_int, ctypes.c_int, f32p, sz, ctypes.c_int,
                                    c_char_pp, ctypes.POINTER(vp)]
    L.xlf_block_json.argtypes = [vp, ctypes.c_char_p, sz, szp]
    L.xlf_block_run.argtypes = [vp, ctypes.POINTER(TensorRef), ctypes.c_int, ctypes.POINTER(TensorRef), ctypes.c_int, ctypes.c_int, vp]
    L.xlf_block_destroy.argtypes = [vp]
    L.xlf_block_destroy.restype = None
    ip, dp = ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)
    L.xlf_shard.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip]
    L.xlf_multi_create.argtypes = [vp, ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p, sz, ctypes.c_int, c_char_pp, ctypes.POINTER(vp)]
    L.xlf_multi_destroy.argtypes = [vp]
    L.xlf_multi_destroy.restype = None
    L.xlf_multi_autotune.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.xlf_multi_run_host.argtypes = [vp, f32p, ctypes.c_int, c_char_pp, f32p, dp]
    L.xlf_multi_time_seeded.argtypes = [vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
    _LIB = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise XlfError(rc, lib().xlf_last_error().decode())


def text_call(fn, *args) -> str:
    need = ctypes.c_size_t()
    check(fn(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(fn(*args, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()
